# full-size 3D parity tests, then the launch list (time, DRAM, FP64 counters) of a C5 apply
export PYTHONPATH=.
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_fp64.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum,sm__sass_thread_inst_executed_ops_dadd_dmul_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__cycles_elapsed.avg.per_second
python -m pytest tests/test_gpu_3d.py -x -q -k "full_size or C5_256" > gpurun_out/t3d_full.log 2>&1; echo "tests rc=$?" >> gpurun_out/t3d_full.log
tail -n 2 gpurun_out/t3d_full.log
python tools/prof_apply.py C5 2 > gpurun_out/plain_m2.log 2>&1 && \
  ncu --metrics $M --clock-control none -s 20 -c 12 --csv --log-file gpurun_out/r2_launches_C5_apply.csv \
  python tools/prof_apply.py C5 2 > gpurun_out/ncu_m2.log 2>&1
echo done
