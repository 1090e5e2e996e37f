# Round-2 profiling pass (run under gpurun, one GPU): FP64 peak, ncu --set full of the two C3 apply
# kernels, and FP64-pipe / DRAM metrics for every launch of a C3 apply, a C3 solve (dense DSTs) and
# a C5 apply.  Each ncu run follows the same command exiting 0 without ncu.
export PYTHONPATH=.
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_fp64.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum,sm__sass_thread_inst_executed_ops_dadd_dmul_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__cycles_elapsed.avg.per_second
./tools/fp64_peak > gpurun_out/fp64_peak.jsonl 2>&1
python tools/prof_apply.py C3 2 > gpurun_out/plain_C3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_inv_sparse|k_sweep" -s 2 -c 2 -o gpurun_out/r2_C3_full \
  python tools/prof_apply.py C3 2 > gpurun_out/ncu_C3_full.log 2>&1
python tools/prof_apply.py C3 2 > gpurun_out/plain_C3b.log 2>&1 && \
  ncu --metrics $M --clock-control none -s 20 -c 12 --csv --log-file gpurun_out/r2_fp64_C3_apply.csv \
  python tools/prof_apply.py C3 2 > gpurun_out/ncu_C3_fp64.log 2>&1
python tools/prof_solve.py C3 1 > gpurun_out/plain_C3s.log 2>&1 && \
  ncu --metrics $M --clock-control none -k regex:"k_dst_dense2" -c 4 --csv --log-file gpurun_out/r2_fp64_C3_dense.csv \
  python tools/prof_solve.py C3 1 > gpurun_out/ncu_C3s_fp64.log 2>&1
python tools/prof_apply.py C5 2 > gpurun_out/plain_C5.log 2>&1 && \
  ncu --metrics $M --clock-control none -s 20 -c 12 --csv --log-file gpurun_out/r2_fp64_C5_apply.csv \
  python tools/prof_apply.py C5 2 > gpurun_out/ncu_C5_fp64.log 2>&1
echo done
