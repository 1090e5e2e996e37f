# Round-2 measurement pass on one B200: bench lines (C3 default, C5), launch lists with DRAM and FP64
# counters of one C3 and one C5 apply, ncu --set full of the two C3 apply kernels.
export PYTHONPATH=.
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_fp64.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum,sm__sass_thread_inst_executed_ops_dadd_dmul_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__cycles_elapsed.avg.per_second
python bench.py > gpurun_out/r2_bench_C3.json 2> gpurun_out/r2_bench_C3.err
python bench.py --config C5 --no-cpu-baseline > gpurun_out/r2_bench_C5.json 2> gpurun_out/r2_bench_C5.err
python tools/prof_apply.py C3 2 > gpurun_out/plain_m1.log 2>&1 && \
  ncu --metrics $M --clock-control none -s 20 -c 12 --csv --log-file gpurun_out/r2_launches_C3_apply.csv \
  python tools/prof_apply.py C3 2 > gpurun_out/ncu_m1.log 2>&1
python tools/prof_apply.py C5 2 > gpurun_out/plain_m2.log 2>&1 && \
  ncu --metrics $M --clock-control none -s 20 -c 12 --csv --log-file gpurun_out/r2_launches_C5_apply.csv \
  python tools/prof_apply.py C5 2 > gpurun_out/ncu_m2.log 2>&1
python tools/prof_apply.py C3 2 > gpurun_out/plain_m3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_inv_sparse|k_sweep" -s 4 -c 2 -o gpurun_out/r2_C3_final \
  python tools/prof_apply.py C3 2 > gpurun_out/ncu_m3.log 2>&1
echo done
