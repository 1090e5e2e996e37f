# the launch list of the bench command itself (ncu --metrics gpu__time_duration.sum, first 400 launches),
# after the same command exits 0 without ncu
export PYTHONPATH=.
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b_ll.json 2> gpurun_out/b_ll.err && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r2_launches_C3_bench_step.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  > gpurun_out/ncu_ll.log 2>&1
echo rc=$?
