PYTHONPATH=. python tools/prof_apply.py C4 3 > gpurun_out/prof_c4.log 2>&1
PYTHONPATH=. python tools/prof_apply.py C5 3 > gpurun_out/prof_c5.log 2>&1
timeout 900 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 900 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
