set -x
mkdir -p gpurun_out/ck
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/ck/tests.log 2>&1
tail -3 gpurun_out/ck/tests.log
timeout 600 python bench.py > gpurun_out/ck/bench_C3.json 2> gpurun_out/ck/bench_C3.err
timeout 900 python bench.py --config C5 --no-cpu-baseline > gpurun_out/ck/bench_C5.json 2> gpurun_out/ck/bench_C5.err
