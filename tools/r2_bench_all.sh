# bench lines of every config on one B200 (C3 is the default line; CPU baselines where the oracle solve is short)
export PYTHONPATH=.
python bench.py --config C1 > gpurun_out/r2_bench_C1.json 2> gpurun_out/r2_bench_C1.err
python bench.py --config C2 > gpurun_out/r2_bench_C2.json 2> gpurun_out/r2_bench_C2.err
python bench.py --config C2 --bc neumann --no-cpu-baseline > gpurun_out/r2_bench_C2N.json 2> gpurun_out/r2_bench_C2N.err
python bench.py --config C4 > gpurun_out/r2_bench_C4.json 2> gpurun_out/r2_bench_C4.err
python bench.py --config C5 --no-cpu-baseline > gpurun_out/r2_bench_C5.json 2> gpurun_out/r2_bench_C5.err
python bench.py > gpurun_out/r2_bench_C3.json 2> gpurun_out/r2_bench_C3.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err
for c in C1 C2 C2N C4 C5 C3 ref; do echo "== $c"; tail -c 400 gpurun_out/r2_bench_$c.json; tail -n 2 gpurun_out/r2_bench_$c.err; done
