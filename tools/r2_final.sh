# final pass: the whole -m gpu suite, smoke(), the default bench line (C3 with the CPU oracle baseline),
# the C5 line and the reference arm
export PYTHONPATH=.
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r2_gputests_all.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2_gputests_all.log
tail -n 3 gpurun_out/r2_gputests_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2_smoke.log
tail -n 2 gpurun_out/r2_smoke.log
python bench.py > gpurun_out/r2_bench_C3_default.json 2> gpurun_out/r2_bench_C3_default.err; echo "bench rc=$?"
python bench.py --config C5 --no-cpu-baseline > gpurun_out/r2_bench_C5.json 2> gpurun_out/r2_bench_C5.err; echo "bench C5 rc=$?"
python bench.py --impl reference > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err; echo "ref rc=$?"
