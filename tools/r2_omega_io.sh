# Ω-compact solve I/O: parity tests, then the C3 bench line (e2e through opts.omega_io)
export PYTHONPATH=.
python -m pytest tests/test_gpu_omega.py tests/test_gpu_2d.py -x -q > gpurun_out/t_omega.log 2>&1; echo "tests rc=$?" >> gpurun_out/t_omega.log
tail -n 3 gpurun_out/t_omega.log
python bench.py --no-cpu-baseline > gpurun_out/r2_bench_C3_omega.json 2> gpurun_out/r2_bench_C3_omega.err
tail -n 2 gpurun_out/r2_bench_C3_omega.err
