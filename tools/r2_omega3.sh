# 3D Ω-compact solve I/O: parity tests (omega + 3D), then the C5 bench line (e2e through opts.omega_io)
export PYTHONPATH=.
python -m pytest tests/test_gpu_omega.py tests/test_gpu_3d.py -x -q -k "not full_size and not C5_256" > gpurun_out/t_omega3.log 2>&1; echo "tests rc=$?" >> gpurun_out/t_omega3.log
tail -n 3 gpurun_out/t_omega3.log
python bench.py --config C5 --no-cpu-baseline > gpurun_out/r2_bench_C5_omega.json 2> gpurun_out/r2_bench_C5_omega.err
python -c "import json; d=json.loads(open('gpurun_out/r2_bench_C5_omega.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['s_per_step'], d['e2e']['value'])"
