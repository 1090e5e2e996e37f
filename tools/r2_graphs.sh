# Arnoldi steps as CUDA graphs: GPU tests, then C1/C2/C3/C5 bench lines (device and e2e)
export PYTHONPATH=.
python -m pytest tests/test_gpu_2d.py tests/test_gpu_3d.py tests/test_gpu_edge.py tests/test_gpu_omega.py tests/test_gpu_grayscott.py -x -q -k "not full_size and not C5_256" > gpurun_out/t_graphs.log 2>&1; echo "tests rc=$?" >> gpurun_out/t_graphs.log
tail -n 2 gpurun_out/t_graphs.log
for cfg in C1 C2 C3 C5; do
  python bench.py --config $cfg --no-cpu-baseline > gpurun_out/b_g_$cfg.json 2> gpurun_out/b_g_$cfg.err
  python -c "import json; d=json.loads(open('gpurun_out/b_g_$cfg.json').read().strip().splitlines()[-1]); print('$cfg', round(d['ms_per_step'],3), round(1e3*d['e2e']['s_per_step'],3), d['gmres_iters'], d['gpu_launches_per_step'])"
done
