# one-step-ahead Arnoldi enqueue: 2D/3D/edge GPU tests, the e2e decomposition and the C3/C5 bench lines
export PYTHONPATH=.
python -m pytest tests/test_gpu_2d.py tests/test_gpu_3d.py tests/test_gpu_edge.py tests/test_gpu_omega.py tests/test_gpu_grayscott.py -x -q -k "not full_size and not C5_256" > gpurun_out/t_spec.log 2>&1; echo "tests rc=$?" >> gpurun_out/t_spec.log
tail -n 2 gpurun_out/t_spec.log
python tools/e2e_decompose.py
python bench.py --no-cpu-baseline > gpurun_out/b_spec_C3.json 2> gpurun_out/b_spec_C3.err
python -c "import json; d=json.loads(open('gpurun_out/b_spec_C3.json').read().strip().splitlines()[-1]); print('C3', d['ms_per_step'], d['e2e']['s_per_step'], d['gmres_iters'], d['n_applies'])"
