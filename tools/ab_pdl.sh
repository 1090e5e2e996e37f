# A/B: programmatic dependent launch of the apply chain and the MGS cluster kernel (default) vs plain
# launches (KFBI_PDL=0); the GPU tests on the default
export PYTHONPATH=.
python -m pytest tests/test_gpu_2d.py tests/test_gpu_3d.py tests/test_gpu_edge.py tests/test_gpu_omega.py tests/test_gpu_setup.py -x -q -k "not full_size and not C5_256" > gpurun_out/t_pdl.log 2>&1; echo "tests rc=$?" >> gpurun_out/t_pdl.log
tail -n 2 gpurun_out/t_pdl.log
for r in 1 2; do for v in 1 0; do for cfg in C3 C2 C5; do
  KFBI_PDL=$v python bench.py --config $cfg --no-cpu-baseline > gpurun_out/b_pdl_$cfg.json 2> /dev/null
  python -c "import json; d=json.loads(open('gpurun_out/b_pdl_$cfg.json').read().strip().splitlines()[-1]); print('pdl=$v $cfg', round(d['ms_per_step'],3), round(1e3*d['e2e']['s_per_step'],3))"
done; done; done
