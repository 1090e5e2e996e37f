# A/B: Arnoldi steps as CUDA graphs (default) vs eager launches (KFBI_GRAPHS=0), bench lines C1/C2/C3
export PYTHONPATH=.
for r in 1 2; do for v in 1 0; do for cfg in C1 C2 C3; do
  KFBI_GRAPHS=$v python bench.py --config $cfg --no-cpu-baseline > gpurun_out/b_ab_$cfg.json 2> /dev/null
  python -c "import json; d=json.loads(open('gpurun_out/b_ab_$cfg.json').read().strip().splitlines()[-1]); print('graphs=$v $cfg', round(d['ms_per_step'],3), round(1e3*d['e2e']['s_per_step'],3))"
done; done; done
