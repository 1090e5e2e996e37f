# A/B of the dense 2D DST-I core: split radix (KFBI_DST_SPLIT=1, default) vs the N-point odd extension (0);
# the 2D GPU tests (fast solve backward-error pins, 8192 eigenfunctions, full-size solve) on the default
export PYTHONPATH=.
python -m pytest tests/test_gpu_2d.py tests/test_gpu_edge.py tests/test_gpu_omega.py tests/test_gpu_grayscott.py -x -q -s > gpurun_out/t2d_split.log 2>&1; echo "tests rc=$?" >> gpurun_out/t2d_split.log
grep -E "N=|eigenfunction|passed|failed" gpurun_out/t2d_split.log | tail -12
for v in 1 0; do
  KFBI_NVCC_EXTRA="-DKFBI_DST_SPLIT=$v" python paper_2404_15249_b200/build.py --force > /dev/null 2>&1 || echo "build failed"
  python bench.py --no-cpu-baseline --steps 10 > gpurun_out/b_split_$v.json 2> gpurun_out/b_split_$v.err
  python -c "import json; d=json.loads(open('gpurun_out/b_split_$v.json').read().strip().splitlines()[-1]); print('split=$v', d['ms_per_step'], d['e2e']['s_per_step'])"
done
