# A/B of k_inv_sparse: staged spectral row (bulk copy, default) vs unstaged (KFBI_INV_STAGE=0),
# (the staged variant was removed after this A/B: DESIGN.md §7 "Round 2 experiments")
# the 2D GPU tests on both
export PYTHONPATH=.
for v in 1 0; do
  KFBI_INV_STAGE=$v python -m pytest tests/test_gpu_2d.py tests/test_gpu_edge.py -x -q > gpurun_out/t2d_$v.log 2>&1; echo "stage=$v tests rc=$?" >> gpurun_out/t2d_$v.log
  tail -n 2 gpurun_out/t2d_$v.log
done
for r in 1 2; do for v in 1 0; do for c in C3 C2; do echo "stage=$v $c"; KFBI_INV_STAGE=$v python tools/prof_apply.py $c 3 2>&1 | tail -n 1; done; done; done
