# A/B of the sparse inverse variants (KFBI_INV = m | sync) + the 2D GPU tests on variant m
# (the KFBI_INV variants were removed after this A/B; the kept kernel is k_inv_sparse — DESIGN.md §7)
export PYTHONPATH=.
KFBI_INV=m python -m pytest tests/test_gpu_2d.py tests/test_gpu_edge.py -x -q > gpurun_out/t2d.log 2>&1; echo "tests rc=$?" >> gpurun_out/t2d.log
tail -n 2 gpurun_out/t2d.log
for m in m sync; do for c in C3 C2 C1; do echo "$m $c"; KFBI_INV=$m python tools/prof_apply.py $c 3 2>&1 | tail -n 1; done; done
