# A/B of the y-inverse: plane-pair k_inv3yp (default build) vs one plane per CTA (-DKFBI_INV3Y_SINGLE),
# (the plane-pair variant was removed after this A/B: DESIGN.md §7, k_inv3y)
# the 3D GPU tests (incl. the full-size C5 apply) on the default
export PYTHONPATH=.
for v in pair single; do
  X=""; [ $v = single ] && X="-DKFBI_INV3Y_SINGLE"
  KFBI_NVCC_EXTRA="$X" python paper_2404_15249_b200/build.py --force > /dev/null 2>&1
  if [ $v = pair ]; then
    python -m pytest tests/test_gpu_3d.py -x -q > gpurun_out/t3d_$v.log 2>&1; echo "tests rc=$?" >> gpurun_out/t3d_$v.log
    tail -n 2 gpurun_out/t3d_$v.log
  fi
  for c in C5 C4; do echo "$v $c"; python tools/prof_apply.py $c 3 2>&1 | tail -n 1; done
done
