# A/B of k_inv3y min-blocks-per-SM (2 = default build, 3 = -DKFBI_INV3Y_MINB=3) + the 3D GPU tests on each
export PYTHONPATH=.
for mb in 2 3; do
  KFBI_NVCC_EXTRA="-DKFBI_INV3Y_MINB=$mb" python paper_2404_15249_b200/build.py --force > /dev/null 2>&1
  python -m pytest tests/test_gpu_3d.py -x -q -k "not full_size and not C5_256" > gpurun_out/t3d_$mb.log 2>&1; echo "tests rc=$?" >> gpurun_out/t3d_$mb.log
  tail -n 2 gpurun_out/t3d_$mb.log
  for c in C5 C4; do echo "minb=$mb $c"; python tools/prof_apply.py $c 3 2>&1 | tail -n 1; done
done
