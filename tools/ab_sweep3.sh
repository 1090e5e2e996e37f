# A/B of the k_sweep3 block split over gridDim.y (1, 2, 4, 8) + the 3D GPU tests on the default (4)
export PYTHONPATH=.
python -m pytest tests/test_gpu_3d.py -x -q -k "not full_size and not C5_256" > gpurun_out/t3d.log 2>&1; echo "tests rc=$?" >> gpurun_out/t3d.log
tail -n 2 gpurun_out/t3d.log
for sp in 1 2 4 8; do
  KFBI_NVCC_EXTRA="-DKFBI_SWEEP3_SPLIT=$sp" python paper_2404_15249_b200/build.py --force > /dev/null 2>&1 || echo "build failed"
  for c in C5 C4; do echo "split=$sp $c"; python tools/prof_apply.py $c 3 2>&1 | tail -n 1; done
done
