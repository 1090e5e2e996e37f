# A/B of k_reduced2 modes per CTA (32 = default build, 16) + the 2D GPU tests on the default
export PYTHONPATH=.
python -m pytest tests/test_gpu_2d.py tests/test_gpu_edge.py -x -q > gpurun_out/t2d.log 2>&1; echo "tests rc=$?" >> gpurun_out/t2d.log
tail -n 2 gpurun_out/t2d.log
for mo in 32 16; do
  KFBI_NVCC_EXTRA="-DKFBI_RED2_MODES=$mo" python paper_2404_15249_b200/build.py --force > /dev/null 2>&1 || echo "build failed"
  for c in C3 C2; do echo "modes=$mo $c"; python tools/prof_apply.py $c 3 2>&1 | tail -n 1; done
done
