# A/B: k_inv_sparse CTA size 256 (QPT 8, 128 registers, default) vs 512 (QPT 4, 64 registers)
export PYTHONPATH=.
for t in 512 256; do
  KFBI_NVCC_EXTRA="-DKFBI_INV_THREADS=$t" python paper_2404_15249_b200/build.py --force > /dev/null 2>&1 || echo "build failed"
  if [ $t = 512 ]; then python -m pytest tests/test_gpu_2d.py -x -q -k "apply or witness" 2>&1 | tail -n 1; fi
  for c in C3 C2; do echo "threads=$t $c"; python tools/prof_apply.py $c 3 2>&1 | tail -n 1; done
done
