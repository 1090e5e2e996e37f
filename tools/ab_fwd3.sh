# A/B of k_fwd3s mode groups per CTA (KFBI_FWD_GROUPS = 4, 8 (default), 16, 32)
export PYTHONPATH=.
for g in 4 8 16 32; do
  KFBI_NVCC_EXTRA="-DKFBI_FWD_GROUPS=$g" python paper_2404_15249_b200/build.py --force > /dev/null 2>&1 || echo "build failed"
  for c in C5 C4; do echo "groups=$g $c"; python tools/prof_apply.py $c 3 2>&1 | tail -n 1; done
done
