# ncu --set full of the two C3 apply kernels (after the same command exits 0 without ncu)
export PYTHONPATH=.
python tools/prof_apply.py C3 2 > gpurun_out/plain_f.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_inv_sparse|k_sweep" -s 4 -c 2 -o gpurun_out/r2_C3_final \
  python tools/prof_apply.py C3 2 > gpurun_out/ncu_f.log 2>&1
echo rc=$?
