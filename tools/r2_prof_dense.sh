# ncu --set full of the two once-per-solve dense DST kernels (C3), after a plain run of the same command
export PYTHONPATH=.
python tools/prof_solve.py C3 1 > gpurun_out/plain_dense.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_dst_dense2" -s 2 -c 2 -o gpurun_out/r2_C3_dense \
  python tools/prof_solve.py C3 1 > gpurun_out/ncu_dense.log 2>&1
echo rc=$?
