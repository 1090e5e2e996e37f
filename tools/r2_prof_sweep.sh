export PYTHONPATH=.
python tools/prof_apply.py C3 2 > gpurun_out/plain_C3c.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_sweep<0>|k_reduced2" -s 2 -c 2 -o gpurun_out/r2_C3_sweep \
  python tools/prof_apply.py C3 2 > gpurun_out/ncu_C3_sweep.log 2>&1
echo rc=$?
