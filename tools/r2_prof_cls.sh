export PYTHONPATH=.
python tools/prof_apply.py C3 2 > gpurun_out/plain_cls.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_inv_cls" -s 2 -c 1 -o gpurun_out/r2_C3_cls \
  python tools/prof_apply.py C3 2 > gpurun_out/ncu_cls.log 2>&1
echo rc=$?
