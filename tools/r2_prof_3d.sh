export PYTHONPATH=.
python tools/prof_apply.py C5 2 > gpurun_out/plain_3d.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_fwd3s|k_inv3y" -s 2 -c 2 -o gpurun_out/r2_C5_full \
  python tools/prof_apply.py C5 2 > gpurun_out/ncu_3d.log 2>&1
echo rc=$?
