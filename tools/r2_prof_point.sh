# ncu --set full of the C3 point kernels (k_spline, k_correct, k_interp), one launch each
export PYTHONPATH=.
python tools/prof_apply.py C3 2 > gpurun_out/plain_pt.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_spline|k_correct|k_interp" -s 6 -c 3 -o gpurun_out/r2_C3_point \
  python tools/prof_apply.py C3 2 > gpurun_out/ncu_pt.log 2>&1
echo rc=$?
