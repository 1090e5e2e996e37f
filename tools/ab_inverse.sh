# A/B of the sparse inverse variants (KFBI_INV = ws | sync | async) + the 2D GPU tests on the default
export PYTHONPATH=.
python -m pytest tests/test_gpu_2d.py tests/test_gpu_edge.py -x -q > gpurun_out/t2d.log 2>&1; echo "tests rc=$?" >> gpurun_out/t2d.log
tail -2 gpurun_out/t2d.log
for m in ws sync async; do for c in C3 C2; do echo "$m $c"; KFBI_INV=$m python tools/prof_apply.py $c 3 2>&1 | tail -1; done; done
for a in 1 2; do echo "async abl=$a"; KFBI_WS_ABL=$a python tools/prof_apply.py C3 3 2>&1 | tail -1; done
