export PYTHONPATH=.
python -m pytest tests/test_gpu_3d.py -x -q -k "not full_size and not C5_256" > gpurun_out/t3d.log 2>&1; echo "tests rc=$?" >> gpurun_out/t3d.log
tail -n 2 gpurun_out/t3d.log
for c in C5 C4; do echo "$c"; python tools/prof_apply.py $c 3 2>&1 | tail -n 1; done
