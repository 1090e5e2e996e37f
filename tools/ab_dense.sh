export PYTHONPATH=.
python -m pytest tests/test_gpu_2d.py -x -q -k "solve" > gpurun_out/t2dd.log 2>&1; echo "tests rc=$?" >> gpurun_out/t2dd.log
tail -n 2 gpurun_out/t2dd.log
python tools/prof_solve.py C3 4 2>&1 | tail -n 3
