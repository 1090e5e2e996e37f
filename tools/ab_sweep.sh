export PYTHONPATH=.
python -m pytest tests/test_gpu_2d.py -x -q -k "apply or fast or partitioned" > gpurun_out/t2d.log 2>&1; echo "tests rc=$?" >> gpurun_out/t2d.log
tail -2 gpurun_out/t2d.log
for r in 0 1; do for pd in 0 1; do echo "remap=$r pad=$pd"; KFBI_SW_REMAP=$r KFBI_SW_PAD=$pd python tools/prof_apply.py C3 3 2>&1 | tail -1; done; done
