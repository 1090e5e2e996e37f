# 2D GPU tests, then ncu --set full of the C3 point kernels
export PYTHONPATH=.
python -m pytest tests/test_gpu_2d.py tests/test_gpu_edge.py tests/test_gpu_grayscott.py -x -q > gpurun_out/t2d.log 2>&1; echo "tests rc=$?" >> gpurun_out/t2d.log
tail -n 2 gpurun_out/t2d.log
for c in C3 C1; do echo "$c"; python tools/prof_apply.py $c 3 2>&1 | tail -n 1; done
bash tools/r2_prof_point.sh
