# Device bounds-check pass (compute-sanitizer is closed on this pool): rebuild with -DKFBI_BOUNDS
# (KFBI_CHECK asserts on the hot kernels' computed indices), run the sanitizer workload and the GPU tests.
KFBI_NVCC_EXTRA=-DKFBI_BOUNDS python -c "from paper_2404_15249_b200.build import build; build(force=True)" || exit 1
export PYTHONPATH=.
python tools/sanitize_run.py > gpurun_out/r2_bounds_workload.log 2>&1; echo "workload rc=$?" >> gpurun_out/r2_bounds_workload.log
python -m pytest tests -m gpu -x -q > gpurun_out/r2_bounds_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2_bounds_tests.log
grep -h "KFBI_CHECK" gpurun_out/r2_bounds_*.log | head
tail -n 3 gpurun_out/r2_bounds_workload.log; tail -n 3 gpurun_out/r2_bounds_tests.log
