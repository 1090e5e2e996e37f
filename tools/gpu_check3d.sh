set -x
timeout 900 python -m pytest tests/test_gpu_3d.py -x -q -m gpu -k "not full_size" 2>&1 | tail -30
