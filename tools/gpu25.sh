set -x
timeout 600 python -m pytest tests/test_gpu_condensed.py -x -q -m gpu --timeout 120 2>&1 | tail -25
