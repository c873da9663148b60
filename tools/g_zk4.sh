timeout 900 python -m pytest tests/test_gpu_zk4.py tests/test_depth_filter.py -x -q 2>&1 | tail -3
