timeout 900 python -m pytest tests/test_volume_ops.py tests/test_color.py -x -q > gpurun_out/g3_pytest.log 2>&1; echo pytest $?
