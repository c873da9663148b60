timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2_parity.py tests/test_gpu_slab.py -x -q > gpurun_out/g4_pytest.log 2>&1; echo pytest $?
STREAMS="1 4" STEPS=600 bash tools/quick.sh
