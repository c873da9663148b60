set -x
timeout 900 python -m pytest tests/test_volume_ops.py tests/test_color.py -x -q > gpurun_out/g2_pytest.log 2>&1; echo pytest $?
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-fft-comparator --streams 1"
timeout 300 $CMD > gpurun_out/g2_plain.log 2>&1; echo plain $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"z_kernel" -s 3 -c 1 -o gpurun_out/g2_z $CMD > gpurun_out/g2_ncu.log 2>&1; echo ncu $?
