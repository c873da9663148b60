# F-y at 512: default library (3 staged tiles, 2 CTAs/SM, no spill) vs variant (2 tiles, 3 CTAs/SM, 392 B spill)
P=paper_1712_03084_b200
cp $P/libvc_b200.so /tmp/libvc_default.so
for v in default var; do
  if [ $v = var ]; then cp $P/libvc_b200_var.so $P/libvc_b200.so; else cp /tmp/libvc_default.so $P/libvc_b200.so; fi
  python bench.py --workload c3 --steps 40 --warmup 3 --no-cpu-baseline --no-fft-comparator > gpurun_out/fy_c3_$v.json 2>&1; echo c3 $v $?
done
python -m pytest tests/test_gpu_parity.py -q -x -k "c3 or 512 or integrate" > gpurun_out/fy_pytest.log 2>&1; echo pytest-var $?
cp /tmp/libvc_default.so $P/libvc_b200.so
python -m pytest tests/test_gpu_parity.py -q -x -k "c3 or 512 or integrate" > gpurun_out/fy_pytest_def.log 2>&1; echo pytest-def $?
