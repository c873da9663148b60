# Z occupancy A/B: default (256: 4 CTAs/SM, 512: 2) vs variant library (256: 5, 512: 3)
P=paper_1712_03084_b200
cp $P/libvc_b200.so /tmp/libvc_default.so
for v in default var; do
  if [ $v = var ]; then cp $P/libvc_b200_var.so $P/libvc_b200.so; else cp /tmp/libvc_default.so $P/libvc_b200.so; fi
  python bench.py --steps 300 --warmup 5 --no-cpu-baseline --no-fft-comparator > gpurun_out/zm_b4_$v.json 2>&1; echo b4 $v $?
  python bench.py --workload c3 --steps 40 --warmup 3 --no-cpu-baseline --no-fft-comparator > gpurun_out/zm_c3_$v.json 2>&1; echo c3 $v $?
done
python -m pytest tests/test_gpu_c2_parity.py -q -x > gpurun_out/zm_pytest.log 2>&1; echo pytest-var $?
cp /tmp/libvc_default.so $P/libvc_b200.so
