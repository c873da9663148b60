for v in 1 0; do
  VC_ZP256=$v python bench.py --steps 300 --warmup 5 --no-cpu-baseline --no-fft-comparator > gpurun_out/zq_b4_$v.json 2>&1; echo b4 $v $?
  VC_ZP256=$v python bench.py --steps 300 --warmup 5 --no-cpu-baseline --no-fft-comparator --streams 1 > gpurun_out/zq_b1_$v.json 2>&1; echo b1 $v $?
done
VC_ZP256=1 python -m pytest tests/test_gpu_c2_parity.py -x -q > gpurun_out/zq_pytest.log 2>&1; echo pytest $?
