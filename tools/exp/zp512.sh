for r in 1 2; do for v in 0 1; do
  VC_ZP512=$v python bench.py --workload c3 --steps 40 --warmup 3 --no-cpu-baseline --no-fft-comparator > gpurun_out/z5_${v}_$r.json 2>&1; echo c3 $v $r $?
done; done
VC_ZP512=1 python -m pytest tests/test_gpu_parity.py -q -x -k "c3 or 512 or integrate" > gpurun_out/z5_pytest.log 2>&1; echo pytest $?
