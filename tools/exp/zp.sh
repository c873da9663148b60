python -m pytest tests -m gpu -x -q > gpurun_out/zp_pytest.log 2>&1; echo pytest $?
for zp in 1 0; do
  VC_ZP=$zp python bench.py --workload c5 --steps 20 --warmup 3 --no-cpu-baseline --no-fft-comparator > gpurun_out/zp_c5_$zp.json 2>&1; echo c5 $zp $?
  VC_ZP=$zp python bench.py --workload c3 --steps 40 --warmup 3 --no-cpu-baseline --no-fft-comparator > gpurun_out/zp_c3_$zp.json 2>&1; echo c3 $zp $?
done
