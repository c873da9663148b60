python -m pytest tests -m gpu -x -q > gpurun_out/fyp_pytest.log 2>&1; echo pytest $?
for r in 1 2; do for v in 1 0; do
  VC_FYP=$v python bench.py --workload c5 --steps 20 --warmup 3 --no-cpu-baseline --no-fft-comparator > gpurun_out/fyp_c5_${v}_$r.json 2>&1; echo c5 $v $r $?
done; done
