python -m pytest tests -m gpu -x -q > gpurun_out/mid_pytest.log 2>&1; echo pytest $?
for r in 1 2; do for v in 1 0; do
  VC_MID_BRANCH=$v python bench.py --steps 1000 --warmup 5 --no-cpu-baseline --no-fft-comparator > gpurun_out/mid4_${v}_$r.json 2>&1; echo s4 $v $r $?
  VC_MID_BRANCH=$v python bench.py --steps 500 --warmup 5 --no-cpu-baseline --no-fft-comparator --streams 1 > gpurun_out/mid1_${v}_$r.json 2>&1; echo s1 $v $r $?
done; done
