for r in 1 2; do for v in 1 0; do
  VC_END_BRANCH=$v python bench.py --steps 1000 --warmup 5 --no-cpu-baseline --no-fft-comparator > gpurun_out/eb4_${v}_$r.json 2>&1; echo s4 $v $r $?
  VC_END_BRANCH=$v python bench.py --steps 500 --warmup 5 --no-cpu-baseline --no-fft-comparator --streams 1 > gpurun_out/eb1_${v}_$r.json 2>&1; echo s1 $v $r $?
done; done
