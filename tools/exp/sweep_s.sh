for r in 1 2; do for s in 3 4 5 6; do
  python bench.py --steps 2000 --warmup 5 --no-cpu-baseline --no-fft-comparator --streams $s > gpurun_out/sw_${s}_$r.json 2>&1; echo S=$s $r $?
done; done
