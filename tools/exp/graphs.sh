for r in 1 2; do for g in 1 0; do
  VC_GRAPHS=$g python bench.py --steps 1000 --warmup 5 --no-cpu-baseline --no-fft-comparator > gpurun_out/gr4_${g}_$r.json 2>&1; echo s4 g=$g $?
done; done
for g in 1 0; do VC_GRAPHS=$g python bench.py --steps 500 --warmup 5 --no-cpu-baseline --no-fft-comparator --streams 1 > gpurun_out/gr1_$g.json 2>&1; echo s1 g=$g $?; done
