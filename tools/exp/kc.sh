for r in 1 2; do
  python bench.py --steps 1000 --warmup 5 --no-cpu-baseline --no-fft-comparator > gpurun_out/kc_new_$r.json 2>&1; echo new $r $?
  VC_KEEP_CLEAR=1 python bench.py --steps 1000 --warmup 5 --no-cpu-baseline --no-fft-comparator > gpurun_out/kc_keep_$r.json 2>&1; echo keep $r $?
done
