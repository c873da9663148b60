for s in 2 3 4 6; do
  python bench.py --workload c3 --steps 200 --warmup 5 --no-cpu-baseline --no-fft-comparator --streams $s > gpurun_out/swc3_$s.json 2>&1; echo S=$s $?
done
