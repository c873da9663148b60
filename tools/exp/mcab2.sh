CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-fft-comparator --streams 1"
for m in 0 1; do
VC_MC=$m ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"mc_|iso_|ix_kernel" -s 40 -c 40 --csv --log-file gpurun_out/mcl_$m.csv $CMD > gpurun_out/mcl_$m.log 2>&1; echo l $m $?
done
