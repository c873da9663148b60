cp build/libvc_exp.so paper_1712_03084_b200/libvc_b200.so
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-fft-comparator --streams 1"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"mc_" -s 20 -c 10 --csv --log-file gpurun_out/g12_mc.csv $CMD > /dev/null 2>&1; echo ncu $?
