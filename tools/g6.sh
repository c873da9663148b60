CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-fft-comparator --streams 1"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"z4_kernel" -s 3 -c 1 -o gpurun_out/g6_z4 $CMD > gpurun_out/g6_ncu.log 2>&1; echo ncu $?
