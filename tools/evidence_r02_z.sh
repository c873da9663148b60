# Round-2 evidence, second call (gpurun copies back at most 64 MiB per call): --set full of the Z pass at 512^3 and 1024^3
mkdir -p gpurun_out/ev
ncu --set full --clock-control none -k regex:"z_kernel" -s 2 -c 1 -o gpurun_out/ev/prof_c3z python bench.py --workload c3 --steps 2 --warmup 3 --no-cpu-baseline --no-fft-comparator --streams 1 > gpurun_out/ev/ncu_c3.log 2>&1; echo ncu_c3 $?
ncu --set full --clock-control none -k regex:"zp_kernel" -s 2 -c 1 -o gpurun_out/ev/prof_c5z python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu-baseline --streams 1 > gpurun_out/ev/ncu_c5.log 2>&1; echo ncu_c5 $?
