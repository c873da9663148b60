# reproduce: C5 (S=2) several times without ncu; then under ncu with S=2 and with S=1
for i in 1 2 3; do python bench.py --workload c5 --steps 40 --warmup 3 --no-cpu-baseline > gpurun_out/cc_$i.json 2> gpurun_out/cc_$i.err; echo plain $i $?; done
ncu --set full --clock-control none -k regex:"zp_kernel" -s 2 -c 1 -o gpurun_out/cc_s2 python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/cc_ncu2.log 2>&1; echo ncu_s2 $?
ncu --set full --clock-control none -k regex:"zp_kernel" -s 2 -c 1 -o gpurun_out/cc_s1 python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu-baseline --streams 1 > gpurun_out/cc_ncu1.log 2>&1; echo ncu_s1 $?
tail -3 gpurun_out/cc_ncu2.log
