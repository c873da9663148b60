# Round-2 evidence: default bench line (incl. CPU baseline), reference arm, C3/C4/C5 lines,
# ncu launch list of one C2 frame and --set full captures (C2 frame kernels, the C3/C5 Z pass).
mkdir -p gpurun_out/ev
python bench.py > gpurun_out/ev/bench.json 2> gpurun_out/ev/bench.err; echo bench $?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev/ref.json 2> gpurun_out/ev/ref.err; echo ref $?
python bench.py --workload c3 --steps 40 --warmup 3 --no-cpu-baseline > gpurun_out/ev/c3.json 2> gpurun_out/ev/c3.err; echo c3 $?
python bench.py --workload c4 --no-cpu-baseline --no-fft-comparator > gpurun_out/ev/c4.json 2> gpurun_out/ev/c4.err; echo c4 $?
python bench.py --workload c5 --steps 40 --warmup 3 --no-cpu-baseline > gpurun_out/ev/c5.json 2> gpurun_out/ev/c5.err; echo c5 $?
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-fft-comparator --streams 1"
$CMD > gpurun_out/ev/plain.log 2>&1; echo plain $?
# the resident stream is rendered first (300 frames x 4 views x 2 kernels): skip those launches
ncu --metrics gpu__time_duration.sum --clock-control none -s 2400 -c 160 --csv --log-file gpurun_out/ev/launches.csv $CMD > gpurun_out/ev/ncu_launch.log 2>&1; echo launches $?
KRE="fx_kernel|fy_kernel|z_kernel|iy_|ix_kernel|splat_weighted|mc_select|mc_count|mc_scan_emit|mc_finish|iso_partial|texture_kernel|pre_points|pre_prefix"
ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s 28 -c 14 -o gpurun_out/ev/prof_full $CMD > gpurun_out/ev/ncu_full.log 2>&1; echo ncu $?
