# Round evidence: default bench line (incl. CPU baseline), reference arm, C5 line,
# ncu launch list and one --set full capture of the main kernels.
python bench.py > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err; echo bench $?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev_ref.json 2> gpurun_out/ev_ref.err; echo ref $?
python bench.py --workload c5 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ev_c5.json 2> gpurun_out/ev_c5.err; echo c5 $?
bash tools/prof_launches.sh
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --streams 1"
ncu --set full --clock-control none --import-source on \
  -k regex:"fx_kernel|fy_kernel|z_kernel|iy_kernel|ix_kernel|splat_weighted|mc_count|mc_emit|texture_kernel|pre_points|sparse_clear" \
  -s 20 -c 11 -o gpurun_out/prof_full $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu $?
