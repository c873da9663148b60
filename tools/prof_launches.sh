# ncu per-kernel durations (launch list) for a short bench run
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --streams 1"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"${LIST_RE:-fx_kernel|fy_kernel|z_kernel|iy_kernel|ix_kernel|mc_|pre_|splat|clear_kernel|iso_|texture_kernel|mesh_f32|rowlist_build}" -s ${SKIP:-56} -c ${COUNT:-84} --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo done $?
