set -x
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --streams 1"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fx_kernel|fy_kernel|z_kernel|iy_kernel|ix_kernel|mc_|pre_|splat|clear_kernel|iso_|texture_kernel|mesh_f32" -s 40 -c 60 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"fx_kernel|fy_kernel|z_kernel|ix_kernel|mc_count|mc_emit" -s 12 -c 6 -o gpurun_out/prof_fft $CMD > gpurun_out/ncu_full.log 2>&1
echo done $?
