# MC variants at S=4: current (count+bsum, scan+emit, finish) / split (count, scan, emit, finish) / var library (round-2 start: count, scan, emit, normals || triangles)
P=paper_1712_03084_b200
cp $P/libvc_b200.so /tmp/libvc_default.so
for r in 1 2; do
  cp /tmp/libvc_default.so $P/libvc_b200.so
  python bench.py --steps 1000 --warmup 5 --no-cpu-baseline --no-fft-comparator > gpurun_out/m3_cur_$r.json 2>&1; echo cur $r $?
  VC_MC_SPLIT=1 python bench.py --steps 1000 --warmup 5 --no-cpu-baseline --no-fft-comparator > gpurun_out/m3_split_$r.json 2>&1; echo split $r $?
  cp $P/libvc_b200_var.so $P/libvc_b200.so
  python bench.py --steps 1000 --warmup 5 --no-cpu-baseline --no-fft-comparator > gpurun_out/m3_old_$r.json 2>&1; echo old $r $?
done
cp /tmp/libvc_default.so $P/libvc_b200.so
