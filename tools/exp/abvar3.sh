# current library vs libvc_b200_var.so (candidate), alternating, S=4 and S=1, no tests
P=paper_1712_03084_b200
cp $P/libvc_b200.so /tmp/libvc_default.so
for r in 1 2; do for v in default var; do
  if [ $v = var ]; then cp $P/libvc_b200_var.so $P/libvc_b200.so; else cp /tmp/libvc_default.so $P/libvc_b200.so; fi
  python bench.py --steps 1000 --warmup 5 --no-cpu-baseline --no-fft-comparator > gpurun_out/a3_4_${v}_$r.json 2>&1
  python bench.py --steps 500 --warmup 5 --no-cpu-baseline --no-fft-comparator --streams 1 > gpurun_out/a3_1_${v}_$r.json 2>&1
  echo $v $r
done; done
cp /tmp/libvc_default.so $P/libvc_b200.so
