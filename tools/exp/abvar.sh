# A/B: current library vs paper_1712_03084_b200/libvc_b200_var.so, alternating, same box
P=paper_1712_03084_b200
cp $P/libvc_b200.so /tmp/libvc_default.so
for r in 1 2; do
for v in default var; do
  if [ $v = var ]; then cp $P/libvc_b200_var.so $P/libvc_b200.so; else cp /tmp/libvc_default.so $P/libvc_b200.so; fi
  python bench.py --steps 1000 --warmup 5 --no-cpu-baseline --no-fft-comparator $ABARGS > gpurun_out/abv_${v}_$r.json 2>&1; echo $v $r $?
done
done
cp /tmp/libvc_default.so $P/libvc_b200.so
