# A/B of the C5 (1024^3) frame: expects paper_1712_03084_b200/libvc_b200_base.so (the build to
# compare against) next to the current build; swaps them in turn.
cd paper_1712_03084_b200 && cp libvc_b200.so libvc_b200_new.so && cd ..
for v in base new base new; do
  cp paper_1712_03084_b200/libvc_b200_$v.so paper_1712_03084_b200/libvc_b200.so
  python bench.py --workload c5 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/c5_$v.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/c5_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['value'],2), {k: round(x,3) for k,x in d['kernel_ms'].items()})"
done
cp paper_1712_03084_b200/libvc_b200_new.so paper_1712_03084_b200/libvc_b200.so
