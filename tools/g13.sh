cp paper_1712_03084_b200/libvc_b200.so /tmp/base.so
for v in base z4 z2; do
  if [ $v = base ]; then cp /tmp/base.so paper_1712_03084_b200/libvc_b200.so; else cp build/libvc_$v.so paper_1712_03084_b200/libvc_b200.so; fi
  timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "integrate" > gpurun_out/g13_$v.log 2>&1; echo $v pytest $? $(tail -1 gpurun_out/g13_$v.log)
  timeout 300 python bench.py --workload c5 --steps 10 --warmup 3 --no-cpu-baseline --no-fft-comparator > gpurun_out/g13_$v.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/g13_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['value'],2), {k: round(v,3) for k,v in d['kernel_ms'].items()})"
done
