timeout 600 python -m pytest tests/test_depth_filter.py -x -q > gpurun_out/g8_pytest.log 2>&1; echo pytest $?; tail -2 gpurun_out/g8_pytest.log
for v in cw8 cw4; do
  if [ $v = cw4 ]; then cp paper_1712_03084_b200/libvc_b200.so /tmp/cw8.so; cp build/libvc_cw4.so paper_1712_03084_b200/libvc_b200.so; fi
  timeout 300 python bench.py --steps 600 --warmup 5 --no-cpu-baseline --streams 1 > gpurun_out/g8_$v.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/g8_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['value'],1), {k: round(v*1000,1) for k,v in d['kernel_ms'].items()})"
  timeout 300 python bench.py --steps 2000 --warmup 5 --no-cpu-baseline > gpurun_out/g8_${v}_s4.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/g8_${v}_s4.json').read().strip().splitlines()[-1]); print('$v S4', round(d['value'],1), round(d['e2e']['value'],1))"
done
timeout 600 python -m pytest tests/test_gpu_c2_parity.py -x -q 2>&1 | tail -2
