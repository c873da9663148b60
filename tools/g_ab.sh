timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2_parity.py tests/test_gpu_slab.py tests/test_volume_ops.py -x -q > gpurun_out/gab_pytest.log 2>&1; echo pytest $? $(tail -1 gpurun_out/gab_pytest.log)
cp paper_1712_03084_b200/libvc_b200.so /tmp/new.so
for rep in 1 2; do for v in new old; do
  if [ $v = new ]; then cp /tmp/new.so paper_1712_03084_b200/libvc_b200.so; else cp build/libvc_oldmc.so paper_1712_03084_b200/libvc_b200.so; fi
  timeout 300 python bench.py --steps 3000 --warmup 5 --no-cpu-baseline --no-fft-comparator > gpurun_out/gab_$v.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/gab_$v.json').read().strip().splitlines()[-1]); print('$v S4', round(d['value'],1), round(d['e2e']['value'],1), d['kernel_ms']['mc'])"
done; done
