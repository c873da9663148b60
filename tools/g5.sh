timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2_parity.py tests/test_gpu_slab.py -x -q > gpurun_out/g5_pytest.log 2>&1; echo pytest $?
for z in 0 1; do
VC_Z2=$z python bench.py --steps 600 --warmup 5 --no-cpu-baseline --streams 1 > gpurun_out/g5_z$z.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/g5_z$z.json').read().strip().splitlines()[-1]); print('Z2=$z', round(d['value'],1), {k: round(v*1000,1) for k,v in d['kernel_ms'].items()})"
done
VC_Z2=1 python bench.py --steps 2000 --warmup 5 --no-cpu-baseline > gpurun_out/g5_s4.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/g5_s4.json').read().strip().splitlines()[-1]); print('S4', round(d['value'],1), round(d['e2e']['value'],1))"
