timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/grgb_pytest.log 2>&1; echo pytest $? $(tail -1 gpurun_out/grgb_pytest.log)
for rep in 1 2; do
timeout 300 python bench.py --steps 3000 --warmup 5 --no-cpu-baseline --no-fft-comparator > gpurun_out/grgb.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/grgb.json').read().strip().splitlines()[-1]); print('S4', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
done
