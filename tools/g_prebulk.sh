timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-fft-comparator --streams 1"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pre_prefix" -s 2 -c 3 --csv --log-file gpurun_out/gpb.csv $CMD > /dev/null 2>&1; echo ncu $?
timeout 300 python bench.py --steps 4000 --warmup 5 --no-cpu-baseline --no-fft-comparator > gpurun_out/gpb4.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/gpb4.json').read().strip().splitlines()[-1]); print('S4', round(d['value'],1), round(d['e2e']['value'],1), d['kernel_ms']['preprocess'])"
