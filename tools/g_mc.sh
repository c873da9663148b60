timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2_parity.py tests/test_gpu_slab.py tests/test_volume_ops.py -x -q 2>&1 | tail -2
timeout 300 python bench.py --steps 600 --warmup 5 --no-cpu-baseline --streams 1 > gpurun_out/gm_s1.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/gm_s1.json').read().strip().splitlines()[-1]); print('S1', round(d['value'],1), {k: round(v*1000,1) for k,v in d['kernel_ms'].items()})"
timeout 300 python bench.py --steps 2000 --warmup 5 --no-cpu-baseline > gpurun_out/gm_s4.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/gm_s4.json').read().strip().splitlines()[-1]); print('S4', round(d['value'],1), round(d['e2e']['value'],1))"
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-fft-comparator --streams 1"
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"mc_count|mc_emit" -s 2 -c 4 --csv --log-file gpurun_out/gm_ncu.csv $CMD > /dev/null 2>&1; echo ncu $?
