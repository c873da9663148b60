timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2_parity.py -x -q > gpurun_out/g9_pytest.log 2>&1; echo pytest $?; tail -2 gpurun_out/g9_pytest.log
timeout 300 python bench.py --steps 600 --warmup 5 --no-cpu-baseline --streams 1 > gpurun_out/g9_s1.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/g9_s1.json').read().strip().splitlines()[-1]); print('S1', round(d['value'],1), {k: round(v*1000,1) for k,v in d['kernel_ms'].items()})"
timeout 300 python bench.py --steps 2000 --warmup 5 --no-cpu-baseline > gpurun_out/g9_s4.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/g9_s4.json').read().strip().splitlines()[-1]); print('S4', round(d['value'],1), round(d['e2e']['value'],1))"
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-fft-comparator --streams 1"
timeout 300 ncu --metrics gpu__time_duration.sum,lts__t_sectors_op_red.sum,lts__t_requests_op_red.sum,lts__t_sectors_op_atom.sum,lts__t_requests_op_atom.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed_op_global_red.sum --clock-control none -k regex:"splat_weighted" -s 3 -c 2 --csv $CMD > gpurun_out/g9_splat_ncu.csv 2>gpurun_out/g9_splat_ncu.err; echo ncu $?
