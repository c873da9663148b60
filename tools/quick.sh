# quick perf check: S=1 and S=4 bench lines + per-kernel ms (profiled replay)
for S in ${STREAMS:-1 4}; do
  python bench.py --steps ${STEPS:-600} --warmup 5 --no-cpu-baseline --streams $S > gpurun_out/q_s$S.json 2>gpurun_out/q_s$S.err
  python -c "import json; d=json.loads(open('gpurun_out/q_s$S.json').read().strip().splitlines()[-1]); print('S=$S', round(d['value'],1), round(d['e2e']['value'],1), d['clocks'].get('sm_mhz'), {k: round(v*1000,1) for k,v in d['kernel_ms'].items()})"
done
