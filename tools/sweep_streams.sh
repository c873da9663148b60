# frames/s vs concurrent frames per GPU (contexts + host threads)
for S in ${STREAMS:-1 2 3 4 6}; do
  python bench.py --steps 600 --warmup 5 --no-cpu-baseline --streams $S > gpurun_out/sweep_s$S.json 2>gpurun_out/sweep_s$S.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/sweep_s$S.json').read().strip().splitlines()[-1]); print('S=$S', round(d['value'],1), round(d['e2e']['value'],1), d['clocks'].get('sm_mhz'))"
done
