# A/B of an environment switch on value and e2e: VAR=name VALUES="a b" [STREAMS=4] bash tools/ab_env_e2e.sh
for v in $VALUES; do
  env $VAR=$v python bench.py --steps 800 --warmup 5 --no-cpu-baseline --streams ${STREAMS:-4} > gpurun_out/ab_e2e_$v.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/ab_e2e_$v.json').read().strip().splitlines()[-1]); print('$VAR=$v', round(d['value'],1), round(d['e2e']['value'],1))"
done
