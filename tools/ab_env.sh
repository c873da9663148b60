# A/B of an environment switch: VAR=name VALUES="a b c" bash tools/ab_env.sh
for v in $VALUES; do
  env $VAR=$v python bench.py --steps 800 --warmup 5 --no-cpu-baseline > gpurun_out/ab_env_$v.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/ab_env_$v.json').read().strip().splitlines()[-1]); k=d['kernel_ms']; print('$VAR=$v', round(d['value'],1), round(d['e2e']['value'],1), k['ifft_y'], k['ifft_x'])"
done
