for S in 3 4 5 6; do
  timeout 300 python bench.py --steps 3000 --warmup 5 --no-cpu-baseline --no-fft-comparator --streams $S > gpurun_out/gsw_$S.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/gsw_$S.json').read().strip().splitlines()[-1]); print('S=$S', round(d['value'],1), round(d['e2e']['value'],1))"
done
