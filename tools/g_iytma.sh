timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for rep in 1 2; do for v in 1 0; do
  VC_IY_TMA=$v timeout 300 python bench.py --steps 600 --warmup 5 --no-cpu-baseline --no-fft-comparator --streams 1 > gpurun_out/git.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/git.json').read().strip().splitlines()[-1]); print('IYTMA=$v S1', round(d['value'],1), d['kernel_ms']['ifft_y'])"
  VC_IY_TMA=$v timeout 300 python bench.py --steps 4000 --warmup 5 --no-cpu-baseline --no-fft-comparator > gpurun_out/git4.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/git4.json').read().strip().splitlines()[-1]); print('IYTMA=$v S4', round(d['value'],1), round(d['e2e']['value'],1))"
done; done
