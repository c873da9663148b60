# A/B of the Nyquist-column packing per pass (VC_NYQ_PACK bits: 2 = Z, 4 = I-y; F-y never packs)
for m in ${MODES:-0 7}; do
  VC_NYQ_PACK=$m python bench.py --steps 600 --warmup 5 --no-cpu-baseline > gpurun_out/ab_$m.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/ab_$m.json').read().strip().splitlines()[-1]); k=d['kernel_ms']; print('mode=$m', round(d['value'],1), k['fft_y'], k['fft_z'], k['ifft_y'])"
done
