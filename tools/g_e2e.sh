python - <<'PY'
import torch, time
x = torch.empty(5210112, dtype=torch.uint8).pin_memory(); y = torch.empty(6138733, dtype=torch.uint8, device='cuda'); xd = torch.empty(5210112, dtype=torch.uint8, device='cuda'); yh = torch.empty(6138733, dtype=torch.uint8).pin_memory()
for name, src, dst in (("h2d", x, xd), ("d2h", y, yh)):
    for _ in range(10): dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize(); t=time.perf_counter()
    for _ in range(200): dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize(); dt=(time.perf_counter()-t)/200
    print(name, round(src.numel()/dt/1e9,1), 'GB/s', round(dt*1e3,3), 'ms/frame')
PY
for S in 4 6 8; do
VC_E2E_SPLIT=1 timeout 300 python bench.py --steps 3000 --warmup 5 --no-cpu-baseline --no-fft-comparator --streams $S > gpurun_out/ge_$S.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/ge_$S.json').read().strip().splitlines()[-1]); print('S=$S', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d.get('e2e_split'))"
done
