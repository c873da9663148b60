"""Per-stage roofline table (markdown) from a bench.py JSON line:
    python tools/stage_table.py profiles/r02_bench_full.jsonl"""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
peak = d["roofline"]["peak"]
ab, km = d["algorithmic_bytes"], d["kernel_ms"]
dense = {"fft_z": d["roofline"]["algorithmic_bytes"]}
print(f"| stage | µs | compulsory bytes | TB/s | of {peak / 1000:.2f} TB/s |")
print("|---|---|---|---|---|")
for k, ms in km.items():
    b = ab.get(k)
    if not b or not ms:
        continue
    tbs = b / (ms * 1e-3) / 1e12
    print(f"| {k} | {ms * 1000:.1f} | {b / 1e6:.1f} MB | {tbs:.2f} | {tbs * 1000 / peak:.2f} |")
tot = sum(v for v in ab.values() if isinstance(v, (int, float)))
print(f"\nframe: {tot / 1e6:.0f} MB compulsory in {d['ms_per_step']:.4f} ms/frame (S={d['config'].get('streams_per_gpu')}) "
      f"= {tot / (d['ms_per_step'] * 1e-3) / 1e12:.2f} TB/s = {tot / (d['ms_per_step'] * 1e-3) / 1e9 / peak:.2f} of peak")
