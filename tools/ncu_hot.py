"""Hot SASS segments of one kernel in an ncu report (needs --set full / source counters).
usage: python tools/ncu_hot.py report.ncu-rep kernel_regex [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--kernel-name", "regex:" + kre, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
iS, iI = hdr.index("Source"), hdr.index("Instructions Executed")
iW = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[iI]) for r in data if len(r) > iI and r[iI].isdigit())
samp = sum(int(r[iW]) for r in data if len(r) > iW and r[iW].isdigit())
print(rows[0][1][:100], "| warp-instructions", tot, "| stall samples", samp)
segs, cur = [], None
for idx, r in enumerate(data):
    if len(r) <= iI or not r[iI].isdigit():
        continue
    n, w = int(r[iI]), int(r[iW]) if r[iW].isdigit() else 0
    op = r[iS].strip().split()[0] if r[iS].strip() else ""
    if op.startswith("@") and len(r[iS].split()) > 1:
        op = r[iS].strip().split()[1]
    if cur and cur[2] == n:
        cur[1] = idx; cur[3] += n; cur[4] += w; cur[5].append(op)
    else:
        cur = [idx, idx, n, n, w, [op]]
        segs.append(cur)
segs.sort(key=lambda s: -(s[3] + s[4] * tot / max(samp, 1)))
for s in segs[:top]:
    c = collections.Counter(x.split(".")[0] for x in s[5])
    print(f"[{s[0]:5d}-{s[1]:5d}] exec/inst={s[2]:7d} inst={100*s[3]/tot:5.1f}% stalls={100*s[4]/max(samp,1):5.1f}% "
          f"{c.most_common(6)}")
