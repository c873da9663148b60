"""Summarise an `ncu --set full` report into profiles/.

    python tools/ncu_summarize.py gpurun_out/prof_full.ncu-rep profiles/r01_ncu_full_summary.json

Writes one record per captured kernel launch (duration, DRAM bytes, occupancy,
issue activity, the main stall ratios, instruction count, shared-memory bank
conflicts) and refreshes profiles/ncu_traffic.json, the per-kernel DRAM bytes
per launch that bench.py reports as `roofline.traffic`.
"""
import csv
import io
import json
import os
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "launch__grid_size", "launch__block_size",
]
BENCH_NAME = {"fx_kernel": "fft_x", "fy_kernel": "fft_y", "z_kernel": "fft_z", "zp_kernel": "fft_z",
              "iy_kernel": "ifft_y", "iy_tma_kernel": "ifft_y", "ix_kernel": "ifft_x",
              "splat_weighted_kernel": "splat", "texture_kernel": "texture", "sparse_clear_kernel": "clear"}
C2_N = 256  # traffic keys: bench name at the C2 grid, "name@N" at an N^3 grid


def short(name: str) -> str:
    n = name.split("(")[0]
    n = n.replace("void ", "").split("::")[-1]
    return n


def main(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    units = rows[1]
    ki = hdr.index("Kernel Name")
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3,
             "msecond": 1e3, "usecond": 1.0, "nsecond": 1e-3}
    recs = []
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        rec = {"kernel": short(r[ki])}
        for m in METRICS:
            if m in hdr:
                j = hdr.index(m)
                v = r[j].replace(",", "")
                try:
                    rec[m] = float(v) * scale.get(units[j], 1.0)  # bytes, microseconds
                except ValueError:
                    rec[m] = v
        recs.append(rec)
    json.dump(recs, open(out, "w"), indent=1)
    tpath = os.path.join(os.path.dirname(out), "ncu_traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for rec in recs:
        base = rec["kernel"].split("<")[0]
        targ = rec["kernel"].split("<")[1].split(">")[0].split(",")[0] if "<" in rec["kernel"] else ""
        n = int(targ) if targ.isdigit() else C2_N
        if base in BENCH_NAME:
            key = BENCH_NAME[base] if n == C2_N else f"{BENCH_NAME[base]}@{n}"
            rb, wb = rec.get("dram__bytes_read.sum", 0.0), rec.get("dram__bytes_write.sum", 0.0)
            # ncu reports (M)bytes per the unit row; raw page units are bytes for these counters
            traffic[key] = {
                "dram_bytes_per_launch": int(rb + wb),
                "ncu_duration_us": rec.get("gpu__time_duration.sum"),
                "source": f"{os.path.basename(rep)}: ncu --set full --clock-control none, "
                          "bench.py --streams 1 (cold cache, serialised)"}
            if n != C2_N:
                traffic[key]["source"] = f"{os.path.basename(rep)}: ncu --set full --clock-control none, bench.py " \
                                         f"--workload {'c3' if n == 512 else 'c5'} (one launch, serialised)"
    json.dump(traffic, open(tpath, "w"), indent=1)
    print(f"{len(recs)} launches -> {out}; traffic table {tpath}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
