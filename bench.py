# SPDX-License-Identifier: Apache-2.0
"""Benchmark of the B200 FTR frame path (BASELINE.json metric):
"reconstructed frames/sec at 256^3 grid, 4x512x424 RGB-D views; per-stage ms/frame".

One step = one reconstructed + textured frame of the 300-frame synthetic kick
stream (config C2: 4 Kinect2-like views 512x424, f=365, 256^3 grid, weighted
splat).  `value` = frames/s with inputs resident in HBM (device views, device
output); `e2e` = frames/s through the same C-ABI call with pinned HOST views
and host output (H2D of the views + D2H of the textured mesh in the timed
region).  Multi-GPU (torchrun): frame-parallel, rank r reconstructs frames
r, r+N, ... (no data-path collective); time = max over ranks.

`--impl reference` times the CPU oracle port of the reference path
(oracle/, restated from /root/reference/proj/core) on the host cores.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "reconstructed frames/sec at 256^3 grid, 4x512x424 RGB-D views; per-stage ms/frame"
STREAM = 300
DIMS = (256, 256, 256)
K_VIEWS, W, H, F = 4, 512, 424, 365.0
WORKLOAD = "C2: 300-frame synthetic kick stream, 4 views 512x424 depth+RGB (f=365, 2500 mm circle rig), 256^3 grid"


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


class Clocks:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    def __init__(self, device):
        self.device, self.samples, self._stop, self._t = device, [], threading.Event(), None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                self.samples.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], None, set()
        for s in self.samples:
            try:
                sm.append(float(s[0]))
                mx = float(s[1])
                for n, v in zip(names, s[3:7]):
                    if v.lower() == "active":
                        reasons.add(n)
            except Exception:
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O
    rig = O.make_circle_rig(K_VIEWS, 0, 2500, 1000, W, H, F)
    threads = O.lib().orc_hardware_threads()

    def frame_inputs(f):
        body = O.kick_body(STREAM, f)
        views = [O.render_frame(rig[k], body, k, f) for k in range(K_VIEWS)]
        return [v.depth for v in views], [v.mask for v in views], [v.rgb for v in views]

    t0 = time.perf_counter()
    inp = frame_inputs(0)
    O.reconstruct_frame(rig, *inp, dims=DIMS, want_volume=False)
    t_frame = time.perf_counter() - t0
    # bounded sample: at most ~150 s of CPU work for the timed steps
    steps = max(1, min(args.steps, int(150.0 / max(t_frame, 1e-3))))
    warm = min(args.warmup, 1)
    for i in range(warm):
        O.reconstruct_frame(rig, *frame_inputs(1 + i), dims=DIMS, want_volume=False)
    stage = {"raw_ms": [], "weights_ms": [], "volumetric_ms": [], "other_ms": [], "blend_ms": [],
             "splat_ms": [], "integrate_ms": [], "iso_ms": [], "mc_ms": []}
    total = 0.0
    for i in range(steps):
        f = (7 * i + 3) % STREAM
        inp = frame_inputs(f)
        t0 = time.perf_counter()
        r = O.reconstruct_frame(rig, *inp, dims=DIMS, want_volume=False)
        total += time.perf_counter() - t0
        assert r.status == 0
        for k in stage:
            stage[k].append(r.timings[k])
    fps = steps / total
    sample = (f"{steps} frame(s) of the C2 stream (of {args.steps} requested steps; bounded to ~150 s), "
              f"CPU oracle restated from proj/core (splat on {threads} threads over z-slabs as splat.cpp:59-78, "
              f"other stages single-threaded as the reference; own fp64 radix-2 FFT instead of FFTW)")
    line = {"metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world, "steps": steps, "warmup": warm,
            "ms_per_step": 1000.0 * total / steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": WORKLOAD, "grid": list(DIMS), "views": K_VIEWS},
            "stages_ms": {k: float(np.mean(v)) for k, v in stage.items()},
            "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline_sample():
    """The oracle on the host (rank 0, N=1): 2 frames of C2 (~10-20 s)."""
    from oracle import oracle as O
    rig = O.make_circle_rig(K_VIEWS, 0, 2500, 1000, W, H, F)
    ts = []
    for f in (10, 200):
        body = O.kick_body(STREAM, f)
        views = [O.render_frame(rig[k], body, k, f) for k in range(K_VIEWS)]
        t0 = time.perf_counter()
        r = O.reconstruct_frame(rig, [v.depth for v in views], [v.mask for v in views], [v.rgb for v in views],
                                dims=DIMS, want_volume=False)
        ts.append(time.perf_counter() - t0)
        assert r.status == 0
    threads = O.lib().orc_hardware_threads()
    return {"value": len(ts) / sum(ts), "unit": "frames/s", "cores": threads, "kind": "port",
            "sample": f"2 frames (#10, #200) of the C2 stream; CPU oracle port of proj/core, splat on {threads} "
                      f"threads (splat.cpp:59-78), other stages single-threaded as the reference, fp64 radix-2 "
                      f"FFT in place of FFTW; {os.cpu_count()} host CPUs"}


# ------------------------------------------------------------------ GPU arm
def sparse_stats(pos, origin, edge, nx, ny, nz):
    """Touched 32-voxel x-chunks and non-empty voxel rows of the splat
    accumulator (the same marking rule as k_splat.cu: rows floor(c)-1..+2 in
    y and z, chunks of x in [floor(cx)-1, floor(cx)+2])."""
    c = (np.asarray(pos) - np.asarray(origin)) / edge
    f = np.floor(c).astype(np.int64)
    keys = []
    for oy in range(4):
        for oz in range(4):
            y = f[:, 1] - 1 + oy
            z = f[:, 2] - 1 + oz
            ok = (y >= 0) & (y < ny) & (z >= 0) & (z < nz) & (f[:, 0] + 2 >= 0) & (f[:, 0] - 1 < nx)
            row = (z * ny + y)[ok]
            c0 = np.maximum(f[ok, 0] - 1, 0) // 32
            c1 = np.minimum(f[ok, 0] + 2, nx - 1) // 32
            keys += [row * 64 + c0, row * 64 + c1]
    keys = np.unique(np.concatenate(keys)) if keys else np.zeros(0, np.int64)
    rows = np.unique(keys // 64)
    return len(keys), len(rows), len(np.unique(rows // ny))


def alg_bytes(nx, ny, nz, P, V, T, k, chunks, nzrows, nzplanes):
    """Compulsory bytes per launch in the fp32 device layout (each tensor read
    once and written once; the sparse clear / F-x / F-y touch only the splat's
    32-voxel chunks and non-empty rows) — SURVEY §8(d) adapted, see DESIGN.md."""
    N = nx * ny * nz
    Nh = nz * ny * (nx // 2 + 1)
    rows = ny * nz
    line = 8 * (nx // 2 + 1)
    return {"clear": 16 * 32 * chunks + 8 * rows, "splat": 16 * 64 * P + 4 * 16 * P,
            "fft_x": 16 * 32 * chunks + 4 * rows + 3 * line * nzrows,
            "fft_y": 3 * line * nzrows + 4 * rows + 2 * line * ny * nzplanes,
            "fft_z": 2 * line * ny * nzplanes + 8 * Nh, "ifft_y": 2 * 8 * Nh, "ifft_x": 8 * Nh + 4 * N + 8 * rows,
            "mc": 8 * rows, "preprocess": k * W * H * 7 + P * 60, "iso": P * 32, "texture": V * (24 + 13 * k)}


def run_gpu(args):
    rank, world, local = dist_env()
    import torch
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1712_03084_b200 import _lib as L
    from paper_1712_03084_b200 import volcap as vc
    lib = L.lib()
    S = max(1, args.streams)
    ctxs = [vc.Context(local) for _ in range(S)]  # one context (stream + buffers) per concurrent frame
    ctx = ctxs[0]
    h = ctx.handle
    dev = torch.device("cuda", local)
    streams = [torch.cuda.ExternalStream(c.stream(), device=dev) for c in ctxs]

    rig = vc.make_circle_rig(K_VIEWS, 0, 2500, W, H, F)
    sensors = rig.c_array(K_VIEWS)
    n_pix = W * H
    per_view = n_pix * 2 + n_pix + n_pix * 3
    frame_bytes = K_VIEWS * per_view
    # device-resident stream (rendered on the GPU) + pinned host copy for e2e
    dbuf = C.c_void_p()
    L.check(lib.vc_device_alloc(h, C.c_size_t(STREAM * frame_bytes), C.byref(dbuf)), h)
    hbuf = C.c_void_p()
    L.check(lib.vc_host_alloc(h, C.c_size_t(STREAM * frame_bytes), C.byref(hbuf)), h)

    def view_ptrs(base, f, k):
        o = base + f * frame_bytes + k * per_view
        return o, o + 2 * n_pix, o + 3 * n_pix

    for f in range(STREAM):
        body = vc.kick_body(STREAM, f)
        for k in range(K_VIEWS):
            d, m, c = view_ptrs(dbuf.value, f, k)
            L.check(lib.vc_synth_render(h, C.byref(sensors[k]), C.byref(body), C.c_double(0.0), C.c_uint64(1),
                                        C.c_double(1.0), k, f, C.c_void_p(d), C.c_void_p(m), C.c_void_p(c),
                                        L.VC_MEM_DEVICE), h)
    L.check(lib.vc_memcpy(h, hbuf, dbuf, C.c_size_t(STREAM * frame_bytes), L.VC_MEM_HOST, L.VC_MEM_DEVICE), h)

    def views_for(base, f, kind):
        arr = (L.View * K_VIEWS)()
        for k in range(K_VIEWS):
            d, m, c = view_ptrs(base, f, k)
            arr[k] = L.View(d, m, c, 0, 0, 0, kind)
        return arr

    dev_views = [views_for(dbuf.value, f, L.VC_MEM_DEVICE) for f in range(STREAM)]
    host_views = [views_for(hbuf.value, f, L.VC_MEM_HOST) for f in range(STREAM)]
    from paper_1712_03084_b200.frame_parallel import max_over_ranks, shard_frames
    cfg = vc.ReconConfig(dims=DIMS).to_c()
    outs = [L.TexturedMesh() for _ in range(S)]
    out = outs[0]
    my_frames = shard_frames(STREAM, rank, world) or [0]
    d2h_acc = [0] * S

    def frame(i, views, s=0):
        o = outs[s]
        L.check(lib.vc_reconstruct_frame(ctxs[s].handle, sensors, views[my_frames[i % len(my_frames)]], K_VIEWS,
                                         C.byref(cfg), C.byref(o), None), ctxs[s].handle)
        d2h_acc[s] += o.vertex_count * (12 + 12 + 24 + 3 + 1 + K_VIEWS * (1 + 8 + 4)) + o.triangle_count * 12

    def run_steps(views, steps):
        """`steps` frames over S host threads, each driving its own context."""
        if S == 1:
            for i in range(steps):
                frame(i, views, 0)
            return
        errs = []

        def worker(s):
            try:
                for i in range(s, steps, S):
                    frame(i, views, s)
            except Exception as e:  # surfaced after join
                errs.append(e)
        ts = [threading.Thread(target=worker, args=(s,)) for s in range(S)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        if errs:
            raise errs[0]

    def timed(views, steps):
        master = torch.cuda.current_stream(dev)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        for i in range(S):
            d2h_acc[i] = 0
        ev0.record(master)
        for st in streams:
            st.wait_event(ev0)
        t0 = time.perf_counter()
        run_steps(views, steps)
        for st in streams:
            e = torch.cuda.Event()
            e.record(st)
            master.wait_event(e)
        ev1.record(master)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        ms = max_over_ranks(ev0.elapsed_time(ev1), device="cuda")
        return ms, wall, sum(d2h_acc) / steps

    # ---- device-resident (value)
    for c in ctxs:
        lib.vc_ctx_set_output(c.handle, L.VC_MEM_DEVICE)
    run_steps(dev_views, max(args.warmup, S))
    with Clocks(local) as clk:
        ms, wall, _ = timed(dev_views, args.steps)
    total_frames = args.steps * world
    value = total_frames / (ms / 1000.0)
    kernels = lib.vc_ctx_kernels_per_frame(h)

    # ---- per-stage / per-kernel timings (profiling replay, separate from the timed loop)
    lib.vc_ctx_set_profiling(h, 1)
    tm = L.StageTimings()
    kt = (C.c_double * 16)()
    acc = {}
    prof_frames = min(20, STREAM)
    ker = np.zeros(11)
    for i in range(prof_frames):
        L.check(lib.vc_reconstruct_frame(h, sensors, dev_views[(i * 13) % STREAM], K_VIEWS, C.byref(cfg),
                                         C.byref(out), C.byref(tm)), h)
        for n, _ in L.StageTimings._fields_:
            acc[n] = acc.get(n, 0.0) + getattr(tm, n) / prof_frames
        lib.vc_ctx_kernel_times(h, kt, 16)
        ker += np.array(kt[:11]) / prof_frames
    lib.vc_ctx_set_profiling(h, 0)
    names = ["preprocess", "clear", "splat", "fft_x", "fft_y", "fft_z", "ifft_y", "ifft_x", "iso", "mc", "texture"]
    kernel_ms = dict(zip(names, ker.tolist()))
    P, V, T = out.point_count, out.vertex_count, out.triangle_count
    pos = np.zeros((P, 3))
    L.check(lib.vc_export_points(h, C.c_void_p(pos.ctypes.data), None, None, None, None), h)
    chunks, nzrows, nzplanes = sparse_stats(pos, out.grid.origin[:], out.grid.edge_mm, *DIMS)
    ab = alg_bytes(*DIMS, P, V, T, K_VIEWS, chunks, nzrows, nzplanes)
    bw = {n: ab[n] / (kernel_ms[n] * 1e-3) / 1e9 for n in names if kernel_ms[n] > 0}
    if not all(n in bw for n in ["clear", "fft_x", "fft_y", "fft_z", "ifft_y", "ifft_x"]):
        raise RuntimeError(f"per-kernel event timings missing: {kernel_ms}")
    pk = peaks()
    hbm = float(pk.get("hbm_gbs", 6650.0))
    fft_names = ["fft_x", "fft_y", "fft_z", "ifft_y", "ifft_x"]
    dom = max(fft_names + ["clear"], key=lambda n: kernel_ms[n])
    try:  # dram bytes per launch of the same kernel from the committed ncu --set full capture
        traffic = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))[dom]["dram_bytes_per_launch"]
    except Exception:
        traffic = None
    roofline = {"bound": "hbm", "kernel": dom, "achieved": bw[dom], "peak": hbm, "unit": "GB/s",
                "frac": bw[dom] / hbm, "traffic": traffic,
                "algorithmic_bytes": ab[dom], "avg_launch_ms": kernel_ms[dom],
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)" if "_fallback" not in pk else "fallback"}

    # ---- e2e through the C-ABI with host buffers
    for c in ctxs:
        lib.vc_ctx_set_output(c.handle, L.VC_MEM_HOST)
    run_steps(host_views, max(args.warmup, S))
    e2e_ms, _, d2h_per = timed(host_views, args.steps)
    e2e_value = total_frames / (e2e_ms / 1000.0)

    if rank == 0:
        cpu = cpu_baseline_sample() if (world == 1 and not args.no_cpu_baseline) else None
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOAD, "grid": list(DIMS), "views": K_VIEWS, "splat": "weighted",
                       "frames_per_rank": args.steps, "parallelism": f"frame-parallel x{world}",
                       "streams_per_gpu": S,
                       "l2": "per-step working set (~0.55 GB volume buffers + 5.2 MB inputs) exceeds the 126 MB L2",
                       "precision": "fp32 splat/FFT, fp64 binning, projections, MC vertices"},
            "e2e": {"value": e2e_value, "unit": "frames/s", "h2d_bytes_per_step": frame_bytes,
                    "d2h_bytes_per_step": int(d2h_per)},
            "gpu_launches": kernels * args.steps,
            "roofline": roofline,
            "stages_ms": {k: round(v, 4) for k, v in acc.items()},
            "kernel_ms": {k: round(v, 4) for k, v in kernel_ms.items()},
            "kernel_gbs": {k: round(v, 1) for k, v in bw.items()},
            "mesh": {"points": P, "vertices": V, "triangles": T},
            "sparsity": {"touched_chunks": chunks, "chunks_total": DIMS[1] * DIMS[2] * (DIMS[0] // 32),
                         "nonzero_rows": nzrows, "rows_total": DIMS[1] * DIMS[2],
                         "nonzero_planes": nzplanes, "planes_total": DIMS[2]},
            "algorithmic_bytes": ab,
            "clocks": clk.summary(),
            "wall_s": wall,
        }
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    lib.vc_device_free(h, dbuf)
    lib.vc_host_free(h, hbuf)
    for c in ctxs:
        c.close()
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--streams", type=int, default=3,
                    help="concurrent frames per GPU (one context + host thread each)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl != "reference":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
