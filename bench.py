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
STREAM = 300            # frames of the synthetic kick stream (make_kick_sequence(300), capsule.cpp:197-219)
W, H, F = 512, 424, 365.0


class Workload:
    """One BASELINE.json config as a bench workload.  `frames` views are kept
    resident (device + pinned host); resident frame j is kick-stream frame
    j * STREAM // frames; global step g reconstructs resident frame
    stream_frame(g, frames) (stride 97, coprime with 300 and 60: any `frames`
    consecutive global steps visit every resident frame once)."""

    def __init__(self, key, metric, dims, k, hd, frames, text, stream=STREAM, host_ring=None):
        self.key, self.metric, self.dims, self.k, self.hd, self.frames, self.text = key, metric, dims, k, hd, frames, text
        self.rgb_w, self.rgb_h = (1920, 1080) if hd else (W, H)
        self.stream = stream        # length of the kick sequence the frames sample (make_kick_sequence(n))
        self.host_ring = host_ring  # e2e leg: pinned host copies of the first `host_ring` frames only

    def kick_frame(self, j):
        return j * self.stream // self.frames

    @property
    def view_bytes(self):
        return W * H * 3 + self.rgb_w * self.rgb_h * 3  # depth u16 + mask u8 + RGB8

    @property
    def frame_bytes(self):
        return self.k * self.view_bytes


WORKLOADS = {
    "c2": Workload("c2", METRIC, (256, 256, 256), 4, False, STREAM,
                   "C2: 300-frame synthetic kick stream, 4 views 512x424 depth+RGB (f=365, 2500 mm circle rig), "
                   "256^3 grid"),
    "c3": Workload("c3", "reconstructed frames/sec at 512^3 grid, 6x512x424 depth + 1920x1080 colour views",
                   (512, 512, 512), 6, True, 60,
                   "C3: 60 frames of the kick stream (every 5th of 300), 6 views 512x424 depth (f=365) + 1920x1080 "
                   "colour (f=1060, 52 mm offset), 512^3 grid"),
    # a 4096-frame kick stream, 256^3, K=4, sharded frame-parallel over the ranks; the
    # views are rendered on the device and stay resident (21 GB); one timed step per frame of the shard
    "c4": Workload("c4", "reconstructed frames/sec over a 4096-frame kick stream at 256^3 grid, 4x512x424 RGB-D views",
                   (256, 256, 256), 4, False, 4096,
                   "C4: 4096-frame kick stream (make_kick_sequence(4096)), 4 views 512x424 depth+RGB, 256^3 grid, "
                   "frame-parallel shards over the ranks; each rank reconstructs its whole shard once",
                   stream=4096, host_ring=512),
    # one GPU: whole 1024^3 frames (two in flight: ~40 GB of buffers each); N>1: run_c5's z-slab decomposition
    "c5": Workload("c5", "reconstructed frames/sec at 1024^3 grid, 4x512x424 RGB-D views", (1024, 1024, 1024), 4, False,
                   4, "C5: 4 views 512x424 of the kick stream (4 resident frames), 1024^3 grid, weighted splat"),
}
WORKLOAD = WORKLOADS["c2"].text
DIMS = WORKLOADS["c2"].dims
K_VIEWS = 4


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
def oracle_rig(O, wl):
    rig = O.make_circle_rig(wl.k, 0, 2500, 1000, W, H, F)
    if wl.hd:  # C3 colour camera; Sensor::rgb_relative, types.hpp:68-76
        for i in range(wl.k):
            rig[i].rgb_intr = O.Intrinsics(1060.0, 1060.0, 959.5, 539.5, 1920, 1080)
            rig[i].rgb_relative.t[0] = 52.0
    return rig


def oracle_inputs(O, rig, wl, j):
    """Views of resident frame j (kick frame wl.kick_frame(j)), rendered by the oracle."""
    f = wl.kick_frame(j)
    body = O.kick_body(wl.stream, f)
    views = [O.render_frame(rig[k], body, k, f) for k in range(wl.k)]
    return [v.depth for v in views], [v.mask for v in views], [v.rgb for v in views]


def cpu_frame_fn(O, wl):
    """The CPU implementation the reference legs time: the REFERENCE's own code
    (proj/core compiled unmodified into oracle/_ref/libref.so; kind "reference")
    when it was built, else the oracle restatement (kind "port").  Returns
    (kind, frame(rig, depths, masks, rgbs) -> seconds, description)."""
    from oracle import ref as R
    if R.available(0):
        def frame(rig, d, m, c):
            t0 = time.perf_counter()
            r = R.reconstruct_frame(rig, d, m, c, dims=wl.dims, want_volume=False)
            dt = time.perf_counter() - t0
            assert r.status == 0
            return dt, None
        return "reference", frame, ("the reference's own proj/core sources (reconstruct_frame + texture.cpp) compiled "
                                    "unmodified into oracle/_ref against the Eigen/doctest shims, its FFTW3 calls "
                                    "served by the oracle's fp64 FFT (FFTW is absent); splat on all host threads "
                                    "(splat.cpp:59-78), other stages single-threaded as written")

    def frame(rig, d, m, c):
        t0 = time.perf_counter()
        r = O.reconstruct_frame(rig, d, m, c, dims=wl.dims, want_volume=False)
        dt = time.perf_counter() - t0
        assert r.status == 0
        return dt, r.timings
    return "port", frame, ("CPU oracle restated from proj/core (splat on all host threads over z-slabs as "
                           "splat.cpp:59-78, other stages single-threaded as the reference; own fp64 radix-2 FFT "
                           "instead of FFTW)")


def run_reference(args):
    """The reference's CPU path on the host cores (its own compiled code when
    oracle/_ref was built, else the oracle restatement) on the same workload,
    frames and metric as the GPU arm."""
    from paper_1712_03084_b200.frame_parallel import stream_frame
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O
    wl = WORKLOADS[args.workload]
    rig = oracle_rig(O, wl)
    threads = O.lib().orc_hardware_threads()
    kind, frame, what = cpu_frame_fn(O, wl)
    t_frame, _ = frame(rig, *oracle_inputs(O, rig, wl, stream_frame(0, wl.frames)))
    # bounded sample: at most ~150 s of CPU work for the timed steps
    steps = max(1, min(args.steps, int(150.0 / max(t_frame, 1e-3))))
    warm = min(args.warmup, 1)
    for i in range(warm):
        frame(rig, *oracle_inputs(O, rig, wl, stream_frame(1 + i, wl.frames)))
    stage = {"raw_ms": [], "weights_ms": [], "volumetric_ms": [], "other_ms": [], "blend_ms": [],
             "splat_ms": [], "integrate_ms": [], "iso_ms": [], "mc_ms": []}
    total = 0.0
    used = []
    for i in range(steps):
        j = stream_frame(i, wl.frames)  # the GPU arm's global-step order
        used.append(wl.kick_frame(j))
        dt, timings = frame(rig, *oracle_inputs(O, rig, wl, j))
        total += dt
        if timings:
            for k in stage:
                stage[k].append(timings[k])
    fps = steps / total
    sample = (f"{steps} frame(s) of the {wl.key.upper()} stream (kick frames {used[:6]}{'...' if steps > 6 else ''}, "
              f"the GPU arm's first global steps; of {args.steps} requested steps; bounded to ~150 s); {what}; "
              f"{threads} host threads")
    line = {"metric": wl.metric, "value": fps, "unit": "frames/s", "n_gpus": world, "steps": steps, "warmup": warm,
            "ms_per_step": 1000.0 * total / steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": wl.text, "grid": list(wl.dims), "views": wl.k},
            "stages_ms": {k: float(np.mean(v)) for k, v in stage.items() if v},
            "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": threads, "kind": kind, "sample": sample},
            "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline_sample(wl):
    """The reference's CPU path on the host (rank 0, N=1): 2 frames of the workload (~10-30 s)."""
    from oracle import oracle as O
    rig = oracle_rig(O, wl)
    kind, frame, what = cpu_frame_fn(O, wl)
    ts = []
    picks = (wl.frames // 30, wl.frames * 2 // 3)
    for j in picks:
        ts.append(frame(rig, *oracle_inputs(O, rig, wl, j))[0])
    threads = O.lib().orc_hardware_threads()
    return {"value": len(ts) / sum(ts), "unit": "frames/s", "cores": threads, "kind": kind,
            "sample": f"2 frames (kick #{wl.kick_frame(picks[0])}, #{wl.kick_frame(picks[1])}) of the "
                      f"{wl.key.upper()} stream; {what}; {os.cpu_count()} host CPUs"}


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
    # (no clear pass: F-x zeroes the chunks it reads — 16 B per voxel written
    # back — and I-x resets the row bits)
    return {"splat": 16 * 64 * P + 4 * 16 * P,
            "fft_x": 2 * 16 * 32 * chunks + 4 * rows + 3 * line * nzrows,
            "fft_y": 3 * line * nzrows + 4 * rows + 2 * line * ny * nzplanes,
            "fft_z": 2 * line * ny * nzplanes + 8 * Nh, "ifft_y": 2 * 8 * Nh, "ifft_x": 8 * Nh + 4 * N + 12 * rows,
            "mc": 8 * rows, "preprocess": k * W * H * 7 + P * 60, "iso": P * 32, "texture": V * (24 + 13 * k)}


def survey_bytes(nx, ny, nz, P, V, T, k):
    """SURVEY.md §8(d) algorithmic bytes per launch (fp32 device layout, each
    tensor read once and written once, dense), with the divergence epilogue
    of Appendix A.4(iv): y-C2C 3 in / 2 out, z-fused 2 in / 1 out."""
    N = nx * ny * nz
    Nh = nz * ny * (nx // 2 + 1)
    return {"preprocess": k * W * H * 7 + P * 32, "splat": 16 * N + 16 * 64 * P, "fft_x": 16 * N + 3 * 8 * Nh,
            "fft_y": 3 * 8 * Nh + 2 * 8 * Nh, "fft_z": 2 * 8 * Nh + 8 * Nh, "ifft_y": 2 * 8 * Nh,
            "ifft_x": 8 * Nh + 4 * N, "iso": P * 44, "mc": 4 * N + V * 24 + T * 12, "texture": V * (15 + 13 * k)}


def profile_kernels(lib, h, sensors, views_list, cfg, dims, out, k=4):
    """Per-stage and per-kernel-group CUDA-event times (profiling replay on
    context h, outside the timed loop) + the roofline of the dominant kernel."""
    from paper_1712_03084_b200 import _lib as L
    lib.vc_ctx_set_output(h, L.VC_MEM_DEVICE)
    lib.vc_ctx_set_profiling(h, 1)
    tm = L.StageTimings()
    kt = (C.c_double * 16)()
    acc = {}
    n = len(views_list)
    ker = np.zeros(11)
    for views in views_list:
        L.check(lib.vc_reconstruct_frame(h, sensors, views, k, C.byref(cfg), C.byref(out), C.byref(tm)), h)
        for nm, _ in L.StageTimings._fields_:
            acc[nm] = acc.get(nm, 0.0) + getattr(tm, nm) / n
        lib.vc_ctx_kernel_times(h, kt, 16)
        ker += np.array(kt[:11]) / n
    lib.vc_ctx_set_profiling(h, 0)
    names = ["preprocess", "clear", "splat", "fft_x", "fft_y", "fft_z", "ifft_y", "ifft_x", "iso", "mc", "texture"]
    kernel_ms = dict(zip(names, ker.tolist()))
    P, V, T = out.point_count, out.vertex_count, out.triangle_count
    pos = np.zeros((P, 3))
    L.check(lib.vc_export_points(h, C.c_void_p(pos.ctypes.data), None, None, None, None), h)
    sp = sparse_stats(pos, out.grid.origin[:], out.grid.edge_mm, *dims)
    ab = alg_bytes(*dims, P, V, T, k, *sp)
    bw = {nm: ab[nm] / (kernel_ms[nm] * 1e-3) / 1e9 for nm in names if nm in ab and kernel_ms[nm] > 0}
    if not all(nm in bw for nm in ["fft_x", "fft_y", "fft_z", "ifft_y", "ifft_x"]):
        raise RuntimeError(f"per-kernel event timings missing: {kernel_ms}")
    pk = peaks()
    hbm = float(pk.get("hbm_gbs", 6650.0))
    fft_names = ["fft_x", "fft_y", "fft_z", "ifft_y", "ifft_x"]
    dom = max(fft_names, key=lambda nm: kernel_ms[nm])
    traffic = None
    tkey = dom if tuple(dims) == DIMS else f"{dom}@{dims[0]}"
    try:  # dram bytes per launch of the same kernel at this grid from the committed ncu --set full capture
        traffic = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))[tkey]["dram_bytes_per_launch"]
    except Exception:
        traffic = None
    sb = survey_bytes(*dims, P, V, T, k)
    alg = sb.get(dom, ab[dom])
    achieved = alg / (kernel_ms[dom] * 1e-3) / 1e9
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": traffic,
                "algorithmic_bytes": alg, "bytes_source": "SURVEY.md §8(d) (divergence epilogue, dense)",
                "compulsory_bytes": ab[dom], "frac_compulsory": bw[dom] / hbm,
                "avg_launch_ms": kernel_ms[dom],
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)" if "_fallback" not in pk else "fallback"}
    return {"stages": acc, "kernel_ms": kernel_ms, "bw": bw, "ab": ab, "roofline": roofline, "P": P, "V": V, "T": T,
            "sparse": sp}


def fft_comparator(lib, device, grids):
    """cuFFT timed as a comparator (north_star): batched R2C of
    the 3 components + one fused filter kernel + C2R (the FFTW calls of
    integrate.cpp:31-34,44,63 on the GPU library) against our chain on the same
    dense pseudo-random field (no sparsity shortcuts), device-resident, CUDA
    events.  Timing only: cuFFT's C2R on the non-Hermitian filtered planes is
    undefined, so parity stays with our kernels."""
    from paper_1712_03084_b200 import _lib as L
    from paper_1712_03084_b200 import volcap as vc
    out = []
    try:
        cmp = C.CDLL(os.path.join(ROOT, "paper_1712_03084_b200", "libvc_cufft_cmp.so"))
    except OSError as e:
        return [{"error": f"libvc_cufft_cmp.so: {e}"}]
    for n in grids:
        iters = 20 if n <= 512 else 5
        ms_c = (C.c_double * 4)()
        rc = cmp.vcx_cufft_integrate_time(device, n, n, n, iters, ms_c)
        ctx = vc.Context(device)
        ms_o = (C.c_double * 6)()
        st = lib.vc_time_integrate(ctx.handle, n, n, n, iters, ms_o)
        ctx.close()
        if rc != 0 or st != 0:
            out.append({"grid": [n] * 3, "error": f"cufft rc={rc}, ours status={st}"})
            continue
        out.append({"grid": [n] * 3, "cufft_ms": ms_c[3], "ours_ms": ms_o[5], "speedup": ms_c[3] / ms_o[5],
                     "cufft_split_ms": {"r2c_x3": ms_c[0], "filter": ms_c[1], "c2r": ms_c[2]},
                     "ours_split_ms": dict(zip(["fft_x", "fft_y", "fft_z", "ifft_y", "ifft_x"], list(ms_o)[:5])),
                     "field": "dense pseudo-random 3-component field (every row/plane non-empty)", "iters": iters})
    return out


def run_gpu(args):
    rank, world, local = dist_env()
    import torch
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1712_03084_b200 import _lib as L
    from paper_1712_03084_b200 import volcap as vc
    from paper_1712_03084_b200.frame_parallel import max_over_ranks, rank_frames, stream_frame
    wl = WORKLOADS[args.workload]
    K, dims = wl.k, wl.dims
    lib = L.lib()
    S = max(1, args.streams if args.streams else (2 if wl.key == "c5" else 4))
    ctxs = [vc.Context(local) for _ in range(S)]  # one context (stream + buffers) per concurrent frame
    ctx = ctxs[0]
    h = ctx.handle
    dev = torch.device("cuda", local)
    streams = [torch.cuda.ExternalStream(c.stream(), device=dev) for c in ctxs]

    rig = vc.make_hd_rig(K) if wl.hd else vc.make_circle_rig(K, 0, 2500, W, H, F)
    sensors = rig.c_array(K)
    n_pix = W * H
    per_view, frame_bytes, NF = wl.view_bytes, wl.frame_bytes, wl.frames
    HF = min(NF, wl.host_ring or NF)  # frames with a pinned host copy (the e2e leg's inputs)
    # device-resident stream (rendered on the GPU) + pinned host copy for e2e
    dbuf = C.c_void_p()
    L.check(lib.vc_device_alloc(h, C.c_size_t(NF * frame_bytes), C.byref(dbuf)), h)
    hbuf = C.c_void_p()
    L.check(lib.vc_host_alloc(h, C.c_size_t(HF * frame_bytes), C.byref(hbuf)), h)

    def view_ptrs(base, j, k):
        o = base + j * frame_bytes + k * per_view
        return o, o + 2 * n_pix, o + 3 * n_pix

    for j in range(NF):
        f = wl.kick_frame(j)
        body = vc.kick_body(wl.stream, f)
        for k in range(K):
            d, m, c = view_ptrs(dbuf.value, j, k)
            L.check(lib.vc_synth_render(h, C.byref(sensors[k]), C.byref(body), C.c_double(0.0), C.c_uint64(1),
                                        C.c_double(1.0), k, f, C.c_void_p(d), C.c_void_p(m), C.c_void_p(c),
                                        L.VC_MEM_DEVICE), h)
    L.check(lib.vc_memcpy(h, hbuf, dbuf, C.c_size_t(HF * frame_bytes), L.VC_MEM_HOST, L.VC_MEM_DEVICE), h)

    def views_for(base, j, kind):
        arr = (L.View * K)()
        for k in range(K):
            d, m, c = view_ptrs(base, j, k)
            arr[k] = L.View(d, m, c, 0, 0, 0, kind)
        return arr

    dev_views = [views_for(dbuf.value, j, L.VC_MEM_DEVICE) for j in range(NF)]
    host_views = [views_for(hbuf.value, j % HF, L.VC_MEM_HOST) for j in range(NF)]
    cfg = vc.ReconConfig(dims=dims).to_c()
    outs = [L.TexturedMesh() for _ in range(S)]
    out = outs[0]
    # global step g = i * world + rank reconstructs resident frame stream_frame(g): every pose is sampled
    if wl.key == "c4":  # one timed step per frame of this rank's shard of the stream
        args.steps = len(range(rank, NF, world))
    my_frames = rank_frames(rank, world, max(args.steps, args.warmup, S), NF)
    d2h_acc = [0] * S

    def frame(i, views, s=0):
        o = outs[s]
        L.check(lib.vc_reconstruct_frame(ctxs[s].handle, sensors, views[my_frames[i % len(my_frames)]], K,
                                         C.byref(cfg), C.byref(o), None), ctxs[s].handle)
        d2h_acc[s] += o.vertex_count * (12 + 12 + 24 + 3 + 1 + K * (1 + 8 + 4)) + o.triangle_count * 12

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

    # ---- per-stage / per-kernel timings (profiling replay of the first 20 global steps, outside the timed loop)
    prof = profile_kernels(lib, h, sensors, [dev_views[stream_frame(i, NF)] for i in range(min(20, NF))], cfg,
                           dims, out, K)
    acc, kernel_ms, bw, ab, roofline = prof["stages"], prof["kernel_ms"], prof["bw"], prof["ab"], prof["roofline"]
    P, V, T = prof["P"], prof["V"], prof["T"]
    chunks, nzrows, nzplanes = prof["sparse"]

    # ---- e2e through the C-ABI with host buffers
    for c in ctxs:
        lib.vc_ctx_set_output(c.handle, L.VC_MEM_HOST)
    run_steps(host_views, max(args.warmup, S))
    e2e_ms, _, d2h_per = timed(host_views, args.steps)
    e2e_value = total_frames / (e2e_ms / 1000.0)
    split = None
    if os.environ.get("VC_E2E_SPLIT"):  # diagnostics: H2D only / D2H only
        for c in ctxs:
            lib.vc_ctx_set_output(c.handle, L.VC_MEM_DEVICE)
        h2d_ms, _, _ = timed(host_views, args.steps)
        for c in ctxs:
            lib.vc_ctx_set_output(c.handle, L.VC_MEM_HOST)
        d2h_ms, _, _ = timed(dev_views, args.steps)
        split = {"h2d_only_fps": total_frames / (h2d_ms / 1000.0), "d2h_only_fps": total_frames / (d2h_ms / 1000.0)}

    if rank == 0:
        cmp = None
        if world == 1 and not args.no_fft_comparator and wl.key != "c5":  # (the C2 line times 1024^3 too)
            cmp = fft_comparator(lib, local, [dims[0], 1024] if dims[0] < 1024 else [dims[0]])
            frame_fft = sum(kernel_ms[k] for k in ("fft_x", "fft_y", "fft_z", "ifft_y", "ifft_x"))
            for c in cmp:
                if c.get("grid") == list(dims):
                    c["ours_in_frame_ms"] = frame_fft  # the frame's chain with the splat's sparsity
        # (none at 1024^3: the reference's CPU path takes minutes per frame there)
        cpu = cpu_baseline_sample(wl) if (world == 1 and not args.no_cpu_baseline and wl.key != "c5") else None
        line = {
            "metric": wl.metric, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": wl.text, "grid": list(dims), "views": K, "splat": "weighted",
                       "frames_per_rank": args.steps, "parallelism": f"frame-parallel x{world}",
                       "frame_order": f"global step g = i*{world} + rank reconstructs resident frame (97 g) mod {NF}",
                       "streams_per_gpu": S,
                       "stream_frames": NF,
                       "e2e_inputs": ("pinned host copies of every resident frame" if HF == NF else
                                      f"pinned host copies of the first {HF} frames (frame j reads copy j mod {HF})"),
                       "l2": "per-step working set (volume buffers >= 0.5 GB + inputs) exceeds the 126 MB L2",
                       "precision": "fp32 splat/FFT, fp64 binning, projections, MC vertices"},
            "e2e": {"value": e2e_value, "unit": "frames/s", "h2d_bytes_per_step": frame_bytes,
                    "d2h_bytes_per_step": int(d2h_per)},
            "gpu_launches": kernels * args.steps,
            "roofline": roofline,
            "stages_ms": {k: round(v, 4) for k, v in acc.items()},
            "kernel_ms": {k: round(v, 4) for k, v in kernel_ms.items()},
            "kernel_gbs": {k: round(v, 1) for k, v in bw.items()},
            "mesh": {"points": P, "vertices": V, "triangles": T},
            "sparsity": {"touched_chunks": chunks, "chunks_total": dims[1] * dims[2] * (dims[0] // 32),
                         "nonzero_rows": nzrows, "rows_total": dims[1] * dims[2],
                         "nonzero_planes": nzplanes, "planes_total": dims[2]},
            "algorithmic_bytes": ab,
            "clocks": clk.summary(),
            "wall_s": wall,
        }
        if cmp is not None:
            line["fft_comparator"] = cmp
        if split:
            line["e2e_split"] = split
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    lib.vc_device_free(h, dbuf)
    lib.vc_host_free(h, hbuf)
    for c in ctxs:
        c.close()
    if world > 1:
        torch.distributed.destroy_process_group()


C5_DIMS = (1024, 1024, 1024)
C5_FRAMES = 4
C5_METRIC = "reconstructed frames/sec at 1024^3 grid, 4x512x424 RGB-D views"


def run_c5(args):
    """Config C5 on N>1 GPUs (torchrun): one 1024^3 frame per step through the
    z-slab decomposition over NCCL (vc_reconstruct_frame_dist), strong
    scaling, time = max over ranks.  (N=1 runs whole frames in run_gpu.)"""
    rank, world, local = dist_env()
    import torch
    from paper_1712_03084_b200 import _lib as L
    from paper_1712_03084_b200 import volcap as vc
    from paper_1712_03084_b200.frame_parallel import max_over_ranks
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    lib = L.lib()
    if world < 2:
        raise SystemExit("run_c5 is the N>1 z-slab path")
    import torch.distributed as dist
    from paper_1712_03084_b200.slab import SlabReconstructor, nccl_unique_id
    dist.init_process_group("nccl", device_id=dev)
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    sr = SlabReconstructor.nccl(world, rank, local, obj[0])
    ctx = sr.contexts[0]
    h = ctx.handle
    stream = torch.cuda.ExternalStream(ctx.stream(), device=dev)
    rig = vc.make_circle_rig(K_VIEWS, 0, 2500, W, H, F)
    sensors = rig.c_array(K_VIEWS)
    n_pix = W * H
    per_view = n_pix * 6
    frame_bytes = K_VIEWS * per_view
    dbuf, hbuf = C.c_void_p(), C.c_void_p()
    L.check(lib.vc_device_alloc(h, C.c_size_t(C5_FRAMES * frame_bytes), C.byref(dbuf)), h)
    L.check(lib.vc_host_alloc(h, C.c_size_t(C5_FRAMES * frame_bytes), C.byref(hbuf)), h)

    def vp(base, f, k):
        o = base + f * frame_bytes + k * per_view
        return o, o + 2 * n_pix, o + 3 * n_pix

    for f in range(C5_FRAMES):
        body = vc.kick_body(STREAM, f * STREAM // C5_FRAMES)
        for k in range(K_VIEWS):
            d, m, c = vp(dbuf.value, f, k)
            L.check(lib.vc_synth_render(h, C.byref(sensors[k]), C.byref(body), C.c_double(0.0), C.c_uint64(1),
                                        C.c_double(1.0), k, f, C.c_void_p(d), C.c_void_p(m), C.c_void_p(c),
                                        L.VC_MEM_DEVICE), h)
    L.check(lib.vc_memcpy(h, hbuf, dbuf, C.c_size_t(C5_FRAMES * frame_bytes), L.VC_MEM_HOST, L.VC_MEM_DEVICE), h)

    def views_for(base, f, kind):
        arr = (L.View * K_VIEWS)()
        for k in range(K_VIEWS):
            d, m, c = vp(base, f, k)
            arr[k] = L.View(d, m, c, 0, 0, 0, kind)
        return arr

    dev_views = [views_for(dbuf.value, f, L.VC_MEM_DEVICE) for f in range(C5_FRAMES)]
    host_views = [views_for(hbuf.value, f, L.VC_MEM_HOST) for f in range(C5_FRAMES)]
    cfg = vc.ReconConfig(dims=C5_DIMS).to_c()
    out = L.TexturedMesh()
    info = L.DistInfo()
    d2h = [0]

    def frame(i, views):
        L.check(lib.vc_reconstruct_frame_dist(sr._h, sensors, views[i % C5_FRAMES], K_VIEWS, C.byref(cfg),
                                              C.byref(out), C.byref(info), None), h)
        d2h[0] += out.vertex_count * (12 + 12 + 24 + 3 + 1 + K_VIEWS * 13) + out.triangle_count * 12

    def timed(views, steps):
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        d2h[0] = 0
        ev0.record(stream)
        for i in range(steps):
            frame(i, views)
        ev1.record(stream)
        torch.cuda.synchronize()
        return max_over_ranks(ev0.elapsed_time(ev1), device="cuda"), d2h[0] / steps

    lib.vc_ctx_set_output(h, L.VC_MEM_DEVICE)
    for i in range(args.warmup):
        frame(i, dev_views)
    with Clocks(local) as clk:
        ms, _ = timed(dev_views, args.steps)
    value = args.steps / (ms / 1000.0)
    tm = L.StageTimings()
    L.check(lib.vc_reconstruct_frame_dist(sr._h, sensors, dev_views[0], K_VIEWS, C.byref(cfg), C.byref(out),
                                          C.byref(info), C.byref(tm)), h)
    stages = {nm: getattr(tm, nm) for nm, _ in L.StageTimings._fields_}
    kernel_ms = None
    # slab integrate: this rank's share of the whole-grid FFT chain bytes over fft_ms (incl. the exchanges)
    nx, ny, nz = C5_DIMS
    Nh = nz * ny * (nx // 2 + 1)
    fft_bytes = (16 * nx * ny * nz + 3 * 8 * Nh + 2 * 3 * 8 * Nh + 4 * 8 * Nh + 2 * 8 * Nh + 8 * Nh
                 + 4 * nx * ny * nz) / world
    pk = peaks()
    hbm = float(pk.get("hbm_gbs", 6650.0))
    ach = fft_bytes / (tm.fft_ms * 1e-3) / 1e9
    roofline = {"bound": "hbm", "kernel": "slab integrate (x/y, all-to-all, z, all-to-all, y/x)",
                "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm, "traffic": None,
                "algorithmic_bytes": fft_bytes, "avg_launch_ms": tm.fft_ms}
    launches = None
    mesh = {"vertices_total": info.vertex_total, "triangles_total": info.triangle_total}
    lib.vc_ctx_set_output(h, L.VC_MEM_HOST)
    for i in range(min(args.warmup, 2)):
        frame(i, host_views)
    e2e_ms, d2h_per = timed(host_views, args.steps)
    if rank == 0:
        line = {"metric": C5_METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": "C5: 4 views 512x424 of the kick stream, 1024^3 grid, weighted splat",
                           "grid": list(C5_DIMS), "parallelism": f"z-slab x{world}",
                           "l2": "working set ~40 GB >> 126 MB L2"},
                "e2e": {"value": args.steps / (e2e_ms / 1000.0), "unit": "frames/s",
                        "h2d_bytes_per_step": frame_bytes, "d2h_bytes_per_step": int(d2h_per)},
                "gpu_launches": launches, "roofline": roofline,
                "stages_ms": {k: round(v, 3) for k, v in stages.items()},
                "kernel_ms": {k: round(v, 3) for k, v in kernel_ms.items()} if kernel_ms else None,
                "mesh": mesh, "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    lib.vc_device_free(h, dbuf)
    lib.vc_host_free(h, hbuf)
    sr.close()
    torch.distributed.destroy_process_group()


def free_port():
    import socket
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    p = so.getsockname()[1]
    so.close()
    return p


def launch_ranks(n):
    """`--gpus N` (N > 1) outside torchrun: re-run this script as N ranks, one
    process per GPU, under torch.distributed.run on 127.0.0.1 (the driver's own
    launch line); rank 0 prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def run_plan(args):
    """--plan: the frame-to-rank assignment this launch would run (no GPU): each
    rank computes its frames, rank 0 gathers them (gloo) and prints one JSON line."""
    from paper_1712_03084_b200.frame_parallel import rank_frames
    rank, world, _ = dist_env()
    wl = WORKLOADS[args.workload]
    if wl.key == "c4":  # as run_gpu: the rank's whole shard
        args.steps = len(range(rank, wl.frames, world))
    mine = [wl.kick_frame(j) for j in rank_frames(rank, world, args.steps, wl.frames)]
    allf = [mine]
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        allf = [None] * world
        dist.all_gather_object(allf, mine)
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"plan": True, "n_gpus": world, "steps": args.steps, "workload": wl.key,
                          "frames_by_rank": allf}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4000)  # ~1 s timed: several clock samples
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fft-comparator", action="store_true")
    ap.add_argument("--workload", default="c2", choices=["c2", "c3", "c4", "c5"],
                    help="c2: the BASELINE metric (256^3 stream, frame-parallel); c3: 512^3, 6 views + HD colour; "
                         "c4: the 4096-frame stream, each rank's shard once (--steps ignored); "
                         "c5: 1024^3 frames (z-slabs on N>1)")
    ap.add_argument("--streams", type=int, default=None,
                    help="concurrent frames per GPU (one context + host thread each; default 4, c5: 2)")
    ap.add_argument("--plan", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl != "reference":
        args.warmup = 3
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(launch_ranks(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} does not match WORLD_SIZE={world}")
    if args.plan:
        run_plan(args)
    elif args.impl == "reference":
        if args.workload == "c5":
            raise SystemExit("--impl reference runs c2/c3 (the CPU path at 1024^3 takes minutes per frame)")
        run_reference(args)
    elif args.workload == "c5" and world > 1:
        run_c5(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
