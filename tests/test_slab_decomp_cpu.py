# SPDX-License-Identifier: Apache-2.0
"""The z-slab decomposition of the frame (vc_dist.cpp) as a
numpy model over a real 2-rank gloo process group: the same buffer layouts
(fy_kernel's send layout [s][zl][yl][H], the z pass's [z][kyl][H], iy_kernel's
receive row map), the same all-to-all block exchange and the same global
vertex numbering (own planes + the next rank's first plane) must reproduce
the whole-grid integrate.cpp:19-74 (the oracle) and the global edge-id order
of marching_cubes.cpp:139-142."""
import os
import socket

import numpy as np
import torch
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def signed_freq(n):
    k = np.arange(n)
    return 2.0 * np.pi * np.where(k <= n // 2, k, k - n) / n


def field(nx, ny, nz, seed=11):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((nz, ny, nx, 3))


def slab_integrate(rank, world, F, a2a):
    """vc_dist.cpp phases P1-P3 on rank `rank`; `a2a(send, recv)` exchanges
    equal blocks along axis 0 (block s of send -> rank s)."""
    nz, ny, nx, _ = F.shape
    nzl, kyl, H = nz // world, ny // world, nx // 2 + 1
    zoff, ky0 = rank * nzl, rank * kyl
    f = F[zoff:zoff + nzl]
    wx, wy, wz = signed_freq(nx)[:H], signed_freq(ny), signed_freq(nz)
    # P1: x-R2C, y-C2C; D = wx X + wy Y, Z (fx_kernel / fy_kernel)
    S = np.fft.fft(np.fft.rfft(f, axis=2), axis=1)  # [zl][y][H][3]
    D = wx[None, None, :] * S[..., 0] + wy[None, :, None] * S[..., 1]
    Z = S[..., 2]
    # send layout [s][zl][yl][H]: row ky of plane zl at ((s*nzl + zl)*kyl + yl)*H
    send = np.stack([D, Z])  # [2][zl][y][H]
    send = send.reshape(2, nzl, world, kyl, H).transpose(2, 0, 1, 3, 4).copy()  # [s][2][zl][yl][H]
    recv = np.empty_like(send)
    a2a(send, recv)  # block s' of recv: planes z = s'*nzl + zl of my ky slab
    R = recv.transpose(1, 0, 2, 3, 4).reshape(2, nz, kyl, H)  # [2][z][kyl][H]
    # P2: z pass (z_kernel): FFT_z, -i/|w|^2 (D + wz Z), inverse FFT_z
    FD, FZ = np.fft.fft(R[0], axis=0), np.fft.fft(R[1], axis=0)
    ky = wy[ky0:ky0 + kyl]
    w2 = wx[None, None, :] ** 2 + ky[None, :, None] ** 2 + wz[:, None, None] ** 2
    s = FD + wz[:, None, None] * FZ
    with np.errstate(divide="ignore", invalid="ignore"):
        out = np.where(w2 == 0, 0, -1j * s / w2)
    out = np.fft.ifft(out, axis=0) * nz  # unnormalised inverse
    # backward: block s (kz planes of rank s) -> rank s; receive [s'][zl][kyl][H]
    send2 = out.reshape(world, nzl, kyl, H).copy()
    recv2 = np.empty_like(send2)
    a2a(send2, recv2)
    # iy_kernel row map: ky row -> block ky // kyl, row ky % kyl
    T = recv2.transpose(1, 0, 2, 3).reshape(nzl, ny, H)
    T = np.fft.ifft(T, axis=1) * ny
    A = np.fft.irfft(T, n=nx, axis=2) * nx / (nx * ny * nz)
    return A  # planes [zoff, zoff+nzl)


def cut_edges(A, L, z_lo, z_hi):
    """Cut edges ((z*ny+y)*nx+x)*3+axis of voxels z in [z_lo, z_hi), global ids ascending."""
    nz, ny, nx = A.shape
    b = A >= L
    ids = []
    for z in range(z_lo, z_hi):
        for y in range(ny):
            for x in range(nx):
                for a, (dz, dy, dx) in enumerate(((0, 0, 1), (0, 1, 0), (1, 0, 0))):
                    zz, yy, xx = z + dz, y + dy, x + dx
                    if zz < nz and yy < ny and xx < nx and b[z, y, x] != b[zz, yy, xx]:
                        ids.append(((z * ny + y) * nx + x) * 3 + a)
    return ids


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def a2a(send, recv):
        s = torch.from_numpy(np.ascontiguousarray(send).view(np.float64).copy())
        r = torch.empty_like(s)
        dist.all_to_all_single(r, s)  # equal blocks along dim 0
        recv[...] = r.numpy().view(np.complex128).reshape(recv.shape)

    F = field(16, 32, 16)
    A = slab_integrate(rank, world, F, a2a)
    # global vertex numbering: count own cut edges, all-gather, then number
    # own planes + the next rank's first plane from this rank's offset
    Afull_pieces = [torch.zeros(A.shape, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(Afull_pieces, torch.from_numpy(A.copy()))
    Afull = np.concatenate([p.numpy() for p in Afull_pieces])
    L = float(np.median(Afull))
    nzl = Afull.shape[0] // world
    own = cut_edges(Afull, L, rank * nzl, (rank + 1) * nzl)
    counts = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(counts, torch.tensor([len(own)]))
    voff = int(sum(c.item() for c in counts[:rank]))
    extra = cut_edges(Afull, L, (rank + 1) * nzl, min((rank + 2) * nzl, (rank + 1) * nzl + 1)) \
        if rank + 1 < world else []
    numbered = {e: voff + i for i, e in enumerate(own + extra)}
    out[rank] = (A, numbered, L)
    dist.barrier()
    dist.destroy_process_group()


def test_slab_decomposition_gloo_two_ranks(O):
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    F = field(16, 32, 16)
    ref = O.integrate_fft(F)
    A = np.concatenate([out[r][0] for r in range(world)])
    assert np.abs(A - ref).max() <= 1e-10 * np.abs(ref).max()
    # global edge-id numbering: every rank's ids (own + next rank's first plane) agree with
    # the rank of the edge in the whole-grid enumeration
    L = out[0][2]
    glob = {e: i for i, e in enumerate(cut_edges(A, L, 0, A.shape[0]))}
    for r in range(world):
        for e, i in out[r][1].items():
            assert glob[e] == i
    assert set().union(*[set(out[r][1]) for r in range(world)]) == set(glob)
