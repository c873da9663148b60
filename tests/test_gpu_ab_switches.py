# SPDX-License-Identifier: Apache-2.0
"""The measured alternatives kept behind environment switches produce the same
results as the default path (the switches are read once per process, so each
variant runs in a child process):

* VC_MC_SPLIT=1 — marching cubes with the split count / look-back scan / emit
  kernels instead of the fused scan + emit (k_mc.cu): same mesh, bit for bit,
  on the same fields (a smooth one, and a noise field past the initial
  capacity, which regrows and reruns).
* VC_ZP=0 / VC_FYP=0 — the staged z_kernel<1024> / fy_kernel<1024> instead of
  the pipelined zp_kernel / fyp_kernel (k_fft.cu): the same per-tile
  arithmetic in the same order (two kernels, so the compiler's FMA
  contraction may differ: rel-L2 < 1e-6)."""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import sys
import numpy as np
from paper_1712_03084_b200 import volcap as vc
ctx = vc.default_context(0)
# marching cubes on fixed fields (the splat's float atomics make a frame's field differ between processes)
n = 96
z, y, x = np.meshgrid(*[np.arange(n)] * 3, indexing="ij")
rng = np.random.default_rng(3)
smooth = (30.0 - np.sqrt((x - 47.3) ** 2 + (y - 45.1) ** 2 + (z - 48.7) ** 2)).astype(np.float32)
smooth += rng.normal(scale=0.3, size=smooth.shape).astype(np.float32)
noise = rng.uniform(-1, 1, (40, 40, 40)).astype(np.float32)   # past the initial capacity: regrow + rerun
g1 = vc.fit_grid((0, 0, 0), (100, 100, 100), (n, n, n))
g2 = vc.fit_grid((0, 0, 0), (40, 40, 40), (40, 40, 40))
m1 = vc.marching_cubes(smooth, g1, 0.0, ctx=ctx)
m2 = vc.marching_cubes(noise, g2, 0.0, ctx=ctx)
f = rng.normal(size=(1024, 4, 8, 3)).astype(np.float32)   # (z, y, x, component): a 1024-plane Z pass
a = vc.integrate_fft(f, ctx=ctx)
f2 = rng.normal(size=(4, 1024, 8, 3)).astype(np.float32)  # a 1024-point F-y pass
a2 = vc.integrate_fft(f2, ctx=ctx)
np.savez(sys.argv[1], v1=m1.vertices, t1=m1.triangles, n1=m1.normals, v2=m2.vertices, t2=m2.triangles, a=a, a2=a2)
print("ok")
'''


def _run(tmp_path, name, env_extra):
    out = tmp_path / f"{name}.npz"
    env = dict(os.environ, PYTHONPATH=ROOT, **env_extra)
    r = subprocess.run([sys.executable, "-c", CHILD, str(out)], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-3000:]
    return np.load(out)


@pytest.mark.gpu
def test_ab_switches_match_default(tmp_path):
    base = _run(tmp_path, "default", {})
    split = _run(tmp_path, "mc_split", {"VC_MC_SPLIT": "1"})
    staged = _run(tmp_path, "staged", {"VC_ZP": "0", "VC_FYP": "0"})
    assert base["v1"].shape[0] > 10000 and base["v2"].shape[0] > 40 ** 3 // 16
    for k in ("v1", "t1", "n1", "v2", "t2"):
        assert np.array_equal(base[k], split[k]), k
    for k in ("a", "a2"):
        a, b = base[k].astype(np.float64), staged[k].astype(np.float64)
        assert np.linalg.norm(a - b) / np.linalg.norm(a) < 1e-6, k
