# SPDX-License-Identifier: Apache-2.0
"""The opt-in TMA-fed Z kernel (VC_ZK=4, k_fft.cu z4_kernel) against the oracle.

The switch is read once per process, so the checks run in a child process:
dense random fields (every plane live: one 32-plane box chain per column) at
64/128/256 planes, and a 256^3 kick frame (sparse live-plane runs: boxes of
32/16/8/4/2/1 planes, dead planes never read) against the staged kernel's
field and the oracle's."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import numpy as np
from oracle import oracle as O
from paper_1712_03084_b200 import volcap as vc
ctx = vc.default_context(0)
rel = lambda a, b: float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))
for shape in [(64, 32, 32), (128, 16, 64), (256, 8, 32), (256, 32, 64)]:
    rng = np.random.default_rng(sum(shape))
    f = rng.normal(size=shape + (3,)).astype(np.float32)
    r = rel(vc.integrate_fft(f, ctx=ctx), O.integrate_fft(f.astype(np.float64)))
    assert r < 1e-5, (shape, r)
rig = vc.make_circle_rig(4, 0, 2500, 512, 424, 365)
body = vc.kick_body(300, 150)
frames = [vc.render_frame(rig, body, k, 150, ctx=ctx) for k in range(4)]
rec = vc.reconstruct_frame(frames, rig, vc.ReconConfig(dims=(256, 256, 256)), ctx=ctx, want_volume=True)
np.save(__import__("sys").argv[1], rec.volume.values)
print("ok")
'''


@pytest.mark.gpu
def test_tma_z_kernel_matches_oracle_and_staged(tmp_path):
    import numpy as np

    from paper_1712_03084_b200 import volcap as vc

    out = tmp_path / "a_zk4.npy"
    env = dict(os.environ, VC_ZK="4", PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", CHILD, str(out)], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-3000:]
    a4 = np.load(out)
    # the same frame through the default (staged) Z kernel in this process
    ctx = vc.default_context(0)
    rig = vc.make_circle_rig(4, 0, 2500, 512, 424, 365)
    body = vc.kick_body(300, 150)
    frames = [vc.render_frame(rig, body, k, 150, ctx=ctx) for k in range(4)]
    a1 = vc.reconstruct_frame(frames, rig, vc.ReconConfig(dims=(256, 256, 256)), ctx=ctx, want_volume=True).volume.values
    rel = np.linalg.norm(a4.astype(np.float64) - a1) / np.linalg.norm(a1.astype(np.float64))
    assert rel < 1e-5, rel  # two fp32 FFT orderings of the same field (and the splat's atomics)
