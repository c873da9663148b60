# SPDX-License-Identifier: Apache-2.0
"""CPU-side checks of the drop-in boundary: libvc_b200.so loads, exports every
function include/vc/vc.h declares, the ctypes mirrors match the header's
struct sizes, and the host-only entry points (fit_grid, synthetic rig/body,
status strings) behave like the reference.  No compute calls (no GPU here)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from paper_1712_03084_b200 import _lib as L
from paper_1712_03084_b200 import volcap as vc


def test_library_exports_every_header_symbol():
    lib = L.lib()
    names = L.header_functions()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert lib.vc_abi_version() == 1


def test_exports_are_exactly_the_header():
    out = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True, text=True, check=True)
    exported = {m.group(1) for m in re.finditer(r" T (vc_\w+)$", out.stdout, re.M)}
    assert exported == set(L.header_functions())


def test_struct_layouts_match_header():
    # sizes of the POD structs as a C compiler lays them out
    src = '#include "vc/vc.h"\n#include <stdio.h>\nint main(){printf("%zu %zu %zu %zu %zu %zu %zu %zu\\n",' \
          'sizeof(vc_sensor),sizeof(vc_view),sizeof(vc_recon_config),sizeof(vc_grid_spec),' \
          'sizeof(vc_stage_timings),sizeof(vc_textured_mesh),sizeof(vc_body),sizeof(vc_intrinsics));return 0;}'
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "s.c")
        open(c, "w").write(src)
        subprocess.run(["gcc", "-I", os.path.join(L.REPO_DIR, "include"), c, "-o", os.path.join(d, "s")], check=True)
        sizes = list(map(int, subprocess.run([os.path.join(d, "s")], capture_output=True, text=True).stdout.split()))
    assert sizes == [C.sizeof(t) for t in (L.Sensor, L.View, L.ReconConfig, L.GridSpec, L.StageTimings,
                                            L.TexturedMesh, L.Body, L.Intrinsics)]


def test_no_device_is_reported_not_faked():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    assert L.lib().vc_ctx_create(0, C.byref(h)) == L.VC_ERR_NO_DEVICE
    with pytest.raises(L.VcError):
        vc.Context(0)


def test_status_strings():
    lib = L.lib()
    assert lib.vc_status_string(2).decode() == "empty foreground in all views"
    assert lib.vc_status_string(0).decode() == "ok"


def test_fit_grid_matches_oracle(O):
    """reconstruct.cpp:16-35 host entry point vs the oracle, bit-exact."""
    rng = np.random.default_rng(4)
    for dims in [(64, 128, 64), (256, 256, 256), (128, 256, 128), (16, 16, 16)]:
        lo = rng.uniform(-900, 0, 3); hi = lo + rng.uniform(100, 1800, 3)
        g = vc.fit_grid(lo, hi, dims, 4)
        o = O.fit_grid(lo, hi, dims, 4)
        assert g.edge_mm == o.edge and list(g.origin) == list(o.origin[:])
    with pytest.raises(ValueError):
        vc.fit_grid([0, 0, 0], [1, 1, 1], (16, 16, 16), 8)


def test_synthetic_rig_and_bodies_match_oracle(O):
    rig = vc.make_circle_rig(4, 2, 2500, 512, 424, 365)
    orc = O.make_circle_rig(4, 2, 2500, 1000, 512, 424, 365)
    for i in range(6):
        a, b = rig.sensors[i].to_c(), orc[i]
        assert bytes(a) == bytes(b)
    assert bytes(vc.xpose_body()) == bytes(O.xpose_body())
    for f in (0, 77, 299):
        assert bytes(vc.kick_body(300, f)) == bytes(O.kick_body(300, f))


def test_reconstruct_rejects_frame_count():
    rig = vc.make_circle_rig(4, 0, 2500, 64, 56, 60)
    with pytest.raises(ValueError):
        vc.reconstruct_frame([], rig, vc.ReconConfig(r=5))


def test_kernels_are_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", L.LIB_PATH], capture_output=True, text=True)
    archs = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert archs == {"100a"}, archs
