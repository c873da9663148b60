# SPDX-License-Identifier: Apache-2.0
"""B200-native FT-reconstruction (FTR) frame path of arXiv 1712.03084.

C-ABI: include/vc/vc.h, implemented by libvc_b200.so (CUDA sm_100a + C++
runtime, built in-tree by __graft_entry__.build()).  `volcap` mirrors the
reference's proj/core reconstruction interface over that ABI.
"""
from . import volcap  # noqa: F401
from ._lib import LIB_PATH, VcEmptyScene, VcError, VcInvalidArgument  # noqa: F401
