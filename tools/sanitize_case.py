"""Small end-to-end cases for compute-sanitizer (one process, every kernel family, n <= 14)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads  # noqa: E402
import paper_2504_17881_b200 as P  # noqa: E402
from paper_2504_17881_b200 import ps  # noqa: E402

for dtype in ("c128", "c64"):
    for n, kind, tb, mode in ((12, "R10", 8, 2), (13, "LOW", 11, 2), (12, "S8", 7, 0), (11, "R4", 6, 1), (12, "R10", 8, 3),
                              (5, "R10", None, 2), (2, "R10", None, 2)):
        codes, ang = workloads.random_layer(n, 60, seed=n, kind=kind)
        x, z = P.pauli_encode_codes(codes)
        with P.State(n, dtype) as st:
            for fusion in (0, 1, 2):
                st.set_option(ps.OPT_FUSION, fusion)
                if tb:
                    st.set_option(ps.OPT_TILE_BITS, tb)
                st.set_option(ps.OPT_TILE_TMA, mode)
                st.init_random(1)
                st.apply_rotations(x, z, ang)
            st.norm()
            st.expectation(x[:10], z[:10], np.ones(10))
            st.get_amplitudes(0, 1 << n)
print("sanitize case ok")
