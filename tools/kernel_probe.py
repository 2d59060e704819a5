"""Runs one family of libps kernels at 30 qubits fp64 for profiling (ncu -k regex:<kernel>):

  python tools/kernel_probe.py stream   # K1 k_stream: a 20-rotation layer at fusion level 0
  python tools/kernel_probe.py reduce   # K5 k_norm, k_inner, k_expect (x = 0 and x != 0 groups)
  python tools/kernel_probe.py swap     # K3 k_p2p_swap, K8 k_xtile and k_permute on 2 virtual ranks
                                        #   (peer pointers into the other slice of the same GPU)
Prints CUDA-event times and algorithmic GB/s per family (ps_get_stats, PS_OPT_PROFILE=1).
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402
import paper_2504_17881_b200 as P  # noqa: E402
from paper_2504_17881_b200 import ps  # noqa: E402


def report(st, label):
    s = st.stats()
    out = {"label": label}
    for k in ps.KERNEL_NAMES:
        if s["launches"][k] and s["kernel_ms"][k] > 0:
            out[k] = {"launches": s["launches"][k], "ms": round(s["kernel_ms"][k], 3),
                      "algo_GBps": round(s["algo_bytes"][k] / (s["kernel_ms"][k] / 1e3) / 1e9, 1)}
    out["nvlink_bytes"] = s["nvlink_bytes"]
    out["nvlink_fused_bytes"] = s["nvlink_fused_bytes"]
    print(json.dumps(out), flush=True)


def main():
    what = sys.argv[1]
    n = int(os.environ.get("PROBE_QUBITS", "30"))
    if what == "stream":
        codes, ang = workloads.random_layer(n, 20, seed=5, kind="R10")
        x, z = P.pauli_encode_codes(codes)
        with P.State(n, "c128") as st:
            st.set_option(ps.OPT_FUSION, 0)
            st.set_option(ps.OPT_PROFILE, 1)
            st.init_random(1)
            st.apply_rotations(x, z, ang)
            st.synchronize()
            st.reset_stats()
            st.apply_rotations(x, z, ang)
            report(st, "K1 fusion 0, 20 rotations")
    elif what == "reduce":
        hc, hco = workloads.jw_hamiltonian(n, 3000, 27.0, seed=2, n_local=n)
        hx, hz = P.pauli_encode_codes(hc)
        sel = np.r_[0:40, len(hc) - 40:len(hc)]  # diagonal terms and a few x-groups
        with P.State(n, "c128") as st, P.State(n, "c128") as st2:
            st.set_option(ps.OPT_PROFILE, 1)
            st.init_random(1)
            st2.init_random(2)
            for _ in range(2):
                st.reset_stats()
                st.norm()
                st.inner(st2)
                st.expectation(hx[sel], hz[sel], hco[sel])
            report(st, "K5 norm + inner + expectation")
    elif what == "swap":
        codes, ang = workloads.random_layer(n, 200, seed=6, kind="R10")
        x, z = P.pauli_encode_codes(codes)
        for fused in (0, 1):
            with P.State(n, "c128", emulate=2) as st:
                st.set_option(ps.OPT_PROFILE, 1)
                st.set_option(ps.OPT_FUSED_EXCHANGE, fused)
                st.init_random(1)
                st.apply_rotations(x, z, ang)
                st.synchronize()
                st.reset_stats()
                st.apply_rotations(x, z, ang)
                st.get_amplitudes(0, 4)  # restore: exchanges + local transpositions (k_permute)
                report(st, f"2 virtual ranks, fused={fused}")
    else:
        raise SystemExit("usage: kernel_probe.py stream|reduce|swap")


if __name__ == "__main__":
    main()
