"""NEXT-3: the Fig. 4 analog -- |Z_0(delta)| = |<b| e^{i delta H~(delta)} |b>|
for one partially randomized second-order step of a JW-shaped Hamiltonian (synthetic; R18),
guiding state a Hartree-Fock-like basis state |b> (the n/2 lowest spin orbitals occupied), on one GPU.

  python tools/z0_curve.py --qubits 30 --terms 60000 --ldet 2000 [--deltas 0.01,0.02,...] [--out f.json]

The curve is checked, where the oracle reaches, against the coset oracle: with --embedded the X
support of every term is confined to 16 qubits (workloads.jw_embedded), so the coset of |b> under
the X masks has 2^16 members and the oracle computes Z_0 of the same sampled circuit exactly
(SURVEY T5).  Without it (the full JW shape), the curve is the Fig. 4 analog itself: as the paper
argues, a wrong implementation would give |Z_0| ~ 2^(-n/2), not amplitudes of order 1.
Var_b(H) (the x-grouped terms on the host) is reported for context: 1 - delta^2 Var_b(H) is the
small-delta expansion of exact evolution under H, which the sampled circuit (one qDRIFT sample of
the randomized part per stage at small delta) does not follow.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402
import paper_2504_17881_b200 as P  # noqa: E402
from paper_2504_17881_b200 import formulas, rpe  # noqa: E402


def basis_variance(H, b: int) -> float:
    """Var_b(H) = sum over x != 0 of |sum_{l: x_l = x} h_l w_l(b)|^2, w_l(b) = i^y (-1)^popc(z_l & b)
    (P|b> = w |b xor x>)."""
    groups: dict = {}
    for x, z, h in zip(H.x.tolist(), H.z.tolist(), H.h.tolist()):
        if x == 0:
            continue
        y = bin(x & z).count("1") & 3
        w = (1j ** y) * (-1) ** (bin(z & b).count("1") & 1)
        groups[x] = groups.get(x, 0) + h * w
    return float(sum(abs(v) ** 2 for v in groups.values()))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--qubits", type=int, default=30)
    ap.add_argument("--terms", type=int, default=60000)
    ap.add_argument("--lam", type=float, default=27.0)
    ap.add_argument("--ldet", type=int, default=2000)
    ap.add_argument("--deltas", default="0.005,0.01,0.02,0.05,0.1,0.2,0.3,0.5")
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--embedded", action="store_true", help="X support on 16 qubits: coset-oracle check")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    n = args.qubits
    if args.embedded:
        pos = list(range(n - 16, n))
        codes, coeffs = workloads.jw_embedded(n, pos, args.terms, args.lam, seed=1)
    else:
        codes, coeffs = workloads.jw_hamiltonian(n, args.terms, args.lam, seed=1)
    x, z = P.pauli_encode_codes(codes)
    H = formulas.from_masks(n, x, z, coeffs)
    HD, HR = formulas.split_deterministic(H, min(args.ldet, len(H)))
    b = sum(1 << q for q in range(n // 2))  # occupied spin orbitals 0 .. n/2-1
    var = basis_variance(H, b)
    rows = []
    with P.State(n, "c128") as st:
        for d in [float(v) for v in args.deltas.split(",")]:
            r = formulas.sample_count(HR.lam, d, 0)
            t0 = time.perf_counter()
            z0 = rpe.z0_basis(n, HD, HR, d, r, args.seed, b, state=st)
            el = time.perf_counter() - t0
            rot = 2 * len(HD) + 2 * r
            row = {"delta": d, "Z0": [z0.real, z0.imag], "abs": abs(z0), "r": r, "rotations": rot,
                   "seconds": el, "exact_evolution_expansion_abs": float(np.sqrt(max(0.0, 1 - d * d * var)))}
            if args.embedded:
                import oracle
                sx, sz, sa = formulas.evolution_stream(HD, HR, d, 1, r, args.seed)
                mem = oracle.coset_members(n, b, np.unique(sx))
                init = (mem == b).astype(np.complex128)
                out = oracle.apply_coset(n, mem, init, oracle.decode_masks(n, sx, sz), sa)
                want = complex(out[np.searchsorted(mem, b)])
                row["oracle"] = [want.real, want.imag]
                row["oracle_err"] = abs(z0 - want)
            rows.append(row)
            print(json.dumps(row), flush=True)
    res = {"qubits": n, "terms": len(H), "lambda": H.lam, "l_det": len(HD), "lambda_R": HR.lam, "b": b,
           "var_b": var, "embedded": args.embedded, "points": rows}
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
