"""Seeded synthetic input generators shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic: it only draws Pauli *words* (letter codes
0=I, 1=X, 2=Y, 3=Z per qubit, leftmost letter = factor 1 = qubit 0) and real angles /
coefficients, with the shapes and structure of the paper's workloads.  Each side encodes the
words itself (the product through ``ps_pauli_encode_codes``, the oracle directly from the
factors).  The recipes are stated in DESIGN.md "Input recipe"; base seed 250417881.

Generators
  random_layer(n, count, seed, kind)      R4 / R10 / D / S8 / LOW random Pauli layers
  jw_hamiltonian(n, n_terms, lam, seed)   Jordan-Wigner-shaped molecular Hamiltonian (Table 3)
  trotter1_angles(coeffs, delta)          first-order Trotter step angles phi_l = delta*h_l
  qaoa_layers(n, p, seed)                 QAOA MaxCut on a random 3-regular graph
  gate_circuit(n, depth, seed)            random brickwork of standard gates (converted by the product)
"""
from __future__ import annotations

import numpy as np

BASE_SEED = 250417881
I, X, Y, Z = 0, 1, 2, 3


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([BASE_SEED, int(seed)])))


def random_layer(n: int, count: int, seed: int = 0, kind: str = "R10", low_k: int = 10,
                 run: int = 8):
    """A layer of `count` random Pauli rotations on n qubits; returns (codes[count, n] uint8, angles).

    kinds:
      R4   each letter i.i.d. uniform over {I, X, Y, Z} (mean weight 3n/4)
      R10  weight w ~ U{1..min(10, n)}, positions a uniform w-subset, letters U{X, Y, Z}
           (config 1 / config 2 of BASELINE.json)
      D    diagonal only: letters i.i.d. over {I, Z}
      S8   runs of `run` rotations sharing their non-diagonal positions (same p1 mask); in a run
           each non-diagonal letter is X or Y at random and every other letter I or Z at random
      LOW  as R10 but all non-diagonal letters inside the low `low_k` qubits; Z letters anywhere
    angles: phi ~ U[-pi, pi)
    """
    kind_id = {"R4": 1, "R10": 2, "D": 3, "S8": 4, "LOW": 5}.get(kind, 0)
    rng = _rng(((kind_id * 1000 + n) * 1_000_003 + count) * 1009 + int(seed))
    codes = np.zeros((count, n), dtype=np.uint8)
    if kind == "R4":
        codes[:] = rng.integers(0, 4, size=(count, n), dtype=np.uint8)
    elif kind in ("R10", "LOW"):
        wmax = min(10, n)
        for l in range(count):
            w = int(rng.integers(1, wmax + 1))
            pos = rng.choice(n, size=w, replace=False)
            codes[l, pos] = rng.integers(1, 4, size=w, dtype=np.uint8)
            if kind == "LOW":
                hi = pos[pos >= low_k]
                # keep the weight: non-diagonal letters above low_k become Z
                codes[l, hi] = np.where(codes[l, hi] != 0, Z, 0)
    elif kind == "D":
        codes[:] = rng.integers(0, 2, size=(count, n), dtype=np.uint8) * Z
    elif kind == "S8":
        l = 0
        while l < count:
            w = int(rng.integers(1, min(10, n) + 1))
            nd = rng.choice(n, size=w, replace=False)
            for _ in range(min(run, count - l)):
                row = rng.integers(0, 2, size=n, dtype=np.uint8) * Z
                row[nd] = rng.integers(1, 3, size=w, dtype=np.uint8)  # X or Y
                codes[l] = row
                l += 1
    else:
        raise ValueError(kind)
    angles = rng.uniform(-np.pi, np.pi, size=count)
    return codes, angles


def _jw_string(n: int, p: int, q: int, lp: int, lq: int) -> np.ndarray:
    """lp on p, lq on q, Z on every qubit strictly between (Jordan-Wigner string)."""
    w = np.zeros(n, dtype=np.uint8)
    a, b = min(p, q), max(p, q)
    w[a + 1:b] = Z
    w[p] = lp
    w[q] = lq
    return w


_EVEN_Y_QUADS = [(X, X, X, X), (X, X, Y, Y), (X, Y, X, Y), (X, Y, Y, X),
                 (Y, X, X, Y), (Y, X, Y, X), (Y, Y, X, X), (Y, Y, Y, Y)]


def jw_hamiltonian(n: int, n_terms: int, lam: float, seed: int = 0, n_local: int | None = None):
    """A Jordan-Wigner-shaped molecular Hamiltonian on n spin-orbital qubits (synthetic; the
    paper's Hamiltonians are not available offline).  Returns (codes[L, n], coeffs[L]).

    Families (spin orbitals interleaved alpha/beta, qubit p):  Z_p;  Z_p Z_q;  same-spin hopping
    X_p Z..Z X_q and Y_p Z..Z Y_q;  hopping times an extra Z_r;  two-body quads on a<b<c<d with
    the 8 even-#Y X/Y patterns and JW Z-strings on (a,b) and (c,d).  One-body families are kept
    whole; hopping-with-Z and quads are subsampled to reach n_terms.  Coefficients: random sign,
    log-uniform magnitude in [1e-4, 1], rescaled so sum|h| = lam (Table 3 lambda column).
    Order: x-major -- grouped by the non-diagonal positions above n_local, then all non-diagonal
    positions, then the rest (reading R14 of P:674 "ordered lexicographically").
    """
    rng = _rng(7_000_000 + n * 1000 + seed)
    rows = []
    for p in range(n):
        w = np.zeros(n, np.uint8); w[p] = Z; rows.append(w)
    for p in range(n):
        for q in range(p + 1, n):
            w = np.zeros(n, np.uint8); w[p] = Z; w[q] = Z; rows.append(w)
    for p in range(n):
        for q in range(p + 2, n, 2):  # same spin
            rows.append(_jw_string(n, p, q, X, X))
            rows.append(_jw_string(n, p, q, Y, Y))
    base = len(rows)
    if base > n_terms:
        raise ValueError("n_terms below the one-body families")
    remaining = n_terms - base
    same_spin_pairs = sum(1 for p in range(n) for q in range(p + 2, n, 2))
    n_hopz = min(remaining // 4, same_spin_pairs * (n - 2) * 2)  # all (p, q, r, letter) choices
    n_quad = remaining - n_hopz
    if n_quad > 8 * (n * (n - 1) * (n - 2) * (n - 3) // 24):
        raise ValueError("n_terms exceeds the JW-shaped families")
    # hopping x Z_r
    hz = set()
    while len(hz) < n_hopz:
        p = int(rng.integers(0, n - 2)); q = int(rng.integers(p + 2, n))
        if (q - p) % 2:
            continue
        r = int(rng.integers(0, n))
        if r in (p, q):
            continue
        lp = int(rng.integers(0, 2))
        hz.add((p, q, r, lp))
    for p, q, r, lp in sorted(hz):
        letter = X if lp == 0 else Y
        w = _jw_string(n, p, q, letter, letter)
        w[r] = I if w[r] == Z else Z
        rows.append(w)
    quads = set()
    while len(quads) < n_quad:
        a, b, c, d = sorted(int(v) for v in rng.choice(n, size=4, replace=False))
        pat = int(rng.integers(0, 8))
        quads.add((a, b, c, d, pat))
    for a, b, c, d, pat in sorted(quads):
        la, lb, lc, ld = _EVEN_Y_QUADS[pat]
        w = np.zeros(n, np.uint8)
        w[a + 1:b] = Z
        w[c + 1:d] = Z
        w[a], w[b], w[c], w[d] = la, lb, lc, ld
        rows.append(w)
    codes = np.stack(rows).astype(np.uint8)
    mag = 10.0 ** rng.uniform(-4, 0, size=len(codes))
    sign = np.where(rng.integers(0, 2, size=len(codes)) == 0, -1.0, 1.0)
    coeffs = sign * mag
    coeffs *= lam / np.abs(coeffs).sum()
    codes, coeffs = order_x_major(codes, coeffs, n_local if n_local is not None else n)
    return codes, coeffs


def _pack_bits(bits: np.ndarray) -> np.ndarray:
    """rows of 0/1 (width <= 64) -> uint64 with column q at bit q"""
    w = bits.shape[1]
    out = np.zeros(bits.shape[0], dtype=np.uint64)
    for q in range(w):
        out |= bits[:, q].astype(np.uint64) << np.uint64(q)
    return out


def order_x_major(codes: np.ndarray, coeffs: np.ndarray, n_local: int):
    """Stable order by (non-diagonal positions >= n_local, all non-diagonal positions, letters)."""
    nd = ((codes == X) | (codes == Y)).astype(np.uint8)
    hi = _pack_bits(nd[:, n_local:]) if n_local < codes.shape[1] else np.zeros(len(codes), np.uint64)
    allnd = _pack_bits(nd)
    yz = _pack_bits(((codes == Y) | (codes == Z)).astype(np.uint8))
    order = np.lexsort((yz, allnd, hi))
    return codes[order], coeffs[order]


def jw_embedded(n_total: int, positions, n_terms: int, lam: float, seed: int = 0, extra_z: float = 0.3,
                n_local: int | None = None):
    """A JW-shaped Hamiltonian on len(positions) qubits placed at `positions` of an n_total-qubit
    register, every term additionally carrying random Z letters on the other qubits (probability
    extra_z each).  The X/Y support stays inside `positions`, so the X-span has rank <= len(positions)
    and the coset oracle can check any n_total (SURVEY T5 parity variant)."""
    positions = list(positions)
    small, coeffs = jw_hamiltonian(len(positions), n_terms, lam, seed=seed, n_local=len(positions))
    rng = _rng(5_000_000 + n_total * 100 + seed)
    codes = np.zeros((len(small), n_total), np.uint8)
    others = np.array([q for q in range(n_total) if q not in set(positions)], dtype=np.int64)
    codes[:, others] = (rng.random((len(small), len(others))) < extra_z).astype(np.uint8) * Z
    codes[:, positions] = small
    return order_x_major(codes, coeffs, n_local if n_local is not None else n_total)


def trotter1_angles(coeffs: np.ndarray, delta: float) -> np.ndarray:
    """First-order Trotter step exp(i delta H) ~ prod_l exp(i delta h_l P_l): phi_l = delta*h_l."""
    return delta * np.asarray(coeffs, dtype=np.float64)


def random_regular3(n: int, seed: int = 0):
    """Edges of a random 3-regular simple graph on n vertices (n even), by the pairing model."""
    rng = _rng(9_000_000 + n * 10 + seed)
    while True:
        stubs = np.repeat(np.arange(n), 3)
        rng.shuffle(stubs)
        e = stubs.reshape(-1, 2)
        if np.any(e[:, 0] == e[:, 1]):
            continue
        es = {tuple(sorted(map(int, r))) for r in e}
        if len(es) == len(e):
            return sorted(es)


def qaoa_layers(n: int, p: int, seed: int = 0):
    """QAOA MaxCut: per layer a Z_uZ_v rotation per edge (gamma) then X_v per vertex (beta)."""
    rng = _rng(8_000_000 + n * 10 + seed)
    edges = random_regular3(n, seed)
    rows, angles = [], []
    for _ in range(p):
        gamma, beta = rng.uniform(-np.pi, np.pi, size=2)
        for u, v in edges:
            w = np.zeros(n, np.uint8); w[u] = Z; w[v] = Z
            rows.append(w); angles.append(gamma)
        for v in range(n):
            w = np.zeros(n, np.uint8); w[v] = X
            rows.append(w); angles.append(beta)
    return np.stack(rows), np.array(angles)


GATES_1Q = ["H", "S", "T", "X", "Z", "RX", "RY", "RZ"]
GATES_2Q = ["CNOT", "CZ", "SWAP", "CPHASE", "RZZ"]


def gate_circuit(n: int, depth: int, seed: int = 0):
    """Random brickwork: each layer a random 1-qubit gate on every qubit, then 2-qubit gates on
    alternating neighbour pairs.  Returns a list of (name, qubits tuple, params tuple)."""
    rng = _rng(6_000_000 + n * 10 + seed)
    gates = []
    for d in range(depth):
        for q in range(n):
            g = GATES_1Q[int(rng.integers(0, len(GATES_1Q)))]
            params = (float(rng.uniform(-np.pi, np.pi)),) if g.startswith("R") else ()
            gates.append((g, (q,), params))
        for q in range(d % 2, n - 1, 2):
            g = GATES_2Q[int(rng.integers(0, len(GATES_2Q)))]
            a, b = (q, q + 1) if rng.integers(0, 2) == 0 else (q + 1, q)
            params = (float(rng.uniform(-np.pi, np.pi)),) if g in ("CPHASE", "RZZ") else ()
            gates.append((g, (a, b), params))
    return gates


def ucc_layers(n: int, n_occ: int | None = None, seed: int = 0, max_doubles: int | None = None):
    """A unitary-coupled-cluster (UCCSD-shaped) VQE ansatz layer under Jordan-Wigner (BASELINE.json
    config 4, "VQE-style layers").  Spin orbitals interleaved (qubit p: spin p % 2); the n_occ lowest
    orbitals occupied.  Singles p -> a (occupied p, virtual a, same spin): exp(theta (a_a^dag a_p -
    h.c.)) = exp(i theta/2 (X_p Z..Z Y_a - Y_p Z..Z X_a)) as two rotations; doubles (p<q) -> (a<b),
    spin conserving: the 8 Pauli strings with an odd number of Y on {p, q, a, b} and Z strings on
    (p, q) and (a, b), angles +-theta/8 (sign + for three X and one Y, - for one X and three Y).
    Amplitudes theta ~ U[-0.1, 0.1] (seeded).  Returns (codes[L, n], angles[L]) in ansatz order."""
    rng = _rng(4_000_000 + n * 10 + seed)
    n_occ = n // 2 if n_occ is None else n_occ
    occ = list(range(n_occ))
    vir = list(range(n_occ, n))
    rows, angles = [], []
    for p in occ:
        for a in vir:
            if (a - p) % 2:
                continue
            th = float(rng.uniform(-0.1, 0.1))
            for lp, la, sg in ((X, Y, 1.0), (Y, X, -1.0)):
                rows.append(_jw_string(n, p, a, lp, la))
                angles.append(sg * th / 2)
    doubles = []
    for i, p in enumerate(occ):
        for q in occ[i + 1:]:
            for j, a in enumerate(vir):
                for b in vir[j + 1:]:
                    if (p % 2) + (q % 2) == (a % 2) + (b % 2):
                        doubles.append((p, q, a, b))
    if max_doubles is not None and len(doubles) > max_doubles:
        pick = np.sort(rng.choice(len(doubles), max_doubles, replace=False))
        doubles = [doubles[k] for k in pick]
    odd_y = [(X, X, X, Y), (X, X, Y, X), (X, Y, X, X), (Y, X, X, X),
             (X, Y, Y, Y), (Y, X, Y, Y), (Y, Y, X, Y), (Y, Y, Y, X)]
    for p, q, a, b in doubles:
        th = float(rng.uniform(-0.1, 0.1))
        for k, (l0, l1, l2, l3) in enumerate(odd_y):
            w = np.zeros(n, np.uint8)
            w[p + 1:q] = Z
            w[a + 1:b] = Z
            w[p], w[q], w[a], w[b] = l0, l1, l2, l3
            rows.append(w)
            angles.append((1.0 if k < 4 else -1.0) * th / 8)
    return np.stack(rows).astype(np.uint8), np.array(angles)


def hardware_efficient_vqe(n: int, depth: int, seed: int = 0):
    """Hardware-efficient VQE ansatz as a gate list: per layer RY and RZ on every qubit, then a CNOT
    ladder (q, q+1) -- converted to rotations by ps_gate_to_rotations."""
    rng = _rng(3_000_000 + n * 10 + seed)
    gates = []
    for _ in range(depth):
        for q in range(n):
            gates.append(("RY", (q,), (float(rng.uniform(-np.pi, np.pi)),)))
            gates.append(("RZ", (q,), (float(rng.uniform(-np.pi, np.pi)),)))
        for q in range(n - 1):
            gates.append(("CNOT", (q, q + 1), ()))
    return gates


def suffix_groups(n: int, count: int, L: int, m: int, seed: int = 0):
    """The paper's benchmark workload: groups of L consecutive rotations sharing a
    common upper string Q~ on the top m qubits (Eq. (1); at least one X/Y letter, so every
    group needs an exchange on m >= 1 partitioned qubits) with random lower strings (R10 recipe on
    the n - m low qubits), `count` rotations in total.  Returns (codes, angles)."""
    if m < 1:
        raise ValueError("suffix groups need m >= 1 upper qubits")
    rng = _rng(2_000_000 + n * 100 + L * 7 + m + seed)
    codes = np.zeros((count, n), dtype=np.uint8)
    low, _ = random_layer(n - m, count, seed=seed + 17, kind="R10")
    codes[:, :n - m] = low
    for g0 in range(0, count, L):
        while True:
            up = rng.integers(0, 4, size=m, dtype=np.uint8)
            if np.any((up == X) | (up == Y)):
                break
        codes[g0:g0 + L, n - m:] = up
    angles = rng.uniform(-np.pi, np.pi, size=count)
    return codes, angles
