"""Host-side tests of libps (``-m "not gpu"``): the C-ABI library loads and exports every symbol
include/ps.h declares; the encoder, gate converter and planner are checked against the oracle
and the paper.  No compute entry point is called (no GPU here)."""
from __future__ import annotations

import math
import os
import re

import numpy as np
import pytest

import oracle
from oracle import dense
import workloads
import paper_2504_17881_b200 as P
from paper_2504_17881_b200 import ps

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "ps.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ps_[a-z_0-9]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    L = P.lib()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(ps.EXPORTS) == syms


def test_status_strings():
    L = P.lib()
    for code in range(-7, 1):
        assert L.ps_status_string(code)


# ---------------------------------------------------------------- encoder (a1)

def _golden(name):
    for raw in open(os.path.join(GOLDEN, name)):
        line = raw.split("#", 1)[0].strip()
        if line:
            yield line


@pytest.mark.parametrize("line", list(_golden("encode_examples.txt")))
def test_encode_golden(line):
    word, p1, p2 = line.split()
    assert P.pauli_encode(word) == (int(p1), int(p2))


def test_encode_roundtrip_against_oracle_decode():
    """Product encoder -> masks -> the oracle's independent decode -> same letters."""
    rng = np.random.default_rng(0)
    for n in (1, 2, 7, 36, 64):
        codes = rng.integers(0, 4, size=(50, n)).astype(np.uint8)
        x, z = P.pauli_encode_codes(codes)
        assert np.array_equal(oracle.decode_masks(n, x, z), codes)
        for row, xx, zz in zip(codes[:5], x, z):
            word = "".join("IXYZ"[c] for c in row)
            assert P.pauli_encode(word) == (int(xx), int(zz))


@pytest.mark.parametrize("bad", ["", "XA", "X" * 65])
def test_encode_errors(bad):
    with pytest.raises(P.PsError):
        P.pauli_encode(bad)


# ---------------------------------------------------------------- gate converter (a1)

_textbook = dense.textbook_gate


@pytest.mark.parametrize("name,qubits,params", [
    ("H", (1,), ()), ("S", (0,), ()), ("T", (2,), ()), ("X", (1,), ()), ("Y", (0,), ()), ("Z", (2,), ()),
    ("RX", (0,), (0.37,)), ("RY", (2,), (-1.1,)), ("RZ", (1,), (2.5,)),
    ("CNOT", (0, 2), ()), ("CNOT", (2, 0), ()), ("CZ", (1, 2), ()), ("SWAP", (0, 1), ()),
    ("CPHASE", (2, 1), (0.77,)), ("RZZ", (0, 2), (-0.4,)),
])
def test_gate_converter_matches_textbook(name, qubits, params):
    n = 3
    x, z, a = P.gate_to_rotations(name, qubits, params)
    f = oracle.decode_masks(n, x, z)
    u = dense.dense_layer(f, a)  # product of expm(i phi P) in application order
    assert np.max(np.abs(u - _textbook(name, qubits, params, n))) <= 1e-13


def test_gate_converter_errors():
    with pytest.raises(P.PsError):
        P.gate_to_rotations("FOO", (0,))
    with pytest.raises(P.PsError):
        P.gate_to_rotations("CNOT", (1, 1))
    with pytest.raises(P.PsError):
        P.gate_to_rotations("RX", (0,))  # missing angle


# ---------------------------------------------------------------- planner host model (a2, a5)

def _apply_phys(a: np.ndarray, r: dict):
    """Test-side model of one physical-coordinate rotation:
    a'_i = c a_i + i s w(i^x) a_(i^x),  w(i) = i^y * sign * (-1)^popc(z & i)."""
    n = len(a)
    idx = np.arange(n, dtype=np.uint64)
    x, z = np.uint64(r["x"]), np.uint64(r["z"])
    par = np.array([bin(int(v)).count("1") & 1 for v in (idx ^ x) & z])
    w = (1j ** r["y"]) * r["sign"] * np.where(par == 1, -1.0, 1.0)
    c, s = math.cos(r["angle"]), math.sin(r["angle"])
    j = (idx ^ x).astype(np.int64)
    return c * a + 1j * s * w * a[j]


def _run_model(n, world, x, z, ang, fusion=2, tile_bits=3, layout=1):
    m = world.bit_length() - 1
    nl = n - m
    plans = [P.plan_describe(n, x, z, ang, world=world, rank=r, fusion=fusion, tile_bits=tile_bits, layout=layout)
             for r in range(world)]
    kinds = [[(o["kind"], o["exch_bit"], o["exch_gx"], o["n_rot"]) for o in ops] for ops, _ in plans]
    assert all(k == kinds[0] for k in kinds), "plans must be SPMD-identical in structure"
    return plans, nl


def _execute(n, world, psi, plans, nl):
    local = [psi[r << nl:(r + 1) << nl].copy() for r in range(world)]
    mirror = [None] * world
    on_mirror = False
    cursors = [0] * world
    ops0 = plans[0][0]
    for t, op in enumerate(ops0):
        if op["kind"] == ps.OP_MIRROR_BEGIN:
            # paper step (i)+(ii): B_k = conj(w_k) A_(k xor gx), Q|k> = w_k|k xor gx>
            gx, gz = op["exch_gx"], op["tile_bits"]
            yq = bin(gx & gz).count("1") % 4
            newA, newB = [], []
            for r in range(world):
                w = (1j ** yq) * (-1.0 if bin(gz & r).count("1") % 2 else 1.0)
                b = np.conj(w) * local[r ^ gx]
                newA.append((local[r] + b) / math.sqrt(2))
                newB.append((local[r] - b) / math.sqrt(2))
            local, mirror = newA, newB
            on_mirror = False
            continue
        if op["kind"] == ps.OP_MIRROR_SWITCH:
            on_mirror = True
            continue
        if op["kind"] == ps.OP_MIRROR_END:
            local = [(a + b) / math.sqrt(2) for a, b in zip(local, mirror)]
            on_mirror = False
            continue
        if op["kind"] in (ps.K_STREAM, ps.K_TILE, ps.K_COSET) and on_mirror:
            for r in range(world):
                for _ in range(op["n_rot"]):
                    mirror[r] = _apply_phys(mirror[r], plans[r][1][cursors[r]])
                    cursors[r] += 1
            continue
        if op["kind"] == ps.K_PERMUTE:
            a, b = op["exch_bit"], op["exch_gx"]
            idx = np.arange(1 << nl)
            swp = idx ^ ((((idx >> a) ^ (idx >> b)) & 1) * ((1 << a) | (1 << b)))
            local = [v[swp] for v in local]
        elif op["kind"] == ps.K_EXCHANGE and op["exch_bit"] >= 0:
            ell, gx = op["exch_bit"], op["exch_gx"]
            g = (gx & -gx).bit_length() - 1
            new = [v.copy() for v in local]
            for r in range(world):
                keep = (r >> g) & 1
                p = r ^ gx
                for slot in range(1 << nl):
                    if ((slot >> ell) & 1) != keep:
                        new[r][slot] = local[p][slot ^ (1 << ell)]
            local = new
        elif op["kind"] == ps.K_EXCHANGE:
            # full exchange of a single rotation: own elements against the partner's old values
            gx = op["exch_gx"]
            new = []
            for r in range(world):
                rr = plans[r][1][cursors[r]]
                cursors[r] += 1
                p = r ^ gx
                idx = np.arange(1 << nl, dtype=np.uint64)
                par = np.array([bin(int(v)).count("1") & 1 for v in idx & np.uint64(rr["z"])])
                w = (1j ** rr["y"]) * rr["sign"] * np.where(par == 1, -1.0, 1.0)  # w(own i)
                c, s = math.cos(rr["angle"]), math.sin(rr["angle"])
                j = (idx ^ np.uint64(rr["x"])).astype(np.int64)
                new.append(c * local[r] + 1j * s * np.conj(w) * local[p][j])
            local = new
        else:
            for r in range(world):
                for _ in range(op["n_rot"]):
                    local[r] = _apply_phys(local[r], plans[r][1][cursors[r]])
                    cursors[r] += 1
    return np.concatenate(local)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("kind", ["R4", "R10", "S8"])
@pytest.mark.parametrize("layout", [0, 1, 2])
def test_planner_model_matches_oracle(world, kind, layout):
    n = 7
    codes, ang = workloads.random_layer(n, 60, seed=world, kind=kind)
    x, z = P.pauli_encode_codes(codes)
    psi = oracle.random_state(3, n)
    want = oracle.apply(n, psi, codes, ang)
    plans, nl = _run_model(n, world, x, z, ang, layout=layout)
    got = _execute(n, world, psi, plans, nl)
    assert np.max(np.abs(got - want)) <= 1e-12


def test_lazy_layout_needs_fewer_exchanges():
    """Belady swaps keep a swapped-in qubit until its slot is needed."""
    n, world = 16, 2
    codes, ang = workloads.random_layer(n, 400, seed=9, kind="R10")
    x, z = P.pauli_encode_codes(codes)
    ex = {}
    for layout in (0, 1):
        ops, _ = P.plan_describe(n, x, z, ang, world=world, rank=0, layout=layout, tile_bits=8)
        ex[layout] = sum(o["kind"] == ps.K_EXCHANGE for o in ops)
    assert ex[1] < 0.75 * ex[0]


@pytest.mark.parametrize("layout", [0, 1])
def test_planner_full_exchange_fallback(layout):
    """A global-X string whose local X-part covers every local bit has no free pivot: the plan
    uses the single-rotation full exchange and still matches the oracle."""
    n, world = 4, 2
    words = ["XXXX", "YXZY", "ZZZZ", "XYXY", "IXIX"]
    codes = oracle.words_to_factors(words)
    x, z = P.pauli_encode_codes(codes)
    ang = np.array([0.3, -1.2, 0.7, 2.0, -0.5])
    psi = oracle.random_state(5, n)
    plans, nl = _run_model(n, world, x, z, ang, layout=layout)
    assert any(o["kind"] == ps.K_EXCHANGE and o["exch_bit"] < 0 for o in plans[0][0])
    got = _execute(n, world, psi, plans, nl)
    assert np.max(np.abs(got - oracle.apply(n, psi, codes, ang))) <= 1e-12


def test_mirror_mode_one_exchange_per_group():
    """PS_OPT_LAYOUT=2: a group sharing the upper string Q costs one exchange, and
    grouped execution equals the sequential product (Eq. (core_state), checked by the model)."""
    n, world = 8, 4
    rng = np.random.default_rng(3)
    L = 25
    codes = np.zeros((L, n), np.uint8)
    codes[:, :6] = rng.integers(0, 4, size=(L, 6))
    codes[:, 6] = 2  # Y on global qubit 6
    codes[:, 7] = 3  # Z on global qubit 7
    x, z = P.pauli_encode_codes(codes)
    ang = rng.uniform(-1, 1, L)
    ops, _ = P.plan_describe(n, x, z, ang, world=world, rank=1, layout=2)
    assert sum(o["kind"] == ps.OP_MIRROR_BEGIN for o in ops) == 1
    plans, nl = _run_model(n, world, x, z, ang, layout=2)
    psi = oracle.random_state(9, n)
    got = _execute(n, world, psi, plans, nl)
    assert np.max(np.abs(got - oracle.apply(n, psi, codes, ang))) <= 1e-12


def test_exchange_economy():
    """Eq. (1): a run sharing the upper X-part needs one exchange (plus the
    swap back); z-only upper support needs none."""
    n, world = 8, 4  # top 2 qubits are global
    rng = np.random.default_rng(1)
    L = 30
    codes = np.zeros((L, n), np.uint8)
    codes[:, :4] = rng.integers(0, 4, size=(L, 4))
    codes[:, 6] = 1  # X on global qubit 6 for every rotation
    codes[:, 7] = rng.integers(0, 2, size=L) * 3  # I/Z on global qubit 7
    x, z = P.pauli_encode_codes(codes)
    for layout in (0, 1):  # one exchange in, one back (lazy layout: back at the restore)
        ops, _ = P.plan_describe(n, x, z, rng.uniform(-1, 1, L), world=world, rank=1, layout=layout)
        assert sum(o["kind"] == ps.K_EXCHANGE for o in ops) == 2
    codes[:, 6] = 3  # now Z only on the global qubits
    x, z = P.pauli_encode_codes(codes)
    for layout in (0, 1):
        ops, _ = P.plan_describe(n, x, z, rng.uniform(-1, 1, L), world=world, rank=1, layout=layout)
        assert sum(o["kind"] == ps.K_EXCHANGE for o in ops) == 0


def test_fusion_levels_cover_every_rotation_in_order():
    n = 16
    codes, ang = workloads.random_layer(n, 300, seed=2, kind="R10")
    x, z = P.pauli_encode_codes(codes)
    for fusion in (0, 1, 2):
        ops, rots = P.plan_describe(n, x, z, ang, fusion=fusion, tile_bits=12)
        covered = []
        for o in ops:
            covered.extend(range(o["first_rot"], o["first_rot"] + o["n_rot"]))
        assert covered == list(range(300))
        if fusion == 0:
            assert len(ops) == 300
    ops2, _ = P.plan_describe(n, x, z, ang, fusion=2, tile_bits=12)
    assert len(ops2) < 300 / 3  # coset tiles fuse random layers


def test_jw_hamiltonian_shape():
    codes, coeffs = workloads.jw_hamiltonian(16, 3000, 27.0, n_local=14)
    assert codes.shape == (3000, 16)
    assert abs(np.abs(coeffs).sum() - 27.0) < 1e-9
    x, z = P.pauli_encode_codes(codes)
    assert len(np.unique(np.stack([x, z], 1), axis=0)) == 3000
