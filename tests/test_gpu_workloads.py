"""1-GPU parity of the structured workloads of BASELINE.json configs 3-4 (``-m gpu``): a JW-shaped
first-order Trotter step (x-major order), QAOA MaxCut layers, a converted gate
brickwork, a UCCSD-shaped VQE layer and a hardware-efficient VQE ansatz, through the C ABI with
default options (and a grid cap so the persistent tile loop runs several tiles per CTA), against
the CPU oracle element by element.  Tolerances: BASELINE.json north_star."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import workloads
import paper_2504_17881_b200 as P
from paper_2504_17881_b200 import ps

pytestmark = pytest.mark.gpu

SEED = 250417881
TOL = {"c128": 1e-10, "c64": 1e-4}
_cache: dict = {}


def _workload(kind, n):
    key = (kind, n)
    if key in _cache:
        return _cache[key]
    if kind == "JW":
        codes, coeffs = workloads.jw_hamiltonian(n, 3000, 27.0, seed=3, n_local=n)
        x, z = P.pauli_encode_codes(codes)
        ang = workloads.trotter1_angles(coeffs, 0.5)
    elif kind == "QAOA":
        codes, ang = workloads.qaoa_layers(n, 4, seed=3)
        x, z = P.pauli_encode_codes(codes)
    elif kind == "UCC":
        codes, ang = workloads.ucc_layers(n, n // 2, seed=3, max_doubles=200)
        x, z = P.pauli_encode_codes(codes)
    elif kind in ("GATES", "HEA"):
        gates = workloads.gate_circuit(n, 8, seed=3) if kind == "GATES" else workloads.hardware_efficient_vqe(n, 4, seed=3)
        x, z, ang = P.circuit_to_rotations(gates)
        codes = oracle.decode_masks(n, x, z)  # the oracle decodes the product's masks itself
    else:
        raise ValueError(kind)
    want = oracle.apply(n, oracle.random_state(SEED, n), codes, ang)
    _cache[key] = (x, z, ang, want)
    return _cache[key]


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("kind", ["JW", "QAOA", "GATES", "UCC", "HEA"])
@pytest.mark.parametrize("cap", [0, 5])
def test_structured_workloads(kind, dtype, cap):
    n = 18
    x, z, ang, want = _workload(kind, n)
    with P.State(n, dtype) as st:
        if cap:
            st.set_option(ps.OPT_GRID_CAP, cap)
        st.init_random(SEED)
        st.apply_rotations(x, z, ang)
        got = st.get_amplitudes()
        stats = st.stats()
    err = float(np.max(np.abs(got - want)))
    assert err <= TOL[dtype], (err, stats["launches"], len(ang))


def test_gate_circuit_against_dense_unitary():
    """The converted gate circuit equals the product of the textbook gate matrices (n = 6), so the
    workload itself -- not just its rotation form -- is what the GPU path applies."""
    from oracle import dense
    n = 6
    gates = workloads.gate_circuit(n, 5, seed=9)
    x, z, ang = P.circuit_to_rotations(gates)
    psi = oracle.random_state(SEED, n)
    want = dense.apply_gates(n, psi, gates)
    with P.State(n, "c128") as st:
        st.init_random(SEED)
        st.apply_rotations(x, z, ang)
        got = st.get_amplitudes()
    assert np.max(np.abs(got - want)) <= 1e-12
