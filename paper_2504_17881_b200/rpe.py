"""Robust-phase-estimation signals on the sharded state (NEXT-3).

  Z_m = <psi| e^{i delta H~(delta) 2^m} |psi>          P:667-671 (Data analysis)

computed with libps: a State holding |psi> is kept, a second State is evolved by 2^m partially
randomized second-order steps (``formulas.evolution_stream``, applied through
``ps_apply_rotations``), and Z_m = <psi|evolved> comes from ``ps_inner`` (fp64 accumulation,
NCCL all-reduce over ranks).  The energy offset (identity term) adds the phase e^{i offset delta 2^m}.

``estimate`` is the RPE phase refinement over rounds m = 0..M (Kimmel et al., cited at P:660; the
update rule is the standard one: each round picks the branch of arg(Z_m)/2^m nearest to the
previous estimate).
"""
from __future__ import annotations

import cmath
import math

import numpy as np

from . import formulas
from .ps import State


def signal(n: int, HD, HR, delta: float, m: int, r: int, seed: int, init="random", init_seed: int = 250417881,
           dtype: str = "c128", world: int = 1, rank: int = 0, offset: float = 0.0, emulate: int = 0) -> complex:
    """Z_m for one sampled circuit (the paper averages repeats for the randomized part).  emulate = G
    runs both states as G virtual ranks on this device (ps_create_emulated)."""
    x, z, a = formulas.evolution_stream(HD, HR, delta, 2 ** m, r, seed)
    kw = dict(emulate=emulate) if emulate else dict(world=world, rank=rank)
    with State(n, dtype, **kw) as psi0, State(n, dtype, **kw) as psi:
        for st in (psi0, psi):
            if init == "random":
                st.init_random(init_seed)
            else:
                st.init_basis(int(init))
        if init == "random":
            psi0.normalize()
            psi.normalize()
        psi.apply_rotations(x, z, a)
        zm = psi0.inner(psi)
    return zm * cmath.exp(1j * offset * delta * (2 ** m))


def estimate(zs, delta: float) -> float:
    """Energy estimate from Z_0..Z_M (phase theta_M / delta in (-pi/delta, pi/delta])."""
    if not len(zs):
        raise ValueError("no rounds")
    theta = cmath.phase(zs[0])
    for m in range(1, len(zs)):
        k = 2 ** m
        base = cmath.phase(zs[m])
        # candidates (base + 2 pi j) / k; choose the one nearest to theta
        j = round((theta * k - base) / (2 * math.pi))
        theta = (base + 2 * math.pi * j) / k
    theta = (theta + math.pi) % (2 * math.pi) - math.pi
    return theta / delta


def z0_basis(n: int, HD, HR, delta: float, r: int, seed: int, b: int, dtype: str = "c128", world: int = 1,
             rank: int = 0, emulate: int = 0, offset: float = 0.0, state=None) -> complex:
    """Z_0 = <b| e^{i delta H~(delta)} |b> for a basis guiding state |b> (Fig. 4):
    one partially randomized second-order step applied to |b> through ps_apply_rotations, then the
    amplitude b read back (no second state: the overlap with a basis state is one amplitude).  A
    caller-provided `state` (a State of n qubits) is reused instead of allocating one."""
    x, z, a = formulas.evolution_stream(HD, HR, delta, 1, r, seed)
    kw = dict(emulate=emulate) if emulate else dict(world=world, rank=rank)
    own = state is None
    st = State(n, dtype, **kw) if own else state
    try:
        st.init_basis(int(b))
        st.apply_rotations(x, z, a)
        z0 = complex(st.get_amplitudes(int(b), 1)[0])
    finally:
        if own:
            st.close()
    return z0 * cmath.exp(1j * offset * delta)
