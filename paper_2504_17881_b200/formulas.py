"""Product-formula rotation streams (NEXT-3, host side): the inputs the application layer feeds to
``ps_apply_rotations``.  These builders only produce (xmask, zmask, angle) arrays; every amplitude
update runs in libps.

  H = sum_l h_l P_l, lambda = sum_l |h_l|
  first-order Trotter  e^{i delta H} ~ prod_l e^{i delta h_l P_l}
  second-order Trotter (forward sweep at delta/2, reverse sweep at delta/2)
  qDRIFT: sample l with probability |h_l|/lambda, rotate by sign(h_l) lambda t / r
  partially randomized split H = H_D + H_R (L_det largest |h_l|)            P:595-601 (Eq. hamil_split)
  step: D forward delta/2; two qDRIFT stages of H_R at delta/2; D reverse delta/2
  samples per stage r = ceil(kappa lambda_R^2 delta^2 2^M), kappa = delta/(0.2 pi)

Ordering: deterministic terms x-major ("ordered lexicographically", R14);
randomized samples are never reordered.  Random draws use a counter-based generator
(splitmix64 of (seed, counter)) so every rank of a sharded run builds the identical stream.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

_GOLDEN = 0x9E3779B97F4A7C15
_M64 = (1 << 64) - 1


@dataclass
class Hamiltonian:
    n: int
    x: np.ndarray        # uint64 xor masks
    z: np.ndarray        # uint64 phase masks
    h: np.ndarray        # float64 coefficients
    offset: float = 0.0  # identity coefficient (a global phase e^{i offset t})

    @property
    def lam(self) -> float:
        return float(np.abs(self.h).sum())

    def __len__(self):
        return len(self.h)

    def take(self, idx) -> "Hamiltonian":
        idx = np.asarray(idx, dtype=np.int64)
        return Hamiltonian(self.n, self.x[idx].copy(), self.z[idx].copy(), self.h[idx].copy(), 0.0)


def from_masks(n, x, z, h, offset: float = 0.0) -> Hamiltonian:
    x = np.ascontiguousarray(x, dtype=np.uint64)
    z = np.ascontiguousarray(z, dtype=np.uint64)
    h = np.ascontiguousarray(h, dtype=np.float64)
    keep = (x != 0) | (z != 0)
    offset += float(h[~keep].sum())  # identity terms -> offset
    return Hamiltonian(n, x[keep], z[keep], h[keep], offset)


def order_lex(H: Hamiltonian, n_local: int | None = None) -> Hamiltonian:
    """x-major order: (upper X-part, X-part, Z-part) -- groups terms sharing the upper X-part."""
    nl = H.n if n_local is None else n_local
    hi = H.x >> np.uint64(nl) if nl < 64 else np.zeros_like(H.x)
    order = np.lexsort((H.z, H.x, hi))
    return H.take(order) if len(H) else H


def split_deterministic(H: Hamiltonian, l_det: int, n_local: int | None = None):
    """(H_D, H_R): the l_det largest-|h| terms (ties by masks) deterministic, x-major ordered."""
    if not 0 <= l_det <= len(H):
        raise ValueError("l_det out of range")
    order = np.lexsort((H.z, H.x, -np.abs(H.h)))
    hd = order_lex(H.take(order[:l_det]), n_local)
    hr = H.take(order[l_det:])
    return hd, hr


def trotter1_step(H: Hamiltonian, delta: float):
    return H.x.copy(), H.z.copy(), delta * H.h


def trotter2_step(H: Hamiltonian, delta: float):
    x = np.concatenate([H.x, H.x[::-1]])
    z = np.concatenate([H.z, H.z[::-1]])
    a = np.concatenate([0.5 * delta * H.h, 0.5 * delta * H.h[::-1]])
    return x, z, a


def splitmix_uniform(seed: int, counters: np.ndarray) -> np.ndarray:
    """u in [0, 1) from splitmix64 output (counter+1) of state `seed` (top 53 bits)."""
    c = (np.asarray(counters, dtype=np.uint64) + np.uint64(1))
    with np.errstate(over="ignore"):
        zz = np.uint64(seed) + c * np.uint64(_GOLDEN)
        zz = (zz ^ (zz >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        zz = (zz ^ (zz >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        zz = zz ^ (zz >> np.uint64(31))
    return (zz >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def qdrift_stage(HR: Hamiltonian, t: float, r: int, seed: int, counter: int):
    """r sampled rotations (P_l, sign(h_l) lambda_R t / r), l ~ |h_l|/lambda_R."""
    if r < 0:
        raise ValueError("r must be >= 0")
    if r == 0 or len(HR) == 0:
        if r > 0 and len(HR) == 0:
            raise ValueError("r > 0 with an empty randomized part")
        return np.zeros(0, np.uint64), np.zeros(0, np.uint64), np.zeros(0)
    lam = HR.lam
    cdf = np.cumsum(np.abs(HR.h)) / lam
    cdf[-1] = 1.0
    u = splitmix_uniform(seed, counter + np.arange(r, dtype=np.uint64))
    idx = np.minimum(np.searchsorted(cdf, u, side="right"), len(HR) - 1)
    ang = np.sign(HR.h[idx]) * lam * t / r
    return HR.x[idx].copy(), HR.z[idx].copy(), ang


def sample_count(lam_r: float, delta: float, m_max: int, kappa: float | None = None, reduction: float = 1.0) -> int:
    """r = ceil(kappa lambda_R^2 delta^2 2^M), kappa = delta / (0.2 pi); an optional
    reduction factor (the paper reduces by up to 3)."""
    if delta <= 0:
        raise ValueError("delta must be positive")
    k = delta / (0.2 * math.pi) if kappa is None else kappa
    return int(math.ceil(k * lam_r * lam_r * delta * delta * (2 ** m_max) * reduction - 1e-12))


def partially_randomized_step(HD: Hamiltonian, HR: Hamiltonian, delta: float, r: int, seed: int, step: int):
    """Second-order partially randomized step: D forward at delta/2, qDRIFT stage,
    qDRIFT stage (fresh samples), D reverse at delta/2.  Counters (step, stage, sample) make the
    stream identical on every rank."""
    if r == 0 and len(HR) > 0:
        raise ValueError("r = 0 would drop a non-empty randomized part")
    xs, zs, as_ = [], [], []
    fx, fz, fa = HD.x, HD.z, 0.5 * delta * HD.h
    xs.append(fx); zs.append(fz); as_.append(fa)
    for stage in range(2):
        cx, cz, ca = qdrift_stage(HR, 0.5 * delta, r, seed, counter=(2 * step + stage) * r)
        xs.append(cx); zs.append(cz); as_.append(ca)
    xs.append(fx[::-1]); zs.append(fz[::-1]); as_.append(fa[::-1])
    return (np.concatenate(xs).astype(np.uint64), np.concatenate(zs).astype(np.uint64),
            np.concatenate(as_).astype(np.float64))


def evolution_stream(HD: Hamiltonian, HR: Hamiltonian, delta: float, steps: int, r: int, seed: int):
    """`steps` independent partially randomized steps (fresh samples each)."""
    parts = [partially_randomized_step(HD, HR, delta, r, seed, s) for s in range(steps)]
    return (np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts]),
            np.concatenate([p[2] for p in parts]))
