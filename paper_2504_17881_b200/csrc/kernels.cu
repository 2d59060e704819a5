// kernels.cu -- sm_100a kernels of libps (all HBM-bound; no contraction, no tensor cores).
//
//   K1 k_stream     streaming pair-rotation pass: one rotation or a same-x run applied to each
//                   pair {i, i xor x} in registers, 256-bit LDG/STG, pair indices by bit
//                   insertion (P:96-101 direct sum of 2x2 blocks; P:119-121 AND/XOR/parity)
//   K2/K7 k_coset   fused tile pass (default): a 2^k-amplitude tile -- contiguous (K2) or a
//                   gathered coset i0 xor span{v_t} of contiguous chunks (K7) -- whose rotations
//                   are applied in sub-groups of <= 4-dimensional xor span, each thread holding a
//                   16-amplitude coset in registers; the first sub-group loads straight from HBM,
//                   the last stores straight back, shared memory carries the tile only between
//                   sub-groups (several rotations per traversal of the array)
//   K2/K7 k_tile    the same pass with the whole tile staged in shared memory by TMA bulk copies
//                   (cp.async.bulk + mbarrier ring; PS_OPT_TILE_TMA=1, kept for A/B evidence)
//   K5 k_norm/k_expect/k_inner   fp64-accumulating reductions
//   K6 k_init_*     seeded counter-based init, basis states
//   K3 k_full_update  single-rotation full-exchange update against a partner chunk
//
// Every kernel applies the SAME per-pair arithmetic (arith.cuh).
#include <cuda_runtime.h>
#include <cstdint>
#include <type_traits>

#include "arith.cuh"
#include "ps_internal.h"

namespace ps {
namespace {

template <typename T>
struct RotK {
    T c, b;
    int real;
};


template <typename T>
__device__ __forceinline__ RotK<T> load_rot(const DevRot* __restrict__ r) {
    RotK<T> k;
    k.c = (T)__ldg(&r->c);
    k.b = (T)__ldg(&r->b);
    k.real = (int)__ldg(&r->real);
    return k;
}

// ------------------------------------------------------------------------------------------
// vector global memory access: V amplitudes of type T per access (32 B = 256-bit when V*2*sizeof(T) == 32)

template <typename T, int V>
struct Vec {
    T r[V], i[V];
};

template <typename T, int V>
__device__ __forceinline__ void ld_vec(const T* p, Vec<T, V>& v);
template <typename T, int V>
__device__ __forceinline__ void st_vec(T* p, const Vec<T, V>& v);

template <>
__device__ __forceinline__ void ld_vec<double, 1>(const double* p, Vec<double, 1>& v) {
    asm volatile("ld.global.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.r[0]), "=d"(v.i[0]) : "l"(p));
}
template <>
__device__ __forceinline__ void st_vec<double, 1>(double* p, const Vec<double, 1>& v) {
    asm volatile("st.global.v2.f64 [%0], {%1,%2};" ::"l"(p), "d"(v.r[0]), "d"(v.i[0]) : "memory");
}
template <>
__device__ __forceinline__ void ld_vec<double, 2>(const double* p, Vec<double, 2>& v) {
    asm volatile("ld.global.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(v.r[0]), "=d"(v.i[0]), "=d"(v.r[1]), "=d"(v.i[1])
                 : "l"(p));
}
template <>
__device__ __forceinline__ void st_vec<double, 2>(double* p, const Vec<double, 2>& v) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v.r[0]), "d"(v.i[0]), "d"(v.r[1]),
                 "d"(v.i[1])
                 : "memory");
}
template <>
__device__ __forceinline__ void ld_vec<float, 1>(const float* p, Vec<float, 1>& v) {
    asm volatile("ld.global.L1::no_allocate.v2.f32 {%0,%1}, [%2];" : "=f"(v.r[0]), "=f"(v.i[0]) : "l"(p));
}
template <>
__device__ __forceinline__ void st_vec<float, 1>(float* p, const Vec<float, 1>& v) {
    asm volatile("st.global.v2.f32 [%0], {%1,%2};" ::"l"(p), "f"(v.r[0]), "f"(v.i[0]) : "memory");
}
template <>
__device__ __forceinline__ void ld_vec<float, 2>(const float* p, Vec<float, 2>& v) {
    asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.r[0]), "=f"(v.i[0]), "=f"(v.r[1]), "=f"(v.i[1])
                 : "l"(p));
}
template <>
__device__ __forceinline__ void st_vec<float, 2>(float* p, const Vec<float, 2>& v) {
    asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.r[0]), "f"(v.i[0]), "f"(v.r[1]),
                 "f"(v.i[1])
                 : "memory");
}
template <>
__device__ __forceinline__ void ld_vec<float, 4>(const float* p, Vec<float, 4>& v) {
    asm volatile("ld.global.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v.r[0]), "=f"(v.i[0]), "=f"(v.r[1]), "=f"(v.i[1]), "=f"(v.r[2]), "=f"(v.i[2]),
                   "=f"(v.r[3]), "=f"(v.i[3])
                 : "l"(p));
}
template <>
__device__ __forceinline__ void st_vec<float, 4>(float* p, const Vec<float, 4>& v) {
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(v.r[0]), "f"(v.i[0]),
                 "f"(v.r[1]), "f"(v.i[1]), "f"(v.r[2]), "f"(v.i[2]), "f"(v.r[3]), "f"(v.i[3])
                 : "memory");
}

// ------------------------------------------------------------------------------------------
// K1: streaming pass.  mode 0: pairs across vectors (pivot >= log2 V); mode 1: pairs inside a
// vector (x0 < V); mode 2: diagonal-only run.  One "unit" = one vector pair (mode 0) or one
// vector (modes 1, 2).  Each thread handles UNROLL units per iteration, loads first.

constexpr int kStreamThreads = 256;

// permutes v[e] <- v[e ^ m] for m < V with selects only (no dynamically indexed registers)
template <typename T, int V>
__device__ __forceinline__ void xor_permute(Vec<T, V>& v, int m) {
#pragma unroll
    for (int b = 1; b < V; b <<= 1) {
        if (m & b) {
#pragma unroll
            for (int e = 0; e < V; ++e) {
                if (e & b) continue;
                const T r = v.r[e], i = v.i[e];
                v.r[e] = v.r[e | b];
                v.i[e] = v.i[e | b];
                v.r[e | b] = r;
                v.i[e | b] = i;
            }
        }
    }
}

template <int REAL, typename T, int V>
__device__ __forceinline__ void pair_vecs(Vec<T, V>& vi, Vec<T, V>& vj, uint64_t ibase, uint64_t z, T c, T b) {
#pragma unroll
    for (int e = 0; e < V; ++e) {
        const int s = par64(z & (ibase + e));
        rot_pair<REAL>(vi.r[e], vi.i[e], vj.r[e], vj.i[e], c, flip(b, s));
    }
}

template <int REAL, typename T, int V>
__device__ __forceinline__ void diag_vec(Vec<T, V>& v, uint64_t base, int xin, uint64_t z, T c, T b) {
#pragma unroll
    for (int e = 0; e < V; ++e) {
        const int s = par64(z & (base + (e ^ xin)));
        rot_diag<REAL>(v.r[e], v.i[e], c, flip(b, s));
    }
}

// vj has been permuted so that vj[e] is the partner of vi[e] (original index jbase + (e ^ xin))
template <typename T, int V>
__device__ __forceinline__ void apply_run_pair(Vec<T, V>& vi, Vec<T, V>& vj, uint64_t ibase, int xin,
                                               uint64_t jbase, const DevRot* __restrict__ rec, int nrec) {
    for (int r = 0; r < nrec; ++r) {
        const uint64_t x = __ldg(&rec[r].x);
        const uint64_t z = __ldg(&rec[r].z);
        const RotK<T> k = load_rot<T>(&rec[r]);
        if (x == 0) {
            if (k.real) {
                diag_vec<1>(vi, ibase, 0, z, k.c, k.b);
                diag_vec<1>(vj, jbase, xin, z, k.c, k.b);
            } else {
                diag_vec<0>(vi, ibase, 0, z, k.c, k.b);
                diag_vec<0>(vj, jbase, xin, z, k.c, k.b);
            }
        } else if (k.real) {
            pair_vecs<1>(vi, vj, ibase, z, k.c, k.b);
        } else {
            pair_vecs<0>(vi, vj, ibase, z, k.c, k.b);
        }
    }
}

template <int REAL, typename T, int V, int X0>
__device__ __forceinline__ void intra_pairs(Vec<T, V>& v, uint64_t base, uint64_t z, T c, T b) {
    constexpr int piv = (X0 >= 2) ? 1 : 0;
#pragma unroll
    for (int e = 0; e < V; ++e) {
        if ((e >> piv) & 1) continue;
        const int f = e ^ X0;
        const int s = par64(z & (base + e));
        rot_pair<REAL>(v.r[e], v.i[e], v.r[f], v.i[f], c, flip(b, s));
    }
}

template <int REAL, typename T, int V>
__device__ __forceinline__ void intra_rot(Vec<T, V>& v, uint64_t base, uint64_t x, uint64_t z, T c, T b) {
    if (x == 0) {
        diag_vec<REAL>(v, base, 0, z, c, b);
    } else if (x == 1) {
        intra_pairs<REAL, T, V, 1>(v, base, z, c, b);
    } else if (V >= 4 && x == 2) {
        intra_pairs<REAL, T, V, (V >= 4 ? 2 : 1)>(v, base, z, c, b);
    } else if (V >= 4) {
        intra_pairs<REAL, T, V, (V >= 4 ? 3 : 1)>(v, base, z, c, b);
    }
}

template <typename T, int V>
__device__ __forceinline__ void apply_run_intra(Vec<T, V>& v, uint64_t base, const DevRot* __restrict__ rec,
                                                int nrec) {
    for (int r = 0; r < nrec; ++r) {
        const uint64_t x = __ldg(&rec[r].x);
        const uint64_t z = __ldg(&rec[r].z);
        const RotK<T> k = load_rot<T>(&rec[r]);
        if (k.real)
            intra_rot<1>(v, base, x, z, k.c, k.b);
        else
            intra_rot<0>(v, base, x, z, k.c, k.b);
    }
}

template <typename T, int V, int UNROLL>
__global__ void __launch_bounds__(kStreamThreads) k_stream(T* __restrict__ a, uint64_t units, int mode,
                                                           int piv, uint64_t x0,
                                                           const DevRot* __restrict__ rec, int nrec) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (mode == 0) {
        const uint64_t xv = x0 & ~(uint64_t)(V - 1);
        const int xin = (int)(x0 & (V - 1));
        for (uint64_t u = t0; u < units; u += stride * UNROLL) {
            Vec<T, V> vi[UNROLL], vj[UNROLL];
            uint64_t ib[UNROLL];
#pragma unroll
            for (int q = 0; q < UNROLL; ++q) {
                const uint64_t uq = u + (uint64_t)q * stride;
                ib[q] = insert0(uq * V, piv);
                if (uq < units) {
                    ld_vec<T, V>(a + 2 * ib[q], vi[q]);
                    ld_vec<T, V>(a + 2 * (ib[q] ^ xv), vj[q]);
                }
            }
#pragma unroll
            for (int q = 0; q < UNROLL; ++q) {
                const uint64_t uq = u + (uint64_t)q * stride;
                if (uq < units) {
                    xor_permute<T, V>(vj[q], xin);
                    apply_run_pair<T, V>(vi[q], vj[q], ib[q], xin, ib[q] ^ xv, rec, nrec);
                    xor_permute<T, V>(vj[q], xin);
                }
            }
#pragma unroll
            for (int q = 0; q < UNROLL; ++q) {
                const uint64_t uq = u + (uint64_t)q * stride;
                if (uq < units) {
                    st_vec<T, V>(a + 2 * ib[q], vi[q]);
                    st_vec<T, V>(a + 2 * (ib[q] ^ xv), vj[q]);
                }
            }
        }
    } else {
        for (uint64_t u = t0; u < units; u += stride * UNROLL) {
            Vec<T, V> v[UNROLL];
#pragma unroll
            for (int q = 0; q < UNROLL; ++q) {
                const uint64_t uq = u + (uint64_t)q * stride;
                if (uq < units) ld_vec<T, V>(a + 2 * uq * V, v[q]);
            }
#pragma unroll
            for (int q = 0; q < UNROLL; ++q) {
                const uint64_t uq = u + (uint64_t)q * stride;
                if (uq < units) apply_run_intra<T, V>(v[q], uq * V, rec, nrec);
            }
#pragma unroll
            for (int q = 0; q < UNROLL; ++q) {
                const uint64_t uq = u + (uint64_t)q * stride;
                if (uq < units) st_vec<T, V>(a + 2 * uq * V, v[q]);
            }
        }
    }
}

// ------------------------------------------------------------------------------------------
// sub-group arithmetic shared by the tile kernels (deferred-scale form, ps_internal.h DevTRot):
// each component update is one fused multiply-add; F = product of the factors is applied when
// the amplitudes leave the registers.

// record loads: read-only global (__ldg) or the kernel's parameter block (PARAM = 1: uniform
// constant-bank loads)
template <int PARAM, typename U>
__device__ __forceinline__ U ldr(const U* p) {
    if constexpr (PARAM) return *p;
    else return __ldg(p);
}

__host__ __device__ constexpr int hibit(int v) { return v >= 8 ? 3 : v >= 4 ? 2 : v >= 2 ? 1 : 0; }

// SFORM = 0: a'_i = a_i + s*Ac a_j, a'_j = a_j + s*Bc a_i with Bc = t (REAL) or i t, Ac = -conj(Bc)
// SFORM = 1: a'_i = t a_i + s*Ac a_j, a'_j = t a_j + s*Bc a_i with Bc = g (REAL) or i g, g = +-1
template <int REAL, int SFORM, typename T>
__device__ __forceinline__ void dpair(T& ir, T& ii, T& jr, T& ji, T t, int neg) {
    if (!SFORM) {
        const T b = flip(t, neg);
        if (REAL) {
            const T nir = pfma(-b, jr, ir), nii = pfma(-b, ji, ii);
            const T njr = pfma(b, ir, jr), nji = pfma(b, ii, ji);
            ir = nir; ii = nii; jr = njr; ji = nji;
        } else {
            const T nir = pfma(-b, ji, ir), nii = pfma(b, jr, ii);
            const T njr = pfma(-b, ii, jr), nji = pfma(b, ir, ji);
            ir = nir; ii = nii; jr = njr; ji = nji;
        }
    } else {
        // g = -1 when neg: cross operands carry the sign, the fixed signs ride on the FMA
        const T gjr = flip(jr, neg), gji = flip(ji, neg), gir = flip(ir, neg), gii = flip(ii, neg);
        if (REAL) {
            const T nir = pfma(t, ir, -gjr), nii = pfma(t, ii, -gji);
            const T njr = pfma(t, jr, gir), nji = pfma(t, ji, gii);
            ir = nir; ii = nii; jr = njr; ji = nji;
        } else {
            const T nir = pfma(t, ir, -gji), nii = pfma(t, ii, gjr);
            const T njr = pfma(t, jr, -gii), nji = pfma(t, ji, gir);
            ir = nir; ii = nii; jr = njr; ji = nji;
        }
    }
}

// diagonal element: a' = a + s*Ac a (SFORM 0) or t a + s*Ac a (SFORM 1)
template <int REAL, int SFORM, typename T>
__device__ __forceinline__ void ddiag(T& r, T& i, T t, int neg) {
    if (!SFORM) {
        const T b = flip(t, neg);
        if (REAL) {
            const T nr = pfma(-b, r, r), ni = pfma(-b, i, i);
            r = nr; i = ni;
        } else {
            const T nr = pfma(-b, i, r), ni = pfma(b, r, i);
            r = nr; i = ni;
        }
    } else {
        const T gr = flip(r, neg), gi = flip(i, neg);
        if (REAL) {
            const T nr = pfma(t, r, -gr), ni = pfma(t, i, -gi);
            r = nr; i = ni;
        } else {
            const T nr = pfma(t, r, -gi), ni = pfma(t, i, gr);
            r = nr; i = ni;
        }
    }
}

// Ms bit d = sigma of element d (1: -1) xor the NEG bit of SFORM rotations
template <int REAL, int SFORM, typename T, int DX>
__device__ __forceinline__ void sub_pairs(T (&vr)[kSubAmps], T (&vi)[kSubAmps], uint32_t Ms, T t) {
    if constexpr (DX < kSubAmps) {
        constexpr int piv = hibit(DX);
#pragma unroll
        for (int d = 0; d < kSubAmps; ++d) {
            if ((d >> piv) & 1) continue;
            const int e = d ^ DX;
            dpair<REAL, SFORM>(vr[d], vi[d], vr[e], vi[e], t, (int)((Ms >> d) & 1u));
        }
    }
}

template <int REAL, int SFORM, typename T>
__device__ __forceinline__ void sub_rotation(T (&vr)[kSubAmps], T (&vi)[kSubAmps], uint32_t dx, uint32_t Ms, T t) {
    switch (dx) {
    case 0:
#pragma unroll
        for (int d = 0; d < kSubAmps; ++d) ddiag<REAL, SFORM>(vr[d], vi[d], t, (int)((Ms >> d) & 1u));
        break;
    case 1: sub_pairs<REAL, SFORM, T, 1>(vr, vi, Ms, t); break;
    case 2: sub_pairs<REAL, SFORM, T, 2>(vr, vi, Ms, t); break;
    case 3: sub_pairs<REAL, SFORM, T, 3>(vr, vi, Ms, t); break;
    case 4: sub_pairs<REAL, SFORM, T, 4>(vr, vi, Ms, t); break;
    case 5: sub_pairs<REAL, SFORM, T, 5>(vr, vi, Ms, t); break;
    case 6: sub_pairs<REAL, SFORM, T, 6>(vr, vi, Ms, t); break;
    case 7: sub_pairs<REAL, SFORM, T, 7>(vr, vi, Ms, t); break;
#if PS_SUBDIM >= 4
    case 8: sub_pairs<REAL, SFORM, T, 8>(vr, vi, Ms, t); break;
    case 9: sub_pairs<REAL, SFORM, T, 9>(vr, vi, Ms, t); break;
    case 10: sub_pairs<REAL, SFORM, T, 10>(vr, vi, Ms, t); break;
    case 11: sub_pairs<REAL, SFORM, T, 11>(vr, vi, Ms, t); break;
    case 12: sub_pairs<REAL, SFORM, T, 12>(vr, vi, Ms, t); break;
    case 13: sub_pairs<REAL, SFORM, T, 13>(vr, vi, Ms, t); break;
    case 14: sub_pairs<REAL, SFORM, T, 14>(vr, vi, Ms, t); break;
    default: sub_pairs<REAL, SFORM, T, 15>(vr, vi, Ms, t); break;
#else
    default: break;
#endif
    }
}

__host__ __device__ constexpr int par4(int v) { return (v ^ (v >> 1) ^ (v >> 2) ^ (v >> 3)) & 1; }

// one CFORM rotation with a compile-time pair pattern (dx = DX) and sign pattern parity(DZ & d):
// four fused multiply-adds per pair, the signs ride on the FMA operands.  PS_SHEAR: every
// two-cycle of components (x, y) is rotated in place by three shears, x -= tau y; y += sg x;
// x -= tau y (tau = tan(theta/2), sg = sin(theta), ps_internal.h kTrUnit): six FMAs per pair and
// no register moves (the 4-FMA form must park one member of each two-cycle in a temporary)
template <typename T>
__device__ __forceinline__ void shear3(T& x, T& y, T tau, T sg) {
    x = pfma(-tau, y, x);
    y = pfma(sg, x, y);
    x = pfma(-tau, y, x);
}

template <int REAL, int DX, int DZ, typename T>
__device__ __forceinline__ void cform_sub(T (&vr)[kSubAmps], T (&vi)[kSubAmps], T t, T sg) {
    if constexpr (DX == 0) {
#pragma unroll
        for (int d = 0; d < kSubAmps; ++d) {
            const T b = par4(DZ & d) ? -t : t;
#if PS_SHEAR
            shear3(vr[d], vi[d], b, par4(DZ & d) ? -sg : sg);
#else
            const T nr = pfma(-b, vi[d], vr[d]), ni = pfma(b, vr[d], vi[d]);
            vr[d] = nr;
            vi[d] = ni;
#endif
        }
    } else if constexpr (DX < kSubAmps) {
        constexpr int piv = hibit(DX);
#pragma unroll
        for (int d = 0; d < kSubAmps; ++d) {
            if ((d >> piv) & 1) continue;
            const int e = d ^ DX;
            const T b = par4(DZ & d) ? -t : t;
#if PS_SHEAR
            const T g = par4(DZ & d) ? -sg : sg;
            if (REAL) {
                shear3(vr[d], vr[e], b, g);
                shear3(vi[d], vi[e], b, g);
            } else {
                shear3(vr[d], vi[e], b, g);
                shear3(vr[e], vi[d], b, g);
            }
#else
            if (REAL) {
                const T nir = pfma(-b, vr[e], vr[d]), nii = pfma(-b, vi[e], vi[d]);
                const T njr = pfma(b, vr[d], vr[e]), nji = pfma(b, vi[d], vi[e]);
                vr[d] = nir; vi[d] = nii; vr[e] = njr; vi[e] = nji;
            } else {
                const T nir = pfma(-b, vi[e], vr[d]), nii = pfma(b, vr[e], vi[d]);
                const T njr = pfma(-b, vi[d], vr[e]), nji = pfma(b, vr[d], vi[e]);
                vr[d] = nir; vi[d] = nii; vr[e] = njr; vi[e] = nji;
            }
#endif
        }
    }
}

#if PS_SHEAR
// the generic kernel's form of the same shear rotation (unit dx, run-time per-pair signs Ms)
template <int REAL, int DX, typename T>
__device__ __forceinline__ void shear_pairs(T (&vr)[kSubAmps], T (&vi)[kSubAmps], uint32_t Ms, T t, T sg) {
#pragma unroll
    for (int d = 0; d < kSubAmps; ++d) {
        const int ng = (int)((Ms >> d) & 1u);
        const T b = flip(t, ng), g = flip(sg, ng);
        if constexpr (DX == 0) {
            shear3(vr[d], vi[d], b, g);
        } else {
            if ((d >> hibit(DX)) & 1) continue;
            const int e = d ^ DX;
            if (REAL) {
                shear3(vr[d], vr[e], b, g);
                shear3(vi[d], vi[e], b, g);
            } else {
                shear3(vr[d], vi[e], b, g);
                shear3(vr[e], vi[d], b, g);
            }
        }
    }
}

template <typename T>
__device__ __forceinline__ void shear_rotation(T (&vr)[kSubAmps], T (&vi)[kSubAmps], uint32_t dx, int real,
                                               uint32_t Ms, T t, T sg) {
    switch (dx | (real ? 16u : 0u)) {
    case 0: shear_pairs<0, 0>(vr, vi, Ms, t, sg); break;
    case 1: shear_pairs<0, 1>(vr, vi, Ms, t, sg); break;
    case 2: shear_pairs<0, 2>(vr, vi, Ms, t, sg); break;
    case 4: shear_pairs<0, 4>(vr, vi, Ms, t, sg); break;
    case 17: shear_pairs<1, 1>(vr, vi, Ms, t, sg); break;
    case 18: shear_pairs<1, 2>(vr, vi, Ms, t, sg); break;
    case 20: shear_pairs<1, 4>(vr, vi, Ms, t, sg); break;
#if PS_SUBDIM >= 4
    case 8: shear_pairs<0, 8>(vr, vi, Ms, t, sg); break;
    case 24: shear_pairs<1, 8>(vr, vi, Ms, t, sg); break;
#endif
    default: break;
    }
}
#endif

// unit cases (ps_internal.h tu_case): diagonal by its 4-bit Dz, unit dx by (real, log2 dx, the three
// Dz bits other than the pivot's); signs and the pair pattern are compile-time
#define PS_UD(Z) case Z: cform_sub<0, 0, Z, T>(vr, vi, t, sg); break;
#define PS_UC(R, XI, Z3) case tu_case(R, XI, tu_dz(XI, Z3)): cform_sub<R, (1 << XI), tu_dz(XI, Z3), T>(vr, vi, t, sg); break;
#define PS_UC8(R, XI) PS_UC(R, XI, 0) PS_UC(R, XI, 1) PS_UC(R, XI, 2) PS_UC(R, XI, 3) PS_UC(R, XI, 4) \
    PS_UC(R, XI, 5) PS_UC(R, XI, 6) PS_UC(R, XI, 7)

#ifndef PS_DISPATCH1
// two-level dispatch (default: +0.9 % R10, +1.9 % JW, +1.7 % gates over one 80-way switch,
// profiles/r02/kernel_ab.md section 7): by case id / 16, then 16-way inner switches
template <typename T>
__device__ __forceinline__ void unit_dispatch(T (&vr)[kSubAmps], T (&vi)[kSubAmps], uint32_t ucase, T t, T sg) {
    switch (ucase >> 4) {
    case 0:
        switch (ucase & 15u) {
        case 0: cform_sub<0, 0, 0, T>(vr, vi, t, sg); break;
        case 1: cform_sub<0, 0, 1, T>(vr, vi, t, sg); break;
        case 2: cform_sub<0, 0, 2, T>(vr, vi, t, sg); break;
        case 3: cform_sub<0, 0, 3, T>(vr, vi, t, sg); break;
        case 4: cform_sub<0, 0, 4, T>(vr, vi, t, sg); break;
        case 5: cform_sub<0, 0, 5, T>(vr, vi, t, sg); break;
        case 6: cform_sub<0, 0, 6, T>(vr, vi, t, sg); break;
        case 7: cform_sub<0, 0, 7, T>(vr, vi, t, sg); break;
        case 8: cform_sub<0, 0, 8, T>(vr, vi, t, sg); break;
        case 9: cform_sub<0, 0, 9, T>(vr, vi, t, sg); break;
        case 10: cform_sub<0, 0, 10, T>(vr, vi, t, sg); break;
        case 11: cform_sub<0, 0, 11, T>(vr, vi, t, sg); break;
        case 12: cform_sub<0, 0, 12, T>(vr, vi, t, sg); break;
        case 13: cform_sub<0, 0, 13, T>(vr, vi, t, sg); break;
        case 14: cform_sub<0, 0, 14, T>(vr, vi, t, sg); break;
        case 15: cform_sub<0, 0, 15, T>(vr, vi, t, sg); break;
        default: break;
        }
        break;
    case 1:
        switch (ucase & 15u) {
        case 0: cform_sub<0, (1 << 0), tu_dz(0, 0), T>(vr, vi, t, sg); break;
        case 1: cform_sub<0, (1 << 0), tu_dz(0, 1), T>(vr, vi, t, sg); break;
        case 2: cform_sub<0, (1 << 0), tu_dz(0, 2), T>(vr, vi, t, sg); break;
        case 3: cform_sub<0, (1 << 0), tu_dz(0, 3), T>(vr, vi, t, sg); break;
        case 4: cform_sub<0, (1 << 0), tu_dz(0, 4), T>(vr, vi, t, sg); break;
        case 5: cform_sub<0, (1 << 0), tu_dz(0, 5), T>(vr, vi, t, sg); break;
        case 6: cform_sub<0, (1 << 0), tu_dz(0, 6), T>(vr, vi, t, sg); break;
        case 7: cform_sub<0, (1 << 0), tu_dz(0, 7), T>(vr, vi, t, sg); break;
        case 8: cform_sub<0, (1 << 1), tu_dz(1, 0), T>(vr, vi, t, sg); break;
        case 9: cform_sub<0, (1 << 1), tu_dz(1, 1), T>(vr, vi, t, sg); break;
        case 10: cform_sub<0, (1 << 1), tu_dz(1, 2), T>(vr, vi, t, sg); break;
        case 11: cform_sub<0, (1 << 1), tu_dz(1, 3), T>(vr, vi, t, sg); break;
        case 12: cform_sub<0, (1 << 1), tu_dz(1, 4), T>(vr, vi, t, sg); break;
        case 13: cform_sub<0, (1 << 1), tu_dz(1, 5), T>(vr, vi, t, sg); break;
        case 14: cform_sub<0, (1 << 1), tu_dz(1, 6), T>(vr, vi, t, sg); break;
        case 15: cform_sub<0, (1 << 1), tu_dz(1, 7), T>(vr, vi, t, sg); break;
        default: break;
        }
        break;
    case 2:
        switch (ucase & 15u) {
        case 0: cform_sub<0, (1 << 2), tu_dz(2, 0), T>(vr, vi, t, sg); break;
        case 1: cform_sub<0, (1 << 2), tu_dz(2, 1), T>(vr, vi, t, sg); break;
        case 2: cform_sub<0, (1 << 2), tu_dz(2, 2), T>(vr, vi, t, sg); break;
        case 3: cform_sub<0, (1 << 2), tu_dz(2, 3), T>(vr, vi, t, sg); break;
        case 4: cform_sub<0, (1 << 2), tu_dz(2, 4), T>(vr, vi, t, sg); break;
        case 5: cform_sub<0, (1 << 2), tu_dz(2, 5), T>(vr, vi, t, sg); break;
        case 6: cform_sub<0, (1 << 2), tu_dz(2, 6), T>(vr, vi, t, sg); break;
        case 7: cform_sub<0, (1 << 2), tu_dz(2, 7), T>(vr, vi, t, sg); break;
        case 8: cform_sub<0, (1 << 3), tu_dz(3, 0), T>(vr, vi, t, sg); break;
        case 9: cform_sub<0, (1 << 3), tu_dz(3, 1), T>(vr, vi, t, sg); break;
        case 10: cform_sub<0, (1 << 3), tu_dz(3, 2), T>(vr, vi, t, sg); break;
        case 11: cform_sub<0, (1 << 3), tu_dz(3, 3), T>(vr, vi, t, sg); break;
        case 12: cform_sub<0, (1 << 3), tu_dz(3, 4), T>(vr, vi, t, sg); break;
        case 13: cform_sub<0, (1 << 3), tu_dz(3, 5), T>(vr, vi, t, sg); break;
        case 14: cform_sub<0, (1 << 3), tu_dz(3, 6), T>(vr, vi, t, sg); break;
        case 15: cform_sub<0, (1 << 3), tu_dz(3, 7), T>(vr, vi, t, sg); break;
        default: break;
        }
        break;
    case 3:
        switch (ucase & 15u) {
        case 0: cform_sub<1, (1 << 0), tu_dz(0, 0), T>(vr, vi, t, sg); break;
        case 1: cform_sub<1, (1 << 0), tu_dz(0, 1), T>(vr, vi, t, sg); break;
        case 2: cform_sub<1, (1 << 0), tu_dz(0, 2), T>(vr, vi, t, sg); break;
        case 3: cform_sub<1, (1 << 0), tu_dz(0, 3), T>(vr, vi, t, sg); break;
        case 4: cform_sub<1, (1 << 0), tu_dz(0, 4), T>(vr, vi, t, sg); break;
        case 5: cform_sub<1, (1 << 0), tu_dz(0, 5), T>(vr, vi, t, sg); break;
        case 6: cform_sub<1, (1 << 0), tu_dz(0, 6), T>(vr, vi, t, sg); break;
        case 7: cform_sub<1, (1 << 0), tu_dz(0, 7), T>(vr, vi, t, sg); break;
        case 8: cform_sub<1, (1 << 1), tu_dz(1, 0), T>(vr, vi, t, sg); break;
        case 9: cform_sub<1, (1 << 1), tu_dz(1, 1), T>(vr, vi, t, sg); break;
        case 10: cform_sub<1, (1 << 1), tu_dz(1, 2), T>(vr, vi, t, sg); break;
        case 11: cform_sub<1, (1 << 1), tu_dz(1, 3), T>(vr, vi, t, sg); break;
        case 12: cform_sub<1, (1 << 1), tu_dz(1, 4), T>(vr, vi, t, sg); break;
        case 13: cform_sub<1, (1 << 1), tu_dz(1, 5), T>(vr, vi, t, sg); break;
        case 14: cform_sub<1, (1 << 1), tu_dz(1, 6), T>(vr, vi, t, sg); break;
        case 15: cform_sub<1, (1 << 1), tu_dz(1, 7), T>(vr, vi, t, sg); break;
        default: break;
        }
        break;
    case 4:
        switch (ucase & 15u) {
        case 0: cform_sub<1, (1 << 2), tu_dz(2, 0), T>(vr, vi, t, sg); break;
        case 1: cform_sub<1, (1 << 2), tu_dz(2, 1), T>(vr, vi, t, sg); break;
        case 2: cform_sub<1, (1 << 2), tu_dz(2, 2), T>(vr, vi, t, sg); break;
        case 3: cform_sub<1, (1 << 2), tu_dz(2, 3), T>(vr, vi, t, sg); break;
        case 4: cform_sub<1, (1 << 2), tu_dz(2, 4), T>(vr, vi, t, sg); break;
        case 5: cform_sub<1, (1 << 2), tu_dz(2, 5), T>(vr, vi, t, sg); break;
        case 6: cform_sub<1, (1 << 2), tu_dz(2, 6), T>(vr, vi, t, sg); break;
        case 7: cform_sub<1, (1 << 2), tu_dz(2, 7), T>(vr, vi, t, sg); break;
        case 8: cform_sub<1, (1 << 3), tu_dz(3, 0), T>(vr, vi, t, sg); break;
        case 9: cform_sub<1, (1 << 3), tu_dz(3, 1), T>(vr, vi, t, sg); break;
        case 10: cform_sub<1, (1 << 3), tu_dz(3, 2), T>(vr, vi, t, sg); break;
        case 11: cform_sub<1, (1 << 3), tu_dz(3, 3), T>(vr, vi, t, sg); break;
        case 12: cform_sub<1, (1 << 3), tu_dz(3, 4), T>(vr, vi, t, sg); break;
        case 13: cform_sub<1, (1 << 3), tu_dz(3, 5), T>(vr, vi, t, sg); break;
        case 14: cform_sub<1, (1 << 3), tu_dz(3, 6), T>(vr, vi, t, sg); break;
        case 15: cform_sub<1, (1 << 3), tu_dz(3, 7), T>(vr, vi, t, sg); break;
        default: break;
        }
        break;
    default: break;
    }
}
#else
template <typename T>
__device__ __forceinline__ void unit_dispatch(T (&vr)[kSubAmps], T (&vi)[kSubAmps], uint32_t ucase, T t, T sg) {
    switch (ucase) {
        PS_UD(0) PS_UD(1) PS_UD(2) PS_UD(3) PS_UD(4) PS_UD(5) PS_UD(6) PS_UD(7)
        PS_UD(8) PS_UD(9) PS_UD(10) PS_UD(11) PS_UD(12) PS_UD(13) PS_UD(14) PS_UD(15)
        PS_UC8(0, 0) PS_UC8(0, 1) PS_UC8(0, 2)
        PS_UC8(1, 0) PS_UC8(1, 1) PS_UC8(1, 2)
#if PS_SUBDIM >= 4
        PS_UC8(0, 3) PS_UC8(1, 3)
#endif
    default: break;
    }
}
#endif

// applies the rotations [rb, rb + nr) of a sub-group to the thread's 16 registers; the next
// record is fetched while the current one is applied.  SPEC = 0: generic (one switch on dx, the
// per-pair signs from M at run time); SPEC = 1: CFORM rotations through the specialised cases.
// applies the rotations [rb, rb + nr) of a sub-group to the thread's 16 registers; the next
// record is fetched while the current one is applied.  SPEC = 0: generic (one switch on dx, the
// per-pair signs from M at run time); SPEC = 1: unit-dx CFORM rotations through the compile-time
// cases.  (Decoding rotation q + 1 -- sign, coefficient, case -- before rotation q's updates was
// measured 3-10 % slower: profiles/r02/kernel_ab.md section 5.)
template <typename T, int SPEC, int PARAM = 0>
__device__ __forceinline__ void sub_apply(T (&vr)[kSubAmps], T (&vi)[kSubAmps], const DevTRot* __restrict__ trots,
                                          int rb, int nr, uint32_t r, uint64_t i0) {
    if (nr <= 0) return;
    const DevTRot* tr = trots + rb;
    uint4 h = ldr<PARAM>(reinterpret_cast<const uint4*>(tr));
    double pn = ldr<PARAM>(&tr->p);
#if PS_SHEAR
    double sn = ldr<PARAM>(&tr->s);
#else
    constexpr double sn = 0.0;
#endif
    for (int q = 0; q < nr; ++q) {
        const uint32_t code = h.x, zr = h.y;
        const uint64_t zt_c = ((uint64_t)h.w << 32) | h.z;
        const double pc = pn, sc = sn;
        if (q + 1 < nr) {
            const DevTRot* tn = trots + rb + q + 1;
            h = ldr<PARAM>(reinterpret_cast<const uint4*>(tn));
            pn = ldr<PARAM>(&tn->p);
#if PS_SHEAR
            sn = ldr<PARAM>(&tn->s);
#endif
        }
        const int s0 = par32(zr & r) ^ par64(zt_c & i0);
        if (SPEC && (code & kTrUnit)) {
            // the thread-wide sign flips t once; the per-pair signs are static
            unit_dispatch<T>(vr, vi, code & 0x7fu, flip((T)pc, s0), flip((T)sc, s0));
        } else {
            uint32_t Ms = (code >> 16) ^ (s0 ? 0xffffu : 0u);
            if (code & kTrNeg) Ms ^= 0xffffu;
            const uint32_t dx = (code >> 8) & 15u;
#if PS_SHEAR
            if (code & kTrUnit) {
                shear_rotation<T>(vr, vi, dx, (code & kTrReal) ? 1 : 0, Ms, (T)pc, (T)sc);
                continue;
            }
#endif
            switch (((code & kTrReal) ? 1u : 0u) | ((code & kTrSform) ? 2u : 0u)) {
            case 0: sub_rotation<0, 0, T>(vr, vi, dx, Ms, (T)pc); break;
            case 1: sub_rotation<1, 0, T>(vr, vi, dx, Ms, (T)pc); break;
            case 2: sub_rotation<0, 1, T>(vr, vi, dx, Ms, (T)pc); break;
            default: sub_rotation<1, 1, T>(vr, vi, dx, Ms, (T)pc); break;
            }
        }
    }
}

template <typename T>
__device__ __forceinline__ void sub_scale(T (&vr)[kSubAmps], T (&vi)[kSubAmps], T F) {
#pragma unroll
    for (int d = 0; d < kSubAmps; ++d) {
        vr[d] = pmul(vr[d], F);
        vi[d] = pmul(vi[d], F);
    }
}

struct SubHdr {
    uint32_t u[kSubDim];
    uint32_t r;  // this thread's coset representative
    int rb, nr;
    double F;
};

// the thread's coset representative r = xor of col[b] over the set bits b of its thread index
template <int PARAM = 0>
__device__ __forceinline__ uint32_t sub_rep(const DevSub* __restrict__ sp, uint32_t tid, int ncols) {
    uint32_t r = 0;
#pragma unroll
    for (int b = 0; b < kMaxCols; ++b)
        if (b < ncols && ((tid >> b) & 1u)) r ^= (uint32_t)ldr<PARAM>(&sp->col[b]);
    return r;
}

template <int PARAM = 0>
__device__ __forceinline__ SubHdr load_sub_hdr(const DevSub* __restrict__ sp) {
    SubHdr h;
#pragma unroll
    for (int b = 0; b < kSubDim; ++b) h.u[b] = ldr<PARAM>(&sp->u[b]);
    h.rb = ldr<PARAM>(&sp->rot_begin);
    h.nr = ldr<PARAM>(&sp->nrot);
    h.F = ldr<PARAM>(&sp->F);
    h.r = 0;
    return h;
}

template <int PARAM = 0>
__device__ __forceinline__ SubHdr load_sub(const DevSub* __restrict__ sp, uint32_t tid, int ncols) {
    SubHdr h = load_sub_hdr<PARAM>(sp);
    h.r = sub_rep<PARAM>(sp, tid, ncols);
    return h;
}

__device__ __forceinline__ uint32_t sub_local(const SubHdr& h, int d) {
    uint32_t l = h.r;
#pragma unroll
    for (int b = 0; b < kSubDim; ++b)
        if ((d >> b) & 1) l ^= h.u[b];
    return l;
}

// global indices of the thread's 16 elements l_d = r xor U(d): the map l -> i0 xor off[l >> c] xor
// (l & cmask) is GF(2)-linear in l (off[] enumerates a span, chunk bits and free bits are
// disjoint), so gi[d] = gi[d without its lowest bit] xor Lin(u_lowest): one 64-bit xor each
__host__ __device__ constexpr int lowbit_index(int d) { return (d & 1) ? 0 : (d & 2) ? 1 : (d & 4) ? 2 : 3; }

// IDX = uint32_t when every local index fits 32 bits (n_local <= 32): one 32-bit xor per element
// and one wide multiply-add for the address instead of two 64-bit ops each
template <typename IDX = uint64_t>
__device__ __forceinline__ void elem_index(IDX (&gi)[kSubAmps], const SubHdr& h, uint64_t i0,
                                           const uint64_t* soff, int cbits, uint32_t cmask) {
    IDX E[kSubDim];
#pragma unroll
    for (int b = 0; b < kSubDim; ++b) E[b] = (IDX)soff[h.u[b] >> cbits] ^ (IDX)(h.u[b] & cmask);
    gi[0] = (IDX)i0 ^ (IDX)soff[h.r >> cbits] ^ (IDX)(h.r & cmask);
#pragma unroll
    for (int d = 1; d < kSubAmps; ++d) gi[d] = gi[d & (d - 1)] ^ E[lowbit_index(d)];
}

__device__ __forceinline__ double2 ld_l2_256(const double2* p) {
    double2 v;
    asm volatile("ld.global.L1::no_allocate.L2::256B.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ float2 ld_l2_256(const float2* p) {
    float2 v;
    asm volatile("ld.global.L1::no_allocate.L2::256B.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
    return v;
}

// one amplitude HBM -> shared memory without a register round trip (LDGSTS), L2 256-B sector hint
__device__ __forceinline__ void cp_async_amp(double2* dst, const double2* src) {
    asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_amp(float2* dst, const float2* src) {
    asm volatile("cp.async.ca.shared.global.L2::256B [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}

template <typename T>
struct SmemAmp;
template <>
struct SmemAmp<double> {
    using V = double2;
};
template <>
struct SmemAmp<float> {
    using V = float2;
};

// free_mask as maximal runs of consecutive set bits: i0 = pdep(tau, free_mask) in a few ops per run
struct BitRuns {
    uint32_t n;
    uint8_t pos[32];
    uint8_t len[32];
};

BitRuns make_runs(uint64_t mask) {
    BitRuns r{};
    int q = 0;
    while (mask >> q) {
        if (!((mask >> q) & 1)) {
            ++q;
            continue;
        }
        int l = 0;
        while (q + l < 64 && ((mask >> (q + l)) & 1)) ++l;
        r.pos[r.n] = (uint8_t)q;
        r.len[r.n] = (uint8_t)l;
        ++r.n;
        q += l;
    }
    return r;
}

__device__ __forceinline__ uint64_t deposit(uint64_t tau, const BitRuns& runs) {
    uint64_t out = 0;
    for (uint32_t k = 0; k < runs.n; ++k) {
        const uint32_t l = runs.len[k];
        out |= (tau & ((1ull << l) - 1)) << runs.pos[k];
        tau >>= l;
    }
    return out;
}

__device__ __forceinline__ uint64_t pdep64(uint64_t v, uint64_t mask) {
    uint64_t out = 0;
    for (uint64_t m = mask; m; m &= m - 1) {
        const uint64_t low = m & (~m + 1);
        if (v & 1) out |= low;
        v >>= 1;
    }
    return out;
}

// ------------------------------------------------------------------------------------------
// K2 / K7 (default): register-direct coset tile pass.
//
// tile tau: i0 = pdep(tau, free_mask); tile-local index l = (u << c) | w <-> global index
// i0 ^ off[u] | w (chunk u of 2^c contiguous amplitudes).  Sub-group 0 gathers its 16
// amplitudes per thread straight from HBM (consecutive threads own consecutive tile-local
// indices, so each warp load covers contiguous 256-B chunks), the last sub-group scatters
// straight back; shared memory holds the tile only between sub-groups.

#ifndef PS_COSET_THREADS
#define PS_COSET_THREADS 256
#endif
constexpr int kCosetThreads = PS_COSET_THREADS;  // 2^12 fp64 tiles: 256 threads x 16 amplitudes

// chunk-offset table size in shared memory, rounded up so the tile that follows is 128-B aligned
__host__ __device__ inline size_t coset_off_bytes(int hbits) {
    return ((sizeof(uint64_t) << hbits) + 127) & ~(size_t)127;
}

// per-thread coset representatives (tile-local, 16 bits) of the first rep_tab sub-groups, computed
// once per CTA (fp64 only: at 8 CTAs per SM the fp32 kernel loses more to the extra shared memory
// than it saves)
__host__ __device__ constexpr int rep_tab(size_t amp_bytes) { return amp_bytes == 16 ? 32 : 0; }

// dynamic shared memory of the register-direct tile kernels: tile (at offset 0, so element
// addresses are plain byte offsets) | representatives | chunk offsets
__host__ __device__ inline size_t coset_rep_bytes(int kbits, size_t amp_bytes) {
    return (((size_t)rep_tab(amp_bytes) << (kbits - kSubDim)) * sizeof(uint16_t) + 127) & ~(size_t)127;
}
__host__ __device__ inline size_t coset_smem_bytes(int kbits, int cbits, size_t amp_bytes) {
    return (amp_bytes << kbits) + coset_rep_bytes(kbits, amp_bytes) + coset_off_bytes(kbits - cbits);
}

// shared-memory byte offsets of the thread's 16 elements l_d = r xor U(d): o_d = o_(d without its
// lowest bit) xor (u_lowest << log2 amp bytes) -- one xor each (the tile sits at offset 0)
template <int LB>
__device__ __forceinline__ void smem_offsets(uint32_t (&o)[kSubAmps], const SubHdr& h) {
    o[0] = h.r << LB;
#pragma unroll
    for (int d = 1; d < kSubAmps; ++d) o[d] = o[d & (d - 1)] ^ (h.u[lowbit_index(d)] << LB);
}

// per-tile handshake flags of the fused exchange (system scope: the partner is another GPU)
__device__ __forceinline__ void flag_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t flag_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// the fused exchange + tile pass (K8, XT = 1): this rank's view of the exchange E(gx, ell)
struct XtArgs {
    const void* peer;        // the partner's slice
    uint32_t* flags;         // raised by the partner: it has read its tile tau of my slots
    uint32_t* peer_flags;    // raised by me for the partner
    uint64_t lbit, keepbit;  // 2^ell and keep * 2^ell
    uint64_t dtau, dtau_dep; // tile-index offset of 2^ell (tau space) and its deposit
    uint32_t epoch, cta, ncta;
};

template <typename T, int SPEC, int PARAM, typename IDX = uint64_t, int XT = 0>
__device__ __forceinline__ void coset_body(T* __restrict__ a, int kbits, int cbits, const BitRuns& runs,
                                           const uint64_t* __restrict__ offs, uint64_t ntiles,
                                           const DevSub* __restrict__ subs, int nsub, const DevTRot* __restrict__ trots,
                                           int l2_prefetch, uint64_t or_mask, uint64_t free_mask,
                                           const XtArgs& xt = XtArgs{}) {
    using V2 = typename SmemAmp<T>::V;
    constexpr int LB = sizeof(V2) == 16 ? 4 : 3;  // log2 bytes per amplitude
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int hbits = kbits - cbits;
    V2* tile = reinterpret_cast<V2*>(smem_raw);
    uint16_t* rtab = reinterpret_cast<uint16_t*>(smem_raw + (sizeof(V2) << kbits));
    uint64_t* soff = reinterpret_cast<uint64_t*>(smem_raw + (sizeof(V2) << kbits) + coset_rep_bytes(kbits, sizeof(V2)));
    const uint32_t tid = threadIdx.x;
    const uint32_t nthr = blockDim.x;
    const uint32_t cmask = (1u << cbits) - 1u;
    const int ncols = kbits - kSubDim;
    for (uint32_t u = tid; u < (1u << hbits); u += nthr) soff[u] = __ldg(&offs[u]);
    // representatives depend on (sub-group, thread) only: once per CTA (each thread reads its own)
    constexpr int kRepTab = rep_tab(sizeof(V2));
    for (int s = 0; s < nsub && s < kRepTab; ++s) rtab[s * nthr + tid] = (uint16_t)sub_rep<PARAM>(subs + s, tid, ncols);
    __syncthreads();
    auto rep = [&](int s) -> uint32_t {
        if (kRepTab > 0 && s < kRepTab) return rtab[s * nthr + tid];
        return sub_rep<PARAM>(subs + s, tid, ncols);
    };
    V2* g = reinterpret_cast<V2*>(a);
    // XT: the element of new slot j lives in my slot j (bit ell of j == keep) or in the partner's
    // slot j ^ 2^ell; the rank with keep = 1 walks tile tau ^ dtau (see k_xtile)
    const V2* gp = reinterpret_cast<const V2*>(xt.peer);
    auto src = [&](uint64_t gi) -> const V2* {
        if (XT && (gi & xt.lbit) != xt.keepbit) return gp + (gi ^ xt.lbit);
        return g + gi;
    };
    const uint32_t cta0 = XT ? xt.cta : blockIdx.x, ncta = XT ? xt.ncta : gridDim.x;
    const uint64_t xorD = XT && xt.keepbit ? xt.dtau_dep : 0, xorT = XT && xt.keepbit ? xt.dtau : 0;
    // tile bases advance in the deposited domain: pdep(tau + G) = ((pdep(tau) | ~M) + pdep(G)) & M
    const uint64_t dstep = deposit((uint64_t)ncta, runs);
    uint64_t dtau = deposit((uint64_t)cta0, runs);
    // tune bit 11 (l2_prefetch & 8): sub-group 0 of the CTA's next tile is copied HBM -> shared
    // memory (LDGSTS, one slot per thread and element) as soon as this tile's last sub-group has
    // its inputs in registers, so the next tile's reads are in flight while this one is computed
    // and stored; sub-group 0 then reads its own slots instead of HBM
    const bool pf = XT || (l2_prefetch & 8) != 0;
    auto prefetch_tile = [&](uint64_t i1) {
        SubHdr h0 = load_sub_hdr<PARAM>(subs);
        h0.r = rep(0);
        IDX gi[kSubAmps];
        elem_index<IDX>(gi, h0, i1, soff, cbits, cmask);
#pragma unroll
        for (int d = 0; d < kSubAmps; ++d) cp_async_amp(&tile[d * nthr + tid], src(gi[d]));
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (pf && cta0 < ntiles) prefetch_tile((dtau ^ xorD) | or_mask);
    for (uint64_t tau = cta0; tau < ntiles; tau += ncta, dtau = ((dtau | ~free_mask) + dstep) & free_mask) {
        const uint64_t i0 = (dtau ^ xorD) | or_mask;
        const uint64_t tau_x = tau ^ xorT;  // this tile's index (flag slot)
        T vr[kSubAmps], vi[kSubAmps];
        for (int s = 0; s < nsub; ++s) {
            SubHdr h = load_sub_hdr<PARAM>(subs + s);
            h.r = rep(s);
            if (s == 0 && pf) {
                asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
                for (int d = 0; d < kSubAmps; ++d) {
                    const V2 v = tile[d * nthr + tid];
                    vr[d] = v.x;
                    vi[d] = v.y;
                }
            } else if (s == 0) {
                IDX gi[kSubAmps];
                elem_index<IDX>(gi, h, i0, soff, cbits, cmask);
                V2 v[kSubAmps];
                if (l2_prefetch & 4) {
#pragma unroll
                    for (int d = 0; d < kSubAmps; ++d) v[d] = ld_l2_256(src(gi[d]));
                } else {
#pragma unroll
                    for (int d = 0; d < kSubAmps; ++d) v[d] = __ldcs(src(gi[d]));
                }
#pragma unroll
                for (int d = 0; d < kSubAmps; ++d) {
                    vr[d] = v[d].x;
                    vi[d] = v[d].y;
                }
            } else {
                uint32_t o[kSubAmps];
                smem_offsets<LB>(o, h);
#pragma unroll
                for (int d = 0; d < kSubAmps; ++d) {
                    const V2 v = *reinterpret_cast<const V2*>(smem_raw + o[d]);
                    vr[d] = v.x;
                    vi[d] = v.y;
                }
            }
            if (pf && (s == 0 || s == nsub - 1)) {
                if (XT && s == 0) {
                    // every thread has its (partly remote) inputs of this tile: the partner may now
                    // overwrite its slots that this tile read
                    __syncthreads();
                    if (tid == 0) flag_release(xt.peer_flags + tau_x, xt.epoch);
                }
                if (XT && s == nsub - 1 && tid == 0) {
                    // before any store of this tile: the partner has read its tile holding my slots
                    uint32_t spins = 0;
                    while (flag_acquire(xt.flags + (tau_x ^ xt.dtau)) != xt.epoch) {
                        __nanosleep(64);
                        if (++spins > (1u << 28)) __trap();
                    }
                }
                // every thread's shared-memory reads of this sub-group are done before the slots
                // (s == 0) or the tile (last sub-group) are overwritten
                __syncthreads();
                if (s == nsub - 1 && tau + ncta < ntiles)
                    prefetch_tile(((((dtau | ~free_mask) + dstep) & free_mask) ^ xorD) | or_mask);
            }
            sub_apply<T, SPEC, PARAM>(vr, vi, trots, h.rb, h.nr, h.r, i0);
            if (h.F != 1.0) sub_scale<T>(vr, vi, (T)h.F);
            if (s == nsub - 1) {
                IDX gi[kSubAmps];
                elem_index<IDX>(gi, h, i0, soff, cbits, cmask);
#pragma unroll
                for (int d = 0; d < kSubAmps; ++d) {
                    V2 v;
                    v.x = vr[d];
                    v.y = vi[d];
                    __stcs(&g[gi[d]], v);
                }
            } else {
                uint32_t o[kSubAmps];
                smem_offsets<LB>(o, h);
#pragma unroll
                for (int d = 0; d < kSubAmps; ++d) {
                    V2 v;
                    v.x = vr[d];
                    v.y = vi[d];
                    *reinterpret_cast<V2*>(smem_raw + o[d]) = v;
                }
                __syncthreads();
            }
        }
        if (nsub > 1 && !pf) __syncthreads();  // last sub-group's shared reads before the next tile's writes
    }
}

template <typename T, int MAXT, int MINB, int SPEC>
__global__ void __launch_bounds__(MAXT, MINB)
    k_coset(T* __restrict__ a, int kbits, int cbits, const __grid_constant__ BitRuns runs, const uint64_t* __restrict__ offs,
            uint64_t ntiles, const DevSub* __restrict__ subs, int nsub, const DevTRot* __restrict__ trots,
            int l2_prefetch, uint64_t or_mask, uint64_t free_mask) {
    coset_body<T, SPEC, 0>(a, kbits, cbits, runs, offs, ntiles, subs, nsub, trots, l2_prefetch, or_mask, free_mask);
}

// the pass's records in the parameter block (passes of <= kParamRots rotations in <= kParamSubs
// sub-groups; 15.4 KB of the 32 KB parameter space): record reads become uniform constant-bank
// loads instead of two LDGs per rotation and thread
constexpr int kParamRots = 256, kParamSubs = 128;
struct PassRecs {
    DevSub subs[kParamSubs];
    DevTRot trots[kParamRots];
};

template <typename T, int MAXT, int MINB, int SPEC = 0, int NARROW = 0>
__global__ void __launch_bounds__(MAXT, MINB)
    k_coset_p(T* __restrict__ a, int kbits, int cbits, const __grid_constant__ BitRuns runs,
              const uint64_t* __restrict__ offs, uint64_t ntiles, int nsub, int l2_prefetch, uint64_t or_mask,
              uint64_t free_mask, const __grid_constant__ PassRecs recs) {
    using IDX = typename std::conditional<NARROW != 0, uint32_t, uint64_t>::type;
    coset_body<T, SPEC, 1, IDX>(a, kbits, cbits, runs, offs, ntiles, recs.subs, nsub, recs.trots, l2_prefetch,
                                or_mask, free_mask);
}

// ------------------------------------------------------------------------------------------
// K8 k_xtile: fused half-vector exchange + tile pass (NEXT-2; api.cpp exchange_fused).  The pass
// runs in the layout AFTER the exchange E(gx, ell): a rank with keep = k finds the element of its
// new slot j in its own slot j (bit ell of j == k) or in the partner's slot j ^ 2^ell.  Each tile's
// sub-group 0 gathers straight from both (remote loads through the peer pointer); the CTA then
// raises the partner's flag for this tile (release, system scope), and before its last sub-group
// stores -- into its own slots, some of which the partner still has to read -- it waits until the
// partner has raised this rank's flag for the partner's tile holding those slots (acquire).  The
// rank with keep = 1 walks tile tau ^ dtau where the other walks tau (dtau: tile-index offset of
// 2^ell), so CTA c of both ranks always waits on CTA c of the other in the same round (no
// deadlock with co-resident grids).  Several ranks (an emulation group) run as one launch:
// blockIdx.x / ctas_per_rank selects the rank.

constexpr int kMaxXRanks = 8;
struct XTileParams {
    XTileRank r[kMaxXRanks];
    BitRuns runs;
    const uint64_t* offs;
    uint64_t ntiles, free_mask, dtau, dtau_dep;
    int nranks, ctas_per_rank, kbits, cbits, nsub, ell;
    uint32_t epoch;
};

template <typename T, int SPEC>
__global__ void __launch_bounds__(kCosetThreads, 2) k_xtile(const __grid_constant__ XTileParams P) {
    const int rk = blockIdx.x / P.ctas_per_rank;
    const XTileRank& R = P.r[rk];
    XtArgs xa;
    xa.peer = R.peer;
    xa.flags = R.flags;
    xa.peer_flags = R.peer_flags;
    xa.lbit = 1ull << P.ell;
    xa.keepbit = (uint64_t)R.keep << P.ell;
    xa.dtau = P.dtau;
    xa.dtau_dep = P.dtau_dep;
    xa.epoch = P.epoch;
    xa.cta = blockIdx.x % P.ctas_per_rank;
    xa.ncta = P.ctas_per_rank;
    // the tile kernel's body with the partner's half gathered through the peer pointer, the
    // LDGSTS next-tile prefetch (remote elements included) and the per-tile handshake
    coset_body<T, SPEC, 0, uint64_t, 1>(reinterpret_cast<T*>(R.a), P.kbits, P.cbits, P.runs, P.offs, P.ntiles, R.subs,
                                        P.nsub, R.trots, 4, 0, P.free_mask, xa);
}

// ------------------------------------------------------------------------------------------
// K2 / K7 (default): TMA-prefetched coset tile pass.  Each persistent CTA double-buffers tiles in
// shared memory: while the sub-groups of tile m run on buffer m&1 (in place, the last one storing
// straight to HBM), the TMA engine fills buffer (m+1)&1 with tile m+1 -- one cp.async.bulk per
// 2^c-amplitude chunk, issued by all threads, completion on an mbarrier (complete_tx).

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
    }
}

template <typename T, int CPASYNC>
__global__ void __launch_bounds__(kCosetThreads, 2)
    k_coset_pf(T* __restrict__ a, int kbits, int cbits, uint64_t free_mask, const uint64_t* __restrict__ offs,
               uint64_t ntiles, const DevSub* __restrict__ subs, int nsub, const DevTRot* __restrict__ trots) {
    using V2 = typename SmemAmp<T>::V;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t mbar[2];
    const int hbits = kbits - cbits;
    const uint32_t tile_bytes = (uint32_t)(2 * sizeof(T)) << kbits;
    const uint32_t chunk_bytes = (uint32_t)(2 * sizeof(T)) << cbits;
    const uint32_t nchunks = 1u << hbits;
    uint64_t* soff = reinterpret_cast<uint64_t*>(smem_raw);
    unsigned char* bufs = smem_raw + coset_off_bytes(hbits);
    const uint32_t tid = threadIdx.x;
    const uint32_t cmask = (1u << cbits) - 1u;
    const uint64_t my_tiles = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    for (uint32_t u = tid; u < nchunks; u += blockDim.x) soff[u] = __ldg(&offs[u]);
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&mbar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&mbar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto prefetch = [&](uint64_t m) {
        const uint64_t i0 = pdep64((uint64_t)blockIdx.x + m * gridDim.x, free_mask);
        const int b = (int)(m & 1);
        unsigned char* dst = bufs + (size_t)b * tile_bytes;
        if (CPASYNC) {
            // 16-byte cp.async (LDGSTS) units: one fp64 amplitude or two fp32 amplitudes
            constexpr uint32_t per = 16 / (2 * sizeof(T));
            const uint32_t units = (1u << kbits) / per;
            for (uint32_t q = tid; q < units; q += blockDim.x) {
                const uint32_t l = q * per;
                const T* src = a + 2 * ((i0 ^ soff[l >> cbits]) | (l & cmask));
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst + (size_t)q * 16)),
                             "l"(src)
                             : "memory");
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
            return;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (tid == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&mbar[b])),
                         "r"(tile_bytes)
                         : "memory");
        for (uint32_t u = tid; u < nchunks; u += blockDim.x) {
            const T* src = a + 2 * (i0 ^ soff[u]);
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_addr(dst + (size_t)u * chunk_bytes)),
                "l"(src), "r"(chunk_bytes), "r"(smem_addr(&mbar[b]))
                : "memory");
        }
    };
    V2* g = reinterpret_cast<V2*>(a);
    if (my_tiles > 0) prefetch(0);
    for (uint64_t m = 0; m < my_tiles; ++m) {
        const bool more = m + 1 < my_tiles;
        if (more) prefetch(m + 1);  // buffer (m+1)&1 was released by the barrier ending tile m-1
        const int b = (int)(m & 1);
        if (CPASYNC) {
            if (more)
                asm volatile("cp.async.wait_group 1;" ::: "memory");
            else
                asm volatile("cp.async.wait_group 0;" ::: "memory");
            __syncthreads();
        } else {
            mbar_wait_parity(&mbar[b], (uint32_t)((m >> 1) & 1));
        }
        V2* tile = reinterpret_cast<V2*>(bufs + (size_t)b * tile_bytes);
        const uint64_t i0 = pdep64((uint64_t)blockIdx.x + m * gridDim.x, free_mask);
        for (int s = 0; s < nsub; ++s) {
            const SubHdr h = load_sub(subs + s, tid, kbits - kSubDim);
            T vr[kSubAmps], vi[kSubAmps];
#pragma unroll
            for (int d = 0; d < kSubAmps; ++d) {
                const V2 v = tile[sub_local(h, d)];
                vr[d] = v.x;
                vi[d] = v.y;
            }
            sub_apply<T, 0>(vr, vi, trots, h.rb, h.nr, h.r, i0);
            if (h.F != 1.0) sub_scale<T>(vr, vi, (T)h.F);
            if (s == nsub - 1) {
#pragma unroll
                for (int d = 0; d < kSubAmps; ++d) {
                    const uint32_t l = sub_local(h, d);
                    V2 v;
                    v.x = vr[d];
                    v.y = vi[d];
                    __stcs(&g[(i0 ^ soff[l >> cbits]) | (l & cmask)], v);
                }
            } else {
#pragma unroll
                for (int d = 0; d < kSubAmps; ++d) {
                    V2 v;
                    v.x = vr[d];
                    v.y = vi[d];
                    tile[sub_local(h, d)] = v;
                }
            }
            __syncthreads();
        }
    }
}

// ------------------------------------------------------------------------------------------
// K2 / K7 (TMA variant): persistent CTAs walk tiles through a 3-stage shared-memory ring filled
// and drained by TMA bulk copies (cp.async.bulk, mbarrier complete_tx; bulk stores with
// bulk_group read-completion before a stage is refilled); every sub-group goes through shared
// memory.

constexpr int kStages = 3;
constexpr int kTileMaxThreads = 512;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}

template <typename T>
__global__ void __launch_bounds__(kTileMaxThreads, 1)
    k_tile(T* __restrict__ a, int kbits, int cbits, uint64_t free_mask, const uint64_t* __restrict__ offs,
           uint64_t ntiles, const DevSub* __restrict__ subs, int nsub, const DevTRot* __restrict__ trots) {
    using V2 = typename SmemAmp<T>::V;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t mbar[kStages];
    const uint32_t tile_amps = 1u << kbits;
    const uint32_t tile_bytes = tile_amps * (uint32_t)(2 * sizeof(T));
    const uint32_t nchunks = 1u << (kbits - cbits);
    const uint32_t chunk_bytes = (uint32_t)(2 * sizeof(T)) << cbits;
    const uint32_t tid = threadIdx.x;
    const uint32_t lane = tid & 31u;
    const bool issuer = tid < 32;
    const uint32_t wmask = blockDim.x >= 32 ? 0xffffffffu : ((1u << blockDim.x) - 1u);
    const uint64_t my_tiles = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    auto stage_ptr = [&](int st) { return reinterpret_cast<T*>(smem_raw + (size_t)st * tile_bytes); };

    if (tid == 0) {
        for (int st = 0; st < kStages; ++st)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar[st])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    auto issue_load = [&](uint64_t m) {
        const uint64_t i0 = pdep64((uint64_t)blockIdx.x + m * gridDim.x, free_mask);
        const int st = (int)(m % kStages);
        T* buf = stage_ptr(st);
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&mbar[st])),
                         "r"(tile_bytes)
                         : "memory");
        __syncwarp(wmask);
        for (uint32_t u = lane; u < nchunks; u += 32) {
            const T* src = a + 2 * (i0 ^ __ldg(&offs[u]));
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(buf + 2 * ((size_t)u << cbits))),
                "l"(src), "r"(chunk_bytes), "r"(smem_u32(&mbar[st]))
                : "memory");
        }
    };
    auto issue_store = [&](uint64_t m) {
        const uint64_t i0 = pdep64((uint64_t)blockIdx.x + m * gridDim.x, free_mask);
        T* buf = stage_ptr((int)(m % kStages));
        for (uint32_t u = lane; u < nchunks; u += 32) {
            T* dst = a + 2 * (i0 ^ __ldg(&offs[u]));
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                         "r"(smem_u32(buf + 2 * ((size_t)u << cbits))), "r"(chunk_bytes)
                         : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    };

    if (issuer && my_tiles > 0) issue_load(0);
    for (uint64_t m = 0; m < my_tiles; ++m) {
        const int st = (int)(m % kStages);
        if (issuer && m + 1 < my_tiles) {
            // stage (m+1)%3 last held tile m-2, whose store group is the older of the two pending
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            __syncwarp(wmask);
            issue_load(m + 1);
        }
        mbar_wait(&mbar[st], (uint32_t)((m / kStages) & 1));
        const uint64_t i0 = pdep64((uint64_t)blockIdx.x + m * gridDim.x, free_mask);
        V2* buf = reinterpret_cast<V2*>(stage_ptr(st));
        for (int s = 0; s < nsub; ++s) {
            const SubHdr h = load_sub(subs + s, tid, kbits - kSubDim);
            T vr[kSubAmps], vi[kSubAmps];
#pragma unroll
            for (int d = 0; d < kSubAmps; ++d) {
                const V2 v = buf[sub_local(h, d)];
                vr[d] = v.x;
                vi[d] = v.y;
            }
            sub_apply<T, 0>(vr, vi, trots, h.rb, h.nr, h.r, i0);
            if (h.F != 1.0) sub_scale<T>(vr, vi, (T)h.F);
#pragma unroll
            for (int d = 0; d < kSubAmps; ++d) {
                V2 v;
                v.x = vr[d];
                v.y = vi[d];
                buf[sub_local(h, d)] = v;
            }
            __syncthreads();
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (issuer) issue_store(m);
    }
    if (issuer) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ------------------------------------------------------------------------------------------
// K3 fallback: own element i (local index base+t) updated against the partner's OLD value at
// local index i ^ x, held in `stage` (partner chunk starting at local index pbase):
//   a'_i = c a_i + sigma A b_(i^x)   (the first half of the pair update)

template <typename T>
__global__ void k_full_update(T* __restrict__ a, const T* __restrict__ stage, uint64_t base,
                              uint64_t count, uint64_t pbase, const DevRot* __restrict__ rec) {
    const uint64_t x = __ldg(&rec->x);
    const uint64_t z = __ldg(&rec->z);
    const RotK<T> k = load_rot<T>(rec);
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = base + t;
        const uint64_t j = (i ^ x) - pbase;
        const T b = flip(k.b, par64(z & i));
        T ir = a[2 * i], ii = a[2 * i + 1];
        T jr = stage[2 * j], ji = stage[2 * j + 1];
        if (k.real)
            rot_pair<1>(ir, ii, jr, ji, k.c, b);
        else
            rot_pair<0>(ir, ii, jr, ji, k.c, b);
        a[2 * i] = ir;
        a[2 * i + 1] = ii;
    }
}

// ------------------------------------------------------------------------------------------
// reductions (fp64 accumulation, deterministic two-stage)

constexpr int kRedThreads = 256;

__device__ __forceinline__ double block_sum(double v) {
    __shared__ double sh[kRedThreads / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = v;
    __syncthreads();
    double s = 0.0;
    if (w == 0) {
        s = (l < kRedThreads / 32) ? sh[l] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    }
    __syncthreads();
    return s;
}

// The reductions read the state once with 256-bit vector loads (V amplitudes per load: 2 fp64,
// 4 fp32; V = 1 below V amplitudes), accumulate in fp64 per thread in a fixed order and sum per
// block (deterministic two-stage sums).  HBM-bound: algorithmic bytes = the bytes read.
template <typename T, int V>
__global__ void __launch_bounds__(kRedThreads) k_norm(const T* __restrict__ a, uint64_t n, double* partial) {
    double acc = 0.0;
    const uint64_t units = n / V;
    for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < units; u += (uint64_t)gridDim.x * blockDim.x) {
        Vec<T, V> v;
        ld_vec<T, V>(a + 2 * u * V, v);
#pragma unroll
        for (int e = 0; e < V; ++e) {
            const double r = (double)v.r[e], m = (double)v.i[e];
            acc = __fma_rn(r, r, __fma_rn(m, m, acc));
        }
    }
    const double s = block_sum(acc);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

template <typename T, int V>
__global__ void __launch_bounds__(kRedThreads) k_inner(const T* __restrict__ a, const T* __restrict__ b, uint64_t n,
                                                       double* partial) {
    double re = 0.0, im = 0.0;
    const uint64_t units = n / V;
    for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < units; u += (uint64_t)gridDim.x * blockDim.x) {
        Vec<T, V> va, vb;
        ld_vec<T, V>(a + 2 * u * V, va);
        ld_vec<T, V>(b + 2 * u * V, vb);
#pragma unroll
        for (int e = 0; e < V; ++e) {
            const double ar = (double)va.r[e], ai = (double)va.i[e];
            const double br = (double)vb.r[e], bi = (double)vb.i[e];
            re = __fma_rn(ar, br, __fma_rn(ai, bi, re));
            im = __fma_rn(ar, bi, __fma_rn(-ai, br, im));
        }
    }
    const double s0 = block_sum(re);
    const double s1 = block_sum(im);
    if (threadIdx.x == 0) {
        partial[2 * blockIdx.x] = s0;
        partial[2 * blockIdx.x + 1] = s1;
    }
}

// the terms of one x-group at pair (i, j = i ^ x0): sum_l sigma_l(i) (kr_l tr + ki_l ti), t = conj(a_j) a_i
__device__ __forceinline__ double expect_pair(double ir, double ii, double jr, double ji, uint64_t i,
                                              const DevTerm* __restrict__ terms, int nt) {
    const double tr = __fma_rn(jr, ir, __dmul_rn(ji, ii));
    const double ti = __fma_rn(jr, ii, __dmul_rn(-ji, ir));
    double acc = 0.0;
    for (int l = 0; l < nt; ++l) {
        const double v = __fma_rn(__ldg(&terms[l].kr), tr, __dmul_rn(__ldg(&terms[l].ki), ti));
        acc += par64(__ldg(&terms[l].z) & i) ? -v : v;
    }
    return acc;
}

// expectation over one x-group: terms[0..nt) share xor mask x0
template <typename T, int V>
__global__ void __launch_bounds__(kRedThreads) k_expect(const T* __restrict__ a, uint64_t nl_amps, uint64_t x0,
                                                        const DevTerm* __restrict__ terms, int nt,
                                                        double* partial) {
    double acc = 0.0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x0 == 0) {
        for (uint64_t u = t0; u < nl_amps / V; u += stride) {
            Vec<T, V> v;
            ld_vec<T, V>(a + 2 * u * V, v);
#pragma unroll
            for (int e = 0; e < V; ++e) {
                const uint64_t i = u * V + e;
                const double r = (double)v.r[e], m = (double)v.i[e];
                const double p = __fma_rn(r, r, __dmul_rn(m, m));
                double w = 0.0;
                for (int l = 0; l < nt; ++l) {
                    const double kr = __ldg(&terms[l].kr);
                    w += par64(__ldg(&terms[l].z) & i) ? -kr : kr;
                }
                acc = __fma_rn(w, p, acc);
            }
        }
    } else if ((1ull << (63 - __clzll(x0))) >= (uint64_t)V) {
        // pairs across vectors: the i-vector has bit piv clear, its partners are the vector at
        // ib ^ (x0 without its in-vector bits), permuted by xin
        const int piv = 63 - __clzll(x0);
        const uint64_t xv = x0 & ~(uint64_t)(V - 1);
        const int xin = (int)(x0 & (V - 1));
        for (uint64_t u = t0; u < (nl_amps >> 1) / V; u += stride) {
            const uint64_t ib = insert0(u * V, piv);
            Vec<T, V> vi, vj;
            ld_vec<T, V>(a + 2 * ib, vi);
            ld_vec<T, V>(a + 2 * (ib ^ xv), vj);
#pragma unroll
            for (int e = 0; e < V; ++e)
                acc += expect_pair((double)vi.r[e], (double)vi.i[e], (double)vj.r[e ^ xin], (double)vj.i[e ^ xin], ib + e,
                                   terms, nt);
        }
    } else {
        // pairs inside one vector (x0 < V)
        const int piv = 63 - __clzll(x0);
        for (uint64_t u = t0; u < nl_amps / V; u += stride) {
            Vec<T, V> v;
            ld_vec<T, V>(a + 2 * u * V, v);
#pragma unroll
            for (int e = 0; e < V; ++e) {
                if ((e >> piv) & 1) continue;
                const int f = e ^ (int)x0;
                acc += expect_pair((double)v.r[e], (double)v.i[e], (double)v.r[f], (double)v.i[f], u * V + e, terms, nt);
            }
        }
    }
    const double s = block_sum(acc);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// sums partial[0..n) (stride `width`, component `comp`) in a fixed order into out[comp]
__global__ void k_final_sum(const double* __restrict__ partial, int n, int width, int comp, double* out) {
    double acc = 0.0;
    for (int t = threadIdx.x; t < n; t += blockDim.x) acc += partial[(size_t)t * width + comp];
    const double s = block_sum(acc);
    if (threadIdx.x == 0) out[comp] = s;
}

// ------------------------------------------------------------------------------------------
// init

__device__ __forceinline__ double gen_u(uint64_t seed, uint64_t k) {
    // splitmix64 output k+1 for state `seed`, top 53 bits -> [-1, 1)
    uint64_t zz = seed + (k + 1) * 0x9E3779B97F4A7C15ull;
    zz = (zz ^ (zz >> 30)) * 0xBF58476D1CE4E5B9ull;
    zz = (zz ^ (zz >> 27)) * 0x94D049BB133111EBull;
    zz = zz ^ (zz >> 31);
    return (double)(zz >> 11) * (1.0 / 4503599627370496.0) - 1.0;
}

template <typename T>
__global__ void k_init_random(T* __restrict__ a, uint64_t n, uint64_t seed, uint64_t goff) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t g = goff + i;
        a[2 * i] = (T)gen_u(seed, 2 * g);
        a[2 * i + 1] = (T)gen_u(seed, 2 * g + 1);
    }
}

template <typename T>
__global__ void k_set_one(T* __restrict__ a, uint64_t idx) {
    a[2 * idx] = (T)1;
    a[2 * idx + 1] = (T)0;
}

template <typename T>
__global__ void k_scale(T* __restrict__ a, uint64_t n, double f) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 2 * n; i += (uint64_t)gridDim.x * blockDim.x)
        a[i] = (T)((double)a[i] * f);
}

// local transposition of bits b1 < b2: swap a[i] <-> a[i ^ (2^b1 | 2^b2)] for bit b1 = 0, b2 = 1
template <typename T>
__global__ void k_permute(T* __restrict__ a, uint64_t quarter, int b1, int b2) {
    using V2 = typename SmemAmp<T>::V;
    V2* g = reinterpret_cast<V2*>(a);
    const uint64_t m = (1ull << b1) | (1ull << b2);
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < quarter; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = insert0(insert0(t, b1), b2) | (1ull << b2);
        const uint64_t j = i ^ m;
        const V2 u = g[i], v = g[j];
        g[i] = v;
        g[j] = u;
    }
}

// NVLink P2P half swap: local region element e (row, col) <-> the partner's matching element.
// Elements are enumerated as e = t with the filter bits (fmask, fval) inserted (fmask = 0: every
// element; else one piece of the region, for the swap/compute overlap), t in [t0, t1).
template <typename T>
__device__ __forceinline__ void swap_index(uint64_t tq, uint64_t row_amps, uint64_t my_off, uint64_t peer_off,
                                           uint64_t fmask, uint64_t fval, uint64_t& li, uint64_t& ri) {
    uint64_t e = tq;
    for (uint64_t m = fmask; m; m &= m - 1) {
        const int b = __ffsll((long long)m) - 1;
        e = insert0(e, b) | (fval & (1ull << b));
    }
    const uint64_t row = e / row_amps, col = e - row * row_amps;
    li = row * 2 * row_amps + my_off + col;
    ri = row * 2 * row_amps + peer_off + col;
}

// U elements in flight per thread (NVLink latency ~2 us).  The full-GPU form (512 threads, U = 8)
// runs alone; the overlap form (128 threads, U = 4, <= 64 registers) fits next to the tile kernel's
// two resident CTAs on every SM (their 2 x 256 x 112 registers leave 8192 = 128 x 64), so the swap
// really runs while the pass runs instead of waiting for whole SMs to drain.
template <typename T, int U, int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB)
k_p2p_swap(T* __restrict__ local, T* __restrict__ peer, uint64_t row_amps, uint64_t my_off,
           uint64_t peer_off, uint64_t t0, uint64_t t1, uint64_t fmask, uint64_t fval) {
    using V2 = typename SmemAmp<T>::V;
    V2* L = reinterpret_cast<V2*>(local);
    V2* R = reinterpret_cast<V2*>(peer);
    const uint64_t stride = (uint64_t)gridDim.x * THREADS;
    for (uint64_t t = t0 + (uint64_t)blockIdx.x * THREADS + threadIdx.x; t < t1; t += U * stride) {
        V2 u[U], v[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
            const uint64_t tq = t + (uint64_t)q * stride;
            if (tq < t1) {
                uint64_t li, ri;
                swap_index<T>(tq, row_amps, my_off, peer_off, fmask, fval, li, ri);
                u[q] = L[li];
                v[q] = __ldcv(&R[ri]);
            }
        }
#pragma unroll
        for (int q = 0; q < U; ++q) {
            const uint64_t tq = t + (uint64_t)q * stride;
            if (tq < t1) {
                uint64_t li, ri;
                swap_index<T>(tq, row_amps, my_off, peer_off, fmask, fval, li, ri);
                L[li] = v[q];
                __stcg(&R[ri], u[q]);
            }
        }
    }
    // the stores into the partner's memory are performed at system scope before this thread
    // retires (the NCCL barrier after the launch then orders them before the partner's next reads)
    __threadfence_system();
}

// TMA form of the overlapped swap: one warp per CTA, lane 0 moves chunks of `chunk_amps`
// contiguous elements (a run inside one region row and one piece) through a kSwapStages ring of
// shared memory: bulk-load the partner's chunk and the own chunk (cp.async.bulk, mbarrier
// complete_tx), then bulk-store them crosswise (bulk_group).  Loads run kSwapStages - 2 chunks
// ahead of the stores; a stage is refilled once its stores have read it.  No data passes through
// registers, so 24 KB per CTA are in flight with one thread and ~32 KB of shared memory -- it fits
// on an SM next to the tile kernel's two resident CTAs.
constexpr int kSwapStages = 4;

template <typename T>
__global__ void __launch_bounds__(32, 1)
k_p2p_swap_tma(T* __restrict__ local, T* __restrict__ peer, uint64_t row_amps, uint64_t my_off, uint64_t peer_off,
               uint64_t t0, uint64_t t1, uint64_t fmask, uint64_t fval, uint32_t chunk_amps) {
    using V2 = typename SmemAmp<T>::V;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t mbar[kSwapStages];
    if (threadIdx.x != 0) return;
    const uint32_t cbytes = chunk_amps * (uint32_t)sizeof(V2);
    for (int st = 0; st < kSwapStages; ++st)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar[st])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    V2* L = reinterpret_cast<V2*>(local);
    V2* R = reinterpret_cast<V2*>(peer);
    const uint64_t nch = (t1 - t0) / chunk_amps;
    const uint64_t mine = nch > blockIdx.x ? (nch - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    auto addr = [&](uint64_t m, V2*& lp, V2*& rp) {
        uint64_t li, ri;
        swap_index<T>(t0 + (blockIdx.x + m * gridDim.x) * (uint64_t)chunk_amps, row_amps, my_off, peer_off, fmask,
                      fval, li, ri);
        lp = L + li;
        rp = R + ri;
    };
    // stage st: [partner's chunk | own chunk]
    auto sbuf = [&](int st, int w) { return smem_raw + ((size_t)(2 * st + w)) * cbytes; };
    constexpr int D = kSwapStages - 2;  // loads ahead of stores
    for (uint64_t m = 0; m < mine + D; ++m) {
        if (m < mine) {
            const int st = (int)(m % kSwapStages);
            // stage st last held chunk m - kSwapStages, whose stores were committed two iterations
            // ago: at most one newer store group may still be reading shared memory
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            V2 *lp, *rp;
            addr(m, lp, rp);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&mbar[st])),
                         "r"(2 * cbytes)
                         : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(sbuf(st, 0))),
                "l"(rp), "r"(cbytes), "r"(smem_u32(&mbar[st]))
                : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(sbuf(st, 1))),
                "l"(lp), "r"(cbytes), "r"(smem_u32(&mbar[st]))
                : "memory");
        }
        if (m >= (uint64_t)D) {
            const uint64_t j = m - D;
            const int st = (int)(j % kSwapStages);
            mbar_wait(&mbar[st], (uint32_t)((j / kSwapStages) & 1));
            V2 *lp, *rp;
            addr(j, lp, rp);
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(lp),
                         "r"(smem_u32(sbuf(st, 0))), "r"(cbytes)
                         : "memory");
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(rp),
                         "r"(smem_u32(sbuf(st, 1))), "r"(cbytes)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    // every store complete (not only read out of shared memory), then system scope for the partner
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __threadfence_system();
}

// pairwise barrier between two ranks over peer memory (the overlapped swap's "both ranks finished
// piece j" / "both halves landed" points): one thread raises the partner's word to `epoch` (system-
// scope release, after this stream's earlier kernels completed) and spins until its own word from
// the partner reaches `epoch` (acquire).  One warp with a few registers: it fits on an SM next to the
// tile kernel's resident CTAs, where an NCCL collective kernel would wait for a whole SM to drain.
// A partner that never arrives traps after ~60 s instead of hanging the GPU.
__global__ void k_pair_barrier(const uint32_t* mine, uint32_t* theirs, uint32_t epoch) {
    if (threadIdx.x != 0) return;
    flag_release(theirs, epoch);
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    uint32_t spins = 0;
    while ((int32_t)(flag_acquire(mine) - epoch) < 0) {
        __nanosleep(256);
        if ((++spins & 1023u) == 0) {
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > 60ull * 1000000000ull) __trap();
        }
    }
}

// Eq. (core_state) helpers (PS_OPT_LAYOUT=2)
// butterfly: b = w B (w = conj(w_k) in {+-1, +-i}); A <- (A + b)/sqrt2, B <- (A - b)/sqrt2
template <typename T>
__global__ void k_butterfly(T* __restrict__ A, T* __restrict__ B, uint64_t n, int wr, int wi) {
    const T h = (T)0.70710678118654752440;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const T ar = A[2 * i], ai = A[2 * i + 1], xr = B[2 * i], xi = B[2 * i + 1];
        const T br = (T)wr * xr - (T)wi * xi, bi = (T)wr * xi + (T)wi * xr;  // exact: w in {+-1, +-i}
        A[2 * i] = (ar + br) * h;
        A[2 * i + 1] = (ai + bi) * h;
        B[2 * i] = (ar - br) * h;
        B[2 * i + 1] = (ai - bi) * h;
    }
}

template <typename T>
__global__ void k_recombine(T* __restrict__ A, const T* __restrict__ B, uint64_t n) {
    const T h = (T)0.70710678118654752440;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 2 * n; i += (uint64_t)gridDim.x * blockDim.x)
        A[i] = (A[i] + B[i]) * h;
}

// dst <- peer's slice (NVLink reads through a CUDA-IPC pointer)
template <typename T>
__global__ void k_p2p_copy(T* __restrict__ dst, const T* __restrict__ src, uint64_t n) {
    using V2 = typename SmemAmp<T>::V;
    V2* d = reinterpret_cast<V2*>(dst);
    const V2* r = reinterpret_cast<const V2*>(src);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        d[i] = __ldcv(&r[i]);
}

int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev & 63;
}

// test knob (PS_OPT_GRID_CAP): caps the persistent tile grid so small states run several tiles per
// CTA (the incremental tile bases and the next-tile prefetch); 0 = no cap
thread_local int t_grid_cap = 0;
uint64_t apply_grid_cap(uint64_t cap) { return (t_grid_cap > 0 && (uint64_t)t_grid_cap < cap) ? (uint64_t)t_grid_cap : cap; }

int g_num_sms = 0;
int num_sms() {
    if (g_num_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    return g_num_sms;
}

template <typename T, int V>
cudaError_t launch_stream_t(T* a, int nl, const Pass& p, const DevRot* d_rots, cudaStream_t s) {
    const DevRot* rec = d_rots + p.rot_begin;
    int mode, piv = 0;
    uint64_t units;
    const uint64_t namps = 1ull << nl;
    if (p.x0 == 0) {
        mode = 2;
        units = namps / V;
    } else {
        piv = highest_bit(p.x0);
        if ((1ull << piv) >= (uint64_t)V) {
            mode = 0;
            units = (namps >> 1) / V;
        } else {
            mode = 1;
            units = namps / V;
        }
    }
    constexpr int UNROLL = 2;
    const uint64_t want = (units + (uint64_t)kStreamThreads * UNROLL - 1) / ((uint64_t)kStreamThreads * UNROLL);
    const uint64_t cap = (uint64_t)num_sms() * 8;
    const unsigned grid = (unsigned)(want < cap ? (want ? want : 1) : cap);
    k_stream<T, V, UNROLL><<<grid, kStreamThreads, 0, s>>>(a, units, mode, piv, p.x0, rec, p.rot_count);
    return cudaGetLastError();
}

template <typename T, int MAXT, int MINB, int SPEC>
cudaError_t launch_coset_k(T* a, int nl, const Pass& p, const DevSub* d_subs, const DevTRot* d_trots,
                           const uint64_t* d_offs, int l2_prefetch, int grid_mult, cudaStream_t s) {
    const size_t smem = coset_smem_bytes(p.kbits, p.cbits, 2 * sizeof(T));
    static uint64_t attr_devices = 0;  // function attributes are per device
    const int dev = current_device();
    if (!((attr_devices >> dev) & 1)) {
        cudaFuncSetAttribute(k_coset<T, MAXT, MINB, SPEC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_devices |= 1ull << dev;
    }
    const int threads = 1 << (p.kbits - kSubDim);
    if (threads > MAXT) return cudaErrorInvalidValue;
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_coset<T, MAXT, MINB, SPEC>, threads, smem);
    if (occ < 1) occ = 1;
    const uint64_t ntiles = 1ull << __builtin_popcountll(p.free_mask);  // == 2^(nl - kbits) unless split
    const uint64_t cap = apply_grid_cap((uint64_t)num_sms() * (uint64_t)occ * (uint64_t)(grid_mult > 0 ? grid_mult : 1));
    const unsigned grid = (unsigned)(ntiles < cap ? ntiles : cap);
    k_coset<T, MAXT, MINB, SPEC><<<grid, threads, smem, s>>>(a, p.kbits, p.cbits, make_runs(p.free_mask),
                                                              d_offs + p.off_begin, ntiles, d_subs + p.sub_begin,
                                                              p.sub_count, d_trots, l2_prefetch, p.or_mask, p.free_mask);
    return cudaGetLastError();
}

// occupancy variants: tune bits 1..3 (>> 1) select the register cap for 128-thread CTAs
template <typename T>
cudaError_t launch_coset_t(T* a, int nl, const Pass& p, const DevSub* d_subs, const DevTRot* d_trots,
                           const uint64_t* d_offs, int l2_prefetch, int grid_mult, int occ_sel, cudaStream_t s) {
    const int threads = 1 << (p.kbits - kSubDim);
    // occ_sel 0 = per-dtype default: fp32 tiles hold half the bytes, so 8 CTAs per SM (64
    // registers) keep more bytes in flight (+7 % at 30q); fp64 spills under any cap
    if (occ_sel == 0 && sizeof(T) == 4 && !p.spec) occ_sel = 3;
    if (threads <= 128 && !p.spec && occ_sel == 3)
        return launch_coset_k<T, 128, 8, 0>(a, nl, p, d_subs, d_trots, d_offs, l2_prefetch, grid_mult, s);
    if constexpr (sizeof(T) == 4)
        if (threads == 256 && !p.spec && occ_sel == 3)  // fp32 2^12 tiles (default): 4 CTAs x 64 registers
            return launch_coset_k<T, 256, 4, 0>(a, nl, p, d_subs, d_trots, d_offs, l2_prefetch, grid_mult, s);
    // tiles of 2^13 (fp64) / 2^13..2^14 (fp32) amplitudes: one CTA of 512 / 1024 threads per SM
    if (threads == 512)
        return launch_coset_k<T, 512, 1, 0>(a, nl, p, d_subs, d_trots, d_offs, l2_prefetch, grid_mult, s);
    if constexpr (sizeof(T) == 4)
        if (threads == 1024)
            return launch_coset_k<T, 1024, 1, 0>(a, nl, p, d_subs, d_trots, d_offs, l2_prefetch, grid_mult, s);
    if (threads > kCosetThreads) return cudaErrorInvalidValue;
#ifndef PS_ONLY_DEFAULT  // (development builds: the default kernels only, fast to compile)
    if (threads <= 128 && !p.spec && occ_sel == 1) return launch_coset_k<T, 128, 5, 0>(a, nl, p, d_subs, d_trots, d_offs, l2_prefetch, grid_mult, s);
    if (threads <= 128 && !p.spec && occ_sel == 2) return launch_coset_k<T, 128, 6, 0>(a, nl, p, d_subs, d_trots, d_offs, l2_prefetch, grid_mult, s);
#endif
#ifndef PS_COSET_MINB
#define PS_COSET_MINB 2
#endif
    if (p.spec && threads <= kCosetThreads)
        return launch_coset_k<T, kCosetThreads, PS_COSET_MINB, 1>(a, nl, p, d_subs, d_trots, d_offs, l2_prefetch, grid_mult, s);
    return launch_coset_k<T, kCosetThreads, PS_COSET_MINB, 0>(a, nl, p, d_subs, d_trots, d_offs, l2_prefetch, grid_mult, s);
}

// the pass's records in the launch's parameter block (tune bit 10; passes of <= kParamRots
// rotations); cudaErrorNotSupported when the pass does not fit
template <typename T, int MAXT, int MINB, int SPEC = 0, int NARROW = 0>
cudaError_t launch_coset_param_k(T* a, const Pass& p, const PassRecs& recs, const uint64_t* d_offs, int l2_prefetch,
                                 int grid_mult, cudaStream_t s) {
    const size_t smem = coset_smem_bytes(p.kbits, p.cbits, 2 * sizeof(T));
    static uint64_t attr_devices = 0;
    const int dev = current_device();
    if (!((attr_devices >> dev) & 1)) {
        cudaFuncSetAttribute(k_coset_p<T, MAXT, MINB, SPEC, NARROW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_devices |= 1ull << dev;
    }
    const int threads = 1 << (p.kbits - kSubDim);
    if (threads > MAXT) return cudaErrorNotSupported;
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_coset_p<T, MAXT, MINB, SPEC, NARROW>, threads, smem);
    if (occ < 1) occ = 1;
    const uint64_t ntiles = 1ull << __builtin_popcountll(p.free_mask);
    const uint64_t cap = apply_grid_cap((uint64_t)num_sms() * (uint64_t)occ * (uint64_t)(grid_mult > 0 ? grid_mult : 1));
    const unsigned grid = (unsigned)(ntiles < cap ? ntiles : cap);
    k_coset_p<T, MAXT, MINB, SPEC, NARROW><<<grid, threads, smem, s>>>(a, p.kbits, p.cbits, make_runs(p.free_mask), d_offs + p.off_begin,
                                                          ntiles, p.sub_count, l2_prefetch, p.or_mask, p.free_mask,
                                                          recs);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_coset_param(T* a, int nl, const Pass& p, const DevSub* h_subs, const DevTRot* h_trots,
                               const uint64_t* d_offs, int l2_prefetch, int grid_mult, int occ_sel, cudaStream_t s) {
    if (p.sub_count < 1 || p.sub_count > kParamSubs) return cudaErrorNotSupported;
    const int base = h_subs[p.sub_begin].rot_begin;
    int nrot = 0;
    for (int t = 0; t < p.sub_count; ++t) nrot += h_subs[p.sub_begin + t].nrot;
    if (nrot > kParamRots) return cudaErrorNotSupported;
    static thread_local PassRecs recs;
    for (int t = 0; t < p.sub_count; ++t) {
        recs.subs[t] = h_subs[p.sub_begin + t];
        recs.subs[t].rot_begin -= base;
    }
    for (int q = 0; q < nrot; ++q) recs.trots[q] = h_trots[base + q];
    const int threads = 1 << (p.kbits - kSubDim);
    // fp32: the default kernels with 32-bit element indices when every local index fits (n_local <=
    // 32): +0.8 %; fp64 keeps 64-bit indices (the 32-bit build takes 128 registers: -1 % R10, -2 % JW;
    // profiles/r02/kernel_ab.md section 6)
#ifdef PS_NO_NARROW
    const bool narrow = false;
#else
    const bool narrow = sizeof(T) == 4 && nl <= 32;
#endif
    if (p.spec && threads <= kCosetThreads) {
        if constexpr (sizeof(T) == 4) {
            if (occ_sel == 0 && threads <= 128)
                return narrow ? launch_coset_param_k<T, 128, 8, 1, 1>(a, p, recs, d_offs, l2_prefetch, grid_mult, s)
                              : launch_coset_param_k<T, 128, 8, 1>(a, p, recs, d_offs, l2_prefetch, grid_mult, s);
            if (occ_sel == 2 && threads <= 128)  // 6 CTAs per SM (85 registers): room for the 80 cases
                return launch_coset_param_k<T, 128, 6, 1>(a, p, recs, d_offs, l2_prefetch, grid_mult, s);
        }
        if (threads <= kCosetThreads) {
            if constexpr (sizeof(T) == 4)
                if (narrow)
                    return launch_coset_param_k<T, kCosetThreads, PS_COSET_MINB, 1, 1>(a, p, recs, d_offs, l2_prefetch,
                                                                                      grid_mult, s);
            return launch_coset_param_k<T, kCosetThreads, PS_COSET_MINB, 1>(a, p, recs, d_offs, l2_prefetch, grid_mult, s);
        }
        return cudaErrorNotSupported;
    }
    if constexpr (sizeof(T) == 4)
        if (occ_sel == 0 && threads <= 128)
            return narrow ? launch_coset_param_k<T, 128, 8, 0, 1>(a, p, recs, d_offs, l2_prefetch, grid_mult, s)
                          : launch_coset_param_k<T, 128, 8>(a, p, recs, d_offs, l2_prefetch, grid_mult, s);
    if constexpr (sizeof(T) == 4)
        if ((occ_sel == 0 || occ_sel == 3) && threads == 256)  // fp32 2^12 tiles (default): 4 CTAs x 64 registers
            return narrow ? launch_coset_param_k<T, 256, 4, 0, 1>(a, p, recs, d_offs, l2_prefetch, grid_mult, s)
                          : launch_coset_param_k<T, 256, 4>(a, p, recs, d_offs, l2_prefetch, grid_mult, s);
    if (threads == 512) return launch_coset_param_k<T, 512, 1>(a, p, recs, d_offs, l2_prefetch, grid_mult, s);
    if constexpr (sizeof(T) == 4)
        if (threads == 1024) return launch_coset_param_k<T, 1024, 1>(a, p, recs, d_offs, l2_prefetch, grid_mult, s);
    if constexpr (sizeof(T) == 4)
        if (narrow) return launch_coset_param_k<T, kCosetThreads, PS_COSET_MINB, 0, 1>(a, p, recs, d_offs, l2_prefetch, grid_mult, s);
    return launch_coset_param_k<T, kCosetThreads, PS_COSET_MINB>(a, p, recs, d_offs, l2_prefetch, grid_mult, s);
}

template <typename T, int CPASYNC>
cudaError_t launch_coset_pf_t(T* a, int nl, const Pass& p, const DevSub* d_subs, const DevTRot* d_trots,
                              const uint64_t* d_offs, cudaStream_t s) {
    const size_t smem = coset_off_bytes(p.kbits - p.cbits) + 2 * ((size_t)(2 * sizeof(T)) << p.kbits);
    static uint64_t attr_devices = 0;
    const int dev = current_device();
    if (!((attr_devices >> dev) & 1)) {
        cudaFuncSetAttribute(k_coset_pf<T, CPASYNC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_devices |= 1ull << dev;
    }
    const int threads = 1 << (p.kbits - kSubDim);
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_coset_pf<T, CPASYNC>, threads, smem);
    if (occ < 1) occ = 1;
    const uint64_t ntiles = 1ull << __builtin_popcountll(p.free_mask);  // == 2^(nl - kbits) unless split
    const uint64_t cap = (uint64_t)num_sms() * (uint64_t)occ;
    const unsigned grid = (unsigned)(ntiles < cap ? ntiles : cap);
    k_coset_pf<T, CPASYNC><<<grid, threads, smem, s>>>(a, p.kbits, p.cbits, p.free_mask, d_offs + p.off_begin, ntiles,
                                              d_subs + p.sub_begin, p.sub_count, d_trots);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_tile_t(T* a, int nl, const Pass& p, const DevSub* d_subs, const DevTRot* d_trots,
                          const uint64_t* d_offs, cudaStream_t s) {
    const size_t stage_bytes = (size_t)(2 * sizeof(T)) << p.kbits;
    const size_t smem = stage_bytes * kStages;
    static uint64_t attr_devices = 0;
    const int dev = current_device();
    if (!((attr_devices >> dev) & 1)) {
        cudaFuncSetAttribute(k_tile<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_devices |= 1ull << dev;
    }
    const int threads = 1 << (p.kbits - kSubDim);
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tile<T>, threads, smem);
    if (occ < 1) occ = 1;
    const uint64_t ntiles = 1ull << __builtin_popcountll(p.free_mask);  // == 2^(nl - kbits) unless split
    const uint64_t cap = (uint64_t)num_sms() * (uint64_t)occ;
    const unsigned grid = (unsigned)(ntiles < cap ? ntiles : cap);
    k_tile<T><<<grid, threads, smem, s>>>(a, p.kbits, p.cbits, p.free_mask, d_offs + p.off_begin, ntiles,
                                          d_subs + p.sub_begin, p.sub_count, d_trots);
    return cudaGetLastError();
}

uint64_t pdep_host(uint64_t v, uint64_t mask) {
    uint64_t out = 0;
    for (uint64_t m = mask; m; m &= m - 1, v >>= 1)
        if (v & 1) out |= m & (~m + 1);
    return out;
}

template <typename T, int SPEC>
cudaError_t launch_xtile_t(const XTileRank* ranks, int nranks, const Pass& p, const uint64_t* d_offs, int ell,
                           uint64_t dtau, uint32_t epoch, cudaStream_t s, int grid_cap) {
    if (nranks < 1 || nranks > kMaxXRanks) return cudaErrorInvalidValue;
    const int threads = 1 << (p.kbits - kSubDim);
    if (threads > kCosetThreads) return cudaErrorInvalidValue;
    const size_t smem = coset_smem_bytes(p.kbits, p.cbits, 2 * sizeof(T));
    static uint64_t attr_devices = 0;
    const int dev = current_device();
    if (!((attr_devices >> dev) & 1)) {
        cudaFuncSetAttribute(k_xtile<T, SPEC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_devices |= 1ull << dev;
    }
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_xtile<T, SPEC>, threads, smem);
    if (occ < 1) return cudaErrorInvalidConfiguration;
    // every CTA of the launch must be resident at once (CTAs wait on each other's flags)
    const uint64_t ntiles = 1ull << __builtin_popcountll(p.free_mask);
    uint64_t per = (uint64_t)num_sms() * (uint64_t)occ / (uint64_t)nranks;
    if (grid_cap > 0 && (uint64_t)grid_cap < per) per = (uint64_t)grid_cap;
    if (per > ntiles) per = ntiles;
    if (per < 1) return cudaErrorInvalidConfiguration;
    XTileParams P{};
    for (int k = 0; k < nranks; ++k) P.r[k] = ranks[k];
    P.runs = make_runs(p.free_mask);
    P.offs = d_offs;
    P.ntiles = ntiles;
    P.free_mask = p.free_mask;
    P.dtau = dtau;
    P.dtau_dep = pdep_host(dtau, p.free_mask);
    P.nranks = nranks;
    P.ctas_per_rank = (int)per;
    P.kbits = p.kbits;
    P.cbits = p.cbits;
    P.nsub = p.sub_count;
    P.ell = ell;
    P.epoch = epoch;
    void* args[] = {&P};
    return cudaLaunchCooperativeKernel((const void*)k_xtile<T, SPEC>, dim3((unsigned)(per * nranks)), dim3(threads), args,
                                       smem, s);
}

template <typename T>
__global__ void __launch_bounds__(256) k_expect_cross(const T* __restrict__ a, const T* __restrict__ stage,
                                                      uint64_t base, uint64_t count, uint64_t pbase, uint64_t xl,
                                                      uint64_t zl, int y, int sgn, double* partial) {
    double acc = 0.0;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = base + t, j = (i ^ xl) - pbase;
        const double ar = (double)a[2 * i], ai = (double)a[2 * i + 1];
        const double br = (double)stage[2 * j], bi = (double)stage[2 * j + 1];
        // conj(b) a, then Re(i^y (.)) with the sign (-1)^popc(z & i)
        const double re = __fma_rn(br, ar, __dmul_rn(bi, ai)), im = __fma_rn(br, ai, __dmul_rn(-bi, ar));
        const double v = y == 0 ? re : y == 1 ? -im : y == 2 ? -re : im;
        acc += (par64(zl & i) ^ sgn) ? -v : v;
    }
    const double s = block_sum(acc);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

unsigned red_grid(uint64_t n) {
    const uint64_t want = (n + kRedThreads - 1) / kRedThreads;
    const uint64_t cap = (uint64_t)num_sms() * 4;
    return (unsigned)(want < cap ? (want ? want : 1) : cap);
}

}  // namespace

// ==========================================================================================
// launchers (host)

int kernel_max_red_blocks() { return num_sms() * 4; }

cudaError_t launch_stream(int dtype, void* a, int nl, const Pass& p, const DevRot* d_rots, int vec256,
                          cudaStream_t s) {
    if (dtype == PS_C128) {
        if (vec256 && nl >= 2) return launch_stream_t<double, 2>((double*)a, nl, p, d_rots, s);
        return launch_stream_t<double, 1>((double*)a, nl, p, d_rots, s);
    }
    if (vec256 && nl >= 3) return launch_stream_t<float, 4>((float*)a, nl, p, d_rots, s);
    if (nl >= 2) return launch_stream_t<float, 2>((float*)a, nl, p, d_rots, s);
    return launch_stream_t<float, 1>((float*)a, nl, p, d_rots, s);
}

cudaError_t launch_tile(int dtype, void* a, int nl, const Pass& p, const DevSub* d_subs, const DevTRot* d_trots,
                        const uint64_t* d_offs, int use_tma, int tune, cudaStream_t s, const DevSub* h_subs,
                        const DevTRot* h_trots, int grid_cap) {
    t_grid_cap = grid_cap;
    // tune: bit 0 = L2 prefetch of the next tile (register-direct kernel); bits 4.. = grid multiplier
    // bit 0: TMA bulk L2 prefetch; bit 8: per-thread L2 prefetch; bit 9: L2::256B load hint
    // bit 11: LDGSTS prefetch of the next tile's first sub-group into shared memory
    const int l2p = ((tune >> 7) & 4) | ((tune >> 8) & 8);
    const int occ_sel = (tune >> 1) & 7;
    const int gm = ((tune >> 4) & 15) ? ((tune >> 4) & 15) : 4;
    if (use_tma == 2 && (tune & 1024) && h_subs) {
        cudaError_t e = dtype == PS_C128
                            ? launch_coset_param<double>((double*)a, nl, p, h_subs, h_trots, d_offs, l2p, gm, occ_sel, s)
                            : launch_coset_param<float>((float*)a, nl, p, h_subs, h_trots, d_offs, l2p, gm, occ_sel, s);
        if (e != cudaErrorNotSupported) return e;
    }
    if (use_tma == 2) {
        if (dtype == PS_C128) return launch_coset_t<double>((double*)a, nl, p, d_subs, d_trots, d_offs, l2p, gm, occ_sel, s);
        return launch_coset_t<float>((float*)a, nl, p, d_subs, d_trots, d_offs, l2p, gm, occ_sel, s);
    }
#ifdef PS_ONLY_DEFAULT
    return cudaErrorNotSupported;
#else
    if (use_tma == 1) {
        if (dtype == PS_C128) return launch_tile_t<double>((double*)a, nl, p, d_subs, d_trots, d_offs, s);
        return launch_tile_t<float>((float*)a, nl, p, d_subs, d_trots, d_offs, s);
    }
    if (use_tma == 3) {
        if (dtype == PS_C128) return launch_coset_pf_t<double, 0>((double*)a, nl, p, d_subs, d_trots, d_offs, s);
        return launch_coset_pf_t<float, 0>((float*)a, nl, p, d_subs, d_trots, d_offs, s);
    }
    if (dtype == PS_C128) return launch_coset_pf_t<double, 1>((double*)a, nl, p, d_subs, d_trots, d_offs, s);
    return launch_coset_pf_t<float, 1>((float*)a, nl, p, d_subs, d_trots, d_offs, s);
#endif
}

cudaError_t launch_full_update(int dtype, void* a, const void* stage, uint64_t base, uint64_t count, uint64_t pbase,
                               const DevRot* rec, cudaStream_t s) {
    const unsigned grid = red_grid(count);
    if (dtype == PS_C128)
        k_full_update<double><<<grid, kRedThreads, 0, s>>>((double*)a, (const double*)stage, base, count, pbase, rec);
    else
        k_full_update<float><<<grid, kRedThreads, 0, s>>>((float*)a, (const float*)stage, base, count, pbase, rec);
    return cudaGetLastError();
}

cudaError_t launch_norm(int dtype, const void* a, uint64_t n, double* d_partial, double* d_out, cudaStream_t s) {
    unsigned grid;
    if (dtype == PS_C128) {
        if (n >= 2) k_norm<double, 2><<<grid = red_grid(n / 2), kRedThreads, 0, s>>>((const double*)a, n, d_partial);
        else k_norm<double, 1><<<grid = red_grid(n), kRedThreads, 0, s>>>((const double*)a, n, d_partial);
    } else {
        if (n >= 4) k_norm<float, 4><<<grid = red_grid(n / 4), kRedThreads, 0, s>>>((const float*)a, n, d_partial);
        else k_norm<float, 1><<<grid = red_grid(n), kRedThreads, 0, s>>>((const float*)a, n, d_partial);
    }
    k_final_sum<<<1, kRedThreads, 0, s>>>(d_partial, (int)grid, 1, 0, d_out);
    return cudaGetLastError();
}

cudaError_t launch_inner(int dtype, const void* a, const void* b, uint64_t n, double* d_partial, double* d_out,
                         cudaStream_t s) {
    unsigned grid;
    if (dtype == PS_C128) {
        if (n >= 2) k_inner<double, 2><<<grid = red_grid(n / 2), kRedThreads, 0, s>>>((const double*)a, (const double*)b, n, d_partial);
        else k_inner<double, 1><<<grid = red_grid(n), kRedThreads, 0, s>>>((const double*)a, (const double*)b, n, d_partial);
    } else {
        if (n >= 4) k_inner<float, 4><<<grid = red_grid(n / 4), kRedThreads, 0, s>>>((const float*)a, (const float*)b, n, d_partial);
        else k_inner<float, 1><<<grid = red_grid(n), kRedThreads, 0, s>>>((const float*)a, (const float*)b, n, d_partial);
    }
    k_final_sum<<<1, kRedThreads, 0, s>>>(d_partial, (int)grid, 2, 0, d_out);
    k_final_sum<<<1, kRedThreads, 0, s>>>(d_partial, (int)grid, 2, 1, d_out);
    return cudaGetLastError();
}

cudaError_t launch_expect(int dtype, const void* a, uint64_t n, uint64_t x0, const DevTerm* terms, int nt,
                          double* d_partial, double* d_out_slot, cudaStream_t s) {
    unsigned grid;
    if (dtype == PS_C128) {
        if (n >= 4) k_expect<double, 2><<<grid = red_grid(n / 2), kRedThreads, 0, s>>>((const double*)a, n, x0, terms, nt, d_partial);
        else k_expect<double, 1><<<grid = red_grid(n), kRedThreads, 0, s>>>((const double*)a, n, x0, terms, nt, d_partial);
    } else {
        if (n >= 8) k_expect<float, 4><<<grid = red_grid(n / 4), kRedThreads, 0, s>>>((const float*)a, n, x0, terms, nt, d_partial);
        else k_expect<float, 1><<<grid = red_grid(n), kRedThreads, 0, s>>>((const float*)a, n, x0, terms, nt, d_partial);
    }
    k_final_sum<<<1, kRedThreads, 0, s>>>(d_partial, (int)grid, 1, 0, d_out_slot);
    return cudaGetLastError();
}

cudaError_t launch_init_random(int dtype, void* a, uint64_t n, uint64_t seed, uint64_t goff, cudaStream_t s) {
    const unsigned grid = red_grid(n) * 2;
    if (dtype == PS_C128)
        k_init_random<double><<<grid, kRedThreads, 0, s>>>((double*)a, n, seed, goff);
    else
        k_init_random<float><<<grid, kRedThreads, 0, s>>>((float*)a, n, seed, goff);
    return cudaGetLastError();
}

cudaError_t launch_set_one(int dtype, void* a, uint64_t idx, cudaStream_t s) {
    if (dtype == PS_C128)
        k_set_one<double><<<1, 1, 0, s>>>((double*)a, idx);
    else
        k_set_one<float><<<1, 1, 0, s>>>((float*)a, idx);
    return cudaGetLastError();
}

cudaError_t launch_permute(int dtype, void* a, int nl, int b1, int b2, cudaStream_t s) {
    const uint64_t quarter = 1ull << (nl - 2);
    const unsigned grid = red_grid(quarter) * 2;
    if (b1 > b2) { const int t = b1; b1 = b2; b2 = t; }
    if (dtype == PS_C128)
        k_permute<double><<<grid, kRedThreads, 0, s>>>((double*)a, quarter, b1, b2);
    else
        k_permute<float><<<grid, kRedThreads, 0, s>>>((float*)a, quarter, b1, b2);
    return cudaGetLastError();
}

cudaError_t launch_p2p_swap(int dtype, void* local, void* peer, uint64_t rows, uint64_t row_amps, uint64_t my_off,
                            uint64_t peer_off, uint64_t t0, uint64_t t1, uint64_t fmask, uint64_t fval, cudaStream_t s,
                            int ctas, int tma_chunk) {
    (void)rows;
    if (t1 <= t0) return cudaSuccess;
    // ctas > 0: that many full-size CTAs; 0: one full-size CTA per SM; < 0: the overlap form,
    // -ctas CTAs per SM if -ctas <= 8, else -ctas CTAs
    if (ctas >= 0) {
        const unsigned grid = ctas > 0 ? (unsigned)ctas : (unsigned)num_sms();
        if (dtype == PS_C128)
            k_p2p_swap<double, 8, 512, 1><<<grid, 512, 0, s>>>((double*)local, (double*)peer, row_amps, my_off,
                                                                peer_off, t0, t1, fmask, fval);
        else
            k_p2p_swap<float, 8, 512, 1><<<grid, 512, 0, s>>>((float*)local, (float*)peer, row_amps, my_off, peer_off,
                                                               t0, t1, fmask, fval);
    } else if (tma_chunk > 0) {
        // TMA form: chunk_amps contiguous elements per chunk, one 32-thread CTA per SM x (-ctas)
        const unsigned grid = -ctas <= 8 ? (unsigned)(-ctas * num_sms()) : (unsigned)(-ctas);
        const size_t amp = dtype == PS_C128 ? 16 : 8;
        const size_t smem = (size_t)2 * kSwapStages * (size_t)tma_chunk * amp;
        if (dtype == PS_C128)
            k_p2p_swap_tma<double><<<grid, 32, smem, s>>>((double*)local, (double*)peer, row_amps, my_off, peer_off,
                                                           t0, t1, fmask, fval, (uint32_t)tma_chunk);
        else
            k_p2p_swap_tma<float><<<grid, 32, smem, s>>>((float*)local, (float*)peer, row_amps, my_off, peer_off, t0,
                                                          t1, fmask, fval, (uint32_t)tma_chunk);
    } else {
        const unsigned grid = -ctas <= 8 ? (unsigned)(-ctas * num_sms()) : (unsigned)(-ctas);
        if (dtype == PS_C128)
            k_p2p_swap<double, 4, 128, 8><<<grid, 128, 0, s>>>((double*)local, (double*)peer, row_amps, my_off,
                                                                peer_off, t0, t1, fmask, fval);
        else
            k_p2p_swap<float, 4, 128, 8><<<grid, 128, 0, s>>>((float*)local, (float*)peer, row_amps, my_off, peer_off,
                                                               t0, t1, fmask, fval);
    }
    return cudaGetLastError();
}

cudaError_t launch_pair_barrier(const uint32_t* mine, uint32_t* theirs, uint32_t epoch, cudaStream_t s) {
    k_pair_barrier<<<1, 32, 0, s>>>(mine, theirs, epoch);
    return cudaGetLastError();
}

cudaError_t launch_butterfly(int dtype, void* A, void* B, uint64_t n, int wr, int wi, cudaStream_t s) {
    const unsigned grid = red_grid(n) * 2;
    if (dtype == PS_C128)
        k_butterfly<double><<<grid, kRedThreads, 0, s>>>((double*)A, (double*)B, n, wr, wi);
    else
        k_butterfly<float><<<grid, kRedThreads, 0, s>>>((float*)A, (float*)B, n, wr, wi);
    return cudaGetLastError();
}

cudaError_t launch_recombine(int dtype, void* A, const void* B, uint64_t n, cudaStream_t s) {
    const unsigned grid = red_grid(n) * 2;
    if (dtype == PS_C128)
        k_recombine<double><<<grid, kRedThreads, 0, s>>>((double*)A, (const double*)B, n);
    else
        k_recombine<float><<<grid, kRedThreads, 0, s>>>((float*)A, (const float*)B, n);
    return cudaGetLastError();
}

cudaError_t launch_p2p_copy(int dtype, void* dst, const void* src, uint64_t n, cudaStream_t s) {
    const unsigned grid = (unsigned)num_sms() * 4;
    if (dtype == PS_C128)
        k_p2p_copy<double><<<grid, 512, 0, s>>>((double*)dst, (const double*)src, n);
    else
        k_p2p_copy<float><<<grid, 512, 0, s>>>((float*)dst, (const float*)src, n);
    return cudaGetLastError();
}

cudaError_t launch_scale(int dtype, void* a, uint64_t n, double f, cudaStream_t s) {
    const unsigned grid = red_grid(n) * 2;
    if (dtype == PS_C128)
        k_scale<double><<<grid, kRedThreads, 0, s>>>((double*)a, n, f);
    else
        k_scale<float><<<grid, kRedThreads, 0, s>>>((float*)a, n, f);
    return cudaGetLastError();
}

// tile-index offset dtau of the coset T xor 2^ell (0 when 2^ell lies in the tile space): the unit
// vector reduced by the pass's gathered basis (RREF, pivot = highest bit) leaves free-mask bits only
static uint64_t xtile_dtau(const Pass& p, const uint64_t* h_offs, int ell) {
    if (ell < p.cbits) return 0;
    uint64_t e = 1ull << ell;
    for (int t = 0; t < p.hbits; ++t) {
        const uint64_t v = h_offs[1u << t];
        if (highest_bit(v) == ell) e ^= v;
    }
    e &= p.free_mask;
    uint64_t out = 0;
    int k = 0;
    for (uint64_t m = p.free_mask; m; m &= m - 1, ++k)
        if (e & m & (~m + 1)) out |= 1ull << k;
    return out;
}

cudaError_t launch_xtile(int dtype, const XTileRank* ranks, int nranks, const Pass& p, const uint64_t* d_offs,
                         const uint64_t* h_offs, int ell, uint32_t epoch, cudaStream_t s, int grid_cap) {
    if (p.or_mask) return cudaErrorInvalidValue;
    const uint64_t dtau = xtile_dtau(p, h_offs, ell);
    if (dtype == PS_C128)
        return p.spec ? launch_xtile_t<double, 1>(ranks, nranks, p, d_offs, ell, dtau, epoch, s, grid_cap)
                      : launch_xtile_t<double, 0>(ranks, nranks, p, d_offs, ell, dtau, epoch, s, grid_cap);
    return p.spec ? launch_xtile_t<float, 1>(ranks, nranks, p, d_offs, ell, dtau, epoch, s, grid_cap)
                  : launch_xtile_t<float, 0>(ranks, nranks, p, d_offs, ell, dtau, epoch, s, grid_cap);
}

cudaError_t launch_expect_cross(int dtype, const void* a, const void* stage, uint64_t base, uint64_t count,
                                uint64_t pbase, uint64_t xl, uint64_t zl, int y, int sgn, double* d_partial,
                                double* d_out_slot, cudaStream_t s) {
    const unsigned grid = red_grid(count);
    if (dtype == PS_C128)
        k_expect_cross<double><<<grid, kRedThreads, 0, s>>>((const double*)a, (const double*)stage, base, count, pbase,
                                                             xl, zl, y, sgn, d_partial);
    else
        k_expect_cross<float><<<grid, kRedThreads, 0, s>>>((const float*)a, (const float*)stage, base, count, pbase,
                                                            xl, zl, y, sgn, d_partial);
    k_final_sum<<<1, kRedThreads, 0, s>>>(d_partial, (int)grid, 1, 0, d_out_slot);
    return cudaGetLastError();
}

}  // namespace ps
