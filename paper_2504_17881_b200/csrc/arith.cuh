// arith.cuh -- the per-pair arithmetic every libps kernel uses (one definition, explicit
// round-to-nearest intrinsics, no contraction freedom), so fused and unfused passes and 1-GPU and
// G-GPU runs produce bitwise-identical amplitudes.
//
// exp(i phi P) = cos(phi) I + i sin(phi) P acts on each pair {i, j = i xor x} as
//     a'_i = c a_i + sigma A a_j,    a'_j = c a_j + sigma B a_i,    A = -conj(B)
// with B = sign sin(phi) i^(y+1) (ps_internal.h DevRot).  B is either real (B = b, A = -b) or
// imaginary (B = i b, A = i b); sigma = +-1 is folded into b by the caller.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace ps {

__device__ __forceinline__ double pmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float pmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double pfma(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float pfma(float a, float b, float c) { return __fmaf_rn(a, b, c); }

// REAL = 1: B = b;  REAL = 0: B = i b
template <int REAL, typename T>
__device__ __forceinline__ void rot_pair(T& ir, T& ii, T& jr, T& ji, T c, T b) {
    if (REAL) {
        const T p0 = pmul(b, jr), p1 = pmul(b, ji), p2 = pmul(b, ir), p3 = pmul(b, ii);
        const T nir = pfma(c, ir, -p0), nii = pfma(c, ii, -p1);
        const T njr = pfma(c, jr, p2), nji = pfma(c, ji, p3);
        ir = nir; ii = nii; jr = njr; ji = nji;
    } else {
        const T p0 = pmul(b, ji), p1 = pmul(b, jr), p2 = pmul(b, ii), p3 = pmul(b, ir);
        const T nir = pfma(c, ir, -p0), nii = pfma(c, ii, p1);
        const T njr = pfma(c, jr, -p2), nji = pfma(c, ji, p3);
        ir = nir; ii = nii; jr = njr; ji = nji;
    }
}

// diagonal element update a' = c a + A a (x = 0 strings have y = 0: B = i b, A = i b)
template <int REAL, typename T>
__device__ __forceinline__ void rot_diag(T& r, T& i, T c, T b) {
    if (REAL) {
        const T p0 = pmul(b, r), p1 = pmul(b, i);
        r = pfma(c, r, -p0);
        i = pfma(c, i, -p1);
    } else {
        const T p0 = pmul(b, i), p1 = pmul(b, r);
        const T nr = pfma(c, r, -p0), ni = pfma(c, i, p1);
        r = nr;
        i = ni;
    }
}

// exact sign flip when neg == 1: one LOP3 on the high word (no select, no DADD)
__device__ __forceinline__ double flip(double v, int neg) {
    return __hiloint2double(__double2hiint(v) ^ (int)((unsigned)neg << 31), __double2loint(v));
}
__device__ __forceinline__ float flip(float v, int neg) {
    return __int_as_float(__float_as_int(v) ^ (int)((unsigned)neg << 31));
}

__device__ __forceinline__ int par64(uint64_t v) { return __popcll(v) & 1; }
__device__ __forceinline__ int par32(uint32_t v) { return __popc(v) & 1; }

__device__ __forceinline__ uint64_t insert0(uint64_t t, int p) {
    const uint64_t lo = t & ((1ull << p) - 1);
    return ((t >> p) << (p + 1)) | lo;
}

}  // namespace ps
