// ps_internal.h -- internal types shared by the planner (host C++), the C-ABI layer and the
// CUDA kernels of libps.  Not part of the public ABI (see include/ps.h).
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/ps.h"

namespace ps {

// ------------------------------------------------------------------------------------------
// Device rotation record (one per rotation per pass), 48 bytes.
//
// A pass applies rotations to pairs {i, i xor x} in PHYSICAL local coordinates.  With
// B = sign * sin(phi) * i^(y+1) (y = popc(x & z) of the ORIGINAL logical string),
// A = -conj(B) and sigma = (-1)^(popc(z & i) [xor tile sign]) the update is
// (R3)
//     a'_i = c a_i + sigma * A a_j      (= c a_i + i sin(phi) w(j) a_j,  w(j) = conj w(i))
//     a'_j = c a_j + sigma * B a_i      (= c a_j + i sin(phi) w(i) a_i)
// where i is the member whose pivot bit (highest bit of x) is 0.  B is purely real
// (y odd: B = b) or purely imaginary (y even: B = i b), so each pair costs 4 multiplies and
// 4 fused multiply-adds.  For x = 0 (diagonal, y = 0) the element update is a' = c a + sigma A a.
struct DevRot {
    uint64_t x;    // xor mask (physical local)
    uint64_t z;    // phase mask in the same coordinates
    uint64_t zt;   // unused by K1 (0)
    double c;      // cos(phi)
    double b;      // B = b (real) or i b (imaginary)
    uint32_t real; // 1: B real, 0: B imaginary
    uint32_t pad;
};
static_assert(sizeof(DevRot) == 48, "DevRot layout");

// Tile passes (K2/K7) apply their rotations in SUB-GROUPS: consecutive rotations whose
// tile-local xor masks span <= kSubDim dimensions.  For a sub-group with basis u_0..u_3
// (tile-local, pivots p_0 < .. < p_3 = highest set bits, reduced row-echelon form) every thread
// owns one coset r xor span{u}: r = xor of col[b] over the set bits b of its thread index (the
// columns span a complement of span{u}, chosen so the lanes of one shared-memory phase hit
// distinct banks), and holds the 16 amplitudes l_d = r xor U(d), U(d) = xor of u_b over the set
// bits b of d, in registers while the sub-group's rotations are applied.
//
// Deferred scaling: each rotation is applied as f * (self_coef * a_self + cross_coef * a_other)
// with the uniform factor f = cos(phi) when |cos| >= 2^-10 |sin| (CFORM: self_coef = 1,
// cross_coef = +-t, t = sin/cos, |t| <= 1024) and f = sign*sin(phi) otherwise (SFORM: self_coef =
// t = cos/(sign*sin), cross_coef = +-1 or +-i), i.e. one fused multiply-add per component; the
// product F of the factors is applied when the amplitudes leave the registers (deferred across
// sub-groups while it stays within [2^-40, 2^40]).  CFORM's per-pair sign pattern parity(Dz & d)
// is a compile-time case of the kernel's switch (code bits 0-8), so its pairs carry no sign
// flips; only the thread-wide sign (the representative's parity) flips t once per rotation.
#ifndef PS_SHEAR
#define PS_SHEAR 0  // 1: unit-case CFORM rotations as three in-place shears (DevTRot p = tau, s = sin)
#endif
#ifndef PS_SUBDIM
#define PS_SUBDIM 4
#endif
constexpr int kSubDim = PS_SUBDIM;  // 4 (16 amplitudes per thread) or 3 (8; A/B build)
constexpr int kSubAmps = 1 << kSubDim;
constexpr int kMaxCols = 12;

struct DevSub {
    uint32_t u[kSubDim];     // basis in tile-local coordinates
    uint16_t col[kMaxCols];  // representative columns (tile-local), one per thread-index bit
    int32_t rot_begin;       // first DevTRot of this sub-group (index into the call's table)
    int32_t nrot;
    double F;                // product of the deferred factors
};
static_assert(sizeof(DevSub) == 56, "DevSub layout");

// one rotation of a sub-group: pair (d, d xor dx) of the thread's 16 registers ("i" member: bit
// highest(dx) of d is 0), sigma = parity(zr & r) xor parity(zt & i0) xor parity(Dz & d),
// Dz_b = parity(Z_loc & u_b).
//   code bits 0-6   (with bit 15) unit case = tu_case(real, log2 dx, Dz pattern) of a CFORM rotation
//                   whose dx is 0 (diagonal) or a unit vector: the specialised kernel applies it with
//                   compile-time per-pair signs
//   code bits 8-11  dx (0: diagonal, imaginary only)
//   code bit  12    REAL: B real (y odd) or imaginary (y even), as in DevRot
//   code bit  13    SFORM (else CFORM)
//   code bit  14    NEG (SFORM only): B/f = -1 (REAL) or -i (imaginary) instead of +1 / +i
//   code bit  15    UNIT: bits 0-6 hold the unit case
//   code bits 16-31 M, bit d = parity(Dz & d) (generic kernel: per-pair sign at run time)
constexpr uint32_t kTrReal = 1u << 12, kTrSform = 1u << 13, kTrNeg = 1u << 14, kTrUnit = 1u << 15;
#ifdef __CUDACC__
#define PS_HD __host__ __device__
#else
#define PS_HD
#endif
constexpr int kSpecMinRots = 16;  // planner: choose_spec (per-pass choice)
// unit case index: 0..15 diagonal (imaginary) by Dz; 16 + ((real * 4 + log2 dx) * 8 + the three Dz
// bits other than the pivot's), dx in {1, 2, 4, 8}
constexpr int kUnitCases = 80;
PS_HD constexpr int tu_case(int real, int dxi, int dz) {
    return dxi < 0 ? (dz & 15)
                   : 16 + ((real * 4 + dxi) << 3) + ((dz & ((1 << dxi) - 1)) | ((dz >> (dxi + 1)) << dxi));
}
// inverse of the pattern compression: the 4-bit Dz (pivot bit clear) of unit case pattern z3
PS_HD constexpr int tu_dz(int dxi, int z3) { return (z3 & ((1 << dxi) - 1)) | ((z3 >> dxi) << (dxi + 1)); }
struct DevTRot {
    uint32_t code;
    uint32_t zr;   // tile-local phase mask (parity with the coset representative r)
    uint64_t zt;   // phase mask on the tile-enumeration bits (parity with the tile base i0)
    double p;      // CFORM: t (B/f = +-t or +-i t); SFORM: t = cos/f (B/f = +-1 or +-i);
                   // PS_SHEAR unit case: tau = tan(theta / 2) of the exact rotation (no factor)
    double s;      // PS_SHEAR unit case: sin(theta); otherwise unused (keeps the record 32 B)
};
static_assert(sizeof(DevTRot) == 32, "DevTRot layout");

// expectation term record: contribution sigma(i) * (kr * tr + ki * ti) per pair (x != 0) with
// t = conj(a_j) a_i, or sigma(i) * kr * |a_i|^2 per element (x = 0)
struct DevTerm {
    uint64_t z;
    double kr;
    double ki;
};

enum PassKind : int {
    PASS_STREAM = PS_K_STREAM,
    PASS_TILE = PS_K_TILE,
    PASS_COSET = PS_K_COSET,
    PASS_EXCHANGE = PS_K_EXCHANGE,
    PASS_PERMUTE = PS_K_PERMUTE,  // local transposition of physical bits ell and ell2
    PASS_MIRROR_BEGIN = PS_OP_MIRROR_BEGIN,
    PASS_MIRROR_SWITCH = PS_OP_MIRROR_SWITCH,
    PASS_MIRROR_END = PS_OP_MIRROR_END,
};

constexpr int kMaxTileHigh = 10;  // at most 2^10 gathered chunks per coset tile

struct Pass {
    int kind = PASS_STREAM;
    int rot_begin = 0;    // first record in the call's DevRot array
    int rot_count = 0;    // records in this pass
    int first_input = 0;  // first input rotation covered
    int n_input = 0;      // input rotations covered
    // STREAM
    uint64_t x0 = 0;      // shared non-zero xor mask of the run (0: diagonal-only run)
    // TILE / COSET: tile = i0 xor off[u] | w, w < 2^cbits, u < 2^hbits, i0 = pdep(tau, free_mask)
    int kbits = 0;        // log2 tile amplitudes = cbits + hbits
    int cbits = 0;        // log2 contiguous chunk amplitudes
    int hbits = 0;        // number of gathered high basis vectors
    uint64_t free_mask = 0;
    uint64_t or_mask = 0;   // bits forced into every tile base (a pass split by one free bit)
    uint64_t touch_mask = 0;  // bits in which elements of one tile can differ (chunk bits | offsets)
    int off_begin = 0;    // first entry of this pass's 2^hbits chunk offsets in the call's table
    int sub_begin = 0;    // first DevSub of this pass
    int sub_count = 0;
    int spec = 0;         // 1: the specialised tile kernel (compile-time sign patterns), see planner
    // EXCHANGE
    uint64_t gx = 0;      // partner = rank xor gx
    int ell = 0;          // local pivot bit
    int keep = 0;         // this rank keeps slots with bit ell == keep
    int full = 0;         // 1: single-rotation full exchange (no free pivot); rot_begin/rot_count valid
    // PERMUTE
    int ell2 = 0;
    // MIRROR_BEGIN: upper string (gx, gz) and this rank's conj(w_k)
    uint64_t gz = 0;
    double wr = 1.0, wi = 0.0;
};

// one rank of a fused exchange + tile pass (kernels.cu k_xtile): its slice, the partner's slice
// (peer pointer), the per-tile handshake flags on both sides and its pass records (device)
struct XTileRank {
    void* a;                  // this rank's local slice (new layout after the pass)
    const void* peer;         // the partner's local slice
    uint32_t* flags;          // this rank's flags: the partner raises flag[tile] after reading it
    uint32_t* peer_flags;     // the partner's flags: raised by this rank
    const DevSub* subs;       // the pass's sub-groups (this rank's signs and factors)
    const DevTRot* trots;     // the call's rotation records (sub-group rot_begin indexes them)
    int rank;
    int keep;                 // this rank keeps its slots with bit ell == keep
};

struct Plan {
    std::vector<Pass> passes;
    std::vector<DevRot> rots;
    std::vector<uint64_t> offsets;
    std::vector<DevSub> subs;
    std::vector<DevTRot> trots;
    std::vector<ps_plan_rot> debug_rots;  // filled when requested (plan dump)
    uint64_t exchanges = 0;
    std::vector<int> perm_out;  // layout after the plan: physical bit -> logical qubit
};

struct PlanConfig {
    int n = 0;          // total qubits
    int n_local = 0;    // local qubits n - m
    int world = 1;
    int rank = 0;
    int fusion = 2;
    int tile_bits = 12;
    int min_chunk_bits = 4;     // coset tiles gather chunks of >= 2^min_chunk_bits amplitudes
    int phase_bits = 3;         // log2 lanes per shared-memory phase (16-B amplitudes: 3, 8-B: 4)
    int max_pass_rots = 1 << 30;
    bool want_debug = false;
    int layout = 1;             // world > 1: 1 lazy qubit swaps (Belady), 0 runs with swap-back
    int specialize = 0;         // tile kernel variant: 0 generic (default), 1 per-pass choice, 2 specialised
    std::vector<int> perm;      // starting layout (physical bit -> logical qubit); empty = canonical
};

// planner.cpp
int validate_rotations(int n, const uint64_t* x, const uint64_t* z, const double* angle,
                       size_t count, std::string* err);
void make_plan(const PlanConfig& cfg, const uint64_t* x, const uint64_t* z, const double* angle,
               size_t count, Plan* plan);
// ops returning layout `perm` to the canonical one (exchanges, then local transpositions);
// appends to plan (does not clear it) and sets plan->perm_out to the identity
void make_restore_plan(const PlanConfig& cfg, const std::vector<int>& perm, Plan* plan);
int popc64(uint64_t v);
int highest_bit(uint64_t v);

// thread-local last error
void set_last_error(const std::string& msg);

}  // namespace ps
