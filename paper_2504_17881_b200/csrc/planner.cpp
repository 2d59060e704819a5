// planner.cpp -- host side of the hot path: Pauli-string encoder, gate converter and the
// order-preserving planner that turns a rotation list into HBM passes and exchanges.
//
//   encoder     P:116-121, P:476-484 (two 64-bit masks; worked example XIY -> (5, 4))
//   converter   P:12, P:37-38 (1- and 2-qubit rotations are universal); R1 sign
//   planner     P:126-148 Eq. (1) (one exchange per run sharing the upper-qubit X-part),
//               P:357-430 (partitioned layout, pairwise exchange k <-> k xor q1),
//               P:403-404 (diagonal upper part: no exchange), P:494-499 (several rotations
//               per traversal of the array).  The planner never reorders rotations.
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstring>
#include <string>

#include "ps_internal.h"

namespace ps {

int popc64(uint64_t v) { return __builtin_popcountll(v); }
int highest_bit(uint64_t v) { return v ? 63 - __builtin_clzll(v) : -1; }
static inline int parity64(uint64_t v) { return __builtin_parityll(v); }

int validate_rotations(int n, const uint64_t* x, const uint64_t* z, const double* angle,
                       size_t count, std::string* err) {
    if (count == 0) return PS_OK;
    if (!x || !z || !angle) {
        *err = "NULL rotation array with count > 0";
        return PS_EINVAL;
    }
    const uint64_t lim = (n >= 64) ? ~0ull : ((1ull << n) - 1);
    for (size_t l = 0; l < count; ++l) {
        if (!std::isfinite(angle[l])) {
            *err = "non-finite angle at index " + std::to_string(l);
            return PS_EINVAL;
        }
        if ((x[l] & ~lim) || (z[l] & ~lim)) {
            *err = "mask bit >= n at index " + std::to_string(l);
            return PS_ERANGE;
        }
    }
    return PS_OK;
}

// ------------------------------------------------------------------------------------------
// record construction

// B = sign * sin(phi) * i^(y+1)   (see DevRot): i^1 = i, i^2 = -1, i^3 = -i, i^4 = 1
static DevRot make_rec(uint64_t x, uint64_t z, uint64_t zt, int y, int sign, double phi) {
    DevRot r{};
    r.x = x;
    r.z = z;
    r.zt = zt;
    const double s = std::sin(phi) * (double)sign;
    switch ((y + 1) & 3) {
    case 0: r.real = 1; r.b = s; break;
    case 1: r.real = 0; r.b = s; break;
    case 2: r.real = 1; r.b = -s; break;
    default: r.real = 0; r.b = -s; break;
    }
    r.c = std::cos(phi);
    r.pad = 0;
    return r;
}

// one rotation in physical local coordinates, before pass formation
struct PhysRot {
    uint64_t x, z;
    int y;       // popc(x & z) mod 4 of the logical string
    int sign;    // +1 / -1
    double phi;
    int input;   // input index
};

// ------------------------------------------------------------------------------------------
// GF(2) basis in reduced row-echelon form keyed by the highest set bit (pivot)

struct Basis {
    std::vector<uint64_t> v;  // each v[t] has a distinct pivot; pivots cleared in all others
    uint64_t pivots = 0;
    uint64_t reduce(uint64_t a) const {
        for (uint64_t b : v) {
            int p = highest_bit(b);
            if ((a >> p) & 1) a ^= b;
        }
        return a;
    }
    // adds a (already reduced, non-zero); keeps RREF
    void add(uint64_t a) {
        int p = highest_bit(a);
        for (auto& b : v)
            if ((b >> p) & 1) b ^= a;
        v.push_back(a);
        pivots |= 1ull << p;
    }
    int dim() const { return (int)v.size(); }
};

// ------------------------------------------------------------------------------------------
// pass formation over one segment of local physical rotations (no exchange inside)

static void emit_stream(const std::vector<PhysRot>& seg, size_t b, size_t e, Plan* plan) {
    Pass p;
    p.kind = PASS_STREAM;
    p.rot_begin = (int)plan->rots.size();
    p.first_input = seg[b].input;
    p.n_input = seg[e - 1].input - seg[b].input + 1;
    uint64_t x0 = 0;
    for (size_t t = b; t < e; ++t) {
        if (seg[t].x) x0 = seg[t].x;
        plan->rots.push_back(make_rec(seg[t].x, seg[t].z, 0, seg[t].y, seg[t].sign, seg[t].phi));
    }
    p.x0 = x0;
    p.rot_count = (int)(e - b);
    plan->passes.push_back(p);
}

// tile-local rotation before sub-grouping
struct LocalRot {
    uint64_t x, z, zt;
    int y, sign;
    double phi;
};

// Representative columns of a sub-group (see DevSub): k - kSubDim vectors spanning a complement
// of span{u}; the first `phase_bits` have linearly independent projections on the low
// phase_bits tile-local bits, so the lanes of one shared-memory phase hit distinct banks, and
// the rest are the lowest possible unit vectors (contiguous global segments for the first/last
// sub-group).
static void choose_columns(const Basis& U, int k, int phase_bits, uint16_t* col) {
    Basis S = U;
    int nc = 0;
    const int ncols = k - kSubDim;
    for (int p = 0; p < phase_bits && p < k && nc < ncols; ++p) {
        uint64_t cand = 1ull << p;
        if (S.reduce(cand) == 0) {
            cand = 0;
            for (int q = k - 1; q >= phase_bits; --q) {
                const uint64_t c2 = (1ull << p) | (1ull << q);
                if (S.reduce(c2)) {
                    cand = c2;
                    break;
                }
            }
        }
        if (!cand) continue;
        S.add(S.reduce(cand));
        col[nc++] = (uint16_t)cand;
    }
    for (int q = 0; q < k && nc < ncols; ++q) {
        const uint64_t cand = 1ull << q;
        const uint64_t r = S.reduce(cand);
        if (!r) continue;
        S.add(r);
        col[nc++] = (uint16_t)cand;
    }
    for (; nc < kMaxCols; ++nc) col[nc] = 0;
}

// Splits a tile pass's rotations into sub-groups of <= kSubDim-dimensional xor span (order
// preserving) and emits DevSub / DevTRot records (see ps_internal.h).  A sub-group is also closed
// when its deferred scale would drop below 2^-20 (long runs of diagonal rotations).
static void make_subgroups(const std::vector<LocalRot>& lr, int k, int phase_bits, Plan* plan, Pass* p) {
    p->sub_begin = (int)plan->subs.size();
    size_t b = 0;
    while (b < lr.size()) {
        Basis S;
        size_t e = b;
        double logF = 0.0;
        for (; e < lr.size(); ++e) {
            const double cc = std::fabs(std::cos(lr[e].phi)), ss = std::fabs(std::sin(lr[e].phi));
            const double lf = std::log2(cc >= std::ldexp(ss, -10) ? cc : ss);  // the factor actually deferred
            if (e > b && logF + lf < -20.0) break;
            const uint64_t r = S.reduce(lr[e].x);
            if (r) {
                if (S.dim() == kSubDim) break;
                S.add(r);
            }
            logF += lf;
        }
        // basis = the sub-group's own first independent xor masks in order (so most rotations get
        // a unit dx and only a few unrolled pair patterns are hot in the instruction cache),
        // padded to kSubDim dimensions with the highest free unit vectors
        std::vector<uint64_t> u;
        {
            Basis T;
            for (size_t t = b; t < e && (int)u.size() < kSubDim; ++t) {
                const uint64_t r = T.reduce(lr[t].x);
                if (r) {
                    T.add(r);
                    u.push_back(lr[t].x);
                }
            }
            for (int q = k - 1; q >= 0 && (int)u.size() < kSubDim; --q) {
                const uint64_t r = T.reduce(1ull << q);
                if (r) {
                    T.add(r);
                    u.push_back(1ull << q);
                }
            }
            S = T;
        }
        DevSub sub{};
        for (int t = 0; t < kSubDim; ++t) sub.u[t] = (uint32_t)u[t];
        choose_columns(S, k, phase_bits, sub.col);
        // coordinates of a mask in the basis u (u is independent; solve by elimination)
        auto coords = [&](uint64_t v) -> uint32_t {
            uint64_t rows[kSubDim];
            uint32_t tags[kSubDim];
            for (int q = 0; q < kSubDim; ++q) {
                rows[q] = u[q];
                tags[q] = 1u << q;
            }
            // Gaussian elimination on (rows | tags), pivot = highest bit
            for (int q = 0; q < kSubDim; ++q) {
                int best = q;
                for (int t = q; t < kSubDim; ++t)
                    if (highest_bit(rows[t]) > highest_bit(rows[best])) best = t;
                std::swap(rows[q], rows[best]);
                std::swap(tags[q], tags[best]);
                const int pq = highest_bit(rows[q]);
                for (int t = 0; t < kSubDim; ++t)
                    if (t != q && ((rows[t] >> pq) & 1)) {
                        rows[t] ^= rows[q];
                        tags[t] ^= tags[q];
                    }
            }
            uint32_t c = 0;
            for (int q = 0; q < kSubDim; ++q)
                if ((v >> highest_bit(rows[q])) & 1) {
                    v ^= rows[q];
                    c ^= tags[q];
                }
            return v == 0 ? c : 0xffffffffu;
        };
        sub.rot_begin = (int)plan->trots.size();
        sub.nrot = (int)(e - b);
        double F = 1.0;
        for (size_t t = b; t < e; ++t) {
            const LocalRot& L = lr[t];
            const uint32_t dx = coords(L.x);
            uint32_t dz = 0;
            for (int q = 0; q < kSubDim; ++q)
                if (parity64(L.z & u[q])) dz |= 1u << q;
            uint32_t M = 0;
            for (int d = 0; d < kSubAmps; ++d)
                if (parity64((uint64_t)(dz & (uint32_t)d))) M |= 1u << d;
            const double c = std::cos(L.phi);
            const double s0 = std::sin(L.phi) * (double)L.sign;
            const int e4 = (L.y + 1) & 3;                 // B = s0 * i^e4
            const int real = (e4 & 1) ? 0 : 1;            // i^0, i^2 real; i^1, i^3 imaginary
            const double ph = (e4 == 0 || e4 == 1) ? 1.0 : -1.0;  // B = s0 * ph * (1 or i)
            DevTRot tr{};
            tr.zr = (uint32_t)L.z;
            tr.zt = L.zt;
            if (std::fabs(c) >= std::ldexp(std::fabs(s0), -10) && !(dx == 0 && real)) {
                // CFORM: f = cos(phi), cross coefficient +-t, t = ph * s0 / c, |t| <= 1024
                tr.code = (dx << 8) | (real ? kTrReal : 0u) | (M << 16);
                if (dx == 0 || (dx & (dx - 1)) == 0)  // diagonal or unit dx: a specialised case exists
                    tr.code |= kTrUnit | (uint32_t)tu_case(real, dx ? __builtin_ctz(dx) : -1, (int)dz);
                tr.p = ph * (s0 / c);
                tr.s = 0.0;
#if PS_SHEAR
                if (tr.code & kTrUnit) {
                    // the pair update c * [[1, -t], [t, 1]] is the exact rotation by theta with
                    // cos theta = c, sin theta = ph * s0: three shears, no deferred factor;
                    // |theta| > pi/2 runs as -R(theta -+ pi) (the -1 joins F)
                    const double sg = ph * s0;
                    if (c >= 0.0) {
                        tr.p = sg / (1.0 + c);
                        tr.s = sg;
                    } else {
                        tr.p = -sg / (1.0 - c);
                        tr.s = -sg;
                        F = -F;
                    }
                    plan->trots.push_back(tr);
                    continue;
                }
#endif
                F *= c;
            } else {
                // SFORM: keeps phi = pi/2 exact (R8)
                tr.code = (dx << 8) | (real ? kTrReal : 0u) | kTrSform | (ph < 0 ? kTrNeg : 0u) | (M << 16);
                tr.p = c / s0;
                tr.s = 0.0;
                F *= s0;
            }
            plan->trots.push_back(tr);
        }
        sub.F = F;
        plan->subs.push_back(sub);
        b = e;
    }
    p->sub_count = (int)plan->subs.size() - p->sub_begin;
    // defer the scale factors across sub-groups (the amplitudes stay linear in them) while the
    // accumulated factor stays within [2^-40, 2^40]; F = 1 means "no scaling pass here"
    double acc = 1.0;
    for (int t = p->sub_begin; t < (int)plan->subs.size(); ++t) {
        acc *= plan->subs[t].F;
        const bool last = t + 1 == (int)plan->subs.size();
        const double next = last ? 1.0 : plan->subs[t + 1].F;
        if (last || std::fabs(std::log2(std::fabs(acc * next))) > 40.0) {
            plan->subs[t].F = acc;
            acc = 1.0;
        } else {
            plan->subs[t].F = 1.0;
        }
    }
}

// Tile-kernel variant of a pass.  The specialised kernel applies CFORM rotations whose dx is a unit
// vector (or 0) with compile-time per-pair signs (80 cases), the rest generically; per-pass choice
// (PS_OPT_SPECIALIZE=1): deep passes where most rotations have such a case.
static void choose_spec(const PlanConfig& cfg, const Plan& plan, Pass* p) {
    if (cfg.specialize != 1) {
        p->spec = cfg.specialize == 2;
        return;
    }
    int nrot = 0, unit = 0;
    for (int t = p->sub_begin; t < p->sub_begin + p->sub_count; ++t) {
        const DevSub& sb = plan.subs[t];
        for (int q = sb.rot_begin; q < sb.rot_begin + sb.nrot; ++q) {
            ++nrot;
            unit += (plan.trots[q].code & kTrUnit) ? 1 : 0;
        }
    }
    p->spec = nrot >= kSpecMinRots && 2 * unit >= nrot;
}

static void emit_tile(const std::vector<PhysRot>& seg, size_t b, size_t e, const PlanConfig& cfg,
                      const Basis& hb, int chunk_min, Plan* plan) {
    const int nl = cfg.n_local;
    const int k = std::min(cfg.tile_bits, nl);
    const uint64_t lmask = (nl >= 64) ? ~0ull : ((1ull << nl) - 1);
    // all x inside the low k bits -> contiguous tile (K2)
    uint64_t xor_all = 0;
    for (size_t t = b; t < e; ++t) xor_all |= seg[t].x;
    Pass p;
    p.rot_begin = (int)plan->rots.size();
    p.first_input = seg[b].input;
    p.n_input = seg[e - 1].input - seg[b].input + 1;
    p.rot_count = (int)(e - b);
    if ((xor_all >> k) == 0) {
        p.kind = PASS_TILE;
        p.kbits = k;
        p.cbits = k;
        p.hbits = 0;
        p.free_mask = lmask & ~((1ull << k) - 1);
        p.off_begin = (int)plan->offsets.size();
        plan->offsets.push_back(0);
        p.touch_mask = (1ull << k) - 1;
        const uint64_t kmask = (1ull << k) - 1;
        std::vector<LocalRot> lr;
        for (size_t t = b; t < e; ++t)
            lr.push_back({seg[t].x, seg[t].z & kmask, seg[t].z & p.free_mask, seg[t].y, seg[t].sign, seg[t].phi});
        make_subgroups(lr, k, cfg.phase_bits, plan, &p);
        choose_spec(cfg, *plan, &p);
        plan->passes.push_back(p);
        return;
    }
    // coset tile: grow the contiguous chunk while the tile dimension stays <= k
    int c = chunk_min;
    auto reduced_dim = [&](int cb) {
        Basis r;
        const uint64_t hi = ~((1ull << cb) - 1);
        for (uint64_t v : hb.v) {
            uint64_t a = r.reduce(v & hi);
            if (a) r.add(a);
        }
        return r;
    };
    Basis vb = reduced_dim(c);
    while (c + 1 <= k) {
        Basis nb = reduced_dim(c + 1);
        if (c + 1 + nb.dim() > k) break;
        c += 1;
        vb = nb;
    }
    p.kind = PASS_COSET;
    p.cbits = c;
    p.hbits = vb.dim();
    p.kbits = c + vb.dim();
    const uint64_t cmask = (1ull << c) - 1;
    p.free_mask = lmask & ~cmask & ~vb.pivots;
    // order basis vectors by pivot so tile-local bit t <-> t-th smallest pivot
    std::vector<uint64_t> vs = vb.v;
    std::sort(vs.begin(), vs.end(), [](uint64_t a, uint64_t bb) { return highest_bit(a) < highest_bit(bb); });
    p.off_begin = (int)plan->offsets.size();
    p.touch_mask = cmask;
    for (uint64_t u = 0; u < (1ull << p.hbits); ++u) {
        uint64_t o = 0;
        for (int t = 0; t < p.hbits; ++t)
            if ((u >> t) & 1) o ^= vs[t];
        plan->offsets.push_back(o);
        p.touch_mask |= o;
    }
    std::vector<LocalRot> lr;
    for (size_t t = b; t < e; ++t) {
        const uint64_t x = seg[t].x, z = seg[t].z;
        const uint64_t xh = x & ~cmask;
        uint64_t coef = 0, zc = 0, chk = 0;
        for (int q = 0; q < p.hbits; ++q) {
            const int piv = highest_bit(vs[q]);
            if ((xh >> piv) & 1) {
                coef |= 1ull << q;
                chk ^= vs[q];
            }
            if (parity64(z & vs[q])) zc |= 1ull << q;
        }
        (void)chk;  // chk == xh by construction (x lies in the tile space)
        const uint64_t xl = (coef << c) | (x & cmask);
        const uint64_t zl = (zc << c) | (z & cmask);
        lr.push_back({xl, zl, z & p.free_mask, seg[t].y, seg[t].sign, seg[t].phi});
    }
    make_subgroups(lr, p.kbits, cfg.phase_bits, plan, &p);
    choose_spec(cfg, *plan, &p);
    plan->passes.push_back(p);
}

static void form_passes(const std::vector<PhysRot>& seg, const PlanConfig& cfg, Plan* plan) {
    if (seg.empty()) return;
    const int nl = cfg.n_local;
    if (cfg.fusion <= 0) {
        for (size_t t = 0; t < seg.size(); ++t) emit_stream(seg, t, t + 1, plan);
        return;
    }
    if (cfg.fusion == 1) {
        size_t b = 0;
        uint64_t x0 = 0;
        for (size_t t = 0; t < seg.size(); ++t) {
            const uint64_t x = seg[t].x;
            if (x == 0 || x0 == 0 || x == x0) {
                if (x) x0 = x;
                continue;
            }
            emit_stream(seg, b, t, plan);
            b = t;
            x0 = x;
        }
        emit_stream(seg, b, seg.size(), plan);
        return;
    }
    // fusion 2: greedy tile spaces (order preserving); a tile needs >= 2^kSubDim amplitudes
    const int k = std::min(cfg.tile_bits, nl);
    if (k < kSubDim) {
        PlanConfig c1 = cfg;
        c1.fusion = 1;
        form_passes(seg, c1, plan);
        return;
    }
    const int chunk_min = std::min(cfg.min_chunk_bits, k);
    const uint64_t low = (1ull << chunk_min) - 1;
    size_t b = 0;
    Basis hb;
    uint64_t x0 = 0;
    bool same_x = true;
    int nrot = 0;
    auto close = [&](size_t e) {
        if (e <= b) return;
        if (same_x)
            emit_stream(seg, b, e, plan);
        else
            emit_tile(seg, b, e, cfg, hb, chunk_min, plan);
    };
    for (size_t t = 0; t < seg.size(); ++t) {
        const uint64_t x = seg[t].x;
        const uint64_t r = hb.reduce(x & ~low);
        const bool fits = (r == 0 || chunk_min + hb.dim() + 1 <= k) && nrot < cfg.max_pass_rots;
        if (!fits) {
            close(t);
            b = t;
            hb = Basis();
            x0 = 0;
            same_x = true;
            nrot = 0;
        }
        const uint64_t r2 = hb.reduce(x & ~low);
        if (r2) hb.add(r2);
        if (x) {
            if (x0 == 0) x0 = x;
            else if (x != x0) same_x = false;
        }
        ++nrot;
    }
    close(seg.size());
}

// ------------------------------------------------------------------------------------------
// full plan: layout (exchanges) then passes

static void clear_plan(Plan* plan) {
    plan->passes.clear();
    plan->rots.clear();
    plan->offsets.clear();
    plan->subs.clear();
    plan->trots.clear();
    plan->debug_rots.clear();
    plan->exchanges = 0;
}

static void push_debug_rot(const PlanConfig& cfg, Plan* plan, const PhysRot& pr) {
    if (!cfg.want_debug) return;
    ps_plan_rot d;
    d.x = pr.x;
    d.z = pr.z;
    d.y = pr.y;
    d.sign = pr.sign;
    d.angle = pr.phi;
    plan->debug_rots.push_back(d);
}

// single-rotation full exchange (no free pivot): rotation given in physical coordinates
static void emit_full_exchange(const PlanConfig& cfg, Plan* plan, uint64_t gx, const PhysRot& pr) {
    Pass p;
    p.kind = PASS_EXCHANGE;
    p.full = 1;
    p.gx = gx;
    p.rot_begin = (int)plan->rots.size();
    p.rot_count = 1;
    p.first_input = pr.input;
    p.n_input = 1;
    push_debug_rot(cfg, plan, pr);
    plan->rots.push_back(make_rec(pr.x, pr.z, 0, pr.y, pr.sign, pr.phi));
    plan->passes.push_back(p);
    plan->exchanges += 1;
}

// transposition of physical rank bit j (global bit nl + j) with local bit ell as a half-vector
// exchange with rank r xor 2^j
static void emit_swap_exchange(const PlanConfig& cfg, Plan* plan, int j, int ell, int first_input) {
    Pass ex;
    ex.kind = PASS_EXCHANGE;
    ex.gx = 1ull << j;
    ex.ell = ell;
    ex.keep = (cfg.rank >> j) & 1;
    ex.first_input = first_input;
    ex.n_input = 0;
    plan->passes.push_back(ex);
    plan->exchanges += 1;
}

static void emit_permute(Plan* plan, int a, int b, int first_input) {
    Pass p;
    p.kind = PASS_PERMUTE;
    p.ell = std::min(a, b);
    p.ell2 = std::max(a, b);
    p.first_input = first_input;
    p.n_input = 0;
    plan->passes.push_back(p);
}

static uint64_t map_mask(uint64_t m, const std::vector<int>& inv) {
    uint64_t out = 0;
    while (m) {
        const int q = __builtin_ctzll(m);
        m &= m - 1;
        out |= 1ull << inv[q];
    }
    return out;
}

void make_restore_plan(const PlanConfig& cfg, const std::vector<int>& perm_in, Plan* plan) {
    const int n = cfg.n, nl = cfg.n_local;
    std::vector<int> perm = perm_in, inv(n);
    if ((int)perm.size() != n) {
        perm.resize(n);
        for (int q = 0; q < n; ++q) perm[q] = q;
    }
    for (int p = 0; p < n; ++p) inv[perm[p]] = p;
    auto swap_pos = [&](int a, int b) {
        std::swap(perm[a], perm[b]);
        inv[perm[a]] = a;
        inv[perm[b]] = b;
    };
    // 1. every global position gets its canonical qubit back (exchanges)
    for (int g = nl; g < n; ++g) {
        if (perm[g] == g) continue;
        int p = inv[g];
        if (p >= nl) {  // canonical qubit sits in another global slot: move it local first
            const int ell = nl - 1;
            emit_swap_exchange(cfg, plan, p - nl, ell, -1);
            swap_pos(p, ell);
            p = ell;
        }
        emit_swap_exchange(cfg, plan, g - nl, p, -1);
        swap_pos(g, p);
    }
    // 2. local transpositions (HBM passes)
    for (int ell = 0; ell < nl; ++ell) {
        if (perm[ell] == ell) continue;
        const int p = inv[ell];
        emit_permute(plan, ell, p, -1);
        swap_pos(ell, p);
    }
    plan->perm_out.assign(n, 0);
    for (int q = 0; q < n; ++q) plan->perm_out[q] = q;
}

// lazy qubit-swap layout: a rotation whose X-part touches a global position first swaps that
// position's qubit with the local qubit whose next X-use is furthest in the future (Belady);
// the layout is not restored at the end (plan->perm_out)
static void plan_lazy(const PlanConfig& cfg, const uint64_t* x, const uint64_t* z, const double* angle,
                      size_t count, Plan* plan) {
    const int n = cfg.n, nl = cfg.n_local;
    const uint64_t lmask = (1ull << nl) - 1;
    const uint64_t rank = (uint64_t)cfg.rank;
    std::vector<int> perm = cfg.perm, inv(n);
    if ((int)perm.size() != n) {
        perm.resize(n);
        for (int q = 0; q < n; ++q) perm[q] = q;
    }
    for (int p = 0; p < n; ++p) inv[perm[p]] = p;
    // next X-use per logical qubit
    std::vector<std::vector<int>> uses(n);
    for (size_t l = 0; l < count; ++l)
        for (uint64_t m = x[l]; m; m &= m - 1) uses[__builtin_ctzll(m)].push_back((int)l);
    std::vector<size_t> ptr(n, 0);
    auto next_use = [&](int q, int after) -> long {
        auto& u = uses[q];
        size_t& k = ptr[q];
        while (k < u.size() && u[k] <= after) ++k;
        return k < u.size() ? (long)u[k] : (long)1 << 40;
    };
    std::vector<PhysRot> seg;
    auto flush = [&]() {
        form_passes(seg, cfg, plan);
        seg.clear();
    };
    for (size_t l = 0; l < count; ++l) {
        uint64_t xp = map_mask(x[l], inv);
        bool full = false;
        while (xp >> nl) {
            const int g = nl + __builtin_ctzll(xp >> nl);
            // candidate local positions whose qubit is not in this rotation's X-part
            int best = -1;
            long best_use = -1;
            for (int ell = nl - 1; ell >= 0; --ell) {
                const int q = perm[ell];
                if ((x[l] >> q) & 1) continue;
                long u = next_use(q, (int)l);
                if (perm[g] == ell && q == g) u += 1;  // tie-break: swaps that restore canonical
                if (u > best_use) {
                    best_use = u;
                    best = ell;
                }
            }
            if (best < 0) {
                full = true;
                break;
            }
            flush();
            emit_swap_exchange(cfg, plan, g - nl, best, (int)l);
            std::swap(perm[g], perm[best]);
            inv[perm[g]] = g;
            inv[perm[best]] = best;
            xp = map_mask(x[l], inv);
        }
        const uint64_t zp = map_mask(z[l], inv);
        PhysRot pr;
        pr.x = xp & lmask;
        pr.z = zp & lmask;
        pr.y = popc64(x[l] & z[l]) & 3;
        pr.sign = parity64((zp >> nl) & rank) ? -1 : 1;
        pr.phi = angle[l];
        pr.input = (int)l;
        if (full) {
            flush();
            emit_full_exchange(cfg, plan, xp >> nl, pr);
            continue;
        }
        seg.push_back(pr);
        push_debug_rot(cfg, plan, pr);
    }
    flush();
    plan->perm_out = perm;
}

static void make_plan_core(const PlanConfig& cfg, const uint64_t* x, const uint64_t* z, const double* angle,
                           size_t count, Plan* plan);

// Identity-string rotations (x = z = 0: global phases e^{i phi}, e.g. the converter's gate phases,
// R5) commute with every rotation, so they are summed into one global-phase rotation applied
// last; everything else keeps its order.
void make_plan(const PlanConfig& cfg, const uint64_t* x, const uint64_t* z, const double* angle,
               size_t count, Plan* plan) {
    size_t nid = 0;
    for (size_t l = 0; l < count; ++l) nid += (x[l] == 0 && z[l] == 0);
    if (nid < 2) {
        make_plan_core(cfg, x, z, angle, count, plan);
        return;
    }
    std::vector<uint64_t> xs, zs;
    std::vector<double> as;
    xs.reserve(count - nid + 1);
    zs.reserve(count - nid + 1);
    as.reserve(count - nid + 1);
    double phase = 0.0;
    for (size_t l = 0; l < count; ++l) {
        if (x[l] == 0 && z[l] == 0) {
            phase += angle[l];
            continue;
        }
        xs.push_back(x[l]);
        zs.push_back(z[l]);
        as.push_back(angle[l]);
    }
    xs.push_back(0);
    zs.push_back(0);
    as.push_back(phase);
    make_plan_core(cfg, xs.data(), zs.data(), as.data(), xs.size(), plan);
}

// the paper's grouped execution: groups of consecutive rotations sharing the
// upper string Q = (gx, gz), gx != 0, run as MIRROR_BEGIN; passes of e^{+i phi P_l} on A;
// MIRROR_SWITCH; passes of e^{-i phi P_l} on B; MIRROR_END.  P_l = the lower strings.
static void plan_mirror(const PlanConfig& cfg, const uint64_t* x, const uint64_t* z, const double* angle,
                        size_t count, Plan* plan) {
    const int nl = cfg.n_local;
    const uint64_t lmask = (1ull << nl) - 1;
    const uint64_t rank = (uint64_t)cfg.rank;
    std::vector<PhysRot> seg;
    auto flush = [&]() {
        form_passes(seg, cfg, plan);
        seg.clear();
    };
    size_t i = 0;
    while (i < count) {
        const uint64_t gx = x[i] >> nl, gz = z[i] >> nl;
        if (gx == 0) {
            PhysRot pr;
            pr.x = x[i] & lmask;
            pr.z = z[i] & lmask;
            pr.y = popc64(x[i] & z[i]) & 3;
            pr.sign = parity64(gz & rank) ? -1 : 1;
            pr.phi = angle[i];
            pr.input = (int)i;
            seg.push_back(pr);
            push_debug_rot(cfg, plan, pr);
            ++i;
            continue;
        }
        size_t j = i;
        while (j < count && (x[j] >> nl) == gx && (z[j] >> nl) == gz) ++j;
        flush();
        Pass b;
        b.kind = PASS_MIRROR_BEGIN;
        b.gx = gx;
        b.gz = gz;
        b.first_input = (int)i;
        b.n_input = (int)(j - i);
        // Q|k> = w_k |k xor gx>, w_k = i^popc(gx&gz) (-1)^popc(gz&k); B holds conj(w_k) A_(k xor gx)
        const int e = ((popc64(gx & gz) & 3) + (parity64(gz & rank) ? 2 : 0)) & 3;
        const double re[4] = {1, 0, -1, 0}, im[4] = {0, 1, 0, -1};
        b.wr = re[e];
        b.wi = -im[e];
        plan->passes.push_back(b);
        plan->exchanges += 1;
        for (int half = 0; half < 2; ++half) {
            if (half == 1) {
                Pass sw;
                sw.kind = PASS_MIRROR_SWITCH;
                sw.first_input = (int)i;
                plan->passes.push_back(sw);
            }
            for (size_t t = i; t < j; ++t) {
                PhysRot pr;
                pr.x = x[t] & lmask;
                pr.z = z[t] & lmask;
                pr.y = popc64(pr.x & pr.z) & 3;  // the lower string's own i^(#Y)
                pr.sign = 1;
                pr.phi = half ? -angle[t] : angle[t];
                pr.input = (int)t;
                seg.push_back(pr);
                push_debug_rot(cfg, plan, pr);
            }
            flush();
        }
        Pass en;
        en.kind = PASS_MIRROR_END;
        en.first_input = (int)i;
        plan->passes.push_back(en);
        i = j;
    }
    flush();
}

static void make_plan_core(const PlanConfig& cfg, const uint64_t* x, const uint64_t* z, const double* angle,
                           size_t count, Plan* plan) {
    clear_plan(plan);
    if (cfg.world > 1 && cfg.layout == 2) {
        plan_mirror(cfg, x, z, angle, count, plan);
        plan->perm_out.clear();
        return;
    }
    if (cfg.world > 1 && cfg.layout == 1) {
        plan_lazy(cfg, x, z, angle, count, plan);
        return;
    }
    if ((int)cfg.perm.size() == cfg.n) {
        for (int q = 0; q < cfg.n; ++q)
            if (cfg.perm[q] != q) {
                // run mode needs the canonical layout: restore first
                make_restore_plan(cfg, cfg.perm, plan);
                break;
            }
    }
    plan->perm_out.clear();
    const int nl = cfg.n_local;
    const uint64_t lmask = (nl >= 64) ? ~0ull : ((1ull << nl) - 1);
    const uint64_t rank = (uint64_t)cfg.rank;
    std::vector<PhysRot> seg;

    auto logical_y = [&](size_t l) { return popc64(x[l] & z[l]) & 3; };
    auto push_debug = [&](const PhysRot& pr) {
        if (cfg.want_debug) {
            ps_plan_rot d;
            d.x = pr.x;
            d.z = pr.z;
            d.y = pr.y;
            d.sign = pr.sign;
            d.angle = pr.phi;
            plan->debug_rots.push_back(d);
        }
    };
    auto flush = [&]() {
        form_passes(seg, cfg, plan);
        seg.clear();
    };

    size_t i = 0;
    while (i < count) {
        const uint64_t gx = x[i] >> nl;
        if (cfg.world == 1 || gx == 0) {
            // local rotation in the canonical layout; z on the rank bits -> per-rank sign
            PhysRot pr;
            pr.x = x[i] & lmask;
            pr.z = z[i] & lmask;
            pr.y = logical_y(i);
            pr.sign = parity64((z[i] >> nl) & rank) ? -1 : 1;
            pr.phi = angle[i];
            pr.input = (int)i;
            seg.push_back(pr);
            push_debug(pr);
            ++i;
            continue;
        }
        // run sharing the upper X-part gx (Eq. (1)): rotations with upper X-part in
        // {0, gx} whose local X-parts leave a free pivot bit
        uint64_t U = 0;
        size_t j = i, last = count;  // last = last rotation with upper part gx
        while (j < count) {
            const uint64_t gj = x[j] >> nl;
            if (gj != 0 && gj != gx) break;
            const uint64_t xl = x[j] & lmask;
            if ((U | xl) == lmask) break;
            U |= xl;
            if (gj == gx) last = j;
            ++j;
        }
        flush();
        if (last == count) {
            // no free pivot even for rotation i alone: single-rotation full exchange
            PhysRot pr;
            pr.x = x[i] & lmask;
            pr.z = z[i] & lmask;
            pr.y = logical_y(i);
            pr.sign = parity64((z[i] >> nl) & rank) ? -1 : 1;
            pr.phi = angle[i];
            pr.input = (int)i;
            emit_full_exchange(cfg, plan, gx, pr);
            ++i;
            continue;
        }
        U = 0;
        for (size_t t = i; t <= last; ++t) U |= x[t] & lmask;
        const int ell = highest_bit(lmask & ~U);
        const int g = __builtin_ctzll(gx);
        const int keep = (int)((rank >> g) & 1);
        Pass ex;
        ex.kind = PASS_EXCHANGE;
        ex.gx = gx;
        ex.ell = ell;
        ex.keep = keep;
        ex.first_input = (int)i;
        ex.n_input = (int)(last - i + 1);
        plan->passes.push_back(ex);
        plan->exchanges += 1;
        const uint64_t el = 1ull << ell;
        for (size_t t = i; t <= last; ++t) {
            const uint64_t xh = x[t] >> nl, xl = x[t] & lmask;
            const uint64_t zh = z[t] >> nl, zl = z[t] & lmask;
            const int kappa = parity64(zh & gx) ^ (int)((zl >> ell) & 1);
            PhysRot pr;
            pr.x = xl ^ (xh ? el : 0);
            pr.z = zl ^ (kappa ? el : 0);
            pr.y = logical_y(t);
            pr.sign = (parity64(zh & rank) ^ (keep & kappa)) ? -1 : 1;
            pr.phi = angle[t];
            pr.input = (int)t;
            seg.push_back(pr);
            push_debug(pr);
        }
        flush();
        plan->passes.push_back(ex);  // swap back to the canonical layout
        plan->exchanges += 1;
        i = last + 1;
    }
    flush();
}

}  // namespace ps

// ==========================================================================================
// C ABI: host-only helpers

using namespace ps;

extern "C" int ps_pauli_encode(const char* word, uint64_t* xmask, uint64_t* zmask) {
    if (!word || !xmask || !zmask) {
        set_last_error("ps_pauli_encode: NULL argument");
        return PS_EINVAL;
    }
    const size_t n = std::strlen(word);
    if (n == 0 || n > 64) {
        set_last_error("ps_pauli_encode: word length must be 1..64");
        return PS_EINVAL;
    }
    uint64_t x = 0, z = 0;
    for (size_t q = 0; q < n; ++q) {
        const char ch = (char)std::toupper((unsigned char)word[q]);
        const uint64_t bit = 1ull << q;  // factor q+1 -> bit q
        switch (ch) {
        case 'I': break;
        case 'X': x |= bit; break;
        case 'Y': x |= bit; z |= bit; break;
        case 'Z': z |= bit; break;
        default:
            set_last_error(std::string("ps_pauli_encode: invalid letter '") + word[q] + "'");
            return PS_EINVAL;
        }
    }
    *xmask = x;
    *zmask = z;
    return PS_OK;
}

extern "C" int ps_pauli_encode_codes(const uint8_t* codes, int n, size_t count, uint64_t* xmask,
                                     uint64_t* zmask) {
    if (n < 1 || n > 64) {
        set_last_error("ps_pauli_encode_codes: n must be 1..64");
        return PS_EINVAL;
    }
    if (count && (!codes || !xmask || !zmask)) {
        set_last_error("ps_pauli_encode_codes: NULL argument");
        return PS_EINVAL;
    }
    for (size_t l = 0; l < count; ++l) {
        uint64_t x = 0, z = 0;
        for (int q = 0; q < n; ++q) {
            const uint8_t c = codes[l * (size_t)n + q];
            if (c > 3) {
                set_last_error("ps_pauli_encode_codes: code > 3");
                return PS_EINVAL;
            }
            if (c == 1 || c == 2) x |= 1ull << q;
            if (c == 2 || c == 3) z |= 1ull << q;
        }
        xmask[l] = x;
        zmask[l] = z;
    }
    return PS_OK;
}

// gate -> rotations (exp(+i phi P) convention, R1); application order
extern "C" int ps_gate_to_rotations(const char* gate, const int* qubits, int nq, const double* params,
                                    int np, uint64_t* xm, uint64_t* zm, double* ang, size_t cap,
                                    size_t* n_out) {
    if (!gate || !n_out || (nq > 0 && !qubits)) {
        set_last_error("ps_gate_to_rotations: NULL argument");
        return PS_EINVAL;
    }
    std::string g(gate);
    for (auto& ch : g) ch = (char)std::toupper((unsigned char)ch);
    if (g == "CX") g = "CNOT";
    const double PI = 3.14159265358979323846;
    struct R { uint64_t x, z; double a; };
    std::vector<R> out;
    auto need = [&](int q, int p) -> bool {
        if (nq != q || np < p || (p > 0 && !params)) return false;
        for (int t = 0; t < q; ++t)
            if (qubits[t] < 0 || qubits[t] > 63) return false;
        if (q == 2 && qubits[0] == qubits[1]) return false;
        return true;
    };
    auto X1 = [&](int t) { return 1ull << qubits[t]; };
    bool ok = true;
    if (g == "RX" || g == "RY" || g == "RZ") {
        ok = need(1, 1);
        if (ok) {
            const uint64_t b = X1(0);
            const double a = -params[0] / 2;
            if (g == "RX") out.push_back({b, 0, a});
            if (g == "RY") out.push_back({b, b, a});
            if (g == "RZ") out.push_back({0, b, a});
        }
    } else if (g == "X" || g == "Y" || g == "Z") {
        ok = need(1, 0);
        if (ok) {
            const uint64_t b = X1(0);
            out.push_back({g == "Z" ? 0 : b, g == "X" ? 0 : b, PI / 2});
            out.push_back({0, 0, -PI / 2});
        }
    } else if (g == "S" || g == "T") {
        ok = need(1, 0);
        if (ok) {
            const double a = (g == "S") ? PI / 4 : PI / 8;
            out.push_back({0, X1(0), -a});
            out.push_back({0, 0, a});
        }
    } else if (g == "H") {
        ok = need(1, 0);
        if (ok) {
            const uint64_t b = X1(0);
            out.push_back({0, b, -PI / 4});
            out.push_back({b, 0, -PI / 4});
            out.push_back({0, b, -PI / 4});
            out.push_back({0, 0, PI / 2});
        }
    } else if (g == "CNOT" || g == "CZ" || g == "CPHASE") {
        ok = need(2, g == "CPHASE" ? 1 : 0);
        if (ok) {
            const double lam = (g == "CPHASE") ? params[0] : PI;
            const uint64_t c = X1(0), t = X1(1);
            const double a = lam / 4;
            out.push_back({0, c, -a});
            if (g == "CNOT") {
                out.push_back({t, 0, -a});
                out.push_back({t, c, a});  // Z_c X_t
            } else {
                out.push_back({0, t, -a});
                out.push_back({0, c | t, a});  // Z_c Z_t
            }
            out.push_back({0, 0, a});
        }
    } else if (g == "SWAP") {
        ok = need(2, 0);
        if (ok) {
            const uint64_t b = X1(0) | X1(1);
            out.push_back({b, 0, PI / 4});
            out.push_back({b, b, PI / 4});
            out.push_back({0, b, PI / 4});
            out.push_back({0, 0, -PI / 4});
        }
    } else if (g == "RZZ") {
        ok = need(2, 1);
        if (ok) out.push_back({0, X1(0) | X1(1), -params[0] / 2});
    } else {
        set_last_error("ps_gate_to_rotations: unknown gate " + g);
        return PS_EINVAL;
    }
    if (!ok) {
        set_last_error("ps_gate_to_rotations: bad qubits/params for " + g);
        return PS_EINVAL;
    }
    *n_out = out.size();
    if (out.size() > cap) {
        set_last_error("ps_gate_to_rotations: cap too small");
        return PS_ERANGE;
    }
    if (!out.empty() && (!xm || !zm || !ang)) {
        set_last_error("ps_gate_to_rotations: NULL output");
        return PS_EINVAL;
    }
    for (size_t t = 0; t < out.size(); ++t) {
        xm[t] = out[t].x;
        zm[t] = out[t].z;
        ang[t] = out[t].a;
    }
    return PS_OK;
}

extern "C" int ps_plan_describe(int n_qubits, int world, int rank, int fusion, int tile_bits, int layout,
                                const uint64_t* xmask, const uint64_t* zmask, const double* angle,
                                size_t count, ps_plan_op* ops, size_t ops_cap, size_t* n_ops,
                                ps_plan_rot* rots, size_t rots_cap, size_t* n_rots) {
    if (n_qubits < 1 || n_qubits > 62 || world < 1 || (world & (world - 1)) || rank < 0 ||
        rank >= world) {
        set_last_error("ps_plan_describe: bad n/world/rank");
        return PS_EINVAL;
    }
    const int m = __builtin_ctz((unsigned)world);
    if (n_qubits - m < 1) {
        set_last_error("ps_plan_describe: world too large for n");
        return PS_EINVAL;
    }
    std::string err;
    int rc = validate_rotations(n_qubits, xmask, zmask, angle, count, &err);
    if (rc) {
        set_last_error(err);
        return rc;
    }
    PlanConfig cfg;
    cfg.n = n_qubits;
    cfg.n_local = n_qubits - m;
    cfg.world = world;
    cfg.rank = rank;
    cfg.fusion = fusion;
    cfg.tile_bits = tile_bits > 0 ? tile_bits : 12;
    cfg.want_debug = true;
    cfg.layout = layout;
    Plan plan;
    make_plan(cfg, xmask, zmask, angle, count, &plan);
    if (!plan.perm_out.empty()) make_restore_plan(cfg, plan.perm_out, &plan);
    if (n_ops) *n_ops = plan.passes.size();
    if (n_rots) *n_rots = plan.debug_rots.size();
    if (ops) {
        for (size_t t = 0; t < plan.passes.size() && t < ops_cap; ++t) {
            const Pass& p = plan.passes[t];
            ps_plan_op o{};
            o.kind = p.kind;
            o.first_rot = p.first_input;
            o.n_rot = (p.kind == PASS_PERMUTE || p.kind >= PASS_MIRROR_BEGIN || (p.kind == PASS_EXCHANGE && !p.full))
                          ? 0
                          : p.n_input;
            o.exch_bit = p.full ? -1 : p.ell;
            o.exch_gx = p.kind == PASS_PERMUTE ? (uint64_t)p.ell2 : p.gx;
            o.tile_bits = (uint32_t)p.kbits;
            o.n_sub = (uint32_t)p.sub_count;
            if (p.kind == PASS_MIRROR_BEGIN) o.tile_bits = (uint32_t)p.gz;
            ops[t] = o;
        }
    }
    if (rots) {
        for (size_t t = 0; t < plan.debug_rots.size() && t < rots_cap; ++t) rots[t] = plan.debug_rots[t];
    }
    return PS_OK;
}
