// Host-side planner and encoder of libps under AddressSanitizer + UndefinedBehaviorSanitizer
// (tests/test_sanitize_host.py builds and runs it; no GPU).  Drives ps_pauli_encode(_codes),
// ps_gate_to_rotations and ps_plan_describe (the planner: passes, tiles, sub-groups, exchanges,
// lazy layouts, restore plans, mirror mode) over random layers and structured edge cases.
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <vector>

#include "../include/ps.h"

namespace ps {
void set_last_error(const std::string&) {}
}

static int check(int rc, int want, const char* what) {
    if (rc != want) {
        std::fprintf(stderr, "%s: rc %d (want %d)\n", what, rc, want);
        std::exit(1);
    }
    return rc;
}

int main() {
    std::mt19937_64 rng(250417881);
    uint64_t x = 0, z = 0;
    check(ps_pauli_encode("XIY", &x, &z), PS_OK, "encode");
    if (x != 5 || z != 4) return 1;
    check(ps_pauli_encode("", &x, &z), PS_EINVAL, "encode empty");
    check(ps_pauli_encode("XQ", &x, &z), PS_EINVAL, "encode bad");
    std::vector<uint8_t> codes(64 * 20);
    for (auto& c : codes) c = (uint8_t)(rng() & 3);
    std::vector<uint64_t> xm(20), zm(20);
    check(ps_pauli_encode_codes(codes.data(), 64, 20, xm.data(), zm.data()), PS_OK, "codes");
    const char* gates[] = {"H", "S", "T", "X", "Y", "Z", "RX", "RY", "RZ", "CNOT", "CZ", "SWAP", "CPHASE", "RZZ"};
    for (const char* g : gates) {
        int q[2] = {3, 5};
        double prm = 0.3;
        uint64_t gx[8], gz[8];
        double ga[8];
        size_t nout = 0;
        const bool two = std::string(g) == "CNOT" || std::string(g) == "CZ" || std::string(g) == "SWAP" ||
                         std::string(g) == "CPHASE" || std::string(g) == "RZZ";
        check(ps_gate_to_rotations(g, q, two ? 2 : 1, &prm, 1, gx, gz, ga, 8, &nout), PS_OK, g);
    }
    std::vector<ps_plan_op> ops(1 << 16);
    std::vector<ps_plan_rot> rots(1 << 17);
    for (int trial = 0; trial < 400; ++trial) {
        const int world = 1 << (int)(rng() % 4);
        const int m = __builtin_ctz(world);
        const int n = m + 1 + (int)(rng() % 30);
        const int rank = (int)(rng() % world);
        const int fusion = (int)(rng() % 3);
        const int tile_bits = 4 + (int)(rng() % 10);
        const int layout = world > 1 ? (int)(rng() % 3) : 1;
        const size_t count = 1 + rng() % 300;
        std::vector<uint64_t> X(count), Z(count);
        std::vector<double> A(count);
        const uint64_t lim = n >= 64 ? ~0ull : ((1ull << n) - 1);
        for (size_t l = 0; l < count; ++l) {
            const int kind = (int)(rng() % 5);
            uint64_t xx = 0, zz = 0;
            if (kind == 0) {  // weight-1..10 random string
                const int w = 1 + (int)(rng() % 10);
                for (int t = 0; t < w; ++t) {
                    const int q = (int)(rng() % n);
                    const int letter = 1 + (int)(rng() % 3);
                    if (letter != 3) xx |= 1ull << q;
                    if (letter != 1) zz |= 1ull << q;
                }
            } else if (kind == 1) {  // dense
                xx = rng() & lim;
                zz = rng() & lim;
            } else if (kind == 2) {  // diagonal / identity
                zz = (rng() % 4) ? (rng() & lim) : 0;
            } else if (kind == 3) {  // every local bit in X (full-exchange fallback)
                xx = lim;
                zz = rng() & lim;
            } else {  // repeat the previous x (same-x runs)
                xx = l ? X[l - 1] : 1;
                zz = rng() & lim;
            }
            X[l] = xx & lim;
            Z[l] = zz & lim;
            A[l] = (rng() % 7 == 0) ? 1.5707963267948966 : std::ldexp((double)(rng() >> 11), -53) * 6.28 - 3.14;
        }
        size_t nops = 0, nrots = 0;
        check(ps_plan_describe(n, world, rank, fusion, tile_bits, layout, X.data(), Z.data(), A.data(), count,
                               ops.data(), ops.size(), &nops, rots.data(), rots.size(), &nrots),
              PS_OK, "plan");
    }
    // argument validation
    size_t nops = 0, nrots = 0;
    uint64_t bx = 1ull << 10, bz = 0;
    double ba = 0.1;
    check(ps_plan_describe(8, 1, 0, 2, 12, 1, &bx, &bz, &ba, 1, nullptr, 0, &nops, nullptr, 0, &nrots), PS_ERANGE,
          "range");
    check(ps_plan_describe(8, 3, 0, 2, 12, 1, &bx, &bz, &ba, 1, nullptr, 0, &nops, nullptr, 0, &nrots), PS_EINVAL,
          "world");
    std::printf("asan/ubsan host run ok\n");
    return 0;
}
