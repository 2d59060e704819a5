/*
 * ps_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of what the hot path
 * computes: the sequential application of Pauli rotations exp(i*phi*P) to a
 * full state vector of 2^n complex amplitudes, in fp64.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (paper_2504_17881_b200/) never links, imports or executes it, and this file
 * shares no code, header, table or helper with it.
 *
 * Citations are to /root/reference/PAPER.md line numbers ("P:n") and the
 * section they fall in.
 *
 *   - State: a_i, i = 0..2^n-1, |psi> = sum_i a_i |i>                 P:350-354 (Mathematical model)
 *   - Pauli string P = P_1 (x) ... (x) P_n, P_k in {I, sx, sy, sz}     P:90-93   (Introduction)
 *   - Factor k acts on bit k-1 of the basis index: the worked example
 *     sx (x) I (x) sy -> p1 = (101)_2 = 5, p2 = (100)_2 = 4            P:483-484 (Mathematical model)
 *   - Rotation: exp(i phi P) = cos(phi) I + i sin(phi) P               P:96-97   (Introduction)
 *   - Sequence: rotations are applied in array order (index 0 first);
 *     the paper does not fix the product order (reading R7).
 *
 * Deliberately NOT used here (so the oracle shares no trick with the GPU path):
 * popcount / parity of masks, the i^(#Y) constant, pair enumeration by bit
 * insertion, in-place pair updates.  Each basis index is decoded qubit by
 * qubit with the 2x2 Pauli matrices written out, into a second vector.
 *
 * Build: gcc -O2 -ffp-contract=off -fopenmp -shared -fPIC (see oracle/build.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* factor codes, one byte per qubit: word letter -> code */
enum { F_I = 0, F_X = 1, F_Y = 2, F_Z = 3 };

/*
 * Decode the paper's two-integer representation (p1, p2) into factor codes.
 * bit k-1 of p1 is set iff P_k is not diagonal (sx or sy);
 *            bit k-1 of p2 is set iff P_k in {sy, sz}.
 * factors[l*n + q] receives the factor acting on qubit q (= P_{q+1}).
 * Returns 0, or -1 if a mask has a bit at position >= n.
 */
int oracle_decode_masks(int n, size_t count, const uint64_t *p1, const uint64_t *p2,
                        uint8_t *factors) {
    for (size_t l = 0; l < count; ++l) {
        for (int q = n; q < 64; ++q) {
            if (((p1[l] >> q) & 1u) || ((p2[l] >> q) & 1u)) return -1;
        }
        for (int q = 0; q < n; ++q) {
            int b1 = (int)((p1[l] >> q) & 1u);
            int b2 = (int)((p2[l] >> q) & 1u);
            uint8_t f;
            if (b1 == 0 && b2 == 0) f = F_I;
            else if (b1 == 1 && b2 == 0) f = F_X;
            else if (b1 == 1 && b2 == 1) f = F_Y;
            else f = F_Z;
            factors[l * (size_t)n + q] = f;
        }
    }
    return 0;
}

/*
 * Action of one Pauli string on one basis state |i>: P|i> = w |j>.
 * Worked out from the 2x2 matrices, qubit by qubit:
 *   I|b> = |b>;  sx|b> = |1-b>;  sy|0> = i|1>, sy|1> = -i|0>;  sz|b> = (-1)^b |b>.
 * The phase w is accumulated as a complex number (wr, wi).
 */
static void pauli_on_basis(int n, const uint8_t *f, uint64_t i, uint64_t *j_out,
                           double *wr_out, double *wi_out) {
    uint64_t j = i;
    double wr = 1.0, wi = 0.0;
    for (int q = 0; q < n; ++q) {
        uint64_t bit = (uint64_t)1 << q;
        int b = (i & bit) ? 1 : 0;
        double tr, ti;
        switch (f[q]) {
        case F_I:
            break;
        case F_X:
            j ^= bit;
            break;
        case F_Y:
            j ^= bit;
            if (b == 0) { /* multiply by +i */
                tr = -wi; ti = wr;
            } else {      /* multiply by -i */
                tr = wi; ti = -wr;
            }
            wr = tr; wi = ti;
            break;
        case F_Z:
            if (b == 1) { wr = -wr; wi = -wi; }
            break;
        default:
            break;
        }
    }
    *j_out = j;
    *wr_out = wr;
    *wi_out = wi;
}

/*
 * (P a) for one Pauli string, out of place: out_j = sum_i <j|P|i> a_i = w(i) a_i with j = j(i).
 * amp and out are interleaved (re, im) arrays of 2^n complex numbers.
 */
static void pauli_apply(int n, const uint8_t *f, const double *amp, double *out) {
    const int64_t dim = (int64_t)1 << n;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < dim; ++i) {
        uint64_t j;
        double wr, wi;
        pauli_on_basis(n, f, (uint64_t)i, &j, &wr, &wi);
        double ar = amp[2 * i], ai = amp[2 * i + 1];
        out[2 * j] = wr * ar - wi * ai;
        out[2 * j + 1] = wr * ai + wi * ar;
    }
}

/*
 * Apply rotations exp(i phi_l P_l), l = 0..count-1 in array order, to amp (in place from the
 * caller's view).  exp(i phi P) a = cos(phi) a + i sin(phi) (P a).
 * factors: count*n codes (qubit q of rotation l at [l*n+q]); angle: count radians.
 * Returns 0 or -1 on allocation failure.
 */
int oracle_apply_factors(int n, double *amp, size_t count, const uint8_t *factors,
                         const double *angle) {
    const int64_t dim = (int64_t)1 << n;
    double *pa = (double *)malloc(sizeof(double) * 2 * (size_t)dim);
    if (!pa) return -1;
    for (size_t l = 0; l < count; ++l) {
        const uint8_t *f = factors + l * (size_t)n;
        double c = cos(angle[l]);
        double s = sin(angle[l]);
        pauli_apply(n, f, amp, pa);
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < dim; ++i) {
            double ar = amp[2 * i], ai = amp[2 * i + 1];
            double pr = pa[2 * i], pi = pa[2 * i + 1];
            /* c*a + i*s*(P a):  i*(pr + i pi) = -pi + i pr */
            amp[2 * i] = c * ar - s * pi;
            amp[2 * i + 1] = c * ai + s * pr;
        }
    }
    free(pa);
    return 0;
}

/* out = P a for a single Pauli string (exposed for expectation values and tests). */
int oracle_pauli_apply(int n, const uint8_t *factors, const double *amp, double *out) {
    pauli_apply(n, factors, amp, out);
    return 0;
}

/* sum_i |a_i|^2 */
double oracle_norm(int n, const double *amp) {
    const int64_t dim = (int64_t)1 << n;
    double acc = 0.0;
    for (int64_t i = 0; i < dim; ++i) acc += amp[2 * i] * amp[2 * i] + amp[2 * i + 1] * amp[2 * i + 1];
    return acc;
}

/* <a|b> = sum_i conj(a_i) b_i, result in out[0] (re), out[1] (im). */
void oracle_inner(int n, const double *a, const double *b, double *out) {
    const int64_t dim = (int64_t)1 << n;
    double re = 0.0, im = 0.0;
    for (int64_t i = 0; i < dim; ++i) {
        double ar = a[2 * i], ai = a[2 * i + 1], br = b[2 * i], bi = b[2 * i + 1];
        re += ar * br + ai * bi;
        im += ar * bi - ai * br;
    }
    out[0] = re;
    out[1] = im;
}

/*
 * sum_l coeff_l * Re <psi|P_l|psi>: the energy-type expectation the application layer reads
 * (P:560-566 H = sum_l h_l P_l; P:667-671 signals are overlaps with |psi>).  Plain: form P|psi>,
 * take the inner product.  Returns 0 or -1 on allocation failure.
 */
int oracle_expectation(int n, const double *amp, size_t count, const uint8_t *factors,
                       const double *coeff, double *out) {
    const int64_t dim = (int64_t)1 << n;
    double *pa = (double *)malloc(sizeof(double) * 2 * (size_t)dim);
    if (!pa) return -1;
    double total = 0.0;
    for (size_t l = 0; l < count; ++l) {
        double ip[2];
        pauli_apply(n, factors + l * (size_t)n, amp, pa);
        oracle_inner(n, amp, pa, ip);
        total += coeff[l] * ip[0];
    }
    free(pa);
    *out = total;
    return 0;
}

/*
 * Seeded synthetic amplitudes (input generation, not the method): the counter-based
 * generator specified in DESIGN.md "Input recipe".  Both this oracle and the CUDA
 * init kernel implement it independently from that text.
 *   h(seed, k): z = seed + (k+1)*0x9E3779B97F4A7C15 (mod 2^64);
 *               z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9;
 *               z = (z ^ (z >> 27)) * 0x94D049BB133111EB;
 *               z =  z ^ (z >> 31)
 *   u(seed, k) = (z >> 11) * 2^-52 - 1      (exact in fp64, in [-1, 1))
 *   a_i = u(seed, 2i) + i u(seed, 2i+1)
 */
static double u_of(uint64_t seed, uint64_t k) {
    uint64_t z = seed + (k + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z = z ^ (z >> 31);
    return (double)(z >> 11) * (1.0 / 4503599627370496.0) - 1.0;
}

void oracle_random_amplitudes(uint64_t seed, uint64_t first, uint64_t count, double *out) {
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < (int64_t)count; ++t) {
        uint64_t i = first + (uint64_t)t;
        out[2 * t] = u_of(seed, 2 * i);
        out[2 * t + 1] = u_of(seed, 2 * i + 1);
    }
}

/* raw 64-bit output of the generator, for pinning it against published splitmix64 values */
uint64_t oracle_generator_raw(uint64_t seed, uint64_t k) {
    uint64_t z = seed + (k + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/*
 * Coset oracle for sizes whose full state does not fit the host (34-36 qubits).
 * Every rotation maps the coset C = i0 + span_GF(2){x_l} onto itself (P|i> is proportional
 * to |i xor p1>), so the restriction of the sequential product to C is exact.
 * The caller passes the coset members explicitly (members[0..m-1], any order, distinct,
 * closed under xor with every p1) and their initial amplitudes; the oracle applies the
 * rotations by the same per-qubit decode as above, looking partners up by binary search
 * in a sorted copy.  Returns 0, -1 on allocation failure, -2 if a partner is not a member.
 */
static int cmp_u64(const void *a, const void *b) {
    uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return (x > y) - (x < y);
}

int oracle_apply_coset(int n, size_t m, const uint64_t *members, double *amp, size_t count,
                       const uint8_t *factors, const double *angle) {
    uint64_t *key = (uint64_t *)malloc(sizeof(uint64_t) * m);
    size_t *pos = (size_t *)malloc(sizeof(size_t) * m);
    double *pa = (double *)malloc(sizeof(double) * 2 * m);
    double *tmp = (double *)malloc(sizeof(double) * 2 * m);
    if (!key || !pos || !pa || !tmp) { free(key); free(pos); free(pa); free(tmp); return -1; }
    /* sorted copy of the member indices; pos[k] = caller slot of key[k] */
    for (size_t t = 0; t < m; ++t) key[t] = members[t];
    qsort(key, m, sizeof(uint64_t), cmp_u64);
    for (size_t t = 0; t < m; ++t) {
        size_t lo = 0, hi = m;
        while (lo < hi) { size_t mid = (lo + hi) / 2; if (key[mid] < members[t]) lo = mid + 1; else hi = mid; }
        pos[lo] = t;
    }
    int rc = 0;
    for (size_t l = 0; l < count && rc == 0; ++l) {
        const uint8_t *f = factors + l * (size_t)n;
        double c = cos(angle[l]), s = sin(angle[l]);
        for (size_t t = 0; t < m && rc == 0; ++t) {
            uint64_t j;
            double wr, wi;
            pauli_on_basis(n, f, members[t], &j, &wr, &wi);
            size_t lo = 0, hi = m;
            while (lo < hi) { size_t mid = (lo + hi) / 2; if (key[mid] < j) lo = mid + 1; else hi = mid; }
            if (lo >= m || key[lo] != j) { rc = -2; break; }
            size_t u = pos[lo];
            double ar = amp[2 * t], ai = amp[2 * t + 1];
            pa[2 * u] = wr * ar - wi * ai;
            pa[2 * u + 1] = wr * ai + wi * ar;
        }
        if (rc) break;
        for (size_t t = 0; t < m; ++t) {
            double ar = amp[2 * t], ai = amp[2 * t + 1];
            tmp[2 * t] = c * ar - s * pa[2 * t + 1];
            tmp[2 * t + 1] = c * ai + s * pa[2 * t];
        }
        memcpy(amp, tmp, sizeof(double) * 2 * m);
    }
    free(key); free(pos); free(pa); free(tmp);
    return rc;
}
