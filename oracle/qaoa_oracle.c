/*
 * qaoa_oracle.c -- CPU restatement of the reference QAOA Max-Cut hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2312_03019_b200/)
 * links, loads or calls this file.  It is the checker that tests/, the
 * __graft_entry__.smoke() self-check and bench.py's cpu_baseline / --impl
 * reference leg compare the CUDA path against.  Parity is pinned: the
 * restatement is checked against golden vectors produced by running the
 * reference itself (tests/golden/make_golden.py writes the fixtures).
 *
 * Every function cites the reference file:line it restates
 * (paths relative to /root/reference/pkg/src/qaoa_maxcut/).
 *
 * Arithmetic contract (bit-exact with the reference on an FMA-capable host):
 *   cost   : amp *= table[E - 2C(x) + E]  with numpy's FMA-form complex multiply
 *            re = fma(ar, pr, -(ai*pi)),  im = fma(ar, pi, ai*pr)
 *   mixer  : RX(-beta) on q = 0..n-1 in increasing order, each product rounded
 *            separately then one add (state.py:118-124 evaluates c*a + ms*b,
 *            where c*a and ms*b each have one exactly-zero cross term).
 * Compile with -ffp-contract=off so gcc never fuses the mixer's mul+add.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_EXPORT __attribute__((visibility("default")))

static int set_threads(int threads) {
#ifdef _OPENMP
    if (threads <= 0) threads = omp_get_max_threads();
    return threads;
#else
    (void)threads;
    return 1;
#endif
}

/* Cut count of one basis state: cost.py:122-128 (cut_edge_count_bitwise) built
 * from the row step cost.py:55-63: popcount(row_mask[i] & (bcast(b_i) ^ b)). */
static inline int64_t cut_count_one(int n, const uint64_t* row_mask, uint64_t b) {
    int64_t c = 0;
    for (int i = 0; i < n; ++i) {
        uint64_t bcast = (uint64_t)0 - ((b >> i) & 1u);   /* broadcast_bit cost.py:49-52 */
        c += __builtin_popcountll(row_mask[i] & (bcast ^ b));
    }
    return c;
}

/* CompressedCostPlan.cut_counts, cost.py:88-99: int64 C(x) for x in [0, 2^n). */
ORC_EXPORT void orc_cut_counts(int n, const uint64_t* row_mask, int64_t* out, int threads) {
    const int64_t size = (int64_t)1 << n;
    threads = set_threads(threads);
#pragma omp parallel for schedule(static) num_threads(threads)
    for (int64_t x = 0; x < size; ++x) out[x] = cut_count_one(n, row_mask, (uint64_t)x);
}

/* init_uniform, circuit.py:42-48: one correctly rounded sqrt(1/2^n), imag 0. */
ORC_EXPORT void orc_init_uniform(int n, double* amps, int threads) {
    const int64_t size = (int64_t)1 << n;
    const double u = sqrt(1.0 / (double)((uint64_t)1 << n));
    threads = set_threads(threads);
#pragma omp parallel for schedule(static) num_threads(threads)
    for (int64_t x = 0; x < size; ++x) { amps[2 * x] = u; amps[2 * x + 1] = 0.0; }
}

/* apply_cost_bitwise, cost.py:162-176: amps[x] *= table[(E - 2C(x)) + E],
 * table = _phase_table(E, gamma) (cost.py:136-139), supplied by the caller as
 * interleaved (re, im) pairs of length 2E+1.  Complex multiply in numpy's
 * FMA form (measured on the survey host). */
ORC_EXPORT void orc_apply_cost(int n, const uint64_t* row_mask, int tot_edge,
                               const double* table, double* amps, int threads) {
    const int64_t size = (int64_t)1 << n;
    threads = set_threads(threads);
#pragma omp parallel for schedule(static) num_threads(threads)
    for (int64_t x = 0; x < size; ++x) {
        const int64_t c = cut_count_one(n, row_mask, (uint64_t)x);
        const int64_t k = (int64_t)tot_edge - 2 * c + tot_edge;
        const double pr = table[2 * k], pi = table[2 * k + 1];
        const double ar = amps[2 * x], ai = amps[2 * x + 1];
        amps[2 * x] = fma(ar, pr, -(ai * pi));
        amps[2 * x + 1] = fma(ar, pi, ai * pr);
    }
}

/* apply_rx, state.py:110-128 with theta = -beta (circuit.py:93):
 *   c = cos(theta/2), s = sin(theta/2), ms = -1j*s  (state.py:114-115)
 *   top = c*a + ms*b ; bot = ms*a + c*b            (state.py:121-124)
 * which rounds to  top = (c*ar + s*bi, c*ai + (-s)*br),
 *                  bot = (s*ai + c*br, (-s)*ar + c*bi).
 * The caller passes c and s as Python's math.cos / math.sin produce them. */
ORC_EXPORT void orc_apply_rx(int n, int q, double c, double s, double* amps, int threads) {
    const int64_t half = (int64_t)1 << (n - 1);
    const int64_t stride = (int64_t)1 << q;
    const double ns = -s;
    threads = set_threads(threads);
#pragma omp parallel for schedule(static) num_threads(threads)
    for (int64_t k = 0; k < half; ++k) {
        const int64_t lo = k & (stride - 1);
        const int64_t i0 = ((k >> q) << (q + 1)) | lo;   /* bit q == 0 */
        const int64_t i1 = i0 | stride;                  /* bit q == 1 */
        const double ar = amps[2 * i0], ai = amps[2 * i0 + 1];
        const double br = amps[2 * i1], bi = amps[2 * i1 + 1];
        const double tr = c * ar + s * bi;
        const double ti = c * ai + ns * br;
        const double ur = s * ai + c * br;
        const double ui = ns * ar + c * bi;
        amps[2 * i0] = tr; amps[2 * i0 + 1] = ti;
        amps[2 * i1] = ur; amps[2 * i1 + 1] = ui;
    }
}

/* apply_h, state.py:91-107: top = (a + b) * k, bot = (a - b) * k with
 * k = 1.0 / sqrt(2.0) (state.py:22); numpy multiplies by the scalar as a
 * complex (k, 0): re*k - im*0 has the value re*k. */
ORC_EXPORT void orc_apply_h(int n, int q, double* amps, int threads) {
    const int64_t half = (int64_t)1 << (n - 1);
    const int64_t stride = (int64_t)1 << q;
    const double k = 1.0 / sqrt(2.0);
    threads = set_threads(threads);
#pragma omp parallel for schedule(static) num_threads(threads)
    for (int64_t j = 0; j < half; ++j) {
        const int64_t i0 = ((j >> q) << (q + 1)) | (j & (stride - 1));
        const int64_t i1 = i0 | stride;
        const double ar = amps[2 * i0], ai = amps[2 * i0 + 1];
        const double br = amps[2 * i1], bi = amps[2 * i1 + 1];
        amps[2 * i0] = (ar + br) * k; amps[2 * i0 + 1] = (ai + bi) * k;
        amps[2 * i1] = (ar - br) * k; amps[2 * i1 + 1] = (ai - bi) * k;
    }
}

/* apply_rzz, state.py:131-149: amps *= where(bit q1 != bit q2, e_diff, e_same),
 * phases = {e_same.re, e_same.im, e_diff.re, e_diff.im} as numpy forms them;
 * numpy's FMA-form complex multiply (as in orc_apply_cost). */
ORC_EXPORT void orc_apply_rzz(int n, int q1, int q2, const double* phases, double* amps,
                              int threads) {
    const int64_t size = (int64_t)1 << n;
    threads = set_threads(threads);
#pragma omp parallel for schedule(static) num_threads(threads)
    for (int64_t x = 0; x < size; ++x) {
        const int d = (int)(((x >> q1) ^ (x >> q2)) & 1);
        const double pr = phases[2 * d], pi = phases[2 * d + 1];
        const double ar = amps[2 * x], ai = amps[2 * x + 1];
        amps[2 * x] = fma(ar, pr, -(ai * pi));
        amps[2 * x + 1] = fma(ar, pi, ai * pr);
    }
}

/* apply_mixer_layer, circuit.py:89-94: RX on every qubit, q = 0..n-1 in order. */
ORC_EXPORT void orc_apply_mixer(int n, double c, double s, double* amps, int threads) {
    for (int q = 0; q < n; ++q) orc_apply_rx(n, q, c, s, amps, threads);
}

/* simulate(..., backend="bitwise", launch_control=True), circuit.py:97-113:
 * init_uniform, then p x (cost layer, mixer layer).  tables holds p phase tables
 * of 2E+1 complex entries each; c[l], s[l] are cos/sin(-beta_l/2). */
ORC_EXPORT void orc_simulate(int n, const uint64_t* row_mask, int tot_edge, int p,
                             const double* tables, const double* c, const double* s,
                             double* amps, int threads) {
    orc_init_uniform(n, amps, threads);
    for (int l = 0; l < p; ++l) {
        orc_apply_cost(n, row_mask, tot_edge, tables + (size_t)l * 2 * (2 * tot_edge + 1), amps,
                       threads);
        orc_apply_mixer(n, c[l], s[l], amps, threads);
    }
}

/* expectation, circuit.py:116-121 with cut_values_array graph.py:144-151:
 * sum_x |a_x|^2 * C(x) for an unweighted graph.  numpy's pairwise sum cannot be
 * bit-matched; blocked double summation here (contract: 1e-10 relative). */
ORC_EXPORT double orc_expectation(int n, const uint64_t* row_mask, const double* amps,
                                  int threads) {
    const int64_t size = (int64_t)1 << n;
    const int64_t block = 1 << 12;
    const int64_t nblocks = (size + block - 1) / block;
    double* partial = (double*)calloc((size_t)nblocks, sizeof(double));
    threads = set_threads(threads);
#pragma omp parallel for schedule(static) num_threads(threads)
    for (int64_t b = 0; b < nblocks; ++b) {
        double acc = 0.0;
        const int64_t hi = (b + 1) * block < size ? (b + 1) * block : size;
        for (int64_t x = b * block; x < hi; ++x) {
            const double ar = amps[2 * x], ai = amps[2 * x + 1];
            acc += (ar * ar + ai * ai) * (double)cut_count_one(n, row_mask, (uint64_t)x);
        }
        partial[b] = acc;
    }
    double total = 0.0;
    for (int64_t b = 0; b < nblocks; ++b) total += partial[b];
    free(partial);
    return total;
}

/* Shard variants for the sharded-host tests: the local state holds global
 * basis indices x_hi | y (y < 2^n_local) of an n_nodes-node graph.  Same
 * arithmetic as orc_apply_cost / orc_expectation (cost.py:162-176,
 * circuit.py:116-121). */
ORC_EXPORT void orc_apply_cost_x(int n_local, int n_nodes, const uint64_t* row_mask, uint64_t x_hi,
                                 int tot_edge, const double* table, double* amps, int threads) {
    const int64_t size = (int64_t)1 << n_local;
    threads = set_threads(threads);
#pragma omp parallel for schedule(static) num_threads(threads)
    for (int64_t y = 0; y < size; ++y) {
        const int64_t c = cut_count_one(n_nodes, row_mask, x_hi | (uint64_t)y);
        const int64_t k = (int64_t)tot_edge - 2 * c + tot_edge;
        const double pr = table[2 * k], pi = table[2 * k + 1];
        const double ar = amps[2 * y], ai = amps[2 * y + 1];
        amps[2 * y] = fma(ar, pr, -(ai * pi));
        amps[2 * y + 1] = fma(ar, pi, ai * pr);
    }
}

ORC_EXPORT double orc_expectation_x(int n_local, int n_nodes, const uint64_t* row_mask,
                                    uint64_t x_hi, const double* amps, int threads) {
    const int64_t size = (int64_t)1 << n_local;
    double total = 0.0;
    threads = set_threads(threads);
#pragma omp parallel for schedule(static) reduction(+ : total) num_threads(threads)
    for (int64_t y = 0; y < size; ++y) {
        const double ar = amps[2 * y], ai = amps[2 * y + 1];
        total += (ar * ar + ai * ai) * (double)cut_count_one(n_nodes, row_mask, x_hi | (uint64_t)y);
    }
    return total;
}

/* StateVector.norm, state.py:50-51. */
ORC_EXPORT double orc_norm(int n, const double* amps, int threads) {
    const int64_t size = (int64_t)1 << n;
    double total = 0.0;
    threads = set_threads(threads);
#pragma omp parallel for schedule(static) reduction(+ : total) num_threads(threads)
    for (int64_t x = 0; x < size; ++x) total += amps[2 * x] * amps[2 * x] + amps[2 * x + 1] * amps[2 * x + 1];
    return sqrt(total);
}

ORC_EXPORT int orc_max_threads(void) { return set_threads(0); }
