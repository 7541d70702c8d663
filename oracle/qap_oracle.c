/*
 * qap_oracle.c -- CPU restatement of the reference PSO hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product path in paper_1504_05158_b200/.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  The
 * product never links or calls it.
 *
 * Every function restates one reference routine (paths relative to
 * /root/reference/pkg/src/qapswarm/) in plain C, with the same loop order and
 * the same floating-point operation order (built with -ffp-contract=off so no
 * multiply-add is fused, matching numba/LLVM's default):
 *
 *   orc_philox4x64_10      numpy Philox4x64-10 block (numpy bit generator used
 *                          by streams.phase_rng, streams.py:38-40)
 *   orc_step_draws         streams.step_draws          (streams.py:53-64)
 *   orc_velocity_many      _batch.velocity_many        (_batch.py:30-58)
 *   orc_aggregate_many     _batch.aggregate_many /     (_batch.py:61-183)
 *                          _aggregate_one
 *   orc_cost_many_{i64,f64}_batch.cost_many            (_batch.py:186-197)
 *
 * The aggregation is the reference's O(n^3) rescan, deliberately NOT the
 * incremental algorithm the CUDA kernel uses, so the two are independent.
 * Particles are independent, so the outer loops run under OpenMP exactly like
 * the reference's numba prange; results do not depend on the thread count.
 */
#include <stdint.h>
#include <string.h>
#include <math.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define PH_M0 0xD2E7470EE14C6C93ULL
#define PH_M1 0xCA5A826395121157ULL
#define PH_W0 0x9E3779B97F4A7C15ULL
#define PH_W1 0xBB67AE8584CAA73BULL

static inline void mulhilo64(uint64_t a, uint64_t b, uint64_t *hi, uint64_t *lo) {
    unsigned __int128 p = (unsigned __int128)a * b;
    *hi = (uint64_t)(p >> 64);
    *lo = (uint64_t)p;
}

/* numpy/random123 Philox4x64 with 10 rounds.  ctr/out may alias. */
void orc_philox4x64_10(const uint64_t ctr_in[4], const uint64_t key_in[2], uint64_t out[4]) {
    uint64_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint64_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; ++r) {
        if (r) { k0 += PH_W0; k1 += PH_W1; }
        uint64_t hi0, lo0, hi1, lo1;
        mulhilo64(PH_M0, c0, &hi0, &lo0);
        mulhilo64(PH_M1, c2, &hi1, &lo1);
        uint64_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* The idx-th double of a freshly keyed numpy Generator(Philox(key)).random():
 * numpy pre-increments the 256-bit counter before each 4-word block, so word
 * idx comes from counter (idx/4 + 1, 0, 0, 0), lane idx % 4; random() is
 * (u64 >> 11) * 2^-53 (numpy's next_double). */
double orc_uniform_at(uint64_t seed, uint64_t word1, uint64_t idx) {
    uint64_t key[2] = {seed, word1};
    uint64_t ctr[4] = {idx / 4 + 1, 0, 0, 0};
    uint64_t out[4];
    orc_philox4x64_10(ctr, key, out);
    return (double)(out[idx % 4] >> 11) * (1.0 / 9007199254740992.0);
}

/* streams.step_draws (streams.py:53-64): key = (seed, PHASE_STEP<<56 | t<<24)
 * (streams.py:30-35), rows p0..p0+P-1 of the (Ptotal, 2+2n) block. */
void orc_step_draws(uint64_t seed, uint64_t t, int64_t p0, int64_t P, int n, double *out) {
    const uint64_t word1 = (2ULL << 56) | (t << 24);
    const int64_t w = 2 + 2 * (int64_t)n;
    #pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < P; ++p) {
        uint64_t key[2] = {seed, word1};
        uint64_t blk[4];
        uint64_t cur = UINT64_MAX;
        for (int64_t c = 0; c < w; ++c) {
            uint64_t idx = (uint64_t)((p0 + p) * w + c);
            if (idx / 4 != cur) {
                uint64_t ctr[4] = {idx / 4 + 1, 0, 0, 0};
                orc_philox4x64_10(ctr, key, blk);
                cur = idx / 4;
            }
            out[p * w + c] = (double)(blk[idx % 4] >> 11) * (1.0 / 9007199254740992.0);
        }
    }
}

/* _batch.velocity_many (_batch.py:30-58), in place on v (P,n,n). */
void orc_velocity_many(double *v, const int8_t *x, const int8_t *pl, const int8_t *pg,
                       int64_t P, int n, int64_t swarm_size, double c1,
                       const double *c2r2, const double *c3r3, double v_max, int normalize) {
    const int64_t nn = (int64_t)n * n;
    #pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < P; ++p) {
        const int64_t s = p / swarm_size;
        double *vp = v + p * nn;
        const int8_t *xp = x + p * nn, *plp = pl + p * nn, *pgp = pg + s * nn;
        for (int i = 0; i < n; ++i) {
            for (int j = 0; j < n; ++j) {
                const int64_t e = (int64_t)i * n + j;
                double lin = c1 * vp[e]
                           + c2r2[p] * ((double)plp[e] - (double)xp[e])
                           + c3r3[p] * ((double)pgp[e] - (double)xp[e]);
                if (lin > v_max) lin = v_max;
                else if (lin < -v_max) lin = -v_max;
                vp[e] = lin;
            }
        }
        if (normalize) {
            for (int j = 0; j < n; ++j) {
                double total = 0.0;
                for (int i = 0; i < n; ++i) total += fabs(vp[(int64_t)i * n + j]);
                if (total > 0.0)
                    for (int i = 0; i < n; ++i) vp[(int64_t)i * n + j] = vp[(int64_t)i * n + j] / total;
            }
        }
    }
}

#define MODE_GLOBAL_MAX 0
#define MODE_PICK_COLUMN 1
#define MODE_SECOND_TARGET 2

/* _batch._aggregate_one (_batch.py:61-175): one particle; consumes draws
 * left to right.  m, order, row_free, col_free are caller scratch. */
static void aggregate_one(const int8_t *x, const double *v, int n, int mode, int depth,
                          const double *draws, int8_t *out_mat, int64_t *out_perm,
                          double *m, int64_t *order, uint8_t *row_free, uint8_t *col_free) {
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            m[i * n + j] = (double)x[i * n + j] + v[i * n + j];
            out_mat[i * n + j] = 0;
        }
    memset(row_free, 1, n);
    memset(col_free, 1, n);
    int cursor = 0;
    for (int i = 0; i < n; ++i) order[i] = i;
    if (mode == MODE_PICK_COLUMN) {
        for (int i = n - 1; i > 0; --i) {
            double u = draws[cursor++];
            int64_t j = (int64_t)(u * (double)(i + 1));
            if (j > i) j = i;
            int64_t tmp = order[i]; order[i] = order[j]; order[j] = tmp;
        }
    }
    for (int rnd = 0; rnd < n; ++rnd) {
        int restrict_ = (mode == MODE_SECOND_TARGET) && rnd < depth;
        double best = -INFINITY;
        int64_t count = 0;
        if (mode == MODE_PICK_COLUMN) {
            int64_t c = order[rnd];
            for (int r = 0; r < n; ++r) {
                if (!row_free[r]) continue;
                double val = m[r * n + c];
                if (val > best) { best = val; count = 1; }
                else if (val == best) count++;
            }
        } else {
            for (int r = 0; r < n; ++r) {
                if (!row_free[r]) continue;
                for (int c = 0; c < n; ++c) {
                    if (!col_free[c]) continue;
                    if (restrict_ && x[r * n + c] == 1) continue;
                    double val = m[r * n + c];
                    if (val > best) { best = val; count = 1; }
                    else if (val == best) count++;
                }
            }
            if (count == 0) {  /* every remaining cell excluded: unrestricted fallback */
                restrict_ = 0;
                for (int r = 0; r < n; ++r) {
                    if (!row_free[r]) continue;
                    for (int c = 0; c < n; ++c) {
                        if (!col_free[c]) continue;
                        double val = m[r * n + c];
                        if (val > best) { best = val; count = 1; }
                        else if (val == best) count++;
                    }
                }
            }
        }
        int64_t pick = 0;
        if (count > 1) {
            double u = draws[cursor++];
            pick = (int64_t)(u * (double)count);
            if (pick >= count) pick = count - 1;
        }
        int64_t seen = 0;
        int sel_r = -1, sel_c = -1;
        if (mode == MODE_PICK_COLUMN) {
            int c = (int)order[rnd];
            for (int r = 0; r < n; ++r) {
                if (row_free[r] && m[r * n + c] == best) {
                    if (seen == pick) { sel_r = r; sel_c = c; break; }
                    seen++;
                }
            }
        } else {
            for (int r = 0; r < n && sel_r < 0; ++r) {
                if (!row_free[r]) continue;
                for (int c = 0; c < n; ++c) {
                    if (!col_free[c]) continue;
                    if (restrict_ && x[r * n + c] == 1) continue;
                    if (m[r * n + c] == best) {
                        if (seen == pick) { sel_r = r; sel_c = c; break; }
                        seen++;
                    }
                }
            }
        }
        out_mat[sel_r * n + sel_c] = 1;
        out_perm[sel_c] = sel_r;
        row_free[sel_r] = 0;
        col_free[sel_c] = 0;
    }
}

/* _batch.aggregate_many (_batch.py:178-183).  draws row p starts at
 * draws + p*draws_stride (the reference passes the (P, 2n) tail of
 * step_draws, i.e. stride 2+2n offset 2, or a plain (P, 2n) array). */
void orc_aggregate_many(const int8_t *x, const double *v, int64_t P, int n, int mode, int depth,
                        const double *draws, int64_t draws_stride,
                        int8_t *out_mat, int64_t *out_perm) {
    const int64_t nn = (int64_t)n * n;
    #pragma omp parallel
    {
        double *m = (double *)malloc(sizeof(double) * nn);
        int64_t *order = (int64_t *)malloc(sizeof(int64_t) * n);
        uint8_t *rf = (uint8_t *)malloc(n), *cf = (uint8_t *)malloc(n);
        #pragma omp for schedule(static)
        for (int64_t p = 0; p < P; ++p)
            aggregate_one(x + p * nn, v + p * nn, n, mode, depth, draws + p * draws_stride,
                          out_mat + p * nn, out_perm + p * n, m, order, rf, cf);
        free(m); free(order); free(rf); free(cf);
    }
}

/* _batch.cost_many (_batch.py:186-197), integer instances: int64 products
 * and sums (two's-complement wrap, as numba's int64). */
void orc_cost_many_i64(const int64_t *perms, const int64_t *flow, const int64_t *dist,
                       int64_t *out, int64_t P, int n) {
    #pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < P; ++p) {
        uint64_t acc = 0;
        const int64_t *pp = perms + p * n;
        for (int i = 0; i < n; ++i) {
            int64_t a = pp[i];
            for (int j = 0; j < n; ++j)
                acc += (uint64_t)flow[i * n + j] * (uint64_t)dist[a * n + pp[j]];
        }
        out[p] = (int64_t)acc;
    }
}

/* Same for float instances: sequential i-major, j-minor, no contraction. */
void orc_cost_many_f64(const int64_t *perms, const double *flow, const double *dist,
                       double *out, int64_t P, int n) {
    #pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < P; ++p) {
        double acc = flow[0] * dist[0] * 0.0;
        const int64_t *pp = perms + p * n;
        for (int i = 0; i < n; ++i) {
            int64_t a = pp[i];
            for (int j = 0; j < n; ++j) acc += flow[i * n + j] * dist[a * n + pp[j]];
        }
        out[p] = acc;
    }
}

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void orc_set_num_threads(int k) {
#ifdef _OPENMP
    if (k > 0) omp_set_num_threads(k);
#else
    (void)k;
#endif
}

/* 2-opt (pairwise facility exchange) local search.  NOT in the reference
 * (SPEC.md:148 lists delta evaluation as a non-goal):
 * this is the north-star extension, and this function is its CPU oracle.
 * Policy, per pass: evaluate every swap (r, s), r < s, with the exact
 * integer delta; take the smallest delta, ties to
 * the lexicographically first (r, s); apply it if it is negative, else stop.
 * Costs use int64 wrap-around arithmetic like cost_many. */
void orc_twoopt_many(int64_t *perms, const int64_t *F, const int64_t *D, int64_t *costs,
                     int64_t P, int n, int passes) {
    #pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < P; ++p) {
        int64_t *pp = perms + p * n;
        for (int pass = 0; pass < passes; ++pass) {
            int64_t best = INT64_MAX;
            int br = -1, bs = -1;
            for (int r = 0; r < n; ++r) {
                for (int s = r + 1; s < n; ++s) {
                    const int64_t pr = pp[r], ps = pp[s];
                    uint64_t d = (uint64_t)(F[r * n + r] - F[s * n + s]) * (uint64_t)(D[ps * n + ps] - D[pr * n + pr])
                               + (uint64_t)(F[r * n + s] - F[s * n + r]) * (uint64_t)(D[ps * n + pr] - D[pr * n + ps]);
                    for (int k = 0; k < n; ++k) {
                        if (k == r || k == s) continue;
                        const int64_t pk = pp[k];
                        d += (uint64_t)(F[k * n + r] - F[k * n + s]) * (uint64_t)(D[pk * n + ps] - D[pk * n + pr])
                           + (uint64_t)(F[r * n + k] - F[s * n + k]) * (uint64_t)(D[ps * n + pk] - D[pr * n + pk]);
                    }
                    if ((int64_t)d < best) { best = (int64_t)d; br = r; bs = s; }
                }
            }
            if (br < 0 || best >= 0) break;
            const int64_t t = pp[br]; pp[br] = pp[bs]; pp[bs] = t;
            costs[p] = (int64_t)((uint64_t)costs[p] + (uint64_t)best);
        }
    }
}
