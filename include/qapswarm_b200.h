/*
 * qapswarm_b200.h -- C ABI of the B200-native multi-swarm PSO step for QAP.
 *
 * Drop-in boundary for the reference package `qapswarm` (arXiv 1504.05158
 * restatement; paths below are relative to
 * /root/reference/pkg/src/qapswarm/).  The reference binds its hot path from
 * Python (engine.step, engine.py:196-208) to four numba kernels; this header
 * exposes the same operations with plain pointers and sizes, no torch types.
 *
 * Two tiers:
 *   1. Reference-layout, host-buffer entry points (qsb_velocity_many,
 *      qsb_aggregate_many, qsb_cost_many_*, qsb_step_draws_host): the same
 *      arguments, layouts and in-place semantics as _batch.velocity_many
 *      (_batch.py:30-58), _batch.aggregate_many (_batch.py:178-183),
 *      _batch.cost_many (_batch.py:186-197) and streams.step_draws
 *      (streams.py:53-64).  They copy host -> device -> host internally and
 *      are synchronous, like the numba calls they replace.
 *   2. Device-resident entry points on a qsb_state (caller-owned device
 *      buffers, stream-ordered, no allocation, graph-capturable) used by the
 *      Python engine: the fused step (phases 1-4a of engine.step), the
 *      swarm/global best reduction (engine.py:216-229), migration
 *      (migration.py:55-86) and helpers.
 *
 * Every function returns QSB_OK or an error code; qsb_strerror() names it.
 * Validation that the reference performs in Python (SolverConfig,
 * PsoCoefficients, engine.py:186-187 depth check) stays in the Python host
 * layer, which raises the reference's ValueError messages.
 */
#ifndef QAPSWARM_B200_H
#define QAPSWARM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QSB_OK 0
#define QSB_EINVAL 1        /* bad argument (size, dtype, null pointer) */
#define QSB_EUNSUPPORTED 2  /* shape not supported by any kernel variant */
#define QSB_ECUDA 3         /* CUDA runtime error (see qsb_last_cuda_error) */
#define QSB_EPERM 4         /* input matrix is not a permutation matrix */

/* element types */
#define QSB_F32 1
#define QSB_F64 2
#define QSB_I64 3
#define QSB_U16 4

/* step phase flags (qsb_step_phases) */
#define QSB_PHASE_VELOCITY 1
#define QSB_PHASE_AGGREGATE 2
#define QSB_PHASE_COST 4
#define QSB_PHASE_PBEST 8
#define QSB_PHASE_STORE_V 16

/* S_x modes, same codes as _batch.MODE_CODES (_batch.py:19-27) */
#define QSB_SX_GLOBAL_MAX 0
#define QSB_SX_PICK_COLUMN 1
#define QSB_SX_SECOND_TARGET 2

/* Device-resident particle state (engine.PopulationState, engine.py:85-124),
 * structure of arrays.  Positions are int16 permutations perm[c] = row of
 * the 1 in column c (core.py:5-6); the 0/1 matrices are never stored. */
typedef struct qsb_state {
  int32_t n;                 /* problem size */
  int32_t vstride;           /* V elements per particle (>= n*n, 16-byte multiple) */
  int32_t v_dtype;           /* QSB_F32 (throughput) or QSB_F64 (parity) */
  int32_t cost_dtype;        /* QSB_I64 (integral instance) or QSB_F64 */
  int64_t num_particles;     /* particles on this device */
  int64_t swarm_size;
  int64_t num_swarms;        /* swarms on this device */
  int64_t particle_offset;   /* global id of local particle 0 */
  int64_t swarm_offset;      /* global id of local swarm 0 */
  void* V;                   /* (P, vstride).  QSB_F64: doubles.  QSB_F32 in
                              * the lazily scaled layout (vcol set): "wide"
                              * 32-bit words, the high word of the double
                              * (sign, 11-bit exponent, 20-bit fraction)
                              * rounded to nearest (fp64's exponent range in
                              * fp32's size); QSB_F32 otherwise: floats. */
  int16_t* perm;             /* (P, n) current position X */
  int16_t* perm_new;         /* (P, n) next position */
  int16_t* pl_perm;          /* (P, n) personal best PL */
  void* cost;                /* (P,) goal of perm_new after a step */
  void* pl_cost;             /* (P,) */
  uint8_t* improved;         /* (P,) scratch: cost < pl_cost this step */
  int16_t* pg_perm;          /* (m, n) swarm best PG */
  void* pg_cost;             /* (m,) */
  int16_t* best_perm;        /* (n,) best solution seen on this device */
  void* best_cost;           /* (1,) */
  int64_t* best_iter;        /* (1,) iteration it first appeared */
  int64_t* best_idx;         /* (1,) global particle id it came from */
  int64_t* iteration;        /* (1,) completed iterations t */
  void* swarm_min;           /* (m,) scratch */
  int64_t* swarm_min_idx;    /* (m,) scratch */
  uint32_t* done;            /* (1,) scratch, zero-initialised */
  uint32_t* work;            /* (1,) scratch for dynamic particle scheduling, or NULL */
  /* Lazily scaled fp32 layout (optional; NULL = V holds v itself).  When set
   * (v_dtype QSB_F32, n <= 64), V holds u and the velocity is v = u * s
   * per column; vcol is (P, 5, vcs) 32-bit words with vcs = n rounded up to
   * a multiple of 4: row 0 the column scale s (a wide word, like V; 1.0 is
   * the bit pattern 0x3FF00000), rows 1-2 the low / high
   * words of the f64 sum of |u| over the column, row 3 the maximum of u over
   * the rows other than zp (a wide word, NaN = unknown), row 4 (int32) count << 16 |
   * first row << 8 | zp, zp being the z row (the position) of the step that
   * wrote them.  Set row 0 to 1.0 (0x3FF00000) and row 3 to NaN whenever V is
   * written from outside the step.  For n > 64 (multi-warp kernels) only row 0 is used:
   * the deferred column normalisation, V holds the unnormalised velocity u
   * (floats) and v = u * s. */
  float* vcol;
  /* (P, 2) scratch for the step's per-particle (c2 * r2, c3 * r3), drawn by a
   * one-thread-per-particle pre-pass; NULL = drawn inside the step kernel. */
  double* step_coef;
} qsb_state;

/* QAP instance on the device (qaplib.QapInstance, qaplib.py:28-69). */
typedef struct qsb_instance {
  int32_t n;
  int32_t mat_dtype;         /* QSB_U16, QSB_I64 or QSB_F64 */
  const void* flow;          /* (n, n) row-major */
  const void* distance;      /* (n, n) row-major */
  int32_t acc32;             /* 1 if n * max(flow) * max(distance) < 2^32 (caller-checked) */
  int32_t reserved;
} qsb_instance;

/* kernels.PsoCoefficients (kernels.py:47-76) plus the run seed. */
typedef struct qsb_coeffs {
  double c1, c2, c3, v_max;
  int32_t normalize;         /* sv_mode == "norm" */
  int32_t sx_mode;           /* QSB_SX_* */
  int32_t depth;
  int32_t hints;             /* QSB_HINT_* bits (caller-guaranteed properties) */
  uint64_t seed;             /* SolverConfig.seed wrapped to uint64 (streams.py:34) */
} qsb_coeffs;

/* |c1 * v| <= v_max holds for every stored velocity entry, so the clamp of
 * the rows untouched by x / pl / pg is a no-op and may be skipped. */
#define QSB_HINT_V_BOUNDED 1
/* st->cost[p] holds the goal of st->perm[p] on entry (true between engine
 * steps), so the new goal may be computed incrementally from the facilities
 * that moved (integral instances). */
#define QSB_HINT_COST_CURRENT 2
/* flow and distance are symmetric (integral instances): the incremental goal
 * counts the unmoved rows' column terms through the moved rows' row terms. */
#define QSB_HINT_SYMMETRIC 4
/* st->step_coef already holds this step's (c2 r2, c3 r3) and st->work is
 * zero: the previous step ended with qsb_best_update_next (same seed, c2,
 * c3), so qsb_step_phases launches no pre-pass. */
#define QSB_HINT_COEF_READY 8
/* Performance only (results are identical either way): the population is
 * past its first iterations, where a bulk step of the aggregation more often
 * leaves more than five free columns; selects the fused kernel variant that
 * chains further bulk steps against the stale column maxima instead of
 * rescanning (the engine sets it from iteration QSB_CHAIN_T0 on). */
#define QSB_HINT_LATE 16

/* One migration event (migration.migrate, migration.py:55-86). */
typedef struct qsb_migration {
  int32_t d;                 /* SolverConfig.migration_depth (engine.py:66-68) */
  int32_t period;            /* run when t % period == 0; 0 = unconditional */
  int32_t mode;              /* 0 single device, 1 plan+pack, 2 apply exchanged records */
  int32_t reserved;
  int64_t num_swarms_total;  /* m over all devices */
  const int32_t* picks;      /* (rows, d): host_rng(seed, t).integers(0, S) per event,
                              * or NULL: the kernel draws them from `seed` (below) */
  int64_t picks_epoch0;      /* epoch (t / period) of picks row 0 */
  int64_t picks_rows;
  const void* all_pg_cost;   /* (m_total,) swarm-best costs in global order */
  int64_t* plan;             /* (d, 4) scratch: src, dst, particle, valid */
  int64_t* records;          /* (d, n+1) donor records for exchange, or NULL */
  double* log;               /* (log_rows, d, 6) MigrationEvent fields, or NULL */
  int64_t log_rows;
  int64_t* log_count;        /* (1,) events logged */
  int32_t* status;           /* (1,) set to 1 when picks has no row for t */
  uint64_t seed;             /* SolverConfig.seed wrapped to uint64; used when picks == NULL */
} qsb_migration;

int qsb_version(void);
const char* qsb_strerror(int code);
int qsb_last_cuda_error(void);

/* Measurement utility: holds `stream` until the host writes a non-zero
 * int32 to host_flag (pinned host memory), or until timeout_ns passes, in
 * which case *timed_out (device or mapped memory, may be NULL) is set to 1.
 * Lets a benchmark enqueue a whole timed window before the device starts it,
 * so host scheduling jitter cannot starve the window. */
int qsb_stream_gate(const int32_t* host_flag, int64_t timeout_ns, int32_t* timed_out, void* stream);

/* 1 if a fused step kernel exists for (n, v_dtype, mat_dtype), else 0. */
int qsb_supported(int32_t n, int32_t v_dtype, int32_t mat_dtype);

/* Elements per particle of the padded V layout for n (16-byte rows). */
int32_t qsb_vstride(int32_t n, int32_t v_dtype);

/* ---------------------------------------------------------------- tier 2
 * Fused step, phases selected by `flags` (QSB_PHASE_*): velocity update
 * (_batch.py:30-58) -> aggregation (_batch.py:61-183) -> goal
 * (_batch.py:186-197) -> personal best (engine.py:211-215).  Draws come from
 * the in-kernel Philox stream of streams.step_draws for iteration
 * t = *state->iteration + 1 (or t_host when state->iteration is NULL), or
 * from `inj_draws` rows (stride inj_stride doubles; r2, r3 at columns 0, 1,
 * aggregation draws from column agg_base) when non-NULL.  `coef` (P, 2)
 * optionally overrides (c2*r2, c3*r3). */
int qsb_step_phases(const qsb_state* st, const qsb_instance* inst, const qsb_coeffs* co,
                    int32_t flags, const double* inj_draws, int64_t inj_stride,
                    int32_t agg_base, const double* coef, uint64_t t_host, void* stream);

/* Swarm bests (argmin over improved particles, strict <) and the global best
 * (argmin over all, strict <), engine.py:216-229; advances *iteration. */
int qsb_best_update(const qsb_state* st, void* stream);

/* qsb_best_update plus the NEXT step's draw pre-pass: (c2 r2, c3 r3) of
 * iteration t + 1 for every particle into st->step_coef, and st->work reset
 * (the pre-pass of qsb_step_phases, folded into the best-update launch).
 * Follow it with qsb_step_phases under QSB_HINT_COEF_READY. */
int qsb_best_update_next(const qsb_state* st, const qsb_coeffs* co, void* stream);

/* One full iteration: qsb_step_phases(all) + qsb_best_update.  The caller
 * swaps perm/perm_new afterwards (engine.py:231-232). */
int qsb_step(const qsb_state* st, const qsb_instance* inst, const qsb_coeffs* co, void* stream);

/* Migration (migration.py:55-86) on the post-swap state.  With
 * mig->picks == NULL the donor offsets are drawn on the device from the
 * reference's host stream host_rng(seed, t) (streams.py:48-50), exactly as
 * numpy's scalar Generator.integers(0, S) would draw them. */
int qsb_migrate(const qsb_state* st, const qsb_migration* mig, void* stream);

/* The d donor offsets of the migration event at iteration t (device int32
 * out): host_rng(seed, t).integers(0, swarm_size) called d times
 * (migration.py:82-84).  Parity / debug entry of the in-kernel draw. */
int qsb_migration_picks(uint64_t seed, uint64_t t, int32_t d, int64_t swarm_size, int32_t* out,
                        void* stream);

/* 2-opt local search (north-star extension; no reference symbol, SURVEY.md
 * 8a a11) on st->perm_new / st->cost, integral instances only.  Per pass the
 * best pairwise facility exchange (smallest integer delta, ties to the
 * lexicographically first (r, s)) is applied if it improves; at most
 * `passes` moves.  QSB_TWOOPT_PBEST also performs the personal-best update
 * (use it with qsb_step_phases without QSB_PHASE_PBEST). */
#define QSB_TWOOPT_PBEST 1
#define QSB_TWOOPT_SYMMETRIC 2   /* caller-checked: flow and distance symmetric, < 2^16 */
#define QSB_TWOOPT_BYTES 4       /* caller-checked: entries < 256 and n*max(F)*max(D) < 2^31 */
int qsb_twoopt(const qsb_state* st, const qsb_instance* inst, int32_t passes, int32_t flags,
               void* stream);

/* Goal of P permutations (int16, device) -> out (int64 or f64, device). */
int qsb_cost(const int16_t* perms, int64_t P, const qsb_instance* inst, void* out, void* stream);

/* Population statistics on the device (stats.collect, stats.py:72-100):
 * hist[bins] = the frozen-range PMF counts, binned exactly as numpy
 * (stats.py:45-47); out[0] = the minimum cost; out[1 + r] = the
 * ranks_k[r]-th smallest cost (0-based; nearest-rank percentile, stats.py:28),
 * r < nranks <= 4.  Values are the cost's raw 64-bit pattern (int64 or f64).
 * `work` is device scratch of qsb_stats_work_bytes() bytes. */
size_t qsb_stats_work_bytes(void);
int qsb_population_stats(const void* cost, int32_t cost_dtype, int64_t P, double lo, double width,
                         int32_t bins, const int64_t* ranks_k, int32_t nranks, void* work,
                         uint32_t* hist, int64_t* out, void* stream);

/* streams.step_draws rows p0 .. p0+P-1 into device memory. */
int qsb_step_draws(uint64_t seed, uint64_t t, int64_t p0, int64_t P, int32_t n, double* out,
                   void* stream);

/* Throughput-mode device initialisation (documented non-reference stream). */
int qsb_init_population_device(const qsb_state* st, uint64_t seed, double amp, void* stream);

/* int16 permutations -> 0/1 matrices X[k, i] = (perm[i] == k) (device). */
int qsb_perm_to_matrix(const int16_t* perm, int64_t P, int32_t n, int8_t* x, void* stream);

/* ---------------------------------------------------------------- tier 1
 * Reference-layout, host-buffer, synchronous drop-ins for _batch / streams. */

/* _batch.velocity_many(v, x, pl, pg, swarm_size, c1, c2r2, c3r3, v_max,
 * normalize) (_batch.py:30-58): v (P,n,n) f64 in place; x, pl (P,n,n) int8;
 * pg (P/swarm_size, n, n) int8; c2r2, c3r3 (P,). */
int qsb_velocity_many(double* v, const int8_t* x, const int8_t* pl, const int8_t* pg, int64_t P,
                      int32_t n, int64_t swarm_size, double c1, const double* c2r2,
                      const double* c3r3, double v_max, int32_t normalize);

/* _batch.aggregate_many(x, v, mode, depth, draws, out_mat, out_perm)
 * (_batch.py:178-183): draws row p at draws + p*draws_stride. */
int qsb_aggregate_many(const int8_t* x, const double* v, int64_t P, int32_t n, int32_t mode,
                       int32_t depth, const double* draws, int64_t draws_stride, int8_t* out_mat,
                       int64_t* out_perm);

/* _batch.cost_many(perms, flow, distance, out) (_batch.py:186-197). */
int qsb_cost_many_i64(const int64_t* perms, const int64_t* flow, const int64_t* distance,
                      int64_t* out, int64_t P, int32_t n);
int qsb_cost_many_f64(const int64_t* perms, const double* flow, const double* distance,
                      double* out, int64_t P, int32_t n);

/* 2-opt on host buffers: perms (P, n) int64 and costs (P,) updated in place. */
int qsb_twoopt_many(int64_t* perms, const int64_t* flow, const int64_t* distance, int64_t* costs,
                    int64_t P, int32_t n, int32_t passes);

/* streams.step_draws(seed, iteration, num_particles, n) (streams.py:53-64). */
int qsb_step_draws_host(uint64_t seed, uint64_t t, int64_t P, int32_t n, double* out);

/* The reference's PopulationState (engine.py:85-124) in HOST memory, in the
 * reference's own layout: float64 velocities, int8 0/1 matrices
 * X[k, i] = (perm[i] == k), int64 permutations, int64 (integral instance)
 * or float64 costs.  Pinned (page-locked) buffers transfer fastest; any
 * host memory works. */
typedef struct qsb_host_population {
  int32_t n;
  int32_t cost_dtype;        /* QSB_I64 or QSB_F64 */
  int64_t num_particles, swarm_size, num_swarms;
  double* V;                 /* (P, n, n) in/out */
  int8_t* X_new;             /* (P, n, n) out: next positions (X is not read:
                              * perms is its exact vector view, core.py:5-6) */
  int8_t* PL;                /* (P, n, n) in/out: rows of improved particles */
  int64_t* perms;            /* (P, n) in: current positions */
  int64_t* perms_new;        /* (P, n) out */
  int64_t* pl_perms;         /* (P, n) in/out */
  void* cost;                /* (P,) out: goal of perms_new */
  void* pl_cost;             /* (P,) in/out */
  uint8_t* improved;         /* (P,) out: cost < pl_cost this step */
  int8_t* pg_mats;           /* (m, n, n) in/out: swarm bests */
  int64_t* pg_perms;         /* (m, n) in/out */
  void* pg_costs;            /* (m,) in/out */
  int64_t* best_perm;        /* (n,) in/out: global best record */
  void* best_cost;           /* (1,) in/out */
  int64_t* best_iteration;   /* (1,) in/out */
} qsb_host_population;

/* A QAP instance in host memory (qaplib.QapInstance): int64 or float64. */
typedef struct qsb_host_instance {
  int32_t n;
  int32_t mat_dtype;         /* QSB_I64 or QSB_F64 */
  const void* flow;
  const void* distance;
} qsb_host_instance;

/* One engine.step (engine.py:181-244) on host buffers: the step draws for
 * iteration t (streams.py:53-64), velocity (_batch.py:30-58), aggregation
 * (_batch.py:61-183), goal (_batch.py:186-197), personal / swarm / global
 * bests (engine.py:210-229) and, when migrate_d > 0, migration
 * (migration.py:55-86, donor picks from host_rng(seed, t)); the caller then
 * swaps X <-> X_new and perms <-> perms_new (engine.py:231-232).  fp64
 * parity arithmetic: results are bit-identical to the reference's step.
 * migration_log (migrate_d x 6 doubles) receives the MigrationEvent fields.
 * Synchronous; the particles stream through the device in swarm-aligned
 * chunks (QSB_HOST_CHUNKS, default 16) with copies and compute overlapped. */
int qsb_step_host(qsb_host_population* hp, const qsb_host_instance* inst, const qsb_coeffs* co,
                  uint64_t t, int32_t migrate_d, double* migration_log);

#ifdef __cplusplus
}
#endif
#endif /* QAPSWARM_B200_H */
