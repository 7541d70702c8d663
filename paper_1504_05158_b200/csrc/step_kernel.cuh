// step_kernel.cuh -- the fused PSO step for one particle per thread group.
//
// One group of G warps owns one particle at a time (persistent loop over the
// particles of this device).  Thread t of the group owns columns
// c = t + k*32G (k < CPL) of the particle's n x n velocity tile, so:
//
//   * the velocity update and the column normalisation are column-local and
//     run in the reference's exact order (_batch.py:39-58);
//   * the aggregation keeps incremental per-column statistics over the free
//     rows instead of the reference's O(n^3) rescan (_batch.py:89-175),
//     reproducing its (max, tie-count) per round, its row-major k-th-tie
//     selection and its draw consumption exactly;
//   * the QAP goal is a per-column partial sum over the smem-resident F, D
//     (_batch.py:186-197), reduced in integer arithmetic.
//
// Aggregation statistics.  In column c the cell (zr, c), zr = perm[c], is
// the only one with x = 1 ("z cell": m = 1 + v); every other cell has
// m = 0 + v.  Each column therefore keeps
//   - (nmax, ncnt, nrow): max / tie count / first row of v over its free
//     non-z rows, compared directly in the velocity type (v1 > v2 on the
//     stored values equals m1 > m2, and -0 == +0 as in m);
//   - zkey: the ordered 64-bit key of 1 + v_z, and whether the z cell is
//     currently eligible (its row free, and not inside the second-target
//     restricted rounds).
// The second-target restriction (_batch.py:90, 110) then only toggles z
// eligibility, and a round costs O(CPL) per thread plus one warp reduction.
//
// The tile is staged global -> smem with one cp.async.bulk (1-D TMA) and the
// updated velocity is written back with one bulk store, so the velocity
// phase touches HBM exactly once in each direction.
#pragma once
#include <type_traits>
#include "common.cuh"

namespace qsb {

enum StepFlags : int {
  F_VELOCITY = 1,     // phase 1: velocity update (+ normalise)
  F_AGGREGATE = 2,    // phase 2: S_x aggregation -> perm_new
  F_COST = 4,         // phase 3: goal of perm_new -> cost
  F_PBEST = 8,        // phase 4a: personal best update + improved flag
  F_STORE_V = 16,     // write the updated velocity tile back to HBM
};

struct StepArgs {
  int n, vstride;
  int64_t P;            // particles on this device
  int64_t S;            // swarm size
  int64_t p0;           // global id of local particle 0 (RNG rows)
  double c1, c2, c3, vmax;
  int normalize, mode, depth, flags;
  uint64_t seed;
  const int64_t* t_dev; // device iteration counter (t = *t_dev + 1); nullable
  uint64_t t_host;      // used when t_dev is null
  void* V;
  const int16_t* perm;  // current X, n per particle (perm[c] = row of the 1)
  int16_t* perm_new;
  int16_t* pl_perm;
  const int16_t* pg_perm;  // per local swarm
  void* cost;
  void* pl_cost;
  uint8_t* improved;
  const void* F;
  const void* D;
  const double* inj_draws;   // optional injected draw rows
  int64_t inj_stride;
  int agg_base;              // column of the first aggregation draw in a row
  const double* coef;        // optional (P, 2): c2*r2, c3*r3 per particle
  int fd_smem;               // 1: stage F, D in smem; 0: read them from global/L2
  int v_bounded;             // host guarantee: |c1 * v| <= v_max for every stored v
  int acc32;                 // host guarantee: n * max(F) * max(D) < 2^32
  int cost_incremental;      // host guarantee: cost[p] == goal(perm[p]) on entry
  int symmetric;             // host guarantee: F and D symmetric (integral instances)
  int late;                  // QSB_HINT_LATE: the late-iteration specialisation is wanted
  unsigned int* work;        // optional zeroed counter: dynamic particle scheduling
  float* vcol;               // fp32 lazily scaled layout: (P, 5, vcstride) column state, or null
  int vcstride;
  int mw_defer;              // n > 64 fp32 with vcol: 1 = deferred column scale (row 0 only,
                             // float tile; QSB_MW_DEFER=1 A/B), 0 = the lazily scaled layout
};

struct Best {
  uint64_t key;
  int cnt;
  int col;
  int row;
};

__device__ __forceinline__ Best best_none() {
  Best b; b.key = 0; b.cnt = 0; b.col = INT_MAX; b.row = -1;
  return b;
}

__device__ __forceinline__ Best best_merge(const Best& a, const Best& b) {
  if (a.key > b.key) return a;
  if (b.key > a.key) return b;
  Best r = a;
  r.cnt = a.cnt + b.cnt;
  if (b.col < a.col) { r.col = b.col; r.row = b.row; }
  return r;
}

// Warp-wide (max key, count at max, min col at max, that col's row).
__device__ __forceinline__ Best warp_best(const Best& b) {
  const unsigned hi = (unsigned)(b.key >> 32), lo = (unsigned)b.key;
  const unsigned mh = __reduce_max_sync(FULL, hi);
  const unsigned ml = __reduce_max_sync(FULL, hi == mh ? lo : 0u);
  const bool match = (hi == mh) && (lo == ml) && b.cnt > 0;
  Best r;
  r.key = ((uint64_t)mh << 32) | ml;
  r.cnt = (int)__reduce_add_sync(FULL, match ? (unsigned)b.cnt : 0u);
  r.col = __reduce_min_sync(FULL, match ? b.col : INT_MAX);
  const unsigned who = __ballot_sync(FULL, match && b.col == r.col);
  r.row = __shfl_sync(FULL, b.row, who ? __ffs(who) - 1 : 0);
  return r;
}

// Fast path: when one lane holds the maximum high word, that lane's local
// best is the answer (two shuffles); otherwise the full reduction.
__device__ __forceinline__ Best warp_best_fast(const Best& b) {
  const unsigned hi = (unsigned)(b.key >> 32);
  const unsigned mh = __reduce_max_sync(FULL, hi);
  const unsigned who = __ballot_sync(FULL, hi == mh && b.cnt > 0);
  if (__popc(who) == 1) {
    const int src = __ffs(who) - 1;
    const unsigned pk = ((unsigned)b.cnt << 16) | ((unsigned)(b.col & 0xff) << 8) |
                        (unsigned)((b.row + 1) & 0xff);
    const unsigned lo = __shfl_sync(FULL, (unsigned)b.key, src);
    const unsigned q = __shfl_sync(FULL, pk, src);
    Best r;
    r.key = ((uint64_t)mh << 32) | lo;
    r.cnt = (int)(q >> 16);
    r.col = (int)((q >> 8) & 0xff);
    r.row = (int)(q & 0xff) - 1;
    return r;
  }
  return warp_best(b);
}

__device__ __forceinline__ int64_t warp_sum_i64(int64_t x) {
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
  return x;
}

// Position of the k-th (0-based) set bit of a 32-bit mask (k < popc(m)).
__device__ __forceinline__ int nth_set_bit32(unsigned m, int k) {
  int pos = 0;
#pragma unroll
  for (int w = 16; w; w >>= 1) {
    const int c = __popc(m & ((1u << w) - 1u));
    if (k >= c) { k -= c; m >>= w; pos += w; }
  }
  return pos;
}

// Per-group shared scratch (one per particle group in the CTA).  Row and
// column indices are < 256, so the per-column arrays are bytes (this keeps
// four one-warp CTAs of four particles resident per SM at n = 50).
// Multi-warp groups only: the bulk step's threshold beside the round's
// group reduction, and its count / retired-row words double-buffered over
// consecutive attempts (so an attempt needs no barrier to reset them).
template <int NMAX, int G>
struct MwScratch {
  uint64_t mslots[2][G];
  unsigned long long rmw2[2][(NMAX + 63) / 64];
  int bcnt[2];
};
struct MwNone {};

template <int NMAX, int G>
struct GroupScratch {
  union {
    uint64_t sbulk[NMAX];    // z keys assigned by bulk steps (pending tie-draw count)
    uint64_t tmask[NMAX];    // per tied column: mask of tied rows (one-warp tie path;
                             // used only after the pending bulk keys were counted)
  };
  unsigned long long rmw[(NMAX + 63) / 64];   // rows retired by a bulk step (multi-warp groups)
  uint64_t bar;
  Best slots[2][G];
  int64_t lslots[G];
  int islots[2][G];
  int ssel[4];
  float sS[NMAX];        // column scales of the fp32 tile (lazily scaled layout; else 1)
  uint16_t srow[NMAX];   // per-row tie counts / pick-column match flags / lists
  uint8_t sperm[NMAX];   // perm_new under construction (aggregation output)
  uint8_t szr[NMAX];     // perm of the current position X (z row per column)
  uint8_t sorder[NMAX];  // pick-column visiting order
  unsigned char stie[NMAX];  // tied-column flags: 1 tied, 2 tied with an eligible z cell
  bool wide;                 // tile entries are wide words (lazily scaled fp32 layout)
  std::conditional_t<(G > 1), MwScratch<NMAX, G>, MwNone> mw;
};

template <int G>
struct GroupSync {
  __device__ __forceinline__ static void sync() {
    if constexpr (G == 1) __syncwarp(); else __syncthreads();
  }
};

// Optional event counters for diagnosis builds (-DQSB_COUNTERS): particles,
// normal rounds, bulk steps, bulk z cells, tie rounds, warp tie paths,
// slow tie paths, rescans; lazily scaled layout: full passes, incremental
// rescans, rescans with unknown column state.
#ifdef QSB_COUNTERS
__device__ unsigned long long qsb_counters[12];
#define QSB_COUNT(i, v) do { if ((threadIdx.x & 31) == 0) atomicAdd(&qsb_counters[i], (unsigned long long)(v)); } while (0)
#else
#define QSB_COUNT(i, v) do { } while (0)
#endif

#ifndef QSB_MINB
#define QSB_MINB 4
#endif

template <typename VT, typename MT, int G, int CPL, int W, bool GT = false>
struct StepKernel {
  static constexpr int NT = 32 * G;          // threads per group
  static constexpr int NMAX = NT * CPL;      // largest n handled
  static constexpr int NW = (NMAX + 63) / 64;
  using Scratch = GroupScratch<NMAX, G>;

  static __host__ __device__ size_t fd_bytes(int n) {
    return align_up(2 * (size_t)n * n * sizeof(MT), 128);
  }
  static __host__ __device__ size_t tile_bytes(int vstride) {
    return GT ? 0 : align_up((size_t)vstride * sizeof(VT), 128);
  }
  // One-warp groups stage the next particle's column data next to its tile
  // (cp.async / bulk copies issued with the tile prefetch): the lazily
  // scaled layout's column state (5 x NMAX words), the perm / pl_perm /
  // pg_perm rows (3 x NMAX int16), (c2 r2, c3 r3) and, double-buffered,
  // (cost, pl_cost).
  static constexpr bool STAGE = G == 1 && !GT;
  static constexpr size_t SCOL = 0, SPERM = 20 * NMAX, SCOEF = SPERM + 6 * NMAX, SCOST = SCOEF + 16;
  static __host__ __device__ size_t stage_bytes() {
    return STAGE ? align_up(SCOST + 32, 128) : 0;
  }
  static __host__ __device__ size_t group_bytes(int vstride) {
    return tile_bytes(vstride) + stage_bytes() + align_up(sizeof(Scratch), 128);
  }
  static __host__ __device__ size_t smem_bytes(int n, int vstride, bool fd) {
    return (fd ? fd_bytes(n) : 0) + W * group_bytes(vstride);
  }
};

// Group-wide best: warp fast path for one-warp groups, smem slots otherwise.
template <int G, typename Scratch>
__device__ __forceinline__ Best group_best(const Best& loc, Scratch& sc, int& par, int lane, int tid) {
  if constexpr (G == 1) {
    return warp_best_fast(loc);
  } else {
    Best b = warp_best(loc);
    if (lane == 0) sc.slots[par][tid >> 5] = b;
    __syncthreads();
    b = sc.slots[par][0];
#pragma unroll
    for (int w = 1; w < G; ++w) b = best_merge(b, sc.slots[par][w]);
    par ^= 1;
    return b;
  }
}

// Multi-warp groups: the round's best candidate and the maximum mx (the bulk
// step's threshold) in one group reduction -- one barrier for both.
template <int G, typename Scratch>
__device__ __forceinline__ Best group_best_max(const Best& loc, uint64_t mx, Scratch& sc, int& par, int lane,
                                               int tid, uint64_t& M) {
  Best b = warp_best(loc);
  const unsigned hi = (unsigned)(mx >> 32);
  const unsigned mh = __reduce_max_sync(FULL, hi);
  const unsigned mlo = __reduce_max_sync(FULL, hi == mh ? (unsigned)mx : 0u);
  if (lane == 0) {
    sc.slots[par][tid >> 5] = b;
    sc.mw.mslots[par][tid >> 5] = ((uint64_t)mh << 32) | mlo;
  }
  __syncthreads();
  b = sc.slots[par][0];
  uint64_t m = sc.mw.mslots[par][0];
#pragma unroll
  for (int w = 1; w < G; ++w) {
    b = best_merge(b, sc.slots[par][w]);
    m = max(m, sc.mw.mslots[par][w]);
  }
  par ^= 1;
  M = m;
  return b;
}

template <int G, typename Scratch>
__device__ __forceinline__ int group_min_int(int x, Scratch& sc, int& ipar, int lane, int tid) {
  x = __reduce_min_sync(FULL, x);
  if constexpr (G > 1) {
    if (lane == 0) sc.islots[ipar][tid >> 5] = x;
    __syncthreads();
#pragma unroll
    for (int w = 0; w < G; ++w) x = min(x, sc.islots[ipar][w]);
    ipar ^= 1;
  }
  return x;
}

// Velocity value of a stored entry.  fp64 tiles hold v itself.  fp32 tiles
// in the lazily scaled layout hold "wide" 32-bit words: the high word of the
// double (sign, 11-bit exponent, 20-bit fraction), rounded to nearest -- the
// byte size of fp32 with the exponent range of fp64, so an entry the
// reference keeps as a tiny non-zero value (it decays by ~1 bit per step
// while x / pl / pg leave it alone) does not flush to zero after ~150 steps
// as an fp32 would, and does not turn into a spurious tie.  The words order
// like floats (sign-magnitude), so stored values are compared with float
// compares on the raw bits (exact for |v| in [2^-1015, 2^1017]; no
// flush-to-zero in this build).  Stored-v fp32 tiles hold plain floats.
// Lazily scaled: v = u * s (s the column scale, 1.0 otherwise); the product
// is exact in double.
// `wide` is a runtime property of the state: true for the lazily scaled
// layout of the one-warp fp32 kernels, false for stored-v fp32 tiles (the
// streaming velocity pass keeps float arithmetic) and for fp64.
template <typename VT>
__device__ __forceinline__ double vval(VT u, float s, bool wide) {
  if constexpr (sizeof(VT) == 8) return u;
  else return wide ? wdec(u) * wdec(s) : (double)u * (double)s;   // wide: the scale is a wide word too
}
template <typename VT>
__device__ __forceinline__ uint64_t nonz_key(VT v, float s, bool wide) {   // key of m = 0.0 + v
  return okey(__dadd_rn(0.0, vval(v, s, wide)));
}
template <typename VT>
__device__ __forceinline__ uint64_t z_key(VT v, float s, bool wide) {      // key of m = 1.0 + v
  return okey(__dadd_rn(1.0, vval(v, s, wide)));
}

// Set of free rows (bit r of word r/64).
template <int NW>
struct RowSet {
  uint64_t w[NW];
  __device__ __forceinline__ bool has(int r) const { return (w[r >> 6] >> (r & 63)) & 1ULL; }
  __device__ __forceinline__ void clear(int r) { w[r >> 6] &= ~(1ULL << (r & 63)); }
  __device__ __forceinline__ int first() const {
#pragma unroll
    for (int i = 0; i < NW; ++i) if (w[i]) return i * 64 + __ffsll((long long)w[i]) - 1;
    return -1;
  }
};

template <typename VT>
__device__ __forceinline__ uint64_t mkey(const VT* tile, const float* sS, int n, int r, int c, int zrc,
                                         bool wide) {
  return okey(__dadd_rn(r == zrc ? 1.0 : 0.0, vval(tile[r * n + c], sS[c], wide)));
}

// ---- rare paths, kept out of line so the round loop stays in I-cache ----

// Group-wide int minimum with its own barriers (callable from any point).
template <int G, typename Scratch>
__device__ __forceinline__ int group_min_sync(int x, Scratch& sc, int lane, int tid) {
  x = __reduce_min_sync(FULL, x);
  if constexpr (G > 1) {
    __syncthreads();
    if (lane == 0) sc.islots[0][tid >> 5] = x;
    __syncthreads();
#pragma unroll
    for (int w = 0; w < G; ++w) x = min(x, sc.islots[0][w]);
    __syncthreads();
  }
  return x;
}

// Tie round: the pick-th tied cell in row-major order (_batch.py:155-170).
// Owners have flagged the tied columns in sc.stie (2 = its z cell is
// eligible) before the call.  Result in sc.ssel[0..1]; flags cleared.
template <typename VT, int G, int NW, typename Scratch>
__device__ __noinline__ void tie_select_slow(const VT* tile, int n, Scratch& sc, RowSet<NW> rf,
                                             uint64_t key, int pick, int tid) {
  constexpr int NT = 32 * G;
  GroupSync<G>::sync();
  for (int r = tid; r < n; r += NT) {
    int cnt = 0;
    if (rf.has(r)) {
      for (int c = 0; c < n; ++c) {
        const int tf = sc.stie[c];
        if (!tf) continue;
        const int zc = sc.szr[c];
        if (r == zc && tf != 2) continue;
        if (mkey(tile, sc.sS, n, r, c, zc, sc.wide) == key) ++cnt;
      }
    }
    sc.srow[r] = cnt;
  }
  GroupSync<G>::sync();
  if (tid == 0) {
    int r = 0, acc = 0;
    while (acc + sc.srow[r] <= pick) { acc += sc.srow[r]; ++r; }
    int q = pick - acc, cc = -1;
    for (int c = 0; c < n; ++c) {
      const int tf = sc.stie[c];
      if (!tf) continue;
      const int zc = sc.szr[c];
      if (r == zc && tf != 2) continue;
      if (mkey(tile, sc.sS, n, r, c, zc, sc.wide) == key) {
        if (q == 0) { cc = c; break; }
        --q;
      }
    }
    sc.ssel[0] = r; sc.ssel[1] = cc;
  }
  GroupSync<G>::sync();
  for (int c = tid; c < n; c += NT) sc.stie[c] = 0;
}

// Unique maximum in column c whose first row is not tracked: scan it.
template <typename VT, int G, int CPL, int NW, typename Scratch>
__device__ __noinline__ int first_row_scan(const VT* tile, int n, Scratch& sc, RowSet<NW> rf,
                                           uint64_t key, int c, bool zok, int tid, int lane) {
  constexpr int NT = 32 * G;
  const int zc = sc.szr[c];
  int found = INT_MAX;
  for (int r = tid; r < n; r += NT)
    if (rf.has(r) && (r != zc || zok) && mkey(tile, sc.sS, n, r, c, zc, sc.wide) == key) found = min(found, r);
  return group_min_sync<G>(found, sc, lane, tid);
}

// Number of distinct keys among the z cells placed by bulk steps (n <= 64:
// two list entries per lane, match.any within each half, a short loop for
// values shared across the halves).
template <typename Scratch>
__device__ __noinline__ int bulk_distinct(const Scratch& sc, int nb, int lane) {
  const bool v0 = lane < nb, v1 = lane + 32 < nb;
  const unsigned long long e0 = v0 ? sc.sbulk[lane] : 0ULL;
  const unsigned long long e1 = v1 ? sc.sbulk[lane + 32] : 0ULL;
  const unsigned m0 = __match_any_sync(FULL, e0);
  const unsigned m1 = __match_any_sync(FULL, e1);
  const bool f0 = v0 && (__ffs(m0) - 1) == lane;
  const bool f1 = v1 && (__ffs(m1) - 1) == lane;
  int distinct = __popc(__ballot_sync(FULL, f0));
  unsigned firsts1 = __ballot_sync(FULL, f1);
  while (firsts1) {
    const int src = __ffs(firsts1) - 1;
    firsts1 &= firsts1 - 1;
    const unsigned long long v = __shfl_sync(FULL, e1, src);
    distinct += __any_sync(FULL, v0 && e0 == v) ? 0 : 1;
  }
  return distinct;
}

// Same for multi-warp groups (n > 64): O(nb^2 / threads) comparisons.
template <int G, typename Scratch>
__device__ __noinline__ int bulk_distinct_group(Scratch& sc, int nb, int tid, int lane) {
  constexpr int NT = 32 * G;
  int firsts = 0;
  for (int i = tid; i < nb; i += NT) {
    const uint64_t ki = sc.sbulk[i];
    bool first = true;
    for (int j = 0; j < i; ++j) if (sc.sbulk[j] == ki) { first = false; break; }
    firsts += first;
  }
  firsts = (int)__reduce_add_sync(FULL, (unsigned)firsts);
  __syncthreads();
  if (lane == 0) sc.islots[0][tid >> 5] = firsts;
  __syncthreads();
  int tot = 0;
  for (int w = 0; w < G; ++w) tot += sc.islots[0][w];
  __syncthreads();
  return tot;
}

// Tie round for one-warp groups (n <= 64): the pick-th tied cell in
// row-major order (_batch.py:155-170).  Owners have flagged the tied columns
// in sc.stie (2 = its z cell is eligible).  Each tied column contributes a
// 64-bit mask of tied rows; a warp prefix sum over per-row counts finds the
// row, and the pick-th tied column of that row (ascending) the cell.
// Returns (row << 8) | col; clears the flags.
template <typename VT, typename Scratch>
__device__ __noinline__ int tie_select_warp(const VT* tile, int n, Scratch& sc, uint64_t rfree,
                                            uint64_t key, int pick, int lane) {
  __syncwarp();
  const int c0 = lane, c1 = lane + 32;
  const bool t0 = sc.stie[c0] != 0;
  const bool t1 = c1 < n && sc.stie[c1] != 0;
  unsigned tb[2] = {__ballot_sync(FULL, t0), __ballot_sync(FULL, t1)};
  int cnt0 = 0, cnt1 = 0;
  const bool r0ok = c0 < n && ((rfree >> c0) & 1ULL);
  const bool r1ok = c1 < n && ((rfree >> c1) & 1ULL);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    unsigned b = tb[h];
    while (b) {
      const int c = h * 32 + __ffs(b) - 1;
      b &= b - 1;
      const int zc = sc.szr[c];
      const bool zok = sc.stie[c] == 2;
      const bool a0 = r0ok && (c0 != zc || zok) && mkey(tile, sc.sS, n, c0, c, zc, sc.wide) == key;
      const bool a1 = r1ok && (c1 != zc || zok) && mkey(tile, sc.sS, n, c1, c, zc, sc.wide) == key;
      const unsigned m0 = __ballot_sync(FULL, a0), m1 = __ballot_sync(FULL, a1);
      cnt0 += a0;
      cnt1 += a1;
      if (lane == 0) sc.tmask[c] = ((uint64_t)m1 << 32) | m0;
    }
  }
  // inclusive prefix of the per-row counts, rows 0..31 then 32..63
  int p0 = cnt0, p1 = cnt1;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u0 = __shfl_up_sync(FULL, p0, o), u1 = __shfl_up_sync(FULL, p1, o);
    if (lane >= o) { p0 += u0; p1 += u1; }
  }
  const int tot0 = __shfl_sync(FULL, p0, 31);
  p1 += tot0;
  const unsigned h0 = __ballot_sync(FULL, cnt0 && p0 - cnt0 <= pick && pick < p0);
  const unsigned h1 = __ballot_sync(FULL, cnt1 && p1 - cnt1 <= pick && pick < p1);
  int row, q;
  if (h0) { row = __ffs(h0) - 1; q = pick - (__shfl_sync(FULL, p0 - cnt0, row)); }
  else { const int l = __ffs(h1) - 1; row = 32 + l; q = pick - (__shfl_sync(FULL, p1 - cnt1, l)); }
  __syncwarp();
  const bool b0 = t0 && ((sc.tmask[c0] >> row) & 1ULL);
  const bool b1 = t1 && ((sc.tmask[c1] >> row) & 1ULL);
  const unsigned w0 = __ballot_sync(FULL, b0), w1 = __ballot_sync(FULL, b1);
  const int n0 = __popc(w0);
  const int col = q < n0 ? nth_set_bit32(w0, q) : 32 + nth_set_bit32(w1, q - n0);
  if (t0) sc.stie[c0] = 0;
  if (t1) sc.stie[c1] = 0;
  __syncwarp();
  return (row << 8) | col;
}

// pick-column S_x (_batch.py:78-88, 93-102, 145-153): Fisher-Yates column
// order from n-1 draws, then per column the max over the free rows with
// uniform tie-breaking in row order.  Writes sc.sperm.
template <typename VT, int G, int NW, typename Scratch>
__device__ __noinline__ void agg_pick_column(const VT* tile, int n, Scratch& sc, RowSet<NW> rf,
                                             DrawKey dk, int cursor, int tid, int lane) {
  constexpr int NT = 32 * G;
  DrawCache dr;
  dr.init(dk);
  GroupSync<G>::sync();
  for (int i = tid; i < n; i += NT) sc.sorder[i] = i;
  GroupSync<G>::sync();
  if (tid == 0) {
    for (int i = n - 1; i > 0; --i) {
      const double u = dr.at(cursor++);
      long long j = (long long)__dmul_rn(u, (double)(i + 1));
      if (j > i) j = i;
      const int tmp = sc.sorder[i]; sc.sorder[i] = sc.sorder[j]; sc.sorder[j] = tmp;
    }
    sc.ssel[3] = cursor;
  }
  GroupSync<G>::sync();
  cursor = sc.ssel[3];
  int par = 0;
  for (int rnd = 0; rnd < n; ++rnd) {
    const int c = sc.sorder[rnd];
    const int zc = sc.szr[c];
    Best rb = best_none();
    for (int r = tid; r < n; r += NT) {
      if (!rf.has(r)) continue;
      const uint64_t key = mkey(tile, sc.sS, n, r, c, zc, sc.wide);
      if (key > rb.key) { rb.key = key; rb.cnt = 1; rb.col = r; }
      else if (key == rb.key) ++rb.cnt;
    }
    const Best b = group_best<G>(rb, sc, par, lane, tid);
    int sel_r = b.col;   // first matching row
    if (b.cnt > 1) {
      const double u = dr.at(cursor++);
      const long long pk = (long long)__dmul_rn(u, (double)b.cnt);
      const int pick = (int)(pk >= b.cnt ? b.cnt - 1 : pk);
      for (int r = tid; r < n; r += NT)
        sc.srow[r] = (rf.has(r) && mkey(tile, sc.sS, n, r, c, zc, sc.wide) == b.key) ? 1 : 0;
      GroupSync<G>::sync();
      if (tid == 0) {
        int q = pick, r = 0;
        for (; r < n; ++r) if (sc.srow[r]) { if (q == 0) break; --q; }
        sc.ssel[0] = r;
      }
      GroupSync<G>::sync();
      sel_r = sc.ssel[0];
      GroupSync<G>::sync();
    }
    rf.clear(sel_r);
    if (tid == 0) sc.sperm[c] = sel_r;
  }
}

// Goal for the general element types (int64 products or a non-integral
// instance, sequential as _batch.py:192-197).  Returns the group total on
// tid 0 (as raw bits for doubles).
template <typename MT, int G, int CPL, typename Scratch>
__device__ __noinline__ int64_t cost_general(const MT* cF, const MT* cD, int n, Scratch& sc,
                                             int tid, int lane, int acc32) {
  constexpr int NT = 32 * G;
  if constexpr (std::is_floating_point<MT>::value) {
    double acc = 0.0;
    if (tid == 0) {
      acc = (double)cF[0] * (double)cD[0] * 0.0;
      for (int i = 0; i < n; ++i) {
        const int pi = sc.sperm[i];
        for (int j = 0; j < n; ++j)
          acc = __dadd_rn(acc, __dmul_rn((double)cF[i * n + j], (double)cD[pi * n + sc.sperm[j]]));
      }
    }
    return __double_as_longlong(acc);
  } else {
    uint64_t part = 0;
    for (int j = tid; j < n; j += NT) {
      const int pj = sc.sperm[j];
      if (sizeof(MT) <= 2 && acc32) {
        // n * max(F) * max(D) < 2^32: the column sum fits 32 bits
        uint32_t p32 = 0;
        for (int i = 0; i < n; ++i)
          p32 += (uint32_t)cF[i * n + j] * (uint32_t)cD[sc.sperm[i] * n + pj];
        part += p32;
      } else {
        for (int i = 0; i < n; ++i) {
          if constexpr (sizeof(MT) <= 2)
            part += (uint64_t)((uint32_t)cF[i * n + j] * (uint32_t)cD[sc.sperm[i] * n + pj]);
          else
            part += (uint64_t)cF[i * n + j] * (uint64_t)cD[sc.sperm[i] * n + pj];
        }
      }
    }
    int64_t tot = warp_sum_i64((int64_t)part);
    if constexpr (G > 1) {
      __syncthreads();
      if (lane == 0) sc.lslots[tid >> 5] = tot;
      __syncthreads();
      tot = 0;
      for (int w = 0; w < G; ++w) tot += sc.lslots[w];
    }
    return tot;
  }
}

// Column statistics for the uncommon cases (raw mode: no scaling; or some
// column summed to 0): optional per-column scaling, then max / tie count /
// first row over the non-z rows.  Out of line to keep the hot kernel small.
template <typename VT, int CPL>
struct ColIn {
  int col[CPL], zr[CPL];
  bool cfree[CPL], scale[CPL];
  VT total[CPL], inv[CPL];
};
template <typename VT, int CPL>
struct ColOut {
  VT m[CPL];
  int c[CPL], r[CPL];
};

template <typename VT, int G, int CPL>
__device__ __noinline__ ColOut<VT, CPL> stats_generic(VT* tile, int n, const ColIn<VT, CPL> in) {
  const VT NINF = (VT)(-INFINITY);
  ColOut<VT, CPL> o;
#pragma unroll
  for (int k = 0; k < CPL; ++k) { o.m[k] = NINF; o.c[k] = 0; o.r[k] = -1; }
  for (int r = 0; r < n; ++r) {
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      if (!in.cfree[k]) continue;
      VT* cell = tile + r * n + in.col[k];
      VT v = *cell;
      if (in.scale[k]) {
        if constexpr (sizeof(VT) == 8) v = __ddiv_rn(v, in.total[k]);
        else v = v * in.inv[k];
        *cell = v;
      }
      const VT w = r == in.zr[k] ? NINF : v;
      const bool gt = w > o.m[k];
      o.c[k] = gt ? 1 : o.c[k] + (w == o.m[k] ? 1 : 0);
      o.r[k] = gt ? r : o.r[k];
      o.m[k] = gt ? w : o.m[k];
    }
  }
  return o;
}

// Column statistics (max / tie count / first row over the non-z rows) of a
// freshly written tile, with the normalisation fused in (smode 1: every live
// column scaled; 2: per-column, via stats_generic; 0: no scaling, the lazily
// scaled layout's full pass).  Out of line for the instruction cache (the
// lazily scaled layout carries these statistics from step to step).
template <typename VT, int G, int CPL>
__device__ __noinline__ ColOut<VT, CPL> stats_pass(VT* tile, int n, const ColIn<VT, CPL> in, int smode) {
  VT nmax[CPL];
  int ncnt[CPL], nrow[CPL], col[CPL], zr[CPL];
  bool cfree[CPL];
  VT total[CPL], inv[CPL];
#pragma unroll
  for (int k = 0; k < CPL; ++k) {
    nmax[k] = (VT)(-INFINITY); ncnt[k] = 0; nrow[k] = -1;
    col[k] = in.col[k]; zr[k] = in.zr[k]; cfree[k] = in.cfree[k];
    total[k] = in.total[k]; inv[k] = in.inv[k];
  }
  auto rescale = [&](VT v, int k) -> VT {
    if constexpr (sizeof(VT) == 8) return __ddiv_rn(v, total[k]);
    else return v * inv[k];
  };
  // Max / tie count / first row over the non-z rows (the z row is masked
  // to -inf; stored values are finite), accumulated separately over even
  // and odd rows (two independent dependency chains) and merged.  A
  // half holding only the z row keeps max = -inf and is ignored.
  const VT NINF = (VT)(-INFINITY);
  VT mB[CPL];
  int cB[CPL], rB[CPL];
#pragma unroll
  for (int k = 0; k < CPL; ++k) { mB[k] = NINF; cB[k] = 0; rB[k] = -1; }
  auto upd = [&](VT v, int r, int k, VT& m, int& c, int& rr) {
    const VT w = r == zr[k] ? NINF : v;
    const bool gt = w > m;
    c = gt ? 1 : c + (w == m ? 1 : 0);
    rr = gt ? r : rr;
    m = gt ? w : m;
  };
  auto stats_rows = [&](auto do_scale) {
    if constexpr (G == 1 && CPL == 2) {
      // branch-free form (see the velocity loop): a dead slot 1 rescans
      // slot 0's column with a unit factor; its statistics are unused
      const bool live1 = cfree[1];
      VT* q0 = tile + col[0];
      VT* q1 = tile + (live1 ? col[1] : col[0]);
      const VT s0 = inv[0], s1 = live1 ? inv[1] : (VT)1;
      // the z cells are parked at -inf during the scan (restored below),
      // so the loop needs no per-row z test
      VT* zp0 = q0 + zr[0] * n;
      VT* zp1 = q1 + (live1 ? zr[1] : zr[0]) * n;
      const VT zv0 = *zp0;
      const VT zv1 = live1 ? *zp1 : (VT)0;
      *zp0 = NINF;
      if (live1) *zp1 = NINF;
      const int z0 = -1, z1 = -1;
      const int n2 = 2 * n;
      auto sc_ = [&](VT v, VT f, int k) -> VT {
        if constexpr (sizeof(VT) == 8) return k == 0 || live1 ? __ddiv_rn(v, total[k]) : v;
        else return v * f;
      };
      auto upd2 = [&](VT w, int r, int, VT& m, int& c, int& rr) {
        const bool gt = w > m;
        c = gt ? 1 : c + (w == m ? 1 : 0);
        rr = gt ? r : rr;
        m = gt ? w : m;
      };
      int r = 0;
      for (; r + 1 < n; r += 2, q0 += n2, q1 += n2) {
        VT a0 = q0[0], a1 = q0[n];
        if constexpr (decltype(do_scale)::value) { a0 = sc_(a0, s0, 0); a1 = sc_(a1, s0, 0); q0[0] = a0; q0[n] = a1; }
        upd2(a0, r, z0, nmax[0], ncnt[0], nrow[0]);
        upd2(a1, r + 1, z0, mB[0], cB[0], rB[0]);
        VT b0 = q1[0], b1 = q1[n];
        if constexpr (decltype(do_scale)::value) { b0 = sc_(b0, s1, 1); b1 = sc_(b1, s1, 1); q1[0] = b0; q1[n] = b1; }
        upd2(b0, r, z1, nmax[1], ncnt[1], nrow[1]);
        upd2(b1, r + 1, z1, mB[1], cB[1], rB[1]);
      }
      if (r < n) {
        VT a0 = q0[0];
        if constexpr (decltype(do_scale)::value) { a0 = sc_(a0, s0, 0); q0[0] = a0; }
        upd2(a0, r, z0, nmax[0], ncnt[0], nrow[0]);
        VT b0 = q1[0];
        if constexpr (decltype(do_scale)::value) { b0 = sc_(b0, s1, 1); q1[0] = b0; }
        upd2(b0, r, z1, nmax[1], ncnt[1], nrow[1]);
      }
      if constexpr (decltype(do_scale)::value) {
        *zp0 = sc_(zv0, s0, 0);
        if (live1) *zp1 = sc_(zv1, s1, 1);
      } else {
        *zp0 = zv0;
        if (live1) *zp1 = zv1;
      }
      return;
    }
    // batches of 8 rows, loads first (latency-bound walk for GT tiles);
    // even rows feed the first chain, odd rows the second, as below
    constexpr int RB = G >= 8 ? 16 : 8;   // deeper for the global-memory tiles (n > 128)
    int r = 0;
    for (; r + RB <= n; r += RB) {
#pragma unroll
      for (int k = 0; k < CPL; ++k) {
        if (!cfree[k]) continue;
        VT* cell = tile + r * n + col[k];
        VT x[RB];
#pragma unroll
        for (int b = 0; b < RB; ++b) x[b] = cell[b * n];
        if constexpr (decltype(do_scale)::value) {
#pragma unroll
          for (int b = 0; b < RB; ++b) { x[b] = rescale(x[b], k); cell[b * n] = x[b]; }
        }
#pragma unroll
        for (int b = 0; b < RB; b += 2) {
          upd(x[b], r + b, k, nmax[k], ncnt[k], nrow[k]);
          upd(x[b + 1], r + b + 1, k, mB[k], cB[k], rB[k]);
        }
      }
    }
    for (; r + 1 < n; r += 2) {
#pragma unroll
      for (int k = 0; k < CPL; ++k) {
        if (!cfree[k]) continue;
        VT* cell = tile + r * n + col[k];
        VT v0 = cell[0], v1 = cell[n];
        if constexpr (decltype(do_scale)::value) {
          v0 = rescale(v0, k); v1 = rescale(v1, k);
          cell[0] = v0; cell[n] = v1;
        }
        upd(v0, r, k, nmax[k], ncnt[k], nrow[k]);
        upd(v1, r + 1, k, mB[k], cB[k], rB[k]);
      }
    }
    if (r < n) {
#pragma unroll
      for (int k = 0; k < CPL; ++k) {
        if (!cfree[k]) continue;
        VT* cell = tile + r * n + col[k];
        VT v0 = cell[0];
        if constexpr (decltype(do_scale)::value) { v0 = rescale(v0, k); cell[0] = v0; }
        upd(v0, r, k, nmax[k], ncnt[k], nrow[k]);
      }
    }
  };
  if (smode == 0) {
    stats_rows(std::false_type{});  // lazily scaled layout: u' = lin stays unscaled
  } else if (smode == 1) {
    stats_rows(std::true_type{});   // the normalised (norm mode) path
  } else {
    const ColOut<VT, CPL> g = stats_generic<VT, G, CPL>(tile, n, in);
#pragma unroll
    for (int k = 0; k < CPL; ++k) { nmax[k] = g.m[k]; ncnt[k] = g.c[k]; nrow[k] = g.r[k]; }
  }
#pragma unroll
  for (int k = 0; k < CPL; ++k) {
    if (!cfree[k]) continue;
    // merge the odd-row half (ties: counts add, first row = smaller row)
    if (nmax[k] == NINF || mB[k] > nmax[k]) { nmax[k] = mB[k]; ncnt[k] = cB[k]; nrow[k] = rB[k]; }
    else if (mB[k] == nmax[k] && mB[k] != NINF) { ncnt[k] += cB[k]; nrow[k] = min(nrow[k], rB[k]); }
  }
  ColOut<VT, CPL> o;
#pragma unroll
  for (int k = 0; k < CPL; ++k) { o.m[k] = nmax[k]; o.c[k] = ncnt[k]; o.r[k] = nrow[k]; }
  return o;
}

// Full fp32 velocity pass (the non-incremental case: every entry c1 v, the
// <= 3 touched rows patched afterwards).  Out of line: in the lazily scaled
// layout it runs only when a column is renormalised, and keeping it out of
// the step kernel's body keeps the per-particle path within the
// instruction cache.  Lazily scaled: v = u * cs, the column factor c1 * cs.
template <int CPL>
struct VelIn {
  int col[CPL], zr[CPL], plr[CPL], pgr[CPL];
  bool cfree[CPL];
  float cs[CPL];
  double csd[CPL];   // the column scale as a double (lazily scaled layout: decoded wide word)
};
template <int CPL>
struct VelOut {
  float total[CPL];
  // with `stats` (multi-warp, deferred normalisation): max / tie count /
  // first row of the new column over its non-z rows
  float m[CPL];
  int c[CPL], r[CPL];
};

template <int G, int CPL>
__device__ __noinline__ VelOut<CPL> vel_full_f32(float* tile, int n, const VelIn<CPL> in, double c1,
                                                 double c2r2, double c3r3, double vmax, int v_bounded,
                                                 bool wide, bool stats = false) {
  // wide (the lazily scaled layout): the tile holds wide words (wdec /
  // wenc), decoded to double, scaled and clamped in double, re-encoded;
  // otherwise plain floats in float arithmetic
  const bool WF = wide;
  VelOut<CPL> o;
  int col[CPL], zr[CPL], plr[CPL], pgr[CPL];
  bool cfree[CPL];
  float cs[CPL];
  double csd[CPL];
#pragma unroll
  for (int k = 0; k < CPL; ++k) {
    col[k] = in.col[k]; zr[k] = in.zr[k]; plr[k] = in.plr[k]; pgr[k] = in.pgr[k];
    cfree[k] = in.cfree[k]; cs[k] = in.cs[k]; csd[k] = in.csd[k]; o.total[k] = 0.0f;
    o.m[k] = -INFINITY; o.c[k] = 0; o.r[k] = -1;
  }
  // throughput mode: bulk rows are c1*v; the <= 3 rows touched by
  // x / pl / pg are patched afterwards (sum order is not significant
  // under the fp32 tolerance).  Lazily scaled layout: v = u * s, the
  // column factor is c1 * s and the result stays unnormalised (u' = lin).
  const float c1f = (float)c1;
  const float vm = (float)vmax;
  float c1k[CPL];
  double c1kd[CPL];
#pragma unroll
  for (int k = 0; k < CPL; ++k) { c1k[k] = c1f * cs[k]; c1kd[k] = (double)c1f * csd[k]; }
  float vx[CPL], vl[CPL], vg[CPL], tot[CPL];
#pragma unroll
  for (int k = 0; k < CPL; ++k) {
    tot[k] = 0.f;
    vx[k] = vl[k] = vg[k] = 0.f;
    if (cfree[k]) {
      vx[k] = tile[zr[k] * n + col[k]];
      vl[k] = tile[plr[k] * n + col[k]];
      vg[k] = tile[pgr[k] * n + col[k]];
    }
  }
  // two partial sums per column (even / odd rows) break the FADD
  // dependency chain; the fp32 tolerance admits any summation order
  float tot2[CPL];
#pragma unroll
  for (int k = 0; k < CPL; ++k) tot2[k] = 0.f;
  // |c1 v| <= v_max guaranteed for every stored v: the clamp is a no-op
  const float vmc = v_bounded ? __int_as_float(0x7f800000) : vm;
  const double vmcd = v_bounded ? (double)__int_as_float(0x7f800000) : vmax;
  // one stored word scaled by the column factor and clamped; returns the
  // word to store, and the value's magnitude for the column sum
  auto step1 = [&](float w, int k, float f, double fd, float& mag) -> float {
    if (WF) {
      const double x = fmin(fmax(fd * wdec(w), -vmcd), vmcd);
      mag = (float)fabs(x);
      return wenc(x);
    } else {
      const float x = fminf(fmaxf(f * w, -vmc), vmc);
      mag = fabsf(x);
      return x;
    }
  };
  if constexpr (G == 1 && CPL == 2) {
    // n in 33..64: slot 0 is live in every lane; a dead slot 1 re-runs
    // slot 0's column with a unit factor (same thread, idempotent),
    // which keeps the loop branch-free.  Running smem pointers.
    const bool live1 = cfree[1];
    float* q0 = reinterpret_cast<float*>(tile) + col[0];
    float* q1 = reinterpret_cast<float*>(tile) + (live1 ? col[1] : col[0]);
    const double f0 = c1kd[0];
    const double f1 = live1 ? c1kd[1] : 1.0;
    const int n2 = 2 * n;
    auto run = [&](auto clampit) {
      auto cl = [&](double x) -> double {
        if constexpr (decltype(clampit)::value) return fmin(fmax(x, -vmcd), vmcd);
        else return x;
      };
      auto clf = [&](float x) -> float {
        if constexpr (decltype(clampit)::value) return fminf(fmaxf(x, -vmc), vmc);
        else return x;
      };
      int r = 0;
      if (WF) {
        for (; r + 1 < n; r += 2, q0 += n2, q1 += n2) {
          const double a0 = cl(f0 * wdec(q0[0])), a1 = cl(f0 * wdec(q0[n]));
          q0[0] = wenc(a0); q0[n] = wenc(a1);
          tot[0] += (float)fabs(a0); tot2[0] += (float)fabs(a1);
          const double b0 = cl(f1 * wdec(q1[0])), b1 = cl(f1 * wdec(q1[n]));
          q1[0] = wenc(b0); q1[n] = wenc(b1);
          tot[1] += (float)fabs(b0); tot2[1] += (float)fabs(b1);
        }
        if (r < n) {
          const double a0 = cl(f0 * wdec(q0[0]));
          q0[0] = wenc(a0); tot[0] += (float)fabs(a0);
          const double b0 = cl(f1 * wdec(q1[0]));
          q1[0] = wenc(b0); tot[1] += (float)fabs(b0);
        }
      } else {
        const float g0 = c1k[0], g1 = live1 ? c1k[1] : 1.0f;
        for (; r + 1 < n; r += 2, q0 += n2, q1 += n2) {
          const float a0 = clf(g0 * q0[0]), a1 = clf(g0 * q0[n]);
          q0[0] = a0; q0[n] = a1;
          tot[0] += fabsf(a0); tot2[0] += fabsf(a1);
          const float b0 = clf(g1 * q1[0]), b1 = clf(g1 * q1[n]);
          q1[0] = b0; q1[n] = b1;
          tot[1] += fabsf(b0); tot2[1] += fabsf(b1);
        }
        if (r < n) {
          const float a0 = clf(g0 * q0[0]);
          q0[0] = a0; tot[0] += fabsf(a0);
          const float b0 = clf(g1 * q1[0]);
          q1[0] = b0; tot[1] += fabsf(b0);
        }
      }
    };
    if (v_bounded) run(std::false_type{});
    else run(std::true_type{});
  } else {
    // batches of 8 rows, loads first: with the tile in global memory (GT)
    // the column walk is latency-bound unless many loads are in flight
    constexpr int RB = G >= 8 ? 16 : 8;   // deeper for the global-memory tiles (n > 128)
    // column statistics of the written values (stats): rows ascend, so a
    // strict > keeps the first row of the maximum
    auto track = [&](float w, int row, int k) {
      if (row == zr[k]) return;
      if (w > o.m[k]) { o.m[k] = w; o.c[k] = 1; o.r[k] = row; }
      else if (w == o.m[k]) ++o.c[k];
    };
    int r = 0;
    for (; r + RB <= n; r += RB) {
#pragma unroll
      for (int k = 0; k < CPL; ++k) {
        if (!cfree[k]) continue;
        float* cell = reinterpret_cast<float*>(tile) + r * n + col[k];
        float x[RB];
#pragma unroll
        for (int b = 0; b < RB; ++b) x[b] = cell[b * n];
#pragma unroll
        for (int b = 0; b < RB; ++b) {
          float mag;
          const float w = step1(x[b], k, c1k[k], c1kd[k], mag);
          cell[b * n] = w;
          if (b & 1) tot2[k] += mag; else tot[k] += mag;
          if (stats) track(w, r + b, k);
        }
      }
    }
    for (; r < n; ++r) {
#pragma unroll
      for (int k = 0; k < CPL; ++k) {
        if (!cfree[k]) continue;
        float* cell = reinterpret_cast<float*>(tile) + r * n + col[k];
        float mag;
        const float w = step1(cell[0], k, c1k[k], c1kd[k], mag);
        cell[0] = w;
        tot[k] += mag;
        if (stats) track(w, r, k);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < CPL; ++k) tot[k] += tot2[k];
#pragma unroll
  for (int k = 0; k < CPL; ++k) {
    if (!cfree[k]) continue;
    const int xr = zr[k], lr = plr[k], gr = pgr[k];
    float* colp = reinterpret_cast<float*>(tile) + col[k];
    bool bad = false;
    auto fix = [&](int r, float v0) {
      const float d2 = (float)((r == lr) - (r == xr));
      const float d3 = (float)((r == gr) - (r == xr));
      // the loop's value for this row (its magnitude is in the sum), then
      // the exact one; in double: the pulls and the inertia term can cancel
      float gmag;
      const float g = step1(v0, k, c1k[k], c1kd[k], gmag);
      const double vd = WF ? wdec(v0) : (double)v0;
      const double l = fma(c3r3, (double)d3, fma(c2r2, (double)d2, c1 * (vd * csd[k])));
      if (WF) {
        const double sp = fmin(fmax(l, -vmax), vmax);
        colp[r * n] = wenc(sp);
        tot[k] += (float)fabs(sp) - gmag;
      } else {
        const float sp = (float)fmin(fmax(l, -vmax), vmax);
        colp[r * n] = sp;
        tot[k] += fabsf(sp) - gmag;
        if (stats && r != xr) {
          // the loop counted g for this row; replace it by sp
          float& M = o.m[k];
          int& cnt = o.c[k];
          int& R = o.r[k];
          if (sp > M) { M = sp; cnt = 1; R = r; }
          else if (g == M) { if (sp < M && (--cnt == 0 || R == r)) bad = true; }
          else if (sp == M) { ++cnt; R = min(R, r); }
        }
      }
    };
    fix(xr, vx[k]);
    if (lr != xr) fix(lr, vl[k]);
    if (gr != xr && gr != lr) fix(gr, vg[k]);
    o.total[k] = tot[k];
    if (stats && bad) {
      // a touched row held the maximum and fell below it: rescan the column
      float M = -INFINITY;
      int cnt = 0, R = -1;
      for (int rr = 0; rr < n; ++rr) {
        if (rr == xr) continue;
        const float w = colp[rr * n];
        if (w > M) { M = w; cnt = 1; R = rr; }
        else if (w == M) ++cnt;
      }
      o.m[k] = M; o.c[k] = cnt; o.r[k] = R;
    }
  }
  return o;
}

// Loads of particle pp into the group's staging area: one bulk copy of the
// tile (and, lazily scaled, its column state) on the group's mbarrier, and
// cp.async copies of the perm / pl_perm / pg_perm rows, (c2 r2, c3 r3) and
// (cost, pl_cost) into buffer `buf`.  Inlined at its two call sites (the
// first particle and the prefetch after the aggregation): an out-of-line
// copy saved 7 KB of SASS but cost 2-3 % (call overhead, register saves).
enum LoadFlags : int { L_LAZY = 1, L_PERM = 2, L_COST = 4, L_PL = 8, L_VEL = 16 };

template <typename K, typename VT>
__device__ __forceinline__ void issue_particle_load(const StepArgs* ap, int64_t pp, int buf, int tid,
                                                 int lane, VT* tile, unsigned char* stg, uint64_t* bar,
                                                 uint32_t tile_bytes, uint32_t col_bytes, int lf,
                                                 double inv_s, int part = 3) {
  // part 1: what the previous step kernel wrote (tile, column state, perm /
  // pl_perm rows, costs); part 2: what the best update and the migration
  // write (the swarm-best row, the step's draws)
  const StepArgs& a = *ap;
  if ((part & 1) && tid == 0) {
    bulk_wait_read();                 // the previous bulk store has left the tile
    const bool lz = K::STAGE && (lf & L_LAZY);
    mbar_arrive_expect_tx(bar, tile_bytes + (lz ? col_bytes : 0u));
    bulk_load(tile, reinterpret_cast<const VT*>(a.V) + pp * a.vstride, tile_bytes, bar);
    if (lz) bulk_load(stg + K::SCOL, a.vcol + pp * 5 * (int64_t)a.vcstride, col_bytes, bar);
  }
  if constexpr (K::STAGE) {
    const int n = a.n;
    int16_t* s_perm = reinterpret_cast<int16_t*>(stg + K::SPERM);
    if (lf & L_PERM) {
      const int nw = n >> 1;
      const int64_t ss = (int64_t)__fma_rn((double)pp, inv_s, 0x1p-26);
#pragma unroll 1
      for (int w = lane; w < nw; w += 32) {
        if (part & 1) {
          cp_async4(s_perm + 2 * w, a.perm + pp * n + 2 * w);
          if (lf & L_VEL) cp_async4(s_perm + K::NMAX + 2 * w, a.pl_perm + pp * n + 2 * w);
        }
        if ((part & 2) && (lf & L_VEL)) cp_async4(s_perm + 2 * K::NMAX + 2 * w, a.pg_perm + ss * n + 2 * w);
      }
    }
    if (lane == 0) {
      int64_t* s_cost = reinterpret_cast<int64_t*>(stg + K::SCOST);
      if ((part & 2) && (lf & L_VEL) && a.coef) cp_async16(stg + K::SCOEF, a.coef + 2 * pp);
      if ((part & 1) && (lf & L_COST)) cp_async8(s_cost + 2 * buf, reinterpret_cast<const int64_t*>(a.cost) + pp);
      if ((part & 1) && (lf & L_PL)) cp_async8(s_cost + 2 * buf + 1, reinterpret_cast<const int64_t*>(a.pl_cost) + pp);
    }
    cp_async_commit();
  }
}

// ------------------------------------------------------------------------
// FAST: the throughput step of a lazily scaled fp32 state with every phase,
// the draw pre-pass, no injected draws and even n (engine.step's common
// case).  Those runtime switches become compile-time constants, so the
// paths of the other modes drop out of the kernel body and the hot code
// packs into fewer instruction-cache lines.
template <typename VT, typename MT, int G, int CPL, int W, bool GT = false, bool FAST = false,
          bool CHAIN = false>
// Minimum resident CTAs: one-warp kernels QSB_MINB * 4 warps per SM; the
// multi-warp groups two 8-warp fp32 CTAs with the tile in global memory (n = 256;
// fp64 would spill, smem tiles allow one CTA anyway) or five
// 4-warp CTAs (n <= 128)
// per SM -- without the bound ptxas spends 168 / 106 registers on them and
// halves their occupancy (config 5's step kernel 0.62 -> 0.86 ms)
__global__ void __launch_bounds__(32 * G * W, (G == 1 ? ((sizeof(VT) == 8 && W > 4) ? 1 : (QSB_MINB * 4 + W - 1) / W)
                                                : (G == 8 ? ((sizeof(VT) == 8 || !GT) ? 1 : 2) : 5)))
step_kernel(const __grid_constant__ StepArgs a) {
  // GT: the particle tile stays in global memory (L1/L2-cached) instead of
  // being staged in smem -- used when an n x n tile exceeds shared memory.
  using K = StepKernel<VT, MT, G, CPL, W, GT>;
  constexpr int NT = K::NT;
  constexpr int NW = K::NW;
  using Scratch = typename K::Scratch;
  using Sync = GroupSync<G>;
  constexpr bool kFloatMat = std::is_floating_point<MT>::value;
  // Lazily scaled fp32 layout (a.vcol set; one-warp groups): the tile holds
  // u with v = u * s per column, and a step rewrites only the <= 3 entries
  // per column that x / pl / pg touch ("lazy column scale").
  // (multi-warp groups too, since round 2: the global-memory tile (GT)
  // included; each thread owns one column and rescans its own column)
  constexpr bool kLazy = sizeof(VT) == 4 && (G > 1 || !GT);
  const bool lazy = FAST || (kLazy && a.vcol != nullptr && (G == 1 || !a.mw_defer));
  const bool wide = lazy;   // lazily scaled fp32 tiles hold wide words (vval)
  // multi-warp fp32 kernels with a column-scale array: deferred column
  // normalisation -- the tile keeps the unnormalised velocity u and row 0
  // of vcol the column scale s (v = u * s), so a step reads and writes every
  // entry once, with no second (rescale) pass over the tile
  const bool defer = !FAST && sizeof(VT) == 4 && G > 1 && a.vcol != nullptr && !lazy;

  // PDL: the prologue below reads only what the previous STEP kernel and
  // the 2-opt wrote (the first particle's tile, rows and costs) and the
  // instance; it overlaps the best update (and migration), whose
  // griddepcontrol.wait covered those writes before it let this grid launch.
  // Everything the best update / migration write (t, the draws, the swarm
  // bests, the particle counter) is read after pdl_wait() below.
  extern __shared__ __align__(128) unsigned char smem[];
  const int n = a.n;
  const int nn = n * n;
  const bool fds = (FAST && G == 1) || a.fd_smem;   // multi-warp: F / D via L1 when incremental
  MT* sF = reinterpret_cast<MT*>(smem);
  MT* sD = sF + nn;
  const int gidx = threadIdx.x / NT;
  const int tid = threadIdx.x % NT;
  const int lane = threadIdx.x & 31;
  unsigned char* gb = smem + (fds ? K::fd_bytes(n) : 0) + (size_t)gidx * K::group_bytes(a.vstride);
  VT* tile = reinterpret_cast<VT*>(gb);   // re-pointed per particle when GT
  unsigned char* stg = gb + K::tile_bytes(a.vstride);
  float* s_col = reinterpret_cast<float*>(stg + K::SCOL);
  int16_t* s_perm = reinterpret_cast<int16_t*>(stg + K::SPERM);
  double* s_coef = reinterpret_cast<double*>(stg + K::SCOEF);
  int64_t* s_cost = reinterpret_cast<int64_t*>(stg + K::SCOST);
  Scratch& sc = *reinterpret_cast<Scratch*>(stg + K::stage_bytes());

  const bool do_vel = FAST || (a.flags & F_VELOCITY);
  const bool do_agg = FAST || (a.flags & F_AGGREGATE);
  const bool do_cost = FAST || (a.flags & F_COST);
  const bool do_pbest = FAST || (a.flags & F_PBEST);
  const bool store_v = FAST || (a.flags & F_STORE_V);
  // FAST also fixes the steady-state properties of that case: norm S_v,
  // second-target S_x with depth > 0, |c1 v| <= v_max, symmetric integral
  // instance with 32-bit goal sums, cost[p] current
  const bool normalize = FAST || a.normalize;
  const bool v_bounded = FAST || a.v_bounded;
  const bool cost_incr = FAST || a.cost_incremental;
  const bool acc32 = FAST || a.acc32;
  const bool symmetric = FAST || a.symmetric;
  const int mode = FAST ? (int)MODE_SECOND_TARGET : a.mode;

  const MT* cF = sF;
  const MT* cD = sD;
  if (tid == 0) { mbar_init(&sc.bar, 1); mbar_fence_init(); }
  for (int c = tid; c < K::NMAX; c += NT) { sc.stie[c] = 0; sc.sS[c] = 1.0f; }
  if (tid == 0) sc.wide = wide;
  __syncthreads();

  const uint32_t tile_bytes = (uint32_t)(a.vstride * sizeof(VT));
  const int64_t ngroups = (int64_t)gridDim.x * W;
  const int row_w = 2 + 2 * n;
  uint32_t phase = 0;
  int par = 0;

  // Particle scheduling: a shared work counter when given (per-particle cost
  // varies with ties and rescans; dynamic assignment removes the tail),
  // else a static grid stride.  The next index is claimed when a particle
  // starts, so the atomic's latency is hidden behind the particle's work.
  auto claim = [&]() -> unsigned {
    // plain atom (not the compiler's warp-aggregated form, whose broadcast
    // would wait for the result right here)
    unsigned q = 0, lid;
    asm volatile("mov.u32 %0, %%laneid;" : "=r"(lid));
    if (lid == 0 && tid < 32)
      asm volatile("atom.global.add.u32 %0, [%1], 1;" : "=r"(q) : "l"(a.work + (lid >> 5)) : "memory");
    return q;
  };
  auto bcast = [&](unsigned q) -> int64_t {
    if constexpr (G == 1) {
      return (int64_t)__shfl_sync(FULL, q, 0);
    } else {
      __syncthreads();
      if (tid == 0) sc.ssel[1] = (int)q;
      __syncthreads();
      return (int64_t)(unsigned)sc.ssel[1];
    }
  };
  // the first particle is static; later ones are claimed from the counter
  // (the best update resets it) and offset past the static ones
  int64_t p = (int64_t)blockIdx.x * W + gidx;
  // The next particle's tile is prefetched as soon as the aggregation has
  // stopped reading the current one, so the load overlaps the goal and
  // personal-best phases; `loaded` says whether p's load is in flight.
  bool loaded = false;
  const int vcs = a.vcstride;
  const uint32_t col_bytes = (uint32_t)(5 * vcs * sizeof(float));
  // staged perm rows need 4-byte aligned rows (n even)
  const bool stage_perm = K::STAGE && (FAST || (n % 2) == 0);
  const bool stage_cost = K::STAGE && do_cost && cost_incr && !kFloatMat;
  const bool stage_pl = K::STAGE && do_pbest && do_cost;
  int cbuf = 0;   // s_cost buffer of the particle being processed
  // p / S via a reciprocal: p < 2^24 (host limit), so p * (1/S) is within
  // 2^-28 of p / S, while a non-zero fractional part of p / S is at least
  // 1 / S >= 2^-24: the 2^-26 nudge makes the truncation exact
  const double inv_s = 1.0 / (double)a.S;
  auto swarm_of = [&](int64_t pp) -> int64_t {
    return (int64_t)__fma_rn((double)pp, inv_s, 0x1p-26);
  };
  const int lflags = (lazy ? L_LAZY : 0) | (stage_perm ? L_PERM : 0) | (stage_cost ? L_COST : 0) |
                     (stage_pl ? L_PL : 0) | (do_vel ? L_VEL : 0);
  auto issue_load = [&](int64_t pp, int buf, int part = 3) {
    issue_particle_load<K, VT>(&a, pp, buf, tid, lane, tile, stg, &sc.bar, tile_bytes, col_bytes, lflags,
                               inv_s, part);
  };
  // the first particle's operands are requested before F and D are staged,
  // so the two loads overlap (each warp's first tile is not prefetched)
  if (!GT && p < a.P) { issue_load(p, cbuf, 1); loaded = true; }
  if (do_cost) {
    const MT* gF = reinterpret_cast<const MT*>(a.F);
    const MT* gD = reinterpret_cast<const MT*>(a.D);
    if (G == 1 || fds) {
      if ((nn * sizeof(MT)) % 16 == 0) {
        // 16-byte copies (sD = sF + nn stays aligned)
        const int nv = (int)(nn * sizeof(MT) / 16);
        const uint4* gF4 = reinterpret_cast<const uint4*>(gF);
        const uint4* gD4 = reinterpret_cast<const uint4*>(gD);
        uint4* sF4 = reinterpret_cast<uint4*>(sF);
        uint4* sD4 = reinterpret_cast<uint4*>(sD);
        for (int i = threadIdx.x; i < nv; i += blockDim.x) { sF4[i] = gF4[i]; sD4[i] = gD4[i]; }
      } else {
        for (int i = threadIdx.x; i < nn; i += blockDim.x) { sF[i] = gF[i]; sD[i] = gD[i]; }
      }
    } else {
      cF = gF; cD = gD;
    }
  }
  // from here on: what the best update / migration wrote
  pdl_wait();
  // a step whose personal best is left to the 2-opt (the engine's 2-opt
  // configs) lets that kernel be placed as this grid's CTAs retire, so its
  // F / D / TMEM prologue overlaps this grid's tail (it waits on this grid
  // before reading the positions); configs 2 / 5 +1.7 %.  Ahead of the best
  // update an early trigger measured 1 % slower (config 3), so it stays at exit.
  if (!do_pbest) pdl_launch();
  const uint64_t t = a.t_dev ? (uint64_t)(*a.t_dev) + 1 : a.t_host;
  const uint64_t word1 = stream_word(2, t);
  if (!GT && p < a.P) issue_load(p, cbuf, 2);
  __syncthreads();
  while (p < a.P) {
    const unsigned q_next = a.work ? claim() : 0u;
    int64_t p_next = -1;
    VT* gV = reinterpret_cast<VT*>(a.V) + p * a.vstride;
    if constexpr (GT) {
      tile = gV;
    } else if (!loaded) {
      issue_load(p, cbuf);
    }
    loaded = false;
    if constexpr (K::STAGE) {
      // this particle's tile, column state and rows are in shared memory
      mbar_wait(&sc.bar, phase);
      phase ^= 1u;
      cp_async_wait_all();
      __syncwarp();
    }

    QSB_COUNT(0, 1);
    // multi-warp groups (n > 64) keep the last Philox block of the draw row
    // in registers: their aggregation can take long runs of tie draws at
    // consecutive cursors (one block serves four); the one-warp kernels are
    // at the register cap and draw rarely
    uint64_t dcb = ~0ULL;
    PhiloxBlock dblk{};
    // the particle's draw row, built where a draw is taken (ties, pick-
    // column, no pre-pass): the key is kernel constants plus p, so it needs
    // no registers across the particle
    auto mkdr = [&]() -> DrawKey {
      DrawKey d;
      d.inj = (!FAST && a.inj_draws) ? a.inj_draws + p * a.inj_stride : nullptr;
      d.seed = a.seed;
      d.word1 = word1;
      d.base = (uint64_t)(a.p0 + p) * (uint64_t)row_w;
      return d;
    };

    // ---- per-column registers.  Every global load of the particle's
    // column data is issued first; the draw block (a dependent Philox chain)
    // runs while they are in flight.
    int zr[CPL], col[CPL], plr[CPL], pgr[CPL];
    bool cfree[CPL];
    const int16_t* gperm = a.perm + p * n;
    const int64_t s = swarm_of(p);
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      col[k] = tid + k * NT;
      cfree[k] = col[k] < n;
      plr[k] = pgr[k] = -1;
      if (stage_perm) {
        zr[k] = cfree[k] ? (int)s_perm[col[k]] : -1;
        if (do_vel && cfree[k]) {
          plr[k] = s_perm[K::NMAX + col[k]];
          pgr[k] = s_perm[2 * K::NMAX + col[k]];
        }
      } else {
        zr[k] = cfree[k] ? (int)gperm[col[k]] : -1;
        if (do_vel && cfree[k]) {
          plr[k] = a.pl_perm[p * n + col[k]];
          pgr[k] = a.pg_perm[s * n + col[k]];
        }
      }
    }
    // lazily scaled layout: column scale s, sum A of |u| over the column,
    // and the max / tie count / first row of u over the rows other than the
    // z row zp of the step that wrote them (M = NaN: not known)
    float cs[CPL], cM[CPL];
    double csd[CPL];   // the column scale (lazily scaled layout: a wide word, decoded)
    double cA[CPL];
    int cCR[CPL];
    float* vcp = lazy ? a.vcol + p * 5 * (int64_t)vcs : nullptr;
    const float* vcr = K::STAGE ? s_col : vcp;   // staged copy when one-warp
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      cs[k] = 1.0f; cA[k] = 0.0; cM[k] = 0.0f; cCR[k] = 0;
      if (defer && cfree[k]) cs[k] = a.vcol[p * 5 * (int64_t)vcs + col[k]];
      if (lazy && cfree[k]) {
        cs[k] = vcr[col[k]];
        cA[k] = __hiloint2double(__float_as_int(vcr[2 * vcs + col[k]]),
                                 __float_as_int(vcr[vcs + col[k]]));
        cM[k] = vcr[3 * vcs + col[k]];
        cCR[k] = __float_as_int(vcr[4 * vcs + col[k]]);
      }
      csd[k] = lazy ? wdec(cs[k]) : (double)cs[k];
    }
    double c2r2 = 0.0, c3r3 = 0.0;
    if (do_vel) {
      if (FAST || a.coef) {
        const double* cf = K::STAGE ? s_coef : a.coef + 2 * p;
        c2r2 = cf[0]; c3r3 = cf[1];
      } else {
        c2r2 = __dmul_rn(a.c2, draw_at(mkdr(), 0));   // engine.py:198-199: c2 * r2, c3 * r3
        c3r3 = __dmul_rn(a.c3, draw_at(mkdr(), 1));
      }
    }
#pragma unroll
    for (int k = 0; k < CPL; ++k)
      if (cfree[k]) sc.szr[col[k]] = zr[k];
    // incremental step: every column's state known and in range, no clamp
    // on the untouched entries, c1 > 0 (else the full pass, which also
    // renormalises: u := v, s := 1 / sum |v|)
    bool incr = false;
    if (lazy && do_vel) {
      bool ok = v_bounded && a.c1 > 0.0;
      const float c1f = (float)a.c1;
      // |lin| of a touched entry is at most lb (the clamp, and c1 + c2 + c3
      // for normalised columns), so u' = lin / (c1 s) stays below 2^125
      const float lb = fminf((float)a.vmax, normalize ? (float)(a.c1 + a.c2 + a.c3) : INFINITY);
#pragma unroll
      for (int k = 0; k < CPL; ++k) {
        if (!cfree[k]) continue;
        // wide scale and words: the range only has to keep u' = lin / (c1 s)
        // and the products u * s inside the double exponent range
        const double c1s = a.c1 * csd[k];
        ok &= cM[k] == cM[k] && csd[k] >= 0x1p-900 && csd[k] <= 0x1p900 && c1s >= 0x1p-900 &&
              c1s <= 0x1p900 && c1s >= (double)lb * 0x1p-900;
      }
      if constexpr (G == 1) incr = __all_sync(FULL, ok);
      else incr = __syncthreads_and(ok);      // one group per CTA (W = 1)
      if (!incr) QSB_COUNT(8, 1);
    }

    if constexpr (!GT && !K::STAGE) {
      mbar_wait(&sc.bar, phase);
      phase ^= 1u;
    }

    // ================= phase 1: velocity update (_batch.py:39-50)
    // Row-outer loops over the CPL owned columns: every column still sums in
    // row order (the reference's order), and the lanes share loop overhead.
    VT total[CPL];
    double c1sdk[CPL];   // incremental lazy step: the column factor c1 * s
    float vnm[CPL];          // column statistics from the velocity walk (deferred
    int vnc[CPL], vnr[CPL];  // normalisation, multi-warp fp32)
    bool vstats = false;
#pragma unroll
    for (int k = 0; k < CPL; ++k) total[k] = (VT)0;
    if (do_vel) {
      if constexpr (sizeof(VT) == 8) {
        // reference order, no contraction: (c1*v + c2r2*(pl-x)) + c3r3*(pg-x)
        const double z2 = __dmul_rn(c2r2, 0.0), z3 = __dmul_rn(c3r3, 0.0);
        double tot[CPL];
#pragma unroll
        for (int k = 0; k < CPL; ++k) tot[k] = 0.0;
        // GT tiles (global memory): loads issued 16 rows ahead; the
        // arithmetic and the column sum stay in row order
        constexpr int RB = GT ? 16 : 1;
        double xb[CPL][RB];
        for (int r = 0; r < n; ++r) {
          if (GT && (r & (RB - 1)) == 0) {
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
              if (!cfree[k]) continue;
#pragma unroll
              for (int b = 0; b < RB; ++b)
                if (r + b < n) xb[k][b] = tile[(r + b) * n + col[k]];
            }
          }
#pragma unroll
          for (int k = 0; k < CPL; ++k) {
            if (!cfree[k]) continue;
            const int xr = zr[k], lr = plr[k], gr = pgr[k];
            double* cell = tile + r * n + col[k];
            double v = GT ? xb[k][0] : *cell;   // smem tiles: direct loads
#pragma unroll
            for (int b = 1; b < RB; ++b) if ((r & (RB - 1)) == b) v = xb[k][b];
            const bool special = r == xr || r == lr || r == gr;
            double lin;
            if (special) {
              const double d2 = (r == lr) ? ((r == xr) ? 0.0 : 1.0) : ((r == xr) ? -1.0 : 0.0);
              const double d3 = (r == gr) ? ((r == xr) ? 0.0 : 1.0) : ((r == xr) ? -1.0 : 0.0);
              lin = __dadd_rn(__dadd_rn(__dmul_rn(a.c1, v), __dmul_rn(c2r2, d2)), __dmul_rn(c3r3, d3));
            } else {
              lin = __dadd_rn(__dadd_rn(__dmul_rn(a.c1, v), z2), z3);
            }
            if (!v_bounded || special) {
              if (lin > a.vmax) lin = a.vmax;
              else if (lin < -a.vmax) lin = -a.vmax;
            }
            *cell = lin;
            tot[k] = __dadd_rn(tot[k], fabs(lin));
          }
        }
#pragma unroll
        for (int k = 0; k < CPL; ++k) total[k] = (VT)tot[k];
      } else if (incr) {
        // lazily scaled layout, incremental: v' = normalise(c1 v + ...) is
        // c1 s u / total on every entry x / pl / pg leave alone, so those
        // keep u and the column scale becomes s' = c1 s / total; the
        // touched entries get u' = lin / (c1 s).  Since total = c1 s A' with
        // A' = sum |u'|, s' = 1 / A'.  The all-rows statistics are updated
        // entry by entry (an entry leaving the maximum forces a rescan).
        const float vm = (float)a.vmax;
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
          if (!cfree[k]) continue;
          const int xr = zr[k], lr = plr[k], gr = pgr[k];
          // lin of a touched entry is formed in double (the pulls and the
          // inertia term can cancel), then rounded once; u' = lin / (c1 s)
          const double c1sd = a.c1 * csd[k];
          const double rcd = drcp_approx(c1sd);       // c1 s in [2^-900, 2^900]
          // statistics over the rows other than zp (the previous step's z row)
          float M = cM[k];
          int cnt = cCR[k] >> 16, R = (cCR[k] >> 8) & 0xff;
          const int zp = cCR[k] & 0xff;
          double Ad = cA[k];
          bool bad = false;
          float* colp = reinterpret_cast<float*>(tile) + col[k];
          float* gcol = reinterpret_cast<float*>(gV) + col[k];   // == colp for GT tiles
          // the touched rows and their pulls c2 r2 (pl - x) + c3 r3 (pg - x):
          //   x row: -c2 r2 [x != pl] - c3 r3 [x != pg] (none: unchanged)
          //   pl row (!= x): c2 r2 + c3 r3 [pl == pg];  pg row (!= x, pl): c3 r3
          const double offx = -(xr != lr ? c2r2 : 0.0) - (xr != gr ? c3r3 : 0.0);
          const double offl = c2r2 + (lr == gr ? c3r3 : 0.0);
          auto upd = [&](int r, double off) {
            const float u = colp[r * n];             // wide word
            const double ud = wdec(u);
            const float lin = fminf(fmaxf((float)fma(c1sd, ud, off), -vm), vm);
            const double u2d = (double)lin * rcd;
            const float u2 = wenc(u2d);
            colp[r * n] = u2;
            if (store_v && !GT) gcol[r * n] = u2;
            Ad += fabs(wdec(u2)) - fabs(ud);
            if (r == zp) return;
            if (u2 > M) { M = u2; cnt = 1; R = r; }
            else if (u == M) { if (u2 < M && (--cnt == 0 || R == r)) bad = true; }
            else if (u2 == M) { ++cnt; R = min(R, r); }
          };
          if (offx != 0.0) upd(xr, offx);
          if (lr != xr) upd(lr, offl);
          if (gr != xr && gr != lr) upd(gr, c3r3);
          if (xr != zp) {
            // the excluded row moves from zp to this step's z row xr
            const float uo = colp[zp * n];
            if (uo > M) { M = uo; cnt = 1; R = zp; }
            else if (uo == M) { ++cnt; R = min(R, zp); }
            if (colp[xr * n] == M && (--cnt == 0 || R == xr)) bad = true;
          }
          // A' is kept in double (exact differences of fp32 values); a
          // column that shrinks sharply is re-summed
          bad |= !(Ad >= 0.0625 * cA[k]);
          cA[k] = Ad;
          cM[k] = M;
          cCR[k] = bad ? -1 : ((cnt << 16) | (R << 8) | xr);
          total[k] = (float)c1sd;   // incremental mode: total carries the column factor c1 * s
          c1sdk[k] = c1sd;
        }
        fence_proxy_async_smem();   // generic tile writes before the next bulk load
      } else {
        VelIn<CPL> vi;
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
          vi.col[k] = col[k]; vi.zr[k] = zr[k]; vi.plr[k] = plr[k]; vi.pgr[k] = pgr[k];
          vi.cfree[k] = cfree[k]; vi.cs[k] = cs[k]; vi.csd[k] = csd[k];
        }
        const VelOut<CPL> vo = vel_full_f32<G, CPL>(reinterpret_cast<float*>(tile), n, vi, a.c1, c2r2,
                                                    c3r3, a.vmax, v_bounded, wide, GT && defer && do_agg);
#pragma unroll
        for (int k = 0; k < CPL; ++k) total[k] = (VT)vo.total[k];
        if (GT && defer && do_agg) {
          // deferred normalisation keeps the written values: their column
          // statistics came out of the velocity walk (no second pass over a
          // global-memory tile; smem tiles keep the two-chain stats pass)
#pragma unroll
          for (int k = 0; k < CPL; ++k) { vnm[k] = vo.m[k]; vnc[k] = vo.c[k]; vnr[k] = vo.r[k]; }
          vstats = true;
        }
      }
    }

    // ================= normalisation (_batch.py:51-58) + initial statistics
    // Per column: max / tie count / first row of v over the non-z rows
    // (the z row is masked to -inf; stored values are finite) and the z key.
    VT nmax[CPL];
    int ncnt[CPL], nrow[CPL];
    uint64_t nk64[CPL], zkey[CPL];
    bool zel[CPL], scale[CPL];
    VT inv[CPL];
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      nmax[k] = (VT)(-INFINITY); ncnt[k] = 0; nrow[k] = -1; nk64[k] = 0; zkey[k] = 0; zel[k] = false;
      scale[k] = !lazy && !defer && cfree[k] && do_vel && normalize && total[k] > (VT)0;
      inv[k] = (VT)1;
      if constexpr (sizeof(VT) == 4) inv[k] = scale[k] ? 1.0f / total[k] : 1.0f;
    }
    auto rescale = [&](VT v, int k) -> VT {
      if constexpr (sizeof(VT) == 8) return __ddiv_rn(v, total[k]);
      else return v * inv[k];
    };
    float sK[CPL];   // column scale of the tile after this phase (v = u * sK)
#pragma unroll
    for (int k = 0; k < CPL; ++k) sK[k] = 1.0f;
    bool stats_done = false;
    if constexpr (sizeof(VT) == 4 && G > 1) {
      if (vstats) {
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
          nmax[k] = vnm[k]; ncnt[k] = cfree[k] ? vnc[k] : 0; nrow[k] = ncnt[k] ? vnr[k] : -1;
        }
        stats_done = true;
      }
    }
    if constexpr (kLazy) {
      if (lazy && do_vel) {
        // incremental step: the non-z statistics were carried through the
        // update; rescan the columns where they became unknown.  Full pass:
        // rescan every column (the sums in double).
        bool need[CPL];
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
          need[k] = cfree[k] && (!incr || cCR[k] < 0);
          if (cfree[k] && !need[k]) {
            nmax[k] = cM[k]; ncnt[k] = cCR[k] >> 16; nrow[k] = (cCR[k] >> 8) & 0xff;
          }
        }
        if constexpr (G == 1) {
        // cooperative rescans (lanes over rows): non-z max / count / first
        // row, and the sum of |u| over all rows
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
          unsigned mask = __ballot_sync(FULL, need[k]);
          while (mask) {
            const int src = __ffs(mask) - 1;
            mask &= mask - 1;
            QSB_COUNT(9, 1);
            const int c = src + k * 32;
            const int zc = __shfl_sync(FULL, zr[k], src);
            if (__shfl_sync(FULL, cCR[k], src) < 0) QSB_COUNT(10, 1);
            unsigned kj[CPL];
            unsigned km = 0;
            double sum = 0.0;
#pragma unroll
            for (int j = 0; j < CPL; ++j) {
              const int r = lane + j * 32;
              kj[j] = 0u;
              if (r >= n) continue;
              const float u = (float)tile[r * n + c];   // wide word
              sum += fabs(wdec(u));
              if (r == zc) continue;
              kj[j] = okey32(__fadd_rn(u, 0.0f));
              km = max(km, kj[j]);
            }
            // the maximum by one reduction, its rows by ballots
            const unsigned M = __reduce_max_sync(FULL, km);
            unsigned tot = 0, rr = INT_MAX;
#pragma unroll
            for (int j = CPL - 1; j >= 0; --j) {
              const unsigned b = __ballot_sync(FULL, M != 0u && kj[j] == M);
              tot += __popc(b);
              if (b) rr = j * 32 + __ffs(b) - 1;
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(FULL, sum, o);
            if (lane == src) {
              ncnt[k] = (int)tot;
              nrow[k] = tot ? (int)rr : -1;
              nmax[k] = tot ? (VT)from_okey32(M) : (VT)0;
              cA[k] = sum;
              cM[k] = (float)nmax[k];
              cCR[k] = tot ? (((int)tot << 16) | ((int)rr << 8) | zc) : -1;
            }
          }
        }
        } else {
          // multi-warp groups: each warp rescans the columns it owns, lanes
          // over rows (rows lane + 32 j), warp reductions only -- no group
          // barrier; the columns of a group are independent
          constexpr int RPL = (K::NMAX + 31) / 32;
#pragma unroll
          for (int k = 0; k < CPL; ++k) {
            unsigned mask = __ballot_sync(FULL, need[k]);
            while (mask) {
              const int src = __ffs(mask) - 1;
              mask &= mask - 1;
              QSB_COUNT(9, 1);
              const int c = __shfl_sync(FULL, col[k], src);
              const int zc = __shfl_sync(FULL, zr[k], src);
              const float* colq = reinterpret_cast<const float*>(tile) + c;
              unsigned kj[RPL];
              unsigned km = 0;
              double sum = 0.0;
#pragma unroll
              for (int j = 0; j < RPL; ++j) {
                const int r = lane + 32 * j;
                kj[j] = 0u;
                if (r >= n) continue;
                const float u = colq[r * n];   // wide word
                sum += fabs(wdec(u));
                if (r == zc) continue;
                kj[j] = okey32(__fadd_rn(u, 0.0f));
                km = max(km, kj[j]);
              }
              const unsigned M = __reduce_max_sync(FULL, km);
              unsigned tot = 0, rr = INT_MAX;
#pragma unroll
              for (int j = RPL - 1; j >= 0; --j) {
                const unsigned bb = __ballot_sync(FULL, M != 0u && kj[j] == M);
                tot += __popc(bb);
                if (bb) rr = j * 32 + __ffs(bb) - 1;
              }
#pragma unroll
              for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(FULL, sum, o);
              if (lane == src) {
                ncnt[k] = (int)tot;
                nrow[k] = tot ? (int)rr : -1;
                nmax[k] = tot ? (VT)from_okey32(M) : (VT)0;
                cA[k] = sum;
                cM[k] = (float)nmax[k];
                cCR[k] = tot ? (((int)tot << 16) | ((int)rr << 8) | zc) : -1;
              }
            }
          }
        }
        // s' = 1 / A' (normalised: v' = lin / total, total = c1 s A' in the
        // incremental step, = A' in the full pass); raw mode or a zero
        // column: no normalisation
#pragma unroll
        for (int k = 0; k < CPL; ++k)
          // the new scale as a wide word (double range, so no renormalising pass)
          sK[k] = wenc((normalize && cA[k] > 0.0) ? drcp_approx(cA[k]) : (incr ? c1sdk[k] : 1.0));
        stats_done = true;
      }
    }
    if (stats_done) {
    } else if (do_agg) {
      ColIn<VT, CPL> in;
      bool all_scale = true;
#pragma unroll
      for (int k = 0; k < CPL; ++k) {
        in.col[k] = col[k]; in.zr[k] = zr[k]; in.cfree[k] = cfree[k]; in.scale[k] = scale[k];
        in.total[k] = total[k]; in.inv[k] = inv[k];
        all_scale &= scale[k] || !cfree[k];
      }
      const int smode = ((kLazy && lazy) || defer) ? 0 : (__all_sync(FULL, all_scale) ? 1 : 2);
      const ColOut<VT, CPL> so = stats_pass<VT, G, CPL>(tile, n, in, smode);
#pragma unroll
      for (int k = 0; k < CPL; ++k) { nmax[k] = so.m[k]; ncnt[k] = so.c[k]; nrow[k] = so.r[k]; }
    } else if (!lazy && !defer) {
      // normalisation only (no aggregation): batches of 16 rows, loads first
      constexpr int RB = 16;
      int r = 0;
#pragma unroll 1
      for (; r + RB <= n; r += RB) {
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
          if (!scale[k]) continue;
          VT* cell = tile + r * n + col[k];
          VT x[RB];
#pragma unroll
          for (int b = 0; b < RB; ++b) x[b] = cell[b * n];
#pragma unroll
          for (int b = 0; b < RB; ++b) cell[b * n] = rescale(x[b], k);
        }
      }
#pragma unroll 1
      for (; r < n; ++r) {
#pragma unroll
        for (int k = 0; k < CPL; ++k)
          if (scale[k]) tile[r * n + col[k]] = rescale(tile[r * n + col[k]], k);
      }
    }
    if constexpr (kLazy) {
      if (lazy) {
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
          if (!cfree[k]) continue;
          if (!do_vel) sK[k] = cs[k];
          sc.sS[col[k]] = sK[k];
        }
      }
    }
    if (defer) {
      // deferred normalisation: s' = 1 / sum |lin| for a normalised live
      // column, 1 otherwise (raw mode, zero column); stored in vcol row 0
      float* vs = a.vcol + p * 5 * (int64_t)vcs;
#pragma unroll
      for (int k = 0; k < CPL; ++k) {
        if (!cfree[k]) continue;
        sK[k] = !do_vel ? cs[k] : ((normalize && total[k] > (VT)0) ? 1.0f / (float)total[k] : 1.0f);
        sc.sS[col[k]] = sK[k];
        if (do_vel && store_v) vs[col[k]] = sK[k];
      }
    }
    if (do_agg) {
#pragma unroll
      for (int k = 0; k < CPL; ++k) {
        if (!cfree[k]) continue;
        nk64[k] = ncnt[k] ? nonz_key(nmax[k], sK[k], wide) : 0;
        zkey[k] = z_key(tile[zr[k] * n + col[k]], sK[k], wide);
      }
    }
    if (!GT && do_vel && store_v && !incr) {
      fence_proxy_async_smem();
      Sync::sync();
      if (tid == 0) bulk_store(gV, tile, tile_bytes);
    } else {
      Sync::sync();
    }
    if constexpr (kLazy) {
      if (lazy && do_vel && store_v) {
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
          if (!cfree[k]) continue;
          vcp[col[k]] = sK[k];
          vcp[vcs + col[k]] = __int_as_float(__double2loint(cA[k]));
          vcp[2 * vcs + col[k]] = __int_as_float(__double2hiint(cA[k]));
          vcp[3 * vcs + col[k]] = cCR[k] < 0 ? __int_as_float(0x7fc00000) : cM[k];
          vcp[4 * vcs + col[k]] = __int_as_float(cCR[k] < 0 ? 0 : cCR[k]);
        }
      }
    }

    // ================= phase 2: aggregation S_x(X + V)
    if (do_agg) {
      RowSet<NW> rf;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const int lo = w * 64;
        rf.w[w] = (n - lo >= 64) ? ~0ULL : (n > lo ? ((1ULL << (n - lo)) - 1) : 0ULL);
      }
      int cursor = a.agg_base;     // next aggregation draw (column in the draw row)

      if (mode == MODE_PICK_COLUMN) {
        agg_pick_column<VT, G, NW>(tile, n, sc, rf, mkdr(), cursor, tid, lane);
      } else {
        bool restricted = (mode == MODE_SECOND_TARGET) && a.depth > 0;
        // cached per-column candidate: (key, tie count, first row) of the
        // column's best eligible cell; recomputed only when its parts change
        uint64_t ck[CPL];
        int cc[CPL], cr[CPL];
        auto recompute = [&](int k) {
          const uint64_t nk = ncnt[k] ? nk64[k] : 0;
          const uint64_t zk = zel[k] ? zkey[k] : 0;
          if (nk > zk) { ck[k] = nk; cc[k] = ncnt[k]; cr[k] = nrow[k]; }
          else if (zk > nk) { ck[k] = zk; cc[k] = 1; cr[k] = zr[k]; }
          else {
            ck[k] = zk;
            cc[k] = zk ? ncnt[k] + 1 : 0;
            cr[k] = nrow[k] < 0 ? -1 : min(nrow[k], zr[k]);
          }
        };
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
          zel[k] = cfree[k] && !restricted;
          ck[k] = 0; cc[k] = 0; cr[k] = -1;
          if (cfree[k]) recompute(k);
        }
        int nbulk = 0;     // z keys placed by bulk steps, tie draws not yet counted
        int bpar = 0;      // multi-warp bulk attempts: buffer parity
        Best pre{};        // multi-warp: the round's reduction, done beside the bulk threshold
        bool have_pre = false;

        for (int rnd = 0; rnd < n; ++rnd) {
          if (restricted && rnd == a.depth) {
            // leaving the restricted rounds: free z cells become candidates
            restricted = false;
#pragma unroll
            for (int k = 0; k < CPL; ++k)
              if (cfree[k]) { zel[k] = rf.has(zr[k]); recompute(k); }
          }
          if constexpr (G == 1 && CPL <= 2) {
            // ---- endgame: with k <= 5 free columns left (after the bulk
            // step, typically 4), lane l holds cell (R[l / k], C[l % k]) of
            // the k x k free submatrix, R / C the free rows / columns in
            // ascending order.  Lane order is row-major, so every remaining
            // round is one warp max and a tie picks the pick-th set bit of
            // the tie ballot (_batch.py:155-170).
            const int kf = n - rnd;
            if (!restricted && kf <= 5) {
              // ascending lists of the free rows (sc.srow) and columns
              // (sc.sorder), each entry written by its owner lane
              const unsigned lt = (1u << lane) - 1u;
              const unsigned rl = (unsigned)rf.w[0], rh = (unsigned)(rf.w[0] >> 32);
              if ((rl >> lane) & 1u) sc.srow[__popc(rl & lt)] = (uint16_t)lane;
              if ((rh >> lane) & 1u) sc.srow[__popc(rl) + __popc(rh & lt)] = (uint16_t)(lane + 32);
              const unsigned cb0 = __ballot_sync(FULL, cfree[0]);
              if (cfree[0]) sc.sorder[__popc(cb0 & lt)] = (uint8_t)col[0];
              if constexpr (CPL == 2) {
                const unsigned cb1 = __ballot_sync(FULL, cfree[1]);
                if (cfree[1]) sc.sorder[__popc(cb0) + __popc(cb1 & lt)] = (uint8_t)col[1];
              }
              __syncwarp();
              const int ei = lane / kf, ej = lane - ei * kf;
              bool act = lane < kf * kf;
              int er = 0, ec = 0;
              uint64_t ekey = 0;
              if (act) {
                er = sc.srow[ei];
                ec = sc.sorder[ej];
                ekey = mkey(tile, sc.sS, n, er, ec, (int)sc.szr[ec], sc.wide);
              }
#pragma unroll 1
              for (int left = kf; left > 0; --left) {
                const uint64_t kk = act ? ekey : 0ULL;
                const unsigned mh = __reduce_max_sync(FULL, (unsigned)(kk >> 32));
                const unsigned ml = __reduce_max_sync(FULL, (unsigned)(kk >> 32) == mh ? (unsigned)kk : 0u);
                const uint64_t M = ((uint64_t)mh << 32) | ml;
                const unsigned tb = __ballot_sync(FULL, act && ekey == M);
                const int cnt = __popc(tb);
                int src = __ffs(tb) - 1;
                if (cnt > 1) {
                  if (nbulk) {
                    cursor += nbulk - bulk_distinct(sc, nbulk, lane);
                    nbulk = 0;
                  }
                  const double u = draw_at(mkdr(), cursor++);
                  const long long pk = (long long)__dmul_rn(u, (double)cnt);
                  src = nth_set_bit32(tb, (int)(pk >= cnt ? cnt - 1 : pk));
                  QSB_COUNT(4, 1);
                }
                if (lane == src) sc.sperm[ec] = (uint8_t)er;
                const int si = __shfl_sync(FULL, ei, src), sj = __shfl_sync(FULL, ej, src);
                act = act && ei != si && ej != sj;
              }
              __syncwarp();
              break;
            }
          }
          bool need[CPL];
#pragma unroll
          for (int k = 0; k < CPL; ++k) need[k] = false;
          bool bulk = false;

          // ---- bulk step (unrestricted rounds, G == 1): every free z cell
          // whose m = 1 + v exceeds the largest free non-z cell is selected
          // before any non-z cell, in an order that does not change the
          // result; a group of g equal keys costs g - 1 tie draws (counted
          // lazily, only if a later round needs a draw).
          if constexpr (G == 1 && CPL <= 2) {
            if constexpr (!CHAIN) {
            if (!restricted) {
              uint64_t ml = 0;
#pragma unroll
              for (int k = 0; k < CPL; ++k)
                if (cfree[k] && ncnt[k] && nk64[k] > ml) ml = nk64[k];
              const unsigned mh = __reduce_max_sync(FULL, (unsigned)(ml >> 32));
              const unsigned mlo = __reduce_max_sync(FULL, (unsigned)(ml >> 32) == mh ? (unsigned)ml : 0u);
              const uint64_t M = ((uint64_t)mh << 32) | mlo;
              bool q[CPL];
              unsigned qb[CPL];
              int nq = 0;
#pragma unroll
              for (int k = 0; k < CPL; ++k) {
                q[k] = cfree[k] && zel[k] && zkey[k] > M;
                qb[k] = __ballot_sync(FULL, q[k]);
                nq += __popc(qb[k]);
              }
              if (nq >= 2) {
                const unsigned lt = (1u << lane) - 1u;
                uint64_t rbits = 0;
                int base = nbulk;
#pragma unroll
                for (int k = 0; k < CPL; ++k) {
                  if (q[k]) {
                    sc.sbulk[base + __popc(qb[k] & lt)] = zkey[k];
                    sc.sperm[col[k]] = zr[k];
                    rbits |= 1ULL << zr[k];
                    cfree[k] = false; zel[k] = false; ck[k] = 0; cc[k] = 0;
                  }
                  base += __popc(qb[k]);
                }
                nbulk = base;
                __syncwarp();
                const unsigned rl = __reduce_or_sync(FULL, (unsigned)rbits);
                const unsigned rh = __reduce_or_sync(FULL, (unsigned)(rbits >> 32));
                const uint64_t rmask = ((uint64_t)rh << 32) | rl;
                rf.w[0] &= ~rmask;
                rnd += nq - 1;
                QSB_COUNT(2, 1);
                QSB_COUNT(3, nq);
                // non-z statistics whose maximum row may have left
#pragma unroll
                for (int k = 0; k < CPL; ++k) {
                  if (!cfree[k] || !ncnt[k]) continue;
                  need[k] = (ncnt[k] == 1 && nrow[k] >= 0) ? ((rmask >> nrow[k]) & 1ULL) : true;
                }
                bulk = true;
              }
            }
            } else {
            // CHAIN (late iterations): after a bulk step that leaves more than
            // five free columns, the retired rows leave the remaining columns'
            // non-z maxima stale, but still upper bounds, so z cells above the
            // stale maximum are still selected first; further attempts run
            // until fewer than two qualify or the endgame is next, with no
            // rescans in between
#pragma unroll 1
            for (int att = 0; !restricted; ++att) {
              uint64_t ml = 0;
#pragma unroll
              for (int k = 0; k < CPL; ++k)
                if (cfree[k] && ncnt[k] && nk64[k] > ml) ml = nk64[k];
              const unsigned mh = __reduce_max_sync(FULL, (unsigned)(ml >> 32));
              const unsigned mlo = __reduce_max_sync(FULL, (unsigned)(ml >> 32) == mh ? (unsigned)ml : 0u);
              const uint64_t M = ((uint64_t)mh << 32) | mlo;
              bool q[CPL];
              unsigned qb[CPL];
              int nq = 0;
#pragma unroll
              for (int k = 0; k < CPL; ++k) {
                q[k] = cfree[k] && zel[k] && zkey[k] > M;
                qb[k] = __ballot_sync(FULL, q[k]);
                nq += __popc(qb[k]);
              }
              if (nq < 2) break;
              {
                const unsigned lt = (1u << lane) - 1u;
                uint64_t rbits = 0;
                int base = nbulk;
#pragma unroll
                for (int k = 0; k < CPL; ++k) {
                  if (q[k]) {
                    sc.sbulk[base + __popc(qb[k] & lt)] = zkey[k];
                    sc.sperm[col[k]] = zr[k];
                    rbits |= 1ULL << zr[k];
                    cfree[k] = false; zel[k] = false; ck[k] = 0; cc[k] = 0;
                    need[k] = false;     // (an earlier chained attempt may have set it)
                  }
                  base += __popc(qb[k]);
                }
                nbulk = base;
                __syncwarp();
                const unsigned rl = __reduce_or_sync(FULL, (unsigned)rbits);
                const unsigned rh = __reduce_or_sync(FULL, (unsigned)(rbits >> 32));
                const uint64_t rmask = ((uint64_t)rh << 32) | rl;
                rf.w[0] &= ~rmask;
                rnd += att == 0 ? nq - 1 : nq;
                QSB_COUNT(2, 1);
                QSB_COUNT(3, nq);
                // non-z statistics whose maximum row may have left
#pragma unroll
                for (int k = 0; k < CPL; ++k) {
                  if (!cfree[k] || !ncnt[k]) continue;
                  need[k] = need[k] || ((ncnt[k] == 1 && nrow[k] >= 0) ? ((rmask >> nrow[k]) & 1ULL) : true);
                }
                bulk = true;
              }
              if (n - (rnd + 1) <= 5) break;
            }
            }
          } else {
            // multi-warp groups: the same bulk step with smem reductions; the
            // threshold M is reduced together with the round's best candidate
            // (used as is when no bulk step happens), and the attempt's count
            // and row words alternate between two buffers: two group barriers
            // per round
            if (!restricted) {
              uint64_t ml = 0;
#pragma unroll
              for (int k = 0; k < CPL; ++k)
                if (cfree[k] && ncnt[k] && nk64[k] > ml) ml = nk64[k];
              Best lc;
              lc.key = ck[0]; lc.cnt = cc[0]; lc.col = col[0]; lc.row = cr[0];
#pragma unroll
              for (int k = 1; k < CPL; ++k) {
                if (ck[k] > lc.key) { lc.key = ck[k]; lc.cnt = cc[k]; lc.col = col[k]; lc.row = cr[k]; }
                else if (ck[k] == lc.key) lc.cnt += cc[k];
              }
              if (lc.cnt == 0) { lc.key = 0; lc.col = INT_MAX; }
              // (this buffer's last reads, two attempts ago, are behind the
              // previous attempt's barriers; the reduction's barrier orders the
              // reset before this attempt's atomics)
              int* bcnt = &sc.mw.bcnt[bpar];
              unsigned long long* rw = sc.mw.rmw2[bpar];
              bpar ^= 1;
              if (tid == 0) *bcnt = 0;
              if (tid < NW) rw[tid] = 0ULL;
              uint64_t M;
              pre = group_best_max<G>(lc, ml, sc, par, lane, tid, M);
              have_pre = true;
              bool q[CPL];
#pragma unroll
              for (int k = 0; k < CPL; ++k) q[k] = cfree[k] && zel[k] && zkey[k] > M;
              // warp-aggregated: one position atomic and one OR per row word
              // per warp (the order of the bulk keys does not matter)
#pragma unroll
              for (int k = 0; k < CPL; ++k) {
                const unsigned qb = __ballot_sync(FULL, q[k]);
                if (!qb) continue;
                int base = 0;
                if (lane == 0) base = atomicAdd(bcnt, __popc(qb));
                base = __shfl_sync(FULL, base, 0);
                if (q[k]) sc.sbulk[nbulk + base + __popc(qb & ((1u << lane) - 1u))] = zkey[k];
#pragma unroll
                for (int w = 0; w < NW; ++w) {
                  const uint64_t bit = (q[k] && (zr[k] >> 6) == w) ? 1ULL << (zr[k] & 63) : 0ULL;
                  const unsigned lo = __reduce_or_sync(FULL, (unsigned)bit);
                  const unsigned hi = __reduce_or_sync(FULL, (unsigned)(bit >> 32));
                  if (lane == 0 && (lo | hi)) atomicOr(&rw[w], ((unsigned long long)hi << 32) | lo);
                }
              }
              __syncthreads();
              const int nq = *bcnt;
              if (nq >= 2) {
                uint64_t rm[NW];
#pragma unroll
                for (int w = 0; w < NW; ++w) { rm[w] = rw[w]; rf.w[w] &= ~rm[w]; }
#pragma unroll
                for (int k = 0; k < CPL; ++k) {
                  if (q[k]) {
                    sc.sperm[col[k]] = zr[k];
                    cfree[k] = false; zel[k] = false; ck[k] = 0; cc[k] = 0;
                  } else if (cfree[k] && ncnt[k]) {
                    need[k] = (ncnt[k] == 1 && nrow[k] >= 0) ? ((rm[nrow[k] >> 6] >> (nrow[k] & 63)) & 1ULL)
                                                             : true;
                  }
                }
                nbulk += nq;
                rnd += nq - 1;
                QSB_COUNT(2, 1);
                QSB_COUNT(3, nq);
                bulk = true;
                have_pre = false;
              }
            }
          }

          if (!bulk) {
            QSB_COUNT(1, 1);
            // ---- one round: lane-local best of the cached candidates, then the group's
            Best loc;
            loc.key = ck[0]; loc.cnt = cc[0]; loc.col = col[0]; loc.row = cr[0];
#pragma unroll
            for (int k = 1; k < CPL; ++k) {
              if (ck[k] > loc.key) { loc.key = ck[k]; loc.cnt = cc[k]; loc.col = col[k]; loc.row = cr[k]; }
              else if (ck[k] == loc.key) loc.cnt += cc[k];
            }
            if (loc.cnt == 0) { loc.key = 0; loc.col = INT_MAX; }
            Best b;
            if constexpr (G > 1) {
              b = have_pre ? pre : group_best<G>(loc, sc, par, lane, tid);
              have_pre = false;
            } else {
              b = group_best<G>(loc, sc, par, lane, tid);
            }

            int sel_r, sel_c;
            if (b.cnt == 1 && b.row >= 0) {
              sel_r = b.row; sel_c = b.col;
            } else if (b.cnt == 0) {
              // every remaining cell is excluded (a 1x1 remainder): the
              // reference falls back to the unrestricted set (_batch.py:118-132)
              sel_r = rf.first();
              int mc = INT_MAX;
#pragma unroll
              for (int k = 0; k < CPL; ++k) if (cfree[k]) mc = min(mc, col[k]);
              sel_c = group_min_sync<G>(mc, sc, lane, tid);
            } else if (b.cnt == 1) {
              // unique maximum in column b.col whose first row is not tracked
              sel_c = b.col;
              GroupSync<G>::sync();
#pragma unroll
              for (int k = 0; k < CPL; ++k) if (col[k] == sel_c) sc.ssel[3] = zel[k];
              GroupSync<G>::sync();
              sel_r = first_row_scan<VT, G, CPL, NW>(tile, n, sc, rf, b.key, sel_c, sc.ssel[3] != 0,
                                                     tid, lane);
            } else {
              // ---- ties: one draw, the pick-th tied cell in row-major order
              if (nbulk) {
                if constexpr (G == 1) cursor += nbulk - bulk_distinct(sc, nbulk, lane);
                else cursor += nbulk - bulk_distinct_group<G>(sc, nbulk, tid, lane);
                nbulk = 0;
              }
              double u;
              if constexpr (G > 1) {
                const int k = cursor++;
                const DrawKey dr = mkdr();
                if (dr.inj) {
                  u = dr.inj[k];
                } else {
                  const uint64_t idx = dr.base + (uint64_t)k;
                  if ((idx >> 2) != dcb) { dblk = philox_block_call((idx >> 2) + 1, dr.seed, dr.word1); dcb = idx >> 2; }
                  u = word_unit(dblk, (unsigned)(idx & 3));
                }
              } else {
                u = draw_at(mkdr(), cursor++);
              }
              const long long pk = (long long)__dmul_rn(u, (double)b.cnt);
              const int pick = (int)(pk >= b.cnt ? b.cnt - 1 : pk);
              QSB_COUNT(4, 1);
              bool fast = false;
              sel_r = sel_c = -1;
              if constexpr (G == 1 && CPL <= 2) {
                // common case: each tied column holds one tied cell with a
                // known row -> the row set is a 64-bit mask and the pick-th
                // set bit is the answer (e.g. x cells tied at 1 + 0)
                bool slow = false;
                uint64_t rm = 0;
#pragma unroll
                for (int k = 0; k < CPL; ++k) {
                  if (cc[k] && ck[k] == b.key) {
                    if (cc[k] == 1 && cr[k] >= 0) rm |= 1ULL << cr[k];
                    else slow = true;
                  }
                }
                const unsigned rl = __reduce_or_sync(FULL, (unsigned)rm);
                const unsigned rh = __reduce_or_sync(FULL, (unsigned)(rm >> 32));
                if (!__any_sync(FULL, slow) && __popc(rl) + __popc(rh) == b.cnt) {
                  const int nl = __popc(rl);
                  sel_r = pick < nl ? nth_set_bit32(rl, pick) : 32 + nth_set_bit32(rh, pick - nl);
                  unsigned owner[CPL];
#pragma unroll
                  for (int k = 0; k < CPL; ++k)
                    owner[k] = __ballot_sync(FULL, cc[k] && ck[k] == b.key && cr[k] == sel_r);
                  sel_c = owner[0] ? __ffs(owner[0]) - 1 : 32 + __ffs(owner[CPL - 1]) - 1;
                } else {
                  // general ties: per-column row masks + warp prefix over rows
#pragma unroll
                  for (int k = 0; k < CPL; ++k)
                    if (cc[k] && ck[k] == b.key) sc.stie[col[k]] = zel[k] ? 2 : 1;
                  QSB_COUNT(5, 1);
                  const int rc = tie_select_warp<VT>(tile, n, sc, rf.w[0], b.key, pick, lane);
                  sel_r = rc >> 8;
                  sel_c = rc & 0xff;
                }
                fast = true;
              }
              if (!fast) {
                GroupSync<G>::sync();
#pragma unroll
                for (int k = 0; k < CPL; ++k)
                  if (cc[k] && ck[k] == b.key) sc.stie[col[k]] = zel[k] ? 2 : 1;
                QSB_COUNT(6, 1);
                tie_select_slow<VT, G, NW>(tile, n, sc, rf, b.key, pick, tid);
                sel_r = sc.ssel[0]; sel_c = sc.ssel[1];
                GroupSync<G>::sync();
              }
            }

            // ---- retire row sel_r and column sel_c; update the statistics
            rf.clear(sel_r);
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
              if (!cfree[k]) continue;
              if (col[k] == sel_c) {
                cfree[k] = false; zel[k] = false; ck[k] = 0; cc[k] = 0;
                sc.sperm[sel_c] = sel_r;
                continue;
              }
              bool chg = false;
              if (zr[k] == sel_r) {                     // this column's z cell left
                chg = zel[k];
                zel[k] = false;
              } else if (ncnt[k] && ((GT && ncnt[k] == 1 && nrow[k] >= 0)
                                         // global tile: a unique maximum with a known
                                         // row needs no L2 read (the shared-memory
                                         // tile's read is cheaper than the test)
                                         ? nrow[k] == sel_r
                                         : tile[sel_r * n + col[k]] == nmax[k])) {
                if (nrow[k] == sel_r) nrow[k] = -1;
                need[k] = --ncnt[k] == 0;
                chg = true;
              }
              if (chg) recompute(k);
            }
          }
          if (rnd >= n - 1) break;
          if constexpr (G == 1 && CPL <= 2) {
            // the next round is the endgame, which needs no column statistics
            if (n - (rnd + 1) <= 5 && !(restricted && rnd + 1 < a.depth)) continue;
          }

          // ---- cooperative rescans of columns whose non-z maximum was retired
          if constexpr (G == 1) {
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
              unsigned mask = __ballot_sync(FULL, need[k]);
              while (mask) {
                const int src = __ffs(mask) - 1;
                mask &= mask - 1;
                QSB_COUNT(7, 1);
                const int c = src + k * 32;
                const int zc = __shfl_sync(FULL, zr[k], src);
                if constexpr (sizeof(VT) == 4) {
                  // fp32: one 32-bit key per cell, three warp reductions
                  // one key per cell (lane = row, + 32 j), the maximum by one
                  // reduction, its rows by ballots: count = popc, first row
                  // = lowest set bit in row order
                  unsigned kj[CPL];
                  unsigned km = 0;
#pragma unroll
                  for (int j = 0; j < CPL; ++j) {
                    const int r = lane + j * 32;
                    kj[j] = (r >= n || r == zc || !rf.has(r)) ? 0u
                            : okey32(__fadd_rn((float)tile[r * n + c], 0.0f));
                    km = max(km, kj[j]);
                  }
                  const unsigned M = __reduce_max_sync(FULL, km);
                  unsigned tot = 0, rr = INT_MAX;
#pragma unroll
                  for (int j = CPL - 1; j >= 0; --j) {
                    const unsigned b = __ballot_sync(FULL, M != 0u && kj[j] == M);
                    tot += __popc(b);
                    if (b) rr = j * 32 + __ffs(b) - 1;
                  }
                  if (lane == src) {
                    ncnt[k] = (int)tot;
                    nrow[k] = tot ? (int)rr : -1;
                    nmax[k] = tot ? (VT)from_okey32(M) : (VT)0;
                    nk64[k] = tot ? nonz_key(nmax[k], sK[k], wide) : 0;
                    recompute(k);
                  }
                } else {
                  Best rb = best_none();
#pragma unroll
                  for (int j = 0; j < CPL; ++j) {
                    const int r = lane + j * 32;
                    if (r >= n || r == zc || !rf.has(r)) continue;
                    const uint64_t key = nonz_key(tile[r * n + c], 1.0f, false);
                    if (key > rb.key) { rb.key = key; rb.cnt = 1; rb.col = r; }
                    else if (key == rb.key) ++rb.cnt;
                  }
                  const Best rr = warp_best(rb);
                  if (lane == src) {
                    ncnt[k] = rr.cnt;
                    nrow[k] = rr.cnt ? rr.col : -1;
                    nk64[k] = rr.cnt ? rr.key : 0;
                    nmax[k] = rr.cnt ? (VT)from_okey(rr.key) : (VT)0;
                    recompute(k);
                  }
                }
              }
            }
          } else {
            // multi-warp groups: each warp rescans the columns it owns,
            // lanes over rows, warp reductions only (no group barrier; the
            // columns of a group are independent)
            constexpr int RPL = (K::NMAX + 31) / 32;
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
              unsigned mask = __ballot_sync(FULL, need[k]);
              while (mask) {
                const int src = __ffs(mask) - 1;
                mask &= mask - 1;
                QSB_COUNT(7, 1);
                const int c = __shfl_sync(FULL, col[k], src);
                const int zc = __shfl_sync(FULL, zr[k], src);
                Best rb = best_none();
#pragma unroll
                for (int j = 0; j < RPL; ++j) {
                  const int r = lane + 32 * j;
                  if (r >= n || r == zc || !rf.has(r)) continue;
                  // ordered by the stored value (the column scale is positive
                  // and u * s is exact in double, so the order and the ties
                  // are those of v); nmax keeps the stored value
                  const uint64_t key = nonz_key(tile[r * n + c], 1.0f, false);
                  if (key > rb.key) { rb.key = key; rb.cnt = 1; rb.col = r; }
                  else if (key == rb.key) ++rb.cnt;
                }
                const Best rr = warp_best(rb);
                if (lane == src) {
                  ncnt[k] = rr.cnt;
                  nrow[k] = rr.cnt ? rr.col : -1;
                  nmax[k] = rr.cnt ? (VT)from_okey(rr.key) : (VT)0;
                  nk64[k] = rr.cnt ? nonz_key(nmax[k], sc.sS[c], sc.wide) : 0;
                  recompute(k);
                }
              }
            }
          }
        }
      }
      Sync::sync();
      if constexpr (!GT) {
        // the tile is no longer read for this particle: prefetch the next one
        p_next = a.work ? bcast(q_next) + ngroups : p + ngroups;
        if (p_next < a.P) { issue_load(p_next, cbuf ^ 1); loaded = true; }
      }
      int16_t* gnew = a.perm_new + p * n;
      #pragma unroll 1
      for (int c = tid; c < n; c += NT) gnew[c] = (int16_t)sc.sperm[c];
    }

    // ================= phase 3: goal  sum_ij F[i,j] * D[perm_i, perm_j]
    bool cost_done = false;
    int64_t ncost = 0;   // the new goal (raw bits for doubles), valid on tid 0 when cost_done
    if constexpr (G == 1 && !kFloatMat) {
      // Incremental goal (integral instances, one-warp groups): most columns
      // keep their row (the bulk step re-selects the z cells), so with C the
      // set of facilities that moved,
      //   cost' - cost = sum_{i in C, all j} F[i][j] (D'[i][j] - D[i][j])
      //                + sum_{i not in C, j in C} F[i][j] (D'[i][j] - D[i][j])
      // with D[i][j] = D[p_i][p_j].  Exact in int64 (mod 2^64, as the full
      // sum).  Needs cost[p] == goal(perm[p]) on entry (host guarantee).
      if (do_cost && cost_incr && sizeof(MT) <= 2 && acc32 && n >= 8) {
        Sync::sync();
        const int c0 = lane, c1 = lane + 32;
        const bool m0 = c0 < n && sc.sperm[c0] != sc.szr[c0];
        const bool m1 = c1 < n && sc.sperm[c1] != sc.szr[c1];
        const unsigned ch[2] = {__ballot_sync(FULL, m0), __ballot_sync(FULL, m1)};
        const int k = __popc(ch[0]) + __popc(ch[1]);
        if (3 * k <= n) {
          uint64_t acc = 0;
          int pjn[CPL], pjo[CPL];
#pragma unroll
          for (int kk = 0; kk < CPL; ++kk) {
            pjn[kk] = col[kk] < n ? sc.sperm[col[kk]] : 0;
            pjo[kk] = col[kk] < n ? sc.szr[col[kk]] : 0;
          }
          const int ro0 = c0 < n ? sc.szr[c0] : 0, ro1 = c1 < n ? sc.szr[c1] : 0;
          int wsym[CPL];
#pragma unroll
          for (int kk = 0; kk < CPL; ++kk) wsym[kk] = (symmetric && !(kk == 0 ? m0 : m1)) ? 2 : 1;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            unsigned b = ch[h];
            while (b) {
              const int i = h * 32 + __ffs(b) - 1;
              b &= b - 1;
              const int pin = sc.sperm[i], pio = sc.szr[i];
              // n max(F) max(D) < 2^32, n >= 8 (host / launch checked): every
              // term F (D' - D) and this facility's <= 2 * CPL terms per lane
              // fit int32
              // (F, D symmetric: an unmoved row's column-i term equals its
              // row-i term, which then counts twice)
              int part = 0;
#pragma unroll
              for (int kk = 0; kk < CPL; ++kk)
                if (col[kk] < n)
                  part += wsym[kk] * (int)cF[i * n + col[kk]] *
                          ((int)cD[pin * n + pjn[kk]] - (int)cD[pio * n + pjo[kk]]);
              if (!symmetric) {
                if (c0 < n && !m0) part += (int)cF[c0 * n + i] * ((int)cD[ro0 * n + pin] - (int)cD[ro0 * n + pio]);
                if (c1 < n && !m1) part += (int)cF[c1 * n + i] * ((int)cD[ro1 * n + pin] - (int)cD[ro1 * n + pio]);
              }
              acc += (uint64_t)(int64_t)part;
            }
          }
          const int64_t delta = warp_sum_i64((int64_t)acc);
          if (tid == 0) {
            int64_t* cp = reinterpret_cast<int64_t*>(a.cost);
            const int64_t old = stage_cost ? s_cost[2 * cbuf] : cp[p];
            ncost = (int64_t)((uint64_t)old + (uint64_t)delta);
            cp[p] = ncost;
          }
          cost_done = true;
        }
      }
    }
    if constexpr (G > 1 && !kFloatMat) {
      // The same incremental goal for multi-warp groups (n > 64): the moved
      // facilities C are listed in shared memory, and every thread adds the
      // terms of its own columns j over i in C (integer sums: the list order
      // does not matter).  At n = 256 |C| is a few, against the n^2 terms of
      // the full goal.
      if (do_cost && cost_incr && sizeof(MT) <= 2 && acc32 && n >= 8) {
        bool mv[CPL];
        if (tid == 0) sc.ssel[2] = 0;
        Sync::sync();
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
          mv[k] = col[k] < n && sc.sperm[col[k]] != sc.szr[col[k]];
          if (mv[k]) sc.srow[atomicAdd(&sc.ssel[2], 1)] = (uint16_t)col[k];
        }
        Sync::sync();
        const int kc = sc.ssel[2];
        if (3 * kc <= n) {
          int64_t acc = 0;
#pragma unroll
          for (int k = 0; k < CPL; ++k) {
            const int j = col[k];
            if (j >= n) continue;
            const int pjn = sc.sperm[j], pjo = sc.szr[j];
            // symmetric F, D: an unmoved column's term for row i in C equals
            // its row's term for column i, which then counts twice
            const int w = (symmetric && !mv[k]) ? 2 : 1;
#pragma unroll 4
            for (int c = 0; c < kc; ++c) {
              const int i = sc.srow[c];
              const int pin = sc.sperm[i], pio = sc.szr[i];
              // n max(F) max(D) < 2^32 and n >= 8: each term fits int32
              acc += (int64_t)(w * (int)cF[i * n + j] * ((int)cD[pin * n + pjn] - (int)cD[pio * n + pjo]));
              if (!symmetric && !mv[k])
                acc += (int64_t)((int)cF[j * n + i] * ((int)cD[pjo * n + pin] - (int)cD[pjo * n + pio]));
            }
          }
          int64_t delta = warp_sum_i64(acc);
          if (lane == 0) sc.lslots[tid >> 5] = delta;
          Sync::sync();
          if (tid == 0) {
            for (int w = 1; w < G; ++w) delta += sc.lslots[w];
            int64_t* cp = reinterpret_cast<int64_t*>(a.cost);
            ncost = (int64_t)((uint64_t)cp[p] + (uint64_t)delta);
            cp[p] = ncost;
          }
          cost_done = true;
        }
      }
    }
    if (do_cost && !cost_done) {
      const int64_t tot = cost_general<MT, G, CPL>(cF, cD, n, sc, tid, lane, acc32);
      if (tid == 0) reinterpret_cast<int64_t*>(a.cost)[p] = tot;   // raw bits for doubles
      ncost = tot;
      cost_done = true;
    }

    // ================= phase 4a: personal best (engine.py:211-215)
    if (do_pbest) {
      Sync::sync();
      if (tid == 0) {
        bool imp;
        // the new goal from this step (register) and the staged pl_cost
        const int64_t cvb = cost_done ? ncost : reinterpret_cast<int64_t*>(a.cost)[p];
        const int64_t plb = stage_pl ? s_cost[2 * cbuf + 1] : reinterpret_cast<int64_t*>(a.pl_cost)[p];
        if constexpr (kFloatMat) {
          const double cv = __longlong_as_double(cvb);
          imp = cv < __longlong_as_double(plb);
          if (imp) reinterpret_cast<double*>(a.pl_cost)[p] = cv;
        } else {
          imp = cvb < plb;
          if (imp) reinterpret_cast<int64_t*>(a.pl_cost)[p] = cvb;
        }
        a.improved[p] = imp ? 1 : 0;
        sc.ssel[2] = imp;
      }
      Sync::sync();
      if (sc.ssel[2]) {
        int16_t* gpl = a.pl_perm + p * n;
        #pragma unroll 1
        for (int c = tid; c < n; c += NT) gpl[c] = (int16_t)sc.sperm[c];
      }
    }
    Sync::sync();
    if (p_next < 0) p_next = a.work ? bcast(q_next) + ngroups : p + ngroups;
    p = p_next;
    cbuf ^= 1;
  }
  if (!GT && tid == 0) bulk_wait_all();
}

}  // namespace qsb
