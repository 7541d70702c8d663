// step_kernel.cuh -- the fused PSO step for one particle per thread group.
//
// One group of G warps owns one particle at a time (persistent loop over the
// particles of this device).  Thread t of the group owns columns
// c = t + k*32G (k < CPL) of the particle's n x n velocity tile, so:
//
//   * the velocity update and the column normalisation are column-local and
//     run in the reference's exact order (_batch.py:39-58);
//   * the aggregation keeps incremental per-column (max, count, first row)
//     statistics over the free rows instead of the reference's O(n^3) rescan
//     (_batch.py:89-175), reproducing its (max, tie-count) per round, its
//     row-major k-th-tie selection and its draw consumption exactly;
//   * the QAP goal is a per-column partial sum over the smem-resident F, D
//     (_batch.py:186-197), reduced in integer arithmetic.
//
// The tile is staged global -> smem with one cp.async.bulk (1-D TMA) and the
// updated velocity is written back with one bulk store, so the velocity
// phase touches HBM exactly once in each direction.
#pragma once
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
};

struct Best {
  uint64_t key;
  int cnt;
  int col;
  int row;
};

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

__device__ __forceinline__ int64_t warp_sum_i64(int64_t x) {
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
  return x;
}

// Per-group shared scratch (one per particle group in the CTA).
template <int NMAX, int G>
struct GroupScratch {
  int sperm[NMAX];     // perm_new under construction (aggregation output)
  int szr[NMAX];       // perm of the current position X (zero row per column)
  int srow[NMAX];      // per-row tie counts / pick-column match flags
  int sorder[NMAX];    // pick-column visiting order
  unsigned char stie[NMAX];  // tied-column flags
  Best slots[2][G];
  int64_t lslots[2][G];
  int ssel[4];
  uint64_t bar;
};

template <int G>
struct GroupSync {
  __device__ __forceinline__ static void sync() {
    if constexpr (G == 1) __syncwarp(); else __syncthreads();
  }
};

template <typename VT, typename MT, int G, int CPL, int W>
struct StepKernel {
  static constexpr int NT = 32 * G;          // threads per group
  static constexpr int NMAX = NT * CPL;      // largest n handled
  static constexpr int NW = (NMAX + 63) / 64;
  using Scratch = GroupScratch<NMAX, G>;

  static __host__ __device__ size_t fd_bytes(int n) {
    return align_up(2 * (size_t)n * n * sizeof(MT), 128);
  }
  static __host__ __device__ size_t tile_bytes(int vstride) {
    return align_up((size_t)vstride * sizeof(VT), 128);
  }
  static __host__ __device__ size_t group_bytes(int vstride) {
    return tile_bytes(vstride) + align_up(sizeof(Scratch), 128);
  }
  static __host__ __device__ size_t smem_bytes(int n, int vstride, bool fd) {
    return (fd ? fd_bytes(n) : 0) + W * group_bytes(vstride);
  }
};

// ------------------------------------------------------------------------
template <typename VT, typename MT, int G, int CPL, int W>
__global__ void __launch_bounds__(32 * G * W)
step_kernel(const StepArgs a) {
  using K = StepKernel<VT, MT, G, CPL, W>;
  constexpr int NT = K::NT;
  constexpr int NW = K::NW;
  using Scratch = typename K::Scratch;
  using Sync = GroupSync<G>;

  extern __shared__ __align__(128) unsigned char smem[];
  const int n = a.n;
  const int nn = n * n;
  const bool fds = a.fd_smem;
  MT* sF = reinterpret_cast<MT*>(smem);
  MT* sD = sF + nn;
  const int gidx = threadIdx.x / NT;
  const int tid = threadIdx.x % NT;
  const int lane = threadIdx.x & 31;
  unsigned char* gb = smem + (fds ? K::fd_bytes(n) : 0) + (size_t)gidx * K::group_bytes(a.vstride);
  VT* tile = reinterpret_cast<VT*>(gb);
  Scratch& sc = *reinterpret_cast<Scratch*>(gb + K::tile_bytes(a.vstride));

  const bool do_vel = a.flags & F_VELOCITY;
  const bool do_agg = a.flags & F_AGGREGATE;
  const bool do_cost = a.flags & F_COST;
  const bool do_pbest = a.flags & F_PBEST;
  const bool store_v = a.flags & F_STORE_V;

  const MT* cF = sF;
  const MT* cD = sD;
  if (do_cost) {
    const MT* gF = reinterpret_cast<const MT*>(a.F);
    const MT* gD = reinterpret_cast<const MT*>(a.D);
    if constexpr (G == 1) {
      for (int i = threadIdx.x; i < nn; i += blockDim.x) { sF[i] = gF[i]; sD[i] = gD[i]; }
    } else {
      if (fds) for (int i = threadIdx.x; i < nn; i += blockDim.x) { sF[i] = gF[i]; sD[i] = gD[i]; }
      else { cF = gF; cD = gD; }
    }
  }
  if (tid == 0) { mbar_init(&sc.bar, 1); mbar_fence_init(); }
  for (int c = tid; c < K::NMAX; c += NT) sc.stie[c] = 0;
  __syncthreads();

  const uint64_t t = a.t_dev ? (uint64_t)(*a.t_dev) + 1 : a.t_host;
  const uint64_t word1 = stream_word(2, t);
  const uint32_t tile_bytes = (uint32_t)(a.vstride * sizeof(VT));
  const int64_t ngroups = (int64_t)gridDim.x * W;
  const int row_w = 2 + 2 * n;
  uint32_t phase = 0;

  for (int64_t p = (int64_t)blockIdx.x * W + gidx; p < a.P; p += ngroups) {
    VT* gV = reinterpret_cast<VT*>(a.V) + p * a.vstride;
    if (tid == 0) {
      bulk_wait_read();                 // previous particle's store has left the tile
      mbar_arrive_expect_tx(&sc.bar, tile_bytes);
      bulk_load(tile, gV, tile_bytes, &sc.bar);
    }

    DrawRow dr;
    dr.inj = a.inj_draws ? a.inj_draws + p * a.inj_stride : nullptr;
    dr.seed = a.seed;
    dr.word1 = word1;
    dr.base = (uint64_t)(a.p0 + p) * (uint64_t)row_w;
    dr.cached = ~0ULL;

    // ---- per-column registers
    int zr[CPL], col[CPL];
    bool cfree[CPL];
    uint64_t ckey[CPL];
    int ccnt[CPL], crow[CPL];
    const int16_t* gperm = a.perm + p * n;
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      col[k] = tid + k * NT;
      cfree[k] = col[k] < n;
      zr[k] = cfree[k] ? (int)gperm[col[k]] : -1;
      if (cfree[k]) sc.szr[col[k]] = zr[k];
      ckey[k] = 0; ccnt[k] = 0; crow[k] = -1;
    }
    const bool restricted0 = (a.mode == MODE_SECOND_TARGET) && a.depth > 0;

    mbar_wait(&sc.bar, phase);
    phase ^= 1u;

    // ================= phase 1: velocity (+ initial column statistics)
    if (do_vel) {
      double c2r2, c3r3;
      if (a.coef) { c2r2 = a.coef[2 * p]; c3r3 = a.coef[2 * p + 1]; }
      else {
        c2r2 = __dmul_rn(a.c2, dr.at(0));   // engine.py:198-199: c2 * r2, c3 * r3
        c3r3 = __dmul_rn(a.c3, dr.at(1));
      }
      const int64_t s = p / a.S;
#pragma unroll
      for (int k = 0; k < CPL; ++k) {
        if (!cfree[k]) continue;
        const int c = col[k];
        const int xr = zr[k];
        const int plr = a.pl_perm[p * n + c];
        const int pgr = a.pg_perm[s * n + c];
        if constexpr (sizeof(VT) == 8) {
          // Reference order, no contraction: (c1*v + c2r2*(pl-x)) + c3r3*(pg-x)
          double total = 0.0;
          for (int r = 0; r < n; ++r) {
            const double v = (double)tile[r * n + c];
            const double d2 = (r == plr) ? ((r == xr) ? 0.0 : 1.0) : ((r == xr) ? -1.0 : 0.0);
            const double d3 = (r == pgr) ? ((r == xr) ? 0.0 : 1.0) : ((r == xr) ? -1.0 : 0.0);
            double lin = __dadd_rn(__dadd_rn(__dmul_rn(a.c1, v), __dmul_rn(c2r2, d2)),
                                   __dmul_rn(c3r3, d3));
            if (lin > a.vmax) lin = a.vmax;
            else if (lin < -a.vmax) lin = -a.vmax;
            tile[r * n + c] = (VT)lin;
            total = __dadd_rn(total, fabs(lin));
          }
          if (a.normalize && total > 0.0)
            for (int r = 0; r < n; ++r) tile[r * n + c] = (VT)__ddiv_rn((double)tile[r * n + c], total);
        } else {
          const float c1f = (float)a.c1, c2f = (float)c2r2, c3f = (float)c3r3;
          const float vm = (float)a.vmax;
          float total = 0.f;
          for (int r = 0; r < n; ++r) {
            const float v = (float)tile[r * n + c];
            const float d2 = (float)((r == plr) - (r == xr));
            const float d3 = (float)((r == pgr) - (r == xr));
            float lin = fmaf(c3f, d3, fmaf(c2f, d2, c1f * v));
            lin = fminf(fmaxf(lin, -vm), vm);
            tile[r * n + c] = (VT)lin;
            total += fabsf(lin);
          }
          if (a.normalize && total > 0.f) {
            const float inv = 1.0f / total;
            for (int r = 0; r < n; ++r) tile[r * n + c] = (VT)((float)tile[r * n + c] * inv);
          }
        }
      }
      if (store_v) {
        fence_proxy_async_smem();
        Sync::sync();
        if (tid == 0) bulk_store(gV, tile, tile_bytes);
      } else {
        Sync::sync();
      }
    }

    // ================= phase 2: aggregation S_x(X + V)
    if (do_agg) {
      uint64_t rfree[NW];
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const int lo = w * 64;
        rfree[w] = (n - lo >= 64) ? ~0ULL : (n > lo ? ((1ULL << (n - lo)) - 1) : 0ULL);
      }
      auto row_is_free = [&](int r) -> bool { return (rfree[r >> 6] >> (r & 63)) & 1ULL; };
      auto mval = [&](int r, int c, int zrc) -> uint64_t {
        return okey(cell_m(tile[r * n + c], r == zrc));
      };
      int cursor = a.agg_base;     // next aggregation draw (column in the draw row)

      if (a.mode != MODE_PICK_COLUMN) {
        bool restricted = restricted0;
        // initial per-column statistics over all rows (skip z cells if restricted)
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
          if (!cfree[k]) continue;
          const int c = col[k];
          uint64_t kk = 0; int cn = 0, cr = -1;
          for (int r = 0; r < n; ++r) {
            if (restricted && r == zr[k]) continue;
            const uint64_t key = mval(r, c, zr[k]);
            if (key > kk) { kk = key; cn = 1; cr = r; }
            else if (key == kk) ++cn;
          }
          ckey[k] = kk; ccnt[k] = cn; crow[k] = cr;
        }

        for (int rnd = 0; rnd < n; ++rnd) {
          if (restricted && rnd == a.depth) {
            // leaving the restricted phase: the z cells become candidates
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
              if (!cfree[k] || !row_is_free(zr[k])) continue;
              const uint64_t key = mval(zr[k], col[k], zr[k]);
              if (key > ckey[k]) { ckey[k] = key; ccnt[k] = 1; crow[k] = zr[k]; }
              else if (key == ckey[k]) { ++ccnt[k]; if (crow[k] >= 0 && zr[k] < crow[k]) crow[k] = zr[k]; }
            }
            restricted = false;
          }
          // ---- (max, count) over the eligible free cells
          Best loc; loc.key = 0; loc.cnt = 0; loc.col = INT_MAX; loc.row = -1;
#pragma unroll
          for (int k = 0; k < CPL; ++k) {
            if (!cfree[k] || ccnt[k] == 0) continue;
            Best b; b.key = ckey[k]; b.cnt = ccnt[k]; b.col = col[k]; b.row = crow[k];
            loc = best_merge(loc, b);
          }
          Best b = warp_best(loc);
          if constexpr (G > 1) {
            const int par = rnd & 1;
            if (lane == 0) sc.slots[par][tid >> 5] = b;
            __syncthreads();
            b = sc.slots[par][0];
#pragma unroll
            for (int w = 1; w < G; ++w) b = best_merge(b, sc.slots[par][w]);
          }

          int sel_r, sel_c;
          if (b.cnt == 0) {
            // every remaining cell is excluded (only a 1x1 remainder): the
            // reference falls back to the unrestricted set (_batch.py:118-132)
            sel_r = -1;
#pragma unroll
            for (int w = 0; w < NW; ++w)
              if (sel_r < 0 && rfree[w]) sel_r = w * 64 + __ffsll((long long)rfree[w]) - 1;
            int mc = INT_MAX;
#pragma unroll
            for (int k = 0; k < CPL; ++k) if (cfree[k]) mc = min(mc, col[k]);
            mc = __reduce_min_sync(FULL, mc);
            if constexpr (G > 1) {
              if (lane == 0) sc.slots[rnd & 1][tid >> 5].col = mc;
              __syncthreads();
              for (int w = 0; w < G; ++w) mc = min(mc, sc.slots[rnd & 1][w].col);
              __syncthreads();
            }
            sel_c = mc;
          } else {
            int pick = 0;
            if (b.cnt > 1) {
              const double u = dr.at(cursor++);
              long long pk = (long long)__dmul_rn(u, (double)b.cnt);
              pick = (int)(pk >= b.cnt ? b.cnt - 1 : pk);
            }
            if (b.cnt == 1 && b.row >= 0) {
              sel_r = b.row; sel_c = b.col;
            } else if (b.cnt == 1) {
              // unique max, but that column's first row is not tracked: scan it
              sel_c = b.col;
              const int zc = sc.szr[sel_c];
              int found = INT_MAX;
#pragma unroll
              for (int j = 0; j < CPL; ++j) {
                const int r = tid + j * NT;
                if (r < n && row_is_free(r) && !(restricted && r == zc) && mval(r, sel_c, zc) == b.key)
                  found = min(found, r);
              }
              found = __reduce_min_sync(FULL, found);
              if constexpr (G > 1) {
                if (lane == 0) sc.slots[rnd & 1][tid >> 5].row = found;
                __syncthreads();
                for (int w = 0; w < G; ++w) found = min(found, sc.slots[rnd & 1][w].row);
                __syncthreads();
              }
              sel_r = found;
            } else {
              // ---- ties: the pick-th tied cell in row-major order
#pragma unroll
              for (int k = 0; k < CPL; ++k)
                if (cfree[k] && ccnt[k] > 0 && ckey[k] == b.key) sc.stie[col[k]] = 1;
              Sync::sync();
#pragma unroll
              for (int j = 0; j < CPL; ++j) {
                const int r = tid + j * NT;
                if (r >= n) continue;
                int cnt = 0;
                if (row_is_free(r)) {
                  for (int c = 0; c < n; ++c) {
                    if (!sc.stie[c]) continue;
                    const int zc = sc.szr[c];
                    if (restricted && r == zc) continue;
                    if (mval(r, c, zc) == b.key) ++cnt;
                  }
                }
                sc.srow[r] = cnt;
              }
              Sync::sync();
              if (tid == 0) {
                int r = 0, acc = 0;
                while (acc + sc.srow[r] <= pick) { acc += sc.srow[r]; ++r; }
                int q = pick - acc, cc = -1;
                for (int c = 0; c < n; ++c) {
                  if (!sc.stie[c]) continue;
                  const int zc = sc.szr[c];
                  if (restricted && r == zc) continue;
                  if (mval(r, c, zc) == b.key) {
                    if (q == 0) { cc = c; break; }
                    --q;
                  }
                }
                sc.ssel[0] = r; sc.ssel[1] = cc;
              }
              Sync::sync();
              sel_r = sc.ssel[0]; sel_c = sc.ssel[1];
#pragma unroll
              for (int k = 0; k < CPL; ++k) if (cfree[k]) sc.stie[col[k]] = 0;
              Sync::sync();
            }
          }

          // ---- retire row sel_r and column sel_c
          rfree[sel_r >> 6] &= ~(1ULL << (sel_r & 63));
          bool need[CPL];
#pragma unroll
          for (int k = 0; k < CPL; ++k) {
            need[k] = false;
            if (!cfree[k]) continue;
            if (col[k] == sel_c) { cfree[k] = false; sc.sperm[sel_c] = sel_r; continue; }
            if (ccnt[k] == 0) continue;
            if (restricted && zr[k] == sel_r) continue;
            if (mval(sel_r, col[k], zr[k]) == ckey[k]) {
              if (crow[k] == sel_r) crow[k] = -1;
              if (--ccnt[k] == 0) need[k] = true;
            }
          }
          if (rnd == n - 1) break;

          // ---- cooperative rescans of columns whose maximum was retired
          if constexpr (G == 1) {
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
              unsigned mask = __ballot_sync(FULL, need[k]);
              while (mask) {
                const int src = __ffs(mask) - 1;
                mask &= mask - 1;
                const int c = src + k * 32;
                const int zc = __shfl_sync(FULL, zr[k], src);
                Best rb; rb.key = 0; rb.cnt = 0; rb.col = INT_MAX; rb.row = -1;
#pragma unroll
                for (int j = 0; j < CPL; ++j) {
                  const int r = lane + j * 32;
                  if (r >= n || !row_is_free(r) || (restricted && r == zc)) continue;
                  const uint64_t key = mval(r, c, zc);
                  if (key > rb.key) { rb.key = key; rb.cnt = 1; rb.col = r; }
                  else if (key == rb.key) ++rb.cnt;
                }
                const Best rr = warp_best(rb);
                if (lane == src) { ckey[k] = rr.key; ccnt[k] = rr.cnt; crow[k] = rr.cnt ? rr.col : -1; }
              }
            }
          } else {
            // generic group: list the columns, then scan each with all threads
            if (tid == 0) sc.ssel[2] = 0;
            __syncthreads();
#pragma unroll
            for (int k = 0; k < CPL; ++k)
              if (need[k]) sc.srow[atomicAdd(&sc.ssel[2], 1)] = k * NT + tid;
            __syncthreads();
            const int cnt = sc.ssel[2];
            for (int i = 0; i < cnt; ++i) {
              const int c = sc.srow[i];
              const int zc = sc.szr[c];
              Best rb; rb.key = 0; rb.cnt = 0; rb.col = INT_MAX; rb.row = -1;
#pragma unroll
              for (int j = 0; j < CPL; ++j) {
                const int r = tid + j * NT;
                if (r >= n || !row_is_free(r) || (restricted && r == zc)) continue;
                const uint64_t key = mval(r, c, zc);
                if (key > rb.key) { rb.key = key; rb.cnt = 1; rb.col = r; }
                else if (key == rb.key) ++rb.cnt;
              }
              Best rr = warp_best(rb);
              const int par = (rnd + i + 1) & 1;
              if (lane == 0) sc.slots[par][tid >> 5] = rr;
              __syncthreads();
              rr = sc.slots[par][0];
              for (int w = 1; w < G; ++w) rr = best_merge(rr, sc.slots[par][w]);
#pragma unroll
              for (int k = 0; k < CPL; ++k)
                if (col[k] == c) { ckey[k] = rr.key; ccnt[k] = rr.cnt; crow[k] = rr.cnt ? rr.col : -1; }
              __syncthreads();
            }
          }
        }
      } else {
        // ---------------- pick-column (_batch.py:78-88, 93-102, 145-153)
        for (int i = tid; i < n; i += NT) sc.sorder[i] = i;
        Sync::sync();
        if (tid == 0) {
          for (int i = n - 1; i > 0; --i) {
            const double u = dr.at(cursor++);
            long long j = (long long)__dmul_rn(u, (double)(i + 1));
            if (j > i) j = i;
            const int tmp = sc.sorder[i]; sc.sorder[i] = sc.sorder[j]; sc.sorder[j] = tmp;
          }
          sc.ssel[3] = cursor;
        }
        Sync::sync();
        cursor = sc.ssel[3];
        for (int rnd = 0; rnd < n; ++rnd) {
          const int c = sc.sorder[rnd];
          const int zc = sc.szr[c];
          Best rb; rb.key = 0; rb.cnt = 0; rb.col = INT_MAX; rb.row = -1;
#pragma unroll
          for (int j = 0; j < CPL; ++j) {
            const int r = tid + j * NT;
            if (r >= n || !row_is_free(r)) continue;
            const uint64_t key = mval(r, c, zc);
            if (key > rb.key) { rb.key = key; rb.cnt = 1; rb.col = r; }
            else if (key == rb.key) ++rb.cnt;
          }
          Best b = warp_best(rb);
          if constexpr (G > 1) {
            const int par = rnd & 1;
            if (lane == 0) sc.slots[par][tid >> 5] = b;
            __syncthreads();
            b = sc.slots[par][0];
            for (int w = 1; w < G; ++w) b = best_merge(b, sc.slots[par][w]);
          }
          int sel_r = b.col;   // first matching row
          if (b.cnt > 1) {
            const double u = dr.at(cursor++);
            long long pk = (long long)__dmul_rn(u, (double)b.cnt);
            const int pick = (int)(pk >= b.cnt ? b.cnt - 1 : pk);
            // pick-th matching free row, ascending
#pragma unroll
            for (int j = 0; j < CPL; ++j) {
              const int r = tid + j * NT;
              if (r < n) sc.srow[r] = (row_is_free(r) && mval(r, c, zc) == b.key) ? 1 : 0;
            }
            Sync::sync();
            if (tid == 0) {
              int q = pick, r = 0;
              for (; r < n; ++r) if (sc.srow[r]) { if (q == 0) break; --q; }
              sc.ssel[0] = r;
            }
            Sync::sync();
            sel_r = sc.ssel[0];
            Sync::sync();
          }
          rfree[sel_r >> 6] &= ~(1ULL << (sel_r & 63));
          if (tid == 0) sc.sperm[c] = sel_r;
        }
      }
      Sync::sync();
      int16_t* gnew = a.perm_new + p * n;
      for (int c = tid; c < n; c += NT) gnew[c] = (int16_t)sc.sperm[c];
    }

    // ================= phase 3: goal  sum_ij F[i,j] * D[perm_i, perm_j]
    if (do_cost) {
      if constexpr (sizeof(MT) == 8 && (MT)0.5 != (MT)0) {
        // non-integral instance: sequential i-major sum, as _batch.py:192-197
        if (tid == 0) {
          double acc = (double)cF[0] * (double)cD[0] * 0.0;
          for (int i = 0; i < n; ++i) {
            const int pi = sc.sperm[i];
            for (int j = 0; j < n; ++j)
              acc = __dadd_rn(acc, __dmul_rn((double)cF[i * n + j], (double)cD[pi * n + sc.sperm[j]]));
          }
          reinterpret_cast<double*>(a.cost)[p] = acc;
        }
      } else {
        uint64_t part = 0;
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
          const int j = col[k];
          if (j >= n) continue;
          const int pj = sc.sperm[j];
          for (int i = 0; i < n; ++i) {
            const int pi = sc.sperm[i];
            if constexpr (sizeof(MT) <= 2)
              part += (uint64_t)((uint32_t)cF[i * n + j] * (uint32_t)cD[pi * n + pj]);
            else
              part += (uint64_t)cF[i * n + j] * (uint64_t)cD[pi * n + pj];
          }
        }
        int64_t tot = warp_sum_i64((int64_t)part);
        if constexpr (G > 1) {
          if (lane == 0) sc.lslots[0][tid >> 5] = tot;
          __syncthreads();
          tot = 0;
          for (int w = 0; w < G; ++w) tot += sc.lslots[0][w];
        }
        if (tid == 0) reinterpret_cast<int64_t*>(a.cost)[p] = tot;
      }
    }

    // ================= phase 4a: personal best (engine.py:211-215)
    if (do_pbest) {
      Sync::sync();
      if (tid == 0) {
        bool imp;
        if constexpr (sizeof(MT) == 8 && (MT)0.5 != (MT)0) {
          const double cv = reinterpret_cast<double*>(a.cost)[p];
          double* pl = reinterpret_cast<double*>(a.pl_cost);
          imp = cv < pl[p];
          if (imp) pl[p] = cv;
        } else {
          const int64_t cv = reinterpret_cast<int64_t*>(a.cost)[p];
          int64_t* pl = reinterpret_cast<int64_t*>(a.pl_cost);
          imp = cv < pl[p];
          if (imp) pl[p] = cv;
        }
        a.improved[p] = imp ? 1 : 0;
        sc.ssel[2] = imp;
      }
      Sync::sync();
      if (sc.ssel[2]) {
        int16_t* gpl = a.pl_perm + p * n;
        for (int c = tid; c < n; c += NT) gpl[c] = (int16_t)sc.sperm[c];
      }
    }
    Sync::sync();
  }
  if (tid == 0) bulk_wait_all();
}

}  // namespace qsb
