// aux_kernels.cuh -- the small kernels around the fused step:
//   swarm/global best reduction (engine.py:216-229), migration
//   (migration.py:55-86), the step-draw dump (streams.py:53-64), the
//   standalone goal evaluation (_batch.py:186-197), layout conversion for
//   the reference-layout entry points, and the device population init.
#pragma once
#include <type_traits>
#include "common.cuh"

namespace qsb {

// ----------------------------------------------------------- best update
struct BestArgs {
  int n;
  int64_t S;            // swarm size
  int64_t m;            // local swarms
  int64_t p0;           // global id of local particle 0 (tie-break key)
  const void* cost;     // (P,) of perm_new
  const uint8_t* improved;
  const int16_t* perm_new;
  int16_t* pg_perm;
  void* pg_cost;
  // global best record
  void* best_cost;
  int16_t* best_perm;
  int64_t* best_iter;
  int64_t* best_idx;     // global particle id of the record (for multi-device merges)
  int64_t* t_dev;        // iteration counter; t = *t_dev + 1, written back at the end
  void* swarm_min;       // (m,) scratch: per-swarm min cost over all particles
  int64_t* swarm_min_idx;
  unsigned* done;        // arrival counter (zero-initialised)
  // the next step's draw pre-pass (qsb_best_update_next), or coef == null
  double* coef;          // (P, 2): c2 r2, c3 r3 of iteration t + 1
  double c2, c3;
  uint64_t seed;
  int64_t P;             // local particles
  unsigned* work;        // the step kernel's particle counter, reset here
};

template <typename CT>
__device__ __forceinline__ bool lex_less(CT a, int64_t ia, CT b, int64_t ib) {
  return a < b || (a == b && ia < ib);
}

template <typename CT>
__device__ __forceinline__ void warp_lexmin(CT& c, int64_t& i) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const CT oc = __shfl_xor_sync(FULL, c, o);
    const int64_t oi = __shfl_xor_sync(FULL, i, o);
    if (lex_less(oc, oi, c, i)) { c = oc; i = oi; }
  }
}

template <typename CT>
__device__ __forceinline__ CT ct_max() {
  if constexpr (std::is_floating_point<CT>::value) return __longlong_as_double(0x7ff0000000000000LL);
  else return (CT)0x7fffffffffffffffLL;
}

// One warp per swarm: argmin over improved particles (first index) replaces
// the swarm best when strictly cheaper; argmin over all particles feeds the
// global best, which the last-arriving block applies (strict <, first index).
template <typename CT, int WPB>
__global__ void __launch_bounds__(32 * WPB) best_kernel(const BestArgs a) {
  pdl_wait();     // costs / improved flags of the step kernel
  pdl_launch();   // the next step's coef_kernel waits on this grid anyway
  const int lane = threadIdx.x & 31;
  const int64_t k = (int64_t)blockIdx.x * WPB + (threadIdx.x >> 5);
  const CT* cost = reinterpret_cast<const CT*>(a.cost);
  const int n = a.n;
  if (a.coef) {
    // the next step's (c2 r2, c3 r3): exactly coef_kernel's stream and
    // arithmetic for iteration t + 1 (this grid advances *t_dev to t at its
    // end, so t + 1 = *t_dev + 2 here), and the particle counter reset
    if (a.work && blockIdx.x == 0 && threadIdx.x == 0) *a.work = 0u;
    const uint64_t word1 = stream_word(2, (uint64_t)(*a.t_dev) + 2);
    const uint64_t w = 2 + 2 * (uint64_t)n;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < a.P;
         p += (int64_t)gridDim.x * blockDim.x) {
      const uint64_t idx = (uint64_t)(a.p0 + p) * w;
      const PhiloxBlock b = philox4x64_10((idx >> 2) + 1, a.seed, word1);
      const unsigned l = (unsigned)(idx & 3);   // w is even: l is 0 or 2
      double u0, u1;
      if (l == 0) { u0 = u64_to_unit(b.v[0]); u1 = u64_to_unit(b.v[1]); }
      else { u0 = u64_to_unit(b.v[2]); u1 = u64_to_unit(b.v[3]); }
      a.coef[2 * p] = __dmul_rn(a.c2, u0);
      a.coef[2 * p + 1] = __dmul_rn(a.c3, u1);
    }
  }
  if (k < a.m) {
    CT bi = ct_max<CT>(), ba = ct_max<CT>();
    int64_t ii = INT64_MAX, ia = INT64_MAX;
    const int64_t lo = k * a.S;
    CT* pgc = reinterpret_cast<CT*>(a.pg_cost);
    const CT pg_old = pgc[k];
    // four loads in flight per lane before any compare (S = 100: one batch)
    for (int64_t q0 = 0; q0 < a.S; q0 += 128) {
      CT cv[4];
      bool iv[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t q = q0 + lane + 32 * j;
        cv[j] = q < a.S ? cost[lo + q] : ct_max<CT>();
        iv[j] = q < a.S ? a.improved[lo + q] != 0 : false;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t q = q0 + lane + 32 * j;
        if (q >= a.S) continue;
        const int64_t i = lo + q;
        if (lex_less(cv[j], i, ba, ia)) { ba = cv[j]; ia = i; }
        if (iv[j] && lex_less(cv[j], i, bi, ii)) { bi = cv[j]; ii = i; }
      }
    }
    warp_lexmin(bi, ii);
    warp_lexmin(ba, ia);
    if (ii != INT64_MAX && bi < pg_old) {
      for (int c = lane; c < n; c += 32) a.pg_perm[k * n + c] = a.perm_new[ii * n + c];
      if (lane == 0) pgc[k] = bi;
    }
    if (lane == 0) {
      reinterpret_cast<CT*>(a.swarm_min)[k] = ba;
      a.swarm_min_idx[k] = ia;
    }
  }
  // last block applies the global best
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(a.done, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  // the other blocks' swarm minima, read from L2 (ld.cg), four per thread in
  // flight before any compare; the best record's inputs fetched alongside
  const CT* sm = reinterpret_cast<const CT*>(a.swarm_min);
  const int64_t* smi = a.swarm_min_idx;
  CT* gb = reinterpret_cast<CT*>(a.best_cost);
  const int64_t t = *a.t_dev + 1;
  const CT gb_old = *gb;
  CT bc = ct_max<CT>();
  int64_t bidx = INT64_MAX;
  for (int64_t q0 = 0; q0 < a.m; q0 += 4 * (int64_t)blockDim.x) {
    CT cv[4];
    int64_t iv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t q = q0 + threadIdx.x + (int64_t)j * blockDim.x;
      cv[j] = q < a.m ? __ldcg(sm + q) : ct_max<CT>();
      iv[j] = q < a.m ? (int64_t)__ldcg((const long long*)smi + q) : INT64_MAX;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (lex_less(cv[j], iv[j], bc, bidx)) { bc = cv[j]; bidx = iv[j]; }
  }
  warp_lexmin(bc, bidx);
  __shared__ CT wc[WPB];
  __shared__ int64_t wi[WPB];
  if (lane == 0) { wc[threadIdx.x >> 5] = bc; wi[threadIdx.x >> 5] = bidx; }
  __syncthreads();
  if (threadIdx.x < 32) {
    bc = lane < WPB ? wc[lane] : ct_max<CT>();
    bidx = lane < WPB ? wi[lane] : INT64_MAX;
    warp_lexmin(bc, bidx);
    const bool upd = bidx != INT64_MAX && bc < gb_old;
    if (upd)
      for (int c = lane; c < n; c += 32) a.best_perm[c] = a.perm_new[bidx * n + c];
    __syncwarp();
    if (lane == 0) {
      if (upd) { *gb = bc; *a.best_iter = t; *a.best_idx = a.p0 + bidx; }
      *a.t_dev = t;
      *a.done = 0;
    }
  }
}

// Measurement gate (qsb_stream_gate): one thread polls a host flag in mapped
// pinned memory, parked between polls, with a wall-clock (globaltimer)
// timeout so a host that never opens the gate cannot hang the device.
__global__ void gate_kernel(const volatile int32_t* flag, long long timeout_ns, int32_t* timed_out) {
  if (threadIdx.x != 0) return;
  long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (*flag == 0) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) {
      if (timed_out) *timed_out = 1;
      return;
    }
    __nanosleep(2000);
  }
}

// ------------------------------------------------------------- migration
struct MigArgs {
  int n;
  int64_t S;             // swarm size
  int64_t m;             // total swarms (global)
  int64_t m0;            // first swarm owned by this device
  int64_t m_local;       // swarms owned by this device
  int d;                 // replacements per event
  int period;            // run only when t % period == 0 (0: unconditional)
  const int64_t* t_dev;  // current iteration (already advanced by best_kernel)
  const int32_t* picks;  // (rows, d) donor offsets j = rng.integers(0, S), or
                         // NULL: drawn here from host_rng(seed, t) (host_picks)
  int64_t picks_e0;      // epoch of row 0 (epoch = t / period, or t if period == 0)
  int64_t picks_rows;
  uint64_t seed;         // SolverConfig.seed wrapped to uint64 (device picks)
  const void* all_pg_cost;   // (m,) global swarm-best costs (== pg_cost on one device)
  const int16_t* perm;   // local current particles (post-swap)
  const void* cost;      // local current costs
  int16_t* pg_perm;      // local swarm bests
  void* pg_cost;
  int64_t* plan;         // (d, 4): src, dst, particle, epoch-valid flag
  int64_t* rec;          // (d, n+1) donor records (multi-device exchange), nullable
  double* log;           // (log_rows, d, 6) migration events, nullable
  int64_t log_rows;
  int64_t* log_count;    // events written so far (device counter)
  int* status;           // set to 1 if the picks table has no row for t
  int mode;              // 0 fused (plan+apply), 1 plan+pack, 2 apply from rec
  size_t picks_smem_off; // byte offset of the device picks in dynamic shared memory
};

constexpr int MIG_SORT_MAX = 8192;   // swarms sorted in shared memory (larger m: rank counting)

// 32-bit draw j of a fresh numpy Generator(Philox(key = (seed, word1))):
// numpy's Philox hands out the low then the high half of each 64-bit word,
// words in counter order starting at counter 1 (numpy increments first).
__device__ __forceinline__ uint32_t host_u32(uint64_t seed, uint64_t word1, uint64_t j) {
  const PhiloxBlock b = philox4x64_10((j >> 3) + 1, seed, word1);
  const uint64_t w = b.v[(j >> 1) & 3];
  return (j & 1) ? (uint32_t)(w >> 32) : (uint32_t)w;
}

// The donor offsets of one migration event: d successive scalar calls
// rng.integers(0, S) on host_rng(seed, t) (migration.py:82-84,
// streams.py:48-50).  numpy bounds a 32-bit draw x by Lemire's method:
// m = x * S, rejected while (m mod 2^32) < (2^32 - S) mod S, value m >> 32.
// Draw k uses 32-bit word k unless an earlier draw was rejected, so every
// thread takes its own word and, in the (probability <= d S / 2^32) case of
// a rejection anywhere, one thread redraws the event sequentially.
// Block-wide: every thread of the block must call it.
__device__ void host_picks(uint64_t seed, uint64_t t, int d, int64_t S, int32_t* out) {
  const uint64_t word1 = stream_word(3, t);
  const uint32_t thr = (uint32_t)((0x100000000ULL - (uint64_t)S) % (uint64_t)S);
  int rej = 0;
  for (int k = threadIdx.x; k < d; k += blockDim.x) {
    const uint64_t m = (uint64_t)host_u32(seed, word1, (uint64_t)k) * (uint64_t)S;
    rej |= (uint32_t)m < thr;
    out[k] = (int32_t)(m >> 32);
  }
  if (__syncthreads_or(rej)) {
    if (threadIdx.x == 0) {
      uint64_t j = 0;
      for (int k = 0; k < d; ++k) {
        uint64_t m;
        do { m = (uint64_t)host_u32(seed, word1, j++) * (uint64_t)S; } while ((uint32_t)m < thr);
        out[k] = (int32_t)(m >> 32);
      }
    }
    __syncthreads();
  }
}

// Debug / parity entry: the picks of iteration t into out (one block).
__global__ void picks_kernel(uint64_t seed, uint64_t t, int d, int64_t S, int32_t* out) {
  host_picks(seed, t, d, S, out);
}

// Stable ascending rank of every swarm cost (np.argsort(kind="stable")),
// then rank k donates to rank m-1-k (migration.py:81-90).
template <typename CT>
__global__ void __launch_bounds__(1024) migrate_kernel(const MigArgs a) {
  extern __shared__ __align__(16) unsigned char msm[];
  pdl_wait();     // swarm minima / bests and t_dev of the best update
  pdl_launch();   // the next step kernel may set up meanwhile (it waits on this grid)
  const int64_t t = *a.t_dev;
  if (a.period > 0 && (t % a.period) != 0) return;
  const int64_t epoch = a.period > 0 ? t / a.period : t;
  const int64_t row = epoch - a.picks_e0;
  if (a.mode != 2 && a.picks && (row < 0 || row >= a.picks_rows)) {
    if (threadIdx.x == 0) *a.status = 1;
    return;
  }
  const int n = a.n;
  const int64_t m = a.m;
  CT* pgc = reinterpret_cast<CT*>(a.pg_cost);
  const CT* lcost = reinterpret_cast<const CT*>(a.cost);
  if (a.mode == 2) {
    for (int k = threadIdx.x; k < a.d; k += blockDim.x) {
      const int64_t dst = a.plan[4 * k + 1] - a.m0;
      if (dst < 0 || dst >= a.m_local) continue;
      const int64_t* r = a.rec + (int64_t)k * (n + 1);
      CT c;
      if constexpr (std::is_floating_point<CT>::value) c = __longlong_as_double(r[0]);
      else c = (CT)r[0];
      pgc[dst] = c;
      for (int q = 0; q < n; ++q) a.pg_perm[dst * n + q] = (int16_t)r[1 + q];
    }
    if (a.log && a.log_count && *a.log_count >= a.d) {
      // complete the events with the donors' costs (known only after the exchange)
      const int64_t row0 = (*a.log_count / a.d - 1) * a.d;
      for (int k = threadIdx.x; k < a.d; k += blockDim.x) {
        const int64_t* r = a.rec + (int64_t)k * (n + 1);
        double c;
        if constexpr (std::is_floating_point<CT>::value) c = __longlong_as_double(r[0]);
        else c = (double)r[0];
        a.log[(row0 + k) * 6 + 5] = c;
      }
    }
    return;
  }
  CT* sc = reinterpret_cast<CT*>(msm);
  int32_t* order = reinterpret_cast<int32_t*>(msm + align_up(m * sizeof(CT), 16));
  // device picks after the sort scratch (qsb_migrate sizes the buffer)
  int32_t* dpk = reinterpret_cast<int32_t*>(msm + a.picks_smem_off);
  if (!a.picks) host_picks(a.seed, (uint64_t)t, a.d, a.S, dpk);
  const CT* allc = reinterpret_cast<const CT*>(a.all_pg_cost);
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) sc[i] = allc[i];
  __syncthreads();
  const int mi = (int)m;
  const int p2 = mi <= 1 ? 1 : 1 << (32 - __clz(mi - 1));
  if (p2 <= MIG_SORT_MAX) {
    // stable ascending order (np.argsort kind="stable") by a bitonic sort of
    // (cost, index) keys in shared memory, padded to a power of two
    CT* kc = reinterpret_cast<CT*>(order + align_up((size_t)p2, 4));   // ki = order: p2 entries
    int32_t* ki = order;
    for (int i = threadIdx.x; i < p2; i += blockDim.x) {
      kc[i] = i < mi ? sc[i] : ct_max<CT>();
      ki[i] = i < mi ? i : INT_MAX;
    }
    __syncthreads();
    for (int size = 2; size <= p2; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = threadIdx.x; i < p2; i += blockDim.x) {
          const int j = i ^ stride;
          if (j <= i) continue;
          const CT ci = kc[i], cj = kc[j];
          const int ii = ki[i], ij = ki[j];
          const bool gt = ci > cj || (ci == cj && ii > ij);
          if (gt == ((i & size) == 0)) { kc[i] = cj; kc[j] = ci; ki[i] = ij; ki[j] = ii; }
        }
        __syncthreads();
      }
    }
  } else {
    // large m: stable rank of each swarm cost, one warp per swarm
    const int lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
    for (int i = threadIdx.x >> 5; i < mi; i += nwarp) {
      const CT ci = sc[i];
      unsigned r = 0;
      for (int j = lane; j < mi; j += 32) {
        const CT cj = sc[j];
        r += (cj < ci) || (cj == ci && j < i);
      }
      r = __reduce_add_sync(0xffffffffu, r);
      if (lane == 0) order[r] = i;
    }
  }
  __syncthreads();
  const int32_t* picks = a.picks ? a.picks + row * a.d : dpk;
  for (int k = threadIdx.x; k < a.d; k += blockDim.x) {
    const int64_t src = order[k];
    const int64_t dst = order[m - 1 - k];
    const int64_t particle = src * a.S + picks[k];
    const int64_t lp = particle - a.m0 * a.S;
    const bool src_local = src >= a.m0 && src < a.m0 + a.m_local;
    const bool dst_local = dst >= a.m0 && dst < a.m0 + a.m_local;
    a.plan[4 * k + 0] = src;
    a.plan[4 * k + 1] = dst;
    a.plan[4 * k + 2] = particle;
    a.plan[4 * k + 3] = 1;
    if (a.log && (*a.log_count / a.d) < a.log_rows) {
      double* e = a.log + ((*a.log_count / a.d) * a.d + k) * 6;
      e[0] = (double)t; e[1] = (double)src; e[2] = (double)dst; e[3] = (double)particle;
      e[4] = (double)sc[dst];
      e[5] = src_local ? (double)lcost[lp] : 0.0;   // multi-device: filled by the host
    }
    if (a.mode == 0) {
      pgc[dst] = lcost[lp];   // one device owns everything: swarm-best cost in place
    } else if (a.rec) {
      int64_t* r = a.rec + (int64_t)k * (n + 1);
      if (src_local) {
        if constexpr (std::is_floating_point<CT>::value) r[0] = __double_as_longlong(lcost[lp]);
        else r[0] = (int64_t)lcost[lp];
      } else {
        r[0] = 0;
      }
    }
    (void)dst_local;
  }
  // the donor permutations, all (event, facility) pairs across the block
  if (a.mode == 0 || a.rec) {
    const int64_t dn = (int64_t)a.d * n;
    for (int64_t e = threadIdx.x; e < dn; e += blockDim.x) {
      const int k = (int)(e / n), q = (int)(e - (int64_t)k * n);
      const int64_t src = order[k];
      const int64_t lp = src * a.S + picks[k] - a.m0 * a.S;
      const bool src_local = src >= a.m0 && src < a.m0 + a.m_local;
      if (a.mode == 0) {
        a.pg_perm[(int64_t)order[m - 1 - k] * n + q] = a.perm[lp * n + q];
      } else {
        a.rec[(int64_t)k * (n + 1) + 1 + q] = src_local ? (int64_t)a.perm[lp * n + q] : 0;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && a.log && (*a.log_count / a.d) < a.log_rows) *a.log_count += a.d;
}

// --------------------------------------------------------- draws (debug)
__global__ void draws_kernel(uint64_t seed, uint64_t t, int64_t p0, int64_t P, int n, double* out) {
  const int64_t w = 2 + 2 * (int64_t)n;
  const int64_t total = P * w;
  const uint64_t word1 = stream_word(2, t);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t idx = (uint64_t)(p0 * w + e);
    const PhiloxBlock b = philox4x64_10((idx >> 2) + 1, seed, word1);
    out[e] = u64_to_unit(b.v[idx & 3]);
  }
}

// Per-particle (c2 * r2, c3 * r3) of iteration t (engine.py:198-199; draw
// columns 0 and 1 of streams.step_draws), one thread per particle, ahead of
// the step kernel: keeps the dependent Philox chain off the step kernel's
// per-particle critical path.
__global__ void coef_kernel(uint64_t seed, const int64_t* t_dev, uint64_t t_host, int64_t p0,
                            int64_t P, int n, double c2, double c3, double* out, unsigned* work) {
  pdl_wait();     // t_dev is advanced by the previous step's best_kernel
  pdl_launch();   // the step kernel may stage its constants meanwhile
  // the step kernel's particle counter, reset here instead of by a memset
  if (work && blockIdx.x == 0 && threadIdx.x == 0) *work = 0u;
  const uint64_t t = t_dev ? (uint64_t)(*t_dev) + 1 : t_host;
  const uint64_t word1 = stream_word(2, t);
  const uint64_t w = 2 + 2 * (uint64_t)n;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P;
       p += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t idx = (uint64_t)(p0 + p) * w;
    const PhiloxBlock b = philox4x64_10((idx >> 2) + 1, seed, word1);
    const unsigned l = (unsigned)(idx & 3);   // w is even: l is 0 or 2
    double u0, u1;
    if (l == 0) { u0 = u64_to_unit(b.v[0]); u1 = u64_to_unit(b.v[1]); }
    else { u0 = u64_to_unit(b.v[2]); u1 = u64_to_unit(b.v[3]); }
    out[2 * p] = __dmul_rn(c2, u0);
    out[2 * p + 1] = __dmul_rn(c3, u1);
  }
}

// ------------------------------------------------------ standalone goal
template <typename MT, typename PT>
__global__ void cost_kernel(const PT* perms, int64_t P, int n, const MT* F, const MT* D, void* out) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t p = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); p < P; p += nw) {
    const PT* pp = perms + p * n;
    if constexpr (std::is_floating_point<MT>::value) {
      if (lane == 0) {
        double acc = (double)F[0] * (double)D[0] * 0.0;
        for (int i = 0; i < n; ++i) {
          const int64_t pi = pp[i];
          for (int j = 0; j < n; ++j)
            acc = __dadd_rn(acc, __dmul_rn((double)F[i * n + j], (double)D[pi * n + pp[j]]));
        }
        reinterpret_cast<double*>(out)[p] = acc;
      }
    } else {
      uint64_t part = 0;
      for (int j = lane; j < n; j += 32) {
        const int64_t pj = pp[j];
        for (int i = 0; i < n; ++i) part += (uint64_t)F[i * n + j] * (uint64_t)D[(int64_t)pp[i] * n + pj];
      }
      for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(FULL, part, o);
      if (lane == 0) reinterpret_cast<int64_t*>(out)[p] = (int64_t)part;
    }
  }
}

// ------------------------------------------------------- layout helpers
// Reference layout X[k, i] = 1 iff k == perm[i] (core.py:5-6) -> perm.
// bad[0] is set when a column does not hold exactly one 1.
__global__ void mat_to_perm_kernel(const int8_t* x, int64_t P, int n, int16_t* perm, int* bad) {
  const int64_t total = P * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = e / n;
    const int c = (int)(e % n);
    const int8_t* xp = x + p * n * n;
    int r1 = -1, ones = 0;
    for (int r = 0; r < n; ++r) if (xp[r * n + c] == 1) { ++ones; r1 = r; }
    if (ones != 1) { atomicExch(bad, 1); r1 = 0; }
    perm[e] = (int16_t)r1;
  }
}

template <typename PT>
__global__ void perm_to_mat_kernel(const PT* perm, int64_t P, int n, int8_t* x) {
  const int64_t total = P * n * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = e / ((int64_t)n * n);
    const int rc = (int)(e % ((int64_t)n * n));
    const int r = rc / n, c = rc % n;
    x[e] = (perm[p * n + c] == r) ? 1 : 0;
  }
}

// -------------------------------------------- device population init
// Throughput-mode initialisation (NOT the reference's init stream): every
// particle draws a Fisher-Yates permutation and U(-amp, amp) velocities from
// Philox keyed (seed, 4<<56); particle rows are counter offsets, so the
// result is independent of the device count.  Global particle p owns words
// p (n^2 + n) + e: e < n^2 the velocity entries (row-major), then n - 1
// shuffle draws, i = n-1 .. 1 swapping perm[i] with perm[min(floor(u (i+1)), i)]
// (the reference's init_population, engine.py:150-156, draws a permuted
// identity and U(-amp, amp) the same way, from its own sequential stream).
template <typename VT>
__global__ void init_kernel(uint64_t seed, int64_t p0, int64_t P, int n, int vstride, double amp,
                            int16_t* perm, VT* V, int wide) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const uint64_t word1 = stream_word(4, 0);
  const int64_t nn = (int64_t)n * n;
  const uint64_t row_w = (uint64_t)(nn + n);
  for (int64_t p = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); p < P; p += nw) {
    const uint64_t base = (uint64_t)(p0 + p) * row_w;
    VT* vp = V + p * vstride;
    for (int64_t e = lane; e < vstride; e += 32) {
      if (e < nn) {
        const uint64_t idx = base + (uint64_t)e;
        const double u = u64_to_unit(philox4x64_10((idx >> 2) + 1, seed, word1).v[idx & 3]);
        // (-amp) + (2 amp) u with separate roundings (no FMA), so the oracle
        // restates it in numpy (oracle.device_init)
        const double v = __dadd_rn(-amp, __dmul_rn(__dmul_rn(2.0, amp), u));
        if constexpr (sizeof(VT) == 4) vp[e] = wide ? (VT)wenc(v) : (VT)v;
        else vp[e] = (VT)v;
      } else {
        vp[e] = (VT)0;
      }
    }
    if (lane == 0) {
      int16_t* pp = perm + p * n;
      for (int i = 0; i < n; ++i) pp[i] = (int16_t)i;
      DrawCache dr;
      dr.init(DrawKey{nullptr, seed, word1, base + (uint64_t)nn});
      for (int i = n - 1; i > 0; --i) {
        long long j = (long long)(dr.at(n - 1 - i) * (double)(i + 1));
        if (j > i) j = i;
        const int16_t tmp = pp[i]; pp[i] = pp[j]; pp[j] = tmp;
      }
    }
  }
}

}  // namespace qsb
