// twoopt.cuh -- 2-opt (pairwise facility exchange) local search, integer.
//
// Not part of the reference (the reference lists delta
// evaluation as a non-goal).  North-star extension, applied to
// each particle's new permutation after S_x and the goal, before the personal
// best.  Policy per pass: evaluate every swap (r, s), r < s, with the exact
// integer delta of SURVEY.md Appendix A4, take the smallest delta with ties
// to the lexicographically first (r, s), apply it if negative, else stop.
// CPU oracle: orc_twoopt_many in oracle/qap_oracle.c.
//
// One CTA per particle.  The permuted distance matrix Dp[i][j] = D[p_i][p_j]
// lives in shared memory, so a delta is a contiguous O(n) sweep; a move
// swaps two rows and two columns of Dp.  All n(n-1)/2 deltas of a pass are
// scored in parallel (pair q -> (r, s) by closed-form unranking) and reduced
// to the lexicographic (delta, q) minimum.
#pragma once
#include <type_traits>
#include "common.cuh"

namespace qsb {

struct TwoOptArgs {
  int n;
  int ldn;          // byte-matrix row stride (dp4a kernel)
  int64_t P;
  int passes;
  int sym;          // F and D symmetric (halves the delta sweep)
  int do_pbest;     // also apply the personal-best update (engine.py:211-215)
  int f_smem;       // F staged in shared memory
  int16_t* perm;    // (P, n) in/out: the particles' new positions
  int64_t* cost;    // (P,) in/out
  int16_t* pl_perm;
  int64_t* pl_cost;
  uint8_t* improved;
  const void* F;
  const void* D;
};

__device__ __forceinline__ void unrank_pair(int64_t q, int n, int& r, int& s) {
  const double t = sqrt((double)(-8 * q + 4 * (int64_t)n * (n - 1) - 7));
  r = n - 2 - (int)floor(t / 2.0 - 0.5);
  s = (int)(q + r + 1 - (int64_t)n * (n - 1) / 2 + (int64_t)(n - r) * (n - r - 1) / 2);
}

template <typename MT, int NT>
__global__ void __launch_bounds__(NT) twoopt_kernel(const TwoOptArgs a) {
  using DT = MT;   // Dp holds D entries, same range
  extern __shared__ __align__(16) unsigned char tsm[];
  const int n = a.n;
  const int nn = n * n;
  DT* Dp = reinterpret_cast<DT*>(tsm);
  size_t off = align_up((size_t)nn * sizeof(DT), 16);
  MT* sF = reinterpret_cast<MT*>(tsm + off);
  if (a.f_smem) off += align_up((size_t)nn * sizeof(MT), 16);
  int* sp = reinterpret_cast<int*>(tsm + off);
  off += align_up((size_t)n * sizeof(int), 16);
  int64_t* rd = reinterpret_cast<int64_t*>(tsm + off);
  int* rq = reinterpret_cast<int*>(rd + NT / 32);
  __shared__ int s_move;

  const MT* gF = reinterpret_cast<const MT*>(a.F);
  const MT* gD = reinterpret_cast<const MT*>(a.D);
  if (a.f_smem)
    for (int i = threadIdx.x; i < nn; i += NT) sF[i] = gF[i];
  const MT* F = a.f_smem ? sF : gF;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t npairs = (int64_t)n * (n - 1) / 2;

  for (int64_t p = blockIdx.x; p < a.P; p += gridDim.x) {
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += NT) sp[i] = a.perm[p * n + i];
    __syncthreads();
    for (int e = threadIdx.x; e < nn; e += NT) Dp[e] = (DT)gD[sp[e / n] * n + sp[e % n]];
    __syncthreads();
    uint64_t cost = (uint64_t)a.cost[p];
    for (int pass = 0; pass < a.passes; ++pass) {
      int64_t best = INT64_MAX;
      int bq = INT_MAX;
      if (a.sym && n >= 96 && sizeof(MT) == 2 && (n % 2) == 0) {
        // large symmetric n: one warp per pair, lanes over k (row streams
        // F[r][.], F[s][.], Dp[r][.], Dp[s][.] are contiguous -> no bank
        // conflicts; two uint16 per 32-bit load)
        const unsigned* F32 = reinterpret_cast<const unsigned*>(F);
        const unsigned* D32 = reinterpret_cast<const unsigned*>(Dp);
        const int h = n / 2;
        for (int64_t q = warp; q < npairs; q += NT / 32) {
          int r, s;
          unrank_pair(q, n, r, s);
          int64_t acc = 0;
          for (int j = lane; j < h; j += 32) {
            const unsigned fr = F32[r * h + j], fs = F32[s * h + j];
            const unsigned dr = D32[r * h + j], ds = D32[s * h + j];
            const int k0 = 2 * j, k1 = 2 * j + 1;
            const int64_t a0 = ((int64_t)(fr & 0xffff) - (int64_t)(fs & 0xffff)) *
                               ((int64_t)(ds & 0xffff) - (int64_t)(dr & 0xffff));
            const int64_t a1 = ((int64_t)(fr >> 16) - (int64_t)(fs >> 16)) *
                               ((int64_t)(ds >> 16) - (int64_t)(dr >> 16));
            acc += (k0 == r || k0 == s) ? 0 : a0;
            acc += (k1 == r || k1 == s) ? 0 : a1;
          }
#pragma unroll
          for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
          const int64_t dd = (int64_t)((uint64_t)((int64_t)F[r * n + r] - F[s * n + s]) *
                                           (uint64_t)((int64_t)Dp[s * n + s] - Dp[r * n + r]) +
                                       2 * (uint64_t)acc);
          if (dd < best) { best = dd; bq = (int)q; }   // q ascends per warp: first wins
        }
      } else
      for (int64_t q = threadIdx.x; q < npairs; q += NT) {
        int r, s;
        unrank_pair(q, n, r, s);
        const DT* Dr = Dp + r * n;
        const DT* Ds = Dp + s * n;
        uint64_t d = (uint64_t)((int64_t)F[r * n + r] - F[s * n + s]) * (uint64_t)((int64_t)Ds[s] - Dr[r]);
        uint64_t acc = 0;
        if (a.sym) {
          // F, D symmetric: both k-terms are equal and the (r,s) cross term vanishes
          for (int k = 0; k < n; ++k) {
            if (k == r || k == s) continue;
            acc += (uint64_t)((int64_t)F[k * n + r] - F[k * n + s]) * (uint64_t)((int64_t)Ds[k] - Dr[k]);
          }
          d += 2 * acc;
        } else {
          d += (uint64_t)((int64_t)F[r * n + s] - F[s * n + r]) * (uint64_t)((int64_t)Ds[r] - Dr[s]);
          for (int k = 0; k < n; ++k) {
            if (k == r || k == s) continue;
            const DT* Dk = Dp + k * n;
            acc += (uint64_t)((int64_t)F[k * n + r] - F[k * n + s]) * (uint64_t)((int64_t)Dk[s] - Dk[r])
                 + (uint64_t)((int64_t)F[r * n + k] - F[s * n + k]) * (uint64_t)((int64_t)Ds[k] - Dr[k]);
          }
          d += acc;
        }
        const int64_t dd = (int64_t)d;
        if (dd < best) { best = dd; bq = (int)q; }   // q ascends per thread: first wins
      }
      // lexicographic (delta, q) minimum over the CTA
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const int64_t ob = __shfl_xor_sync(FULL, best, o);
        const int oq = __shfl_xor_sync(FULL, bq, o);
        if (ob < best || (ob == best && oq < bq)) { best = ob; bq = oq; }
      }
      if (lane == 0) { rd[warp] = best; rq[warp] = bq; }
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int w = 1; w < NT / 32; ++w)
          if (rd[w] < rd[0] || (rd[w] == rd[0] && rq[w] < rq[0])) { rd[0] = rd[w]; rq[0] = rq[w]; }
        s_move = (rq[0] != INT_MAX && rd[0] < 0) ? rq[0] : -1;
      }
      __syncthreads();
      const int mq = s_move;
      if (mq < 0) break;
      cost += (uint64_t)rd[0];
      int r, s;
      unrank_pair(mq, n, r, s);
      // swap facilities r and s: rows r, s then columns r, s of Dp
      for (int j = threadIdx.x; j < n; j += NT) {
        const DT t = Dp[r * n + j]; Dp[r * n + j] = Dp[s * n + j]; Dp[s * n + j] = t;
      }
      __syncthreads();
      for (int i = threadIdx.x; i < n; i += NT) {
        const DT t = Dp[i * n + r]; Dp[i * n + r] = Dp[i * n + s]; Dp[i * n + s] = t;
      }
      if (threadIdx.x == 0) { const int t = sp[r]; sp[r] = sp[s]; sp[s] = t; }
      __syncthreads();
    }
    for (int i = threadIdx.x; i < n; i += NT) a.perm[p * n + i] = (int16_t)sp[i];
    if (a.do_pbest) {
      // one thread decides (strict <, engine.py:211), then all copy
      __syncthreads();
      if (threadIdx.x == 0) {
        const bool imp = (int64_t)cost < a.pl_cost[p];
        if (imp) a.pl_cost[p] = (int64_t)cost;
        a.improved[p] = imp ? 1 : 0;
        s_move = imp;
      }
      __syncthreads();
      if (s_move)
        for (int i = threadIdx.x; i < n; i += NT) a.pl_perm[p * n + i] = (int16_t)sp[i];
    }
    if (threadIdx.x == 0) a.cost[p] = (int64_t)cost;
  }
}


// ---------------------------------------------------------------------------
// 2-opt for symmetric instances with byte-sized entries (n * max(F) * max(D)
// < 2^31), as packed 4-way byte dot products.  For symmetric F and D the
// permuted distance matrix P = D[p][p] is symmetric and
//   sum_{k != r,s} (F_kr - F_ks)(P_ks - P_kr)
//     = G[r][s] + G[s][r] - G[r][r] - G[s][s] - T_r - T_s,
//   G[a][b] = sum_k F[a][k] P[b][k]   (rows: contiguous k),
//   T_r = (F_rr - F_rs)(P_rs - P_rr),  T_s = (F_sr - F_ss)(P_ss - P_sr),
// so delta(r, s) = (F_rr - F_ss)(P_ss - P_rr) + 2 * that sum -- the value
// twoopt_kernel's symmetric sweep computes, exact in int64 (G < 2^31).
// Each thread owns a 4 x 4 block pair (rows r0.., s0..) of the upper
// triangle and accumulates G[r][s] and G[s][r] with __dp4a.  The byte
// matrices live in shared memory in a 4-row interleaved layout: the four
// rows of a block share 16-byte chunks, so one 128-bit load fetches word w
// of all four rows, and an odd chunk stride per block keeps the loads of
// consecutive blocks in distinct banks.
__device__ __forceinline__ int bidx(int r, int c, int ldw) {
  return ((((r >> 2) * ldw + (c >> 2)) << 4) | ((r & 3) << 2) | (c & 3));
}

template <int NT>
__global__ void __launch_bounds__(NT) twoopt_dp4a_kernel(const TwoOptArgs a) {
  extern __shared__ __align__(16) unsigned char tsm[];
  const int n = a.n;
  const int ldw = a.ldn >> 2;          // 16-byte chunks per 4-row block (odd)
  const int nb = (n + 3) >> 2;         // 4-row blocks
  const int nr = nb * 4;
  const size_t mbytes = (size_t)nb * ldw * 16;
  uint8_t* F8 = tsm;
  uint8_t* D8 = F8 + mbytes;
  uint8_t* P8 = D8 + mbytes;
  int* sp = reinterpret_cast<int*>(P8 + mbytes);
  int* gd = sp + nr;
  int64_t* rd = reinterpret_cast<int64_t*>(gd + nr + (nr & 1));
  int* rq = reinterpret_cast<int*>(rd + NT / 32);
  __shared__ int s_move;
  const uint4* F128 = reinterpret_cast<const uint4*>(F8);
  const uint4* P128 = reinterpret_cast<const uint4*>(P8);
  const uint16_t* gF = reinterpret_cast<const uint16_t*>(a.F);
  const uint16_t* gD = reinterpret_cast<const uint16_t*>(a.D);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ncols = ldw * 4;
  for (int e = threadIdx.x; e < nr * ncols; e += NT) {
    const int r = e / ncols, c = e - r * ncols;
    const bool in = r < n && c < n;
    const int i = bidx(r, c, ldw);
    F8[i] = in ? (uint8_t)gF[r * n + c] : 0;
    D8[i] = in ? (uint8_t)gD[r * n + c] : 0;
    P8[i] = 0;
  }
  const int nbp = nb * (nb + 1) / 2;
  for (int64_t p = blockIdx.x; p < a.P; p += gridDim.x) {
    __syncthreads();
    for (int i = threadIdx.x; i < nr; i += NT) sp[i] = i < n ? a.perm[p * n + i] : 0;
    __syncthreads();
    for (int e = threadIdx.x; e < n * n; e += NT) {
      const int r = e / n, c = e - r * n;
      P8[bidx(r, c, ldw)] = D8[bidx(sp[r], sp[c], ldw)];
    }
    __syncthreads();
    uint64_t cost = (uint64_t)a.cost[p];
    for (int pass = 0; pass < a.passes; ++pass) {
      // G[r][r] for every row
      for (int r = threadIdx.x; r < n; r += NT) {
        const unsigned* F32 = reinterpret_cast<const unsigned*>(F8);
        const unsigned* P32 = reinterpret_cast<const unsigned*>(P8);
        unsigned acc = 0;
        for (int w = 0; w < ldw; ++w) {
          const int wi = (((r >> 2) * ldw + w) << 2) | (r & 3);
          acc = __dp4a(F32[wi], P32[wi], acc);
        }
        gd[r] = (int)acc;
      }
      __syncthreads();
      int64_t best = INT64_MAX;
      int bq = INT_MAX;
      for (int bp = threadIdx.x; bp < nbp; bp += NT) {
        // block pair (bi <= bj) from its upper-triangle rank
        int bi = (int)((2.0f * nb + 1.0f - sqrtf((2.0f * nb + 1.0f) * (2.0f * nb + 1.0f) - 8.0f * bp)) * 0.5f);
        bi = max(0, min(bi, nb - 1));
        while (bi > 0 && bi * nb - bi * (bi - 1) / 2 > bp) --bi;
        while (bi + 1 < nb && (bi + 1) * nb - (bi + 1) * bi / 2 <= bp) ++bi;
        const int bj = bi + bp - (bi * nb - bi * (bi - 1) / 2);
        unsigned gA[4][4], gB[4][4];
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) { gA[x][y] = 0; gB[x][y] = 0; }
        const uint4* fr = F128 + bi * ldw;
        const uint4* pr = P128 + bi * ldw;
        const uint4* fs = F128 + bj * ldw;
        const uint4* ps = P128 + bj * ldw;
#pragma unroll 2
        for (int w = 0; w < ldw; ++w) {
          const uint4 a_fr = fr[w], a_pr = pr[w], a_fs = fs[w], a_ps = ps[w];
          const unsigned f_r[4] = {a_fr.x, a_fr.y, a_fr.z, a_fr.w};
          const unsigned p_r[4] = {a_pr.x, a_pr.y, a_pr.z, a_pr.w};
          const unsigned f_s[4] = {a_fs.x, a_fs.y, a_fs.z, a_fs.w};
          const unsigned p_s[4] = {a_ps.x, a_ps.y, a_ps.z, a_ps.w};
#pragma unroll
          for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) {
              gA[x][y] = __dp4a(f_r[x], p_s[y], gA[x][y]);   // G[r][s]
              gB[x][y] = __dp4a(f_s[y], p_r[x], gB[x][y]);   // G[s][r]
            }
        }
        const int r0 = 4 * bi, s0 = 4 * bj;
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) {
            const int r = r0 + x, s = s0 + y;
            if (r >= s || s >= n) continue;
            const int64_t Frr = F8[bidx(r, r, ldw)], Fss = F8[bidx(s, s, ldw)], Frs = F8[bidx(r, s, ldw)];
            const int64_t Prr = P8[bidx(r, r, ldw)], Pss = P8[bidx(s, s, ldw)], Prs = P8[bidx(r, s, ldw)];
            const int64_t sum = (int64_t)gA[x][y] + (int64_t)gB[x][y] - gd[r] - gd[s]
                                - (Frr - Frs) * (Prs - Prr) - (Frs - Fss) * (Pss - Prs);
            const int64_t dd = (Frr - Fss) * (Pss - Prr) + 2 * sum;
            const int q = r * n - r * (r + 1) / 2 + (s - r - 1);
            if (dd < best || (dd == best && q < bq)) { best = dd; bq = q; }
          }
      }
      // lexicographic (delta, q) minimum over the CTA
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const int64_t ob = __shfl_xor_sync(FULL, best, o);
        const int oq = __shfl_xor_sync(FULL, bq, o);
        if (ob < best || (ob == best && oq < bq)) { best = ob; bq = oq; }
      }
      if (lane == 0) { rd[warp] = best; rq[warp] = bq; }
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int w = 1; w < NT / 32; ++w)
          if (rd[w] < rd[0] || (rd[w] == rd[0] && rq[w] < rq[0])) { rd[0] = rd[w]; rq[0] = rq[w]; }
        s_move = (rq[0] != INT_MAX && rd[0] < 0) ? rq[0] : -1;
      }
      __syncthreads();
      const int mq = s_move;
      if (mq < 0) break;
      cost += (uint64_t)rd[0];
      int r, s;
      unrank_pair(mq, n, r, s);
      // swap facilities r and s: rows r, s then columns r, s of P
      for (int j = threadIdx.x; j < n; j += NT) {
        const int ir = bidx(r, j, ldw), is = bidx(s, j, ldw);
        const uint8_t t = P8[ir]; P8[ir] = P8[is]; P8[is] = t;
      }
      __syncthreads();
      for (int i = threadIdx.x; i < n; i += NT) {
        const int ir = bidx(i, r, ldw), is = bidx(i, s, ldw);
        const uint8_t t = P8[ir]; P8[ir] = P8[is]; P8[is] = t;
      }
      if (threadIdx.x == 0) { const int t = sp[r]; sp[r] = sp[s]; sp[s] = t; }
      __syncthreads();
    }
    for (int i = threadIdx.x; i < n; i += NT) a.perm[p * n + i] = (int16_t)sp[i];
    if (a.do_pbest) {
      __syncthreads();
      if (threadIdx.x == 0) {
        const bool imp = (int64_t)cost < a.pl_cost[p];
        if (imp) a.pl_cost[p] = (int64_t)cost;
        a.improved[p] = imp ? 1 : 0;
        s_move = imp;
      }
      __syncthreads();
      if (s_move)
        for (int i = threadIdx.x; i < n; i += NT) a.pl_perm[p * n + i] = (int16_t)sp[i];
    }
    if (threadIdx.x == 0) a.cost[p] = (int64_t)cost;
  }
}


// ---------------------------------------------------------------------------
// 2-opt on the 5th-generation tensor cores (symmetric instances, byte
// entries).  The O(n^3) part of a pass is H[r][s] = G[r][s] + G[s][r] of the
// dp4a kernel above, and H is one GEMM:
//   H = F P^T + P F^T = [F | P] [P | F]^T        (K = 2n),
// unsigned 8-bit operands with exact s32 accumulation (tcgen05.mma
// kind::i8; every H entry is < 2 n 255^2 < 2^32 and non-negative, read as
// uint32).  F and P sit in shared memory in the canonical K-major,
// no-swizzle UMMA layout (8-row x 16-byte core matrices); H lands in tensor
// memory, one TMEM lane per row r, and the epilogue threads read their row
// with tcgen05.ld and score the swaps (r, s > r) exactly as the dp4a kernel
// (same int64 delta, same lexicographic (delta, q) order), so the two
// kernels are interchangeable bit for bit.
//
// One CTA per particle at a time; one thread issues the MMAs of a pass
// (M = 128 rows per tile, 1 or 2 tiles; N = n rounded up to 16; K in steps
// of 32 bytes) and commits them to an mbarrier the CTA waits on.

// byte offset of (row r, byte k) in the canonical layout with kb bytes per row
__device__ __forceinline__ int cl_off(int r, int k, int kb) {
  return (r >> 3) * (kb << 3) + ((k >> 4) << 7) + ((r & 7) << 4) + (k & 15);
}

// shared-memory matrix descriptor: K-major, no swizzle (layout type 0),
// LBO = byte distance of K-adjacent core matrices, SBO = of 8-row groups
__device__ __forceinline__ uint64_t umma_smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ULL << 46);   // descriptor version 1 (sm_100)
}

// instruction descriptor: u8 x u8 -> s32, both K-major, M x N
__host__ __device__ constexpr uint32_t umma_idesc_u8(int M, int N) {
  return (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void umma_i8(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
      :: "r"(d_tmem), "l"(a), "l"(b), "r"(idesc), "r"(accumulate) : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               :: "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// 16 consecutive 32-bit TMEM columns of this thread's lane
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

struct TwoOptTc {
  int kb;       // bytes per operand row: n rounded up to 32
  int npad;     // N: n rounded up to 16
  int tiles;    // M tiles of 128 rows
  int tcols;    // allocated TMEM columns (power of two >= 32)
  static __host__ __device__ size_t smem_bytes(int n, int kb, int tiles, int NT) {
    const size_t mb = (size_t)tiles * 128 * kb;
    return 2 * mb + align_up((size_t)n * (n + 1), 16) + align_up((size_t)n * 4, 16) +
           (size_t)(n + 15) / 16 * 256 + (NT / 32) * 12 + 64;
  }
};

template <int NT>
__global__ void __launch_bounds__(NT) twoopt_tc_kernel(const TwoOptArgs a, const TwoOptTc g) {
  extern __shared__ __align__(1024) unsigned char tsm[];
  const int n = a.n, kb = g.kb, npad = g.npad, tiles = g.tiles;
  const size_t mb = (size_t)tiles * 128 * kb;
  uint8_t* F8 = tsm;                      // canonical layout, rows >= n and bytes >= n zero
  uint8_t* P8 = F8 + mb;                  // P = D[p][p], same layout
  uint8_t* D8 = P8 + mb;                  // D row-major, row stride n + 1, column n zero
  const int dn = n + 1;
  int* sp = reinterpret_cast<int*>(D8 + align_up((size_t)n * dn, 16));
  int4* sv = reinterpret_cast<int4*>(sp + align_up((size_t)n, 4));   // per row: {G[r][r], F_rr, P_rr, 0}
  int64_t* rd = reinterpret_cast<int64_t*>(sv + (n + 15) / 16 * 16);
  int* rq = reinterpret_cast<int*>(rd + NT / 32);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t s_tmem;
  __shared__ int s_move;
  __shared__ unsigned s_mx[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint16_t* gF = reinterpret_cast<const uint16_t*>(a.F);
  const uint16_t* gD = reinterpret_cast<const uint16_t*>(a.D);

  if (tid < 2) s_mx[tid] = 0;
  {
    uint4* z = reinterpret_cast<uint4*>(F8);
    const int nz = (int)(2 * mb / 16);
    for (int i = tid; i < nz; i += NT) z[i] = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  unsigned mf = 0, md = 0;
  for (int e = tid; e < n * n; e += NT) {
    const int r = e / n, c = e - r * n;
    F8[cl_off(r, c, kb)] = (uint8_t)gF[e];
    D8[r * dn + c] = (uint8_t)gD[e];
    mf = max(mf, (unsigned)gF[e]);
    md = max(md, (unsigned)gD[e]);
  }
  for (int r = tid; r < n; r += NT) D8[r * dn + n] = 0;
  atomicMax(&s_mx[0], mf);
  atomicMax(&s_mx[1], md);
  if (tid == 0) { mbar_init(&bar, 1); mbar_fence_init(); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32(&s_tmem)), "r"(g.tcols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  const uint32_t idesc = umma_idesc_u8(128, npad);
  const uint32_t sbo = (uint32_t)kb * 8;
  const int ksteps = kb / 32;
  uint32_t phase = 0;

  // epilogue role of this warp: tile t, lane quarter q, column chunks c = h, h + cs, ...
  const int q = warp & 3;
  const int t = (NT == 256 && tiles == 2) ? (warp >> 2) : 0;
  const int h = (NT == 256 && tiles == 1) ? (warp >> 2) : 0;
  const int cs = (NT == 256 && tiles == 1) ? 2 : 1;
  const int rbase = t * 128 + q * 32;
  const int r = rbase + lane;
  const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(t * npad);
  const int nchunks = npad / 16;
  // n max(F) max(D) < 2^28: every H, G[r][r] and delta fits int32
  const bool narrow = (double)n * (double)s_mx[0] * (double)s_mx[1] < 268435456.0;

  for (int64_t p = blockIdx.x; p < a.P; p += gridDim.x) {
    __syncthreads();
    for (int i = tid; i < n; i += NT) sp[i] = a.perm[p * n + i];
    __syncthreads();
    {
      // P = D[p][p], 16 bytes per store: a thread keeps one 16-column chunk
      // (its sp entries in registers) and walks rows; bytes >= n stay zero
      const int nck = kb >> 4;
      const int c = tid % nck;
      int spc[16];
#pragma unroll
      for (int b = 0; b < 16; ++b) spc[b] = c * 16 + b < n ? sp[c * 16 + b] : n;   // n: the zero column
      for (int i = tid / nck; i < n; i += NT / nck) {
        const uint8_t* drow = D8 + sp[i] * dn;
        unsigned w[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          const unsigned b0 = drow[spc[4 * x]], b1 = drow[spc[4 * x + 1]];
          const unsigned b2 = drow[spc[4 * x + 2]], b3 = drow[spc[4 * x + 3]];
          w[x] = __byte_perm(__byte_perm(b0, b1, 0x0040), __byte_perm(b2, b3, 0x0040), 0x5410);
        }
        *reinterpret_cast<uint4*>(P8 + cl_off(i, c * 16, kb)) = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
    uint64_t cost = (uint64_t)a.cost[p];
    for (int pass = 0; pass < a.passes; ++pass) {
      __syncthreads();
      // G[r][r] (4-way byte dot products over the row's 16-byte chunks)
      for (int rr = tid; rr < n; rr += NT) {
        unsigned acc = 0;
        for (int c = 0; c < kb; c += 16) {
          const uint4 f = *reinterpret_cast<const uint4*>(F8 + cl_off(rr, c, kb));
          const uint4 d = *reinterpret_cast<const uint4*>(P8 + cl_off(rr, c, kb));
          acc = __dp4a(f.x, d.x, acc); acc = __dp4a(f.y, d.y, acc);
          acc = __dp4a(f.z, d.z, acc); acc = __dp4a(f.w, d.w, acc);
        }
        sv[rr] = make_int4((int)acc, F8[cl_off(rr, rr, kb)], P8[cl_off(rr, rr, kb)], 0);
      }
      fence_proxy_async_smem();   // P8 (generic writes) -> tensor-core reads
      tc_fence_before();
      __syncthreads();
      if (tid == 0) {
        tc_fence_after();
        const uint32_t fa = smem_u32(F8), pa = smem_u32(P8);
        for (int tt = 0; tt < tiles; ++tt) {
          const uint32_t aoff = (uint32_t)(tt * 16) * sbo;   // 128 rows = 16 row groups
          for (int j = 0; j < 2 * ksteps; ++j) {
            const bool lo = j < ksteps;
            const uint32_t ko = (uint32_t)(lo ? j : j - ksteps) * 256;
            const uint64_t ad = umma_smem_desc((lo ? fa : pa) + aoff + ko, 128, sbo);
            const uint64_t bd = umma_smem_desc((lo ? pa : fa) + ko, 128, sbo);
            umma_i8(tmem + (uint32_t)(tt * npad), ad, bd, idesc, j > 0 ? 1u : 0u);
          }
        }
        umma_commit(&bar);
      }
      mbar_wait(&bar, phase);
      phase ^= 1u;
      tc_fence_after();

      // delta(r, s) = 2 (H - G_rr - G_ss) + (2 F_rs - F_rr - F_ss)(2 P_rs - P_rr - P_ss),
      // the dp4a kernel's delta regrouped; a thread walks s upwards, so a
      // strict < keeps the first q of its row
      int bd = INT_MAX, bs = -1;                 // narrow: int32 deltas
      int64_t wbd = INT64_MAX;
      if (rbase < n) {
        const int4 mine = r < n ? sv[r] : make_int4(0, 0, 0, 0);
        const int gdr = mine.x, Frr = mine.y, Prr = mine.z;
        for (int c = h; c < nchunks; c += cs) {
          if (c * 16 + 15 <= rbase) continue;   // whole chunk on or below the diagonal (warp-uniform)
          uint32_t v[16];
          tmem_ld16(trow + (uint32_t)(c * 16), v);
          if (r >= n) continue;
          const uint4 fr = *reinterpret_cast<const uint4*>(F8 + cl_off(r, c * 16, kb));
          const uint4 pr = *reinterpret_cast<const uint4*>(P8 + cl_off(r, c * 16, kb));
          const unsigned fw[4] = {fr.x, fr.y, fr.z, fr.w};
          const unsigned pw[4] = {pr.x, pr.y, pr.z, pr.w};
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int s = c * 16 + j;
            const int4 o = sv[s];
            const int Frs = (int)__byte_perm(fw[j >> 2], 0u, 0x4440 | (j & 3));
            const int Prs = (int)__byte_perm(pw[j >> 2], 0u, 0x4440 | (j & 3));
            const int t = (2 * Frs - Frr - o.y) * (2 * Prs - Prr - o.z);   // |t| < 2^18
            const bool ok = s > r && s < n;
            if (narrow) {
              // n max(F) max(D) < 2^28: H, G and the delta fit int32
              const int dd = 2 * ((int)v[j] - gdr - o.x) + t;
              if (ok && dd < bd) { bd = dd; bs = s; }
            } else {
              const int64_t dd = 2 * ((int64_t)v[j] - gdr - o.x) + t;
              if (ok && dd < wbd) { wbd = dd; bs = s; }
            }
          }
        }
      }
      const int qr = r * n - r * (r + 1) / 2 - r - 1;   // q = qr + s
      int64_t best = bs < 0 ? INT64_MAX : (narrow ? (int64_t)bd : wbd);
      int bq = bs < 0 ? INT_MAX : qr + bs;
      tc_fence_before();
      // lexicographic (delta, q) minimum over the CTA
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const int64_t ob = __shfl_xor_sync(FULL, best, o);
        const int oq = __shfl_xor_sync(FULL, bq, o);
        if (ob < best || (ob == best && oq < bq)) { best = ob; bq = oq; }
      }
      if (lane == 0) { rd[warp] = best; rq[warp] = bq; }
      __syncthreads();
      if (tid == 0) {
        for (int w = 1; w < NT / 32; ++w)
          if (rd[w] < rd[0] || (rd[w] == rd[0] && rq[w] < rq[0])) { rd[0] = rd[w]; rq[0] = rq[w]; }
        s_move = (rq[0] != INT_MAX && rd[0] < 0) ? rq[0] : -1;
      }
      __syncthreads();
      const int mq = s_move;
      if (mq < 0) break;
      cost += (uint64_t)rd[0];
      int r0, s0;
      unrank_pair(mq, n, r0, s0);
      // swap facilities r0 and s0: rows, then columns of P
      for (int j = tid; j < n; j += NT) {
        const int ir = cl_off(r0, j, kb), is = cl_off(s0, j, kb);
        const uint8_t x = P8[ir]; P8[ir] = P8[is]; P8[is] = x;
      }
      __syncthreads();
      for (int i = tid; i < n; i += NT) {
        const int ir = cl_off(i, r0, kb), is = cl_off(i, s0, kb);
        const uint8_t x = P8[ir]; P8[ir] = P8[is]; P8[is] = x;
      }
      if (tid == 0) { const int x = sp[r0]; sp[r0] = sp[s0]; sp[s0] = x; }
    }
    __syncthreads();
    for (int i = tid; i < n; i += NT) a.perm[p * n + i] = (int16_t)sp[i];
    if (a.do_pbest) {
      if (tid == 0) {
        const bool imp = (int64_t)cost < a.pl_cost[p];
        if (imp) a.pl_cost[p] = (int64_t)cost;
        a.improved[p] = imp ? 1 : 0;
        s_move = imp;
      }
      __syncthreads();
      if (s_move)
        for (int i = tid; i < n; i += NT) a.pl_perm[p * n + i] = (int16_t)sp[i];
    }
    if (tid == 0) a.cost[p] = (int64_t)cost;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(g.tcols) : "memory");
  }
}


// ---------------------------------------------------------------------------
// Pipelined tensor-core 2-opt, one pass, 128 < n <= 256 (config 5).
//
// twoopt_tc_kernel above runs P-build -> MMA -> epilogue of one particle
// after the other in one CTA, so the tensor core idles while the CTA builds
// P = D[p][p] and scores the swaps, and the scalar pipes idle during the
// MMA.  Here the roles are warp-specialised and consecutive particles
// overlap:
//   * 4 builder warps gather P = D[p][p] of the NEXT particle from D in
//     shared memory into the (single) shared P buffer, with G[r][r], F_rr,
//     P_rr per row;
//   * one builder lane issues the particle's MMAs and then copies P into
//     tensor memory (tcgen05.cp), so the P buffer is free for the next
//     particle as soon as the tensor core is done with it;
//   * 12 epilogue warps score the swaps from TMEM (H and the P copy) and F
//     in shared memory, and apply the best move.
// H is symmetric and only s > r is read: row tile 0 (r < 128) needs columns
// 0..npad-1, row tile 1 (r >= 128) only columns 128..npad-1, so the MMAs are
// M = 128 x N = npad and M = 128 x N = npad - 128 (3/4 of the full GEMM)
// into TMEM columns [0, 2 npad - 128) <= 384; the P copy takes columns
// 384..511 (row r at lane r mod 128, 64 columns per 128-row tile).
// Epilogue warps are spread over the four TMEM lane quarters 4 / 3 / 3 / 2
// because low rows have more s > r.  Bit-identical to twoopt_tc_kernel.
// Barriers (CTA mbarriers): full[b] (builders -> MMA issuer and epilogue:
// P, sv[b], sp[b] written), mma0 / mma_done (tile-0 / tile-1 MMA + copy
// commits -> epilogue; mma_done also -> builders: P readable again),
// hfree0 / hfree (epilogue done with tile 0's / tile 1's H columns and P
// copy: the next particle's tile-0 MMA overlaps this particle's tile-1
// scoring and reduction, its tile-1 MMA the tile-0 scoring of the
// particle before), bfree[b] (epilogue done with sv[b], sp[b]).
constexpr int TCP_NT = 768;          // 24 warps, 80 registers each
constexpr int TCP_EPI = 16;          // epilogue warps
constexpr int TCP_BLD = 8;           // builder warps (warp 15 issues the MMAs)
constexpr uint32_t TCP_PCOL = 384;   // TMEM column of the P copy
// warp w: TMEM lane quarter q = w & 3, index jq = w >> 2 within the quarter
// (six per quarter).  The first TCP_EQ[q] of a quarter score swaps (5 / 4 /
// 4 / 3: low rows have more s > r), the rest build: warps 15, 17 .. 23.
__host__ __device__ constexpr int tcp_eq(int q) { return q == 0 ? 5 : q == 3 ? 3 : 4; }

struct TwoOptTcp {
  int kb, npad;
  unsigned sleep_epi, sleep_bld;   // ns parked between polls (epilogue / builder waits)
  int ts;                          // 1: second MMA half with A = the P copy in TMEM
  // D row stride in bytes: an odd number of 4-byte words, so 32 consecutive
  // D rows read at one column fall into 32 distinct banks
  static __host__ __device__ int dstride(int n) { return (((n + 3) / 4) | 1) * 4; }
  static __host__ __device__ size_t smem_bytes(int n, int kb) {
    return 2 * (size_t)256 * kb + align_up((size_t)n * dstride(n), 16) + 2 * 256 * 16 + 2 * 256 * 2 +
           2 * 256 * 2 + 2 * TCP_EPI * 16 + 2 * 256 * 4;
  }
};

// one lane of a converged warp (elect.sync): issues a single-thread
// tcgen05 instruction while the operands stay warp-uniform
__device__ __forceinline__ bool elect_one() {
  uint32_t e;
  asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}\n" : "=r"(e));
  return e != 0;
}

__device__ __forceinline__ void mbar_arrive1(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}

// mbarrier wait that parks the warp (try_wait with a suspend-time hint, so
// waiting warps do not steal issue slots from the working roles), with a
// deadlock guard: a launch error (trap) instead of a hung GPU after 2^24
// unsuccessful polls (each followed by a 64 ns sleep)
__device__ __forceinline__ void mbar_wait_guard(uint64_t* bar, uint32_t parity, unsigned sleep_ns = 128) {
  const uint32_t a = smem_u32(bar);
#pragma unroll 1
  for (uint32_t spins = 0;; ++spins) {
    uint32_t ok;
    asm volatile("{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n"
                 "selp.u32 %0, 1, 0, P1;\n}\n" : "=r"(ok) : "r"(a), "r"(parity), "r"(1000u) : "memory");
    if (ok) return;
    __nanosleep(sleep_ns);  // a parked warp issues nothing (try_wait alone returned after ~100 cycles)
    if (spins > (1u << 24)) __trap();
  }
}

// 128 rows x 32 bytes of a canonical K-major operand -> TMEM lanes 0..127,
// 8 columns
__device__ __forceinline__ void tmem_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" :: "r"(taddr), "l"(sdesc) : "memory");
}

#ifdef QSB_TCP_TIMING
// diagnosis build: clock64 stamps of the pipeline events of CTA 0's first
// 64 particles (read with qsb_debug_tcp_stamps)
__device__ long long qsb_tcp_ts[64][10];
#define TCP_TS(i, k) do { if (blockIdx.x == 0 && (i) < 64) qsb_tcp_ts[(i)][(k)] = clock64(); } while (0)
#else
#define TCP_TS(i, k) do { } while (0)
#endif

// One row tile's MMAs (H += F P^T over K steps, then P F^T) and the P copy
// into TMEM, issued by one elected lane of a converged warp.  KS K steps of
// 32 bytes; a K step is +16 in a no-swizzle descriptor's address field.
// A operand from tensor memory (the P copy, row r at lane r mod 128, 8
// columns per 32-byte K step), B from shared memory
__device__ __forceinline__ void umma_i8_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n"
      :: "r"(d_tmem), "r"(a_tmem), "l"(b), "r"(idesc), "r"(accumulate) : "memory");
}

// Split issue (TS mode): H = F P^T from shared memory plus the P copy first
// (after which the P buffer is free for the next particle's builders), then
// H += P F^T with P read back from tensor memory.
template <int KS>
__device__ __forceinline__ void tcp_issue_fp(uint32_t dt, uint64_t f0, uint64_t p0, uint32_t idd, uint32_t pcol) {
  if (elect_one()) {
#pragma unroll
    for (int j = 0; j < KS; ++j) umma_i8(dt, f0 + 16 * j, p0 + 16 * j, idd, j > 0 ? 1u : 0u);
#pragma unroll
    for (int k = 0; k < KS; ++k) tmem_cp_128x256b(pcol + 8 * k, p0 + 16 * k);
  }
  __syncwarp();
}
template <int KS>
__device__ __forceinline__ void tcp_issue_pf(uint32_t dt, uint32_t pcol, uint64_t f0, uint32_t idd) {
  if (elect_one()) {
#pragma unroll
    for (int j = 0; j < KS; ++j) umma_i8_ts(dt, pcol + 8 * j, f0 + 16 * j, idd, 1u);
  }
  __syncwarp();
}

template <int KS>
__device__ __forceinline__ void tcp_issue_tile(uint32_t dt, uint64_t f0, uint64_t p0, uint32_t idd,
                                               uint32_t pcol) {
  if (elect_one()) {
#pragma unroll
    for (int j = 0; j < KS; ++j) umma_i8(dt, f0 + 16 * j, p0 + 16 * j, idd, j > 0 ? 1u : 0u);
#pragma unroll
    for (int j = 0; j < KS; ++j) umma_i8(dt, p0 + 16 * j, f0 + 16 * j, idd, 1u);
    // the epilogue's copy of P: 32 bytes (8 columns) of 128 rows per copy
#pragma unroll
    for (int k = 0; k < KS; ++k) tmem_cp_128x256b(pcol + 8 * k, p0 + 16 * k);
  }
  __syncwarp();
}

__global__ void __launch_bounds__(TCP_NT, 1) twoopt_tcp_kernel(const TwoOptArgs a, const TwoOptTcp g) {
  extern __shared__ __align__(1024) unsigned char tsm[];
  const int n = a.n, kb = g.kb, npad = g.npad;
  const size_t mb = (size_t)256 * kb;
  const int dn = TwoOptTcp::dstride(n);
  uint8_t* F8 = tsm;                                          // canonical layout, 256 rows
  uint8_t* P8 = F8 + mb;                                      // P = D[p][p], same layout
  uint8_t* D8 = P8 + mb;                                      // D row-major, stride dn
  int4* svb = reinterpret_cast<int4*>(D8 + align_up((size_t)n * dn, 16));   // [2][256] {G_rr, F_rr, P_rr, 0}
  int16_t* spb = reinterpret_cast<int16_t*>(svb + 512);      // [2][256] the particle's perm
  int16_t* pinvb = spb + 512;                                 // [2][256] inverse perm (builders)
  int64_t* redd = reinterpret_cast<int64_t*>(pinvb + 512);   // [2][TCP_EPI]
  int* redq = reinterpret_cast<int*>(redd + 2 * TCP_EPI);    // [2][TCP_EPI]
  int* spwb = redq + 2 * TCP_EPI;                             // [2][256] the perm as words (builders)
  __shared__ __align__(8) uint64_t full[2], bfree[2], mma0, mma_done, hfree0, hfree, pfree;
  __shared__ uint32_t s_tmem;
  __shared__ unsigned s_mx[2];
  __shared__ unsigned s_arr[2];   // epilogue warps done with particle idx (buffer b)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint16_t* gF = reinterpret_cast<const uint16_t*>(a.F);
  const uint16_t* gD = reinterpret_cast<const uint16_t*>(a.D);

  // ---- prologue: zero the operands, F (canonical) and D (row-major) as bytes
  if (tid < 2) { s_mx[tid] = 0; s_arr[tid] = 0; }
  {
    uint4* z = reinterpret_cast<uint4*>(F8);
    const int nz = (int)(2 * mb / 16);
    for (int i = tid; i < nz; i += TCP_NT) z[i] = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  unsigned mf = 0, md = 0;
  if ((n & 7) == 0) {
    const int cw = n >> 3;                  // 8-entry chunks per row (16-byte loads)
    for (int e = tid; e < n * cw; e += TCP_NT) {
      const int r = e / cw, c = e - r * cw;
      const uint4 f = *reinterpret_cast<const uint4*>(gF + (size_t)r * n + 8 * c);
      const uint4 d = *reinterpret_cast<const uint4*>(gD + (size_t)r * n + 8 * c);
      *reinterpret_cast<uint2*>(F8 + cl_off(r, 8 * c, kb)) =
          make_uint2(__byte_perm(f.x, f.y, 0x6420), __byte_perm(f.z, f.w, 0x6420));
      const uint32_t dl = __byte_perm(d.x, d.y, 0x6420), dh = __byte_perm(d.z, d.w, 0x6420);
      uint8_t* drow = D8 + r * dn + 8 * c;  // stride n + 1: byte stores
#pragma unroll
      for (int x = 0; x < 4; ++x) { drow[x] = (uint8_t)(dl >> (8 * x)); drow[4 + x] = (uint8_t)(dh >> (8 * x)); }
      const uint32_t fm = __vmaxu2(__vmaxu2(f.x, f.y), __vmaxu2(f.z, f.w));
      const uint32_t dm = __vmaxu2(__vmaxu2(d.x, d.y), __vmaxu2(d.z, d.w));
      mf = max(mf, max(fm & 0xffffu, fm >> 16));
      md = max(md, max(dm & 0xffffu, dm >> 16));
    }
  } else {
    for (int e = tid; e < n * n; e += TCP_NT) {
      const int r = e / n, c = e - r * n;
      F8[cl_off(r, c, kb)] = (uint8_t)gF[e];
      D8[r * dn + c] = (uint8_t)gD[e];
      mf = max(mf, (unsigned)gF[e]);
      md = max(md, (unsigned)gD[e]);
    }
  }
  mf = __reduce_max_sync(FULL, mf);
  md = __reduce_max_sync(FULL, md);
  if (lane == 0) { atomicMax(&s_mx[0], mf); atomicMax(&s_mx[1], md); }
  if (tid == 0) {
    mbar_init(&full[0], TCP_BLD); mbar_init(&full[1], TCP_BLD);
    mbar_init(&bfree[0], 1); mbar_init(&bfree[1], 1);
    mbar_init(&mma0, 1); mbar_init(&mma_done, 1); mbar_init(&pfree, 1);
    mbar_init(&hfree0, TCP_EPI); mbar_init(&hfree, TCP_EPI);
    mbar_fence_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32(&s_tmem)), "r"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_proxy_async_smem();     // F8 / zeroed P (generic writes) -> tensor-core reads
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  const bool narrow = (double)n * (double)s_mx[0] * (double)s_mx[1] < 268435456.0;
  const int nch = npad >> 4;
  // PDL: the prologue above overlaps the step kernel's launch tail; the
  // particles' positions and costs are read after it completes
  pdl_wait();
  pdl_launch();   // the best update may be placed meanwhile (it waits on this grid)

  if ((warp >> 2) >= tcp_eq(warp & 3)) {
    // =========================== builders (+ the MMA issuer, warp 15 lane 0)
    const int bt = (warp == 15 ? 0 : warp - 16) * 32 + lane;   // builder thread 0..255
    const uint32_t sbo = (uint32_t)kb * 8;
    const int ksteps = kb / 32;
    const uint32_t id0 = umma_idesc_u8(128, npad), id1 = umma_idesc_u8(128, npad - 128);
    const int nck = kb >> 4;                 // 16-byte chunks per row (<= 16)
    int idx = 0;
    for (int64_t p = blockIdx.x; p < a.P; p += gridDim.x, ++idx) {
      const int b = idx & 1;
      int16_t* sp = spb + 256 * b;
      int16_t* pinv = pinvb + 256 * b;      // double-buffered: a fast builder thread may
                                            // start the next particle while others still read
      int4* sv = svb + 256 * b;
      int* spw = spwb + 256 * b;
      if (idx >= 2) mbar_wait_guard(&bfree[b], ((idx >> 1) - 1) & 1, g.sleep_bld);    // sv[b], sp[b] free
      for (int i = bt; i < n; i += TCP_BLD * 32) {
        const int16_t v = a.perm[p * n + i];
        sp[i] = v;
        spw[i] = v;
        pinv[v] = (int16_t)i;
      }
      if (idx >= 1) mbar_wait_guard(&pfree, (idx - 1) & 1, g.sleep_bld);   // P read by MMA + copy
      asm volatile("bar.sync 2, %0;" :: "r"(TCP_BLD * 32) : "memory");
      if (bt == 0) TCP_TS(idx, 0);
      // P[i] = D[p_i][p] built by SOURCE row: thread d owns D row d, i.e.
      // P row i = pinv[d], and the warp's 32 consecutive D rows read column
      // p_j in 32 distinct banks (odd word stride).  G[i][i] = F[i] . P[i]
      // and P_ii come out of the same pass.
      // the thread's D rows d = bt (+ 32 TCP_BLD ...), interleaved chunk by chunk
      {
        constexpr int NR = (256 + TCP_BLD * 32 - 1) / (TCP_BLD * 32);
        int dr[NR], ir[NR];
        const uint8_t* drow[NR];
        unsigned acc[NR], pii[NR];
#pragma unroll
        for (int h = 0; h < NR; ++h) {
          dr[h] = bt + h * TCP_BLD * 32;
          ir[h] = dr[h] < n ? pinv[dr[h]] : 0;
          drow[h] = D8 + (dr[h] < n ? dr[h] : 0) * dn;
          acc[h] = 0;
          pii[h] = dr[h] < n ? drow[h][dr[h]] : 0u;   // P_ii = D[p_i][p_i], p_i = d
        }
        // full chunks: the 16 column indices as words (four broadcast
        // loads), one add and one byte load per entry, no bounds tests
        const int nfull = n >> 4;
#pragma unroll 1
        for (int c = 0; c < nfull; ++c) {
          const int4* q4 = reinterpret_cast<const int4*>(spw + 16 * c);
          int pj[16];
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            const int4 qq = q4[x];
            pj[4 * x] = qq.x; pj[4 * x + 1] = qq.y; pj[4 * x + 2] = qq.z; pj[4 * x + 3] = qq.w;
          }
#pragma unroll
          for (int h = 0; h < NR; ++h) {
            unsigned bb[16];
#pragma unroll
            for (int y = 0; y < 16; ++y) bb[y] = drow[h][pj[y]];
            unsigned w[4];
#pragma unroll
            for (int x = 0; x < 4; ++x)
              w[x] = __byte_perm(__byte_perm(bb[4 * x], bb[4 * x + 1], 0x0040),
                                 __byte_perm(bb[4 * x + 2], bb[4 * x + 3], 0x0040), 0x5410);
            if (dr[h] >= n) continue;
            const int i = ir[h];
            *reinterpret_cast<uint4*>(P8 + cl_off(i, 16 * c, kb)) = make_uint4(w[0], w[1], w[2], w[3]);
            const uint4 f = *reinterpret_cast<const uint4*>(F8 + cl_off(i, 16 * c, kb));
            acc[h] = __dp4a(f.x, w[0], acc[h]); acc[h] = __dp4a(f.y, w[1], acc[h]);
            acc[h] = __dp4a(f.z, w[2], acc[h]); acc[h] = __dp4a(f.w, w[3], acc[h]);
          }
        }
        // the partial chunk and the zero padding up to kb
#pragma unroll 1
        for (int c = nfull; c < nck; ++c) {
          const uint4 i0 = *reinterpret_cast<const uint4*>(sp + 16 * c);       // p_j, j = 16c .. 16c+7
          const uint4 i1 = *reinterpret_cast<const uint4*>(sp + 16 * c + 8);   // (broadcast loads)
          const unsigned iw[8] = {i0.x, i0.y, i0.z, i0.w, i1.x, i1.y, i1.z, i1.w};
          unsigned w[NR][4];
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            unsigned bb[NR][4];
#pragma unroll
            for (int y = 0; y < 4; ++y) {
              const int j = 16 * c + 4 * x + y;
              const unsigned pj = (iw[(4 * x + y) >> 1] >> (16 * (y & 1))) & 0xffffu;
#pragma unroll
              for (int h = 0; h < NR; ++h) bb[h][y] = j < n ? (unsigned)drow[h][pj] : 0u;
            }
#pragma unroll
            for (int h = 0; h < NR; ++h)
              w[h][x] = __byte_perm(__byte_perm(bb[h][0], bb[h][1], 0x0040),
                                    __byte_perm(bb[h][2], bb[h][3], 0x0040), 0x5410);
          }
#pragma unroll
          for (int h = 0; h < NR; ++h) {
            if (dr[h] >= n) continue;
            const int i = ir[h];
            *reinterpret_cast<uint4*>(P8 + cl_off(i, 16 * c, kb)) = make_uint4(w[h][0], w[h][1], w[h][2], w[h][3]);
            const uint4 f = *reinterpret_cast<const uint4*>(F8 + cl_off(i, 16 * c, kb));
            acc[h] = __dp4a(f.x, w[h][0], acc[h]); acc[h] = __dp4a(f.y, w[h][1], acc[h]);
            acc[h] = __dp4a(f.z, w[h][2], acc[h]); acc[h] = __dp4a(f.w, w[h][3], acc[h]);
          }
        }
#pragma unroll
        for (int h = 0; h < NR; ++h)
          if (dr[h] < n) sv[ir[h]] = make_int4((int)acc[h], F8[cl_off(ir[h], ir[h], kb)], (int)pii[h], 2 * (int)acc[h]);
      }
      if (bt == 0) TCP_TS(idx, 1);
      fence_proxy_async_smem();                    // P (generic writes) -> tensor-core reads
      __syncwarp();
      if (lane == 0) mbar_arrive1(&full[b]);
      if (warp == 15) {
        // the whole warp runs the issue loop (warp-uniform descriptors stay
        // in uniform registers); one elected lane issues each instruction
        {
          if (lane == 0) TCP_TS(idx, 2);
          mbar_wait_guard(&full[b], (idx >> 1) & 1);
          if (lane == 0) TCP_TS(idx, 3);
          // descriptors of F and P at the tile's row offset; a K step of 32
          // bytes is 2 core matrices = +16 in the descriptor's address field
          // (no carry: shared addresses stay below 2^18), so each MMA is one
          // add and the instruction
          const uint64_t dF = umma_smem_desc(smem_u32(F8), 128, sbo);
          const uint64_t dP = umma_smem_desc(smem_u32(P8), 128, sbo);
          // tile 0: rows 0..127 x columns 0..npad-1; tile 1: rows 128.. x columns 128..
          if (g.ts) {
            // per tile: F P^T and the P copy, then P F^T with P read from
            // tensor memory; the P buffer is released after tile 1's F P^T
            // and copy, so the builders overlap tile 1's P F^T
            const uint32_t pc0 = tmem + TCP_PCOL, pc1 = pc0 + 64;
            const uint32_t dt0 = tmem, dt1 = tmem + (uint32_t)npad;
            const uint64_t f1 = dF + (uint64_t)sbo, p1 = dP + (uint64_t)sbo;   // row 128: (16 sbo) >> 4
#define TCP_KS(fn, args) switch (ksteps) { case 5: fn<5> args; break; case 6: fn<6> args; break; \
                                           case 7: fn<7> args; break; default: fn<8> args; break; }
            if (idx >= 1) mbar_wait_guard(&hfree0, (idx - 1) & 1);
            if (lane == 0) TCP_TS(idx, 4);
            tc_fence_after();
            TCP_KS(tcp_issue_fp, (dt0, dF, dP, id0, pc0));
            TCP_KS(tcp_issue_pf, (dt0, pc0, dF, id0));
            if (elect_one()) umma_commit(&mma0);
            __syncwarp();
            if (idx >= 1) mbar_wait_guard(&hfree, (idx - 1) & 1);
            tc_fence_after();
            TCP_KS(tcp_issue_fp, (dt1, f1, p1, id1, pc1));
            if (elect_one()) umma_commit(&pfree);
            __syncwarp();
            TCP_KS(tcp_issue_pf, (dt1, pc1, f1, id1));
            if (elect_one()) umma_commit(&mma_done);
            __syncwarp();
#undef TCP_KS
          } else {
#pragma unroll 1
          for (int tt = 0; tt < 2; ++tt) {
            // the tile's H columns and P copy drained by the previous particle
            if (idx >= 1) mbar_wait_guard(tt ? &hfree : &hfree0, (idx - 1) & 1);
            if (tt == 0 && lane == 0) TCP_TS(idx, 4);
            tc_fence_after();
            const uint64_t offd = (uint64_t)(tt * sbo);          // (16 sbo bytes) >> 4
            const uint64_t f0 = dF + offd, p0 = dP + offd;
            const uint32_t dt = tmem + (uint32_t)(tt * npad), idd = tt ? id1 : id0;
            const uint32_t pc = tmem + TCP_PCOL + (uint32_t)(64 * tt);
            switch (ksteps) {   // kb = 160 .. 256: fully unrolled issue sequences
              case 5: tcp_issue_tile<5>(dt, f0, p0, idd, pc); break;
              case 6: tcp_issue_tile<6>(dt, f0, p0, idd, pc); break;
              case 7: tcp_issue_tile<7>(dt, f0, p0, idd, pc); break;
              default: tcp_issue_tile<8>(dt, f0, p0, idd, pc); break;
            }
            if (elect_one()) umma_commit(tt ? &mma_done : &mma0);
            if (tt && elect_one()) umma_commit(&pfree);
            __syncwarp();
          }
          }
          if (lane == 0) TCP_TS(idx, 5);
        }
        __syncwarp();
      }
    }
  } else {
    // =========================== epilogue warps
    const int q = warp & 3;                 // TMEM lane quarter
    const int jw = warp >> 2;               // index among this quarter's epilogue warps
    const int Wq = tcp_eq(q);
    const int e = warp < 15 ? warp : 15;    // epilogue index (warp 16 -> 15)
    const int r0 = 32 * q + lane, r1 = 128 + r0;
    const int len0 = max(0, nch - 2 * q);                                // tile-0 chunks c >= 2q
    const int len1 = (128 + 32 * q < n) ? max(0, nch - 8 - 2 * q) : 0;   // tile-1 chunks c >= 8 + 2q
    const uint32_t tl = tmem + ((uint32_t)(32 * q) << 16);
    const int qr0 = r0 * n - r0 * (r0 + 1) / 2 - r0 - 1;
    const int qr1 = r1 * n - r1 * (r1 + 1) / 2 - r1 - 1;
    int idx = 0;
    for (int64_t p = blockIdx.x; p < a.P; p += gridDim.x, ++idx) {
      const int b = idx & 1;
      mbar_wait_guard(&full[b], (idx >> 1) & 1, g.sleep_epi);
      mbar_wait_guard(&mma0, idx & 1, g.sleep_epi);
      tc_fence_after();
      if (lane == 0 && warp == 0) TCP_TS(idx, 6);
      const int4* sv = svb + 256 * b;
      // a thread visits its pairs in increasing q (tile-0 row before its
      // tile-1 row, chunks ascending), so a strict < keeps the first q of
      // equal deltas
      int bd = INT_MAX, bs = INT_MAX;                 // narrow: int32 deltas, bs = q index
      int64_t wbd = INT64_MAX;
      // TMEM loads run one chunk ahead of the scoring (two register sets;
      // tcgen05.wait::ld names the registers, so no use moves above it)
      const int L = len0 + len1;
      auto issue = [&](int k, uint32_t (&v)[16], uint32_t (&pw)[4]) {
        const bool t1 = k >= len0;
        const int c = t1 ? 8 + 2 * q + (k - len0) : 2 * q + k;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(tl + (uint32_t)(t1 ? npad + (c - 8) * 16 : c * 16)));
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(pw[0]), "=r"(pw[1]), "=r"(pw[2]), "=r"(pw[3])
                     : "r"(tl + TCP_PCOL + (uint32_t)((t1 ? 64 : 0) + 4 * c)));
      };
      auto wait = [&](uint32_t (&v)[16], uint32_t (&pw)[4]) {
        asm volatile("tcgen05.wait::ld.sync.aligned;"
                     : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]),
                       "+r"(v[7]), "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]),
                       "+r"(v[14]), "+r"(v[15]), "+r"(pw[0]), "+r"(pw[1]), "+r"(pw[2]), "+r"(pw[3])
                     :: "memory");
      };
      auto score = [&](int k, const uint32_t (&v)[16], const uint32_t (&pw)[4]) {
        const bool t1 = k >= len0;
        const int c = t1 ? 8 + 2 * q + (k - len0) : 2 * q + k;
        const int r = t1 ? r1 : r0;
        if (r >= n) return;
        const int4 mine = sv[r];
        const int gdr = mine.x, Frr = mine.y, Prr = mine.z;
        const uint4 fr = *reinterpret_cast<const uint4*>(F8 + cl_off(r, c * 16, kb));
        const unsigned fw[4] = {fr.x, fr.y, fr.z, fr.w};
        const int qr = t1 ? qr1 : qr0;
        // chunks strictly right of the warp's rows and inside n (warp-
        // uniform): no pair tests, and the row's -2 G_rr is added once per
        // chunk (it does not change the argmin within the row), so a pair is
        // d = (2 H - 2 G_ss) + t; the chunk's first minimum then competes
        // with the running best under the same strict <
        if (narrow && 16 * c >= 32 * q + 32 + (t1 ? 128 : 0) && 16 * c + 16 <= n) {
          int cb = INT_MAX, cj = 0;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int4 o = sv[c * 16 + j];
            const int Frs = (int)__byte_perm(fw[j >> 2], 0u, 0x4440 | (j & 3));
            const int Prs = (int)__byte_perm(pw[j >> 2], 0u, 0x4440 | (j & 3));
            const int t = (2 * Frs - Frr - o.y) * (2 * Prs - Prr - o.z);
            const int d = ((int)v[j] + (int)v[j] - o.w) + t;
            if (d < cb) { cb = d; cj = j; }
          }
          const int dd = cb - 2 * gdr;
          if (dd < bd) { bd = dd; bs = qr + c * 16 + cj; }
          return;
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int s = c * 16 + j;
          const int4 o = sv[s];
          const int Frs = (int)__byte_perm(fw[j >> 2], 0u, 0x4440 | (j & 3));
          const int Prs = (int)__byte_perm(pw[j >> 2], 0u, 0x4440 | (j & 3));
          const int t = (2 * Frs - Frr - o.y) * (2 * Prs - Prr - o.z);   // |t| < 2^18
          const bool ok = s > r && s < n;
          if (narrow) {
            const int dd = 2 * ((int)v[j] - gdr - o.x) + t;
            if (ok && dd < bd) { bd = dd; bs = qr + s; }
          } else {
            const int64_t dd = 2 * ((int64_t)v[j] - gdr - o.x) + t;
            if (ok && dd < wbd) { wbd = dd; bs = qr + s; }
          }
        }
      };
      // tile 1's MMA is awaited before the warp's first tile-1 load; tile
      // 0's region is released after the wait of its last tile-0 load
      bool have1 = false, rel0 = false;
      auto need = [&](int kk) {
        if (kk >= len0 && !have1) {
          mbar_wait_guard(&mma_done, idx & 1);
          tc_fence_after();
          have1 = true;
        }
      };
      auto release0 = [&]() {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive1(&hfree0);
        rel0 = true;
      };
      uint32_t va[16], pa[4], vb[16], pb[4];
      int k = jw;
      if (k < L) { need(k); issue(k, va, pa); }
      while (k < L) {
        wait(va, pa);
        const int k2 = k + Wq;
        if (!rel0 && k2 >= len0) release0();
        if (k2 < L) { need(k2); issue(k2, vb, pb); }
        score(k, va, pa);
        if (k2 >= L) break;
        wait(vb, pb);
        const int k3 = k2 + Wq;
        if (!rel0 && k3 >= len0) release0();
        if (k3 < L) { need(k3); issue(k3, va, pa); }
        score(k2, vb, pb);
        k = k3;
      }
      if (!rel0) release0();
      // H and the P copy drained: the next particle's MMAs may overwrite them
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive1(&hfree);
      if (lane == 0 && warp == 0) TCP_TS(idx, 7);
      if (lane == 0 && warp == 3) TCP_TS(idx, 8);
      int64_t best = bs == INT_MAX ? INT64_MAX : (narrow ? (int64_t)bd : wbd);
      int bq = bs;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const int64_t ob = __shfl_xor_sync(FULL, best, o);
        const int oq = __shfl_xor_sync(FULL, bq, o);
        if (ob < best || (ob == best && oq < bq)) { best = ob; bq = oq; }
      }
      // the last epilogue warp to finish the particle reduces the sixteen
      // minima and applies the move; the others go on to the next particle
      unsigned arr = 0;
      if (lane == 0) {
        redd[TCP_EPI * b + e] = best;
        redq[TCP_EPI * b + e] = bq;
        __threadfence_block();
        arr = atomicAdd(&s_arr[b], 1u);
      }
      arr = __shfl_sync(FULL, arr, 0);
      if (arr == TCP_EPI - 1) {
        __threadfence_block();
        // (s_arr[b] is next used at particle idx + 2, whose sv[b] the
        // builders write only after this warp's bfree[b] arrival)
        if (lane == 0) s_arr[b] = 0;
        const int64_t cost0 = a.cost[p];
        const int64_t pl0 = a.do_pbest ? a.pl_cost[p] : 0;
        best = lane < TCP_EPI ? redd[TCP_EPI * b + lane] : INT64_MAX;
        bq = lane < TCP_EPI ? redq[TCP_EPI * b + lane] : INT_MAX;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          const int64_t ob = __shfl_xor_sync(FULL, best, o);
          const int oq = __shfl_xor_sync(FULL, bq, o);
          if (ob < best || (ob == best && oq < bq)) { best = ob; bq = oq; }
        }
        const bool move = bq != INT_MAX && best < 0;
        int rs = -1, ss = -1;
        if (move) unrank_pair(bq, n, rs, ss);
        const int64_t cost = cost0 + (move ? best : 0);
        const int16_t* sp = spb + 256 * b;
        const bool imp = a.do_pbest && cost < pl0;
        for (int et = lane; et < n; et += 32) {
          const int src = et == rs ? ss : (et == ss ? rs : et);
          const int16_t val = sp[src];
          a.perm[p * n + et] = val;
          if (imp) a.pl_perm[p * n + et] = val;
        }
        if (lane == 0) {
          a.cost[p] = cost;
          if (a.do_pbest) {
            if (imp) a.pl_cost[p] = cost;
            a.improved[p] = imp ? 1 : 0;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive1(&bfree[b]);
        if (lane == 0) TCP_TS(idx, 9);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(512) : "memory");
  }
}


// Small instances (n <= 32): four particles per CTA, one warp each, share
// one MMA batch.  Rows 32 w .. 32 w + 31 of the stacked operands belong to
// warp w's particle, so
//   H_stack = [F_4 | P_stack] [P_stack | F_4]^T      (M = N = 128, K = 64)
// holds every particle's H as a diagonal 32 x 32 block (the off-diagonal
// blocks are computed and ignored: the tensor core is not the bottleneck
// here, the per-particle round trips are).  Warp w reads TMEM lanes
// 32 w .. 32 w + 31 (its lane quarter), columns 32 w .. 32 w + 31, scores
// its particle's swaps and applies its move itself; the CTA repeats the
// MMA while any of its particles still moved and passes remain.
template <int NT>
__global__ void __launch_bounds__(NT) twoopt_tc4_kernel(const TwoOptArgs a) {
  static_assert(NT == 128, "one warp per particle, four particles per CTA");
  constexpr int KB = 32, ROWS = 128;
  extern __shared__ __align__(1024) unsigned char tsm[];
  const int n = a.n;
  const int dn = n + 1;
  uint8_t* F8 = tsm;                         // 4 stacked copies of F (canonical layout)
  uint8_t* P8 = F8 + ROWS * KB;              // the 4 particles' P = D[p][p]
  uint8_t* D8 = P8 + ROWS * KB;              // D row-major, stride n + 1, column n zero
  int* spall = reinterpret_cast<int*>(D8 + align_up((size_t)n * dn, 16));   // [4][32]
  int4* svall = reinterpret_cast<int4*>(spall + 128);                          // [4][32]
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t s_tmem;
  __shared__ unsigned s_mx[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint16_t* gF = reinterpret_cast<const uint16_t*>(a.F);
  const uint16_t* gD = reinterpret_cast<const uint16_t*>(a.D);
  int* sp = spall + 32 * warp;
  int4* sv = svall + 32 * warp;

  if (tid < 2) s_mx[tid] = 0;
  {
    uint4* z = reinterpret_cast<uint4*>(F8);
    for (int i = tid; i < 2 * ROWS * KB / 16; i += NT) z[i] = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  unsigned mf = 0, md = 0;
  // a warp per row, a lane per column (n <= 32): no index division
  for (int r = warp; r < n; r += NT / 32) {
    if (lane < n) {
      const unsigned f = gF[r * n + lane], d = gD[r * n + lane];
#pragma unroll
      for (int w = 0; w < 4; ++w) F8[cl_off(32 * w + r, lane, KB)] = (uint8_t)f;
      D8[r * dn + lane] = (uint8_t)d;
      mf = max(mf, f);
      md = max(md, d);
    }
  }
  for (int r = tid; r < n; r += NT) D8[r * dn + n] = 0;
  atomicMax(&s_mx[0], mf);
  atomicMax(&s_mx[1], md);
  if (tid == 0) { mbar_init(&bar, 1); mbar_fence_init(); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32(&s_tmem)), "r"(128) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  const uint32_t idesc = umma_idesc_u8(ROWS, ROWS);
  const bool narrow = (double)n * (double)s_mx[0] * (double)s_mx[1] < 268435456.0;
  const uint32_t trow = tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)(32 * warp);
  const int r = lane;                        // this lane's facility (row)
  uint32_t phase = 0;

  // PDL: the prologue above (F, D, TMEM) overlaps the step kernel's launch
  // tail; the particles' positions and costs are read after it completes
  pdl_wait();
  pdl_launch();   // the best update may be placed meanwhile (it waits on this grid)
  // the next group's permutation entry and cost are loaded one round ahead
  const int64_t gstride = (int64_t)gridDim.x * 4;
  int nperm = 0;
  int64_t ncost = 0, npl = 0;
  {
    const int64_t p0 = (int64_t)blockIdx.x * 4 + warp;
    if (p0 < a.P) {
      if (lane < n) nperm = a.perm[p0 * n + lane];
      ncost = a.cost[p0];
      if (a.do_pbest) npl = a.pl_cost[p0];
    }
  }
  for (int64_t base = (int64_t)blockIdx.x * 4; base < a.P; base += gstride) {
    const int64_t p = base + warp;
    const bool valid = p < a.P;
    const int myperm = nperm;
    uint64_t cost = valid ? (uint64_t)ncost : 0;
    const int64_t mypl = npl;
    {
      const int64_t pn = p + gstride;
      if (pn < a.P) {
        if (lane < n) nperm = a.perm[pn * n + lane];
        ncost = a.cost[pn];
        if (a.do_pbest) npl = a.pl_cost[pn];
      }
    }
    __syncwarp();
    sp[lane] = myperm;
    __syncwarp();
    {
      // row r of this particle's P: bytes j < n gathered (column index from
      // lane j's register; j >= n and rows r >= n read D's zero column n)
      unsigned w[8];
      const uint8_t* drow = D8 + (r < n ? myperm : 0) * dn;
#pragma unroll
      for (int x = 0; x < 8; ++x) {
        unsigned b[4];
#pragma unroll
        for (int y = 0; y < 4; ++y) {
          const int j = 4 * x + y;
          const int pj = __shfl_sync(FULL, myperm, j);
          b[y] = (unsigned)drow[(j < n && r < n) ? pj : n];
        }
        w[x] = __byte_perm(__byte_perm(b[0], b[1], 0x0040), __byte_perm(b[2], b[3], 0x0040), 0x5410);
      }
      *reinterpret_cast<uint4*>(P8 + cl_off(32 * warp + r, 0, KB)) = make_uint4(w[0], w[1], w[2], w[3]);
      *reinterpret_cast<uint4*>(P8 + cl_off(32 * warp + r, 16, KB)) = make_uint4(w[4], w[5], w[6], w[7]);
    }
    bool active = valid && a.passes > 0;
    for (int pass = 0; pass < a.passes; ++pass) {
      // G[r][r] and the diagonals of this lane's row
      {
        const uint4 f0 = *reinterpret_cast<const uint4*>(F8 + cl_off(32 * warp + r, 0, KB));
        const uint4 f1 = *reinterpret_cast<const uint4*>(F8 + cl_off(32 * warp + r, 16, KB));
        const uint4 d0 = *reinterpret_cast<const uint4*>(P8 + cl_off(32 * warp + r, 0, KB));
        const uint4 d1 = *reinterpret_cast<const uint4*>(P8 + cl_off(32 * warp + r, 16, KB));
        unsigned acc = 0;
        acc = __dp4a(f0.x, d0.x, acc); acc = __dp4a(f0.y, d0.y, acc);
        acc = __dp4a(f0.z, d0.z, acc); acc = __dp4a(f0.w, d0.w, acc);
        acc = __dp4a(f1.x, d1.x, acc); acc = __dp4a(f1.y, d1.y, acc);
        acc = __dp4a(f1.z, d1.z, acc); acc = __dp4a(f1.w, d1.w, acc);
        sv[r] = make_int4((int)acc, F8[cl_off(32 * warp + r, r, KB)], P8[cl_off(32 * warp + r, r, KB)], 0);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncthreads();
      if (tid == 0) {
        tc_fence_after();
        const uint32_t fa = smem_u32(F8), pa = smem_u32(P8);
        umma_i8(tmem, umma_smem_desc(fa, 128, KB * 8), umma_smem_desc(pa, 128, KB * 8), idesc, 0u);
        umma_i8(tmem, umma_smem_desc(pa, 128, KB * 8), umma_smem_desc(fa, 128, KB * 8), idesc, 1u);
        umma_commit(&bar);
      }
      mbar_wait(&bar, phase);
      phase ^= 1u;
      tc_fence_after();
      uint32_t v0[16], v1[16];
      tmem_ld16(trow, v0);
      tmem_ld16(trow + 16u, v1);
      tc_fence_before();
      int bd = INT_MAX, bs = -1;
      int64_t wbd = INT64_MAX;
      if (active && r < n) {
        const int4 mine = sv[r];
        const int gdr = mine.x, Frr = mine.y, Prr = mine.z;
        const uint4 fr0 = *reinterpret_cast<const uint4*>(F8 + cl_off(32 * warp + r, 0, KB));
        const uint4 fr1 = *reinterpret_cast<const uint4*>(F8 + cl_off(32 * warp + r, 16, KB));
        const uint4 pr0 = *reinterpret_cast<const uint4*>(P8 + cl_off(32 * warp + r, 0, KB));
        const uint4 pr1 = *reinterpret_cast<const uint4*>(P8 + cl_off(32 * warp + r, 16, KB));
        const unsigned fw[8] = {fr0.x, fr0.y, fr0.z, fr0.w, fr1.x, fr1.y, fr1.z, fr1.w};
        const unsigned pw[8] = {pr0.x, pr0.y, pr0.z, pr0.w, pr1.x, pr1.y, pr1.z, pr1.w};
#pragma unroll
        for (int s = 0; s < 32; ++s) {
          const int4 o = sv[s];
          const int Frs = (int)__byte_perm(fw[s >> 2], 0u, 0x4440 | (s & 3));
          const int Prs = (int)__byte_perm(pw[s >> 2], 0u, 0x4440 | (s & 3));
          const int t = (2 * Frs - Frr - o.y) * (2 * Prs - Prr - o.z);
          const uint32_t h = s < 16 ? v0[s & 15] : v1[s & 15];
          const bool ok = s > r && s < n;
          if (narrow) {
            const int dd = 2 * ((int)h - gdr - o.x) + t;
            if (ok && dd < bd) { bd = dd; bs = s; }
          } else {
            const int64_t dd = 2 * ((int64_t)h - gdr - o.x) + t;
            if (ok && dd < wbd) { wbd = dd; bs = s; }
          }
        }
      }
      const int64_t mine_best = bs < 0 ? INT64_MAX : (narrow ? (int64_t)bd : wbd);
      const int mine_q = bs < 0 ? INT_MAX : r * n - r * (r + 1) / 2 + (bs - r - 1);
      int64_t best = mine_best;
      int bq = mine_q;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const int64_t ob = __shfl_xor_sync(FULL, best, o);
        const int oq = __shfl_xor_sync(FULL, bq, o);
        if (ob < best || (ob == best && oq < bq)) { best = ob; bq = oq; }
      }
      if (active && bq != INT_MAX && best < 0) {
        cost += (uint64_t)best;
        // (r0, s0): the row is the lane holding the winning q (one q per lane)
        const int r0 = __ffs(__ballot_sync(FULL, mine_q == bq)) - 1;
        const int s0 = __shfl_sync(FULL, bs, r0);
        // swap facilities r0 and s0 of this warp's P: rows, then columns
        if (lane < KB) {
          const int ir = cl_off(32 * warp + r0, lane, KB), is = cl_off(32 * warp + s0, lane, KB);
          const uint8_t x = P8[ir]; P8[ir] = P8[is]; P8[is] = x;
        }
        __syncwarp();
        {
          const int ir = cl_off(32 * warp + lane, r0, KB), is = cl_off(32 * warp + lane, s0, KB);
          const uint8_t x = P8[ir]; P8[ir] = P8[is]; P8[is] = x;
        }
        if (lane == 0) { const int x = sp[r0]; sp[r0] = sp[s0]; sp[s0] = x; }
        __syncwarp();
      } else {
        active = false;
      }
      // another pass only while some particle of the CTA still moved (the
      // last pass needs no vote: the group's closing barrier follows)
      if (pass + 1 == a.passes) break;
      if (!__syncthreads_or(active)) break;
    }
    __syncwarp();
    if (valid) {
      if (lane < n) a.perm[p * n + lane] = (int16_t)sp[lane];
      bool imp = false;
      if (a.do_pbest) {
        imp = (int64_t)cost < mypl;
        if (lane == 0) {
          if (imp) a.pl_cost[p] = (int64_t)cost;
          a.improved[p] = imp ? 1 : 0;
        }
        if (imp && lane < n) a.pl_perm[p * n + lane] = (int16_t)sp[lane];
      }
      if (lane == 0) a.cost[p] = (int64_t)cost;
    }
    __syncthreads();   // P8 / sp reused by the next group
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(128) : "memory");
  }
}

}  // namespace qsb
