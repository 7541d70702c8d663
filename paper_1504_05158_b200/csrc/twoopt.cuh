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

}  // namespace qsb
