// twoopt_pair.cuh -- 2-opt on a CTA pair (cta_group::2), one pass, 128 < n <= 256.
//
// twoopt_tcp_kernel (twoopt.cuh) pipelines P-build and scoring on one SM, but
// the MMA of a particle still runs alone: H needs 384 of the 512 TMEM
// columns and its P copy the rest, so H cannot be double-buffered.  Here a
// cluster of two CTAs (two SMs of a TPC) shares each particle:
//   * each CTA holds half the rows of F and of P (rows 128 c .. 128 c + 127
//     in CTA c), so shared memory per particle halves and P is
//     double-buffered in shared memory (no TMEM copy);
//   * CTA 0 issues tcgen05.mma.cta_group::2 (M = 256, N = 256, K = 2n in
//     32-byte steps): each CTA contributes its 128 rows of A = [F | P] and of
//     B = [P | F] and receives its 128 rows of H = [F|P][P|F]^T in its own
//     TMEM, 256 columns, so H is double-buffered (512 columns);
//   * the pairs s > r are split evenly: CTA 0 scores rows r < 128 against
//     s < 192, CTA 1 rows R >= 128 against s > R plus (through the symmetry
//     of H, F and P) the pairs (r, R) with R >= 192 from its own rows;
//   * the per-row terms {G_rr, F_rr, P_rr} of both halves are exchanged
//     through distributed shared memory, and so are the two halves' best
//     (delta, q).
// Particle i's P-build, particle i-1's MMA and particle i-2's scoring
// overlap.  Deltas, tie order and results are bit-identical to
// twoopt_tc_kernel.
//
// Barriers (mbarriers at the same offset in both CTAs; remote arrives with
// release.cluster, waits with acquire.cluster):
//   full[b]     both halves of P(b), sv(b), sp(b) written    (8 + 8 builder warps)
//   mma_done[b] H(b) complete (tcgen05.commit multicast to both CTAs)
//   hfree[b]    (CTA 0) both CTAs' epilogues read H(b)        (16 + 16 epilogue warps)
//   bfree[b]    both epilogues done with P(b), sv(b), sp(b)  (16 + 16 epilogue warps)
//   pairbar[b]  both CTAs' best (delta, q) exchanged          (1 + 1)
#pragma once
#include "twoopt.cuh"

namespace qsb {

constexpr int TP2_NT = 768;          // 24 warps, 80 registers
constexpr int TP2_EPI = 16;
constexpr int TP2_BLD = 8;

// epilogue warps per TMEM lane quarter, by CTA rank: CTA 0 rows r < 128 score
// 12 / 10 / 8 / 6 chunk-rows per quarter, CTA 1 rows R >= 128 8 / 6 / 12 / 10
__host__ __device__ constexpr int tp2_eq(int rank, int q) {
  return rank == 0 ? (q == 0 ? 5 : q == 3 ? 3 : 4) : (q == 1 ? 3 : q == 2 ? 5 : 4);
}

struct TwoOptPair {
  int kb;     // bytes per operand row: n rounded up to 32
  static __host__ __device__ int dstride(int n) { return (((n + 3) / 4) | 1) * 4; }
  static __host__ __device__ size_t smem_bytes(int n, int kb) {
    return 3 * (size_t)128 * kb + align_up((size_t)n * dstride(n), 16) + 2 * 256 * 16 + 2 * 256 * 2 +
           2 * 256 * 2 + 256 * 2 + 2 * TP2_EPI * 16 + 64;
  }
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on the mbarrier at this smem address in CTA `rank` of the cluster
__device__ __forceinline__ void mbar_arrive_at(uint64_t* bar, uint32_t rank) {
  const uint32_t ra = mapa_shared(smem_u32(bar), rank);
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" :: "r"(ra) : "memory");
}
__device__ __forceinline__ void mbar_wait_cl(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
#pragma unroll 1
  for (uint32_t spins = 0;; ++spins) {
    uint32_t ok;
    asm volatile("{\n.reg .pred P1;\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%1], %2, %3;\n"
                 "selp.u32 %0, 1, 0, P1;\n}\n" : "=r"(ok) : "r"(a), "r"(parity), "r"(1000u) : "memory");
    if (ok) return;
    __nanosleep(128);
    if (spins > (1u << 24)) __trap();
  }
}
__device__ __forceinline__ void st_cluster_v4(void* p, uint32_t rank, int4 v) {
  const uint32_t ra = mapa_shared(smem_u32(p), rank);
  asm volatile("st.shared::cluster.v4.s32 [%0], {%1, %2, %3, %4};"
               :: "r"(ra), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void st_cluster_b64(void* p, uint32_t rank, int64_t v) {
  const uint32_t ra = mapa_shared(smem_u32(p), rank);
  asm volatile("st.shared::cluster.b64 [%0], %1;" :: "r"(ra), "l"(v) : "memory");
}
__device__ __forceinline__ void st_cluster_b32(void* p, uint32_t rank, int v) {
  const uint32_t ra = mapa_shared(smem_u32(p), rank);
  asm volatile("st.shared::cluster.b32 [%0], %1;" :: "r"(ra), "r"(v) : "memory");
}
__device__ __forceinline__ void umma_i8_pair(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n"
      :: "r"(d_tmem), "l"(a), "l"(b), "r"(idesc), "r"(accumulate) : "memory");
}
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               :: "r"(smem_u32(bar)), "h"((uint16_t)3) : "memory");
}

#ifdef QSB_TCP_TIMING
__device__ long long qsb_pair_ts[64][12];
#define TP2_TS(i, k) do { if (blockIdx.x == 0 && (i) < 64) qsb_pair_ts[(i)][(k)] = clock64(); } while (0)
#else
#define TP2_TS(i, k) do { } while (0)
#endif

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TP2_NT, 1)
twoopt_pair_kernel(const TwoOptArgs a, const TwoOptPair g) {
  extern __shared__ __align__(1024) unsigned char tsm[];
  const int n = a.n, kb = g.kb;
  const size_t mb = (size_t)128 * kb;
  const int dn = TwoOptPair::dstride(n);
  const uint32_t rank = cluster_rank(), peer = rank ^ 1u;
  const int rbase = 128 * (int)rank;          // first global row of this CTA's half
  uint8_t* F8 = tsm;                          // rows rbase .. rbase + 127 of F (canonical)
  uint8_t* P8b[2] = {F8 + mb, F8 + 2 * mb};   // the same rows of P, double-buffered
  uint8_t* D8 = F8 + 3 * mb;                  // all of D, row-major, stride dn
  int4* svb = reinterpret_cast<int4*>(D8 + align_up((size_t)n * dn, 16));   // [2][256] {G_rr, F_rr, P_rr}
  int16_t* spb = reinterpret_cast<int16_t*>(svb + 512);      // [2][256] the particle's perm
  int16_t* pinvb = spb + 512;                                 // [2][256] its inverse
  int16_t* mine = pinvb + 512;                                // [256] D rows whose P row is in this half
  int64_t* redd = reinterpret_cast<int64_t*>(mine + 256);    // [2][TP2_EPI]
  int* redq = reinterpret_cast<int*>(redd + 2 * TP2_EPI);    // [2][TP2_EPI]
  __shared__ __align__(8) uint64_t full[2], bfree[2], mma_done[2], hfree[2], pairbar[2];
  __shared__ __align__(8) int64_t pair_d[2][2];
  __shared__ int pair_q[2][2];
  __shared__ int s_cnt[TP2_BLD + 1];
  __shared__ uint32_t s_tmem;
  __shared__ unsigned s_mx[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint16_t* gF = reinterpret_cast<const uint16_t*>(a.F);
  const uint16_t* gD = reinterpret_cast<const uint16_t*>(a.D);

  // ---- prologue: this half of F (canonical), all of D (bytes), max F / D
  if (tid < 2) s_mx[tid] = 0;
  {
    uint4* z = reinterpret_cast<uint4*>(F8);
    const int nz = (int)(3 * mb / 16);
    for (int i = tid; i < nz; i += TP2_NT) z[i] = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  unsigned mf = 0, md = 0;
  for (int e = tid; e < n * n; e += TP2_NT) {
    const int r = e / n, c = e - r * n;
    const unsigned f = gF[e], d = gD[e];
    if (r >= rbase && r < rbase + 128) F8[cl_off(r - rbase, c, kb)] = (uint8_t)f;
    D8[r * dn + c] = (uint8_t)d;
    mf = max(mf, f);
    md = max(md, d);
  }
  mf = __reduce_max_sync(FULL, mf);
  md = __reduce_max_sync(FULL, md);
  if (lane == 0) { atomicMax(&s_mx[0], mf); atomicMax(&s_mx[1], md); }
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&full[b], 2 * TP2_BLD);
      mbar_init(&bfree[b], 2 * TP2_EPI);
      mbar_init(&mma_done[b], 1);
      mbar_init(&hfree[b], 2 * TP2_EPI);
      mbar_init(&pairbar[b], 2);
    }
    mbar_fence_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32(&s_tmem)), "r"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  fence_proxy_async_smem();     // F8 / zeroed P (generic writes) -> tensor-core reads
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();           // both CTAs' barriers initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  const bool narrow = (double)n * (double)s_mx[0] * (double)s_mx[1] < 268435456.0;
  const int64_t npairs = gridDim.x >> 1;
  const int64_t pair0 = blockIdx.x >> 1;
  const int q = warp & 3, jq = warp >> 2;

  if (jq >= tp2_eq((int)rank, q)) {
    // =========================== builders (+ the MMA issuer: CTA 0's first builder lane)
    int bi = 0;                               // index among this CTA's builder warps
    for (int w = 0; w < warp; ++w) bi += (w >> 2) >= tp2_eq((int)rank, w & 3);
    const int bt = bi * 32 + lane;            // 0 .. 255
    const bool issuer_warp = bi == 0 && rank == 0;
    const uint32_t sbo = (uint32_t)kb * 8;
    const int ksteps = kb / 32;
    const uint32_t idesc = umma_idesc_u8(256, 256);
    const int nck = kb >> 4;
    int idx = 0;
    for (int64_t p = pair0; p < a.P; p += npairs, ++idx) {
      const int b = idx & 1;
      int16_t* sp = spb + 256 * b;
      int16_t* pinv = pinvb + 256 * b;
      int4* sv = svb + 256 * b;
      uint8_t* P8 = P8b[b];
      if (idx >= 2) mbar_wait_cl(&bfree[b], ((idx >> 1) - 1) & 1);   // both epilogues done with b
      if (bt == 0) TP2_TS(idx, 0);
      for (int i = bt; i < n; i += TP2_BLD * 32) {
        const int16_t v = a.perm[p * n + i];
        sp[i] = v;
        pinv[v] = (int16_t)i;
      }
      asm volatile("bar.sync 2, %0;" :: "r"(TP2_BLD * 32) : "memory");
      // the D rows d whose P row pinv[d] is in this half, ascending (32
      // consecutive list entries read a column in mostly distinct banks)
      {
        const bool f = bt < n && (pinv[bt] >> 7) == (int)rank;
        const unsigned bal = __ballot_sync(FULL, f);
        if (lane == 0) s_cnt[bi] = __popc(bal);
        asm volatile("bar.sync 2, %0;" :: "r"(TP2_BLD * 32) : "memory");
        int base = 0;
        for (int w = 0; w < bi; ++w) base += s_cnt[w];
        if (f) mine[base + __popc(bal & ((1u << lane) - 1u))] = (int16_t)bt;
        if (bt == TP2_BLD * 32 - 1) s_cnt[TP2_BLD] = base + __popc(bal);
        asm volatile("bar.sync 2, %0;" :: "r"(TP2_BLD * 32) : "memory");
      }
      const int cnt = s_cnt[TP2_BLD];
      if (bt == 0) TP2_TS(idx, 1);
      // two threads per P row (even / odd 16-byte chunks), G_ii and P_ii
      // from the same pass
      {
        const int k = bt >> 1, h = bt & 1;
        unsigned acc = 0, pii = 0;
        int i = -1, li = 0;
        if (k < cnt) {
          const int d = mine[k];
          i = pinv[d];
          li = i - rbase;
          const uint8_t* drow = D8 + d * dn;
#pragma unroll 1
          for (int c = h; c < nck; c += 2) {
            const uint4 i0 = *reinterpret_cast<const uint4*>(sp + 16 * c);
            const uint4 i1 = *reinterpret_cast<const uint4*>(sp + 16 * c + 8);
            const unsigned iw[8] = {i0.x, i0.y, i0.z, i0.w, i1.x, i1.y, i1.z, i1.w};
            unsigned w[4];
#pragma unroll
            for (int x = 0; x < 4; ++x) {
              unsigned bb[4];
#pragma unroll
              for (int y = 0; y < 4; ++y) {
                const int j = 16 * c + 4 * x + y;
                const unsigned pj = (iw[(4 * x + y) >> 1] >> (16 * (y & 1))) & 0xffffu;
                bb[y] = j < n ? (unsigned)drow[pj] : 0u;
              }
              w[x] = __byte_perm(__byte_perm(bb[0], bb[1], 0x0040), __byte_perm(bb[2], bb[3], 0x0040), 0x5410);
            }
            *reinterpret_cast<uint4*>(P8 + cl_off(li, 16 * c, kb)) = make_uint4(w[0], w[1], w[2], w[3]);
            const uint4 f = *reinterpret_cast<const uint4*>(F8 + cl_off(li, 16 * c, kb));
            acc = __dp4a(f.x, w[0], acc); acc = __dp4a(f.y, w[1], acc);
            acc = __dp4a(f.z, w[2], acc); acc = __dp4a(f.w, w[3], acc);
            if ((i >> 4) == c) {
              const int o = i & 15;
              const unsigned ww = o < 4 ? w[0] : o < 8 ? w[1] : o < 12 ? w[2] : w[3];
              pii = (ww >> (8 * (o & 3))) & 0xffu;
            }
          }
        }
        acc += __shfl_xor_sync(FULL, acc, 1);
        pii += __shfl_xor_sync(FULL, pii, 1);     // only the thread holding chunk i >> 4 has it
        if (h == 0 && i >= 0) {
          const int4 v = make_int4((int)acc, F8[cl_off(li, i, kb)], (int)pii, 0);
          sv[i] = v;
          st_cluster_v4(sv + i, peer, v);         // the peer scores pairs against row i too
        }
      }
      fence_proxy_async_smem();                   // P (generic writes) -> tensor-core reads
      __syncwarp();
      if (bt == 0) TP2_TS(idx, 2);
      if (lane == 0) { mbar_arrive_at(&full[b], rank); mbar_arrive_at(&full[b], peer); }
      if (issuer_warp) {
        if (lane == 0) {
          mbar_wait_cl(&full[b], (idx >> 1) & 1);               // both halves built
          TP2_TS(idx, 3);
          if (idx >= 2) mbar_wait_cl(&hfree[b], ((idx >> 1) - 1) & 1);   // H(b) drained
          TP2_TS(idx, 4);
          tc_fence_after();
          const uint32_t fa = smem_u32(F8), pa = smem_u32(P8);
          for (int j = 0; j < 2 * ksteps; ++j) {
            const bool lo = j < ksteps;
            const uint32_t ko = (uint32_t)(lo ? j : j - ksteps) * 256;
            const uint64_t ad = umma_smem_desc((lo ? fa : pa) + ko, 128, sbo);
            const uint64_t bd = umma_smem_desc((lo ? pa : fa) + ko, 128, sbo);
            umma_i8_pair(tmem + (uint32_t)(256 * b), ad, bd, idesc, j > 0 ? 1u : 0u);
          }
          umma_commit_pair(&mma_done[b]);
          TP2_TS(idx, 5);
        }
        __syncwarp();
      }
    }
  } else {
    // =========================== epilogue warps
    const int Wq = tp2_eq((int)rank, q);
    int e = 0;                                // index among this CTA's epilogue warps
    for (int w = 0; w < warp; ++w) e += (w >> 2) < tp2_eq((int)rank, w & 3);
    const int lr = 32 * q + lane;             // local row = TMEM lane
    const int R = rbase + lr;                 // global row
    // chunk list of this quarter, in increasing q order per thread:
    //   CTA 0: own-half chunks c = 2q .. 7 (s > r), then cross chunks 8 .. 11
    //   CTA 1: cross chunks 0 .. 7 (pairs (r, R), R >= 192), then c = 8 + 2q .. 15
    const int nown = rank == 0 ? 8 - 2 * q : 8 - 2 * q;
    const int ncross = rank == 0 ? 4 : (q >= 2 ? 8 : 0);
    const int L = nown + ncross;
    const uint32_t tl = tmem + ((uint32_t)(32 * q) << 16);
    int idx = 0;
    for (int64_t p = pair0; p < a.P; p += npairs, ++idx) {
      const int b = idx & 1;
      // the particle's goal and personal best (read early: their latency
      // overlaps the wait; one thread rewrites them after the exchange)
      const int64_t cost0 = a.cost[p];
      const int64_t pl0 = a.do_pbest ? a.pl_cost[p] : 0;
      mbar_wait_cl(&full[b], (idx >> 1) & 1);
      mbar_wait_cl(&mma_done[b], (idx >> 1) & 1);
      tc_fence_after();
      if (warp == 0 && lane == 0) TP2_TS(idx, 6);
      const uint8_t* P8 = P8b[b];
      const int4* sv = svb + 256 * b;
      int bd = INT_MAX, bs = INT_MAX;
      int64_t wbd = INT64_MAX;
      const int4 mrow = R < n ? sv[R] : make_int4(0, 0, 0, 0);
      const int gdr = mrow.x, Frr = mrow.y, Prr = mrow.z;
      // the thread visits its pairs in increasing q (strict < keeps the first
      // of equal deltas): CTA 1's cross chunks hold pairs (s, R), s < 128 <=
      // R, ascending in s; then every row's pairs (R, s), s > R ascending.
      // bs records the column (or, for cross pairs, the column + 1024); q is
      // formed once at the end.
      const int qrow = R * n - R * (R + 1) / 2 - R - 1;   // q(R, s) = qrow + s
      for (int k = jq; k < L; k += Wq) {
        int c;                                 // column chunk (columns 16 c .. 16 c + 15)
        bool cross1;                           // CTA 1 cross chunk: pairs (s, R)
        if (rank == 0) { c = k < nown ? 2 * q + k : 8 + (k - nown); cross1 = false; }
        else { cross1 = k < ncross; c = cross1 ? k : 8 + 2 * q + (k - ncross); }
        uint32_t v[16];
        tmem_ld16(tl + (uint32_t)(256 * b + 16 * c), v);
        if (R >= n) continue;
        const uint4 fr = *reinterpret_cast<const uint4*>(F8 + cl_off(lr, 16 * c, kb));
        const uint4 pr = *reinterpret_cast<const uint4*>(P8 + cl_off(lr, 16 * c, kb));
        const unsigned fw[4] = {fr.x, fr.y, fr.z, fr.w};
        const unsigned pw[4] = {pr.x, pr.y, pr.z, pr.w};
        const int tag = cross1 ? 1024 : 0;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int s = 16 * c + j;
          const int4 o = sv[s];
          const int Frs = (int)__byte_perm(fw[j >> 2], 0u, 0x4440 | (j & 3));
          const int Prs = (int)__byte_perm(pw[j >> 2], 0u, 0x4440 | (j & 3));
          const int t = (2 * Frs - Frr - o.y) * (2 * Prs - Prr - o.z);   // |t| < 2^18
          const bool ok = cross1 || (s > R && s < n);
          if (narrow) {
            const int dd = 2 * ((int)v[j] - gdr - o.x) + t;
            if (ok && dd < bd) { bd = dd; bs = s + tag; }
          } else {
            const int64_t dd = 2 * ((int64_t)v[j] - gdr - o.x) + t;
            if (ok && dd < wbd) { wbd = dd; bs = s + tag; }
          }
        }
      }
      if (bs != INT_MAX) {
        if (bs >= 1024) {
          const int lo = bs - 1024;
          bs = lo * n - lo * (lo + 1) / 2 + (R - lo - 1);
        } else {
          bs = qrow + bs;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_at(&hfree[b], 0);   // H(b) drained (counted by CTA 0's issuer)
      if (warp == 0 && lane == 0) TP2_TS(idx, 7);
      if (warp == 3 && lane == 0) TP2_TS(idx, 8);
      int64_t best = bs == INT_MAX ? INT64_MAX : (narrow ? (int64_t)bd : wbd);
      int bq = bs;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const int64_t ob = __shfl_xor_sync(FULL, best, o);
        const int oq = __shfl_xor_sync(FULL, bq, o);
        if (ob < best || (ob == best && oq < bq)) { best = ob; bq = oq; }
      }
      if (lane == 0) { redd[TP2_EPI * b + e] = best; redq[TP2_EPI * b + e] = bq; }
      asm volatile("bar.sync 1, %0;" :: "r"(32 * TP2_EPI) : "memory");
      // the epilogue warps' minima: lane l < TP2_EPI takes warp l's, then a
      // shuffle reduction (every warp computes the same result)
      best = lane < TP2_EPI ? redd[TP2_EPI * b + lane] : INT64_MAX;
      bq = lane < TP2_EPI ? redq[TP2_EPI * b + lane] : INT_MAX;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const int64_t ob = __shfl_xor_sync(FULL, best, o);
        const int oq = __shfl_xor_sync(FULL, bq, o);
        if (ob < best || (ob == best && oq < bq)) { best = ob; bq = oq; }
      }
      // the two halves' best, exchanged through distributed shared memory
      if (e == 0 && lane == 0) {
        pair_d[b][rank] = best; pair_q[b][rank] = bq;
        st_cluster_b64(&pair_d[b][rank], peer, best);
        st_cluster_b32(&pair_q[b][rank], peer, bq);
        mbar_arrive_at(&pairbar[b], rank);
        mbar_arrive_at(&pairbar[b], peer);
      }
      if (warp == 0 && lane == 0) TP2_TS(idx, 9);
      mbar_wait_cl(&pairbar[b], (idx >> 1) & 1);
      if (warp == 0 && lane == 0) TP2_TS(idx, 10);
      {
        const int64_t o0 = pair_d[b][0], o1 = pair_d[b][1];
        const int q0 = pair_q[b][0], q1 = pair_q[b][1];
        if (o1 < o0 || (o1 == o0 && q1 < q0)) { best = o1; bq = q1; } else { best = o0; bq = q0; }
      }
      const bool move = bq != INT_MAX && best < 0;
      int rs = -1, ss = -1;
      if (move) unrank_pair(bq, n, rs, ss);
      const int64_t cost = cost0 + (move ? best : 0);
      const bool imp = a.do_pbest && cost < pl0;
      const int16_t* sp = spb + 256 * b;
      const int i = rbase + 32 * e + lane;          // this thread's perm entry (its CTA's half)
      if (32 * e + lane < 128 && i < n) {
        const int src = i == rs ? ss : (i == ss ? rs : i);
        const int16_t val = sp[src];
        a.perm[p * n + i] = val;
        if (imp) a.pl_perm[p * n + i] = val;
      }
      if (rank == 0 && e == 0 && lane == 0) {
        a.cost[p] = cost;
        if (a.do_pbest) {
          if (imp) a.pl_cost[p] = cost;
          a.improved[p] = imp ? 1 : 0;
        }
      }
      __syncwarp();
      if (lane == 0) { mbar_arrive_at(&bfree[b], rank); mbar_arrive_at(&bfree[b], peer); }
      if (warp == 0 && lane == 0) TP2_TS(idx, 11);
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();           // no remote arrive or store may target an exited CTA
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(512) : "memory");
  }
}

}  // namespace qsb
