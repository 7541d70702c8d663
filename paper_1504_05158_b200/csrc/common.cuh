// common.cuh -- device helpers shared by the qapswarm-b200 kernels (sm_100a).
//
//  * numpy-compatible Philox4x64-10 stream (streams.py:30-64 of the reference)
//  * order-preserving 64-bit keys for the aggregation compares
//  * mbarrier + cp.async.bulk (1-D TMA) wrappers for staging particle tiles
#pragma once
#include <cstdint>
#include <climits>
#include <cuda_runtime.h>

namespace qsb {

constexpr int MODE_GLOBAL_MAX = 0;     // _batch.py:19
constexpr int MODE_PICK_COLUMN = 1;    // _batch.py:20
constexpr int MODE_SECOND_TARGET = 2;  // _batch.py:21

constexpr unsigned FULL = 0xffffffffu;

// ----------------------------------------------------------------- Philox
// numpy's Philox4x64 (random123 constants), 10 rounds.  A fresh
// Generator(Philox(key)) yields word idx from counter (idx/4 + 1, 0, 0, 0),
// lane idx % 4 (numpy increments the counter before each block);
// Generator.random() maps a word to (u >> 11) * 2^-53.
struct PhiloxBlock { uint64_t v[4]; };

__device__ __forceinline__ PhiloxBlock philox4x64_10(uint64_t c0, uint64_t k0, uint64_t k1) {
  uint64_t c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += 0x9E3779B97F4A7C15ULL; k1 += 0xBB67AE8584CAA73BULL; }
    const uint64_t lo0 = 0xD2E7470EE14C6C93ULL * c0, hi0 = __umul64hi(0xD2E7470EE14C6C93ULL, c0);
    const uint64_t lo1 = 0xCA5A826395121157ULL * c2, hi1 = __umul64hi(0xCA5A826395121157ULL, c2);
    const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  PhiloxBlock b; b.v[0] = c0; b.v[1] = c1; b.v[2] = c2; b.v[3] = c3;
  return b;
}

// Out-of-line copy for the per-particle draw rows: the block is evaluated a
// few times per particle, and inlining 10 rounds at every call site bloats
// the step kernel beyond the instruction cache.
__device__ __noinline__ PhiloxBlock philox_block_call(uint64_t c0, uint64_t k0, uint64_t k1) {
  // rounds kept rolled: this copy serves tie draws inside the step kernel,
  // where a small code footprint matters more than the loop overhead
  uint64_t c1 = 0, c2 = 0, c3 = 0;
#pragma unroll 1
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += 0x9E3779B97F4A7C15ULL; k1 += 0xBB67AE8584CAA73BULL; }
    const uint64_t lo0 = 0xD2E7470EE14C6C93ULL * c0, hi0 = __umul64hi(0xD2E7470EE14C6C93ULL, c0);
    const uint64_t lo1 = 0xCA5A826395121157ULL * c2, hi1 = __umul64hi(0xCA5A826395121157ULL, c2);
    const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  PhiloxBlock b; b.v[0] = c0; b.v[1] = c1; b.v[2] = c2; b.v[3] = c3;
  return b;
}

__device__ __forceinline__ double u64_to_unit(uint64_t u) {
  return (double)(u >> 11) * (1.0 / 9007199254740992.0);
}

// Key word of streams._key (streams.py:30-35): phase << 56 | t << 24.
__host__ __device__ __forceinline__ uint64_t stream_word(uint64_t phase, uint64_t t) {
  return (phase << 56) | (t << 24);
}

// Per-particle draw row of streams.step_draws: column k of particle row
// `row` is word row*(2+2n)+k.  DrawKey is plain values (it stays in
// registers; an address-taken object would live in local memory, which the
// per-particle hot path then writes every particle).  draw_at evaluates one
// Philox block per call -- tie draws are rare; sequential runs of draws
// (pick-column shuffles, the device init) use DrawCache, which keeps the
// last block.  Injected rows (tests replaying fixed draws, the
// reference-layout aggregate entry point) bypass Philox.
struct DrawKey {
  const double* inj;   // nullable
  uint64_t seed, word1;
  uint64_t base;       // first word index of this particle's row
};

__device__ __forceinline__ double word_unit(const PhiloxBlock& b, unsigned l) {
  const uint64_t w = l == 0 ? b.v[0] : l == 1 ? b.v[1] : l == 2 ? b.v[2] : b.v[3];
  return u64_to_unit(w);
}

// out of line: several call sites (tie draws) in the step kernel
__device__ __noinline__ double draw_at(const double* inj, uint64_t seed, uint64_t word1, uint64_t base,
                                       int k) {
  if (inj) return inj[k];
  const uint64_t idx = base + (uint64_t)k;
  return word_unit(philox_block_call((idx >> 2) + 1, seed, word1), (unsigned)(idx & 3));
}

__device__ __forceinline__ double draw_at(const DrawKey& d, int k) {
  return draw_at(d.inj, d.seed, d.word1, d.base, k);
}

struct DrawCache {
  DrawKey key;
  uint64_t cached;     // block index held in blk (UINT64_MAX = none)
  PhiloxBlock blk;
  __device__ __forceinline__ void init(const DrawKey& k) { key = k; cached = ~0ULL; }
  __device__ __forceinline__ double at(int k) {
    if (key.inj) return key.inj[k];
    const uint64_t idx = key.base + (uint64_t)k;
    const uint64_t b = idx >> 2;
    if (b != cached) { blk = philox_block_call(b + 1, key.seed, key.word1); cached = b; }
    return word_unit(blk, (unsigned)(idx & 3));
  }
};

// --------------------------------------------------------- ordered keys
// Aggregation compares m = f64(x) + v (_batch.py:68).  m is finite and never
// -0.0 (x + v with x in {0.0, 1.0} canonicalises a negative zero), so the
// usual sign-flip map is a strict order isomorphism and key equality is
// value equality.  Key 0 is never produced and means "no candidate".
__device__ __forceinline__ uint64_t okey(double m) {
  const uint64_t b = (uint64_t)__double_as_longlong(m);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}

__device__ __forceinline__ unsigned okey32(float f) {
  const unsigned b = __float_as_uint(f);
  return (b >> 31) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ float from_okey32(unsigned k) {
  return __uint_as_float((k >> 31) ? (k & 0x7fffffffu) : ~k);
}

__device__ __forceinline__ double from_okey(uint64_t k) {
  const uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffULL) : ~k;
  return __longlong_as_double((long long)b);
}

template <typename VT>
__device__ __forceinline__ double cell_m(VT v, bool x_one) {
  return __dadd_rn(x_one ? 1.0 : 0.0, (double)v);
}

// ------------------------------------------------ wide 32-bit velocity words
// fp32 velocity tiles in the lazily scaled layout (every fp32 state with a
// column-state array, n <= 256; step_kernel.cuh, vval) store the high word of
// the double (sign, 11-bit exponent, 20-bit fraction), rounded to nearest:
// fp32's size with fp64's exponent range.  The throughput-mode init writes
// these words when the state is lazily scaled.
constexpr int WIDE_MAX_N = 256;
__device__ __forceinline__ double wdec(float w) { return __hiloint2double(__float_as_int(w), 0); }
__device__ __forceinline__ float wenc(double d) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(d) + 0x80000000ULL;
  return __int_as_float((int)(unsigned)(b >> 32));
}

// Approximate reciprocal (MUFU.RCP, <= 1 ulp; deterministic).  Used where
// the lazily scaled layout only needs a consistent scale, not the IEEE
// rounded quotient (the column sums are tracked from the stored values).
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// Approximate reciprocal of a positive normal double (mantissa by MUFU.RCP,
// exponent by integer arithmetic; deterministic, relative error ~2^-23):
// the lazily scaled layout's wide column scales span the double range.
__device__ __forceinline__ double drcp_approx(double x) {
  const long long b = __double_as_longlong(x);
  const long long e = ((b >> 52) & 0x7ff) - 1023;
  const double m = __longlong_as_double((b & 0x000fffffffffffffLL) | (1023LL << 52));   // [1, 2)
  const double r = (double)rcp_approx((float)m);                                        // (0.5, 1]
  return __longlong_as_double(__double_as_longlong(r) - (e << 52));
}

// -------------------------------------------------- mbarrier / bulk copy
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// Programmatic dependent launch (PDL).  A kernel launched with the
// programmatic-stream-serialization attribute may start while the previous
// kernel in the stream is still running; pdl_wait() blocks until that kernel
// has finished and its writes are visible, so every PDL kernel calls it
// before touching memory a predecessor may write.  pdl_launch() lets the
// next PDL kernel in the stream start early.  Both are no-ops without the
// attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" :: "r"(a), "r"(phase) : "memory");
}

// 1-D bulk copy global -> shared, completion signalled on bar (tx bytes).
__device__ __forceinline__ void bulk_load(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      :: "r"(smem_u32(dst_smem)), "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// 1-D bulk copy shared -> global, tracked by the issuing thread's bulk group.
__device__ __forceinline__ void bulk_store(void* dst_gmem, const void* src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
               :: "l"(dst_gmem), "r"(smem_u32(src_smem)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// Wait until prior bulk stores of this thread have finished READING smem.
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// Wait until prior bulk stores of this thread are complete (globally visible).
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Non-bulk async copies global -> shared (cp.async), per thread.
__device__ __forceinline__ void cp_async4(void* dst_smem, const void* src_gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(smem_u32(dst_smem)), "l"(src_gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst_smem, const void* src_gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(smem_u32(dst_smem)), "l"(src_gmem) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst_smem, const void* src_gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(smem_u32(dst_smem)), "l"(src_gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// Make generic-proxy smem writes visible to the async (bulk copy) proxy.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__host__ __device__ __forceinline__ size_t align_up(size_t x, size_t a) {
  return (x + a - 1) / a * a;
}

}  // namespace qsb
