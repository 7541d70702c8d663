// qsb_api.cu -- extern "C" entry points of libqsb (include/qapswarm_b200.h).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <utility>
#include <vector>

#include "../../include/qapswarm_b200.h"
#include "aux_kernels.cuh"
#include "step_kernel.cuh"
#include "twoopt.cuh"
#include "twoopt_pair.cuh"
#include "stats.cuh"

using namespace qsb;

static thread_local int g_last_cuda = 0;

static int cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return QSB_OK;
  g_last_cuda = (int)e;
  return QSB_ECUDA;
}

static int launch_status() { return cuda_status(cudaGetLastError()); }

// CUDA errors of the other translation unit (host_step.cu)
void qsb_note_cuda_error(int e) { g_last_cuda = e; }

// Launch-time caches (SM counts, shared-memory limits, function attributes,
// occupancy) are kept per device, so one process may drive several GPUs.
constexpr int MAX_DEV = 64;
static int cur_dev() {
  int d = 0;
  cudaGetDevice(&d);
  return d < 0 ? 0 : (d >= MAX_DEV ? MAX_DEV - 1 : d);
}

static int num_sms() {
  static int sms[MAX_DEV] = {};
  const int d = cur_dev();
  if (!sms[d]) {
    cudaDeviceGetAttribute(&sms[d], cudaDevAttrMultiProcessorCount, d);
    if (sms[d] <= 0) sms[d] = 148;
  }
  return sms[d];
}

// Launch with programmatic stream serialization (PDL) so the kernel's launch
// overlaps the tail of the previous kernel in the stream; the kernel itself
// calls pdl_wait() before reading anything.  QSB_NO_PDL=1 launches plainly
// (A/B knob).
static bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("QSB_NO_PDL");
    v = (e && e[0] == '1') ? 0 : 1;
  }
  return v == 1;
}

template <typename... KArgs, typename... Act>
static int launch_pdl(void (*fn)(KArgs...), int grid, int block, size_t smem, cudaStream_t s,
                      Act&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cuda_status(cudaLaunchKernelEx(&cfg, fn, std::forward<Act>(args)...));
}

static size_t smem_optin() {
  static int v[MAX_DEV] = {};
  const int d = cur_dev();
  if (!v[d]) {
    cudaDeviceGetAttribute(&v[d], cudaDevAttrMaxSharedMemoryPerBlockOptin, d);
    if (v[d] <= 0) v[d] = 227 * 1024;
  }
  return (size_t)v[d];
}

// QSB_MW_DEFER=1 (A/B): fp32 states with n > 64 keep the pre-round-2
// deferred column scale instead of the lazily scaled layout; the Python
// engine reads the same variable (engine._LAZY_MAX_N)
static int mw_defer() {
  static int v = -1;
  if (v < 0) { const char* e = getenv("QSB_MW_DEFER"); v = (e && e[0] == '1') ? 1 : 0; }
  return v;
}

// ------------------------------------------------------------ fused step
template <typename VT, typename MT, int G, int CPL, int W, bool GT = false, bool FAST = false,
          bool CHAIN = false>
static int launch_step(const StepArgs& a, cudaStream_t s) {
  using K = StepKernel<VT, MT, G, CPL, W, GT>;
  StepArgs b = a;
  const bool need_fd = (a.flags & F_COST) != 0;
  // one-warp kernels stage F and D once per SM (one 16-warp CTA); the
  // multi-warp groups (one particle per CTA, several CTAs per SM) read them
  // through L1 when the goal is incremental (a few rows per step) instead of
  // spending shared memory -- and CTAs per SM -- on a copy per CTA
  b.fd_smem = need_fd && (G == 1 || (!a.cost_incremental && K::smem_bytes(a.n, a.vstride, true) <= smem_optin()));
  const size_t smem = K::smem_bytes(a.n, a.vstride, b.fd_smem);
  if (smem > smem_optin()) return QSB_EUNSUPPORTED;
  auto fn = step_kernel<VT, MT, G, CPL, W, GT, FAST, CHAIN>;
  static size_t attr_smem[MAX_DEV] = {};
  static size_t occ_smem[MAX_DEV] = {};
  static int occ_blocks[MAX_DEV] = {};
  const int d = cur_dev();
  if (smem > attr_smem[d]) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_status(e);
    attr_smem[d] = smem;
  }
  if (occ_smem[d] != smem) {
    int bps = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, fn, 32 * G * W, smem);
    if (e != cudaSuccess) return cuda_status(e);
    occ_blocks[d] = bps > 0 ? bps : 1;
    occ_smem[d] = smem;
  }
  if (a.P <= 0) return QSB_OK;
  const int64_t want = (a.P + W - 1) / W;
  const int64_t cap = (int64_t)num_sms() * occ_blocks[d];
  const int grid = (int)(want < cap ? want : cap);
  return launch_pdl(fn, grid, 32 * G * W, smem, s, b);
}

// The steady-state throughput case (lazily scaled fp32 state, every phase,
// draw pre-pass, no injected draws, norm S_v, second-target S_x, bounded
// velocity, symmetric integral instance with 32-bit goal sums, current
// costs, even n) runs compile-time specialised kernels (step_kernel FAST).
// The late-iteration specialisation (chained bulk steps, step_kernel CHAIN):
// chosen by the caller's QSB_HINT_LATE; QSB_CHAIN=0 / 1 forces it off / on
// for A/B runs.
static bool chain_wanted(const StepArgs& a) {
  static int force = -2;
  if (force == -2) {
    const char* e = getenv("QSB_CHAIN");
    force = e ? (e[0] == '1' ? 1 : 0) : -1;
  }
  if (force >= 0) return force == 1;
  return a.late != 0;
}

static bool fast_case(const StepArgs& a, size_t mt_size) {
  return a.vcol && !a.mw_defer && a.coef && !a.inj_draws && (a.n % 2) == 0 &&
         a.flags == (F_VELOCITY | F_AGGREGATE | F_COST | F_PBEST | F_STORE_V) &&
         a.mode == MODE_SECOND_TARGET && a.depth > 0 && a.normalize && a.v_bounded &&
         a.cost_incremental && a.acc32 && a.symmetric && mt_size <= 2;
}

template <typename VT, typename MT, bool DRY>
static int dispatch_n(const StepArgs& a, cudaStream_t s) {
  constexpr bool kFastType = sizeof(VT) == 4 && sizeof(MT) == 2;
  const bool fast = kFastType && fast_case(a, sizeof(MT));
  const bool chain = fast && chain_wanted(a);
  // one-warp groups: fp32 tiles run 16 particles per CTA where they fit (one
  // CTA per SM, F / D staged once per SM), else 8; fp64 tiles 9 per CTA at
  // n = 33..64 where they fit, else 4
  if (a.n <= 64) {
    if constexpr (sizeof(VT) == 4) {
      if (a.n <= 32) {
        if (StepKernel<VT, MT, 1, 1, 16>::smem_bytes(a.n, a.vstride, true) <= smem_optin()) {
          // (n <= 32 keeps the default kernel late too: its chained
          // variant needs a stack frame and was slower at config 1)
          if constexpr (kFastType)
            if (fast) return DRY ? QSB_OK : launch_step<VT, MT, 1, 1, 16, false, true>(a, s);
          return DRY ? QSB_OK : launch_step<VT, MT, 1, 1, 16>(a, s);
        }
      } else if (StepKernel<VT, MT, 1, 2, 16>::smem_bytes(a.n, a.vstride, true) <= smem_optin()) {
        if constexpr (kFastType) {
          if (chain) return DRY ? QSB_OK : launch_step<VT, MT, 1, 2, 16, false, true, true>(a, s);
          if (fast) return DRY ? QSB_OK : launch_step<VT, MT, 1, 2, 16, false, true>(a, s);
        }
        return DRY ? QSB_OK : launch_step<VT, MT, 1, 2, 16>(a, s);
      } else if (StepKernel<VT, MT, 1, 2, 8>::smem_bytes(a.n, a.vstride, true) <= smem_optin()) {
        return DRY ? QSB_OK : launch_step<VT, MT, 1, 2, 8>(a, s);
      }
    }
    if (a.n <= 32) {
      if constexpr (DRY) return StepKernel<VT, MT, 1, 1, 4>::smem_bytes(a.n, a.vstride, true) <= smem_optin() ? QSB_OK : QSB_EUNSUPPORTED;
      else return launch_step<VT, MT, 1, 1, 4>(a, s);
    }
    if constexpr (sizeof(VT) == 8) {
      // fp64 tiles (n = 33..64): nine particles in one CTA (one CTA per SM,
      // F / D staged once) where they fit, against 2 x 4 otherwise
      if (StepKernel<VT, MT, 1, 2, 9>::smem_bytes(a.n, a.vstride, true) <= smem_optin())
        return DRY ? QSB_OK : launch_step<VT, MT, 1, 2, 9>(a, s);
    }
    if constexpr (DRY) return StepKernel<VT, MT, 1, 2, 4>::smem_bytes(a.n, a.vstride, true) <= smem_optin() ? QSB_OK : QSB_EUNSUPPORTED;
    else return launch_step<VT, MT, 1, 2, 4>(a, s);
  }
  if (a.n <= 128) {
    if constexpr (DRY) return StepKernel<VT, MT, 4, 1, 1>::smem_bytes(a.n, a.vstride, false) <= smem_optin() ? QSB_OK : QSB_EUNSUPPORTED;
    else {
      if constexpr (kFastType)
        if (fast) return launch_step<VT, MT, 4, 1, 1, false, true>(a, s);
      return launch_step<VT, MT, 4, 1, 1>(a, s);
    }
  }
  if (a.n <= 256) {
    const bool fits = StepKernel<VT, MT, 8, 1, 1>::smem_bytes(a.n, a.vstride, false) <= smem_optin();
    if constexpr (DRY) return QSB_OK;
    else {
      if constexpr (kFastType)
        if (fast) return fits ? launch_step<VT, MT, 8, 1, 1, false, true>(a, s)
                              : launch_step<VT, MT, 8, 1, 1, true, true>(a, s);
      return fits ? launch_step<VT, MT, 8, 1, 1>(a, s) : launch_step<VT, MT, 8, 1, 1, true>(a, s);
    }
  }
  return QSB_EUNSUPPORTED;
}

template <bool DRY>
static int dispatch(int v_dtype, int mat_dtype, const StepArgs& a, cudaStream_t s) {
  if (v_dtype == QSB_F32) {
    if (mat_dtype == QSB_U16) return dispatch_n<float, uint16_t, DRY>(a, s);
    if (mat_dtype == QSB_I64) return dispatch_n<float, int64_t, DRY>(a, s);
    if (mat_dtype == QSB_F64) return dispatch_n<float, double, DRY>(a, s);
  } else if (v_dtype == QSB_F64) {
    if (mat_dtype == QSB_U16) return dispatch_n<double, uint16_t, DRY>(a, s);
    if (mat_dtype == QSB_I64) return dispatch_n<double, int64_t, DRY>(a, s);
    if (mat_dtype == QSB_F64) return dispatch_n<double, double, DRY>(a, s);
  }
  return QSB_EINVAL;
}

static int32_t vstride_of(int32_t n, int32_t v_dtype) {
  const int32_t per16 = v_dtype == QSB_F64 ? 2 : 4;
  const int32_t nn = n * n;
  return (nn + per16 - 1) / per16 * per16;
}

// 2-opt on the state's perm_new / cost (north-star extension, twoopt.cuh)
template <typename MT, int NT>
static int launch_twoopt(TwoOptArgs t, cudaStream_t s) {
  using DT = MT;
  const size_t nn = (size_t)t.n * t.n;
  const size_t base = align_up(nn * sizeof(DT), 16) + align_up((size_t)t.n * 4, 16) + (NT / 32) * 12 + 64;
  size_t smem = base + align_up(nn * sizeof(MT), 16);
  t.f_smem = 1;
  if (smem > smem_optin()) { smem = base; t.f_smem = 0; }
  if (smem > smem_optin()) return QSB_EUNSUPPORTED;
  auto fn = twoopt_kernel<MT, NT>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_status(e);
  }
  int bps = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, fn, NT, smem);
  if (bps < 1) bps = 1;
  const int64_t cap = (int64_t)num_sms() * bps;
  const int grid = (int)(t.P < cap ? t.P : cap);
  if (grid <= 0) return QSB_OK;
  fn<<<grid, NT, smem, s>>>(t);
  return launch_status();
}

// byte-matrix dp4a kernel (symmetric, entries < 256, n * max * max < 2^31)
template <int NT>
static int launch_twoopt_dp4a(TwoOptArgs t, cudaStream_t s) {
  const int nr = (t.n + 3) / 4 * 4;
  int ldw = nr / 4;                       // 16-byte chunks per 4-row block
  if ((ldw & 1) == 0) ldw += 1;           // odd: consecutive blocks in distinct banks
  t.ldn = 4 * ldw;
  const size_t smem = 3 * (size_t)(nr / 4) * ldw * 16 + 2 * (size_t)nr * 4 + 8 + (NT / 32) * 12 + 16;
  if (smem > smem_optin()) return QSB_EUNSUPPORTED;
  auto fn = twoopt_dp4a_kernel<NT>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_status(e);
  }
  int bps = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, fn, NT, smem);
  if (bps < 1) bps = 1;
  const int64_t cap = (int64_t)num_sms() * bps;
  const int grid = (int)(t.P < cap ? t.P : cap);
  if (grid <= 0) return QSB_OK;
  fn<<<grid, NT, smem, s>>>(t);
  return launch_status();
}

// tensor-core kernel (symmetric, entries < 256, n <= 256): H = [F|P][P|F]^T
// as one u8 GEMM per pass (twoopt.cuh).  TMEM columns bound the CTAs per SM
// (a CTA that cannot allocate would spin), so the launch raises its shared
// memory request until at most 512 / tcols CTAs fit on an SM.
template <int NT>
static int launch_twoopt_tc(TwoOptArgs t, cudaStream_t s) {
  TwoOptTc g{};
  g.kb = (t.n + 31) / 32 * 32;
  g.npad = (t.n + 15) / 16 * 16;
  g.tiles = (t.n + 127) / 128;
  const int need = g.tiles * g.npad;
  g.tcols = need <= 32 ? 32 : need <= 64 ? 64 : need <= 128 ? 128 : need <= 256 ? 256 : 512;
  if (g.tiles > 2 || (g.tiles == 2 && NT != 256)) return QSB_EUNSUPPORTED;
  auto fn = twoopt_tc_kernel<NT>;
  static size_t dyn_max_dev[MAX_DEV] = {};
  size_t& dyn_max = dyn_max_dev[cur_dev()];
  if (!dyn_max) {
    cudaFuncAttributes fa{};
    cudaError_t e = cudaFuncGetAttributes(&fa, fn);
    if (e != cudaSuccess) return cuda_status(e);
    dyn_max = smem_optin() - fa.sharedSizeBytes;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn_max);
    if (e != cudaSuccess) return cuda_status(e);
  }
  size_t smem = TwoOptTc::smem_bytes(t.n, g.kb, g.tiles, NT);
  if (smem > dyn_max) return QSB_EUNSUPPORTED;
  // CTAs per SM from registers, shared memory and TMEM columns (the occupancy
  // API reports 1 for this kernel, so the limits are applied directly)
  static int regs = 0, stat = 0;
  if (!regs) {
    cudaFuncAttributes fa{};
    cudaError_t e = cudaFuncGetAttributes(&fa, fn);
    if (e != cudaSuccess) return cuda_status(e);
    regs = fa.numRegs; stat = (int)fa.sharedSizeBytes;
  }
  const int warp_regs = (regs * 32 + 255) / 256 * 256;
  const int by_regs = 65536 / (warp_regs * (NT / 32));
  const int by_smem = (int)((smem_optin() + 1024) / (smem + stat + 1024));
  int bps = by_regs < by_smem ? by_regs : by_smem;
  if (bps > 512 / g.tcols) bps = 512 / g.tcols;
  if (bps < 1) bps = 1;
  const int64_t cap = (int64_t)num_sms() * bps;
  const int grid = (int)(t.P < cap ? t.P : cap);
  if (grid <= 0) return QSB_OK;
  fn<<<grid, NT, smem, s>>>(t, g);
  return launch_status();
}

// 128 < n <= 256, one pass: the pipelined, warp-specialised kernel
// (twoopt_tcp_kernel), one CTA per SM (its shared memory allows no more)
static int launch_twoopt_tcp(TwoOptArgs t, cudaStream_t s) {
  TwoOptTcp g{};
  g.kb = (t.n + 31) / 32 * 32;
  g.npad = (t.n + 15) / 16 * 16;
  if (t.n <= 128 || t.n > 256 || t.passes != 1) return QSB_EUNSUPPORTED;
  // polling pauses of the parked roles (A/B knobs QSB_TCP_SLEEP_EPI / _BLD, ns)
  static int sl[2] = {-1, -1};
  if (sl[0] < 0) {
    const char* e0 = getenv("QSB_TCP_SLEEP_EPI");
    const char* e1 = getenv("QSB_TCP_SLEEP_BLD");
    sl[0] = e0 ? atoi(e0) : 128;
    sl[1] = e1 ? atoi(e1) : 128;
  }
  g.sleep_epi = (unsigned)sl[0];
  g.sleep_bld = (unsigned)sl[1];
  // second MMA half with A from the tensor-memory copy of P (QSB_TCP_TS=0: both from shared memory)
  static int ts = -1;
  if (ts < 0) { const char* e = getenv("QSB_TCP_TS"); ts = (e && e[0] == '0') ? 0 : 1; }
  g.ts = ts;
  const size_t smem = TwoOptTcp::smem_bytes(t.n, g.kb);
  static size_t attr_dev[MAX_DEV] = {};
  size_t& attr = attr_dev[cur_dev()];
  if (smem > attr) {
    cudaFuncAttributes fa{};
    cudaError_t e = cudaFuncGetAttributes(&fa, twoopt_tcp_kernel);
    if (e != cudaSuccess) return cuda_status(e);
    if (smem + fa.sharedSizeBytes > smem_optin()) return QSB_EUNSUPPORTED;
    e = cudaFuncSetAttribute(twoopt_tcp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_status(e);
    attr = smem;
  }
  const int64_t cap = num_sms();
  const int grid = (int)(t.P < cap ? t.P : cap);
  if (grid <= 0) return QSB_OK;
  return launch_pdl(twoopt_tcp_kernel, grid, TCP_NT, smem, s, t, g);
}

// 128 < n <= 256, one pass, QSB_TWOOPT_KERNEL=pair: the CTA-pair kernel
// (twoopt_pair.cuh), one pair per two SMs
static int launch_twoopt_pair(TwoOptArgs t, cudaStream_t s) {
  if (t.n <= 128 || t.n > 256 || t.passes != 1) return QSB_EUNSUPPORTED;
  TwoOptPair g{};
  g.kb = (t.n + 31) / 32 * 32;
  const size_t smem = TwoOptPair::smem_bytes(t.n, g.kb);
  static size_t attr_dev[MAX_DEV] = {};
  size_t& attr = attr_dev[cur_dev()];
  if (smem > attr) {
    cudaFuncAttributes fa{};
    cudaError_t e = cudaFuncGetAttributes(&fa, twoopt_pair_kernel);
    if (e != cudaSuccess) return cuda_status(e);
    if (smem + fa.sharedSizeBytes > smem_optin()) return QSB_EUNSUPPORTED;
    e = cudaFuncSetAttribute(twoopt_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_status(e);
    attr = smem;
  }
  const int64_t cap = num_sms() / 2;
  const int64_t pairs = t.P < cap ? t.P : cap;
  if (pairs <= 0) return QSB_OK;
  twoopt_pair_kernel<<<(int)(2 * pairs), TP2_NT, smem, s>>>(t, g);
  return launch_status();
}

// n <= 32: four particles per CTA share one MMA batch (twoopt_tc4_kernel)
static int launch_twoopt_tc4(TwoOptArgs t, cudaStream_t s) {
  constexpr int NT = 128;
  auto fn = twoopt_tc4_kernel<NT>;
  static int regs = 0, stat = 0;
  if (!regs) {
    cudaFuncAttributes fa{};
    cudaError_t e = cudaFuncGetAttributes(&fa, fn);
    if (e != cudaSuccess) return cuda_status(e);
    regs = fa.numRegs; stat = (int)fa.sharedSizeBytes;
  }
  const size_t smem = 2 * 128 * 32 + align_up((size_t)t.n * (t.n + 1), 16) + 128 * 4 + 128 * 16 + 64;
  const int warp_regs = (regs * 32 + 255) / 256 * 256;
  const int by_regs = 65536 / (warp_regs * (NT / 32));
  const int by_smem = (int)((smem_optin() + 1024) / (smem + stat + 1024));
  int bps = by_regs < by_smem ? by_regs : by_smem;
  if (bps > 4) bps = 4;                   // 128 TMEM columns per CTA
  if (bps < 1) bps = 1;
  const int64_t groups = (t.P + 3) / 4;
  const int64_t cap = (int64_t)num_sms() * bps;
  const int grid = (int)(groups < cap ? groups : cap);
  if (grid <= 0) return QSB_OK;
  return launch_pdl(fn, grid, NT, smem, s, t);
}

// QSB_TWOOPT_KERNEL=dp4a | tc | pair (A/B knobs): the dp4a kernel, the
// unpipelined tensor-core kernel for every n, or the CTA-pair kernel
// (twoopt_pair.cuh; correct, slower than the one-SM pipeline so far)
// instead of twoopt_tcp_kernel at 128 < n <= 256
static int twoopt_knob() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("QSB_TWOOPT_KERNEL");
    v = (e && strcmp(e, "dp4a") == 0) ? 1 : (e && strcmp(e, "tc") == 0) ? 2
      : (e && strcmp(e, "pair") == 0) ? 3 : 0;
  }
  return v;
}
static bool twoopt_use_dp4a() { return twoopt_knob() == 1; }

template <typename MT>
static int dispatch_twoopt(const TwoOptArgs& t, cudaStream_t s, bool bytes = false) {
  if constexpr (sizeof(MT) == 2) {
    if (bytes && t.sym && t.n <= 256 && !twoopt_use_dp4a()) {
      int rc = QSB_EUNSUPPORTED;
      if (t.n > 128 && t.passes == 1 && twoopt_knob() == 3) rc = launch_twoopt_pair(t, s);
      if (rc == QSB_EUNSUPPORTED && t.n > 128 && t.passes == 1 && (twoopt_knob() == 0 || twoopt_knob() == 3))
        rc = launch_twoopt_tcp(t, s);
      if (rc == QSB_EUNSUPPORTED)
        rc = t.n <= 32 ? launch_twoopt_tc4(t, s)
           : t.n <= 128 ? launch_twoopt_tc<128>(t, s) : launch_twoopt_tc<256>(t, s);
      if (rc != QSB_EUNSUPPORTED) return rc;
    }
    if (bytes && t.sym) {
      const int rc = t.n <= 32 ? launch_twoopt_dp4a<64>(t, s)
                   : t.n <= 64 ? launch_twoopt_dp4a<128>(t, s)
                   : (t.n <= 128 ? launch_twoopt_dp4a<256>(t, s) : launch_twoopt_dp4a<512>(t, s));
      if (rc != QSB_EUNSUPPORTED) return rc;
    }
  }
  return t.n <= 64 ? launch_twoopt<MT, 128>(t, s) : launch_twoopt<MT, 256>(t, s);
}

extern "C" {

int qsb_version(void) { return 10000; }

#ifdef QSB_TCP_TIMING
int qsb_debug_tcp_stamps(long long* out) {   // 64 x 10 clock64 stamps (diagnosis build only)
  return cuda_status(cudaMemcpyFromSymbol(out, qsb_tcp_ts, sizeof(long long) * 640));
}
int qsb_debug_pair_stamps(long long* out) {  // 64 x 12 clock64 stamps (diagnosis build only)
  return cuda_status(cudaMemcpyFromSymbol(out, qsb_pair_ts, sizeof(long long) * 768));
}
#endif

const char* qsb_strerror(int code) {
  switch (code) {
    case QSB_OK: return "ok";
    case QSB_EINVAL: return "invalid argument";
    case QSB_EUNSUPPORTED: return "problem size not supported by the fused kernel";
    case QSB_ECUDA: return cudaGetErrorString((cudaError_t)g_last_cuda);
    case QSB_EPERM: return "input is not a permutation matrix";
    default: return "unknown error";
  }
}

int qsb_last_cuda_error(void) { return g_last_cuda; }

#ifdef QSB_COUNTERS
// diagnosis builds only: read and reset the step-kernel event counters
int qsb_debug_counters(unsigned long long* out12) {
  cudaError_t e = cudaMemcpyFromSymbol(out12, qsb_counters, 12 * sizeof(unsigned long long));
  if (e != cudaSuccess) return cuda_status(e);
  unsigned long long z[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  return cuda_status(cudaMemcpyToSymbol(qsb_counters, z, sizeof(z)));
}
#endif

int32_t qsb_vstride(int32_t n, int32_t v_dtype) { return vstride_of(n, v_dtype); }

int qsb_stream_gate(const int32_t* host_flag, int64_t timeout_ns, int32_t* timed_out, void* stream) {
  if (!host_flag || timeout_ns <= 0) return QSB_EINVAL;
  void* dflag = nullptr;
  cudaError_t e = cudaHostGetDevicePointer(&dflag, const_cast<int32_t*>(host_flag), 0);
  if (e != cudaSuccess) return cuda_status(e);
  int32_t* dto = nullptr;
  if (timed_out) {
    cudaPointerAttributes pa{};
    e = cudaPointerGetAttributes(&pa, timed_out);
    if (e != cudaSuccess) return cuda_status(e);
    if (pa.type == cudaMemoryTypeHost) {
      e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&dto), timed_out, 0);
      if (e != cudaSuccess) return cuda_status(e);
    } else {
      dto = timed_out;
    }
  }
  gate_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(reinterpret_cast<const volatile int32_t*>(dflag),
                                                   (long long)timeout_ns, dto);
  return launch_status();
}

int qsb_supported(int32_t n, int32_t v_dtype, int32_t mat_dtype) {
  if (n < 2) return 0;
  StepArgs a{};
  a.n = n;
  a.vstride = vstride_of(n, v_dtype);
  return dispatch<true>(v_dtype, mat_dtype, a, nullptr) == QSB_OK ? 1 : 0;
}

static void fill_args(StepArgs& a, const qsb_state* st, const qsb_instance* inst, const qsb_coeffs* co) {
  a.n = st->n;
  a.vstride = st->vstride;
  a.P = st->num_particles;
  a.S = st->swarm_size;
  a.p0 = st->particle_offset;
  a.c1 = co->c1; a.c2 = co->c2; a.c3 = co->c3; a.vmax = co->v_max;
  a.normalize = co->normalize;
  a.mode = co->sx_mode;
  a.depth = co->depth;
  a.seed = co->seed;
  a.V = st->V;
  a.perm = st->perm;
  a.perm_new = st->perm_new;
  a.pl_perm = st->pl_perm;
  a.pg_perm = st->pg_perm;
  a.cost = st->cost;
  a.pl_cost = st->pl_cost;
  a.improved = st->improved;
  a.F = inst ? inst->flow : nullptr;
  a.D = inst ? inst->distance : nullptr;
  a.acc32 = inst ? inst->acc32 : 0;
  a.v_bounded = (co->hints & QSB_HINT_V_BOUNDED) ? 1 : 0;
  a.cost_incremental = (co->hints & QSB_HINT_COST_CURRENT) ? 1 : 0;
  a.symmetric = (co->hints & QSB_HINT_SYMMETRIC) ? 1 : 0;
  a.late = (co->hints & QSB_HINT_LATE) ? 1 : 0;
  a.vcol = st->v_dtype == QSB_F32 ? st->vcol : nullptr;
  a.mw_defer = mw_defer();
  a.vcstride = (st->n + 3) / 4 * 4;
}

int qsb_step_phases(const qsb_state* st, const qsb_instance* inst, const qsb_coeffs* co,
                    int32_t flags, const double* inj_draws, int64_t inj_stride, int32_t agg_base,
                    const double* coef, uint64_t t_host, void* stream) {
  if (!st || !co || st->n < 2 || st->vstride < st->n * st->n) return QSB_EINVAL;
  if ((flags & (QSB_PHASE_COST | QSB_PHASE_PBEST)) && !(flags & QSB_PHASE_AGGREGATE)) return QSB_EINVAL;
  if ((flags & QSB_PHASE_COST) && (!inst || inst->n != st->n)) return QSB_EINVAL;
  if (co->sx_mode < 0 || co->sx_mode > 2) return QSB_EINVAL;
  StepArgs a{};
  fill_args(a, st, inst, co);
  a.flags = flags;
  a.t_dev = st->iteration;
  a.t_host = t_host;
  a.inj_draws = inj_draws;
  a.inj_stride = inj_stride;
  a.agg_base = agg_base;
  a.coef = coef;
  bool work_reset = false;
  if (!coef && !inj_draws && (flags & QSB_PHASE_VELOCITY) && st->step_coef && (co->hints & QSB_HINT_COEF_READY)) {
    // the previous step's best update drew this step's coefficients
    a.coef = st->step_coef;
    work_reset = true;
  } else if (!coef && !inj_draws && (flags & QSB_PHASE_VELOCITY) && st->step_coef && st->num_particles > 0) {
    // the step's (c2 r2, c3 r3) from a one-thread-per-particle pre-pass
    const int64_t P = st->num_particles;
    const int grid = (int)((P + 255) / 256 < 4 * num_sms() ? (P + 255) / 256 : 4 * num_sms());
    const int rc = launch_pdl(coef_kernel, grid, 256, 0, (cudaStream_t)stream, co->seed,
                              (const int64_t*)st->iteration, t_host, st->particle_offset, P, st->n,
                              co->c2, co->c3, st->step_coef, (unsigned*)st->work);
    if (rc) return rc;
    a.coef = st->step_coef;
    work_reset = true;   // coef_kernel zeroed the particle counter
  }
  a.work = st->work;
  if (a.work && !work_reset) {
    cudaError_t e = cudaMemsetAsync(a.work, 0, sizeof(unsigned int), (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_status(e);
  }
  const int mat = inst ? inst->mat_dtype : QSB_U16;
  return dispatch<false>(st->v_dtype, mat, a, (cudaStream_t)stream);
}

static int best_update(const qsb_state* st, const qsb_coeffs* co, void* stream);

int qsb_best_update(const qsb_state* st, void* stream) { return best_update(st, nullptr, stream); }

int qsb_best_update_next(const qsb_state* st, const qsb_coeffs* co, void* stream) {
  if (!co || !st || !st->step_coef) return QSB_EINVAL;
  return best_update(st, co, stream);
}

static int best_update(const qsb_state* st, const qsb_coeffs* co, void* stream) {
  if (!st || !st->iteration || !st->done) return QSB_EINVAL;
  BestArgs b{};
  if (co) {
    b.coef = st->step_coef;
    b.c2 = co->c2;
    b.c3 = co->c3;
    b.seed = co->seed;
    b.P = st->num_particles;
    b.work = (unsigned*)st->work;
  }
  b.n = st->n;
  b.S = st->swarm_size;
  b.m = st->num_swarms;
  b.p0 = st->particle_offset;
  b.cost = st->cost;
  b.improved = st->improved;
  b.perm_new = st->perm_new;
  b.pg_perm = st->pg_perm;
  b.pg_cost = st->pg_cost;
  b.best_cost = st->best_cost;
  b.best_perm = st->best_perm;
  b.best_iter = st->best_iter;
  b.best_idx = st->best_idx;
  b.t_dev = st->iteration;
  b.swarm_min = st->swarm_min;
  b.swarm_min_idx = st->swarm_min_idx;
  b.done = st->done;
  static int wpb = -1;
  if (wpb < 0) {
    const char* e = std::getenv("QSB_BEST_WPB");
    wpb = (e && e[0] == '4') ? 4 : 8;
  }
  const int grid = (int)((b.m + wpb - 1) / wpb);
  if (grid <= 0) return QSB_EINVAL;
  if (wpb == 4) {
    if (st->cost_dtype == QSB_I64)
      return launch_pdl(best_kernel<int64_t, 4>, grid, 32 * 4, 0, (cudaStream_t)stream, b);
    if (st->cost_dtype == QSB_F64)
      return launch_pdl(best_kernel<double, 4>, grid, 32 * 4, 0, (cudaStream_t)stream, b);
    return QSB_EINVAL;
  }
  if (st->cost_dtype == QSB_I64)
    return launch_pdl(best_kernel<int64_t, 8>, grid, 32 * 8, 0, (cudaStream_t)stream, b);
  if (st->cost_dtype == QSB_F64)
    return launch_pdl(best_kernel<double, 8>, grid, 32 * 8, 0, (cudaStream_t)stream, b);
  return QSB_EINVAL;
}

int qsb_step(const qsb_state* st, const qsb_instance* inst, const qsb_coeffs* co, void* stream) {
  int rc = qsb_step_phases(st, inst, co,
                           QSB_PHASE_VELOCITY | QSB_PHASE_AGGREGATE | QSB_PHASE_COST |
                               QSB_PHASE_PBEST | QSB_PHASE_STORE_V,
                           nullptr, 0, 2, nullptr, 0, stream);
  if (rc) return rc;
  return qsb_best_update(st, stream);
}

int qsb_migrate(const qsb_state* st, const qsb_migration* mig, void* stream) {
  if (!st || !mig || !st->iteration || mig->d < 0) return QSB_EINVAL;
  if (mig->d == 0) return QSB_OK;
  if (2 * (int64_t)mig->d >= mig->num_swarms_total) return QSB_EINVAL;
  MigArgs a{};
  a.n = st->n;
  a.S = st->swarm_size;
  a.m = mig->num_swarms_total;
  a.m0 = st->swarm_offset;
  a.m_local = st->num_swarms;
  a.d = mig->d;
  a.period = mig->period;
  a.t_dev = st->iteration;
  a.picks = mig->picks;
  a.picks_e0 = mig->picks_epoch0;
  a.picks_rows = mig->picks_rows;
  a.all_pg_cost = mig->all_pg_cost ? mig->all_pg_cost : st->pg_cost;
  a.perm = st->perm;
  a.cost = st->cost;
  a.pg_perm = st->pg_perm;
  a.pg_cost = st->pg_cost;
  a.plan = mig->plan;
  a.rec = mig->records;
  a.log = mig->log;
  a.log_rows = mig->log_rows;
  a.log_count = mig->log_count;
  a.status = mig->status;
  a.mode = mig->mode;
  a.seed = mig->seed;
  if (!a.plan || !a.status || (a.log && !a.log_count)) return QSB_EINVAL;
  if (a.mode == 0 && (a.m0 != 0 || a.m_local != a.m)) return QSB_EINVAL;
  if (a.mode == 2 && !a.rec) return QSB_EINVAL;
  const size_t csz = st->cost_dtype == QSB_F64 ? 8 : 8;
  size_t p2 = 1;
  while (p2 < (size_t)a.m) p2 <<= 1;
  a.picks_smem_off = align_up(align_up((size_t)a.m * csz, 16) +
                       (p2 <= (size_t)MIG_SORT_MAX ? align_up(p2, 4) * 4 + p2 * 8 : (size_t)a.m * 4), 16);
  const size_t smem = a.picks_smem_off + (mig->picks ? 0 : align_up((size_t)a.d * 4, 16));
  if (smem > smem_optin()) return QSB_EUNSUPPORTED;
  cudaStream_t s = (cudaStream_t)stream;
  if (st->cost_dtype == QSB_I64) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(migrate_kernel<int64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    return launch_pdl(migrate_kernel<int64_t>, 1, 1024, smem, s, a);
  }
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(migrate_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  return launch_pdl(migrate_kernel<double>, 1, 1024, smem, s, a);
}

int qsb_migration_picks(uint64_t seed, uint64_t t, int32_t d, int64_t swarm_size, int32_t* out,
                        void* stream) {
  if (!out || d < 0 || swarm_size < 1 || swarm_size > 0xFFFFFFFFLL) return QSB_EINVAL;
  if (d == 0) return QSB_OK;
  picks_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(seed, t, d, swarm_size, out);
  return launch_status();
}

size_t qsb_stats_work_bytes(void) { return sizeof(StatsWork); }

int qsb_population_stats(const void* cost, int32_t cost_dtype, int64_t P, double lo, double width,
                         int32_t bins, const int64_t* ranks_k, int32_t nranks, void* work,
                         uint32_t* hist, int64_t* out, void* stream) {
  if (!cost || !work || !hist || !out || P <= 0 || bins < 1 || nranks < 0 || nranks > STATS_RANKS ||
      !(width > 0.0))
    return QSB_EINVAL;
  if (nranks && !ranks_k) return QSB_EINVAL;
  unsigned long long k[STATS_RANKS] = {0, 0, 0, 0};
  for (int r = 0; r < nranks; ++r) {
    if (ranks_k[r] < 0 || ranks_k[r] >= P) return QSB_EINVAL;
    k[r] = (unsigned long long)ranks_k[r];
  }
  cudaStream_t s = (cudaStream_t)stream;
  StatsWork* w = (StatsWork*)work;
  cudaError_t e = cudaMemsetAsync(w, 0, sizeof(StatsWork), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(hist, 0, sizeof(uint32_t) * (size_t)bins, s);
  if (e != cudaSuccess) return cuda_status(e);
  stats_init_kernel<<<1, 1, 0, s>>>(w, k[0], k[1], k[2], k[3]);
  const int threads = 256;
  const int grid = (int)((P + threads - 1) / threads < 2 * num_sms() ? (P + threads - 1) / threads : 2 * num_sms());
  const size_t hsmem = sizeof(unsigned int) * (size_t)bins;
  if (hsmem > smem_optin()) return QSB_EUNSUPPORTED;
  if (cost_dtype == QSB_I64) {
    auto hk = stats_hist_kernel<int64_t>;
    if (hsmem > 48 * 1024) cudaFuncSetAttribute(hk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsmem);
    hk<<<grid, threads, hsmem, s>>>((const int64_t*)cost, P, lo, width, bins, hist, w);
    for (int shift = 56; nranks && shift >= 0; shift -= 8)
      stats_select_kernel<int64_t><<<grid, threads, 0, s>>>((const int64_t*)cost, P, shift, nranks, w);
    stats_finish_kernel<int64_t><<<1, 1, 0, s>>>(w, nranks, (long long*)out);
  } else if (cost_dtype == QSB_F64) {
    auto hk = stats_hist_kernel<double>;
    if (hsmem > 48 * 1024) cudaFuncSetAttribute(hk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsmem);
    hk<<<grid, threads, hsmem, s>>>((const double*)cost, P, lo, width, bins, hist, w);
    for (int shift = 56; nranks && shift >= 0; shift -= 8)
      stats_select_kernel<double><<<grid, threads, 0, s>>>((const double*)cost, P, shift, nranks, w);
    stats_finish_kernel<double><<<1, 1, 0, s>>>(w, nranks, (long long*)out);
  } else {
    return QSB_EINVAL;
  }
  return launch_status();
}

int qsb_cost(const int16_t* perms, int64_t P, const qsb_instance* inst, void* out, void* stream) {
  if (!perms || !inst || !out || P < 0 || inst->n < 2) return QSB_EINVAL;
  if (P == 0) return QSB_OK;
  const int grid = (int)((P + 7) / 8 < 4 * num_sms() ? (P + 7) / 8 : 4 * num_sms());
  cudaStream_t s = (cudaStream_t)stream;
  switch (inst->mat_dtype) {
    case QSB_U16:
      cost_kernel<uint16_t, int16_t><<<grid, 256, 0, s>>>(perms, P, inst->n, (const uint16_t*)inst->flow,
                                                         (const uint16_t*)inst->distance, out);
      break;
    case QSB_I64:
      cost_kernel<int64_t, int16_t><<<grid, 256, 0, s>>>(perms, P, inst->n, (const int64_t*)inst->flow,
                                                        (const int64_t*)inst->distance, out);
      break;
    case QSB_F64:
      cost_kernel<double, int16_t><<<grid, 256, 0, s>>>(perms, P, inst->n, (const double*)inst->flow,
                                                       (const double*)inst->distance, out);
      break;
    default:
      return QSB_EINVAL;
  }
  return launch_status();
}

int qsb_step_draws(uint64_t seed, uint64_t t, int64_t p0, int64_t P, int32_t n, double* out, void* stream) {
  if (!out || P < 0 || n < 1) return QSB_EINVAL;
  if (P == 0) return QSB_OK;
  const int64_t total = P * (2 + 2 * (int64_t)n);
  const int grid = (int)((total + 255) / 256 < 8 * num_sms() ? (total + 255) / 256 : 8 * num_sms());
  draws_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(seed, t, p0, P, n, out);
  return launch_status();
}

int qsb_init_population_device(const qsb_state* st, uint64_t seed, double amp, void* stream) {
  if (!st || !st->perm || !st->V) return QSB_EINVAL;
  // wide words iff the state is lazily scaled (engine.PopulationState.v_wide)
  const int wide = st->v_dtype == QSB_F32 && st->vcol && st->n <= WIDE_MAX_N && (st->n <= 64 || !mw_defer());
  const int grid = (int)((st->num_particles + 7) / 8 < 8 * num_sms() ? (st->num_particles + 7) / 8 : 8 * num_sms());
  if (grid <= 0) return QSB_OK;
  if (st->v_dtype == QSB_F32)
    init_kernel<float><<<grid, 256, 0, (cudaStream_t)stream>>>(seed, st->particle_offset, st->num_particles,
                                                                st->n, st->vstride, amp, st->perm, (float*)st->V, wide);
  else
    init_kernel<double><<<grid, 256, 0, (cudaStream_t)stream>>>(seed, st->particle_offset, st->num_particles,
                                                                 st->n, st->vstride, amp, st->perm, (double*)st->V, 0);
  return launch_status();
}

int qsb_perm_to_matrix(const int16_t* perm, int64_t P, int32_t n, int8_t* x, void* stream) {
  if (!perm || !x || P < 0 || n < 1) return QSB_EINVAL;
  if (P == 0) return QSB_OK;
  const int64_t total = P * n * n;
  const int grid = (int)((total + 255) / 256 < 8 * num_sms() ? (total + 255) / 256 : 8 * num_sms());
  perm_to_mat_kernel<int16_t><<<grid, 256, 0, (cudaStream_t)stream>>>(perm, P, n, x);
  return launch_status();
}

int qsb_twoopt(const qsb_state* st, const qsb_instance* inst, int32_t passes, int32_t flags,
               void* stream) {
  if (!st || !inst || st->n < 2 || inst->n != st->n || passes < 0) return QSB_EINVAL;
  if (st->cost_dtype != QSB_I64 || inst->mat_dtype == QSB_F64) return QSB_EINVAL;
  TwoOptArgs t{};
  t.n = st->n;
  t.P = st->num_particles;
  t.passes = passes;
  t.sym = (flags & QSB_TWOOPT_SYMMETRIC) ? 1 : 0;
  t.do_pbest = (flags & QSB_TWOOPT_PBEST) ? 1 : 0;
  t.perm = st->perm_new;
  t.cost = (int64_t*)st->cost;
  t.pl_perm = st->pl_perm;
  t.pl_cost = (int64_t*)st->pl_cost;
  t.improved = st->improved;
  t.F = inst->flow;
  t.D = inst->distance;
  if (t.P == 0 || (passes == 0 && !t.do_pbest)) return QSB_OK;
  if (t.do_pbest && (!t.pl_perm || !t.pl_cost || !t.improved)) return QSB_EINVAL;
  if (inst->mat_dtype == QSB_U16)
    return dispatch_twoopt<uint16_t>(t, (cudaStream_t)stream, (flags & QSB_TWOOPT_BYTES) != 0);
  return dispatch_twoopt<int64_t>(t, (cudaStream_t)stream);
}

}  // extern "C"

// ------------------------------------------------- tier 1: host buffers
namespace {

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  int ensure(size_t bytes) {
    if (bytes <= cap) return QSB_OK;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc(&p, bytes ? bytes : 16);
    if (e != cudaSuccess) return cuda_status(e);
    cap = bytes;
    return QSB_OK;
  }
};

struct HostCtx {
  std::mutex mu;
  cudaStream_t stream = nullptr;
  DevBuf b[10];
  int init() {
    if (!stream) {
      cudaError_t e = cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking);
      if (e != cudaSuccess) return cuda_status(e);
    }
    return QSB_OK;
  }
};

HostCtx& hctx() {
  static HostCtx c;
  return c;
}

#define QSB_TRY(x) do { int _rc = (x); if (_rc) return _rc; } while (0)
#define QSB_CUDA(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) return cuda_status(_e); } while (0)

}  // namespace

extern "C" {

int qsb_velocity_many(double* v, const int8_t* x, const int8_t* pl, const int8_t* pg, int64_t P, int32_t n,
                      int64_t swarm_size, double c1, const double* c2r2, const double* c3r3, double v_max,
                      int32_t normalize) {
  if (!v || !x || !pl || !pg || !c2r2 || !c3r3 || n < 1 || P < 0 || swarm_size < 1) return QSB_EINVAL;
  if (P == 0) return QSB_OK;
  if (n < 2) return QSB_EUNSUPPORTED;
  HostCtx& h = hctx();
  std::lock_guard<std::mutex> lock(h.mu);
  QSB_TRY(h.init());
  const int64_t nn = (int64_t)n * n;
  const int64_t m = (P + swarm_size - 1) / swarm_size;
  const int32_t vs = vstride_of(n, QSB_F64);
  cudaStream_t s = h.stream;
  QSB_TRY(h.b[0].ensure(P * vs * 8));
  QSB_TRY(h.b[1].ensure((P * 2 + m) * nn));
  QSB_TRY(h.b[2].ensure((P * 2 + m) * n * 2));
  QSB_TRY(h.b[3].ensure(P * 16));
  QSB_TRY(h.b[4].ensure(16));
  double* dV = (double*)h.b[0].p;
  int8_t* dx = (int8_t*)h.b[1].p;
  int8_t* dpl = dx + P * nn;
  int8_t* dpg = dpl + P * nn;
  int16_t* pp = (int16_t*)h.b[2].p;
  int16_t* ppl = pp + P * n;
  int16_t* ppg = ppl + P * n;
  double* dcoef = (double*)h.b[3].p;
  int* bad = (int*)h.b[4].p;
  QSB_CUDA(cudaMemcpy2DAsync(dV, vs * 8, v, nn * 8, nn * 8, P, cudaMemcpyHostToDevice, s));
  QSB_CUDA(cudaMemcpyAsync(dx, x, P * nn, cudaMemcpyHostToDevice, s));
  QSB_CUDA(cudaMemcpyAsync(dpl, pl, P * nn, cudaMemcpyHostToDevice, s));
  QSB_CUDA(cudaMemcpyAsync(dpg, pg, m * nn, cudaMemcpyHostToDevice, s));
  QSB_CUDA(cudaMemcpy2DAsync(dcoef, 16, c2r2, 8, 8, P, cudaMemcpyHostToDevice, s));
  QSB_CUDA(cudaMemcpy2DAsync(dcoef + 1, 16, c3r3, 8, 8, P, cudaMemcpyHostToDevice, s));
  QSB_CUDA(cudaMemsetAsync(bad, 0, 4, s));
  const int grid = 4 * num_sms();
  mat_to_perm_kernel<<<grid, 256, 0, s>>>(dx, 2 * P + m, n, pp, bad);
  QSB_TRY(launch_status());
  int hbad = 0;
  QSB_CUDA(cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, s));
  QSB_CUDA(cudaStreamSynchronize(s));
  if (hbad) return QSB_EPERM;
  qsb_state st{};
  st.n = n; st.vstride = vs; st.v_dtype = QSB_F64; st.cost_dtype = QSB_I64;
  st.num_particles = P; st.swarm_size = swarm_size; st.num_swarms = m;
  st.V = dV; st.perm = pp; st.pl_perm = ppl; st.pg_perm = ppg;
  qsb_coeffs co{};
  co.c1 = c1; co.v_max = v_max; co.normalize = normalize; co.sx_mode = 0; co.depth = 1;
  QSB_TRY(qsb_step_phases(&st, nullptr, &co, QSB_PHASE_VELOCITY | QSB_PHASE_STORE_V, nullptr, 0, 2, dcoef, 1, s));
  QSB_CUDA(cudaMemcpy2DAsync(v, nn * 8, dV, vs * 8, nn * 8, P, cudaMemcpyDeviceToHost, s));
  QSB_CUDA(cudaStreamSynchronize(s));
  return QSB_OK;
}

int qsb_aggregate_many(const int8_t* x, const double* v, int64_t P, int32_t n, int32_t mode, int32_t depth,
                       const double* draws, int64_t draws_stride, int8_t* out_mat, int64_t* out_perm) {
  if (!x || !v || !draws || !out_mat || !out_perm || n < 1 || P < 0 || mode < 0 || mode > 2) return QSB_EINVAL;
  if (draws_stride < 2 * (int64_t)n) return QSB_EINVAL;
  if (P == 0) return QSB_OK;
  if (n < 2) return QSB_EUNSUPPORTED;
  HostCtx& h = hctx();
  std::lock_guard<std::mutex> lock(h.mu);
  QSB_TRY(h.init());
  const int64_t nn = (int64_t)n * n;
  const int32_t vs = vstride_of(n, QSB_F64);
  cudaStream_t s = h.stream;
  QSB_TRY(h.b[0].ensure(P * vs * 8));
  QSB_TRY(h.b[1].ensure(P * nn));
  QSB_TRY(h.b[2].ensure(P * n * 2 * 2));
  QSB_TRY(h.b[3].ensure(P * draws_stride * 8));
  QSB_TRY(h.b[4].ensure(16));
  QSB_TRY(h.b[5].ensure(P * nn));
  double* dV = (double*)h.b[0].p;
  int8_t* dx = (int8_t*)h.b[1].p;
  int16_t* pp = (int16_t*)h.b[2].p;
  int16_t* pnew = pp + P * n;
  double* dd = (double*)h.b[3].p;
  int* bad = (int*)h.b[4].p;
  int8_t* dmat = (int8_t*)h.b[5].p;
  QSB_CUDA(cudaMemcpy2DAsync(dV, vs * 8, v, nn * 8, nn * 8, P, cudaMemcpyHostToDevice, s));
  QSB_CUDA(cudaMemcpyAsync(dx, x, P * nn, cudaMemcpyHostToDevice, s));
  QSB_CUDA(cudaMemcpyAsync(dd, draws, P * draws_stride * 8, cudaMemcpyHostToDevice, s));
  QSB_CUDA(cudaMemsetAsync(bad, 0, 4, s));
  mat_to_perm_kernel<<<4 * num_sms(), 256, 0, s>>>(dx, P, n, pp, bad);
  QSB_TRY(launch_status());
  int hbad = 0;
  QSB_CUDA(cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, s));
  QSB_CUDA(cudaStreamSynchronize(s));
  if (hbad) return QSB_EPERM;
  qsb_state st{};
  st.n = n; st.vstride = vs; st.v_dtype = QSB_F64; st.cost_dtype = QSB_I64;
  st.num_particles = P; st.swarm_size = P; st.num_swarms = 1;
  st.V = dV; st.perm = pp; st.perm_new = pnew;
  qsb_coeffs co{};
  co.sx_mode = mode; co.depth = depth;
  QSB_TRY(qsb_step_phases(&st, nullptr, &co, QSB_PHASE_AGGREGATE, dd, draws_stride, 0, nullptr, 1, s));
  QSB_TRY(qsb_perm_to_matrix(pnew, P, n, dmat, s));
  std::vector<int16_t> hp((size_t)(P * n));
  QSB_CUDA(cudaMemcpyAsync(hp.data(), pnew, P * n * 2, cudaMemcpyDeviceToHost, s));
  QSB_CUDA(cudaMemcpyAsync(out_mat, dmat, P * nn, cudaMemcpyDeviceToHost, s));
  QSB_CUDA(cudaStreamSynchronize(s));
  for (int64_t i = 0; i < P * n; ++i) out_perm[i] = hp[(size_t)i];
  return QSB_OK;
}

static int cost_many_host(const int64_t* perms, const void* flow, const void* dist, void* out, int64_t P,
                          int32_t n, int mat_dtype) {
  if (!perms || !flow || !dist || !out || n < 1 || P < 0) return QSB_EINVAL;
  if (P == 0) return QSB_OK;
  HostCtx& h = hctx();
  std::lock_guard<std::mutex> lock(h.mu);
  QSB_TRY(h.init());
  const int64_t nn = (int64_t)n * n;
  cudaStream_t s = h.stream;
  QSB_TRY(h.b[6].ensure(P * n * 8));
  QSB_TRY(h.b[7].ensure(2 * nn * 8));
  QSB_TRY(h.b[8].ensure(P * 8));
  int64_t* dp = (int64_t*)h.b[6].p;
  char* dm = (char*)h.b[7].p;
  QSB_CUDA(cudaMemcpyAsync(dp, perms, P * n * 8, cudaMemcpyHostToDevice, s));
  QSB_CUDA(cudaMemcpyAsync(dm, flow, nn * 8, cudaMemcpyHostToDevice, s));
  QSB_CUDA(cudaMemcpyAsync(dm + nn * 8, dist, nn * 8, cudaMemcpyHostToDevice, s));
  const int grid = (int)((P + 7) / 8 < 4 * num_sms() ? (P + 7) / 8 : 4 * num_sms());
  if (mat_dtype == QSB_I64)
    cost_kernel<int64_t, int64_t><<<grid, 256, 0, s>>>(dp, P, n, (const int64_t*)dm,
                                                      (const int64_t*)(dm + nn * 8), h.b[8].p);
  else
    cost_kernel<double, int64_t><<<grid, 256, 0, s>>>(dp, P, n, (const double*)dm,
                                                     (const double*)(dm + nn * 8), h.b[8].p);
  QSB_TRY(launch_status());
  QSB_CUDA(cudaMemcpyAsync(out, h.b[8].p, P * 8, cudaMemcpyDeviceToHost, s));
  QSB_CUDA(cudaStreamSynchronize(s));
  return QSB_OK;
}

int qsb_cost_many_i64(const int64_t* perms, const int64_t* flow, const int64_t* distance, int64_t* out,
                      int64_t P, int32_t n) {
  return cost_many_host(perms, flow, distance, out, P, n, QSB_I64);
}

int qsb_cost_many_f64(const int64_t* perms, const double* flow, const double* distance, double* out,
                      int64_t P, int32_t n) {
  return cost_many_host(perms, flow, distance, out, P, n, QSB_F64);
}

int qsb_step_draws_host(uint64_t seed, uint64_t t, int64_t P, int32_t n, double* out) {
  if (!out || P < 0 || n < 1) return QSB_EINVAL;
  if (P == 0) return QSB_OK;
  HostCtx& h = hctx();
  std::lock_guard<std::mutex> lock(h.mu);
  QSB_TRY(h.init());
  const int64_t bytes = P * (2 + 2 * (int64_t)n) * 8;
  QSB_TRY(h.b[9].ensure(bytes));
  QSB_TRY(qsb_step_draws(seed, t, 0, P, n, (double*)h.b[9].p, h.stream));
  QSB_CUDA(cudaMemcpyAsync(out, h.b[9].p, bytes, cudaMemcpyDeviceToHost, h.stream));
  QSB_CUDA(cudaStreamSynchronize(h.stream));
  return QSB_OK;
}

int qsb_twoopt_many(int64_t* perms, const int64_t* flow, const int64_t* distance, int64_t* costs,
                    int64_t P, int32_t n, int32_t passes) {
  if (!perms || !flow || !distance || !costs || n < 2 || P < 0 || passes < 0) return QSB_EINVAL;
  if (P == 0) return QSB_OK;
  HostCtx& h = hctx();
  std::lock_guard<std::mutex> lock(h.mu);
  QSB_TRY(h.init());
  const int64_t nn = (int64_t)n * n;
  cudaStream_t s = h.stream;
  // symmetric instances use the halved delta sweep (exact: products < 2^63)
  bool sym = true;
  for (int i = 0; i < n && sym; ++i)
    for (int j = 0; j < i; ++j)
      if (flow[i * n + j] != flow[j * n + i] || distance[i * n + j] != distance[j * n + i]) { sym = false; break; }
  int64_t mx = 0;
  for (int64_t i = 0; i < nn; ++i) { if (flow[i] > mx) mx = flow[i]; if (distance[i] > mx) mx = distance[i]; }
  if (mx >= (1 << 16)) sym = false;
  const bool bytes = mx < 256 && (double)n * (double)mx * (double)mx < 2147483648.0;
  QSB_TRY(h.b[6].ensure(P * n * 2 + P * 8 + 16));
  QSB_TRY(h.b[7].ensure(2 * nn * 8));
  const bool narrow = mx < (1 << 16);   // uint16 device matrices when exact
  int16_t* dp = (int16_t*)h.b[6].p;
  int64_t* dc = (int64_t*)((char*)h.b[6].p + align_up(P * n * 2, 16));
  std::vector<int16_t> hp((size_t)(P * n));
  for (int64_t i = 0; i < P * n; ++i) hp[(size_t)i] = (int16_t)perms[i];
  QSB_CUDA(cudaMemcpyAsync(dp, hp.data(), P * n * 2, cudaMemcpyHostToDevice, s));
  QSB_CUDA(cudaMemcpyAsync(dc, costs, P * 8, cudaMemcpyHostToDevice, s));
  std::vector<uint16_t> narrow_fd;
  if (narrow) {
    narrow_fd.resize((size_t)(2 * nn));
    for (int64_t i = 0; i < nn; ++i) { narrow_fd[(size_t)i] = (uint16_t)flow[i]; narrow_fd[(size_t)(nn + i)] = (uint16_t)distance[i]; }
    QSB_CUDA(cudaMemcpyAsync(h.b[7].p, narrow_fd.data(), 2 * nn * 2, cudaMemcpyHostToDevice, s));
  } else {
    QSB_CUDA(cudaMemcpyAsync(h.b[7].p, flow, nn * 8, cudaMemcpyHostToDevice, s));
    QSB_CUDA(cudaMemcpyAsync((char*)h.b[7].p + nn * 8, distance, nn * 8, cudaMemcpyHostToDevice, s));
  }
  TwoOptArgs t{};
  t.n = n; t.P = P; t.passes = passes; t.sym = sym ? 1 : 0; t.do_pbest = 0;
  t.perm = dp; t.cost = dc;
  t.F = h.b[7].p;
  t.D = (char*)h.b[7].p + nn * (narrow ? 2 : 8);
  if (narrow) QSB_TRY(dispatch_twoopt<uint16_t>(t, s, bytes));
  else QSB_TRY(dispatch_twoopt<int64_t>(t, s));
  QSB_CUDA(cudaMemcpyAsync(hp.data(), dp, P * n * 2, cudaMemcpyDeviceToHost, s));
  QSB_CUDA(cudaMemcpyAsync(costs, dc, P * 8, cudaMemcpyDeviceToHost, s));
  QSB_CUDA(cudaStreamSynchronize(s));
  for (int64_t i = 0; i < P * n; ++i) perms[i] = hp[(size_t)i];
  return QSB_OK;
}

}  // extern "C"

