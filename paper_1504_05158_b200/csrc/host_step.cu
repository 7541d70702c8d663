// host_step.cu -- qsb_step_host: one engine.step on the reference's HOST
// buffers (engine.PopulationState, engine.py:85-124; step, engine.py:181-244).
//
// This is the Level-1 drop-in a maintainer binds when the population stays
// in host memory in the reference layout (float64 V, int8 0/1 matrices,
// int64 permutations).  Every call moves the state through PCIe: the
// particles are cut into swarm-aligned chunks and three streams overlap the
// host->device copy of chunk c+1, the fused fp64 step of chunk c and the
// device->host copy of chunk c-1.  The arithmetic is the parity mode
// (bit-identical to the reference); draws, goal, bests and migration all run
// on the device, the host only copies rows it must (PL rows of improved
// particles, swarm-best matrices).
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/qapswarm_b200.h"

void qsb_note_cuda_error(int e);   // qsb_api.cu

namespace {

__global__ void narrow_kernel(const int64_t* __restrict__ in, int16_t* __restrict__ out, int64_t count) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int16_t)in[i];
}

__global__ void widen_kernel(const int16_t* __restrict__ in, int64_t* __restrict__ out, int64_t count) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int64_t)in[i];
}

int cu(cudaError_t e) {
  if (e == cudaSuccess) return QSB_OK;
  qsb_note_cuda_error((int)e);     // reported by qsb_strerror / qsb_last_cuda_error
  return QSB_ECUDA;
}

#define HS_TRY(x) do { int _rc = (x); if (_rc) return _rc; } while (0)
#define HS_CUDA(x) do { int _rc = cu(x); if (_rc) return _rc; } while (0)

int grid_for(int64_t count) {
  const int64_t g = (count + 255) / 256;
  return (int)(g < 1184 ? (g > 0 ? g : 1) : 1184);
}

struct Buf {
  void* p = nullptr;
  size_t cap = 0;
  int ensure(size_t bytes) {
    if (bytes <= cap) return QSB_OK;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    HS_CUDA(cudaMalloc(&p, bytes ? bytes : 16));
    cap = bytes;
    return QSB_OK;
  }
  template <typename T> T* as(size_t off_bytes = 0) const { return (T*)((char*)p + off_bytes); }
};

constexpr int MAX_CHUNKS = 64;

struct Ctx {
  std::mutex mu;
  cudaStream_t s_in = nullptr, s_comp = nullptr, s_out = nullptr;
  cudaEvent_t ev_in[MAX_CHUNKS], ev_comp[MAX_CHUNKS], ev_out[MAX_CHUNKS], ev_pg;
  bool init_done = false;
  Buf V, perm, perm_new, pl_perm, in64, pl64, cost, pl_cost, improved, xnew;
  Buf pg_perm, pg64, pg_cost, best, iters, swarm_min, swarm_min_idx, misc, coef, fd, mig;
  int64_t* h_iters = nullptr;   // pinned: per-chunk t - 1
  int init() {
    if (init_done) return QSB_OK;
    HS_CUDA(cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking));
    HS_CUDA(cudaStreamCreateWithFlags(&s_comp, cudaStreamNonBlocking));
    HS_CUDA(cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking));
    for (int c = 0; c < MAX_CHUNKS; ++c) {
      HS_CUDA(cudaEventCreateWithFlags(&ev_in[c], cudaEventDisableTiming));
      HS_CUDA(cudaEventCreateWithFlags(&ev_comp[c], cudaEventDisableTiming));
      HS_CUDA(cudaEventCreateWithFlags(&ev_out[c], cudaEventDisableTiming));
    }
    HS_CUDA(cudaEventCreateWithFlags(&ev_pg, cudaEventDisableTiming));
    HS_CUDA(cudaMallocHost(&h_iters, MAX_CHUNKS * sizeof(int64_t)));
    init_done = true;
    return QSB_OK;
  }
};

Ctx& ctx() {
  static Ctx c;
  return c;
}

int chunks_wanted() {
  const char* e = std::getenv("QSB_HOST_CHUNKS");
  int k = e ? std::atoi(e) : 16;   // 16: best of 8 / 16 / 32 / 64 at config 3 (profiles/r02/host_e2e_sweep.json)
  if (k < 1) k = 1;
  if (k > MAX_CHUNKS) k = MAX_CHUNKS;
  return k;
}

}  // namespace

extern "C" {

int qsb_step_host(qsb_host_population* hp, const qsb_host_instance* hi, const qsb_coeffs* co,
                  uint64_t t, int32_t migrate_d, double* migration_log) {
  if (!hp || !hi || !co) return QSB_EINVAL;
  const int n = hp->n;
  const int64_t P = hp->num_particles, S = hp->swarm_size, m = hp->num_swarms;
  if (n < 2 || hi->n != n || S < 1 || m < 1 || P != m * S) return QSB_EINVAL;
  if (hp->cost_dtype != QSB_I64 && hp->cost_dtype != QSB_F64) return QSB_EINVAL;
  if (!hp->V || !hp->X_new || !hp->PL || !hp->perms || !hp->perms_new || !hp->pl_perms || !hp->improved ||
      !hp->cost || !hp->pl_cost || !hp->pg_mats || !hp->pg_perms || !hp->pg_costs ||
      !hp->best_perm || !hp->best_cost || !hp->best_iteration || !hi->flow || !hi->distance)
    return QSB_EINVAL;
  if (migrate_d < 0 || (migrate_d > 0 && (2 * (int64_t)migrate_d >= m || !migration_log)))
    return QSB_EINVAL;
  if (co->sx_mode < 0 || co->sx_mode > 2) return QSB_EINVAL;
  Ctx& c = ctx();
  std::lock_guard<std::mutex> lock(c.mu);
  HS_TRY(c.init());
  const int64_t nn = (int64_t)n * n;
  const int32_t vs = qsb_vstride(n, QSB_F64);
  const size_t csz = 8;

  // ---- device buffers (grown on demand, kept between calls)
  HS_TRY(c.V.ensure((size_t)P * vs * 8));
  HS_TRY(c.perm.ensure((size_t)P * n * 2));
  HS_TRY(c.perm_new.ensure((size_t)P * n * 2));
  HS_TRY(c.pl_perm.ensure((size_t)P * n * 2));
  HS_TRY(c.in64.ensure((size_t)P * n * 8));
  HS_TRY(c.pl64.ensure((size_t)P * n * 8));
  HS_TRY(c.cost.ensure((size_t)P * csz));
  HS_TRY(c.pl_cost.ensure((size_t)P * csz));
  HS_TRY(c.improved.ensure((size_t)P));
  HS_TRY(c.xnew.ensure((size_t)P * nn));
  HS_TRY(c.pg_perm.ensure((size_t)m * n * 2));
  HS_TRY(c.pg64.ensure((size_t)(m + 1) * n * 8));       // + the best permutation
  HS_TRY(c.pg_cost.ensure((size_t)m * csz));
  HS_TRY(c.best.ensure(64 + (size_t)n * 2));             // cost, iter, idx, perm
  HS_TRY(c.iters.ensure(MAX_CHUNKS * 8));
  HS_TRY(c.swarm_min.ensure((size_t)m * csz));
  HS_TRY(c.swarm_min_idx.ensure((size_t)m * 8));
  HS_TRY(c.misc.ensure(64));                             // done, work
  HS_TRY(c.coef.ensure((size_t)P * 16));
  // instance in the narrowest exact device format (instance.device_format)
  int mat = hi->mat_dtype;
  bool u16 = false;
  int64_t fmax = 0, dmax = 0;
  if (mat == QSB_I64) {
    const int64_t* f = (const int64_t*)hi->flow;
    const int64_t* d = (const int64_t*)hi->distance;
    bool ok = true;
    for (int64_t i = 0; i < nn; ++i) {
      if (f[i] < 0 || f[i] >= 65536 || d[i] < 0 || d[i] >= 65536) { ok = false; break; }
      if (f[i] > fmax) fmax = f[i];
      if (d[i] > dmax) dmax = d[i];
    }
    u16 = ok;
  } else if (mat != QSB_F64) {
    return QSB_EINVAL;
  }
  HS_TRY(c.fd.ensure((size_t)2 * nn * 8));
  static thread_local std::vector<uint16_t> fd16;
  if (u16) {
    fd16.resize((size_t)2 * nn);
    const int64_t* f = (const int64_t*)hi->flow;
    const int64_t* d = (const int64_t*)hi->distance;
    for (int64_t i = 0; i < nn; ++i) { fd16[i] = (uint16_t)f[i]; fd16[nn + i] = (uint16_t)d[i]; }
    HS_CUDA(cudaMemcpyAsync(c.fd.p, fd16.data(), (size_t)2 * nn * 2, cudaMemcpyHostToDevice, c.s_comp));
  } else {
    HS_CUDA(cudaMemcpyAsync(c.fd.p, hi->flow, (size_t)nn * 8, cudaMemcpyHostToDevice, c.s_comp));
    HS_CUDA(cudaMemcpyAsync(c.fd.as<char>((size_t)nn * 8), hi->distance, (size_t)nn * 8,
                            cudaMemcpyHostToDevice, c.s_comp));
  }
  qsb_instance inst{};
  inst.n = n;
  inst.mat_dtype = u16 ? QSB_U16 : mat;
  inst.flow = c.fd.p;
  inst.distance = c.fd.as<char>((size_t)nn * (u16 ? 2 : 8));
  inst.acc32 = u16 ? (int)((double)n * (double)fmax * (double)dmax < 4294967296.0) : 0;
  if (!qsb_supported(n, QSB_F64, inst.mat_dtype)) return QSB_EUNSUPPORTED;

  // ---- swarm-aligned chunks
  int K = chunks_wanted();
  if (K > m) K = (int)m;
  const int64_t cs = (m + K - 1) / K;
  K = (int)((m + cs - 1) / cs);

  // swarm bests and the best record (needed by every chunk's best update)
  HS_CUDA(cudaMemcpyAsync(c.pg64.p, hp->pg_perms, (size_t)m * n * 8, cudaMemcpyHostToDevice, c.s_comp));
  HS_CUDA(cudaMemcpyAsync(c.pg64.as<int64_t>((size_t)m * n * 8), hp->best_perm, (size_t)n * 8,
                          cudaMemcpyHostToDevice, c.s_comp));
  HS_CUDA(cudaMemcpyAsync(c.pg_cost.p, hp->pg_costs, (size_t)m * csz, cudaMemcpyHostToDevice, c.s_comp));
  HS_CUDA(cudaMemcpyAsync(c.best.p, hp->best_cost, 8, cudaMemcpyHostToDevice, c.s_comp));
  HS_CUDA(cudaMemcpyAsync(c.best.as<char>(8), hp->best_iteration, 8, cudaMemcpyHostToDevice, c.s_comp));
  narrow_kernel<<<grid_for((m + 1) * n), 256, 0, c.s_comp>>>(c.pg64.as<int64_t>(), c.pg_perm.as<int16_t>(),
                                                             m * n);
  narrow_kernel<<<grid_for(n), 256, 0, c.s_comp>>>(c.pg64.as<int64_t>((size_t)m * n * 8),
                                                   c.best.as<int16_t>(32), n);
  HS_CUDA(cudaMemsetAsync(c.misc.p, 0, 64, c.s_comp));
  for (int k = 0; k < K; ++k) c.h_iters[k] = (int64_t)t - 1;
  HS_CUDA(cudaMemcpyAsync(c.iters.p, c.h_iters, (size_t)K * 8, cudaMemcpyHostToDevice, c.s_comp));

  qsb_state base{};
  base.n = n; base.vstride = vs; base.v_dtype = QSB_F64; base.cost_dtype = hp->cost_dtype;
  base.swarm_size = S;
  qsb_coeffs cf = *co;
  cf.hints = 0;     // host state: no velocity bound or current-goal guarantee is assumed
  const int flags = QSB_PHASE_VELOCITY | QSB_PHASE_AGGREGATE | QSB_PHASE_COST | QSB_PHASE_PBEST |
                    QSB_PHASE_STORE_V;

  for (int k = 0; k < K; ++k) {
    const int64_t s0 = k * cs, s1 = (s0 + cs < m) ? s0 + cs : m;
    const int64_t p0 = s0 * S, pc = (s1 - s0) * S;
    // host -> device: V, positions, personal bests
    if (vs == nn) {
      HS_CUDA(cudaMemcpyAsync(c.V.as<double>((size_t)p0 * vs * 8), hp->V + p0 * nn, (size_t)pc * nn * 8,
                              cudaMemcpyHostToDevice, c.s_in));
    } else {
      HS_CUDA(cudaMemcpy2DAsync(c.V.as<double>((size_t)p0 * vs * 8), (size_t)vs * 8, hp->V + p0 * nn,
                                (size_t)nn * 8, (size_t)nn * 8, (size_t)pc, cudaMemcpyHostToDevice, c.s_in));
    }
    HS_CUDA(cudaMemcpyAsync(c.in64.as<int64_t>((size_t)p0 * n * 8), hp->perms + p0 * n, (size_t)pc * n * 8,
                            cudaMemcpyHostToDevice, c.s_in));
    HS_CUDA(cudaMemcpyAsync(c.pl64.as<int64_t>((size_t)p0 * n * 8), hp->pl_perms + p0 * n,
                            (size_t)pc * n * 8, cudaMemcpyHostToDevice, c.s_in));
    HS_CUDA(cudaMemcpyAsync(c.pl_cost.as<char>((size_t)p0 * csz), (const char*)hp->pl_cost + p0 * csz,
                            (size_t)pc * csz, cudaMemcpyHostToDevice, c.s_in));
    HS_CUDA(cudaEventRecord(c.ev_in[k], c.s_in));

    // device: narrow, fused step (fp64 parity arithmetic), bests, X_new, widen
    HS_CUDA(cudaStreamWaitEvent(c.s_comp, c.ev_in[k], 0));
    narrow_kernel<<<grid_for(pc * n), 256, 0, c.s_comp>>>(c.in64.as<int64_t>((size_t)p0 * n * 8),
                                                          c.perm.as<int16_t>((size_t)p0 * n * 2), pc * n);
    narrow_kernel<<<grid_for(pc * n), 256, 0, c.s_comp>>>(c.pl64.as<int64_t>((size_t)p0 * n * 8),
                                                          c.pl_perm.as<int16_t>((size_t)p0 * n * 2), pc * n);
    qsb_state st = base;
    st.num_particles = pc;
    st.num_swarms = s1 - s0;
    st.particle_offset = p0;
    st.swarm_offset = s0;
    st.V = c.V.as<double>((size_t)p0 * vs * 8);
    st.perm = c.perm.as<int16_t>((size_t)p0 * n * 2);
    st.perm_new = c.perm_new.as<int16_t>((size_t)p0 * n * 2);
    st.pl_perm = c.pl_perm.as<int16_t>((size_t)p0 * n * 2);
    st.cost = c.cost.as<char>((size_t)p0 * csz);
    st.pl_cost = c.pl_cost.as<char>((size_t)p0 * csz);
    st.improved = c.improved.as<uint8_t>((size_t)p0);
    st.pg_perm = c.pg_perm.as<int16_t>((size_t)s0 * n * 2);
    st.pg_cost = c.pg_cost.as<char>((size_t)s0 * csz);
    st.best_cost = c.best.p;
    st.best_iter = c.best.as<int64_t>(8);
    st.best_idx = c.best.as<int64_t>(16);
    st.best_perm = c.best.as<int16_t>(32);
    st.swarm_min = c.swarm_min.as<char>((size_t)s0 * csz);
    st.swarm_min_idx = c.swarm_min_idx.as<int64_t>((size_t)s0 * 8);
    st.done = c.misc.as<uint32_t>(0);
    st.work = c.misc.as<uint32_t>(8);
    st.step_coef = c.coef.as<double>((size_t)p0 * 16);
    st.vcol = nullptr;
    st.iteration = nullptr;                        // the step reads t from t_host
    HS_TRY(qsb_step_phases(&st, &inst, &cf, flags, nullptr, 0, 2, nullptr, t, c.s_comp));
    st.iteration = c.iters.as<int64_t>((size_t)k * 8);   // t - 1, advanced to t by the update
    HS_TRY(qsb_best_update(&st, c.s_comp));
    HS_TRY(qsb_perm_to_matrix(st.perm_new, pc, n, c.xnew.as<int8_t>((size_t)p0 * nn), c.s_comp));
    widen_kernel<<<grid_for(pc * n), 256, 0, c.s_comp>>>(st.perm_new, c.in64.as<int64_t>((size_t)p0 * n * 8),
                                                         pc * n);
    widen_kernel<<<grid_for(pc * n), 256, 0, c.s_comp>>>(st.pl_perm, c.pl64.as<int64_t>((size_t)p0 * n * 8),
                                                         pc * n);
    HS_CUDA(cudaGetLastError());
    HS_CUDA(cudaEventRecord(c.ev_comp[k], c.s_comp));

    // device -> host
    HS_CUDA(cudaStreamWaitEvent(c.s_out, c.ev_comp[k], 0));
    if (vs == nn) {
      HS_CUDA(cudaMemcpyAsync(hp->V + p0 * nn, c.V.as<double>((size_t)p0 * vs * 8), (size_t)pc * nn * 8,
                              cudaMemcpyDeviceToHost, c.s_out));
    } else {
      HS_CUDA(cudaMemcpy2DAsync(hp->V + p0 * nn, (size_t)nn * 8, c.V.as<double>((size_t)p0 * vs * 8),
                                (size_t)vs * 8, (size_t)nn * 8, (size_t)pc, cudaMemcpyDeviceToHost, c.s_out));
    }
    HS_CUDA(cudaMemcpyAsync(hp->X_new + p0 * nn, c.xnew.as<int8_t>((size_t)p0 * nn), (size_t)pc * nn,
                            cudaMemcpyDeviceToHost, c.s_out));
    HS_CUDA(cudaMemcpyAsync(hp->perms_new + p0 * n, c.in64.as<int64_t>((size_t)p0 * n * 8),
                            (size_t)pc * n * 8, cudaMemcpyDeviceToHost, c.s_out));
    HS_CUDA(cudaMemcpyAsync(hp->pl_perms + p0 * n, c.pl64.as<int64_t>((size_t)p0 * n * 8),
                            (size_t)pc * n * 8, cudaMemcpyDeviceToHost, c.s_out));
    HS_CUDA(cudaMemcpyAsync((char*)hp->cost + p0 * csz, c.cost.as<char>((size_t)p0 * csz), (size_t)pc * csz,
                            cudaMemcpyDeviceToHost, c.s_out));
    HS_CUDA(cudaMemcpyAsync((char*)hp->pl_cost + p0 * csz, c.pl_cost.as<char>((size_t)p0 * csz),
                            (size_t)pc * csz, cudaMemcpyDeviceToHost, c.s_out));
    HS_CUDA(cudaMemcpyAsync(hp->improved + p0, c.improved.as<uint8_t>((size_t)p0), (size_t)pc,
                            cudaMemcpyDeviceToHost, c.s_out));
    HS_CUDA(cudaEventRecord(c.ev_out[k], c.s_out));
  }

  // migration (migration.py:55-86) on the post-step positions, picks drawn
  // on the device from host_rng(seed, t)
  if (migrate_d > 0) {
    HS_TRY(c.mig.ensure((size_t)migrate_d * (4 * 8 + 6 * 8) + 64));
    int64_t* plan = c.mig.as<int64_t>();
    double* log = c.mig.as<double>((size_t)migrate_d * 32);
    int64_t* log_count = c.mig.as<int64_t>((size_t)migrate_d * 80);
    int32_t* status = c.mig.as<int32_t>((size_t)migrate_d * 80 + 8);
    HS_CUDA(cudaMemsetAsync(log_count, 0, 16, c.s_comp));
    qsb_state st = base;
    st.num_particles = P; st.num_swarms = m; st.particle_offset = 0; st.swarm_offset = 0;
    st.perm = c.perm_new.as<int16_t>();           // current positions after the swap
    st.cost = c.cost.p;
    st.pg_perm = c.pg_perm.as<int16_t>();
    st.pg_cost = c.pg_cost.p;
    st.iteration = c.iters.as<int64_t>((size_t)(K - 1) * 8);    // == t
    qsb_migration mg{};
    mg.d = migrate_d; mg.period = 0; mg.mode = 0;
    mg.num_swarms_total = m;
    mg.picks = nullptr;
    mg.seed = co->seed;
    mg.all_pg_cost = c.pg_cost.p;
    mg.plan = plan; mg.records = nullptr;
    mg.log = log; mg.log_rows = 1; mg.log_count = log_count; mg.status = status;
    HS_TRY(qsb_migrate(&st, &mg, c.s_comp));
    HS_CUDA(cudaMemcpyAsync(migration_log, log, (size_t)migrate_d * 48, cudaMemcpyDeviceToHost, c.s_comp));
  }
  widen_kernel<<<grid_for(m * n), 256, 0, c.s_comp>>>(c.pg_perm.as<int16_t>(), c.pg64.as<int64_t>(), m * n);
  widen_kernel<<<grid_for(n), 256, 0, c.s_comp>>>(c.best.as<int16_t>(32),
                                                  c.pg64.as<int64_t>((size_t)m * n * 8), n);
  HS_CUDA(cudaGetLastError());
  HS_CUDA(cudaMemcpyAsync(hp->pg_perms, c.pg64.p, (size_t)m * n * 8, cudaMemcpyDeviceToHost, c.s_comp));
  HS_CUDA(cudaMemcpyAsync(hp->best_perm, c.pg64.as<int64_t>((size_t)m * n * 8), (size_t)n * 8,
                          cudaMemcpyDeviceToHost, c.s_comp));
  HS_CUDA(cudaMemcpyAsync(hp->pg_costs, c.pg_cost.p, (size_t)m * csz, cudaMemcpyDeviceToHost, c.s_comp));
  HS_CUDA(cudaMemcpyAsync(hp->best_cost, c.best.p, 8, cudaMemcpyDeviceToHost, c.s_comp));
  HS_CUDA(cudaMemcpyAsync(hp->best_iteration, c.best.as<char>(8), 8, cudaMemcpyDeviceToHost, c.s_comp));
  HS_CUDA(cudaEventRecord(c.ev_pg, c.s_comp));

  // host: personal-best matrices of the improved particles (engine.py:212),
  // chunk by chunk as their copies land
  for (int k = 0; k < K; ++k) {
    HS_CUDA(cudaEventSynchronize(c.ev_out[k]));
    const int64_t s0 = k * cs, s1 = (s0 + cs < m) ? s0 + cs : m;
    for (int64_t p = s0 * S; p < s1 * S; ++p)
      if (hp->improved[p]) std::memcpy(hp->PL + p * nn, hp->X_new + p * nn, (size_t)nn);
  }
  // swarm-best matrices from their permutations (X[k, i] = 1 iff k == perm[i])
  HS_CUDA(cudaEventSynchronize(c.ev_pg));
  std::memset(hp->pg_mats, 0, (size_t)m * nn);
  for (int64_t s = 0; s < m; ++s)
    for (int i = 0; i < n; ++i) hp->pg_mats[s * nn + hp->pg_perms[s * n + i] * n + i] = 1;
  return QSB_OK;
}

}  // extern "C"
