// frb_kernels.cu -- the C-ABI entry points (include/frb200.h), launch-group
// dispatch, and the one-shot force / arithmetic self-test kernels.  The
// relaxation kernel itself is frb_relax.cuh, instantiated per CTA size in
// frb_k256.cu, frb_k512.cu, frb_k768.cu, frb_k1024.cu and frb_kenergy.cu.

#include "frb_relax.cuh"

namespace frb_tu {
thread_local char g_err[512] = "";
thread_local int g_launches = 0;
}  // namespace frb_tu

using frb_tu::g_err;

namespace {

// One-shot forces for every node of problem blockIdx.x (reference
// internal_forces, microsolver.py:221-238), same element math as the solver.
__global__ void __launch_bounds__(256) frb_forces_kernel(const __grid_constant__ frb_batch b, const double* __restrict__ u,
                                                          double* __restrict__ f) {
  __shared__ Scalars sc;
  __shared__ Net n;
  __shared__ Rank rk;
  __shared__ int any_bad;
  const int p = blockIdx.x;
  if (threadIdx.x == 0) {
    load_views(n, rk, b, p, 0);
    any_bad = 0;
  }
  __syncthreads();
  const PosGlobal pos{n.X, u + 3 * n.node_base};
  double* fp = f + 3 * n.node_base;
  bool bad = false;
  for (int i = threadIdx.x; i < n.N; i += blockDim.x) {
    double fx, fy, fz;
    bad |= node_force_csr(n, pos, i, fx, fy, fz);
    fp[3 * i] = fx;
    fp[3 * i + 1] = fy;
    fp[3 * i + 2] = fz;
  }
  if (bad) any_bad = 1;
  __syncthreads();
  int badi = -1;
  if (any_bad) badi = singular_argmin(n, pos, sc);
  if (threadIdx.x == 0) {
    b.results[p].status = badi >= 0 ? FRB_STATUS_SINGULAR : FRB_STATUS_CONVERGED;
    b.results[p].bad_element = badi;
  }
}

// out[6*i + ...]: div_fast, div ok flag, __ddiv_rn, sqrt_fast, sqrt ok flag, __dsqrt_rn
__global__ void arith_selftest_kernel(const double* a, const double* b, int n, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool ok;
  out[6 * i] = frb_arith::div_fast(a[i], b[i], ok);
  out[6 * i + 1] = ok ? 1.0 : 0.0;
  out[6 * i + 2] = __ddiv_rn(a[i], b[i]);
  out[6 * i + 3] = frb_arith::sqrt_fast(a[i], ok);
  out[6 * i + 4] = ok ? 1.0 : 0.0;
  out[6 * i + 5] = __dsqrt_rn(a[i]);
}

}  // namespace


extern "C" {

int frb_abi_version(void) { return FRB_ABI_VERSION; }

const char* frb_last_error(void) { return g_err; }

int frb_solve_launches(void) { return frb_tu::g_launches; }

int frb_device_info(int device, int* n_sm, int* smem_optin, int* cc_major, int* cc_minor) {
  cudaDeviceProp prop;
  int rc = cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
  if (rc) return rc;
  if (n_sm) *n_sm = prop.multiProcessorCount;
  if (smem_optin) *smem_optin = static_cast<int>(prop.sharedMemPerBlockOptin);
  if (cc_major) *cc_major = prop.major;
  if (cc_minor) *cc_minor = prop.minor;
  return FRB_OK;
}

int64_t frb_rank_smem_bytes(int32_t n_pos, int32_t n_own, int32_t n_act, int32_t n_slots, int32_t n_prog,
                            int32_t mode) {
  const int64_t nf = 3 * static_cast<int64_t>(n_own);
  return 8 * (3 * static_cast<int64_t>(n_pos) + ((mode & 1) ? 1 : 2) * nf + (nf > n_act ? nf : n_act) +
              ((mode & 2) ? 1 : 2) * n_own +
              3 * static_cast<int64_t>(n_slots) + 160) +
         4 * ((static_cast<int64_t>(n_prog) + 1) & ~1LL);
}

int frb_max_dofs_per_thread(int block_threads, int fprv_global) { return dofs_cap(block_threads, fprv_global != 0); }

}  // extern "C"

namespace {

// One launch group on stream s (validated, dispatched to its instantiation).
// alone: the group has the GPU to itself, so its virtual clusters (which
// need all their CTAs resident at once) can count on the SMs its hardware
// clusters leave idle; groups running concurrently never use them.
int launch_one(const frb_batch* batch, const frb_config* cfg, int gi, int optin, cudaStream_t s, bool alone) {
  frb_group g = batch->groups[gi];
  if (!alone) g.flags |= FRB_GF_NO_VIRTUAL;
  int rc = FRB_OK;
  if (g.cluster < 1 || g.cluster > FRB_MAX_CLUSTER) return set_err(FRB_E_INVALID, "cluster size out of range");
  if (g.block_threads < 32 || g.block_threads > kMaxThreads || g.block_threads % 32)
    return set_err(FRB_E_INVALID, "block_threads must be a multiple of 32 in [32, 1024]");
  if (g.smem_bytes > optin) return set_err(FRB_E_TOO_LARGE, "a rank exceeds shared memory per CTA");
  int32_t* q = batch->queue + gi;
  if (cfg->energy_check_interval > 0) {
    // work-ledger kernels (a diagnostic, kept out of the production
    // kernels' code): CTAs of at most 512 threads, up to 16 DOFs each
    const int T = g.block_threads < 512 ? g.block_threads : 512;
    const int ke = (g.max_own_dofs + T - 1) / T;
    if (ke > 16) return set_err(FRB_E_TOO_LARGE, "too many free DOFs per thread for the ledger kernels");
    return frb_tu::dispatch_energy(batch, cfg, g, q, s, T, ke);
  }
  // production kernels run with exactly MAXT threads (the template's CTA
  // size, >= block_threads): DOFs per thread follow from that
  const int tpl = g.block_threads <= 256 ? 256 : g.block_threads <= 512 ? 512 : g.block_threads <= 768 ? 768 : 1024;
  const int k = (g.max_own_dofs + tpl - 1) / tpl;
  if (k > dofs_cap(g.block_threads, g.fprv_global != 0)) return set_err(FRB_E_TOO_LARGE, "too many free DOFs per thread");
  if (g.block_threads <= 256) rc = frb_tu::dispatch_256(batch, cfg, g, q, s, k);
  else if (g.block_threads <= 512) rc = frb_tu::dispatch_512(batch, cfg, g, q, s, k);
  else if (g.block_threads <= 768) rc = frb_tu::dispatch_768(batch, cfg, g, q, s, k);
  else rc = frb_tu::dispatch_1024(batch, cfg, g, q, s, k);
  return rc;
}

}  // namespace

extern "C" {

int frb_solve_batch(const frb_batch* batch, const frb_config* cfg, void* stream) {
  if (!batch || !cfg) return set_err(FRB_E_INVALID, "null batch or config");
  frb_tu::g_launches = 0;
  if (batch->n_problems < 0 || batch->n_groups < 0) return set_err(FRB_E_INVALID, "negative counts");
  if (batch->n_problems == 0) return FRB_OK;
  if (!batch->groups || !batch->queue || !batch->work) return set_err(FRB_E_INVALID, "groups/queue/work missing");
  if (cfg->max_iters <= 0) return set_err(FRB_E_INVALID, "max_iters must be > 0");
  int dev = 0, optin = 0;
  int rc = cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  if (rc) return rc;
  rc = cuda_check(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev),
                  "cudaDeviceGetAttribute");
  if (rc) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int n_live = 0;
  bool serial = false;
  for (int gi = 0; gi < batch->n_groups; ++gi) {
    n_live += batch->groups[gi].count > 0;
    serial |= (batch->groups[gi].flags & FRB_GF_SERIAL) != 0;
  }
  if (n_live <= 1 || serial) {
    for (int gi = 0; gi < batch->n_groups; ++gi)
      if (batch->groups[gi].count > 0 && (rc = launch_one(batch, cfg, gi, optin, s, n_live <= 1))) return rc;
    return FRB_OK;
  }
  // Several cluster sizes (heterogeneous batch).  Groups of 16-CTA clusters
  // that may use virtual clusters run last, one after another, each alone
  // (7 hardware clusters + virtual clusters on the 36 SMs they leave idle);
  // concurrently with smaller groups those 36 SMs were all the small
  // networks got (c4: 2.27 s against 0.52 s + the 16-CTA groups alone).
  // The other groups run concurrently on forked streams, largest clusters
  // launched first, joined back into s.
  auto last = [&](const frb_group& g) {
    return g.cluster >= 16 && g.gm_cap > 0 && batch->xchg && !(g.flags & FRB_GF_NO_VIRTUAL) &&
           cfg->energy_check_interval <= 0 && !batch->phase_cycles;
  };
  cudaEvent_t fork;
  rc = cuda_check(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming), "cudaEventCreate");
  if (rc) return rc;
  rc = cuda_check(cudaEventRecord(fork, s), "cudaEventRecord");
  for (int gi = batch->n_groups - 1; gi >= 0 && !rc; --gi) {
    if (batch->groups[gi].count == 0 || last(batch->groups[gi])) continue;
    cudaStream_t gs;
    cudaEvent_t join;
    rc = cuda_check(cudaStreamCreateWithFlags(&gs, cudaStreamNonBlocking), "cudaStreamCreate");
    if (rc) break;
    rc = cuda_check(cudaStreamWaitEvent(gs, fork, 0), "cudaStreamWaitEvent");
    if (!rc) rc = launch_one(batch, cfg, gi, optin, gs, false);
    if (!rc) rc = cuda_check(cudaEventCreateWithFlags(&join, cudaEventDisableTiming), "cudaEventCreate");
    if (!rc) {
      rc = cuda_check(cudaEventRecord(join, gs), "cudaEventRecord");
      if (!rc) rc = cuda_check(cudaStreamWaitEvent(s, join, 0), "cudaStreamWaitEvent");
      cudaEventDestroy(join);  // released once recorded work completes
    }
    cudaStreamDestroy(gs);     // likewise: pending work still runs
  }
  cudaEventDestroy(fork);
  for (int gi = batch->n_groups - 1; gi >= 0 && !rc; --gi)  // after every forked group (stream order on s)
    if (batch->groups[gi].count > 0 && last(batch->groups[gi])) rc = launch_one(batch, cfg, gi, optin, s, true);
  return rc;
}

int frb_selftest_arith(const double* a, const double* b, int n, double* out, void* stream) {
  if (n <= 0) return FRB_OK;
  if (!a || !b || !out) return set_err(FRB_E_INVALID, "null argument");
  arith_selftest_kernel<<<(n + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(a, b, n, out);
  return cuda_check(cudaGetLastError(), "arith_selftest_kernel launch");
}

int frb_internal_forces(const frb_batch* batch, const double* u, double* f, void* stream) {
  if (!batch || !u || !f) return set_err(FRB_E_INVALID, "null argument");
  if (batch->n_problems <= 0) return FRB_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int rc = cuda_check(cudaMemsetAsync(batch->results, 0, sizeof(frb_result) * batch->n_problems, s),
                      "cudaMemsetAsync");
  if (rc) return rc;
  frb_forces_kernel<<<batch->n_problems, 256, 0, s>>>(*batch, u, f);
  return cuda_check(cudaGetLastError(), "frb_forces_kernel launch");
}

}  // extern "C"
