// frb_naive.cu -- the NaiveLoop strategy on the device: one kernel launch per
// line of the reference's Fig. 1 loop, problems strictly one after another.
//
// This is the paper's per-operation baseline (Figs. 2 and 4)
// and the spec's NaiveLoop: "within each Fig. 1 line, the
// per-DOF/element loop is split across all workers with a full cross-worker
// barrier per line (models one kernel dispatch per operation)".  Here the
// workers are every thread of the GPU and the barrier is the kernel boundary;
// the host drives the iteration and reads the convergence flag after every
// iteration, as a naive accelerator port does.  It exists to be measured
// against the persistent team kernel (frb_relax.cuh), not to be fast.
//
// Per iteration (reference pkg/src/fibrelax/microsolver.py:434-530):
//   nv_coefs    _element_force_coefficients (:196-211), every element
//   nv_forces   _scatter_forces (:214-218) as the per-node gather in element
//               order (role a then role b), free nodes
//   nv_dofs     adaptive-damping terms k_hat, (u k_hat) u, (u m) u and f f
//               (:467-489); f becomes f_prev
//   nv_reduce   the three np.sum pairwise trees (plan.py) and the scalar
//               bookkeeping: c, residual, r_ref / threshold, convergence
//   nv_update   accelerations, the second half-kick, the next half-kick and
//               drift, the BC ramp (:443-454, :501-507)
// Every operation is the fused kernel's, in the same order, with the same
// correctly rounded intrinsics, so the results are bit-identical to
// TeamBatched (tests/test_gpu_naive.py).

#include "frb_relax.cuh"

namespace {

// Device-side scalars of the problem being solved.
struct NaiveState {
  double c, residual, r_ref, threshold, alpha;
  int done, converged, singular, it;
};

constexpr int kNT = 256;

__device__ __forceinline__ void load_net(Net& n, Rank& r, const frb_batch& b, int p) {
  if (threadIdx.x == 0) load_views(n, r, b, p, 0);
  __syncthreads();
}

// positions X + u of every node (u holds the fixed nodes' prescribed values)
struct PosXU {
  const double* X;
  const double* u;
  __device__ __forceinline__ double operator()(int node, int axis) const {
    return dadd(X[3 * node + axis], u[3 * node + axis]);
  }
};

// u of the fixed nodes for ramp factor alpha (alpha < 0: zero before the ramp)
__global__ void __launch_bounds__(kNT) nv_fixed(const __grid_constant__ frb_batch b, int p, double alpha, int ramp) {
  __shared__ Net n;
  __shared__ Rank r;
  load_net(n, r, b, p);
  double* u = b.u + 3 * n.node_base;
  for (int i = n.NF + blockIdx.x * blockDim.x + threadIdx.x; i < n.N; i += gridDim.x * blockDim.x)
    for (int j = 0; j < 3; ++j) u[3 * i + j] = fixed_u(n, i, j, alpha, ramp != 0);
}

// element coefficients EA (l - L) / (L l) and the singular test l < 1e-12 L
__global__ void __launch_bounds__(kNT) nv_coefs(const __grid_constant__ frb_batch b, int p, double* coef,
                                                NaiveState* st) {
  __shared__ Net n;
  __shared__ Rank r;
  load_net(n, r, b, p);
  const PosXU pos{n.X, b.u + 3 * n.node_base};
  bool bad = false;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n.M; e += gridDim.x * blockDim.x) {
    const int2 ab = n.eab[e];
    const double dx = dsub(pos(ab.y, 0), pos(ab.x, 0));
    const double dy = dsub(pos(ab.y, 1), pos(ab.x, 1));
    const double dz = dsub(pos(ab.y, 2), pos(ab.x, 2));
    const double l = seg_len(dx, dy, dz);
    const double L = n.EL[e];
    coef[e] = ddiv(dmul(elem_ea(n, e), dsub(l, L)), dmul(L, l));
    bad |= l < dmul(kCollapse, L);
  }
  if (bad) st->singular = 1;
}

// f at every free node: role-a incidences 0 - nd - nd ..., role b 0 + nd ...,
// nd = d * coef with d recomputed from the positions (bincount order)
__global__ void __launch_bounds__(kNT) nv_forces(const __grid_constant__ frb_batch b, int p, const double* coef,
                                                 double* fcur) {
  __shared__ Net n;
  __shared__ Rank r;
  load_net(n, r, b, p);
  const PosXU pos{n.X, b.u + 3 * n.node_base};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n.NF; i += gridDim.x * blockDim.x) {
    const int2 meta = n.incn[i];
    const int na = meta.y & 0xffff, nb = (meta.y >> 16) & 0xffff;
    const double px = pos(i, 0), py = pos(i, 1), pz = pos(i, 2);
    double ax = 0.0, ay = 0.0, az = 0.0, bx = 0.0, by = 0.0, bz = 0.0;
    for (int k = 0; k < na + nb; ++k) {
      const int2 e = n.inc[meta.x + k];
      const double cf = coef[e.y];
      if (k < na) {
        ax = dsub(ax, dmul(dsub(pos(e.x, 0), px), cf));
        ay = dsub(ay, dmul(dsub(pos(e.x, 1), py), cf));
        az = dsub(az, dmul(dsub(pos(e.x, 2), pz), cf));
      } else {
        bx = dadd(bx, dmul(dsub(px, pos(e.x, 0)), cf));
        by = dadd(by, dmul(dsub(py, pos(e.x, 1)), cf));
        bz = dadd(bz, dmul(dsub(pz, pos(e.x, 2)), cf));
      }
    }
    fcur[3 * i] = dadd(ax, bx);
    fcur[3 * i + 1] = dadd(ay, by);
    fcur[3 * i + 2] = dadd(az, bz);
  }
}

// per free DOF: k_hat, sq = (u k_hat) u, sq2 = (u m) u, ff = f f; f -> f_prev
__global__ void __launch_bounds__(kNT) nv_dofs(const __grid_constant__ frb_batch b, int p, const double* fcur,
                                               const double* v, double* sq, double* sq2, double* ff, int adaptive) {
  __shared__ Net n;
  __shared__ Rank r;
  load_net(n, r, b, p);
  const double* u = b.u + 3 * n.node_base;
  double* fprv = b.f + 3 * n.node_base;
  for (int d = blockIdx.x * blockDim.x + threadIdx.x; d < 3 * n.NF; d += gridDim.x * blockDim.x) {
    const double f = fcur[d];
    if (adaptive) {
      const double den = dmul(n.dt, v[d]);
      double kh = den != 0.0 ? ddiv(dsub(f, fprv[d]), den) : 0.0;
      kh = (kh > 0.0 || isnan(kh)) ? kh : 0.0;  // np.maximum(k_hat, 0)
      sq[d] = dmul(dmul(u[d], kh), u[d]);
      sq2[d] = dmul(dmul(u[d], n.mass[d / 3]), u[d]);
    }
    ff[d] = dmul(f, f);
    fprv[d] = f;
  }
}

// numpy's pairwise sum of a[0:nf] through the plan (plan.py): one thread per
// leaf (8 stride-8 chains, fold, tail), then the combine levels
__device__ double plan_sum(const int* plan, const double* a, double* slots) {
  const int L = plan[0], H = plan[1], root = plan[2];
  if (L == 0) return 0.0;
  const int* leaf_start = plan + 4;
  const int* leaf_size = leaf_start + L;
  const int* level_off = leaf_size + L;
  const int K = L - 1;
  const int* op_dst = level_off + H + 1;
  const int* op_l = op_dst + K;
  const int* op_r = op_l + K;
  for (int l = threadIdx.x; l < L; l += blockDim.x) {
    const double* x = a + leaf_start[l];
    const int size = leaf_size[l];
    double s = 0.0;
    int body = 0;
    if (size >= 8) {
      body = size - size % 8;
      double rr[8];
      for (int j = 0; j < 8; ++j) rr[j] = x[j];
      for (int i = 8; i < body; i += 8)
        for (int j = 0; j < 8; ++j) rr[j] = dadd(rr[j], x[i + j]);
      s = dadd(dadd(dadd(rr[0], rr[1]), dadd(rr[2], rr[3])), dadd(dadd(rr[4], rr[5]), dadd(rr[6], rr[7])));
    }
    for (int i = body; i < size; ++i) s = dadd(s, x[i]);
    slots[l] = s;
  }
  __syncthreads();
  for (int h = 0; h < H; ++h) {
    for (int k = level_off[h] + threadIdx.x; k < level_off[h + 1]; k += blockDim.x)
      slots[op_dst[k]] = dadd(slots[op_l[k]], slots[op_r[k]]);
    __syncthreads();
  }
  const double out = slots[root];
  __syncthreads();
  return out;
}

// the three reductions and the scalar bookkeeping (one block)
__global__ void __launch_bounds__(kNT) nv_reduce(const __grid_constant__ frb_batch b,
                                                 const __grid_constant__ frb_config cfg, int p, const double* sq,
                                                 const double* sq2, const double* ff, double* slots, NaiveState* st) {
  __shared__ Net n;
  __shared__ Rank r;
  load_net(n, r, b, p);
  const bool adaptive = cfg.damping == FRB_DAMPING_ADAPTIVE;
  double s_sq = 0.0, s_m = 0.0;
  if (adaptive) {
    s_sq = plan_sum(n.plan, sq, slots);
    s_m = plan_sum(n.plan, sq2, slots);
  }
  const double s_f = plan_sum(n.plan, ff, slots);
  if (threadIdx.x != 0 || st->singular) return;
  // np.sum adds the pairwise result to the identity 0.0
  const double mq = dadd(0.0, s_m), lsq = dadd(0.0, s_sq), res = dsqrt(dadd(0.0, s_f));
  double c = cfg.damping_c;
  if (adaptive) {
    const double lam = ddiv(lsq, mq);
    c = (mq > 0.0 && lam > 0.0) ? dmul(2.0, dsqrt(lam)) : 0.0;
  }
  const int it = st->it;
  const int full_bc_iter = cfg.bc_ramp_iters > 0 ? cfg.bc_ramp_iters - 1 : 0;
  if (it == full_bc_iter) {
    st->r_ref = res;
    const double th = dmul(cfg.tol_rel, res);
    st->threshold = th > cfg.tol_abs ? th : cfg.tol_abs;  // max(tol_abs, .)
  }
  int done = 0, conv = 0;
  if (it >= full_bc_iter && res <= st->threshold) {
    done = conv = 1;
  } else if (it + 1 >= cfg.max_iters) {
    done = 1;
  }
  st->c = c;
  st->residual = res;
  st->done = done;
  st->converged = conv;
}

// first half-kick and drift of iteration 0 (prologue), from f_prev = f(u0)
__global__ void __launch_bounds__(kNT) nv_first_kick(const __grid_constant__ frb_batch b, int p, double* v) {
  __shared__ Net n;
  __shared__ Rank r;
  load_net(n, r, b, p);
  double* u = b.u + 3 * n.node_base;
  const double* f = b.f + 3 * n.node_base;
  for (int d = blockIdx.x * blockDim.x + threadIdx.x; d < 3 * n.NF; d += gridDim.x * blockDim.x) {
    const double a = ddiv(-f[d], n.mass[d / 3]);
    v[d] = dadd(0.0, dmul(n.hdt, a));
    u[d] = dadd(0.0, dmul(n.dt, v[d]));
  }
}

// accelerations, second half-kick; unless done, the next half-kick + drift
__global__ void __launch_bounds__(kNT) nv_update(const __grid_constant__ frb_batch b, int p, double* v,
                                                 const NaiveState* st) {
  __shared__ Net n;
  __shared__ Rank r;
  load_net(n, r, b, p);
  double* u = b.u + 3 * n.node_base;
  const double* f = b.f + 3 * n.node_base;  // f_prev = f of this iteration
  const double c = st->c;
  const bool done = st->done != 0;
  for (int d = blockIdx.x * blockDim.x + threadIdx.x; d < 3 * n.NF; d += gridDim.x * blockDim.x) {
    const double a = dsub(ddiv(-f[d], n.mass[d / 3]), dmul(c, v[d]));
    double vd = dadd(v[d], dmul(n.hdt, a));
    if (!done) {
      vd = dadd(vd, dmul(n.hdt, a));
      u[d] = dadd(u[d], dmul(n.dt, vd));
    }
    v[d] = vd;
  }
}

// epilogue (one block): positions to global scratch, reactions and sigma
// at the fixed nodes, the result record -- or the singular record
__global__ void __launch_bounds__(kNT) nv_finish(const __grid_constant__ frb_batch b,
                                                 const __grid_constant__ frb_config cfg, int p, const NaiveState* st) {
  __shared__ Net n;
  __shared__ Rank r;
  __shared__ Scalars sc;
  load_net(n, r, b, p);
  const double* u = b.u + 3 * n.node_base;
  for (int d = threadIdx.x; d < 3 * n.N; d += blockDim.x) n.posg[d] = dadd(n.X[d], u[d]);
  if (threadIdx.x == 0) {
    sc.converged = st->converged;
    sc.residual = st->residual;
    sc.r_ref = st->r_ref;
  }
  __syncthreads();
  const bool ramp = cfg.bc_ramp_iters > 0;
  if (st->singular) {
    const int bad = singular_argmin(n, PosGlobalAll{n.posg}, sc);
    if (threadIdx.x == 0) write_singular(b, p, bad, st->it);
    return;
  }
  const int full_bc_iter = ramp ? cfg.bc_ramp_iters - 1 : 0;
  double w[4] = {0.0, 0.0, 0.0, 0.0};
  fixed_forces_and_stress(b, p, n, sc, st->it, st->alpha, ramp, full_bc_iter, false, w);
}

__global__ void nv_reset(NaiveState* st, double alpha) {
  st->c = 0.0;
  st->residual = st->r_ref = 0.0;
  st->threshold = __longlong_as_double(0x7ff0000000000000ULL);
  st->alpha = alpha;
  st->done = st->converged = st->singular = 0;
  st->it = 0;
}

__global__ void nv_set_it(NaiveState* st, int it, double alpha) {
  st->it = it;
  st->alpha = alpha;
}

double host_ramp_alpha(int it_plus_1, int ramp) {
  const double x = static_cast<double>(it_plus_1) / static_cast<double>(ramp);
  return x < 1.0 ? x : 1.0;
}

}  // namespace

extern "C" int frb_naive_solve(const frb_batch* batch, const frb_config* cfg, int32_t problem, double* scratch,
                               int64_t scratch_doubles, void* stream) {
  if (!batch || !cfg || !scratch) return set_err(FRB_E_INVALID, "null argument");
  if (problem < 0 || problem >= batch->n_problems) return set_err(FRB_E_INVALID, "problem index out of range");
  if (cfg->max_iters <= 0) return set_err(FRB_E_INVALID, "max_iters must be > 0");
  if (cfg->energy_check_interval > 0)
    return set_err(FRB_E_UNSUPPORTED, "the work ledger is not provided on the NaiveLoop path");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  frb_problem P;
  int rc = cuda_check(cudaMemcpyAsync(&P, batch->problems + problem, sizeof P, cudaMemcpyDeviceToHost, s),
                      "cudaMemcpyAsync(problem)");
  if (!rc) rc = cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize");
  if (rc) return rc;
  const int64_t N = P.n_nodes, M = P.n_elems, nf = 3 * static_cast<int64_t>(P.n_free_nodes);
  const int64_t L = nf / 8 + 2 * (nf / 128) + 8;  // >= plan leaves + internal slots
  const int64_t need = M + 6 * (3 * N) + 2 * L + 64;
  if (scratch_doubles < need) return set_err(FRB_E_INVALID, "naive scratch too small");
  double* coef = scratch;
  double* fcur = coef + M;
  double* v = fcur + 3 * N;
  double* sq = v + 3 * N;
  double* sq2 = sq + 3 * N;
  double* ff = sq2 + 3 * N;
  double* slots = ff + 3 * N;
  NaiveState* st = reinterpret_cast<NaiveState*>(slots + 2 * L + 8);
  const int ramp_n = cfg->bc_ramp_iters;
  const bool ramp = ramp_n > 0;
  const int adaptive = cfg->damping == FRB_DAMPING_ADAPTIVE;
  const int grid_e = static_cast<int>((M + kNT - 1) / kNT) > 0 ? static_cast<int>((M + kNT - 1) / kNT) : 1;
  const int grid_n = static_cast<int>((N + kNT - 1) / kNT) > 0 ? static_cast<int>((N + kNT - 1) / kNT) : 1;
  const int grid_d = static_cast<int>((nf + kNT - 1) / kNT) > 0 ? static_cast<int>((nf + kNT - 1) / kNT) : 1;
  const frb_batch& b = *batch;
  double alpha = ramp ? -1.0 : 1.0;
  NaiveState hst;
  auto host_state = [&]() {
    int e = cuda_check(cudaMemcpyAsync(&hst, st, sizeof hst, cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync(state)");
    return e ? e : cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize");
  };
  // ---- prologue (microsolver.py:400-430) ----
  nv_reset<<<1, 1, 0, s>>>(st, alpha);
  if ((rc = cuda_check(cudaMemsetAsync(b.u + 3 * P.node_base, 0, 3 * N * sizeof(double), s), "memset u"))) return rc;
  if ((rc = cuda_check(cudaMemsetAsync(v, 0, 3 * N * sizeof(double), s), "memset v"))) return rc;
  nv_fixed<<<grid_n, kNT, 0, s>>>(b, problem, alpha, ramp);
  nv_coefs<<<grid_e, kNT, 0, s>>>(b, problem, coef, st);
  nv_forces<<<grid_n, kNT, 0, s>>>(b, problem, coef, b.f + 3 * P.node_base);
  if ((rc = cuda_check(cudaGetLastError(), "naive prologue launch"))) return rc;
  if ((rc = host_state())) return rc;
  int it = 0;
  if (!hst.singular) {
    nv_first_kick<<<grid_d, kNT, 0, s>>>(b, problem, v);
    if (ramp) {
      alpha = host_ramp_alpha(1, ramp_n);
      nv_fixed<<<grid_n, kNT, 0, s>>>(b, problem, alpha, 1);
    }
    // ---- relaxation loop (microsolver.py:434-530): one launch per line ----
    for (;; ++it) {
      nv_set_it<<<1, 1, 0, s>>>(st, it, alpha);
      nv_coefs<<<grid_e, kNT, 0, s>>>(b, problem, coef, st);
      nv_forces<<<grid_n, kNT, 0, s>>>(b, problem, coef, fcur);
      nv_dofs<<<grid_d, kNT, 0, s>>>(b, problem, fcur, v, sq, sq2, ff, adaptive);
      nv_reduce<<<1, kNT, 0, s>>>(b, *cfg, problem, sq, sq2, ff, slots, st);
      if ((rc = cuda_check(cudaGetLastError(), "naive iteration launch"))) return rc;
      if ((rc = host_state())) return rc;
      if (hst.singular) break;
      nv_update<<<grid_d, kNT, 0, s>>>(b, problem, v, st);
      if (hst.done) break;
      if (ramp && alpha < 1.0) {
        alpha = host_ramp_alpha(it + 2, ramp_n);
        nv_fixed<<<grid_n, kNT, 0, s>>>(b, problem, alpha, 1);
      }
    }
  }
  nv_set_it<<<1, 1, 0, s>>>(st, it, alpha);
  nv_finish<<<1, kNT, 0, s>>>(b, *cfg, problem, st);
  return cuda_check(cudaGetLastError(), "naive epilogue launch");
}

extern "C" int64_t frb_naive_scratch_doubles(int32_t n_nodes, int32_t n_elems, int32_t n_free_nodes) {
  const int64_t nf = 3 * static_cast<int64_t>(n_free_nodes);
  const int64_t L = nf / 8 + 2 * (nf / 128) + 8;
  return n_elems + 6 * (3 * static_cast<int64_t>(n_nodes)) + 2 * L + 64;
}
