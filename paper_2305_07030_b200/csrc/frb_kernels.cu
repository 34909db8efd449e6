// frb_kernels.cu -- persistent dynamic-relaxation kernel for sm_100a.
//
// One CTA owns one fiber network at a time, pulled from a device work queue
// (the spec's TeamBatched strategy; the paper's "one team per
// sub-problem" kernel).  The whole Fig.-1 loop of the
// reference (_relax, pkg/src/fibrelax/microsolver.py:379-530) runs inside
// the kernel; finalize_result (:549-564) runs in its epilogue.
//
// Bit-exactness contract.  Every FP64 operation is an
// explicit __d{add,sub,mul,div,sqrt}_rn intrinsic, so no FMA contraction or
// reassociation can occur; the evaluation order of each reference line is
// reproduced literally:
//   * fiber length sqrt((dx*dx + dz*dz) + dy*dy)        (einsum, :206)
//   * coef = (EA*(l-L)) / (L*l), nd = d*coef           (:210-211)
//   * per node f = A + B, A = 0 - nd_e1 - nd_e2 ... over role-a elements in
//     ascending id, B = 0 + nd... over role b          (bincount, :214-218)
//   * the three reductions follow NumPy's pairwise tree (plan.py): each
//     thread accumulates one stride-8 chain of one leaf in order, the
//     8 chains of a leaf sit in 8 consecutive lanes and fold with xor
//     shuffles 1,2,4 (= ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))), tails are
//     added in order, then leaves combine level by level in SMEM.
//
// Memory layout per CTA (dynamic SMEM, FP64):
//   pos  [3N]   current positions X+u of every node (the gather source)
//   fbuf [2][nf] internal force on free DOFs, ping-pong (current / previous)
//   slot [3][2L-1] pairwise-tree slots for the three reductions
// Thread-private registers hold u and v for the <= 17 DOFs a thread owns
// (its pairwise chain plus at most one tail element), so the state of the
// relaxation never round-trips through HBM.  Read-only network data
// (X, mass, incidence lists, L, EA) is streamed through L1/L2.

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "frb200.h"

namespace {

constexpr int kMaxThreads = 512;
constexpr int kMaxOwn = 17;          // 16 chain elements + 1 tail element
constexpr int kMaxWarps = kMaxThreads / 32;
constexpr double kCollapse = 1e-12;  // microsolver.py:30

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double dsqrt(double a) { return __dsqrt_rn(a); }

// sqrt(einsum("ij,ij->i", d, d)) for 3 columns == sqrt((x*x + z*z) + y*y)
__device__ __forceinline__ double seg_len(double dx, double dy, double dz) {
  return dsqrt(dadd(dadd(dmul(dx, dx), dmul(dz, dz)), dmul(dy, dy)));
}

struct Plan {
  int n_leaves, n_levels, root;
  const int* leaf_start;
  const int* leaf_size;
  const int* level_off;
  const int* op_dst;
  const int* op_left;
  const int* op_right;
};

__device__ __forceinline__ Plan load_plan(const int* flat) {
  Plan p;
  p.n_leaves = flat[0];
  p.n_levels = flat[1];
  p.root = flat[2];
  const int L = p.n_leaves, H = p.n_levels, K = L > 0 ? L - 1 : 0;
  p.leaf_start = flat + 4;
  p.leaf_size = p.leaf_start + L;
  p.level_off = p.leaf_size + L;
  p.op_dst = p.level_off + H + 1;
  p.op_left = p.op_dst + K;
  p.op_right = p.op_left + K;
  return p;
}

struct Net {
  int N, NF, nf, M;
  double dt, hdt, volume;
  double g[9];  // F - I
  const double* X;
  const double* mass;
  const int2* incn;
  const int2* inc;
  const int2* eab;
  const double* EL;
  const double* EA;
  Plan plan;
};

__device__ __forceinline__ Net load_net(const frb_batch& b, int p) {
  const frb_problem& P = b.problems[p];
  Net n;
  n.N = P.n_nodes;
  n.NF = P.n_free_nodes;
  n.nf = 3 * P.n_free_nodes;
  n.M = P.n_elems;
  n.dt = P.dt;
  n.hdt = dmul(0.5, P.dt);
  n.volume = P.volume;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      n.g[3 * r + c] = dsub(P.F[3 * r + c], r == c ? 1.0 : 0.0);
  n.X = b.X + 3 * P.node_base;
  n.mass = b.node_mass + P.node_base;
  n.incn = reinterpret_cast<const int2*>(b.inc_node) + P.node_base;
  n.inc = reinterpret_cast<const int2*>(b.inc) + P.inc_base;
  n.eab = reinterpret_cast<const int2*>(b.elem_ab) + P.elem_base;
  n.EL = b.elem_L + P.elem_base;
  n.EA = b.elem_EA + P.elem_base;
  n.plan = load_plan(b.plans + P.plan_base);
  return n;
}

// u_presc[i][j] = x @ (F-I)^T as OpenBLAS evaluates it (microsolver.py:320-322):
// t = x0*g[j][0]; t = fma(x1, g[j][1], t); t = fma(x2, g[j][2], t)
__device__ __forceinline__ double presc(const Net& n, int node, int j) {
  const double x0 = n.X[3 * node], x1 = n.X[3 * node + 1], x2 = n.X[3 * node + 2];
  double t = dmul(x0, n.g[3 * j]);
  t = __fma_rn(x1, n.g[3 * j + 1], t);
  return __fma_rn(x2, n.g[3 * j + 2], t);
}

// Fixed-node displacement given the ramp factor (microsolver.py:409-410, 453).
// alpha < 0 encodes "untouched initial zero" (ramp > 0 before iteration 0).
__device__ __forceinline__ double fixed_u(const Net& n, int node, int j, double alpha, bool ramp) {
  if (!ramp) return presc(n, node, j);
  if (alpha < 0.0) return 0.0;
  return dmul(alpha, presc(n, node, j));
}

// Position sources: the solver's SMEM array, or X + u recomputed from global
// memory (one-shot internal_forces).  Both yield the same rounded X + u.
struct PosSmem {
  const double* p;
  __device__ __forceinline__ double operator()(int node, int axis) const { return p[3 * node + axis]; }
};
struct PosGlobal {
  const double* X;
  const double* u;
  __device__ __forceinline__ double operator()(int node, int axis) const {
    return dadd(X[3 * node + axis], u[3 * node + axis]);
  }
};

// Internal force at node i (gather over its incidence lists, element order
// per role).  Returns true if an incident element collapsed (l < 1e-12 L).
template <class Pos>
__device__ __forceinline__ bool node_force(const Net& n, const Pos& pos, int i, double& fx,
                                           double& fy, double& fz) {
  const int2 meta = n.incn[i];
  const int first = meta.x;
  const int na = meta.y & 0xffff;
  const int nb = (meta.y >> 16) & 0xffff;
  const double px = pos(i, 0), py = pos(i, 1), pz = pos(i, 2);
  double ax = 0.0, ay = 0.0, az = 0.0, bx = 0.0, by = 0.0, bz = 0.0;
  bool bad = false;
  for (int k = 0; k < na + nb; ++k) {
    const int2 e = n.inc[first + k];
    const double ox = pos(e.x, 0), oy = pos(e.x, 1), oz = pos(e.x, 2);
    const bool role_a = k < na;
    // d = P[b] - P[a]
    const double dx = role_a ? dsub(ox, px) : dsub(px, ox);
    const double dy = role_a ? dsub(oy, py) : dsub(py, oy);
    const double dz = role_a ? dsub(oz, pz) : dsub(pz, oz);
    const double L = __ldg(n.EL + e.y);
    const double EA = __ldg(n.EA + e.y);
    const double l = seg_len(dx, dy, dz);
    bad |= l < dmul(kCollapse, L);
    const double coef = ddiv(dmul(EA, dsub(l, L)), dmul(L, l));
    const double ndx = dmul(dx, coef), ndy = dmul(dy, coef), ndz = dmul(dz, coef);
    if (role_a) {  // bincount(ia, -nd): A = 0 + (-nd) + ...
      ax = dsub(ax, ndx);
      ay = dsub(ay, ndy);
      az = dsub(az, ndz);
    } else {       // bincount(ib, nd)
      bx = dadd(bx, ndx);
      by = dadd(by, ndy);
      bz = dadd(bz, ndz);
    }
  }
  fx = dadd(ax, bx);
  fy = dadd(ay, by);
  fz = dadd(az, bz);
  return bad;
}

// numpy argmin over (l - eps) with NaN-first semantics: a precedes b?
__device__ __forceinline__ bool argmin_before(double va, int ia, double vb, int ib) {
  const bool na = isnan(va), nb = isnan(vb);
  if (na != nb) return na;
  if (!na && va != vb) return va < vb;
  return ia < ib;
}

struct Scalars {
  double c, residual, r_ref, threshold;
  double red[kMaxWarps * 9];
  int ired[kMaxWarps];
  int problem, done, converged, singular;
};

// Block-wide deterministic sum of 9 per-thread values (fixed shuffle tree,
// then warps in order).  Result valid in thread 0.
__device__ void block_sum9(double v[9], Scalars& sc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int r = 0; r < 9; ++r) {
    double x = v[r];
    for (int o = 16; o > 0; o >>= 1) x = dadd(x, __shfl_down_sync(0xffffffffu, x, o));
    if (lane == 0) sc.red[warp * 9 + r] = x;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    for (int r = 0; r < 9; ++r) {
      double s = sc.red[r];
      for (int w = 1; w < nw; ++w) s = dadd(s, sc.red[w * 9 + r]);
      v[r] = s;
    }
  }
  __syncthreads();
}

// Singular-element path: reference raises SingularElementError naming
// argmin(length - eps_len) over all elements (microsolver.py:207-209).
template <class Pos>
__device__ int singular_argmin(const Net& n, const Pos& pos, Scalars& sc) {
  double best = 0.0;
  int besti = 0x7fffffff;
  for (int e = threadIdx.x; e < n.M; e += blockDim.x) {
    const int2 ab = n.eab[e];
    const double dx = dsub(pos(ab.y, 0), pos(ab.x, 0));
    const double dy = dsub(pos(ab.y, 1), pos(ab.x, 1));
    const double dz = dsub(pos(ab.y, 2), pos(ab.x, 2));
    const double L = n.EL[e];
    const double v = dsub(seg_len(dx, dy, dz), dmul(kCollapse, L));
    if (besti == 0x7fffffff || argmin_before(v, e, best, besti)) {
      best = v;
      besti = e;
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_down_sync(0xffffffffu, best, o);
    const int oi = __shfl_down_sync(0xffffffffu, besti, o);
    if (oi != 0x7fffffff && (besti == 0x7fffffff || argmin_before(ov, oi, best, besti))) {
      best = ov;
      besti = oi;
    }
  }
  if (lane == 0) {
    sc.red[warp] = best;
    sc.ired[warp] = besti;
  }
  __syncthreads();
  int result = 0;
  if (threadIdx.x == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    double b = sc.red[0];
    int bi = sc.ired[0];
    for (int w = 1; w < nw; ++w) {
      const int oi = sc.ired[w];
      if (oi != 0x7fffffff && (bi == 0x7fffffff || argmin_before(sc.red[w], oi, b, bi))) {
        b = sc.red[w];
        bi = oi;
      }
    }
    result = bi;
  }
  __syncthreads();
  return result;
}

// Check every element's current length (init and ramp iterations, when
// fixed-fixed elements move).  Sets sc.singular.
__device__ void check_all_elements(const Net& n, const double* pos, Scalars& sc) {
  bool bad = false;
  for (int e = threadIdx.x; e < n.M; e += blockDim.x) {
    const int2 ab = n.eab[e];
    const double dx = dsub(pos[3 * ab.y], pos[3 * ab.x]);
    const double dy = dsub(pos[3 * ab.y + 1], pos[3 * ab.x + 1]);
    const double dz = dsub(pos[3 * ab.y + 2], pos[3 * ab.x + 2]);
    bad |= seg_len(dx, dy, dz) < dmul(kCollapse, n.EL[e]);
  }
  if (bad) sc.singular = 1;
}

__device__ __forceinline__ void set_fixed_positions(const Net& n, double* pos, double alpha,
                                                    bool ramp) {
  for (int i = n.NF + threadIdx.x; i < n.N; i += blockDim.x)
    for (int j = 0; j < 3; ++j) pos[3 * i + j] = dadd(n.X[3 * i + j], fixed_u(n, i, j, alpha, ramp));
}

__device__ __forceinline__ double ramp_alpha(int it_plus_1, int ramp) {
  // Python: min(1.0, (it + 1) / ramp)
  const double x = ddiv(static_cast<double>(it_plus_1), static_cast<double>(ramp));
  return x < 1.0 ? x : 1.0;
}

__device__ void solve_one(const frb_batch& b, const frb_config& cfg, int p, double* smem,
                          Scalars& sc) {
  const Net n = load_net(b, p);
  const int T = blockDim.x, t = threadIdx.x, lane = t & 31;
  const int L = n.plan.n_leaves;
  double* pos = smem;
  double* fb0 = pos + 3 * n.N;
  double* fb1 = fb0 + n.nf;
  double* slot = fb1 + n.nf;

  const bool adaptive = cfg.damping == FRB_DAMPING_ADAPTIVE;
  const int ramp_n = cfg.bc_ramp_iters;
  const bool ramp = ramp_n > 0;
  const int full_bc_iter = ramp ? ramp_n - 1 : 0;
  const double dt = n.dt, hdt = n.hdt;
  double alpha = ramp ? -1.0 : 1.0;  // -1: fixed nodes still at their zero init

  // ---- DOF ownership: thread t <-> chain (leaf t/8, lane j = t%8) --------
  const bool chain = t < 8 * L;
  const int leaf = t >> 3, j = t & 7;
  int lstart = 0, q = 0, body = 0, nt = 0;
  if (chain) {
    lstart = n.plan.leaf_start[leaf];
    const int lsize = n.plan.leaf_size[leaf];
    q = lsize >= 8 ? (lsize >> 3) : 0;
    body = 8 * q;
    nt = lsize - body;
  }
  const int nown = chain ? q + (j < nt ? 1 : 0) : 0;
  double u[kMaxOwn], v[kMaxOwn];

  if (t == 0) {
    sc.singular = 0;
    sc.done = 0;
    sc.converged = 0;
    sc.threshold = __longlong_as_double(0x7ff0000000000000ULL);  // +inf until set
  }
  // ---- prologue: BCs, initial positions (microsolver.py:400-411) ---------
  for (int k = t; k < 3 * n.NF; k += T) pos[k] = dadd(n.X[k], 0.0);
  set_fixed_positions(n, pos, alpha, ramp);
  __syncthreads();
  check_all_elements(n, pos, sc);
  __syncthreads();
  if (sc.singular) {
    const int bad = singular_argmin(n, PosSmem{pos}, sc);
    if (t == 0) {
      frb_result& r = b.results[p];
      r.status = FRB_STATUS_SINGULAR;
      r.bad_element = bad;
      r.iters = 0;
      r.converged = 0;
    }
    __syncthreads();
    return;
  }
  // initial internal forces on free nodes (:413-420)
  for (int i = t; i < n.NF; i += T) {
    double fx, fy, fz;
    node_force(n, PosSmem{pos}, i, fx, fy, fz);
    fb0[3 * i] = fx;
    fb0[3 * i + 1] = fy;
    fb0[3 * i + 2] = fz;
  }
  __syncthreads();
  // a = -f/m (:428-430), then iteration 0's kick + drift (:443-448)
#pragma unroll
  for (int k = 0; k < kMaxOwn; ++k) {
    if (k < nown) {
      const int d = k < q ? lstart + j + 8 * k : lstart + body + j;
      const double a = ddiv(-fb0[d], n.mass[d / 3]);
      v[k] = dadd(0.0, dmul(hdt, a));
      u[k] = dadd(0.0, dmul(dt, v[k]));
      pos[d] = dadd(n.X[d], u[k]);
    }
  }
  if (ramp) {  // iteration 0's ramp step (:449-453)
    alpha = ramp_alpha(1, ramp_n);
    set_fixed_positions(n, pos, alpha, ramp);
  }
  __syncthreads();

  // ---- relaxation loop (microsolver.py:434-530) ---------------------------
  int cur = 1;
  int it = 0;
  for (;; ++it) {
    double* fcur = cur ? fb1 : fb0;
    const double* fprev = cur ? fb0 : fb1;

    // internal forces at the drifted positions (:456-465)
    bool bad = false;
    for (int i = t; i < n.NF; i += T) {
      double fx, fy, fz;
      bad |= node_force(n, PosSmem{pos}, i, fx, fy, fz);
      fcur[3 * i] = fx;
      fcur[3 * i + 1] = fy;
      fcur[3 * i + 2] = fz;
    }
    if (bad) sc.singular = 1;
    if (ramp && it < ramp_n) check_all_elements(n, pos, sc);
    __syncthreads();
    if (sc.singular) {
      const int badi = singular_argmin(n, PosSmem{pos}, sc);
      if (t == 0) {
        frb_result& r = b.results[p];
        r.status = FRB_STATUS_SINGULAR;
        r.bad_element = badi;
        r.iters = it;
        r.converged = 0;
      }
      __syncthreads();
      return;
    }

    // per-DOF damping / residual terms + pairwise chains (:467-499)
    if ((t & ~31) < 8 * L) {  // warp holds at least one chain
      double r0 = 0.0, r1 = 0.0, r2 = 0.0;     // chains: u k u, u m u, f f
      double t0 = 0.0, t1 = 0.0, t2 = 0.0;     // this lane's tail element
#pragma unroll
      for (int k = 0; k < kMaxOwn; ++k) {
        if (k < nown) {
          const int d = k < q ? lstart + j + 8 * k : lstart + body + j;
          const double f = fcur[d];
          const double ff = dmul(f, f);
          double sq = 0.0, sq2 = 0.0;
          if (adaptive) {
            const double den = dmul(dt, v[k]);
            const double num = dsub(f, fprev[d]);
            double kh = den != 0.0 ? ddiv(num, den) : 0.0;
            kh = (kh > 0.0 || isnan(kh)) ? kh : 0.0;  // np.maximum(kh, 0.0)
            sq = dmul(dmul(u[k], kh), u[k]);
            sq2 = dmul(dmul(u[k], n.mass[d / 3]), u[k]);
          }
          if (k < q) {
            if (k == 0) {
              r0 = sq;
              r1 = sq2;
              r2 = ff;
            } else {
              r0 = dadd(r0, sq);
              r1 = dadd(r1, sq2);
              r2 = dadd(r2, ff);
            }
          } else {
            t0 = sq;
            t1 = sq2;
            t2 = ff;
          }
        }
      }
      // fold the 8 chains of the leaf: xor 1, 2, 4
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) {
        r0 = dadd(r0, __shfl_xor_sync(0xffffffffu, r0, o));
        r1 = dadd(r1, __shfl_xor_sync(0xffffffffu, r1, o));
        r2 = dadd(r2, __shfl_xor_sync(0xffffffffu, r2, o));
      }
      // tails in order (tail i lives on lane i of the group)
      const int base = lane & ~7;
      const int my_nt = chain ? nt : 0;
#pragma unroll
      for (int i = 0; i < 7; ++i) {
        const double a0 = __shfl_sync(0xffffffffu, t0, base + i);
        const double a1 = __shfl_sync(0xffffffffu, t1, base + i);
        const double a2 = __shfl_sync(0xffffffffu, t2, base + i);
        if (i < my_nt) {
          r0 = dadd(r0, a0);
          r1 = dadd(r1, a1);
          r2 = dadd(r2, a2);
        }
      }
      if (chain && j == 0) {
        slot[3 * leaf] = r0;
        slot[3 * leaf + 1] = r1;
        slot[3 * leaf + 2] = r2;
      }
    }
    __syncthreads();

    // tree combine + scalar bookkeeping (warp 0)
    if (t < 32) {
      const Plan& pl = n.plan;
      for (int lev = 0; lev < pl.n_levels; ++lev) {
        for (int k = pl.level_off[lev] + lane; k < pl.level_off[lev + 1]; k += 32) {
          const int dd = pl.op_dst[k], la = pl.op_left[k], rb = pl.op_right[k];
          slot[3 * dd] = dadd(slot[3 * la], slot[3 * rb]);
          slot[3 * dd + 1] = dadd(slot[3 * la + 1], slot[3 * rb + 1]);
          slot[3 * dd + 2] = dadd(slot[3 * la + 2], slot[3 * rb + 2]);
        }
        __syncwarp();
      }
      if (t == 0) {
        double s_sq = 0.0, s_m = 0.0, s_f = 0.0;
        if (L > 0) {
          s_sq = slot[3 * pl.root];
          s_m = slot[3 * pl.root + 1];
          s_f = slot[3 * pl.root + 2];
        }
        // np.sum adds the pairwise result to the identity 0.0
        s_sq = dadd(0.0, s_sq);
        s_m = dadd(0.0, s_m);
        s_f = dadd(0.0, s_f);
        double c = cfg.damping_c;
        if (adaptive) {
          if (s_m > 0.0) {
            const double lam = ddiv(s_sq, s_m);
            c = lam > 0.0 ? dmul(2.0, dsqrt(lam)) : 0.0;
          } else {
            c = 0.0;
          }
        }
        const double res = dsqrt(s_f);
        if (it == full_bc_iter) {
          sc.r_ref = res;
          const double th = dmul(cfg.tol_rel, res);
          sc.threshold = th > cfg.tol_abs ? th : cfg.tol_abs;  // max(tol_abs, .)
        }
        int done = 0, conv = 0;
        if (it >= full_bc_iter && res <= sc.threshold) {
          done = 1;
          conv = 1;
        } else if (it + 1 >= cfg.max_iters) {
          done = 1;
        }
        sc.c = c;
        sc.residual = res;
        sc.done = done;
        sc.converged = conv;
      }
    }
    __syncthreads();

    // accelerations, second half-kick (:501-507); then the next iteration's
    // first half-kick and drift (:443-453) unless finished
    const double c = sc.c;
    const bool done = sc.done != 0;
#pragma unroll
    for (int k = 0; k < kMaxOwn; ++k) {
      if (k < nown) {
        const int d = k < q ? lstart + j + 8 * k : lstart + body + j;
        const double a = dsub(ddiv(-fcur[d], n.mass[d / 3]), dmul(c, v[k]));
        v[k] = dadd(v[k], dmul(hdt, a));
        if (!done) {
          v[k] = dadd(v[k], dmul(hdt, a));
          u[k] = dadd(u[k], dmul(dt, v[k]));
          pos[d] = dadd(n.X[d], u[k]);
        }
      }
    }
    if (!done && ramp && alpha < 1.0) {
      alpha = ramp_alpha(it + 2, ramp_n);
      set_fixed_positions(n, pos, alpha, ramp);
    }
    cur ^= 1;
    __syncthreads();
    if (done) break;
  }

  // ---- epilogue: outputs in solver order + stress (:549-564, :285-299) ----
  const double* ffin = cur ? fb0 : fb1;  // toggled after the last iteration
  double* uo = b.u + 3 * b.problems[p].node_base;
  double* fo = b.f + 3 * b.problems[p].node_base;
#pragma unroll
  for (int k = 0; k < kMaxOwn; ++k) {
    if (k < nown) {
      const int d = k < q ? lstart + j + 8 * k : lstart + body + j;
      uo[d] = u[k];
    }
  }
  for (int d = t; d < n.nf; d += T) fo[d] = ffin[d];
  double s9[9];
#pragma unroll
  for (int r = 0; r < 9; ++r) s9[r] = 0.0;
  for (int i = n.NF + t; i < n.N; i += T) {
    double f3[3];
    node_force(n, PosSmem{pos}, i, f3[0], f3[1], f3[2]);
    for (int jj = 0; jj < 3; ++jj) {
      uo[3 * i + jj] = fixed_u(n, i, jj, alpha, ramp);
      fo[3 * i + jj] = f3[jj];
    }
    // S = r^T x over boundary nodes, x = X + u (= pos)
    for (int a = 0; a < 3; ++a)
      for (int c3 = 0; c3 < 3; ++c3) s9[3 * a + c3] = dadd(s9[3 * a + c3], dmul(f3[a], pos[3 * i + c3]));
  }
  block_sum9(s9, sc);
  if (t == 0) {
    frb_result& r = b.results[p];
    const double two_v = dmul(2.0, n.volume);
    for (int a = 0; a < 3; ++a)
      for (int c3 = 0; c3 < 3; ++c3)
        r.avg_stress[3 * a + c3] = ddiv(dadd(s9[3 * a + c3], s9[3 * c3 + a]), two_v);
    r.status = sc.converged ? FRB_STATUS_CONVERGED : FRB_STATUS_MAX_ITERS;
    r.converged = sc.converged;
    r.iters = it + 1;
    r.bad_element = -1;
    r.final_residual = sc.residual;
    r.r_ref = (full_bc_iter <= it) ? sc.r_ref : __longlong_as_double(0x7ff8000000000000ULL);
    r.energy_residual = __longlong_as_double(0x7ff8000000000000ULL);
    for (int e = 0; e < 4; ++e) r.energy[e] = 0.0;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kMaxThreads, 1)
    frb_relax_cta_kernel(frb_batch b, frb_config cfg) {
  extern __shared__ __align__(16) double smem[];
  __shared__ Scalars sc;
  for (;;) {
    if (threadIdx.x == 0) sc.problem = atomicAdd(b.queue, 1);
    __syncthreads();
    const int idx = sc.problem;
    __syncthreads();
    if (idx >= b.n_problems) break;
    const int p = b.order ? b.order[idx] : idx;
    solve_one(b, cfg, p, smem, sc);
  }
}

// One-shot forces for every node of problem blockIdx.x (reference
// internal_forces, microsolver.py:221-238), same gather code as the solver.
__global__ void __launch_bounds__(kMaxThreads)
    frb_forces_kernel(frb_batch b, const double* __restrict__ u, double* __restrict__ f) {
  __shared__ Scalars sc;
  const int p = blockIdx.x;
  const frb_problem& P = b.problems[p];
  const Net n = load_net(b, p);
  const PosGlobal pos{n.X, u + 3 * P.node_base};
  double* fp = f + 3 * P.node_base;
  if (threadIdx.x == 0) sc.singular = 0;
  __syncthreads();
  bool bad = false;
  for (int i = threadIdx.x; i < n.N; i += blockDim.x) {
    double fx, fy, fz;
    bad |= node_force(n, pos, i, fx, fy, fz);
    fp[3 * i] = fx;
    fp[3 * i + 1] = fy;
    fp[3 * i + 2] = fz;
  }
  if (bad) sc.singular = 1;
  __syncthreads();
  int badi = -1;
  if (sc.singular) badi = singular_argmin(n, pos, sc);
  if (threadIdx.x == 0) {
    b.results[p].status = badi >= 0 ? FRB_STATUS_SINGULAR : FRB_STATUS_CONVERGED;
    b.results[p].bad_element = badi;
  }
}

thread_local char g_err[512] = "";

int set_err(int code, const char* fmt, const char* what) {
  snprintf(g_err, sizeof g_err, fmt, what);
  return code;
}

int cuda_check(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return FRB_OK;
  snprintf(g_err, sizeof g_err, "%s: %s", where, cudaGetErrorString(e));
  return FRB_E_CUDA;
}

}  // namespace

extern "C" {

int frb_abi_version(void) { return FRB_ABI_VERSION; }

const char* frb_last_error(void) { return g_err; }

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

int64_t frb_cta_smem_bytes(int32_t n_nodes, int32_t n_free_nodes, int32_t n_leaves) {
  const int64_t slots = n_leaves > 0 ? 2 * static_cast<int64_t>(n_leaves) - 1 : 1;
  return 8 * (3 * static_cast<int64_t>(n_nodes) + 6 * static_cast<int64_t>(n_free_nodes) + 3 * slots);
}

int frb_solve_batch(const frb_batch* batch, const frb_config* cfg, int block_threads, int grid_ctas,
                    void* stream) {
  if (!batch || !cfg) return set_err(FRB_E_INVALID, "%s", "null batch or config");
  if (batch->n_problems < 0) return set_err(FRB_E_INVALID, "%s", "negative problem count");
  if (batch->n_problems == 0) return FRB_OK;
  if (block_threads < 32 || block_threads > kMaxThreads || block_threads % 32)
    return set_err(FRB_E_INVALID, "%s", "block_threads must be a multiple of 32 in [32, 512]");
  if (cfg->energy_check_interval > 0)
    return set_err(FRB_E_UNSUPPORTED, "%s", "energy ledger not in this build");
  if (cfg->max_iters <= 0) return set_err(FRB_E_INVALID, "%s", "max_iters must be > 0");
  const int smem = batch->smem_bytes;
  int dev = 0;
  int rc = cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  if (rc) return rc;
  int optin = 0, nsm = 0;
  rc = frb_device_info(dev, &nsm, &optin, nullptr, nullptr);
  if (rc) return rc;
  if (smem > optin) return set_err(FRB_E_TOO_LARGE, "%s", "problem exceeds shared memory per CTA");
  rc = cuda_check(cudaFuncSetAttribute(frb_relax_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem),
                  "cudaFuncSetAttribute");
  if (rc) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (grid_ctas <= 0) {
    int per_sm = 0;
    rc = cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, frb_relax_cta_kernel, block_threads, smem),
                    "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
    if (rc) return rc;
    if (per_sm < 1) return set_err(FRB_E_TOO_LARGE, "%s", "kernel does not fit on an SM");
    grid_ctas = per_sm * nsm;
  }
  if (grid_ctas > batch->n_problems) grid_ctas = batch->n_problems;
  rc = cuda_check(cudaMemsetAsync(batch->queue, 0, sizeof(int32_t), s), "cudaMemsetAsync");
  if (rc) return rc;
  frb_relax_cta_kernel<<<grid_ctas, block_threads, smem, s>>>(*batch, *cfg);
  return cuda_check(cudaGetLastError(), "frb_relax_cta_kernel launch");
}

int frb_internal_forces(const frb_batch* batch, const double* u, double* f, void* stream) {
  if (!batch || !u || !f) return set_err(FRB_E_INVALID, "%s", "null argument");
  if (batch->n_problems <= 0) return FRB_OK;
  frb_forces_kernel<<<batch->n_problems, 256, 0, static_cast<cudaStream_t>(stream)>>>(*batch, u, f);
  return cuda_check(cudaGetLastError(), "frb_forces_kernel launch");
}

}  // extern "C"
