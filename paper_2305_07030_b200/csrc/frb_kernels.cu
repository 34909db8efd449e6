// frb_kernels.cu -- persistent dynamic-relaxation kernel for sm_100a (K1).
//
// One CTA owns one fiber network at a time, pulled from a device work queue
// (the spec's TeamBatched strategy; the paper's "one team per
// sub-problem" kernel).  The whole Fig.-1 loop of the
// reference (_relax, pkg/src/fibrelax/microsolver.py:379-530) runs inside
// the kernel; finalize_result (:549-564) runs in its epilogue.
//
// Bit-exactness contract.  Every FP64 operation is an
// explicit round-to-nearest operation (intrinsics, or the branch-free
// fast paths of frb_arith.cuh that are bit-identical to them), so no FMA
// contraction or reassociation can occur; each reference line keeps its
// evaluation order:
//   * fiber length sqrt((dx*dx + dz*dz) + dy*dy)        (einsum, :206)
//   * coef = (EA*(l-L)) / (L*l), nd = d*coef           (:210-211)
//   * per node f = A + B, A = 0 - nd_e1 - nd_e2 ... over role-a elements in
//     ascending id, B = 0 + nd... over role b          (bincount, :214-218)
//   * the three reductions follow NumPy's pairwise tree (plan.py): thread
//     8*leaf + j sums the stride-8 chain j of its leaf in order, the 8
//     chains of a leaf sit in 8 consecutive lanes and fold with xor shuffles
//     1, 2, 4 (= ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))), tails are added in
//     order, then leaves combine level by level in SMEM.
//
// Work split per iteration (one CTA, T threads, DOF d owned by thread d % T):
//   F  force    thread per free node: gather over its incidence slots -> f
//   A  per DOF  k_hat, sq = (u k_hat) u, sq2 = (u m) u, ff = f f
//   C  chains   thread per (leaf, chain): ordered sums of sq, sq2, ff
//   T  tree     warp 0: pairwise combine, c, residual, convergence
//   U  per DOF  a = -f/m - c v, two half kicks, drift, new positions
// Only C is sequential, and only over <= 16 additions per thread; all
// divisions / square roots run DOF- or node-parallel.
//
// Memory layout per CTA (dynamic SMEM, FP64, nf = 3 * free nodes):
//   pos  [3][NF]  free-node positions X+u (SoA; conflict-free gathers).
//                 Between F and U it is dead and holds sq (flat, by DOF).
//   fcur [nf]     f from F; after A it holds ff
//   fprv [nf]     f of the previous iteration; after A the current f
//   sq2  [nf]
//   slot [2L-1][3] pairwise-tree slots
// u and v of a thread's <= 8 DOFs live in registers.  Fixed-node positions
// (constant unless the BC ramps) sit in global scratch and are read through
// L1, as are masses, X and the slot-major incidence table.

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "frb200.h"
#include "frb_arith.cuh"

namespace {

constexpr int kMaxThreads = 1024;
constexpr int kMaxWarps = kMaxThreads / 32;
constexpr double kCollapse = 1e-12;  // microsolver.py:30

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double dsqrt(double a) { return __dsqrt_rn(a); }
__device__ __forceinline__ double qnan() { return __longlong_as_double(0x7ff8000000000000ULL); }

// sqrt(einsum("ij,ij->i", d, d)) for 3 columns == sqrt((x*x + z*z) + y*y)
__device__ __forceinline__ double len2(double dx, double dy, double dz) {
  return dadd(dadd(dmul(dx, dx), dmul(dz, dz)), dmul(dy, dy));
}
__device__ __forceinline__ double seg_len(double dx, double dy, double dz) { return dsqrt(len2(dx, dy, dz)); }

// ------------------------------------------------------------------ problem view

struct Net {
  int N, NF, nf, M;
  int S, SA, SB, ea_uniform;
  int L;  // pairwise leaves
  int n_levels, root;
  double dt, hdt, volume, ea;
  double g[9];  // F - I
  const double* X;
  const double* mass;
  const int2* incn;
  const int2* inc;
  const int2* eab;
  const double* EL;
  const double* EA;
  const int* ell_o;
  const double* ell_L;
  const double* ell_EA;
  const int* ell_c;
  const int2* ff_ab;
  const double* ff_L;
  const double* ff_EA;
  int n_ff;
  const int* leaf_start;
  const int* leaf_size;
  const int* level_off;
  const int* op_dst;
  const int* op_left;
  const int* op_right;
  double* pfix;  // fixed-node positions, AoS [N-NF][3] (global scratch)
  int64_t node_base;
};

__device__ void load_net(Net& n, const frb_batch& b, int p) {
  const frb_problem& P = b.problems[p];
  n.N = P.n_nodes;
  n.NF = P.n_free_nodes;
  n.nf = 3 * P.n_free_nodes;
  n.M = P.n_elems;
  n.S = P.ell_stride;
  n.SA = P.ell_slots_a;
  n.SB = P.ell_slots_b;
  n.ea_uniform = P.flags & FRB_PF_EA_UNIFORM;
  n.dt = P.dt;
  n.hdt = dmul(0.5, P.dt);
  n.volume = P.volume;
  n.ea = P.ea;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) n.g[3 * r + c] = dsub(P.F[3 * r + c], r == c ? 1.0 : 0.0);
  n.node_base = P.node_base;
  n.X = b.X + 3 * P.node_base;
  n.mass = b.node_mass + P.node_base;
  n.incn = reinterpret_cast<const int2*>(b.inc_node) + P.node_base;
  n.inc = reinterpret_cast<const int2*>(b.inc) + P.inc_base;
  n.eab = reinterpret_cast<const int2*>(b.elem_ab) + P.elem_base;
  n.EL = b.elem_L + P.elem_base;
  n.EA = b.elem_EA + P.elem_base;
  n.ell_o = b.ell_other + P.ell_base;
  n.ell_L = b.ell_L + P.ellv_base;
  n.ell_EA = b.ell_EA ? b.ell_EA + P.ellv_base : nullptr;
  n.ell_c = b.ell_c + P.ell_base;
  n.ff_ab = reinterpret_cast<const int2*>(b.ff_ab) + P.ff_base;
  n.ff_L = b.ff_L + P.ffv_base;
  n.ff_EA = b.ff_EA ? b.ff_EA + P.ffv_base : nullptr;
  n.n_ff = P.n_ff;
  n.pfix = b.work ? b.work + 3 * P.node_base : nullptr;
  const int* flat = b.plans + P.plan_base;
  n.L = flat[0];
  n.n_levels = flat[1];
  n.root = flat[2];
  const int K = n.L > 0 ? n.L - 1 : 0;
  n.leaf_start = flat + 4;
  n.leaf_size = n.leaf_start + n.L;
  n.level_off = n.leaf_size + n.L;
  n.op_dst = n.level_off + n.n_levels + 1;
  n.op_left = n.op_dst + K;
  n.op_right = n.op_left + K;
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

// ------------------------------------------------------------------ positions

// Solver positions: free nodes from SMEM (SoA), fixed nodes from the global
// scratch (AoS).
struct PosSolver {
  const double* p;     // [3][NF]
  const double* pfix;  // [N-NF][3]
  int NF;
  __device__ __forceinline__ double operator()(int node, int axis) const {
    return node < NF ? p[axis * NF + node] : pfix[3 * (node - NF) + axis];
  }
};
// X + u recomputed from global memory (one-shot internal_forces).
struct PosGlobal {
  const double* X;
  const double* u;
  __device__ __forceinline__ double operator()(int node, int axis) const {
    return dadd(X[3 * node + axis], u[3 * node + axis]);
  }
};

// ------------------------------------------------------------------ gathers

// One element's end-force vector nd = d*coef with d = P[b] - P[a] (exact
// intrinsics; used off the hot path).  Returns true when it collapsed.
__device__ __forceinline__ bool element_force(double dx, double dy, double dz, double L, double EA,
                                              double& nx, double& ny, double& nz) {
  const double l = seg_len(dx, dy, dz);
  const double coef = ddiv(dmul(EA, dsub(l, L)), dmul(L, l));
  nx = dmul(dx, coef);
  ny = dmul(dy, coef);
  nz = dmul(dz, coef);
  return l < dmul(kCollapse, L);
}

// Internal force at node i from the CSR incidence lists (all nodes; used by
// the epilogue, the singular path and internal_forces).
template <class Pos>
__device__ __forceinline__ bool node_force_csr(const Net& n, const Pos& pos, int i, double& fx,
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
    double nx, ny, nz;
    if (k < na) {
      bad |= element_force(dsub(ox, px), dsub(oy, py), dsub(oz, pz), n.EL[e.y], n.EA[e.y], nx, ny, nz);
      ax = dsub(ax, nx);  // bincount(ia, -nd): 0 + (-nd) + ...
      ay = dsub(ay, ny);
      az = dsub(az, nz);
    } else {
      bad |= element_force(dsub(px, ox), dsub(py, oy), dsub(pz, oz), n.EL[e.y], n.EA[e.y], nx, ny, nz);
      bx = dadd(bx, nx);  // bincount(ib, nd)
      by = dadd(by, ny);
      bz = dadd(bz, nz);
    }
  }
  fx = dadd(ax, bx);
  fy = dadd(ay, by);
  fz = dadd(az, bz);
  return bad;
}

// Exact (intrinsic) fallbacks, kept out of line so the rare path does not
// inflate the register allocation of the hot loops.  Results come back by
// value (references would force the caller's values through local memory).
struct LenCoef {
  double l, coef;
};
__device__ __noinline__ LenCoef exact_len_coef(double dx, double dy, double dz, double L, double EA) {
  LenCoef r;
  r.l = seg_len(dx, dy, dz);
  r.coef = ddiv(dmul(EA, dsub(r.l, L)), dmul(L, r.l));
  return r;
}
__device__ __noinline__ double exact_div(double a, double b) { return ddiv(a, b); }

// a / b through the branch-free fast path, exact fallback out of line.
__device__ __forceinline__ double div_rn(double a, double b) {
  bool ok;
  const double q = frb_arith::div_fast(a, b, ok);
  return ok ? q : exact_div(a, b);
}

// Length and force coefficient of one element through the fast paths.
__device__ __forceinline__ LenCoef len_coef(double dx, double dy, double dz, double L, double EA) {
  bool ok1, ok2;
  LenCoef r;
  r.l = frb_arith::sqrt_fast(len2(dx, dy, dz), ok1);
  r.coef = frb_arith::div_fast(dmul(EA, dsub(r.l, L)), dmul(L, r.l), ok2);
  if (!(ok1 && ok2)) r = exact_len_coef(dx, dy, dz, L, EA);
  return r;
}

// Slot-major incidence view of the free nodes (see frb200.h: ell_*).
struct Ell {
  const int* __restrict__ o;      // other endpoint, -1 = padding
  const int* __restrict__ c;      // free-free element index, -1 = other is fixed
  const double* __restrict__ L;   // reference length (used when c < 0)
  const double* __restrict__ EA;  // E*A per slot, nullptr when uniform
  double ea;
  int SA, SB, S;
};

// Sum over one role's slots of free node i, in slot (= element) order:
// role a accumulates 0 - nd - nd ..., role b 0 + nd + nd ...  Elements to a
// free neighbour take the coefficient computed once in phase F1 (coef[c])
// and recompute d = P[b] - P[a] from the same operands, so nd is bitwise the
// value the reference's per-element pass produces; elements to a fixed
// neighbour are evaluated here.  Padding slots are skipped (exact: the
// reference adds nothing there).
template <bool ROLE_A>
__device__ __forceinline__ void ell_role(const Ell& E, const double* __restrict__ coef, int k0, int k1, int i,
                                         const PosSolver& pos, double px, double py, double pz, double& sx,
                                         double& sy, double& sz, bool& bad) {
  for (int k = k0; k < k1; ++k) {
    const int o = __ldg(E.o + k * E.S + i);
    if (o < 0) continue;
    const int c = __ldg(E.c + k * E.S + i);
    const double ox = pos(o, 0), oy = pos(o, 1), oz = pos(o, 2);
    const double dx = ROLE_A ? dsub(ox, px) : dsub(px, ox);
    const double dy = ROLE_A ? dsub(oy, py) : dsub(py, oy);
    const double dz = ROLE_A ? dsub(oz, pz) : dsub(pz, oz);
    double cf;
    if (c >= 0) {
      cf = coef[c];
    } else {
      const double L = __ldg(E.L + k * E.S + i);
      const double EA = E.EA ? __ldg(E.EA + k * E.S + i) : E.ea;
      const LenCoef lc = len_coef(dx, dy, dz, L, EA);
      bad |= lc.l < dmul(kCollapse, L);
      cf = lc.coef;
    }
    if (ROLE_A) {  // bincount(ia, -nd): 0 + (-nd) + ...
      sx = dsub(sx, dmul(dx, cf));
      sy = dsub(sy, dmul(dy, cf));
      sz = dsub(sz, dmul(dz, cf));
    } else {  // bincount(ib, nd)
      sx = dadd(sx, dmul(dx, cf));
      sy = dadd(sy, dmul(dy, cf));
      sz = dadd(sz, dmul(dz, cf));
    }
  }
}

// Internal force at free node i (phase F2).
__device__ __forceinline__ bool node_force_ell(const Ell& E, const double* __restrict__ coef,
                                               const PosSolver& pos, int i, double& fx, double& fy,
                                               double& fz) {
  const double px = pos(i, 0), py = pos(i, 1), pz = pos(i, 2);
  double ax = 0.0, ay = 0.0, az = 0.0, bx = 0.0, by = 0.0, bz = 0.0;
  bool bad = false;
  ell_role<true>(E, coef, 0, E.SA, i, pos, px, py, pz, ax, ay, az, bad);
  ell_role<false>(E, coef, E.SA, E.SA + E.SB, i, pos, px, py, pz, bx, by, bz, bad);
  fx = dadd(ax, bx);
  fy = dadd(ay, by);
  fz = dadd(az, bz);
  return bad;
}

// Phase F1: coefficient EA (l - L) / (L l) of every free-free element, once
// per iteration, fiber-parallel (microsolver.py:196-211).
__device__ __forceinline__ bool free_free_coefs(const Net& n, const double* __restrict__ pos, int NF,
                                                double* __restrict__ coef) {
  bool bad = false;
  for (int e = threadIdx.x; e < n.n_ff; e += blockDim.x) {
    const int2 ab = __ldg(n.ff_ab + e);
    const double L = __ldg(n.ff_L + e);
    const double EA = n.ff_EA ? __ldg(n.ff_EA + e) : n.ea;
    const double dx = dsub(pos[ab.y], pos[ab.x]);
    const double dy = dsub(pos[NF + ab.y], pos[NF + ab.x]);
    const double dz = dsub(pos[2 * NF + ab.y], pos[2 * NF + ab.x]);
    const LenCoef lc = len_coef(dx, dy, dz, L, EA);
    bad |= lc.l < dmul(kCollapse, L);
    coef[e] = lc.coef;
  }
  return bad;
}

// ------------------------------------------------------------------ block helpers

struct Scalars {
  double c, residual, r_ref, threshold;
  double red[kMaxWarps * 9];
  int ired[kMaxWarps];
  int problem, done, converged, singular;
};

// numpy argmin over (l - eps) with NaN-first semantics: does (va, ia) come first?
__device__ __forceinline__ bool argmin_before(double va, int ia, double vb, int ib) {
  const bool na = isnan(va), nb = isnan(vb);
  if (na != nb) return na;
  if (!na && va != vb) return va < vb;
  return ia < ib;
}

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

// Singular-element path: the reference raises SingularElementError naming
// argmin(length - eps_len) over all elements (microsolver.py:207-209).
template <class Pos>
__device__ int singular_argmin(const Net& n, const Pos& pos, Scalars& sc) {
  constexpr int kNone = 0x7fffffff;
  double best = 0.0;
  int besti = kNone;
  for (int e = threadIdx.x; e < n.M; e += blockDim.x) {
    const int2 ab = n.eab[e];
    const double dx = dsub(pos(ab.y, 0), pos(ab.x, 0));
    const double dy = dsub(pos(ab.y, 1), pos(ab.x, 1));
    const double dz = dsub(pos(ab.y, 2), pos(ab.x, 2));
    const double v = dsub(seg_len(dx, dy, dz), dmul(kCollapse, n.EL[e]));
    if (besti == kNone || argmin_before(v, e, best, besti)) {
      best = v;
      besti = e;
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_down_sync(0xffffffffu, best, o);
    const int oi = __shfl_down_sync(0xffffffffu, besti, o);
    if (oi != kNone && (besti == kNone || argmin_before(ov, oi, best, besti))) {
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
      if (oi != kNone && (bi == kNone || argmin_before(sc.red[w], oi, b, bi))) {
        b = sc.red[w];
        bi = oi;
      }
    }
    result = bi;
  }
  __syncthreads();
  return result;
}

// Length check of every element (init and ramp iterations, when elements
// between fixed nodes move).  Sets sc.singular.
__device__ void check_all_elements(const Net& n, const PosSolver& pos, Scalars& sc) {
  bool bad = false;
  for (int e = threadIdx.x; e < n.M; e += blockDim.x) {
    const int2 ab = n.eab[e];
    const double dx = dsub(pos(ab.y, 0), pos(ab.x, 0));
    const double dy = dsub(pos(ab.y, 1), pos(ab.x, 1));
    const double dz = dsub(pos(ab.y, 2), pos(ab.x, 2));
    bad |= seg_len(dx, dy, dz) < dmul(kCollapse, n.EL[e]);
  }
  if (bad) sc.singular = 1;
}

__device__ __forceinline__ void set_fixed_positions(const Net& n, double alpha, bool ramp) {
  for (int i = n.NF + threadIdx.x; i < n.N; i += blockDim.x)
    for (int j = 0; j < 3; ++j) n.pfix[3 * (i - n.NF) + j] = dadd(n.X[3 * i + j], fixed_u(n, i, j, alpha, ramp));
}

__device__ __forceinline__ double ramp_alpha(int it_plus_1, int ramp) {
  // Python: min(1.0, (it + 1) / ramp)
  const double x = ddiv(static_cast<double>(it_plus_1), static_cast<double>(ramp));
  return x < 1.0 ? x : 1.0;
}

__device__ void write_singular(const frb_batch& b, int p, int bad, int iters) {
  if (threadIdx.x == 0) {
    frb_result& r = b.results[p];
    r.status = FRB_STATUS_SINGULAR;
    r.bad_element = bad;
    r.iters = iters;
    r.converged = 0;
    r.final_residual = qnan();
    r.r_ref = qnan();
    r.energy_residual = qnan();
  }
}

// Quotients num(k)/den(k) for the DOFs k < MAXK a thread owns (has(k)); use
// (k, q) consumes them in DOF order.  den(k) == 0 yields q = 0 (the caller
// decides what a zero denominator means).
template <int MAXK, class Has, class Num, class Den, class Use>
__device__ __forceinline__ void batched_div(Has has, Num num, Den den, Use use) {
#pragma unroll
  for (int k = 0; k < MAXK; ++k) {
    if (has(k)) {
      const double dk = den(k);
      use(k, dk == 0.0 ? 0.0 : div_rn(num(k), dk));
    }
  }
}

// ------------------------------------------------------------------ the solve

template <int MAXK>
__device__ void solve_one(const frb_batch& b, const frb_config& cfg, int p, double* smem, Scalars& sc,
                          const Net& n) {
  const int T = blockDim.x, t = threadIdx.x, lane = t & 31;
  const int NF = n.NF, nf = n.nf, L = n.L;
  double* pos = smem;        // [3][NF]; sq between phases F and U
  double* fcur = pos + nf;   // [nf]
  double* fprv = fcur + nf;  // [nf]
  double* sq2 = fprv + nf;   // [max(nf, n_ff)]: F1 coefficients, then sq2
  double* slot = sq2 + (nf > n.n_ff ? nf : n.n_ff);  // [2L-1][3]
  const PosSolver P{pos, n.pfix, NF};
  // the tree's combine program lives in SMEM (warp 0 walks it every iteration)
  const int n_ops = L > 0 ? L - 1 : 0;
  int* prog = reinterpret_cast<int*>(slot + 3 * (L > 0 ? 2 * L - 1 : 1));  // [levels+1][3*ops]
  int* lvl_s = prog;
  int* dst_s = lvl_s + n.n_levels + 1;
  int* lft_s = dst_s + n_ops;
  int* rgt_s = lft_s + n_ops;
  for (int k = t; k <= n.n_levels; k += T) lvl_s[k] = n.level_off[k];
  for (int k = t; k < n_ops; k += T) {
    dst_s[k] = n.op_dst[k];
    lft_s[k] = n.op_left[k];
    rgt_s[k] = n.op_right[k];
  }

  const bool adaptive = cfg.damping == FRB_DAMPING_ADAPTIVE;
  const int ramp_n = cfg.bc_ramp_iters;
  const bool ramp = ramp_n > 0;
  const int full_bc_iter = ramp ? ramp_n - 1 : 0;
  const double dt = n.dt, hdt = n.hdt;
  double alpha = ramp ? -1.0 : 1.0;  // -1: fixed nodes still at their zero init

  // thread t owns DOFs d = t + k*T (k < MAXK)
  auto has = [&](int k) { return t + k * T < nf; };
  double u[MAXK], v[MAXK];
#pragma unroll
  for (int k = 0; k < MAXK; ++k) u[k] = v[k] = 0.0;

  // pairwise-chain role: thread t < 8L sums chain j of leaf t/8
  const bool chain = t < 8 * L;
  const int leaf = t >> 3, j = t & 7;
  int lstart = 0, q = 0, nt = 0;
  if (chain) {
    lstart = n.leaf_start[leaf];
    const int lsize = n.leaf_size[leaf];
    q = lsize >= 8 ? (lsize >> 3) : 0;
    nt = lsize - 8 * q;
  }

  // ---- prologue: BCs, initial positions (microsolver.py:400-411) ---------
  for (int i = t; i < NF; i += T)
    for (int a = 0; a < 3; ++a) pos[a * NF + i] = dadd(n.X[3 * i + a], 0.0);
  set_fixed_positions(n, alpha, ramp);
  __syncthreads();
  check_all_elements(n, P, sc);
  __syncthreads();
  if (sc.singular) {
    write_singular(b, p, singular_argmin(n, P, sc), 0);
    __syncthreads();
    return;
  }
  // hot loop-invariant views of the incidence table
  const Ell E{n.ell_o, n.ell_c, n.ell_L, n.ea_uniform ? nullptr : n.ell_EA, n.ea, n.SA, n.SB, n.S};
  const double* __restrict__ Xg = n.X;
  const double* __restrict__ mass = n.mass;
  // initial internal forces on free nodes (:413-420), kept as f_prev
  free_free_coefs(n, pos, NF, sq2);
  __syncthreads();
  for (int i = t; i < NF; i += T) {
    double fx, fy, fz;
    node_force_ell(E, sq2, P, i, fx, fy, fz);
    fprv[3 * i] = fx;
    fprv[3 * i + 1] = fy;
    fprv[3 * i + 2] = fz;
  }
  __syncthreads();
  // a = -f/m (:428-430), then iteration 0's kick + drift (:443-448)
  batched_div<MAXK>(
      has, [&](int k) { return -fprv[t + k * T]; }, [&](int k) { return __ldg(mass + (t + k * T) / 3); },
      [&](int k, double a) {
        const int d = t + k * T;
        v[k] = dadd(0.0, dmul(hdt, a));
        u[k] = dadd(0.0, dmul(dt, v[k]));
        const int node = d / 3;
        pos[(d - 3 * node) * NF + node] = dadd(__ldg(Xg + d), u[k]);
      });
  if (ramp) {  // iteration 0's ramp step (:449-453)
    alpha = ramp_alpha(1, ramp_n);
    set_fixed_positions(n, alpha, ramp);
  }
  __syncthreads();

  // ---- relaxation loop (microsolver.py:434-530) ---------------------------
  int it = 0;
  for (;; ++it) {
    // F: internal forces at the drifted positions (:456-465): F1 element
    // coefficients into the sq2 buffer, then F2 per-node gathers
    bool bad = free_free_coefs(n, pos, NF, sq2);
    __syncthreads();
    for (int i = t; i < NF; i += T) {
      double fx, fy, fz;
      bad |= node_force_ell(E, sq2, P, i, fx, fy, fz);
      fcur[3 * i] = fx;
      fcur[3 * i + 1] = fy;
      fcur[3 * i + 2] = fz;
    }
    if (bad) sc.singular = 1;
    if (ramp && it < ramp_n) check_all_elements(n, P, sc);
    __syncthreads();
    if (sc.singular) {
      write_singular(b, p, singular_argmin(n, P, sc), it);
      __syncthreads();
      return;
    }

    // A: k_hat = (f - f_prev)/(dt v) where dt v != 0 else 0, clamped with
    // np.maximum(k_hat, 0) (:468-476); sq = (u k_hat) u, sq2 = (u m) u,
    // ff = f f (:489).  Outputs: sq -> pos (flat), sq2, ff -> fcur, f -> fprv.
    batched_div<MAXK>(
        has, [&](int k) { return dsub(fcur[t + k * T], fprv[t + k * T]); },
        [&](int k) { return adaptive ? dmul(dt, v[k]) : 0.0; },
        [&](int k, double kh) {
          const int d = t + k * T;
          const double f = fcur[d];
          if (adaptive) {
            kh = (kh > 0.0 || isnan(kh)) ? kh : 0.0;
            pos[d] = dmul(dmul(u[k], kh), u[k]);
            sq2[d] = dmul(dmul(u[k], __ldg(mass + d / 3)), u[k]);
          }
          fcur[d] = dmul(f, f);
          fprv[d] = f;
        });
    __syncthreads();

    // C: ordered chain sums of one leaf chain + fold + tails -> leaf slots
    if ((t & ~31) < 8 * L) {  // warp holds at least one chain
      double r0 = 0.0, r1 = 0.0, r2 = 0.0;
      double t0 = 0.0, t1 = 0.0, t2 = 0.0;
      if (chain) {
        int d = lstart + j;
        if (q > 0) {
          r0 = pos[d];
          r1 = sq2[d];
          r2 = fcur[d];
          for (int k = 1; k < q; ++k) {
            d += 8;
            r0 = dadd(r0, pos[d]);
            r1 = dadd(r1, sq2[d]);
            r2 = dadd(r2, fcur[d]);
          }
        }
        if (j < nt) {
          const int dtail = lstart + 8 * q + j;
          t0 = pos[dtail];
          t1 = sq2[dtail];
          t2 = fcur[dtail];
        }
        if (!adaptive) r0 = r1 = t0 = t1 = 0.0;
      }
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) {
        r0 = dadd(r0, __shfl_xor_sync(0xffffffffu, r0, o));
        r1 = dadd(r1, __shfl_xor_sync(0xffffffffu, r1, o));
        r2 = dadd(r2, __shfl_xor_sync(0xffffffffu, r2, o));
      }
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

    // T: tree combine + scalar bookkeeping (warp 0)
    if (t < 32) {
      for (int lev = 0; lev < n.n_levels; ++lev) {
        const int k1 = lvl_s[lev + 1];
        for (int k = lvl_s[lev] + lane; k < k1; k += 32) {
          const int dd = dst_s[k], la = lft_s[k], rb = rgt_s[k];
          slot[3 * dd] = dadd(slot[3 * la], slot[3 * rb]);
          slot[3 * dd + 1] = dadd(slot[3 * la + 1], slot[3 * rb + 1]);
          slot[3 * dd + 2] = dadd(slot[3 * la + 2], slot[3 * rb + 2]);
        }
        __syncwarp();
      }
      if (t == 0) {
        double s_sq = 0.0, s_m = 0.0, s_f = 0.0;
        if (L > 0) {
          s_sq = slot[3 * n.root];
          s_m = slot[3 * n.root + 1];
          s_f = slot[3 * n.root + 2];
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

    // U: accelerations and second half-kick (:501-507); then the next
    // iteration's first half-kick and drift (:443-453) unless finished
    const double c = sc.c;
    const bool done = sc.done != 0;
    batched_div<MAXK>(
        has, [&](int k) { return -fprv[t + k * T]; }, [&](int k) { return __ldg(mass + (t + k * T) / 3); },
        [&](int k, double fm) {
          const double a = dsub(fm, dmul(c, v[k]));
          v[k] = dadd(v[k], dmul(hdt, a));
          if (!done) {
            const int d = t + k * T;
            v[k] = dadd(v[k], dmul(hdt, a));
            u[k] = dadd(u[k], dmul(dt, v[k]));
            const int node = d / 3;
            pos[(d - 3 * node) * NF + node] = dadd(__ldg(Xg + d), u[k]);
          }
        });
    if (!done && ramp && alpha < 1.0) {
      alpha = ramp_alpha(it + 2, ramp_n);
      set_fixed_positions(n, alpha, ramp);
    }
    __syncthreads();
    if (done) break;
  }

  // ---- epilogue: outputs in solver order + stress (:549-564, :285-299) ----
  double* uo = b.u + 3 * n.node_base;
  double* fo = b.f + 3 * n.node_base;
#pragma unroll
  for (int k = 0; k < MAXK; ++k) {
    if (has(k)) {
      const int d = t + k * T;
      uo[d] = u[k];
      fo[d] = fprv[d];
      const int node = d / 3;
      pos[(d - 3 * node) * NF + node] = dadd(__ldg(Xg + d), u[k]);  // pos held sq
    }
  }
  __syncthreads();
  double s9[9];
#pragma unroll
  for (int r = 0; r < 9; ++r) s9[r] = 0.0;
  for (int i = NF + t; i < n.N; i += T) {
    double f3[3];
    node_force_csr(n, P, i, f3[0], f3[1], f3[2]);
    for (int jj = 0; jj < 3; ++jj) {
      uo[3 * i + jj] = fixed_u(n, i, jj, alpha, ramp);
      fo[3 * i + jj] = f3[jj];
    }
    // S = r^T x over boundary nodes (sorted ids == solver order), x = X + u
    for (int a = 0; a < 3; ++a)
      for (int c3 = 0; c3 < 3; ++c3) s9[3 * a + c3] = dadd(s9[3 * a + c3], dmul(f3[a], P(i, c3)));
  }
  block_sum9(s9, sc);
  if (t == 0) {
    frb_result& r = b.results[p];
    const double two_v = dmul(2.0, n.volume);
    for (int a = 0; a < 3; ++a)
      for (int c3 = 0; c3 < 3; ++c3) r.avg_stress[3 * a + c3] = ddiv(dadd(s9[3 * a + c3], s9[3 * c3 + a]), two_v);
    r.status = sc.converged ? FRB_STATUS_CONVERGED : FRB_STATUS_MAX_ITERS;
    r.converged = sc.converged;
    r.iters = it + 1;
    r.bad_element = -1;
    r.final_residual = sc.residual;
    r.r_ref = (full_bc_iter <= it) ? sc.r_ref : qnan();
    r.energy_residual = qnan();
    for (int e = 0; e < 4; ++e) r.energy[e] = 0.0;
  }
  __syncthreads();
}

template <int MAXK, int MAXT>
__global__ void __launch_bounds__(MAXT, 1) frb_relax_cta_kernel(frb_batch b, frb_config cfg) {
  extern __shared__ __align__(16) double smem[];
  __shared__ Scalars sc;
  __shared__ Net net;
  for (;;) {
    if (threadIdx.x == 0) {
      const int idx = atomicAdd(b.queue, 1);
      sc.problem = idx;
      if (idx < b.n_problems) {
        load_net(net, b, b.order ? b.order[idx] : idx);
        sc.singular = 0;
        sc.done = 0;
        sc.converged = 0;
        sc.threshold = __longlong_as_double(0x7ff0000000000000ULL);  // +inf until set
      }
    }
    __syncthreads();
    const int idx = sc.problem;
    if (idx >= b.n_problems) break;
    solve_one<MAXK>(b, cfg, b.order ? b.order[idx] : idx, smem, sc, net);
  }
}

// One-shot forces for every node of problem blockIdx.x (reference
// internal_forces, microsolver.py:221-238), same gather code as the solver.
__global__ void __launch_bounds__(256) frb_forces_kernel(frb_batch b, const double* __restrict__ u,
                                                          double* __restrict__ f) {
  __shared__ Scalars sc;
  __shared__ Net n;
  const int p = blockIdx.x;
  if (threadIdx.x == 0) {
    load_net(n, b, p);
    sc.singular = 0;
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
  if (bad) sc.singular = 1;
  __syncthreads();
  int badi = -1;
  if (sc.singular) badi = singular_argmin(n, pos, sc);
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

thread_local char g_err[512] = "";

int set_err(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

int cuda_check(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return FRB_OK;
  snprintf(g_err, sizeof g_err, "%s: %s", where, cudaGetErrorString(e));
  return FRB_E_CUDA;
}

template <int MAXK, int MAXT>
int launch_cta(const frb_batch* batch, const frb_config* cfg, int threads, int grid, cudaStream_t s) {
  const int smem = batch->smem_bytes;
  auto kern = frb_relax_cta_kernel<MAXK, MAXT>;
  int rc = cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem),
                      "cudaFuncSetAttribute");
  if (rc) return rc;
  if (grid <= 0) {
    int dev = 0, nsm = 0, per_sm = 0;
    rc = cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    if (rc) return rc;
    rc = cuda_check(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev), "cudaDeviceGetAttribute");
    if (rc) return rc;
    rc = cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem),
                    "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
    if (rc) return rc;
    if (per_sm < 1) return set_err(FRB_E_TOO_LARGE, "kernel does not fit on an SM");
    grid = per_sm * nsm;
  }
  if (grid > batch->n_problems) grid = batch->n_problems;
  rc = cuda_check(cudaMemsetAsync(batch->queue, 0, sizeof(int32_t), s), "cudaMemsetAsync");
  if (rc) return rc;
  kern<<<grid, threads, smem, s>>>(*batch, *cfg);
  return cuda_check(cudaGetLastError(), "frb_relax_cta_kernel launch");
}

template <int MAXT>
int dispatch_k(const frb_batch* batch, const frb_config* cfg, int threads, int grid, cudaStream_t s, int k) {
  if (k <= 1) return launch_cta<1, MAXT>(batch, cfg, threads, grid, s);
  if (k <= 2) return launch_cta<2, MAXT>(batch, cfg, threads, grid, s);
  if (k <= 4) return launch_cta<4, MAXT>(batch, cfg, threads, grid, s);
  if (k <= 6) return launch_cta<6, MAXT>(batch, cfg, threads, grid, s);
  return launch_cta<FRB_MAX_DOFS_PER_THREAD, MAXT>(batch, cfg, threads, grid, s);
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

int64_t frb_cta_smem_bytes(int32_t n_free_nodes, int32_t n_ff, int32_t n_leaves) {
  const int64_t nf = 3 * static_cast<int64_t>(n_free_nodes);
  const int64_t L = n_leaves;
  const int64_t slots = L > 0 ? 2 * L - 1 : 1;
  const int64_t levels = L > 1 ? 64 - __builtin_clzll(static_cast<uint64_t>(L - 1)) + 1 : 0;  // >= tree height
  const int64_t prog_ints = (levels + 1) + 3 * (L > 0 ? L - 1 : 0);
  return 8 * (3 * nf + (nf > n_ff ? nf : n_ff) + 3 * slots) + 4 * ((prog_ints + 1) & ~1LL);
}

int frb_solve_batch(const frb_batch* batch, const frb_config* cfg, int block_threads, int grid_ctas,
                    void* stream) {
  if (!batch || !cfg) return set_err(FRB_E_INVALID, "null batch or config");
  if (batch->n_problems < 0) return set_err(FRB_E_INVALID, "negative problem count");
  if (batch->n_problems == 0) return FRB_OK;
  if (block_threads < 32 || block_threads > kMaxThreads || block_threads % 32)
    return set_err(FRB_E_INVALID, "block_threads must be a multiple of 32 in [32, 1024]");
  if (!batch->work) return set_err(FRB_E_INVALID, "work buffer missing");
  if (cfg->energy_check_interval > 0) return set_err(FRB_E_UNSUPPORTED, "energy ledger not in this build");
  if (cfg->max_iters <= 0) return set_err(FRB_E_INVALID, "max_iters must be > 0");
  int dev = 0, optin = 0;
  int rc = cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  if (rc) return rc;
  rc = cuda_check(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev),
                  "cudaDeviceGetAttribute");
  if (rc) return rc;
  if (batch->smem_bytes > optin) return set_err(FRB_E_TOO_LARGE, "problem exceeds shared memory per CTA");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // u, v register arrays sized for the DOFs per thread of the largest problem;
  // the launch bound (and with it the register budget) follows the CTA size
  const int per_thread = (batch->max_nf + block_threads - 1) / block_threads;
  if (per_thread > FRB_MAX_DOFS_PER_THREAD)
    return set_err(FRB_E_TOO_LARGE, "more than FRB_MAX_DOFS_PER_THREAD free DOFs per thread");
  if (block_threads <= 256) return dispatch_k<256>(batch, cfg, block_threads, grid_ctas, s, per_thread);
  if (block_threads <= 512) return dispatch_k<512>(batch, cfg, block_threads, grid_ctas, s, per_thread);
  if (block_threads <= 768) return dispatch_k<768>(batch, cfg, block_threads, grid_ctas, s, per_thread);
  return dispatch_k<1024>(batch, cfg, block_threads, grid_ctas, s, per_thread);
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
