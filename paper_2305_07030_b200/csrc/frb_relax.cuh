#pragma once
// frb_relax.cuh -- persistent dynamic-relaxation cluster kernel for sm_100a.
//
// A thread-block cluster of C CTAs ("ranks") owns one fiber network at a time,
// pulled from a device work queue (the spec's TeamBatched strategy,
// SPEC.md:361; the paper's "one team per sub-problem" kernel,
// PAPER.md:76-82).  C = 1 for networks that fit one SM; larger networks are
// split over the cluster by node range.  The whole Fig.-1 loop of the
// reference (_relax, pkg/src/fibrelax/microsolver.py:379-530) runs inside the
// kernel; finalize_result (:549-564) runs in its epilogue.
//
// Bit-exactness contract.  Every FP64 operation is an
// explicit round-to-nearest operation (intrinsics, or the branch-free fast
// paths of frb_arith.cuh that are bit-identical to them), so no FMA
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
//     order; aligned 4-leaf subtrees fold in the same warp (quad mode); the
//     rank evaluates the subtrees of its own leaves (local program), exports
//     their roots to every rank, and every rank replays the same top program
//     over all exports (plan.tree_split), so all ranks take the same
//     decisions.
//
// Work per iteration on each rank (T threads; own DOF d owned by thread d%T):
//   F1 coefs   per active element (>= 1 own endpoint): EA (l-L)/(L l)
//   F2 gather  per own node: f = A + B from the coefficients
//   A  per DOF k_hat, sq = (u k_hat) u, sq2 = (u m) u
//   C  chains  per (own leaf, chain): ordered sums of sq, sq2, f f, folds -> local tree slots
//   T  tree    warp 0: local program, exports (+ flags, ledger partials) to the
//              peers, wait, top program, c / residual / convergence; warps
//              1.. meanwhile form (-f)/m of every own DOF
//   U  per DOF a = (-f)/m - c v, two half kicks, drift, positions (+ halo push)
//
// Cluster exchange (C > 1).  Halo positions (U -> next F) and tree exports
// (T) travel as st.async stores into the peers' shared memory, each
// completing a transaction on the receiver's mbarrier; a rank waits on its
// own mbarriers only.  There is no cluster-wide barrier inside the loop: a
// cluster barrier's acquire invalidates L1 (CCTL.IVALL), which evicted the
// read-only tables the loop streams through L1 (profiles/r01_v4_ncu_c2.md).
// Each rank posts the byte count it expects for a phase (arrive.expect_tx)
// before any peer can send into that phase: the next halo phase is posted in
// A (peers send halos only after receiving this rank's exports of T), the
// next export phase right after the current one completes (peers send
// exports only after this rank's halo push of U).  When a problem ends, the
// two phases posted for an iteration that will not happen are completed
// locally (mbarrier.complete_tx) so the barriers are idle for the next
// problem.
//
// Shared memory per rank (offsets identical on every rank of a problem so a
// peer's buffer is addressed by the same offset; Layout):
//   pos   [PN][3]  positions (AoS) of own, halo and fixed local nodes; an own
//                  DOF's slot holds its sq between A and C.
//   fcur  [NFO]    f from F2 (C squares it where it sums f f); (-f)/m after T
//   fprv  [NFO]    f of the previous iteration; the current f after A (in
//                  global memory instead for networks too large for it)
//   cf    [CF]     F1 element coefficients, then sq2
//   lslot [LS][3]  local tree slots
//   tslot [2][TS][3], flag [2][64]  top tree slots and the peers' singular
//                  flags [16] + work-ledger partials [16][3], double-buffered
//                  by iteration parity: a peer that is not a halo neighbour
//                  can run one iteration ahead and send its next exports
//                  while this rank still reads the current ones (it cannot
//                  run two ahead: that needs this rank's next exports)
//   fin  [16]      per-rank final kinetic-energy partials (epilogue)
//   ack  [16]      halo-copy acknowledgements from the receiving ranks
//   rm    [NFO/3]  refined reciprocal (div_fast's r2) of each own node's
//                  mass: (-f)/m then costs 3 FP64 ops instead of 9 + MUFU
//   ms    [NFO/3]  the own nodes' masses (A and (-f)/m read them on chip)
//   prog           the rank's tree block (programs, exports)
// u, v and the reference coordinates of a thread's own DOFs live in registers.

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <type_traits>

#include "frb200.h"
#include "frb_arith.cuh"

namespace cg = cooperative_groups;

namespace frb_tu {
extern thread_local char g_err[512];
extern thread_local int g_launches;  // frb_solve_launches()
}

namespace {

constexpr int kMaxThreads = 1024;
constexpr int kMaxWarps = kMaxThreads / 32;
constexpr double kCollapse = 1e-12;  // microsolver.py:30
#ifndef FRB_KCHUNK
#define FRB_KCHUNK 4
#endif
constexpr int kChunk = FRB_KCHUNK;
// instrumentation slots (frb_batch.phase_cycles): F1, F2, A, C, T local tree +
// exports, T exchange wait, T top tree + scalars, U, epilogue, prologue, halo wait
constexpr int kPhases = 12;
enum { PH_F1, PH_F2, PH_A, PH_C, PH_TL, PH_TW, PH_TT, PH_U, PH_EPI, PH_PRO, PH_HALO, PH_TLP };  // per-DOF phases process a thread's DOFs in chunks of this many

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

// ------------------------------------------------------------------ cluster primitives

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// shared::cluster address of the same variable in CTA `rank`
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// 8-byte store into a peer's shared memory, completing 8 transaction bytes
// on the peer's mbarrier
__device__ __forceinline__ void st_async(uint32_t addr, double v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];"
               :
               : "r"(addr), "l"(__double_as_longlong(v)), "r"(bar)
               : "memory");
}
// Bulk copy (TMA engine) of `bytes` from this CTA's shared memory into a
// peer's, completing `bytes` transaction bytes on the peer's mbarrier.
// Addresses and size are 16-byte multiples (partition.py lays out the halo).
__device__ __forceinline__ void bulk_copy_to_peer(uint32_t dst, uint32_t src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :
               : "r"(dst), "r"(src), "r"(bytes), "r"(bar)
               : "memory");
}
// Generic-proxy shared-memory writes become visible to the async proxy (the
// bulk copies read what the threads wrote).
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" : : "r"(smem_u32(bar)), "r"(count) : "memory");
}
// this CTA's arrival for the current phase + the bytes the phase waits for
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               :
               : "r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// complete `bytes` of the current phase locally (no data will arrive)
__device__ __forceinline__ void mbar_complete(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.complete_tx.shared::cluster.relaxed.cluster.b64 [%0], %1;"
               :
               : "r"(mapa(smem_u32(bar), cg::this_cluster().block_rank())), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}

// ------------------------------------------------------------------ global-memory exchange
//
// Virtual clusters (kGM): a 16-CTA cluster must sit inside one GPC, so only
// 7 of them fit the GPU (112 of 148 SMs).  The remaining SMs run "virtual
// clusters": C independent CTAs (one per SM, no cluster launch) that solve a
// network together exchanging through L2 instead of DSMEM, with the same
// tables, layout and arithmetic.  Each virtual cluster owns a slice of the
// caller's exchange scratch (frb_batch.xchg, frb_group.xchg_off):
//   cnt [32][32] int  one 128-byte line per counter (pollers of one counter
//                     do not contend with the atomics of another): line r <
//                     16 halo bytes received by rank r, 16 exports arrived,
//                     17 barrier arrivals, 18 current problem
//   ex  [2][ex_stride] top-slot image (3 TS doubles) + 64 flag words, by
//                     iteration parity
//   mir [C][2][mir_stride/2] each rank's halo mirror: the bytes peers copy
//                     into its position array, by iteration parity
// Counters only grow: every wait is "counter >= the running expected value",
// so nothing is reset between problems.  Spins are bounded (trap after ~20 s)
// so a scheduling failure cannot hang the GPU.
struct Gx {
  int* cnt;
  double* ex;
  double* mir;
  int ex_stride, mir_stride;
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void gm_spin(const int* p, int target) {
  const long long t0 = clock64();
  while (ld_acquire(p) < target) {
    __nanosleep(20);  // back off: fewer polls contending with the producers' atomics
    if (clock64() - t0 > 40000000000LL) __trap();  // ~20 s: a virtual cluster that never assembled
  }
}

// ------------------------------------------------------------------ problem views

struct Net {
  int N, NF, M, C;
  int L, n_levels, root, ea_uniform;
  double dt, hdt, volume, ea;
  double g[9];  // F - I
  const double* X;
  const double* mass;   // per node
  const int2* incn;
  const int2* inc;
  const int2* eab;
  const double* EL;
  const double* EA;
  const int* plan;
  double* posg;  // [N][3] positions scratch (init checks, singular path, epilogue)
  int64_t node_base;
};

struct Rank {
  int node0, n_own, n_local, n_fix, n_act, n_int;
  int S, SA, SB, leaf0, n_leaves;
  int PN, NFO, CF;  // uniform SMEM extents of the problem (max over ranks)
  int LS, TS, PI;   // tree: local slots, top slots, block words (uniform)
  int tree_len, n_exp, root_top;
  uint32_t halo_bytes, leaf_bytes;  // transaction bytes this rank receives per phase
  uint32_t ack_from;                // ranks that copy halo positions to this one
  int n_runs, n_dst;                // outgoing halo copies, distinct ranks they go to
  const int4* runs;                 // (dst rank, src byte, dst byte, bytes)
  const int* tree;
  const uint32_t* ell;
  const uint32_t* act_ab;
  const double* act_L;
  const double* act_EA;
  const int* halo_g;
  const int* fix_g;
};

__device__ void load_views(Net& n, Rank& R, const frb_batch& b, int p, int r) {
  const frb_problem& P = b.problems[p];
  n.N = P.n_nodes;
  n.NF = P.n_free_nodes;
  n.M = P.n_elems;
  n.C = P.cluster;
  n.ea_uniform = P.flags & FRB_PF_EA_UNIFORM;
  n.dt = P.dt;
  n.hdt = dmul(0.5, P.dt);
  n.volume = P.volume;
  n.ea = P.ea;
  for (int i = 0; i < 3; ++i)
    for (int c = 0; c < 3; ++c) n.g[3 * i + c] = dsub(P.F[3 * i + c], i == c ? 1.0 : 0.0);
  n.node_base = P.node_base;
  n.X = b.X + 3 * P.node_base;
  n.mass = b.node_mass + P.node_base;
  n.incn = reinterpret_cast<const int2*>(b.inc_node) + P.tnode_base;
  n.inc = reinterpret_cast<const int2*>(b.inc) + P.inc_base;
  n.eab = reinterpret_cast<const int2*>(b.elem_ab) + P.telem_base;
  n.EL = b.elem_L + P.elem_base;
  n.EA = b.elem_EA ? b.elem_EA + P.elem_base : nullptr;
  n.plan = b.plans + P.plan_base;
  n.L = n.plan[0];
  n.n_levels = n.plan[1];
  n.root = n.plan[2];
  n.posg = b.work + 3 * P.node_base;
  const frb_part& Q = b.parts[P.part_base + r];
  R.node0 = Q.node0;
  R.n_own = Q.n_own;
  R.n_local = Q.n_local;
  R.n_fix = Q.n_fix;
  R.n_act = Q.n_act;
  R.n_int = Q.n_int;
  R.S = Q.ell_stride;
  R.SA = Q.slots_a;
  R.SB = Q.slots_b;
  R.leaf0 = Q.leaf0;
  R.n_leaves = Q.n_leaves;
  R.tree = b.trees + Q.tree_base;
  R.tree_len = Q.tree_len;
  R.LS = R.tree[0];
  R.TS = R.tree[1];
  R.PI = R.tree[2];
  R.n_exp = R.tree[6];
  R.root_top = R.tree[7];
  R.halo_bytes = static_cast<uint32_t>(Q.halo_bytes);
  R.ack_from = Q.ack_from;
  R.n_runs = Q.n_runs;
  R.runs = reinterpret_cast<const int4*>(b.runs) + Q.runs_base;
  {
    uint32_t dst = 0;
    for (int i = 0; i < Q.n_runs; ++i) dst |= 1u << R.runs[i].x;
    R.n_dst = __popc(dst);
  }
  R.leaf_bytes = 24u * static_cast<uint32_t>(R.tree[8] - R.n_exp) + 8u * static_cast<uint32_t>(n.C - 1);
  // uniform extents: maxima over the problem's ranks
  R.PN = R.NFO = R.CF = 0;
  for (int q = 0; q < n.C; ++q) {
    const frb_part& Qq = b.parts[P.part_base + q];
    R.PN = max(R.PN, Qq.n_local + Qq.n_fix);
    R.NFO = max(R.NFO, 3 * Qq.n_own);
    R.CF = max(R.CF, Qq.n_act);
  }
  R.CF = max(R.CF, R.NFO);
  R.ell = b.ell + Q.ell_base;
  R.act_ab = b.act_ab + Q.act_base;
  R.act_L = b.act_L + P.actv_base + Q.actv_off;
  R.act_EA = (b.act_EA && !n.ea_uniform) ? b.act_EA + P.actv_base + Q.actv_off : nullptr;
  R.halo_g = b.halo_g + Q.halo_base;
  R.fix_g = b.fix_g + Q.fix_base;
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

// Solver numbering, all positions from global memory.
struct PosGlobalAll {
  const double* posg;
  __device__ __forceinline__ double operator()(int node, int axis) const { return posg[3 * node + axis]; }
};
// X + u recomputed from global memory (one-shot internal_forces).
struct PosGlobal {
  const double* X;
  const double* u;
  __device__ __forceinline__ double operator()(int node, int axis) const {
    return dadd(X[3 * node + axis], u[3 * node + axis]);
  }
};
// Fixed nodes only: X + fixed_u(alpha), evaluated on the fly.
struct PosFixed {
  const Net* n;
  double alpha;
  bool ramp;
  __device__ __forceinline__ double operator()(int node, int axis) const {
    return dadd(n->X[3 * node + axis], fixed_u(*n, node, axis, alpha, ramp));
  }
};

// ------------------------------------------------------------------ element math

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

// E*A of element e: the descriptor's value when uniform (the per-element
// array is then not uploaded: frb_batch.elem_EA may be null)
__device__ __forceinline__ double elem_ea(const Net& n, int e) { return n.ea_uniform ? n.ea : n.EA[e]; }

// Internal force at node i from the CSR incidence lists (all nodes, solver
// numbering; used by the epilogue, the singular path and internal_forces).
template <class Pos>
__device__ __noinline__ bool node_force_csr(const Net& n, const Pos& pos, int i, double& fx, double& fy,
                                            double& fz) {
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
      bad |= element_force(dsub(ox, px), dsub(oy, py), dsub(oz, pz), n.EL[e.y], elem_ea(n, e.y), nx, ny, nz);
      ax = dsub(ax, nx);  // bincount(ia, -nd): 0 + (-nd) + ...
      ay = dsub(ay, ny);
      az = dsub(az, nz);
    } else {
      bad |= element_force(dsub(px, ox), dsub(py, oy), dsub(pz, oz), n.EL[e.y], elem_ea(n, e.y), nx, ny, nz);
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

// The rank's dynamic shared memory.  Hot loops index it with integer
// offsets (never through generic pointers), so every access is an LDS/STS
// with the CTA's shared window base held in one register.
extern __shared__ __align__(16) double g_smem[];

// Phase F1: coefficient EA (l - L) / (L l) of every active element of the
// rank, once per iteration (microsolver.py:196-211).  Elements cut by a rank
// boundary are evaluated by both ranks from identical operands.
#ifndef FRB_KELEM
#define FRB_KELEM 3
#endif
constexpr int kElem = FRB_KELEM;  // elements a thread keeps in flight in F1

__device__ __noinline__ LenCoef exact_elem(int o_pos, uint32_t ab, double L, double EA) {
  const double* pa = &g_smem[o_pos + 3 * static_cast<int>(ab & 0xffffu)];
  const double* pb = &g_smem[o_pos + 3 * static_cast<int>(ab >> 16)];
  return exact_len_coef(dsub(pb[0], pa[0]), dsub(pb[1], pa[1]), dsub(pb[2], pa[2]), L, EA);
}

// Active elements [first, end) of the rank: the interior ones (no halo
// endpoint, partition.py orders them first) overlap the halo copies, the cut
// ones follow the halo wait.
__device__ __forceinline__ bool element_coefs(int T, int first, int n_act, const uint32_t* __restrict__ act_ab,
                                              const double* __restrict__ act_L, const double* __restrict__ act_EA,
                                              double ea, int o_pos, int o_cf) {
  bool bad = false;
  if (first >= n_act) return bad;
  const int last = n_act - 1;
  for (int e0 = first + threadIdx.x; e0 < n_act; e0 += kElem * T) {
    uint32_t ab[kElem];
    double L[kElem], EA[kElem], l[kElem], cf[kElem];
    bool ok[kElem];
#pragma unroll
    for (int q = 0; q < kElem; ++q) {  // table loads of the whole group first
      const int e = min(e0 + q * T, last);
      ab[q] = __ldg(act_ab + e);
      L[q] = __ldg(act_L + e);
      EA[q] = act_EA ? __ldg(act_EA + e) : ea;
    }
#pragma unroll
    for (int q = 0; q < kElem; ++q) {  // independent chains: the scheduler interleaves them
      const double* pa = &g_smem[o_pos + 3 * static_cast<int>(ab[q] & 0xffffu)];
      const double* pb = &g_smem[o_pos + 3 * static_cast<int>(ab[q] >> 16)];
      const double dx = dsub(pb[0], pa[0]);
      const double dy = dsub(pb[1], pa[1]);
      const double dz = dsub(pb[2], pa[2]);
      bool ok1, ok2;
      l[q] = frb_arith::sqrt_fast(len2(dx, dy, dz), ok1);
      cf[q] = frb_arith::div_fast(dmul(EA[q], dsub(l[q], L[q])), dmul(L[q], l[q]), ok2);
      ok[q] = ok1 && ok2;
    }
    bool all_ok = true;
#pragma unroll
    for (int q = 0; q < kElem; ++q) all_ok &= ok[q];
    if (!all_ok) {  // one branch per group: the rare exact fallbacks
#pragma unroll
      for (int q = 0; q < kElem; ++q) {
        if (!ok[q]) {
          const LenCoef r = exact_elem(o_pos, ab[q], L[q], EA[q]);
          l[q] = r.l;
          cf[q] = r.coef;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < kElem; ++q) {
      const int e = e0 + q * T;
      const bool in = e < n_act;
      bad |= in & (l[q] < dmul(kCollapse, L[q]));
      if (in) g_smem[o_cf + e] = cf[q];
    }
  }
  return bad;
}

// Phase F2: internal force at own node i, summed over its slots in slot
// (= element) order: role a accumulates 0 - nd - nd ..., role b
// 0 + nd + nd ...  nd = d * coef with d = P[b] - P[a] recomputed from the
// operands F1 used, so it is bitwise the reference's per-element value.
// Padding slots point at node i itself (partition.py RankTables.ell): their
// d is +0 and they add a signed zero, which leaves the sums unchanged, so
// the gather is branch-free.  The slot words of a group are loaded up front
// so their latencies overlap.
constexpr int kSlots = 3;

// kOne: at most kSlots slots per role, a single unrolled group; kFull:
// exactly kSlots per role (lattices: 3 + 3), no padding selects
template <bool kRoleA, bool kOne, bool kFull>
__device__ __forceinline__ void gather_role(const uint32_t* __restrict__ ell_i, int S, int n_slots, int i,
                                            int o_pos, int o_cf, double px, double py, double pz, double& sx,
                                            double& sy, double& sz) {
  for (int k0 = 0; k0 < (kOne ? 1 : n_slots); k0 += kSlots) {
    if (kOne && n_slots == 0) break;
    uint32_t w[kSlots];
    w[0] = __ldg(ell_i + k0 * S);
    // slots past the end become self-padding of node i (a +-0 contribution)
    const uint32_t self_pad = (static_cast<uint32_t>(i) << 16) | (w[0] & 0xffffu);
#pragma unroll
    for (int q = 1; q < kSlots; ++q) w[q] = kFull || k0 + q < n_slots ? __ldg(ell_i + (k0 + q) * S) : self_pad;
#pragma unroll
    for (int q = 0; q < kSlots; ++q) {
      const double* po = &g_smem[o_pos + 3 * static_cast<int>(w[q] >> 16)];
      const double coef = g_smem[o_cf + static_cast<int>(w[q] & 0xffffu)];
      if (kRoleA) {  // bincount(ia, -nd): 0 + (-nd) + ...,  d = P[o] - P[i]
        sx = dsub(sx, dmul(dsub(po[0], px), coef));
        sy = dsub(sy, dmul(dsub(po[1], py), coef));
        sz = dsub(sz, dmul(dsub(po[2], pz), coef));
      } else {  // bincount(ib, nd),  d = P[i] - P[o]
        sx = dadd(sx, dmul(dsub(px, po[0]), coef));
        sy = dadd(sy, dmul(dsub(py, po[1]), coef));
        sz = dadd(sz, dmul(dsub(pz, po[2]), coef));
      }
    }
  }
}

// f of every own node into g_smem[o_out + 3 i + axis]; a thread gathers two
// of its nodes together so their load latencies overlap
template <bool kOne, bool kFull>
__device__ __forceinline__ void node_force(const uint32_t* __restrict__ ell, int S, int SA, int SB, int o_pos,
                                           int o_cf, int o_out, int i) {
  const double px = g_smem[o_pos + 3 * i], py = g_smem[o_pos + 3 * i + 1], pz = g_smem[o_pos + 3 * i + 2];
  double ax = 0.0, ay = 0.0, az = 0.0, bx = 0.0, by = 0.0, bz = 0.0;
  gather_role<true, kOne, kFull>(ell + i, S, SA, i, o_pos, o_cf, px, py, pz, ax, ay, az);
  gather_role<false, kOne, kFull>(ell + SA * S + i, S, SB, i, o_pos, o_cf, px, py, pz, bx, by, bz);
  g_smem[o_out + 3 * i] = dadd(ax, bx);
  g_smem[o_out + 3 * i + 1] = dadd(ay, by);
  g_smem[o_out + 3 * i + 2] = dadd(az, bz);
}

template <bool kOne, bool kFull>
__device__ __forceinline__ void node_forces_t(int T, int n_own, const uint32_t* __restrict__ ell, int S, int SA,
                                              int SB, int o_pos, int o_cf, int o_out) {
  int i = threadIdx.x;
  for (; i + T < n_own; i += 2 * T) {
    node_force<kOne, kFull>(ell, S, SA, SB, o_pos, o_cf, o_out, i);
    node_force<kOne, kFull>(ell, S, SA, SB, o_pos, o_cf, o_out, i + T);
  }
  if (i < n_own) node_force<kOne, kFull>(ell, S, SA, SB, o_pos, o_cf, o_out, i);
}

__device__ __forceinline__ void node_forces(int T, int n_own, const uint32_t* __restrict__ ell, int S, int SA, int SB,
                                            int o_pos, int o_cf, int o_out) {
  if (SA == kSlots && SB == kSlots) {  // a lattice's 3 + 3 incidences
    node_forces_t<true, true>(T, n_own, ell, S, SA, SB, o_pos, o_cf, o_out);
  } else if (SA <= kSlots && SB <= kSlots) {
    node_forces_t<true, false>(T, n_own, ell, S, SA, SB, o_pos, o_cf, o_out);
  } else {
    node_forces_t<false, false>(T, n_own, ell, S, SA, SB, o_pos, o_cf, o_out);
  }
}

// ------------------------------------------------------------------ block helpers

struct Scalars {
  long long clk[kPhases];  // per-phase cycle totals (thread 0, when instrumented)
  long long t_last;
  double c, residual, r_ref, threshold;
  double red[kMaxWarps * 9];
  int ired[kMaxWarps];
  int problem, done, converged, singular;
  int gx_h, gx_s, gx_b;                  // kGM: expected counter values (thread 0)
  // tree-phase context (warp 0 re-reads it from shared memory each
  // iteration: held in registers across the loop it spilled to local memory,
  // and every reload cost an L2 round trip on the serial critical path)
  int tp_lprog, tp_tprog, tp_exps, tp_n_exp, tp_root, tp_lslot, tp_tslot, tp_flag, tp_TS;
  uint32_t peer_smem[FRB_MAX_CLUSTER];  // shared::cluster base of each rank's dynamic SMEM
  uint32_t peer_bar_h[FRB_MAX_CLUSTER]; // each rank's halo mbarrier
  uint32_t peer_bar_s[FRB_MAX_CLUSTER]; // each rank's leaf-sum mbarrier
  uint32_t peer_bar_a[FRB_MAX_CLUSTER]; // each rank's halo-copy acknowledgement mbarrier
};

// Phase timing: thread 0 charges the cycles since the previous mark to
// phase `ph` (called right after a barrier, so it measures the critical path).
__device__ __forceinline__ void mark(Scalars& sc, bool on, int ph) {
  if (on && threadIdx.x == 0) {
    const long long now = clock64();
    sc.clk[ph] += now - sc.t_last;
    sc.t_last = now;
  }
}

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
__device__ __noinline__ int singular_argmin(const Net& n, const Pos& pos, Scalars& sc) {
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

// Length check of elements whose endpoints are both fixed (their only motion
// is the BC ramp; every other element is checked in F1).  With all_elements,
// every element is checked.
template <class Pos>
__device__ __noinline__ bool check_elements(const Net& n, const Pos& pos, bool all_elements) {
  bool bad = false;
  for (int e = threadIdx.x; e < n.M; e += blockDim.x) {
    const int2 ab = n.eab[e];
    if (!all_elements && (ab.x < n.NF || ab.y < n.NF)) continue;
    const double dx = dsub(pos(ab.y, 0), pos(ab.x, 0));
    const double dy = dsub(pos(ab.y, 1), pos(ab.x, 1));
    const double dz = dsub(pos(ab.y, 2), pos(ab.x, 2));
    bad |= seg_len(dx, dy, dz) < dmul(kCollapse, n.EL[e]);
  }
  return bad;
}

// Fixed-node positions into global scratch, split over the cluster's ranks.
__device__ __noinline__ void set_fixed_positions(const Net& n, int rank, double alpha, bool ramp) {
  for (int i = n.NF + rank * blockDim.x + threadIdx.x; i < n.N; i += n.C * blockDim.x)
    for (int j = 0; j < 3; ++j) n.posg[3 * i + j] = dadd(n.X[3 * i + j], fixed_u(n, i, j, alpha, ramp));
}

// Fixed-node positions of the rank's local copies (SMEM).
__device__ __forceinline__ void set_local_fixed(const Net& n, const Rank& R, double* pos, double alpha, bool ramp) {
  for (int k = threadIdx.x; k < R.n_fix; k += blockDim.x) {
    const int g = __ldg(R.fix_g + k);
    double* p = pos + 3 * (R.n_local + k);
    for (int j = 0; j < 3; ++j) p[j] = dadd(n.X[3 * g + j], fixed_u(n, g, j, alpha, ramp));
  }
}

__device__ __forceinline__ double ramp_alpha(int it_plus_1, int ramp) {
  // Python: min(1.0, (it + 1) / ramp)
  const double x = ddiv(static_cast<double>(it_plus_1), static_cast<double>(ramp));
  return x < 1.0 ? x : 1.0;
}

// Cluster-wide barrier with release/acquire semantics (DSMEM and global
// memory writes before it are visible after it); a CTA barrier when C == 1.
// Used once or twice per problem, never inside the relaxation loop.
__device__ __forceinline__ void csync(int C) {
  if (C > 1) {
    cg::this_cluster().sync();
  } else {
    __syncthreads();
  }
}

// Barrier over the ranks of a problem: cluster barrier, or (virtual
// cluster) an arrival counter in global memory.
template <bool kGM>
__device__ __forceinline__ void gsync(int C, Scalars& sc, const Gx& gx) {
  if constexpr (kGM) {
    __threadfence();  // every thread's global writes (positions, outputs) before the arrival
    __syncthreads();
    if (threadIdx.x == 0) {
      atomicAdd(gx.cnt + 32 * 17, 1);
      sc.gx_b += C;
      gm_spin(gx.cnt + 32 * 17, sc.gx_b);
      __threadfence();
    }
    __syncthreads();
  } else {
    csync(C);
  }
}

template <class T>
__device__ __forceinline__ T* peer(T* p, int q) {
  return cg::this_cluster().map_shared_rank(p, q);
}

// Epilogue on rank 0: reactions at the fixed nodes from the final positions
// (posg), their displacements, sigma = sym(sum r (x) x)/V (microsolver.py:
// 285-299; deterministic order, tolerance-only vs the reference's BLAS) and
// the result record.
__device__ __noinline__ void fixed_forces_and_stress(const frb_batch& b, int p, const Net& n, Scalars& sc,
                                                     int it, double alpha, bool ramp, int full_bc_iter,
                                                     bool energy, const double* w) {
  const int T = blockDim.x, t = threadIdx.x;
  double* uo = b.u + 3 * n.node_base;
  double* fo = b.f + 3 * n.node_base;
  double s9[9];
#pragma unroll
  for (int r = 0; r < 9; ++r) s9[r] = 0.0;
  const PosGlobalAll G{n.posg};
  for (int i = n.NF + t; i < n.N; i += T) {
    double f3[3];
    node_force_csr(n, G, i, f3[0], f3[1], f3[2]);
    for (int jj = 0; jj < 3; ++jj) {
      uo[3 * i + jj] = fixed_u(n, i, jj, alpha, ramp);
      fo[3 * i + jj] = f3[jj];
    }
    // S = r^T x over boundary nodes (sorted ids == solver order), x = X + u
    for (int a = 0; a < 3; ++a)
      for (int c3 = 0; c3 < 3; ++c3) s9[3 * a + c3] = dadd(s9[3 * a + c3], dmul(f3[a], G(i, c3)));
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
    // energy_balance (microsolver.py:274-282): w = {w_kin, w_int, w_damp, w_ext}
    r.energy_residual = qnan();
    for (int e = 0; e < 4; ++e) r.energy[e] = energy ? w[e] : 0.0;
    if (energy) {
      const double defect = fabs(dsub(dsub(dsub(w[3], w[1]), w[0]), w[2]));
      double den = fabs(w[3]);
      if (fabs(w[1]) > den) den = fabs(w[1]);
      if (w[0] > den) den = w[0];
      if (1e-30 > den) den = 1e-30;  // ENERGY_FLOOR, microsolver.py:29
      r.energy_residual = ddiv(defect, den);
    }
  }
}

// Work ledger terms at the fixed nodes (rank 0, every thread; positions of
// all nodes in posg): the reactions f_fix from the incidence lists, then
//   mode 0: sum f_fix . u_presc                        (initial BC step)
//   mode 1: store f_fix as the previous reactions       (ramp, iteration -1)
//   mode 2: sum f_fix . du and sum f_prev_fix . du with du = d_alpha u_presc,
//           then store f_fix                            (ramp iterations)
// f_prev_fix lives in the fixed-DOF part of the u output (written only by
// the epilogue).  Returns {sum1, sum2} in thread 0 (any order: the
// reference's np.dot is BLAS-ordered, the ledger is tolerance-only).
__device__ __noinline__ void energy_fixed(const frb_batch& b, const Net& n, Scalars& sc, int mode, double d_alpha,
                                          double* out) {
  double s9[9];
#pragma unroll
  for (int r = 0; r < 9; ++r) s9[r] = 0.0;
  double* fprev_fix = b.u + 3 * n.node_base;
  const PosGlobalAll G{n.posg};
  for (int i = n.NF + threadIdx.x; i < n.N; i += blockDim.x) {
    double f3[3];
    node_force_csr(n, G, i, f3[0], f3[1], f3[2]);
    for (int j = 0; j < 3; ++j) {
      const double up = presc(n, i, j);
      if (mode == 0) {
        s9[0] = dadd(s9[0], dmul(f3[j], up));
      } else if (mode == 2) {
        const double du = dmul(d_alpha, up);
        s9[0] = dadd(s9[0], dmul(f3[j], du));
        s9[1] = dadd(s9[1], dmul(fprev_fix[3 * i + j], du));
      }
      fprev_fix[3 * i + j] = f3[j];
    }
  }
  block_sum9(s9, sc);
  if (threadIdx.x == 0) {
    out[0] = s9[0];
    out[1] = s9[1];
  }
}

__device__ __forceinline__ void write_singular(const frb_batch& b, int p, int bad, int iters) {
  frb_result& r = b.results[p];
  r.status = FRB_STATUS_SINGULAR;
  r.bad_element = bad;
  r.iters = iters;
  r.converged = 0;
  r.final_residual = r.r_ref = r.energy_residual = qnan();
}

// ------------------------------------------------------------------ the solve

// SMEM layout of a problem, in doubles from g_smem (identical on every
// rank of the problem, so a peer's buffer is addressed by the same offset).
struct Layout {
  int pos, fcur, fprv, cf, lslot, tslot, flag, rm, ms, prog;  // prog: int32 index
};

// kFG (the networks too large for on-chip f_prev) also read the node masses
// from global memory: a runtime switch between the two cost 20 % on C3 (the
// extra live state spills)
template <bool kFG>
__device__ __forceinline__ Layout layout(const Rank& R) {
  Layout o;
  o.pos = 0;
  o.fcur = 3 * R.PN;
  o.fprv = o.fcur + R.NFO;
  o.cf = o.fprv + (kFG ? 0 : R.NFO);
  o.lslot = o.cf + R.CF;
  o.tslot = o.lslot + 3 * R.LS;
  o.flag = o.tslot + 6 * R.TS;  // two parity buffers of top slots
  o.rm = o.flag + 2 * 64 + 32;    // two parity buffers of flags[16] + partials[16][3]; fin[16]; ack[16]
  o.ms = o.rm + R.NFO / 3;                    // refined reciprocal masses of the own nodes
  o.prog = 2 * (o.ms + (kFG ? 0 : R.NFO / 3));  // the own nodes' masses (on chip unless kFG)
  return o;
}

// Replay one combine program (plan.py _program: warp rounds of up to 32
// independent ops, lane-packed, slot indices premultiplied by 3, idle lanes
// folding their own scratch slots, one idle pad round) on g_smem[o_slot + ...] with
// the calling warp: no branch in the loop, the next round's op is fetched
// while the current one runs.  Not unrolled: a single warp runs it while
// the rest of the CTA waits, so its code must stay small.
__device__ __forceinline__ void run_prog(const int* prog, int o_slot, int lane) {
  const int nr = prog[0];
  const int2* w = reinterpret_cast<const int2*>(prog + 2) + lane;  // 8-byte aligned (plan.py _program)
  double* const sl = &g_smem[o_slot];
  int2 cur = w[0];
#pragma unroll 1
  for (int r = 0; r < nr; ++r) {
    w += 32;
    const int2 nxt = w[0];
    const double* pa = sl + (cur.y & 0xffff);
    const double* pb = sl + (cur.y >> 16);
    const double a0 = pa[0], a1 = pa[1], a2 = pa[2];
    const double b0 = pb[0], b1 = pb[1], b2 = pb[2];
    double* pd = sl + cur.x;
    pd[0] = dadd(a0, b0);
    pd[1] = dadd(a1, b1);
    pd[2] = dadd(a2, b2);
    __syncwarp();
    cur = nxt;
  }
}

struct Mbar {
  uint64_t* h;   // halo positions (bulk copies from the peers)
  uint64_t* s;   // leaf sums + flags
  uint64_t* a;   // acknowledgements of this rank's outgoing halo copies
  uint32_t ph_h, ph_s, ph_a;
};

// Complete the two phases posted for an iteration that will not run, so the
// barriers are idle for the next problem (see the header comment).
__device__ __forceinline__ void drain(Mbar& mb, uint32_t halo_bytes, uint32_t leaf_bytes) {
  if (threadIdx.x == 0) {
    mbar_complete(mb.h, halo_bytes);
    mbar_complete(mb.s, leaf_bytes);
  }
  mbar_wait(mb.h, mb.ph_h);
  mbar_wait(mb.s, mb.ph_s);
  mb.ph_h ^= 1u;
  mb.ph_s ^= 1u;
}

template <int MAXK, bool kFG, bool kEnergy, int kT, bool kGM>
__device__ void solve_problem(const frb_batch& b, const frb_config& cfg, int p, int rank, Scalars& sc, Mbar& mb,
                              const Net& n, const Rank& R, const Gx& gx) {
  static_assert(!(kGM && kEnergy), "the work ledger runs on hardware clusters only");
  // kT > 0: the kernel is launched with exactly kT threads, so every
  // DOF-strided index t + k T folds its stride into immediate offsets
  const int T = kT > 0 ? kT : static_cast<int>(blockDim.x);
  const int t = threadIdx.x, lane = t & 31;
  const int C = n.C, L = n.L, n_own = R.n_own, nfo = 3 * n_own;
  const Layout o = layout<kFG>(R);
  const double* __restrict__ Xg = n.X;
  const double* __restrict__ nmass = n.mass + R.node0;  // own nodes' masses
  const int dof0 = 3 * R.node0;
  // clamp for unconditional per-DOF loads of read-only data (X, masses);
  // data other threads write (f, f_prev) is only read for owned DOFs
  const int dl_max = nfo > 0 ? nfo - 1 : 0;
  const int nk = t < nfo ? (nfo - 1 - t) / T + 1 : 0;  // DOFs this thread owns
  const int dl_last = t + (nk > 0 ? nk - 1 : 0) * T;
  // hot per-rank tables and sizes, held in registers
  const uint32_t* __restrict__ ell = R.ell;
  const int S = R.S, SA = R.SA, SB = R.SB, n_act = R.n_act;
  const uint32_t* __restrict__ act_ab = R.act_ab;
  const double* __restrict__ act_L = R.act_L;
  const double* __restrict__ act_EA = R.act_EA;
  const double ea = n.ea;
  const uint32_t peer_pos = 8u * o.pos;  // byte offsets in a peer's dynamic SMEM
  // f_prev of own DOF dl: SMEM, or the `f` output array for networks too
  // large for the cluster's SMEM (it ends up holding the final f either way)
  double* const fprv_g = b.f + 3 * n.node_base + dof0;
  // (value getter / setter: a generic reference into shared memory would
  // hide the address space from the compiler)
  auto FPRV = [&](int dl) -> double { return kFG ? fprv_g[dl] : g_smem[o.fprv + dl]; };
  auto SET_FPRV = [&](int dl, double x) {
    if (kFG) {
      fprv_g[dl] = x;
    } else {
      g_smem[o.fprv + dl] = x;
    }
  };

  // the rank's tree block (local + top programs, exports) lives in SMEM
  int* const prog = reinterpret_cast<int*>(g_smem) + o.prog;
  for (int k = t; k < R.tree_len; k += T) prog[k] = __ldg(R.tree + k);
  // kFG: the one per-node SMEM slot holds the mass itself (A reads it every
  // iteration); (-f)/m then runs the full division in the shadow of the tree
  // phase.  Otherwise both the mass and its refined reciprocal are on chip.
  for (int i = t; i < n_own; i += T) {
    const double m = __ldg(nmass + i);
    if constexpr (kFG) {
      g_smem[o.rm + i] = m;
    } else {
      g_smem[o.ms + i] = m;
      g_smem[o.rm + i] = frb_arith::rcp_refined(m);
    }
  }
  auto MASS = [&](int i) -> double { return g_smem[(kFG ? o.rm : o.ms) + i]; };
  if (t == 0) {
    sc.tp_lprog = o.prog + R.tree[3];
    sc.tp_tprog = o.prog + R.tree[4];
    sc.tp_exps = o.prog + R.tree[5];
    sc.tp_n_exp = R.n_exp;
    sc.tp_root = R.root_top;
    sc.tp_lslot = o.lslot;
    sc.tp_tslot = o.tslot;
    sc.tp_flag = o.flag;
    sc.tp_TS = R.TS;
  }
  const bool quad_mode = (R.tree[9] & 4) != 0;  // plan.py MODE_QUAD

  const bool adaptive = cfg.damping == FRB_DAMPING_ADAPTIVE;
  const int ramp_n = cfg.bc_ramp_iters;
  const bool ramp = ramp_n > 0;
  const int full_bc_iter = ramp ? ramp_n - 1 : 0;
  const double dt = n.dt, hdt = n.hdt;
  double alpha = ramp ? -1.0 : 1.0;  // -1: fixed nodes still at their zero init
  const bool prof = b.phase_cycles != nullptr;
  // work ledger (energy_check_interval > 0, used as a flag like the
  // reference, microsolver.py:395, 510): rank 0's thread 0 keeps
  // w = {w_kin, w_int, w_damp, w_ext}; the other ranks send it their
  // per-iteration partial dots with the exchange
  constexpr bool energy = kEnergy;  // == (cfg.energy_check_interval > 0), dispatched per kernel
  const bool eramp = energy && ramp;  // reactions at the ramped fixed nodes each ramp step
  const uint32_t leaf_bytes = R.leaf_bytes + ((energy && rank == 0) ? 24u * static_cast<uint32_t>(C - 1) : 0u);
  double w[4] = {0.0, 0.0, 0.0, 0.0};
  double alpha_prev = 0.0;  // alpha of the previous step (d_alpha, microsolver.py:451)

  // own DOF dl = t + k*T (local DOF; global DOF dof0 + dl)
  double u[MAXK], v[MAXK];
#pragma unroll
  for (int k = 0; k < MAXK; ++k) u[k] = v[k] = 0.0;

  // pairwise-chain role: in chain round k thread t sums chain j = t % 8 of
  // own leaf t / 8 + k T / 8; the leaves' (start, size) come from the tree
  // block in shared memory each round (no per-problem registers)
  const int j = t & 7;
  const int2* const leaf_tab = reinterpret_cast<const int2*>(prog + R.tree[10]);

  // reference coordinates of the own DOFs stay in registers (re-reading
  // them from global memory in U measured slower: C3 wave 63.3 vs 58.9 ms)
  double xr[MAXK];
#pragma unroll
  for (int k = 0; k < MAXK; ++k) xr[k] = __ldg(Xg + dof0 + min(t + k * T, dl_max));

  auto put_local = [&](int dl, double x) {
    g_smem[o.pos + dl] = x;
    if (eramp && alpha < 1.0) n.posg[dof0 + dl] = x;  // ramp reactions read every position
  };
  // Halo exchange (thread 0, after every thread's position writes, a proxy
  // fence and a CTA barrier): one bulk DSMEM copy per run of own nodes a peer
  // keeps as halo, completing on the peer's halo mbarrier; the peers
  // acknowledge receipt on this rank's ack mbarrier, which A waits for
  // before it reuses the own position slots as sq scratch.
  const uint32_t smem_base = smem_u32(g_smem);
  auto issue_halo = [&]() {
    if constexpr (kGM) return;  // see gm_send_halo
    if (R.n_dst > 0) mbar_expect(mb.a, 8u * static_cast<uint32_t>(R.n_dst));
    for (int i = 0; i < R.n_runs; ++i) {
      const int4 run = __ldg(R.runs + i);
      bulk_copy_to_peer(sc.peer_smem[run.x] + static_cast<uint32_t>(run.z), smem_base + static_cast<uint32_t>(run.y),
                        static_cast<uint32_t>(run.w), sc.peer_bar_h[run.x]);
    }
  };
  auto ack_halo = [&]() {  // thread 0, after the halo wait
    if constexpr (kGM) return;  // the mirrors are double-buffered: nothing to acknowledge
    for (uint32_t bits = R.ack_from; bits; bits &= bits - 1) {
      const int qr = __ffs(bits) - 1;
      st_async(sc.peer_smem[qr] + 8u * static_cast<uint32_t>(o.flag + 144 + rank), 0.0, sc.peer_bar_a[qr]);
    }
  };

  // kGM halo exchange: every thread copies its share of the outgoing runs
  // into the receivers' mirrors (16-byte stores), then thread 0 publishes the
  // bytes with a release add on each receiver's counter; a receiver waits
  // for its running total and copies its halo slots back from its mirror.
  auto gm_send_halo = [&]() {
    if constexpr (kGM) {
      const int par = static_cast<int>(mb.ph_h);
      for (int i = 0; i < R.n_runs; ++i) {
        const int4 run = __ldg(R.runs + i);
        const double2* src = reinterpret_cast<const double2*>(&g_smem[o.pos] + run.y / 8);
        double2* dst = reinterpret_cast<double2*>(gx.mir + static_cast<int64_t>(run.x) * gx.mir_stride +
                                                  par * (gx.mir_stride / 2) + run.z / 8);
        for (int k = t; k < run.w / 16; k += T) dst[k] = src[k];
      }
      __threadfence();  // each thread's mirror stores visible GPU-wide before the release below
      __syncthreads();
      if (t == 0) {
        for (int i = 0; i < R.n_runs; ++i) {
          const int4 run = __ldg(R.runs + i);
          atomicAdd(gx.cnt + 32 * run.x, run.w);
        }
      }
    }
  };
  auto gm_recv_halo = [&]() {
    if constexpr (kGM) {
      const int par = static_cast<int>(mb.ph_h);
      if (t == 0) {
        sc.gx_h += static_cast<int>(R.halo_bytes);
        gm_spin(gx.cnt + 32 * rank, sc.gx_h);
        __threadfence();
      }
      __syncthreads();
      const double* src = gx.mir + static_cast<int64_t>(rank) * gx.mir_stride + par * (gx.mir_stride / 2);
      const int hi = 3 * R.n_local;
      for (int k0 = 3 * n_own + t; k0 < hi; k0 += 8 * T) {  // 8 L2 loads in flight per thread
        double tmp[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) tmp[q] = k0 + q * T < hi ? __ldcg(src + k0 + q * T) : 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (k0 + q * T < hi) g_smem[o.pos + k0 + q * T] = tmp[q];
      }
      __syncthreads();
    }
  };

  // (-f)/m of every own DOF into its f slot of SMEM (free once C has
  // consumed f f): threads first .. first + n - 1 cover all DOFs, four per
  // step so the divisions overlap; rare exact fallback.  In the loop the
  // warps other than warp 0 do it while warp 0 runs the tree phase.
  auto accel = [&](int first, int nthr) {
    for (int d0 = t - first; d0 < nfo; d0 += kChunk * nthr) {
      double q[kChunk];
      bool ok[kChunk];
#pragma unroll
      for (int kk = 0; kk < kChunk; ++kk) {
        // past the end: re-read this thread's own DOF d0 (it rewrites it
        // below, in program order), never another thread's slot
        const int dl = d0 + kk * nthr < nfo ? d0 + kk * nthr : d0;
        const int i = dl / 3;  // f of this iteration, left in fcur by A
        if constexpr (kFG) {
          q[kk] = frb_arith::div_fast(-g_smem[o.fcur + dl], MASS(i), ok[kk]);
        } else {
          q[kk] = frb_arith::div_fast_r(-g_smem[o.fcur + dl], MASS(i), g_smem[o.rm + i], ok[kk]);
        }
      }
      bool all_ok = true;
#pragma unroll
      for (int kk = 0; kk < kChunk; ++kk) all_ok &= ok[kk];
      if (!all_ok) {  // one branch per chunk: the rare exact fallbacks
#pragma unroll
        for (int kk = 0; kk < kChunk; ++kk) {
          const int dl = d0 + kk * nthr;
          if (!ok[kk] && dl < nfo) q[kk] = exact_div(-g_smem[o.fcur + dl], MASS(dl / 3));
        }
      }
#pragma unroll
      for (int kk = 0; kk < kChunk; ++kk) {
        const int dl = d0 + kk * nthr;
        if (dl < nfo) g_smem[o.fcur + dl] = q[kk];
      }
    }
  };

  // ---- prologue: BCs, initial positions (microsolver.py:400-411) ---------
  // post the first halo and leaf-sum phases before any peer may send
  if (!kGM && C > 1 && t == 0) {
    mbar_expect(mb.h, R.halo_bytes);
    mbar_expect(mb.s, leaf_bytes);
  }
  for (int l = t; l < R.n_local; l += T) {
    const int g = l < n_own ? R.node0 + l : R.halo_g[l - n_own];
    for (int a = 0; a < 3; ++a) g_smem[o.pos + 3 * l + a] = dadd(Xg[3 * g + a], 0.0);
  }
  set_local_fixed(n, R, &g_smem[o.pos], alpha, ramp);
  set_fixed_positions(n, rank, alpha, ramp);
  // initial free positions to global too (the all-element check reads posg)
  for (int l = t; l < n_own; l += T)
    for (int a = 0; a < 3; ++a) n.posg[3 * (R.node0 + l) + a] = dadd(Xg[3 * (R.node0 + l) + a], 0.0);
  gsync<kGM>(C, sc, gx);
  if (check_elements(n, PosGlobalAll{n.posg}, true)) sc.singular = 1;
  __syncthreads();
  if (sc.singular) {
    if (!kGM && C > 1) drain(mb, R.halo_bytes, leaf_bytes);
    const int bad = singular_argmin(n, PosGlobalAll{n.posg}, sc);
    if (rank == 0 && t == 0) write_singular(b, p, bad, 0);
    return;
  }
  // initial internal forces on own nodes (:413-420), kept as f_prev
  element_coefs(T, 0, n_act, act_ab, act_L, act_EA, ea, o.pos, o.cf);
  __syncthreads();
  node_forces(T, n_own, ell, S, SA, SB, o.pos, o.cf, o.fcur);
  __syncthreads();
  for (int dl = t; dl < nfo; dl += T) SET_FPRV(dl, g_smem[o.fcur + dl]);
  __syncthreads();
  if (energy && rank == 0) {  // initial BC step work (:421-425), or the reactions before the ramp
    double e2[2];
    energy_fixed(b, n, sc, ramp ? 1 : 0, 0.0, e2);
    if (t == 0 && !ramp) {
      const double step = dmul(0.5, e2[0]);
      w[3] = dadd(w[3], step);
      w[1] = dadd(w[1], step);
    }
  }
  if (eramp) csync(C);  // rank 0 has read the initial positions before any rank drifts (ledger: clusters only)

  // a = -f/m (:428-430), then iteration 0's kick + drift (:443-448)
  accel(0, T);
  __syncthreads();
#pragma unroll
  for (int k = 0; k < MAXK; ++k) {
    const int dl = t + k * T;
    if (dl < nfo) {
      v[k] = dadd(0.0, dmul(hdt, g_smem[o.fcur + dl]));
      u[k] = dadd(0.0, dmul(dt, v[k]));
      put_local(dl, dadd(xr[k], u[k]));
    }
  }
  if (ramp) {  // iteration 0's ramp step (:449-453)
    alpha = ramp_alpha(1, ramp_n);
    set_local_fixed(n, R, &g_smem[o.pos], alpha, ramp);
    if (energy) set_fixed_positions(n, rank, alpha, ramp);
  }
  if (C > 1) fence_proxy_async();
  __syncthreads();

  // ---- relaxation loop (microsolver.py:434-530) ---------------------------
  mark(sc, prof, PH_PRO);
  int it = 0;
  for (;; ++it) {
    double wfix = 0.0;  // ramp work at the fixed nodes this step (rank 0, thread 0)
    if (eramp && it < ramp_n) {
      csync(C);  // every rank's positions of this step are in posg
      if (rank == 0) {
        double e2[2];
        energy_fixed(b, n, sc, 2, dsub(alpha, alpha_prev), e2);
        if (t == 0) wfix = dmul(0.5, dadd(e2[0], e2[1]));
      }
      alpha_prev = alpha;
    }
    // F: internal forces at the drifted positions (:456-465).  With peers:
    // send this rank's halo copies, evaluate the interior elements while
    // they fly, then wait for the peers' copies, acknowledge them and
    // evaluate the elements cut by the rank boundary.
    if (C > 1 && t == 0) issue_halo();
    if (C > 1) gm_send_halo();
    bool bad = element_coefs(T, 0, C > 1 ? R.n_int : n_act, act_ab, act_L, act_EA,
                             ea, o.pos, o.cf);
    if (C > 1) {
      mark(sc, prof, PH_F1);
      if constexpr (kGM) {
        gm_recv_halo();
      } else {
        mbar_wait(mb.h, mb.ph_h);
      }
      mb.ph_h ^= 1u;
      if (t == 0) ack_halo();
      mark(sc, prof, PH_HALO);
      bad |= element_coefs(T, R.n_int, n_act, act_ab, act_L, act_EA, ea,
                           o.pos, o.cf);
    }
    if (ramp && it < ramp_n && rank == 0) bad |= check_elements(n, PosFixed{&n, alpha, ramp}, false);
    __syncthreads();
    mark(sc, prof, PH_F1);
    node_forces(T, n_own, ell, S, SA, SB, o.pos, o.cf, o.fcur);
    if (bad) sc.singular = 1;
    __syncthreads();
    mark(sc, prof, PH_F2);

    // A: k_hat = (f - f_prev)/(dt v) where dt v != 0 else 0, clamped with
    // np.maximum(k_hat, 0) (:468-476); sq = (u k_hat) u, sq2 = (u m) u,
    // f f (:489) is formed by C.  Outputs: sq -> own position slot, sq2 -> cf,
    // f stays in fcur and is copied to fprv.
    if (!kGM && C > 1 && t == 0) mbar_expect(mb.h, R.halo_bytes);  // next halo phase
    if (!kGM && C > 1 && R.n_dst > 0) {  // the peers have read this rank's positions (they become sq below)
      mbar_wait(mb.a, mb.ph_a);
      mb.ph_a ^= 1u;
    }
    double es[3] = {0.0, 0.0, 0.0};
    // damping mode hoisted out of the per-DOF loop (one copy per mode)
    auto a_phase = [&](auto ad) {
      constexpr bool kAd = decltype(ad)::value;
      if (nk > 0)
#pragma unroll
      for (int k0 = 0; k0 < MAXK; k0 += kChunk) {
        constexpr int KC = MAXK < kChunk ? MAXK : kChunk;
        double f[KC], kh[KC], m[KC];
        bool ok[KC];
#pragma unroll
        for (int kk = 0; kk < KC; ++kk) {
          // unowned slots re-read the thread's own last DOF (written only by
          // this thread, later in program order): no other thread's data
          const int dl = k0 + kk < nk ? t + (k0 + kk) * T : dl_last;
          f[kk] = g_smem[o.fcur + dl];
          kh[kk] = FPRV(dl);  // f_prev, until the quotient replaces it
          m[kk] = MASS(dl / 3);
        }
        if constexpr (kAd) {
#pragma unroll
          for (int kk = 0; kk < KC; ++kk) {
            const double vk = k0 + kk < MAXK ? v[k0 + kk] : 0.0;
            const double den = dmul(dt, vk);
            const double num = dsub(f[kk], kh[kk]);
            kh[kk] = frb_arith::div_fast(num, den, ok[kk]);
            if (den == 0.0) {
              kh[kk] = 0.0;
              ok[kk] = true;
            }
          }
          bool all_ok = true;
#pragma unroll
          for (int kk = 0; kk < KC; ++kk) all_ok &= ok[kk];
          if (!all_ok) {  // one branch per chunk: the rare exact fallbacks
#pragma unroll
            for (int kk = 0; kk < KC; ++kk) {
              const int dl = t + (k0 + kk) * T;
              if (!ok[kk] && dl < nfo) kh[kk] = exact_div(dsub(f[kk], FPRV(dl)), dmul(dt, v[k0 + kk]));
            }
          }
        }
#pragma unroll
        for (int kk = 0; kk < KC; ++kk) {
          const int k = k0 + kk, dl = t + k * T;
          if (k < MAXK && dl < nfo) {
            if constexpr (kAd) {
              const double khc = (kh[kk] > 0.0 || isnan(kh[kk])) ? kh[kk] : 0.0;
              g_smem[o.pos + dl] = dmul(dmul(u[k], khc), u[k]);
              g_smem[o.cf + dl] = dmul(dmul(u[k], m[kk]), u[k]);
            }
            if (energy) {  // f . v_half, f_prev . v_half, (m v_half) . v_half (:538-544)
              const double vh = v[k];
              es[0] = dadd(es[0], dmul(f[kk], vh));
              es[1] = dadd(es[1], dmul(FPRV(dl), vh));
              es[2] = dadd(es[2], dmul(dmul(m[kk], vh), vh));
            }
            SET_FPRV(dl, f[kk]);
          }
        }
      }
    };
    if (adaptive) {
      a_phase(std::true_type{});
    } else {
      a_phase(std::false_type{});
    }
    if (energy) {  // warp partials of the ledger dots -> sc.red
#pragma unroll
      for (int e = 0; e < 3; ++e) {
        double x = es[e];
        for (int sh = 16; sh > 0; sh >>= 1) x = dadd(x, __shfl_down_sync(0xffffffffu, x, sh));
        if (lane == 0) sc.red[(t >> 5) * 9 + e] = x;
      }
    }
    __syncthreads();
    mark(sc, prof, PH_A);

    // C: ordered chain sums of one leaf chain + fold + tails -> every rank's
    // slots; the singular flag travels with them.  Round 0 covers leaves
    // 0 .. T/8 - 1 with the chain role cached in registers; ranks with more
    // leaves than T/8 (a 512-thread CTA on a 16-rank 32^3 network) run
    // further rounds, warp w taking leaves 4w + k T/8 .. (quads stay aligned:
    // T/8 is a multiple of 4).
    auto chain_round = [&](int lloc, bool has, int ls, int qn, int ntl) {
      double r0 = 0.0, r1 = 0.0, r2 = 0.0;
      double t0 = 0.0, t1 = 0.0, t2 = 0.0;
      if (has) {
        int dl = ls + j;
        if (qn > 0) {
          r0 = g_smem[o.pos + dl];
          r1 = g_smem[o.cf + dl];
          const double f0 = g_smem[o.fcur + dl];
          r2 = dmul(f0, f0);  // f f (microsolver.py:494), squared where it is summed
#pragma unroll 4
          for (int k = 1; k < qn; ++k) {
            dl += 8;
            r0 = dadd(r0, g_smem[o.pos + dl]);
            r1 = dadd(r1, g_smem[o.cf + dl]);
            const double fk = g_smem[o.fcur + dl];
            r2 = dadd(r2, dmul(fk, fk));
          }
        }
        if (j < ntl) {
          const int dtl = ls + 8 * qn + j;
          t0 = g_smem[o.pos + dtl];
          t1 = g_smem[o.cf + dtl];
          const double ft = g_smem[o.fcur + dtl];
          t2 = dmul(ft, ft);
        }
        if (!adaptive) r0 = r1 = t0 = t1 = 0.0;
      }
#pragma unroll
      for (int sh = 1; sh < 8; sh <<= 1) {
        r0 = dadd(r0, __shfl_xor_sync(0xffffffffu, r0, sh));
        r1 = dadd(r1, __shfl_xor_sync(0xffffffffu, r1, sh));
        r2 = dadd(r2, __shfl_xor_sync(0xffffffffu, r2, sh));
      }
      const int base = lane & ~7;
      const int my_nt = has ? ntl : 0;
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
      if (quad_mode) {  // lanes 0, 8, 16, 24 hold leaves 4w .. 4w+3: ((l0 + l1) + (l2 + l3))
        const double p0 = __shfl_down_sync(0xffffffffu, r0, 8);
        const double p1 = __shfl_down_sync(0xffffffffu, r1, 8);
        const double p2 = __shfl_down_sync(0xffffffffu, r2, 8);
        if ((lane & 15) == 0) {
          r0 = dadd(r0, p0);
          r1 = dadd(r1, p1);
          r2 = dadd(r2, p2);
        }
        const double q0 = __shfl_down_sync(0xffffffffu, r0, 16);
        const double q1 = __shfl_down_sync(0xffffffffu, r1, 16);
        const double q2 = __shfl_down_sync(0xffffffffu, r2, 16);
        if (lane == 0) {
          const int sl = o.lslot + 3 * (lloc >> 2);  // local slot = the quad of the warp's leaves
          g_smem[sl] = dadd(r0, q0);
          g_smem[sl + 1] = dadd(r1, q1);
          g_smem[sl + 2] = dadd(r2, q2);
        }
      } else if (has && j == 0) {
        const int sl = o.lslot + 3 * lloc;  // local leaf lloc
        g_smem[sl] = r0;
        g_smem[sl + 1] = r1;
        g_smem[sl + 2] = r2;
      }
    };
    for (int l0 = (t & ~31) >> 3; l0 < R.n_leaves; l0 += T >> 3) {  // warps holding a chain; rare extra rounds
      const int ll = l0 + (lane >> 3);
      const bool has = ll < R.n_leaves;
      int ls = 0, qn = 0, ntl = 0;
      if (has) {
        const int2 li = leaf_tab[ll];
        ls = li.x;
        qn = li.y >= 8 ? (li.y >> 3) : 0;
        ntl = li.y - 8 * qn;
      }
      chain_round(ll, has, ls, qn, ntl);
    }
    __syncthreads();
    mark(sc, prof, PH_C);

    // T (warp 0): local subtrees of this rank's leaves, their roots to every
    // rank (with this rank's singular flag), the top tree over all ranks'
    // exports, then the scalar bookkeeping.  Meanwhile the other warps
    // compute U's c-independent part, fm = (-f)/m (warp 0 does after T).
#ifndef FRB_NO_SHADOW
    // the shadow work starts once warp 0 has run its local program and sent
    // the exports (named barrier 1): run concurrently, its shared-memory
    // traffic tripled the program's latency (2.7k against 0.55k cycles
    // alone, 16-rank 32^3)
    if (T > 32 && t >= 32) {
      asm volatile("bar.sync 1, %0;" : : "r"(T) : "memory");
      accel(32, T - 32);
    }
#endif
    if (t < 32) {
      const volatile Scalars& vs = sc;
      const int* const gi = reinterpret_cast<const int*>(g_smem);
      const int* const lprog = gi + vs.tp_lprog;
      const int* const tprog = gi + vs.tp_tprog;
      const int* const exps = gi + vs.tp_exps;
      const int n_exp = vs.tp_n_exp, root_top = vs.tp_root, o_lslot = vs.tp_lslot, TSv = vs.tp_TS;
      const int ob = static_cast<int>(mb.ph_s);  // exchange buffer of this iteration's parity
      const int o_ts = vs.tp_tslot + ob * 3 * TSv, o_fl = vs.tp_flag + ob * 64;
      run_prog(lprog, o_lslot, lane);
      mark(sc, prof, PH_TLP);
      // every (export, rank) pair on its own lane: the own copy for qr ==
      // rank, three st.async into the peer's top slots otherwise
      // kGM: each export once into the virtual cluster's top-slot image (the
      // own copy too: every rank reads the whole image back)
      double* const gx_ex = kGM ? gx.ex + static_cast<int64_t>(mb.ph_s) * gx.ex_stride : nullptr;
#pragma unroll 1
      for (int x = lane; x < n_exp * (kGM ? 1 : C); x += 32) {
        if constexpr (kGM) {
          const int ls = o_lslot + 3 * exps[2 * x], ts = 3 * exps[2 * x + 1];
          gx_ex[ts] = g_smem[ls];
          gx_ex[ts + 1] = g_smem[ls + 1];
          gx_ex[ts + 2] = g_smem[ls + 2];
          continue;
        }
        const int e = x / C, qr = x - e * C;
        const int ls = o_lslot + 3 * exps[2 * e], ts = 3 * exps[2 * e + 1];
        const double v0 = g_smem[ls], v1 = g_smem[ls + 1], v2 = g_smem[ls + 2];
        if (qr == rank) {
          g_smem[o_ts + ts] = v0;
          g_smem[o_ts + ts + 1] = v1;
          g_smem[o_ts + ts + 2] = v2;
        } else {
          const uint32_t ad = sc.peer_smem[qr] + 8u * (o_ts + ts);
          st_async(ad, v0, sc.peer_bar_s[qr]);
          st_async(ad + 8, v1, sc.peer_bar_s[qr]);
          st_async(ad + 16, v2, sc.peer_bar_s[qr]);
        }
      }
      mark(sc, prof, PH_TL);
      if (energy && lane == 0) {  // this rank's ledger dots: own slot, and rank 0's
        double e3[3] = {0.0, 0.0, 0.0};
        for (int wp = 0; wp < (T + 31) / 32; ++wp)
          for (int e = 0; e < 3; ++e) e3[e] = dadd(e3[e], sc.red[wp * 9 + e]);
        for (int e = 0; e < 3; ++e) g_smem[o_fl + 16 + 3 * rank + e] = e3[e];
        if (rank != 0)
          for (int e = 0; e < 3; ++e)
            st_async(sc.peer_smem[0] + 8u * (o_fl + 16 + 3 * rank + e), e3[e], sc.peer_bar_s[0]);
      }
      if (kGM) {  // flag, then publish this rank's exports with a release add
        if (lane == 0) gx_ex[3 * TSv + rank] = sc.singular ? 1.0 : 0.0;
        __threadfence();  // every lane's export stores
        __syncwarp();
        if (lane == 0) atomicAdd(gx.cnt + 32 * 16, 1);
      } else if (C > 1) {
        if (lane < C && lane != rank)  // this rank's singular flag, lane q -> rank q
          st_async(sc.peer_smem[lane] + 8u * (o_fl + rank), sc.singular ? 1.0 : 0.0, sc.peer_bar_s[lane]);
      }
#ifndef FRB_NO_SHADOW
      if (T > 32) asm volatile("bar.arrive 1, %0;" : : "r"(T) : "memory");  // exports out: shadow work may start
#endif
      if constexpr (kGM) {  // every rank's exports: wait for the count, copy the image back
        if (lane == 0) {
          sc.gx_s += C;
          gm_spin(gx.cnt + 32 * 16, sc.gx_s);
          __threadfence();
        }
        __syncwarp();
        const int n_top = 3 * R.tree[8];  // the exported slots of the top array
        for (int k0 = lane; k0 < n_top; k0 += 8 * 32) {  // 8 L2 loads in flight per lane
          double tmp[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) tmp[q] = k0 + 32 * q < n_top ? __ldcg(gx_ex + k0 + 32 * q) : 0.0;
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (k0 + 32 * q < n_top) g_smem[o_ts + k0 + 32 * q] = tmp[q];
        }
        if (lane < C) g_smem[o_fl + lane] = __ldcg(gx_ex + 3 * TSv + lane);
        __syncwarp();
        mark(sc, prof, PH_TW);
      } else if (C > 1) {
        mbar_wait(mb.s, mb.ph_s);  // every peer's exports and flag
        if (lane == 0) mbar_expect(mb.s, leaf_bytes);  // next exchange phase
        mark(sc, prof, PH_TW);
      }
      __syncwarp();
      // the peers' singular flags, one per lane (a loop over the ranks cost
      // 2.3k cycles per iteration on 16 ranks: serial shared-memory loads)
      const bool peer_bad = lane < C && lane != rank && g_smem[o_fl + lane] != 0.0;
      const bool singular = (sc.singular != 0) | __any_sync(0xffffffffu, peer_bad);
      if (!singular) run_prog(tprog, o_ts, lane);
      double s_sq = 0.0, s_m = 0.0, s_f = 0.0;  // the three pairwise sums
      if (root_top >= 0) {
        s_sq = g_smem[o_ts + 3 * root_top];
        s_m = g_smem[o_ts + 3 * root_top + 1];
        s_f = g_smem[o_ts + 3 * root_top + 2];
      }
      // lanes 0 and 1 run the same instructions (no divergence): lane 0
      // lam = s_sq / s_m and c = 2 sqrt(lam); lane 1 s_f / 1 = s_f and the
      // residual sqrt(s_f), threshold and convergence test
      if (lane < 2) {
        if (singular) {
          if (lane == 0) sc.singular = 1;
        } else {
          // np.sum adds the pairwise result to the identity 0.0
          s_sq = dadd(0.0, s_sq);
          s_m = dadd(0.0, s_m);
          s_f = dadd(0.0, s_f);
          const double qv = ddiv(lane == 0 ? s_sq : s_f, lane == 0 ? s_m : 1.0);
          const double rv = dsqrt(qv);
          if (lane == 0) {
            double c = cfg.damping_c;
            if (adaptive) c = (s_m > 0.0 && qv > 0.0) ? dmul(2.0, rv) : 0.0;
            sc.c = c;
            if (energy && rank == 0) {  // _accumulate_energy (microsolver.py:533-546), ranks in order
              double d[3] = {0.0, 0.0, 0.0};
              for (int qr = 0; qr < C; ++qr)
                for (int e = 0; e < 3; ++e) d[e] = dadd(d[e], g_smem[o_fl + 16 + 3 * qr + e]);
              w[1] = dadd(w[1], dmul(0.5, dmul(dt, dadd(d[0], d[1]))));
              if (wfix != 0.0 || (ramp && it < ramp_n)) {
                w[1] = dadd(w[1], wfix);
                w[3] = dadd(w[3], wfix);
              }
              w[2] = dadd(w[2], dmul(dmul(c, dt), d[2]));
            }
          } else {
            const double res = rv;
            double thr = sc.threshold;
            if (it == full_bc_iter) {
              sc.r_ref = res;
              const double th = dmul(cfg.tol_rel, res);
              thr = th > cfg.tol_abs ? th : cfg.tol_abs;  // max(tol_abs, .)
              sc.threshold = thr;
            }
            int done = 0, conv = 0;
            if (it >= full_bc_iter && res <= thr) {
              done = 1;
              conv = 1;
            } else if (it + 1 >= cfg.max_iters) {
              done = 1;
            }
            sc.residual = res;
            sc.done = done;
            sc.converged = conv;
          }
        }
      }
#ifndef FRB_NO_SHADOW
      if (T <= 32) accel(0, T);
#endif
    }
    mb.ph_s ^= 1u;
    __syncthreads();
#ifdef FRB_NO_SHADOW  // experiment: (-f)/m after the tree phase, by every warp
    accel(0, T);
    __syncthreads();
#endif
    mark(sc, prof, PH_TT);
    if (sc.singular) {
      if (!kGM && C > 1) drain(mb, R.halo_bytes, leaf_bytes);
      // positions of every node to global memory, then the argmin over all
      // elements (each rank redundantly; rank 0 reports)
#pragma unroll
      for (int k = 0; k < MAXK; ++k)
        if (t + k * T < nfo) n.posg[dof0 + t + k * T] = dadd(xr[k], u[k]);
      set_fixed_positions(n, rank, alpha, ramp);
      gsync<kGM>(C, sc, gx);
      const int badi = singular_argmin(n, PosGlobalAll{n.posg}, sc);
      if (rank == 0 && t == 0) write_singular(b, p, badi, it);
      return;
    }

    // U: accelerations and second half-kick (:501-507); then the next
    // iteration's first half-kick and drift (:443-453) unless finished
    const double c = sc.c;
    const bool done = sc.done != 0;
#pragma unroll
    for (int k = 0; k < MAXK; ++k) {
      const int dl = t + k * T;
      if (dl < nfo) {
        const double a = dsub(g_smem[o.fcur + dl], dmul(c, v[k]));
        v[k] = dadd(v[k], dmul(hdt, a));
        if (!done) {
          v[k] = dadd(v[k], dmul(hdt, a));
          u[k] = dadd(u[k], dmul(dt, v[k]));
          put_local(dl, dadd(xr[k], u[k]));
        }
      }
    }
    if (!done && ramp && alpha < 1.0) {
      alpha = ramp_alpha(it + 2, ramp_n);
      set_local_fixed(n, R, &g_smem[o.pos], alpha, ramp);
      if (energy) set_fixed_positions(n, rank, alpha, ramp);
    }
    if (done) break;
    if (C > 1) fence_proxy_async();  // the positions feed the next halo copies
    __syncthreads();
    mark(sc, prof, PH_U);
  }
  if (!kGM && C > 1) drain(mb, R.halo_bytes, leaf_bytes);
  mark(sc, prof, PH_U);

  // ---- epilogue: outputs in solver order + stress (:549-564, :285-299) ----
  double* uo = b.u + 3 * n.node_base;
  double* fo = b.f + 3 * n.node_base;
#pragma unroll
  for (int k = 0; k < MAXK; ++k) {
    const int dl = t + k * T;
    if (dl < nfo) {
      const int d = dof0 + dl;
      uo[d] = u[k];
      if (!kFG) fo[d] = g_smem[o.fprv + dl];
      n.posg[d] = dadd(xr[k], u[k]);  // x = X + u, all free nodes
    }
  }
  set_fixed_positions(n, rank, alpha, ramp);
  if (energy) {  // w_kin = 0.5 (m v) . v (:546): rank partials into rank 0's slots
    double ek = 0.0;
#pragma unroll
    for (int k = 0; k < MAXK; ++k)
      if (t + k * T < nfo) ek = dadd(ek, dmul(dmul(__ldg(nmass + (t + k * T) / 3), v[k]), v[k]));
    for (int sh = 16; sh > 0; sh >>= 1) ek = dadd(ek, __shfl_down_sync(0xffffffffu, ek, sh));
    if (lane == 0) sc.red[(t >> 5) * 9] = ek;
    __syncthreads();
    if (t == 0) {
      double e = 0.0;
      for (int wp = 0; wp < (T + 31) / 32; ++wp) e = dadd(e, sc.red[wp * 9]);
      double* dst = &g_smem[o.flag + 128 + rank];  // fin[rank]
      *(C > 1 ? peer(dst, 0) : dst) = e;
    }
  }
  gsync<kGM>(C, sc, gx);
  if (rank == 0 && energy && t == 0) {
    double e = 0.0;
    for (int qr = 0; qr < C; ++qr) e = dadd(e, g_smem[o.flag + 128 + qr]);
    w[0] = dmul(0.5, e);
  }
  if (rank == 0) fixed_forces_and_stress(b, p, n, sc, it, alpha, ramp, full_bc_iter, energy, w);
  __syncthreads();
  mark(sc, prof, PH_EPI);
}

template <int MAXK, int MAXT, bool kFG, bool kEnergy, bool kGM = false>
__global__ void __launch_bounds__(MAXT, 1)
    frb_relax_kernel(const __grid_constant__ frb_batch b, const __grid_constant__ frb_config cfg, int first,
                     int count, int32_t* queue, const __grid_constant__ frb_group grp) {
  __shared__ Scalars sc;
  __shared__ Net net;
  __shared__ Rank rk;
  __shared__ uint64_t bars[3];
  // hardware cluster: its size and rank; virtual cluster (kGM): C
  // consecutive CTAs of a non-cluster launch and their slice of the scratch
  const int C = kGM ? grp.cluster : static_cast<int>(cg::this_cluster().num_blocks());
  const int rank = kGM ? static_cast<int>(blockIdx.x) % C : (C > 1 ? static_cast<int>(cg::this_cluster().block_rank()) : 0);
  Gx gx{nullptr, nullptr, nullptr, 0, 0};
  if constexpr (kGM) {
    const int vg = static_cast<int>(blockIdx.x) / C;
    char* base = reinterpret_cast<char*>(b.xchg) + grp.xchg_off;
    gx.ex_stride = grp.gm_ex_stride;
    gx.mir_stride = grp.gm_mir_stride;
    gx.cnt = reinterpret_cast<int*>(base + 4096 * static_cast<int64_t>(vg));
    double* ex0 = reinterpret_cast<double*>(base + 4096 * static_cast<int64_t>(grp.gm_cap));
    gx.ex = ex0 + static_cast<int64_t>(vg) * 2 * gx.ex_stride;
    gx.mir = ex0 + static_cast<int64_t>(grp.gm_cap) * 2 * gx.ex_stride +
             static_cast<int64_t>(vg) * C * gx.mir_stride;
  }
  if (threadIdx.x == 0) {
    for (int k = 0; k < kPhases; ++k) sc.clk[k] = 0;
    sc.t_last = clock64();
    sc.gx_h = sc.gx_s = sc.gx_b = 0;
    if (!kGM && C > 1) {
      mbar_init(&bars[0], 1);
      mbar_init(&bars[1], 1);
      mbar_init(&bars[2], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      for (int q = 0; q < C; ++q) {
        sc.peer_smem[q] = mapa(smem_u32(g_smem), q);
        sc.peer_bar_h[q] = mapa(smem_u32(&bars[0]), q);
        sc.peer_bar_s[q] = mapa(smem_u32(&bars[1]), q);
        sc.peer_bar_a[q] = mapa(smem_u32(&bars[2]), q);
      }
    }
  }
  Mbar mb{&bars[0], &bars[1], &bars[2], 0u, 0u, 0u};
  gsync<kGM>(C, sc, gx);  // barriers initialised cluster-wide before any remote use
  for (;;) {
    if (rank == 0 && threadIdx.x == 0) {
      const int idx = atomicAdd(queue, 1);
      if constexpr (kGM) {
        gx.cnt[32 * 18] = idx;  // published by the barrier's release
      } else {
        for (int q = 0; q < C; ++q) *(C > 1 ? peer(&sc.problem, q) : &sc.problem) = idx;
      }
    }
    gsync<kGM>(C, sc, gx);
    if constexpr (kGM) {
      if (threadIdx.x == 0) sc.problem = ld_acquire(gx.cnt + 32 * 18);
      __syncthreads();
    }
    const int idx = sc.problem;
    if (idx >= count) break;
    const int p = b.order[first + idx];
    if (threadIdx.x == 0) {
      load_views(net, rk, b, p, rank);
      sc.singular = 0;
      sc.done = 0;
      sc.converged = 0;
      sc.threshold = __longlong_as_double(0x7ff0000000000000ULL);  // +inf until set
    }
    __syncthreads();
    solve_problem<MAXK, kFG, kEnergy, kEnergy ? 0 : MAXT, kGM>(b, cfg, p, rank, sc, mb, net, rk, gx);
    gsync<kGM>(C, sc, gx);  // no rank reuses its SMEM (or the problem slot) before every peer is done with it
  }
  if (b.phase_cycles && threadIdx.x == 0) {
    for (int k = 0; k < kPhases; ++k) b.phase_cycles[kPhases * blockIdx.x + k] = sc.clk[k];
  }
}


int set_err(int code, const char* msg) {
  snprintf(frb_tu::g_err, sizeof frb_tu::g_err, "%s", msg);
  return code;
}

int cuda_check(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return FRB_OK;
  snprintf(frb_tu::g_err, sizeof frb_tu::g_err, "%s: %s", where, cudaGetErrorString(e));
  return FRB_E_CUDA;
}

// most register-held DOFs per thread a CTA size instantiates (24 only for
// the global-f_prev kernels of 256 threads, 16 otherwise up to 512 threads)
int dofs_cap(int threads, bool fg) { return threads > 768 ? 8 : threads > 512 ? 12 : (threads > 256 || !fg) ? 16 : 24; }

// Kernel attributes every launch of an instantiation needs.
template <class K>
int prepare_kernel(K kern, int smem_bytes, int C, bool cluster) {
  int rc = cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes),
                      "cudaFuncSetAttribute(smem)");
  if (rc) return rc;
  // smallest SMEM carveout that holds the rank: the rest of the 256 KB
  // array is L1, which holds the loop's read-only tables
  cudaFuncAttributes fa;
  rc = cuda_check(cudaFuncGetAttributes(&fa, kern), "cudaFuncGetAttributes");
  if (rc) return rc;
  const int need = smem_bytes + static_cast<int>(fa.sharedSizeBytes) + 1024;
  const int pct = (100 * need + 228 * 1024 - 1) / (228 * 1024);
  rc = cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, pct < 100 ? pct : 100),
                  "cudaFuncSetAttribute(carveout)");
  if (rc) return rc;
  if (cluster && C > 8)
    rc = cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
                    "cudaFuncSetAttribute(non-portable cluster)");
  return rc;
}

template <int MAXK, int MAXT, bool kFG, bool kEnergy = false>
int launch_group(const frb_batch* batch, const frb_config* cfg, const frb_group& g, int32_t* queue,
                 cudaStream_t s, int threads = 0) {
  auto kern = frb_relax_kernel<MAXK, MAXT, kFG, kEnergy, false>;
  const int C = g.cluster;
  int rc = prepare_kernel(kern, g.smem_bytes, C, true);
  if (rc) return rc;
  cudaLaunchConfig_t lc = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.blockDim = dim3(threads > 0 ? threads : (kEnergy ? g.block_threads : MAXT));
  lc.dynamicSmemBytes = g.smem_bytes;
  lc.stream = s;
  lc.attrs = attr;
  lc.numAttrs = 1;
  int clusters = g.grid_clusters;
  if (clusters <= 0) {
    lc.gridDim = dim3(C);
    rc = cuda_check(cudaOccupancyMaxActiveClusters(&clusters, kern, &lc), "cudaOccupancyMaxActiveClusters");
    if (rc) return rc;
    if (clusters < 1) return set_err(FRB_E_TOO_LARGE, "cluster does not fit on the GPU");
  }
  if (clusters > g.count) clusters = g.count;
  // virtual clusters on the SMs the hardware clusters leave idle (a cluster
  // of 8+ CTAs sits in one GPC: 7 clusters of 16 use 112 of 148 SMs)
  int gm = 0;
  if constexpr (!kEnergy && (MAXT == 512 || MAXT == 768)) {
    if (C >= 8 && batch->xchg && g.gm_cap > 0 && g.grid_clusters <= 0 && !(g.flags & FRB_GF_NO_VIRTUAL) &&
        (!batch->phase_cycles || (g.flags & FRB_GF_VIRTUAL_ONLY))) {  // (phase profiles: hardware clusters)
      int dev = 0, nsm = 0;
      rc = cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
      if (!rc) rc = cuda_check(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev), "sm count");
      if (rc) return rc;
      if (g.flags & FRB_GF_VIRTUAL_ONLY) clusters = 0;  // experiment: virtual clusters only
      gm = (nsm - clusters * C) / C;
      if (gm > g.gm_cap) gm = g.gm_cap;
      if (gm > g.count - clusters) gm = g.count - clusters;
      if (gm < 0) gm = 0;
    }
  }
  lc.gridDim = dim3(clusters * C);
  rc = cuda_check(cudaMemsetAsync(queue, 0, sizeof(int32_t), s), "cudaMemsetAsync");
  if (rc) return rc;
  if (gm > 0) {
    rc = cuda_check(cudaMemsetAsync(reinterpret_cast<char*>(batch->xchg) + g.xchg_off, 0, 4096 * g.gm_cap, s),
                    "cudaMemsetAsync(xchg)");
    if (rc) return rc;
  }
  if constexpr (!kEnergy && (MAXT == 512 || MAXT == 768)) {
    if (gm > 0) {  // forked stream: both kernels pull from the same queue
      auto vkern = frb_relax_kernel<MAXK, MAXT, kFG, kEnergy, true>;
      rc = prepare_kernel(vkern, g.smem_bytes, C, false);
      if (rc) return rc;
      cudaEvent_t ev0, ev1;
      cudaStream_t gs;
      rc = cuda_check(cudaEventCreateWithFlags(&ev0, cudaEventDisableTiming), "cudaEventCreate");
      if (rc) return rc;
      rc = cuda_check(cudaEventCreateWithFlags(&ev1, cudaEventDisableTiming), "cudaEventCreate");
      if (!rc) rc = cuda_check(cudaStreamCreateWithFlags(&gs, cudaStreamNonBlocking), "cudaStreamCreate");
      if (!rc) rc = cuda_check(cudaEventRecord(ev0, s), "cudaEventRecord");
      if (!rc) rc = cuda_check(cudaStreamWaitEvent(gs, ev0, 0), "cudaStreamWaitEvent");
      if (!rc && clusters > 0)
        rc = cuda_check(cudaLaunchKernelEx(&lc, kern, *batch, *cfg, g.first, g.count, queue, g), "cudaLaunchKernelEx");
      cudaLaunchConfig_t vc = lc;
      vc.gridDim = dim3(gm * C);
      vc.stream = gs;
      vc.attrs = nullptr;
      vc.numAttrs = 0;
      if (!rc) frb_tu::g_launches += clusters > 0;
      if (!rc) rc = cuda_check(cudaLaunchKernelEx(&vc, vkern, *batch, *cfg, g.first, g.count, queue, g),
                               "cudaLaunchKernelEx(virtual clusters)");
      if (!rc) ++frb_tu::g_launches;
      if (!rc) rc = cuda_check(cudaEventRecord(ev1, gs), "cudaEventRecord");
      if (!rc) rc = cuda_check(cudaStreamWaitEvent(s, ev1, 0), "cudaStreamWaitEvent");
      cudaEventDestroy(ev0);
      cudaEventDestroy(ev1);
      cudaStreamDestroy(gs);
      if (rc) return rc;
      return cuda_check(cudaGetLastError(), "frb_relax_kernel launch");
    }
  }
  rc = cuda_check(cudaLaunchKernelEx(&lc, kern, *batch, *cfg, g.first, g.count, queue, g), "cudaLaunchKernelEx");
  if (rc) return rc;
  ++frb_tu::g_launches;
  return cuda_check(cudaGetLastError(), "frb_relax_kernel launch");
}

template <int MAXT>
int dispatch_k(const frb_batch* batch, const frb_config* cfg, const frb_group& g, int32_t* queue,
               cudaStream_t s, int k) {
  if (g.fprv_global) {  // large networks: CTAs of 256 / 512 / 768 / 1024 threads
    if constexpr (MAXT == 256) {
      if (k <= 16) return launch_group<16, MAXT, true>(batch, cfg, g, queue, s);
      if (k <= 20) return launch_group<20, MAXT, true>(batch, cfg, g, queue, s);
      if (k <= 24) return launch_group<24, MAXT, true>(batch, cfg, g, queue, s);
    }
    if constexpr (MAXT == 512) {
      if (k <= 8) return launch_group<8, MAXT, true>(batch, cfg, g, queue, s);
      if (k <= 11) return launch_group<11, MAXT, true>(batch, cfg, g, queue, s);  // 32^3 on 16 ranks
      if (k <= 12) return launch_group<12, MAXT, true>(batch, cfg, g, queue, s);
      if (k <= 14) return launch_group<14, MAXT, true>(batch, cfg, g, queue, s);
      if (k <= 16) return launch_group<16, MAXT, true>(batch, cfg, g, queue, s);
    }
    if constexpr (MAXT >= 768) {
      if (k <= 4) return launch_group<4, MAXT, true>(batch, cfg, g, queue, s);
      if (k <= 6) return launch_group<6, MAXT, true>(batch, cfg, g, queue, s);
      if (k <= 7) return launch_group<7, MAXT, true>(batch, cfg, g, queue, s);  // 32^3 on 16 ranks
      if (k <= 8) return launch_group<8, MAXT, true>(batch, cfg, g, queue, s);
      if constexpr (MAXT <= 768) {
        if (k <= 10) return launch_group<10, MAXT, true>(batch, cfg, g, queue, s);
        if (k <= 12) return launch_group<12, MAXT, true>(batch, cfg, g, queue, s);
      }
    }
    return set_err(FRB_E_TOO_LARGE, "too many free DOFs per thread for this CTA size");
  }
  if (k <= 1) return launch_group<1, MAXT, false>(batch, cfg, g, queue, s);
  if (k <= 4) return launch_group<4, MAXT, false>(batch, cfg, g, queue, s);
  if (k <= 6) return launch_group<6, MAXT, false>(batch, cfg, g, queue, s);
  if (k <= 8) return launch_group<8, MAXT, false>(batch, cfg, g, queue, s);
  if constexpr (MAXT <= 768) {
    if (k <= 10) return launch_group<10, MAXT, false>(batch, cfg, g, queue, s);
    if (k <= 12) return launch_group<12, MAXT, false>(batch, cfg, g, queue, s);
  }
  if constexpr (MAXT <= 512) {
    if (k <= 14) return launch_group<14, MAXT, false>(batch, cfg, g, queue, s);
    if (k <= 16) return launch_group<16, MAXT, false>(batch, cfg, g, queue, s);
  }
  return set_err(FRB_E_TOO_LARGE, "too many free DOFs per thread for this CTA size");
}

}  // namespace

// the solver kernels of one CTA-size template, one translation unit each
// (frb_k256.cu ... frb_k1024.cu, frb_kenergy.cu) so they compile in parallel
namespace frb_tu {
int dispatch_256(const frb_batch*, const frb_config*, const frb_group&, int32_t*, cudaStream_t, int k);
int dispatch_512(const frb_batch*, const frb_config*, const frb_group&, int32_t*, cudaStream_t, int k);
int dispatch_768(const frb_batch*, const frb_config*, const frb_group&, int32_t*, cudaStream_t, int k);
int dispatch_1024(const frb_batch*, const frb_config*, const frb_group&, int32_t*, cudaStream_t, int k);
int dispatch_energy(const frb_batch*, const frb_config*, const frb_group&, int32_t*, cudaStream_t, int T, int ke);
}  // namespace frb_tu
