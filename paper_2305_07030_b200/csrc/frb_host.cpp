// frb_host.cpp -- native host setup of one network (the per-network part of
// the reference's build_problem, pkg/src/fibrelax/microsolver.py:302-335),
// written straight into the packed batch arrays.
//
// Called once per network from a pool of host threads (ctypes releases the
// GIL), so packing a batch of thousands of networks scales over the host
// cores.  Every floating-point value is bit-identical to the reference's
// numpy evaluation (compiled with -ffp-contract=off: no FMA contraction;
// sqrt and / are IEEE correctly rounded in C):
//   * reference length   L = sqrt((dx*dx + dz*dz) + dy*dy)   (network.py:171-172,
//                        numpy's 3-column einsum order)
//   * lumped mass        half = ((rho*A)*L)/2 added with np.add.at semantics:
//                        role a in element order, then role b (microsolver.py:175-178)
//   * time step base     min_e L_e * sqrt(rho_e / E_e)       (microsolver.py:185-193)
//   * RVE volume         bounding-box product span0*span1*span2, 1 if <= 0
//                        (network.py:154-165)

#include <math.h>
#include <stdint.h>
#include <string.h>

#include <atomic>
#include <thread>
#include <vector>

#include "frb200.h"

extern "C" int frb_setup_problem(int32_t n_nodes, int32_t n_elems, const double* coords, const int64_t* elements,
                                 const double* materials, int32_t n_materials, const int64_t* node_order,
                                 const int64_t* act_elem, int64_t n_act, double* X_out, double* mass_out,
                                 double* L_out, double* EA_out, double* act_L_out, double* act_EA_out,
                                 double* scalars_out, double* mass_scratch) {
  if (n_nodes < 0 || n_elems < 0 || n_act < 0 || !scalars_out) return FRB_E_INVALID;
  if (n_nodes > 0 && (!coords || !node_order)) return FRB_E_INVALID;
  if (n_elems > 0 && (!elements || !materials || !L_out || !EA_out || !mass_scratch)) return FRB_E_INVALID;
  // reference lengths, E*A, dt base (original element order)
  bool any_nan = false;
  double dt_min = INFINITY;
  for (int32_t e = 0; e < n_elems; ++e) {
    const int64_t a = elements[3 * e], b = elements[3 * e + 1], m = elements[3 * e + 2];
    if (a < 0 || a >= n_nodes || b < 0 || b >= n_nodes || m < 0 || m >= n_materials) return FRB_E_INVALID;
    const double dx = coords[3 * b] - coords[3 * a];
    const double dy = coords[3 * b + 1] - coords[3 * a + 1];
    const double dz = coords[3 * b + 2] - coords[3 * a + 2];
    const double L = sqrt((dx * dx + dz * dz) + dy * dy);
    const double E = materials[3 * m], A = materials[3 * m + 1], rho = materials[3 * m + 2];
    L_out[e] = L;
    EA_out[e] = E * A;
    const double t = L * sqrt(rho / E);
    if (isnan(t)) any_nan = true;  // np.min propagates NaN
    else if (t < dt_min) dt_min = t;
  }
  const double dt_base = any_nan ? NAN : dt_min;
  // lumped node mass, original node order: role a in element order, then role b
  double* nm = mass_scratch;
  if (n_elems > 0 || n_nodes > 0) {
    if (n_nodes > 0 && !nm) return FRB_E_INVALID;
    for (int32_t i = 0; i < n_nodes; ++i) nm[i] = 0.0;
    for (int role = 0; role < 2; ++role)
      for (int32_t e = 0; e < n_elems; ++e) {
        const int64_t m = elements[3 * e + 2];
        const double half = ((materials[3 * m + 2] * materials[3 * m + 1]) * L_out[e]) / 2.0;
        nm[elements[3 * e + role]] += half;
      }
  }
  int64_t zero_mass = -1;
  for (int32_t i = 0; i < n_nodes; ++i)
    if (nm[i] <= 0.0) {  // np.any(node_mass <= 0) -> np.argmin: the first minimum
      if (zero_mass < 0 || nm[i] < nm[zero_mass]) zero_mass = i;
    }
  // solver-order coordinates and masses
  for (int32_t s = 0; s < n_nodes; ++s) {
    const int64_t o = node_order[s];
    if (o < 0 || o >= n_nodes) return FRB_E_INVALID;
    if (X_out) memcpy(X_out + 3 * s, coords + 3 * o, 3 * sizeof(double));
    if (mass_out) mass_out[s] = nm[o];
  }
  // per-rank active-element values (partition.py RankTables.act_elem)
  for (int64_t k = 0; k < n_act; ++k) {
    const int64_t e = act_elem[k];
    if (e < 0 || e >= n_elems) return FRB_E_INVALID;
    if (act_L_out) act_L_out[k] = L_out[e];
    if (act_EA_out) act_EA_out[k] = EA_out[e];
  }
  // bounding-box volume
  double span[3] = {0.0, 0.0, 0.0};
  if (n_nodes > 0) {
    for (int c = 0; c < 3; ++c) {
      double lo = coords[c], hi = coords[c];
      for (int32_t i = 1; i < n_nodes; ++i) {
        const double x = coords[3 * i + c];
        if (x < lo) lo = x;
        if (x > hi) hi = x;
      }
      span[c] = hi - lo;
    }
  }
  const double box = (span[0] * span[1]) * span[2];
  scalars_out[0] = n_elems > 0 ? dt_base : NAN;
  scalars_out[1] = box > 0.0 ? box : 1.0;
  scalars_out[2] = static_cast<double>(zero_mass);
  return FRB_OK;
}

static_assert(sizeof(frb_setup_item) == 144, "frb_setup_item layout (SETUP_ITEM_DTYPE in _native.py)");

// Every network of a batch on n_threads host threads (work-stealing over the
// items); per-item status in items[i].rc.  Returns FRB_E_INVALID if any item
// was malformed, else FRB_OK.
extern "C" int frb_setup_batch(frb_setup_item* items, int32_t n_items, int32_t n_threads) {
  if (n_items < 0 || (n_items > 0 && !items)) return FRB_E_INVALID;
  std::atomic<int32_t> next{0};
  auto work = [&]() {
    for (int32_t i = next.fetch_add(1); i < n_items; i = next.fetch_add(1)) {
      frb_setup_item& it = items[i];
      it.rc = frb_setup_problem(it.n_nodes, it.n_elems, it.coords, it.elements, it.materials, it.n_materials,
                                it.node_order, it.act_elem, it.n_act, it.X_out, it.mass_out, it.L_out,
                                it.EA_out, it.act_L_out, it.act_EA_out, it.scalars, it.mass_scratch);
    }
  };
  int32_t nt = n_threads < 1 ? 1 : n_threads;
  if (nt > n_items) nt = n_items;
  std::vector<std::thread> pool;
  for (int32_t k = 1; k < nt; ++k) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
  for (int32_t i = 0; i < n_items; ++i)
    if (items[i].rc != FRB_OK) return FRB_E_INVALID;
  return FRB_OK;
}
