// fused2d.hpp — one-launch D-SKI MVM for 2-D grids with gradients (C1, C2, C4).
#pragma once

#include "pcg_fused.hpp"

#include <vector>

#include "gk_common.hpp"

namespace gk {

// Geometry of a d = 2 D-SKI operator in its internal (cell-sorted) layout.
struct Fused2dGeom {
  int T = 6;                 // stencil taps (6 quintic, 4 cubic)
  int m0 = 0, m1 = 0;        // grid nodes per axis
  int nb0 = 0, nb1 = 0;      // base cells per axis (m - T + 1)
  int n = 0;                 // points
  const int4* base = nullptr;        // [n] (base0, base1, -, -)
  const double2* wd = nullptr;       // [n][2][T] (w, dw) pairs, axis 0 then axis 1
  const double2* rec = nullptr;      // [n][2T+1] (w, dw) pairs then the int4 base (scatter staging records)
  const int* cell_start = nullptr;   // [nb0*nb1 + 1]
  const double* t0 = nullptr;        // axis-0 Toeplitz sequence (carries s²)
  const double* t1 = nullptr;        // axis-1 Toeplitz sequence
  int band0 = 0, band1 = 0;
  double nv2 = 0.0, ng2 = 0.0;
};

// Work decomposition of the four phases for one right-hand-side count,
// computed on the host from the cell occupancy (so every staging buffer is
// sized for the fullest window) and cached per operator.
struct Fused2dPlan {
  bool ok = false;
  int nrhs = 0, RP = 1, BRP = 0, BR = 0, chunks = 0;  // RP right-hand sides per thread
  int s_TC = 0, s_strips = 0, s_L = 0, s_segs = 0, s_pmax = 0, s_csw = 0;
  int g_TC = 0, g_strips = 0, g_L = 0, g_segs = 0, g_pmax = 0, g_nw = 0;
  int t_split = 1;
  int t_wide = 0;  // Toeplitz phases: 16-column items
  int s_mode = 0, g_mode = 0;  // 0 staged rolling, 1 direct-load variants
  int s_nspl = 2;
  int s_nst = 3;                // staged scatter: cell rows in flight              // staged scatter: threads splitting one column's points
  int s_nbuf = 1;              // direct scatter: partial grid buffers (pbuf holds s_nbuf × M × nrhs)
  int tuning_gen = -1;  // g_tuning.gen the plan was built under
  int grid = 0;
  int minb = 2;  // __launch_bounds__ min blocks of the instantiation used
  size_t smem = 0;
  DevBuf<unsigned long long> bar;  // grid-barrier counter (monotonic, this plan only)
  DevBuf<unsigned long long> prof; // [grid][8] phase stamps (tuning "fused_prof")
};

void fused2d_plan(const Fused2dGeom& g, const std::vector<int>& cell_start_h, int nrhs, int device,
                  Fused2dPlan& p);
// out = B K_UU B^T v (+ noise): u, h, y1, w are M×nrhs grid scratch buffers
// (h holds the scatter's segment-boundary halo rows).
// skip: bitmask of phases to leave out (1 scatter, 2 mode 1, 4 mode 0, 8
// gather), OR-ed with the debug knob: the split launches of the grid-slab MVM
// run the scatter alone (14) and the rest alone (1) around an all-reduce of
// [u; h].
void fused2d_mvm(const Fused2dGeom& g, Fused2dPlan& p, const double* v, double* out, double* u,
                 double* h, double* y1, double* w, double* pbuf, bool noise, cudaStream_t s, int skip = 0);

// Persistent PCG (PCG with this operator's one-launch MVM and the rows-resident
// vector step in one cooperative kernel, up to `iters` iterations). False when
// the plans are incompatible (then the caller uses the per-iteration path).
bool fused2d_pcg_persist(const Fused2dGeom& g, Fused2dPlan& p, PcgVecPlan& vp, PcgVecArgs va, const double* P,
                         double* AP, double* u, double* h, double* y1, double* w, double* pbuf, int iters,
                         cudaStream_t s);

}  // namespace gk
