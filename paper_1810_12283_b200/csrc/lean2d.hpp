// lean2d.hpp — lean one-launch D-SKI MVM for 2-D grids with gradients (C1, C2:
// grids up to 128 nodes per axis, up to 64 right-hand sides).
#pragma once

#include "fused2d.hpp"

namespace gk {

struct Lean2dPlan {
  bool ok = false;
  int nrhs = 0, RP = 1, BRP = 0, L = 5, nseg = 0, grid = 0;
  int kp1 = 0, mt1 = 0, nt1 = 0, ms1 = 0, dlo1 = 0, nd1 = 0;
  int kp0 = 0, mt0 = 0, nt0 = 0, ms0 = 0, dlo0 = 0, nd0 = 0;
  size_t smem = 0;
  int tuning_gen = -1;
  DevBuf<unsigned long long> bar;   // grid-barrier counter (this plan only)
  DevBuf<unsigned long long> prof;  // [grid][8] phase stamps (tuning "fused_prof")
};

void lean2d_plan(const Fused2dGeom& g, int nrhs, int device, Lean2dPlan& p);
// out = B K_UU Bᵀ v (+ noise); uu: 2×M×nrhs (segment-parity scatter slots),
// y1, w: M×nrhs grid scratch.
void lean2d_mvm(const Fused2dGeom& g, Lean2dPlan& p, const double* v, double* out, double* uu,
                double* y1, double* w, bool noise, cudaStream_t s);

}  // namespace gk
