// pcg_fused.hpp — one-launch PCG vector step (everything but the MVM).
#pragma once

#include "gk_common.hpp"

namespace gk {

// Per-column PCG state on the device (linalg.cpp:85-131 run for nrhs columns).
struct PcgState {
  double* bnorm;
  double* rz;
  double* alpha;
  double* beta;
  double* hist;  // [(maxit+1)][nrhs]
  int* active;
  int* upd;
  int* its;
  int* conv;
  int* nactive;  // single int
  int maxit;
  double tol;
  int nrhs;
};

struct PcgVecArgs {
  PcgState st;
  double* X;
  double* R;
  double* P;
  const double* AP;
  double* Z;
  const double* q1;    // [N][k] preconditioner basis (null: no preconditioner, z = r)
  const double* dinv;  // [N] D^{-1/2}
  int k;
  i64 N;
  int nrhs;
  int rch;        // filled by pcg_vec_launch: staged row chunk
  double* part;
  double* tpart;
  double* T;
  unsigned long long* bar;
  double* red_out;           // [3][nrhs] published column reductions
  unsigned long long* rctr;  // reduce-barrier counters (arrivals, releases)
  unsigned long long* prof;  // debug: [grid][8] phase stamps or null
};

struct PcgVecPlan {
  bool v2 = false;  // rows-resident variant (k_pcg_vec2)
  bool r1 = false;  // single-RHS streamed-GEMV variant (k_pcg_vec_r1)
  int grid = 0;
  int rch = 1;
  size_t smem = 0;
  DevBuf<double> part, tpart, T;
  DevBuf<unsigned long long> bar;
  DevBuf<double> red_out;
  DevBuf<unsigned long long> rctr;
  DevBuf<unsigned long long> prof;
  int launches = 0;
};

bool pcg_vec_supported(int nrhs, int k);
void pcg_vec_prepare(PcgVecPlan& p, i64 N, int nrhs, int k, int device);
void pcg_vec_launch(PcgVecPlan& p, PcgVecArgs a, cudaStream_t s);
void pcg_vec_dump(PcgVecPlan& p);  // debug (GK_PCG_PROF): phase times of the last launch

}  // namespace gk
