// Controller logic of the SuperMann / CP loop (proj/src/solver.cpp:189-350),
// one thread: the graph loop's controller kernels (loop.cu, G = true: also set
// the graph's conditional handles) and the CTA-resident small-tree loop
// (small.cu, G = false: the branch decisions are read from the state).
#pragma once

#include <cuda_runtime.h>

#include "../../include/spock_b200.h"
#include "aa.cuh"
#include "loop.hpp"

namespace spock {

__device__ __forceinline__ void set_cond(unsigned long long h, unsigned int v) {
  cudaGraphSetConditional(static_cast<cudaGraphConditionalHandle>(h), v);
}

__device__ __forceinline__ int ring(int i, int n) { return ((i % n) + n) % n; }

// top of iteration k (solver.cpp:233-290): M-norm, xi thresholds, termination,
// Anderson direction coefficients, K0 test; selects the branch body
template <bool G>
__device__ void ctl_begin(const LoopArgs& A) {
  LoopState& S = *A.st;
  const LoopParams& P = A.P;
  const double* red = A.red;
  if (P.supermann) {
    S.h += 1;
    S.aa_cols = min(S.aa_cols + 1, P.m);
  }
  int reason = -1;
  if (!S.have_omega) {
    const double rad = red[0] - 2.0 * P.alpha * red[1] + red[2];
    if (rad < -1e-12 * fmax(1.0, red[0] + red[2])) reason = -2;  // solver.cpp:171-172
    S.omega = sqrt(fmax(0.0, rad));
    if (S.k == 0) S.zeta = S.omega_safe = S.omega;
  }
  const double n1 = red[4], n2 = red[5];
  if (S.k == 0) {
    S.th1 = fmax(P.eps_abs, P.eps_rel * n1);
    S.th2 = fmax(P.eps_abs, P.eps_rel * n2);
  }
  S.xi1 = n1;
  S.xi2 = n2;
  ++S.n_Lt;
  if (reason < 0) {
    if (!isfinite(n1) || !isfinite(n2) || !isfinite(S.omega))
      reason = SPOCK_STALLED;
    else if (n1 <= S.th1 && n2 <= S.th2)
      reason = SPOCK_CONVERGED;
    else if (S.k >= P.max_iters)
      reason = SPOCK_MAX_ITERS;
  }
  if (reason != -1) {
    S.reason = reason;
    S.sw = 0;
    S.refresh = 0;
    if (G) set_cond(A.h_sw, 0);
    if (G) set_cond(A.h_ref, 0);
    if (G) set_cond(A.h_loop, 0);
    return;
  }
  if (S.k < A.cap) A.rnorm[S.k] = S.omega;
  if (!P.supermann) {  // CP: v <- T(v)
    S.sw = 3;
    S.refresh = 1;
    S.act = 'K';
    if (G) set_cond(A.h_sw, 3);
    if (G) set_cond(A.h_ref, 1);
    return;
  }
  // Anderson direction (solver.cpp:64-76)
  const int kk = S.aa_k++;
  S.cpsi[0] = -1.0;
  S.ncpsi = 1;
  // Gram ring update: row / column of the newest difference (slot of head h)
  const int cols = S.aa_cols, m = P.m, s0 = ring(S.h, m);
  for (int b = 0; b < cols; ++b) {
    const int sb = ring(S.h - b, m);
    const double hi = red[8 + 2 * b], lo = red[8 + 2 * b + 1];
    S.gh[s0 + sb * kLoopMaxMem] = S.gh[sb + s0 * kLoopMaxMem] = hi;
    S.gl[s0 + sb * kLoopMaxMem] = S.gl[sb + s0 * kLoopMaxMem] = lo;
  }
  if (kk > P.m) {
    dd G[kLoopMaxMem * kLoopMaxMem], gr[kLoopMaxMem];
    double kap[kLoopMaxMem];
    for (int a = 0; a < cols; ++a) {
      const int sa = ring(S.h - a, m);
      for (int b = 0; b < cols; ++b) {
        const int sb = ring(S.h - b, m);
        G[a + b * cols] = {S.gh[sa + sb * kLoopMaxMem], S.gl[sa + sb * kLoopMaxMem]};
      }
      gr[a] = {red[8 + 2 * (cols + a)], red[8 + 2 * (cols + a) + 1]};
    }
    aa_kappa_dd<kLoopMaxMem>(G, gr, cols, A.nv, kap);
    for (int c = 0; c < cols; ++c) S.cpsi[c + 1] = -kap[c];
    S.ncpsi = cols + 1;
  }
  if (S.omega <= P.c0 * S.zeta) {  // K0
    S.zeta = S.omega;
    S.act = '0';
    ++S.k0;
    S.sw = 1;
    S.refresh = 1;
    if (G) set_cond(A.h_sw, 1);
    if (G) set_cond(A.h_ref, 1);
  } else {  // line search with M psi (solver.cpp:287-290)
    ++S.n_Lt;
    ++S.n_L;
    S.tau = 1.0;
    S.backtracks = 0;
    S.sw = 2;
    if (G) set_cond(A.h_sw, 2);
  }
}

// line-search trial decision (solver.cpp:295-338)
template <bool G>
__device__ void ctl_ls(const LoopArgs& A) {
  LoopState& S = *A.st;
  const LoopParams& P = A.P;
  const double* red = A.red;
  ++S.n_T;
  ++S.n_L;
  const double rad = red[0] - 2.0 * P.alpha * red[1] + red[2];
  if (rad < -1e-12 * fmax(1.0, red[0] + red[2])) {
    S.reason = -2;
    S.act = 'S';
    S.sw = 0;
    S.ls_more = 0;
    if (G) set_cond(A.h_ls, 0);
    if (G) set_cond(A.h_act, 0);
    if (G) set_cond(A.h_ref, 0);
    if (G) set_cond(A.h_loop, 0);
    return;
  }
  const double omt = sqrt(fmax(0.0, rad));
  S.omt = omt;
  if ((S.omega <= S.omega_safe && omt <= P.c1 * S.omega) || omt == 0.0) {  // K1
    S.omega_safe = omt + pow(P.c2, double(S.k));
    S.act = '1';
    ++S.k1;
    S.omega = omt;  // carried to the next iteration
    S.have_omega = 1;
    S.refresh = 0;
    S.ls_more = 0;
    if (G) set_cond(A.h_ls, 0);
    if (G) set_cond(A.h_act, 1);
    if (G) set_cond(A.h_ref, 0);
    return;
  }
  const double rho = omt * omt - S.tau * (red[3] + red[4]);
  if (rho >= P.sigma * omt * S.omega) {  // K2
    S.coef = P.lambda * rho / (omt * omt);
    S.act = '2';
    ++S.k2;
    S.refresh = 1;
    S.ls_more = 0;
    if (G) set_cond(A.h_ls, 0);
    if (G) set_cond(A.h_act, 2);
    if (G) set_cond(A.h_ref, 1);
    return;
  }
  S.tau *= P.beta;
  if (++S.backtracks > P.max_backtracks) {  // KM fallback
    S.act = 'S';
    ++S.stalled;
    S.refresh = 1;
    S.ls_more = 0;
    if (G) set_cond(A.h_ls, 0);
    if (G) set_cond(A.h_act, 3);
    if (G) set_cond(A.h_ref, 1);
    return;
  }
  S.ls_more = 1;
  if (G) set_cond(A.h_ls, 1);
  if (G) set_cond(A.h_act, 0);
}

// end of iteration k: branch record, refresh bookkeeping, loop condition
template <bool G>
__device__ void ctl_end(const LoopArgs& A) {
  LoopState& S = *A.st;
  if (S.reason != -1) {
    if (G) set_cond(A.h_loop, 0);
    return;
  }
  if (S.k < A.cap) A.branch[S.k] = char(S.act);
  if (S.refresh) {
    S.have_omega = 0;
    ++S.n_T;
    ++S.n_L;
  }
  ++S.k;
  if (G) set_cond(A.h_loop, S.k < S.k_stop ? 1 : 0);
}

}  // namespace spock
