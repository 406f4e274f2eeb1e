// Device-resident SuperMann / CP loop: controller kernels (loop.hpp).
//
// Each controller is a single thread that reads the reductions of the current
// iteration from HBM (M-norm dots, xi norms, Anderson Gram, line-search dots),
// runs the branch logic of proj/src/solver.cpp:238-349 exactly as the host
// loop does (Engine::solve_b), writes the scalars the next kernels read
// (psi coefficients, tau, K2 coefficient) and sets the graph's conditional
// handles.  The vector kernels read their coefficients from the state, so one
// captured graph serves every iteration.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>

#include "../../include/spock_b200.h"
#include "kernels.hpp"
#include "loop.hpp"

namespace spock {

namespace {

__device__ __forceinline__ void set_cond(unsigned long long h, unsigned int v) {
  cudaGraphSetConditional(static_cast<cudaGraphConditionalHandle>(h), v);
}

__device__ __forceinline__ int ring(int i, int n) { return ((i % n) + n) % n; }

// Anderson least squares from the Gram matrix by column-pivoted Cholesky (the
// R factor of the column-pivoted QR of M_d), as Engine's host aa_kappa.
__device__ void aa_kappa_dev(const double* G, const double* gr, int cols, double* kap) {
  constexpr int M = kLoopMaxMem;
  int piv[M];
  double W[M * M], Rm[M * M], cv[M];
  for (int a = 0; a < cols; ++a) piv[a] = a;
  for (int e = 0; e < cols * cols; ++e) W[e] = G[e], Rm[e] = 0.0;
  double maxd = 0.0;
  for (int a = 0; a < cols; ++a) maxd = fmax(maxd, G[a + a * cols]);
  const double floor_rel = 64.0 * 2.220446049250313e-16;
  int rank = 0;
  double maxpiv = 0.0;
  for (int t = 0; t < cols; ++t) {
    int best = t;
    for (int a = t + 1; a < cols; ++a)
      if (W[piv[a] + piv[a] * cols] > W[piv[best] + piv[best] * cols]) best = a;
    const int tmp = piv[t];
    piv[t] = piv[best];
    piv[best] = tmp;
    const int pt = piv[t];
    const double dd = W[pt + pt * cols];
    if (!(dd > floor_rel * maxd)) break;
    const double rkk = sqrt(dd);
    Rm[t + pt * cols] = rkk;
    maxpiv = fmax(maxpiv, rkk);
    for (int a = t + 1; a < cols; ++a) Rm[t + piv[a] * cols] = W[pt + piv[a] * cols] / rkk;
    double ct = gr[pt];
    for (int s = 0; s < t; ++s) ct -= Rm[s + pt * cols] * cv[s];
    cv[t] = ct / rkk;
    for (int a = t + 1; a < cols; ++a)
      for (int b = t + 1; b < cols; ++b) W[piv[a] + piv[b] * cols] -= Rm[t + piv[a] * cols] * Rm[t + piv[b] * cols];
    ++rank;
  }
  int np = 0;
  for (int t = 0; t < rank; ++t) np += (Rm[t + piv[t] * cols] > 1e-12 * maxpiv) ? 1 : 0;
  for (int a = 0; a < cols; ++a) kap[a] = 0.0;
  for (int t = np - 1; t >= 0; --t) {
    double s = cv[t];
    for (int a = t + 1; a < np; ++a) s -= Rm[t + piv[a] * cols] * kap[piv[a]];
    kap[piv[t]] = s / Rm[t + piv[t] * cols];
  }
}

// history push for iteration k (solver.cpp:57-63): newest slot hn = h + 1
__global__ void k_push(const __grid_constant__ LoopArgs A) {
  const LoopState& S = *A.st;
  const int m = A.P.m, hn = S.h + 1;
  double* rn = A.RH[ring(hn, m + 1)];
  const double* rp = A.RH[ring(hn - 1, m + 1)];
  double* dn = A.DH[ring(hn, m)];
  const bool first = S.aa_k == 0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < A.nv; i += int64_t(gridDim.x) * blockDim.x) {
    const double r = A.R[i];
    dn[i] = first ? r : r - rp[i];
    rn[i] = r;
  }
}

// Gram of the difference columns and M_d' r: pairs (a <= b) row-major, then a
__global__ void __launch_bounds__(kRedThreads) k_gram(const __grid_constant__ LoopArgs A, double* __restrict__ partial,
                                                      double* out) {
  constexpr int MD = kLoopMaxMem * (kLoopMaxMem + 1) / 2 + kLoopMaxMem;
  __shared__ double sm[MD][kRedThreads / 32];
  const LoopState& S = *A.st;
  const int m = A.P.m, hn = S.h + 1, cols = min(S.aa_cols + 1, m);
  const double* X[MD];
  const double* Y[MD];
  int nd = 0;
  for (int a = 0; a < cols; ++a)
    for (int b = a; b < cols; ++b) {
      X[nd] = A.DH[ring(hn - a, m)];
      Y[nd] = A.DH[ring(hn - b, m)];
      ++nd;
    }
  for (int a = 0; a < cols; ++a) {
    X[nd] = A.DH[ring(hn - a, m)];
    Y[nd] = A.R;
    ++nd;
  }
  double acc[MD];
#pragma unroll
  for (int j = 0; j < MD; ++j) acc[j] = 0.0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < A.nv; i += stride) {
#pragma unroll
    for (int j = 0; j < MD; ++j)
      if (j < nd) acc[j] += X[j][i] * Y[j][i];
  }
  const int w = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < MD; ++j) {
    double v = acc[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sm[j][w] = v;
  }
  __syncthreads();
  if (threadIdx.x < MD) {
    double s = 0.0;
    for (int k = 0; k < kRedThreads / 32; ++k) s += sm[threadIdx.x][k];
    partial[size_t(threadIdx.x) * gridDim.x + blockIdx.x] = s;
  }
  grid_finalize<false>(partial, MD, out, red_counter(partial));
}


// top of iteration k (solver.cpp:233-290): M-norm, xi thresholds, termination,
// Anderson direction coefficients, K0 test; selects the branch body
__global__ void k_begin(const __grid_constant__ LoopArgs A) {
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
    set_cond(A.h_sw, 0);
    set_cond(A.h_ref, 0);
    set_cond(A.h_loop, 0);
    return;
  }
  if (S.k < A.cap) A.rnorm[S.k] = S.omega;
  if (!P.supermann) {  // CP: v <- T(v)
    S.sw = 3;
    S.refresh = 1;
    S.act = 'K';
    set_cond(A.h_sw, 3);
    set_cond(A.h_ref, 1);
    return;
  }
  // Anderson direction (solver.cpp:64-76)
  const int kk = S.aa_k++;
  S.cpsi[0] = -1.0;
  S.ncpsi = 1;
  if (kk > P.m) {
    const int cols = S.aa_cols;
    double G[kLoopMaxMem * kLoopMaxMem], gr[kLoopMaxMem], kap[kLoopMaxMem];
    int j = 0;
    for (int a = 0; a < cols; ++a)
      for (int b = a; b < cols; ++b) {
        G[a + b * cols] = G[b + a * cols] = red[8 + j];
        ++j;
      }
    for (int a = 0; a < cols; ++a) gr[a] = red[8 + j++];
    aa_kappa_dev(G, gr, cols, kap);
    for (int c = 0; c < cols; ++c) S.cpsi[c + 1] = -kap[c];
    S.ncpsi = cols + 1;
  }
  if (S.omega <= P.c0 * S.zeta) {  // K0
    S.zeta = S.omega;
    S.act = '0';
    ++S.k0;
    S.sw = 1;
    S.refresh = 1;
    set_cond(A.h_sw, 1);
    set_cond(A.h_ref, 1);
  } else {  // line search with M psi (solver.cpp:287-290)
    ++S.n_Lt;
    ++S.n_L;
    S.tau = 1.0;
    S.backtracks = 0;
    S.sw = 2;
    set_cond(A.h_sw, 2);
  }
}

// first kernel of the line-search branch: arm its WHILE (the handle lives in
// that branch's body graph)
__global__ void k_ls_init(const __grid_constant__ LoopArgs A) { set_cond(A.h_ls, 1); }

__global__ void k_copy(double* __restrict__ dst, const double* __restrict__ src, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

// psi = cpsi[0] r + sum_c cpsi[c+1] r_{k-1-c}  (history head already advanced)
__global__ void k_psi(const __grid_constant__ LoopArgs A) {
  const LoopState& S = *A.st;
  const int m = A.P.m, h = S.h, nc = S.ncpsi;
  const double* src[kLoopMaxMem + 1];
  double cf[kLoopMaxMem + 1];
  src[0] = A.R;
  cf[0] = S.cpsi[0];
  for (int c = 1; c < nc; ++c) {
    src[c] = A.RH[ring(h - c, m + 1)];
    cf[c] = S.cpsi[c];
  }
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < A.nv; i += int64_t(gridDim.x) * blockDim.x) {
    double s = cf[0] * src[0][i];
    for (int c = 1; c < nc; ++c) s += cf[c] * src[c][i];
    A.PSI[i] = s;
  }
}

__global__ void k_axpy_tau(const __grid_constant__ LoopArgs A) {  // C = V + tau psi
  const double tau = A.st->tau;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < A.nv; i += int64_t(gridDim.x) * blockDim.x)
    A.C[i] = A.V[i] + tau * A.PSI[i];
}

// line-search trial decision (solver.cpp:295-338)
__global__ void k_ls(const __grid_constant__ LoopArgs A) {
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
    set_cond(A.h_ls, 0);
    set_cond(A.h_act, 0);
    set_cond(A.h_ref, 0);
    set_cond(A.h_loop, 0);
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
    set_cond(A.h_ls, 0);
    set_cond(A.h_act, 1);
    set_cond(A.h_ref, 0);
    return;
  }
  const double rho = omt * omt - S.tau * (red[3] + red[4]);
  if (rho >= P.sigma * omt * S.omega) {  // K2
    S.coef = P.lambda * rho / (omt * omt);
    S.act = '2';
    ++S.k2;
    S.refresh = 1;
    set_cond(A.h_ls, 0);
    set_cond(A.h_act, 2);
    set_cond(A.h_ref, 1);
    return;
  }
  S.tau *= P.beta;
  if (++S.backtracks > P.max_backtracks) {  // KM fallback
    S.act = 'S';
    ++S.stalled;
    S.refresh = 1;
    set_cond(A.h_ls, 0);
    set_cond(A.h_act, 3);
    set_cond(A.h_ref, 1);
    return;
  }
  set_cond(A.h_ls, 1);
  set_cond(A.h_act, 0);
}

__global__ void k_k2(const __grid_constant__ LoopArgs A) {  // v <- v - coef r~
  const double coef = A.st->coef;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < A.nv; i += int64_t(gridDim.x) * blockDim.x)
    A.V[i] -= coef * A.CR[i];
}

// end of iteration k: branch record, refresh bookkeeping, loop condition
__global__ void k_end(const __grid_constant__ LoopArgs A) {
  LoopState& S = *A.st;
  if (S.reason != -1) {
    set_cond(A.h_loop, 0);
    return;
  }
  if (S.k < A.cap) A.branch[S.k] = char(S.act);
  if (S.refresh) {
    S.have_omega = 0;
    ++S.n_T;
    ++S.n_L;
  }
  ++S.k;
  set_cond(A.h_loop, S.k < S.k_stop ? 1 : 0);
}

inline int vec_blocks(int64_t n) { return int(std::min<int64_t>((n + 255) / 256, 4 * 148)); }

}  // namespace

void loop_push(const LoopArgs& A, cudaStream_t st) { k_push<<<vec_blocks(A.nv), 256, 0, st>>>(A); }
void loop_gram(const LoopArgs& A, double* partial, double* out, cudaStream_t st) {
  k_gram<<<kRedBlocks, kRedThreads, 0, st>>>(A, partial, out);
}
void loop_begin(const LoopArgs& A, cudaStream_t st) { k_begin<<<1, 1, 0, st>>>(A); }
void loop_psi(const LoopArgs& A, cudaStream_t st) { k_psi<<<vec_blocks(A.nv), 256, 0, st>>>(A); }
void loop_axpy_tau(const LoopArgs& A, cudaStream_t st) { k_axpy_tau<<<vec_blocks(A.nv), 256, 0, st>>>(A); }
void loop_ls(const LoopArgs& A, cudaStream_t st) { k_ls<<<1, 1, 0, st>>>(A); }
void loop_k2(const LoopArgs& A, cudaStream_t st) { k_k2<<<vec_blocks(A.nv), 256, 0, st>>>(A); }
void loop_end(const LoopArgs& A, cudaStream_t st) { k_end<<<1, 1, 0, st>>>(A); }
void loop_ls_init(const LoopArgs& A, cudaStream_t st) { k_ls_init<<<1, 1, 0, st>>>(A); }
void loop_copy(double* dst, const double* src, int64_t n, cudaStream_t st) {
  k_copy<<<vec_blocks(n), 256, 0, st>>>(dst, src, n);
}

}  // namespace spock
