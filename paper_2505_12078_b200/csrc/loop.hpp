// Device-resident SuperMann / CP loop (loop.cu): the iteration of
// proj/src/solver.cpp:189-350 as one CUDA graph with conditional nodes (WHILE
// over iterations, SWITCH over the K0 / line-search / CP branches, WHILE over
// line-search trials, SWITCH over K1 / K2 / KM, IF for the refresh).  Branch
// decisions run in single-thread controller kernels on the reduction results
// already in HBM, so the host launches one graph per solve.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace spock {

constexpr int kLoopMaxMem = 10;  // Anderson memory handled by the graph loop (the Gram update in one launch)
constexpr int kAaHostMax = 64;   // Anderson memory of the host-driven loop (Gram update in chunks)
// double-double Gram update: 2 * cols dots of (hi, lo) per block, then the
// arrival counter of the last-block finalize
constexpr int kGramRegion = 4 * kLoopMaxMem * 296 + 2;

// solve state in device memory (read back by the host at the end)
struct LoopState {
  int k;           // iteration index of the next top-of-iteration check
  int k_stop;      // the graph returns to the host when k reaches k_stop
  int reason;      // -1 running, else SPOCK_* status; -2: negative M-norm radicand
  int have_omega;  // omega carried from a K1 step
  int aa_k, aa_cols, h;  // Anderson calls, history columns, history head (pushes so far)
  int backtracks;
  int n_T, n_L, n_Lt, k0, k1, k2, stalled;
  int sw, act, refresh;  // branch decisions (mirrors of the conditional handles)
  int ls_more;           // line search continues (mirror of the line-search WHILE handle)
  double omega, zeta, omega_safe, th1, th2, tau, omt, coef;
  double xi1, xi2;
  double cpsi[kLoopMaxMem + 1];  // psi = cpsi[0] r + sum_j cpsi[j+1] r_{k-1-j}
  int ncpsi;
  // Gram of the difference history in double-double, indexed by ring slot
  double gh[kLoopMaxMem * kLoopMaxMem], gl[kLoopMaxMem * kLoopMaxMem];
};

struct LoopParams {
  double eps_abs, eps_rel, c0, c1, c2, beta, sigma, lambda, alpha;
  int max_iters, max_backtracks, m, supermann;
};

struct LoopArgs {
  LoopState* st;
  LoopParams P;
  const double* red;  // reduction results: [0..3) M-norm dots, [3..5) <r~, M psi>, [4..6) xi norms,
                      // [8..) Gram update as (hi, lo) pairs: <d_new, d_b>, then <d_b, r>, b = 0..cols-1
  double* rnorm;      // per-iteration ||r||_M
  char* branch;       // per-iteration branch character
  int cap;            // capacity of rnorm / branch
  int64_t nz, nv;
  double* V;
  double* TV;
  double* R;
  double* C;
  double* CR;
  double* PSI;
  double* RH[kLoopMaxMem + 1];  // residual history ring (m + 1 slots)
  double* DH[kLoopMaxMem];      // difference history ring (m slots)
  unsigned long long h_loop, h_sw, h_ls, h_act, h_ref;  // cudaGraphConditionalHandle values
};

// kernels launched (and captured) by Engine::solve_graph
void loop_push(const LoopArgs& A, cudaStream_t st);                       // history push (before Gram)
void loop_gram(const LoopArgs& A, double* partial, double* out, cudaStream_t st);  // Gram update (double-double)
void loop_begin(const LoopArgs& A, cudaStream_t st);                      // termination, Anderson, branch
void loop_psi(const LoopArgs& A, cudaStream_t st);                        // psi from the device coefficients
void loop_axpy_tau(const LoopArgs& A, cudaStream_t st);                   // C = V + tau psi
void loop_ls(const LoopArgs& A, cudaStream_t st);                         // line-search decision
void loop_k2(const LoopArgs& A, cudaStream_t st);                         // V -= coef CR
void loop_end(const LoopArgs& A, cudaStream_t st);                        // bookkeeping, loop condition
void loop_ls_init(const LoopArgs& A, cudaStream_t st);                    // arm the line-search WHILE
void loop_copy(double* dst, const double* src, int64_t n, cudaStream_t st);

// The host-driven loop's Gram update: (hi, lo) of <dnew, D[b]> for b < cols,
// then <D[b], r>, with optional 0/1 weights w (sharded solve: the entries this
// rank counts); cols <= kLoopMaxMem per launch.
struct GramArgs {
  const double* dnew;
  const double* r;
  const double* D[kLoopMaxMem];
  const double* w;
  int cols;
  int64_t n;
};
void launch_gram_dd(const GramArgs& A, double* partial, double* out, cudaStream_t st);

}  // namespace spock
