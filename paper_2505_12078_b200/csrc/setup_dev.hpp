// Device-side setup: the SOC epigraph data of every node,
// soc_data_quadlin (proj/src/problem.cpp:113-161) per block of blkdiag(Q, R),
// as batched kernels: one CTA per symmetric eigendecomposition (parallel-order
// cyclic Jacobi in shared memory, canonical output), then the reduced
// square-root factor, the head map H = (S'MS)^{1/2} S' (and its transpose),
// the kernel component q - S S'q and the translation a, written straight into
// the per-node HBM layout the T kernels stream.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace spock {

constexpr int kEigMaxN = 112;  // a (n2 x n2) and U (n x n) in shared memory: 2 * 112^2 * 8 B = 196 KB

// one symmetric eigendecomposition: M (n x n, column-major, only read) ->
// W ascending (n), V (n x n, column-major, column k = eigenvector of W[k],
// largest-|entry| positive)
struct EigJob {
  const double* M;
  double* W;
  double* V;
  int n;
  int pad_;
};
int eig_smem_bytes(int n);
cudaError_t eig_configure(int nmax);
void launch_sym_eig(const EigJob* jobs, int njobs, int nmax, cudaStream_t st);

// per node: ranks of the x / u blocks from their eigenvalues (threshold
// 1e-10 lambda_max over both blocks, PSD check), lambda_max, and the merged
// ascending order of the kept eigenvalues (the boundary row permutation)
struct SocRankArgs {
  const double* Wx;  // [nb][nx]
  const double* Wu;  // [nb][nu] (nullptr: leaf blocks, no u part)
  int nb, nx, nu;
  int* px;           // [nb]
  int* pu;           // [nb]
  int* perm;         // [nb][nx + nu]
  double* lmax;      // [nb]
  int* err;          // set to 1 when a block is not positive semidefinite
};
void launch_soc_rank(const SocRankArgs& a, cudaStream_t st);

// one block of soc_data_quadlin: S = V(:, n-p..n), SMS = S'MS
struct SocBlockJob {
  const double* M;   // n x n
  const double* v;   // n (linear term)
  const double* V;   // n x n eigenvectors (ascending)
  double* sms;       // p x p  (S'MS; then its eigendecomposition)
  double* W2;        // p
  double* U2;        // p x p
  double* H;         // p x n, column-major (row k of the head map)
  double* HT;        // n x p, column-major
  double* qk;        // n: v - S S'v
  double* w;         // p: (S'MS)^{-1/2} S'v
  int n, p;
};
void launch_soc_sms(const SocBlockJob* jobs, int njobs, int nmax, cudaStream_t st);
void launch_soc_build(const SocBlockJob* jobs, int njobs, int nmax, cudaStream_t st);

// per node: translation a = (-w/2, -|w|^2/8 + 1/2, -|w|^2/8 - 1/2) and |qk|^2
struct SocTailArgs {
  const double* w;       // [nb][nx + nu] (x part then u part, p used)
  const int* px;
  const int* pu;         // nullptr: leaves
  const int64_t* a_off;  // [nb] offset of the node's translation in a
  double* a;
  const double* qk;      // [nb][qk_stride]
  int qk_stride;
  double* qk2;           // [nb]
  int nb, nx, nu;
};
void launch_soc_tail(const SocTailArgs& t, cudaStream_t st);

// P[b] = I (n x n) for b < count (zero-filled first)
void launch_eye(double* P, int64_t count, int n, cudaStream_t st);

}  // namespace spock
