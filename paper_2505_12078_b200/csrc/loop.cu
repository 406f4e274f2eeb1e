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
#include "aa.cuh"
#include "loop.hpp"
#include "loop_ctl.cuh"

namespace spock {

static_assert(kGramRegion == 4 * kLoopMaxMem * kRedBlocks + 2, "Gram partial region");

namespace {


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

// Gram update of the Anderson history in double-double (aa.cuh): per thread,
// error-free products accumulated by two-sum; per block, a fixed-order warp and
// warp-to-warp reduction; the last block to arrive sums the block partials in
// block order.  Outputs (hi, lo) of <dnew, D[b]> (b < cols), then <D[b], r>.
__device__ __forceinline__ dd warp_sum_dd(dd v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const dd u = {__shfl_xor_sync(0xffffffffu, v.hi, o), __shfl_xor_sync(0xffffffffu, v.lo, o)};
    v = (threadIdx.x & o) ? dd_add(u, v) : dd_add(v, u);  // same operand order on both lanes
  }
  return v;
}

// push (graph loop): the history push fused in -- dnew = first ? r : r - rp is
// written to the new difference column as it is read, and r to the new
// residual slot; ctl: the controller (ctl_begin) runs in the last block
struct GramPush {
  double* dn;
  double* rn;
  const double* rp;
  int first;
  const LoopArgs* ctl;
};
__device__ void gram_dd_body(const double* __restrict__ dnew, const double* __restrict__ r,
                             const double* const* D, const double* __restrict__ w, int cols, int64_t n,
                             double* __restrict__ partial, double* out, const GramPush* push = nullptr) {
  constexpr int M = kLoopMaxMem;
  constexpr int NW = kRedThreads / 32;
  __shared__ double sh[2 * M][NW], sl[2 * M][NW];
  __shared__ int last;
  dd acc[2 * M];
#pragma unroll
  for (int j = 0; j < 2 * M; ++j) acc[j] = {0.0, 0.0};
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += stride) {
    // entries with weight 0 may hold anything (another rank computes them): skipped, not multiplied
    if (w && w[i] == 0.0) continue;
    const double rr = r[i];
    double x;
    if (push) {
      x = push->first ? rr : rr - push->rp[i];
      push->dn[i] = x;
      push->rn[i] = rr;
    } else {
      x = dnew[i];
    }
#pragma unroll
    for (int b = 0; b < M; ++b)
      if (b < cols) {
        const double db = (push && b == 0) ? x : D[b][i];  // push: column 0 is the one being written
        acc[b] = dd_fma(acc[b], x, db);
        acc[M + b] = dd_fma(acc[M + b], db, rr);
      }
  }
  const int wp = threadIdx.x >> 5, nd = 2 * cols;
#pragma unroll
  for (int j = 0; j < 2 * M; ++j) {
    if ((j < M ? j : j - M) >= cols) continue;  // only the 2 cols sums in use (warp-uniform)
    const dd v = warp_sum_dd(acc[j]);
    if ((threadIdx.x & 31) == 0) sh[j][wp] = v.hi, sl[j][wp] = v.lo;
  }
  __syncthreads();
  const int nb = gridDim.x;
  if (threadIdx.x < nd) {
    const int j = threadIdx.x < cols ? threadIdx.x : M + threadIdx.x - cols;
    dd s = {sh[j][0], sl[j][0]};
    for (int k = 1; k < NW; ++k) s = dd_add(s, {sh[j][k], sl[j][k]});
    partial[size_t(2 * threadIdx.x) * nb + blockIdx.x] = s.hi;
    partial[size_t(2 * threadIdx.x + 1) * nb + blockIdx.x] = s.lo;
  }
  // last block: partials in block order (thread-strided, warp tree, warps in order)
  unsigned int* counter = reinterpret_cast<unsigned int*>(partial + size_t(4 * M) * kRedBlocks);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == unsigned(nb - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int j = 0; j < nd; ++j) {
    dd s = {0.0, 0.0};
    for (int k = threadIdx.x; k < nb; k += blockDim.x)
      s = dd_add(s, {__ldcg(partial + size_t(2 * j) * nb + k), __ldcg(partial + size_t(2 * j + 1) * nb + k)});
    s = warp_sum_dd(s);
    if ((threadIdx.x & 31) == 0) sh[0][wp] = s.hi, sl[0][wp] = s.lo;
    __syncthreads();
    if (threadIdx.x == 0) {
      dd o = {sh[0][0], sl[0][0]};
      for (int k = 1; k < NW; ++k) o = dd_add(o, {sh[0][k], sl[0][k]});
      out[2 * j] = o.hi;
      out[2 * j + 1] = o.lo;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *counter = 0u;
    if (push && push->ctl) ctl_begin<true>(*push->ctl);
  }
}

// graph loop: the history columns come from the device ring (head hn = h + 1)
__global__ void __launch_bounds__(kRedThreads) k_gram(const __grid_constant__ LoopArgs A, double* __restrict__ partial,
                                                      double* out) {
  const LoopState& S = *A.st;
  const int m = A.P.m, hn = S.h + 1, cols = min(S.aa_cols + 1, m);
  const double* D[kLoopMaxMem];
#pragma unroll
  for (int b = 0; b < kLoopMaxMem; ++b) D[b] = A.DH[ring(hn - min(b, cols - 1), m)];
  const GramPush P{A.DH[ring(hn, m)], A.RH[ring(hn, m + 1)], A.RH[ring(hn - 1, m + 1)], S.aa_k == 0 ? 1 : 0, &A};
  gram_dd_body(D[0], A.R, D, nullptr, cols, A.nv, partial, out, &P);
}

__global__ void __launch_bounds__(kRedThreads) k_gram_args(const __grid_constant__ GramArgs G, double* __restrict__ partial,
                                                           double* out) {
  gram_dd_body(G.dnew, G.r, G.D, G.w, G.cols, G.n, partial, out);
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

__global__ void k_begin(const __grid_constant__ LoopArgs A) { ctl_begin<true>(A); }
__global__ void k_ls(const __grid_constant__ LoopArgs A) { ctl_ls<true>(A); }
__global__ void k_end(const __grid_constant__ LoopArgs A) { ctl_end<true>(A); }

__global__ void k_k2(const __grid_constant__ LoopArgs A) {  // v <- v - coef r~
  const double coef = A.st->coef;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < A.nv; i += int64_t(gridDim.x) * blockDim.x)
    A.V[i] -= coef * A.CR[i];
}

inline int vec_blocks(int64_t n) { return int(std::min<int64_t>((n + 255) / 256, 4 * 148)); }

}  // namespace

void loop_push(const LoopArgs& A, cudaStream_t st) { k_push<<<vec_blocks(A.nv), 256, 0, st>>>(A); }
void loop_gram(const LoopArgs& A, double* partial, double* out, cudaStream_t st) {
  k_gram<<<kRedBlocks, kRedThreads, 0, st>>>(A, partial, out);
}
void launch_gram_dd(const GramArgs& A, double* partial, double* out, cudaStream_t st) {
  k_gram_args<<<kRedBlocks, kRedThreads, 0, st>>>(A, partial, out);
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
