// One CP application T as a single persistent dataflow kernel (sm_100a).
//
// Replaces the per-stage launches of the S1 sweeps (proj/src/projections.cpp:
// 142-187, 2N+2 fork-joins on the CPU) together with L* (tree_operator.cpp:
// 65-114), S2 (projections.cpp:189-210), L (tree_operator.cpp:20-63) and S3 +
// the Moreau step (projections.cpp:212-244, solver.cpp:159-163).
//
// Work items, handed out in this order by a global ticket counter:
//   [0, nn)             backward item of node nn-1 ... 0 (children first)
//   [nn, nn+nnl)        S2 of parent i (no dependencies; needed by forward items)
//   [nn+nnl, 2nn+nnl)   forward item of node 0 ... nn-1 (parents first)
// An item only waits on items with smaller tickets.  A CTA holds at most two
// items: the one it computes and the next one, whose operands are already in
// flight into the other half of a two-slot shared-memory ring: the node's
// matrices by TMA bulk copies (cp.async.bulk + mbarrier) and every operand
// that does not depend on other items (z and eta segments, box data, SOC
// translations, ...) by cp.async.  The smallest unfinished item is always
// either being computed or the prefetched next item of a CTA whose current
// item is done, so the schedule cannot deadlock.  Completion is published per
// node with release/acquire flags (CTA barrier + one fenced release store).
//
// Backward item (node i), restructured Alg. 2 (see kernels.cu header):
//   adj_i = H_i' head_i - rsum_i/2 qk_i                 (own stage SOC, for the parent)
//   xbar_i = z_x - a(G_x' ec_i + sum_c adj_c,x)          (L* and the CP primal step)
//   q_i = sum_c [Abar_c' q_c] - xbar_i - K_i' ubar_i + h_i ;  leaf: q_i = -xbar_i
//   d_i = Rt_i^{-1}(ubar_i - sum_c [B_c' q_c] - g_i)
//   [Abar_i' q_i; B_i' q_i] -> T12_i for the parent
// with every child-independent term computed before the flag wait and the
// rest as one parallel GEMV round: T12_i = [M1_i' | M1_i'K_i'] v, d_i = dc - Rt^-1 w.
// Forward item (node c), one GEMV with F_c = [M1_c; K_c M1_c]:
//   [x_c; u_c - d_c] = F_c [x_anc; d_anc] + [c_c; K_c c_c]  (flag released here)
//   then every dual segment owned by c: eta+ = p - a Pi_S3(p / a),
//   p = eta + a L(2 z+ - z).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "dev.cuh"
#include "fused.hpp"

namespace spock {

namespace fused256 {
#define FUSED_FT 256
#define FUSED_REG 0
#include "fused_impl.cuh"
#undef FUSED_REG
#undef FUSED_FT
}  // namespace fused256

// the register-resident GEMV variant (~250 registers per thread: one CTA of
// 256 threads per SM, the two-slot configuration)
namespace fused256r {
#define FUSED_FT 256
#define FUSED_REG 1
#include "fused_impl.cuh"
#undef FUSED_REG
#undef FUSED_FT
}  // namespace fused256r

namespace fused128 {
#define FUSED_FT 128
#define FUSED_REG 0
#include "fused_impl.cuh"
#undef FUSED_REG
#undef FUSED_FT
}  // namespace fused128

namespace {
// Offline combined blocks of the fused sweeps (one CTA per non-root node):
//   Bm = [M1' | M1' K'] (m x m), Fm = [M1; K M1] (m x m), fc = [c; K c]
// (leaves: only the M1 part; K is the node's own feedback gain).
__global__ void k_build_combined(Dev D, double* Bm, double* Fm, double* fc, int64_t cs) {
  const int c = blockIdx.x + 1;
  const int nx = D.nx, nu = D.nu, m = nx + nu;
  const bool leaf = D.cc[c] == 0;
  const double* M1 = D.M1 + size_t(c - 1) * D.m1_stride;   // nx x m
  const double* M1T = D.M1T + size_t(c - 1) * D.m1_stride; // m x nx
  const double* K = leaf ? nullptr : D.K + size_t(c) * D.k_stride;   // nu x nx
  const double* KT = leaf ? nullptr : D.KT + size_t(c) * D.k_stride; // nx x nu
  double* B = Bm + size_t(c - 1) * cs;
  double* Fo = Fm + size_t(c - 1) * cs;
  const double* cv = D.cvec + size_t(c - 1) * nx;
  double* f = fc + size_t(c - 1) * m;
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    const int r = e % m, col = e / m;
    double b = 0.0, fo = 0.0;
    if (col < nx) {
      b = M1T[r + size_t(col) * m];
    } else if (!leaf) {
      for (int k = 0; k < nx; ++k) b += M1T[r + size_t(k) * m] * KT[k + size_t(col - nx) * nx];
    }
    if (r < nx) {
      fo = M1[r + size_t(col) * nx];
    } else if (!leaf) {
      for (int k = 0; k < nx; ++k) fo += K[(r - nx) + size_t(k) * nu] * M1[k + size_t(col) * nx];
    }
    B[e] = b;
    Fo[e] = fo;
  }
  for (int r = threadIdx.x; r < m; r += blockDim.x) {
    double v = 0.0;
    if (r < nx) {
      v = cv[r];
    } else if (!leaf) {
      for (int k = 0; k < nx; ++k) v += K[(r - nx) + size_t(k) * nu] * cv[k];
    }
    f[r] = v;
  }
}
constexpr int kSlotD = kMaxD + 8;
constexpr int kScratchSlots = 6;
}  // namespace

int fused_smem_bytes(const FusedArgs& F) {
  return int(sizeof(double) * (size_t(F.nslots) * (size_t(F.mat_doubles) + F.vec_doubles) +
                               kScratchSlots * kSlotD + size_t(F.red_doubles)));
}

const void* fused_kernel_ptr(int threads, int reg) {
  if (threads == 128) return reinterpret_cast<const void*>(&fused128::k_T_fused);
  return reg ? reinterpret_cast<const void*>(&fused256r::k_T_fused)
             : reinterpret_cast<const void*>(&fused256::k_T_fused);
}

cudaError_t fused_configure(int smem_bytes, int threads, int reg) {
  const void* f = fused_kernel_ptr(threads, reg);
  // every kernel of the engine prefers the maximum shared-memory carveout, so
  // consecutive launches never wait for an SM to change its L1 / smem split
  cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  return set_smem_limit(f, smem_bytes);
}


namespace {
__global__ void k_hand_clear(double* h, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    h[i] = __longlong_as_double((long long)fused256::kHandEmpty);
}
}  // namespace

void launch_hand_clear(double* hand, int64_t n, cudaStream_t st) {
  if (n > 0) k_hand_clear<<<int(std::min<int64_t>((n + 255) / 256, 1184)), 256, 0, st>>>(hand, n);
}

void launch_build_combined(const Dev& D, double* Bm, double* Fm, double* fc, int64_t stride, cudaStream_t st) {
  if (D.nr > 0) k_build_combined<<<D.nr, 256, 0, st>>>(D, Bm, Fm, fc, stride);
}

void launch_T_fused(const FusedArgs& F, int grid, cudaStream_t st) {
  if (F.threads == 128)
    fused128::k_T_fused<<<grid, 128, fused_smem_bytes(F), st>>>(F);
  else if (F.reg_gemv)
    fused256r::k_T_fused<<<grid, 256, fused_smem_bytes(F), st>>>(F);
  else
    fused256::k_T_fused<<<grid, 256, fused_smem_bytes(F), st>>>(F);
}

}  // namespace spock
