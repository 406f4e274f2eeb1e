// One CP application T as a single persistent dataflow kernel (sm_100a).
//
// Replaces the per-stage launches of the S1 sweeps (proj/src/projections.cpp:
// 142-187, 2N+2 fork-joins on the CPU) together with L* (tree_operator.cpp:
// 65-114), S2 (projections.cpp:189-210), L (tree_operator.cpp:20-63) and S3 +
// the Moreau step (projections.cpp:212-244, solver.cpp:159-163).
//
// Work items, handed out in this order by a global ticket counter:
//   [0, nnl)            S2 of parent i (no dependencies)
//   [nnl, nnl+nn)       backward item of node nn-1 ... 0 (children first)
//   [nnl+nn, nnl+2nn)   forward item of node 0 ... nn-1 (parents first)
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
// Forward item (node c):
//   x_c = [Abar_c B_c][x_anc; d_anc] + c_c,  u_c = K_c x_c + d_c  (flag released here)
//   then every dual segment owned by c: eta+ = p - a Pi_S3(p / a),
//   p = eta + a L(2 z+ - z).
#include <cuda_runtime.h>

#include <cstdint>

#include "dev.cuh"
#include "fused.hpp"

namespace spock {

namespace fused256 {
#define FUSED_FT 256
#include "fused_impl.cuh"
#undef FUSED_FT
}  // namespace fused256

namespace fused128 {
#define FUSED_FT 128
#include "fused_impl.cuh"
#undef FUSED_FT
}  // namespace fused128

namespace {
constexpr int kSlotD = kMaxD + 8;
constexpr int kScratchSlots = 6;
}  // namespace

int fused_smem_bytes(const FusedArgs& F) {
  return int(sizeof(double) * (size_t(F.nslots) * (size_t(F.mat_doubles) + F.vec_doubles) +
                               kScratchSlots * kSlotD + 2 * 256));
}

cudaError_t fused_configure(int smem_bytes, int threads) {
  if (threads == 128)
    return cudaFuncSetAttribute(fused128::k_T_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  return cudaFuncSetAttribute(fused256::k_T_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
}

const void* fused_kernel_ptr(int threads) {
  return threads == 128 ? reinterpret_cast<const void*>(&fused128::k_T_fused)
                        : reinterpret_cast<const void*>(&fused256::k_T_fused);
}

void launch_T_fused(const FusedArgs& F, int grid, cudaStream_t st) {
  if (F.threads == 128)
    fused128::k_T_fused<<<grid, 128, fused_smem_bytes(F), st>>>(F);
  else
    fused256::k_T_fused<<<grid, 256, fused_smem_bytes(F), st>>>(F);
}

}  // namespace spock
