// Persistent dataflow kernel for one CP application T (fused.cu).
#pragma once

#include <cuda_runtime.h>

#include "dev.cuh"

namespace spock {

// Operand base arrays of the per-item records (offsets are relative to these).
enum FusedBase : int {
  FB_Z = 0, FB_ETA, FB_HXT, FB_HUT, FB_M1T, FB_KT, FB_RINV, FB_HNT, FB_QK, FB_GD, FB_H, FB_G, FB_QKN, FB_GND,
  FB_M1, FB_HX, FB_HU, FB_K, FB_HN, FB_CVEC, FB_A, FB_LO, FB_HI, FB_RB, FB_AN, FB_LON, FB_HIN, FB_BM, FB_FM,
  FB_FC, FB_COUNT
};
constexpr int kRecMats = 6;
constexpr int kRecSpans = 20;

// Precomputed per-item prefetch plan and metadata (built once on the host;
// one cooperative 512-byte load per item on the device).
struct alignas(16) ItemRec {
  int32_t kind, node, nmat, nspan;
  int32_t px, pu, pN, nc, ny, nch, c0, anc;
  int32_t s1o, s2o, s3o, yo;
  int64_t moff[kRecMats];
  int32_t mcnt[kRecMats];
  int64_t voff[kRecSpans];
  int32_t vcnt[kRecSpans];
  uint8_t mbase[kRecMats];
  uint8_t vbase[kRecSpans];
  uint8_t mcrit;  // bit k: matrix k is on the critical path (staged in critical-only mode)
  uint8_t pad_[5];
};
static_assert(sizeof(ItemRec) <= 512, "ItemRec must fit the 512-byte cooperative load");

struct FusedArgs {
  Dev D;
  const double* z;
  const double* eta;
  double* zo;
  double* eo;
  double alpha;
  unsigned long long* ticket;  // reset to 0 before each launch
  int* flagS2;                 // [nnl], reset to 0 before each launch
  int* flagB;                  // [nn]
  int* flagF;                  // [nn]
  int mat_doubles;             // shared-memory matrix staging area per ring slot (doubles)
  int vec_doubles;             // prefetched vector operands per ring slot (doubles)
  int stage_smem;              // 1: TMA bulk staging of node blocks into shared memory
  int stage_all;               // 1: stage every block; 0: only the critical-path blocks
  int nslots;                  // 1 or 2 (prefetch ring depth)
  int threads;                 // 128 or 256 threads per CTA
  int reg_gemv;                // 256 threads: register-resident critical-path GEMVs
  int red_doubles;             // shared scratch of the CTA GEMVs: (threads / 32) * max GEMV rows
  const ItemRec* items;        // [nnl + 2 nn]
  double* hand;                // optional [nn - 1] x 2m child -> parent slots (T12, adj), empty between launches
  double* fhand;               // optional [nn - 1] x (m + nu) parent -> child slots (x+, d, u+), likewise
  unsigned long long* trace;   // optional: 4 globaltimer stamps per item (debug/profiling)
  const double* base[FB_COUNT];
};

int fused_smem_bytes(const FusedArgs& F);
cudaError_t fused_configure(int smem_bytes, int threads, int reg);
void launch_T_fused(const FusedArgs& F, int grid, cudaStream_t st);
void launch_hand_clear(double* hand, int64_t n, cudaStream_t st);
void launch_build_combined(const Dev& D, double* Bm, double* Fm, double* fc, int64_t stride, cudaStream_t st);
const void* fused_kernel_ptr(int threads, int reg);

}  // namespace spock
