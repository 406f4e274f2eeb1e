// Persistent dataflow kernel for one CP application T (fused.cu).
#pragma once

#include <cuda_runtime.h>

#include "dev.cuh"

namespace spock {

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
};

int fused_smem_bytes(const FusedArgs& F);
cudaError_t fused_configure(int smem_bytes);
void launch_T_fused(const FusedArgs& F, int grid, cudaStream_t st);
const void* fused_kernel_ptr();

}  // namespace spock
