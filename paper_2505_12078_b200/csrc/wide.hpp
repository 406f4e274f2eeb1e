// Streaming dataflow T for wide trees (wide.cu).
#pragma once

#include <cuda_runtime.h>

#include "dev.cuh"

namespace spock {

struct WideArgs {
  Dev D;
  const double* z;
  const double* eta;
  double* zo;
  double* eo;
  double alpha;
  int* flagB;   // [nn]  backward item of node i done (T12_i, adj_i, d_i); zeroed before each launch
  int* flagS2;  // [nnl] S2 of parent i done
  int* flagF;   // [nn]  forward (x+, u+) of node i done
  int slots;    // ring slots per warp
  int chunk;    // doubles per ring slot (even)
  int warps;    // warps per CTA
  int vecd;     // doubles per per-warp vector buffer (two per warp)
  unsigned long long* prof;  // optional [10] cycle counters (SPOCK_WIDE_PROF)
};

int wide_smem_bytes(int warps, int slots, int chunk, int vecd);
int wide_rows(const Dev& D, int max_nc);  // register row groups (template parameter)
cudaError_t wide_configure(int rows, int ctas, int smem_bytes);
const void* wide_kernel_ptr(int rows, int ctas);
void launch_T_wide(const WideArgs& A, int rows, int ctas, int grid, cudaStream_t st);

}  // namespace spock
