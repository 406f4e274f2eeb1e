// Microbenchmark: cluster barrier and DSMEM access costs on B200 (cluster of C
// CTAs x 256 threads).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cluster_mb tools/cluster_mb.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ int cl_rank() { unsigned r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return int(r); }
__device__ __forceinline__ int cl_size() { unsigned r; asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r)); return int(r); }
template <class T> __device__ __forceinline__ T* cl_map(T* p, int rank) {
  uint64_t r; asm volatile("mapa.u64 %0, %1, %2;" : "=l"(r) : "l"(p), "r"(rank)); return reinterpret_cast<T*>(r);
}
__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void csync_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}

__global__ void k(int mode, int iters, long long* out) {
  __shared__ double buf[4096];
  const int r = cl_rank(), C = cl_size(), t = threadIdx.x;
  for (int i = t; i < 4096; i += blockDim.x) buf[i] = i;
  csync();
  double* peer = cl_map(buf, (r + 1) % C);
  double acc = 0.0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (mode == 1) { peer[t] = it; peer[t + 256] = it; }
    if (mode == 2) { acc += peer[t] + peer[t + 256]; }
    if (mode == 3) { buf[t] = it; buf[t + 256] = it; }
    if (mode == 5) { acc += peer[(t * 7 + it) & 4095]; }
    if (mode == 4) csync_relaxed(); else csync();
  }
  long long t1 = clock64();
  if (t == 0 && r == 0) out[mode] = (t1 - t0) / iters;
  if (acc == -1.0) out[7] = 1;
}

int main() {
  long long* d; cudaMalloc(&d, 64); cudaMemset(d, 0, 64);
  for (int C : {2, 4, 8}) {
    for (int mode = 0; mode < 6; ++mode) {
      cudaLaunchConfig_t cfg{}; cfg.gridDim = dim3(C); cfg.blockDim = dim3(256);
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = C;
      at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1; cfg.attrs = at; cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, k, mode, 10000, d);
      cudaDeviceSynchronize();
      long long h[8]; cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
      const char* nm[] = {"barrier only", "2 remote stores + barrier", "2 remote loads + barrier", "2 local stores + barrier", "relaxed barrier", "1 remote load + barrier"};
      printf("C=%d %-28s %lld cycles\n", C, nm[mode], h[mode]);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
