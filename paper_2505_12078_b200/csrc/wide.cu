// Wide-tree streaming T (the kernel body lives in wide_impl.cuh; each row
// count is instantiated in its own translation unit, wide_r*.cu, so the five
// instantiations compile in parallel): launchers, configuration, and the
// exchange kernels of the subtree-sharded T.
#include "wide_impl.cuh"

namespace spock {

const void* wide_ptr_r1(int ctas);
const void* wide_ptr_r2(int ctas);
const void* wide_ptr_r3(int ctas);
const void* wide_ptr_r4(int ctas);
const void* wide_ptr_r5(int ctas);
const void* wide_ptr_r8(int ctas);
cudaError_t wide_launch_r1(const cudaLaunchConfig_t* cfg, int ctas, const WideArgs& A);
cudaError_t wide_launch_r2(const cudaLaunchConfig_t* cfg, int ctas, const WideArgs& A);
cudaError_t wide_launch_r3(const cudaLaunchConfig_t* cfg, int ctas, const WideArgs& A);
cudaError_t wide_launch_r4(const cudaLaunchConfig_t* cfg, int ctas, const WideArgs& A);
cudaError_t wide_launch_r5(const cudaLaunchConfig_t* cfg, int ctas, const WideArgs& A);
cudaError_t wide_launch_r8(const cudaLaunchConfig_t* cfg, int ctas, const WideArgs& A);

namespace {

// one warp per stage-ts node of this rank: record -> exchange buffer slot
__global__ void k_shard_pack(const __grid_constant__ ShardXArgs X) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, l = lane_id();
  const int c = X.b0 + w;
  if (c >= X.b1) return;
  const int m = X.D.nx + X.D.nu;
  const int k = c - X.bfirst;
  double* o = X.xbuf + size_t(k) * X.E;
  for (int r = l; r < m; r += 32) {
    o[r] = X.D.adj[size_t(c - 1) * m + r];
    o[m + r] = X.D.T12[size_t(c - 1) * m + r];
  }
  if (l < 6 && X.vec) {
    const int64_t ix = X.xidx[size_t(k) * 6 + l];
    o[2 * m + l] = ix < 0 ? 0.0 : (l < 2 ? X.z[ix] : X.eta[ix]);
  }
}

// remote stage-ts nodes: exchange buffer -> adj, T12, the inputs' tau/s entries; backward flag
__global__ void k_shard_unpack(const __grid_constant__ ShardXArgs X) {
  const int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, l = lane_id();
  if (k >= X.nbound) return;
  const int c = X.bfirst + k;
  if (c >= X.b0 && c < X.b1) return;
  const int m = X.D.nx + X.D.nu;
  const double* o = X.xbuf + size_t(k) * X.E;
  for (int r = l; r < m; r += 32) {
    X.D.adj[size_t(c - 1) * m + r] = o[r];
    X.D.T12[size_t(c - 1) * m + r] = o[m + r];
  }
  if (l < 6 && X.vec) {
    const int64_t ix = X.xidx[size_t(k) * 6 + l];
    if (ix >= 0) (l < 2 ? const_cast<double*>(X.z) : const_cast<double*>(X.eta))[ix] = o[2 * m + l];
  }
  __syncwarp();
  if (l == 0) {
    __threadfence();
    X.flagB[c] = 1;  // visible to the next launch (stream order)
  }
}

}  // namespace

void launch_shard_pack(const ShardXArgs& X, cudaStream_t st) {
  const int n = X.b1 - X.b0;
  if (n > 0) k_shard_pack<<<(n + 7) / 8, 256, 0, st>>>(X);
}
void launch_shard_unpack(const ShardXArgs& X, cudaStream_t st) {
  if (X.nbound > 0) k_shard_unpack<<<(X.nbound + 7) / 8, 256, 0, st>>>(X);
}

int wide_smem_bytes(const WideArgs& A) {
  return int(sizeof(double) * size_t(A.warps) * warp_doubles(A.slots, A.chunk, A.vrec, A.vecd));
}

int wide_rows(const Dev& D, int max_nc) {
  const int need = std::max(D.nx + D.nu, max_nc);
  const int r = (need + 31) / 32;
  if (r <= 1) return 1;
  if (r <= 2) return 2;
  if (r <= 3) return 3;
  if (r <= 4) return 4;
  if (r <= 5) return 5;  // n_x + n_u = 150 (c5: n_x 100, n_u 50)
  return 8;
}

const void* wide_kernel_ptr(int rows, int ctas) {
  switch (rows) {
    case 1: return wide_ptr_r1(ctas);
    case 2: return wide_ptr_r2(ctas);
    case 3: return wide_ptr_r3(ctas);
    case 4: return wide_ptr_r4(ctas);
    case 5: return wide_ptr_r5(ctas);
    default: return wide_ptr_r8(ctas);
  }
}

cudaError_t wide_configure(int rows, int ctas, int smem_bytes) {
  cudaFuncSetAttribute(wide_kernel_ptr(rows, ctas), cudaFuncAttributePreferredSharedMemoryCarveout,
                       cudaSharedmemCarveoutMaxShared);
  cudaFuncSetAttribute(reinterpret_cast<const void*>(&k_shard_pack), cudaFuncAttributePreferredSharedMemoryCarveout,
                       cudaSharedmemCarveoutMaxShared);
  cudaFuncSetAttribute(reinterpret_cast<const void*>(&k_shard_unpack),
                       cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  return set_smem_limit(wide_kernel_ptr(rows, ctas), smem_bytes);
}

// Items spin on the flags of smaller tickets and tickets are dealt round-robin
// by warp index, so every CTA of the grid must be resident at once: the launch
// is cooperative, which makes the runtime guarantee co-residency (or fail the
// launch) even when other kernels -- a concurrent solver's stream, another
// process under MPS -- hold part of the device.
cudaError_t launch_T_wide(const WideArgs& A, int rows, int ctas, int grid, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(32 * A.warps);
  cfg.dynamicSmemBytes = size_t(wide_smem_bytes(A));
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  switch (rows) {
    case 1: return wide_launch_r1(&cfg, ctas, A);
    case 2: return wide_launch_r2(&cfg, ctas, A);
    case 3: return wide_launch_r3(&cfg, ctas, A);
    case 4: return wide_launch_r4(&cfg, ctas, A);
    case 5: return wide_launch_r5(&cfg, ctas, A);
    default: return wide_launch_r8(&cfg, ctas, A);
  }
}

}  // namespace spock
