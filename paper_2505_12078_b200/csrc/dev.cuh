// Device-side data layout of the B200 SPOCK solver.
//
// Everything lives in HBM, node-major, one contiguous block per node so that a
// warp streams a node's matrix with coalesced 256 B requests (lanes walk the
// rows of a column-major block).  Where a kernel needs the transpose of a
// block (L* against L, the backward against the forward sweep), the block is
// stored twice: each launch still reads every matrix once.
//
// Vectors z (primal) and eta (dual) use the reference's PrimalLayout and
// DualLayout (proj/include/spock/layout.hpp:14-52) except that the head rows
// of each stage-cost SOC segment are ordered [x rows; u rows] (the reference
// orders them by ascending eigenvalue); spock_* boundary calls permute.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace spock {

// Opt-in maximum dynamic shared memory per block on the current device.  The
// MaxDynamicSharedMemorySize attribute of a kernel is process-global, not per
// solver: each kernel gets this maximum (once it is known to cover the launch)
// so that a later solver with smaller blocks never lowers the limit under an
// earlier solver's launches.  Occupancy follows the launch's own byte count.
inline int smem_optin_max() {
  int dev = 0, v = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return v;
}
inline cudaError_t set_smem_limit(const void* f, int need) {
  cudaFuncAttributes fa{};
  const cudaError_t e = cudaFuncGetAttributes(&fa, f);
  if (e != cudaSuccess) return e;
  const int mx = smem_optin_max() - int(fa.sharedSizeBytes);  // dynamic + static <= opt-in
  if (need > mx) return cudaErrorInvalidValue;
  return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
}

constexpr int kWarps = 8;          // warps per CTA in warp-per-node kernels
constexpr int kMaxD = 256;         // max nx+nu (and any per-node GEMV length)
constexpr int kMaxR = kMaxD / 32;  // rows per lane

// S2 closed forms (kernel of M = [E' -I -I], MM' = a I + b 11')
enum S2Kind : int { S2_AVAR = 0, S2_MAX = 1, S2_EQ = 2, S2_DENSE = 3 };

struct Dev {
  int nn, nnl, nl, nr, nx, nu, N;
  int nz, neta;
  // tree (proj/include/spock/tree.hpp:82-87)
  const int* anc;
  const int* cf;  // child_first
  const int* cc;  // child_count
  // primal layout
  int u_base, tau_base, s_base, y_base;
  const int* y_off;
  const int* y_dim;
  // dual layout
  const int* s1_off;
  const int* s1_nc;
  const int* s1_ydim;
  const int* s2_off;
  const int* s2_dim;
  const int* s3_off;
  const int* s3_nc;
  const int* s3_socdim;
  // stage-cost SOC data per non-root (index node-1)
  const int* px;
  const int* pu;
  const int64_t* hx_off;  // into Hx/HxT (px*nx each)
  const int64_t* hu_off;  // into Hu/HuT (pu*nu each)
  const double* Hx;       // px x nx col-major (L)
  const double* HxT;      // nx x px col-major (L*)
  const double* Hu;
  const double* HuT;
  const double* qk;      // (nx+nu) per non-root
  const int64_t* a_off;  // translation a (p+2) per non-root
  const double* a;
  // terminal SOC data per leaf
  const int* pN;
  const int64_t* hn_off;
  const double* HN;   // pN x nx
  const double* HNT;  // nx x pN
  const double* qkN;  // nx per leaf
  const int64_t* aN_off;
  const double* aN;
  // stage constraints per non-leaf: diagonal fast path or dense
  int g_diag;          // 1: every [Gx Gu] is square diagonal -> gd
  const double* gd;    // (nx+nu) per non-leaf
  const int64_t* g_off;  // row offsets
  const double* Gx;      // nc x nx
  const double* Gu;      // nc x nu
  const double* GxT;     // nx x nc
  const double* GuT;     // nu x nc
  const double* lo;      // box per non-leaf, at g_off
  const double* hi;
  // terminal constraints per leaf
  int gN_diag;
  const double* gNd;  // nx per leaf
  const int64_t* gN_off;
  const double* GN;   // ncN x nx
  const double* GNT;  // nx x ncN
  const double* loN;
  const double* hiN;
  // risk per non-leaf: b at (y_off - y_base); dual cone of the y-copy rows
  const double* rb;
  const int* yc_nonneg;  // >=0: leading nonneg rows then free rows; -1: general parts
  const int* yc_poff;    // general parts [yc_poff[i], yc_poff[i+1])
  const int* yc_kind;
  const int* yc_dim;
  // S2 per non-leaf
  const int* s2_kind;
  const double* s2_gamma;
  const int64_t* s2p_off;
  const double* s2P;  // dense projectors (dim x dim)
  // offline factors (Alg. 1) restructured for one-pass sweeps (see kernels.cu)
  // per-node strides of the factor blocks (even numbers of doubles: 16 B
  // aligned blocks for TMA bulk copies)
  int64_t m1_stride, k_stride, r_stride;
  const double* M1;   // [Abar B] nx x (nx+nu) per non-root (forward)
  const double* M1T;  // (nx+nu) x nx per non-root (backward)
  const double* cvec; // nx per non-root
  const double* K;    // nu x nx per non-leaf (forward)
  const double* KT;   // nx x nu per non-leaf (backward)
  const double* Rinv; // nu x nu per non-leaf
  const double* g;    // nu per non-leaf: sum_c B_c' P_c c_c
  const double* h;    // nx per non-leaf: sum_c Abar_c' P_c c_c
  const double* xinit;  // scaled x_init (nx)
  // scratch
  double* T12;  // (nx+nu) per non-root: [Abar' q; B' q] of the child sweep
  double* adj;  // (nx+nu) per non-root: L* stage-cost child terms
  double* dvec; // nu per non-leaf
};

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Tail of a deterministic grid reduction.  Every block has written its
// per-value partials partial[j * gridDim.x + block]; the last block to arrive
// (arrival counter in global memory, reset here for the next launch) combines
// them in a fixed order -- thread-strided, then warp tree, then warps in index
// order -- and writes out[j].  MAX: maximum with NaN propagation, else sum.
// Replaces a separate one-thread-per-value finalize launch whose serial loop
// over the partials cost ~10 us of L2 latency per reduction.
template <bool MAX>
__device__ void grid_finalize(const double* partial, int nvals, double* out, unsigned int* counter) {
  __shared__ int last;
  __shared__ double wsum[32];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int nparts = gridDim.x, nw = blockDim.x >> 5, w = threadIdx.x >> 5;
  for (int j = 0; j < nvals; ++j) {
    double s = 0.0;
    bool nan = false;
    for (int k = threadIdx.x; k < nparts; k += blockDim.x) {
      const double v = __ldcg(partial + size_t(j) * nparts + k);
      if (MAX) {
        nan |= isnan(v);
        s = fmax(s, v);
      } else {
        s += v;
      }
    }
    if (MAX) {
      s = warp_max(s);
      if (__any_sync(0xffffffffu, nan)) s = NAN;
    } else {
      s = warp_sum(s);
    }
    if ((threadIdx.x & 31) == 0) wsum[w] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double o = wsum[0];
      for (int k = 1; k < nw; ++k) o = MAX ? ((isnan(o) || isnan(wsum[k])) ? NAN : fmax(o, wsum[k])) : o + wsum[k];
      out[j] = o;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *counter = 0u;
}

// acc[k] += sum_c A[(lane + 32k) + c*lda] * x[c]  for rows < m, columns < n.
// A is column-major; each column is read by the warp as one coalesced run.
__device__ __forceinline__ void warp_gemv(const double* __restrict__ A, int m, int n, int lda,
                                          const double* x, double (&acc)[kMaxR]) {
  const int l = lane_id();
  int c = 0;
  for (; c + 4 <= n; c += 4) {
    const double x0 = x[c], x1 = x[c + 1], x2 = x[c + 2], x3 = x[c + 3];
    const double* c0 = A + size_t(c) * lda;
#pragma unroll
    for (int k = 0; k < kMaxR; ++k) {
      const int r = l + 32 * k;
      if (k * 32 < m && r < m) {
        const double a0 = c0[r], a1 = c0[lda + r], a2 = c0[2 * lda + r],
                     a3 = c0[3 * lda + r];
        acc[k] = fma(a0, x0, acc[k]);
        acc[k] = fma(a1, x1, acc[k]);
        acc[k] = fma(a2, x2, acc[k]);
        acc[k] = fma(a3, x3, acc[k]);
      }
    }
  }
  for (; c < n; ++c) {
    const double xc = x[c];
    const double* col = A + size_t(c) * lda;
#pragma unroll
    for (int k = 0; k < kMaxR; ++k) {
      const int r = l + 32 * k;
      if (k * 32 < m && r < m) acc[k] = fma(col[r], xc, acc[k]);
    }
  }
}

__device__ __forceinline__ void zero_acc(double (&acc)[kMaxR]) {
#pragma unroll
  for (int k = 0; k < kMaxR; ++k) acc[k] = 0.0;
}

}  // namespace spock
