// Latency-optimised standalone L and L* for narrow trees (sm_100a).
//
// TreeOperator::apply / apply_adjoint (proj/src/tree_operator.cpp:20-114) as
// used by the SuperMann loop outside T (M-norm, xi residuals, M psi).  One CTA
// per node (grid-stride): the whole CTA issues the node's coalesced block loads
// at once, so a node costs about one HBM round trip instead of the ~10 a single
// warp needs (kernels.cu).  Same arithmetic and ascending sibling order as the
// warp-per-node kernels.
#include <cuda_runtime.h>

#include "dev.cuh"
#include "kernels.hpp"

namespace spock {

namespace {

constexpr int kT = 256;
constexpr int kV = kMaxD + 8;

// y[r] = (acc ? y[r] : 0) + sum_c A[r + c*lda] x[c]; A in global memory
__device__ void gemv_g(const double* __restrict__ A, int m, int n, int lda, const double* x, double* y, bool acc,
                       double* red) {
  const int t = threadIdx.x;
  if (m <= 0) return;
  if (m > kT) {
    for (int r = t; r < m; r += kT) {
      double v = acc ? y[r] : 0.0;
      for (int c = 0; c < n; ++c) v = fma(__ldg(A + r + size_t(c) * lda), x[c], v);
      y[r] = v;
    }
    __syncthreads();
    return;
  }
  const int slices = max(1, kT / m);
  const int r = t % m, s = t / m;
  double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
  if (s < slices) {
    int c = s;
    for (; c + 3 * slices < n; c += 4 * slices) {
      const double a0 = __ldg(A + r + size_t(c) * lda), a1 = __ldg(A + r + size_t(c + slices) * lda);
      const double a2 = __ldg(A + r + size_t(c + 2 * slices) * lda), a3 = __ldg(A + r + size_t(c + 3 * slices) * lda);
      v0 = fma(a0, x[c], v0);
      v1 = fma(a1, x[c + slices], v1);
      v2 = fma(a2, x[c + 2 * slices], v2);
      v3 = fma(a3, x[c + 3 * slices], v3);
    }
    for (; c < n; c += slices) v0 = fma(__ldg(A + r + size_t(c) * lda), x[c], v0);
  }
  if (t < m * slices) red[t] = (v0 + v1) + (v2 + v3);
  __syncthreads();
  if (t < m) {
    double o = acc ? y[t] : 0.0;
    for (int j = 0; j < slices; ++j) o += red[t + j * m];
    y[t] = o;
  }
  __syncthreads();
}

__device__ double bsum(double v, double* red) {
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < kT / 32; ++k) s += red[k];
  __syncthreads();
  return s;
}

__device__ __forceinline__ int sidx(const Dev& D, int node) { return node == 0 ? 0 : D.s_base + node - 1; }

// eta = L w, w = z (one CTA per node)
__global__ void __launch_bounds__(kT) k_L_cta(Dev D, const double* __restrict__ z, double* __restrict__ eta) {
  __shared__ double xs[kV], ys[kV], red[kT];
  const int t = threadIdx.x, nx = D.nx, nu = D.nu, m = nx + nu;
  for (int i = blockIdx.x; i < D.nn; i += gridDim.x) {
    if (i < D.nnl) {
      const int ny = D.y_dim[i], yo = D.y_off[i], so = D.s1_off[i], nc = D.s1_nc[i];
      const double* rb = D.rb + (yo - D.y_base);
      double part = 0.0;
      for (int r = t; r < ny; r += kT) {
        const double yv = z[yo + r];
        part += rb[r] * yv;
        eta[so + r] = yv;
      }
      for (int r = t; r < m; r += kT) xs[r] = r < nx ? z[1 + size_t(i) * nx + r] : z[D.u_base + size_t(i) * nu + r - nx];
      const double by = bsum(part, red);
      if (t == 0) eta[so + ny] = z[sidx(D, i)] - by;
      if (D.g_diag) {
        const double* gd = D.gd + size_t(i) * m;
        for (int r = t; r < nc; r += kT) eta[so + ny + 1 + r] = gd[r] * xs[r];
      } else {
        gemv_g(D.Gx + D.g_off[i] * nx, nc, nx, nc, xs, ys, false, red);
        gemv_g(D.Gu + D.g_off[i] * nu, nc, nu, nc, xs + nx, ys, true, red);
        for (int r = t; r < nc; r += kT) eta[so + ny + 1 + r] = ys[r];
      }
      __syncthreads();
    }
    if (i > 0) {
      const int k = i - 1, an = D.anc[i], px = D.px[k], pu = D.pu[k], p = px + pu, o2 = D.s2_off[k];
      for (int r = t; r < m; r += kT) xs[r] = r < nx ? z[1 + size_t(an) * nx + r] : z[D.u_base + size_t(an) * nu + r - nx];
      __syncthreads();
      const double* qk = D.qk + size_t(k) * m;
      double part = 0.0;
      for (int r = t; r < m; r += kT) part += qk[r] * xs[r];
      const double qd = bsum(part, red);
      gemv_g(D.Hx + D.hx_off[k], px, nx, px, xs, ys, false, red);
      gemv_g(D.Hu + D.hu_off[k], pu, nu, pu, xs + nx, ys + px, false, red);
      for (int r = t; r < p; r += kT) eta[o2 + r] = ys[r];
      if (t == 0) {
        const double row = 0.5 * z[D.tau_base + k] - 0.5 * qd;
        eta[o2 + p] = row;
        eta[o2 + p + 1] = row;
      }
      __syncthreads();
    }
    if (i >= D.nnl) {
      const int j = i - D.nnl, nc = D.s3_nc[j], p = D.pN[j], eo = D.s3_off[j];
      for (int r = t; r < nx; r += kT) xs[r] = z[1 + size_t(i) * nx + r];
      __syncthreads();
      if (D.gN_diag) {
        const double* gd = D.gNd + size_t(j) * nx;
        for (int r = t; r < nc; r += kT) eta[eo + r] = gd[r] * xs[r];
      } else {
        gemv_g(D.GN + D.gN_off[j] * nx, nc, nx, nc, xs, ys, false, red);
        for (int r = t; r < nc; r += kT) eta[eo + r] = ys[r];
      }
      const double* qk = D.qkN + size_t(j) * nx;
      double part = 0.0;
      for (int r = t; r < nx; r += kT) part += qk[r] * xs[r];
      const double qd = bsum(part, red);
      gemv_g(D.HN + D.hn_off[j], p, nx, p, xs, ys, false, red);
      for (int r = t; r < p; r += kT) eta[eo + nc + r] = ys[r];
      if (t == 0) {
        const double row = 0.5 * z[D.s_base + i - 1] - 0.5 * qd;
        eta[eo + nc + p] = row;
        eta[eo + nc + p + 1] = row;
      }
      __syncthreads();
    }
  }
}

// L* part 1: per non-root child, adj = H' head - rsum/2 qk, and the tau slot
__global__ void __launch_bounds__(kT) k_Lt_child_cta(Dev D, const double* __restrict__ eta, double* __restrict__ zo) {
  __shared__ double xs[kV], ys[kV], red[kT];
  const int t = threadIdx.x, nx = D.nx, nu = D.nu, m = nx + nu;
  for (int k = blockIdx.x; k < D.nr; k += gridDim.x) {
    const int px = D.px[k], pu = D.pu[k], p = px + pu, o2 = D.s2_off[k];
    for (int r = t; r < p; r += kT) xs[r] = eta[o2 + r];
    const double rsum = eta[o2 + p] + eta[o2 + p + 1];
    const double* qk = D.qk + size_t(k) * m;
    for (int r = t; r < m; r += kT) ys[r] = -0.5 * rsum * qk[r];
    __syncthreads();
    gemv_g(D.HxT + D.hx_off[k], nx, px, nx, xs, ys, true, red);
    gemv_g(D.HuT + D.hu_off[k], nu, pu, nu, xs + px, ys + nx, true, red);
    double* adj = D.adj + size_t(k) * m;
    for (int r = t; r < m; r += kT) adj[r] = ys[r];
    if (t == 0) zo[D.tau_base + k] = 0.5 * rsum;
    __syncthreads();
  }
}

// L* part 2: per node, own segments + ascending sum of the children's adj
__global__ void __launch_bounds__(kT) k_Lt_node_cta(Dev D, const double* __restrict__ eta, double* __restrict__ zo) {
  __shared__ double xs[kV], ys[kV], red[kT];
  const int t = threadIdx.x, nx = D.nx, nu = D.nu, m = nx + nu;
  for (int i = blockIdx.x; i < D.nn; i += gridDim.x) {
    if (i < D.nnl) {
      const int ny = D.y_dim[i], yo = D.y_off[i], so = D.s1_off[i], nc = D.s1_nc[i];
      const double sc = eta[so + ny];
      const double* rb = D.rb + (yo - D.y_base);
      for (int r = t; r < ny; r += kT) zo[yo + r] = eta[so + r] - sc * rb[r];
      if (t == 0) zo[sidx(D, i)] = sc;
      const double* ec = eta + so + ny + 1;
      if (D.g_diag) {
        const double* gd = D.gd + size_t(i) * m;
        for (int r = t; r < m; r += kT) ys[r] = gd[r] * ec[r];
        __syncthreads();
      } else {
        for (int r = t; r < nc; r += kT) xs[r] = ec[r];
        __syncthreads();
        gemv_g(D.GxT + D.g_off[i] * nx, nx, nc, nx, xs, ys, false, red);
        gemv_g(D.GuT + D.g_off[i] * nu, nu, nc, nu, xs, ys + nx, false, red);
      }
      const int c0 = D.cf[i], nch = D.cc[i];
      for (int r = t; r < m; r += kT) {
        double v = ys[r];
        for (int c = 0; c < nch; ++c) v += D.adj[size_t(c0 + c - 1) * m + r];
        if (r < nx)
          zo[1 + size_t(i) * nx + r] = v;
        else
          zo[D.u_base + size_t(i) * nu + r - nx] = v;
      }
      __syncthreads();
    } else {
      const int j = i - D.nnl, nc = D.s3_nc[j], p = D.pN[j];
      const double* ec = eta + D.s3_off[j];
      const double* hd = ec + nc;
      const double rsum = hd[p] + hd[p + 1];
      if (D.gN_diag) {
        const double* gd = D.gNd + size_t(j) * nx;
        for (int r = t; r < nx; r += kT) ys[r] = gd[r] * ec[r];
        __syncthreads();
      } else {
        for (int r = t; r < nc; r += kT) xs[r] = ec[r];
        __syncthreads();
        gemv_g(D.GNT + D.gN_off[j] * nx, nx, nc, nx, xs, ys, false, red);
      }
      for (int r = t; r < p; r += kT) xs[r] = hd[r];
      __syncthreads();
      gemv_g(D.HNT + D.hn_off[j], nx, p, nx, xs, ys, true, red);
      const double* qk = D.qkN + size_t(j) * nx;
      for (int r = t; r < nx; r += kT) zo[1 + size_t(i) * nx + r] = ys[r] - 0.5 * rsum * qk[r];
      if (t == 0) zo[D.s_base + i - 1] = 0.5 * rsum;
      __syncthreads();
    }
  }
}

}  // namespace

void set_carveout_narrow() {
  cudaFuncSetAttribute(k_L_cta, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  cudaFuncSetAttribute(k_Lt_child_cta, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  cudaFuncSetAttribute(k_Lt_node_cta, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
}

void launch_L_narrow(const Dev& D, const double* z, double* eta, cudaStream_t st) {
  k_L_cta<<<std::min(D.nn, 4 * 148), kT, 0, st>>>(D, z, eta);
}

void launch_Lt_narrow(const Dev& D, const double* eta, double* z, cudaStream_t st) {
  if (D.nr > 0) k_Lt_child_cta<<<std::min(D.nr, 4 * 148), kT, 0, st>>>(D, eta, z);
  k_Lt_node_cta<<<std::min(D.nn, 4 * 148), kT, 0, st>>>(D, eta, z);
}

}  // namespace spock
