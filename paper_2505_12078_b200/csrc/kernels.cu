// Hot-path kernels of the B200 SPOCK solver (sm_100a, fp64).
//
// Mapping of the reference's CPU loops (arxiv/paper_2505_12078):
//   k_Lt_child / k_Lt_node  <- TreeOperator::apply_adjoint  proj/src/tree_operator.cpp:65-114
//   k_L (PLAIN / DUAL)      <- TreeOperator::apply          proj/src/tree_operator.cpp:20-63
//                              + proj_s3 and the Moreau step proj/src/projections.cpp:212-244,
//                                                             proj/src/solver.cpp:159-163
//   k_s1_back / k_s1_fwd    <- proj_s1 Alg. 2               proj/src/projections.cpp:142-187
//   k_s2                    <- proj_s2                      proj/src/projections.cpp:189-210
//   k_s3                    <- proj_s3                      proj/src/projections.cpp:212-244
//   k_dots / k_xi           <- SuperMann reductions          proj/src/solver.cpp:169,240-256,320
//   factorisation kernels   <- make_solver_cache Alg. 1     proj/src/projections.cpp:59-140
//
// All kernels are warp-per-node: a warp streams a node's column-major block
// with coalesced loads (lanes over rows), the input vector sits in shared
// memory, sibling sums run in ascending child order (bitwise deterministic),
// and reductions use a fixed grid with a fixed-order final pass.
//
// S1 restructuring.  With e_c = P_c c_c, g_i = sum_c B_c'e_c, h_i = sum_c
// Abar_c'e_c the reference recursion (projections.cpp:150-174) becomes
//   q_i = sum_c Abar_c' q_c - xbar_i - K_i' ubar_i + h_i
//   d_i = Rt_i^{-1} (ubar_i - sum_c B_c' q_c - g_i)
// because sum_c Abar_c' P_c B_c = -K_i' exactly (K_i = -Rt_i^{-1} sum B'PA,
// Rt_i = I + sum B'PB); the d-dependence of q cancels.  One warp per node
// then needs only [Abar_c B_c]' of its own block plus K_i, Rt_i^{-1} of the
// parent, and P never has to be read per iteration.
#include <cuda_runtime.h>

#include <cstdio>

#include "dev.cuh"
#include "kernels.hpp"
#include "loop_ctl.cuh"

namespace spock {

namespace {

__device__ __forceinline__ int s_index(const Dev& D, int node) { return node == 0 ? 0 : D.s_base + node - 1; }

// Translated SOC projection of v = (head rows in acc (p of them), vp, vp1):
// the cone head is rows 0..p (p+1 entries), the axis is vp1 (layout:
// [head; tau/2 row; tau/2 row]).  proj_soc_inplace, projections.cpp:11-24.
__device__ __forceinline__ void soc_project(double (&v)[kMaxR], int p, double& vp, double& vp1,
                                            const double* __restrict__ a) {
  const int l = lane_id();
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < kMaxR; ++k) {
    const int r = l + 32 * k;
    if (k * 32 < p && r < p) {
      v[k] -= a[r];
      s += v[k] * v[k];
    }
  }
  vp -= a[p];
  vp1 -= a[p + 1];
  s = warp_sum(s) + vp * vp;
  const double hn = sqrt(s), t = vp1;
  if (hn <= t) {
    // inside the cone: unchanged
  } else if (hn <= -t) {
#pragma unroll
    for (int k = 0; k < kMaxR; ++k) v[k] = 0.0;
    vp = 0.0;
    vp1 = 0.0;
  } else {
    const double f = (hn + t) / (2.0 * hn);
#pragma unroll
    for (int k = 0; k < kMaxR; ++k) v[k] *= f;
    vp *= f;
    vp1 = 0.5 * (hn + t);
  }
#pragma unroll
  for (int k = 0; k < kMaxR; ++k) {
    const int r = l + 32 * k;
    if (k * 32 < p && r < p) v[k] += a[r];
  }
  vp += a[p];
  vp1 += a[p + 1];
}

// Dual-cone projection of the y-copy rows of node i, in place on t[0..ny)
// (proj_cone_inplace, projections.cpp:39-57, over dual_cone(K_i)).
__device__ void ycone_project(const Dev& D, int i, double* t, int ny) {
  const int l = lane_id();
  const int nn = D.yc_nonneg[i];
  if (nn >= 0) {  // AV@R forms: leading orthant rows, remaining rows free
    for (int r = l; r < nn; r += 32) t[r] = fmax(t[r], 0.0);
    return;
  }
  int off = 0;
  for (int pi = D.yc_poff[i]; pi < D.yc_poff[i + 1]; ++pi) {
    const int kind = D.yc_kind[pi], dim = D.yc_dim[pi];
    if (kind == 0) {  // Zero
      for (int r = l; r < dim; r += 32) t[off + r] = 0.0;
    } else if (kind == 1) {  // NonnegOrthant
      for (int r = l; r < dim; r += 32) t[off + r] = fmax(t[off + r], 0.0);
    } else if (kind == 2) {  // SOC, axis last
      double s = 0.0;
      for (int r = l; r < dim - 1; r += 32) s += t[off + r] * t[off + r];
      const double hn = sqrt(warp_sum(s));
      const double tt = t[off + dim - 1];
      __syncwarp();
      if (hn <= tt) {
      } else if (hn <= -tt) {
        for (int r = l; r < dim; r += 32) t[off + r] = 0.0;
      } else {
        const double f = (hn + tt) / (2.0 * hn);
        for (int r = l; r < dim - 1; r += 32) t[off + r] *= f;
        if (l == 0) t[off + dim - 1] = 0.5 * (hn + tt);
      }
    }
    __syncwarp();
    off += dim;
  }
}

// ---------------------------------------------------------------------------
// L* part 1: per non-root child c, adj_c = H_c' head_c - rsum/2 qk_c and the
// tau slot (tree_operator.cpp:80-88).
__device__ __forceinline__ void lt_child_body(const Dev& D, int k, const double* __restrict__ eta, const double* __restrict__ zin, double* __restrict__ zout, double a, double b, double* __restrict__ xs) {
  const int l = lane_id();
  const int px = D.px[k], pu = D.pu[k], p = px + pu;
  const double* seg = eta + D.s2_off[k];
  for (int r = l; r < p; r += 32) xs[r] = seg[r];
  const double rsum = seg[p] + seg[p + 1];
  __syncwarp();
  const double* qk = D.qk + size_t(k) * (D.nx + D.nu);
  double* adj = D.adj + size_t(k) * (D.nx + D.nu);
  double acc[kMaxR];
#pragma unroll
  for (int kk = 0; kk < kMaxR; ++kk) {
    const int r = l + 32 * kk;
    acc[kk] = (r < D.nx) ? -0.5 * rsum * qk[r] : 0.0;
  }
  warp_gemv(D.HxT + D.hx_off[k], D.nx, px, D.nx, xs, acc);
#pragma unroll
  for (int kk = 0; kk < kMaxR; ++kk) {
    const int r = l + 32 * kk;
    if (r < D.nx) adj[r] = acc[kk];
  }
#pragma unroll
  for (int kk = 0; kk < kMaxR; ++kk) {
    const int r = l + 32 * kk;
    acc[kk] = (r < D.nu) ? -0.5 * rsum * qk[D.nx + r] : 0.0;
  }
  warp_gemv(D.HuT + D.hu_off[k], D.nu, pu, D.nu, xs + px, acc);
#pragma unroll
  for (int kk = 0; kk < kMaxR; ++kk) {
    const int r = l + 32 * kk;
    if (r < D.nu) adj[D.nx + r] = acc[kk];
  }
  if (l == 0) {
    const int ti = D.tau_base + k;
    const double lt = 0.5 * rsum;
    zout[ti] = (a == 0.0 ? 0.0 : a * zin[ti]) + b * lt;
  }
}

__global__ void __launch_bounds__(32 * kWarps) k_Lt_child(Dev D, const double* __restrict__ eta,
                                                         const double* __restrict__ zin, double* __restrict__ zout,
                                                         double a, double b) {
  __shared__ double sh[kWarps][kMaxD];
  const int w = threadIdx.x >> 5;
  const int k = blockIdx.x * kWarps + w;
  if (k >= D.nr) return;
  lt_child_body(D, k, eta, zin, zout, a, b, sh[w]);
}

// L* part 2: per node, own segments + ascending sum of the children's adj
// (tree_operator.cpp:75-79,89-113).  zout = a*zin + b*L*eta (+c0 at s0).
__device__ __forceinline__ void lt_node_body(const Dev& D, int i, const double* __restrict__ eta, const double* __restrict__ zin, double* __restrict__ zout, double a, double b, double c0, double* __restrict__ xs) {
  const int l = lane_id();
  const int nx = D.nx, nu = D.nu;
  auto emit = [&](int idx, double lt) { zout[idx] = (a == 0.0 ? 0.0 : a * zin[idx]) + b * lt; };
  double acc[kMaxR];
  if (i < D.nnl) {
    const int ny = D.y_dim[i], yo = D.y_off[i], so = D.s1_off[i];
    const double sc = eta[so + ny];
    const double* rb = D.rb + (yo - D.y_base);
    for (int r = l; r < ny; r += 32) emit(yo + r, eta[so + r] - sc * rb[r]);
    const int nc = D.s1_nc[i];
    const double* ec = eta + so + ny + 1;
    if (l == 0) {
      const int si = s_index(D, i);
      double v = (a == 0.0 ? 0.0 : a * zin[si]) + b * sc;
      if (i == 0) v += c0;
      zout[si] = v;
    }
    // x part
    zero_acc(acc);
    if (D.g_diag) {
      const double* gd = D.gd + size_t(i) * (nx + nu);
#pragma unroll
      for (int k = 0; k < kMaxR; ++k) {
        const int r = l + 32 * k;
        if (r < nx) acc[k] = gd[r] * ec[r];
      }
    } else {
      for (int r = l; r < nc; r += 32) xs[r] = ec[r];
      __syncwarp();
      warp_gemv(D.GxT + D.g_off[i] * nx, nx, nc, nx, xs, acc);
    }
    const int c0i = D.cf[i], nch = D.cc[i];
    for (int c = 0; c < nch; ++c) {
      const double* ad = D.adj + size_t(c0i + c - 1) * (nx + nu);
#pragma unroll
      for (int k = 0; k < kMaxR; ++k) {
        const int r = l + 32 * k;
        if (r < nx) acc[k] += ad[r];
      }
    }
#pragma unroll
    for (int k = 0; k < kMaxR; ++k) {
      const int r = l + 32 * k;
      if (r < nx) emit(1 + i * nx + r, acc[k]);
    }
    // u part
    zero_acc(acc);
    if (D.g_diag) {
      const double* gd = D.gd + size_t(i) * (nx + nu);
#pragma unroll
      for (int k = 0; k < kMaxR; ++k) {
        const int r = l + 32 * k;
        if (r < nu) acc[k] = gd[nx + r] * ec[nx + r];
      }
    } else {
      warp_gemv(D.GuT + D.g_off[i] * nu, nu, nc, nu, xs, acc);
    }
    for (int c = 0; c < nch; ++c) {
      const double* ad = D.adj + size_t(c0i + c - 1) * (nx + nu) + nx;
#pragma unroll
      for (int k = 0; k < kMaxR; ++k) {
        const int r = l + 32 * k;
        if (r < nu) acc[k] += ad[r];
      }
    }
#pragma unroll
    for (int k = 0; k < kMaxR; ++k) {
      const int r = l + 32 * k;
      if (r < nu) emit(D.u_base + i * nu + r, acc[k]);
    }
  } else {
    const int j = i - D.nnl;
    const int nc = D.s3_nc[j], p = D.pN[j];
    const double* ec = eta + D.s3_off[j];
    const double* hd = ec + nc;
    const double rsum = hd[p] + hd[p + 1];
    zero_acc(acc);
    if (D.gN_diag) {
      const double* gd = D.gNd + size_t(j) * nx;
#pragma unroll
      for (int k = 0; k < kMaxR; ++k) {
        const int r = l + 32 * k;
        if (r < nx) acc[k] = gd[r] * ec[r];
      }
    } else {
      for (int r = l; r < nc; r += 32) xs[r] = ec[r];
      __syncwarp();
      warp_gemv(D.GNT + D.gN_off[j] * nx, nx, nc, nx, xs, acc);
      __syncwarp();
    }
    for (int r = l; r < p; r += 32) xs[r] = hd[r];
    __syncwarp();
    warp_gemv(D.HNT + D.hn_off[j], nx, p, nx, xs, acc);
    const double* qk = D.qkN + size_t(j) * nx;
#pragma unroll
    for (int k = 0; k < kMaxR; ++k) {
      const int r = l + 32 * k;
      if (r < nx) emit(1 + i * nx + r, acc[k] - 0.5 * rsum * qk[r]);
    }
    if (l == 0) emit(D.s_base + i - 1, 0.5 * rsum);
  }
}

__global__ void __launch_bounds__(32 * kWarps) k_Lt_node(Dev D, const double* __restrict__ eta,
                                                        const double* __restrict__ zin, double* __restrict__ zout,
                                                        double a, double b, double c0) {
  __shared__ double sh[kWarps][kMaxD];
  const int w = threadIdx.x >> 5;
  const int i = blockIdx.x * kWarps + w;
  if (i >= D.nn) return;
  lt_node_body(D, i, eta, zin, zout, a, b, c0, sh[w]);
}

// ---------------------------------------------------------------------------
// L applied to w = a1*z1 + a2*z2.  PLAIN: eta_out = L w.  DUAL: the CP dual
// half with the S3 projection fused: p = eta + alpha L w, eta_out =
// p - alpha Pi_S3(p/alpha)  (solver.cpp:159-163).
template <bool DUAL>
__device__ __forceinline__ void L_node_body(const Dev& D, int i, const double* __restrict__ z1, double a1, const double* __restrict__ z2, double a2, const double* __restrict__ eta_in, double* __restrict__ eta_out, double alpha, double* __restrict__ xs) {
  const int l = lane_id();
  const int nx = D.nx, nu = D.nu;
  auto W = [&](int idx) { return z2 ? a1 * z1[idx] + a2 * z2[idx] : a1 * z1[idx]; };
  auto fin = [&](int idx, double val) -> double {  // before projection
    return DUAL ? eta_in[idx] + alpha * val : val;
  };
  double acc[kMaxR];
  if (i < D.nnl) {
    const int ny = D.y_dim[i], yo = D.y_off[i], so = D.s1_off[i];
    const double* rb = D.rb + (yo - D.y_base);
    // y-copy rows and the risk scalar s - b'y
    double part = 0.0;
    for (int r = l; r < ny; r += 32) {
      const double yv = W(yo + r);
      part += rb[r] * yv;
      const double pv = fin(so + r, yv);
      if (DUAL)
        eta_out[so + r] = pv / alpha;  // staged: projected below
      else
        eta_out[so + r] = pv;
    }
    const double by = warp_sum(part);
    if (DUAL) {
      __syncwarp();
      ycone_project(D, i, eta_out + so, ny);
      __syncwarp();
      for (int r = l; r < ny; r += 32) {
        const double pv = eta_in[so + r] + alpha * W(yo + r);
        eta_out[so + r] = pv - alpha * eta_out[so + r];
      }
    }
    if (l == 0) {
      const double sv = W(s_index(D, i)) - by;
      const double pv = fin(so + ny, sv);
      eta_out[so + ny] = DUAL ? pv - alpha * fmax(0.0, pv / alpha) : pv;
    }
    // constraint rows Gx x + Gu u
    const int nc = D.s1_nc[i];
    for (int r = l; r < nx; r += 32) xs[r] = W(1 + i * nx + r);
    for (int r = l; r < nu; r += 32) xs[nx + r] = W(D.u_base + i * nu + r);
    __syncwarp();
    zero_acc(acc);
    if (D.g_diag) {
      const double* gd = D.gd + size_t(i) * (nx + nu);
#pragma unroll
      for (int k = 0; k < kMaxR; ++k) {
        const int r = l + 32 * k;
        if (r < nc) acc[k] = gd[r] * xs[r];
      }
    } else {
      warp_gemv(D.Gx + D.g_off[i] * nx, nc, nx, nc, xs, acc);
      warp_gemv(D.Gu + D.g_off[i] * nu, nc, nu, nc, xs + nx, acc);
    }
    const double* lo = D.lo + D.g_off[i];
    const double* hi = D.hi + D.g_off[i];
    const int co = so + ny + 1;
#pragma unroll
    for (int k = 0; k < kMaxR; ++k) {
      const int r = l + 32 * k;
      if (r < nc) {
        const double pv = fin(co + r, acc[k]);
        eta_out[co + r] = DUAL ? pv - alpha * fmin(fmax(pv / alpha, lo[r]), hi[r]) : pv;
      }
    }
    __syncwarp();
  }
  if (i > 0) {  // stage-cost SOC block of (x_anc, u_anc, tau_i)
    const int k = i - 1, an = D.anc[i];
    const int px = D.px[k], pu = D.pu[k], p = px + pu;
    for (int r = l; r < nx; r += 32) xs[r] = W(1 + an * nx + r);
    for (int r = l; r < nu; r += 32) xs[nx + r] = W(D.u_base + an * nu + r);
    __syncwarp();
    const double* qk = D.qk + size_t(k) * (nx + nu);
    double part = 0.0;
    for (int r = l; r < nx + nu; r += 32) part += qk[r] * xs[r];
    const double qd = warp_sum(part);
    const double row = 0.5 * W(D.tau_base + k) - 0.5 * qd;
    zero_acc(acc);
    // rows [0, px): Hx x ; rows [px, p): Hu u -- gathered per lane
    double accx[kMaxR], accu[kMaxR];
    zero_acc(accx);
    zero_acc(accu);
    warp_gemv(D.Hx + D.hx_off[k], px, nx, px, xs, accx);
    warp_gemv(D.Hu + D.hu_off[k], pu, nu, pu, xs + nx, accu);
    const int so = D.s2_off[k];
    __syncwarp();
    // stage through shared memory to realign the u rows after the x rows
#pragma unroll
    for (int kk = 0; kk < kMaxR; ++kk) {
      const int r = l + 32 * kk;
      if (r < px) xs[r] = accx[kk];
    }
#pragma unroll
    for (int kk = 0; kk < kMaxR; ++kk) {
      const int r = l + 32 * kk;
      if (r < pu) xs[px + r] = accu[kk];
    }
    __syncwarp();
#pragma unroll
    for (int kk = 0; kk < kMaxR; ++kk) {
      const int r = l + 32 * kk;
      acc[kk] = (r < p) ? fin(so + r, xs[r]) : 0.0;
    }
    double vp = fin(so + p, row), vp1 = fin(so + p + 1, row);
    if (DUAL) {
      const double* av = D.a + D.a_off[k];
      double t[kMaxR];
#pragma unroll
      for (int kk = 0; kk < kMaxR; ++kk) t[kk] = acc[kk] / alpha;
      double tp = vp / alpha, tp1 = vp1 / alpha;
      soc_project(t, p, tp, tp1, av);
#pragma unroll
      for (int kk = 0; kk < kMaxR; ++kk) acc[kk] = acc[kk] - alpha * t[kk];
      vp = vp - alpha * tp;
      vp1 = vp1 - alpha * tp1;
    }
#pragma unroll
    for (int kk = 0; kk < kMaxR; ++kk) {
      const int r = l + 32 * kk;
      if (r < p) eta_out[so + r] = acc[kk];
    }
    if (l == 0) {
      eta_out[so + p] = vp;
      eta_out[so + p + 1] = vp1;
    }
    __syncwarp();
  }
  if (i >= D.nnl) {  // leaf: GN x and the terminal SOC block of (x, s)
    const int j = i - D.nnl;
    const int nc = D.s3_nc[j], p = D.pN[j];
    for (int r = l; r < nx; r += 32) xs[r] = W(1 + i * nx + r);
    __syncwarp();
    const int eo = D.s3_off[j];
    zero_acc(acc);
    if (D.gN_diag) {
      const double* gd = D.gNd + size_t(j) * nx;
#pragma unroll
      for (int k = 0; k < kMaxR; ++k) {
        const int r = l + 32 * k;
        if (r < nc) acc[k] = gd[r] * xs[r];
      }
    } else {
      warp_gemv(D.GN + D.gN_off[j] * nx, nc, nx, nc, xs, acc);
    }
    const double* lo = D.loN + D.gN_off[j];
    const double* hi = D.hiN + D.gN_off[j];
#pragma unroll
    for (int k = 0; k < kMaxR; ++k) {
      const int r = l + 32 * k;
      if (r < nc) {
        const double pv = fin(eo + r, acc[k]);
        eta_out[eo + r] = DUAL ? pv - alpha * fmin(fmax(pv / alpha, lo[r]), hi[r]) : pv;
      }
    }
    const double* qk = D.qkN + size_t(j) * nx;
    double part = 0.0;
    for (int r = l; r < nx; r += 32) part += qk[r] * xs[r];
    const double qd = warp_sum(part);
    const double row = 0.5 * W(D.s_base + i - 1) - 0.5 * qd;
    zero_acc(acc);
    warp_gemv(D.HN + D.hn_off[j], p, nx, p, xs, acc);
    const int so = eo + nc;
#pragma unroll
    for (int kk = 0; kk < kMaxR; ++kk) {
      const int r = l + 32 * kk;
      acc[kk] = (r < p) ? fin(so + r, acc[kk]) : 0.0;
    }
    double vp = fin(so + p, row), vp1 = fin(so + p + 1, row);
    if (DUAL) {
      const double* av = D.aN + D.aN_off[j];
      double t[kMaxR];
#pragma unroll
      for (int kk = 0; kk < kMaxR; ++kk) t[kk] = acc[kk] / alpha;
      double tp = vp / alpha, tp1 = vp1 / alpha;
      soc_project(t, p, tp, tp1, av);
#pragma unroll
      for (int kk = 0; kk < kMaxR; ++kk) acc[kk] = acc[kk] - alpha * t[kk];
      vp = vp - alpha * tp;
      vp1 = vp1 - alpha * tp1;
    }
#pragma unroll
    for (int kk = 0; kk < kMaxR; ++kk) {
      const int r = l + 32 * kk;
      if (r < p) eta_out[so + r] = acc[kk];
    }
    if (l == 0) {
      eta_out[so + p] = vp;
      eta_out[so + p + 1] = vp1;
    }
  }
}

template <bool DUAL>
__global__ void __launch_bounds__(32 * kWarps) k_L(Dev D, const double* __restrict__ z1, double a1,
                                                  const double* __restrict__ z2, double a2,
                                                  const double* __restrict__ eta_in, double* __restrict__ eta_out,
                                                  double alpha) {
  __shared__ double sh[kWarps][kMaxD];
  const int w = threadIdx.x >> 5;
  const int i = blockIdx.x * kWarps + w;
  if (i >= D.nn) return;
  L_node_body<DUAL>(D, i, z1, a1, z2, a2, eta_in, eta_out, alpha, sh[w]);
}

// Standalone S3 projection in place (proj_s3, projections.cpp:212-244).
__device__ __forceinline__ void s3_node_body(const Dev& D, int i, double* __restrict__ eta, double* __restrict__ xs) {
  const int l = lane_id();
  double acc[kMaxR];
  if (i < D.nnl) {
    const int ny = D.y_dim[i], so = D.s1_off[i];
    ycone_project(D, i, eta + so, ny);
    if (l == 0) eta[so + ny] = fmax(0.0, eta[so + ny]);
    const int nc = D.s1_nc[i], co = so + ny + 1;
    const double* lo = D.lo + D.g_off[i];
    const double* hi = D.hi + D.g_off[i];
    for (int r = l; r < nc; r += 32) eta[co + r] = fmin(fmax(eta[co + r], lo[r]), hi[r]);
  }
  if (i > 0) {
    const int k = i - 1, p = D.px[k] + D.pu[k], so = D.s2_off[k];
#pragma unroll
    for (int kk = 0; kk < kMaxR; ++kk) {
      const int r = l + 32 * kk;
      acc[kk] = r < p ? eta[so + r] : 0.0;
    }
    double vp = eta[so + p], vp1 = eta[so + p + 1];
    __syncwarp();
    soc_project(acc, p, vp, vp1, D.a + D.a_off[k]);
#pragma unroll
    for (int kk = 0; kk < kMaxR; ++kk) {
      const int r = l + 32 * kk;
      if (r < p) eta[so + r] = acc[kk];
    }
    if (l == 0) {
      eta[so + p] = vp;
      eta[so + p + 1] = vp1;
    }
  }
  if (i >= D.nnl) {
    const int j = i - D.nnl, nc = D.s3_nc[j], eo = D.s3_off[j], p = D.pN[j], so = eo + nc;
    const double* lo = D.loN + D.gN_off[j];
    const double* hi = D.hiN + D.gN_off[j];
    for (int r = l; r < nc; r += 32) eta[eo + r] = fmin(fmax(eta[eo + r], lo[r]), hi[r]);
#pragma unroll
    for (int kk = 0; kk < kMaxR; ++kk) {
      const int r = l + 32 * kk;
      acc[kk] = r < p ? eta[so + r] : 0.0;
    }
    double vp = eta[so + p], vp1 = eta[so + p + 1];
    __syncwarp();
    soc_project(acc, p, vp, vp1, D.aN + D.aN_off[j]);
#pragma unroll
    for (int kk = 0; kk < kMaxR; ++kk) {
      const int r = l + 32 * kk;
      if (r < p) eta[so + r] = acc[kk];
    }
    if (l == 0) {
      eta[so + p] = vp;
      eta[so + p + 1] = vp1;
    }
  }
}

__global__ void __launch_bounds__(32 * kWarps) k_s3(Dev D, double* __restrict__ eta) {
  __shared__ double sh[kWarps][kMaxD];
  const int w = threadIdx.x >> 5;
  const int i = blockIdx.x * kWarps + w;
  if (i >= D.nn) return;
  s3_node_body(D, i, eta, sh[w]);
}

// ---------------------------------------------------------------------------
// S1 backward, one launch per stage (nodes [b, e)), in place on z's (x, u).
__device__ __forceinline__ void s1_back_body(const Dev& D, int i, const double* __restrict__ z, double* __restrict__ xs) {
  const int l = lane_id();
  const int nx = D.nx, nu = D.nu;
  double q[kMaxR];
  const double* xb = z + 1 + size_t(i) * nx;
  if (D.cc[i] == 0) {
#pragma unroll
    for (int k = 0; k < kMaxR; ++k) {
      const int r = l + 32 * k;
      q[k] = r < nx ? -xb[r] : 0.0;
    }
  } else {
    const double* ub = z + D.u_base + size_t(i) * nu;
    for (int r = l; r < nu; r += 32) xs[r] = ub[r];
    __syncwarp();
    double t[kMaxR];
    zero_acc(t);
    warp_gemv(D.KT + size_t(i) * D.k_stride, nx, nu, nx, xs, t);  // K' ubar
    const double* h = D.h + size_t(i) * nx;
#pragma unroll
    for (int k = 0; k < kMaxR; ++k) {
      const int r = l + 32 * k;
      q[k] = r < nx ? h[r] - xb[r] - t[k] : 0.0;
    }
    // rhs = ubar - g - sum_c B_c' q_c  (ascending children)
    const double* gv = D.g + size_t(i) * nu;
    double rhs[kMaxR];
#pragma unroll
    for (int k = 0; k < kMaxR; ++k) {
      const int r = l + 32 * k;
      rhs[k] = r < nu ? xs[r] - gv[r] : 0.0;
    }
    const int c0 = D.cf[i], nch = D.cc[i];
    for (int c = 0; c < nch; ++c) {
      const double* T = D.T12 + size_t(c0 + c - 1) * (nx + nu);
#pragma unroll
      for (int k = 0; k < kMaxR; ++k) {
        const int r = l + 32 * k;
        if (r < nx) q[k] += T[r];
        if (r < nu) rhs[k] -= T[nx + r];
      }
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < kMaxR; ++k) {
      const int r = l + 32 * k;
      if (r < nu) xs[r] = rhs[k];
    }
    __syncwarp();
    zero_acc(t);
    warp_gemv(D.Rinv + size_t(i) * D.r_stride, nu, nu, nu, xs, t);
    double* dv = D.dvec + size_t(i) * nu;
#pragma unroll
    for (int k = 0; k < kMaxR; ++k) {
      const int r = l + 32 * k;
      if (r < nu) dv[r] = t[k];
    }
    __syncwarp();
  }
  if (i > 0) {
#pragma unroll
    for (int k = 0; k < kMaxR; ++k) {
      const int r = l + 32 * k;
      if (r < nx) xs[r] = q[k];
    }
    __syncwarp();
    double t[kMaxR];
    zero_acc(t);
    warp_gemv(D.M1T + size_t(i - 1) * D.m1_stride, nx + nu, nx, nx + nu, xs, t);
    double* T = D.T12 + size_t(i - 1) * (nx + nu);
#pragma unroll
    for (int k = 0; k < kMaxR; ++k) {
      const int r = l + 32 * k;
      if (r < nx + nu) T[r] = t[k];
    }
  }
}

__global__ void __launch_bounds__(32 * kWarps) k_s1_back(Dev D, int b, int e, const double* __restrict__ z) {
  __shared__ double sh[kWarps][kMaxD];
  const int w = threadIdx.x >> 5;
  const int i = b + blockIdx.x * kWarps + w;
  if (i >= e) return;
  s1_back_body(D, i, z, sh[w]);
}

// S1 forward, one launch per stage: x_c = [Abar B][x_anc; d_anc] + c_c,
// u_c = K_c x_c + d_c (projections.cpp:176-186).
__device__ __forceinline__ void s1_fwd_body(const Dev& D, int i, double* __restrict__ z, double* __restrict__ xs) {
  const int l = lane_id();
  const int nx = D.nx, nu = D.nu;
  double x[kMaxR];
  if (i == 0) {
#pragma unroll
    for (int k = 0; k < kMaxR; ++k) {
      const int r = l + 32 * k;
      x[k] = r < nx ? D.xinit[r] : 0.0;
    }
  } else {
    const int an = D.anc[i];
    for (int r = l; r < nx; r += 32) xs[r] = z[1 + size_t(an) * nx + r];
    for (int r = l; r < nu; r += 32) xs[nx + r] = D.dvec[size_t(an) * nu + r];
    __syncwarp();
    const double* cv = D.cvec + size_t(i - 1) * nx;
#pragma unroll
    for (int k = 0; k < kMaxR; ++k) {
      const int r = l + 32 * k;
      x[k] = 0.0;
      (void)r;
    }
    warp_gemv(D.M1 + size_t(i - 1) * D.m1_stride, nx, nx + nu, nx, xs, x);
#pragma unroll
    for (int k = 0; k < kMaxR; ++k) {
      const int r = l + 32 * k;
      if (r < nx) x[k] += cv[r];
    }
  }
#pragma unroll
  for (int k = 0; k < kMaxR; ++k) {
    const int r = l + 32 * k;
    if (r < nx) z[1 + size_t(i) * nx + r] = x[k];
  }
  if (D.cc[i] > 0) {
    __syncwarp();
#pragma unroll
    for (int k = 0; k < kMaxR; ++k) {
      const int r = l + 32 * k;
      if (r < nx) xs[r] = x[k];
    }
    __syncwarp();
    double u[kMaxR];
    zero_acc(u);
    warp_gemv(D.K + size_t(i) * D.k_stride, nu, nx, nu, xs, u);
    const double* dv = D.dvec + size_t(i) * nu;
#pragma unroll
    for (int k = 0; k < kMaxR; ++k) {
      const int r = l + 32 * k;
      if (r < nu) z[D.u_base + size_t(i) * nu + r] = u[k] + dv[r];
    }
  }
}

__global__ void __launch_bounds__(32 * kWarps) k_s1_fwd(Dev D, int b, int e, double* __restrict__ z) {
  __shared__ double sh[kWarps][kMaxD];
  const int w = threadIdx.x >> 5;
  const int i = b + blockIdx.x * kWarps + w;
  if (i >= e) return;
  s1_fwd_body(D, i, z, sh[w]);
}

// ---------------------------------------------------------------------------
// S2: projection of (y_i, tau_[i], s_[i]) onto ker [E' -I -I] per non-leaf.
__device__ __forceinline__ void s2_node_body(const Dev& D, int i, double* __restrict__ z, double* __restrict__ xs) {
  const int l = lane_id();
  const int n = D.cc[i], c0 = D.cf[i], ny = D.y_dim[i];
  double* y = z + D.y_off[i];
  double* tau = z + D.tau_base + (c0 - 1);
  double* s = z + D.s_base + (c0 - 1);  // children are non-root
  const int kind = D.s2_kind[i];
  if (kind == S2_DENSE) {
    const int dim = ny + 2 * n;
    for (int r = l; r < ny; r += 32) xs[r] = y[r];
    for (int r = l; r < n; r += 32) {
      xs[ny + r] = tau[r];
      xs[ny + n + r] = s[r];
    }
    __syncwarp();
    double acc[kMaxR];
    zero_acc(acc);
    warp_gemv(D.s2P + D.s2p_off[i], dim, dim, dim, xs, acc);
#pragma unroll
    for (int k = 0; k < kMaxR; ++k) {
      const int r = l + 32 * k;
      if (r < ny)
        y[r] = acc[k];
      else if (r < ny + n)
        tau[r - ny] = acc[k];
      else if (r < dim)
        s[r - ny - n] = acc[k];
    }
    return;
  }
  const double gam = D.s2_gamma[i];
  double A, Bc;
  if (kind == S2_AVAR) {
    A = gam * gam + 3.0;
    Bc = 1.0;
  } else if (kind == S2_MAX) {
    A = 3.0;
    Bc = 1.0;
  } else {
    A = 3.0;
    Bc = 0.0;
  }
  const double ylast = kind == S2_AVAR ? y[2 * n] : (kind == S2_MAX ? y[n] : 0.0);
  auto ety = [&](int k) -> double {
    if (kind == S2_AVAR) return gam * y[k] - y[n + k] + ylast;
    if (kind == S2_MAX) return -y[k] + ylast;
    return y[k];
  };
  double part = 0.0;
  for (int k = l; k < n; k += 32) part += ety(k) - tau[k] - s[k];
  const double S = warp_sum(part);
  const double den = A + Bc * n;
  const double shift = Bc * S / den;
  for (int k = l; k < n; k += 32) {
    const double v = ety(k) - tau[k] - s[k];
    const double lam = (v - shift) / A;
    if (kind == S2_AVAR) {
      y[k] -= gam * lam;
      y[n + k] += lam;
    } else if (kind == S2_MAX) {
      y[k] += lam;
    } else {
      y[k] -= lam;
    }
    tau[k] += lam;
    s[k] += lam;
  }
  __syncwarp();
  if (l == 0 && kind != S2_EQ) {
    const double lsum = S / den;  // sum_k lambda_k
    if (kind == S2_AVAR)
      y[2 * n] = ylast - lsum;
    else
      y[n] = ylast - lsum;
  }
}

__global__ void __launch_bounds__(32 * kWarps) k_s2(Dev D, double* __restrict__ z) {
  __shared__ double sh[kWarps][kMaxD];
  const int w = threadIdx.x >> 5;
  const int i = blockIdx.x * kWarps + w;
  if (i >= D.nnl) return;
  s2_node_body(D, i, z, sh[w]);
}

// ---------------------------------------------------------------------------
// Vector kernels.
__global__ void k_axpby(int n, double a, const double* __restrict__ x, double b, const double* __restrict__ y,
                        double* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = y ? a * x[i] + b * y[i] : a * x[i];
}

// out = c0*x0 + sum_j c_j x_j (j < nv <= 16)
__global__ void k_lincomb(int n, int nv, LinCombArgs A, double* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double s = A.c[0] * A.x[0][i];
    for (int j = 1; j < nv; ++j) s += A.c[j] * A.x[j][i];
    out[i] = s;
  }
}

__global__ void k_gather(int n, const int* __restrict__ perm, const double* __restrict__ src,
                         double* __restrict__ dst) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[i] = src[perm[i]];
}
__global__ void k_scatter(int n, const int* __restrict__ perm, const double* __restrict__ src,
                          double* __restrict__ dst) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[perm[i]] = src[i];
}

// Deterministic multi-dot: block partials over a fixed grid, then one block
// sums them in index order.
__global__ void __launch_bounds__(kRedThreads) k_dots(DotArgs A, double* __restrict__ partial, double* out) {
  __shared__ double sm[kMaxDots][kRedThreads / 32];
  double acc[kMaxDots];
#pragma unroll
  for (int j = 0; j < kMaxDots; ++j) acc[j] = 0.0;
  const int stride = gridDim.x * blockDim.x;
  for (int j = 0; j < A.ndots; ++j) {
    const double* x = A.x[j];
    const double* y = A.y[j];
    const double* w = A.w[j];
    const int n = A.n[j];
    double s = 0.0;
    if (w) {  // entries with weight 0 may hold anything (another rank computes them): skipped, not multiplied
      for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        if (w[i] != 0.0) s += x[i] * y[i];
      }
    } else {
      for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) s += x[i] * y[i];
    }
    acc[j] = s;
  }
  const int w = threadIdx.x >> 5;
  for (int j = 0; j < A.ndots; ++j) {
    const double v = warp_sum(acc[j]);
    if ((threadIdx.x & 31) == 0) sm[j][w] = v;
  }
  __syncthreads();
  if (threadIdx.x < A.ndots) {
    double s = 0.0;
    for (int k = 0; k < kRedThreads / 32; ++k) s += sm[threadIdx.x][k];
    partial[size_t(threadIdx.x) * gridDim.x + blockIdx.x] = s;
  }
  grid_finalize<false>(partial, A.ndots, out, red_counter(partial));
}

// xi infinity norms: max_i |(x_i / alpha - y_i) * d_i| for two (x, y, d)
// triples; NaN flagged through a separate count.
__global__ void __launch_bounds__(kRedThreads) k_xi(XiArgs A, double* __restrict__ partial, double* out) {
  __shared__ double sm[2][kRedThreads / 32];
  __shared__ int nanflag;
  if (threadIdx.x == 0) nanflag = 0;
  __syncthreads();
  double m[2] = {0.0, 0.0};
  bool bad = false;
  const int stride = gridDim.x * blockDim.x;
  for (int t = 0; t < 2; ++t) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < A.n[t]; i += stride) {
      if (A.w[t] && A.w[t][i] == 0.0) continue;
      double v = A.x[t][i] / A.alpha - A.y[t][i];
      if (A.d[t]) v *= A.d[t][i];
      if (isnan(v)) bad = true;
      m[t] = fmax(m[t], fabs(v));
    }
  }
  if (bad) atomicExch(&nanflag, 1);
  const int w = threadIdx.x >> 5;
  for (int t = 0; t < 2; ++t) {
    const double v = warp_max(m[t]);
    if ((threadIdx.x & 31) == 0) sm[t][w] = v;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double s = 0.0;
    for (int k = 0; k < kRedThreads / 32; ++k) s = fmax(s, sm[threadIdx.x][k]);
    partial[size_t(threadIdx.x) * gridDim.x + blockIdx.x] = nanflag ? NAN : s;
  }
  grid_finalize<true>(partial, 2, out, red_counter(partial));
}

// ---------------------------------------------------------------------------
// Offline factorisation helpers (Alg. 1), one CTA per batch item.
// C = alpha * op(A) op(B) + beta * C with A m x k, B k x n (after op).
__global__ void k_bgemm(BGemmArgs G) {
  const int b = blockIdx.x;
  const double* A = G.A[b];
  const double* B = G.B[b];
  double* C = G.C[b];
  const int m = G.m, n = G.n, k = G.k;
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
    const int i = e % m, j = e / m;
    double s = 0.0;
    for (int t = 0; t < k; ++t) {
      const double a = G.ta ? A[t + size_t(i) * G.lda] : A[i + size_t(t) * G.lda];
      const double bb = G.tb ? B[j + size_t(t) * G.ldb] : B[t + size_t(j) * G.ldb];
      s = fma(a, bb, s);
    }
    C[i + size_t(j) * G.ldc] = G.alpha * s + (G.beta == 0.0 ? 0.0 : G.beta * C[i + size_t(j) * G.ldc]);
  }
}

// Parent step of Alg. 1: Rt = I + sum_c rt_c (ascending), Cholesky (error flag
// on failure, projections.cpp:96-98), Rinv = Rt^{-1}, K = -Rinv sum_c kt_c,
// g = sum_c ge_c.  One CTA per parent; nu <= 128.
__global__ void k_alg1_parent(Alg1Args P) {
  extern __shared__ double smem[];
  const int i = P.b + blockIdx.x;
  const int nu = P.nu, nx = P.nx;
  double* L = smem;              // nu x nu
  double* Ri = smem + nu * nu;   // nu x nu
  double* kt = Ri + nu * nu;     // nu x nx
  const int c0 = P.cf[i], nch = P.cc[i];
  for (int e = threadIdx.x; e < nu * nu; e += blockDim.x) {
    const int r = e % nu, c = e / nu;
    double s = (r == c) ? 1.0 : 0.0;
    for (int ch = 0; ch < nch; ++ch) s += P.rt[size_t(c0 + ch - 1) * nu * nu + e];
    L[e] = s;
    if (P.Rt_out) P.Rt_out[size_t(i) * nu * nu + e] = s;
  }
  for (int e = threadIdx.x; e < nu * nx; e += blockDim.x) {
    double s = 0.0;
    for (int ch = 0; ch < nch; ++ch) s += P.kt[size_t(c0 + ch - 1) * nu * nx + e];
    kt[e] = s;
  }
  for (int e = threadIdx.x; e < nu; e += blockDim.x) {
    double s = 0.0;
    for (int ch = 0; ch < nch; ++ch) s += P.ge[size_t(c0 + ch - 1) * nu + e];
    P.g[size_t(i) * nu + e] = s;
  }
  __syncthreads();
  // right-looking Cholesky in shared memory (lower)
  for (int j = 0; j < nu; ++j) {
    __shared__ double piv;
    if (threadIdx.x == 0) {
      const double d = L[j + j * nu];
      if (!(d > 0.0)) {
        *P.err = 1;
        piv = 1.0;
      } else {
        piv = sqrt(d);
      }
      L[j + j * nu] = piv;
    }
    __syncthreads();
    for (int r = j + 1 + threadIdx.x; r < nu; r += blockDim.x) L[r + j * nu] /= piv;
    __syncthreads();
    for (int e = threadIdx.x; e < (nu - j - 1) * (nu - j - 1); e += blockDim.x) {
      const int r = j + 1 + e % (nu - j - 1), c = j + 1 + e / (nu - j - 1);
      if (r >= c) L[r + c * nu] -= L[r + j * nu] * L[c + j * nu];
    }
    __syncthreads();
  }
  // inverse: solve L L' X = I, one column per thread
  for (int c = threadIdx.x; c < nu; c += blockDim.x) {
    for (int r = 0; r < nu; ++r) {
      double s = (r == c) ? 1.0 : 0.0;
      for (int t = 0; t < r; ++t) s -= L[r + t * nu] * Ri[t + c * nu];
      Ri[r + c * nu] = s / L[r + r * nu];
    }
    for (int r = nu - 1; r >= 0; --r) {
      double s = Ri[r + c * nu];
      for (int t = r + 1; t < nu; ++t) s -= L[t + r * nu] * Ri[t + c * nu];
      Ri[r + c * nu] = s / L[r + r * nu];
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nu * nu; e += blockDim.x) P.Rinv[size_t(i) * P.r_stride + e] = Ri[e];
  // K = -Rinv kt (nu x nx), stored as K (nu x nx) and K' (nx x nu)
  for (int e = threadIdx.x; e < nu * nx; e += blockDim.x) {
    const int r = e % nu, c = e / nu;
    double s = 0.0;
    for (int t = 0; t < nu; ++t) s += Ri[r + t * nu] * kt[t + c * nu];
    P.K[size_t(i) * P.k_stride + e] = -s;
    P.KT[size_t(i) * P.k_stride + c + size_t(r) * nx] = -s;
  }
}

// Parent step 2: P_i = I + K'K + sum_c pt_c ; h_i = sum_c he_c.
__global__ void k_alg1_parent2(Alg1Args P) {
  const int i = P.b + blockIdx.x;
  const int nu = P.nu, nx = P.nx;
  const int c0 = P.cf[i], nch = P.cc[i];
  const double* K = P.K + size_t(i) * P.k_stride;
  for (int e = threadIdx.x; e < nx * nx; e += blockDim.x) {
    const int r = e % nx, c = e / nx;
    double s = (r == c) ? 1.0 : 0.0;
    double kk = 0.0;
    for (int t = 0; t < nu; ++t) kk += K[t + r * nu] * K[t + c * nu];
    s += kk;
    for (int ch = 0; ch < nch; ++ch) s += P.pt[size_t(c0 + ch - 1) * nx * nx + e];
    P.P[size_t(i) * nx * nx + e] = s;
  }
  for (int e = threadIdx.x; e < nx; e += blockDim.x) {
    double s = 0.0;
    for (int ch = 0; ch < nch; ++ch) s += P.he[size_t(c0 + ch - 1) * nx + e];
    P.h[size_t(i) * nx + e] = s;
  }
}

// Child step: Abar = A + B K_anc written into M1 = [Abar B] and M1' ; e = P c
__global__ void k_alg1_child_abar(Alg1Args P) {
  const int c = P.b + blockIdx.x;  // node
  const int k = c - 1, nx = P.nx, nu = P.nu, an = P.anc[c];
  const double* A = P.A + size_t(k) * nx * nx;
  const double* B = P.B + size_t(k) * nx * nu;
  const double* K = P.K + size_t(an) * P.k_stride;
  double* M1 = P.M1 + size_t(k) * P.m1_stride;
  double* M1T = P.M1T + size_t(k) * P.m1_stride;
  for (int e = threadIdx.x; e < nx * nx; e += blockDim.x) {
    const int r = e % nx, col = e / nx;
    double s = A[e];
    for (int t = 0; t < nu; ++t) s += B[r + t * nx] * K[t + col * nu];
    M1[e] = s;
    M1T[col + size_t(r) * (nx + nu)] = s;
    if (P.Abar_out) P.Abar_out[size_t(k) * nx * nx + e] = s;
  }
  for (int e = threadIdx.x; e < nx * nu; e += blockDim.x) {
    const int r = e % nx, col = e / nx;
    M1[size_t(nx) * nx + e] = B[e];
    M1T[(nx + col) + size_t(r) * (nx + nu)] = B[e];
  }
}

#include "small.cuh"
#include "cluster.cuh"

}  // namespace

// ===========================================================================
// Launchers
static inline int blocks_for(int n, int per) { return (n + per - 1) / per; }

void launch_Lt(const Dev& D, const double* eta, const double* zin, double* zout, double a, double b, double c0,
               cudaStream_t st) {
  const int T = 32 * kWarps;
  if (D.nr > 0) k_Lt_child<<<blocks_for(D.nr, kWarps), T, 0, st>>>(D, eta, zin, zout, a, b);
  k_Lt_node<<<blocks_for(D.nn, kWarps), T, 0, st>>>(D, eta, zin, zout, a, b, c0);
}

void launch_L(const Dev& D, const double* z1, double a1, const double* z2, double a2, const double* eta_in,
              double* eta_out, double alpha, bool dual, cudaStream_t st) {
  const int T = 32 * kWarps;
  if (dual)
    k_L<true><<<blocks_for(D.nn, kWarps), T, 0, st>>>(D, z1, a1, z2, a2, eta_in, eta_out, alpha);
  else
    k_L<false><<<blocks_for(D.nn, kWarps), T, 0, st>>>(D, z1, a1, z2, a2, eta_in, eta_out, alpha);
}

void launch_s1(const Dev& D, const int* stage_start, double* z, cudaStream_t st) {
  const int T = 32 * kWarps;
  for (int t = D.N; t >= 0; --t) {
    const int b = stage_start[t], e = stage_start[t + 1];
    k_s1_back<<<blocks_for(e - b, kWarps), T, 0, st>>>(D, b, e, z);
  }
  for (int t = 0; t <= D.N; ++t) {
    const int b = stage_start[t], e = stage_start[t + 1];
    k_s1_fwd<<<blocks_for(e - b, kWarps), T, 0, st>>>(D, b, e, z);
  }
}

void launch_s2(const Dev& D, double* z, cudaStream_t st) {
  if (D.nnl > 0) k_s2<<<blocks_for(D.nnl, kWarps), 32 * kWarps, 0, st>>>(D, z);
}

void launch_s3(const Dev& D, double* eta, cudaStream_t st) {
  k_s3<<<blocks_for(D.nn, kWarps), 32 * kWarps, 0, st>>>(D, eta);
}

int cluster_static_smem() {
  cudaFuncAttributes fa{};
  if (cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(&k_cluster_solve)) != cudaSuccess) return 48 * 1024;
  return int(fa.sharedSizeBytes);
}

// attributes are process-wide per function: set once, to the device's opt-in
// maximum, so concurrent solvers with different arenas never lower each
// other's limit between attribute and launch
static cudaError_t cluster_attrs_once() {
  static cudaError_t err = [] {
    const void* fn = reinterpret_cast<const void*>(&k_cluster_solve);
    int dev = 0, optin = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - cluster_static_smem());
    if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    return e;
  }();
  return err;
}

static cudaLaunchConfig_t cluster_cfg(int ctas, int arena_bytes, cudaStream_t st, cudaLaunchAttribute* at) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(kSmallThreads);
  cfg.dynamicSmemBytes = size_t(arena_bytes);
  cfg.stream = st;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = unsigned(ctas);
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cfg;
}

int cluster_max_active(int ctas, int arena_bytes) {
  if (cluster_attrs_once() != cudaSuccess) return 0;
  cudaLaunchAttribute at[1];
  cudaLaunchConfig_t cfg = cluster_cfg(ctas, arena_bytes, nullptr, at);
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, reinterpret_cast<const void*>(&k_cluster_solve), &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

cudaError_t launch_cluster_solve(const ClusterArgs& A, int ctas, int arena_bytes, cudaStream_t st) {
  if (cudaError_t e = cluster_attrs_once(); e != cudaSuccess) return e;
  cudaLaunchAttribute at[1];
  cudaLaunchConfig_t cfg = cluster_cfg(ctas, arena_bytes, st, at);
  return cudaLaunchKernelEx(&cfg, k_cluster_solve, A);
}

void launch_small_solve(const SmallArgs& A, cudaStream_t st) {
  static_assert(kSmallThreads == kSmallThreadsHost, "small solve block size");
  // the per-node blocks are read through L1 every iteration: give the SM's
  // unified L1 / shared memory to L1 (the kernel needs ~22 KB of shared memory)
  static bool once = [] {
    cudaFuncSetAttribute(reinterpret_cast<const void*>(&k_small_solve), cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxL1);
    return true;
  }();
  (void)once;
  k_small_solve<<<1, kSmallThreads, 0, st>>>(A);
}

void launch_axpby(int n, double a, const double* x, double b, const double* y, double* out, cudaStream_t st) {
  k_axpby<<<std::min(blocks_for(n, 256), 4 * 148), 256, 0, st>>>(n, a, x, b, y, out);
}

void launch_lincomb(int n, int nv, const LinCombArgs& A, double* out, cudaStream_t st) {
  k_lincomb<<<std::min(blocks_for(n, 256), 4 * 148), 256, 0, st>>>(n, nv, A, out);
}

void launch_gather(int n, const int* perm, const double* src, double* dst, cudaStream_t st) {
  k_gather<<<std::min(blocks_for(n, 256), 4 * 148), 256, 0, st>>>(n, perm, src, dst);
}
void launch_scatter(int n, const int* perm, const double* src, double* dst, cudaStream_t st) {
  k_scatter<<<std::min(blocks_for(n, 256), 4 * 148), 256, 0, st>>>(n, perm, src, dst);
}

void launch_dots(const DotArgs& A, double* partial, double* out, cudaStream_t st) {
  k_dots<<<kRedBlocks, kRedThreads, 0, st>>>(A, partial, out);
}

void launch_xi(const XiArgs& A, double* partial, double* out, cudaStream_t st) {
  k_xi<<<kRedBlocks, kRedThreads, 0, st>>>(A, partial, out);
}

void launch_bgemm(const BGemmArgs& G, int count, cudaStream_t st) {
  if (count > 0) k_bgemm<<<count, 256, 0, st>>>(G);
}

void launch_alg1_parent(const Alg1Args& P, int count, cudaStream_t st) {
  if (count <= 0) return;
  const size_t sm = sizeof(double) * (2 * P.nu * P.nu + P.nu * P.nx);
  k_alg1_parent<<<count, 128, sm, st>>>(P);
}
void launch_alg1_parent2(const Alg1Args& P, int count, cudaStream_t st) {
  if (count > 0) k_alg1_parent2<<<count, 256, 0, st>>>(P);
}
void launch_alg1_child_abar(const Alg1Args& P, int count, cudaStream_t st) {
  if (count > 0) k_alg1_child_abar<<<count, 256, 0, st>>>(P);
}

// every kernel of the engine prefers the maximum shared-memory carveout (see fused.cu)
void set_carveout_all() {
  const void* fs[] = {
      reinterpret_cast<const void*>(&k_Lt_child), reinterpret_cast<const void*>(&k_Lt_node),
      reinterpret_cast<const void*>(&k_L<true>), reinterpret_cast<const void*>(&k_L<false>),
      reinterpret_cast<const void*>(&k_s3), reinterpret_cast<const void*>(&k_s1_back),
      reinterpret_cast<const void*>(&k_s1_fwd), reinterpret_cast<const void*>(&k_s2),
      reinterpret_cast<const void*>(&k_axpby), reinterpret_cast<const void*>(&k_lincomb),
      reinterpret_cast<const void*>(&k_gather), reinterpret_cast<const void*>(&k_scatter),
      reinterpret_cast<const void*>(&k_dots), reinterpret_cast<const void*>(&k_xi)};
  for (const void* f : fs)
    cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
}

cudaError_t set_alg1_smem(int bytes) {
  return set_smem_limit(reinterpret_cast<const void*>(&k_alg1_parent), bytes);
}

}  // namespace spock
