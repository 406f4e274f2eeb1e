// One CP application T for wide trees as a persistent, warp-granular dataflow
// kernel with per-warp TMA streaming rings (sm_100a).
//
// Same items, order and arithmetic as the CTA-granular kernel of fused.cu
// (backward nn-1..0, S2 of every parent, forward 0..nn-1; an item only waits
// on items with smaller tickets), but sized for trees whose matrices do not fit
// on chip and whose per-T cost is streaming them once from HBM:
//
//  * one item per WARP, tickets assigned round-robin (ticket = warp + k*NW), so
//    the whole schedule of a warp is known in advance and no CTA barrier sits
//    on any path (a warp waits only on its own ring and on dependency flags);
//  * every node matrix streams through a per-warp ring of S shared-memory
//    slots, one cp.async.bulk (TMA bulk copy, mbarrier completion) per column
//    chunk.  Lane 0 runs the producer S chunks ahead of the consumer, across
//    item boundaries and across dependency waits, so HBM sees S*W chunks per
//    SM in flight regardless of what the warps are computing;
//  * lanes own rows (r = lane + 32k), the chunk is read from shared memory
//    column by column with the input vector broadcast: fixed summation order,
//    bitwise run-to-run deterministic.
//
// Reference map (arxiv/paper_2505_12078): backward = L* (tree_operator.cpp:
// 65-114) + the CP primal step (solver.cpp:150-156) + S1 backward sweep
// (projections.cpp:147-174, restructured as in kernels.cu); S2 = proj_s2
// (projections.cpp:189-210, closed form); forward = S1 forward sweep
// (projections.cpp:176-186) + L (tree_operator.cpp:20-63) + S3 and the Moreau
// dual step (projections.cpp:212-244, solver.cpp:157-163).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "dev.cuh"
#include "kernels.hpp"
#include "wide.hpp"

namespace spock {

namespace {

constexpr int kMaxSlots = 8;

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(su32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// data produced by other warps of this launch: L2 only (no stale L1 lines)
__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }

__device__ void wait_flag(const int* f) {
  for (int k = 0; k < 32; ++k)
    if (ld_acquire(f) >= 1) return;
  while (ld_acquire(f) < 1) __nanosleep(64);
}
// warp barrier (orders every lane's writes before lane 0's), then one release
// store by lane 0 (st.release is cumulative over the writes it has observed)
__device__ __forceinline__ void w_release(int* f) {
  __syncwarp();
  if (lane_id() == 0) st_release(f, 1);
}

struct MatD {
  const double* p;
  int rows, cols;
};

// ticket -> (kind, node): 0 backward (node nn-1..0), 1 S2 (parent 0..nnl-1), 2 forward (0..nn-1)
__device__ __forceinline__ void decode(const Dev& D, int tk, int& kind, int& node) {
  if (tk < D.nn) {
    kind = 0;
    node = D.nn - 1 - tk;
  } else if (tk < D.nn + D.nnl) {
    kind = 1;
    node = tk - D.nn;
  } else {
    kind = 2;
    node = tk - D.nn - D.nnl;
  }
}

// The streamed matrices of an item, in the order the item consumes them.
// Producer and consumer both enumerate this list, so it is the one contract
// between them.
__device__ int item_mats(const Dev& D, int kind, int i, MatD* md) {
  int n = 0;
  const int nx = D.nx, nu = D.nu, m = nx + nu;
  const bool root = i == 0, leaf = D.cc[i] == 0;
  if (kind == 0) {
    if (!root) {
      const int k = i - 1;
      md[n++] = {D.HxT + D.hx_off[k], nx, D.px[k]};
      md[n++] = {D.HuT + D.hu_off[k], nu, D.pu[k]};
    }
    if (leaf) {
      const int j = i - D.nnl;
      md[n++] = {D.HNT + D.hn_off[j], nx, D.pN[j]};
    } else {
      md[n++] = {D.KT + size_t(i) * D.k_stride, nx, nu};
      md[n++] = {D.Rinv + size_t(i) * D.r_stride, nu, nu};
    }
    if (!root) md[n++] = {D.M1T + size_t(i - 1) * D.m1_stride, m, nx};
  } else if (kind == 2) {
    if (!root) md[n++] = {D.M1 + size_t(i - 1) * D.m1_stride, nx, m};
    if (!leaf) md[n++] = {D.K + size_t(i) * D.k_stride, nu, nx};
    if (!root) {
      const int k = i - 1;
      md[n++] = {D.Hx + D.hx_off[k], D.px[k], nx};
      md[n++] = {D.Hu + D.hu_off[k], D.pu[k], nu};
    }
    if (leaf) {
      const int j = i - D.nnl;
      md[n++] = {D.HN + D.hn_off[j], D.pN[j], nx};
    }
  }
  return n;
}

__device__ __forceinline__ int chunk_cols(int rows, int chunk) { return max(2, (chunk / rows) & ~1); }

// producer cursor of a warp's ring (shared memory, touched by lane 0 only)
struct Prod {
  uint32_t prod;  // chunks issued
  int tp, mi, co, nm;
  MatD md[6];
};

struct Ring {
  double* buf;
  uint64_t* bar;
  Prod* ps;
  int S, chunk, stride, total;
  uint32_t cons;  // chunks consumed (uniform across the warp)
  long long t_ring, t_flag;  // optional profile: cycles waiting on chunks / dependency flags
};

// lane 0: keep S chunks in flight, walking this warp's tickets ahead of the consumer
__device__ __noinline__ void refill(const Dev& D, Prod* __restrict__ P, uint32_t cons, int S, int chunk,
                                    double* buf, uint64_t* bar, int stride, int total) {
  while (P->prod < cons + uint32_t(S)) {
    for (;;) {
      if (P->tp >= total) return;
      if (P->mi < P->nm) {
        const MatD& M = P->md[P->mi];
        if (M.rows > 0 && P->co < M.cols) break;
        ++P->mi;
        P->co = 0;
        continue;
      }
      P->tp += stride;
      if (P->tp >= total) return;
      int kind, node;
      decode(D, P->tp, kind, node);
      P->nm = item_mats(D, kind, node, P->md);
      P->mi = 0;
      P->co = 0;
    }
    const MatD M = P->md[P->mi];
    const int cc = min(chunk_cols(M.rows, chunk), M.cols - P->co);
    const uint32_t bytes = (uint32_t(cc) * uint32_t(M.rows) * 8u + 15u) & ~15u;
    const int slot = int(P->prod % uint32_t(S));
    fence_proxy_async();
    mbar_expect_tx(&bar[slot], bytes);
    bulk_g2s(buf + size_t(slot) * chunk, M.p + size_t(P->co) * M.rows, bytes, &bar[slot]);
    ++P->prod;
    P->co += cc;
  }
}

// acc[k] += sum_{c < cc} A[(lane + 32k) + c*rows] x[c], A in shared memory
template <int RR>
__device__ __forceinline__ void gemv_cols(const double* A, int rows, int cc, const double* x, double (&acc)[RR]) {
  const int l = lane_id();
  int c = 0;
  for (; c + 4 <= cc; c += 4) {
    const double x0 = x[c], x1 = x[c + 1], x2 = x[c + 2], x3 = x[c + 3];
    const double* a = A + c * rows;
#pragma unroll
    for (int k = 0; k < RR; ++k) {
      const int r = l + 32 * k;
      if (r < rows) {
        acc[k] = fma(a[r], x0, acc[k]);
        acc[k] = fma(a[r + rows], x1, acc[k]);
        acc[k] = fma(a[r + 2 * rows], x2, acc[k]);
        acc[k] = fma(a[r + 3 * rows], x3, acc[k]);
      }
    }
  }
  for (; c < cc; ++c) {
    const double xc = x[c];
    const double* a = A + c * rows;
#pragma unroll
    for (int k = 0; k < RR; ++k) {
      const int r = l + 32 * k;
      if (r < rows) acc[k] = fma(a[r], xc, acc[k]);
    }
  }
}

// consume the chunks of one streamed matrix: acc += M x
template <int RR>
__device__ __forceinline__ void sgemv(const Dev& D, Ring& R, const MatD M, const double* x, double (&acc)[RR]) {
  if (M.rows <= 0) return;
  const int ccmax = chunk_cols(M.rows, R.chunk);
  for (int co = 0; co < M.cols; co += ccmax) {
    const int cc = min(ccmax, M.cols - co);
    const int slot = int(R.cons % uint32_t(R.S));
    const uint32_t par = (R.cons / uint32_t(R.S)) & 1u;
    if (!mbar_try_wait(&R.bar[slot], par)) {
      const long long t0 = clock64();
      while (!mbar_try_wait(&R.bar[slot], par)) {
      }
      R.t_ring += clock64() - t0;
    }
    gemv_cols<RR>(R.buf + size_t(slot) * R.chunk, M.rows, cc, x + co, acc);
    __syncwarp();
    ++R.cons;
    if (lane_id() == 0) refill(D, R.ps, R.cons, R.S, R.chunk, R.buf, R.bar, R.stride, R.total);
  }
}

// acc += A x with A column-major in global memory (dense G / G_N paths)
template <int RR>
__device__ void gemv_glob(const double* __restrict__ A, int m, int n, int lda, const double* x, double (&acc)[RR]) {
  const int l = lane_id();
  for (int c = 0; c < n; ++c) {
    const double xc = x[c];
    const double* col = A + size_t(c) * lda;
#pragma unroll
    for (int k = 0; k < RR; ++k) {
      const int r = l + 32 * k;
      if (r < m) acc[k] = fma(__ldg(col + r), xc, acc[k]);
    }
  }
}

template <int RR>
__device__ __forceinline__ void zero(double (&a)[RR]) {
#pragma unroll
  for (int k = 0; k < RR; ++k) a[k] = 0.0;
}

// translated SOC projection (proj_soc_inplace, projections.cpp:11-24) of
// (v rows < p, vp, vp1) about a; cone head = rows 0..p, axis vp1
template <int RR>
__device__ void soc_proj(double (&v)[RR], int p, double& vp, double& vp1, const double* __restrict__ a) {
  const int l = lane_id();
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < RR; ++k) {
    const int r = l + 32 * k;
    if (r < p) {
      v[k] -= a[r];
      s += v[k] * v[k];
    }
  }
  vp -= a[p];
  vp1 -= a[p + 1];
  s = warp_sum(s) + vp * vp;
  const double hn = sqrt(s), t = vp1;
  if (hn <= t) {
  } else if (hn <= -t) {
#pragma unroll
    for (int k = 0; k < RR; ++k) v[k] = 0.0;
    vp = 0.0;
    vp1 = 0.0;
  } else {
    const double f = (hn + t) / (2.0 * hn);
#pragma unroll
    for (int k = 0; k < RR; ++k) v[k] *= f;
    vp *= f;
    vp1 = 0.5 * (hn + t);
  }
#pragma unroll
  for (int k = 0; k < RR; ++k) {
    const int r = l + 32 * k;
    if (r < p) v[k] += a[r];
  }
  vp += a[p];
  vp1 += a[p + 1];
}

// dual cone of the y-copy rows, in place on t[0..ny) (proj_cone_inplace,
// projections.cpp:39-57)
__device__ void ycone(const Dev& D, int i, double* t) {
  const int l = lane_id();
  const int nn0 = D.yc_nonneg[i];
  if (nn0 >= 0) {
    for (int r = l; r < nn0; r += 32) t[r] = fmax(t[r], 0.0);
    __syncwarp();
    return;
  }
  int off = 0;
  for (int pi = D.yc_poff[i]; pi < D.yc_poff[i + 1]; ++pi) {
    const int kind = D.yc_kind[pi], dim = D.yc_dim[pi];
    if (kind == 0) {
      for (int r = l; r < dim; r += 32) t[off + r] = 0.0;
    } else if (kind == 1) {
      for (int r = l; r < dim; r += 32) t[off + r] = fmax(t[off + r], 0.0);
    } else if (kind == 2) {
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
// Backward item of node i.
template <int RR>
__device__ void w_back(const WideArgs& A, Ring& R, int i, double* xs, double* xs2) {
  const Dev& D = A.D;
  const int l = lane_id(), nx = D.nx, nu = D.nu, m = nx + nu;
  const double al = A.alpha;
  const double* __restrict__ z = A.z;
  const double* __restrict__ eta = A.eta;
  const bool root = i == 0, leaf = D.cc[i] == 0;
  // streamed matrices, consumed in item_mats order:
  //   HxT, HuT (non-root) | HNT (leaf) or KT, Rinv (non-leaf) | M1T (non-root)
  double acc[RR];
  if (!root) {  // own stage-SOC adjoint term for the parent (tree_operator.cpp:80-88)
    const int k = i - 1, px = D.px[k], pu = D.pu[k], p = px + pu;
    const double* seg = eta + D.s2_off[k];
    for (int r = l; r < p; r += 32) xs[r] = seg[r];
    const double rsum = seg[p] + seg[p + 1];
    const double* qk = D.qk + size_t(k) * m;
    double* adj = D.adj + size_t(k) * m;
    __syncwarp();
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      acc[kk] = r < nx ? -0.5 * rsum * qk[r] : 0.0;
    }
    sgemv<RR>(D, R, MatD{D.HxT + D.hx_off[k], nx, px}, xs, acc);
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < nx) adj[r] = acc[kk];
    }
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      acc[kk] = r < nu ? -0.5 * rsum * qk[nx + r] : 0.0;
    }
    sgemv<RR>(D, R, MatD{D.HuT + D.hu_off[k], nu, pu}, xs + px, acc);
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < nu) adj[nx + r] = acc[kk];
    }
    __syncwarp();
  }
  const double* zx = z + 1 + size_t(i) * nx;
  if (leaf) {  // L* leaf rows, then q = -xbar and T12 = M1' q
    const int j = i - D.nnl, nc = D.s3_nc[j], pN = D.pN[j];
    const double* ec = eta + D.s3_off[j];
    const double* hd = ec + nc;
    const double rsumN = hd[pN] + hd[pN + 1];
    zero(acc);
    if (D.gN_diag) {
      const double* gd = D.gNd + size_t(j) * nx;
#pragma unroll
      for (int kk = 0; kk < RR; ++kk) {
        const int r = l + 32 * kk;
        if (r < nx) acc[kk] = gd[r] * ec[r];
      }
    } else {
      for (int r = l; r < nc; r += 32) xs[r] = ec[r];
      __syncwarp();
      gemv_glob<RR>(D.GNT + D.gN_off[j] * nx, nx, nc, nx, xs, acc);
      __syncwarp();
    }
    for (int r = l; r < pN; r += 32) xs2[r] = hd[r];
    __syncwarp();
    sgemv<RR>(D, R, MatD{D.HNT + D.hn_off[j], nx, pN}, xs2, acc);
    const double* qk = D.qkN + size_t(j) * nx;
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < nx) xs[r] = -(zx[r] - al * (acc[kk] - 0.5 * rsumN * qk[r]));
    }
    __syncwarp();
    if (!root) {
      zero(acc);
      sgemv<RR>(D, R, MatD{D.M1T + size_t(i - 1) * D.m1_stride, m, nx}, xs, acc);
      double* T12 = D.T12 + size_t(i - 1) * m;
#pragma unroll
      for (int kk = 0; kk < RR; ++kk) {
        const int r = l + 32 * kk;
        if (r < m) T12[r] = acc[kk];
      }
    }
    w_release(A.flagB + i);
    return;
  }
  // non-leaf: G' ec (before the children), then the children's adj and T12
  const int nc = D.s1_nc[i], ny = D.y_dim[i], so = D.s1_off[i];
  const double* ec = eta + so + ny + 1;
  double vx[RR], vu[RR];
  zero(vx);
  zero(vu);
  if (D.g_diag) {
    const double* gd = D.gd + size_t(i) * m;
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < nx) vx[kk] = gd[r] * ec[r];
      if (r < nu) vu[kk] = gd[nx + r] * ec[nx + r];
    }
  } else {
    for (int r = l; r < nc; r += 32) xs[r] = ec[r];
    __syncwarp();
    gemv_glob<RR>(D.GxT + D.g_off[i] * nx, nx, nc, nx, xs, vx);
    gemv_glob<RR>(D.GuT + D.g_off[i] * nu, nu, nc, nu, xs, vu);
    __syncwarp();
  }
  const int c0 = D.cf[i], nch = D.cc[i];
  {
    const long long t0 = clock64();
    for (int k = l; k < nch; k += 32) wait_flag(A.flagB + c0 + k);
    __syncwarp();
    R.t_flag += clock64() - t0;
  }
  double sx[RR], su[RR];
  zero(sx);
  zero(su);
  for (int c = 0; c < nch; ++c) {  // ascending child order (tree_operator.cpp:106-113)
    const double* ad = D.adj + size_t(c0 + c - 1) * m;
    const double* T = D.T12 + size_t(c0 + c - 1) * m;
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < nx) {
        vx[kk] += ldcg(ad + r);
        sx[kk] += ldcg(T + r);
      }
      if (r < nu) {
        vu[kk] += ldcg(ad + nx + r);
        su[kk] += ldcg(T + nx + r);
      }
    }
  }
  // (xbar, ubar) = (z_x, z_u) - alpha L* eta on the node's (x, u) rows
  const double* zu = z + D.u_base + size_t(i) * nu;
  const double* gv = D.g + size_t(i) * nu;
#pragma unroll
  for (int kk = 0; kk < RR; ++kk) {
    const int r = l + 32 * kk;
    if (r < nu) {
      const double ub = zu[r] - al * vu[kk];
      xs[r] = ub;
      xs2[r] = ub - gv[r] - su[kk];
    }
  }
  __syncwarp();
  zero(acc);
  sgemv<RR>(D, R, MatD{D.KT + size_t(i) * D.k_stride, nx, nu}, xs, acc);  // K' ubar
  const double* h = D.h + size_t(i) * nx;
  double q[RR];
#pragma unroll
  for (int kk = 0; kk < RR; ++kk) {
    const int r = l + 32 * kk;
    q[kk] = r < nx ? h[r] - (zx[r] - al * vx[kk]) - acc[kk] + sx[kk] : 0.0;
  }
  zero(acc);
  sgemv<RR>(D, R, MatD{D.Rinv + size_t(i) * D.r_stride, nu, nu}, xs2, acc);  // d = Rt^-1 (ubar - g - sum B'q)
  double* dv = D.dvec + size_t(i) * nu;
#pragma unroll
  for (int kk = 0; kk < RR; ++kk) {
    const int r = l + 32 * kk;
    if (r < nu) dv[r] = acc[kk];
  }
  if (!root) {
    __syncwarp();
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < nx) xs[r] = q[kk];
    }
    __syncwarp();
    zero(acc);
    sgemv<RR>(D, R, MatD{D.M1T + size_t(i - 1) * D.m1_stride, m, nx}, xs, acc);  // T12 = [Abar' q; B' q]
    double* T12 = D.T12 + size_t(i - 1) * m;
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < m) T12[r] = acc[kk];
    }
  } else if (l == 0) {
    A.zo[0] = z[0] - al * eta[so + ny] - al;  // CP primal step on s0 (solver.cpp:153-154)
  }
  w_release(A.flagB + i);
}

// S2 of parent i on w = z - alpha L* eta (closed forms of kernels.cu k_s2)
__device__ void w_s2(const WideArgs& A, int i, double* xs) {
  const Dev& D = A.D;
  const int l = lane_id();
  const int n = D.cc[i], c0 = D.cf[i], ny = D.y_dim[i], yo = D.y_off[i], so = D.s1_off[i];
  const double al = A.alpha;
  const double* __restrict__ z = A.z;
  const double* __restrict__ eta = A.eta;
  double* zo = A.zo;
  const double* rb = D.rb + (yo - D.y_base);
  const double sc = eta[so + ny];
  auto wy = [&](int r) { return z[yo + r] - al * (eta[so + r] - sc * rb[r]); };
  auto wtau = [&](int k) {
    const int c = c0 + k;
    const int o2 = D.s2_off[c - 1], p = D.px[c - 1] + D.pu[c - 1];
    return z[D.tau_base + c - 1] - al * (0.5 * (eta[o2 + p] + eta[o2 + p + 1]));
  };
  auto ws = [&](int k) {
    const int c = c0 + k;
    double lt;
    if (D.cc[c] > 0) {
      lt = eta[D.s1_off[c] + D.y_dim[c]];
    } else {
      const int j = c - D.nnl, p = D.pN[j], o3 = D.s3_off[j] + D.s3_nc[j];
      lt = 0.5 * (eta[o3 + p] + eta[o3 + p + 1]);
    }
    return z[D.s_base + c - 1] - al * lt;
  };
  const int kind = D.s2_kind[i];
  if (kind == S2_DENSE) {
    const int dim = ny + 2 * n;
    for (int r = l; r < dim; r += 32) xs[r] = r < ny ? wy(r) : (r < ny + n ? wtau(r - ny) : ws(r - ny - n));
    __syncwarp();
    const double* P = D.s2P + D.s2p_off[i];
    for (int r = l; r < dim; r += 32) {
      double o = 0.0;
      for (int c = 0; c < dim; ++c) o = fma(__ldg(P + r + size_t(c) * dim), xs[c], o);
      if (r < ny)
        zo[yo + r] = o;
      else if (r < ny + n)
        zo[D.tau_base + c0 + (r - ny) - 1] = o;
      else
        zo[D.s_base + c0 + (r - ny - n) - 1] = o;
    }
    w_release(A.flagS2 + i);
    return;
  }
  const double gam = D.s2_gamma[i];
  const double Aa = kind == S2_AVAR ? gam * gam + 3.0 : 3.0;
  const double Bc = kind == S2_EQ ? 0.0 : 1.0;
  const double ylast = kind == S2_AVAR ? wy(2 * n) : (kind == S2_MAX ? wy(n) : 0.0);
  auto ety = [&](int k) -> double {
    if (kind == S2_AVAR) return gam * wy(k) - wy(n + k) + ylast;
    if (kind == S2_MAX) return -wy(k) + ylast;
    return wy(k);
  };
  double part = 0.0;
  for (int k = l; k < n; k += 32) part += ety(k) - wtau(k) - ws(k);
  const double S = warp_sum(part);
  const double den = Aa + Bc * n;
  const double shift = Bc * S / den;
  for (int k = l; k < n; k += 32) {
    const double yk = wy(k), tk = wtau(k), sk = ws(k);
    const double v = ety(k) - tk - sk;
    const double lam = (v - shift) / Aa;
    if (kind == S2_AVAR) {
      zo[yo + k] = yk - gam * lam;
      zo[yo + n + k] = wy(n + k) + lam;
    } else if (kind == S2_MAX) {
      zo[yo + k] = yk + lam;
    } else {
      zo[yo + k] = yk - lam;
    }
    zo[D.tau_base + c0 + k - 1] = tk + lam;
    zo[D.s_base + c0 + k - 1] = sk + lam;
  }
  if (l == 0 && kind != S2_EQ) {
    const double lsum = S / den;
    if (kind == S2_AVAR)
      zo[yo + 2 * n] = ylast - lsum;
    else
      zo[yo + n] = ylast - lsum;
  }
  w_release(A.flagS2 + i);
}

// ---------------------------------------------------------------------------
// Forward item of node c: S1 forward step, then every dual segment owned by c.
template <int RR>
__device__ void w_fwd(const WideArgs& A, Ring& R, int c, double* xs, double* xs2) {
  const Dev& D = A.D;
  const int l = lane_id(), nx = D.nx, nu = D.nu;
  const double al = A.alpha;
  const double* __restrict__ z = A.z;
  const double* __restrict__ eta = A.eta;
  double* zo = A.zo;
  double* eo = A.eo;
  const bool root = c == 0, leaf = D.cc[c] == 0;
  // streamed matrices, consumed in item_mats order:
  //   M1 (non-root) | K (non-leaf) | Hx, Hu (non-root) | HN (leaf)
  double x[RR], u[RR];
  zero(u);
  const int an = root ? 0 : D.anc[c];
  if (root) {
    const long long t0 = clock64();
    if (l == 0) wait_flag(A.flagB);
    __syncwarp();
    R.t_flag += clock64() - t0;
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      x[kk] = r < nx ? D.xinit[r] : 0.0;
    }
  } else {
    const long long t0 = clock64();
    if (l == 0) wait_flag(A.flagF + an);
    __syncwarp();
    R.t_flag += clock64() - t0;
    for (int r = l; r < nx; r += 32) xs[r] = ldcg(zo + 1 + size_t(an) * nx + r);
    for (int r = l; r < nu; r += 32) xs[nx + r] = ldcg(D.dvec + size_t(an) * nu + r);
    __syncwarp();
    zero(x);
    sgemv<RR>(D, R, MatD{D.M1 + size_t(c - 1) * D.m1_stride, nx, nx + nu}, xs, x);  // [Abar B][x_anc; d_anc]
    const double* cv = D.cvec + size_t(c - 1) * nx;
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < nx) x[kk] += cv[r];
    }
  }
#pragma unroll
  for (int kk = 0; kk < RR; ++kk) {
    const int r = l + 32 * kk;
    if (r < nx) zo[1 + size_t(c) * nx + r] = x[kk];
  }
  if (!leaf) {
    __syncwarp();
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < nx) xs2[r] = x[kk];
    }
    __syncwarp();
    sgemv<RR>(D, R, MatD{D.K + size_t(c) * D.k_stride, nu, nx}, xs2, u);  // K x
    const double* dv = D.dvec + size_t(c) * nu;
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < nu) {
        u[kk] += ldcg(dv + r);
        zo[D.u_base + size_t(c) * nu + r] = u[kk];
      }
    }
  }
  w_release(A.flagF + c);  // children need only (x+, u+) and d
  // ---- dual update on the segments owned by c (k_L<DUAL>): p = eta + a L w,
  // w = 2 z+ - z, eta+ = p - a Pi_S3(p / a)
  {
    const long long t0 = clock64();
    if (l == 0 && !leaf) wait_flag(A.flagS2 + c);
    if (l == 1 && !root) wait_flag(A.flagS2 + an);
    __syncwarp();
    R.t_flag += clock64() - t0;
  }
  auto W = [&](int idx) { return 2.0 * ldcg(zo + idx) - z[idx]; };
  // own (x^, u^) in registers
  double hx[RR], hu[RR];
  {
    const double* zx = z + 1 + size_t(c) * nx;
    const double* zu = z + D.u_base + size_t(c) * nu;
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      hx[kk] = r < nx ? 2.0 * x[kk] - zx[r] : 0.0;
      hu[kk] = (!leaf && r < nu) ? 2.0 * u[kk] - zu[r] : 0.0;
    }
  }
  double acc[RR];
  if (!leaf) {
    const int ny = D.y_dim[c], yo = D.y_off[c], so = D.s1_off[c];
    const double* rb = D.rb + (yo - D.y_base);
    double part = 0.0;
    for (int r = l; r < ny; r += 32) {
      const double yv = W(yo + r);
      part += rb[r] * yv;
      eo[so + r] = (eta[so + r] + al * yv) / al;  // staged p/a, projected below
    }
    const double by = warp_sum(part);
    __syncwarp();
    ycone(D, c, eo + so);
    for (int r = l; r < ny; r += 32) {
      const double pv = eta[so + r] + al * W(yo + r);
      eo[so + r] = pv - al * eo[so + r];
    }
    if (l == 0) {
      const double sv = W(root ? 0 : D.s_base + c - 1) - by;
      const double pv = eta[so + ny] + al * sv;
      eo[so + ny] = pv - al * fmax(0.0, pv / al);
    }
    const int nc = D.s1_nc[c];
    zero(acc);
    if (D.g_diag) {
      const double* gd = D.gd + size_t(c) * (nx + nu);
      // constraint row r < nx uses x^_r, rows nx.. use u^ (diagonal [Gx Gu])
#pragma unroll
      for (int kk = 0; kk < RR; ++kk) {
        const int r = l + 32 * kk;
        if (r < nx) xs[r] = hx[kk];
        if (r < nu) xs[nx + r] = hu[kk];
      }
      __syncwarp();
#pragma unroll
      for (int kk = 0; kk < RR; ++kk) {
        const int r = l + 32 * kk;
        if (r < nc) acc[kk] = gd[r] * xs[r];
      }
    } else {
#pragma unroll
      for (int kk = 0; kk < RR; ++kk) {
        const int r = l + 32 * kk;
        if (r < nx) xs[r] = hx[kk];
        if (r < nu) xs[nx + r] = hu[kk];
      }
      __syncwarp();
      gemv_glob<RR>(D.Gx + D.g_off[c] * nx, nc, nx, nc, xs, acc);
      gemv_glob<RR>(D.Gu + D.g_off[c] * nu, nc, nu, nc, xs + nx, acc);
    }
    const double* lo = D.lo + D.g_off[c];
    const double* hi = D.hi + D.g_off[c];
    const int co = so + ny + 1;
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < nc) {
        const double pv = eta[co + r] + al * acc[kk];
        eo[co + r] = pv - al * fmin(fmax(pv / al, lo[r]), hi[r]);
      }
    }
    __syncwarp();
  }
  if (!root) {  // stage-cost SOC block of (x^_anc, u^_anc, tau^_c)
    const int k = c - 1, px = D.px[k], pu = D.pu[k], p = px + pu;
    for (int r = l; r < nx; r += 32) xs[r] = W(1 + an * nx + r);
    for (int r = l; r < nu; r += 32) xs[nx + r] = W(D.u_base + an * nu + r);
    __syncwarp();
    const double* qk = D.qk + size_t(k) * (nx + nu);
    double part = 0.0;
    for (int r = l; r < nx + nu; r += 32) part += qk[r] * xs[r];
    const double qd = warp_sum(part);
    const double row = 0.5 * W(D.tau_base + k) - 0.5 * qd;
    double ax[RR], au[RR];
    zero(ax);
    zero(au);
    sgemv<RR>(D, R, MatD{D.Hx + D.hx_off[k], px, nx}, xs, ax);       // Hx x^
    sgemv<RR>(D, R, MatD{D.Hu + D.hu_off[k], pu, nu}, xs + nx, au);  // Hu u^
    __syncwarp();
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < px) xs2[r] = ax[kk];
      if (r < pu) xs2[px + r] = au[kk];
    }
    __syncwarp();
    const int so = D.s2_off[k];
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      acc[kk] = r < p ? eta[so + r] + al * xs2[r] : 0.0;
    }
    double vp = eta[so + p] + al * row, vp1 = eta[so + p + 1] + al * row;
    double t[RR];
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) t[kk] = acc[kk] / al;
    double tp = vp / al, tp1 = vp1 / al;
    soc_proj<RR>(t, p, tp, tp1, D.a + D.a_off[k]);
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < p) eo[so + r] = acc[kk] - al * t[kk];
    }
    if (l == 0) {
      eo[so + p] = vp - al * tp;
      eo[so + p + 1] = vp1 - al * tp1;
    }
    __syncwarp();
  }
  if (leaf) {  // G_N x^ (box) and the terminal SOC block of (x^, s^)
    const int j = c - D.nnl, nc = D.s3_nc[j], p = D.pN[j], eo3 = D.s3_off[j];
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < nx) xs[r] = hx[kk];
    }
    __syncwarp();
    zero(acc);
    if (D.gN_diag) {
      const double* gd = D.gNd + size_t(j) * nx;
#pragma unroll
      for (int kk = 0; kk < RR; ++kk) {
        const int r = l + 32 * kk;
        if (r < nc) acc[kk] = gd[r] * xs[r];
      }
    } else {
      gemv_glob<RR>(D.GN + D.gN_off[j] * nx, nc, nx, nc, xs, acc);
    }
    const double* lo = D.loN + D.gN_off[j];
    const double* hi = D.hiN + D.gN_off[j];
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < nc) {
        const double pv = eta[eo3 + r] + al * acc[kk];
        eo[eo3 + r] = pv - al * fmin(fmax(pv / al, lo[r]), hi[r]);
      }
    }
    const double* qk = D.qkN + size_t(j) * nx;
    double part = 0.0;
    for (int r = l; r < nx; r += 32) part += qk[r] * xs[r];
    const double qd = warp_sum(part);
    const double row = 0.5 * W(D.s_base + c - 1) - 0.5 * qd;
    zero(acc);
    sgemv<RR>(D, R, MatD{D.HN + D.hn_off[j], p, nx}, xs, acc);  // H_N x^
    const int so = eo3 + nc;
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      acc[kk] = r < p ? eta[so + r] + al * acc[kk] : 0.0;
    }
    double vp = eta[so + p] + al * row, vp1 = eta[so + p + 1] + al * row;
    double t[RR];
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) t[kk] = acc[kk] / al;
    double tp = vp / al, tp1 = vp1 / al;
    soc_proj<RR>(t, p, tp, tp1, D.aN + D.aN_off[j]);
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < p) eo[so + r] = acc[kk] - al * t[kk];
    }
    if (l == 0) {
      eo[so + p] = vp - al * tp;
      eo[so + p + 1] = vp1 - al * tp1;
    }
  }
}

template <int RR, int MINB>
__global__ void __launch_bounds__(256, MINB) k_T_wide(const __grid_constant__ WideArgs A) {
  extern __shared__ __align__(128) double wsm[];
  const Dev& D = A.D;
  const int w = threadIdx.x >> 5, l = lane_id();
  const int W = A.warps, S = A.slots, CH = A.chunk, VD = A.vecd;
  double* ring = wsm + size_t(w) * S * CH;
  double* xs = wsm + size_t(W) * S * CH + size_t(w) * 2 * VD;
  double* xs2 = xs + VD;
  uint64_t* bars = reinterpret_cast<uint64_t*>(wsm + size_t(W) * S * CH + size_t(W) * 2 * VD) + w * kMaxSlots;
  __shared__ Prod prods[8];
  Prod* P = &prods[w];
  Ring R;
  R.ps = P;
  R.buf = ring;
  R.bar = bars;
  R.S = S;
  R.chunk = CH;
  R.stride = gridDim.x * W;
  R.total = D.nn + D.nnl + D.nn;
  R.cons = 0;
  R.t_ring = 0;
  R.t_flag = 0;
  const int gw = blockIdx.x * W + w;
  if (l == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    P->prod = 0;
    P->tp = gw;
    P->mi = 0;
    P->co = 0;
    P->nm = 0;
    if (gw < R.total) {
      int kind, node;
      decode(D, gw, kind, node);
      P->nm = item_mats(D, kind, node, P->md);
    }
    refill(D, P, 0u, S, CH, ring, bars, R.stride, R.total);
  }
  __syncwarp();
  long long t_kind[3] = {0, 0, 0};
  int n_kind[3] = {0, 0, 0};
  const long long t_start = clock64();
  for (int tk = gw; tk < R.total; tk += R.stride) {
    int kind, node;
    decode(D, tk, kind, node);
    const long long t0 = clock64();
    if (kind == 0)
      w_back<RR>(A, R, node, xs, xs2);
    else if (kind == 1)
      w_s2(A, node, xs);
    else
      w_fwd<RR>(A, R, node, xs, xs2);
    __syncwarp();
    t_kind[kind] += clock64() - t0;
    ++n_kind[kind];
  }
  if (A.prof && l == 0) {  // optional: per-warp cycle accounting, summed over warps
    unsigned long long* pf = A.prof;
    atomicAdd(pf + 0, (unsigned long long)(clock64() - t_start));
    atomicAdd(pf + 1, (unsigned long long)R.t_ring);
    atomicAdd(pf + 2, (unsigned long long)R.t_flag);
    for (int k = 0; k < 3; ++k) {
      atomicAdd(pf + 3 + k, (unsigned long long)t_kind[k]);
      atomicAdd(pf + 6 + k, (unsigned long long)n_kind[k]);
    }
    atomicAdd(pf + 9, 1ull);
  }
}

}  // namespace

int wide_smem_bytes(int warps, int slots, int chunk, int vecd) {
  return int(sizeof(double) * (size_t(warps) * slots * chunk + size_t(warps) * 2 * vecd) +
             sizeof(uint64_t) * size_t(warps) * kMaxSlots);
}

int wide_rows(const Dev& D, int max_nc) {
  const int need = std::max(D.nx + D.nu, max_nc);
  const int r = (need + 31) / 32;
  if (r <= 1) return 1;
  if (r <= 2) return 2;
  if (r <= 3) return 3;
  if (r <= 4) return 4;
  return 8;
}

#define WIDE_SWITCH(rows, ctas, F)                    \
  do {                                                \
    if (ctas >= 2) {                                  \
      switch (rows) {                                 \
        case 1: F(1, 2); break;                       \
        case 2: F(2, 2); break;                       \
        case 3: F(3, 2); break;                       \
        case 4: F(4, 2); break;                       \
        default: F(8, 2); break;                      \
      }                                               \
    } else {                                          \
      switch (rows) {                                 \
        case 1: F(1, 1); break;                       \
        case 2: F(2, 1); break;                       \
        case 3: F(3, 1); break;                       \
        case 4: F(4, 1); break;                       \
        default: F(8, 1); break;                      \
      }                                               \
    }                                                 \
  } while (0)

const void* wide_kernel_ptr(int rows, int ctas) {
  const void* p = nullptr;
#define WPTR(R, M) p = reinterpret_cast<const void*>(&k_T_wide<R, M>)
  WIDE_SWITCH(rows, ctas, WPTR);
#undef WPTR
  return p;
}

cudaError_t wide_configure(int rows, int ctas, int smem_bytes) {
  return cudaFuncSetAttribute(wide_kernel_ptr(rows, ctas), cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
}

void launch_T_wide(const WideArgs& A, int rows, int ctas, int grid, cudaStream_t st) {
  const int smem = wide_smem_bytes(A.warps, A.slots, A.chunk, A.vecd);
  const int threads = 32 * A.warps;
#define WLAUNCH(R, M) k_T_wide<R, M><<<grid, threads, smem, st>>>(A)
  WIDE_SWITCH(rows, ctas, WLAUNCH);
#undef WLAUNCH
}

}  // namespace spock
