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
// An item only waits on items with smaller tickets, which were taken by CTAs
// that are already running, so the schedule cannot deadlock whatever the
// residency.  Each CTA issues TMA bulk copies (cp.async.bulk, mbarrier
// completion) of its node's matrices into shared memory *before* it waits on
// the completion flags of its children (backward) or parent (forward); the
// flag wait then overlaps the HBM traffic and the dependent chain of 2N+2
// levels costs one flag hop plus a shared-memory GEMV per level.
//
// Backward item (node i), restructured Alg. 2 (see kernels.cu header):
//   adj_i = H_i' head_i - rsum_i/2 qk_i                 (own stage SOC, for the parent)
//   xbar_i = z_x - a(G_x' ec_i + sum_c adj_c,x)          (L* and the CP primal step)
//   q_i = sum_c [Abar_c' q_c] - xbar_i - K_i' ubar_i + h_i ;  leaf: q_i = -xbar_i
//   d_i = Rt_i^{-1}(ubar_i - sum_c [B_c' q_c] - g_i)
//   [Abar_i' q_i; B_i' q_i] -> T12_i for the parent
// Forward item (node c):
//   x_c = [Abar_c B_c][x_anc; d_anc] + c_c,  u_c = K_c x_c + d_c
//   then every dual segment owned by c: eta+ = p - a Pi_S3(p / a),
//   p = eta + a L(2 z+ - z).
#include <cuda_runtime.h>

#include <cstdint>

#include "dev.cuh"
#include "fused.hpp"

namespace spock {

namespace {

constexpr int kFT = 256;  // threads per CTA
constexpr int kSlot = kMaxD + 8;  // doubles per vector slot in shared memory
constexpr int kSlots = 6;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
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
// loads of data produced by other CTAs in this launch: L2 only (no stale L1)
__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }

struct Smem {
  uint64_t bar;
  int item;
  int pad_;
  double* mat;  // matrix staging area (dynamic smem)
  double* vec;  // vector scratch
  double* red;  // 2*kFT doubles
};

// y[r] = (acc ? y[r] : 0) + sum_c A[r + c*lda] x[c], r < m <= kFT; every
// thread of the CTA participates (column slices reduced in fixed order).
__device__ void cta_gemv(const double* A, int m, int n, int lda, const double* x, double* y, bool acc,
                         double* red) {
  const int t = threadIdx.x;
  if (m <= 0) return;
  const int slices = max(1, kFT / m);
  const int r = t % m, s = t / m;
  double v = 0.0;
  if (s < slices && n > 0)
    for (int c = s; c < n; c += slices) v = fma(A[r + size_t(c) * lda], x[c], v);
  if (t < m * slices) red[t] = v;
  __syncthreads();
  if (t < m) {
    double o = acc ? y[t] : 0.0;
    for (int j = 0; j < slices; ++j) o += red[t + j * m];
    y[t] = o;
  }
  __syncthreads();
}

// sum over the CTA, result broadcast to all threads
__device__ double cta_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int k = 0; k < kFT / 32; ++k) s += red[k];
  __syncthreads();
  return s;
}

// translated SOC projection of v[0..d) (axis last) in place: v <- a + Pi_SOC(v - a)
__device__ void cta_soc_project(double* v, const double* a, int d, double* red) {
  const int t = threadIdx.x;
  double s = 0.0;
  for (int r = t; r < d; r += kFT) {
    v[r] -= a[r];
    if (r < d - 1) s += v[r] * v[r];
  }
  const double hn = sqrt(cta_sum(s, red));
  const double tt = v[d - 1];
  __syncthreads();
  if (hn <= tt) {
  } else if (hn <= -tt) {
    for (int r = t; r < d; r += kFT) v[r] = 0.0;
  } else {
    const double f = (hn + tt) / (2.0 * hn);
    for (int r = t; r < d - 1; r += kFT) v[r] *= f;
    if (t == 0) v[d - 1] = 0.5 * (hn + tt);
  }
  __syncthreads();
  for (int r = t; r < d; r += kFT) v[r] += a[r];
  __syncthreads();
}

__device__ void wait_flag(const int* f, int epoch) {
  while (ld_acquire(f) < epoch) __nanosleep(32);
}

// ---------------------------------------------------------------------------
__device__ void item_s2(const FusedArgs& F, int i, double* red, double* vec) {
  const Dev& D = F.D;
  const int t = threadIdx.x;
  const int n = D.cc[i], c0 = D.cf[i], ny = D.y_dim[i], yo = D.y_off[i], so = D.s1_off[i];
  const double al = F.alpha;
  const double* z = F.z;
  const double* eta = F.eta;
  double* zo = F.zo;
  const double* rb = D.rb + (yo - D.y_base);
  const double sc = eta[so + ny];
  // w = z - alpha L* eta on (y_i, tau_c, s_c)
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
    double* w = vec;  // dim <= kMaxD
    for (int r = t; r < dim; r += kFT) w[r] = r < ny ? wy(r) : (r < ny + n ? wtau(r - ny) : ws(r - ny - n));
    __syncthreads();
    double* o = w + kSlot;
    cta_gemv(D.s2P + D.s2p_off[i], dim, dim, dim, w, o, false, red);
    for (int r = t; r < dim; r += kFT) {
      if (r < ny)
        zo[yo + r] = o[r];
      else if (r < ny + n)
        zo[D.tau_base + c0 + (r - ny) - 1] = o[r];
      else
        zo[D.s_base + c0 + (r - ny - n) - 1] = o[r];
    }
    __syncthreads();
    return;
  }
  const double gam = D.s2_gamma[i];
  const double A = kind == S2_AVAR ? gam * gam + 3.0 : 3.0;
  const double Bc = kind == S2_EQ ? 0.0 : 1.0;
  const double ylast = kind == S2_AVAR ? wy(2 * n) : (kind == S2_MAX ? wy(n) : 0.0);
  auto ety = [&](int k) -> double {
    if (kind == S2_AVAR) return gam * wy(k) - wy(n + k) + ylast;
    if (kind == S2_MAX) return -wy(k) + ylast;
    return wy(k);
  };
  double part = 0.0;
  for (int k = t; k < n; k += kFT) part += ety(k) - wtau(k) - ws(k);
  const double S = cta_sum(part, red);
  const double den = A + Bc * n;
  const double shift = Bc * S / den;
  for (int k = t; k < n; k += kFT) {
    const double yk = wy(k), tk = wtau(k), sk = ws(k);
    const double v = ety(k) - tk - sk;
    const double lam = (v - shift) / A;
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
  if (t == 0 && kind != S2_EQ) {
    const double lsum = S / den;
    if (kind == S2_AVAR)
      zo[yo + 2 * n] = ylast - lsum;
    else
      zo[yo + n] = ylast - lsum;
  }
  __syncthreads();
}

// release a completion flag: CTA barrier, then one fenced release store
// (the semaphore pattern of CUTLASS's GenericBarrier)
__device__ __forceinline__ void cta_release(int* flag) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    st_release(flag, 1);
  }
}

// issue the bulk copies of one item's blocks (thread 0); returns staged (or
// global) pointers through `out`
__device__ void stage_blocks(const FusedArgs& F, Smem& S, const double* const* src, const int* doubles, int n,
                             const double** out) {
  if (threadIdx.x != 0) return;
  if (!F.stage_smem) {
    for (int k = 0; k < n; ++k) out[k] = src[k];
    return;
  }
  fence_proxy_async();
  uint32_t total = 0;
  for (int k = 0; k < n; ++k) total += uint32_t((doubles[k] + 1) & ~1) * 8u;
  if (total)
    mbar_expect_tx(&S.bar, total);
  else
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&S.bar)) : "memory");
  int off = 0;
  for (int k = 0; k < n; ++k) {
    if (doubles[k] <= 0) {
      out[k] = src[k];
      continue;
    }
    const int padded = (doubles[k] + 1) & ~1;
    bulk_g2s(S.mat + off, src[k], uint32_t(padded) * 8u, &S.bar);
    out[k] = S.mat + off;
    off += padded;
  }
}

__device__ __forceinline__ void wait_blocks(const FusedArgs& F, Smem& S, uint32_t& phase) {
  if (!F.stage_smem) return;
  while (!mbar_try_wait(&S.bar, phase)) {
  }
  phase ^= 1u;
}

__device__ void item_back(const FusedArgs& F, int i, Smem& S, uint32_t& phase) {
  const Dev& D = F.D;
  const int t = threadIdx.x, nx = D.nx, nu = D.nu, m = nx + nu;
  const bool leaf = D.cc[i] == 0, root = i == 0;
  const double al = F.alpha;
  const double* z = F.z;
  const double* eta = F.eta;
  int px = 0, pu = 0, pN = 0;
  if (!root) px = D.px[i - 1], pu = D.pu[i - 1];
  if (leaf) pN = D.pN[i - D.nnl];
  // ---- 1. prefetch this node's blocks: H_x', H_u' (own stage SOC), M1' (own
  // sweep block), K', Rt^-1 (non-leaf) or H_N' (leaf)
  __shared__ const double* sp[6];
  {
    const double* src[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    int dbl[6] = {0, 0, 0, 0, 0, 0};
    if (!root) {
      src[0] = D.HxT + D.hx_off[i - 1], dbl[0] = px * nx;
      src[1] = D.HuT + D.hu_off[i - 1], dbl[1] = pu * nu;
      src[2] = D.M1T + size_t(i - 1) * D.m1_stride, dbl[2] = m * nx;
    }
    if (!leaf) {
      src[3] = D.KT + size_t(i) * D.k_stride, dbl[3] = nx * nu;
      src[4] = D.Rinv + size_t(i) * D.r_stride, dbl[4] = nu * nu;
    } else {
      src[5] = D.HNT + D.hn_off[i - D.nnl], dbl[5] = pN * nx;
    }
    stage_blocks(F, S, src, dbl, 6, sp);
  }
  double* V = S.vec;
  double* head = V;          // own stage-SOC head (p), later the leaf head (pN)
  double* gx = head + kSlot; // G' ec (+ leaf terms): L* (x, u) without the children
  double* xb = gx + kSlot;   // z (x, u) of this node
  double* q = xb + kSlot;    // q (nx)
  double* tv = q + kSlot;    // scratch (m)
  double* rhs = tv + kSlot;  // scratch (m)
  double* red = S.red;
  // ---- 2. everything that does not depend on the children
  double rsum = 0.0, rsumN = 0.0;
  if (!root) {
    const int o2 = D.s2_off[i - 1], p = px + pu;
    for (int r = t; r < p; r += kFT) head[r] = eta[o2 + r];
    rsum = eta[o2 + p] + eta[o2 + p + 1];
  }
  for (int r = t; r < (leaf ? nx : m); r += kFT)
    xb[r] = r < nx ? z[1 + size_t(i) * nx + r] : z[D.u_base + size_t(i) * nu + (r - nx)];
  if (!leaf) {
    const int ny = D.y_dim[i], nc = D.s1_nc[i];
    const double* ec = eta + D.s1_off[i] + ny + 1;
    if (D.g_diag) {
      const double* gd = D.gd + size_t(i) * m;
      for (int r = t; r < m; r += kFT) gx[r] = gd[r] * ec[r];
    } else {
      for (int r = t; r < nc; r += kFT) rhs[r] = ec[r];
      __syncthreads();
      cta_gemv(D.GxT + D.g_off[i] * nx, nx, nc, nx, rhs, gx, false, red);
      cta_gemv(D.GuT + D.g_off[i] * nu, nu, nc, nu, rhs, gx + nx, false, red);
    }
  } else {
    const int j = i - D.nnl, nc = D.s3_nc[j];
    const double* ec = eta + D.s3_off[j];
    if (D.gN_diag) {
      const double* gd = D.gNd + size_t(j) * nx;
      for (int r = t; r < nx; r += kFT) gx[r] = gd[r] * ec[r];
    } else {
      for (int r = t; r < nc; r += kFT) rhs[r] = ec[r];
      __syncthreads();
      cta_gemv(D.GNT + D.gN_off[j] * nx, nx, nc, nx, rhs, gx, false, red);
    }
  }
  __syncthreads();
  const double *HxT = sp[0], *HuT = sp[1], *M1T = sp[2], *KT = sp[3], *Ri = sp[4], *HNT = sp[5];
  wait_blocks(F, S, phase);
  if (!root) {  // own stage-SOC adjoint term for the parent: adj_i = H' head - rsum/2 qk
    const double* qkv = D.qk + size_t(i - 1) * m;
    for (int r = t; r < m; r += kFT) tv[r] = -0.5 * rsum * qkv[r];
    __syncthreads();
    cta_gemv(HxT, nx, px, nx, head, tv, true, red);
    cta_gemv(HuT, nu, pu, nu, head + px, tv + nx, true, red);
    double* adj = D.adj + size_t(i - 1) * m;
    for (int r = t; r < m; r += kFT) adj[r] = tv[r];
  }
  if (leaf) {  // terminal SOC term of L* (x part): + H_N' head_N - rsum_N/2 qk_N
    const int j = i - D.nnl;
    const double* hd = eta + D.s3_off[j] + D.s3_nc[j];
    __syncthreads();
    for (int r = t; r < pN; r += kFT) head[r] = hd[r];
    rsumN = hd[pN] + hd[pN + 1];
    __syncthreads();
    cta_gemv(HNT, nx, pN, nx, head, gx, true, red);
    const double* qk = D.qkN + size_t(j) * nx;
    for (int r = t; r < nx; r += kFT) {
      gx[r] -= 0.5 * rsumN * qk[r];
      q[r] = -(xb[r] - al * gx[r]);  // leaf: q = -xbar
    }
    __syncthreads();
  } else {
    // ---- 3. children (flags), then q, d
    const int c0 = D.cf[i], nch = D.cc[i];
    if (t == 0)
      for (int c = 0; c < nch; ++c) wait_flag(F.flagB + c0 + c, 1);
    __syncthreads();
    const double* h = D.h + size_t(i) * nx;
    const double* gv = D.g + size_t(i) * nu;
    for (int r = t; r < m; r += kFT) {
      double lt = gx[r], tq = 0.0;
      for (int c = 0; c < nch; ++c) {
        const size_t o = size_t(c0 + c - 1) * m + r;
        lt += ldcg(D.adj + o);
        tq += ldcg(D.T12 + o);
      }
      const double w = xb[r] - al * lt;  // (xbar, ubar)
      if (r < nx) {
        q[r] = h[r] - w + tq;
      } else {
        xb[r] = w;  // ubar
        rhs[r - nx] = w - gv[r - nx] - tq;
      }
    }
    __syncthreads();
    cta_gemv(KT, nx, nu, nx, xb + nx, tv, false, red);  // K' ubar
    for (int r = t; r < nx; r += kFT) q[r] -= tv[r];
    cta_gemv(Ri, nu, nu, nu, rhs, tv + nx, false, red);  // d
    double* dv = D.dvec + size_t(i) * nu;
    for (int r = t; r < nu; r += kFT) dv[r] = tv[nx + r];
    __syncthreads();
  }
  if (!root) {
    cta_gemv(M1T, m, nx, m, q, tv, false, red);
    double* T12 = D.T12 + size_t(i - 1) * m;
    for (int r = t; r < m; r += kFT) T12[r] = tv[r];
  } else if (t == 0) {
    const double sc = eta[D.s1_off[0] + D.y_dim[0]];
    F.zo[0] = z[0] - al * sc - al;  // CP primal step on s0 (solver.cpp:153-154)
  }
  cta_release(F.flagB + i);
}

__device__ void item_fwd(const FusedArgs& F, int c, Smem& S, uint32_t& phase) {
  const Dev& D = F.D;
  const int t = threadIdx.x, nx = D.nx, nu = D.nu, m = nx + nu;
  const bool leaf = D.cc[c] == 0, root = c == 0;
  const double al = F.alpha;
  const double* z = F.z;
  const double* eta = F.eta;
  double* zo = F.zo;
  double* eo = F.eo;
  int px = 0, pu = 0, pN = 0;
  if (!root) px = D.px[c - 1], pu = D.pu[c - 1];
  if (leaf) pN = D.pN[c - D.nnl];
  __shared__ const double* sp[5];
  {
    const double* src[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    int dbl[5] = {0, 0, 0, 0, 0};
    if (!root) {
      src[0] = D.M1 + size_t(c - 1) * D.m1_stride, dbl[0] = nx * m;
      src[1] = D.Hx + D.hx_off[c - 1], dbl[1] = px * nx;
      src[2] = D.Hu + D.hu_off[c - 1], dbl[2] = pu * nu;
    }
    if (!leaf)
      src[3] = D.K + size_t(c) * D.k_stride, dbl[3] = nu * nx;
    else
      src[4] = D.HN + D.hn_off[c - D.nnl], dbl[4] = pN * nx;
    stage_blocks(F, S, src, dbl, 5, sp);
  }
  double* V = S.vec;
  double* xd = V;              // [x_anc+; d_anc]
  double* xn = xd + kSlot;     // own (x+, u+)
  double* zown = xn + kSlot;   // own (x, u) of z
  double* ahat = zown + kSlot; // anc (x^, u^)
  double* val = ahat + kSlot;  // segment values
  double* pv = val + kSlot;    // p / alpha
  double* red = S.red;
  // independent of the parent
  for (int r = t; r < (leaf ? nx : m); r += kFT)
    zown[r] = r < nx ? z[1 + size_t(c) * nx + r] : z[D.u_base + size_t(c) * nu + (r - nx)];
  const int an = root ? 0 : D.anc[c];
  if (!root)
    for (int r = t; r < m; r += kFT)
      ahat[r] = -(r < nx ? z[1 + size_t(an) * nx + r] : z[D.u_base + size_t(an) * nu + (r - nx)]);
  double dself = 0.0;  // own d entry for thread t < nu
  __syncthreads();
  const double *M1 = sp[0], *Hx = sp[1], *Hu = sp[2], *K = sp[3], *HN = sp[4];
  wait_blocks(F, S, phase);
  // ---- parent forward (root: own backward)
  if (t == 0) wait_flag(root ? F.flagB : F.flagF + an, 1);
  __syncthreads();
  if (!leaf && t < nu) dself = ldcg(D.dvec + size_t(c) * nu + t);
  if (!root) {
    for (int r = t; r < m; r += kFT) {
      if (r < nx) {
        const double xp = ldcg(zo + 1 + size_t(an) * nx + r);
        xd[r] = xp;
        ahat[r] += 2.0 * xp;
      } else {
        xd[r] = ldcg(D.dvec + size_t(an) * nu + (r - nx));
        ahat[r] += 2.0 * ldcg(zo + D.u_base + size_t(an) * nu + (r - nx));
      }
    }
    __syncthreads();
    cta_gemv(M1, nx, m, nx, xd, xn, false, red);
    const double* cv = D.cvec + size_t(c - 1) * nx;
    for (int r = t; r < nx; r += kFT) xn[r] += cv[r];
  } else {
    for (int r = t; r < nx; r += kFT) xn[r] = D.xinit[r];
  }
  __syncthreads();
  if (!leaf) {
    cta_gemv(K, nu, nx, nu, xn, xn + nx, false, red);
    if (t < nu) xn[nx + t] += dself;
    __syncthreads();
  }
  for (int r = t; r < (leaf ? nx : m); r += kFT) {
    if (r < nx)
      zo[1 + size_t(c) * nx + r] = xn[r];
    else
      zo[D.u_base + size_t(c) * nu + (r - nx)] = xn[r];
  }
  // children need only (x+, u+) and d: release before the dual work
  cta_release(F.flagF + c);
  for (int r = t; r < (leaf ? nx : m); r += kFT) zown[r] = 2.0 * xn[r] - zown[r];  // own (x^, u^)
  if (t == 0) {
    if (!leaf) wait_flag(F.flagS2 + c, 1);
    if (!root) wait_flag(F.flagS2 + an, 1);
  }
  __syncthreads();
  const double* hat = zown;
  auto dual = [&](int off, int d) {
    for (int r = t; r < d; r += kFT) {
      const double p = eta[off + r] + al * val[r];
      val[r] = p;
      pv[r] = p / al;
    }
    __syncthreads();
  };
  auto hatv = [&](int idx) { return 2.0 * ldcg(zo + idx) - z[idx]; };
  if (!root) {  // stage-cost SOC block of (x_anc, u_anc, tau_c)
    const int k = c - 1, p = px + pu, o2 = D.s2_off[k];
    const double* qk = D.qk + size_t(k) * m;
    double part = 0.0;
    for (int r = t; r < m; r += kFT) part += qk[r] * ahat[r];
    const double qd = cta_sum(part, red);
    cta_gemv(Hx, px, nx, px, ahat, val, false, red);
    cta_gemv(Hu, pu, nu, pu, ahat + nx, val + px, false, red);
    if (t == 0) {
      const double row = 0.5 * hatv(D.tau_base + k) - 0.5 * qd;
      val[p] = row;
      val[p + 1] = row;
    }
    __syncthreads();
    dual(o2, p + 2);
    cta_soc_project(pv, D.a + D.a_off[k], p + 2, red);
    for (int r = t; r < p + 2; r += kFT) eo[o2 + r] = val[r] - al * pv[r];
    __syncthreads();
  }
  if (!leaf) {  // y-copy rows (dual cone), risk scalar (R+), constraint rows (box)
    const int ny = D.y_dim[c], yo = D.y_off[c], so = D.s1_off[c], nc = D.s1_nc[c];
    const double* rb = D.rb + (yo - D.y_base);
    const int nn0 = D.yc_nonneg[c];
    double part = 0.0;
    for (int r = t; r < ny; r += kFT) {
      const double yh = hatv(yo + r);
      part += rb[r] * yh;
      const double p = eta[so + r] + al * yh;
      double tp = p / al;
      if (nn0 >= 0) {
        if (r < nn0) tp = fmax(tp, 0.0);
        eo[so + r] = p - al * tp;
      } else {
        eo[so + r] = tp;  // staged, general cone projected below
      }
    }
    const double by = cta_sum(part, red);
    if (nn0 < 0) {
      int off = 0;
      for (int pi = D.yc_poff[c]; pi < D.yc_poff[c + 1]; ++pi) {
        const int kind = D.yc_kind[pi], dim = D.yc_dim[pi];
        double* pvg = eo + so + off;
        if (kind == 0) {
          for (int r = t; r < dim; r += kFT) pvg[r] = 0.0;
        } else if (kind == 1) {
          for (int r = t; r < dim; r += kFT) pvg[r] = fmax(pvg[r], 0.0);
        } else if (kind == 2) {
          double ss = 0.0;
          for (int r = t; r < dim - 1; r += kFT) ss += pvg[r] * pvg[r];
          const double hn = sqrt(cta_sum(ss, red));
          const double tt = pvg[dim - 1];
          __syncthreads();
          if (hn <= tt) {
          } else if (hn <= -tt) {
            for (int r = t; r < dim; r += kFT) pvg[r] = 0.0;
          } else {
            const double f = (hn + tt) / (2.0 * hn);
            for (int r = t; r < dim - 1; r += kFT) pvg[r] *= f;
            if (t == 0) pvg[dim - 1] = 0.5 * (hn + tt);
          }
        }
        __syncthreads();
        off += dim;
      }
      for (int r = t; r < ny; r += kFT) {
        const double p = eta[so + r] + al * hatv(yo + r);
        eo[so + r] = p - al * eo[so + r];
      }
    }
    if (t == 0) {
      const double sv = hatv(c == 0 ? 0 : D.s_base + c - 1) - by;
      const double p = eta[so + ny] + al * sv;
      eo[so + ny] = p - al * fmax(0.0, p / al);
    }
    __syncthreads();
    // constraint rows G [x^; u^] with box projection
    if (D.g_diag) {
      const double* gd = D.gd + size_t(c) * m;
      for (int r = t; r < nc; r += kFT) val[r] = gd[r] * hat[r];
    } else {
      cta_gemv(D.Gx + D.g_off[c] * nx, nc, nx, nc, hat, val, false, red);
      cta_gemv(D.Gu + D.g_off[c] * nu, nc, nu, nc, hat + nx, val, true, red);
    }
    __syncthreads();
    const int co = so + ny + 1;
    const double* lo = D.lo + D.g_off[c];
    const double* hi = D.hi + D.g_off[c];
    for (int r = t; r < nc; r += kFT) {
      const double p = eta[co + r] + al * val[r];
      eo[co + r] = p - al * fmin(fmax(p / al, lo[r]), hi[r]);
    }
    __syncthreads();
  } else {  // leaf: G_N x^ (box) and the terminal SOC block of (x, s)
    const int j = c - D.nnl, nc = D.s3_nc[j], eo3 = D.s3_off[j], p = pN;
    if (D.gN_diag) {
      const double* gd = D.gNd + size_t(j) * nx;
      for (int r = t; r < nc; r += kFT) val[r] = gd[r] * hat[r];
    } else {
      cta_gemv(D.GN + D.gN_off[j] * nx, nc, nx, nc, hat, val, false, red);
    }
    __syncthreads();
    const double* lo = D.loN + D.gN_off[j];
    const double* hi = D.hiN + D.gN_off[j];
    for (int r = t; r < nc; r += kFT) {
      const double pp = eta[eo3 + r] + al * val[r];
      eo[eo3 + r] = pp - al * fmin(fmax(pp / al, lo[r]), hi[r]);
    }
    __syncthreads();
    const double* qk = D.qkN + size_t(j) * nx;
    double part = 0.0;
    for (int r = t; r < nx; r += kFT) part += qk[r] * hat[r];
    const double qd = cta_sum(part, red);
    cta_gemv(HN, p, nx, p, hat, val, false, red);
    if (t == 0) {
      const double row = 0.5 * hatv(D.s_base + c - 1) - 0.5 * qd;
      val[p] = row;
      val[p + 1] = row;
    }
    __syncthreads();
    const int so = eo3 + nc;
    dual(so, p + 2);
    cta_soc_project(pv, D.aN + D.aN_off[j], p + 2, red);
    for (int r = t; r < p + 2; r += kFT) eo[so + r] = val[r] - al * pv[r];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kFT, 1) k_T_fused(FusedArgs F) {
  extern __shared__ __align__(1024) double dsm[];
  __shared__ Smem S;
  __shared__ int ticket;
  const int t = threadIdx.x;
  if (t == 0) {
    mbar_init(&S.bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    S.mat = dsm;
    S.vec = dsm + F.mat_doubles;
    S.red = S.vec + kSlots * kSlot;
  }
  __syncthreads();
  uint32_t phase = 0;
  const int nnl = F.D.nnl, nn = F.D.nn, total = nnl + 2 * nn;
  for (;;) {
    if (t == 0) ticket = int(atomicAdd(F.ticket, 1ull));
    __syncthreads();
    const int it = ticket;
    __syncthreads();
    if (it >= total) break;
    if (it < nnl) {
      item_s2(F, it, S.red, S.vec);
      __threadfence();
      __syncthreads();
      if (t == 0) st_release(F.flagS2 + it, 1);
    } else if (it < nnl + nn) {
      item_back(F, nn - 1 - (it - nnl), S, phase);
    } else {
      item_fwd(F, it - nnl - nn, S, phase);
    }
  }
}

}  // namespace

int fused_smem_bytes(const FusedArgs& F) {
  return int(sizeof(double) * (F.mat_doubles + kSlots * kSlot + 2 * kFT));
}

cudaError_t fused_configure(int smem_bytes) {
  return cudaFuncSetAttribute(k_T_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
}

const void* fused_kernel_ptr() { return reinterpret_cast<const void*>(&k_T_fused); }

void launch_T_fused(const FusedArgs& F, int grid, cudaStream_t st) {
  k_T_fused<<<grid, kFT, fused_smem_bytes(F), st>>>(F);
}

}  // namespace spock
