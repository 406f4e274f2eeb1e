// (wide_impl.cuh: the kernel body, included by wide.cu and the wide_r*.cu
// instantiation units.)
// One CP application T for wide trees as a persistent, warp-granular dataflow
// kernel with per-warp TMA streaming rings (sm_100a).
//
// Same items, order and arithmetic as the CTA-granular kernel of fused.cu
// (backward nn-1..0, S2 of every parent, forward 0..nn-1; an item only waits
// on items with smaller tickets), but sized for trees whose matrices do not fit
// on chip and whose per-T cost is streaming them once from HBM:
//
//  * one item per WARP, tickets assigned round-robin (ticket = warp + j*NW), so
//    the whole schedule of a warp is known in advance and no CTA barrier sits
//    on any path (a warp waits only on its own ring and on dependency flags);
//  * per ticket a 256-byte host-built record (WRec) arrives by bulk copy three
//    tickets ahead: node metadata, the matrices to stream, the vector spans;
//  * every node matrix streams through a per-warp ring of S shared-memory
//    slots, one cp.async.bulk (TMA bulk copy, mbarrier completion) per column
//    chunk.  Lane 0 runs the producer S chunks ahead of the consumer, across
//    item boundaries and across dependency waits;
//  * the item's independent vector operands (z and eta segments, SOC data,
//    boxes, ...) are staged by bulk copies (16-byte aligned supersets) when the
//    item starts, in parallel with the dependency-flag waits and the loads of
//    what other items produced, so an item pays about one memory round trip
//    before its arithmetic;
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
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "dev.cuh"
#include "kernels.hpp"
#include "wide.hpp"

namespace spock {

namespace {

constexpr int kMaxSlots = 16;
constexpr int kRecSlots = 4;  // record ring: tickets j .. j+3

// span ids (WRec::voff/vcnt/vbase index); leaf items alias the non-leaf ids
enum : int { B_HEAD = 0, B_QK, B_ZX, B_ZU, B_EC, B_GD, B_H, B_G };
enum : int { B_SEG3 = B_ZU, B_GDN = B_GD, B_QKN = B_H };
enum : int { F_ZX = 0, F_ZU, F_AX, F_AU, F_CV, F_SEG2, F_A, F_QK, F_SEG1, F_RB, F_GD, F_LO, F_HI, F_ZY, F_ZT, F_ZS };
enum : int { F_SEG3 = F_SEG1, F_AN = F_RB, F_QKN = F_GD, F_GDN = F_LO, F_LON = F_HI, F_HIN = F_ZY };
// standalone L (kind 3), L* child terms (kind 4), L* node rows (kind 5)
enum : int { L_ZX = 0, L_ZU, L_AX, L_AU, L_QK, L_ZT, L_ZS, L_Y, L_RB, L_GD, L_QKN };
enum : int { L_GDN = L_GD };
enum : int { LC_HEAD = 0, LC_QK };
enum : int { LN_SEG1 = 0, LN_RB, LN_GD, LN_QKN };
enum : int { LN_SEG3 = LN_SEG1, LN_GDN = LN_GD };

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
// bulk prefetch of [src, src + bytes) into L2 (no shared memory involved)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
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

__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// poll relaxed (an acquire load invalidates L1 on every poll), then one acquire
// load of the released value
__device__ void wait_flag(const int* f) {
  int k = 0;
  while (ld_relaxed(f) < 1)
    if (++k > 16) __nanosleep(64);
  (void)ld_acquire(f);
}
// warp barrier (orders every lane's writes before lane 0's), then one release
// store by lane 0 (st.release is cumulative over the writes it has observed)
__device__ __forceinline__ void w_release(int* f) {
  __syncwarp();
  if (lane_id() == 0) st_release(f, 1);
}

struct MatD {
  const double* p;
  int rows, cols, cc;
};

// producer cursor of a warp's ring (shared memory, touched by lane 0 only)
struct Prod {
  uint32_t prod;  // chunks issued
  int jp;         // ticket index (of this warp) the producer is on
  int have;       // matrix list of ticket jp copied from its record
  int mi, co, nm;
  MatD md[kWMats];
};

struct Ring {
  double* buf;
  uint64_t* bar;
  Prod* ps;
  WRec* rb;  // record ring (kRecSlots)
  uint64_t* rbar;
  const WRec* rc;  // record of the item being consumed
  int mk;          // next streamed matrix of that item
  int S, sshift, chunk, stride, total, gw;
  bool prof;
  int jc;         // ticket index the consumer is on
  uint32_t cons;  // chunks consumed (uniform across the warp)
  long long t_ring, t_flag;  // optional profile: cycles waiting on chunks / dependency flags
  long long t_span, t_refill;  // ... on staged spans / in the producer
};

// lane 0: keep S chunks in flight, walking this warp's tickets ahead of the
// consumer (at most two tickets ahead: records are requested three ahead)
__device__ __forceinline__ void refill(Prod* __restrict__ P, WRec* rb, uint64_t* rbar, uint32_t cons, int jc, int S,
                                    int chunk, double* buf, uint64_t* bar, int stride, int total, int gw) {
  // S is a power of two
  while (P->prod < cons + uint32_t(S)) {
    for (;;) {
      if (gw + P->jp * stride >= total) return;
      if (!P->have) {
        if (P->jp > jc + 2) return;
        const int s = P->jp & (kRecSlots - 1);
        const uint32_t par = uint32_t(P->jp / kRecSlots) & 1u;
        while (!mbar_try_wait(&rbar[s], par)) {
        }
        const WRec& rc = rb[s];
        P->nm = rc.nmat;
        for (int k = 0; k < rc.nmat; ++k) P->md[k] = MatD{rc.mp[k], rc.mrows[k], rc.mcols[k], rc.mcc[k]};
        P->mi = 0;
        P->co = 0;
        P->have = 1;
      }
      if (P->mi < P->nm) {
        const MatD& M = P->md[P->mi];
        if (M.rows > 0 && P->co < M.cols) break;
        ++P->mi;
        P->co = 0;
        continue;
      }
      ++P->jp;
      P->have = 0;
    }
    const MatD M = P->md[P->mi];
    const int cc = min(M.cc, M.cols - P->co);
    const uint32_t bytes = (uint32_t(cc) * uint32_t(M.rows) * 8u + 15u) & ~15u;
    const int slot = int(P->prod & uint32_t(S - 1));
    fence_proxy_async();
    mbar_expect_tx(&bar[slot], bytes);
    bulk_g2s(buf + size_t(slot) * chunk, M.p + size_t(P->co) * M.rows, bytes, &bar[slot]);
    ++P->prod;
    P->co += cc;
  }
}

__device__ __forceinline__ void refill_lane0(Ring& R) {
  long long t0 = 0;
  if (R.prof) t0 = clock64();
  if (lane_id() == 0) refill(R.ps, R.rb, R.rbar, R.cons, R.jc, R.S, R.chunk, R.buf, R.bar, R.stride, R.total, R.gw);
  if (R.prof) {
    __syncwarp();
    R.t_refill += clock64() - t0;
  }
}

// acc[k] += sum_{c < cc} A[(lane + 32k) + c*rows] x[c], A in shared memory
// (a second, interleaved accumulator chain measured no faster: the warp is not
// bound by the DFMA chain but by the instructions around it)
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

// consume the chunks of the item's next streamed matrix (record order): acc += M x
template <int RR>
__device__ __forceinline__ void sgemv(Ring& R, const double* x, double (&acc)[RR]) {
  const int k = R.mk++;
  const int rows = R.rc->mrows[k], cols = R.rc->mcols[k], ccmax = R.rc->mcc[k];
  if (rows <= 0) return;
  for (int co = 0; co < cols; co += ccmax) {
    const int cc = min(ccmax, cols - co);
    const int slot = int(R.cons & uint32_t(R.S - 1));
    const uint32_t par = (R.cons >> R.sshift) & 1u;
    if (R.prof) {
      const long long t0 = clock64();  // try_wait may suspend: time the whole wait
      while (!mbar_try_wait(&R.bar[slot], par)) {
      }
      R.t_ring += clock64() - t0;
    } else {
      while (!mbar_try_wait(&R.bar[slot], par)) {
      }
    }
    gemv_cols<RR>(R.buf + size_t(slot) * R.chunk, rows, cc, x + co, acc);
    __syncwarp();
    ++R.cons;
    refill_lane0(R);
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
__device__ void soc_proj(double (&v)[RR], int p, double& vp, double& vp1, const double* a) {
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
// Staged vector operands of one item.
struct Spans {
  const WideArgs* A;
  const WRec* rc;
  const double* vrec;
  const int* doff;
  __device__ __forceinline__ const double* base(int b) const {
    return b == WB_Z ? A->z : (b == WB_ETA ? A->eta : A->vb[b]);
  }
  __device__ __forceinline__ const double* operator()(int id) const {
    if ((rc->unstaged >> id) & 1) return base(rc->vbase[id]) + rc->voff[id];
    return vrec + doff[id];
  }
};

// bulk-copy the item's staged spans (16-byte aligned supersets) into vrec, one
// span per lane (offsets by a warp prefix sum); one mbarrier phase per item
// (completes at once when nothing is staged)
__device__ void stage_spans(const WideArgs& A, const WRec& rc, double* vrec, int* doff, uint64_t* sbar) {
  const int l = lane_id();
  // z / eta may be 8-byte aligned sub-vectors (SuperMann's stacked (z | eta)):
  // the alignment shift is taken from the address
  int nn = 0, sh = 0;
  const double* src = nullptr;
  if (l < rc.nspan) {
    const int n = rc.vcnt[l];
    if (!(((rc.unstaged >> l) & 1) || n == 0)) {
      const int b = rc.vbase[l];
      src = (b == WB_Z ? A.z : (b == WB_ETA ? A.eta : A.vb[b])) + rc.voff[l];
      sh = int((reinterpret_cast<uintptr_t>(src) >> 3) & 1);
      nn = (n + sh + 1) & ~1;
    }
  }
  int incl = nn;  // inclusive prefix sum over the lanes (span order)
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (l >= o) incl += v;
  }
  const int off = incl - nn;
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  if (l < rc.nspan) doff[l] = nn ? off + sh : 0;
  if (l == 0) {
    fence_proxy_async();
    mbar_expect_tx(sbar, uint32_t(total) * 8u);
  }
  __syncwarp();
  if (nn) {
    fence_proxy_async();
    bulk_g2s(vrec + off, src - sh, uint32_t(nn) * 8u, sbar);
  }
}

struct SpanWait {
  uint64_t* bar;
  uint32_t parity;
};
__device__ __forceinline__ void spans_ready(Ring& R, const SpanWait& W) {
  long long t0 = 0;
  if (R.prof) t0 = clock64();
  while (!mbar_try_wait(W.bar, W.parity)) {
  }
  // the lanes' dependency loads into shared scratch (xs, dep) are read by other
  // lanes from here on: order them explicitly (independent thread scheduling)
  __syncwarp();
  if (R.prof) R.t_span += clock64() - t0;
}

// ---------------------------------------------------------------------------
// Backward item of node i.  Streamed (record order): HxT, HuT (non-root) |
// HNT (leaf) or KT, Rinv (non-leaf) | M1T (non-root).
template <int RR>
__device__ void w_back(const WideArgs& A, Ring& R, const WRec& rc, const Spans& sp, const SpanWait& W, double* xs,
                       double* xs2) {
  const Dev& D = A.D;
  const int l = lane_id(), nx = D.nx, nu = D.nu, m = nx + nu;
  const double al = A.alpha;
  const int i = rc.node;
  const bool root = i == 0, leaf = rc.nch == 0;
  // children: flags, then their adj (L* stage-cost terms) and T12 sums
  double vx[RR], vu[RR], sx[RR], su[RR];
  zero(vx);
  zero(vu);
  zero(sx);
  zero(su);
  if (!leaf) {
    const int c0 = rc.c0, nch = rc.nch;
    long long t0 = 0;
    if (R.prof) t0 = clock64();
    for (int k = l; k < nch; k += 32) wait_flag(A.flagB + c0 + k);
    __syncwarp();
    if (R.prof) R.t_flag += clock64() - t0;
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
  }
  spans_ready(R, W);
  double acc[RR];
  if (!root) {  // own stage-SOC adjoint term for the parent (tree_operator.cpp:80-88)
    const int k = i - 1, px = rc.px, pu = rc.pu, p = px + pu;
    const double* head = sp(B_HEAD);
    const double rsum = head[p] + head[p + 1];
    const double* qk = sp(B_QK);
    double* adj = D.adj + size_t(k) * m;
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      acc[kk] = r < nx ? -0.5 * rsum * qk[r] : 0.0;
    }
    sgemv<RR>(R, head, acc);
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
    sgemv<RR>(R, head + px, acc);
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < nu) adj[nx + r] = acc[kk];
    }
  }
  const double* zx = sp(B_ZX);
  if (leaf) {  // L* leaf rows, then q = -xbar and T12 = M1' q
    const int j = i - D.nnl, nc = rc.nc, pN = rc.pN;
    const double* ec = sp(B_SEG3);
    const double* hd = ec + nc;
    const double rsumN = hd[pN] + hd[pN + 1];
    zero(acc);
    if (D.gN_diag) {
      const double* gd = sp(B_GDN);
#pragma unroll
      for (int kk = 0; kk < RR; ++kk) {
        const int r = l + 32 * kk;
        if (r < nx) acc[kk] = gd[r] * ec[r];
      }
    } else {
      gemv_glob<RR>(D.GNT + D.gN_off[j] * nx, nx, nc, nx, ec, acc);
    }
    sgemv<RR>(R, hd, acc);
    const double* qk = sp(B_QKN);
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < nx) xs[r] = -(zx[r] - al * (acc[kk] - 0.5 * rsumN * qk[r]));
    }
    __syncwarp();
    if (!root) {
      zero(acc);
      sgemv<RR>(R, xs, acc);
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
  // non-leaf: (xbar, ubar) = (z_x, z_u) - alpha (G' ec + sum_c adj_c)
  const int nc = rc.nc;
  const double* ecs = sp(B_EC);  // [s-row; constraint rows]
  const double* ec = ecs + 1;
  double gx[RR], gu[RR];
  zero(gx);
  zero(gu);
  if (D.g_diag) {
    const double* gd = sp(B_GD);
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < nx) gx[kk] = gd[r] * ec[r];
      if (r < nu) gu[kk] = gd[nx + r] * ec[nx + r];
    }
  } else {
    gemv_glob<RR>(D.GxT + D.g_off[i] * nx, nx, nc, nx, ec, gx);
    gemv_glob<RR>(D.GuT + D.g_off[i] * nu, nu, nc, nu, ec, gu);
  }
  const double* zu = sp(B_ZU);
  const double* gv = sp(B_G);
#pragma unroll
  for (int kk = 0; kk < RR; ++kk) {
    const int r = l + 32 * kk;
    if (r < nu) {
      const double ub = zu[r] - al * (gu[kk] + vu[kk]);
      xs[r] = ub;
      xs2[r] = ub - gv[r] - su[kk];
    }
  }
  __syncwarp();
  zero(acc);
  sgemv<RR>(R, xs, acc);  // K' ubar
  const double* h = sp(B_H);
  double q[RR];
#pragma unroll
  for (int kk = 0; kk < RR; ++kk) {
    const int r = l + 32 * kk;
    q[kk] = r < nx ? h[r] - (zx[r] - al * (gx[kk] + vx[kk])) - acc[kk] + sx[kk] : 0.0;
  }
  zero(acc);
  sgemv<RR>(R, xs2, acc);  // d = Rt^-1 (ubar - g - sum B'q)
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
    sgemv<RR>(R, xs, acc);  // T12 = [Abar' q; B' q]
    double* T12 = D.T12 + size_t(i - 1) * m;
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < m) T12[r] = acc[kk];
    }
  } else if (l == 0) {
    A.zo[0] = A.z[0] - al * ecs[0] - al;  // CP primal step on s0 (solver.cpp:153-154)
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
// Streamed (record order): M1 (non-root) | K (non-leaf) | Hx, Hu (non-root) |
// HN (leaf).  dep: [u+_anc (nu) | d_c (nu) | tau+_c | s+_c | y+_c (ny <= ycap)]
template <int RR>
__device__ void w_fwd(const WideArgs& A, Ring& R, const WRec& rc, const Spans& sp, const SpanWait& W, double* xs,
                      double* xs2, double* dep) {
  const Dev& D = A.D;
  const int l = lane_id(), nx = D.nx, nu = D.nu;
  const double al = A.alpha;
  double* zo = A.zo;
  double* eo = A.eo;
  const int c = rc.node;
  const bool root = c == 0, leaf = rc.nch == 0;
  const int an = root ? 0 : rc.anc;
  const int ny = leaf ? 0 : rc.ny;
  const bool ystage = ny <= A.ycap;
  // dependencies: parent forward (root: the root's backward item), S2 of c and of the parent
  {
    long long t0 = 0;
    if (R.prof) t0 = clock64();
    if (l == 0) wait_flag(root ? A.flagB : A.flagF + an);
    if (l == 1 && !leaf) wait_flag(A.flagS2 + c);
    if (l == 2 && !root) wait_flag(A.flagS2 + an);
    __syncwarp();
    if (R.prof) R.t_flag += clock64() - t0;
  }
  // everything other items produced for this one, in one batch of L2 loads
  if (!root) {
    for (int r = l; r < nx; r += 32) xs[r] = ldcg(zo + 1 + size_t(an) * nx + r);
    for (int r = l; r < nu; r += 32) {
      xs[nx + r] = ldcg(D.dvec + size_t(an) * nu + r);
      dep[r] = ldcg(zo + D.u_base + size_t(an) * nu + r);
    }
    if (l == 0) dep[2 * nu] = ldcg(zo + D.tau_base + c - 1);
  }
  if (!leaf)
    for (int r = l; r < nu; r += 32) dep[nu + r] = ldcg(D.dvec + size_t(c) * nu + r);
  if (l == 0) dep[2 * nu + 1] = ldcg(zo + (root ? 0 : D.s_base + c - 1));
  if (ystage)
    for (int r = l; r < ny; r += 32) dep[2 * nu + 2 + r] = ldcg(zo + rc.yo + r);
  spans_ready(R, W);
  double x[RR], u[RR];
  zero(u);
  if (root) {
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      x[kk] = r < nx ? D.xinit[r] : 0.0;
    }
  } else {
    zero(x);
    sgemv<RR>(R, xs, x);  // [Abar B][x_anc; d_anc]
    const double* cv = sp(F_CV);
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
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < nx) xs2[r] = x[kk];
    }
    __syncwarp();
    sgemv<RR>(R, xs2, u);  // K x
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < nu) {
        u[kk] += dep[nu + r];
        zo[D.u_base + size_t(c) * nu + r] = u[kk];
      }
    }
  }
  w_release(A.flagF + c);  // children need only (x+, u+) and d
  // ---- dual update on the segments owned by c (k_L<DUAL>): p = eta + a L w,
  // w = 2 z+ - z, eta+ = p - a Pi_S3(p / a)
  double hx[RR], hu[RR];
  {
    const double* zx = sp(F_ZX);
    const double* zu = leaf ? nullptr : sp(F_ZU);
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      hx[kk] = r < nx ? 2.0 * x[kk] - zx[r] : 0.0;
      hu[kk] = (!leaf && r < nu) ? 2.0 * u[kk] - zu[r] : 0.0;
    }
  }
  const double hs = 2.0 * dep[2 * nu + 1] - sp(F_ZS)[0];  // w on s_c
  double acc[RR];
  if (!leaf) {
    const int so = rc.so;
    const double* seg1 = sp(F_SEG1);
    const double* rb = sp(F_RB);
    const double* zy = sp(F_ZY);
    auto hy = [&](int r) { return 2.0 * (ystage ? dep[2 * nu + 2 + r] : ldcg(zo + rc.yo + r)) - zy[r]; };
    double part = 0.0;
    for (int r = l; r < ny; r += 32) {
      const double yv = hy(r);
      part += rb[r] * yv;
      eo[so + r] = (seg1[r] + al * yv) / al;  // staged p/a, projected below
    }
    const double by = warp_sum(part);
    __syncwarp();
    ycone(D, c, eo + so);
    for (int r = l; r < ny; r += 32) {
      const double pv = seg1[r] + al * hy(r);
      eo[so + r] = pv - al * eo[so + r];
    }
    if (l == 0) {
      const double pv = seg1[ny] + al * (hs - by);
      eo[so + ny] = pv - al * fmax(0.0, pv / al);
    }
    const int nc = rc.nc;
    zero(acc);
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < nx) xs2[r] = hx[kk];
      if (r < nu) xs2[nx + r] = hu[kk];
    }
    __syncwarp();
    if (D.g_diag) {  // constraint row r uses [x^; u^]_r (diagonal [Gx Gu])
      const double* gd = sp(F_GD);
#pragma unroll
      for (int kk = 0; kk < RR; ++kk) {
        const int r = l + 32 * kk;
        if (r < nc) acc[kk] = gd[r] * xs2[r];
      }
    } else {
      gemv_glob<RR>(D.Gx + D.g_off[c] * nx, nc, nx, nc, xs2, acc);
      gemv_glob<RR>(D.Gu + D.g_off[c] * nu, nc, nu, nc, xs2 + nx, acc);
    }
    const double* lo = sp(F_LO);
    const double* hi = sp(F_HI);
    const double* ec = seg1 + ny + 1;
    const int co = so + ny + 1;
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < nc) {
        const double pv = ec[r] + al * acc[kk];
        eo[co + r] = pv - al * fmin(fmax(pv / al, lo[r]), hi[r]);
      }
    }
    __syncwarp();
  }
  if (!root) {  // stage-cost SOC block of (x^_anc, u^_anc, tau^_c)
    const int px = rc.px, pu = rc.pu, p = px + pu, so = rc.s2o;
    const double* zax = sp(F_AX);
    const double* zau = sp(F_AU);
    // xs holds [x+_anc; d_anc]: w_anc = [2 x+_anc - z_x; 2 u+_anc - z_u] into xs2
    for (int r = l; r < nx; r += 32) xs2[r] = 2.0 * xs[r] - zax[r];
    for (int r = l; r < nu; r += 32) xs2[nx + r] = 2.0 * dep[r] - zau[r];
    __syncwarp();
    const double* qk = sp(F_QK);
    double part = 0.0;
    for (int r = l; r < nx + nu; r += 32) part += qk[r] * xs2[r];
    const double qd = warp_sum(part);
    const double row = 0.5 * (2.0 * dep[2 * nu] - sp(F_ZT)[0]) - 0.5 * qd;
    double ax[RR], au[RR];
    zero(ax);
    zero(au);
    sgemv<RR>(R, xs2, ax);       // Hx x^
    sgemv<RR>(R, xs2 + nx, au);  // Hu u^
    // realign [Hx x^; Hu u^] (p rows) through shared memory
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < px) xs[r] = ax[kk];
      if (r < pu) xs[px + r] = au[kk];
    }
    __syncwarp();
    const double* seg2 = sp(F_SEG2);
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      acc[kk] = r < p ? seg2[r] + al * xs[r] : 0.0;
    }
    double vp = seg2[p] + al * row, vp1 = seg2[p + 1] + al * row;
    double t[RR];
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) t[kk] = acc[kk] / al;
    double tp = vp / al, tp1 = vp1 / al;
    soc_proj<RR>(t, p, tp, tp1, sp(F_A));
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
    const int j = c - D.nnl, nc = rc.nc, p = rc.pN, eo3 = rc.so;
    const double* seg3 = sp(F_SEG3);
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < nx) xs2[r] = hx[kk];
    }
    __syncwarp();
    zero(acc);
    if (D.gN_diag) {
      const double* gd = sp(F_GDN);
#pragma unroll
      for (int kk = 0; kk < RR; ++kk) {
        const int r = l + 32 * kk;
        if (r < nc) acc[kk] = gd[r] * xs2[r];
      }
    } else {
      gemv_glob<RR>(D.GN + D.gN_off[j] * nx, nc, nx, nc, xs2, acc);
    }
    const double* lo = sp(F_LON);
    const double* hi = sp(F_HIN);
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < nc) {
        const double pv = seg3[r] + al * acc[kk];
        eo[eo3 + r] = pv - al * fmin(fmax(pv / al, lo[r]), hi[r]);
      }
    }
    const double* qk = sp(F_QKN);
    double part = 0.0;
    for (int r = l; r < nx; r += 32) part += qk[r] * xs2[r];
    const double qd = warp_sum(part);
    const double row = 0.5 * hs - 0.5 * qd;
    zero(acc);
    sgemv<RR>(R, xs2, acc);  // H_N x^
    const double* hseg = seg3 + nc;
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      acc[kk] = r < p ? hseg[r] + al * acc[kk] : 0.0;
    }
    double vp = hseg[p] + al * row, vp1 = hseg[p + 1] + al * row;
    double t[RR];
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) t[kk] = acc[kk] / al;
    double tp = vp / al, tp1 = vp1 / al;
    soc_proj<RR>(t, p, tp, tp1, sp(F_AN));
    const int so = eo3 + nc;
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

// ---------------------------------------------------------------------------
// Standalone L (TreeOperator::apply, tree_operator.cpp:20-63): eta_out = L z,
// all rows owned by node i.  Streamed: Hx, Hu (non-root) | HN (leaf).
template <int RR>
__device__ void w_L(const WideArgs& A, Ring& R, const WRec& rc, const Spans& sp, const SpanWait& W, double* xs,
                    double* xs2) {
  const Dev& D = A.D;
  const int l = lane_id(), nx = D.nx, nu = D.nu;
  double* eo = A.eo;
  const int i = rc.node;
  const bool root = i == 0, leaf = rc.nch == 0;
  spans_ready(R, W);
  double acc[RR];
  if (!leaf) {  // y-copy rows, risk scalar s - b'y, constraint rows G [x; u]
    const int ny = rc.ny, so = rc.so, nc = rc.nc;
    const double* zy = sp(L_Y);
    const double* rb = sp(L_RB);
    double part = 0.0;
    for (int r = l; r < ny; r += 32) {
      const double yv = zy[r];
      part += rb[r] * yv;
      eo[so + r] = yv;
    }
    const double by = warp_sum(part);
    if (l == 0) eo[so + ny] = sp(L_ZS)[0] - by;
    const double* zx = sp(L_ZX);
    const double* zu = sp(L_ZU);
    for (int r = l; r < nx; r += 32) xs[r] = zx[r];
    for (int r = l; r < nu; r += 32) xs[nx + r] = zu[r];
    __syncwarp();
    zero(acc);
    if (D.g_diag) {
      const double* gd = sp(L_GD);
#pragma unroll
      for (int kk = 0; kk < RR; ++kk) {
        const int r = l + 32 * kk;
        if (r < nc) acc[kk] = gd[r] * xs[r];
      }
    } else {
      gemv_glob<RR>(D.Gx + D.g_off[i] * nx, nc, nx, nc, xs, acc);
      gemv_glob<RR>(D.Gu + D.g_off[i] * nu, nc, nu, nc, xs + nx, acc);
    }
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < nc) eo[so + ny + 1 + r] = acc[kk];
    }
    __syncwarp();
  }
  if (!root) {  // stage-cost SOC block of (x_anc, u_anc, tau_i)
    const int px = rc.px, pu = rc.pu, p = px + pu, o2 = rc.s2o;
    const double* zax = sp(L_AX);
    const double* zau = sp(L_AU);
    for (int r = l; r < nx; r += 32) xs2[r] = zax[r];
    for (int r = l; r < nu; r += 32) xs2[nx + r] = zau[r];
    __syncwarp();
    const double* qk = sp(L_QK);
    double part = 0.0;
    for (int r = l; r < nx + nu; r += 32) part += qk[r] * xs2[r];
    const double qd = warp_sum(part);
    double ax[RR], au[RR];
    zero(ax);
    zero(au);
    sgemv<RR>(R, xs2, ax);       // Hx x_anc
    sgemv<RR>(R, xs2 + nx, au);  // Hu u_anc
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < px) eo[o2 + r] = ax[kk];
      if (r < pu) eo[o2 + px + r] = au[kk];
    }
    if (l == 0) {
      const double row = 0.5 * sp(L_ZT)[0] - 0.5 * qd;
      eo[o2 + p] = row;
      eo[o2 + p + 1] = row;
    }
    __syncwarp();
  }
  if (leaf) {  // G_N x and the terminal SOC block of (x, s)
    const int j = i - D.nnl, nc = rc.nc, p = rc.pN, e3 = rc.so;
    const double* zx = sp(L_ZX);
    for (int r = l; r < nx; r += 32) xs[r] = zx[r];
    __syncwarp();
    zero(acc);
    if (D.gN_diag) {
      const double* gd = sp(L_GDN);
#pragma unroll
      for (int kk = 0; kk < RR; ++kk) {
        const int r = l + 32 * kk;
        if (r < nc) acc[kk] = gd[r] * xs[r];
      }
    } else {
      gemv_glob<RR>(D.GN + D.gN_off[j] * nx, nc, nx, nc, xs, acc);
    }
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < nc) eo[e3 + r] = acc[kk];
    }
    const double* qk = sp(L_QKN);
    double part = 0.0;
    for (int r = l; r < nx; r += 32) part += qk[r] * xs[r];
    const double qd = warp_sum(part);
    zero(acc);
    sgemv<RR>(R, xs, acc);  // H_N x
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < p) eo[e3 + nc + r] = acc[kk];
    }
    if (l == 0) {
      const double row = 0.5 * sp(L_ZS)[0] - 0.5 * qd;
      eo[e3 + nc + p] = row;
      eo[e3 + nc + p + 1] = row;
    }
  }
}

// L* child terms of node i (tree_operator.cpp:80-88): adj_i = H_i' head_i -
// rsum/2 qk_i for the parent, and the tau_i slot.  Streamed: HxT, HuT.
template <int RR>
__device__ void w_Lt_child(const WideArgs& A, Ring& R, const WRec& rc, const Spans& sp, const SpanWait& W) {
  const Dev& D = A.D;
  const int l = lane_id(), nx = D.nx, nu = D.nu, m = nx + nu;
  const int i = rc.node, k = i - 1, px = rc.px, pu = rc.pu, p = px + pu;
  spans_ready(R, W);
  const double* head = sp(LC_HEAD);
  const double rsum = head[p] + head[p + 1];
  const double* qk = sp(LC_QK);
  double* adj = D.adj + size_t(k) * m;
  double acc[RR];
#pragma unroll
  for (int kk = 0; kk < RR; ++kk) {
    const int r = l + 32 * kk;
    acc[kk] = r < nx ? -0.5 * rsum * qk[r] : 0.0;
  }
  sgemv<RR>(R, head, acc);
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
  sgemv<RR>(R, head + px, acc);
#pragma unroll
  for (int kk = 0; kk < RR; ++kk) {
    const int r = l + 32 * kk;
    if (r < nu) adj[nx + r] = acc[kk];
  }
  if (l == 0) A.zo[D.tau_base + k] = 0.5 * rsum;
  w_release(A.flagB + i);
}

// L* rows of node i (tree_operator.cpp:75-79,89-113): own segments plus the
// ascending sum of the children's adj.  Streamed: HNT (leaf).
template <int RR>
__device__ void w_Lt_node(const WideArgs& A, Ring& R, const WRec& rc, const Spans& sp, const SpanWait& W) {
  const Dev& D = A.D;
  const int l = lane_id(), nx = D.nx, nu = D.nu, m = nx + nu;
  double* zo = A.zo;
  const int i = rc.node;
  const bool leaf = rc.nch == 0;
  double vx[RR], vu[RR];
  zero(vx);
  zero(vu);
  if (!leaf) {
    const int c0 = rc.c0, nch = rc.nch;
    long long t0 = 0;
    if (R.prof) t0 = clock64();
    for (int k = l; k < nch; k += 32) wait_flag(A.flagB + c0 + k);
    __syncwarp();
    if (R.prof) R.t_flag += clock64() - t0;
    for (int c = 0; c < nch; ++c) {  // ascending child order
      const double* ad = D.adj + size_t(c0 + c - 1) * m;
#pragma unroll
      for (int kk = 0; kk < RR; ++kk) {
        const int r = l + 32 * kk;
        if (r < nx) vx[kk] += ldcg(ad + r);
        if (r < nu) vu[kk] += ldcg(ad + nx + r);
      }
    }
  }
  spans_ready(R, W);
  if (!leaf) {
    const int ny = rc.ny, yo = rc.yo, nc = rc.nc;
    const double* seg1 = sp(LN_SEG1);
    const double* rb = sp(LN_RB);
    const double sc = seg1[ny];
    for (int r = l; r < ny; r += 32) zo[yo + r] = seg1[r] - sc * rb[r];
    if (l == 0) zo[i == 0 ? 0 : D.s_base + i - 1] = sc;
    const double* ec = seg1 + ny + 1;
    double gx[RR], gu[RR];
    zero(gx);
    zero(gu);
    if (D.g_diag) {
      const double* gd = sp(LN_GD);
#pragma unroll
      for (int kk = 0; kk < RR; ++kk) {
        const int r = l + 32 * kk;
        if (r < nx) gx[kk] = gd[r] * ec[r];
        if (r < nu) gu[kk] = gd[nx + r] * ec[nx + r];
      }
    } else {
      gemv_glob<RR>(D.GxT + D.g_off[i] * nx, nx, nc, nx, ec, gx);
      gemv_glob<RR>(D.GuT + D.g_off[i] * nu, nu, nc, nu, ec, gu);
    }
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < nx) zo[1 + size_t(i) * nx + r] = gx[kk] + vx[kk];
      if (r < nu) zo[D.u_base + size_t(i) * nu + r] = gu[kk] + vu[kk];
    }
  } else {
    const int j = i - D.nnl, nc = rc.nc, p = rc.pN;
    const double* ec = sp(LN_SEG3);
    const double* hd = ec + nc;
    const double rsum = hd[p] + hd[p + 1];
    double acc[RR];
    zero(acc);
    if (D.gN_diag) {
      const double* gd = sp(LN_GDN);
#pragma unroll
      for (int kk = 0; kk < RR; ++kk) {
        const int r = l + 32 * kk;
        if (r < nx) acc[kk] = gd[r] * ec[r];
      }
    } else {
      gemv_glob<RR>(D.GNT + D.gN_off[j] * nx, nx, nc, nx, ec, acc);
    }
    sgemv<RR>(R, hd, acc);
    const double* qk = sp(LN_QKN);
#pragma unroll
    for (int kk = 0; kk < RR; ++kk) {
      const int r = l + 32 * kk;
      if (r < nx) zo[1 + size_t(i) * nx + r] = acc[kk] - 0.5 * rsum * qk[r];
    }
    if (l == 0) zo[D.s_base + i - 1] = 0.5 * rsum;
  }
}

// per-warp shared-memory footprint in doubles (16-byte multiples)
__host__ __device__ __forceinline__ size_t warp_doubles(int S, int CH, int VR, int VD) {
  return size_t(S) * CH + size_t(VR) + 3 * size_t(VD) + kRecSlots * 32 + 8 /*doff*/ + kMaxSlots + kRecSlots + 2;
}

template <int RR, int MINB>
__global__ void __launch_bounds__(256, MINB) k_T_wide(const __grid_constant__ WideArgs A) {
  extern __shared__ __align__(128) double wsm[];
  const int w = threadIdx.x >> 5, l = lane_id();
  const int S = A.slots, CH = A.chunk, VR = A.vrec, VD = A.vecd;
  double* ring = wsm + size_t(w) * warp_doubles(S, CH, VR, VD);
  double* vrec = ring + size_t(S) * CH;
  double* xs = vrec + VR;
  double* xs2 = xs + VD;
  double* dep = xs2 + VD;
  WRec* rb = reinterpret_cast<WRec*>(dep + VD);
  int* doff = reinterpret_cast<int*>(reinterpret_cast<double*>(rb) + kRecSlots * 32);
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<double*>(doff) + 8);
  uint64_t* rbar = bars + kMaxSlots;
  uint64_t* sbar = rbar + kRecSlots;
  __shared__ Prod prods[8];
  Prod* P = &prods[w];
  Ring R;
  R.ps = P;
  R.buf = ring;
  R.bar = bars;
  R.rb = rb;
  R.rbar = rbar;
  R.S = S;
  R.sshift = __ffs(S) - 1;
  R.chunk = CH;
  R.prof = A.prof != nullptr;
  R.rc = nullptr;
  R.mk = 0;
  R.stride = gridDim.x * A.warps;
  R.total = A.ntick;
  R.gw = blockIdx.x * A.warps + w;
  R.jc = 0;
  R.cons = 0;
  R.t_ring = 0;
  R.t_flag = 0;
  R.t_span = 0;
  R.t_refill = 0;
  long long t_rec = 0;
  auto request = [&](int j) {  // lane 0: bulk copy of the record of ticket index j
    const int tk = R.gw + j * R.stride;
    if (tk >= R.total) return;
    const int s = j & (kRecSlots - 1);
    fence_proxy_async();
    mbar_expect_tx(&rbar[s], uint32_t(sizeof(WRec)));
    bulk_g2s(&rb[s], A.recs + tk, uint32_t(sizeof(WRec)), &rbar[s]);
  };
  if (l == 0) {
    for (int s = 0; s < kMaxSlots; ++s) mbar_init(&bars[s], 1);
    for (int s = 0; s < kRecSlots; ++s) mbar_init(&rbar[s], 1);
    mbar_init(sbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    P->prod = 0;
    P->jp = 0;
    P->have = 0;
    P->mi = P->co = P->nm = 0;
    request(0);
    request(1);
    request(2);
  }
  __syncwarp();
  long long t_kind[3] = {0, 0, 0};  // backward / S2 / forward (+ L, L* items counted as forward)
  int n_kind[3] = {0, 0, 0};
  const long long t_start = R.prof ? clock64() : 0;
  for (int j = 0; R.gw + j * R.stride < R.total; ++j) {
    R.jc = j;
    if (l == 0) {
      request(j + 3);
      // L2 prefetch of the next ticket's matrices: the smem ring only runs S
      // chunks ahead, L2 holds the rest of the next item so its chunks arrive at
      // L2 rather than HBM latency (record j+1 was requested two items ago)
      if (A.l2_prefetch && R.gw + (j + 1) * R.stride < R.total) {
        const int s1 = (j + 1) & (kRecSlots - 1);
        if (mbar_try_wait(&rbar[s1], uint32_t((j + 1) / kRecSlots) & 1u)) {
          const WRec& rn = rb[s1];
          for (int k = 0; k < rn.nmat; ++k) {
            const uint32_t bytes = (uint32_t(rn.mrows[k]) * uint32_t(rn.mcols[k]) * 8u + 15u) & ~15u;
            if (bytes) bulk_prefetch_l2(rn.mp[k], bytes);
          }
        }
      }
    }
    refill_lane0(R);
    const int s = j & (kRecSlots - 1);
    const uint32_t par = uint32_t(j / kRecSlots) & 1u;
    {
      long long t0 = 0;
      if (R.prof) t0 = clock64();
      while (!mbar_try_wait(&rbar[s], par)) {
      }
      if (R.prof) t_rec += clock64() - t0;
    }
    const WRec& rc = rb[s];
    long long t0 = 0;
    if (R.prof) t0 = clock64();
    const int kind = rc.kind;
    R.rc = &rc;
    R.mk = 0;
    stage_spans(A, rc, vrec, doff, sbar);
    __syncwarp();
    const SpanWait W{sbar, uint32_t(j) & 1u};
    Spans sp{&A, &rc, vrec, doff};
    switch (kind) {
      case 0: w_back<RR>(A, R, rc, sp, W, xs, xs2); break;
      case 1: w_s2(A, rc.node, xs); break;
      case 2: w_fwd<RR>(A, R, rc, sp, W, xs, xs2, dep); break;
      case 3: w_L<RR>(A, R, rc, sp, W, xs, xs2); break;
      case 4: w_Lt_child<RR>(A, R, rc, sp, W); break;
      default: w_Lt_node<RR>(A, R, rc, sp, W); break;
    }
    if (kind == 1) spans_ready(R, W);  // keep the span barrier's phase in step
    __syncwarp();
    if (R.prof) {
      t_kind[min(kind, 2)] += clock64() - t0;
      ++n_kind[min(kind, 2)];
    }
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
    atomicAdd(pf + 10, (unsigned long long)R.t_span);
    atomicAdd(pf + 11, (unsigned long long)R.t_refill);
    atomicAdd(pf + 12, (unsigned long long)t_rec);
  }
}

}  // namespace

// one translation unit per row count RR (wide_r*.cu) instantiates k_T_wide
#define SPOCK_WIDE_TU(RR)                                                                          \
  const void* wide_ptr_r##RR(int ctas) {                                                           \
    return ctas >= 2 ? reinterpret_cast<const void*>(&k_T_wide<RR, 2>)                            \
                     : reinterpret_cast<const void*>(&k_T_wide<RR, 1>);                            \
  }                                                                                                \
  cudaError_t wide_launch_r##RR(const cudaLaunchConfig_t* cfg, int ctas, const WideArgs& A) {      \
    return ctas >= 2 ? cudaLaunchKernelEx(cfg, k_T_wide<RR, 2>, A) : cudaLaunchKernelEx(cfg, k_T_wide<RR, 1>, A); \
  }

}  // namespace spock
