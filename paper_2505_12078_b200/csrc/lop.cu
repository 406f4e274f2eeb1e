// Standalone L and L* for narrow trees: one CTA per node, every operand
// staged at once (sm_100a).
//
// TreeOperator::apply / apply_adjoint (proj/src/tree_operator.cpp:20-114), as
// the SuperMann loop uses them outside T (M-norm, xi residuals, M psi).  On a
// narrow tree there is about one node per SM, so the time of a launch is the
// latency of one node: the CTA loads the node's 256-byte record (the same
// host-built records the streaming kernel uses, wide.hpp), then issues every
// matrix block (cp.async 16 B) and vector span (cp.async 8 B) of the node in one
// batch, waits once, and computes from shared memory with warp-column-block
// GEMVs (fixed summation order).  L* is parent-centric: node i also computes
// its children's stage-cost adjoint terms (their blocks are staged with its
// own), so one launch has no inter-CTA dependency.
#include <cuda_runtime.h>

#include <cstdint>

#include "dev.cuh"
#include "kernels.hpp"
#include "wide.hpp"

namespace spock {

namespace {

constexpr int kT = 256;
constexpr int kNW = kT / 32;
// span ids of the record kinds (same as wide.cu)
enum : int { L_ZX = 0, L_ZU, L_AX, L_AU, L_QK, L_ZT, L_ZS, L_Y, L_RB, L_GD, L_QKN };
enum : int { LC_HEAD = 0, LC_QK };
enum : int { LN_SEG1 = 0, LN_RB, LN_GD, LN_QKN };

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(su32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_wait_all() {
  asm volatile("cp.async.commit_group;\n cp.async.wait_group 0;" ::: "memory");
}

struct LopArgs {
  Dev D;
  const double* z;
  const double* eta;
  double* out;
  const WRec* lrec;   // kind 3, node i at i
  const WRec* ltrec;  // kind 4 for nodes 1..nn-1 at i-1, then kind 5 for node i at nr + i
  const double* vb[WB_COUNT];
  int mat_cap;  // doubles of matrix staging per CTA
  int vec_cap;  // doubles of vector staging per CTA
  int rows;     // max(nx + nu, constraint rows): GEMV partial slabs are kNW * (rows + 64)
};

__device__ __forceinline__ const double* span_src(const LopArgs& A, const WRec& R, int k) {
  const int b = R.vbase[k];
  return (b == WB_Z ? A.z : (b == WB_ETA ? A.eta : A.vb[b])) + R.voff[k];
}

// stage every span of R into vec[off..]; returns the offsets through so[] (or
// leaves global pointers for unstaged spans)
__device__ int stage_rec_spans(const LopArgs& A, const WRec& R, double* vec, int off, const double** sp) {
  for (int k = 0; k < R.nspan; ++k) {
    const int n = R.vcnt[k];
    const double* src = span_src(A, R, k);
    if (((R.unstaged >> k) & 1) || n == 0 || off + n > A.vec_cap) {
      if (threadIdx.x == 0) sp[k] = src;
      continue;
    }
    double* dst = vec + off;
    for (int e = threadIdx.x; e < n; e += kT) cp8(dst + e, src + e);
    if (threadIdx.x == 0) sp[k] = dst;
    off += (n + 1) & ~1;
  }
  return off;
}

// stage matrix k of R (padded even, 16-byte aligned) if it fits
__device__ const double* stage_mat(const WRec& R, int k, double* mat, int& off, int cap) {
  const int n = int(R.mrows[k]) * int(R.mcols[k]);
  const int n2 = (n + 1) & ~1;
  if (n2 == 0 || off + n2 > cap) return R.mp[k];
  double* dst = mat + off;
  for (int e = 2 * threadIdx.x; e < n2; e += 2 * kT) cp16(dst + e, R.mp[k] + e);
  off += n2;
  return dst;
}

// warp-column-block GEMV partials: red[w*m + r] = sum_{c in block w} A[r + c*lda] x[c]
__device__ __forceinline__ void cols_partial(const double* A, int m, int n, int lda, const double* x, double* red) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int cb = (n + kNW - 1) / kNW;
  const int c0 = min(n, w * cb), c1 = min(n, c0 + cb);
  for (int rb = 0; rb < m; rb += 128) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    const int r0 = rb + l, r1 = r0 + 32, r2 = r0 + 64, r3 = r0 + 96;
    for (int c = c0; c < c1; ++c) {
      const double xc = x[c];
      const double* col = A + size_t(c) * lda;
      if (r0 < m) a0 = fma(col[r0], xc, a0);
      if (r1 < m) a1 = fma(col[r1], xc, a1);
      if (r2 < m) a2 = fma(col[r2], xc, a2);
      if (r3 < m) a3 = fma(col[r3], xc, a3);
    }
    double* rw = red + size_t(w) * m;
    if (r0 < m) rw[r0] = a0;
    if (r1 < m) rw[r1] = a1;
    if (r2 < m) rw[r2] = a2;
    if (r3 < m) rw[r3] = a3;
  }
}

// y[r] = base[r] + sum_w red[w*m + r] for r < m (base may be null)
__device__ __forceinline__ void cols_reduce(const double* red, int m, const double* base, double* y) {
  for (int r = threadIdx.x; r < m; r += kT) {
    double o = base ? base[r] : 0.0;
#pragma unroll
    for (int w = 0; w < kNW; ++w) o += red[size_t(w) * m + r];
    y[r] = o;
  }
}

__device__ double bsum(double v, double* red) {
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < kNW; ++k) s += red[k];
  __syncthreads();
  return s;
}

__device__ void load_rec(WRec* dst, const WRec* src) {
  if (threadIdx.x < 16) reinterpret_cast<int4*>(dst)[threadIdx.x] = __ldg(reinterpret_cast<const int4*>(src) + threadIdx.x);
}

// ---------------------------------------------------------------------------
// eta = L z, CTA per node
__global__ void __launch_bounds__(kT) k_L_node(const __grid_constant__ LopArgs A) {
  extern __shared__ __align__(16) double sm[];
  __shared__ WRec R;
  __shared__ const double* sp[kWSpans];
  __shared__ const double* mp[kWMats];
  const Dev& D = A.D;
  const int i = blockIdx.x, t = threadIdx.x, nx = D.nx, nu = D.nu;
  double* mat = sm;
  double* vec = mat + A.mat_cap;
  double* red = vec + A.vec_cap;  // kNW * (rows + 64) + rows
  load_rec(&R, A.lrec + i);
  __syncthreads();
  // every operand of the node in one batch
  stage_rec_spans(A, R, vec, 0, sp);
  {
    int off = 0;
    for (int k = 0; k < R.nmat; ++k) {
      const double* p = stage_mat(R, k, mat, off, A.mat_cap);
      if (t == 0) mp[k] = p;
    }
  }
  cp_wait_all();
  __syncthreads();
  double* eo = A.out;
  const bool root = i == 0, leaf = R.nch == 0;
  if (!leaf) {  // y-copy rows, risk scalar, constraint rows
    const int ny = R.ny, so = R.so, nc = R.nc;
    const double* zy = sp[L_Y];
    const double* rb = sp[L_RB];
    double part = 0.0;
    for (int r = t; r < ny; r += kT) {
      const double yv = zy[r];
      part += rb[r] * yv;
      eo[so + r] = yv;
    }
    const double by = bsum(part, red);
    if (t == 0) eo[so + ny] = sp[L_ZS][0] - by;
    const double* zx = sp[L_ZX];
    const double* zu = sp[L_ZU];
    if (D.g_diag) {
      const double* gd = sp[L_GD];
      for (int r = t; r < nc; r += kT) eo[so + ny + 1 + r] = gd[r] * (r < nx ? zx[r] : zu[r - nx]);
    } else {
      cols_partial(D.Gx + D.g_off[i] * nx, nc, nx, nc, zx, red);
      __syncthreads();
      double* tmp = red + kNW * (A.rows + 64);
      cols_reduce(red, nc, nullptr, tmp);
      __syncthreads();
      cols_partial(D.Gu + D.g_off[i] * nu, nc, nu, nc, zu, red);
      __syncthreads();
      cols_reduce(red, nc, tmp, eo + so + ny + 1);
    }
    __syncthreads();
  }
  int mk = 0;
  if (!root) {  // stage-cost SOC block of (x_anc, u_anc, tau_i)
    const int px = R.px, pu = R.pu, p = px + pu, o2 = R.s2o;
    const double* zax = sp[L_AX];
    const double* zau = sp[L_AU];
    const double* qk = sp[L_QK];
    double part = 0.0;
    for (int r = t; r < nx + nu; r += kT) part += qk[r] * (r < nx ? zax[r] : zau[r - nx]);
    const double qd = bsum(part, red);
    double* red2 = red + size_t(kNW) * px;  // Hu partials after Hx's
    cols_partial(mp[mk], px, nx, px, zax, red);
    cols_partial(mp[mk + 1], pu, nu, pu, zau, red2);
    mk += 2;
    __syncthreads();
    cols_reduce(red, px, nullptr, eo + o2);
    cols_reduce(red2, pu, nullptr, eo + o2 + px);

    if (t == 0) {
      const double row = 0.5 * sp[L_ZT][0] - 0.5 * qd;
      eo[o2 + p] = row;
      eo[o2 + p + 1] = row;
    }
    __syncthreads();
  }
  if (leaf) {  // G_N x and the terminal SOC block of (x, s)
    const int j = i - D.nnl, nc = R.nc, p = R.pN, e3 = R.so;
    const double* zx = sp[L_ZX];
    if (D.gN_diag) {
      const double* gd = sp[L_GD];
      for (int r = t; r < nc; r += kT) eo[e3 + r] = gd[r] * zx[r];
    } else {
      cols_partial(D.GN + D.gN_off[j] * nx, nc, nx, nc, zx, red);
      __syncthreads();
      cols_reduce(red, nc, nullptr, eo + e3);
    }
    const double* qk = sp[L_QKN];
    double part = 0.0;
    for (int r = t; r < nx; r += kT) part += qk[r] * zx[r];
    const double qd = bsum(part, red);
    cols_partial(mp[mk], p, nx, p, zx, red);
    __syncthreads();
    cols_reduce(red, p, nullptr, eo + e3 + nc);
    if (t == 0) {
      const double row = 0.5 * sp[L_ZS][0] - 0.5 * qd;
      eo[e3 + nc + p] = row;
      eo[e3 + nc + p + 1] = row;
    }
  }
}

// ---------------------------------------------------------------------------
// z = L* eta, CTA per node, parent-centric: node i's rows and the stage-cost
// adjoint terms (and tau slots) of its children
__global__ void __launch_bounds__(kT) k_Lt_node(const __grid_constant__ LopArgs A, int nr) {
  extern __shared__ __align__(16) double sm[];
  __shared__ WRec R;
  __shared__ WRec RC;
  __shared__ const double* sp[kWSpans];
  __shared__ const double* spc[kWSpans];
  __shared__ const double* mp[kWMats];
  const Dev& D = A.D;
  const int i = blockIdx.x, t = threadIdx.x, nx = D.nx, nu = D.nu, m = nx + nu;
  double* mat = sm;
  double* vec = mat + A.mat_cap;
  double* red = vec + A.vec_cap;            // kNW * (rows + 64)
  double* acc = red + kNW * (A.rows + 64);  // m: sum of the children's adj (ascending)
  double* zo = A.out;
  load_rec(&R, A.ltrec + nr + i);
  __syncthreads();
  const bool leaf = R.nch == 0;
  const int c0 = R.c0, nch = R.nch;
  for (int r = t; r < m; r += kT) acc[r] = 0.0;
  // children, one at a time; the first child's operands are staged together
  // with the node's own, the rest overlap nothing but stay one round trip each
  int voff = stage_rec_spans(A, R, vec, 0, sp);
  {
    int off = 0;
    for (int k = 0; k < R.nmat; ++k) {
      const double* p = stage_mat(R, k, mat, off, A.mat_cap / 2);
      if (t == 0) mp[k] = p;
    }
  }
  for (int c = 0; c < nch; ++c) {
    const int ch = c0 + c;
    __syncthreads();
    load_rec(&RC, A.ltrec + (ch - 1));
    __syncthreads();
    stage_rec_spans(A, RC, vec, voff, spc);
    int off = A.mat_cap / 2;
    const double* HxT = stage_mat(RC, 0, mat, off, A.mat_cap);
    const double* HuT = stage_mat(RC, 1, mat, off, A.mat_cap);
    cp_wait_all();
    __syncthreads();
    const int px = RC.px, pu = RC.pu, p = px + pu;
    const double* head = spc[LC_HEAD];
    const double* qk = spc[LC_QK];
    const double rsum = head[p] + head[p + 1];
    // adj_c = [HxT head_x; HuT head_u] - rsum/2 qk, accumulated in child order
    cols_partial(HxT, nx, px, nx, head, red);
    __syncthreads();
    for (int r = t; r < nx; r += kT) {
      double o = -0.5 * rsum * qk[r];
#pragma unroll
      for (int w = 0; w < kNW; ++w) o += red[size_t(w) * nx + r];
      acc[r] += o;
    }
    __syncthreads();
    cols_partial(HuT, nu, pu, nu, head + px, red);
    __syncthreads();
    for (int r = t; r < nu; r += kT) {
      double o = -0.5 * rsum * qk[nx + r];
#pragma unroll
      for (int w = 0; w < kNW; ++w) o += red[size_t(w) * nu + r];
      acc[nx + r] += o;
    }
    if (t == 0) zo[D.tau_base + ch - 1] = 0.5 * rsum;
  }
  cp_wait_all();
  __syncthreads();
  if (!leaf) {
    const int ny = R.ny, yo = R.yo, nc = R.nc;
    const double* seg1 = sp[LN_SEG1];
    const double* rb = sp[LN_RB];
    const double sc = seg1[ny];
    for (int r = t; r < ny; r += kT) zo[yo + r] = seg1[r] - sc * rb[r];
    if (t == 0) zo[i == 0 ? 0 : D.s_base + i - 1] = sc;
    const double* ec = seg1 + ny + 1;
    if (D.g_diag) {
      const double* gd = sp[LN_GD];
      for (int r = t; r < m; r += kT) {
        const double v = gd[r] * ec[r] + acc[r];
        if (r < nx)
          zo[1 + size_t(i) * nx + r] = v;
        else
          zo[D.u_base + size_t(i) * nu + r - nx] = v;
      }
    } else {
      cols_partial(D.GxT + D.g_off[i] * nx, nx, nc, nx, ec, red);
      __syncthreads();
      cols_reduce(red, nx, acc, zo + 1 + size_t(i) * nx);
      __syncthreads();
      cols_partial(D.GuT + D.g_off[i] * nu, nu, nc, nu, ec, red);
      __syncthreads();
      cols_reduce(red, nu, acc + nx, zo + D.u_base + size_t(i) * nu);
    }
  } else {
    const int j = i - D.nnl, nc = R.nc, p = R.pN;
    const double* ec = sp[LN_SEG1];
    const double* hd = ec + nc;
    const double rsum = hd[p] + hd[p + 1];
    const double* qk = sp[LN_QKN];
    double* gx = acc;  // no children: reuse
    if (D.gN_diag) {
      const double* gd = sp[LN_GD];
      for (int r = t; r < nx; r += kT) gx[r] = gd[r] * ec[r];
    } else {
      cols_partial(D.GNT + D.gN_off[j] * nx, nx, nc, nx, ec, red);
      __syncthreads();
      cols_reduce(red, nx, nullptr, gx);
    }
    __syncthreads();
    cols_partial(mp[0], nx, p, nx, hd, red);
    __syncthreads();
    for (int r = t; r < nx; r += kT) {
      double o = gx[r];
#pragma unroll
      for (int w = 0; w < kNW; ++w) o += red[size_t(w) * nx + r];
      zo[1 + size_t(i) * nx + r] = o - 0.5 * rsum * qk[r];
    }
    if (t == 0) zo[D.s_base + i - 1] = 0.5 * rsum;
  }
}

}  // namespace

int lop_smem_bytes(int rows, int mat_cap, int vec_cap) {
  return int(sizeof(double) * (size_t(mat_cap) + vec_cap + kNW * (rows + 64) + rows + 8));
}

cudaError_t lop_configure(int bytes) {
  cudaFuncSetAttribute(k_L_node, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  cudaFuncSetAttribute(k_Lt_node, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  cudaError_t e = set_smem_limit(reinterpret_cast<const void*>(&k_L_node), bytes);
  if (e != cudaSuccess) return e;
  return set_smem_limit(reinterpret_cast<const void*>(&k_Lt_node), bytes);
}

void launch_L_lop(const Dev& D, const WideArgs& W, const WRec* lrec, const double* z, double* eta, int rows,
                  int mat_cap, int vec_cap, cudaStream_t st) {
  LopArgs A{};
  A.D = D, A.z = z, A.eta = nullptr, A.out = eta, A.lrec = lrec, A.ltrec = nullptr;
  for (int k = 0; k < WB_COUNT; ++k) A.vb[k] = W.vb[k];
  A.mat_cap = mat_cap, A.vec_cap = vec_cap, A.rows = rows;
  k_L_node<<<D.nn, kT, lop_smem_bytes(rows, mat_cap, vec_cap), st>>>(A);
}

void launch_Lt_lop(const Dev& D, const WideArgs& W, const WRec* ltrec, const double* eta, double* z, int rows,
                   int mat_cap, int vec_cap, cudaStream_t st) {
  LopArgs A{};
  A.D = D, A.z = nullptr, A.eta = eta, A.out = z, A.lrec = nullptr, A.ltrec = ltrec;
  for (int k = 0; k < WB_COUNT; ++k) A.vb[k] = W.vb[k];
  A.mat_cap = mat_cap, A.vec_cap = vec_cap, A.rows = rows;
  k_Lt_node<<<D.nn, kT, lop_smem_bytes(rows, mat_cap, vec_cap), st>>>(A, D.nr);
}

}  // namespace spock
