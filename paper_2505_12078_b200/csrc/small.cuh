// CTA-resident SuperMann / CP solve for small trees (included by kernels.cu,
// which holds the warp-per-node operator bodies it runs).
//
// On a tree whose per-node blocks fit in one SM's L1 (c1: 31 nodes, ~0.3 MB per
// CP application) a solve is bound by latency, not bandwidth: the device-resident
// graph loop pays ~25 graph nodes and 2N+2 dependent tree levels of
// inter-CTA flag hand-offs per iteration (~90 us per CP iteration on c1, twice
// the CPU's).  Here ONE CTA runs the whole solve: every operator phase (L* child
// and node terms, S1 backward and forward stage by stage, S2, L with S3 and the
// dual step) is a warp-per-node loop over the phase's nodes followed by
// __syncthreads, the reductions are fixed-order block reductions, and thread 0
// runs the same controller as the graph loop (loop_ctl.cuh: termination,
// Anderson in double-double, K0 / line search / K1 / K2 / KM) on a shared-memory
// copy of the state.  Matrices are read through L1 (__ldg), where they stay
// resident across iterations.  Same algorithm, same operator arithmetic as the
// per-stage kernels; only the reduction grids differ.
//
// Reference map: the loop is proj/src/solver.cpp:189-350 (SuperMann) and
// 182-187 (CP); T is solver.cpp:148-164 over tree_operator.cpp:20-114 and
// projections.cpp:142-244.

constexpr int kSmallThreads = 256;
constexpr int kSW = kSmallThreads / 32;

// ---- CTA building blocks (all threads call them; each ends with a barrier) --
__device__ void cta_Lt(const Dev& D, const double* eta, const double* zin, double* zout, double a, double b,
                       double c0, double* xs) {
  const int w = threadIdx.x >> 5;
  for (int k = w; k < D.nr; k += kSW) {
    lt_child_body(D, k, eta, zin, zout, a, b, xs);
    __syncwarp();
  }
  __syncthreads();
  for (int i = w; i < D.nn; i += kSW) {
    lt_node_body(D, i, eta, zin, zout, a, b, c0, xs);
    __syncwarp();
  }
  __syncthreads();
}

__device__ void cta_L(const Dev& D, const double* z, double* eta, double* xs) {
  const int w = threadIdx.x >> 5;
  for (int i = w; i < D.nn; i += kSW) {
    L_node_body<false>(D, i, z, 1.0, nullptr, 0.0, nullptr, eta, 0.0, xs);
    __syncwarp();
  }
  __syncthreads();
}

// one CP application, the per-stage schedule of Engine::T (launch_Lt, launch_s1,
// launch_s2, launch_L<DUAL>) with a barrier per launch
__device__ void cta_T(const Dev& D, const int* ss, const double* z, const double* eta, double* zo, double* eo,
                      double alpha, double* xs) {
  const int w = threadIdx.x >> 5;
  cta_Lt(D, eta, z, zo, 1.0, -alpha, -alpha, xs);
  for (int t = D.N; t >= 0; --t) {
    for (int i = ss[t] + w; i < ss[t + 1]; i += kSW) {
      s1_back_body(D, i, zo, xs);
      __syncwarp();
    }
    __syncthreads();
  }
  for (int t = 0; t <= D.N; ++t) {
    for (int i = ss[t] + w; i < ss[t + 1]; i += kSW) {
      s1_fwd_body(D, i, zo, xs);
      __syncwarp();
    }
    __syncthreads();
  }
  for (int i = w; i < D.nnl; i += kSW) {
    s2_node_body(D, i, zo, xs);
    __syncwarp();
  }
  __syncthreads();
  for (int i = w; i < D.nn; i += kSW) {
    L_node_body<true>(D, i, zo, 2.0, z, -1.0, eta, eo, alpha, xs);
    __syncwarp();
  }
  __syncthreads();
}

// fixed-order block sums of NV per-thread values into out[0..NV)
template <int NV>
__device__ void cta_sums(double (&v)[NV], double* wred, double* out) {
  const int w = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const double s = warp_sum(v[j]);
    if ((threadIdx.x & 31) == 0) wred[j * kSW + w] = s;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double s = 0.0;
    for (int k = 0; k < kSW; ++k) s += wred[threadIdx.x * kSW + k];
    out[threadIdx.x] = s;
  }
  __syncthreads();
}

// M-norm dots of (r, L r_z): <r_z, r_z>, <r_eta, L r_z>, <r_eta, r_eta> -> out[0..3)
__device__ void cta_mnorm(const double* r, const double* lrz, int64_t nz, int64_t ne, double* wred, double* out) {
  double v[3] = {0.0, 0.0, 0.0};
  for (int64_t i = threadIdx.x; i < nz; i += kSmallThreads) v[0] += r[i] * r[i];
  for (int64_t i = threadIdx.x; i < ne; i += kSmallThreads) {
    const double e = r[nz + i];
    v[1] += e * lrz[i];
    v[2] += e * e;
  }
  cta_sums<3>(v, wred, out);
}

// termination residual norms (solver.cpp:240-244): max |(x / alpha - y) d| per part, NaN propagated
__device__ void cta_xi(const double* r, const double* lsre, const double* lrz, const double* d1, const double* d2,
                       int64_t nz, int64_t ne, double alpha, double* wred, double* out) {
  double m[2] = {0.0, 0.0};
  int bad = 0;
  for (int64_t i = threadIdx.x; i < nz; i += kSmallThreads) {
    const double v = (r[i] / alpha - lsre[i]) * d1[i];
    bad |= isnan(v);
    m[0] = fmax(m[0], fabs(v));
  }
  for (int64_t i = threadIdx.x; i < ne; i += kSmallThreads) {
    const double v = (r[nz + i] / alpha - lrz[i]) * d2[i];
    bad |= isnan(v);
    m[1] = fmax(m[1], fabs(v));
  }
  const int w = threadIdx.x >> 5;
  const int anybad = __syncthreads_or(bad);
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const double s = warp_max(m[j]);
    if ((threadIdx.x & 31) == 0) wred[j * kSW + w] = s;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double s = 0.0;
    for (int k = 0; k < kSW; ++k) s = fmax(s, wred[threadIdx.x * kSW + k]);
    out[threadIdx.x] = anybad ? NAN : s;
  }
  __syncthreads();
}

// Anderson Gram update in double-double (as loop.cu's gram_dd_body, one block)
__device__ void cta_gram(const LoopArgs& A, const LoopState& S, double* wred, double* out) {
  constexpr int M = kLoopMaxMem;
  const int m = A.P.m, hn = S.h + 1, cols = min(S.aa_cols + 1, m);
  const double* D0[M];
#pragma unroll
  for (int b = 0; b < M; ++b) D0[b] = A.DH[ring(hn - min(b, cols - 1), m)];
  const double* dnew = D0[0];
  dd acc[2 * M];
#pragma unroll
  for (int j = 0; j < 2 * M; ++j) acc[j] = {0.0, 0.0};
  for (int64_t i = threadIdx.x; i < A.nv; i += kSmallThreads) {
    const double x = dnew[i], rr = A.R[i];
#pragma unroll
    for (int b = 0; b < M; ++b)
      if (b < cols) {
        const double db = D0[b][i];
        acc[b] = dd_fma(acc[b], x, db);
        acc[M + b] = dd_fma(acc[M + b], db, rr);
      }
  }
  const int w = threadIdx.x >> 5;
  double* wl = wred + 2 * M * kSW;
#pragma unroll
  for (int j = 0; j < 2 * M; ++j) {
    if ((j < M ? j : j - M) >= cols) continue;  // only the 2 cols sums in use (block-uniform)
    dd v = acc[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const dd u = {__shfl_xor_sync(0xffffffffu, v.hi, o), __shfl_xor_sync(0xffffffffu, v.lo, o)};
      v = dd_add(v, u);
    }
    if ((threadIdx.x & 31) == 0) wred[j * kSW + w] = v.hi, wl[j * kSW + w] = v.lo;
  }
  __syncthreads();
  if (threadIdx.x < 2 * cols) {
    const int j = threadIdx.x < cols ? threadIdx.x : M + threadIdx.x - cols;
    dd s = {wred[j * kSW], wl[j * kSW]};
    for (int k = 1; k < kSW; ++k) s = dd_add(s, {wred[j * kSW + k], wl[j * kSW + k]});
    out[2 * threadIdx.x] = s.hi;
    out[2 * threadIdx.x + 1] = s.lo;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kSmallThreads, 1) k_small_solve(const __grid_constant__ SmallArgs A) {
  __shared__ double xs_all[kSW][kMaxD];
  __shared__ double red[8 + 4 * kLoopMaxMem];
  __shared__ double wred[4 * kLoopMaxMem * kSW];
  __shared__ LoopState S;
  __shared__ LoopArgs LA;
  const int t = threadIdx.x, w = t >> 5;
  double* xs = xs_all[w];
  if (t == 0) {
    S = *A.L.st;
    LA = A.L;
    LA.st = &S;
    LA.red = red;
  }
  __syncthreads();
  const Dev& D = A.D;
  const int* ss = A.stage_start;
  const int64_t nz = A.L.nz, nv = A.L.nv, ne = nv - nz;
  const double alpha = A.L.P.alpha;
  double *V = A.L.V, *TV = A.L.TV, *R = A.L.R, *C = A.L.C, *CR = A.L.CR, *PSI = A.L.PSI;
  double *TC = A.TC, *PV = A.PV, *Lrz = A.Lrz, *cLrz = A.cLrz;
  const bool sm = A.supermann != 0;
  const int m = A.L.P.m;
  long long tprev = clock64();
  long long tacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // T, L, L*, reductions, gram, controller, vector ops, other
  auto tick = [&](int cls) {
    if (A.prof && t == 0) {
      const long long now = clock64();
      tacc[cls] += now - tprev;
      tprev = now;
    }
  };
  auto vec = [&](auto&& f) {
    for (int64_t i = t; i < nv; i += kSmallThreads) f(i);
    __syncthreads();
  };
  // r = v - T v, L r_z and the M-norm dots of (r, L r_z)
  auto refresh = [&](const double* v, double* tv, double* r, double* lrz) {
    tick(7);
    cta_T(D, ss, v, v + nz, tv, tv + nz, alpha, xs);
    tick(0);
    vec([&](int64_t i) { r[i] = v[i] - tv[i]; });
    tick(6);
    cta_L(D, r, lrz, xs);
    tick(1);
    cta_mnorm(r, lrz, nz, ne, wred, red);
    tick(3);
  };
  refresh(V, TV, R, Lrz);  // prologue (solver.cpp:211-235)
  for (;;) {
    // top of the iteration: L* r_eta, xi norms, Anderson push and Gram
    tick(7);
    cta_Lt(D, R + nz, nullptr, A.Lsre, 0.0, 1.0, 0.0, xs);
    tick(2);
    cta_xi(R, A.Lsre, Lrz, A.d1, A.d2, nz, ne, alpha, wred, red + 4);
    tick(3);
    if (sm) {
      const int hn = S.h + 1;
      double* rn = LA.RH[ring(hn, m + 1)];
      const double* rp = LA.RH[ring(hn - 1, m + 1)];
      double* dn = LA.DH[ring(hn, m)];
      const bool first = S.aa_k == 0;
      vec([&](int64_t i) {
        const double r = R[i];
        dn[i] = first ? r : r - rp[i];
        rn[i] = r;
      });
      tick(6);
      cta_gram(LA, S, wred, red + 8);
      tick(4);
    }
    if (t == 0) ctl_begin<false>(LA);
    __syncthreads();
    tick(5);
    if (S.sw == 0) break;
    if (sm) {  // psi = cpsi[0] r + sum_c cpsi[c] r_{k-1-c}
      const int h = S.h, nc = S.ncpsi;
      vec([&](int64_t i) {
        double s = S.cpsi[0] * R[i];
        for (int c = 1; c < nc; ++c) s += S.cpsi[c] * LA.RH[ring(h - c, m + 1)][i];
        PSI[i] = s;
      });
    }
    const int sw = S.sw;
    if (sw == 1) {  // K0
      vec([&](int64_t i) { V[i] += PSI[i]; });
    } else if (sw == 2) {  // M psi, then the line search (solver.cpp:287-338)
      cta_Lt(D, PSI + nz, nullptr, A.tmpz, 0.0, 1.0, 0.0, xs);
      cta_L(D, PSI, A.tmpe, xs);
      vec([&](int64_t i) { PV[i] = i < nz ? PSI[i] - alpha * A.tmpz[i] : PSI[i] - alpha * A.tmpe[i - nz]; });
      for (;;) {
        const double tau = S.tau;
        vec([&](int64_t i) { C[i] = V[i] + tau * PSI[i]; });
        refresh(C, TC, CR, cLrz);
        {
          double v[2] = {0.0, 0.0};
          for (int64_t i = t; i < nz; i += kSmallThreads) v[0] += CR[i] * PV[i];
          for (int64_t i = t; i < ne; i += kSmallThreads) v[1] += CR[nz + i] * PV[nz + i];
          cta_sums<2>(v, wred, red + 3);
        }
        if (t == 0) ctl_ls<false>(LA);
        __syncthreads();
        if (!S.ls_more) break;
      }
      if (S.reason == -2) break;
      const int act = S.act;
      if (act == '1') {
        vec([&](int64_t i) {
          V[i] = C[i];
          TV[i] = TC[i];
          R[i] = CR[i];
          if (i < ne) Lrz[i] = cLrz[i];
        });
      } else if (act == '2') {
        const double coef = S.coef;
        vec([&](int64_t i) { V[i] -= coef * CR[i]; });
      } else {  // KM fallback
        vec([&](int64_t i) { V[i] = TV[i]; });
      }
    } else {  // CP: v <- T v
      vec([&](int64_t i) { V[i] = TV[i]; });
    }
    if (S.refresh) refresh(V, TV, R, Lrz);
    if (t == 0) ctl_end<false>(LA);
    __syncthreads();
    if (S.reason != -1 || S.k >= S.k_stop) break;
  }
  __syncthreads();
  if (t == 0) *A.L.st = S;
  if (A.prof && t == 0)
    for (int k = 0; k < 8; ++k) A.prof[k] += (unsigned long long)tacc[k];
}
