// Cluster-resident SuperMann / CP solve for small trees (included by
// kernels.cu after small.cuh, whose operator phases it distributes).
//
// On a tree whose whole device image -- per-node blocks, layouts, iterates,
// history rings -- fits in the shared memory of a few SMs (c1: 31 nodes,
// ~0.5 MB), a solve is bound by the latency of its dependent phases, not by
// bandwidth.  One thread-block cluster of C CTAs runs the whole solve:
//
//  * at launch every CTA copies its share of the device allocations (host-
//    packed, whole allocations per CTA) into its shared memory, and each CTA
//    rewrites its copy of the argument block so every pointer addresses the
//    distributed shared-memory copy (generic addresses from map_shared_rank):
//    from then on the solve touches HBM only for the per-iteration ||r||_M and
//    branch records;
//  * every operator phase (L* child and node terms, S1 backward and forward
//    stage by stage, S2, L with S3 and the dual step) is a warp-per-node loop
//    over the cluster's C x 8 warps, closed by a cluster barrier
//    (barrier.cluster arrive.release / wait.acquire, ~0.2 us) instead of a
//    kernel boundary or an inter-CTA flag round trip through L2;
//  * reductions are fixed-order: warps in index order inside a CTA, CTAs in
//    rank order in CTA 0 (bitwise run-to-run deterministic);
//  * thread 0 of CTA 0 runs the graph loop's controller (loop_ctl.cuh) on the
//    state in its shared memory; the other CTAs read the branch scalars through
//    DSMEM after the barrier that follows it.
//
// Same algorithm and operator arithmetic as small.cuh and the per-stage kernels
// (only the reduction partition differs).  Reference map: the loop is
// proj/src/solver.cpp:189-350 (SuperMann) and 182-187 (CP); T is
// solver.cpp:148-164 over tree_operator.cpp:20-114 and projections.cpp:142-244.

__device__ __forceinline__ int cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return int(r);
}
__device__ __forceinline__ int cl_size() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return int(r);
}
// generic address of the same shared-memory location in CTA `rank` of the cluster
template <class Ty>
__device__ __forceinline__ Ty* cl_map(Ty* p, int rank) {
  uint64_t r;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(r) : "l"(p), "r"(rank));
  return reinterpret_cast<Ty*>(r);
}

__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

struct CDist {  // this thread's share of the cluster's work
  int rank, C, gw, GW, gt, GT;
  int w, n0, n1;  // warp in the CTA; the CTA's node range (operator phases)
  int nred;  // reductions so far: partial tables alternate between two halves, so a
             // CTA writing the next reduction's partials never overwrites the ones CTA 0
             // is still summing (the two uses of a half are a cluster barrier apart)
};
__device__ __forceinline__ double* part_half(CDist& c, double* part0) {
  return part0 + (c.nred++ & 1) * (kClusterMax * 64);
}

// operator phases: CTA c runs the nodes it owns ([n0, n1): their blocks sit in
// its shared memory), one warp per node
__device__ void cl_Lt(const CDist& c, const Dev& D, const double* eta, const double* zin, double* zout, double a,
                      double b, double c0, double* xs) {
  for (int k = max(c.n0 - 1, 0) + c.w; k < min(c.n1 - 1, D.nr); k += kSW) {  // child node k + 1
    lt_child_body(D, k, eta, zin, zout, a, b, xs);
    __syncwarp();
  }
  csync();
  for (int i = c.n0 + c.w; i < c.n1; i += kSW) {
    lt_node_body(D, i, eta, zin, zout, a, b, c0, xs);
    __syncwarp();
  }
  csync();
}

__device__ void cl_L(const CDist& c, const Dev& D, const double* z, double* eta, double* xs) {
  for (int i = c.n0 + c.w; i < c.n1; i += kSW) {
    L_node_body<false>(D, i, z, 1.0, nullptr, 0.0, nullptr, eta, 0.0, xs);
    __syncwarp();
  }
  csync();
}

__device__ void cl_T(const CDist& c, const Dev& D, const int* ss, const double* z, const double* eta, double* zo,
                     double* eo, double alpha, double* xs) {
  cl_Lt(c, D, eta, z, zo, 1.0, -alpha, -alpha, xs);
  for (int t = D.N; t >= 0; --t) {
    for (int i = max(ss[t], c.n0) + c.w; i < min(ss[t + 1], c.n1); i += kSW) {
      s1_back_body(D, i, zo, xs);
      __syncwarp();
    }
    csync();
  }
  for (int t = 0; t <= D.N; ++t) {
    for (int i = max(ss[t], c.n0) + c.w; i < min(ss[t + 1], c.n1); i += kSW) {
      s1_fwd_body(D, i, zo, xs);
      __syncwarp();
    }
    csync();
  }
  for (int i = c.n0 + c.w; i < min(c.n1, D.nnl); i += kSW) {
    s2_node_body(D, i, zo, xs);
    __syncwarp();
  }
  csync();
  for (int i = c.n0 + c.w; i < c.n1; i += kSW) {
    L_node_body<true>(D, i, zo, 2.0, z, -1.0, eta, eo, alpha, xs);
    __syncwarp();
  }
  csync();
}

// NV cluster-wide sums (op 0) or maxima (op 1, NaN propagated by `bad`) into
// red[0..NV) of CTA 0: warps in index order, then CTAs in rank order
template <int NV>
__device__ void cl_reduce(CDist& c, double (&v)[NV], int op, int bad, double* wred, double* partb,
                          double* red0) {
  double* part0 = part_half(c, partb);
  const int w = threadIdx.x >> 5;
  const int anybad = op == 1 ? __syncthreads_or(bad) : 0;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const double s = op == 0 ? warp_sum(v[j]) : warp_max(v[j]);
    if ((threadIdx.x & 31) == 0) wred[j * kSW + w] = s;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    const int j = threadIdx.x;
    double s = wred[j * kSW];
    for (int k = 1; k < kSW; ++k) s = op == 0 ? s + wred[j * kSW + k] : fmax(s, wred[j * kSW + k]);
    if (anybad) s = NAN;
    part0[c.rank * 64 + j] = s;  // CTA 0's partial table (DSMEM)
  }
  csync();
  if (c.rank == 0 && threadIdx.x < NV) {
    const int j = threadIdx.x;
    double s = part0[j];
    for (int r = 1; r < c.C; ++r) {
      const double x = part0[r * 64 + j];
      s = op == 0 ? s + x : ((isnan(s) || isnan(x)) ? NAN : fmax(s, x));
    }
    red0[j] = s;
  }
  __syncthreads();
}

// Anderson Gram update in double-double (as cta_gram), partials per CTA in rank order
__device__ void cl_gram(CDist& c, const LoopArgs& A, const LoopState* S, double* wred, double* partb,
                        double* out0) {
  double* part0 = part_half(c, partb);
  constexpr int M = kLoopMaxMem;
  const int m = A.P.m, hn = S->h + 1, cols = min(S->aa_cols + 1, m);
  const double* D0[M];
#pragma unroll
  for (int b = 0; b < M; ++b) D0[b] = A.DH[ring(hn - min(b, cols - 1), m)];
  const double* dnew = D0[0];
  dd acc[2 * M];
#pragma unroll
  for (int j = 0; j < 2 * M; ++j) acc[j] = {0.0, 0.0};
  for (int64_t i = c.gt; i < A.nv; i += c.GT) {
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
    part0[c.rank * 64 + 2 * threadIdx.x] = s.hi;
    part0[c.rank * 64 + 2 * threadIdx.x + 1] = s.lo;
  }
  csync();
  if (c.rank == 0 && threadIdx.x < 2 * cols) {
    const int q = threadIdx.x;
    dd s = {part0[2 * q], part0[2 * q + 1]};
    for (int r = 1; r < c.C; ++r) s = dd_add(s, {part0[r * 64 + 2 * q], part0[r * 64 + 2 * q + 1]});
    out0[2 * q] = s.hi;
    out0[2 * q + 1] = s.lo;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kSmallThreads, 1) k_cluster_solve(const __grid_constant__ ClusterArgs CA) {
  extern __shared__ __align__(16) unsigned char arena[];
  __shared__ double xs_all[kSW][kMaxD];
  __shared__ double wred[4 * kLoopMaxMem * kSW];
  __shared__ double part[2 * kClusterMax * 64];  // CTA 0's: per-rank reduction partials, two halves
  __shared__ double red[8 + 4 * kLoopMaxMem];
  __shared__ LoopState S;  // CTA 0's is the live state
  __shared__ SmallArgs A;  // this CTA's arguments, pointers relocated into the cluster's shared memory
  CDist c;
  c.rank = cl_rank();
  c.C = cl_size();
  const int t = threadIdx.x, w = t >> 5;
  c.gw = c.rank * kSW + w;
  c.GW = c.C * kSW;
  c.gt = c.rank * kSmallThreads + t;
  c.GT = c.C * kSmallThreads;
  c.nred = 0;
  c.w = w;
  c.n0 = CA.own[c.rank];
  c.n1 = CA.own[c.rank + 1];
  double* xs = xs_all[w];
  // stage this CTA's allocations (8-byte granules; every allocation is 16-byte aligned)
  for (int p = 0; p < CA.nplace; ++p) {
    const ClusterPlace P = CA.place[p];
    if (P.cta != c.rank) continue;
    const double* src = reinterpret_cast<const double*>(P.src);
    double* dst = reinterpret_cast<double*>(arena + P.off);
    for (int64_t i = t; i < P.bytes / 8; i += kSmallThreads) dst[i] = src[i];
  }
  if (t == 0) {
    A = CA.S;
    for (int f = 0; f < CA.nfield; ++f) {
      const ClusterField F = CA.field[f];
      if (F.cta >= 0 && F.cta != c.rank) continue;
      const ClusterPlace P = CA.place[F.place];
      char* base = reinterpret_cast<char*>(cl_map(arena + P.off, P.cta));
      *reinterpret_cast<char**>(reinterpret_cast<char*>(&A) + F.field) = base + F.delta;
    }
    if (c.rank == 0) S = *CA.S.L.st;
    A.L.st = cl_map(&S, 0);
    A.L.red = cl_map(red, 0);
  }
  __syncthreads();
  csync();
  LoopState* Sp = A.L.st;  // CTA 0's state (DSMEM for the other CTAs)
  double* part0 = cl_map(part, 0);
  double* red0 = cl_map(red, 0);
  const Dev& D = A.D;
  const int* ss = A.stage_start;
  const int64_t nz = A.L.nz, nv = A.L.nv, ne = nv - nz;
  const double alpha = A.L.P.alpha;
  double *V = A.L.V, *TV = A.L.TV, *R = A.L.R, *C = A.L.C, *CR = A.L.CR, *PSI = A.L.PSI;
  double *TC = A.TC, *PV = A.PV, *Lrz = A.Lrz, *cLrz = A.cLrz;
  const bool sm = A.supermann != 0;
  const int m = A.L.P.m;
  const bool ctl = c.rank == 0 && t == 0;
  // optional phase profile (SPOCK_SMALL_PROF=1): clock64 totals on CTA 0, thread 0
  long long tprev = clock64();
  long long tacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // T, L, L*, reductions, gram, controller, vector ops, other
  auto tick = [&](int cls) {
    if (A.prof && ctl) {
      const long long now = clock64();
      tacc[cls] += now - tprev;
      tprev = now;
    }
  };
  auto vec = [&](auto&& f) {
    tick(7);
    for (int64_t i = c.gt; i < nv; i += c.GT) f(i);
    csync();
    tick(6);
  };
  auto mnorm = [&](const double* r, const double* lrz) {
    double v[3] = {0.0, 0.0, 0.0};
    for (int64_t i = c.gt; i < nz; i += c.GT) v[0] += r[i] * r[i];
    for (int64_t i = c.gt; i < ne; i += c.GT) {
      const double e = r[nz + i];
      v[1] += e * lrz[i];
      v[2] += e * e;
    }
    cl_reduce<3>(c, v, 0, 0, wred, part0, red0);
  };
  auto refresh = [&](const double* v, double* tv, double* r, double* lrz) {
    tick(7);
    cl_T(c, D, ss, v, v + nz, tv, tv + nz, alpha, xs);
    tick(0);
    vec([&](int64_t i) { r[i] = v[i] - tv[i]; });
    cl_L(c, D, r, lrz, xs);
    tick(1);
    mnorm(r, lrz);
    tick(3);
  };
  refresh(V, TV, R, Lrz);  // prologue (solver.cpp:211-235)
  for (;;) {
    tick(7);
    cl_Lt(c, D, R + nz, nullptr, A.Lsre, 0.0, 1.0, 0.0, xs);
    tick(2);
    {  // termination residual norms (solver.cpp:240-244)
      double mx[2] = {0.0, 0.0};
      int bad = 0;
      const double* d1 = A.d1;
      const double* d2 = A.d2;
      const double* lsre = A.Lsre;
      for (int64_t i = c.gt; i < nz; i += c.GT) {
        const double v = (R[i] / alpha - lsre[i]) * d1[i];
        bad |= isnan(v);
        mx[0] = fmax(mx[0], fabs(v));
      }
      for (int64_t i = c.gt; i < ne; i += c.GT) {
        const double v = (R[nz + i] / alpha - Lrz[i]) * d2[i];
        bad |= isnan(v);
        mx[1] = fmax(mx[1], fabs(v));
      }
      cl_reduce<2>(c, mx, 1, bad, wred, part0, red0 + 4);
      tick(3);
    }
    if (sm) {
      const int hn = Sp->h + 1;
      double* rn = A.L.RH[ring(hn, m + 1)];
      const double* rp = A.L.RH[ring(hn - 1, m + 1)];
      double* dn = A.L.DH[ring(hn, m)];
      const bool first = Sp->aa_k == 0;
      vec([&](int64_t i) {
        const double r = R[i];
        dn[i] = first ? r : r - rp[i];
        rn[i] = r;
      });
      cl_gram(c, A.L, Sp, wred, part0, red0 + 8);
      tick(4);
    }
    if (ctl) ctl_begin<false>(A.L);
    csync();
    tick(5);
    const int sw = Sp->sw;
    if (sw == 0) break;
    if (sm) {  // psi = cpsi[0] r + sum_c cpsi[c] r_{k-1-c}
      const int h = Sp->h, nc = Sp->ncpsi;
      double cp[kLoopMaxMem + 1];
      for (int j = 0; j < nc; ++j) cp[j] = Sp->cpsi[j];
      vec([&](int64_t i) {
        double s = cp[0] * R[i];
        for (int q = 1; q < nc; ++q) s += cp[q] * A.L.RH[ring(h - q, m + 1)][i];
        PSI[i] = s;
      });
    }
    if (sw == 1) {  // K0
      vec([&](int64_t i) { V[i] += PSI[i]; });
    } else if (sw == 2) {  // M psi, then the line search (solver.cpp:287-338)
      cl_Lt(c, D, PSI + nz, nullptr, A.tmpz, 0.0, 1.0, 0.0, xs);
      cl_L(c, D, PSI, A.tmpe, xs);
      vec([&](int64_t i) { PV[i] = i < nz ? PSI[i] - alpha * A.tmpz[i] : PSI[i] - alpha * A.tmpe[i - nz]; });
      for (;;) {
        const double tau = Sp->tau;
        vec([&](int64_t i) { C[i] = V[i] + tau * PSI[i]; });
        refresh(C, TC, CR, cLrz);
        {
          double v[2] = {0.0, 0.0};
          for (int64_t i = c.gt; i < nz; i += c.GT) v[0] += CR[i] * PV[i];
          for (int64_t i = c.gt; i < ne; i += c.GT) v[1] += CR[nz + i] * PV[nz + i];
          cl_reduce<2>(c, v, 0, 0, wred, part0, red0 + 3);
        }
        if (ctl) ctl_ls<false>(A.L);
        csync();
        if (!Sp->ls_more) break;
      }
      if (Sp->reason == -2) break;
      const int act = Sp->act;
      if (act == '1') {
        vec([&](int64_t i) {
          V[i] = C[i];
          TV[i] = TC[i];
          R[i] = CR[i];
          if (i < ne) Lrz[i] = cLrz[i];
        });
      } else if (act == '2') {
        const double coef = Sp->coef;
        vec([&](int64_t i) { V[i] -= coef * CR[i]; });
      } else {  // KM fallback
        vec([&](int64_t i) { V[i] = TV[i]; });
      }
    } else {  // CP: v <- T v
      vec([&](int64_t i) { V[i] = TV[i]; });
    }
    if (Sp->refresh) refresh(V, TV, R, Lrz);
    if (ctl) ctl_end<false>(A.L);
    csync();
    if (Sp->reason != -1 || Sp->k >= Sp->k_stop) break;
  }
  csync();
  // results back to HBM: the state (CTA 0) and every writable allocation
  if (c.rank == 0 && t == 0) *CA.S.L.st = S;
  if (A.prof && ctl)
    for (int k = 0; k < 8; ++k) A.prof[k] += (unsigned long long)tacc[k];
  for (int p = 0; p < CA.nplace; ++p) {
    const ClusterPlace P = CA.place[p];
    if (P.cta != c.rank || !P.writable) continue;
    double* dst = const_cast<double*>(reinterpret_cast<const double*>(P.src));
    const double* src = reinterpret_cast<const double*>(arena + P.off);
    for (int64_t i = t; i < P.bytes / 8; i += kSmallThreads) dst[i] = src[i];
  }
  csync();  // no CTA leaves while others may still read its shared memory
}
