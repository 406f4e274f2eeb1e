// Device code of the fused T kernel, instantiated per CTA size by fused.cu
// (FUSED_FT threads per CTA).  See fused.cu for the design notes.

constexpr int kFT = FUSED_FT;  // threads per CTA
constexpr bool kReg = FUSED_REG != 0;  // register-resident critical-path GEMVs (RegGemv)
constexpr int kSlot = kMaxD + 8;  // doubles per scratch vector slot
constexpr int kScratch = 6;       // scratch slots per CTA

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
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
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
// child -> parent hand-off slots (FusedArgs::hand): an empty slot holds
// kHandEmpty, a NaN payload no stored value carries (hand_canon maps every NaN
// to the canonical one), so a parent polls its children's values themselves:
// each 8-byte value is read whole or not yet, and nothing else the parent
// reads comes from the child, so no fence or flag sits on this hop
constexpr unsigned long long kHandEmpty = 0x7FF4DEAD7FF4DEADull;
__device__ __forceinline__ double hand_canon(double v) {
  return v != v ? __longlong_as_double(0x7FF8000000000000ll) : v;
}
__device__ __forceinline__ void st_relaxed(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ double ld_relaxed(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ bool hand_empty(double v) {
  return (unsigned long long)__double_as_longlong(v) == kHandEmpty;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void stamp(const FusedArgs& F, int item, int k) {
  // slots 0..3: %globaltimer (ns, cross-SM ordering); 4..7: clock64 (intra-item phases)
  if (F.trace && threadIdx.x == 0) F.trace[size_t(item) * 8 + k] = k < 4 ? gtimer() : (unsigned long long)clock64();
}

__device__ void wait_flag(const int* f) {
  // tight spin first (the producer is usually one hop away), then back off
  for (int k = 0; k < 64; ++k)
    if (ld_acquire(f) >= 1) return;
  while (ld_acquire(f) < 1) __nanosleep(32);
}
// CTA barrier, then one release store.  bar.sync makes every thread's prior
// writes performed with respect to thread 0, and st.release.gpu is cumulative,
// so a consumer that acquires the flag sees all of them (PTX memory model;
// the extra fence.sc of __threadfence() is not needed).
__device__ __forceinline__ void cta_release(int* flag) {
  __syncthreads();
  if (threadIdx.x == 0) st_release(flag, 1);
}

// Partial GEMV of one warp over its column block [c0, c1): lanes own rows
// (r = lane + 32k), RB independent accumulators per pass, partial sums to
// red[w * ldr + r].  Used by cta_gemv / cta_gemv2 below.
template <int RB>
__device__ __forceinline__ void warp_cols_gemv(const double* A, int m, int lda, const double* x, int c0, int c1,
                                               double* redw) {
  const int l = threadIdx.x & 31;
  for (int rb = 0; rb < m; rb += 32 * RB) {
    double a[RB];
#pragma unroll
    for (int k = 0; k < RB; ++k) a[k] = 0.0;
    int c = c0;
    for (; c + 2 <= c1; c += 2) {
      const double x0 = x[c], x1 = x[c + 1];
      const double* col0 = A + size_t(c) * lda;
      const double* col1 = col0 + lda;
#pragma unroll
      for (int k = 0; k < RB; ++k) {
        const int r = rb + l + 32 * k;
        if (r < m) {
          a[k] = fma(col0[r], x0, a[k]);
          a[k] = fma(col1[r], x1, a[k]);
        }
      }
    }
    for (; c < c1; ++c) {
      const double xc = x[c];
      const double* col = A + size_t(c) * lda;
#pragma unroll
      for (int k = 0; k < RB; ++k) {
        const int r = rb + l + 32 * k;
        if (r < m) a[k] = fma(col[r], xc, a[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < RB; ++k) {
      const int r = rb + l + 32 * k;
      if (r < m) redw[r] = a[k];
    }
  }
}

// y[r] = (acc ? y[r] : 0) + sum_c A[r + c*lda] x[c].  The columns are split in
// kFT/32 contiguous blocks, one per warp (lanes over rows, independent
// accumulators), and the warp partials are summed in warp order: a short
// dependent chain per thread and a fixed, run-to-run identical summation order.
// red holds (kFT/32) * m doubles.
__device__ void cta_gemv(const double* A, int m, int n, int lda, const double* x, double* y, bool acc,
                         double* red) {
  constexpr int NW = kFT / 32;
  if (m <= 0) return;
  const int w = threadIdx.x >> 5;
  const int cb = (n + NW - 1) / NW;
  const int c0 = min(n, w * cb), c1 = min(n, c0 + cb);
  warp_cols_gemv<4>(A, m, lda, x, c0, c1, red + size_t(w) * m);
  __syncthreads();
  for (int t = threadIdx.x; t < m; t += kFT) {
    double o = acc ? y[t] : 0.0;
#pragma unroll
    for (int j = 0; j < NW; ++j) o += red[size_t(j) * m + t];
    y[t] = o;
  }
  __syncthreads();
}

// y1 = A1 x1 (m1 rows) and y2 = A2 x2 (m2 rows) in one pass and one barrier
// pair: every warp takes a column block of each product.  red holds
// (kFT/32) * (m1 + m2) doubles.
__device__ void cta_gemv2(const double* A1, int m1, int n1, int lda1, const double* x1, double* y1,
                          const double* A2, int m2, int n2, int lda2, const double* x2, double* y2, double* red) {
  constexpr int NW = kFT / 32;
  const int w = threadIdx.x >> 5, m = m1 + m2;
  const int cb1 = (n1 + NW - 1) / NW, cb2 = (n2 + NW - 1) / NW;
  const int a0 = min(n1, w * cb1), a1 = min(n1, a0 + cb1);
  const int b0 = min(n2, w * cb2), b1 = min(n2, b0 + cb2);
  warp_cols_gemv<4>(A1, m1, lda1, x1, a0, a1, red + size_t(w) * m);
  warp_cols_gemv<2>(A2, m2, lda2, x2, b0, b1, red + size_t(w) * m + m1);
  __syncthreads();
  for (int t = threadIdx.x; t < m; t += kFT) {
    double o = 0.0;
#pragma unroll
    for (int j = 0; j < NW; ++j) o += red[size_t(j) * m + t];
    if (t < m1)
      y1[t] = o;
    else
      y2[t - m1] = o;
  }
  __syncthreads();
}

// Register-resident GEMV pair for the critical path: the matrix entries a
// thread needs are loaded from shared memory into registers BEFORE the
// dependency wait, so after it only the FMAs over the (new) input vectors, one
// partial store and the ordered partial sums remain.  Stacked rows [A1; A2]:
// P1 threads per row of A1 and P2 per row of A2, each over a contiguous column
// chunk of at most kRegCols; the per-row partials are summed in chunk order.
constexpr int kRegCols = 32;
struct RegGemv {
  double a[kRegCols];
  int row;   // stacked output row (-1: idle thread)
  int c0;    // first column
  int cnt;   // columns held
  int slot;  // partial index: part * (m1 + m2) + row
  int p1, p2;
};
// plan + load; false when a chunk would exceed kRegCols (caller keeps cta_gemv2)
__device__ __forceinline__ bool reg_gemv_load(RegGemv& G, const double* A1, int m1, int n1, int lda1,
                                              const double* A2, int m2, int n2, int lda2) {
  int best = 1 << 30, p1b = 0, p2b = 0;
  constexpr int NW = kFT / 32;  // partials fit the cta_gemv scratch: at most NW per row
  for (int p1 = 1; p1 * m1 <= kFT && p1 <= n1 && p1 <= NW; ++p1) {
    const int p2 = m2 > 0 ? min(min((kFT - p1 * m1) / m2, n2), NW) : 0;
    if (m2 > 0 && p2 < 1) break;
    const int c = max((n1 + p1 - 1) / p1, m2 > 0 ? (n2 + p2 - 1) / p2 : 0);
    if (c < best) best = c, p1b = p1, p2b = p2;
  }
  if (best > kRegCols) return false;
  G.p1 = p1b, G.p2 = p2b;
  const int t = threadIdx.x, m = m1 + m2;
  const double* src = nullptr;
  int lda = 0;
  G.row = -1, G.cnt = 0, G.c0 = 0, G.slot = 0;
  if (t < p1b * m1) {
    const int part = t / m1, cb = (n1 + p1b - 1) / p1b;
    G.row = t - part * m1;
    G.c0 = part * cb;
    G.cnt = max(0, min(cb, n1 - G.c0));
    G.slot = part * m + G.row;
    src = A1 + G.row, lda = lda1;
  } else if (t - p1b * m1 < p2b * m2) {
    const int u = t - p1b * m1, part = u / m2, cb = (n2 + p2b - 1) / p2b;
    const int r = u - part * m2;
    G.row = m1 + r;
    G.c0 = part * cb;
    G.cnt = max(0, min(cb, n2 - G.c0));
    G.slot = part * m + G.row;
    src = A2 + r, lda = lda2;
  }
#pragma unroll
  for (int k = 0; k < kRegCols; ++k) G.a[k] = k < G.cnt ? src[size_t(G.c0 + k) * lda] : 0.0;
  return true;
}
// y1 = A1 x1, y2 = A2 x2 from the registers of reg_gemv_load (two barriers)
__device__ __forceinline__ void reg_gemv_run(const RegGemv& G, int m1, const double* x1, double* y1, int m2,
                                             const double* x2, double* y2, double* red) {
  const int m = m1 + m2;
  if (G.row >= 0) {
    const double* x = (G.row < m1 ? x1 : x2) + G.c0;
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int k = 0; k < kRegCols; k += 2) {
      if (k < G.cnt) s0 = fma(G.a[k], x[k], s0);
      if (k + 1 < G.cnt) s1 = fma(G.a[k + 1], x[k + 1], s1);
    }
    red[G.slot] = s0 + s1;
  }
  __syncthreads();
  for (int r = threadIdx.x; r < m; r += kFT) {
    const int np = r < m1 ? G.p1 : G.p2;
    double o = 0.0;
    for (int j = 0; j < np; ++j) o += red[size_t(j) * m + r];
    if (r < m1)
      y1[r] = o;
    else
      y2[r - m1] = o;
  }
  __syncthreads();
}

__device__ double cta_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < kFT / 32; ++k) s += red[k];
  __syncthreads();
  return s;
}

// v <- a + Pi_SOC(v - a), axis last, in place (projections.cpp:11-37)
__device__ void cta_soc_project(double* v, const double* a, int d, double* red) {
  const int t = threadIdx.x;
  double s = 0.0;
  for (int r = t; r < d; r += kFT) {
    v[r] -= a[r];
    if (r < d - 1) s += v[r] * v[r];
  }
  const double hn = sqrt(cta_sum(s, red));
  const double tt = v[d - 1];
  __syncthreads();  // every thread has read v[d-1] before thread 0 rewrites it
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

// ---------------------------------------------------------------------------
// Span ids of the per-item records (host: Engine::setup_fused).
enum Span : int {
  // backward
  B_HEAD = 0, B_QK, B_ZX, B_ZU, B_EC, B_GD, B_H, B_G, B_HEADN, B_QKN,
  // forward
  F_ZX = 0, F_ZU, F_AX, F_AU, F_FC, F_SEG2, F_A, F_QK, F_GD, F_LO, F_HI, F_SEG3, F_AN, F_QKN, F_GND, F_LON,
  F_HIN, F_SEG1, F_RB
};

struct Slot {
  double* mat;
  double* vec;
  uint64_t* bar;
  int voff[kRecSpans];      // span offsets in vec
  const double* mp[kRecMats];  // staged (or global) matrix pointers
};

// cooperative load of one 512-byte item record into shared memory
__device__ __forceinline__ void load_rec(const FusedArgs& F, int it, ItemRec* dst) {
  const int t = threadIdx.x;
  constexpr int W = int(sizeof(ItemRec) / 16);
  if (t < W) reinterpret_cast<int4*>(dst)[t] = __ldg(reinterpret_cast<const int4*>(F.items + it) + t);
}

// issue the prefetch of an item into a slot: vector spans by cp.async (all
// threads, one commit group per item), matrices by TMA bulk copies (thread 0)
__device__ void issue(const FusedArgs& F, const ItemRec& R, Slot& S) {
  const int t = threadIdx.x;
  int off = 0;
  for (int k = 0; k < R.nspan; ++k) {
    const int n = R.vcnt[k];
    if (n > 0) {
      const double* src = F.base[R.vbase[k]] + R.voff[k];
      double* dst = S.vec + off;
      for (int e = t; e < n; e += kFT) cp_async8(dst + e, src + e);
    }
    if (t == 0) S.voff[k] = off;
    off += (n + 1) & ~1;
  }
  cp_async_commit();
  if (t == 0) {
    const bool stage = F.stage_smem && R.nmat > 0;
    if (stage) {
      fence_proxy_async();
      uint32_t total = 0;
      for (int k = 0; k < R.nmat; ++k)
        if (F.stage_all || (R.mcrit & (1 << k))) total += uint32_t((R.mcnt[k] + 1) & ~1) * 8u;
      if (total)
        mbar_expect_tx(S.bar, total);
      else
        mbar_arrive(S.bar);
    }
    int mo = 0;
    for (int k = 0; k < R.nmat; ++k) {
      const double* src = F.base[R.mbase[k]] + R.moff[k];
      if (!stage || R.mcnt[k] <= 0 || !(F.stage_all || (R.mcrit & (1 << k)))) {
        S.mp[k] = src;
        continue;
      }
      const int padded = (R.mcnt[k] + 1) & ~1;
      bulk_g2s(S.mat + mo, src, uint32_t(padded) * 8u, S.bar);
      S.mp[k] = S.mat + mo;
      mo += padded;
    }
  }
}

// wait on up to kFT flags in parallel (one thread each), then CTA barrier
__device__ __forceinline__ void wait_flags_par(const int* f, int n) {
  const int t = threadIdx.x;
  for (int k = t; k < n; k += kFT) wait_flag(f + k);
  __syncthreads();
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
    double* w = vec;
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

// Backward item.  Everything that does not depend on the children is done
// before the flag wait (own adjoint term, G' ec, cst = h - z_x + a gx - K'(z_u - a gu),
// dc = Rt^-1(z_u - a gu - g)); after it, one parallel GEMV round:
//   T12_i = [M1_i' | M1_i' K_i'] [S_T1 + a S_adjx + cst ; a S_adju],  d_i = dc - Rt^-1 (a S_adju + S_T2)
// (offline B_i = [M1_i' | M1_i' K_i'], Engine::build_combined).
__device__ void item_back(const FusedArgs& F, const ItemRec& P, const Slot& S, double* sc_, double* red) {
  const Dev& D = F.D;
  const int i = P.node;
  const int t = threadIdx.x, nx = D.nx, nu = D.nu, m = nx + nu;
  const bool leaf = P.nch == 0, root = i == 0;
  const double al = F.alpha;
  const double* V = S.vec;
  auto sp = [&](int id) { return V + S.voff[id]; };
  double* gx = sc_;           // G' ec (+ leaf terms)
  double* q = gx + kSlot;     // leaf q / nonleaf v = [v_x; v_u]
  double* tv = q + kSlot;     // scratch (m)
  double* rhs = tv + kSlot;   // scratch: ubc, w
  double* dc = rhs + kSlot;   // Rt^-1 (ubc - g)
  double* rhs2 = dc + kSlot;  // ubc - g
  const int px = P.px, pu = P.pu;
  int mk = 0;
  const double* HxT = root ? nullptr : S.mp[mk++];
  const double* HuT = root ? nullptr : S.mp[mk++];
  const double* Mb = root ? nullptr : S.mp[mk++];  // M1' (leaf) or [M1' | M1'K'] (non-leaf)
  const double* KT = leaf ? nullptr : S.mp[mk++];
  const double* Ri = leaf ? nullptr : S.mp[mk++];
  const double* HNT = leaf ? S.mp[mk++] : nullptr;
  const int item = F.D.nn - 1 - i;  // ticket of this backward item
  if (!leaf) {
    const int nc = P.nc;
    const double* ec = sp(B_EC);
    if (D.g_diag) {
      const double* gd = sp(B_GD);
      for (int r = t; r < m; r += kFT) gx[r] = gd[r] * ec[r];
      __syncthreads();
    } else {
      cta_gemv(D.GxT + D.g_off[i] * nx, nx, nc, nx, ec, gx, false, red);
      cta_gemv(D.GuT + D.g_off[i] * nu, nu, nc, nu, ec, gx + nx, false, red);
    }
  } else {
    const int j = i - D.nnl, nc = P.nc, pN = P.pN;
    const double* ec = sp(B_EC);
    if (D.gN_diag) {
      const double* gd = sp(B_GD);
      for (int r = t; r < nx; r += kFT) gx[r] = gd[r] * ec[r];
      __syncthreads();
    } else {
      cta_gemv(D.GNT + D.gN_off[j] * nx, nx, nc, nx, ec, gx, false, red);
    }
    const double* hd = sp(B_HEADN);
    cta_gemv(HNT, nx, pN, nx, hd, gx, true, red);
    const double rsumN = hd[pN] + hd[pN + 1];
    const double* qk = sp(B_QKN);
    const double* zx = sp(B_ZX);
    for (int r = t; r < nx; r += kFT) q[r] = -(zx[r] - al * (gx[r] - 0.5 * rsumN * qk[r]));  // q = -xbar
  }
  if (!root) {  // own stage-SOC adjoint term for the parent: adj_i = H' head - rsum/2 qk
    const double* head = sp(B_HEAD);
    const double rsum = head[px + pu] + head[px + pu + 1];
    const double* qkv = sp(B_QK);
    for (int r = t; r < m; r += kFT) tv[r] = -0.5 * rsum * qkv[r];
    __syncthreads();
    cta_gemv(HxT, nx, px, nx, head, tv, true, red);
    cta_gemv(HuT, nu, pu, nu, head + px, tv + nx, true, red);
    if (F.hand) {
      double* h = F.hand + size_t(i - 1) * 2 * m + m;
      for (int r = t; r < m; r += kFT) st_relaxed(h + r, hand_canon(tv[r]));
    } else {
      double* adj = D.adj + size_t(i - 1) * m;
      for (int r = t; r < m; r += kFT) adj[r] = tv[r];
    }
  }
  if (leaf) {
    __syncthreads();
    cta_gemv(Mb, m, nx, m, q, tv, false, red);  // T12 = M1' q
    if (F.hand) {
      double* h = F.hand + size_t(i - 1) * 2 * m;
      for (int r = t; r < m; r += kFT) st_relaxed(h + r, hand_canon(tv[r]));
    } else {
      double* T12 = D.T12 + size_t(i - 1) * m;
      for (int r = t; r < m; r += kFT) T12[r] = tv[r];
    }
    cta_release(F.flagB + i);
    stamp(F, item, 2);
    return;
  }
  // ---- non-leaf, before the children: ubc, cst, dc
  {
    const double* zx = sp(B_ZX);
    const double* zu = sp(B_ZU);
    const double* h = sp(B_H);
    const double* gv = sp(B_G);
    for (int r = t; r < nu; r += kFT) {
      const double ubc = zu[r] - al * gx[nx + r];
      rhs[r] = ubc;
      rhs2[r] = ubc - gv[r];
    }
    __syncthreads();
    cta_gemv2(KT, nx, nu, nx, rhs, tv, Ri, nu, nu, nu, rhs2, dc, red);  // K' ubc ; dc
    for (int r = t; r < nx; r += kFT) q[r] = h[r] - zx[r] + al * gx[r] - tv[r];  // cst (into v_x)
    __syncthreads();
  }
  // ---- children (the GEMV round's matrix entries into registers first)
  RegGemv G;
  const bool rg = kReg && !root && reg_gemv_load(G, Mb, m, m, m, Ri, nu, nu, nu);
  const int c0 = P.c0, nch = P.nch;
  if (!F.hand) wait_flags_par(F.flagB + c0, nch);
  stamp(F, item, 1);
  stamp(F, item, 4);
  for (int r = t; r < m; r += kFT) {
    // children terms: up to four children's loads in flight at once (one L2
    // round trip instead of one per child), summed in child order
    double sa = 0.0, st = 0.0;
    for (int c = 0; c < nch; c += 4) {
      double va[4], vt[4];
      if (F.hand) {  // poll the children's slots, then empty them for the next T
        bool full;
        do {
          full = true;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const double* h = F.hand + size_t(c0 + c + k - 1) * 2 * m + r;
            vt[k] = c + k < nch ? ld_relaxed(h) : 0.0;
            va[k] = c + k < nch ? ld_relaxed(h + m) : 0.0;
            full = full && !hand_empty(vt[k]) && !hand_empty(va[k]);
          }
        } while (!full);  // (a backed-off poll measured slower)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (c + k < nch) {
            double* h = F.hand + size_t(c0 + c + k - 1) * 2 * m + r;
            h[0] = __longlong_as_double((long long)kHandEmpty);
            h[m] = __longlong_as_double((long long)kHandEmpty);
          }
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const size_t o = size_t(c0 + c + k - 1) * m + r;
          va[k] = c + k < nch ? ldcg(D.adj + o) : 0.0;
          vt[k] = c + k < nch ? ldcg(D.T12 + o) : 0.0;
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (c + k < nch) {
          sa += va[k];
          st += vt[k];
        }
    }
    if (r < nx) {
      q[r] += st + al * sa;  // v_x
    } else {
      q[r] = al * sa;               // v_u
      rhs[r - nx] = al * sa + st;   // w
    }
  }
  __syncthreads();
  stamp(F, item, 5);
  if (rg)
    reg_gemv_run(G, m, q, tv, nu, rhs, gx, red);  // T12 ; Rt^-1 w
  else if (!root)
    cta_gemv2(Mb, m, m, m, q, tv, Ri, nu, nu, nu, rhs, gx, red);
  else
    cta_gemv(Ri, nu, nu, nu, rhs, gx, false, red);
  stamp(F, item, 6);
  double* dv = D.dvec + size_t(i) * nu;
  for (int r = t; r < nu; r += kFT) dv[r] = dc[r] - gx[r];
  if (!root && F.hand) {
    double* h = F.hand + size_t(i - 1) * 2 * m;
    for (int r = t; r < m; r += kFT) st_relaxed(h + r, hand_canon(tv[r]));
  } else if (!root) {
    double* T12 = D.T12 + size_t(i - 1) * m;
    for (int r = t; r < m; r += kFT) T12[r] = tv[r];
  } else if (t == 0) {
    const double sc = F.eta[P.s1o + P.ny];
    F.zo[0] = F.z[0] - al * sc - al;  // CP primal step on s0 (solver.cpp:153-154)
  }
  stamp(F, item, 7);
  cta_release(F.flagB + i);
  stamp(F, item, 2);
}

__device__ void item_fwd(const FusedArgs& F, const ItemRec& P, const Slot& S, double* sc_, double* red) {
  const Dev& D = F.D;
  const int c = P.node;
  const int t = threadIdx.x, nx = D.nx, nu = D.nu, m = nx + nu;
  const bool leaf = P.nch == 0, root = c == 0;
  const double al = F.alpha;
  const double* z = F.z;
  const double* eta = F.eta;
  double* zo = F.zo;
  double* eo = F.eo;
  const double* V = S.vec;
  auto sp = [&](int id) { return V + S.voff[id]; };
  double* xd = sc_;            // [x_anc+; d_anc]
  double* xn = xd + kSlot;     // own (x+, u+), then (x^, u^)
  double* ahat = xn + kSlot;   // anc (x^, u^)
  double* val = ahat + kSlot;  // segment values
  double* pv = val + kSlot;    // p / alpha
  double* early = pv + kSlot;    // own d (nu), then hat tau_c, hat s_c (loaded early)
  const int px = P.px, pu = P.pu;
  int mk = 0;
  const double* Mf = root ? nullptr : S.mp[mk++];  // M1 (leaf) or [M1; K M1] (non-leaf)
  const double* Hx = root ? nullptr : S.mp[mk++];
  const double* Hu = root ? nullptr : S.mp[mk++];
  const double* K = root ? S.mp[mk++] : nullptr;   // root: u0 = K x_init + d0
  const double* HN = leaf ? S.mp[mk++] : nullptr;
  const int an = root ? 0 : P.anc;
  if (root) {  // before the dependency: K x_init
    for (int r = t; r < nx; r += kFT) xn[r] = D.xinit[r];
    __syncthreads();
    cta_gemv(K, nu, nx, nu, xn, xn + nx, false, red);
  }
  // ---- parent forward (root: own backward), S2 of self and parent; the
  // GEMV's matrix entries into registers first
  RegGemv G;
  const int mr = leaf ? nx : m;
  const bool rg = kReg && !root && reg_gemv_load(G, Mf, mr, m, mr, nullptr, 0, 0, 0);
  const bool fh = F.fhand != nullptr;  // parent values by hand-off slot instead of flagF + L2
  if (t == 0 && (root || !fh)) wait_flag(root ? F.flagB : F.flagF + an);
  else if (t == 32 && !leaf) wait_flag(F.flagS2 + c);
  else if (t == 64 && !root) wait_flag(F.flagS2 + an);
  // own d: with hand-offs no flag chain runs from this node's backward item
  // through the root to here, so a non-leaf acquires its own backward flag
  else if (t == 96 && (F.hand || fh) && !leaf && !root) wait_flag(F.flagB + c);
  __syncthreads();
  stamp(F, F.D.nn + F.D.nnl + c, 1);
  if (!root) {
    const double* zax = sp(F_AX);
    const double* zau = sp(F_AU);
    // hat tau_c, hat s_c (written by the parent's S2): in the same load round
    if (t == kFT - 1) early[nu] = 2.0 * ldcg(zo + D.tau_base + c - 1) - z[D.tau_base + c - 1];
    if (t == kFT - 2) early[nu + 1] = 2.0 * ldcg(zo + D.s_base + c - 1) - z[D.s_base + c - 1];
    // the parent's slot for this node: [x_anc+ | d_anc | u_anc+], emptied after the read
    double* hs = fh ? F.fhand + size_t(c - 1) * (m + nu) : nullptr;
    auto take = [&](int k) {
      double v;
      while (hand_empty(v = ld_relaxed(hs + k))) {
      }
      hs[k] = __longlong_as_double((long long)kHandEmpty);
      return v;
    };
    for (int r = t; r < m; r += kFT) {
      if (r < nx) {
        const double xp = fh ? take(r) : ldcg(zo + 1 + size_t(an) * nx + r);
        xd[r] = xp;
        ahat[r] = 2.0 * xp - zax[r];
      } else {
        xd[r] = fh ? take(r) : ldcg(D.dvec + size_t(an) * nu + (r - nx));
        // own d in the same load round (final: every backward item precedes the root forward)
        if (!leaf) early[r - nx] = ldcg(D.dvec + size_t(c) * nu + (r - nx));
        const double up = fh ? take(m + r - nx) : ldcg(zo + D.u_base + size_t(an) * nu + (r - nx));
        ahat[r] = 2.0 * up - zau[r - nx];
      }
    }
    __syncthreads();
    if (rg)
      reg_gemv_run(G, mr, xd, xn, 0, nullptr, nullptr, red);  // [x; u - d] = Mf xd
    else
      cta_gemv(Mf, mr, m, mr, xd, xn, false, red);
    // one owner per entry: u rows get their own d in the same pass (a second
    // pass indexed by r - nx would race with this one on xn[nx..m))
    const double* fc = sp(F_FC);
    for (int r = t; r < (leaf ? nx : m); r += kFT) {
      double v = xn[r] + fc[r];
      if (!leaf && r >= nx) v += early[r - nx];
      xn[r] = v;
    }
  } else {
    for (int r = t; r < nu; r += kFT) {
      const double d0 = ldcg(D.dvec + r);
      early[r] = d0;  // (own d, for the children's slots)
      xn[nx + r] += d0;
    }
  }
  __syncthreads();
  for (int r = t; r < (leaf ? nx : m); r += kFT) {
    if (r < nx)
      zo[1 + size_t(c) * nx + r] = xn[r];
    else
      zo[D.u_base + size_t(c) * nu + (r - nx)] = xn[r];
  }
  if (fh) {  // children's slots [x+ | d | u+]: no fence, no flag on this hop
    for (int k = 0; k < P.nch; ++k) {
      double* hs = F.fhand + size_t(P.c0 + k - 1) * (m + nu);
      for (int r = t; r < m + nu; r += kFT)
        st_relaxed(hs + r, hand_canon(r < nx ? xn[r] : (r < m ? early[r - nx] : xn[nx + r - m])));
    }
    __syncthreads();  // (xn is doubled in place below)
  } else {
    // children need only (x+, u+) and d: publish before the dual work
    cta_release(F.flagF + c);
  }
  stamp(F, F.D.nn + F.D.nnl + c, 2);
  {
    const double* zx = sp(F_ZX);
    const double* zu = sp(F_ZU);
    for (int r = t; r < (leaf ? nx : m); r += kFT) xn[r] = 2.0 * xn[r] - (r < nx ? zx[r] : zu[r - nx]);
  }
  const double* hat = xn;
  __syncthreads();
  auto hatv = [&](int idx) { return 2.0 * ldcg(zo + idx) - z[idx]; };
  if (!root) {  // stage-cost SOC block of (x_anc, u_anc, tau_c)
    const int p = px + pu, o2 = P.s2o;
    const double* qk = sp(F_QK);
    double part = 0.0;
    for (int r = t; r < m; r += kFT) part += qk[r] * ahat[r];
    const double qd = cta_sum(part, red);
    cta_gemv(Hx, px, nx, px, ahat, val, false, red);
    cta_gemv(Hu, pu, nu, pu, ahat + nx, val + px, false, red);
    if (t == 0) {
      const double row = 0.5 * early[nu] - 0.5 * qd;  // hat tau_c
      val[p] = row;
      val[p + 1] = row;
    }
    __syncthreads();
    const double* seg = sp(F_SEG2);
    for (int r = t; r < p + 2; r += kFT) {
      const double pp = seg[r] + al * val[r];
      val[r] = pp;
      pv[r] = pp / al;
    }
    __syncthreads();
    cta_soc_project(pv, sp(F_A), p + 2, red);
    for (int r = t; r < p + 2; r += kFT) eo[o2 + r] = val[r] - al * pv[r];
    __syncthreads();
  }
  if (!leaf) {  // y-copy rows (dual cone), risk scalar (R+), constraint rows (box)
    const int ny = P.ny, yo = P.yo, so = P.s1o, nc = P.nc;
    const bool pre = P.vcnt[F_SEG1] > 0;
    const double* seg1 = pre ? sp(F_SEG1) : eta + so;
    const double* rb = pre ? sp(F_RB) : D.rb + (yo - D.y_base);
    const int nn0 = D.yc_nonneg[c];
    double part = 0.0;
    for (int r = t; r < ny; r += kFT) {
      const double yh = hatv(yo + r);
      part += rb[r] * yh;
      const double pp = seg1[r] + al * yh;
      double tp = pp / al;
      if (nn0 >= 0) {
        if (r < nn0) tp = fmax(tp, 0.0);
        eo[so + r] = pp - al * tp;
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
        const double pp = seg1[r] + al * hatv(yo + r);
        eo[so + r] = pp - al * eo[so + r];
      }
    }
    if (t == 0) {
      const double sv = (c == 0 ? hatv(0) : early[nu + 1]) - by;
      const double pp = seg1[ny] + al * sv;
      eo[so + ny] = pp - al * fmax(0.0, pp / al);
    }
    // constraint rows G [x^; u^] with box projection
    if (D.g_diag) {
      const double* gd = sp(F_GD);
      for (int r = t; r < nc; r += kFT) val[r] = gd[r] * hat[r];
      __syncthreads();
    } else {
      cta_gemv(D.Gx + D.g_off[c] * nx, nc, nx, nc, hat, val, false, red);
      cta_gemv(D.Gu + D.g_off[c] * nu, nc, nu, nc, hat + nx, val, true, red);
    }
    const double* lo = sp(F_LO);
    const double* hi = sp(F_HI);
    const double* ec = seg1 + ny + 1;
    for (int r = t; r < nc; r += kFT) {
      const double pp = ec[r] + al * val[r];
      eo[so + ny + 1 + r] = pp - al * fmin(fmax(pp / al, lo[r]), hi[r]);
    }
    __syncthreads();
  } else {  // leaf: G_N x^ (box) and the terminal SOC block of (x, s)
    const int j = c - D.nnl, nc = P.nc, eo3 = P.s3o, p = P.pN;
    const double* seg3 = sp(F_SEG3);
    if (D.gN_diag) {
      const double* gd = sp(F_GND);
      for (int r = t; r < nc; r += kFT) val[r] = gd[r] * hat[r];
      __syncthreads();
    } else {
      cta_gemv(D.GN + D.gN_off[j] * nx, nc, nx, nc, hat, val, false, red);
    }
    const double* lo = sp(F_LON);
    const double* hi = sp(F_HIN);
    for (int r = t; r < nc; r += kFT) {
      const double pp = seg3[r] + al * val[r];
      eo[eo3 + r] = pp - al * fmin(fmax(pp / al, lo[r]), hi[r]);
    }
    __syncthreads();
    const double* qk = sp(F_QKN);
    double part = 0.0;
    for (int r = t; r < nx; r += kFT) part += qk[r] * hat[r];
    const double qd = cta_sum(part, red);
    cta_gemv(HN, p, nx, p, hat, val, false, red);
    if (t == 0) {
      const double row = 0.5 * early[nu + 1] - 0.5 * qd;  // hat s_c
      val[p] = row;
      val[p + 1] = row;
    }
    __syncthreads();
    const double* hs = seg3 + nc;
    for (int r = t; r < p + 2; r += kFT) {
      const double pp = hs[r] + al * val[r];
      val[r] = pp;
      pv[r] = pp / al;
    }
    __syncthreads();
    cta_soc_project(pv, sp(F_AN), p + 2, red);
    for (int r = t; r < p + 2; r += kFT) eo[eo3 + nc + r] = val[r] - al * pv[r];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kFT, 1) k_T_fused(FusedArgs F) {
  extern __shared__ __align__(1024) double dsm[];
  __shared__ uint64_t bars[2];
  __shared__ Slot slots[2];
  __shared__ int tk[2];
  __shared__ ItemRec recs[2];
  const int t = threadIdx.x;
  double* scratch = dsm + F.nslots * (size_t(F.mat_doubles) + F.vec_doubles);
  double* red = scratch + kScratch * kSlot;  // F.red_doubles (GEMV warp partials, CTA sums)
  if (t == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < 2; ++s) {
      slots[s].mat = dsm + (F.nslots > 1 ? s : 0) * (size_t(F.mat_doubles) + F.vec_doubles);
      slots[s].vec = slots[s].mat + F.mat_doubles;
      slots[s].bar = &bars[s];
    }
    tk[0] = int(atomicAdd(F.ticket, 1ull));
  }
  uint32_t phase[2] = {0u, 0u};
  const int total = F.D.nnl + 2 * F.D.nn;

  __syncthreads();
  int cur = 0;
  if (tk[0] < total) {
    load_rec(F, tk[0], &recs[0]);
    __syncthreads();
    issue(F, recs[0], slots[0]);
  } else {
    cp_async_commit();
  }
  const bool ring = F.nslots > 1;
  for (;;) {
    const int it = tk[cur];
    if (it >= total) break;
    const int nxt = ring ? cur ^ 1 : cur;
    // take and prefetch the next item into the other slot (two-slot ring)
    if (ring) {
      if (t == 0) tk[nxt] = int(atomicAdd(F.ticket, 1ull));
      __syncthreads();
      const int itn = tk[nxt];
      if (itn < total) {
        load_rec(F, itn, &recs[nxt]);
        __syncthreads();
        issue(F, recs[nxt], slots[nxt]);
      } else {
        cp_async_commit();  // keep one group per item in flight
      }
    } else {
      cp_async_commit();
    }
    // wait for the current item's operands (all but the newest cp.async group)
    cp_async_wait<1>();
    const ItemRec& P = recs[cur];
    if (P.kind != 0 && F.stage_smem && P.nmat > 0) {
      while (!mbar_try_wait(slots[cur].bar, phase[cur])) {
      }
      phase[cur] ^= 1u;
    }
    __syncthreads();
    stamp(F, it, 0);
    if (P.kind == 0) {
      item_s2(F, P.node, red, scratch);
      cta_release(F.flagS2 + P.node);
    } else if (P.kind == 1) {
      item_back(F, P, slots[cur], scratch, red);
    } else {
      item_fwd(F, P, slots[cur], scratch, red);
    }
    __syncthreads();
    stamp(F, it, 3);
    if (!ring) {  // single slot: take and prefetch the next item now
      if (t == 0) tk[cur] = int(atomicAdd(F.ticket, 1ull));
      __syncthreads();
      if (tk[cur] < total) {
        load_rec(F, tk[cur], &recs[cur]);
        __syncthreads();
        issue(F, recs[cur], slots[cur]);
      }
    }
    cur = nxt;
  }
  cp_async_wait<0>();
}

