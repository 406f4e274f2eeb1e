// Device engine of the B200 SPOCK solver (see engine.hpp).
//
// Reference map (arxiv/paper_2505_12078):
//   Engine::Engine       <- SpockSolver::SpockSolver   proj/src/solver.cpp:79-114
//   Engine::factorize    <- make_solver_cache Alg. 1   proj/src/projections.cpp:59-140 (on device)
//   Engine::power_iteration <- estimate_norm           proj/src/tree_operator.cpp:157-212 (on device)
//   Engine::T            <- SpockSolver::apply_T       proj/src/solver.cpp:148-164
//   Engine::solve_b      <- SpockSolver::run           proj/src/solver.cpp:189-350
#include "engine.hpp"
#include "aa.cuh"
#include "setup_dev.hpp"
#include "nccl_dl.hpp"

#include <chrono>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>

namespace spock {

#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) throw CudaError(std::string("CUDA error: ") + cudaGetErrorString(e_) + \
                                           " at " #x);                                         \
  } while (0)

namespace {
inline int64_t pad2(int64_t n) { return (n + 1) & ~int64_t(1); }
void require(bool c, const char* m) {
  if (!c) throw std::invalid_argument(m);
}
bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}
}  // namespace

void Params::validate() const {  // proj/src/solver.cpp:9-19
  if (eps_abs <= 0.0 || eps_rel < 0.0) throw std::invalid_argument("SpockParams: bad tolerances");
  if (alpha < 0.0) throw std::invalid_argument("SpockParams: alpha must be >= 0");
  if (aa_memory < 1) throw std::invalid_argument("SpockParams: aa_memory must be >= 1");
  if (c0 < 0.0 || c0 >= 1.0 || c1 < 0.0 || c1 >= 1.0 || c2 < 0.0 || c2 >= 1.0)
    throw std::invalid_argument("SpockParams: c0, c1, c2 must be in [0, 1)");
  if (beta <= 0.0 || beta >= 1.0 || sigma <= 0.0 || sigma >= 1.0)
    throw std::invalid_argument("SpockParams: beta, sigma must be in (0, 1)");
  if (lambda <= 0.0 || lambda >= 2.0) throw std::invalid_argument("SpockParams: lambda must be in (0, 2)");
  if (max_iters < 1 || max_backtracks < 1) throw std::invalid_argument("SpockParams: bad iteration caps");
  if (aa_memory > kAaHostMax) throw std::invalid_argument("SpockParams: aa_memory above 64 is not supported on device");
}

template <class Ty>
Ty* Engine::dalloc(size_t n) {
  void* p = nullptr;
  // two spare elements: aligned 16-byte bulk copies of a trailing odd element stay in bounds
  const size_t bytes = (std::max<size_t>(n, 1) + 2) * sizeof(Ty);
  CK(cudaMalloc(&p, bytes));
  CK(cudaMemsetAsync(p, 0, bytes, st_));
  allocs_.push_back(p);
  alloc_bytes_[reinterpret_cast<uintptr_t>(p)] = bytes;
  return static_cast<Ty*>(p);
}
double* Engine::dupload(const BigVec& h) {
  double* d = dalloc<double>(h.size());
  if (!h.empty()) CK(cudaMemcpyAsync(d, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice, st_));
  return d;
}
template <class Ty>
Ty* Engine::dupload(const std::vector<Ty>& h) {
  Ty* d = dalloc<Ty>(h.size());
  if (!h.empty()) CK(cudaMemcpyAsync(d, h.data(), h.size() * sizeof(Ty), cudaMemcpyHostToDevice, st_));
  return d;
}

Engine::Engine(const spock_problem_desc* desc, const Params& prm) : prm_(prm) {
  // SPOCK_DEBUG_SETUP=1: wall time of each setup phase on stderr
  const bool dbg = std::getenv("SPOCK_DEBUG_SETUP") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!dbg) return;
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[setup] %-22s %8.1f ms\n", what,
                 std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  };
  prm_.validate();
  p_ = problem_from_desc(desc);
  raw_xinit_ = p_.x_init;  // the unscaled initial state (the solve default)
  mark("problem_from_desc");
  pc_ = prm_.use_preconditioner ? precondition_inplace(p_) : identity_precond(p_);
  mark("precondition");
  require(p_.nx + p_.nu <= kMaxD, "spock-b200: nx + nu above 256 is not supported");
  CK(cudaGetDevice(&dev_));
  CK(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
  {
    // SOC epigraph data on the device (SPOCK_HOST_SOC=1: the host restatement)
    const char* hs = std::getenv("SPOCK_HOST_SOC");
    soc_dev_ = !(hs && hs[0] == '1') && p_.nx <= kEigMaxN && p_.tree.nn() > 1;
    if (soc_dev_) {
      soc_device_ranks();
    } else {
      soc_ = soc_epigraph_data(p_);
    }
  }
  mark(soc_dev_ ? "soc ranks (device)" : "soc_epigraph_data");
  lay_ = make_layouts(p_, soc_);
  stage_start_ = p_.tree.stage_start;
  set_carveout_all();
  set_carveout_narrow();
  mark("layouts + stream");
  upload();
  CK(cudaStreamSynchronize(st_));
  mark("upload");
  narrow_ = p_.tree.nn() < 4096;
  if (const char* nv = std::getenv("SPOCK_NARROW")) narrow_ = nv[0] == '1';
  factorize();
  CK(cudaStreamSynchronize(st_));
  mark("factorize (Alg. 1)");
  norm_.analytic_bound = analytic_norm_bound(p_, soc_);
  mark("analytic bound");
  compute_pool();
  mark("pooled blocks");
  setup_fused();
  setup_wide(false);
  CK(cudaStreamSynchronize(st_));
  mark("fused / wide records");
  power_iteration();
  alpha_ = prm_.alpha > 0.0 ? prm_.alpha : 0.99 / std::max(norm_.estimate, 1e-300);
  {  // CTA-resident loop (small.cuh) for trees whose CP application streams little
    const char* env = std::getenv("SPOCK_SMALL");
    double b[5];
    traffic(b);
    // default off: measured slower than the graph loop on c1 (127 vs 91 us per CP
    // iteration): one SM cannot hold c1's ~0.2 MB of blocks plus iterates in
    // L1, so every warp-per-node body pays a chain of L2 round trips (~5 k
    // cycles per node; SPOCK_SMALL_PROF=1 breakdown in DESIGN.md §5)
    small_ok_ = env && env[0] == '1';
    // cluster-resident loop: on when the small loop's whole device image fits
    // in the shared memory of a cluster (SPOCK_CLUSTER=0 disables it)
    const char* cenv = std::getenv("SPOCK_CLUSTER");
    const int64_t nv = lay_.nz + lay_.neta;
    const double image = b[4] + 8.0 * double(nv) * (13 + 2 * prm_.aa_memory);
    int cl_ok = 0;
    CK(cudaDeviceGetAttribute(&cl_ok, cudaDevAttrClusterLaunch, dev_));
    if (!small_ok_ && !(cenv && cenv[0] == '0') && cl_ok && prm_.aa_memory <= kLoopMaxMem &&
        image < double(kClusterMax) * 150e3) {
      small_alloc();
      cluster_ok_ = cluster_plan(prm_.aa_memory);
    }
  }
  CK(cudaStreamSynchronize(st_));
  mark("power iteration");
  // the per-node blocks now live on the device: release the host copies (GBs on
  // wide trees; several ranks of a sharded run share one host)
  p_.A = BigVec();
  p_.B = BigVec();
  p_.Q = BigVec();
  p_.R = BigVec();
  p_.QN = BigVec();
  p_.Gx = BigVec();
  p_.Gu = BigVec();
  p_.GN = BigVec();
}

// Persistent dataflow T (fused.cu): flags, ticket, shared-memory staging size
// and grid.  Falls back to the per-stage kernels only for shapes the fused
// kernel does not cover (constraint rows above 256) or on request
// (SPOCK_T_UNFUSED=1, used by the tests that compare both paths).
void Engine::setup_fused() {
  const Tree& tr = p_.tree;
  const int nn = tr.nn(), nnl = tr.nnl(), nx = p_.nx, nu = p_.nu, m = nx + nu;
  fused_ok_ = true;
  for (int i = 0; i < nnl; ++i)
    if (p_.nc[i] > kMaxD) fused_ok_ = false;
  for (int j = 0; j < tr.nl(); ++j)
    if (p_.ncN[j] > kMaxD) fused_ok_ = false;
  // Measured on B200 (profiles/r01_fused_configs.md): the dataflow kernel
  // wins on narrow trees (c2, 223 nodes: 0.105 ms vs 1.21 ms per T), the
  // stage-parallel kernels on wide ones (c3, 36085 nodes: 3.05 ms vs 3.30 ms).
  const char* env = std::getenv("SPOCK_T_UNFUSED");
  const char* fenv = std::getenv("SPOCK_T_FUSED");
  if (env && env[0] == '1') fused_ok_ = false;
  if (!(fenv && fenv[0] == '1') && nn >= 4096) fused_ok_ = false;
  if (!fused_ok_) return;
  // largest per-item set of staged blocks and prefetched vector spans (even
  // doubles each), mirroring make_plan in fused.cu
  auto knob = [](const char* name, int dflt) {
    const char* v = std::getenv(name);
    return (v && v[0]) ? std::atoi(v) : dflt;
  };
  // defaults: wide trees stream more bytes per SM with 128-thread CTAs and
  // critical-only staging; narrow trees favour a 256-thread ring
  const bool wide = nn >= 4096;
  const int sall = knob("SPOCK_FUSED_STAGEALL", wide ? 0 : 1);
  // measured in the SuperMann loop (tools/e2e_probe.py): 2 slots on c2 (252 vs 280 ms / 500 it),
  // 1 slot (two CTAs per SM) on c2p (215 vs 259 ms / 300 it)
  const int nslots = knob("SPOCK_FUSED_SLOTS", nn < 512 ? 2 : 1);
  const int threads = knob("SPOCK_FUSED_FT", wide ? 128 : 256) == 128 ? 128 : 256;
  int64_t mx = 0, vx = 0;
  for (int i = 0; i < nn; ++i) {
    const bool leaf = tr.leaf(i), root = i == 0;
    int64_t b = 0, f = 0, vb = pad2(nx), vf = pad2(nx);
    if (!root) {
      const int px = soc_.stage[i - 1].px, pu = soc_.stage[i - 1].pu, p = px + pu;
      const int64_t mb = leaf ? int64_t(m) * nx : int64_t(m) * m;  // M1' or [M1' | M1'K']
      const int64_t mf = leaf ? int64_t(nx) * m : int64_t(m) * m;  // M1 or [M1; K M1]
      b += (sall ? pad2(int64_t(px) * nx) + pad2(int64_t(pu) * nu) : 0) + pad2(mb);
      f += pad2(mf) + (sall ? pad2(int64_t(px) * nx) + pad2(int64_t(pu) * nu) : 0);
      vb += pad2(p + 2) + pad2(m);
      vf += pad2(nx) + pad2(nu) + pad2(m) + 2 * pad2(p + 2) + pad2(m);
    }
    if (!leaf) {
      const int nc = p_.nc[i], ny = lay_.y_dim[i];
      b += pad2(int64_t(nx) * nu) + pad2(int64_t(nu) * nu);
      if (root) f += pad2(int64_t(nu) * nx);
      vb += pad2(nu) + pad2(nc) + (D_.g_diag ? pad2(m) : 0) + pad2(nx) + pad2(nu);
      vf += pad2(nu) + (D_.g_diag ? pad2(m) : 0) + 2 * pad2(nc);
      if (ny + 1 + nc <= kMaxD) vf += pad2(ny + 1 + nc) + pad2(ny);
    } else {
      const int j = i - tr.nnl(), pN = soc_.leaf[j].px, nc = p_.ncN[j];
      b += sall ? pad2(int64_t(pN) * nx) : 0;
      f += sall ? pad2(int64_t(pN) * nx) : 0;
      vb += pad2(nc) + (D_.gN_diag ? pad2(nx) : 0) + pad2(pN + 2) + pad2(nx);
      vf += pad2(nc + pN + 2) + pad2(pN + 2) + pad2(nx) + (D_.gN_diag ? pad2(nx) : 0) + 2 * pad2(nc);
    }
    mx = std::max(mx, std::max(b, f));
    vx = std::max(vx, std::max(vb, vf));
  }
  FusedArgs& F = fargs_;
  F = FusedArgs{};
  F.stage_smem = 1;
  F.stage_all = sall;
  F.nslots = nslots > 1 ? 2 : 1;
  F.threads = threads;
  F.mat_doubles = int(mx);
  F.vec_doubles = int(vx);
  {
    int rows = std::max(m + nu, 64);  // cta_gemv2 stacks m + nu rows; cta_sum needs 8
    for (int i = 0; i < nnl; ++i) rows = std::max(rows, p_.nc[i]);
    for (int j = 0; j < tr.nl(); ++j) rows = std::max(rows, p_.ncN[j]);
    rows = std::max(rows, max_dense_s2_);
    F.red_doubles = int(pad2((threads / 32) * int64_t(rows)));
  }
  int dev = 0, sms = 148, smem_optin = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const char* ns = std::getenv("SPOCK_FUSED_NOSTAGE");
  if ((ns && ns[0] == '1') || fused_smem_bytes(F) + 8192 > smem_optin) {  // stream blocks from L2/HBM
    F.stage_smem = 0;
    F.mat_doubles = 0;
  }
  if (fused_smem_bytes(F) + 8192 > smem_optin) {  // even the vector ring does not fit
    fused_ok_ = false;
    return;
  }
  const int bytes = fused_smem_bytes(F);
  // register-resident GEMVs (~250 registers per thread): with the two-slot
  // ring a CTA fills an SM's shared memory anyway; measured on c2 (m = 75):
  // GEMV round 1.9 k -> 1.0 k cycles per tree level, T 82.5 -> 77.6 us
  {
    const int r = knob("SPOCK_FUSED_REG", -1);
    F.reg_gemv = r >= 0 ? (r != 0 && F.threads == 256) : (F.threads == 256 && F.nslots == 2 && m >= 32);
  }
  CK(fused_configure(bytes, F.threads, F.reg_gemv));
  int occ = 0;
  F.D = D_;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fused_kernel_ptr(F.threads, F.reg_gemv), F.threads, bytes));
  const int occ_cap = std::max(1, knob("SPOCK_FUSED_OCC", 4));
  fused_grid_ = std::max(1, std::min(occ, occ_cap)) * sms;
  const int total = nnl + 2 * nn;
  fused_grid_ = std::min(fused_grid_, total);
  fused_grid_full_ = fused_grid_;
  if (const int cap = knob("SPOCK_FUSED_GRID", 0); cap > 0) fused_grid_ = std::min(fused_grid_, cap);
  const size_t fb = 8 + sizeof(int) * size_t(nnl + 2 * nn);
  fused_sync_bytes_ = fb;
  char* buf = dalloc<char>(fb);
  F.ticket = reinterpret_cast<unsigned long long*>(buf);
  F.flagS2 = reinterpret_cast<int*>(buf + 8);
  F.flagB = F.flagS2 + nnl;
  F.flagF = F.flagB + nn;
  // child -> parent hand-off slots: a parent polls its children's T12 and L*
  // terms themselves, with no release fence and no flag on that hop
  // (bit 0: backward sweep; bit 1: forward sweep, parent -> child (x+, d, u+))
  const int hand = nn > 1 ? knob("SPOCK_FUSED_HAND", 3) : 0;
  if (hand & 1) {
    F.hand = dalloc<double>(size_t(nn - 1) * 2 * m);
    launch_hand_clear(F.hand, int64_t(nn - 1) * 2 * m, st_);
  }
  if (hand & 2) {
    F.fhand = dalloc<double>(size_t(nn - 1) * (m + nu));
    launch_hand_clear(F.fhand, int64_t(nn - 1) * (m + nu), st_);
  }
  // offline combined blocks B = [M1' | M1'K'], F = [M1; K M1], f = [c; K c]
  const int64_t cs = pad2(int64_t(m) * m);
  double* dBm = dalloc<double>(size_t(std::max(nn - 1, 1)) * cs);
  double* dFm = dalloc<double>(size_t(std::max(nn - 1, 1)) * cs);
  double* dfc = dalloc<double>(size_t(std::max(nn - 1, 1)) * m);
  launch_build_combined(D_, dBm, dFm, dfc, cs, st_);
  CK(cudaGetLastError());
  // per-item records (prefetch plans + metadata), mirroring the span ids of fused.cu
  enum { B_HEAD = 0, B_QK, B_ZX, B_ZU, B_EC, B_GD, B_H, B_G, B_HEADN, B_QKN };
  enum { F_ZX = 0, F_ZU, F_AX, F_AU, F_FC, F_SEG2, F_A, F_QK, F_GD, F_LO, F_HI, F_SEG3, F_AN, F_QKN, F_GND,
         F_LON, F_HIN, F_SEG1, F_RB };
  // ticket order: [backward nn-1..0][S2 of each parent][forward 0..nn-1]
  std::vector<ItemRec> recs(size_t(nnl) + 2 * size_t(nn));
  std::vector<int64_t> hx_off(nn - 1), hu_off(nn - 1), a_off(nn - 1), hn_off(tr.nl()), aN_off(tr.nl());
  {
    int64_t sx = 0, su = 0, sa = 0;
    for (int k = 0; k < nn - 1; ++k) {
      hx_off[k] = sx, hu_off[k] = su, a_off[k] = sa;
      sx += pad2(int64_t(soc_.stage[k].px) * nx);
      su += pad2(int64_t(soc_.stage[k].pu) * nu);
      sa += soc_.stage[k].px + soc_.stage[k].pu + 2;
    }
    int64_t sh = 0, sb = 0;
    for (int j = 0; j < tr.nl(); ++j) {
      hn_off[j] = sh, aN_off[j] = sb;
      sh += pad2(int64_t(soc_.leaf[j].px) * nx);
      sb += soc_.leaf[j].px + 2;
    }
  }
  auto fill_meta = [&](ItemRec& R, int i) {
    R.node = i;
    R.nch = tr.child_count[i];
    R.c0 = tr.child_first[i];
    R.anc = tr.anc[i];
    R.px = i > 0 ? soc_.stage[i - 1].px : 0;
    R.pu = i > 0 ? soc_.stage[i - 1].pu : 0;
    R.s2o = i > 0 ? lay_.seg2_off[i - 1] : 0;
    if (i < nnl) {
      R.nc = p_.nc[i], R.ny = lay_.y_dim[i], R.s1o = lay_.seg1_off[i], R.yo = lay_.y_off[i];
    } else {
      const int j = i - nnl;
      R.nc = p_.ncN[j], R.pN = soc_.leaf[j].px, R.s3o = lay_.seg3_off[j];
    }
  };
  auto mat = [&](ItemRec& R, int base, int64_t off, int64_t cnt, bool crit) {
    if (crit) R.mcrit |= uint8_t(1u << R.nmat);
    R.mbase[R.nmat] = uint8_t(base);
    R.moff[R.nmat] = off;
    R.mcnt[R.nmat] = int32_t(cnt);
    ++R.nmat;
  };
  auto vec = [&](ItemRec& R, int id, int base, int64_t off, int64_t cnt) {
    R.vbase[id] = uint8_t(base);
    R.voff[id] = off;
    R.vcnt[id] = int32_t(cnt);
    R.nspan = std::max(R.nspan, id + 1);
  };
  for (int it = 0; it < nnl; ++it) {
    ItemRec& R = recs[size_t(nn) + it];
    std::memset(&R, 0, sizeof(R));
    R.kind = 0;
    fill_meta(R, it);
  }
  for (int k = 0; k < nn; ++k) {  // backward items: node nn-1 ... 0
    const int i = nn - 1 - k;
    ItemRec& R = recs[size_t(k)];
    std::memset(&R, 0, sizeof(R));
    R.kind = 1;
    fill_meta(R, i);
    const bool leaf = tr.leaf(i), root = i == 0;
    if (!root) {
      const int px = R.px, pu = R.pu;
      mat(R, FB_HXT, hx_off[i - 1], int64_t(px) * nx, false);
      mat(R, FB_HUT, hu_off[i - 1], int64_t(pu) * nu, false);
      if (leaf)
        mat(R, FB_M1T, int64_t(i - 1) * D_.m1_stride, int64_t(m) * nx, true);
      else
        mat(R, FB_BM, int64_t(i - 1) * cs, int64_t(m) * m, true);
      vec(R, B_HEAD, FB_ETA, lay_.seg2_off[i - 1], px + pu + 2);
      vec(R, B_QK, FB_QK, int64_t(i - 1) * m, m);
    }
    vec(R, B_ZX, FB_Z, 1 + int64_t(i) * nx, nx);
    if (!leaf) {
      mat(R, FB_KT, int64_t(i) * D_.k_stride, int64_t(nx) * nu, true);
      mat(R, FB_RINV, int64_t(i) * D_.r_stride, int64_t(nu) * nu, true);
      vec(R, B_ZU, FB_Z, lay_.u_base + int64_t(i) * nu, nu);
      vec(R, B_EC, FB_ETA, lay_.seg1_off[i] + lay_.y_dim[i] + 1, p_.nc[i]);
      if (D_.g_diag) vec(R, B_GD, FB_GD, int64_t(i) * m, m);
      vec(R, B_H, FB_H, int64_t(i) * nx, nx);
      vec(R, B_G, FB_G, int64_t(i) * nu, nu);
    } else {
      const int j = i - nnl, pN = R.pN, nc = R.nc;
      mat(R, FB_HNT, hn_off[j], int64_t(pN) * nx, false);
      vec(R, B_EC, FB_ETA, lay_.seg3_off[j], nc);
      if (D_.gN_diag) vec(R, B_GD, FB_GND, int64_t(j) * nx, nx);
      vec(R, B_HEADN, FB_ETA, lay_.seg3_off[j] + nc, pN + 2);
      vec(R, B_QKN, FB_QKN, int64_t(j) * nx, nx);
    }
  }
  for (int c = 0; c < nn; ++c) {  // forward items: node 0 ... nn-1
    ItemRec& R = recs[size_t(nn) + nnl + c];
    std::memset(&R, 0, sizeof(R));
    R.kind = 2;
    fill_meta(R, c);
    const bool leaf = tr.leaf(c), root = c == 0;
    vec(R, F_ZX, FB_Z, 1 + int64_t(c) * nx, nx);
    if (!leaf) vec(R, F_ZU, FB_Z, lay_.u_base + int64_t(c) * nu, nu);
    if (!root) {
      const int px = R.px, pu = R.pu, an = R.anc, p = px + pu;
      if (leaf)
        mat(R, FB_M1, int64_t(c - 1) * D_.m1_stride, int64_t(nx) * m, true);
      else
        mat(R, FB_FM, int64_t(c - 1) * cs, int64_t(m) * m, true);
      mat(R, FB_HX, hx_off[c - 1], int64_t(px) * nx, false);
      mat(R, FB_HU, hu_off[c - 1], int64_t(pu) * nu, false);
      vec(R, F_AX, FB_Z, 1 + int64_t(an) * nx, nx);
      vec(R, F_AU, FB_Z, lay_.u_base + int64_t(an) * nu, nu);
      vec(R, F_FC, FB_FC, int64_t(c - 1) * m, leaf ? nx : m);
      vec(R, F_SEG2, FB_ETA, lay_.seg2_off[c - 1], p + 2);
      vec(R, F_A, FB_A, a_off[c - 1], p + 2);
      vec(R, F_QK, FB_QK, int64_t(c - 1) * m, m);
    }
    if (root) mat(R, FB_K, int64_t(c) * D_.k_stride, int64_t(nu) * nx, true);
    if (!leaf) {
      const int nc = p_.nc[c], ny = lay_.y_dim[c];
      const int64_t go = p_.g_off[c];
      if (D_.g_diag) vec(R, F_GD, FB_GD, int64_t(c) * m, m);
      vec(R, F_LO, FB_LO, go, nc);
      vec(R, F_HI, FB_HI, go, nc);
      if (ny + 1 + nc <= kMaxD) {
        vec(R, F_SEG1, FB_ETA, lay_.seg1_off[c], ny + 1 + nc);
        vec(R, F_RB, FB_RB, lay_.y_off[c] - D_.y_base, ny);
      }
    } else {
      const int j = c - nnl, pN = R.pN, nc = R.nc;
      const int64_t go = p_.gN_off[j];
      mat(R, FB_HN, hn_off[j], int64_t(pN) * nx, false);
      vec(R, F_SEG3, FB_ETA, lay_.seg3_off[j], nc + pN + 2);
      vec(R, F_AN, FB_AN, aN_off[j], pN + 2);
      vec(R, F_QKN, FB_QKN, int64_t(j) * nx, nx);
      if (D_.gN_diag) vec(R, F_GND, FB_GND, int64_t(j) * nx, nx);
      vec(R, F_LON, FB_LON, go, nc);
      vec(R, F_HIN, FB_HIN, go, nc);
    }
  }
  ItemRec* drec = nullptr;
  CK(cudaMalloc(&drec, sizeof(ItemRec) * recs.size()));
  allocs_.push_back(drec);
  CK(cudaMemcpyAsync(drec, recs.data(), sizeof(ItemRec) * recs.size(), cudaMemcpyHostToDevice, st_));
  F.items = drec;
  const double* bases[FB_COUNT] = {};
  bases[FB_HXT] = D_.HxT, bases[FB_HUT] = D_.HuT, bases[FB_M1T] = D_.M1T, bases[FB_KT] = D_.KT;
  bases[FB_RINV] = D_.Rinv, bases[FB_HNT] = D_.HNT, bases[FB_QK] = D_.qk, bases[FB_GD] = D_.gd;
  bases[FB_H] = D_.h, bases[FB_G] = D_.g, bases[FB_QKN] = D_.qkN, bases[FB_GND] = D_.gNd;
  bases[FB_M1] = D_.M1, bases[FB_HX] = D_.Hx, bases[FB_HU] = D_.Hu, bases[FB_K] = D_.K, bases[FB_HN] = D_.HN;
  bases[FB_CVEC] = D_.cvec, bases[FB_A] = D_.a, bases[FB_LO] = D_.lo, bases[FB_HI] = D_.hi, bases[FB_RB] = D_.rb;
  bases[FB_AN] = D_.aN, bases[FB_LON] = D_.loN, bases[FB_HIN] = D_.hiN;
  bases[FB_BM] = dBm, bases[FB_FM] = dFm, bases[FB_FC] = dfc;
  for (int k = 0; k < FB_COUNT; ++k) F.base[k] = bases[k];
}

// Streaming dataflow T for wide trees (wide.cu): warp-granular items with
// per-warp TMA rings.  Default for trees the CTA-granular kernel does not take
// (>= 4096 nodes); SPOCK_T_WIDE=0 selects the per-stage kernels instead,
// SPOCK_T_WIDE=1 forces it on any tree the fused kernel is not used for.
// Pooled blocks: nodes whose per-node matrices are bitwise identical share one
// copy in the streaming kernel's records.  The generators share A, B, Q, R per
// event (generators.cpp:89-95); on an iid tree every node of the same stage and
// event then has the same subtree, hence the same Alg. 1 factors.  Exact
// classes, bottom-up: a node's class is (its A, B, Q, R [, QN], its children's
// classes in order); its blocks (H, H', M1, M1', K, K', R~^-1) depend only on
// its class and its parent's class, so nodes agreeing on both stream the same
// matrices (from L2 after the first).  Per-node perturbed problems have no
// duplicates (every node is its own class) and are unchanged.
void Engine::compute_pool() {
  const Tree& tr = p_.tree;
  const int nn = tr.nn(), nnl = tr.nnl(), N = tr.horizon;
  const size_t nx = p_.nx, nu = p_.nu;
  pool_rep_.resize(size_t(nn));
  for (int i = 0; i < nn; ++i) pool_rep_[i] = i;
  const char* env = std::getenv("SPOCK_POOL");
  if (env && env[0] == '0') return;
  struct Blk {
    const double* p;
    size_t n;
  };
  auto blocks = [&](int i, Blk (&b)[5]) {
    int k = 0;
    if (i > 0) {
      const size_t r = size_t(i - 1);
      b[k++] = {&p_.A[r * nx * nx], nx * nx};
      b[k++] = {&p_.B[r * nx * nu], nx * nu};
      b[k++] = {&p_.Q[r * nx * nx], nx * nx};
      b[k++] = {&p_.R[r * nu * nu], nu * nu};
    }
    if (i >= nnl) b[k++] = {&p_.QN[size_t(i - nnl) * nx * nx], nx * nx};
    return k;
  };
  std::vector<uint64_t> dh(size_t(nn), 0);
  parallel_for(nn, [&](int64_t ii) {
    Blk b[5];
    const int nb = blocks(int(ii), b);
    uint64_t h = 0x9E3779B97F4A7C15ull ^ uint64_t(nb);
    for (int q = 0; q < nb; ++q) {
      const uint64_t* w = reinterpret_cast<const uint64_t*>(b[q].p);
      for (size_t t = 0; t < b[q].n; ++t) {
        h = (h ^ w[t]) * 0xFF51AFD7ED558CCDull;
        h ^= h >> 31;
      }
    }
    dh[size_t(ii)] = h;
  });
  auto same_data = [&](int a, int b) {
    Blk x[5], y[5];
    const int na = blocks(a, x), nb = blocks(b, y);
    if (na != nb) return false;
    for (int q = 0; q < na; ++q)
      if (std::memcmp(x[q].p, y[q].p, sizeof(double) * x[q].n) != 0) return false;
    return true;
  };
  // exact classes bottom-up (stage by stage, leaves first)
  std::vector<int> cls(size_t(nn), -1);
  std::vector<int> rep_of_cls;
  std::unordered_map<uint64_t, std::vector<int>> cand;  // signature hash -> class ids
  for (int t = N; t >= 0; --t) {
    for (int i = tr.stage_start[t]; i < tr.stage_start[t + 1]; ++i) {
      const int c0 = tr.child_first[i], nc = tr.child_count[i];
      uint64_t h = dh[size_t(i)] ^ (uint64_t(nc) << 48);
      for (int c = 0; c < nc; ++c) h = (h ^ uint64_t(cls[size_t(c0 + c)] + 1)) * 0x9E3779B97F4A7C15ull;
      int found = -1;
      for (int k : cand[h]) {
        const int r = rep_of_cls[size_t(k)];
        if (tr.child_count[r] != nc || !same_data(i, r)) continue;
        bool ok = true;
        for (int c = 0; c < nc && ok; ++c) ok = cls[size_t(c0 + c)] == cls[size_t(tr.child_first[r] + c)];
        if (ok) {
          found = k;
          break;
        }
      }
      if (found < 0) {
        found = int(rep_of_cls.size());
        rep_of_cls.push_back(i);
        cand[h].push_back(found);
      }
      cls[size_t(i)] = found;
    }
  }
  // blocks of node i depend on (class of i, class of its parent)
  std::map<std::pair<int, int>, int> first;
  int shared = 0;
  for (int i = 0; i < nn; ++i) {
    const std::pair<int, int> key{cls[size_t(i)], i > 0 ? cls[size_t(tr.anc[i])] : -1};
    auto it = first.find(key);
    if (it == first.end()) {
      first.emplace(key, i);
    } else {
      pool_rep_[size_t(i)] = it->second;
      ++shared;
    }
  }
  pool_unique_ = nn - shared;
  if (std::getenv("SPOCK_DEBUG_SETUP"))
    std::fprintf(stderr, "[pool] %d nodes, %d classes, %d distinct block sets\n", nn, int(rep_of_cls.size()),
                 pool_unique_);
}

void Engine::setup_wide(bool force) {
  wide_ok_ = false;
  t_wide_ = false;
  const Tree& tr = p_.tree;
  const int nn = tr.nn(), nnl = tr.nnl(), nx = p_.nx, nu = p_.nu, m = nx + nu;
  auto knob = [](const char* name, int dflt) {
    const char* v = std::getenv(name);
    return (v && v[0]) ? std::atoi(v) : dflt;
  };
  // T runs on this kernel when the CTA-granular one is not used and the tree is
  // wide (or on request); so do the standalone L / L* on wide trees (measured:
  // on narrow trees one item per warp is latency-bound, narrow.cu's CTA-per-node
  // kernels win -- profiles/r01_wide_configs.md; SPOCK_LOP_WIDE=0/1 overrides)
  const int want = knob("SPOCK_T_WIDE", -1);
  const bool t_wide = !fused_ok_ && want != 0 && (want > 0 || nn >= 4096);
  lop_wide_ = knob("SPOCK_LOP_WIDE", nn >= 4096 ? 1 : 0) != 0;
  lop_narrow_ = knob("SPOCK_LOP_NARROW", 1) != 0;  // 0: narrow.cu's kernels instead of lop.cu
  (void)force;  // the records also feed lop.cu's narrow L / L*, so they are always built
  int max_nc = 0, max_ny = 0;
  for (int i = 0; i < nnl; ++i) max_nc = std::max(max_nc, p_.nc[i]);
  for (int j = 0; j < tr.nl(); ++j) max_nc = std::max(max_nc, p_.ncN[j]);
  for (int i = 0; i < nnl; ++i) max_ny = std::max(max_ny, lay_.y_dim[i]);
  if (max_nc > kMaxD) return;
  WideArgs& A = wargs_;
  A = WideArgs{};
  A.warps = std::max(1, std::min(8, knob("SPOCK_WIDE_WARPS", 8)));
  // deep narrow trees: fewer items per level than resident warps
  const bool latency_mode = double(nn) / double(tr.horizon + 1) < 148.0 * 2 * 6;
  {
    // Deep, narrow trees (a 100-stage horizon: ~1 000 items per level for ~1 800
    // resident warps) are bound by the latency of one item per level, not by
    // bandwidth: a 4-slot ring per warp (fewer warps) shortens each item
    // (measured (100, 10, 3): 6.14 -> 5.31 ms per T; wide levels prefer 2 slots)
    const int lat_slots = latency_mode ? 4 : 2;
    const int sl = std::max(1, std::min(16, knob("SPOCK_WIDE_SLOTS", lat_slots)));
    A.slots = sl >= 16 ? 16 : (sl >= 8 ? 8 : (sl >= 4 ? 4 : (sl >= 2 ? 2 : 1)));  // power of two
  }
  A.chunk = std::max(256, knob("SPOCK_WIDE_CHUNK", 512)) & ~1;
  // staging capacities sized for the common items: rare wide parents (a 100-way
  // fan-out has 201-row risk blocks) read their large spans in place, so they
  // do not inflate every warp's shared memory (fewer resident warps)
  A.ycap = std::min(max_ny, 64);
  A.l2_prefetch = knob("SPOCK_WIDE_L2PF", 0);  // measured slower (c3 1.80 vs 1.40 ms)
  A.vecd = int((std::max({m, max_nc, max_dense_s2_, 2 * nu + 2 + A.ycap}) + 2 + 7) & ~7);
  // one CTA of 8 warps per SM on deep narrow trees: ~1 200 warps for ~1 000
  // items per level, each warp's ring less contended (measured (100, 10, 3):
  // 4.89 -> 4.67 ms per T; 6 or 7 warps per CTA, 8 slots or 2 slots lose)
  wide_ctas_ = knob("SPOCK_WIDE_CTAS", latency_mode ? 1 : 2) >= 2 ? 2 : 1;
  wide_rows_ = wide_rows(D_, max_nc);
  // ---- per-ticket records: [backward nn-1..0][S2 0..nnl-1][forward 0..nn-1]
  std::vector<int64_t> hxo(std::max(nn - 1, 1)), huo(std::max(nn - 1, 1)), ao(std::max(nn - 1, 1));
  std::vector<int64_t> hno(std::max(tr.nl(), 1)), aNo(std::max(tr.nl(), 1));
  {
    int64_t sx = 0, su = 0, sa = 0;
    for (int k = 0; k < nn - 1; ++k) {
      hxo[k] = sx, huo[k] = su, ao[k] = sa;
      sx += pad2(int64_t(soc_.stage[k].px) * nx);
      su += pad2(int64_t(soc_.stage[k].pu) * nu);
      sa += soc_.stage[k].px + soc_.stage[k].pu + 2;
    }
    int64_t sh = 0, sb = 0;
    for (int j = 0; j < tr.nl(); ++j) {
      hno[j] = sh, aNo[j] = sb;
      sh += pad2(int64_t(soc_.leaf[j].px) * nx);
      sb += soc_.leaf[j].px + 2;
    }
  }
  const int total = nn + nnl + nn;
  std::vector<WRec> recs(static_cast<size_t>(total));
  auto meta = [&](WRec& R, int kind, int i) {
    std::memset(&R, 0, sizeof(R));
    R.kind = kind;
    R.node = i;
    R.nch = tr.child_count[i];
    R.c0 = tr.child_first[i];
    R.anc = tr.anc[i];
    if (i > 0) {
      R.px = soc_.stage[i - 1].px;
      R.pu = soc_.stage[i - 1].pu;
      R.s2o = lay_.seg2_off[i - 1];
    }
    if (i < nnl) {
      R.nc = p_.nc[i], R.ny = lay_.y_dim[i], R.so = lay_.seg1_off[i], R.yo = lay_.y_off[i];
    } else {
      const int j = i - nnl;
      R.nc = p_.ncN[j], R.pN = soc_.leaf[j].px, R.so = lay_.seg3_off[j];
    }
  };
  auto mat = [&](WRec& R, const double* p, int rows, int cols) {
    R.mp[R.nmat] = p;
    R.mrows[R.nmat] = int16_t(rows);
    R.mcols[R.nmat] = int16_t(cols);
    ++R.nmat;
  };
  // Only the iterate spans (z, eta) are staged: the per-node constants (boxes,
  // diagonal G, q_kernel, translations, c, g, h, risk b) are read in place, which
  // shrinks every warp's staging buffer (c4: 814 -> 358 doubles) and fits 8 warps
  // per CTA instead of 6 (c4 T 3.31 -> 3.06 ms, c5s 13.4 -> 11.8 ms).  Deep narrow
  // trees keep them staged: there every item is on the latency-bound critical
  // path ((100, 10, 3): 5.31 ms staged, 6.34 ms in place)
  int max_fan = 0;
  for (int i = 0; i < nnl; ++i) max_fan = std::max(max_fan, tr.child_count[i]);
  // latency-sensitive shapes keep the constants staged: deep or narrow trees (many
  // dependent levels) and wide fan-outs (slow parents on the critical path).
  // Measured: staged wins on (48, 3, 7) 3.27 vs 3.60 ms, (12, 100, 2) 4.12 vs 4.41,
  // (100, 10, 3) 4.94 vs 6.32; in place wins on c3, c4, (12, 4, 7) and c5s.
  const bool lat_sensitive = latency_mode || tr.horizon >= 40 || max_fan >= 50;
  const bool stage_const = knob("SPOCK_WIDE_STAGE_CONST", lat_sensitive ? 1 : 0) != 0;
  auto span = [&](WRec& R, int id, int base, int64_t off, int64_t cnt) {
    R.vbase[id] = uint8_t(base);
    R.voff[id] = int32_t(off);
    if (cnt > 160 || off > INT32_MAX || (!stage_const && base != WB_Z && base != WB_ETA)) {  // read in place
      R.unstaged |= 1 << id;
      R.vcnt[id] = 0;
    } else {
      R.vcnt[id] = uint16_t(cnt);
    }
    R.nspan = std::max(R.nspan, id + 1);
  };
  require(lay_.neta < INT32_MAX && lay_.nz < INT32_MAX, "spock-b200: wide T needs vectors below 2^31 entries");
  enum { B_HEAD = 0, B_QK, B_ZX, B_ZU, B_EC, B_GD, B_H, B_G };
  enum { B_SEG3 = B_ZU, B_GDN = B_GD, B_QKN = B_H };
  enum { F_ZX = 0, F_ZU, F_AX, F_AU, F_CV, F_SEG2, F_A, F_QK, F_SEG1, F_RB, F_GD, F_LO, F_HI, F_ZY, F_ZT, F_ZS };
  enum { F_SEG3 = F_SEG1, F_AN = F_RB, F_QKN = F_GD, F_GDN = F_LO, F_LON = F_HI, F_HIN = F_ZY };
  const std::vector<int>& pr = pool_rep_;  // matrix blocks: the node's pooled representative
  for (int k = 0; k < nn; ++k) {  // backward items
    const int i = nn - 1 - k;
    WRec& R = recs[size_t(k)];
    meta(R, 0, i);
    const bool leaf = tr.leaf(i), root = i == 0;
    if (!root) {
      mat(R, D_.HxT + hxo[pr[i] - 1], nx, R.px);
      mat(R, D_.HuT + huo[pr[i] - 1], nu, R.pu);
      span(R, B_HEAD, WB_ETA, R.s2o, R.px + R.pu + 2);
      span(R, B_QK, WB_QK, int64_t(i - 1) * m, m);
    }
    span(R, B_ZX, WB_Z, 1 + int64_t(i) * nx, nx);
    if (leaf) {
      const int j = i - nnl;
      mat(R, D_.HNT + hno[pr[i] - nnl], nx, R.pN);
      span(R, B_SEG3, WB_ETA, R.so, R.nc + R.pN + 2);
      if (D_.gN_diag) span(R, B_GDN, WB_GDN, int64_t(j) * nx, nx);
      span(R, B_QKN, WB_QKN, int64_t(j) * nx, nx);
    } else {
      mat(R, D_.KT + size_t(pr[i]) * D_.k_stride, nx, nu);
      mat(R, D_.Rinv + size_t(pr[i]) * D_.r_stride, nu, nu);
      span(R, B_ZU, WB_Z, lay_.u_base + int64_t(i) * nu, nu);
      span(R, B_EC, WB_ETA, R.so + R.ny, 1 + R.nc);
      if (D_.g_diag) span(R, B_GD, WB_GD, int64_t(i) * m, m);
      span(R, B_H, WB_H, int64_t(i) * nx, nx);
      span(R, B_G, WB_G, int64_t(i) * nu, nu);
    }
    if (!root) mat(R, D_.M1T + size_t(pr[i] - 1) * D_.m1_stride, m, nx);
  }
  for (int i = 0; i < nnl; ++i) meta(recs[size_t(nn) + i], 1, i);
  for (int c = 0; c < nn; ++c) {  // forward items
    WRec& R = recs[size_t(nn) + nnl + c];
    meta(R, 2, c);
    const bool leaf = tr.leaf(c), root = c == 0;
    const int an = R.anc;
    span(R, F_ZX, WB_Z, 1 + int64_t(c) * nx, nx);
    if (!leaf) span(R, F_ZU, WB_Z, lay_.u_base + int64_t(c) * nu, nu);
    if (!root) {
      mat(R, D_.M1 + size_t(pr[c] - 1) * D_.m1_stride, nx, m);
      span(R, F_AX, WB_Z, 1 + int64_t(an) * nx, nx);
      span(R, F_AU, WB_Z, lay_.u_base + int64_t(an) * nu, nu);
      span(R, F_CV, WB_CV, int64_t(c - 1) * nx, nx);
      span(R, F_SEG2, WB_ETA, R.s2o, R.px + R.pu + 2);
      span(R, F_A, WB_A, ao[c - 1], R.px + R.pu + 2);
      span(R, F_QK, WB_QK, int64_t(c - 1) * m, m);
      span(R, F_ZT, WB_Z, lay_.tau_base + c - 1, 1);
    }
    if (!leaf) mat(R, D_.K + size_t(pr[c]) * D_.k_stride, nu, nx);
    if (!root) {
      mat(R, D_.Hx + hxo[pr[c] - 1], R.px, nx);
      mat(R, D_.Hu + huo[pr[c] - 1], R.pu, nu);
    }
    span(R, F_ZS, WB_Z, root ? 0 : lay_.s_base + c - 1, 1);
    if (!leaf) {
      const int64_t go = p_.g_off[c];
      span(R, F_SEG1, WB_ETA, R.so, R.ny + 1 + R.nc);
      span(R, F_RB, WB_RB, R.yo - D_.y_base, R.ny);
      if (D_.g_diag) span(R, F_GD, WB_GD, int64_t(c) * m, m);
      span(R, F_LO, WB_LO, go, R.nc);
      span(R, F_HI, WB_HI, go, R.nc);
      span(R, F_ZY, WB_Z, R.yo, R.ny);
    } else {
      const int j = c - nnl;
      const int64_t go = p_.gN_off[j];
      mat(R, D_.HN + hno[pr[c] - nnl], R.pN, nx);
      span(R, F_SEG3, WB_ETA, R.so, R.nc + R.pN + 2);
      span(R, F_AN, WB_AN, aNo[j], R.pN + 2);
      span(R, F_QKN, WB_QKN, int64_t(j) * nx, nx);
      if (D_.gN_diag) span(R, F_GDN, WB_GDN, int64_t(j) * nx, nx);
      span(R, F_LON, WB_LON, go, R.nc);
      span(R, F_HIN, WB_HIN, go, R.nc);
    }
  }
  // standalone L (kind 3) and L* (kind 4: child terms of nodes 1..nn-1, then
  // kind 5: node rows of 0..nn-1) for the SuperMann loop outside T
  enum { L_ZX = 0, L_ZU, L_AX, L_AU, L_QK, L_ZT, L_ZS, L_Y, L_RB, L_GD, L_QKN };
  enum { LC_HEAD = 0, LC_QK };
  enum { LN_SEG1 = 0, LN_RB, LN_GD, LN_QKN };
  std::vector<WRec> lrecs(static_cast<size_t>(nn)), ltrecs;
  for (int i = 0; i < nn; ++i) {
    WRec& R = lrecs[size_t(i)];
    meta(R, 3, i);
    const bool leaf = tr.leaf(i), root = i == 0;
    span(R, L_ZX, WB_Z, 1 + int64_t(i) * nx, nx);
    if (!leaf) {
      span(R, L_ZU, WB_Z, lay_.u_base + int64_t(i) * nu, nu);
      span(R, L_Y, WB_Z, R.yo, R.ny);
      span(R, L_RB, WB_RB, R.yo - D_.y_base, R.ny);
      if (D_.g_diag) span(R, L_GD, WB_GD, int64_t(i) * m, m);
      span(R, L_ZS, WB_Z, root ? 0 : lay_.s_base + i - 1, 1);
    }
    if (!root) {
      const int an = R.anc;
      mat(R, D_.Hx + hxo[pr[i] - 1], R.px, nx);
      mat(R, D_.Hu + huo[pr[i] - 1], R.pu, nu);
      span(R, L_AX, WB_Z, 1 + int64_t(an) * nx, nx);
      span(R, L_AU, WB_Z, lay_.u_base + int64_t(an) * nu, nu);
      span(R, L_QK, WB_QK, int64_t(i - 1) * m, m);
      span(R, L_ZT, WB_Z, lay_.tau_base + i - 1, 1);
    }
    if (leaf) {
      const int j = i - nnl;
      mat(R, D_.HN + hno[pr[i] - nnl], R.pN, nx);
      if (D_.gN_diag) span(R, L_GD, WB_GDN, int64_t(j) * nx, nx);
      span(R, L_QKN, WB_QKN, int64_t(j) * nx, nx);
      span(R, L_ZS, WB_Z, lay_.s_base + i - 1, 1);
    }
  }
  for (int i = 1; i < nn; ++i) {
    WRec R;
    meta(R, 4, i);
    mat(R, D_.HxT + hxo[pr[i] - 1], nx, R.px);
    mat(R, D_.HuT + huo[pr[i] - 1], nu, R.pu);
    span(R, LC_HEAD, WB_ETA, R.s2o, R.px + R.pu + 2);
    span(R, LC_QK, WB_QK, int64_t(i - 1) * m, m);
    ltrecs.push_back(R);
  }
  for (int i = 0; i < nn; ++i) {
    WRec R;
    meta(R, 5, i);
    if (!tr.leaf(i)) {
      span(R, LN_SEG1, WB_ETA, R.so, R.ny + 1 + R.nc);
      span(R, LN_RB, WB_RB, R.yo - D_.y_base, R.ny);
      if (D_.g_diag) span(R, LN_GD, WB_GD, int64_t(i) * m, m);
    } else {
      const int j = i - nnl;
      mat(R, D_.HNT + hno[pr[i] - nnl], nx, R.pN);
      span(R, LN_SEG1, WB_ETA, R.so, R.nc + R.pN + 2);
      if (D_.gN_diag) span(R, LN_GD, WB_GDN, int64_t(j) * nx, nx);
      span(R, LN_QKN, WB_QKN, int64_t(j) * nx, nx);
    }
    ltrecs.push_back(R);
  }
  int64_t vmax = 2;
  for (const std::vector<WRec>* L : {&recs, &lrecs, &ltrecs})
    for (const WRec& R : *L) {
      int64_t t = 0;
      for (int k = 0; k < R.nspan; ++k)
        if (R.vcnt[k]) t += pad2(R.vcnt[k] + 1);  // + alignment shift (taken from the address)
      vmax = std::max(vmax, t);
    }
  A.vrec = int(pad2(vmax));
  int dev = 0, sms = 148, smem_optin = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const int budget = smem_optin / wide_ctas_ - 2048;
  while (wide_smem_bytes(A) > budget && A.chunk > 512) A.chunk = (A.chunk / 2) & ~1;
  while (wide_smem_bytes(A) > budget && A.warps > 1) --A.warps;
  const int bytes = wide_smem_bytes(A);
  if (bytes > smem_optin) return;
  for (std::vector<WRec>* L : {&recs, &lrecs, &ltrecs})
    for (WRec& R : *L)  // columns per ring chunk (even; a chunk holds >= 2 columns)
      for (int k = 0; k < R.nmat; ++k)
        R.mcc[k] = int16_t(R.mrows[k] > 0 ? std::max(2, (A.chunk / R.mrows[k]) & ~1) : 2);
  CK(wide_configure(wide_rows_, wide_ctas_, bytes));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, wide_kernel_ptr(wide_rows_, wide_ctas_), 32 * A.warps,
                                                   bytes));
  if (occ < 1) return;
  // every CTA must be resident (items spin on flags of smaller tickets)
  wide_grid_ = occ * sms;
  if (std::getenv("SPOCK_DEBUG_SETUP"))
    std::fprintf(stderr, "[wide] rows %d ctas %d warps %d slots %d chunk %d vrec %d vecd %d smem %d B occ %d grid %d\n",
                 wide_rows_, wide_ctas_, A.warps, A.slots, A.chunk, A.vrec, A.vecd, bytes, occ, wide_grid_);
  // latency configuration for launches with about one item per warp (standalone
  // L / L* on narrow trees): one CTA per SM, few warps, 16-slot rings so a
  // warp's whole item is requested at once instead of one chunk per round trip
  wlat_ = A;
  wlat_.slots = 16;
  wlat_.warps = 4;
  while (wlat_.warps > 1 && wide_smem_bytes(wlat_) > smem_optin - 2048) --wlat_.warps;
  while (wide_smem_bytes(wlat_) > smem_optin - 2048 && wlat_.slots > 2) wlat_.slots /= 2;
  {
    const int lb = wide_smem_bytes(wlat_);
    CK(wide_configure(wide_rows_, 1, wide_ctas_ == 1 ? std::max(lb, bytes) : lb));
    int occl = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occl, wide_kernel_ptr(wide_rows_, 1), 32 * wlat_.warps, lb));
    wide_grid_lat_ = std::max(1, occl) * sms;
  }
  WRec* drec = nullptr;
  CK(cudaMalloc(&drec, sizeof(WRec) * recs.size()));
  allocs_.push_back(drec);
  CK(cudaMemcpyAsync(drec, recs.data(), sizeof(WRec) * recs.size(), cudaMemcpyHostToDevice, st_));
  CK(cudaStreamSynchronize(st_));
  A.recs = drec;
  A.ntick = total;
  wrecs_ = std::move(recs);
  lrec_ = dalloc<WRec>(lrecs.size());
  ltrec_ = dalloc<WRec>(ltrecs.size());
  CK(cudaMemcpyAsync(lrec_, lrecs.data(), sizeof(WRec) * lrecs.size(), cudaMemcpyHostToDevice, st_));
  CK(cudaMemcpyAsync(ltrec_, ltrecs.data(), sizeof(WRec) * ltrecs.size(), cudaMemcpyHostToDevice, st_));
  nlrec_ = int(lrecs.size());
  nltrec_ = int(ltrecs.size());
  lrecs_h_ = lrecs;
  ltrecs_h_ = ltrecs;
  CK(cudaStreamSynchronize(st_));
  // lop.cu (narrow trees): staging capacities from the records
  {
    auto staged = [](const WRec& R) {
      int64_t t = 0;
      for (int k = 0; k < R.nspan; ++k)
        if (!((R.unstaged >> k) & 1)) t += pad2(R.vcnt[k]);
      return t;
    };
    auto mats = [](const WRec& R) {
      int64_t t = 0;
      for (int k = 0; k < R.nmat; ++k) t += pad2(int64_t(R.mrows[k]) * R.mcols[k]);
      return t;
    };
    int64_t vL = 0, v4 = 0, v5 = 0, mL = 0, m4 = 0, m5 = 0;
    for (const WRec& R : lrecs) vL = std::max(vL, staged(R)), mL = std::max(mL, mats(R));
    for (const WRec& R : ltrecs) {
      if (R.kind == 4) v4 = std::max(v4, staged(R)), m4 = std::max(m4, mats(R));
      else v5 = std::max(v5, staged(R)), m5 = std::max(m5, mats(R));
    }
    lop_rows_ = std::max(m, max_nc);
    lop_vec_ = int(pad2(std::max(vL, v4 + v5) + 2));
    lop_mat_ = int(pad2(std::max(mL, 2 * std::max(m4, m5))));
    // matrices that do not fit are read from global memory inside the GEMVs
    while (lop_smem_bytes(lop_rows_, lop_mat_, lop_vec_) > smem_optin - 2048 && lop_mat_ > 0)
      lop_mat_ = int(pad2(lop_mat_ / 2));
    CK(lop_configure(lop_smem_bytes(lop_rows_, lop_mat_, lop_vec_)));
  }
  A.vb[WB_QK] = D_.qk, A.vb[WB_GD] = D_.gd, A.vb[WB_H] = D_.h, A.vb[WB_G] = D_.g, A.vb[WB_QKN] = D_.qkN;
  A.vb[WB_GDN] = D_.gNd, A.vb[WB_CV] = D_.cvec, A.vb[WB_A] = D_.a, A.vb[WB_LO] = D_.lo, A.vb[WB_HI] = D_.hi;
  A.vb[WB_RB] = D_.rb, A.vb[WB_AN] = D_.aN, A.vb[WB_LON] = D_.loN, A.vb[WB_HIN] = D_.hiN;
  wide_flag_bytes_ = sizeof(int) * size_t(total);
  wide_flags_ = dalloc<int>(size_t(total));
  A.flagB = wide_flags_;
  A.flagS2 = wide_flags_ + nn;
  A.flagF = wide_flags_ + nn + nnl;
  if (knob("SPOCK_WIDE_PROF", 0)) A.prof = dalloc<unsigned long long>(16);
  wide_ok_ = true;
  t_wide_ = t_wide;
  // Split T for trees with a narrow top: stages whose nodes are fewer than the
  // latency configuration's warps run in their own launch with 16-slot rings
  // (a whole item prefetched at once); the wide stages stay on the throughput
  // configuration.  L1: backward of the wide stages + every S2; L2: the top's
  // backward then forward; L3: forward of the wide stages.
  const int split_min = knob("SPOCK_T_SPLIT_NODES", wide_grid_lat_ * wlat_.warps);
  t_split_ = 0;
  if (t_wide_ && split_min > 0 && knob("SPOCK_T_SPLIT", 0)) {  // measured slower: c3 1.50 vs 1.40 ms
    int s = 0;
    while (s <= tr.horizon && tr.stage_start[s + 1] - tr.stage_start[s] < split_min) ++s;
    if (s >= 2 && s <= tr.horizon) {
      const int top = tr.stage_start[s];
      std::vector<WRec> l1, l2, l3;
      for (int k = 0; k < nn; ++k) {  // backward, node nn-1 .. 0
        const int i = nn - 1 - k;
        (i >= top ? l1 : l2).push_back(wrecs_[size_t(k)]);
      }
      for (int i = 0; i < nnl; ++i) l1.push_back(wrecs_[size_t(nn) + i]);
      for (int c = 0; c < nn; ++c) (c >= top ? l3 : l2).push_back(wrecs_[size_t(nn) + nnl + c]);
      auto up = [&](const std::vector<WRec>& v, WRec*& d, int& n) {
        d = dalloc<WRec>(v.size());
        CK(cudaMemcpyAsync(d, v.data(), sizeof(WRec) * v.size(), cudaMemcpyHostToDevice, st_));
        n = int(v.size());
      };
      up(l1, tsplit_rec_[0], tsplit_n_[0]);
      up(l2, tsplit_rec_[1], tsplit_n_[1]);
      up(l3, tsplit_rec_[2], tsplit_n_[2]);
      CK(cudaStreamSynchronize(st_));
      t_split_ = s;
    }
  }
}

// ---------------------------------------------------------------------------
// Subtree sharding of T.  The host (paper_2505_12078_b200/shard.py)
// chooses a split stage ts and gives this rank the stage-ts nodes [b0, b1) with
// their subtrees; stages < ts are computed redundantly on every rank.  One T:
//   phase A  backward items of the rank's subtrees (stages >= ts), then the
//            boundary records of its stage-ts nodes are packed into its slice
//            of the exchange buffer;
//   (host)   all-gather of the exchange buffer across ranks (NCCL / gloo);
//   phase B  remote stage-ts records are unpacked (their adj and T12 terms,
//            the z / eta entries S2 of their parent reads) and their backward
//            flags set; then the top backward items, S2 of every parent the
//            rank holds, and the forward items of the top and of its subtrees.
// Each rank's iterates are valid on the top and on its own subtrees.
void Engine::shard_setup(int G, int rank, int ts, const int* back_a, int na, const int* back_b, int nb,
                         const int* s2, int ns2, const int* fwd, int nf, double* xbuf) {
  const Tree& tr = p_.tree;
  const int nn = tr.nn(), nnl = tr.nnl();
  require(G >= 1 && rank >= 0 && rank < G, "spock_shard_setup: bad rank / world size");
  require(ts >= 1 && ts <= tr.horizon, "spock_shard_setup: split stage must be in [1, N]");
  if (!wide_ok_) setup_wide(true);
  require(wide_ok_, "spock_shard_setup: the streaming T kernel is not available for this problem");
  shard_ = ShardState{};
  ShardState& S = shard_;
  S.G = G, S.rank = rank, S.ts = ts;
  S.bfirst = tr.stage_start[ts];
  S.nbound = tr.stage_start[ts + 1] - S.bfirst;
  S.q = (S.nbound + G - 1) / G;
  S.b0 = S.bfirst + std::min(rank * S.q, S.nbound);
  S.b1 = S.bfirst + std::min((rank + 1) * S.q, S.nbound);
  S.E = 2 * (p_.nx + p_.nu) + 6;
  S.xbuf = xbuf;
  auto pick = [&](const int* nodes, int n, int kind) {
    std::vector<WRec> out;
    out.reserve(size_t(n));
    for (int k = 0; k < n; ++k) {
      const int i = nodes[k];
      require(i >= 0 && i < (kind == 1 ? nnl : nn), "spock_shard_setup: node index out of range");
      const size_t t = kind == 0 ? size_t(nn - 1 - i) : (kind == 1 ? size_t(nn) + i : size_t(nn) + nnl + i);
      out.push_back(wrecs_[t]);
    }
    return out;
  };
  std::vector<WRec> ra = pick(back_a, na, 0), rb = pick(back_b, nb, 0);
  const std::vector<WRec> r2 = pick(s2, ns2, 1), rf = pick(fwd, nf, 2);
  rb.insert(rb.end(), r2.begin(), r2.end());
  rb.insert(rb.end(), rf.begin(), rf.end());
  S.nA = int(ra.size());
  S.nB = int(rb.size());
  S.recA = dalloc<WRec>(std::max<size_t>(ra.size(), 1));
  S.recB = dalloc<WRec>(std::max<size_t>(rb.size(), 1));
  if (!ra.empty()) CK(cudaMemcpyAsync(S.recA, ra.data(), sizeof(WRec) * ra.size(), cudaMemcpyHostToDevice, st_));
  if (!rb.empty()) CK(cudaMemcpyAsync(S.recB, rb.data(), sizeof(WRec) * rb.size(), cudaMemcpyHostToDevice, st_));
  // per stage-ts node: where S2 of its parent reads its tau / s inputs
  std::vector<int64_t> idx(size_t(S.nbound) * 6);
  for (int k = 0; k < S.nbound; ++k) {
    const int c = S.bfirst + k;
    const int p = soc_.stage[c - 1].px + soc_.stage[c - 1].pu;
    int64_t* x = &idx[size_t(k) * 6];
    x[0] = lay_.tau_base + c - 1;               // z tau_c
    x[1] = lay_.s_base + c - 1;                 // z s_c
    x[2] = lay_.seg2_off[c - 1] + p;            // eta tau rows of c's stage-SOC segment
    x[3] = x[2] + 1;
    if (c < nnl) {
      x[4] = lay_.seg1_off[c] + lay_.y_dim[c];  // eta risk scalar row of c
      x[5] = -1;
    } else {
      const int j = c - nnl;
      x[4] = lay_.seg3_off[j] + p_.ncN[j] + soc_.leaf[j].px;  // eta terminal SOC tau rows
      x[5] = x[4] + 1;
    }
  }
  S.xidx = dupload(idx);
  // nodes whose iterate entries this rank computes: the top and its subtrees
  S.owned.assign(size_t(nn), 0);
  std::vector<int> root_ts(size_t(nn), -1);
  for (int i = 0; i < nn; ++i) {
    if (i < S.bfirst) {
      S.owned[i] = 1;
      continue;
    }
    root_ts[i] = tr.stage[i] == ts ? i : root_ts[tr.anc[i]];
    S.owned[i] = (root_ts[i] >= S.b0 && root_ts[i] < S.b1) ? 1 : 0;
  }
  // sharded solve: L / L* item subsets, entry masks and exclusive weights
  {
    std::vector<WRec> lo, la, lb;
    for (int i = 0; i < nn; ++i)
      if (S.owned[i]) lo.push_back(lrecs_h_[size_t(i)]);
    for (int i = 1; i < nn; ++i)
      if (S.owned[i]) la.push_back(ltrecs_h_[size_t(i - 1)]);
    for (int i = 0; i < nn; ++i)
      if (S.owned[i]) lb.push_back(ltrecs_h_[size_t(nn - 1 + i)]);
    auto up = [&](const std::vector<WRec>& v, WRec*& d, int& n) {
      d = dalloc<WRec>(std::max<size_t>(v.size(), 1));
      if (!v.empty()) CK(cudaMemcpyAsync(d, v.data(), sizeof(WRec) * v.size(), cudaMemcpyHostToDevice, st_));
      n = int(v.size());
    };
    up(lo, S.recL, S.nL);
    up(la, S.recLtA, S.nLtA);
    up(lb, S.recLtB, S.nLtB);
    std::vector<uint8_t> zm(size_t(lay_.nz)), em(size_t(lay_.neta)), zx(zm.size()), ex(em.size());
    S.on = true;  // shard_masks needs it
    shard_masks(zm.data(), em.data());
    shard_weights(zx.data(), ex.data());
    std::vector<double> mz(zm.begin(), zm.end()), me(em.begin(), em.end()), wz(zx.begin(), zx.end()),
        we(ex.begin(), ex.end());
    std::vector<double> wv(wz);
    wv.insert(wv.end(), we.begin(), we.end());
    S.mz = dupload(mz), S.me = dupload(me), S.wz = dupload(wz), S.we = dupload(we), S.wv = dupload(wv);
  }
  CK(cudaStreamSynchronize(st_));
  S.on = true;
}

void Engine::shard_set_collectives(CollFn fn, void* user) {
  require(shard_.on, "spock_shard_set_collectives: call spock_shard_setup first");
  shard_.coll = fn;
  shard_.coll_user = user;
}

// Host-loop Gram of the Anderson difference history by position (newest 0),
// double-double: shift every entry one position, then row / column 0 from this
// iteration's update dots (launch_gram_dd, chunks of kLoopMaxMem columns:
// [<dnew, D_b> | <D_b, r>] as (hi, lo) pairs per chunk).  Sharded: the ranks'
// partial sums are all-gathered and added in rank order, so the double-double
// precision survives the cross-rank sum (an all-reduce of hi and lo would not).
void Engine::gram_update(int cols, bool sharded) {
  const int n = 4 * cols;
  const double* src = gram_out_;
  int G = 1;
  if (sharded && shard_coll_on() && shard_.G > 1) {
    G = shard_.G;
    if (!gram_gather_) gram_gather_ = dalloc<double>(size_t(G) * 4 * kAaHostMax);
    CK(cudaMemcpyAsync(gram_gather_ + size_t(shard_.rank) * n, gram_out_, sizeof(double) * n,
                       cudaMemcpyDeviceToDevice, st_));
    coll(3, gram_gather_, n);
    src = gram_gather_;
  }
  std::vector<double> h(size_t(G) * n);
  CK(cudaMemcpyAsync(h.data(), src, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, st_));
  sync();
  std::vector<dd> nd(cols, dd{0.0, 0.0}), rd(cols, dd{0.0, 0.0});
  for (int g = 0; g < G; ++g) {
    const double* q = h.data() + size_t(g) * n;
    for (int c0 = 0; c0 < cols; c0 += kLoopMaxMem) {
      const int cc = std::min(kLoopMaxMem, cols - c0);
      const double* z = q + 4 * c0;
      for (int b = 0; b < cc; ++b) {
        nd[c0 + b] = dd_add(nd[c0 + b], dd{z[2 * b], z[2 * b + 1]});
        rd[c0 + b] = dd_add(rd[c0 + b], dd{z[2 * (cc + b)], z[2 * (cc + b) + 1]});
      }
    }
  }
  constexpr int K = kAaHostMax;
  const int m = prm_.aa_memory;
  for (int a = m - 1; a >= 1; --a)
    for (int b = m - 1; b >= 1; --b) gram_h_[a + b * K] = gram_h_[(a - 1) + (b - 1) * K];
  for (int b = 0; b < cols; ++b) {
    gram_h_[b * K] = gram_h_[b] = nd[b];
    gram_r_[b] = rd[b];
  }
}

// Cancellation of a sharded solve is a collective decision: each rank polls its
// own callback and the ranks all-reduce the flags with MAX, so either every rank
// stops at this iteration or none does (a lone rank leaving would strand the
// others in their next collective).  Unsharded: the callback's own answer.
bool Engine::agree_cancel(bool mine) {
  if (!shard_solving_ || !shard_coll_on() || shard_.G == 1) return mine;
  if (!cancel_dev_) cancel_dev_ = dalloc<double>(1);
  host_red_[511] = mine ? 1.0 : 0.0;
  CK(cudaMemcpyAsync(cancel_dev_, host_red_ + 511, sizeof(double), cudaMemcpyHostToDevice, st_));
  coll(2, cancel_dev_, 1);
  CK(cudaMemcpyAsync(host_red_ + 511, cancel_dev_, sizeof(double), cudaMemcpyDeviceToHost, st_));
  sync();
  return host_red_[511] != 0.0;
}

void Engine::shard_nccl_init(const void* id, int nranks, int rank) {
  require(shard_.on, "spock_shard_nccl_init: call spock_shard_setup first");
  require(nranks == shard_.G && rank == shard_.rank, "spock_shard_nccl_init: world / rank differ from the shard plan");
  const NcclDl& N = nccl_dl();
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  ncclComm_t c = nullptr;
  nccl_check(N.CommInitRank(&c, nranks, u, rank), "ncclCommInitRank");
  shard_.nccl = c;
}

void Engine::coll(int op, double* buf, int64_t n) {
  if (n <= 0) return;
  if (shard_.nccl) {  // on the solver stream, ordered after the kernels that wrote buf
    const NcclDl& N = nccl_dl();
    ncclComm_t c = static_cast<ncclComm_t>(shard_.nccl);
    if (op == 0 || op == 3) {  // all-gather in place: rank r's slice at r * count
      const size_t cnt = op == 0 ? size_t(n / shard_.G) : size_t(n);
      nccl_check(N.AllGather(buf + size_t(shard_.rank) * cnt, buf, cnt, ncclDouble, c, st_), "ncclAllGather");
    } else {
      nccl_check(N.AllReduce(buf, buf, size_t(n), ncclDouble, op == 1 ? ncclSum : ncclMax, c, st_),
                 "ncclAllReduce");
    }
    return;
  }
  if (!shard_.coll || shard_.G == 1) return;
  if (shard_.coll(shard_.coll_user, op, buf, n) != 0) throw std::runtime_error("sharded solve: collective failed");
}

// one T of the sharded solve: phase A, all-gather, phase B
void Engine::shard_T(const double* z, const double* eta, double* zo, double* eo) {
  shard_T_A(z, eta, zo, eo);
  coll(0, shard_.xbuf, int64_t(shard_.G) * shard_.q * shard_.E);
  shard_T_B(z, eta, zo, eo);
}

// L* of the sharded solve: child terms of the rank's nodes, all-gather of the
// stage-ts adj terms, node rows of the rank's nodes
void Engine::shard_Lt(const double* eta, double* z) {
  const ShardState& S = shard_;
  WideArgs A = wargs_;
  A.D = D_, A.eta = eta, A.zo = z;
  CK(cudaMemsetAsync(wide_flags_, 0, sizeof(int) * size_t(p_.tree.nn()), st_));
  if (S.nLtA > 0) launch_wide(A, S.recLtA, S.nLtA);
  ShardXArgs X{D_, nullptr, eta, S.xidx, S.xbuf, S.bfirst, S.b0, S.b1, S.E, nullptr, 0, 0};
  launch_shard_pack(X, st_);
  coll(0, S.xbuf, int64_t(S.G) * S.q * S.E);
  X.flagB = wargs_.flagB;
  X.nbound = S.nbound;
  launch_shard_unpack(X, st_);
  if (S.nLtB > 0) launch_wide(A, S.recLtB, S.nLtB);
}

void Engine::shard_L(const double* z, double* eta) {
  WideArgs A = wargs_;
  A.D = D_, A.z = z, A.eo = eta;
  if (shard_.nL > 0) launch_wide(A, shard_.recL, shard_.nL);
}

// exclusive weights: like shard_masks, but an entry computed on every rank (its
// owner node is in the replicated top) belongs to rank 0 only, so the ranks'
// weighted vectors sum to the whole vector and weighted dots to the whole dot
void Engine::shard_weights(uint8_t* zm, uint8_t* em) {
  ShardState& S = shard_;
  require(S.on, "spock_shard_weights: call spock_shard_setup first");
  if (S.rank == 0) {
    shard_masks(zm, em);
    return;
  }
  const std::vector<uint8_t> saved = S.owned;
  for (int i = 0; i < S.bfirst; ++i) S.owned[i] = 0;
  shard_masks(zm, em);
  S.owned = saved;
}

// validity masks of this rank's iterates in the boundary layouts (1: computed here)
void Engine::shard_masks(uint8_t* zm, uint8_t* em) const {
  const ShardState& S = shard_;
  require(S.on, "spock_shard_masks: call spock_shard_setup first");
  const Tree& tr = p_.tree;
  const int nn = tr.nn(), nnl = tr.nnl(), nx = p_.nx, nu = p_.nu;
  if (zm) {
    std::memset(zm, 0, size_t(lay_.nz));
    zm[0] = S.owned[0];  // s0 belongs to the root (top)
    for (int i = 0; i < nn; ++i) {
      const uint8_t o = S.owned[i];
      std::memset(zm + 1 + size_t(i) * nx, o, size_t(nx));
      if (i < nnl) {
        std::memset(zm + lay_.u_base + size_t(i) * nu, o, size_t(nu));
        std::memset(zm + lay_.y_off[i], o, size_t(lay_.y_dim[i]));
      }
      if (i > 0) {
        // tau_i, s_i: T writes them in S2 of the parent (every rank holding the
        // parent), L* in node i's own items -- both on node i's owner
        zm[lay_.tau_base + i - 1] = o;
        zm[lay_.s_base + i - 1] = o;
      }
    }
  }
  if (em) {
    std::memset(em, 0, size_t(lay_.neta));
    for (int i = 0; i < nn; ++i) {
      const uint8_t o = S.owned[i];
      if (i < nnl) std::memset(em + lay_.seg1_off[i], o, size_t(lay_.y_dim[i] + 1 + p_.nc[i]));
      if (i > 0) {
        const int k = i - 1;
        std::memset(em + lay_.seg2_off[k], o, size_t(soc_.stage[k].px + soc_.stage[k].pu + 2));
      }
      if (i >= nnl) {
        const int j = i - nnl;
        std::memset(em + lay_.seg3_off[j], o, size_t(p_.ncN[j] + soc_.leaf[j].px + 2));
      }
    }
  }
}

// boundary-layout sharded T, in two calls around the host's all-gather
void Engine::shard_apply_T_b(int phase, const double* z, const double* eta, double* zo, double* eo) {
  double *iz = scratch_z_[0], *ie = scratch_e_[0], *oz = scratch_z_[1], *oe = scratch_e_[1];
  if (phase == 2) {  // the whole sharded T with the exchange in C++ (NCCL)
    require(shard_.nccl != nullptr, "spock_shard_apply_T phase 2 needs spock_shard_nccl_init");
    copy_in_z(z, iz);
    to_internal_eta(eta, ie);
    shard_T(iz, ie, oz, oe);
    copy_out(oz, zo, lay_.nz);
    from_internal_eta(oe, eo);
    sync();
    return;
  }
  if (phase == 0) {
    copy_in_z(z, iz);
    to_internal_eta(eta, ie);
    shard_T_A(iz, ie, oz, oe);
  } else {
    shard_T_B(iz, ie, oz, oe);
    copy_out(oz, zo, lay_.nz);
    from_internal_eta(oe, eo);
    sync();
  }
}

// device-resident ping-pong between the scratch iterates (bench helper)
void Engine::shard_bench(int phase, int parity) {
  double *z0 = scratch_z_[parity], *e0 = scratch_e_[parity], *z1 = scratch_z_[1 - parity],
         *e1 = scratch_e_[1 - parity];
  if (phase == 2) {
    require(shard_.nccl != nullptr, "spock_shard_bench phase 2 needs spock_shard_nccl_init");
    shard_T(z0, e0, z1, e1);
  } else if (phase == 0) {
    shard_T_A(z0, e0, z1, e1);
  } else {
    shard_T_B(z0, e0, z1, e1);
  }
}

void Engine::shard_T_A(const double* z, const double* eta, double* zo, double* eo) {
  const ShardState& S = shard_;
  require(S.on, "spock_shard_T: call spock_shard_setup first");
  WideArgs A = wargs_;
  A.D = D_, A.z = z, A.eta = eta, A.zo = zo, A.eo = eo, A.alpha = alpha_;
  A.recs = S.recA;
  A.ntick = S.nA;
  CK(cudaMemsetAsync(wide_flags_, 0, wide_flag_bytes_, st_));
  if (S.nA > 0) launch_wide(A, S.recA, S.nA);
  ShardXArgs X{D_, z, eta, S.xidx, S.xbuf, S.bfirst, S.b0, S.b1, S.E, nullptr, 0, 1};
  launch_shard_pack(X, st_);
}

void Engine::shard_T_B(const double* z, const double* eta, double* zo, double* eo) {
  const ShardState& S = shard_;
  require(S.on, "spock_shard_T: call spock_shard_setup first");
  // remote stage-ts records -> adj, T12, the inputs' tau / s entries, backward flags
  ShardXArgs X{D_, z, eta, S.xidx, S.xbuf, S.bfirst, S.b0, S.b1, S.E, wargs_.flagB, S.nbound, 1};
  launch_shard_unpack(X, st_);
  WideArgs A = wargs_;
  A.D = D_, A.z = z, A.eta = eta, A.zo = zo, A.eo = eo, A.alpha = alpha_;
  A.recs = S.recB;
  A.ntick = S.nB;
  if (S.nB > 0) launch_wide(A, S.recB, S.nB);
}

void Engine::wide_profile(unsigned long long* out) {
  for (int k = 0; k < 13; ++k) out[k] = 0;
  if (!wargs_.prof) return;
  CK(cudaStreamSynchronize(st_));
  CK(cudaMemcpy(out, wargs_.prof, sizeof(unsigned long long) * 13, cudaMemcpyDeviceToHost));
}

void Engine::set_grid_cap(int ctas) {
  if (ctas < 0) throw std::invalid_argument("set_grid_cap: negative CTA count");
  if (gloop_[0].exec || gloop_[1].exec || bench_graph_ || small_solved_)
    throw std::invalid_argument("set_grid_cap: must be called before the first solve or bench");
  if (!fused_ok_) return;  // the streaming schedules are HBM-bound: nothing to share
  fused_grid_ = ctas > 0 ? std::min(fused_grid_full_, ctas) : fused_grid_full_;
}

Engine::~Engine() {
  for (GraphLoop& G : gloop_)
    if (G.exec) cudaGraphExecDestroy(G.exec);
  if (shard_.nccl) {
    try {
      nccl_dl().CommDestroy(static_cast<ncclComm_t>(shard_.nccl));
    } catch (...) {
    }
  }
  if (wargs_.prof) {  // SPOCK_WIDE_PROF=1: per-warp cycle shares of the wide kernel
    unsigned long long p[13] = {};
    try {
      wide_profile(p);
    } catch (...) {
    }
    const double tot = double(p[0] ? p[0] : 1);
    std::fprintf(stderr,
                 "[wide prof] warps*launches=%llu total=%.3g cyc  ring-wait %.1f%%  flag-wait %.1f%%  back %.1f%% "
                 "(%llu, %.0f cyc/item)  s2 %.1f%% (%llu, %.0f)  fwd %.1f%% (%llu, %.0f)  span-wait %.1f%%  "
                 "refill %.1f%%  record-wait %.1f%%\n",
                 p[9], tot, 100.0 * p[1] / tot, 100.0 * p[2] / tot, 100.0 * p[3] / tot, p[6],
                 p[6] ? double(p[3]) / p[6] : 0.0, 100.0 * p[4] / tot, p[7], p[7] ? double(p[4]) / p[7] : 0.0,
                 100.0 * p[5] / tot, p[8], p[8] ? double(p[5]) / p[8] : 0.0, 100.0 * p[10] / tot,
                 100.0 * p[11] / tot, 100.0 * p[12] / tot);
  }
  if (bench_graph_) cudaGraphExecDestroy(bench_graph_);
  if (st_) cudaStreamSynchronize(st_);
  for (void* p : allocs_) cudaFree(p);
  if (host_red_) cudaFreeHost(host_red_);
  if (st_) cudaStreamDestroy(st_);
}

// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// Device-side SOC epigraph data (soc_data_quadlin, proj/src/problem.cpp:113-161,
// per block of blkdiag(Q, R) as the host restatement soc_block in model.cpp).
// Pass 1 (before the layouts): eigendecompositions of every Q_k, R_k, QN_j
// (one CTA each) and, per node, the ranks, lambda_max and the merged row order
// the boundary permutation needs.  Pass 2 (upload): S'MS, its square root by a
// second eigendecomposition, the head maps H and H', q_kernel and the
// translation a, written into the per-node layout.
namespace {
template <class Ty>
Ty* tmp_alloc(std::vector<void*>& owned, size_t n) {
  void* p = nullptr;
  CK(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(Ty)));
  owned.push_back(p);
  return static_cast<Ty*>(p);
}
template <class Ty>
Ty* tmp_upload(std::vector<void*>& owned, const Ty* h, size_t n, cudaStream_t st) {
  Ty* d = tmp_alloc<Ty>(owned, n);
  if (n) CK(cudaMemcpyAsync(d, h, n * sizeof(Ty), cudaMemcpyHostToDevice, st));
  return d;
}
}  // namespace

void Engine::soc_device_ranks() {
  const Tree& tr = p_.tree;
  const int nn = tr.nn(), nr = nn - 1, nl = tr.nl(), nx = p_.nx, nu = p_.nu;
  SocScratch& S = socs_;
  auto& own = S.owned;
  S.Q = tmp_upload(own, p_.Q.data(), p_.Q.size(), st_);
  S.R = tmp_upload(own, p_.R.data(), p_.R.size(), st_);
  S.q = tmp_upload(own, p_.q.data(), p_.q.size(), st_);
  S.r = tmp_upload(own, p_.r.data(), p_.r.size(), st_);
  S.QN = tmp_upload(own, p_.QN.data(), p_.QN.size(), st_);
  S.qN = tmp_upload(own, p_.qN.data(), p_.qN.size(), st_);
  const int nbx = nr + nl;  // x blocks: stage Q_k, then terminal QN_j
  S.Wx = tmp_alloc<double>(own, size_t(nbx) * nx);
  S.Vx = tmp_alloc<double>(own, size_t(nbx) * nx * nx);
  S.Wu = tmp_alloc<double>(own, size_t(nr) * nu);
  S.Vu = tmp_alloc<double>(own, size_t(nr) * nu * nu);
  CK(eig_configure(std::max(nx, nu)));
  std::vector<EigJob> jx(static_cast<size_t>(nbx)), ju(static_cast<size_t>(nr));
  for (int b = 0; b < nbx; ++b) {
    const double* M = b < nr ? S.Q + size_t(b) * nx * nx : S.QN + size_t(b - nr) * nx * nx;
    jx[b] = EigJob{M, S.Wx + size_t(b) * nx, S.Vx + size_t(b) * nx * nx, nx, 0};
  }
  for (int k = 0; k < nr; ++k) ju[k] = EigJob{S.R + size_t(k) * nu * nu, S.Wu + size_t(k) * nu,
                                              S.Vu + size_t(k) * nu * nu, nu, 0};
  std::vector<void*> jobs_own;
  const EigJob* djx = tmp_upload(jobs_own, jx.data(), jx.size(), st_);
  const EigJob* dju = tmp_upload(jobs_own, ju.data(), ju.size(), st_);
  launch_sym_eig(djx, nbx, nx, st_);
  CK(cudaGetLastError());
  launch_sym_eig(dju, nr, nu, st_);
  CK(cudaGetLastError());
  // ranks, lambda_max, merged order
  const int pw = nx + nu;
  int* dpx = tmp_alloc<int>(jobs_own, size_t(nbx));
  int* dpu = tmp_alloc<int>(jobs_own, size_t(nr));
  int* dperm = tmp_alloc<int>(jobs_own, size_t(nbx) * pw);
  double* dlm = tmp_alloc<double>(jobs_own, size_t(nbx));
  int* derr = tmp_alloc<int>(jobs_own, 1);
  CK(cudaMemsetAsync(derr, 0, sizeof(int), st_));
  launch_soc_rank(SocRankArgs{S.Wx, S.Wu, nr, nx, nu, dpx, dpu, dperm, dlm, derr}, st_);
  launch_soc_rank(SocRankArgs{S.Wx + size_t(nr) * nx, nullptr, nl, nx, nu, dpx + nr, nullptr,
                              dperm + size_t(nr) * pw, dlm + nr, derr},
                  st_);
  CK(cudaGetLastError());
  std::vector<int> hpx(nbx), hpu(std::max(nr, 1)), hperm(size_t(nbx) * pw);
  std::vector<double> hlm(nbx);
  int herr = 0;
  CK(cudaMemcpyAsync(hpx.data(), dpx, sizeof(int) * nbx, cudaMemcpyDeviceToHost, st_));
  if (nr) CK(cudaMemcpyAsync(hpu.data(), dpu, sizeof(int) * nr, cudaMemcpyDeviceToHost, st_));
  CK(cudaMemcpyAsync(hperm.data(), dperm, sizeof(int) * hperm.size(), cudaMemcpyDeviceToHost, st_));
  CK(cudaMemcpyAsync(hlm.data(), dlm, sizeof(double) * nbx, cudaMemcpyDeviceToHost, st_));
  CK(cudaMemcpyAsync(&herr, derr, sizeof(int), cudaMemcpyDeviceToHost, st_));
  CK(cudaStreamSynchronize(st_));
  for (void* q : jobs_own) cudaFree(q);
  require(herr == 0, "soc_data_quadlin: Q must be positive semidefinite");
  soc_.stage.assign(static_cast<size_t>(nr), SocBlock{});
  soc_.leaf.assign(static_cast<size_t>(nl), SocBlock{});
  for (int k = 0; k < nr; ++k) {
    SocBlock& b = soc_.stage[k];
    b.px = hpx[k], b.pu = hpu[k], b.lambda_max = hlm[k];
    b.perm.assign(hperm.begin() + size_t(k) * pw, hperm.begin() + size_t(k) * pw + b.px + b.pu);
  }
  for (int j = 0; j < nl; ++j) {
    SocBlock& b = soc_.leaf[j];
    b.px = hpx[nr + j], b.lambda_max = hlm[nr + j];
    b.perm.resize(b.px);
    for (int r = 0; r < b.px; ++r) b.perm[r] = r;
  }
}

void Engine::soc_device_build(const std::vector<int64_t>& hxo, const std::vector<int64_t>& huo,
                              const std::vector<int64_t>& ao, const std::vector<int64_t>& hno,
                              const std::vector<int64_t>& aNo) {
  const Tree& tr = p_.tree;
  const int nn = tr.nn(), nr = nn - 1, nl = tr.nl(), nx = p_.nx, nu = p_.nu, pw = nx + nu;
  SocScratch& S = socs_;
  auto& own = S.owned;
  const int nbx = nr + nl;
  double* smsx = tmp_alloc<double>(own, size_t(nbx) * nx * nx);
  double* u2x = tmp_alloc<double>(own, size_t(nbx) * nx * nx);
  double* w2x = tmp_alloc<double>(own, size_t(nbx) * nx);
  double* smsu = tmp_alloc<double>(own, size_t(nr) * nu * nu);
  double* u2u = tmp_alloc<double>(own, size_t(nr) * nu * nu);
  double* w2u = tmp_alloc<double>(own, size_t(nr) * nu);
  double* wst = tmp_alloc<double>(own, size_t(nr) * pw);
  double* wlf = tmp_alloc<double>(own, size_t(nl) * pw);
  std::vector<SocBlockJob> jx(static_cast<size_t>(nbx)), ju(static_cast<size_t>(nr));
  std::vector<EigJob> ex(static_cast<size_t>(nbx)), eu(static_cast<size_t>(nr));
  for (int b = 0; b < nbx; ++b) {
    SocBlockJob& J = jx[b];
    const bool leaf = b >= nr;
    const int k = leaf ? b - nr : b;
    J.n = nx;
    J.p = leaf ? soc_.leaf[k].px : soc_.stage[k].px;
    J.M = leaf ? S.QN + size_t(k) * nx * nx : S.Q + size_t(k) * nx * nx;
    J.v = leaf ? S.qN + size_t(k) * nx : S.q + size_t(k) * nx;
    J.V = S.Vx + size_t(b) * nx * nx;
    J.sms = smsx + size_t(b) * nx * nx;
    J.U2 = u2x + size_t(b) * nx * nx;
    J.W2 = w2x + size_t(b) * nx;
    J.H = const_cast<double*>(leaf ? D_.HN + hno[k] : D_.Hx + hxo[k]);
    J.HT = const_cast<double*>(leaf ? D_.HNT + hno[k] : D_.HxT + hxo[k]);
    J.qk = const_cast<double*>(leaf ? D_.qkN + size_t(k) * nx : D_.qk + size_t(k) * pw);
    J.w = leaf ? wlf + size_t(k) * pw : wst + size_t(k) * pw;
    ex[b] = EigJob{J.sms, J.W2, J.U2, J.p, 0};
  }
  for (int k = 0; k < nr; ++k) {
    SocBlockJob& J = ju[k];
    J.n = nu;
    J.p = soc_.stage[k].pu;
    J.M = S.R + size_t(k) * nu * nu;
    J.v = S.r + size_t(k) * nu;
    J.V = S.Vu + size_t(k) * nu * nu;
    J.sms = smsu + size_t(k) * nu * nu;
    J.U2 = u2u + size_t(k) * nu * nu;
    J.W2 = w2u + size_t(k) * nu;
    J.H = const_cast<double*>(D_.Hu + huo[k]);
    J.HT = const_cast<double*>(D_.HuT + huo[k]);
    J.qk = const_cast<double*>(D_.qk + size_t(k) * pw + nx);
    J.w = wst + size_t(k) * pw + nx;
    eu[k] = EigJob{J.sms, J.W2, J.U2, J.p, 0};
  }
  const SocBlockJob* djx = tmp_upload(own, jx.data(), jx.size(), st_);
  const SocBlockJob* dju = tmp_upload(own, ju.data(), ju.size(), st_);
  const EigJob* dex = tmp_upload(own, ex.data(), ex.size(), st_);
  const EigJob* deu = tmp_upload(own, eu.data(), eu.size(), st_);
  launch_soc_sms(djx, nbx, nx, st_);
  launch_soc_sms(dju, nr, nu, st_);
  launch_sym_eig(dex, nbx, nx, st_);
  launch_sym_eig(deu, nr, nu, st_);
  launch_soc_build(djx, nbx, nx, st_);
  launch_soc_build(dju, nr, nu, st_);
  CK(cudaGetLastError());
  // translations and |qk|^2 (analytic norm bound)
  int* dpx = tmp_alloc<int>(own, size_t(nbx));
  int* dpu = tmp_alloc<int>(own, size_t(std::max(nr, 1)));
  {
    std::vector<int> hpx(nbx), hpu(std::max(nr, 1));
    for (int k = 0; k < nr; ++k) hpx[k] = soc_.stage[k].px, hpu[k] = soc_.stage[k].pu;
    for (int j = 0; j < nl; ++j) hpx[nr + j] = soc_.leaf[j].px;
    CK(cudaMemcpyAsync(dpx, hpx.data(), sizeof(int) * nbx, cudaMemcpyHostToDevice, st_));
    CK(cudaMemcpyAsync(dpu, hpu.data(), sizeof(int) * hpu.size(), cudaMemcpyHostToDevice, st_));
    CK(cudaStreamSynchronize(st_));  // host vectors go out of scope
  }
  const int64_t* dao = tmp_upload(own, ao.data(), ao.size(), st_);
  const int64_t* daNo = tmp_upload(own, aNo.data(), aNo.size(), st_);
  double* qk2 = tmp_alloc<double>(own, size_t(nbx));
  launch_soc_tail(SocTailArgs{wst, dpx, dpu, dao, const_cast<double*>(D_.a), D_.qk, pw, qk2, nr, nx, nu}, st_);
  launch_soc_tail(SocTailArgs{wlf, dpx + nr, nullptr, daNo, const_cast<double*>(D_.aN), D_.qkN, nx, qk2 + nr, nl,
                              nx, nu},
                  st_);
  CK(cudaGetLastError());
  std::vector<double> h2(nbx);
  CK(cudaMemcpyAsync(h2.data(), qk2, sizeof(double) * nbx, cudaMemcpyDeviceToHost, st_));
  CK(cudaStreamSynchronize(st_));
  for (int k = 0; k < nr; ++k) soc_.stage[k].qk2 = h2[k];
  for (int j = 0; j < nl; ++j) soc_.leaf[j].qk2 = h2[nr + j];
  for (void* q : own) cudaFree(q);
  own.clear();
  S = SocScratch{};
}

void Engine::upload() {
  const Tree& tr = p_.tree;
  const int nn = tr.nn(), nnl = tr.nnl(), nl = tr.nl(), nr = nn - 1, nx = p_.nx, nu = p_.nu;
  Dev& D = D_;
  D.nn = nn, D.nnl = nnl, D.nl = nl, D.nr = nr, D.nx = nx, D.nu = nu, D.N = tr.horizon;
  D.nz = int(lay_.nz), D.neta = int(lay_.neta);
  D.anc = dupload(tr.anc);
  D.cf = dupload(tr.child_first);
  D.cc = dupload(tr.child_count);
  D.u_base = lay_.u_base, D.tau_base = lay_.tau_base, D.s_base = lay_.s_base;
  D.y_base = lay_.u_base + nnl * nu;
  D.y_off = dupload(lay_.y_off);
  D.y_dim = dupload(lay_.y_dim);
  D.s1_off = dupload(lay_.seg1_off);
  D.s1_nc = dupload(lay_.seg1_nc);
  D.s1_ydim = dupload(lay_.seg1_ydim);
  D.s2_off = dupload(lay_.seg2_off);
  D.s2_dim = dupload(lay_.seg2_dim);
  D.s3_off = dupload(lay_.seg3_off);
  D.s3_nc = dupload(lay_.seg3_nc);
  D.s3_socdim = dupload(lay_.seg3_socdim);

  // stage-cost SOC data
  std::vector<int64_t> shxo, shuo, sao;
  {
    std::vector<int> px(nr), pu(nr);
    std::vector<int64_t> hxo(nr), huo(nr), ao(nr);
    int64_t sx = 0, su = 0, sa = 0;
    for (int k = 0; k < nr; ++k) {
      px[k] = soc_.stage[k].px;
      pu[k] = soc_.stage[k].pu;
      hxo[k] = sx;
      huo[k] = su;
      ao[k] = sa;
      sx += pad2(int64_t(px[k]) * nx);
      su += pad2(int64_t(pu[k]) * nu);
      sa += px[k] + pu[k] + 2;
    }
    std::vector<double> Hx, HxT, Hu, HuT, qk, a;
    if (!soc_dev_) {
      Hx.resize(sx), HxT.resize(sx), Hu.resize(su), HuT.resize(su), qk.resize(size_t(nr) * (nx + nu)), a.resize(sa);
    }
    for (int k = 0; k < nr && !soc_dev_; ++k) {
      const SocBlock& b = soc_.stage[k];
      for (int j = 0; j < nx; ++j)
        for (int r = 0; r < b.px; ++r) {
          const double v = b.Hx[r + size_t(j) * b.px];
          Hx[hxo[k] + r + size_t(j) * b.px] = v;
          HxT[hxo[k] + j + size_t(r) * nx] = v;
        }
      for (int j = 0; j < nu; ++j)
        for (int r = 0; r < b.pu; ++r) {
          const double v = b.Hu[r + size_t(j) * b.pu];
          Hu[huo[k] + r + size_t(j) * b.pu] = v;
          HuT[huo[k] + j + size_t(r) * nu] = v;
        }
      std::copy(b.qk.begin(), b.qk.end(), qk.begin() + size_t(k) * (nx + nu));
      std::copy(b.a.begin(), b.a.end(), a.begin() + ao[k]);
    }
    D.px = dupload(px);
    D.pu = dupload(pu);
    D.hx_off = dupload(hxo);
    D.hu_off = dupload(huo);
    D.a_off = dupload(ao);
    hxo_ = hxo, huo_ = huo, ao_ = ao;
    if (soc_dev_) {
      D.Hx = dalloc<double>(sx);
      D.HxT = dalloc<double>(sx);
      D.Hu = dalloc<double>(su);
      D.HuT = dalloc<double>(su);
      D.qk = dalloc<double>(size_t(nr) * (nx + nu));
      D.a = dalloc<double>(sa);
    } else {
      D.Hx = dupload(Hx);
      D.HxT = dupload(HxT);
      D.Hu = dupload(Hu);
      D.HuT = dupload(HuT);
      D.qk = dupload(qk);
      D.a = dupload(a);
    }
    shxo = std::move(hxo), shuo = std::move(huo), sao = std::move(ao);
  }
  // terminal SOC data
  {
    std::vector<int> pN(nl);
    std::vector<int64_t> ho(nl), ao(nl);
    int64_t sh = 0, sa = 0;
    for (int j = 0; j < nl; ++j) {
      pN[j] = soc_.leaf[j].px;
      ho[j] = sh;
      ao[j] = sa;
      sh += pad2(int64_t(pN[j]) * nx);
      sa += pN[j] + 2;
    }
    std::vector<double> HN, HNT, qk, a;
    if (!soc_dev_) HN.resize(sh), HNT.resize(sh), qk.resize(size_t(nl) * nx), a.resize(sa);
    for (int j = 0; j < nl && !soc_dev_; ++j) {
      const SocBlock& b = soc_.leaf[j];
      for (int c = 0; c < nx; ++c)
        for (int r = 0; r < b.px; ++r) {
          const double v = b.Hx[r + size_t(c) * b.px];
          HN[ho[j] + r + size_t(c) * b.px] = v;
          HNT[ho[j] + c + size_t(r) * nx] = v;
        }
      std::copy(b.qk.begin(), b.qk.begin() + nx, qk.begin() + size_t(j) * nx);
      std::copy(b.a.begin(), b.a.end(), a.begin() + ao[j]);
    }
    D.pN = dupload(pN);
    D.hn_off = dupload(ho);
    D.aN_off = dupload(ao);
    hno_ = ho, aNo_ = ao;
    if (soc_dev_) {
      D.HN = dalloc<double>(sh);
      D.HNT = dalloc<double>(sh);
      D.qkN = dalloc<double>(size_t(nl) * nx);
      D.aN = dalloc<double>(sa);
      soc_device_build(shxo, shuo, sao, ho, ao);
    } else {
      D.HN = dupload(HN);
      D.HNT = dupload(HNT);
      D.qkN = dupload(qk);
      D.aN = dupload(a);
    }
  }
  // boundary permutation of eta (stage SOC head rows)
  {
    std::vector<int> perm(lay_.neta);
    for (int64_t i = 0; i < lay_.neta; ++i) perm[i] = int(i);
    perm_identity_ = true;
    for (int k = 0; k < nr; ++k) {
      const SocBlock& b = soc_.stage[k];
      for (int r = 0; r < b.px + b.pu; ++r) {
        perm[lay_.seg2_off[k] + r] = lay_.seg2_off[k] + b.perm[r];
        if (b.perm[r] != r) perm_identity_ = false;
      }
    }
    perm_eta_ = dupload(perm);
  }
  // constraints
  {
    std::vector<uint8_t> nd(static_cast<size_t>(std::max(nnl, 1)), 0);  // node i: [Gx Gu] not square diagonal
    parallel_for(nnl, [&](int64_t ii) {
      const int i = int(ii);
      if (p_.nc[i] != nx + nu) {
        nd[i] = 1;
        return;
      }
      const size_t o = size_t(p_.g_off[i]);
      const int nc = p_.nc[i];
      for (int c = 0; c < nx; ++c)
        for (int r = 0; r < nc; ++r)
          if (r != c && p_.Gx[o * nx + r + size_t(c) * nc] != 0.0) {
            nd[i] = 1;
            return;
          }
      for (int c = 0; c < nu; ++c)
        for (int r = 0; r < nc; ++r)
          if (r != nx + c && p_.Gu[o * nu + r + size_t(c) * nc] != 0.0) {
            nd[i] = 1;
            return;
          }
    });
    bool gdiag = true;
    for (int i = 0; i < nnl; ++i) gdiag = gdiag && !nd[i];
    D.g_diag = gdiag ? 1 : 0;
    const int64_t rows = p_.g_off[nnl];
    std::vector<int64_t> goff(p_.g_off.begin(), p_.g_off.end() - 1);
    D.g_off = dupload(goff);
    D.lo = dupload(p_.C_lo);
    D.hi = dupload(p_.C_hi);
    if (gdiag) {
      std::vector<double> gd(size_t(nnl) * (nx + nu));
      parallel_for(nnl, [&](int64_t ii) {
        const int i = int(ii);
        const size_t o = size_t(p_.g_off[i]);
        const int nc = p_.nc[i];
        for (int r = 0; r < nx; ++r) gd[size_t(i) * (nx + nu) + r] = p_.Gx[o * nx + r + size_t(r) * nc];
        for (int r = 0; r < nu; ++r) gd[size_t(i) * (nx + nu) + nx + r] = p_.Gu[o * nu + nx + r + size_t(r) * nc];
      });
      D.gd = dupload(gd);
    } else {
      std::vector<double> GxT(size_t(rows) * nx), GuT(size_t(rows) * nu);
      for (int i = 0; i < nnl; ++i) {
        const size_t o = size_t(p_.g_off[i]);
        const int nc = p_.nc[i];
        for (int c = 0; c < nx; ++c)
          for (int r = 0; r < nc; ++r) GxT[o * nx + c + size_t(r) * nx] = p_.Gx[o * nx + r + size_t(c) * nc];
        for (int c = 0; c < nu; ++c)
          for (int r = 0; r < nc; ++r) GuT[o * nu + c + size_t(r) * nu] = p_.Gu[o * nu + r + size_t(c) * nc];
      }
      D.Gx = dupload(p_.Gx);
      D.Gu = dupload(p_.Gu);
      D.GxT = dupload(GxT);
      D.GuT = dupload(GuT);
    }
    bool gndiag = true;
    for (int j = 0; j < nl && gndiag; ++j) {
      if (p_.ncN[j] != nx) {
        gndiag = false;
        break;
      }
      const size_t o = size_t(p_.gN_off[j]);
      for (int c = 0; c < nx && gndiag; ++c)
        for (int r = 0; r < nx; ++r)
          if (r != c && p_.GN[o * nx + r + size_t(c) * nx] != 0.0) {
            gndiag = false;
            break;
          }
    }
    D.gN_diag = gndiag ? 1 : 0;
    std::vector<int64_t> gnoff(p_.gN_off.begin(), p_.gN_off.end() - 1);
    D.gN_off = dupload(gnoff);
    D.loN = dupload(p_.CN_lo);
    D.hiN = dupload(p_.CN_hi);
    if (gndiag) {
      std::vector<double> gd(size_t(nl) * nx);
      for (int j = 0; j < nl; ++j) {
        const size_t o = size_t(p_.gN_off[j]);
        for (int r = 0; r < nx; ++r) gd[size_t(j) * nx + r] = p_.GN[o * nx + r + size_t(r) * nx];
      }
      D.gNd = dupload(gd);
    } else {
      const int64_t rN = p_.gN_off[nl];
      std::vector<double> GNT(size_t(rN) * nx);
      for (int j = 0; j < nl; ++j) {
        const size_t o = size_t(p_.gN_off[j]);
        const int nc = p_.ncN[j];
        for (int c = 0; c < nx; ++c)
          for (int r = 0; r < nc; ++r) GNT[o * nx + c + size_t(r) * nx] = p_.GN[o * nx + r + size_t(c) * nc];
      }
      D.GN = dupload(p_.GN);
      D.GNT = dupload(GNT);
    }
  }
  // risk: b, dual cone of the y-copy rows, S2 kind
  {
    std::vector<double> rb;
    std::vector<int> ycn(nnl), ypo(nnl + 1, 0), ykind, ydim, s2k(nnl);
    std::vector<double> s2g(nnl, 0.0);
    std::vector<int64_t> s2po(nnl, 0);
    std::vector<double> s2P;
    for (int i = 0; i < nnl; ++i) {
      const Risk& rs = p_.risk[i];
      rb.insert(rb.end(), rs.b.begin(), rs.b.end());
      std::vector<ConePart> dk;
      for (const auto& cp : rs.cone) {
        if (cp.kind == SPOCK_CONE_ZERO)
          dk.push_back({SPOCK_CONE_FREE, cp.dim});
        else if (cp.kind == SPOCK_CONE_FREE)
          dk.push_back({SPOCK_CONE_ZERO, cp.dim});
        else
          dk.push_back(cp);
      }
      bool simple = true;
      int nonneg = 0;
      for (size_t t = 0; t < dk.size(); ++t) {
        if (t == 0 && dk[t].kind == SPOCK_CONE_NONNEG)
          nonneg = dk[t].dim;
        else if (dk[t].kind != SPOCK_CONE_FREE)
          simple = false;
      }
      ycn[i] = simple ? nonneg : -1;
      for (const auto& cp : dk) {
        ykind.push_back(cp.kind);
        ydim.push_back(cp.dim);
      }
      ypo[i + 1] = int(ykind.size());
      // S2 closed form detection on E (exact structure of the AV@R forms)
      const int n = rs.n, ny = rs.rows;
      auto E = [&](int r, int c) { return rs.E[r + size_t(c) * ny]; };
      int kind = S2_DENSE;
      double gam = 0.0;
      if (rs.nnu == 0) {
        if (ny == 2 * n + 1 && E(0, 0) > 0.0) {
          gam = E(0, 0);
          bool ok = true;
          for (int c = 0; c < n && ok; ++c)
            for (int r = 0; r < ny; ++r) {
              double want = 0.0;
              if (r < n) want = (r == c) ? gam : 0.0;
              else if (r < 2 * n) want = (r - n == c) ? -1.0 : 0.0;
              else want = 1.0;
              if (E(r, c) != want) {
                ok = false;
                break;
              }
            }
          if (ok) kind = S2_AVAR;
        } else if (ny == n + 1) {
          bool ok = true;
          for (int c = 0; c < n && ok; ++c)
            for (int r = 0; r < ny; ++r) {
              const double want = r < n ? ((r == c) ? -1.0 : 0.0) : 1.0;
              if (E(r, c) != want) {
                ok = false;
                break;
              }
            }
          if (ok) kind = S2_MAX;
        } else if (ny == n) {
          bool ok = true;
          for (int c = 0; c < n && ok; ++c)
            for (int r = 0; r < ny; ++r)
              if (E(r, c) != (r == c ? 1.0 : 0.0)) {
                ok = false;
                break;
              }
          if (ok) kind = S2_EQ;
        }
      }
      s2k[i] = kind;
      s2g[i] = gam;
      if (kind == S2_DENSE) {
        // projector onto ker M, M = [E' -I -I; F' 0 0] (projections.cpp:114-137):
        // N = I - M'(MM')^+ M with a relative eigenvalue threshold on MM'
        const int dim = ny + 2 * n, mr = n + rs.nnu;
        require(dim <= kMaxD, "spock-b200: general risk spec with y+2*children above 256 is not supported");
        max_dense_s2_ = std::max(max_dense_s2_, dim);
        Mat M(mr, dim);
        for (int c = 0; c < n; ++c) {
          for (int r = 0; r < ny; ++r) M(c, r) = E(r, c);
          M(c, ny + c) = -1.0;
          M(c, ny + n + c) = -1.0;
        }
        for (int c = 0; c < rs.nnu; ++c)
          for (int r = 0; r < ny; ++r) M(n + c, r) = rs.F[r + size_t(c) * ny];
        Mat MM(mr, mr);
        for (int a2 = 0; a2 < mr; ++a2)
          for (int b2 = 0; b2 < mr; ++b2) {
            double s = 0.0;
            for (int t = 0; t < dim; ++t) s += M(a2, t) * M(b2, t);
            MM(a2, b2) = s;
          }
        Vec w;
        Mat V;
        sym_eig(MM, w, V);
        const double lmax = w.empty() ? 0.0 : w.back();
        Mat Pinv(mr, mr);
        for (int t = 0; t < mr; ++t) {
          if (!(w[t] > 1e-14 * lmax)) continue;
          for (int b2 = 0; b2 < mr; ++b2)
            for (int a2 = 0; a2 < mr; ++a2) Pinv(a2, b2) += V(a2, t) * V(b2, t) / w[t];
        }
        s2po[i] = int64_t(s2P.size());
        s2P.resize(s2P.size() + size_t(dim) * dim);
        double* N = &s2P[s2po[i]];
        for (int c = 0; c < dim; ++c)
          for (int r = 0; r < dim; ++r) {
            double s = (r == c) ? 1.0 : 0.0;
            for (int a2 = 0; a2 < mr; ++a2) {
              double t2 = 0.0;
              for (int b2 = 0; b2 < mr; ++b2) t2 += Pinv(a2, b2) * M(b2, c);
              s -= M(a2, r) * t2;
            }
            N[r + size_t(c) * dim] = s;
          }
      }
    }
    D.rb = dupload(rb);
    D.yc_nonneg = dupload(ycn);
    D.yc_poff = dupload(ypo);
    D.yc_kind = dupload(ykind);
    D.yc_dim = dupload(ydim);
    D.s2_kind = dupload(s2k);
    D.s2_gamma = dupload(s2g);
    D.s2p_off = dupload(s2po);
    D.s2P = dupload(s2P);
  }
  // factor buffers (filled by factorize) and scratch
  D.m1_stride = pad2(int64_t(nx) * (nx + nu));
  D.k_stride = pad2(int64_t(nx) * nu);
  D.r_stride = pad2(int64_t(nu) * nu);
  D.M1 = dalloc<double>(size_t(nr) * D.m1_stride);
  D.M1T = dalloc<double>(size_t(nr) * D.m1_stride);
  D.cvec = dupload(p_.c);
  D.K = dalloc<double>(size_t(nnl) * D.k_stride);
  D.KT = dalloc<double>(size_t(nnl) * D.k_stride);
  D.Rinv = dalloc<double>(size_t(nnl) * D.r_stride);
  D.g = dalloc<double>(size_t(nnl) * nu);
  D.h = dalloc<double>(size_t(nnl) * nx);
  xinit_ = dalloc<double>(nx);
  D.xinit = xinit_;
  D.T12 = dalloc<double>(size_t(nr) * (nx + nu));
  D.adj = dalloc<double>(size_t(nr) * (nx + nu));
  D.dvec = dalloc<double>(size_t(nnl) * nu);
  // termination scalings d1 (z) and d2 (eta), proj/src/solver.cpp:100-109
  {
    std::vector<double> d1(lay_.nz, 1.0), d2(lay_.neta, 1.0);
    if (!pc_.is_identity) {
      for (int i = 0; i < nn; ++i) {
        const Vec& s = tr.leaf(i) ? pc_.sxN : pc_.sx;
        for (int k = 0; k < nx; ++k) d1[1 + size_t(i) * nx + k] = s[k];
        if (i < nnl)
          for (int k = 0; k < nu; ++k) d1[lay_.u_base + size_t(i) * nu + k] = pc_.su[k];
      }
      for (int i = 0; i < nnl; ++i)
        for (int k = 0; k < lay_.seg1_nc[i]; ++k)
          d2[lay_.seg1_off[i] + lay_.seg1_ydim[i] + 1 + k] = pc_.cstr_scale[i];
    }
    d1_ = dupload(d1);
    d2_ = dupload(d2);
  }
  partial_ = dalloc<double>(size_t(4) * kRedRegion);
  red_out_ = dalloc<double>(512);
  gram_partial_ = dalloc<double>(size_t(kGramRegion));
  gram_out_ = dalloc<double>(size_t(4 * kAaHostMax));
  gram_h_.assign(size_t(kAaHostMax) * kAaHostMax, dd{0.0, 0.0});
  gram_r_.assign(size_t(kAaHostMax), dd{0.0, 0.0});
  CK(cudaMallocHost(&host_red_, 512 * sizeof(double)));
  for (int t = 0; t < 3; ++t) {
    scratch_z_[t] = dalloc<double>(lay_.nz);
    scratch_e_[t] = dalloc<double>(lay_.neta);
  }
  set_xinit(raw_xinit_.data());
}

void Engine::set_xinit(const double* x) {
  std::vector<double> xs(p_.nx);
  for (int k = 0; k < p_.nx; ++k) xs[k] = pc_.is_identity ? x[k] : pc_.sx[k] * x[k];
  CK(cudaMemcpyAsync(xinit_, xs.data(), sizeof(double) * p_.nx, cudaMemcpyHostToDevice, st_));
  CK(cudaStreamSynchronize(st_));
}

// ---------------------------------------------------------------------------
// Alg. 1 on device, stage by stage (projections.cpp:77-112), followed by the
// per-iteration factors of the restructured sweep (see kernels.cu).
void Engine::factorize() {
  const Tree& tr = p_.tree;
  const int nn = tr.nn(), nr = nn - 1, nx = p_.nx, nu = p_.nu, N = tr.horizon;
  std::vector<void*> tmp;
  auto talloc = [&](size_t n) {
    void* p = nullptr;
    CK(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(double)));
    tmp.push_back(p);
    return static_cast<double*>(p);
  };
  double* dA = talloc(size_t(nr) * nx * nx);
  double* dB = talloc(size_t(nr) * nx * nu);
  CK(cudaMemcpyAsync(dA, p_.A.data(), sizeof(double) * p_.A.size(), cudaMemcpyHostToDevice, st_));
  CK(cudaMemcpyAsync(dB, p_.B.data(), sizeof(double) * p_.B.size(), cudaMemcpyHostToDevice, st_));
  double* P = talloc(size_t(nn) * nx * nx);
  double* PB = talloc(size_t(nr) * nx * nu);
  double* PA = talloc(size_t(nr) * nx * nx);
  double* e = talloc(size_t(nr) * nx);
  double* rt = talloc(size_t(nr) * nu * nu);
  double* kt = talloc(size_t(nr) * nu * nx);
  double* ge = talloc(size_t(nr) * nu);
  double* tt = talloc(size_t(nr) * nx * nx);
  double* pt = talloc(size_t(nr) * nx * nx);
  double* he = talloc(size_t(nr) * nx);
  int* derr = nullptr;
  CK(cudaMalloc(&derr, sizeof(int)));
  tmp.push_back(derr);
  CK(cudaMemsetAsync(derr, 0, sizeof(int), st_));
  // leaves: P = I
  CK(cudaMemsetAsync(P, 0, sizeof(double) * size_t(nn) * nx * nx, st_));
  launch_eye(P + size_t(tr.stage_start[N]) * nx * nx, nn - tr.stage_start[N], nx, st_);
  CK(cudaGetLastError());
  // pointer arrays for batched GEMMs (rebuilt per stage)
  const size_t maxw = size_t(nr) + 1;
  const double** hA = new const double*[maxw];
  const double** hBp = new const double*[maxw];
  double** hC = new double*[maxw];
  const double** dAp = nullptr;
  const double** dBp = nullptr;
  double** dCp = nullptr;
  CK(cudaMalloc(&dAp, sizeof(void*) * maxw));
  CK(cudaMalloc(&dBp, sizeof(void*) * maxw));
  CK(cudaMalloc(&dCp, sizeof(void*) * maxw));
  tmp.push_back(dAp);
  tmp.push_back(dBp);
  tmp.push_back(dCp);
  auto gemm = [&](int cnt, int m, int n, int k, int lda, int ldb, int ldc, int ta, int tb, double alpha,
                  double beta) {
    if (cnt <= 0) return;
    CK(cudaMemcpyAsync(dAp, hA, sizeof(void*) * cnt, cudaMemcpyHostToDevice, st_));
    CK(cudaMemcpyAsync(dBp, hBp, sizeof(void*) * cnt, cudaMemcpyHostToDevice, st_));
    CK(cudaMemcpyAsync(dCp, hC, sizeof(void*) * cnt, cudaMemcpyHostToDevice, st_));
    BGemmArgs G{dAp, dBp, dCp, m, n, k, lda, ldb, ldc, ta, tb, alpha, beta};
    launch_bgemm(G, cnt, st_);
    CK(cudaStreamSynchronize(st_));  // host pointer arrays are reused
  };
  Alg1Args A1{};
  A1.nx = nx;
  A1.nu = nu;
  A1.m1_stride = D_.m1_stride;
  A1.k_stride = D_.k_stride;
  A1.r_stride = D_.r_stride;
  A1.cf = D_.cf;
  A1.cc = D_.cc;
  A1.anc = D_.anc;
  A1.A = dA;
  A1.B = dB;
  A1.rt = rt;
  A1.kt = kt;
  A1.ge = ge;
  A1.pt = pt;
  A1.he = he;
  A1.P = P;
  A1.K = const_cast<double*>(D_.K);
  A1.KT = const_cast<double*>(D_.KT);
  A1.Rinv = const_cast<double*>(D_.Rinv);
  A1.g = const_cast<double*>(D_.g);
  A1.h = const_cast<double*>(D_.h);
  A1.M1 = const_cast<double*>(D_.M1);
  A1.M1T = const_cast<double*>(D_.M1T);
  A1.err = derr;
  const int smem = int(sizeof(double) * (2 * nu * nu + nu * nx));
  if (smem > 48 * 1024) CK(set_alg1_smem(smem));
  const double* dcv = D_.cvec;
  for (int t = N - 1; t >= 0; --t) {
    const int cb = tr.stage_start[t + 1], ce = tr.stage_start[t + 2], cnt = ce - cb;
    const int pb = tr.stage_start[t], pe = tr.stage_start[t + 1];
    // PB = P_c B, PA = P_c A, e = P_c c
    for (int c = cb; c < ce; ++c) {
      hA[c - cb] = P + size_t(c) * nx * nx;
      hBp[c - cb] = dB + size_t(c - 1) * nx * nu;
      hC[c - cb] = PB + size_t(c - 1) * nx * nu;
    }
    gemm(cnt, nx, nu, nx, nx, nx, nx, 0, 0, 1.0, 0.0);
    for (int c = cb; c < ce; ++c) {
      hBp[c - cb] = dA + size_t(c - 1) * nx * nx;
      hC[c - cb] = PA + size_t(c - 1) * nx * nx;
    }
    gemm(cnt, nx, nx, nx, nx, nx, nx, 0, 0, 1.0, 0.0);
    for (int c = cb; c < ce; ++c) {
      hBp[c - cb] = dcv + size_t(c - 1) * nx;
      hC[c - cb] = e + size_t(c - 1) * nx;
    }
    gemm(cnt, nx, 1, nx, nx, nx, nx, 0, 0, 1.0, 0.0);
    // rt = B'PB, kt = B'PA, ge = B'e
    for (int c = cb; c < ce; ++c) {
      hA[c - cb] = dB + size_t(c - 1) * nx * nu;
      hBp[c - cb] = PB + size_t(c - 1) * nx * nu;
      hC[c - cb] = rt + size_t(c - 1) * nu * nu;
    }
    gemm(cnt, nu, nu, nx, nx, nx, nu, 1, 0, 1.0, 0.0);
    for (int c = cb; c < ce; ++c) {
      hBp[c - cb] = PA + size_t(c - 1) * nx * nx;
      hC[c - cb] = kt + size_t(c - 1) * nu * nx;
    }
    gemm(cnt, nu, nx, nx, nx, nx, nu, 1, 0, 1.0, 0.0);
    for (int c = cb; c < ce; ++c) {
      hBp[c - cb] = e + size_t(c - 1) * nx;
      hC[c - cb] = ge + size_t(c - 1) * nu;
    }
    gemm(cnt, nu, 1, nx, nx, nx, nu, 1, 0, 1.0, 0.0);
    // parents: Rt, Cholesky, Rinv, K, g
    A1.b = pb;
    launch_alg1_parent(A1, pe - pb, st_);
    // children: Abar = A + B K_anc -> M1, M1'
    A1.b = cb;
    launch_alg1_child_abar(A1, cnt, st_);
    // tt = P_c Abar ; pt = Abar' tt ; he = Abar' e
    for (int c = cb; c < ce; ++c) {
      hA[c - cb] = P + size_t(c) * nx * nx;
      hBp[c - cb] = D_.M1 + size_t(c - 1) * D_.m1_stride;
      hC[c - cb] = tt + size_t(c - 1) * nx * nx;
    }
    gemm(cnt, nx, nx, nx, nx, nx, nx, 0, 0, 1.0, 0.0);
    for (int c = cb; c < ce; ++c) {
      hA[c - cb] = D_.M1 + size_t(c - 1) * D_.m1_stride;
      hBp[c - cb] = tt + size_t(c - 1) * nx * nx;
      hC[c - cb] = pt + size_t(c - 1) * nx * nx;
    }
    gemm(cnt, nx, nx, nx, nx, nx, nx, 1, 0, 1.0, 0.0);
    for (int c = cb; c < ce; ++c) {
      hBp[c - cb] = e + size_t(c - 1) * nx;
      hC[c - cb] = he + size_t(c - 1) * nx;
    }
    gemm(cnt, nx, 1, nx, nx, nx, nx, 1, 0, 1.0, 0.0);
    // parents: P = I + K'K + sum pt ; h = sum he
    A1.b = pb;
    launch_alg1_parent2(A1, pe - pb, st_);
  }
  CK(cudaGetLastError());
  int herr = 0;
  CK(cudaMemcpyAsync(&herr, derr, sizeof(int), cudaMemcpyDeviceToHost, st_));
  CK(cudaStreamSynchronize(st_));
  delete[] hA;
  delete[] hBp;
  delete[] hC;
  for (void* p : tmp) cudaFree(p);
  if (herr) throw std::runtime_error("make_solver_cache: Cholesky failed (corrupt dynamics data)");
}

// ---------------------------------------------------------------------------
void Engine::sync() { CK(cudaStreamSynchronize(st_)); }

// standalone L / L*: CTA-per-node kernels on narrow trees (latency), warp-per-
// node kernels on wide ones (throughput); same arithmetic
// one launch of the streaming kernel over a ticket list: the throughput
// configuration, or the latency one when there is about one item per warp
void Engine::launch_wide(WideArgs A, const WRec* recs, int ntick) {
  A.recs = recs;
  A.ntick = ntick;
  if (ntick <= wide_grid_lat_ * wlat_.warps) {
    A.warps = wlat_.warps, A.slots = wlat_.slots;
    CK(launch_T_wide(A, wide_rows_, 1, std::min(wide_grid_lat_, (ntick + A.warps - 1) / A.warps), st_));
  } else {
    CK(launch_T_wide(A, wide_rows_, wide_ctas_, std::min(wide_grid_, (ntick + A.warps - 1) / A.warps), st_));
  }
}

void Engine::L(const double* z, double* eta) {
  if (shard_solving_) {
    shard_L(z, eta);
    return;
  }
  if (wide_ok_ && !lop_wide_ && lop_narrow_) {
    launch_L_lop(D_, wargs_, lrec_, z, eta, lop_rows_, lop_mat_, lop_vec_, st_);
    CK(cudaGetLastError());
    return;
  }
  if (wide_ok_ && lop_wide_) {  // warp-granular streaming items (wide.cu, kind 3)
    WideArgs A = wargs_;
    A.D = D_, A.z = z, A.eo = eta;
    launch_wide(A, lrec_, nlrec_);
    CK(cudaGetLastError());
    return;
  }
  if (narrow_)
    launch_L_narrow(D_, z, eta, st_);
  else
    launch_L(D_, z, 1.0, nullptr, 0.0, nullptr, eta, 0.0, false, st_);
  CK(cudaGetLastError());
}

void Engine::Lt(const double* eta, double* z) {
  if (shard_solving_) {
    shard_Lt(eta, z);
    return;
  }
  if (wide_ok_ && !lop_wide_ && lop_narrow_) {
    launch_Lt_lop(D_, wargs_, ltrec_, eta, z, lop_rows_, lop_mat_, lop_vec_, st_);
    CK(cudaGetLastError());
    return;
  }
  if (wide_ok_ && lop_wide_) {  // kinds 4 (child terms, flagged) then 5 (node rows)
    WideArgs A = wargs_;
    A.D = D_, A.eta = eta, A.zo = z;
    CK(cudaMemsetAsync(wide_flags_, 0, sizeof(int) * size_t(p_.tree.nn()), st_));
    launch_wide(A, ltrec_, nltrec_);
    CK(cudaGetLastError());
    return;
  }
  if (narrow_)
    launch_Lt_narrow(D_, eta, z, st_);
  else
    launch_Lt(D_, eta, nullptr, z, 0.0, 1.0, 0.0, st_);
  CK(cudaGetLastError());
}

// one CP application (solver.cpp:148-164), internal layout; zo/eo must not
// alias z/eta
void Engine::T(const double* z, const double* eta, double* zo, double* eo) {
  if (shard_solving_) {
    shard_T(z, eta, zo, eo);
    return;
  }
  if (fused_ok_) {
    FusedArgs F = fargs_;
    F.D = D_;
    F.z = z;
    F.eta = eta;
    F.zo = zo;
    F.eo = eo;
    F.base[FB_Z] = z;
    F.base[FB_ETA] = eta;
    F.alpha = alpha_;
    CK(cudaMemsetAsync(F.ticket, 0, fused_sync_bytes_, st_));
    launch_T_fused(F, fused_grid_, st_);
    CK(cudaGetLastError());
    return;
  }
  if (t_wide_) {
    WideArgs A = wargs_;
    A.D = D_;
    A.z = z;
    A.eta = eta;
    A.zo = zo;
    A.eo = eo;
    A.alpha = alpha_;
    CK(cudaMemsetAsync(wide_flags_, 0, wide_flag_bytes_, st_));
    if (t_split_) {
      for (int k = 0; k < 3; ++k) launch_wide(A, tsplit_rec_[k], tsplit_n_[k]);
      CK(cudaGetLastError());
      return;
    }
    A.recs = wargs_.recs;
    A.ntick = wargs_.ntick;
    CK(launch_T_wide(A, wide_rows_, wide_ctas_, wide_grid_, st_));
    CK(cudaGetLastError());
    return;
  }
  launch_Lt(D_, eta, z, zo, 1.0, -alpha_, -alpha_, st_);
  launch_s1(D_, stage_start_.data(), zo, st_);
  launch_s2(D_, zo, st_);
  launch_L(D_, zo, 2.0, z, -1.0, eta, eo, alpha_, true, st_);
  CK(cudaGetLastError());
}

void Engine::dots(std::initializer_list<std::pair<const double*, const double*>> pairs, int64_t n_default,
                  const std::vector<int64_t>& ns, double* host_out) {
  DotArgs A{};
  int j = 0;
  for (const auto& pr : pairs) {
    A.x[j] = pr.first;
    A.y[j] = pr.second;
    A.n[j] = int(j < int(ns.size()) ? ns[j] : n_default);
    ++j;
  }
  A.ndots = j;
  launch_dots(A, partial_, red_out_, st_);
  CK(cudaMemcpyAsync(host_red_, red_out_, sizeof(double) * j, cudaMemcpyDeviceToHost, st_));
  sync();
  for (int k = 0; k < j; ++k) host_out[k] = host_red_[k];
}

// power iteration on L*L (tree_operator.cpp:157-205) with device operators
void Engine::power_iteration() {
  const int64_t nz = lay_.nz, ne = lay_.neta;
  std::vector<double> v(nz);
  philox_normals(0x9E3779B97F4A7C15ull, nz, v.data());
  double vn = 0.0;
  for (double x : v) vn += x * x;
  vn = std::sqrt(vn);
  for (auto& x : v) x /= vn;
  double* dv = scratch_z_[0];
  double* du = scratch_e_[0];
  double* dw = scratch_z_[1];
  CK(cudaMemcpyAsync(dv, v.data(), sizeof(double) * nz, cudaMemcpyHostToDevice, st_));
  const double tol = 1e-6;
  const int max_iters = 500;
  double prev = 0.0, prev_change = 0.0;
  for (int it = 1; it <= max_iters; ++it) {
    L(dv, du);
    double r;
    dots({{du, du}}, ne, {}, &r);
    const double est = std::sqrt(r);
    norm_.estimate = est;
    norm_.iterations = it;
    if (std::getenv("SPOCK_DEBUG_NORM")) std::fprintf(stderr, "[power] it %d est %.17g\n", it, est);
    if (est == 0.0) {
      norm_.converged = true;
      break;
    }
    if (it > 2) {
      const double change = std::fabs(est - prev);
      double ratio = prev_change > 0.0 ? change / prev_change : 0.0;
      ratio = std::min(ratio, 0.999);
      const double remaining = change * ratio / (1.0 - ratio);
      if (change + remaining <= tol * est) {
        norm_.converged = true;
        break;
      }
      prev_change = change;
    } else if (it == 2) {
      prev_change = std::fabs(est - prev);
    }
    prev = est;
    Lt(du, dw);
    double wn2;
    dots({{dw, dw}}, nz, {}, &wn2);
    const double wn = std::sqrt(wn2);
    if (wn == 0.0) {
      norm_.converged = true;
      break;
    }
    launch_axpby(int(nz), 1.0 / wn, dw, 0.0, nullptr, dv, st_);
  }
}

// ---------------------------------------------------------------------------
// boundary conversions
void Engine::copy_in_z(const double* src, double* dst) {
  CK(cudaMemcpyAsync(dst, src, sizeof(double) * lay_.nz, cudaMemcpyDefault, st_));
}
void Engine::to_internal_eta(const double* src, double* dst) {
  if (perm_identity_) {
    CK(cudaMemcpyAsync(dst, src, sizeof(double) * lay_.neta, cudaMemcpyDefault, st_));
    return;
  }
  const double* s = src;
  if (!is_device_ptr(src)) {
    CK(cudaMemcpyAsync(scratch_e_[2], src, sizeof(double) * lay_.neta, cudaMemcpyHostToDevice, st_));
    s = scratch_e_[2];
  }
  launch_gather(int(lay_.neta), perm_eta_, s, dst, st_);
}
void Engine::from_internal_eta(const double* src, double* dst) {
  if (perm_identity_) {
    CK(cudaMemcpyAsync(dst, src, sizeof(double) * lay_.neta, cudaMemcpyDefault, st_));
    return;
  }
  if (is_device_ptr(dst)) {
    launch_scatter(int(lay_.neta), perm_eta_, src, dst, st_);
  } else {
    launch_scatter(int(lay_.neta), perm_eta_, src, scratch_e_[2], st_);
    CK(cudaMemcpyAsync(dst, scratch_e_[2], sizeof(double) * lay_.neta, cudaMemcpyDeviceToHost, st_));
  }
}
void Engine::copy_out(const double* src, double* dst, int64_t n) {
  CK(cudaMemcpyAsync(dst, src, sizeof(double) * n, cudaMemcpyDefault, st_));
}

void Engine::apply_T_b(const double* z, const double* eta, double* zo, double* eo) {
  double *iz = scratch_z_[0], *ie = scratch_e_[0], *oz = scratch_z_[1], *oe = scratch_e_[1];
  copy_in_z(z, iz);
  to_internal_eta(eta, ie);
  T(iz, ie, oz, oe);
  copy_out(oz, zo, lay_.nz);
  from_internal_eta(oe, eo);
  sync();
}
void Engine::apply_L_b(const double* z, double* eta) {
  copy_in_z(z, scratch_z_[0]);
  L(scratch_z_[0], scratch_e_[0]);
  from_internal_eta(scratch_e_[0], eta);
  sync();
}
void Engine::apply_Lt_b(const double* eta, double* z) {
  to_internal_eta(eta, scratch_e_[0]);
  Lt(scratch_e_[0], scratch_z_[0]);
  copy_out(scratch_z_[0], z, lay_.nz);
  sync();
}
double Engine::m_norm_b(const double* z, const double* eta, double alpha) {  // tree_operator.cpp:214-222
  copy_in_z(z, scratch_z_[0]);
  to_internal_eta(eta, scratch_e_[0]);
  L(scratch_z_[0], scratch_e_[1]);
  double r[3];
  dots({{scratch_z_[0], scratch_z_[0]}, {scratch_e_[0], scratch_e_[1]}, {scratch_e_[0], scratch_e_[0]}}, 0,
       {lay_.nz, lay_.neta, lay_.neta}, r);
  const double rad = r[0] - 2.0 * alpha * r[1] + r[2];
  if (rad < -1e-12 * std::max(1.0, r[0] + r[2]))
    throw std::runtime_error("m_norm: negative radicand (alpha violates alpha*||L|| < 1)");
  return std::sqrt(std::max(0.0, rad));
}
void Engine::proj_s1_b(double* z) {
  copy_in_z(z, scratch_z_[0]);
  launch_s1(D_, stage_start_.data(), scratch_z_[0], st_);
  copy_out(scratch_z_[0], z, lay_.nz);
  sync();
}
void Engine::proj_s2_b(double* z) {
  copy_in_z(z, scratch_z_[0]);
  launch_s2(D_, scratch_z_[0], st_);
  copy_out(scratch_z_[0], z, lay_.nz);
  sync();
}
void Engine::proj_s3_b(double* eta) {
  to_internal_eta(eta, scratch_e_[0]);
  launch_s3(D_, scratch_e_[0], st_);
  from_internal_eta(scratch_e_[0], eta);
  sync();
}
void Engine::unscale_b(const double* zs, double* z) {  // solver.cpp:116-130
  std::vector<double> h(lay_.nz);
  CK(cudaMemcpyAsync(h.data(), zs, sizeof(double) * lay_.nz, cudaMemcpyDefault, st_));
  sync();
  if (!pc_.is_identity) {
    const Tree& tr = p_.tree;
    for (int i = 0; i < tr.nn(); ++i) {
      const Vec& s = tr.leaf(i) ? pc_.sxN : pc_.sx;
      for (int k = 0; k < p_.nx; ++k) h[1 + size_t(i) * p_.nx + k] /= s[k];
      if (i < tr.nnl())
        for (int k = 0; k < p_.nu; ++k) h[lay_.u_base + size_t(i) * p_.nu + k] /= pc_.su[k];
    }
  }
  CK(cudaMemcpyAsync(z, h.data(), sizeof(double) * lay_.nz, cudaMemcpyDefault, st_));
  sync();
}

// ---------------------------------------------------------------------------
// CTA-resident loop for small trees (small.cuh): the whole solve in one CTA,
// operator phases separated by __syncthreads, the graph loop's controller on a
// shared-memory state.  Chosen when a CP application streams little enough
// that one SM's L1 holds the blocks (Engine::traffic <= kSmallBytes) and the
// per-stage operator kernels cover the shape.  SPOCK_SMALL=0 disables it,
// SPOCK_SMALL=1 forces it (tests).
bool Engine::small_eligible() const {
  const char* genv = std::getenv("SPOCK_SOLVE_GRAPH");  // 0: the host-driven loop (no device-resident loop)
  if (genv && genv[0] == '0') return false;
  if (prm_.cancelled || prm_.aa_memory > kLoopMaxMem) return false;
  return small_ok_ || cluster_ok_;
}

// Pointer fields of SmallArgs the cluster solve relocates into shared memory
// (f: the field, writable: copied back to HBM after the solve).
template <class F>
static void for_each_small_ptr(SmallArgs& A, int m, F&& f) {
  Dev& D = A.D;
  // (auto&: a reference to the pointer field itself, not to a converted temporary)
  auto c = [&](auto& p) { f(static_cast<const void**>(static_cast<void*>(&p)), false); };
  auto w = [&](auto& p) { f(static_cast<const void**>(static_cast<void*>(&p)), true); };
  c(D.anc), c(D.cf), c(D.cc), c(D.y_off), c(D.y_dim), c(D.s1_off), c(D.s1_nc), c(D.s1_ydim), c(D.s2_off);
  c(D.s2_dim), c(D.s3_off), c(D.s3_nc), c(D.s3_socdim), c(D.px), c(D.pu), c(D.hx_off), c(D.hu_off), c(D.Hx);
  c(D.HxT), c(D.Hu), c(D.HuT), c(D.qk), c(D.a_off), c(D.a), c(D.pN), c(D.hn_off), c(D.HN), c(D.HNT), c(D.qkN);
  c(D.aN_off), c(D.aN), c(D.gd), c(D.g_off), c(D.Gx), c(D.Gu), c(D.GxT), c(D.GuT), c(D.lo), c(D.hi), c(D.gNd);
  c(D.gN_off), c(D.GN), c(D.GNT), c(D.loN), c(D.hiN), c(D.rb), c(D.yc_nonneg), c(D.yc_poff), c(D.yc_kind);
  c(D.yc_dim), c(D.s2_kind), c(D.s2_gamma), c(D.s2p_off), c(D.s2P), c(D.M1), c(D.M1T), c(D.cvec), c(D.K);
  c(D.KT), c(D.Rinv), c(D.g), c(D.h), c(D.xinit);
  w(D.T12), w(D.adj), w(D.dvec);
  c(A.stage_start), c(A.d1), c(A.d2);
  w(A.TC), w(A.PV), w(A.Lrz), w(A.cLrz), w(A.Lsre), w(A.tmpz), w(A.tmpe);
  LoopArgs& L = A.L;
  w(L.V), w(L.TV), w(L.R), w(L.C), w(L.CR), w(L.PSI);
  for (int j = 0; j <= m; ++j) w(L.RH[j]);
  for (int j = 0; j < m; ++j) w(L.DH[j]);
}

// Pack the small loop's device image into the shared memory of a cluster of C
// CTAs.  CTA c owns the contiguous node range [own[c], own[c+1]) and runs every
// operator phase for those nodes, so each node-indexed block array (H, M1, K,
// R~^-1, translations, boxes, ...) is split: CTA c holds the slice of its nodes
// in its own shared memory and its pointer is rebased onto that slice (local
// latency).  Small read-only tables (tree, layouts, offsets) are replicated in
// every CTA; everything else -- iterates, history rings, the child-to-parent
// scratch -- is placed whole (largest first, least-filled CTA) and reached
// through DSMEM by the other CTAs.  False: does not fit.
bool Engine::cluster_plan(int m) {
  if (cplace_d_ && cplan_m_ == m) return true;
  SmallArgs A = small_;
  int dev = 0, smem_optin = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const int cap = ((smem_optin - cluster_static_smem() - 1024) / 16) * 16;
  if (cap <= 0) return false;
  const Tree& tr = p_.tree;
  const int nn = tr.nn(), nnl = tr.nnl(), nx = p_.nx, nu = p_.nu;
  const int64_t mm = nx + nu;
  using Span = std::pair<int64_t, int64_t>;  // (first element, count) of node i's block; count 0: none
  std::map<uintptr_t, std::function<Span(int)>> split;
  auto sp = [&](const double* base, std::function<Span(int)> f) {
    if (base) split[reinterpret_cast<uintptr_t>(base)] = std::move(f);
  };
  auto nr_ = [&](int i, auto f) -> Span { return i > 0 ? f(i - 1) : Span{0, 0}; };
  auto nl_ = [&](int i, auto f) -> Span { return i < nnl ? f(i) : Span{0, 0}; };
  auto lf_ = [&](int i, auto f) -> Span { return i >= nnl ? f(i - nnl) : Span{0, 0}; };
  const Dev& D = D_;
  const auto& px = soc_.stage;
  sp(D.Hx, [&](int i) { return nr_(i, [&](int k) { return Span{hxo_[k], pad2(int64_t(px[k].px) * nx)}; }); });
  sp(D.HxT, [&](int i) { return nr_(i, [&](int k) { return Span{hxo_[k], pad2(int64_t(px[k].px) * nx)}; }); });
  sp(D.Hu, [&](int i) { return nr_(i, [&](int k) { return Span{huo_[k], pad2(int64_t(px[k].pu) * nu)}; }); });
  sp(D.HuT, [&](int i) { return nr_(i, [&](int k) { return Span{huo_[k], pad2(int64_t(px[k].pu) * nu)}; }); });
  sp(D.qk, [&](int i) { return nr_(i, [&](int k) { return Span{k * mm, mm}; }); });
  sp(D.a, [&](int i) { return nr_(i, [&](int k) { return Span{ao_[k], px[k].px + px[k].pu + 2}; }); });
  sp(D.M1, [&](int i) { return nr_(i, [&](int k) { return Span{k * D.m1_stride, D.m1_stride}; }); });
  sp(D.M1T, [&](int i) { return nr_(i, [&](int k) { return Span{k * D.m1_stride, D.m1_stride}; }); });
  sp(D.cvec, [&](int i) { return nr_(i, [&](int k) { return Span{int64_t(k) * nx, nx}; }); });
  sp(D.HN, [&](int i) { return lf_(i, [&](int j) { return Span{hno_[j], pad2(int64_t(soc_.leaf[j].px) * nx)}; }); });
  sp(D.HNT, [&](int i) { return lf_(i, [&](int j) { return Span{hno_[j], pad2(int64_t(soc_.leaf[j].px) * nx)}; }); });
  sp(D.qkN, [&](int i) { return lf_(i, [&](int j) { return Span{int64_t(j) * nx, nx}; }); });
  sp(D.aN, [&](int i) { return lf_(i, [&](int j) { return Span{aNo_[j], soc_.leaf[j].px + 2}; }); });
  sp(D.gNd, [&](int i) { return lf_(i, [&](int j) { return Span{int64_t(j) * nx, nx}; }); });
  sp(D.GN, [&](int i) { return lf_(i, [&](int j) { return Span{p_.gN_off[j] * nx, int64_t(p_.ncN[j]) * nx}; }); });
  sp(D.GNT, [&](int i) { return lf_(i, [&](int j) { return Span{p_.gN_off[j] * nx, int64_t(p_.ncN[j]) * nx}; }); });
  sp(D.loN, [&](int i) { return lf_(i, [&](int j) { return Span{p_.gN_off[j], p_.ncN[j]}; }); });
  sp(D.hiN, [&](int i) { return lf_(i, [&](int j) { return Span{p_.gN_off[j], p_.ncN[j]}; }); });
  sp(D.gd, [&](int i) { return nl_(i, [&](int q) { return Span{q * mm, mm}; }); });
  sp(D.Gx, [&](int i) { return nl_(i, [&](int q) { return Span{p_.g_off[q] * nx, int64_t(p_.nc[q]) * nx}; }); });
  sp(D.GxT, [&](int i) { return nl_(i, [&](int q) { return Span{p_.g_off[q] * nx, int64_t(p_.nc[q]) * nx}; }); });
  sp(D.Gu, [&](int i) { return nl_(i, [&](int q) { return Span{p_.g_off[q] * nu, int64_t(p_.nc[q]) * nu}; }); });
  sp(D.GuT, [&](int i) { return nl_(i, [&](int q) { return Span{p_.g_off[q] * nu, int64_t(p_.nc[q]) * nu}; }); });
  sp(D.lo, [&](int i) { return nl_(i, [&](int q) { return Span{p_.g_off[q], p_.nc[q]}; }); });
  sp(D.hi, [&](int i) { return nl_(i, [&](int q) { return Span{p_.g_off[q], p_.nc[q]}; }); });
  sp(D.K, [&](int i) { return nl_(i, [&](int q) { return Span{q * D.k_stride, D.k_stride}; }); });
  sp(D.KT, [&](int i) { return nl_(i, [&](int q) { return Span{q * D.k_stride, D.k_stride}; }); });
  sp(D.Rinv, [&](int i) { return nl_(i, [&](int q) { return Span{q * D.r_stride, D.r_stride}; }); });
  sp(D.g, [&](int i) { return nl_(i, [&](int q) { return Span{int64_t(q) * nu, nu}; }); });
  sp(D.h, [&](int i) { return nl_(i, [&](int q) { return Span{int64_t(q) * nx, nx}; }); });
  sp(D.rb, [&](int i) {
    return nl_(i, [&](int q) { return Span{int64_t(lay_.y_off[q]) - D.y_base, lay_.y_dim[q]}; });
  });
  // every pointer field: allocation, delta, writable
  struct Fld {
    int field;
    uintptr_t ptr, base;
    size_t abytes;
    bool wr;
  };
  std::vector<Fld> flds;
  bool ok = true;
  for_each_small_ptr(A, m, [&](const void** f, bool wr) {
    const uintptr_t p = reinterpret_cast<uintptr_t>(*f);
    if (!p || !ok) return;
    auto it = alloc_bytes_.upper_bound(p);
    if (it == alloc_bytes_.begin() || p >= std::prev(it)->first + std::prev(it)->second) {
      ok = false;
      return;
    }
    --it;
    flds.push_back(Fld{int(reinterpret_cast<const char*>(f) - reinterpret_cast<const char*>(&A)), p, it->first,
                       it->second, wr});
  });
  if (!ok) return false;
  const char* ce = std::getenv("SPOCK_CLUSTER_CTAS");
  // smallest cluster tried: 8 CTAs (c1: CP 64 vs 67 us and SuperMann 199 vs
  // 216 us per iteration at 4; 2-3 CTAs 80 us; tools/c1_cluster_ctas.py)
  int want = ce && ce[0] ? std::atoi(ce) : 8;
  want = std::max(1, std::min(kClusterMax, want));
  for (int C = want; C <= kClusterMax; ++C) {
    std::vector<int> own(size_t(C) + 1);
    for (int c = 0; c <= C; ++c) own[c] = int(int64_t(nn) * c / C);
    std::vector<size_t> used(size_t(C), 0);
    std::vector<ClusterPlace> pl;
    std::vector<ClusterField> fl;
    bool fits = true;
    auto put = [&](int c, uintptr_t src, size_t bytes, bool wr) -> int {  // -> placement index (16-aligned)
      size_t off = (used[c] + 15) & ~size_t(15);
      off += src & 15;  // keep the 16-byte phase of the source (8-byte granules)
      if (off + bytes > size_t(cap)) {
        fits = false;
        return -1;
      }
      used[c] = off + bytes;
      // whole 8-byte granules inside the allocation (every dalloc allocation
      // carries two spare elements, so the last data element is covered)
      pl.push_back(ClusterPlace{reinterpret_cast<const char*>(src), int64_t(bytes & ~size_t(7)), c, int(off),
                                wr ? 1 : 0, 0});
      return int(pl.size()) - 1;
    };
    // 1. split block arrays: each CTA's node slice
    std::map<uintptr_t, bool> done;
    for (const Fld& F : flds) {
      auto sit = split.find(F.ptr);
      if (sit == split.end() || F.wr) continue;
      for (int c = 0; c < C && fits; ++c) {
        int64_t lo = INT64_MAX, hi = -1;
        for (int i = own[c]; i < own[c + 1]; ++i) {
          const Span s2 = sit->second(i);
          if (s2.second <= 0) continue;
          lo = std::min(lo, s2.first);
          hi = std::max(hi, s2.first + s2.second);
        }
        if (hi < 0) continue;  // no node of this CTA has a block here: never dereferenced by it
        const int pi = put(c, F.ptr + uintptr_t(lo) * 8, size_t(hi - lo) * 8, false);
        if (pi >= 0) fl.push_back(ClusterField{F.field, pi, -lo * 8, c});
      }
      done[F.ptr] = true;
    }
    // 2. small read-only tables: replicated
    for (const Fld& F : flds) {
      if (done.count(F.ptr) || F.wr || F.abytes > 16384) continue;
      for (int c = 0; c < C && fits; ++c) {
        const int pi = put(c, F.base, F.abytes, false);
        if (pi >= 0) fl.push_back(ClusterField{F.field, pi, int64_t(F.ptr - F.base), c});
      }
    }
    // 3. the rest: whole allocations, largest first, least-filled CTA
    std::map<uintptr_t, int> whole;  // allocation base -> placement
    std::vector<const Fld*> rest;
    for (const Fld& F : flds)
      if (!(done.count(F.ptr) && !F.wr) && (F.wr || F.abytes > 16384)) rest.push_back(&F);
    std::vector<uintptr_t> bases;
    std::map<uintptr_t, std::pair<size_t, bool>> abyte;
    for (const Fld* F : rest) {
      auto& e = abyte[F->base];
      e.first = F->abytes;
      e.second = e.second || F->wr;
    }
    for (auto& kv : abyte) bases.push_back(kv.first);
    std::sort(bases.begin(), bases.end(), [&](uintptr_t x, uintptr_t y) { return abyte[x].first > abyte[y].first; });
    for (uintptr_t b : bases) {
      if (!fits) break;
      int best = 0;
      for (int c = 1; c < C; ++c)
        if (used[c] < used[best]) best = c;
      whole[b] = put(best, b, abyte[b].first, abyte[b].second);
    }
    for (const Fld* F : rest)
      if (fits && whole.count(F->base)) fl.push_back(ClusterField{F->field, whole[F->base], int64_t(F->ptr - F->base), -1});
    if (!fits) continue;
    size_t arena = 16;
    for (size_t u : used) arena = std::max(arena, (u + 15) & ~size_t(15));
    if (cluster_max_active(C, int(arena)) < 1) continue;  // the device cannot co-schedule this cluster
    cplace_d_ = dupload(pl);
    cfield_d_ = dupload(fl);
    cplace_n_ = int(pl.size());
    cfield_n_ = int(fl.size());
    cluster_ctas_ = C;
    cluster_arena_ = int(arena);
    cown_.assign(own.begin(), own.end());
    cplan_m_ = m;
    CK(cudaStreamSynchronize(st_));
    if (std::getenv("SPOCK_DEBUG_SETUP"))
      std::fprintf(stderr, "[cluster] ctas %d arena %zu B placements %d fields %d\n", C, arena, cplace_n_, cfield_n_);
    return true;
  }
  return false;
}

const char* Engine::loop_path() const {
  if (shard_.on && shard_coll_on()) return "host";
  if (small_eligible()) return cluster_ok_ ? "cluster" : "small";
  const char* env = std::getenv("SPOCK_SOLVE_GRAPH");
  if (prm_.cancelled || prm_.aa_memory > kLoopMaxMem || (env && env[0] == '0')) return "host";
  return "graph";
}

void Engine::small_alloc() {
  SmallArgs& A = small_;
  if (A.L.V) return;  // buffers, built once per engine
  const int64_t nz = lay_.nz, ne = lay_.neta, nv = nz + ne;
  auto pair = [&]() { return dalloc<double>(size_t(nv)); };
  A.L.V = pair(), A.L.TV = pair(), A.L.R = pair(), A.L.C = pair(), A.L.CR = pair(), A.L.PSI = pair();
  A.TC = pair(), A.PV = pair();
  A.Lrz = dalloc<double>(size_t(ne));
  A.cLrz = dalloc<double>(size_t(ne));
  A.Lsre = dalloc<double>(size_t(nz));
  A.tmpz = dalloc<double>(size_t(nz));
  A.tmpe = dalloc<double>(size_t(ne));
  for (int j = 0; j < kLoopMaxMem + 1; ++j) A.L.RH[j] = pair();
  for (int j = 0; j < kLoopMaxMem; ++j) A.L.DH[j] = pair();
  A.L.st = dalloc<LoopState>(1);
  A.stage_start = dupload(stage_start_);
  A.D = D_;
  A.d1 = d1_;
  A.d2 = d2_;
  small_cap_ = 0;
}

bool Engine::solve_small(const double* x_init, const double* wz, const double* we, double* oz, double* ozs,
                         double* oe, bool supermann, Status& st) {
  if (!small_eligible()) return false;
  const int m = prm_.aa_memory;
  const int64_t nz = lay_.nz, ne = lay_.neta, nv = nz + ne;
  set_xinit(x_init ? x_init : raw_xinit_.data());
  SmallArgs& A = small_;
  small_alloc();
  const int cap = prm_.max_iters + 2;
  if (small_cap_ < cap) {
    A.L.rnorm = dalloc<double>(size_t(cap));
    A.L.branch = dalloc<char>(size_t(cap));
    small_cap_ = cap;
  }
  A.L.P = LoopParams{prm_.eps_abs, prm_.eps_rel, prm_.c0, prm_.c1, prm_.c2, prm_.beta, prm_.sigma, prm_.lambda,
                     alpha_, prm_.max_iters, prm_.max_backtracks, m, supermann ? 1 : 0};
  A.L.cap = cap;
  A.L.nz = nz;
  A.L.nv = nv;
  A.D = D_;
  A.d1 = d1_;
  A.d2 = d2_;
  A.supermann = supermann ? 1 : 0;
  double* V = A.L.V;
  CK(cudaMemsetAsync(V, 0, sizeof(double) * nv, st_));
  if (wz || we) {
    if (!wz || !we) throw std::invalid_argument("solve: warm start has wrong dimensions");
    copy_in_z(wz, V);
    to_internal_eta(we, V + nz);
  }
  LoopState S0{};
  S0.reason = -1;
  S0.n_T = 1;
  S0.n_L = 1;
  S0.k_stop = prm_.max_iters + 1;
  CK(cudaMemcpyAsync(A.L.st, &S0, sizeof(S0), cudaMemcpyHostToDevice, st_));
  const char* pe = std::getenv("SPOCK_SMALL_PROF");
  if (pe && pe[0] == '1' && !A.prof) {
    A.prof = dalloc<unsigned long long>(8);
  }
  small_solved_ = true;
  if (cluster_ok_) {
    if (!cluster_plan(m)) return false;  // (cannot happen after a successful plan at construction)
    ClusterArgs CA{};
    CA.S = A;
    CA.place = cplace_d_;
    CA.nplace = cplace_n_;
    CA.field = cfield_d_;
    CA.nfield = cfield_n_;
    for (int c = 0; c <= cluster_ctas_; ++c) CA.own[c] = cown_[c];
    CK(launch_cluster_solve(CA, cluster_ctas_, cluster_arena_, st_));
  } else {
    launch_small_solve(A, st_);
  }
  CK(cudaGetLastError());
  if (A.prof) {
    unsigned long long h[8];
    CK(cudaMemcpyAsync(h, A.prof, sizeof(h), cudaMemcpyDeviceToHost, st_));
    CK(cudaStreamSynchronize(st_));
    std::fprintf(stderr, "[small prof] cycles T %llu L %llu L* %llu red %llu gram %llu ctl %llu vec %llu other %llu\n",
                 h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
  }
  LoopState Sh{};
  CK(cudaMemcpyAsync(&Sh, A.L.st, sizeof(Sh), cudaMemcpyDeviceToHost, st_));
  CK(cudaStreamSynchronize(st_));
  if (Sh.reason == -2) throw std::runtime_error("spock: negative M-norm radicand (alpha too large)");
  const int iters = Sh.k;
  std::vector<double> rn(size_t(std::max(iters, 1)));
  std::vector<char> br(size_t(std::max(iters, 1)));
  if (iters > 0) {
    CK(cudaMemcpy(rn.data(), A.L.rnorm, sizeof(double) * iters, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(br.data(), A.L.branch, size_t(iters), cudaMemcpyDeviceToHost));
  }
  st.iterations = iters;
  st.reason = Sh.reason < 0 ? SPOCK_MAX_ITERS : Sh.reason;
  st.xi1 = Sh.xi1;
  st.xi2 = Sh.xi2;
  st.k0 = Sh.k0, st.k1 = Sh.k1, st.k2 = Sh.k2, st.stalled = Sh.stalled;
  st.n_T = Sh.n_T, st.n_L = Sh.n_L, st.n_Lt = Sh.n_Lt;
  st.rnorm.assign(rn.begin(), rn.begin() + iters);
  st.branches.assign(br.begin(), br.begin() + iters);
  if (prm_.progress)  // replayed after the kernel (as for the graph loop)
    for (int k = 0; k < iters; ++k) prm_.progress(k, rn[k], br[k]);
  if (ozs) copy_out(A.L.TV, ozs, nz);
  if (oe) from_internal_eta(A.L.TV + nz, oe);
  sync();
  if (oz) unscale_b(A.L.TV, oz);
  return true;
}

// ---------------------------------------------------------------------------
// Device-resident loop (loop.cu): one CUDA graph per solve.
//   WHILE(h_loop) {
//     L*(r_eta), xi norms, [history push, Gram]      -> k_begin (termination,
//     Anderson coefficients, branch) -> [psi]
//     SWITCH(h_sw) { 0: done | 1: K0 v += psi | 2: M psi, WHILE(h_ls) { trial
//       v + tau psi, refresh, dots, k_ls }, SWITCH(h_act) { K1 copies | K2 |
//       KM } | 3: CP v <- T v }
//     IF(h_ref) { refresh(v), M-norm dots }
//     k_end (branch record, counters, loop condition)
//   }
// The host only launches the graph (in chunks of iterations) and reads the
// state back; the arithmetic is the host loop's (solve_b) kernel for kernel.
bool Engine::solve_graph(const double* x_init, const double* wz, const double* we, double* oz, double* ozs,
                         double* oe, bool supermann, Status& st) {
  const int m = prm_.aa_memory;
  if (prm_.cancelled || m > kLoopMaxMem) return false;
  const char* env = std::getenv("SPOCK_SOLVE_GRAPH");
  if (env && env[0] == '0') return false;
  const int64_t nz = lay_.nz, ne = lay_.neta, nv = nz + ne;
  set_xinit(x_init ? x_init : raw_xinit_.data());
  GraphLoop& G = gloop_[supermann ? 1 : 0];
  if (!G.exec) build_loop_graph(G, supermann);
  const LoopArgs& A = G.A;
  double *V = A.V, *TV = A.TV, *R = A.R;
  CK(cudaMemsetAsync(V, 0, sizeof(double) * nv, st_));
  if (wz || we) {
    if (!wz || !we) throw std::invalid_argument("solve: warm start has wrong dimensions");
    copy_in_z(wz, V);
    to_internal_eta(we, V + nz);
  }
  // prologue (solver.cpp:211-235): r = v - T v and its M-norm dots
  T(V, V + nz, TV, TV + nz);
  launch_axpby(int(nv), 1.0, V, -1.0, TV, R, st_);
  L(R, G.Lrz);
  {
    DotArgs D{};
    D.x[0] = R, D.y[0] = R, D.n[0] = int(nz);
    D.x[1] = R + nz, D.y[1] = G.Lrz, D.n[1] = int(ne);
    D.x[2] = R + nz, D.y[2] = R + nz, D.n[2] = int(ne);
    D.ndots = 3;
    launch_dots(D, partial_, red_out_, st_);
  }
  LoopState S0{};
  S0.reason = -1;
  S0.n_T = 1;
  S0.n_L = 1;
  S0.k_stop = prm_.max_iters + 1;
  CK(cudaMemcpyAsync(A.st, &S0, sizeof(S0), cudaMemcpyHostToDevice, st_));
  CK(cudaGraphLaunch(G.exec, st_));
  LoopState Sh{};
  CK(cudaMemcpyAsync(&Sh, A.st, sizeof(Sh), cudaMemcpyDeviceToHost, st_));
  CK(cudaStreamSynchronize(st_));
  if (Sh.reason == -2) throw std::runtime_error("spock: negative M-norm radicand (alpha too large)");
  const int iters = Sh.k;
  std::vector<double> rn(size_t(std::max(iters, 1)));
  std::vector<char> br(size_t(std::max(iters, 1)));
  if (iters > 0) {
    CK(cudaMemcpy(rn.data(), A.rnorm, sizeof(double) * iters, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(br.data(), A.branch, size_t(iters), cudaMemcpyDeviceToHost));
  }
  st.iterations = iters;
  st.reason = Sh.reason < 0 ? SPOCK_MAX_ITERS : Sh.reason;
  st.xi1 = Sh.xi1;
  st.xi2 = Sh.xi2;
  st.k0 = Sh.k0, st.k1 = Sh.k1, st.k2 = Sh.k2, st.stalled = Sh.stalled;
  st.n_T = Sh.n_T, st.n_L = Sh.n_L, st.n_Lt = Sh.n_Lt;
  st.rnorm.assign(rn.begin(), rn.begin() + iters);
  st.branches.assign(br.begin(), br.begin() + iters);
  if (prm_.progress)  // replayed after the graph (the one behavioural difference)
    for (int k = 0; k < iters; ++k) prm_.progress(k, rn[k], br[k]);
  if (ozs) copy_out(TV, ozs, nz);
  if (oe) from_internal_eta(TV + nz, oe);
  sync();
  if (oz) unscale_b(TV, oz);
  return true;
}

// Buffers and the instantiated graph of the device-resident loop, built on the
// first solve of each kind (SuperMann / CP) and reused: pointers are baked in.
void Engine::build_loop_graph(GraphLoop& G, bool supermann) {
  const int m = prm_.aa_memory;
  const int64_t nz = lay_.nz, ne = lay_.neta, nv = nz + ne;
  auto pair = [&]() { return dalloc<double>(size_t(nv)); };
  LoopArgs& A = G.A;
  A = LoopArgs{};
  double *V = pair(), *TV = pair(), *R = pair(), *C = pair(), *TC = pair(), *CR = pair(), *PV = pair(),
         *PSI = pair();
  double* Lrz = dalloc<double>(size_t(ne));
  double* cLrz = dalloc<double>(size_t(ne));
  double* Lsre = dalloc<double>(size_t(nz));
  double* tmpz = dalloc<double>(size_t(nz));
  double* tmpe = dalloc<double>(size_t(ne));
  G.Lrz = Lrz;
  for (int j = 0; j < m + 1 && supermann; ++j) A.RH[j] = pair();
  for (int j = 0; j < m && supermann; ++j) A.DH[j] = pair();
  const int cap = prm_.max_iters + 2;
  A.rnorm = dalloc<double>(size_t(cap));
  A.branch = dalloc<char>(size_t(cap));
  A.st = dalloc<LoopState>(1);
  const double alpha = alpha_;
  A.P = LoopParams{prm_.eps_abs, prm_.eps_rel, prm_.c0, prm_.c1, prm_.c2, prm_.beta, prm_.sigma, prm_.lambda,
                   alpha, prm_.max_iters, prm_.max_backtracks, m, supermann ? 1 : 0};
  A.red = red_out_;
  A.cap = cap;
  A.nz = nz;
  A.nv = nv;
  A.V = V, A.TV = TV, A.R = R, A.C = C, A.CR = CR, A.PSI = PSI;
  auto refresh = [&](const double* v, double* tv, double* r, double* lrz) {  // T, r = v - Tv, L rz
    T(v, v + nz, tv, tv + nz);
    launch_axpby(int(nv), 1.0, v, -1.0, tv, r, st_);
    L(r, lrz);
  };
  auto mnorm = [&](const double* r, const double* lrz) {
    DotArgs D{};
    D.x[0] = r, D.y[0] = r, D.n[0] = int(nz);
    D.x[1] = r + nz, D.y[1] = lrz, D.n[1] = int(ne);
    D.x[2] = r + nz, D.y[2] = r + nz, D.n[2] = int(ne);
    D.ndots = 3;
    launch_dots(D, partial_, red_out_, st_);
  };
  std::vector<cudaGraph_t> owned;
  auto capture = [&](auto&& f) {
    cudaGraph_t c;
    CK(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal));
    f();
    CK(cudaStreamEndCapture(st_, &c));
    owned.push_back(c);
    return c;
  };
  auto child = [&](cudaGraph_t parent, cudaGraph_t c, cudaGraphNode_t dep) {
    cudaGraphNode_t n;
    CK(cudaGraphAddChildGraphNode(&n, parent, dep ? &dep : nullptr, dep ? 1 : 0, c));
    return n;
  };
  auto cond = [&](cudaGraph_t parent, cudaGraphConditionalHandle h, cudaGraphConditionalNodeType type,
                  unsigned size, cudaGraphNode_t dep, cudaGraph_t* bodies) {
    cudaGraphNodeParams np{};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = type;
    np.conditional.size = size;
    cudaGraphNode_t n;
    CK(cudaGraphAddNode(&n, parent, dep ? &dep : nullptr, dep ? 1 : 0, &np));
    for (unsigned k = 0; k < size; ++k) bodies[k] = np.conditional.phGraph_out[k];
    return n;
  };
  cudaGraph_t g;
  CK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h_loop, h_sw, h_ls, h_act, h_ref;
  CK(cudaGraphConditionalHandleCreate(&h_loop, g, 1, cudaGraphCondAssignDefault));
  cudaGraph_t body;
  cond(g, h_loop, cudaGraphCondTypeWhile, 1, nullptr, &body);
  // handles live on the graph that holds their node; the kernels that set a
  // handle are captured after it exists (A is copied into their arguments)
  CK(cudaGraphConditionalHandleCreate(&h_sw, body, 0, cudaGraphCondAssignDefault));
  CK(cudaGraphConditionalHandleCreate(&h_ref, body, 0, cudaGraphCondAssignDefault));
  A.h_loop = (unsigned long long)h_loop;
  A.h_sw = (unsigned long long)h_sw;
  A.h_ref = (unsigned long long)h_ref;
  cudaGraph_t gtop = capture([&] {
    Lt(R + nz, Lsre);
    XiArgs X{};
    X.x[0] = R, X.y[0] = Lsre, X.d[0] = d1_, X.n[0] = int(nz);
    X.x[1] = R + nz, X.y[1] = Lrz, X.d[1] = d2_, X.n[1] = int(ne);
    X.alpha = alpha;
    launch_xi(X, partial_ + kRedRegion, red_out_ + 4, st_);
    if (supermann) {  // history push, Gram update and the controller in one launch
      loop_gram(A, gram_partial_, red_out_ + 8, st_);
    } else {
      loop_begin(A, st_);
    }
    if (supermann) loop_psi(A, st_);
  });
  cudaGraphNode_t n_top = child(body, gtop, nullptr);
  cudaGraph_t sw[4];
  cudaGraphNode_t n_sw = cond(body, h_sw, cudaGraphCondTypeSwitch, 4, n_top, sw);
  CK(cudaGraphConditionalHandleCreate(&h_ls, sw[2], 0, cudaGraphCondAssignDefault));
  CK(cudaGraphConditionalHandleCreate(&h_act, sw[2], 0, cudaGraphCondAssignDefault));
  A.h_ls = (unsigned long long)h_ls;
  A.h_act = (unsigned long long)h_act;
  // case 1 (K0): v += psi
  child(sw[1], capture([&] { launch_axpby(int(nv), 1.0, V, 1.0, PSI, V, st_); }), nullptr);
  // case 2: M psi, line search, K1 / K2 / KM
  {
    cudaGraph_t gm = capture([&] {
      loop_ls_init(A, st_);
      Lt(PSI + nz, tmpz);
      launch_axpby(int(nz), 1.0, PSI, -alpha, tmpz, PV, st_);
      L(PSI, tmpe);
      launch_axpby(int(ne), 1.0, PSI + nz, -alpha, tmpe, PV + nz, st_);
    });
    cudaGraphNode_t n_m = child(sw[2], gm, nullptr);
    cudaGraph_t lsb;
    cudaGraphNode_t n_ls = cond(sw[2], h_ls, cudaGraphCondTypeWhile, 1, n_m, &lsb);
    child(lsb, capture([&] {
            loop_axpy_tau(A, st_);
            refresh(C, TC, CR, cLrz);
            // the candidate's M-norm dots and <r~, M psi> in one launch: red[0..3), red[3..5)
            DotArgs D{};
            D.x[0] = CR, D.y[0] = CR, D.n[0] = int(nz);
            D.x[1] = CR + nz, D.y[1] = cLrz, D.n[1] = int(ne);
            D.x[2] = CR + nz, D.y[2] = CR + nz, D.n[2] = int(ne);
            D.x[3] = CR, D.y[3] = PV, D.n[3] = int(nz);
            D.x[4] = CR + nz, D.y[4] = PV + nz, D.n[4] = int(ne);
            D.ndots = 5;
            launch_dots(D, partial_, red_out_, st_);
            loop_ls(A, st_);
          }),
          nullptr);
    cudaGraph_t act[4];
    cond(sw[2], h_act, cudaGraphCondTypeSwitch, 4, n_ls, act);
    child(act[1], capture([&] {  // K1: the candidate becomes the iterate
            loop_copy(V, C, nv, st_);
            loop_copy(TV, TC, nv, st_);
            loop_copy(R, CR, nv, st_);
            loop_copy(Lrz, cLrz, ne, st_);
          }),
          nullptr);
    child(act[2], capture([&] { loop_k2(A, st_); }), nullptr);
    child(act[3], capture([&] { loop_copy(V, TV, nv, st_); }), nullptr);
  }
  // case 3 (CP): v <- T v
  child(sw[3], capture([&] { loop_copy(V, TV, nv, st_); }), nullptr);
  cudaGraph_t rb;
  cudaGraphNode_t n_ref = cond(body, h_ref, cudaGraphCondTypeIf, 1, n_sw, &rb);
  child(rb, capture([&] {
          refresh(V, TV, R, Lrz);
          mnorm(R, Lrz);
        }),
        nullptr);
  child(body, capture([&] { loop_end(A, st_); }), n_ref);
  CK(cudaGraphInstantiate(&G.exec, g, 0));
  for (cudaGraph_t c : owned) cudaGraphDestroy(c);
  cudaGraphDestroy(g);
}

// ---------------------------------------------------------------------------
// SuperMann / CP loop (proj/src/solver.cpp:189-350).  State lives on device;
// one host round trip per iteration (omega, xi norms and the Anderson Gram
// matrix come back together) plus one per line-search trial.
void Engine::solve_b(const double* x_init, const double* wz, const double* we, double* oz, double* ozs, double* oe,
                     bool supermann, Status& st) {
  // sharded solve: host-driven loop, T / L / L* over this rank's
  // items with the exchanges, every reduction over this rank's entries and
  // all-reduced (sums of dots, max of the xi norms) through the host's collectives
  const bool sharded = shard_.on && shard_coll_on();
  struct Flag {
    bool& f;
    ~Flag() { f = false; }
  } flag_guard{shard_solving_};
  shard_solving_ = sharded;
  const double* w_z = sharded ? shard_.wz : nullptr;
  const double* w_e = sharded ? shard_.we : nullptr;
  const double* w_v = sharded ? shard_.wv : nullptr;
  if (!sharded && solve_small(x_init, wz, we, oz, ozs, oe, supermann, st)) return;
  if (!sharded && solve_graph(x_init, wz, we, oz, ozs, oe, supermann, st)) return;
  const int64_t nz = lay_.nz, ne = lay_.neta, nv = nz + ne;
  set_xinit(x_init ? x_init : raw_xinit_.data());
  const int m = prm_.aa_memory;
  // pair buffers: [z | eta] contiguous so Anderson works on the stacked vector
  std::vector<double*> bufs;
  auto pair = [&]() {
    double* p = nullptr;
    CK(cudaMallocAsync(&p, sizeof(double) * (nv + 2), st_));
    bufs.push_back(p);
    return p;
  };
  double *V = pair(), *TV = pair(), *R = pair(), *C = pair(), *TC = pair(), *CR = pair(), *PV = pair(),
         *PSI = pair();
  double *Lrz = nullptr, *cLrz = nullptr, *Lsre = nullptr, *tmpz = nullptr, *tmpe = nullptr;
  CK(cudaMallocAsync(&Lrz, sizeof(double) * ne, st_));
  CK(cudaMallocAsync(&cLrz, sizeof(double) * ne, st_));
  CK(cudaMallocAsync(&Lsre, sizeof(double) * nz, st_));
  CK(cudaMallocAsync(&tmpz, sizeof(double) * nz, st_));
  CK(cudaMallocAsync(&tmpe, sizeof(double) * ne, st_));
  std::vector<double*> RH(m + 1), DH(m);  // residual / difference history, newest at index 0
  for (auto& p : RH) p = pair();
  for (auto& p : DH) p = pair();
  CK(cudaMemsetAsync(V, 0, sizeof(double) * nv, st_));
  if (wz || we) {
    if (!wz || !we) throw std::invalid_argument("solve: warm start has wrong dimensions");
    copy_in_z(wz, V);
    to_internal_eta(we, V + nz);
  }
  auto cleanup = [&]() {
    for (double* p : bufs) cudaFreeAsync(p, st_);
    cudaFreeAsync(Lrz, st_);
    cudaFreeAsync(cLrz, st_);
    cudaFreeAsync(Lsre, st_);
    cudaFreeAsync(tmpz, st_);
    cudaFreeAsync(tmpe, st_);
    cudaStreamSynchronize(st_);
  };
  const double alpha = alpha_;
  auto refresh = [&](const double* v, double* tv, double* r, double* lrz) {  // T, r = v - Tv, L rz
    T(v, v + nz, tv, tv + nz);
    ++st.n_T;
    launch_axpby(int(nv), 1.0, v, -1.0, tv, r, st_);
    L(r, lrz);
    ++st.n_L;
  };
  // queue the M-norm dots of (r, lrz) into red_out_[base..base+3)
  auto queue_mnorm = [&](const double* r, const double* lrz, int base) {
    DotArgs A{};
    A.x[0] = r, A.y[0] = r, A.n[0] = int(nz), A.w[0] = w_z;
    A.x[1] = r + nz, A.y[1] = lrz, A.n[1] = int(ne), A.w[1] = w_e;
    A.x[2] = r + nz, A.y[2] = r + nz, A.n[2] = int(ne), A.w[2] = w_e;
    A.ndots = 3;
    launch_dots(A, partial_, red_out_ + base, st_);
  };
  auto mnorm_of = [&](const double* h) {  // solver.cpp:166-174
    const double rad = h[0] - 2.0 * alpha * h[1] + h[2];
    if (rad < -1e-12 * std::max(1.0, h[0] + h[2]))
      throw std::runtime_error("spock: negative M-norm radicand (alpha too large)");
    return std::sqrt(std::max(0.0, rad));
  };
  auto fetch = [&](int n) {
    CK(cudaMemcpyAsync(host_red_, red_out_, sizeof(double) * n, cudaMemcpyDeviceToHost, st_));
    sync();
  };
  int aa_k = 0;  // Anderson call counter
  int aa_cols = 0;
  std::fill(gram_h_.begin(), gram_h_.end(), dd{0.0, 0.0});
  std::fill(gram_r_.begin(), gram_r_.end(), dd{0.0, 0.0});
  try {
    refresh(V, TV, R, Lrz);
    queue_mnorm(R, Lrz, 0);
    bool have_omega = false;
    double omega = 0.0, zeta = 0.0, omega_safe = 0.0, th1 = 0.0, th2 = 0.0;
    for (int k = 0;; ++k) {
      // xi residuals (solver.cpp:240-244)
      Lt(R + nz, Lsre);
      ++st.n_Lt;
      XiArgs X{};
      X.x[0] = R, X.y[0] = Lsre, X.d[0] = d1_, X.n[0] = int(nz);
      X.x[1] = R + nz, X.y[1] = Lrz, X.d[1] = d2_, X.n[1] = int(ne);
      X.alpha = alpha;
      if (sharded) X.w[0] = shard_.mz, X.w[1] = shard_.me;
      launch_xi(X, partial_ + kRedRegion, red_out_ + 4, st_);
      // Anderson push (solver.cpp:57-63) and the Gram update of the newest
      // difference in double-double (aa.cuh; Gram kept by history position)
      if (supermann) {
        std::rotate(RH.begin(), RH.end() - 1, RH.end());
        std::rotate(DH.begin(), DH.end() - 1, DH.end());
        CK(cudaMemcpyAsync(RH[0], R, sizeof(double) * nv, cudaMemcpyDeviceToDevice, st_));
        if (aa_k == 0)
          CK(cudaMemcpyAsync(DH[0], R, sizeof(double) * nv, cudaMemcpyDeviceToDevice, st_));
        else
          launch_axpby(int(nv), 1.0, RH[0], -1.0, RH[1], DH[0], st_);
        aa_cols = std::min(aa_cols + 1, m);
        for (int c0 = 0; c0 < aa_cols; c0 += kLoopMaxMem) {
          GramArgs A{};
          A.dnew = DH[0], A.r = R, A.w = w_v, A.n = nv;
          A.cols = std::min(kLoopMaxMem, aa_cols - c0);
          for (int b = 0; b < A.cols; ++b) A.D[b] = DH[c0 + b];
          launch_gram_dd(A, gram_partial_, gram_out_ + 4 * c0, st_);
        }
      }
      if (sharded) {  // this iteration's fresh partials, summed (max for xi) over the ranks
        if (!have_omega) coll(1, red_out_, 3);
        coll(2, red_out_ + 4, 2);
      }
      fetch(8);
      if (supermann) gram_update(aa_cols, sharded);
      if (!have_omega) {
        omega = mnorm_of(host_red_);
        have_omega = true;
        if (k == 0) zeta = omega_safe = omega;  // solver.cpp:233-235
      }
      const double n1 = host_red_[4], n2 = host_red_[5];
      if (k == 0) {
        th1 = std::max(prm_.eps_abs, prm_.eps_rel * n1);
        th2 = std::max(prm_.eps_abs, prm_.eps_rel * n2);
      }
      st.iterations = k;
      st.xi1 = n1;
      st.xi2 = n2;
      int reason = -1;
      if (!std::isfinite(n1) || !std::isfinite(n2) || !std::isfinite(omega))
        reason = SPOCK_STALLED;
      else if (n1 <= th1 && n2 <= th2)
        reason = SPOCK_CONVERGED;
      else if (k >= prm_.max_iters)
        reason = SPOCK_MAX_ITERS;
      else if (prm_.cancelled && (k % std::max(1, prm_.poll_every) == 0) && agree_cancel(prm_.cancelled()))
        reason = SPOCK_CANCELLED;
      if (reason >= 0) {
        st.reason = reason;
        if (ozs) copy_out(TV, ozs, nz);
        if (oe) from_internal_eta(TV + nz, oe);
        sync();
        if (oz) unscale_b(TV, oz);
        cleanup();
        return;
      }
      st.rnorm.push_back(omega);
      if (!supermann) {
        std::swap(V, TV);
        st.branches.push_back('K');
        if (prm_.progress) prm_.progress(k, omega, 'K');
        refresh(V, TV, R, Lrz);
        queue_mnorm(R, Lrz, 0);
        have_omega = false;
        continue;
      }
      // Anderson direction (solver.cpp:64-76)
      const int kk = aa_k++;
      if (kk <= m) {
        launch_axpby(int(nv), -1.0, R, 0.0, nullptr, PSI, st_);
      } else {
        // kappa = argmin ||M_d kappa - r|| by column-pivoted Cholesky of the
        // Gram matrix (the R factor of a column-pivoted QR of M_d)
        const int cols = aa_cols;
        std::vector<dd> G(size_t(cols) * cols);
        for (int a = 0; a < cols; ++a)
          for (int b = 0; b < cols; ++b) G[a + b * cols] = gram_h_[a + b * kAaHostMax];
        std::vector<double> kap(cols);
        aa_kappa_dd<kAaHostMax>(G.data(), gram_r_.data(), cols, nv, kap.data());
        // psi = -r - sum_j kappa_j (M_r - M_d)_j, (M_r - M_d)_j = r_{k-1-j} = RH[j+1]
        LinCombArgs A{};
        A.x[0] = R;
        A.c[0] = -1.0;
        for (int c = 0; c < cols; ++c) {
          A.x[c + 1] = RH[c + 1];
          A.c[c + 1] = -kap[c];
        }
        launch_lincomb(int(nv), cols + 1, A, PSI, st_);
      }
      char branch;
      bool carried = false;
      double omega_next = 0.0;
      if (omega <= prm_.c0 * zeta) {  // K0
        launch_axpby(int(nv), 1.0, V, 1.0, PSI, V, st_);
        zeta = omega;
        branch = '0';
        ++st.k0;
      } else {
        // M psi (solver.cpp:287-290)
        Lt(PSI + nz, tmpz);
        ++st.n_Lt;
        launch_axpby(int(nz), 1.0, PSI, -alpha, tmpz, PV, st_);
        L(PSI, tmpe);
        ++st.n_L;
        launch_axpby(int(ne), 1.0, PSI + nz, -alpha, tmpe, PV + nz, st_);
        double tau = 1.0;
        int backtracks = 0;
        for (;;) {
          launch_axpby(int(nv), 1.0, V, tau, PSI, C, st_);
          refresh(C, TC, CR, cLrz);
          queue_mnorm(CR, cLrz, 0);
          {
            DotArgs A{};
            A.x[0] = CR, A.y[0] = PV, A.n[0] = int(nz), A.w[0] = w_z;
            A.x[1] = CR + nz, A.y[1] = PV + nz, A.n[1] = int(ne), A.w[1] = w_e;
            A.ndots = 2;
            launch_dots(A, partial_ + 3 * kRedRegion, red_out_ + 3, st_);
          }
          if (sharded) coll(1, red_out_, 5);
          fetch(5);
          const double omt = mnorm_of(host_red_);
          if ((omega <= omega_safe && omt <= prm_.c1 * omega) || omt == 0.0) {  // K1
            std::swap(V, C);
            std::swap(TV, TC);
            std::swap(R, CR);
            std::swap(Lrz, cLrz);
            omega_safe = omt + std::pow(prm_.c2, k);
            branch = '1';
            ++st.k1;
            carried = true;
            omega_next = omt;
            break;
          }
          const double rho = omt * omt - tau * (host_red_[3] + host_red_[4]);
          if (rho >= prm_.sigma * omt * omega) {  // K2
            const double coef = prm_.lambda * rho / (omt * omt);
            launch_axpby(int(nv), 1.0, V, -coef, CR, V, st_);
            branch = '2';
            ++st.k2;
            break;
          }
          tau *= prm_.beta;
          if (++backtracks > prm_.max_backtracks) {  // KM fallback
            CK(cudaMemcpyAsync(V, TV, sizeof(double) * nv, cudaMemcpyDeviceToDevice, st_));
            branch = 'S';
            ++st.stalled;
            break;
          }
        }
      }
      st.branches.push_back(branch);
      if (prm_.progress) prm_.progress(k, omega, branch);
      if (carried) {
        omega = omega_next;
        have_omega = true;
      } else {
        refresh(V, TV, R, Lrz);
        queue_mnorm(R, Lrz, 0);
        have_omega = false;
      }
    }
  } catch (...) {
    cleanup();
    throw;
  }
}

// k back-to-back T applications on device-resident iterates (bench helper).
// With flush, a 256 MiB buffer is rewritten between applications (outside the
// per-application event pair) so no application reads the previous one's
// L2-resident data; the result is the sum of per-application device times.
void Engine::flush_l2() {
  const size_t n = size_t(256) << 20;
  if (!flush_buf_) flush_buf_ = dalloc<double>(n / sizeof(double));
  CK(cudaMemsetAsync(flush_buf_, int(0x5a), n, st_));
}

// SPOCK_FUSED_TRACE=<file>: one traced fused T (4 globaltimer stamps per item,
// int64 little endian) written to <file>; used by tools/trace_fused.py
static void dump_trace_if_requested(const FusedArgs& F0, int grid, cudaStream_t st, int nitems) {
  const char* path = std::getenv("SPOCK_FUSED_TRACE");
  if (!path || !path[0]) return;
  FusedArgs F = F0;
  unsigned long long* d = nullptr;
  CK(cudaMalloc(&d, sizeof(unsigned long long) * 8 * size_t(nitems)));
  CK(cudaMemsetAsync(d, 0, sizeof(unsigned long long) * 8 * size_t(nitems), st));
  F.trace = d;
  launch_T_fused(F, grid, st);
  std::vector<unsigned long long> h(8 * size_t(nitems));
  CK(cudaMemcpyAsync(h.data(), d, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  cudaFree(d);
  if (FILE* f = std::fopen(path, "wb")) {
    std::fwrite(h.data(), sizeof(unsigned long long), h.size(), f);
    std::fclose(f);
  }
}

double Engine::bench_T(int k, bool graph, bool flush) {
  double *z[2] = {scratch_z_[0], scratch_z_[1]}, *e[2] = {scratch_e_[0], scratch_e_[1]};
  CK(cudaMemsetAsync(z[0], 0, sizeof(double) * lay_.nz, st_));
  CK(cudaMemsetAsync(e[0], 0, sizeof(double) * lay_.neta, st_));
  if (fused_ok_ && std::getenv("SPOCK_FUSED_TRACE")) {
    FusedArgs F = fargs_;
    F.D = D_;
    F.z = z[0], F.eta = e[0], F.zo = z[1], F.eo = e[1], F.alpha = alpha_;
    F.base[FB_Z] = z[0];
    F.base[FB_ETA] = e[0];
    flush_l2();
    CK(cudaMemsetAsync(F.ticket, 0, fused_sync_bytes_, st_));
    dump_trace_if_requested(F, fused_grid_, st_, D_.nnl + 2 * D_.nn);
  }
  if (graph && !bench_graph_) {
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal));
    T(z[0], e[0], z[1], e[1]);
    T(z[1], e[1], z[0], e[0]);
    CK(cudaStreamEndCapture(st_, &g));
    CK(cudaGraphInstantiate(&bench_graph_, g, 0));
    cudaGraphDestroy(g);
  }
  std::vector<cudaEvent_t> ev(2 * ((k + 1) / 2) + 2);
  for (auto& x : ev) CK(cudaEventCreate(&x));
  const int pairs = (k + 1) / 2;
  double total = 0.0;
  if (flush) {
    for (int i = 0; i < pairs; ++i) {
      for (int h = 0; h < 2; ++h) {
        flush_l2();
        CK(cudaEventRecord(ev[2 * i + h], st_));
        T(z[h], e[h], z[1 - h], e[1 - h]);
        CK(cudaEventRecord(ev[ev.size() - 1], st_));
        CK(cudaEventSynchronize(ev[ev.size() - 1]));
        float ms = 0.0f;
        CK(cudaEventElapsedTime(&ms, ev[2 * i + h], ev[ev.size() - 1]));
        total += ms;
      }
    }
  } else {
    CK(cudaEventRecord(ev[0], st_));
    for (int i = 0; i < pairs; ++i) {
      if (graph) {
        CK(cudaGraphLaunch(bench_graph_, st_));
      } else {
        T(z[0], e[0], z[1], e[1]);
        T(z[1], e[1], z[0], e[0]);
      }
    }
    CK(cudaEventRecord(ev[1], st_));
    CK(cudaEventSynchronize(ev[1]));
    float ms = 0.0f;
    CK(cudaEventElapsedTime(&ms, ev[0], ev[1]));
    total = ms;
  }
  for (auto& x : ev) cudaEventDestroy(x);
  CK(cudaGetLastError());
  return total * double(k) / double(2 * pairs);
}

// average device ms per launch class over k repetitions:
// ms[0] L* (standalone), ms[1] S1 sweeps (per-stage path only), ms[2] S2,
// ms[3] L (standalone), ms[4] whole T (fused kernel or per-stage sequence)
void Engine::bench_kernels(int k, bool flush, double* ms) {
  double *z0 = scratch_z_[0], *e0 = scratch_e_[0], *z1 = scratch_z_[1], *e1 = scratch_e_[1];
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int c = 0; c < 5; ++c) ms[c] = 0.0;
  for (int i = 0; i < k; ++i) {
    for (int c = 0; c < 5; ++c) {
      if (c == 1 && fused_ok_) continue;
      if (flush) flush_l2();
      CK(cudaEventRecord(a, st_));
      switch (c) {
        case 0: Lt(e0, z1); break;
        case 1: launch_s1(D_, stage_start_.data(), z1, st_); break;
        case 2: launch_s2(D_, z1, st_); break;
        case 3: L(z0, e1); break;
        case 4: T(z0, e0, z1, e1); break;
      }
      CK(cudaEventRecord(b, st_));
      CK(cudaEventSynchronize(b));
      float t = 0.0f;
      CK(cudaEventElapsedTime(&t, a, b));
      ms[c] += t;
    }
  }
  for (int c = 0; c < 5; ++c) ms[c] /= std::max(k, 1);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  CK(cudaGetLastError());
}

// Algorithmic bytes per launch class (each operand read or written once per
// launch): [L*, S1 sweeps, S2, L, T].  T is the sum
// of the fused phases: L* matrices + S1 blocks + L matrices + every vector
// segment once (the dual update reads eta and the a/box data, writes eta+).
void Engine::traffic(double* out) const {
  const Tree& tr = p_.tree;
  const int nn = tr.nn(), nnl = tr.nnl(), nx = p_.nx, nu = p_.nu, m = nx + nu;
  double lt = 0, s1 = 0, s2 = 0, l = 0, dual = 0;
  for (int k = 0; k < nn - 1; ++k) {
    const int px = soc_.stage[k].px, pu = soc_.stage[k].pu, p = px + pu;
    const double H = double(px) * nx + double(pu) * nu;
    lt += H + m + (p + 2) + m + 1;            // H', qk, eta seg, adj out, tau out
    l += H + m + 2.0 * m + 1 + (p + 2);       // H, qk, (x,u)_anc, tau, eta seg out
    dual += 2.0 * (p + 2);                    // eta in (p+2) and translation a (p+2) of the dual update
    s1 += double(m) * nx + (nx + m)           // backward: M1', q in, T12 out
          + double(nx) * m + m + 2 * nx;      // forward: M1, (x,d)_anc, c, x out
  }
  for (int i = 0; i < nnl; ++i) {
    const int ny = lay_.y_dim[i], nc = p_.nc[i], nch = tr.child_count[i];
    const double g = D_.g_diag ? m : double(nc) * m;
    lt += (ny + 1 + nc) + ny + g + double(nch) * m + (m + ny + 1);  // eta seg, b, G, adj sums, z out
    l += ny + ny + g + m + 1 + (ny + 1 + nc);                          // y, b, G, (x,u), s, eta out
    dual += 2.0 * nc;                                                  // box lo/hi
    s1 += double(nx) * nu + nx + nu + double(nu) * nu + double(nch) * m + nu  // KT, h, g, Rinv, T12 sums, d
          + double(nu) * nx + nu + nu + nu;                                  // forward K, d, u out
    s2 += 2.0 * (ny + 2 * nch);
  }
  for (int j = 0; j < nn - nnl; ++j) {
    const int pN = soc_.leaf[j].px, nc = p_.ncN[j];
    const double g = D_.gN_diag ? nx : double(nc) * nx;
    lt += nc + g + double(pN) * nx + (pN + 2) + nx + (nx + 1);
    l += g + double(pN) * nx + nx + nx + 1 + (nc + pN + 2);
    dual += 2.0 * (pN + 2) + 2.0 * nc;
  }
  out[0] = 8.0 * lt;
  out[1] = 8.0 * s1;
  out[2] = 8.0 * s2;
  out[3] = 8.0 * l;
  out[4] = out[0] + out[1] + out[2] + out[3] + 8.0 * dual;
}

}  // namespace spock
