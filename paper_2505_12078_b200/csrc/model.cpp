// Host-side setup of the B200 SPOCK solver (see model.hpp for the reference map).
#include "model.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <limits>
#include <thread>
#include <unordered_map>

namespace spock {

namespace {
void require(bool c, const char* m) {
  if (!c) throw std::invalid_argument(m);
}
constexpr double kProbTol = 1e-12;

// Parallel loop over [0, n) on host threads (setup only; deterministic since
// every index writes its own slot).
void host_parallel(int64_t n, const std::function<void(int64_t)>& f) {
  int nt = int(std::thread::hardware_concurrency());
  nt = std::max(1, std::min<int>(nt, 32));
  if (n < 64 || nt == 1) {
    for (int64_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::vector<std::thread> th;
  const int64_t per = (n + nt - 1) / nt;
  for (int t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      for (int64_t i = t * per; i < std::min(n, (t + 1) * per); ++i) f(i);
    });
  for (auto& x : th) x.join();
}

uint64_t fnv(const void* p, size_t n, uint64_t h = 1469598103934665603ull) {
  const unsigned char* b = static_cast<const unsigned char*>(p);
  for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  return h;
}
}  // namespace

// ---------------------------------------------------------------------------
// Symmetric eigendecomposition: cyclic Jacobi with a decreasing rotation
// threshold; ascending eigenvalues (Eigen::SelfAdjointEigenSolver order, ties
// keep position order); every eigenvector's largest-|.| entry positive.
void sym_eig(const Mat& A0, Vec& w, Mat& V) {
  const int n = A0.r;
  std::vector<double> A(size_t(n) * n), U(size_t(n) * n, 0.0);
  auto a = [&](int i, int j) -> double& { return A[size_t(i) + size_t(j) * n]; };
  auto u = [&](int i, int j) -> double& { return U[size_t(i) + size_t(j) * n]; };
  for (int j = 0; j < n; ++j) {
    u(j, j) = 1.0;
    for (int i = 0; i < n; ++i) a(i, j) = 0.5 * (A0(i, j) + A0(j, i));
  }
  const double eps = std::numeric_limits<double>::epsilon();
  for (int sweep = 0; sweep < 100; ++sweep) {
    bool any = false;
    for (int p = 0; p < n - 1; ++p) {
      for (int q = p + 1; q < n; ++q) {
        const double apq = a(p, q);
        if (apq == 0.0) continue;
        const double app = a(p, p), aqq = a(q, q);
        const double small = eps * 1e-3;
        if (std::fabs(apq) <= small * std::sqrt(std::fabs(app) * std::fabs(aqq)) &&
            std::fabs(apq) <= 1e-300 + small * std::max(std::fabs(app), std::fabs(aqq))) {
          a(p, q) = a(q, p) = 0.0;
          continue;
        }
        any = true;
        const double th = (aqq - app) / (2.0 * apq);
        const double t = std::fabs(th) > 1e150 ? 0.5 / th
                                               : (th >= 0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {
          const double kp = a(k, p), kq = a(k, q);
          a(k, p) = c * kp - s * kq;
          a(k, q) = s * kp + c * kq;
        }
        for (int k = 0; k < n; ++k) {
          const double pk = a(p, k), qk = a(q, k);
          a(p, k) = c * pk - s * qk;
          a(q, k) = s * pk + c * qk;
        }
        a(p, q) = a(q, p) = 0.0;
        for (int k = 0; k < n; ++k) {
          const double kp = u(k, p), kq = u(k, q);
          u(k, p) = c * kp - s * kq;
          u(k, q) = s * kp + c * kq;
        }
      }
    }
    if (!any) break;
  }
  std::vector<int> ord(n);
  for (int i = 0; i < n; ++i) ord[i] = i;
  std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return a(x, x) < a(y, y); });
  w.resize(n);
  V = Mat(n, n);
  for (int k = 0; k < n; ++k) {
    const int o = ord[k];
    w[k] = a(o, o);
    int im = 0;
    for (int i = 1; i < n; ++i)
      if (std::fabs(u(i, o)) > std::fabs(u(im, o)) * (1.0 + 1e-12)) im = i;
    const double sg = u(im, o) < 0 ? -1.0 : 1.0;
    for (int i = 0; i < n; ++i) V(i, k) = sg * u(i, o);
  }
}

// ---------------------------------------------------------------------------
void Tree::finalize() {  // proj/src/tree.cpp:24-83
  const int n = nn();
  require(n > 0, "ScenarioTree: empty tree");
  require(anc[0] == -1, "ScenarioTree: node 0 must be the root");
  stage.assign(n, 0);
  for (int i = 1; i < n; ++i) {
    const int a = anc[i];
    require(a >= 0 && a < i, "ScenarioTree: ancestors must precede children");
    stage[i] = stage[a] + 1;
    require(stage[i] >= stage[i - 1], "ScenarioTree: node numbering must be stage-contiguous");
  }
  horizon = stage[n - 1];
  child_first.assign(n, n);
  child_count.assign(n, 0);
  for (int i = 1; i < n; ++i) {
    const int a = anc[i];
    if (child_count[a] == 0)
      child_first[a] = i;
    else
      require(child_first[a] + child_count[a] == i, "ScenarioTree: children of a node must be contiguous");
    ++child_count[a];
  }
  stage_start.assign(horizon + 2, 0);
  for (int i = 0; i < n; ++i) ++stage_start[stage[i] + 1];
  for (int t = 0; t <= horizon; ++t) stage_start[t + 1] += stage_start[t];
  for (int i = 0; i < n; ++i)
    require((child_count[i] == 0) == (stage[i] == horizon),
            "ScenarioTree: leaves must be exactly the horizon-stage nodes");
  require(stop_stage >= 0 && stop_stage <= horizon, "ScenarioTree: stop stage outside [0, horizon]");
  for (int t = stop_stage; t < horizon; ++t)
    for (int i = stage_start[t]; i < stage_start[t + 1]; ++i)
      require(child_count[i] == 1, "ScenarioTree: nodes past the stop stage must have one child");
  require(std::fabs(prob[0] - 1.0) <= kProbTol, "ScenarioTree: root probability must be 1");
  for (int i = 1; i < n; ++i) {
    require(prob[i] >= 1e-15, "ScenarioTree: node probability below 1e-15");
    require(std::fabs(prob[i] - prob[anc[i]] * cond_prob[i]) <= kProbTol,
            "ScenarioTree: prob(i) must equal prob(anc)*cond_prob(i)");
  }
  for (int t = 0; t <= horizon; ++t) {
    double s = 0.0;
    for (int i = stage_start[t]; i < stage_start[t + 1]; ++i) s += prob[i];
    require(std::fabs(s - 1.0) <= kProbTol, "ScenarioTree: stage probabilities must sum to 1");
  }
}

void Risk::validate() const {  // proj/src/risk.cpp:45-63
  require(n > 0, "RiskSpec: n must be positive");
  int cd = 0;
  for (const auto& p : cone) cd += p.dim;
  require(cd == rows, "RiskSpec: cone/E row mismatch");
  if (kind == SPOCK_RISK_AVAR) {
    require(int(pi.size()) == n, "RiskSpec: avar pi has wrong length");
    require(nnu == 0, "RiskSpec: avar specs carry no nu variables");
    const bool standard = rows == 2 * n + 1;
    const bool max_form = gamma == 0.0 && rows == n + 1;
    const bool eq_form = gamma == 1.0 && rows == n;
    require(standard || max_form || eq_form, "RiskSpec: malformed avar representation");
  }
}

namespace {
void check_symmetric(const double* M, int n, const char* what) {
  double mx = 0.0;
  for (int k = 0; k < n * n; ++k) mx = std::max(mx, std::fabs(M[k]));
  const double scale = std::max(1.0, mx);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i)
      if (std::fabs(M[i + j * n] - M[j + i * n]) > 1e-12 * scale)
        throw std::invalid_argument(std::string(what) + ": matrix must be symmetric");
}
bool chol_pd(const double* M, int n) {
  std::vector<double> L(size_t(n) * n, 0.0);
  for (int j = 0; j < n; ++j) {
    double d = 0.5 * (M[j + j * n] + M[j + j * n]);
    for (int k = 0; k < j; ++k) d -= L[j + k * n] * L[j + k * n];
    if (!(d > 0.0)) return false;
    d = std::sqrt(d);
    L[j + j * n] = d;
    for (int i = j + 1; i < n; ++i) {
      double s = 0.5 * (M[i + j * n] + M[j + i * n]);
      for (int k = 0; k < j; ++k) s -= L[i + k * n] * L[j + k * n];
      L[i + j * n] = s / d;
    }
  }
  return true;
}
}  // namespace

void Problem::validate() const {  // proj/src/problem.cpp:39-86
  const int nn = tree.nn(), nnl = tree.nnl(), nl = tree.nl();
  require(nx > 0 && nu > 0, "Raocp: dimensions must be positive");
  // per-node checks on host threads; the first failing node (in node order)
  // raises the reference's exception on this thread
  std::vector<uint8_t> bad(static_cast<size_t>(std::max(nn - 1, 1)), 0);
  host_parallel(nn - 1, [&](int64_t k) {
    try {
      check_symmetric(&Q[size_t(k) * nx * nx], nx, "Raocp Q");
      check_symmetric(&R[size_t(k) * nu * nu], nu, "Raocp R");
      if (!chol_pd(&R[size_t(k) * nu * nu], nu)) bad[k] = 1;
    } catch (const std::invalid_argument&) {
      bad[k] = 1;
    }
  });
  for (int i = 1; i < nn; ++i) {
    if (!bad[i - 1]) continue;
    check_symmetric(&Q[size_t(i - 1) * nx * nx], nx, "Raocp Q");
    check_symmetric(&R[size_t(i - 1) * nu * nu], nu, "Raocp R");
    require(chol_pd(&R[size_t(i - 1) * nu * nu], nu), "Raocp: R must be positive definite");
  }
  for (int i = 0; i < nnl; ++i) {
    risk[i].validate();
    require(risk[i].n == tree.child_count[i], "Raocp: risk spec size must match child count");
    for (int k = 0; k < nc[i]; ++k)
      require(C_lo[box_off[i] + k] <= C_hi[box_off[i] + k], "Box: lower bound above upper bound");
  }
  std::vector<uint8_t> badN(static_cast<size_t>(std::max(nl, 1)), 0);
  host_parallel(nl, [&](int64_t j) {
    try {
      check_symmetric(&QN[size_t(j) * nx * nx], nx, "Raocp QN");
    } catch (const std::invalid_argument&) {
      badN[j] = 1;
    }
  });
  for (int j = 0; j < nl; ++j) {
    if (badN[j]) check_symmetric(&QN[size_t(j) * nx * nx], nx, "Raocp QN");
    for (int k = 0; k < ncN[j]; ++k)
      require(CN_lo[boxN_off[j] + k] <= CN_hi[boxN_off[j] + k], "Box: lower bound above upper bound");
  }
}

BigVec::BigVec(const double* src, size_t count) : p(count ? new double[count] : nullptr), n(count) {
  const int64_t slab = int64_t(1) << 20;
  host_parallel((int64_t(count) + slab - 1) / slab, [&](int64_t b) {
    const size_t o = size_t(b) * slab;
    std::memcpy(p.get() + o, src + o, sizeof(double) * std::min<size_t>(slab, count - o));
  });
}

BigVec BigVec::transposed(const double* src, size_t nb, int rows, int cols) {
  BigVec v;
  const size_t bs = size_t(rows) * cols;
  v.n = nb * bs;
  v.p.reset(v.n ? new double[v.n] : nullptr);
  double* dst = v.p.get();
  host_parallel(int64_t(nb), [&](int64_t b) {
    const double* s = src + size_t(b) * bs;
    double* o = dst + size_t(b) * bs;
    for (int j = 0; j < cols; ++j)
      for (int i = 0; i < rows; ++i) o[i + size_t(j) * rows] = s[size_t(i) * cols + j];
  });
  return v;
}

BigVec BigVec::repeated(const double* blk, size_t nb, int rows, int cols) {
  BigVec v;
  const size_t bs = size_t(rows) * cols;
  v.n = nb * bs;
  v.p.reset(v.n ? new double[v.n] : nullptr);
  double* dst = v.p.get();
  host_parallel(int64_t(nb), [&](int64_t b) { std::memcpy(dst + size_t(b) * bs, blk, sizeof(double) * bs); });
  return v;
}

Problem problem_from_desc(const spock_problem_desc* d) {
  require(d != nullptr, "spock: null problem description");
  Problem P;
  const int nn = d->num_nodes;
  require(nn > 0, "ScenarioTree: empty tree");
  require(d->anc && d->prob && d->cond_prob && d->event, "ScenarioTree: missing tree arrays");
  Tree& t = P.tree;
  t.anc.assign(d->anc, d->anc + nn);
  t.event.assign(d->event, d->event + nn);
  t.prob.assign(d->prob, d->prob + nn);
  t.cond_prob.assign(d->cond_prob, d->cond_prob + nn);
  t.stop_stage = d->stop_stage;
  t.num_events = d->num_events;
  t.finalize();
  require(t.horizon == d->horizon, "from_arrays: horizon mismatch");
  P.nx = d->nx;
  P.nu = d->nu;
  require(P.nx > 0 && P.nu > 0, "Raocp: dimensions must be positive");
  const size_t nx = P.nx, nu = P.nu, nr = nn - 1, nnl = t.nnl(), nl = t.nl();
  auto cp = [](const double* s, size_t n) {
    require(n == 0 || s != nullptr, "Raocp: missing data array");
    return Vec(s, s + n);
  };
  require((d->layout & ~(SPOCK_LAYOUT_ROW_MAJOR | SPOCK_LAYOUT_SHARED_G)) == 0, "Raocp: unknown layout flags");
  const bool rowm = (d->layout & SPOCK_LAYOUT_ROW_MAJOR) != 0;
  // nb per-node blocks of rows x cols, column-major in the problem
  auto big = [&](const double* s, size_t nb, int rows, int cols) {
    require(nb == 0 || s != nullptr, "Raocp: missing data array");
    return rowm ? BigVec::transposed(s, nb, rows, cols) : BigVec(s, nb * size_t(rows) * cols);
  };
  P.A = big(d->A, nr, int(nx), int(nx));
  P.B = big(d->B, nr, int(nx), int(nu));
  P.c = cp(d->c, nr * nx);
  // Q, R, QN must be symmetric (validate() rejects them otherwise), so their
  // row-major and column-major images coincide: plain parallel copies
  auto sym = [&](const double* s, size_t nb, int n) {
    require(nb == 0 || s != nullptr, "Raocp: missing data array");
    return BigVec(s, nb * size_t(n) * n);
  };
  P.Q = sym(d->Q, nr, int(nx));
  P.R = sym(d->R, nr, int(nu));
  P.q = cp(d->q, nr * nx);
  P.r = cp(d->r, nr * nu);
  P.QN = sym(d->QN, nl, int(nx));
  P.qN = cp(d->qN, nl * nx);
  P.nc.assign(d->nc, d->nc + nnl);
  P.ncN.assign(d->ncN, d->ncN + nl);
  P.g_off.resize(nnl + 1);
  P.box_off.resize(nnl + 1);
  int64_t go = 0, bo = 0;
  for (size_t i = 0; i < nnl; ++i) {
    require(P.nc[i] >= 0, "Raocp: negative constraint rows");
    P.g_off[i] = go;
    P.box_off[i] = bo;
    go += int64_t(P.nc[i]);
    bo += P.nc[i];
  }
  P.g_off[nnl] = go;
  P.box_off[nnl] = bo;
  // constraint blocks: nc[i] x cols per node at row offset off[i]
  auto gbig = [&](const double* s, const std::vector<int>& ncv, const std::vector<int64_t>& off, int cols) {
    const size_t nb = ncv.size();
    const int64_t rows_total = off[nb];
    require(rows_total == 0 || s != nullptr, "Raocp: missing data array");
    if (d->layout & SPOCK_LAYOUT_SHARED_G) {
      const int r0 = nb ? ncv[0] : 0;
      for (size_t i = 0; i < nb; ++i) require(ncv[i] == r0, "Raocp: shared constraint block needs equal row counts");
      std::vector<double> blk(size_t(r0) * cols);
      for (int j = 0; j < cols; ++j)
        for (int i = 0; i < r0; ++i) blk[i + size_t(j) * r0] = rowm ? s[size_t(i) * cols + j] : s[i + size_t(j) * r0];
      return BigVec::repeated(blk.data(), nb, r0, cols);
    }
    if (!rowm) return BigVec(s, size_t(rows_total) * cols);
    BigVec v(nullptr, 0);
    v.n = size_t(rows_total) * cols;
    v.p.reset(v.n ? new double[v.n] : nullptr);
    double* dst = v.p.get();
    host_parallel(int64_t(nb), [&](int64_t b) {
      const int r = ncv[b];
      const double* sb = s + size_t(off[b]) * cols;
      double* o = dst + size_t(off[b]) * cols;
      for (int j = 0; j < cols; ++j)
        for (int i = 0; i < r; ++i) o[i + size_t(j) * r] = sb[size_t(i) * cols + j];
    });
    return v;
  };
  P.Gx = gbig(d->Gx, P.nc, P.g_off, int(nx));
  P.Gu = gbig(d->Gu, P.nc, P.g_off, int(nu));
  P.C_lo = cp(d->C_lo, bo);
  P.C_hi = cp(d->C_hi, bo);
  P.gN_off.resize(nl + 1);
  P.boxN_off.resize(nl + 1);
  go = bo = 0;
  for (size_t j = 0; j < nl; ++j) {
    require(P.ncN[j] >= 0, "Raocp: negative constraint rows");
    P.gN_off[j] = go;
    P.boxN_off[j] = bo;
    go += P.ncN[j];
    bo += P.ncN[j];
  }
  P.gN_off[nl] = go;
  P.boxN_off[nl] = bo;
  P.GN = gbig(d->GN, P.ncN, P.gN_off, int(nx));
  P.CN_lo = cp(d->CN_lo, bo);
  P.CN_hi = cp(d->CN_hi, bo);
  const double *E = d->risk_E, *F = d->risk_F, *b = d->risk_b, *pi = d->risk_pi;
  const int *ck = d->cone_kind, *cd = d->cone_dim;
  for (size_t i = 0; i < nnl; ++i) {
    Risk rs;
    rs.kind = d->risk_kind[i];
    rs.n = t.child_count[i];
    rs.rows = d->risk_rows[i];
    rs.nnu = d->risk_nnu[i];
    require(rs.rows >= 0 && rs.nnu >= 0, "RiskSpec: bad dimensions");
    rs.E.assign(E, E + size_t(rs.rows) * rs.n);
    E += size_t(rs.rows) * rs.n;
    if (rs.nnu > 0) {
      rs.F.assign(F, F + size_t(rs.rows) * rs.nnu);
      F += size_t(rs.rows) * rs.nnu;
    }
    rs.b.assign(b, b + rs.rows);
    b += rs.rows;
    rs.gamma = d->risk_gamma[i];
    if (rs.kind == SPOCK_RISK_AVAR) {
      rs.pi.assign(pi, pi + rs.n);
      pi += rs.n;
    }
    for (int k = 0; k < d->cone_nparts[i]; ++k) rs.cone.push_back({*ck++, *cd++});
    P.risk.push_back(std::move(rs));
  }
  require(d->x_init != nullptr, "Raocp: x_init has wrong length");
  P.x_init.assign(d->x_init, d->x_init + nx);
  P.validate();
  return P;
}

// ---------------------------------------------------------------------------
Precond identity_precond(const Problem& p) {
  Precond pc;
  pc.sx.assign(p.nx, 1.0);
  pc.su.assign(p.nu, 1.0);
  pc.sxN.assign(p.nx, 1.0);
  pc.cstr_scale.assign(p.tree.nnl(), 1.0);
  pc.c_hat = 1.0;
  pc.is_identity = true;
  return pc;
}

Precond precondition_inplace(Problem& p) {  // proj/src/problem.cpp:249-326
  const Tree& tr = p.tree;
  const int nn = tr.nn(), nnl = tr.nnl(), nl = tr.nl(), nx = p.nx, nu = p.nu;
  int max_ch = 1;
  for (int i = 0; i < nnl; ++i) max_ch = std::max(max_ch, tr.child_count[i]);
  Precond pc;
  pc.is_identity = false;
  pc.c_hat = std::sqrt(double(max_ch));
  pc.sx.assign(nx, 1.0);
  pc.su.assign(nu, 1.0);
  pc.sxN.assign(nx, 1.0);
  for (int i = 1; i < nn; ++i) {
    const double* Q = &p.Q[size_t(i - 1) * nx * nx];
    const double* R = &p.R[size_t(i - 1) * nu * nu];
    for (int k = 0; k < nx; ++k) pc.sx[k] = std::max(pc.sx[k], std::sqrt(std::max(0.0, Q[k + k * nx])));
    for (int k = 0; k < nu; ++k) pc.su[k] = std::max(pc.su[k], std::sqrt(std::max(0.0, R[k + k * nu])));
  }
  for (auto& v : pc.sx) v *= pc.c_hat;
  for (auto& v : pc.su) v *= pc.c_hat;
  for (int j = 0; j < nl; ++j) {
    const double* Q = &p.QN[size_t(j) * nx * nx];
    for (int k = 0; k < nx; ++k) pc.sxN[k] = std::max(pc.sxN[k], std::sqrt(std::max(0.0, Q[k + k * nx])));
  }
  Vec isx(nx), isu(nu), isxN(nx);
  for (int k = 0; k < nx; ++k) isx[k] = 1.0 / pc.sx[k], isxN[k] = 1.0 / pc.sxN[k];
  for (int k = 0; k < nu; ++k) isu[k] = 1.0 / pc.su[k];
  host_parallel(nn - 1, [&](int64_t k) {
    const int i = int(k) + 1;
    const Vec& cs = tr.leaf(i) ? pc.sxN : pc.sx;
    double* A = &p.A[size_t(k) * nx * nx];
    double* B = &p.B[size_t(k) * nx * nu];
    double* c = &p.c[size_t(k) * nx];
    double* Q = &p.Q[size_t(k) * nx * nx];
    double* R = &p.R[size_t(k) * nu * nu];
    for (int j = 0; j < nx; ++j)
      for (int r = 0; r < nx; ++r) A[r + j * nx] = cs[r] * A[r + j * nx] * isx[j];
    for (int j = 0; j < nu; ++j)
      for (int r = 0; r < nx; ++r) B[r + j * nx] = cs[r] * B[r + j * nx] * isu[j];
    for (int r = 0; r < nx; ++r) c[r] = cs[r] * c[r];
    for (int j = 0; j < nx; ++j)
      for (int r = 0; r < nx; ++r) Q[r + j * nx] = isx[r] * Q[r + j * nx] * isx[j];
    for (int j = 0; j < nu; ++j)
      for (int r = 0; r < nu; ++r) R[r + j * nu] = isu[r] * R[r + j * nu] * isu[j];
    for (int r = 0; r < nx; ++r) p.q[size_t(k) * nx + r] *= isx[r];
    for (int r = 0; r < nu; ++r) p.r[size_t(k) * nu + r] *= isu[r];
  });
  for (int j = 0; j < nl; ++j) {
    double* Q = &p.QN[size_t(j) * nx * nx];
    for (int jj = 0; jj < nx; ++jj)
      for (int r = 0; r < nx; ++r) Q[r + jj * nx] = isxN[r] * Q[r + jj * nx] * isxN[jj];
    for (int r = 0; r < nx; ++r) p.qN[size_t(j) * nx + r] *= isxN[r];
  }
  // per non-leaf constraint row scaling by max(1, ||[Gx/sx Gu/su]||_2), per node
  // on host threads.  When every row of the scaled block has at most one
  // nonzero (box selectors: every generated problem) the columns have disjoint
  // supports, S'S is diagonal and the norm is the largest column norm; else
  // the dense S'S and its largest eigenvalue
  pc.cstr_scale.assign(nnl, 1.0);
  host_parallel(nnl, [&](int64_t ii) {
    const int i = int(ii);
    const int nc = p.nc[i], m = nx + nu;
    const size_t o = size_t(p.g_off[i]);
    auto S = [&](int r, int j) {
      return j < nx ? p.Gx[o * nx + r + size_t(j) * nc] * isx[j] : p.Gu[o * nu + r + size_t(j - nx) * nc] * isu[j - nx];
    };
    bool sel = true;
    for (int r = 0; r < nc && sel; ++r) {
      int nz = 0;
      for (int j = 0; j < m; ++j) nz += S(r, j) != 0.0;
      sel = nz <= 1;
    }
    double emax = 0.0;
    if (sel) {
      for (int j = 0; j < m; ++j) {
        double s2 = 0.0;
        for (int r = 0; r < nc; ++r) s2 += S(r, j) * S(r, j);
        emax = std::max(emax, s2);
      }
    } else {
      Mat G(m, m);
      bool diag = true;
      for (int j = 0; j < m; ++j)
        for (int k = 0; k < m; ++k) {
          double s2 = 0.0;
          for (int r = 0; r < nc; ++r) s2 += S(r, j) * S(r, k);
          G(j, k) = s2;
          if (j != k && s2 != 0.0) diag = false;
        }
      if (diag) {
        for (int j = 0; j < m; ++j) emax = std::max(emax, G(j, j));
      } else {
        Vec w;
        Mat V;
        sym_eig(G, w, V);
        emax = w.empty() ? 0.0 : w.back();
      }
    }
    pc.cstr_scale[i] = std::max(1.0, std::sqrt(std::max(0.0, emax)));
  });
  host_parallel(nnl, [&](int64_t ii) {
    const int i = int(ii), nc = p.nc[i];
    const size_t o = size_t(p.g_off[i]);
    const double a = pc.cstr_scale[i];
    for (int j = 0; j < nx; ++j)
      for (int r = 0; r < nc; ++r) {
        double& g = p.Gx[o * nx + r + size_t(j) * nc];
        g = g * isx[j] / a;
      }
    for (int j = 0; j < nu; ++j)
      for (int r = 0; r < nc; ++r) {
        double& g = p.Gu[o * nu + r + size_t(j) * nc];
        g = g * isu[j] / a;
      }
    for (int r = 0; r < nc; ++r) {
      p.C_lo[p.box_off[i] + r] /= a;
      p.C_hi[p.box_off[i] + r] /= a;
    }
  });
  for (int j = 0; j < nl; ++j) {
    const size_t o = size_t(p.gN_off[j]);
    const int nc = p.ncN[j];
    for (int jj = 0; jj < nx; ++jj)
      for (int r = 0; r < nc; ++r) p.GN[o * nx + r + size_t(jj) * nc] *= isxN[jj];
  }
  for (int k = 0; k < nx; ++k) p.x_init[k] *= pc.sx[k];
  return pc;
}

// ---------------------------------------------------------------------------
// soc_data_quadlin (proj/src/problem.cpp:113-161) for blkdiag(Q, R) with
// linear term (q, r), decomposed per block.  R may be absent (nu = 0: leaf).
SocBlock soc_block(const double* Q, int nx, const double* R, int nu, const double* q, const double* r) {
  SocBlock out;
  Vec wx, wu;
  Mat Vx, Vu;
  {
    Mat M(nx, nx);
    std::memcpy(M.a.data(), Q, sizeof(double) * nx * nx);
    sym_eig(M, wx, Vx);
  }
  if (nu > 0) {
    Mat M(nu, nu);
    std::memcpy(M.a.data(), R, sizeof(double) * nu * nu);
    sym_eig(M, wu, Vu);
  }
  double lmax = 0.0, lmin = std::numeric_limits<double>::infinity();
  for (double v : wx) lmax = std::max(lmax, v), lmin = std::min(lmin, v);
  for (double v : wu) lmax = std::max(lmax, v), lmin = std::min(lmin, v);
  if (nx + nu == 0) lmin = 0.0;
  require(lmin >= -1e-10 * std::max(lmax, 1.0), "soc_data_quadlin: Q must be positive semidefinite");
  const double thresh = 1e-10 * lmax;
  out.lambda_max = lmax;
  // merged ascending order of the kept eigenvalues (x block first on ties)
  std::vector<int> kx, ku;
  for (int k = 0; k < nx; ++k)
    if (wx[k] > thresh) kx.push_back(k);
  for (int k = 0; k < nu; ++k)
    if (wu[k] > thresh) ku.push_back(k);
  out.px = int(kx.size());
  out.pu = int(ku.size());
  const int p = out.px + out.pu;
  out.perm.resize(p);
  {
    int ix = 0, iu = 0, pos = 0;
    while (ix < out.px || iu < out.pu) {
      const bool takex = iu >= out.pu || (ix < out.px && wx[kx[ix]] <= wu[ku[iu]]);
      if (takex)
        out.perm[ix++] = pos++;
      else
        out.perm[out.px + iu++] = pos++;
    }
  }
  // per block: H = (S'MS)^{1/2} S', qk = v - S S'v, w = (S'MS)^{-1/2} S' v
  auto block = [&](const double* M, int n, const Vec& wv, const Mat& V, const std::vector<int>& keep,
                   const double* v, Vec& H, double* qk, double* wout) {
    const int pb = int(keep.size());
    H.assign(size_t(pb) * n, 0.0);
    for (int i = 0; i < n; ++i) qk[i] = v[i];
    if (pb == 0) return;
    Mat S(n, pb);
    for (int k = 0; k < pb; ++k)
      for (int i = 0; i < n; ++i) S(i, k) = V(i, keep[k]);
    Mat SMS(pb, pb);
    for (int b = 0; b < pb; ++b)
      for (int a2 = 0; a2 < pb; ++a2) {
        double s = 0.0;
        for (int j = 0; j < n; ++j) {
          double t = 0.0;
          for (int i = 0; i < n; ++i) t += S(i, a2) * M[i + j * n];
          s += t * S(j, b);
        }
        SMS(a2, b) = s;
      }
    Vec e2;
    Mat U;
    sym_eig(SMS, e2, U);
    Mat sq(pb, pb), isq(pb, pb);
    for (int j = 0; j < pb; ++j)
      for (int i = 0; i < pb; ++i) {
        double s = 0.0, si = 0.0;
        for (int k = 0; k < pb; ++k) {
          const double ev = std::sqrt(std::max(0.0, e2[k]));
          s += U(i, k) * ev * U(j, k);
          si += U(i, k) * (ev > 0 ? 1.0 / ev : 0.0) * U(j, k);
        }
        sq(i, j) = s;
        isq(i, j) = si;
      }
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < pb; ++i) {
        double s = 0.0;
        for (int k = 0; k < pb; ++k) s += sq(i, k) * S(j, k);
        H[i + size_t(j) * pb] = s;
      }
    Vec Sv(pb, 0.0);
    for (int k = 0; k < pb; ++k)
      for (int i = 0; i < n; ++i) Sv[k] += S(i, k) * v[i];
    for (int k = 0; k < pb; ++k)
      for (int i = 0; i < n; ++i) qk[i] -= S(i, k) * Sv[k];
    (void)wv;
    for (int i = 0; i < pb; ++i) {
      double s = 0.0;
      for (int k = 0; k < pb; ++k) s += isq(i, k) * Sv[k];
      wout[i] = s;
    }
  };
  out.qk.assign(nx + nu, 0.0);
  Vec w(p, 0.0);
  block(Q, nx, wx, Vx, kx, q, out.Hx, out.qk.data(), w.data());
  if (nu > 0) block(R, nu, wu, Vu, ku, r, out.Hu, out.qk.data() + nx, w.data() + out.px);
  double qn2 = 0.0;
  for (double v : w) qn2 += v * v;
  out.a.assign(p + 2, 0.0);
  for (int k = 0; k < p; ++k) out.a[k] = -0.5 * w[k];
  out.a[p] = -0.125 * qn2 + 0.5;
  out.a[p + 1] = -0.125 * qn2 - 0.5;
  return out;
}

void parallel_for(int64_t n, const std::function<void(int64_t)>& f) { host_parallel(n, f); }

SocData soc_epigraph_data(const Problem& p) {  // proj/src/problem.cpp:216-236
  const int nn = p.tree.nn(), nnl = p.tree.nnl(), nl = p.tree.nl(), nx = p.nx, nu = p.nu;
  SocData d;
  d.stage.resize(nn - 1);
  d.leaf.resize(nl);
  // memoise identical (Q, R, q, r) blocks (generators share them per event)
  std::vector<int> rep(nn - 1);
  {
    std::unordered_map<uint64_t, int> memo;
    for (int k = 0; k < nn - 1; ++k) {
      uint64_t h = fnv(&p.Q[size_t(k) * nx * nx], sizeof(double) * nx * nx);
      h = fnv(&p.R[size_t(k) * nu * nu], sizeof(double) * nu * nu, h);
      h = fnv(&p.q[size_t(k) * nx], sizeof(double) * nx, h);
      h = fnv(&p.r[size_t(k) * nu], sizeof(double) * nu, h);
      auto it = memo.find(h);
      const int o = it == memo.end() ? -1 : it->second;
      if (o >= 0 && !std::memcmp(&p.Q[size_t(o) * nx * nx], &p.Q[size_t(k) * nx * nx], sizeof(double) * nx * nx) &&
          !std::memcmp(&p.R[size_t(o) * nu * nu], &p.R[size_t(k) * nu * nu], sizeof(double) * nu * nu) &&
          !std::memcmp(&p.q[size_t(o) * nx], &p.q[size_t(k) * nx], sizeof(double) * nx) &&
          !std::memcmp(&p.r[size_t(o) * nu], &p.r[size_t(k) * nu], sizeof(double) * nu)) {
        rep[k] = o;
      } else {
        memo[h] = k;
        rep[k] = k;
      }
    }
  }
  host_parallel(nn - 1, [&](int64_t k) {
    if (rep[k] != k) return;
    d.stage[k] = soc_block(&p.Q[size_t(k) * nx * nx], nx, &p.R[size_t(k) * nu * nu], nu, &p.q[size_t(k) * nx],
                           &p.r[size_t(k) * nu]);
  });
  for (int k = 0; k < nn - 1; ++k)
    if (rep[k] != k) d.stage[k] = d.stage[rep[k]];
  std::vector<int> repl(nl);
  {
    std::unordered_map<uint64_t, int> memo;
    for (int j = 0; j < nl; ++j) {
      uint64_t h = fnv(&p.QN[size_t(j) * nx * nx], sizeof(double) * nx * nx);
      h = fnv(&p.qN[size_t(j) * nx], sizeof(double) * nx, h);
      auto it = memo.find(h);
      const int o = it == memo.end() ? -1 : it->second;
      if (o >= 0 && !std::memcmp(&p.QN[size_t(o) * nx * nx], &p.QN[size_t(j) * nx * nx], sizeof(double) * nx * nx) &&
          !std::memcmp(&p.qN[size_t(o) * nx], &p.qN[size_t(j) * nx], sizeof(double) * nx)) {
        repl[j] = o;
      } else {
        memo[h] = j;
        repl[j] = j;
      }
    }
  }
  host_parallel(nl, [&](int64_t j) {
    if (repl[j] != j) return;
    d.leaf[j] = soc_block(&p.QN[size_t(j) * nx * nx], nx, nullptr, 0, &p.qN[size_t(j) * nx], nullptr);
  });
  for (int j = 0; j < nl; ++j)
    if (repl[j] != j) d.leaf[j] = d.leaf[repl[j]];
  (void)nnl;
  return d;
}

Layouts make_layouts(const Problem& p, const SocData& soc) {
  const Tree& tr = p.tree;
  const int nn = tr.nn(), nnl = tr.nnl(), nl = tr.nl();
  Layouts L;
  int64_t off = 1 + int64_t(nn) * p.nx;
  L.u_base = int(off);
  off += int64_t(nnl) * p.nu;
  L.y_off.resize(nnl);
  L.y_dim.resize(nnl);
  for (int i = 0; i < nnl; ++i) {
    L.y_off[i] = int(off);
    L.y_dim[i] = p.risk[i].rows;
    off += L.y_dim[i];
  }
  L.tau_base = int(off);
  off += nn - 1;
  L.s_base = int(off);
  off += nn - 1;
  L.nz = off;
  require(off < (int64_t(1) << 31), "spock: primal vector exceeds 2^31 entries");
  off = 0;
  L.seg1_off.resize(nnl);
  L.seg1_nc.resize(nnl);
  L.seg1_ydim.resize(nnl);
  for (int i = 0; i < nnl; ++i) {
    L.seg1_off[i] = int(off);
    L.seg1_ydim[i] = p.risk[i].rows;
    L.seg1_nc[i] = p.nc[i];
    off += L.seg1_ydim[i] + 1 + L.seg1_nc[i];
  }
  L.seg2_off.resize(nn - 1);
  L.seg2_dim.resize(nn - 1);
  for (int i = 1; i < nn; ++i) {
    L.seg2_off[i - 1] = int(off);
    L.seg2_dim[i - 1] = soc.stage[i - 1].px + soc.stage[i - 1].pu + 2;
    off += L.seg2_dim[i - 1];
  }
  L.seg3_off.resize(nl);
  L.seg3_nc.resize(nl);
  L.seg3_socdim.resize(nl);
  for (int j = 0; j < nl; ++j) {
    L.seg3_off[j] = int(off);
    L.seg3_nc[j] = p.ncN[j];
    L.seg3_socdim[j] = soc.leaf[j].px + 2;
    off += L.seg3_nc[j] + L.seg3_socdim[j];
  }
  L.neta = off;
  require(off < (int64_t(1) << 31), "spock: dual vector exceeds 2^31 entries");
  return L;
}

namespace {
double holder(const double* A, int r, int c) {
  if (r == 0 || c == 0) return 0.0;
  double n1 = 0.0, ni = 0.0;
  for (int j = 0; j < c; ++j) {
    double s = 0.0;
    for (int i = 0; i < r; ++i) s += std::fabs(A[i + size_t(j) * r]);
    n1 = std::max(n1, s);
  }
  for (int i = 0; i < r; ++i) {
    double s = 0.0;
    for (int j = 0; j < c; ++j) s += std::fabs(A[i + size_t(j) * r]);
    ni = std::max(ni, s);
  }
  return std::sqrt(n1 * ni);
}
}  // namespace

double analytic_norm_bound(const Problem& p, const SocData& soc) {
  const Tree& tr = p.tree;
  const int nn = tr.nn(), nnl = tr.nnl(), nx = p.nx, nu = p.nu;
  int max_ch = 1;
  for (int i = 0; i < nnl; ++i) max_ch = std::max(max_ch, tr.child_count[i]);
  // per-node maxima on host threads, then one max (order-independent)
  std::vector<double> per(static_cast<size_t>(nn), 0.0);
  host_parallel(nn, [&](int64_t ii) {
    const int i = int(ii);
    double mx = 0.0;
    if (i < nnl) {
      mx = std::max(mx, 1.0);
      double bb = 0.0;
      for (double v : p.risk[i].b) bb += v * v;
      mx = std::max(mx, std::sqrt(1.0 + bb));
      const int nc = p.nc[i];
      std::vector<double> g(size_t(nc) * (nx + nu));
      std::memcpy(g.data(), &p.Gx[size_t(p.g_off[i]) * nx], sizeof(double) * nc * nx);
      std::memcpy(g.data() + size_t(nc) * nx, &p.Gu[size_t(p.g_off[i]) * nu], sizeof(double) * nc * nu);
      mx = std::max(mx, holder(g.data(), nc, nx + nu));
    }
    if (i > 0) {
      const auto& d = soc.stage[i - 1];
      double qq = d.qk2;
      if (qq < 0.0) {
        qq = 0.0;
        for (double v : d.qk) qq += v * v;
      }
      mx = std::max(mx, std::sqrt(d.lambda_max + 0.5 * (1.0 + qq)));
    }
    if (i >= nnl) {
      const int j = i - nnl;
      const auto& d = soc.leaf[j];
      mx = std::max(mx, holder(&p.GN[size_t(p.gN_off[j]) * nx], p.ncN[j], nx));
      double qq = d.qk2;
      if (qq < 0.0) {
        qq = 0.0;
        for (double v : d.qk) qq += v * v;
      }
      mx = std::max(mx, std::sqrt(d.lambda_max + 0.5 * (1.0 + qq)));
    }
    per[size_t(i)] = mx;
  });
  double mx = 0.0;
  for (double v : per) mx = std::max(mx, v);
  return std::sqrt(1.0 + double(max_ch)) * mx;
}

// Philox4x32-10 (proj/src/rng.cpp:10-103): normals for the power-iteration start
void philox_normals(uint64_t seed, int64_t n, double* out) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
  uint32_t ctr[4] = {0, 0, 0, 0}, key[2] = {uint32_t(seed), uint32_t(seed >> 32)}, blk[4];
  int pos = 4;
  auto u32 = [&]() -> uint32_t {
    if (pos >= 4) {
      uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3], k0 = key[0], k1 = key[1];
      for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = uint64_t(M0) * c0, p1 = uint64_t(M1) * c2;
        const uint32_t n0 = uint32_t(p1 >> 32) ^ c1 ^ k0, n1 = uint32_t(p1);
        const uint32_t n2 = uint32_t(p0 >> 32) ^ c3 ^ k1, n3 = uint32_t(p0);
        c0 = n0, c1 = n1, c2 = n2, c3 = n3;
        k0 += W0;
        k1 += W1;
      }
      blk[0] = c0, blk[1] = c1, blk[2] = c2, blk[3] = c3;
      if (++ctr[0] == 0)
        if (++ctr[1] == 0)
          if (++ctr[2] == 0) ++ctr[3];
      pos = 0;
    }
    return blk[pos++];
  };
  auto uni = [&]() {
    const uint64_t lo = u32();
    const uint64_t hi = u32();
    return double(((hi << 32) | lo) >> 11) * 0x1.0p-53;
  };
  bool have = false;
  double spare = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    if (have) {
      have = false;
      out[i] = spare;
      continue;
    }
    double u1 = uni();
    while (u1 <= 0.0) u1 = uni();
    const double u2 = uni();
    const double mag = std::sqrt(-2.0 * std::log(u1)), ang = 2.0 * M_PI * u2;
    spare = mag * std::sin(ang);
    have = true;
    out[i] = mag * std::cos(ang);
  }
}

}  // namespace spock
