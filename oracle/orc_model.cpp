// TEST INFRASTRUCTURE ONLY -- parity oracle (see orc.hpp).
// Restates proj/src/tree.cpp, risk.cpp, problem.cpp, layout.cpp.
#include <algorithm>

#include "orc.hpp"

namespace orc {

namespace {
void require(bool c, const char* m) {
  if (!c) throw std::invalid_argument(m);
}
constexpr double kProbTol = 1e-12;

Mat check_symmetric(const Mat& M, const char* what) {  // problem.cpp:16-22
  require(M.r == M.c, "matrix must be square");
  double mx = 0.0;
  for (double v : M.a) mx = std::max(mx, std::fabs(v));
  const double scale = std::max(1.0, mx);
  Mat S(M.r, M.c);
  for (int j = 0; j < M.c; ++j)
    for (int i = 0; i < M.r; ++i) {
      if (std::fabs(M(i, j) - M(j, i)) > 1e-12 * scale)
        throw std::invalid_argument(std::string(what) + ": matrix must be symmetric");
      S(i, j) = 0.5 * (M(i, j) + M(j, i));
    }
  return S;
}
}  // namespace

// ScenarioTree::finalize_topology, proj/src/tree.cpp:24-83
void Tree::finalize() {
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
    for (int i = sb(t); i < se(t); ++i)
      require(child_count[i] == 1, "ScenarioTree: nodes past the stop stage must have one child");
  require(std::fabs(prob[0] - 1.0) <= kProbTol, "ScenarioTree: root probability must be 1");
  for (int i = 1; i < n; ++i) {
    require(prob[i] >= 1e-15, "ScenarioTree: node probability below 1e-15");
    require(std::fabs(prob[i] - prob[anc[i]] * cond_prob[i]) <= kProbTol,
            "ScenarioTree: prob(i) must equal prob(anc)*cond_prob(i)");
  }
  for (int t = 0; t <= horizon; ++t) {
    double s = 0.0;
    for (int i = sb(t); i < se(t); ++i) s += prob[i];
    require(std::fabs(s - 1.0) <= kProbTol, "ScenarioTree: stage probabilities must sum to 1");
  }
}

void stage_parallel_for(const Tree& t, int st, const std::function<void(int)>& body, uint64_t flops) {
  parallel_for(t.sb(st), t.se(st), body, flops);  // tree.cpp:227-230
}

std::vector<ConePart> dual_cone(const std::vector<ConePart>& c) {  // risk.cpp:25-43
  std::vector<ConePart> d;
  for (const auto& p : c) {
    if (p.kind == ZERO)
      d.push_back({FREE, p.dim});
    else if (p.kind == FREE)
      d.push_back({ZERO, p.dim});
    else
      d.push_back(p);
  }
  return d;
}

void Risk::validate() const {  // risk.cpp:45-63
  require(n > 0, "RiskSpec: n must be positive");
  require(E.c == n, "RiskSpec: E must have n columns");
  require(int(b.size()) == E.r, "RiskSpec: b/E row mismatch");
  require(F.c == 0 || F.r == E.r, "RiskSpec: F/E row mismatch");
  int cd = 0;
  for (const auto& p : cone) cd += p.dim;
  require(cd == E.r, "RiskSpec: cone/E row mismatch");
  if (kind == 0) {
    require(int(pi.size()) == n, "RiskSpec: avar pi has wrong length");
    require(F.c == 0, "RiskSpec: avar specs carry no nu variables");
    const bool standard = E.r == 2 * n + 1;
    const bool max_form = gamma == 0.0 && E.r == n + 1;
    const bool eq_form = gamma == 1.0 && E.r == n;
    require(standard || max_form || eq_form, "RiskSpec: malformed avar representation");
  }
}

void Raocp::validate() const {  // problem.cpp:39-86
  require(tree != nullptr, "Raocp: missing tree");
  require(nx > 0 && nu > 0, "Raocp: dimensions must be positive");
  const int nn = tree->nn(), nnl = tree->nnl(), nl = tree->nl();
  require(int(A.size()) == nn - 1 && int(B.size()) == nn - 1 && int(c.size()) == nn - 1,
          "Raocp: dynamics arrays must cover all non-root nodes");
  require(int(Q.size()) == nn - 1 && int(R.size()) == nn - 1 && int(q.size()) == nn - 1 &&
              int(r.size()) == nn - 1,
          "Raocp: stage cost arrays must cover all non-root nodes");
  require(int(QN.size()) == nl && int(qN.size()) == nl, "Raocp: terminal cost arrays must cover all leaves");
  require(int(Gx.size()) == nnl && int(Gu.size()) == nnl && int(C.size()) == nnl && int(risk.size()) == nnl,
          "Raocp: constraint/risk arrays must cover all non-leaf nodes");
  require(int(GN.size()) == nl && int(CN.size()) == nl,
          "Raocp: terminal constraint arrays must cover all leaves");
  require(int(x_init.size()) == nx, "Raocp: x_init has wrong length");
  for (int i = 1; i < nn; ++i) {
    require(A[i - 1].r == nx && A[i - 1].c == nx, "Raocp: A dimension mismatch");
    require(B[i - 1].r == nx && B[i - 1].c == nu, "Raocp: B dimension mismatch");
    require(int(c[i - 1].size()) == nx, "Raocp: c dimension mismatch");
    require(Q[i - 1].r == nx && Q[i - 1].c == nx, "Raocp: Q dimension mismatch");
    require(R[i - 1].r == nu && R[i - 1].c == nu, "Raocp: R dimension mismatch");
    require(int(q[i - 1].size()) == nx && int(r[i - 1].size()) == nu, "Raocp: q/r dimension mismatch");
    check_symmetric(Q[i - 1], "Raocp Q");
    Mat L;
    require(cholesky(check_symmetric(R[i - 1], "Raocp R"), L), "Raocp: R must be positive definite");
  }
  for (int i = 0; i < nnl; ++i) {
    risk[i].validate();
    require(risk[i].n == tree->child_count[i], "Raocp: risk spec size must match child count");
    require(C[i].lo.size() == C[i].hi.size(), "Box: bound length mismatch");
    for (int k = 0; k < C[i].dim(); ++k) require(C[i].lo[k] <= C[i].hi[k], "Box: lower bound above upper bound");
    require(Gx[i].r == C[i].dim() && Gx[i].c == nx, "Raocp: Gx dimension mismatch");
    require(Gu[i].r == C[i].dim() && Gu[i].c == nu, "Raocp: Gu dimension mismatch");
  }
  for (int j = 0; j < nl; ++j) {
    require(QN[j].r == nx && QN[j].c == nx, "Raocp: QN dimension mismatch");
    require(int(qN[j].size()) == nx, "Raocp: qN dimension mismatch");
    check_symmetric(QN[j], "Raocp QN");
    require(CN[j].lo.size() == CN[j].hi.size(), "Box: bound length mismatch");
    for (int k = 0; k < CN[j].dim(); ++k) require(CN[j].lo[k] <= CN[j].hi[k], "Box: lower bound above upper bound");
    require(GN[j].r == CN[j].dim() && GN[j].c == nx, "Raocp: GN dimension mismatch");
  }
}

// soc_data_quadlin, proj/src/problem.cpp:113-161
SocQuadLin soc_data_quadlin(const Mat& Qin, const Vec& q) {
  const Mat Q = check_symmetric(Qin, "soc_data_quadlin");
  const int n = Q.r;
  require(int(q.size()) == n, "soc_data_quadlin: q dimension mismatch");
  Vec ev;
  Mat V;
  sym_eig(Q, ev, V);
  double lmax = 0.0;
  for (double v : ev) lmax = std::max(lmax, v);
  double lmin = ev.empty() ? 0.0 : *std::min_element(ev.begin(), ev.end());
  require(lmin >= -1e-10 * std::max(lmax, 1.0), "soc_data_quadlin: Q must be positive semidefinite");
  const double thresh = 1e-10 * lmax;
  SocQuadLin d;
  d.n = n;
  d.lambda_max = lmax;
  std::vector<int> keep;
  for (int k = 0; k < n; ++k)
    if (ev[k] > thresh) keep.push_back(k);
  d.p = int(keep.size());
  d.S = Mat(n, d.p);
  for (int k = 0; k < d.p; ++k)
    for (int i = 0; i < n; ++i) d.S(i, k) = V(i, keep[k]);
  d.a.assign(d.p + 2, 0.0);
  double qn2 = 0.0;
  if (d.p > 0) {
    Mat SQS = matmul_tn(d.S, matmul(Q, d.S));
    Vec e2;
    Mat U;
    sym_eig(SQS, e2, U);
    d.sqrt_factor = Mat(d.p, d.p);
    for (int j = 0; j < d.p; ++j)
      for (int i = 0; i < d.p; ++i) {
        double s = 0.0;
        for (int k = 0; k < d.p; ++k) s += U(i, k) * std::sqrt(std::max(0.0, e2[k])) * U(j, k);
        d.sqrt_factor(i, j) = s;
      }
    d.head_map = matmul(d.sqrt_factor, transpose(d.S));
    Vec Sq(d.p, 0.0);
    matvec_t_acc(d.S, q.data(), Sq.data());
    d.q_kernel = q;
    for (int k = 0; k < d.p; ++k)
      for (int i = 0; i < n; ++i) d.q_kernel[i] -= d.S(i, k) * Sq[k];
    Mat Lc;
    require(cholesky(d.sqrt_factor, Lc), "soc_data_quadlin: reduced factor not PD");
    Vec w = Sq;
    chol_solve(Lc, w.data());
    for (int k = 0; k < d.p; ++k) d.a[k] = -0.5 * w[k];
    qn2 = sqnorm(w);
  } else {
    d.sqrt_factor = Mat(0, 0);
    d.head_map = Mat(0, n);
    d.q_kernel = q;
  }
  d.a[d.p] = -0.125 * qn2 + 0.5;
  d.a[d.p + 1] = -0.125 * qn2 - 0.5;
  return d;
}

SocData soc_epigraph_data(const Raocp& p) {  // problem.cpp:216-236
  const int nn = p.tree->nn(), nnl = p.tree->nnl();
  SocData d;
  d.stage.resize(nn - 1);
  d.leaf.resize(nn - nnl);
  const int n = p.nx + p.nu;
  parallel_for(1, nn, [&](int i) {
    Mat Qf(n, n);
    for (int j = 0; j < p.nx; ++j)
      for (int k = 0; k < p.nx; ++k) Qf(k, j) = p.Q[i - 1](k, j);
    for (int j = 0; j < p.nu; ++j)
      for (int k = 0; k < p.nu; ++k) Qf(p.nx + k, p.nx + j) = p.R[i - 1](k, j);
    Vec qf(n);
    for (int k = 0; k < p.nx; ++k) qf[k] = p.q[i - 1][k];
    for (int k = 0; k < p.nu; ++k) qf[p.nx + k] = p.r[i - 1][k];
    d.stage[i - 1] = soc_data_quadlin(Qf, qf);
  }, 1000000);
  parallel_for(nnl, nn, [&](int j) { d.leaf[j - nnl] = soc_data_quadlin(p.QN[j - nnl], p.qN[j - nnl]); },
               1000000);
  return d;
}

Precond identity_precond(const Raocp& p) {  // problem.cpp:238-247
  Precond pc;
  pc.sx.assign(p.nx, 1.0);
  pc.su.assign(p.nu, 1.0);
  pc.sxN.assign(p.nx, 1.0);
  pc.cstr_scale.assign(p.tree->nnl(), 1.0);
  pc.c_hat = 1.0;
  pc.is_identity = true;
  return pc;
}

// precondition, proj/src/problem.cpp:249-326
void precondition(const Raocp& p, Raocp& s, Precond& pc) {
  const Tree& tr = *p.tree;
  const int nn = tr.nn(), nnl = tr.nnl(), nl = tr.nl();
  int max_ch = 1;
  for (int i = 0; i < nnl; ++i) max_ch = std::max(max_ch, tr.child_count[i]);
  pc = Precond{};
  pc.c_hat = std::sqrt(double(max_ch));
  pc.sx.assign(p.nx, 1.0);
  pc.su.assign(p.nu, 1.0);
  pc.sxN.assign(p.nx, 1.0);
  for (int i = 1; i < nn; ++i) {
    for (int k = 0; k < p.nx; ++k) pc.sx[k] = std::max(pc.sx[k], std::sqrt(std::max(0.0, p.Q[i - 1](k, k))));
    for (int k = 0; k < p.nu; ++k) pc.su[k] = std::max(pc.su[k], std::sqrt(std::max(0.0, p.R[i - 1](k, k))));
  }
  for (auto& v : pc.sx) v *= pc.c_hat;
  for (auto& v : pc.su) v *= pc.c_hat;
  for (int j = 0; j < nl; ++j)
    for (int k = 0; k < p.nx; ++k) pc.sxN[k] = std::max(pc.sxN[k], std::sqrt(std::max(0.0, p.QN[j](k, k))));
  Vec isx(p.nx), isu(p.nu), isxN(p.nx);
  for (int k = 0; k < p.nx; ++k) isx[k] = 1.0 / pc.sx[k], isxN[k] = 1.0 / pc.sxN[k];
  for (int k = 0; k < p.nu; ++k) isu[k] = 1.0 / pc.su[k];
  s = p;
  for (int i = 1; i < nn; ++i) {
    const int k = i - 1;
    const Vec& cs = tr.leaf(i) ? pc.sxN : pc.sx;
    for (int jj = 0; jj < p.nx; ++jj)
      for (int ii = 0; ii < p.nx; ++ii) s.A[k](ii, jj) = cs[ii] * p.A[k](ii, jj) * isx[jj];
    for (int jj = 0; jj < p.nu; ++jj)
      for (int ii = 0; ii < p.nx; ++ii) s.B[k](ii, jj) = cs[ii] * p.B[k](ii, jj) * isu[jj];
    for (int ii = 0; ii < p.nx; ++ii) s.c[k][ii] = cs[ii] * p.c[k][ii];
    for (int jj = 0; jj < p.nx; ++jj)
      for (int ii = 0; ii < p.nx; ++ii) s.Q[k](ii, jj) = isx[ii] * p.Q[k](ii, jj) * isx[jj];
    for (int jj = 0; jj < p.nu; ++jj)
      for (int ii = 0; ii < p.nu; ++ii) s.R[k](ii, jj) = isu[ii] * p.R[k](ii, jj) * isu[jj];
    for (int ii = 0; ii < p.nx; ++ii) s.q[k][ii] = isx[ii] * p.q[k][ii];
    for (int ii = 0; ii < p.nu; ++ii) s.r[k][ii] = isu[ii] * p.r[k][ii];
  }
  for (int j = 0; j < nl; ++j) {
    for (int jj = 0; jj < p.nx; ++jj)
      for (int ii = 0; ii < p.nx; ++ii) s.QN[j](ii, jj) = isxN[ii] * p.QN[j](ii, jj) * isxN[jj];
    for (int ii = 0; ii < p.nx; ++ii) s.qN[j][ii] = isxN[ii] * p.qN[j][ii];
  }
  pc.cstr_scale.assign(nnl, 1.0);
  for (int i = 0; i < nnl; ++i) {
    const int nc = p.Gx[i].r;
    Mat st(nc, p.nx + p.nu);
    for (int j = 0; j < p.nx; ++j)
      for (int r = 0; r < nc; ++r) st(r, j) = p.Gx[i](r, j) * isx[j];
    for (int j = 0; j < p.nu; ++j)
      for (int r = 0; r < nc; ++r) st(r, p.nx + j) = p.Gu[i](r, j) * isu[j];
    Vec ev;
    Mat V;
    sym_eig(matmul_tn(st, st), ev, V);
    double emax = ev.empty() ? 0.0 : *std::max_element(ev.begin(), ev.end());
    const double a = std::max(1.0, std::sqrt(std::max(0.0, emax)));
    pc.cstr_scale[i] = a;
    for (int j = 0; j < p.nx; ++j)
      for (int r = 0; r < nc; ++r) s.Gx[i](r, j) = st(r, j) / a;
    for (int j = 0; j < p.nu; ++j)
      for (int r = 0; r < nc; ++r) s.Gu[i](r, j) = st(r, p.nx + j) / a;
    for (int r = 0; r < nc; ++r) {
      s.C[i].lo[r] = p.C[i].lo[r] / a;
      s.C[i].hi[r] = p.C[i].hi[r] / a;
    }
  }
  for (int j = 0; j < nl; ++j)
    for (int jj = 0; jj < p.nx; ++jj)
      for (int r = 0; r < p.GN[j].r; ++r) s.GN[j](r, jj) = p.GN[j](r, jj) * isxN[jj];
  for (int k = 0; k < p.nx; ++k) s.x_init[k] = pc.sx[k] * p.x_init[k];
}

PrimalLayout make_primal_layout(const Raocp& p) {  // layout.cpp:5-30
  const Tree& tr = *p.tree;
  PrimalLayout L;
  L.nx = p.nx;
  L.nu = p.nu;
  L.num_nodes = tr.nn();
  L.num_nonleaf = tr.nnl();
  int off = 1 + L.num_nodes * L.nx;
  L.u_base = off;
  off += L.num_nonleaf * L.nu;
  L.y_off.resize(L.num_nonleaf);
  L.y_dim.resize(L.num_nonleaf);
  for (int i = 0; i < L.num_nonleaf; ++i) {
    L.y_off[i] = off;
    L.y_dim[i] = p.risk[i].rows();
    off += L.y_dim[i];
  }
  L.tau_base = off;
  off += L.num_nodes - 1;
  L.s_base = off;
  off += L.num_nodes - 1;
  L.n = off;
  return L;
}

DualLayout make_dual_layout(const Raocp& p, const SocData& soc) {  // layout.cpp:32-67
  const Tree& tr = *p.tree;
  DualLayout L;
  L.num_nodes = tr.nn();
  L.num_nonleaf = tr.nnl();
  int off = 0;
  L.seg1_off.resize(L.num_nonleaf);
  L.seg1_nc.resize(L.num_nonleaf);
  L.seg1_ydim.resize(L.num_nonleaf);
  for (int i = 0; i < L.num_nonleaf; ++i) {
    L.seg1_off[i] = off;
    L.seg1_ydim[i] = p.risk[i].rows();
    L.seg1_nc[i] = p.C[i].dim();
    off += L.seg1_ydim[i] + 1 + L.seg1_nc[i];
  }
  L.seg2_off.resize(L.num_nodes - 1);
  L.seg2_dim.resize(L.num_nodes - 1);
  for (int i = 1; i < L.num_nodes; ++i) {
    L.seg2_off[i - 1] = off;
    L.seg2_dim[i - 1] = soc.stage[i - 1].p + 2;
    off += L.seg2_dim[i - 1];
  }
  const int nl = tr.nl();
  L.seg3_off.resize(nl);
  L.seg3_nc.resize(nl);
  L.seg3_socdim.resize(nl);
  for (int j = 0; j < nl; ++j) {
    L.seg3_off[j] = off;
    L.seg3_nc[j] = p.CN[j].dim();
    L.seg3_socdim[j] = soc.leaf[j].p + 2;
    off += L.seg3_nc[j] + L.seg3_socdim[j];
  }
  L.n = off;
  return L;
}

}  // namespace orc
