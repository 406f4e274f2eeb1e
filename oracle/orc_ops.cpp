// TEST INFRASTRUCTURE ONLY -- parity oracle (see orc.hpp).
// Restates proj/src/projections.cpp and proj/src/tree_operator.cpp.
#include <algorithm>

#include "orc.hpp"

namespace orc {

// proj_soc_inplace, projections.cpp:11-24
void proj_soc_inplace(double* v, int d) {
  if (d < 2) throw std::invalid_argument("proj_soc: dimension must be >= 2");
  const double t = v[d - 1];
  const double hn = std::sqrt(dot(v, v, d - 1));
  if (hn <= t) return;
  if (hn <= -t) {
    for (int k = 0; k < d; ++k) v[k] = 0.0;
    return;
  }
  const double f = (hn + t) / (2.0 * hn);
  for (int k = 0; k < d - 1; ++k) v[k] *= f;
  v[d - 1] = 0.5 * (hn + t);
}

// proj_cone_inplace, projections.cpp:39-57
void proj_cone_inplace(const std::vector<ConePart>& cone, double* v) {
  int off = 0;
  for (const auto& p : cone) {
    if (p.kind == ZERO)
      for (int k = 0; k < p.dim; ++k) v[off + k] = 0.0;
    else if (p.kind == NONNEG)
      for (int k = 0; k < p.dim; ++k) v[off + k] = std::max(v[off + k], 0.0);
    else if (p.kind == SOC)
      proj_soc_inplace(v + off, p.dim);
    off += p.dim;
  }
}

// make_solver_cache, projections.cpp:59-140
SolverCache make_solver_cache(const Raocp& p) {
  const Tree& tr = *p.tree;
  const int nn = tr.nn(), nnl = tr.nnl(), N = tr.horizon, nx = p.nx, nu = p.nu;
  SolverCache c;
  c.P.resize(nn);
  c.K.resize(nnl);
  c.Rt.resize(nnl);
  c.RtL.resize(nnl);
  c.Abar.resize(nn - 1);
  c.s2_proj.resize(nnl);
  c.q_scr.assign(nn, Vec(nx, 0.0));
  c.d_scr.assign(nnl, Vec(nu, 0.0));
  c.term_u.assign(nn - 1, Vec(nu, 0.0));
  c.term_x.assign(nn - 1, Vec(nx, 0.0));
  const uint64_t dyn = 2ull * nx * nx * (nx + nu);
  stage_parallel_for(tr, N, [&](int j) { c.P[j] = Mat::eye(nx); });
  std::vector<Mat> rt_term(nn - 1), k_term(nn - 1), p_term(nn - 1);
  for (int t = N - 1; t >= 0; --t) {
    stage_parallel_for(tr, t + 1, [&](int ip) {
      const Mat pb = matmul(c.P[ip], p.B[ip - 1]);
      rt_term[ip - 1] = matmul_tn(p.B[ip - 1], pb);
      k_term[ip - 1] = matmul_tn(p.B[ip - 1], matmul(c.P[ip], p.A[ip - 1]));
    }, 2 * dyn);
    stage_parallel_for(tr, t, [&](int i) {
      Mat rt = Mat::eye(nu), kt(nu, nx);
      for (int k = 0; k < tr.child_count[i]; ++k) {
        const int ip = tr.child_first[i] + k;
        rt = add(rt, rt_term[ip - 1]);
        kt = add(kt, k_term[ip - 1]);
      }
      c.Rt[i] = rt;
      if (!cholesky(rt, c.RtL[i]))
        throw std::runtime_error("make_solver_cache: Cholesky failed (corrupt dynamics data)");
      Mat K(nu, nx);
      for (int j = 0; j < nx; ++j) {
        Vec col(kt.col(j), kt.col(j) + nu);
        chol_solve(c.RtL[i], col.data());
        for (int r = 0; r < nu; ++r) K(r, j) = -col[r];
      }
      c.K[i] = K;
    }, dyn);
    stage_parallel_for(tr, t + 1, [&](int ip) {
      const int i = tr.anc[ip];
      c.Abar[ip - 1] = add(p.A[ip - 1], matmul(p.B[ip - 1], c.K[i]));
      p_term[ip - 1] = matmul_tn(c.Abar[ip - 1], matmul(c.P[ip], c.Abar[ip - 1]));
    }, 2 * dyn);
    stage_parallel_for(tr, t, [&](int i) {
      Mat pi = add(Mat::eye(nx), matmul_tn(c.K[i], c.K[i]));
      for (int k = 0; k < tr.child_count[i]; ++k) pi = add(pi, p_term[tr.child_first[i] + k - 1]);
      c.P[i] = pi;
    }, dyn);
  }
  parallel_for(0, nnl, [&](int i) {
    const Risk& rs = p.risk[i];
    const int nch = tr.child_count[i], ny = rs.rows(), nnu = rs.F.c, dim = ny + 2 * nch;
    Mat M(nch + nnu, dim);
    for (int j = 0; j < ny; ++j)
      for (int k = 0; k < nch; ++k) M(k, j) = rs.E(j, k);
    for (int k = 0; k < nch; ++k) {
      M(k, ny + k) = -1.0;
      M(k, ny + nch + k) = -1.0;
    }
    for (int j = 0; j < ny; ++j)
      for (int k = 0; k < nnu; ++k) M(nch + k, j) = rs.F(j, k);
    c.s2_proj[i] = kernel_projector(M);
  }, 100000);
  return c;
}

// proj_s1, projections.cpp:142-187
void proj_s1(const Raocp& p, SolverCache& c, const PrimalLayout& zl, const Vec& x_init, double* z) {
  const Tree& tr = *p.tree;
  const int N = tr.horizon, nx = zl.nx, nu = zl.nu;
  const uint64_t mv = 2ull * nx * (nx + nu);
  stage_parallel_for(tr, N, [&](int j) {
    for (int k = 0; k < nx; ++k) c.q_scr[j][k] = -z[zl.x(j) + k];
  }, nx);
  for (int t = N - 1; t >= 0; --t) {
    stage_parallel_for(tr, t + 1, [&](int ip) {
      Vec tmp = c.q_scr[ip];
      matvec_acc(c.P[ip], p.c[ip - 1].data(), tmp.data());
      Vec& tu = c.term_u[ip - 1];
      std::fill(tu.begin(), tu.end(), 0.0);
      matvec_t_acc(p.B[ip - 1], tmp.data(), tu.data());
    }, mv);
    stage_parallel_for(tr, t, [&](int i) {
      Vec dbar(nu, 0.0);
      for (int k = 0; k < tr.child_count[i]; ++k) {
        const Vec& tu = c.term_u[tr.child_first[i] + k - 1];
        for (int r = 0; r < nu; ++r) dbar[r] += tu[r];
      }
      Vec d(nu);
      for (int r = 0; r < nu; ++r) d[r] = z[zl.u(i) + r] - dbar[r];
      chol_solve(c.RtL[i], d.data());
      c.d_scr[i] = d;
    }, mv);
    stage_parallel_for(tr, t + 1, [&](int ip) {
      const int i = tr.anc[ip];
      Vec bd = matvec(p.B[ip - 1], c.d_scr[i].data());
      for (int k = 0; k < nx; ++k) bd[k] += p.c[ip - 1][k];
      Vec pv = matvec(c.P[ip], bd.data());
      for (int k = 0; k < nx; ++k) pv[k] += c.q_scr[ip][k];
      Vec& tx = c.term_x[ip - 1];
      std::fill(tx.begin(), tx.end(), 0.0);
      matvec_t_acc(c.Abar[ip - 1], pv.data(), tx.data());
    }, 2 * mv);
    stage_parallel_for(tr, t, [&](int i) {
      Vec du(nu);
      for (int r = 0; r < nu; ++r) du[r] = c.d_scr[i][r] - z[zl.u(i) + r];
      Vec qi(nx, 0.0);
      matvec_t_acc(c.K[i], du.data(), qi.data());
      for (int k = 0; k < nx; ++k) qi[k] -= z[zl.x(i) + k];
      for (int kk = 0; kk < tr.child_count[i]; ++kk) {
        const Vec& tx = c.term_x[tr.child_first[i] + kk - 1];
        for (int k = 0; k < nx; ++k) qi[k] += tx[k];
      }
      c.q_scr[i] = qi;
    }, mv);
  }
  for (int k = 0; k < nx; ++k) z[zl.x(0) + k] = x_init[k];
  for (int t = 0; t < N; ++t) {
    stage_parallel_for(tr, t, [&](int i) {
      Vec u = matvec(c.K[i], z + zl.x(i));
      for (int r = 0; r < nu; ++r) z[zl.u(i) + r] = u[r] + c.d_scr[i][r];
    }, mv);
    stage_parallel_for(tr, t + 1, [&](int ip) {
      const int i = tr.anc[ip];
      Vec x = matvec(p.A[ip - 1], z + zl.x(i));
      matvec_acc(p.B[ip - 1], z + zl.u(i), x.data());
      for (int k = 0; k < nx; ++k) z[zl.x(ip) + k] = x[k] + p.c[ip - 1][k];
    }, mv);
  }
}

// proj_s2, projections.cpp:189-210
void proj_s2(const Raocp& p, const SolverCache& c, const PrimalLayout& zl, double* z) {
  const Tree& tr = *p.tree;
  uint64_t fl = 0;
  for (int i = 0; i < tr.nnl(); ++i) {
    const uint64_t d = uint64_t(zl.y_dim[i]) + 2 * tr.child_count[i];
    fl = std::max(fl, 2 * d * d);
  }
  parallel_for(0, tr.nnl(), [&](int i) {
    const int nch = tr.child_count[i], ny = zl.y_dim[i], cf = tr.child_first[i];
    Vec w(ny + 2 * nch);
    for (int k = 0; k < ny; ++k) w[k] = z[zl.y(i) + k];
    for (int k = 0; k < nch; ++k) {
      w[ny + k] = z[zl.tau(cf + k)];
      w[ny + nch + k] = z[zl.s(cf + k)];
    }
    const Vec o = matvec(c.s2_proj[i], w.data());
    for (int k = 0; k < ny; ++k) z[zl.y(i) + k] = o[k];
    for (int k = 0; k < nch; ++k) {
      z[zl.tau(cf + k)] = o[ny + k];
      z[zl.s(cf + k)] = o[ny + nch + k];
    }
  }, fl);
}

// proj_s3, projections.cpp:212-244
void proj_s3(const Raocp& p, const SocData& soc, const DualLayout& el,
             const std::vector<std::vector<ConePart>>& dk, double* eta) {
  const Tree& tr = *p.tree;
  const int nn = tr.nn(), nnl = tr.nnl();
  parallel_for(0, nn, [&](int i) {
    if (i < nnl) {
      proj_cone_inplace(dk[i], eta + el.y_copy(i));
      double& sc = eta[el.risk_scalar(i)];
      sc = std::max(0.0, sc);
      double* e = eta + el.cstr(i);
      for (int k = 0; k < el.seg1_nc[i]; ++k) e[k] = std::min(std::max(e[k], p.C[i].lo[k]), p.C[i].hi[k]);
    }
    if (i > 0) {
      const auto& d = soc.stage[i - 1];
      double* seg = eta + el.stage_soc(i);
      const int dim = el.seg2_dim[i - 1];
      for (int k = 0; k < dim; ++k) seg[k] -= d.a[k];
      proj_soc_inplace(seg, dim);
      for (int k = 0; k < dim; ++k) seg[k] += d.a[k];
    }
    if (i >= nnl) {
      const int j = i - nnl;
      double* e = eta + el.leaf_cstr(j);
      for (int k = 0; k < el.seg3_nc[j]; ++k) e[k] = std::min(std::max(e[k], p.CN[j].lo[k]), p.CN[j].hi[k]);
      const auto& d = soc.leaf[j];
      double* seg = eta + el.leaf_soc(j);
      const int dim = el.seg3_socdim[j];
      for (int k = 0; k < dim; ++k) seg[k] -= d.a[k];
      proj_soc_inplace(seg, dim);
      for (int k = 0; k < dim; ++k) seg[k] += d.a[k];
    }
  }, 8ull * (p.nx + p.nu));
}

// ---------------- TreeOperator, proj/src/tree_operator.cpp ----------------
TreeOperator::TreeOperator(const Raocp& p, const SocData& soc)
    : p_(&p), soc_(&soc), zl_(make_primal_layout(p)), el_(make_dual_layout(p, soc)) {
  for (int i = 0; i < p.tree->nnl(); ++i) dk_.push_back(dual_cone(p.risk[i].cone));
  adj_.assign(p.tree->nn() - 1, Vec(p.nx + p.nu, 0.0));
  mscr_.resize(el_.n);
}

// TreeOperator::apply, tree_operator.cpp:20-63
void TreeOperator::apply(const Vec& z, Vec& eta) const {
  const Raocp& p = *p_;
  const Tree& tr = *p.tree;
  const int nn = tr.nn(), nnl = tr.nnl(), nx = p.nx, nu = p.nu;
  eta.assign(el_.n, 0.0);
  parallel_for(0, nn, [&](int i) {
    if (i < nnl) {
      const int ny = el_.seg1_ydim[i];
      for (int k = 0; k < ny; ++k) eta[el_.y_copy(i) + k] = z[zl_.y(i) + k];
      eta[el_.risk_scalar(i)] = z[zl_.s(i)] - dot(p.risk[i].b.data(), z.data() + zl_.y(i), ny);
      double* e = eta.data() + el_.cstr(i);
      Vec g = matvec(p.Gx[i], z.data() + zl_.x(i));
      matvec_acc(p.Gu[i], z.data() + zl_.u(i), g.data());
      for (int k = 0; k < el_.seg1_nc[i]; ++k) e[k] = g[k];
    }
    if (i > 0) {
      const auto& d = soc_->stage[i - 1];
      const int a = tr.anc[i];
      const double* x = z.data() + zl_.x(a);
      const double* u = z.data() + zl_.u(a);
      double* seg = eta.data() + el_.stage_soc(i);
      for (int r = 0; r < d.p; ++r) {
        double s = 0.0;
        for (int k = 0; k < nx; ++k) s += d.head_map(r, k) * x[k];
        double s2 = 0.0;
        for (int k = 0; k < nu; ++k) s2 += d.head_map(r, nx + k) * u[k];
        seg[r] = s + s2;
      }
      const double row = 0.5 * z[zl_.tau(i)] -
                         0.5 * (dot(d.q_kernel.data(), x, nx) + dot(d.q_kernel.data() + nx, u, nu));
      seg[d.p] = row;
      seg[d.p + 1] = row;
    }
    if (i >= nnl) {
      const int j = i - nnl;
      const double* x = z.data() + zl_.x(i);
      Vec g = matvec(p.GN[j], x);
      for (int k = 0; k < el_.seg3_nc[j]; ++k) eta[el_.leaf_cstr(j) + k] = g[k];
      const auto& d = soc_->leaf[j];
      double* seg = eta.data() + el_.leaf_soc(j);
      if (d.p > 0) {
        Vec h = matvec(d.head_map, x);
        for (int r = 0; r < d.p; ++r) seg[r] = h[r];
      }
      const double row = 0.5 * z[zl_.s(i)] - 0.5 * dot(d.q_kernel.data(), x, nx);
      seg[d.p] = row;
      seg[d.p + 1] = row;
    }
  }, 4ull * (nx + nu) * (nx + nu));
}

// TreeOperator::apply_adjoint, tree_operator.cpp:65-114
void TreeOperator::apply_adjoint(const Vec& eta, Vec& z) const {
  const Raocp& p = *p_;
  const Tree& tr = *p.tree;
  const int nn = tr.nn(), nnl = tr.nnl(), nx = p.nx, nu = p.nu;
  z.assign(zl_.n, 0.0);
  parallel_for(0, nn, [&](int i) {
    if (i < nnl) {
      const int ny = el_.seg1_ydim[i];
      const double sc = eta[el_.risk_scalar(i)];
      for (int k = 0; k < ny; ++k) z[zl_.y(i) + k] = eta[el_.y_copy(i) + k] - sc * p.risk[i].b[k];
      z[zl_.s(i)] += sc;
      const double* ec = eta.data() + el_.cstr(i);
      matvec_t_acc(p.Gx[i], ec, z.data() + zl_.x(i));
      matvec_t_acc(p.Gu[i], ec, z.data() + zl_.u(i));
    }
    if (i > 0) {
      const auto& d = soc_->stage[i - 1];
      const double* seg = eta.data() + el_.stage_soc(i);
      const double rsum = seg[d.p] + seg[d.p + 1];
      Vec& t = adj_[i - 1];
      for (int k = 0; k < nx + nu; ++k) t[k] = -0.5 * rsum * d.q_kernel[k];
      if (d.p > 0) matvec_t_acc(d.head_map, seg, t.data());
      z[zl_.tau(i)] = 0.5 * rsum;
    }
    if (i >= nnl) {
      const int j = i - nnl;
      const auto& d = soc_->leaf[j];
      const double* seg = eta.data() + el_.leaf_soc(j);
      const double rsum = seg[d.p] + seg[d.p + 1];
      double* zx = z.data() + zl_.x(i);
      matvec_t_acc(p.GN[j], eta.data() + el_.leaf_cstr(j), zx);
      if (d.p > 0) matvec_t_acc(d.head_map, seg, zx);
      for (int k = 0; k < nx; ++k) zx[k] -= 0.5 * rsum * d.q_kernel[k];
      z[zl_.s(i)] += 0.5 * rsum;
    }
  }, 4ull * (nx + nu) * (nx + nu));
  parallel_for(0, nnl, [&](int i) {
    for (int k = 0; k < tr.child_count[i]; ++k) {
      const Vec& t = adj_[tr.child_first[i] + k - 1];
      for (int r = 0; r < nx; ++r) z[zl_.x(i) + r] += t[r];
      for (int r = 0; r < nu; ++r) z[zl_.u(i) + r] += t[nx + r];
    }
  }, uint64_t(nx + nu));
}

namespace {
double holder_bound(const Mat& A) {  // tree_operator.cpp:116-124
  if (A.a.empty()) return 0.0;
  double n1 = 0.0, ninf = 0.0;
  for (int j = 0; j < A.c; ++j) {
    double s = 0.0;
    for (int i = 0; i < A.r; ++i) s += std::fabs(A(i, j));
    n1 = std::max(n1, s);
  }
  for (int i = 0; i < A.r; ++i) {
    double s = 0.0;
    for (int j = 0; j < A.c; ++j) s += std::fabs(A(i, j));
    ninf = std::max(ninf, s);
  }
  return std::sqrt(n1 * ninf);
}
}  // namespace

// analytic_norm_bound, tree_operator.cpp:126-155
double TreeOperator::analytic_norm_bound() const {
  const Raocp& p = *p_;
  const Tree& tr = *p.tree;
  const int nn = tr.nn(), nnl = tr.nnl();
  int max_ch = 1;
  for (int i = 0; i < nnl; ++i) max_ch = std::max(max_ch, tr.child_count[i]);
  double mx = 0.0;
  for (int i = 0; i < nn; ++i) {
    if (i < nnl) {
      mx = std::max(mx, 1.0);
      mx = std::max(mx, std::sqrt(1.0 + sqnorm(p.risk[i].b)));
      Mat g(p.Gx[i].r, p.nx + p.nu);
      for (int j = 0; j < p.nx; ++j)
        for (int r = 0; r < g.r; ++r) g(r, j) = p.Gx[i](r, j);
      for (int j = 0; j < p.nu; ++j)
        for (int r = 0; r < g.r; ++r) g(r, p.nx + j) = p.Gu[i](r, j);
      mx = std::max(mx, holder_bound(g));
    }
    if (i > 0) {
      const auto& d = soc_->stage[i - 1];
      mx = std::max(mx, std::sqrt(d.lambda_max + 0.5 * (1.0 + sqnorm(d.q_kernel))));
    }
    if (i >= nnl) {
      const auto& d = soc_->leaf[i - nnl];
      mx = std::max(mx, holder_bound(p.GN[i - nnl]));
      mx = std::max(mx, std::sqrt(d.lambda_max + 0.5 * (1.0 + sqnorm(d.q_kernel))));
    }
  }
  return std::sqrt(1.0 + double(max_ch)) * mx;
}

// estimate_norm, tree_operator.cpp:157-205
OpNormEstimate estimate_norm(int nz, int neta, const std::function<void(const Vec&, Vec&)>& apply,
                             const std::function<void(const Vec&, Vec&)>& adj, double bound, double tol,
                             int max_iters) {
  Philox rng(0x9E3779B97F4A7C15ull);
  Vec v(nz);
  for (int k = 0; k < nz; ++k) v[k] = rng.normal();
  double vn = std::sqrt(sqnorm(v));
  for (auto& x : v) x /= vn;
  Vec u(neta), w(nz);
  OpNormEstimate out;
  out.analytic_bound = bound;
  double prev = 0.0, prev_change = 0.0;
  for (int it = 1; it <= max_iters; ++it) {
    apply(v, u);
    const double est = std::sqrt(sqnorm(u));
    out.estimate = est;
    out.iterations = it;
    if (est == 0.0) {
      out.converged = true;
      break;
    }
    if (it > 2) {
      const double change = std::fabs(est - prev);
      double ratio = prev_change > 0.0 ? change / prev_change : 0.0;
      ratio = std::min(ratio, 0.999);
      const double remaining = change * ratio / (1.0 - ratio);
      if (change + remaining <= tol * est) {
        out.converged = true;
        break;
      }
      prev_change = change;
    } else if (it == 2) {
      prev_change = std::fabs(est - prev);
    }
    prev = est;
    adj(u, w);
    const double wn = std::sqrt(sqnorm(w));
    if (wn == 0.0) {
      out.converged = true;
      break;
    }
    for (int k = 0; k < nz; ++k) v[k] = w[k] / wn;
  }
  return out;
}

OpNormEstimate TreeOperator::estimate_norm(double tol, int max_iters) const {
  return orc::estimate_norm(
      zl_.n, el_.n, [this](const Vec& z, Vec& e) { apply(z, e); },
      [this](const Vec& e, Vec& z) { apply_adjoint(e, z); }, analytic_norm_bound(), tol, max_iters);
}

// m_norm, tree_operator.cpp:214-222
double TreeOperator::m_norm(const Vec& z, const Vec& eta, double alpha) const {
  apply(z, mscr_);
  const double zz = sqnorm(z), ee = sqnorm(eta);
  const double rad = zz - 2.0 * alpha * dot(eta.data(), mscr_.data(), eta.size()) + ee;
  if (rad < -1e-12 * std::max(1.0, zz + ee))
    throw std::runtime_error("m_norm: negative radicand (alpha violates alpha*||L|| < 1)");
  return std::sqrt(std::max(0.0, rad));
}

}  // namespace orc
