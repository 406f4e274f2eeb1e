// TEST INFRASTRUCTURE ONLY -- parity oracle (see orc.hpp).
// Flat C interface of the oracle.  It takes the same spock_problem_desc as the
// product's C-ABI (include/spock_b200.h) so tests feed both byte-identical
// problems.  Functions are prefixed oracle_ and mirror spock_*.
#include <chrono>
#include <cstring>
#include <thread>

#include "../include/spock_b200.h"
#include "orc.hpp"

using namespace orc;

namespace {
thread_local std::string g_err;

Mat take(const double*& p, int r, int c) {
  Mat m(r, c);
  std::memcpy(m.a.data(), p, sizeof(double) * size_t(r) * c);
  p += size_t(r) * c;
  return m;
}
Vec takev(const double*& p, int n) {
  Vec v(p, p + n);
  p += n;
  return v;
}

Raocp from_desc(const spock_problem_desc* d) {
  Raocp P;
  auto tr = std::make_shared<Tree>();
  const int nn = d->num_nodes;
  if (nn <= 0) throw std::invalid_argument("ScenarioTree: empty tree");
  tr->anc.assign(d->anc, d->anc + nn);
  tr->event.assign(d->event, d->event + nn);
  tr->prob.assign(d->prob, d->prob + nn);
  tr->cond_prob.assign(d->cond_prob, d->cond_prob + nn);
  tr->stop_stage = d->stop_stage;
  tr->num_events = d->num_events;
  tr->finalize();
  if (tr->horizon != d->horizon) throw std::invalid_argument("from_arrays: horizon mismatch");
  P.tree = tr;
  P.nx = d->nx;
  P.nu = d->nu;
  const int nx = d->nx, nu = d->nu, nnl = tr->nnl(), nl = tr->nl();
  if (nx <= 0 || nu <= 0) throw std::invalid_argument("Raocp: dimensions must be positive");
  const double *A = d->A, *B = d->B, *c = d->c, *Q = d->Q, *R = d->R, *q = d->q, *r = d->r;
  for (int i = 1; i < nn; ++i) {
    P.A.push_back(take(A, nx, nx));
    P.B.push_back(take(B, nx, nu));
    P.c.push_back(takev(c, nx));
    P.Q.push_back(take(Q, nx, nx));
    P.R.push_back(take(R, nu, nu));
    P.q.push_back(takev(q, nx));
    P.r.push_back(takev(r, nu));
  }
  const double *QN = d->QN, *qN = d->qN;
  for (int j = 0; j < nl; ++j) {
    P.QN.push_back(take(QN, nx, nx));
    P.qN.push_back(takev(qN, nx));
  }
  const double *Gx = d->Gx, *Gu = d->Gu, *lo = d->C_lo, *hi = d->C_hi;
  const double *E = d->risk_E, *F = d->risk_F, *b = d->risk_b, *pi = d->risk_pi;
  const int *ck = d->cone_kind, *cd = d->cone_dim;
  for (int i = 0; i < nnl; ++i) {
    const int nc = d->nc[i];
    P.Gx.push_back(take(Gx, nc, nx));
    P.Gu.push_back(take(Gu, nc, nu));
    Box bx;
    bx.lo = takev(lo, nc);
    bx.hi = takev(hi, nc);
    P.C.push_back(bx);
    Risk rs;
    rs.kind = d->risk_kind[i];
    rs.n = tr->child_count[i];
    const int rows = d->risk_rows[i], nnu = d->risk_nnu[i];
    rs.E = take(E, rows, rs.n);
    rs.F = nnu > 0 ? take(F, rows, nnu) : Mat(rows, 0);
    rs.b = takev(b, rows);
    rs.gamma = d->risk_gamma[i];
    if (rs.kind == 0) rs.pi = takev(pi, rs.n);
    for (int k = 0; k < d->cone_nparts[i]; ++k) rs.cone.push_back({*ck++, *cd++});
    P.risk.push_back(rs);
  }
  const double *GN = d->GN, *lN = d->CN_lo, *hN = d->CN_hi;
  for (int j = 0; j < nl; ++j) {
    const int nc = d->ncN[j];
    P.GN.push_back(take(GN, nc, nx));
    Box bx;
    bx.lo = takev(lN, nc);
    bx.hi = takev(hN, nc);
    P.CN.push_back(bx);
  }
  P.x_init.assign(d->x_init, d->x_init + nx);
  return P;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return SPOCK_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return SPOCK_EINVAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SPOCK_ERUNTIME;
  }
}

struct OSolver {
  std::unique_ptr<SpockSolver> s;
  Raocp raw;
  spock_params prm;
};

Params to_params(const spock_params* p) {
  Params q;
  if (!p) return q;
  q.eps_abs = p->eps_abs;
  q.eps_rel = p->eps_rel;
  q.alpha = p->alpha;
  q.aa_memory = p->aa_memory;
  q.c0 = p->c0, q.c1 = p->c1, q.c2 = p->c2;
  q.beta = p->beta, q.sigma = p->sigma, q.lambda = p->lambda;
  q.max_iters = p->max_iters;
  q.max_backtracks = p->max_backtracks;
  q.use_preconditioner = p->use_preconditioner != 0;
  if (p->progress) {
    auto f = p->progress;
    void* u = p->user;
    q.progress = [f, u](int k, double w, char b) { f(k, w, b, u); };
  }
  if (p->cancelled) {
    auto f = p->cancelled;
    void* u = p->user;
    q.cancelled = [f, u]() { return f(u) != 0; };
  }
  return q;
}

void fill_status(const Status& s, spock_status* o) {
  if (!o) return;
  o->iterations = s.iterations;
  o->reason = s.reason;
  o->xi1_inf = s.xi1_inf;
  o->xi2_inf = s.xi2_inf;
  o->k0_steps = s.k0;
  o->k1_steps = s.k1;
  o->k2_steps = s.k2;
  o->stalled_steps = s.stalled;
  o->alpha = s.alpha;
  o->op_norm_estimate = s.op_norm.estimate;
  o->op_norm_iterations = s.op_norm.iterations;
  o->op_norm_analytic_bound = s.op_norm.analytic_bound;
  o->op_norm_converged = s.op_norm.converged;
  const int n = int(s.rnorm_history.size());
  int w = 0;
  for (; w < n && w < o->history_capacity; ++w) {
    if (o->rnorm_history) o->rnorm_history[w] = s.rnorm_history[w];
    if (o->branch_history) o->branch_history[w] = s.branches[w];
  }
  o->history_len = n;
  o->n_T = s.n_T;
  o->n_L = s.n_L;
  o->n_Lt = s.n_Lt;
}
}  // namespace

extern "C" {

const char* oracle_last_error(void) { return g_err.c_str(); }
void oracle_set_num_threads(int n) { set_num_threads(n); }
int oracle_num_threads(void) { return num_threads(); }

int oracle_solver_create(const spock_problem_desc* d, const spock_params* p, void** out) {
  return guard([&] {
    auto os = std::make_unique<OSolver>();
    os->raw = from_desc(d);
    os->s = std::make_unique<SpockSolver>(os->raw, to_params(p));
    *out = os.release();
  });
}
void oracle_solver_destroy(void* h) { delete static_cast<OSolver*>(h); }

static SpockSolver& S(void* h) { return *static_cast<OSolver*>(h)->s; }

int oracle_solver_dims(void* h, int64_t* nz, int64_t* ne) {
  *nz = S(h).oper().zlay().n;
  *ne = S(h).oper().elay().n;
  return 0;
}
double oracle_solver_alpha(void* h) { return S(h).alpha(); }
void oracle_opnorm(void* h, double* est, int* iters, double* bound, int* conv) {
  const auto& n = S(h).op_norm();
  *est = n.estimate;
  *iters = n.iterations;
  *bound = n.analytic_bound;
  *conv = n.converged;
}

static int do_solve(void* h, const double* x0, const double* wz, const double* we, double* oz, double* ozs,
                    double* oe, spock_status* st, bool sm) {
  return guard([&] {
    SpockSolver& s = S(h);
    const int nx = s.scaled().nx;
    Vec x = x0 ? Vec(x0, x0 + nx) : s.x_init_orig();
    const int nz = s.oper().zlay().n, ne = s.oper().elay().n;
    Vec vz, ve;
    if (wz) vz.assign(wz, wz + nz);
    if (we) ve.assign(we, we + ne);
    SolveResult r = s.solve(x, wz ? &vz : nullptr, we ? &ve : nullptr, sm);
    if (oz) std::memcpy(oz, r.z.data(), sizeof(double) * nz);
    if (ozs) std::memcpy(ozs, r.z_scaled.data(), sizeof(double) * nz);
    if (oe) std::memcpy(oe, r.eta.data(), sizeof(double) * ne);
    fill_status(r.status, st);
  });
}
int oracle_solver_solve(void* h, const double* x0, const double* wz, const double* we, double* oz, double* ozs,
                        double* oe, spock_status* st) {
  return do_solve(h, x0, wz, we, oz, ozs, oe, st, true);
}
int oracle_solver_solve_cp(void* h, const double* x0, const double* wz, const double* we, double* oz,
                           double* ozs, double* oe, spock_status* st) {
  return do_solve(h, x0, wz, we, oz, ozs, oe, st, false);
}

int oracle_apply_T(void* h, const double* z, const double* e, double* zo, double* eo) {
  return guard([&] {
    SpockSolver& s = S(h);
    const int nz = s.oper().zlay().n, ne = s.oper().elay().n;
    Vec a(z, z + nz), b(e, e + ne), c, d;
    s.apply_T(a, b, c, d);
    std::memcpy(zo, c.data(), sizeof(double) * nz);
    std::memcpy(eo, d.data(), sizeof(double) * ne);
  });
}
// Times k back-to-back CP applications v <- T(v) (CPU baseline); returns ms.
int oracle_bench_T(void* h, int k, double* ms) {
  return guard([&] {
    SpockSolver& s = S(h);
    const int nz = s.oper().zlay().n, ne = s.oper().elay().n;
    Vec z(nz, 0.0), e(ne, 0.0), z2, e2;
    const auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < k; ++i) {
      s.apply_T(z, e, z2, e2);
      z.swap(z2);
      e.swap(e2);
    }
    *ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  });
}
int oracle_apply_L(void* h, const double* z, double* e) {
  return guard([&] {
    SpockSolver& s = S(h);
    Vec a(z, z + s.oper().zlay().n), o;
    s.oper().apply(a, o);
    std::memcpy(e, o.data(), sizeof(double) * o.size());
  });
}
int oracle_apply_Lt(void* h, const double* e, double* z) {
  return guard([&] {
    SpockSolver& s = S(h);
    Vec a(e, e + s.oper().elay().n), o;
    s.oper().apply_adjoint(a, o);
    std::memcpy(z, o.data(), sizeof(double) * o.size());
  });
}
int oracle_m_norm(void* h, const double* z, const double* e, double alpha, double* out) {
  return guard([&] {
    SpockSolver& s = S(h);
    Vec a(z, z + s.oper().zlay().n), b(e, e + s.oper().elay().n);
    *out = s.oper().m_norm(a, b, alpha);
  });
}
int oracle_proj_s1(void* h, double* z) {
  return guard([&] {
    SpockSolver& s = S(h);
    proj_s1(s.scaled(), s.cache(), s.oper().zlay(), s.scaled().x_init, z);
  });
}
int oracle_proj_s2(void* h, double* z) {
  return guard([&] { proj_s2(S(h).scaled(), S(h).cache(), S(h).oper().zlay(), z); });
}
int oracle_proj_s3(void* h, double* e) {
  return guard([&] {
    SpockSolver& s = S(h);
    proj_s3(s.scaled(), s.soc(), s.oper().elay(), s.oper().dual_cones(), e);
  });
}
int oracle_unscale_primal(void* h, const double* zs, double* z) {
  return guard([&] {
    SpockSolver& s = S(h);
    Vec a(zs, zs + s.oper().zlay().n);
    Vec o = s.unscale_primal(a);
    std::memcpy(z, o.data(), sizeof(double) * o.size());
  });
}

// ---- setup exports for parity tests ----
// primal layout: u_base, tau_base, s_base; y_off[nnl], y_dim[nnl]
void oracle_primal_layout(void* h, int* bases, int* y_off, int* y_dim) {
  const auto& zl = S(h).oper().zlay();
  bases[0] = zl.u_base;
  bases[1] = zl.tau_base;
  bases[2] = zl.s_base;
  for (int i = 0; i < zl.num_nonleaf; ++i) y_off[i] = zl.y_off[i], y_dim[i] = zl.y_dim[i];
}
// dual layout arrays: seg1_off/nc/ydim [nnl], seg2_off/dim [nn-1], seg3_off/nc/socdim [nl]
void oracle_dual_layout(void* h, int* s1o, int* s1n, int* s1y, int* s2o, int* s2d, int* s3o, int* s3n, int* s3s) {
  const auto& el = S(h).oper().elay();
  for (int i = 0; i < el.num_nonleaf; ++i) s1o[i] = el.seg1_off[i], s1n[i] = el.seg1_nc[i], s1y[i] = el.seg1_ydim[i];
  for (int i = 0; i < el.num_nodes - 1; ++i) s2o[i] = el.seg2_off[i], s2d[i] = el.seg2_dim[i];
  for (size_t j = 0; j < el.seg3_off.size(); ++j)
    s3o[j] = el.seg3_off[j], s3n[j] = el.seg3_nc[j], s3s[j] = el.seg3_socdim[j];
}
// SOC data of one node: which = 0 stage (index node-1), 1 leaf (index j)
int oracle_soc_dims(void* h, int which, int idx, int* n, int* p, double* lmax) {
  const auto& d = which == 0 ? S(h).soc().stage[idx] : S(h).soc().leaf[idx];
  *n = d.n;
  *p = d.p;
  *lmax = d.lambda_max;
  return 0;
}
void oracle_soc_data(void* h, int which, int idx, double* head_map, double* q_kernel, double* a, double* sqrt_factor) {
  const auto& d = which == 0 ? S(h).soc().stage[idx] : S(h).soc().leaf[idx];
  if (head_map) std::memcpy(head_map, d.head_map.a.data(), sizeof(double) * d.head_map.a.size());
  if (q_kernel) std::memcpy(q_kernel, d.q_kernel.data(), sizeof(double) * d.q_kernel.size());
  if (a) std::memcpy(a, d.a.data(), sizeof(double) * d.a.size());
  if (sqrt_factor) std::memcpy(sqrt_factor, d.sqrt_factor.a.data(), sizeof(double) * d.sqrt_factor.a.size());
}
void oracle_precond(void* h, double* sx, double* su, double* sxN, double* cstr, double* chat, int* ident) {
  const auto& pc = S(h).precond();
  std::memcpy(sx, pc.sx.data(), sizeof(double) * pc.sx.size());
  std::memcpy(su, pc.su.data(), sizeof(double) * pc.su.size());
  std::memcpy(sxN, pc.sxN.data(), sizeof(double) * pc.sxN.size());
  std::memcpy(cstr, pc.cstr_scale.data(), sizeof(double) * pc.cstr_scale.size());
  *chat = pc.c_hat;
  *ident = pc.is_identity;
}
// scaled problem matrices: which 0 A,1 B,2 Q,3 R (idx node-1); 4 QN (leaf idx); 5 Gx, 6 Gu (nonleaf)
void oracle_scaled_mat(void* h, int which, int idx, double* out) {
  const Raocp& p = S(h).scaled();
  const Mat* m = nullptr;
  switch (which) {
    case 0: m = &p.A[idx]; break;
    case 1: m = &p.B[idx]; break;
    case 2: m = &p.Q[idx]; break;
    case 3: m = &p.R[idx]; break;
    case 4: m = &p.QN[idx]; break;
    case 5: m = &p.Gx[idx]; break;
    case 6: m = &p.Gu[idx]; break;
    default: return;
  }
  std::memcpy(out, m->a.data(), sizeof(double) * m->a.size());
}
// offline cache: which 0 P (node), 1 K (nonleaf), 2 Rt (nonleaf), 3 Abar (node-1), 4 s2_proj (nonleaf)
int oracle_cache_mat(void* h, int which, int idx, double* out, int* rows, int* cols) {
  SolverCache& c = S(h).cache();
  const Mat* m = nullptr;
  switch (which) {
    case 0: m = &c.P[idx]; break;
    case 1: m = &c.K[idx]; break;
    case 2: m = &c.Rt[idx]; break;
    case 3: m = &c.Abar[idx]; break;
    case 4: m = &c.s2_proj[idx]; break;
    default: return 1;
  }
  *rows = m->r;
  *cols = m->c;
  if (out) std::memcpy(out, m->a.data(), sizeof(double) * m->a.size());
  return 0;
}

// ---- free-standing kernels for known-answer tests ----
int oracle_proj_soc(double* v, int d) {
  return guard([&] { proj_soc_inplace(v, d); });
}
int oracle_soc_quadlin(const double* Q, const double* q, int n, int* p, double* head_map, double* q_kernel,
                       double* a, double* sqrt_factor) {
  return guard([&] {
    Mat Qm(n, n);
    std::memcpy(Qm.a.data(), Q, sizeof(double) * n * n);
    SocQuadLin d = soc_data_quadlin(Qm, Vec(q, q + n));
    *p = d.p;
    if (head_map) std::memcpy(head_map, d.head_map.a.data(), sizeof(double) * d.head_map.a.size());
    if (q_kernel) std::memcpy(q_kernel, d.q_kernel.data(), sizeof(double) * n);
    if (a) std::memcpy(a, d.a.data(), sizeof(double) * (d.p + 2));
    if (sqrt_factor) std::memcpy(sqrt_factor, d.sqrt_factor.a.data(), sizeof(double) * d.p * d.p);
  });
}
void* oracle_aa_create(int m) { return new Anderson(m); }
void oracle_aa_destroy(void* a) { delete static_cast<Anderson*>(a); }
void oracle_aa_direction(void* a, const double* r, int n, double* psi) {
  Vec o = static_cast<Anderson*>(a)->direction(Vec(r, r + n));
  std::memcpy(psi, o.data(), sizeof(double) * n);
}
// The Anderson least squares alone (solver.cpp:73-75): Eigen's ColPivHouseholderQR
// solve with threshold 1e-12 on a column-major rows x cols matrix
void oracle_colpiv_qr_solve(const double* A, int rows, int cols, const double* b, double* x) {
  Mat M(rows, cols);
  for (int c = 0; c < cols; ++c)
    for (int i = 0; i < rows; ++i) M(i, c) = A[size_t(c) * rows + i];
  const Vec k = colpiv_qr_solve(M, Vec(b, b + rows), 1e-12);
  std::memcpy(x, k.data(), sizeof(double) * cols);
}
// Power iteration on an identity operator of size n (test_oper.cpp:159-163)
double oracle_estimate_norm_identity(int n) {
  auto ident = [](const Vec& v, Vec& o) { o = v; };
  return estimate_norm(n, n, ident, ident, 1.0).estimate;
}
void oracle_philox_normals(uint64_t seed, int n, double* out) {
  Philox r(seed);
  for (int i = 0; i < n; ++i) out[i] = r.normal();
}
void oracle_philox_u64(uint64_t seed, int n, uint64_t* out) {
  Philox r(seed);
  for (int i = 0; i < n; ++i) out[i] = r.next_u64();
}

}  // extern "C"
