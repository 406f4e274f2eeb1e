// C-ABI of the B200 SPOCK solver (include/spock_b200.h).  Each entry point
// forwards to the Engine and maps C++ exceptions onto the reference's error
// kinds: std::invalid_argument -> SPOCK_EINVAL, numerical std::runtime_error
// -> SPOCK_ERUNTIME, CUDA failures -> SPOCK_ECUDA.
#include <cstring>
#include <string>
#include <vector>

#include "../../include/spock_b200.h"
#include "engine.hpp"
#include "nccl_dl.hpp"

struct spock_solver {
  spock::Engine* eng = nullptr;
  spock::OpNorm norm;
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return SPOCK_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return SPOCK_EINVAL;
  } catch (const spock::CudaError& e) {
    g_err = e.what();
    return SPOCK_ECUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SPOCK_ERUNTIME;
  }
}

spock::Params to_params(const spock_params* p) {
  spock::Params q;
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
  q.poll_every = p->poll_every > 0 ? p->poll_every : 1;
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

int check(spock_solver* s) {
  if (!s || !s->eng) {
    g_err = "spock: null solver handle";
    return SPOCK_EINVAL;
  }
  // the current device is per host thread: run on the solver's own device
  // whatever thread calls (BatchSolver workers, user threads)
  if (cudaSetDevice(s->eng->device()) != cudaSuccess) {
    g_err = "spock: cannot make the solver's device current";
    return SPOCK_ECUDA;
  }
  return SPOCK_OK;
}
}  // namespace

extern "C" {

const char* spock_last_error(void) { return g_err.c_str(); }

void spock_params_default(spock_params* p) {
  if (!p) return;
  std::memset(p, 0, sizeof(*p));
  p->eps_abs = 1e-6;
  p->eps_rel = 1e-6;
  p->alpha = 0.0;
  p->aa_memory = 3;
  p->c0 = p->c1 = p->c2 = 0.99;
  p->beta = 0.5;
  p->sigma = 0.1;
  p->lambda = 1.0;
  p->max_iters = 50000;
  p->max_backtracks = 40;
  p->use_preconditioner = 1;
  p->poll_every = 1;
}

int spock_solver_create(const spock_problem_desc* desc, const spock_params* params, spock_solver** out) {
  return guard([&] {
    if (!out) throw std::invalid_argument("spock: null output handle");
    auto* s = new spock_solver;
    try {
      s->eng = new spock::Engine(desc, to_params(params));
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

void spock_solver_destroy(spock_solver* s) {
  if (!s) return;
  if (s->eng) cudaSetDevice(s->eng->device());
  delete s->eng;
  delete s;
}

int spock_solver_dims(const spock_solver* s, int64_t* nz, int64_t* neta) {
  if (!s || !s->eng) return SPOCK_EINVAL;
  if (nz) *nz = s->eng->nz();
  if (neta) *neta = s->eng->neta();
  return SPOCK_OK;
}

double spock_solver_alpha(const spock_solver* s) { return (s && s->eng) ? s->eng->alpha() : 0.0; }

static int do_solve(spock_solver* s, const double* x0, const double* wz, const double* we, double* oz,
                    double* ozs, double* oe, spock_status* st, bool sm) {
  if (int rc = check(s)) return rc;
  return guard([&] {
    spock::Status S;
    s->eng->solve_b(x0, wz, we, oz, ozs, oe, sm, S);
    if (!st) return;
    st->iterations = S.iterations;
    st->reason = S.reason;
    st->xi1_inf = S.xi1;
    st->xi2_inf = S.xi2;
    st->k0_steps = S.k0;
    st->k1_steps = S.k1;
    st->k2_steps = S.k2;
    st->stalled_steps = S.stalled;
    st->alpha = s->eng->alpha();
    const auto& nrm = s->eng->op_norm();
    st->op_norm_estimate = nrm.estimate;
    st->op_norm_iterations = nrm.iterations;
    st->op_norm_analytic_bound = nrm.analytic_bound;
    st->op_norm_converged = nrm.converged;
    const int n = int(S.rnorm.size());
    for (int w = 0; w < n && w < st->history_capacity; ++w) {
      if (st->rnorm_history) st->rnorm_history[w] = S.rnorm[w];
      if (st->branch_history) st->branch_history[w] = S.branches[w];
    }
    st->history_len = n;
    st->n_T = S.n_T;
    st->n_L = S.n_L;
    st->n_Lt = S.n_Lt;
  });
}

int spock_solver_solve(spock_solver* s, const double* x_init, const double* wz, const double* we, double* oz,
                       double* ozs, double* oe, spock_status* st) {
  return do_solve(s, x_init, wz, we, oz, ozs, oe, st, true);
}
int spock_solver_solve_cp(spock_solver* s, const double* x_init, const double* wz, const double* we, double* oz,
                          double* ozs, double* oe, spock_status* st) {
  return do_solve(s, x_init, wz, we, oz, ozs, oe, st, false);
}

int spock_solver_apply_T(spock_solver* s, const double* z, const double* eta, double* zo, double* eo) {
  if (int rc = check(s)) return rc;
  return guard([&] { s->eng->apply_T_b(z, eta, zo, eo); });
}
int spock_op_apply(spock_solver* s, const double* z, double* eta) {
  if (int rc = check(s)) return rc;
  return guard([&] { s->eng->apply_L_b(z, eta); });
}
int spock_op_apply_adjoint(spock_solver* s, const double* eta, double* z) {
  if (int rc = check(s)) return rc;
  return guard([&] { s->eng->apply_Lt_b(eta, z); });
}
int spock_op_m_norm(spock_solver* s, const double* z, const double* eta, double alpha, double* out) {
  if (int rc = check(s)) return rc;
  return guard([&] { *out = s->eng->m_norm_b(z, eta, alpha); });
}
int spock_proj_s1(spock_solver* s, double* z) {
  if (int rc = check(s)) return rc;
  return guard([&] { s->eng->proj_s1_b(z); });
}
int spock_proj_s2(spock_solver* s, double* z) {
  if (int rc = check(s)) return rc;
  return guard([&] { s->eng->proj_s2_b(z); });
}
int spock_proj_s3(spock_solver* s, double* eta) {
  if (int rc = check(s)) return rc;
  return guard([&] { s->eng->proj_s3_b(eta); });
}
int spock_solver_unscale_primal(spock_solver* s, const double* zs, double* z) {
  if (int rc = check(s)) return rc;
  return guard([&] { s->eng->unscale_b(zs, z); });
}
int spock_bench_T(spock_solver* s, int32_t k, int32_t use_graph, int32_t flush_l2, double* ms_out) {
  if (int rc = check(s)) return rc;
  return guard([&] { *ms_out = s->eng->bench_T(k, use_graph != 0, flush_l2 != 0); });
}
int spock_bench_kernels(spock_solver* s, int32_t k, int32_t flush_l2, double* ms5) {
  if (int rc = check(s)) return rc;
  return guard([&] { s->eng->bench_kernels(k, flush_l2 != 0, ms5); });
}
int spock_traffic_model(spock_solver* s, double* bytes5, int32_t* launches_per_T) {
  if (int rc = check(s)) return rc;
  return guard([&] {
    s->eng->traffic(bytes5);
    if (launches_per_T) *launches_per_T = s->eng->launches_per_T();
  });
}

int spock_shard_setup(spock_solver* s, int32_t world, int32_t rank, int32_t split_stage, const int32_t* back_a,
                      int32_t na, const int32_t* back_b, int32_t nb, const int32_t* s2, int32_t ns2,
                      const int32_t* fwd, int32_t nf, double* xbuf_dev) {
  if (int rc = check(s)) return rc;
  return guard([&] {
    s->eng->shard_setup(world, rank, split_stage, back_a, na, back_b, nb, s2, ns2, fwd, nf, xbuf_dev);
  });
}

int spock_shard_apply_T(spock_solver* s, int32_t phase, const double* z, const double* eta, double* z_out,
                        double* eta_out) {
  if (int rc = check(s)) return rc;
  return guard([&] { s->eng->shard_apply_T_b(phase, z, eta, z_out, eta_out); });
}

int spock_nccl_unique_id(void* id_out) {
  return guard([&] {
    if (!id_out) throw std::invalid_argument("spock_nccl_unique_id: null output");
    ncclUniqueId u;
    spock::nccl_check(spock::nccl_dl().GetUniqueId(&u), "ncclGetUniqueId");
    std::memcpy(id_out, &u, sizeof(u));
  });
}

int spock_shard_nccl_init(spock_solver* s, const void* id, int32_t nranks, int32_t rank) {
  if (int rc = check(s)) return rc;
  return guard([&] {
    if (!id) throw std::invalid_argument("spock_shard_nccl_init: null id");
    s->eng->shard_nccl_init(id, nranks, rank);
  });
}

int spock_shard_bench(spock_solver* s, int32_t phase, int32_t parity) {
  if (int rc = check(s)) return rc;
  return guard([&] { s->eng->shard_bench(phase, parity & 1); });
}

int spock_shard_masks(spock_solver* s, uint8_t* z_mask, uint8_t* eta_mask) {
  if (int rc = check(s)) return rc;
  return guard([&] { s->eng->shard_masks(z_mask, eta_mask); });
}

int spock_shard_weights(spock_solver* s, uint8_t* z_w, uint8_t* eta_w) {
  if (int rc = check(s)) return rc;
  return guard([&] { s->eng->shard_weights(z_w, eta_w); });
}

int spock_shard_set_collectives(spock_solver* s, spock_collective_fn fn, void* user) {
  if (int rc = check(s)) return rc;
  return guard([&] { s->eng->shard_set_collectives(reinterpret_cast<spock::Engine::CollFn>(fn), user); });
}

void* spock_solver_stream(const spock_solver* s) {
  return (s && s->eng) ? reinterpret_cast<void*>(s->eng->stream()) : nullptr;
}

const char* spock_solver_t_path(const spock_solver* s) { return (s && s->eng) ? s->eng->t_path() : ""; }

const char* spock_solver_loop_path(const spock_solver* s) { return (s && s->eng) ? s->eng->loop_path() : ""; }

int spock_solver_set_grid_cap(spock_solver* s, int32_t ctas) {
  if (int rc = check(s)) return rc;
  return guard([&] { s->eng->set_grid_cap(ctas); });
}

int spock_anderson_lstsq(const double* Md, int64_t rows, int32_t cols, const double* r, double* kappa) {
  return guard([&] {
    if (!Md || !r || !kappa || rows < 1 || cols < 1 || cols > spock::kAaHostMax)
      throw std::invalid_argument("spock_anderson_lstsq: bad arguments");
    std::vector<spock::dd> G(size_t(cols) * cols, spock::dd{0.0, 0.0}), g(size_t(cols), spock::dd{0.0, 0.0});
    for (int a = 0; a < cols; ++a) {
      const double* x = Md + size_t(a) * rows;
      for (int b = a; b < cols; ++b) {
        const double* y = Md + size_t(b) * rows;
        spock::dd s{0.0, 0.0};
        for (int64_t i = 0; i < rows; ++i) s = spock::dd_fma(s, x[i], y[i]);
        G[a + size_t(b) * cols] = G[b + size_t(a) * cols] = s;
      }
      spock::dd s{0.0, 0.0};
      for (int64_t i = 0; i < rows; ++i) s = spock::dd_fma(s, x[i], r[i]);
      g[a] = s;
    }
    spock::aa_kappa_dd<spock::kAaHostMax>(G.data(), g.data(), cols, rows, kappa);
  });
}

int32_t spock_solver_grid(const spock_solver* s) { return (s && s->eng) ? s->eng->fused_grid() : 0; }

}  // extern "C"
