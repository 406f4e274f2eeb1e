/*
 * spock_b200.h -- C-ABI drop-in boundary of the B200-native SPOCK solver.
 *
 * The reference (arxiv/paper_2505_12078, CPU C++20/Eigen) exposes a C++ API:
 *   SpockSolver(const Raocp&, SpockParams)      proj/include/spock/solver.hpp:99
 *   SpockSolver::solve / solve_cp / apply_T     proj/include/spock/solver.hpp:103-112
 *   TreeOperator::apply / apply_adjoint / m_norm proj/include/spock/tree_operator.hpp:38-52
 *   proj_s1 / proj_s2 / proj_s3                  proj/include/spock/projections.hpp:49-65
 * Every entry point below replaces one of those (cited per function).  The C++
 * host layer of this package keeps the reference's semantics and error kinds
 * behind these plain-pointer functions; no Eigen/torch types cross the ABI.
 *
 * Vectors are exchanged in the reference's PrimalLayout / DualLayout order
 * (proj/include/spock/layout.hpp:14-52).  Pointers may be host or device
 * memory; the library detects which (cudaPointerGetAttributes).
 *
 * Matrices are column-major (Eigen's default storage), packed back to back in
 * node order with the reference's indexing: per non-root node at offset
 * node-1, per leaf at node-num_nonleaf, per non-leaf at node
 * (proj/include/spock/problem.hpp:25-58).
 *
 * Return codes map 1:1 onto the reference's exception kinds:
 *   SPOCK_EINVAL   <- std::invalid_argument  (bad parameters / dimensions / data)
 *   SPOCK_ERUNTIME <- std::runtime_error     (Cholesky failure, negative M-norm radicand)
 * spock_last_error() returns the message of the last failure on this thread.
 */
#ifndef SPOCK_B200_H_
#define SPOCK_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPOCK_OK 0
#define SPOCK_EINVAL 1
#define SPOCK_ERUNTIME 2
#define SPOCK_ECUDA 3

/* ConeKind, proj/include/spock/risk.hpp:8 */
#define SPOCK_CONE_ZERO 0
#define SPOCK_CONE_NONNEG 1
#define SPOCK_CONE_SOC 2
#define SPOCK_CONE_FREE 3

/* RiskSpec::Kind, proj/include/spock/risk.hpp:27 */
#define SPOCK_RISK_AVAR 0
#define SPOCK_RISK_GENERAL 1

/* SpockTermination, proj/include/spock/solver.hpp:37 */
#define SPOCK_CONVERGED 0
#define SPOCK_MAX_ITERS 1
#define SPOCK_STALLED 2
#define SPOCK_CANCELLED 3

/* spock_problem_desc.layout flags (extensions; 0 = the reference's layout).
 * ROW_MAJOR: the per-node blocks A, B, Q, R, QN, Gx, Gu, GN are row-major (C
 *   order, e.g. numpy stacks) instead of column-major.
 * SHARED_G: Gx / Gu hold ONE block shared by every non-leaf node and GN one
 *   block shared by every leaf (every nc[i] equal, every ncN[j] equal; the
 *   generators' box selectors, generators.cpp:99-109). */
#define SPOCK_LAYOUT_ROW_MAJOR 1
#define SPOCK_LAYOUT_SHARED_G 2

/* Flat description of a Raocp (proj/include/spock/problem.hpp:29-58) on a
 * ScenarioTree given by raw arrays (ScenarioTree::from_arrays,
 * proj/include/spock/tree.hpp:72-74).  All pointers are host memory. */
typedef struct spock_problem_desc {
  int32_t num_nodes, nx, nu;
  int32_t horizon, stop_stage, num_events;
  const int32_t* anc;       /* [nn], anc[0] = -1 */
  const int32_t* event;     /* [nn] */
  const double* prob;       /* [nn] */
  const double* cond_prob;  /* [nn] */
  /* per non-root node (nn-1 entries each) */
  const double* A; /* nx*nx */
  const double* B; /* nx*nu */
  const double* c; /* nx */
  const double* Q; /* nx*nx */
  const double* R; /* nu*nu */
  const double* q; /* nx */
  const double* r; /* nu */
  /* per leaf */
  const double* QN; /* nx*nx */
  const double* qN; /* nx */
  /* per non-leaf: nc[i] constraint rows */
  const int32_t* nc;
  const double* Gx;   /* packed nc[i]*nx */
  const double* Gu;   /* packed nc[i]*nu */
  const double* C_lo; /* packed nc[i] */
  const double* C_hi;
  /* per leaf: ncN[j] terminal constraint rows */
  const int32_t* ncN;
  const double* GN; /* packed ncN[j]*nx */
  const double* CN_lo;
  const double* CN_hi;
  /* per non-leaf risk spec (proj/include/spock/risk.hpp:26-48); n = children */
  const int32_t* risk_kind;   /* SPOCK_RISK_* */
  const int32_t* risk_rows;   /* rows of E */
  const int32_t* risk_nnu;    /* columns of F */
  const double* risk_E;       /* packed rows*n */
  const double* risk_F;       /* packed rows*nnu */
  const double* risk_b;       /* packed rows */
  const double* risk_gamma;   /* [nnl], Avar only */
  const double* risk_pi;      /* packed n, Avar only */
  const int32_t* cone_nparts; /* [nnl] */
  const int32_t* cone_kind;   /* packed parts */
  const int32_t* cone_dim;    /* packed parts */
  const double* x_init;       /* nx */
  int32_t layout;             /* SPOCK_LAYOUT_* flags */
} spock_problem_desc;

/* SpockParams, proj/include/spock/solver.hpp:15-35.  std::function callbacks
 * become (fnptr, user) pairs; they are polled every `poll_every` iterations
 * (1 = every iteration, the reference's behaviour). */
typedef struct spock_params {
  double eps_abs, eps_rel;
  double alpha; /* 0: 0.99 / power-iteration estimate of ||L|| */
  int32_t aa_memory;
  double c0, c1, c2;
  double beta, sigma, lambda;
  int32_t max_iters;
  int32_t max_backtracks;
  int32_t use_preconditioner;
  void (*progress)(int32_t iter, double rnorm, char branch, void* user);
  int32_t (*cancelled)(void* user);
  void* user;
  int32_t poll_every;
} spock_params;

/* SpockStatus, proj/include/spock/solver.hpp:41-49.  History buffers are
 * caller-owned (capacity entries); *_len reports how many were written. */
typedef struct spock_status {
  int32_t iterations;
  int32_t reason; /* SPOCK_CONVERGED ... */
  double xi1_inf, xi2_inf;
  int32_t k0_steps, k1_steps, k2_steps, stalled_steps;
  double alpha;
  double op_norm_estimate;
  int32_t op_norm_iterations;
  double op_norm_analytic_bound;
  int32_t op_norm_converged;
  double* rnorm_history;
  char* branch_history;
  int32_t history_capacity;
  int32_t history_len;
  /* operator applications issued by the solve (diagnostics) */
  int64_t n_T, n_L, n_Lt;
} spock_status;

typedef struct spock_solver spock_solver;

const char* spock_last_error(void);
void spock_params_default(spock_params* p);

/* SpockSolver::SpockSolver (proj/src/solver.cpp:79-114): validate, precondition,
 * SOC epigraph data, layouts, offline factorisation (on device), ||L|| power
 * iteration (on device), alpha, termination scalings. */
int spock_solver_create(const spock_problem_desc* desc, const spock_params* params,
                        spock_solver** out);
void spock_solver_destroy(spock_solver* s);

/* sizes of z (PrimalLayout::n) and eta (DualLayout::n) */
int spock_solver_dims(const spock_solver* s, int64_t* nz, int64_t* neta);
double spock_solver_alpha(const spock_solver* s);

/* SpockSolver::solve(x_init, warm) (proj/src/solver.cpp:178-180,189-350).
 * x_init may be NULL (problem's x_init); warm_z_scaled/warm_eta may be NULL
 * (zero start).  Outputs (any may be NULL): z (original variables), z_scaled,
 * eta. */
int spock_solver_solve(spock_solver* s, const double* x_init, const double* warm_z_scaled,
                       const double* warm_eta, double* out_z, double* out_z_scaled,
                       double* out_eta, spock_status* status);
/* SpockSolver::solve_cp (proj/src/solver.cpp:182-187): plain KM iterations */
int spock_solver_solve_cp(spock_solver* s, const double* x_init, const double* warm_z_scaled,
                          const double* warm_eta, double* out_z, double* out_z_scaled,
                          double* out_eta, spock_status* status);

/* SpockSolver::apply_T (proj/src/solver.cpp:148-164), scaled coordinates */
int spock_solver_apply_T(spock_solver* s, const double* z, const double* eta, double* z_out,
                         double* eta_out);
/* TreeOperator::apply / apply_adjoint (proj/src/tree_operator.cpp:20-114) on
 * the solver's (scaled) problem */
int spock_op_apply(spock_solver* s, const double* z, double* eta);
int spock_op_apply_adjoint(spock_solver* s, const double* eta, double* z);
/* TreeOperator::m_norm (proj/src/tree_operator.cpp:214-222) */
int spock_op_m_norm(spock_solver* s, const double* z, const double* eta, double alpha,
                    double* out);
/* proj_s1 / proj_s2 / proj_s3 (proj/src/projections.cpp:142-244), in place,
 * on the solver's (scaled) problem; s1 uses the scaled x_init */
int spock_proj_s1(spock_solver* s, double* z);
int spock_proj_s2(spock_solver* s, double* z);
int spock_proj_s3(spock_solver* s, double* eta);
/* SpockSolver::unscale_primal / scale_primal (proj/src/solver.cpp:116-146) */
int spock_solver_unscale_primal(spock_solver* s, const double* z_scaled, double* z);

/* Benchmark helpers (not part of the reference API).
 * spock_bench_T: k back-to-back CP applications v <- T(v) on device-resident
 * iterates; with flush_l2 a 256 MiB buffer is rewritten between applications
 * outside the timed events.  Returns total device milliseconds.
 * spock_bench_kernels: average device ms of [L*, S1 sweeps, S2, L+S3, T].
 * spock_traffic_model: algorithmic bytes of the same five launch classes and
 * the number of kernel launches per T.
 * spock_solver_t_path: which device schedule computes T -- "fused" (CTA-
 * granular dataflow kernel, narrow trees), "wide" (warp-granular streaming
 * dataflow kernel) or "stages" (one launch per tree stage). */
int spock_bench_T(spock_solver* s, int32_t k, int32_t use_graph, int32_t flush_l2, double* ms_out);
int spock_bench_kernels(spock_solver* s, int32_t k, int32_t flush_l2, double* ms5);
int spock_traffic_model(spock_solver* s, double* bytes5, int32_t* launches_per_T);
const char* spock_solver_t_path(const spock_solver* s);
/* Which loop spock_solver_solve / _solve_cp run (extension): "small" -- the
 * whole solve in one CTA (trees whose CP application streams <= 2 MB),
 * "graph" -- one CUDA graph with conditional nodes per solve, "host" -- the
 * host-driven loop (cancellation callback, Anderson memory > 10, sharded). */
const char* spock_solver_loop_path(const spock_solver* s);

/* Concurrent solves (batched multi-x_init; no reference
 * counterpart -- the reference solves one x_init at a time, solver.hpp:104-105).
 * Narrow trees are latency-bound, so several solvers, each on its own stream
 * (spock_solver_stream), solve side by side when each T launch is capped to a
 * share of the SMs.  spock_solver_set_grid_cap caps the CTAs of the fused T
 * launch (0 = the full-device default); it must precede the first solve or
 * bench of the solver (SPOCK_EINVAL otherwise) and is a no-op on the wide and
 * per-stage schedules.  spock_solver_grid returns the current fused T grid
 * (0 when T does not run on the fused kernel). */
int spock_solver_set_grid_cap(spock_solver* s, int32_t ctas);
int32_t spock_solver_grid(const spock_solver* s);

/* Subtree sharding of T over G ranks (no reference counterpart: the reference
 * runs one process).  The host picks a split stage ts; the rank
 * owns the stage-ts nodes [b0, b1) = [bfirst + rank*q, bfirst + (rank+1)*q)
 * (q = ceil(|stage ts| / G)) with their subtrees, and computes the stages < ts
 * redundantly.  The node lists give the rank's items in dependency order:
 * back_a = its subtrees' backward items (descending), back_b = the top's
 * backward items (descending), s2 = parents whose S2 it computes, fwd = forward
 * items (ascending).  xbuf_dev is a device buffer of G*q*(2(nx+nu)+6) doubles,
 * all-gathered by the host between the two phases of spock_shard_apply_T
 * (phase 0: rank's slice written; phase 1: completes T, host pointers in the
 * boundary layouts; entries outside spock_shard_masks are not computed).
 * spock_solver_stream returns the cudaStream_t the solver enqueues on. */
int spock_shard_setup(spock_solver* s, int32_t world, int32_t rank, int32_t split_stage, const int32_t* back_a,
                      int32_t na, const int32_t* back_b, int32_t nb, const int32_t* s2, int32_t ns2,
                      const int32_t* fwd, int32_t nf, double* xbuf_dev);
int spock_shard_apply_T(spock_solver* s, int32_t phase, const double* z, const double* eta, double* z_out,
                        double* eta_out);
int spock_shard_bench(spock_solver* s, int32_t phase, int32_t parity);
int spock_shard_masks(spock_solver* s, uint8_t* z_mask, uint8_t* eta_mask);
/* Sharded solve / solve_cp: once collectives are set, spock_solver_solve and
 * spock_solver_solve_cp on every rank run one SuperMann / CP solve together
 * (host-driven loop; T, L and L* over the rank's items with the stage-ts
 * exchanges; every reduction over the rank's entries, completed by the host's
 * collectives on device buffers, enqueued on spock_solver_stream's stream:
 * op 0 all-gather of the n-double exchange buffer (equal slices per rank),
 * op 1 all-reduce sum, op 2 all-reduce max, op 3 all-gather of n doubles per
 * rank in place -- dev_buf holds world * n, this rank's at [rank n, (rank+1) n),
 * used for the double-double Anderson Gram; return 0 on success).  Outputs
 * are valid on spock_shard_masks' entries. */
typedef int (*spock_collective_fn)(void* user, int32_t op, double* dev_buf, int64_t n);
/* spock_shard_weights: spock_shard_masks restricted to one rank per entry (the
 * replicated top belongs to rank 0): the ranks' weighted outputs sum to the
 * whole vector. */
int spock_shard_weights(spock_solver* s, uint8_t* z_w, uint8_t* eta_w);
int spock_shard_set_collectives(spock_solver* s, spock_collective_fn fn, void* user);
/* Native collectives instead of the callback: rank 0 gets a 128-byte NCCL
 * unique id (spock_nccl_unique_id), the host broadcasts it, and every rank
 * calls spock_shard_nccl_init (after spock_shard_setup, same world / rank).
 * From then on the exchanges and the sharded solves' reductions are
 * ncclAllGather / ncclAllReduce calls enqueued by the library on
 * spock_solver_stream's stream (no host round trip), and phase 2 of
 * spock_shard_apply_T / spock_shard_bench runs a whole sharded T (phase 0,
 * all-gather, phase 1) in one call.  NCCL is loaded at run time
 * (libnccl.so.2). */
int spock_nccl_unique_id(void* id_out);
int spock_shard_nccl_init(spock_solver* s, const void* id, int32_t nranks, int32_t rank);
void* spock_solver_stream(const spock_solver* s);

/* The least-squares step of AndersonAccelerator::direction
 * (proj/src/solver.cpp:67-76: ColPivHouseholderQR(M_d).setThreshold(1e-12)
 * .solve(r)) as the solver computes it on device: Gram M_d'M_d and M_d'r in
 * double-double, column-pivoted Cholesky with Eigen's pivot order and rank
 * rules (aa.cuh).  Host-only (no device needed): M_d column-major rows x cols,
 * cols <= 64. */
int spock_anderson_lstsq(const double* Md, int64_t rows, int32_t cols, const double* r, double* kappa);

#ifdef __cplusplus
}
#endif

#endif /* SPOCK_B200_H_ */
