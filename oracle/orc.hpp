// TEST INFRASTRUCTURE ONLY -- the parity oracle.  Not part of the product.
//
// A CPU restatement (C++20, no Eigen) of the reference SPOCK implementation
// arxiv/paper_2505_12078 (proj/src/*.cpp).  Each function cites the reference
// file:line it follows.  The reference itself cannot be compiled here (Eigen3
// and doctest are absent; proj/CMakeLists.txt:10), so this restatement is the
// checker.  It is pinned against every known-answer test and property test of
// the reference suite (tests/test_oracle_*.py) before it is trusted.
//
// Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and the
// --impl reference arm) may load it.
#pragma once

#include <cmath>
#include <cstdint>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

using Vec = std::vector<double>;

// Dense column-major matrix (Eigen's default storage order).
struct Mat {
  int r = 0, c = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(int rows, int cols, double v = 0.0) : r(rows), c(cols), a(size_t(rows) * cols, v) {}
  double& operator()(int i, int j) { return a[size_t(i) + size_t(j) * r]; }
  double operator()(int i, int j) const { return a[size_t(i) + size_t(j) * r]; }
  double* col(int j) { return a.data() + size_t(j) * r; }
  const double* col(int j) const { return a.data() + size_t(j) * r; }
  static Mat eye(int n) {
    Mat m(n, n);
    for (int i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
  }
};

// ---- small dense linear-algebra kit (replaces the Eigen call sites) ----
Mat matmul(const Mat& A, const Mat& B);
Mat matmul_tn(const Mat& A, const Mat& B);  // A' B
Mat transpose(const Mat& A);
Mat add(const Mat& A, const Mat& B, double sb = 1.0);
Vec matvec(const Mat& A, const double* x);                 // A x
void matvec_acc(const Mat& A, const double* x, double* y);  // y += A x
void matvec_t_acc(const Mat& A, const double* x, double* y);  // y += A' x
double dot(const double* a, const double* b, size_t n);
double sqnorm(const Vec& v);
// Cholesky (Eigen::LLT, lower).  Returns false when not PD.
bool cholesky(const Mat& A, Mat& L);
void chol_solve(const Mat& L, double* b);  // in place
// Symmetric eigendecomposition (cyclic Jacobi) with eigenvalues ascending
// (Eigen::SelfAdjointEigenSolver order) and each eigenvector's largest-|.|
// entry made positive (canonical sign; Eigen's is implementation-defined).
void sym_eig(const Mat& A, Vec& evals, Mat& evecs);
// Column-pivoted Householder QR least squares with relative pivot threshold,
// restating Eigen::ColPivHouseholderQR::{computeInPlace,solve} as used at
// proj/src/solver.cpp:73-75.
Vec colpiv_qr_solve(const Mat& A, const Vec& b, double threshold);
// Orthogonal projector onto ker M (I - V1 V1'), V1 the right singular vectors
// with sigma > 1e-12 sigma_max (proj/src/projections.cpp:127-136); one-sided
// Jacobi SVD of M'.
Mat kernel_projector(const Mat& M);

// ---- Philox4x32-10 (proj/src/rng.cpp) ----
class Philox {
 public:
  explicit Philox(uint64_t seed, uint64_t stream = 0);
  uint32_t next_u32();
  uint64_t next_u64();
  double uniform();
  double normal();
 private:
  void refill();
  uint32_t key_[2], ctr_[4], blk_[4];
  int pos_ = 4;
  bool have_spare_ = false;
  double spare_ = 0.0;
};

// ---- thread pool (proj/src/parallel.cpp) ----
void set_num_threads(int n);
int num_threads();
void parallel_for(int begin, int end, const std::function<void(int)>& body, uint64_t body_flops = 0);

// ---- model (proj/src/tree.cpp, risk.cpp, problem.cpp) ----
enum ConeKind { ZERO = 0, NONNEG = 1, SOC = 2, FREE = 3 };
struct ConePart {
  int kind;
  int dim;
};
std::vector<ConePart> dual_cone(const std::vector<ConePart>& c);

struct Tree {
  int horizon = 0, stop_stage = 0, num_events = 0;
  std::vector<int> anc, event, stage, child_first, child_count, stage_start;
  Vec prob, cond_prob;
  int nn() const { return int(anc.size()); }
  int nnl() const { return stage_start[horizon]; }
  int nl() const { return nn() - nnl(); }
  int sb(int t) const { return stage_start[t]; }
  int se(int t) const { return stage_start[t + 1]; }
  bool leaf(int i) const { return child_count[i] == 0; }
  void finalize();  // ScenarioTree::finalize_topology, tree.cpp:24-83
};
void stage_parallel_for(const Tree& t, int stage, const std::function<void(int)>& body,
                        uint64_t flops = 0);

struct Risk {
  int kind = 1;  // 0 avar, 1 general
  int n = 0;
  Mat E, F;
  Vec b;
  std::vector<ConePart> cone;
  double gamma = 1.0;
  Vec pi;
  int rows() const { return E.r; }
  void validate() const;  // risk.cpp:45-63
};

struct Box {
  Vec lo, hi;
  int dim() const { return int(lo.size()); }
};

struct Raocp {
  std::shared_ptr<Tree> tree;
  int nx = 0, nu = 0;
  std::vector<Mat> A, B, Q, R;
  std::vector<Vec> c, q, r;
  std::vector<Mat> QN;
  std::vector<Vec> qN;
  std::vector<Mat> Gx, Gu;
  std::vector<Box> C;
  std::vector<Risk> risk;
  std::vector<Mat> GN;
  std::vector<Box> CN;
  Vec x_init;
  void validate() const;  // problem.cpp:39-86
};

struct SocQuadLin {  // problem.hpp:74-90
  int n = 0, p = 0;
  Mat S, sqrt_factor, head_map;
  Vec q_kernel, a;
  double lambda_max = 0.0;
};
SocQuadLin soc_data_quadlin(const Mat& Q, const Vec& q);  // problem.cpp:113-161
struct SocData {
  std::vector<SocQuadLin> stage, leaf;
};
SocData soc_epigraph_data(const Raocp& p);  // problem.cpp:216-236

struct Precond {  // problem.hpp:132-145
  Vec sx, su, sxN;
  Vec cstr_scale;
  double c_hat = 1.0;
  bool is_identity = false;
};
Precond identity_precond(const Raocp& p);
void precondition(const Raocp& p, Raocp& s, Precond& pc);  // problem.cpp:249-326

// ---- layouts (proj/src/layout.cpp) ----
struct PrimalLayout {
  int n = 0, nx = 0, nu = 0, num_nodes = 0, num_nonleaf = 0;
  int u_base = 0, tau_base = 0, s_base = 0;
  std::vector<int> y_off, y_dim;
  int x(int i) const { return 1 + i * nx; }
  int u(int i) const { return u_base + i * nu; }
  int y(int i) const { return y_off[i]; }
  int tau(int i) const { return tau_base + (i - 1); }
  int s(int i) const { return i == 0 ? 0 : s_base + (i - 1); }
};
struct DualLayout {
  int n = 0, num_nodes = 0, num_nonleaf = 0;
  std::vector<int> seg1_off, seg1_nc, seg1_ydim, seg2_off, seg2_dim, seg3_off, seg3_nc, seg3_socdim;
  int y_copy(int i) const { return seg1_off[i]; }
  int risk_scalar(int i) const { return seg1_off[i] + seg1_ydim[i]; }
  int cstr(int i) const { return seg1_off[i] + seg1_ydim[i] + 1; }
  int stage_soc(int i) const { return seg2_off[i - 1]; }
  int leaf_cstr(int j) const { return seg3_off[j]; }
  int leaf_soc(int j) const { return seg3_off[j] + seg3_nc[j]; }
};
PrimalLayout make_primal_layout(const Raocp& p);
DualLayout make_dual_layout(const Raocp& p, const SocData& soc);

// ---- projections + offline cache (proj/src/projections.cpp) ----
void proj_soc_inplace(double* v, int d);
void proj_cone_inplace(const std::vector<ConePart>& cone, double* v);
struct SolverCache {
  std::vector<Mat> P, K, Rt, RtL, Abar, s2_proj;
  std::vector<Vec> q_scr, d_scr, term_u, term_x;
};
SolverCache make_solver_cache(const Raocp& p);
void proj_s1(const Raocp& p, SolverCache& c, const PrimalLayout& zl, const Vec& x_init, double* z);
void proj_s2(const Raocp& p, const SolverCache& c, const PrimalLayout& zl, double* z);
void proj_s3(const Raocp& p, const SocData& soc, const DualLayout& el,
             const std::vector<std::vector<ConePart>>& dk, double* eta);

// ---- tree operator (proj/src/tree_operator.cpp) ----
struct OpNormEstimate {
  double estimate = 0.0;
  int iterations = 0;
  double analytic_bound = 0.0;
  bool converged = false;
};
OpNormEstimate estimate_norm(int nz, int neta, const std::function<void(const Vec&, Vec&)>& apply,
                             const std::function<void(const Vec&, Vec&)>& adj, double bound,
                             double tol = 1e-6, int max_iters = 500);
class TreeOperator {
 public:
  TreeOperator(const Raocp& p, const SocData& soc);
  const PrimalLayout& zlay() const { return zl_; }
  const DualLayout& elay() const { return el_; }
  const std::vector<std::vector<ConePart>>& dual_cones() const { return dk_; }
  void apply(const Vec& z, Vec& eta) const;
  void apply_adjoint(const Vec& eta, Vec& z) const;
  double analytic_norm_bound() const;
  OpNormEstimate estimate_norm(double tol = 1e-6, int max_iters = 500) const;
  double m_norm(const Vec& z, const Vec& eta, double alpha) const;
 private:
  const Raocp* p_;
  const SocData* soc_;
  PrimalLayout zl_;
  DualLayout el_;
  std::vector<std::vector<ConePart>> dk_;
  mutable std::vector<Vec> adj_;
  mutable Vec mscr_;
};

// ---- solver (proj/src/solver.cpp) ----
struct Params {
  double eps_abs = 1e-6, eps_rel = 1e-6, alpha = 0.0;
  int aa_memory = 3;
  double c0 = 0.99, c1 = 0.99, c2 = 0.99, beta = 0.5, sigma = 0.1, lambda = 1.0;
  int max_iters = 50000, max_backtracks = 40;
  bool use_preconditioner = true;
  std::function<void(int, double, char)> progress;
  std::function<bool()> cancelled;
  void validate() const;
};
struct Status {
  int iterations = 0, reason = 1;
  double xi1_inf = 0, xi2_inf = 0;
  int k0 = 0, k1 = 0, k2 = 0, stalled = 0;
  Vec rnorm_history;
  std::string branches;
  double alpha = 0;
  OpNormEstimate op_norm;
  long n_T = 0, n_L = 0, n_Lt = 0;
};
struct SolveResult {
  Vec z, z_scaled, eta;
  Status status;
};

class Anderson {  // solver.cpp:45-77
 public:
  explicit Anderson(int m);
  Vec direction(const Vec& r);
 private:
  int m_, k_ = 0;
  std::vector<Vec> res_, diff_;
};

class SpockSolver {
 public:
  SpockSolver(const Raocp& problem, Params params);
  SolveResult solve(const Vec& x_init, const Vec* wz, const Vec* we, bool supermann);
  void apply_T(const Vec& z, const Vec& eta, Vec& z_out, Vec& eta_out);
  double alpha() const { return alpha_; }
  const OpNormEstimate& op_norm() const { return norm_; }
  const Raocp& scaled() const { return scaled_; }
  const Precond& precond() const { return pc_; }
  const TreeOperator& oper() const { return *op_; }
  const SocData& soc() const { return soc_; }
  SolverCache& cache() { return cache_; }
  Vec unscale_primal(const Vec& zs) const;
  const Vec& x_init_orig() const { return x_init_orig_; }
  Raocp& scaled_mut() { return scaled_; }
 private:
  double mnorm_cached(const Vec& rz, const Vec& re, Vec& Lrz, Status& st) const;
  Params prm_;
  Raocp scaled_;
  Precond pc_;
  SocData soc_;
  std::unique_ptr<TreeOperator> op_;
  SolverCache cache_;
  OpNormEstimate norm_;
  double alpha_ = 0;
  Vec x_init_orig_, d1_, d2_;
  Vec tz_, te_, tz2_, te2_;
};

}  // namespace orc
