// Host-side problem model and one-time setup of the B200 SPOCK solver.
//
// Mirrors the reference's data model and setup (arxiv/paper_2505_12078):
//   ScenarioTree::finalize_topology   proj/src/tree.cpp:24-83
//   RiskSpec::validate / dual_cone    proj/src/risk.cpp:25-63
//   Raocp::validate                   proj/src/problem.cpp:39-86
//   soc_data_quadlin / epigraph data  proj/src/problem.cpp:113-161,216-236
//   precondition                      proj/src/problem.cpp:249-326
//   make_primal/dual_layout           proj/src/layout.cpp:5-67
// and lays the result out for the device (column-major per-node blocks packed
// back to back, 64-bit offsets).  The stage-cost SOC head map is built block
// separated (Q and R decomposed separately), which is exactly the structure of
// the reference's eigendecomposition of blkdiag(Q, R); the device keeps the
// head rows of each stage segment as [x rows; u rows] and the boundary
// permutation restores the reference's ascending-eigenvalue row order.
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <functional>
#include <vector>

#include "../../include/spock_b200.h"

namespace spock {

using Vec = std::vector<double>;

struct Mat {  // column-major
  int r = 0, c = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(int rr, int cc, double v = 0.0) : r(rr), c(cc), a(size_t(rr) * cc, v) {}
  double& operator()(int i, int j) { return a[size_t(i) + size_t(j) * r]; }
  double operator()(int i, int j) const { return a[size_t(i) + size_t(j) * r]; }
};

// cyclic Jacobi; ascending eigenvalues, canonical signs (largest |entry| > 0)
void sym_eig(const Mat& A, Vec& w, Mat& V);

struct ConePart {
  int kind, dim;
};

struct Tree {
  int horizon = 0, stop_stage = 0, num_events = 0;
  std::vector<int> anc, event, stage, child_first, child_count, stage_start;
  Vec prob, cond_prob;
  int nn() const { return int(anc.size()); }
  int nnl() const { return stage_start[horizon]; }
  int nl() const { return nn() - nnl(); }
  bool leaf(int i) const { return child_count[i] == 0; }
  void finalize();
};

struct Risk {
  int kind = 1, n = 0, rows = 0, nnu = 0;
  std::vector<double> E, F, b, pi;  // E rows x n col-major, F rows x nnu
  double gamma = 1.0;
  std::vector<ConePart> cone;
  void validate() const;
};

// Raw problem (host copy of the spock_problem_desc), per-node blocks packed.
// Large per-node arrays of the problem (GBs on wide trees): an uninitialised
// allocation filled by parallel slab copies -- std::vector would zero-fill
// the whole range on one thread first
struct BigVec {
  std::unique_ptr<double[]> p;
  size_t n = 0;
  BigVec() = default;
  BigVec(const double* src, size_t count);
  BigVec(BigVec&&) = default;
  BigVec& operator=(BigVec&&) = default;
  BigVec(const BigVec& o) : BigVec(o.data(), o.n) {}
  BigVec& operator=(const BigVec& o) {
    if (this != &o) *this = BigVec(o.data(), o.n);
    return *this;
  }
  // count = nb blocks of rows x cols; src row-major per block -> column-major
  static BigVec transposed(const double* src, size_t nb, int rows, int cols);
  // nb copies of one column-major block of rows x cols
  static BigVec repeated(const double* blk, size_t nb, int rows, int cols);
  double* data() { return p.get(); }
  const double* data() const { return p.get(); }
  size_t size() const { return n; }
  bool empty() const { return n == 0; }
  double& operator[](size_t i) { return p[i]; }
  const double& operator[](size_t i) const { return p[i]; }
};

struct Problem {
  Tree tree;
  int nx = 0, nu = 0;
  BigVec A, B, Q, R;        // per non-root, stride nx*nx etc.
  Vec c, q, r;
  BigVec QN;                // per leaf
  Vec qN;
  std::vector<int> nc, ncN;
  std::vector<int64_t> g_off, gN_off, box_off, boxN_off;  // offsets into Gx/Gu (by rows) and boxes
  BigVec Gx, Gu, GN;
  Vec C_lo, C_hi, CN_lo, CN_hi;
  std::vector<Risk> risk;
  Vec x_init;
  void validate() const;
};
Problem problem_from_desc(const spock_problem_desc* d);

struct Precond {
  Vec sx, su, sxN, cstr_scale;
  double c_hat = 1.0;
  bool is_identity = true;
};
// scales `p` in place (proj/src/problem.cpp:249-326)
Precond precondition_inplace(Problem& p);
Precond identity_precond(const Problem& p);

// SOC epigraph data of one quadratic block-diagonal cost, block separated.
struct SocBlock {
  int px = 0, pu = 0;       // rank of the x / u block
  Vec Hx, Hu;               // px x nx, pu x nu (col-major)
  Vec qk;                   // kernel component of (q, r), length nx+nu
  Vec a;                    // translation, internal row order [x rows; u rows; 2]
  std::vector<int> perm;    // perm[k] = boundary row of internal head row k
  double lambda_max = 0.0;
  double qk2 = -1.0;         // |qk|^2 when qk itself stays on the device (device-side setup)
};
SocBlock soc_block(const double* Q, int nx, const double* R, int nu, const double* q, const double* r);

struct SocData {
  std::vector<SocBlock> stage, leaf;
};
SocData soc_epigraph_data(const Problem& p);
// parallel loop over [0, n) on host threads (setup only; every index must
// write its own slot)
void parallel_for(int64_t n, const std::function<void(int64_t)>& f);

struct Layouts {
  // primal (layout.cpp:5-30)
  int64_t nz = 0;
  int u_base = 0, tau_base = 0, s_base = 0;
  std::vector<int> y_off, y_dim;
  // dual (layout.cpp:32-67)
  int64_t neta = 0;
  std::vector<int> seg1_off, seg1_nc, seg1_ydim, seg2_off, seg2_dim, seg3_off, seg3_nc, seg3_socdim;
};
Layouts make_layouts(const Problem& p, const SocData& soc);

// analytic ||L|| bound (proj/src/tree_operator.cpp:126-155)
double analytic_norm_bound(const Problem& p, const SocData& soc);

// Philox4x32-10 normal stream (proj/src/rng.cpp), for the power-iteration start
void philox_normals(uint64_t seed, int64_t n, double* out);

struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

}  // namespace spock
