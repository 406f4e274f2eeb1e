// Device engine of the B200 SPOCK solver: owns the preconditioned problem,
// its device image, the offline factors and all iteration buffers.  One
// instance runs one solve at a time (as the reference's SpockSolver,
// proj/include/spock/solver.hpp:95-145).
#pragma once

#include <cuda_runtime.h>

#include <functional>
#include <map>
#include <unordered_map>
#include <string>
#include <vector>

#include "aa.cuh"
#include "dev.cuh"
#include "fused.hpp"
#include "kernels.hpp"
#include "loop.hpp"
#include "model.hpp"
#include "wide.hpp"

namespace spock {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct OpNorm {
  double estimate = 0.0, analytic_bound = 0.0;
  int iterations = 0;
  bool converged = false;
};

struct Params {
  double eps_abs = 1e-6, eps_rel = 1e-6, alpha = 0.0;
  int aa_memory = 3;
  double c0 = 0.99, c1 = 0.99, c2 = 0.99, beta = 0.5, sigma = 0.1, lambda = 1.0;
  int max_iters = 50000, max_backtracks = 40;
  bool use_preconditioner = true;
  std::function<void(int, double, char)> progress;
  std::function<bool()> cancelled;
  int poll_every = 1;
  void validate() const;
};

struct Status {
  int iterations = 0, reason = SPOCK_MAX_ITERS;
  double xi1 = 0, xi2 = 0;
  int k0 = 0, k1 = 0, k2 = 0, stalled = 0;
  std::vector<double> rnorm;
  std::string branches;
  int64_t n_T = 0, n_L = 0, n_Lt = 0;
};

class Engine {
 public:
  Engine(const spock_problem_desc* desc, const Params& prm);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  int64_t nz() const { return lay_.nz; }
  int64_t neta() const { return lay_.neta; }
  double alpha() const { return alpha_; }
  const OpNorm& op_norm() const { return norm_; }

  // boundary-layout entry points (host or device pointers)
  void apply_T_b(const double* z, const double* eta, double* zo, double* eo);
  void apply_L_b(const double* z, double* eta);
  void apply_Lt_b(const double* eta, double* z);
  double m_norm_b(const double* z, const double* eta, double alpha);
  void proj_s1_b(double* z);
  void proj_s2_b(double* z);
  void proj_s3_b(double* eta);
  void unscale_b(const double* zs, double* z);
  void solve_b(const double* x_init, const double* wz, const double* we, double* oz, double* ozs, double* oe,
               bool supermann, Status& st);
  // device-resident loop (CUDA graph with conditional nodes); false: not applicable
  // (cancellation callback, Anderson memory above kLoopMaxMem, SPOCK_SOLVE_GRAPH=0)
  bool solve_graph(const double* x_init, const double* wz, const double* we, double* oz, double* ozs, double* oe,
                   bool supermann, Status& st);
  struct GraphLoop {
    cudaGraphExec_t exec = nullptr;
    LoopArgs A{};
    double* Lrz = nullptr;
  };
  GraphLoop gloop_[2];  // CP, SuperMann
  // CTA-resident loop for small trees (small.cuh)
  static constexpr double kSmallBytes = 2.0e6;  // algorithmic bytes per T at most (one SM's L1 / L2 share)
  bool small_eligible() const;
  // which loop a solve runs: "small" (CTA-resident), "graph" (device-resident graph) or "host"
  const char* loop_path() const;
  bool solve_small(const double* x_init, const double* wz, const double* we, double* oz, double* ozs, double* oe,
                   bool supermann, Status& st);
  SmallArgs small_{};
  bool small_ok_ = false;  // decided at construction (SPOCK_SMALL=0/1 overrides)
  int small_cap_ = 0;
  // cluster-resident loop (cluster.cuh): the small loop's allocations packed
  // into the shared memory of a thread-block cluster (SPOCK_CLUSTER=0/1)
  bool cluster_ok_ = false;
  bool small_solved_ = false;  // a small / cluster solve ran (set_grid_cap is then rejected, as after a graph solve)
  bool cluster_plan(int m);
  void small_alloc();
  ClusterPlace* cplace_d_ = nullptr;
  ClusterField* cfield_d_ = nullptr;
  int cplace_n_ = 0, cfield_n_ = 0, cluster_ctas_ = 0, cluster_arena_ = 0, cplan_m_ = -1;
  std::vector<int> cown_;  // node range of each CTA
  std::map<uintptr_t, size_t> alloc_bytes_;  // every dalloc allocation: base -> bytes
  std::vector<int64_t> hxo_, huo_, ao_, hno_, aNo_;  // host copies of the SOC block offsets
  void build_loop_graph(GraphLoop& G, bool supermann);
  double bench_T(int k, bool graph, bool flush);
  void bench_kernels(int k, bool flush, double* ms);
  void traffic(double* bytes) const;
  // subtree sharding (see engine.cu)
  void shard_setup(int G, int rank, int ts, const int* back_a, int na, const int* back_b, int nb, const int* s2,
                   int ns2, const int* fwd, int nf, double* xbuf);
  void shard_T_A(const double* z, const double* eta, double* zo, double* eo);
  void shard_T_B(const double* z, const double* eta, double* zo, double* eo);
  void shard_masks(uint8_t* zm, uint8_t* em) const;
  void shard_weights(uint8_t* zm, uint8_t* em);
  void shard_apply_T_b(int phase, const double* z, const double* eta, double* zo, double* eo);
  void shard_bench(int phase, int parity);
  // sharded solve: the host provides the collectives (op 0: all-gather of the
  // exchange buffer, 1: all-reduce sum, 2: all-reduce max, on device buffers)
  typedef int (*CollFn)(void* user, int op, double* buf, int64_t n);
  void shard_set_collectives(CollFn fn, void* user);
  // NCCL communicator over the ranks of the sharded solver (id: ncclUniqueId
  // from rank 0); afterwards T, L*, the solves' reductions and the exchange all
  // enqueue ncclAllGather / ncclAllReduce on the solver stream
  void shard_nccl_init(const void* id, int nranks, int rank);
  bool shard_coll_on() const { return shard_.coll != nullptr || shard_.nccl != nullptr; }
  cudaStream_t stream() const { return st_; }
  int device() const { return dev_; }
  double* scratch_z(int k) const { return scratch_z_[k]; }
  double* scratch_e(int k) const { return scratch_e_[k]; }
  int launches_per_T() const {
    return fused_ok_ ? 1 : (t_wide_ ? (t_split_ ? 3 : 1) : 2 + 2 * (p_.tree.horizon + 1) + 1 + 1);
  }
  // SPOCK_WIDE_PROF=1: cycle counters of the wide kernel (summed over warps and launches)
  void wide_profile(unsigned long long* out10);
  const char* t_path() const { return fused_ok_ ? "fused" : (t_wide_ ? "wide" : "stages"); }
  // CTAs of the fused T launch; a cap lets several solvers share the SMs
  // (concurrent solves on their own streams).  Must precede the first solve /
  // bench: the cached graphs hold the launch configuration.
  int fused_grid() const { return fused_ok_ ? fused_grid_ : 0; }
  void set_grid_cap(int ctas);

 private:
  void upload();
  // device-side SOC epigraph data (setup_dev.cu): eigenvalues,
  // ranks and the merged row order first (the layouts need the ranks), then
  // the head maps, kernel components and translations straight into D_
  bool soc_dev_ = false;
  struct SocScratch {
    double *Q = nullptr, *R = nullptr, *q = nullptr, *r = nullptr, *QN = nullptr, *qN = nullptr;
    double *Wx = nullptr, *Vx = nullptr, *Wu = nullptr, *Vu = nullptr;
    std::vector<void*> owned;
  } socs_;
  void soc_device_ranks();
  void soc_device_build(const std::vector<int64_t>& hxo, const std::vector<int64_t>& huo,
                        const std::vector<int64_t>& ao, const std::vector<int64_t>& hno,
                        const std::vector<int64_t>& aNo);
  void setup_fused();
  void setup_wide(bool force);
  void compute_pool();
  std::vector<int> pool_rep_;  // node whose matrix blocks the streaming kernel reads for node i
  int pool_unique_ = 0;
  void factorize();
  void power_iteration();
  void set_xinit(const double* x_orig_host);
  // internal-layout device operations
  void T(const double* z, const double* eta, double* zo, double* eo);
  void L(const double* z, double* eta);
  void Lt(const double* eta, double* z);
  void dots(std::initializer_list<std::pair<const double*, const double*>> pairs, int64_t n_default,
            const std::vector<int64_t>& ns, double* host_out);
  void sync();
  void to_internal_eta(const double* src_any, double* dst_dev);
  void from_internal_eta(const double* src_dev, double* dst_any);
  void copy_in_z(const double* src_any, double* dst_dev);
  void copy_out(const double* src_dev, double* dst_any, int64_t n);
  template <class Ty>
  Ty* dalloc(size_t n);
  template <class Ty>
  Ty* dupload(const std::vector<Ty>& h);
  double* dupload(const BigVec& h);

  Params prm_;
  Problem p_;
  Vec raw_xinit_;
  Precond pc_;
  SocData soc_;
  Layouts lay_;
  Dev D_{};
  std::vector<int> stage_start_;
  cudaStream_t st_ = nullptr;
  int dev_ = 0;  // the device current at construction; every C-ABI entry makes it current again
  std::vector<void*> allocs_;
  OpNorm norm_;
  double alpha_ = 0.0;
  // internal buffers
  int* perm_eta_ = nullptr;  // internal index -> boundary index
  bool perm_identity_ = true;
  double* d1_ = nullptr;
  double* d2_ = nullptr;
  double* xinit_ = nullptr;
  double* partial_ = nullptr;
  double* red_out_ = nullptr;
  double* host_red_ = nullptr;  // pinned
  double* scratch_z_[3] = {};
  double* scratch_e_[3] = {};
  cudaGraphExec_t bench_graph_ = nullptr;
  bool fused_ok_ = false;
  bool narrow_ = true;
  FusedArgs fargs_{};
  int fused_grid_ = 0, fused_grid_full_ = 0;
  size_t fused_sync_bytes_ = 0;
  bool wide_ok_ = false;  // streaming kernel set up (records, smem, grid)
  bool t_wide_ = false;   // T runs on it
  int t_split_ = 0;       // > 0: T in three launches, the stages below t_split_ on the latency configuration
  WRec* tsplit_rec_[3] = {};
  int tsplit_n_[3] = {};
  bool lop_wide_ = true;  // standalone L / L* run on it
  bool lop_narrow_ = true;  // else lop.cu (CTA per node, one-shot staging)
  int lop_rows_ = 0, lop_mat_ = 0, lop_vec_ = 0;
  WideArgs wlat_{};
  int wide_grid_lat_ = 0;
  void launch_wide(WideArgs A, const WRec* recs, int ntick);
  WRec* lrec_ = nullptr;
  WRec* ltrec_ = nullptr;
  int nlrec_ = 0, nltrec_ = 0;
  WideArgs wargs_{};
  int wide_grid_ = 0, wide_rows_ = 0, wide_ctas_ = 1;
  int max_dense_s2_ = 0;
  int* wide_flags_ = nullptr;
  std::vector<WRec> wrecs_;  // host copy of the full ticket list (shard subsets are drawn from it)
  struct ShardState {
    bool on = false;
    void* nccl = nullptr;  // ncclComm_t: the collectives run from C++ on the solver stream (shard_nccl_init)
    int G = 1, rank = 0, ts = 0, bfirst = 0, nbound = 0, q = 0, b0 = 0, b1 = 0, E = 0, nA = 0, nB = 0;
    WRec* recA = nullptr;
    WRec* recB = nullptr;
    int64_t* xidx = nullptr;
    double* xbuf = nullptr;
    std::vector<uint8_t> owned;
    WRec* recL = nullptr;
    WRec* recLtA = nullptr;
    WRec* recLtB = nullptr;
    int nL = 0, nLtA = 0, nLtB = 0;
    double *mz = nullptr, *me = nullptr, *wz = nullptr, *we = nullptr, *wv = nullptr;
    CollFn coll = nullptr;
    void* coll_user = nullptr;
  } shard_;
  bool shard_solving_ = false;
  std::vector<WRec> lrecs_h_, ltrecs_h_;
  void coll(int op, double* buf, int64_t n);
  bool agree_cancel(bool mine);
  void gram_update(int cols, bool sharded);
  double* gram_partial_ = nullptr;  // block partials of the double-double Gram update
  double* gram_out_ = nullptr;      // its (hi, lo) results (host loop)
  double* gram_gather_ = nullptr;   // sharded: every rank's results
  std::vector<dd> gram_h_, gram_r_;  // host loop: Gram by history position, M_d' r
  double* cancel_dev_ = nullptr;
  void shard_T(const double* z, const double* eta, double* zo, double* eo);
  void shard_L(const double* z, double* eta);
  void shard_Lt(const double* eta, double* z);
  size_t wide_flag_bytes_ = 0;
  double* flush_buf_ = nullptr;
  void flush_l2();
};

}  // namespace spock
