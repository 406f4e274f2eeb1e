// Host-callable launchers of the B200 SPOCK kernels (kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include "dev.cuh"
#include "loop.hpp"

namespace spock {

constexpr int kRedBlocks = 2 * 148;  // fixed grid => run-to-run identical reductions
constexpr int kRedThreads = 256;
constexpr int kMaxDots = 16;
// one reduction scratch region: kMaxDots x kRedBlocks block partials, then the
// arrival counter of the last-block finalize (grid_finalize, dev.cuh)
constexpr int kRedRegion = kMaxDots * kRedBlocks + 2;
__host__ __device__ inline unsigned int* red_counter(double* partial) {
  return reinterpret_cast<unsigned int*>(partial + size_t(kMaxDots) * kRedBlocks);
}

struct LinCombArgs {
  const double* x[16];
  double c[16];
};
struct DotArgs {
  const double* x[kMaxDots];
  const double* y[kMaxDots];
  int n[kMaxDots];
  int ndots;
  const double* w[kMaxDots];  // optional 0/1 weights (sharded solve: entries this rank counts)
};
struct XiArgs {
  const double* x[2];
  const double* y[2];
  const double* d[2];
  int n[2];
  double alpha;
  const double* w[2];  // optional 0/1 masks (sharded solve: entries this rank computes)
};
struct BGemmArgs {
  const double* const* A;
  const double* const* B;
  double* const* C;
  int m, n, k, lda, ldb, ldc, ta, tb;
  double alpha, beta;
};
struct Alg1Args {
  int b;  // first node of the launch range
  int nx, nu;
  int64_t m1_stride, k_stride, r_stride;
  const int* cf;
  const int* cc;
  const int* anc;
  const double* A;   // per non-root
  const double* B;
  const double* rt;  // per non-root temporaries
  const double* kt;
  const double* ge;
  const double* pt;
  const double* he;
  double* P;     // per node
  double* K;     // per non-leaf
  double* KT;
  double* Rinv;
  double* g;
  double* h;
  double* M1;    // per non-root
  double* M1T;
  double* Rt_out;    // optional per non-leaf
  double* Abar_out;  // optional per non-root
  int* err;
};

// CTA-resident SuperMann / CP solve for small trees (small.cuh)
struct SmallArgs {
  LoopArgs L;  // state (device copy of the initial LoopState), parameters, history rings, V TV R C CR PSI
  Dev D;
  const int* stage_start;  // [N + 2]
  double *TC, *PV, *Lrz, *cLrz, *Lsre, *tmpz, *tmpe;
  const double *d1, *d2;  // termination scalings
  int supermann;
  unsigned long long* prof;  // optional [8] clock64 totals per phase class (SPOCK_SMALL_PROF=1)
};
void launch_small_solve(const SmallArgs& A, cudaStream_t st);
constexpr int kSmallThreadsHost = 256;

// Cluster-resident solve (cluster.cuh): the device allocations the small loop
// touches, packed whole into the shared memory of a thread-block cluster.
constexpr int kClusterMax = 16;
struct ClusterPlace {  // one device allocation staged into CTA `cta`'s arena
  const char* src;
  int64_t bytes;  // multiple of 8
  int32_t cta, off;  // arena offset (16-byte aligned)
  int32_t writable;  // copied back to HBM at the end of the solve
  int32_t pad_;
};
struct ClusterField {  // a pointer field of SmallArgs, relocated into a placement
  int32_t field;  // byte offset of the pointer inside SmallArgs
  int32_t place;
  int64_t delta;  // byte offset from the placement's start (negative: a rebased node slice)
  int32_t cta;    // -1: every CTA applies it; else only that CTA
  int32_t pad_;
};
struct ClusterArgs {
  SmallArgs S;  // global pointers (the staging sources); relocated per CTA in the kernel
  const ClusterPlace* place;
  int nplace;
  const ClusterField* field;
  int nfield;
  int own[kClusterMax + 1];  // CTA c runs the operator phases of nodes [own[c], own[c+1])
};
int cluster_static_smem();
// arena bytes per CTA and cluster size; returns the launch error (cluster
// launches fail, e.g., when the arena does not fit)
cudaError_t launch_cluster_solve(const ClusterArgs& A, int ctas, int arena_bytes, cudaStream_t st);
// clusters of this shape the device can hold at once (0: it cannot launch)
int cluster_max_active(int ctas, int arena_bytes);

void launch_Lt(const Dev& D, const double* eta, const double* zin, double* zout, double a, double b, double c0,
               cudaStream_t st);
void launch_L(const Dev& D, const double* z1, double a1, const double* z2, double a2, const double* eta_in,
              double* eta_out, double alpha, bool dual, cudaStream_t st);
void launch_s1(const Dev& D, const int* stage_start, double* z, cudaStream_t st);
void launch_s2(const Dev& D, double* z, cudaStream_t st);
void launch_s3(const Dev& D, double* eta, cudaStream_t st);
void launch_axpby(int n, double a, const double* x, double b, const double* y, double* out, cudaStream_t st);
void launch_lincomb(int n, int nv, const LinCombArgs& A, double* out, cudaStream_t st);
void launch_gather(int n, const int* perm, const double* src, double* dst, cudaStream_t st);
void launch_scatter(int n, const int* perm, const double* src, double* dst, cudaStream_t st);
void launch_dots(const DotArgs& A, double* partial, double* out, cudaStream_t st);
void launch_xi(const XiArgs& A, double* partial, double* out, cudaStream_t st);
void launch_bgemm(const BGemmArgs& G, int count, cudaStream_t st);
void launch_alg1_parent(const Alg1Args& P, int count, cudaStream_t st);
void launch_alg1_parent2(const Alg1Args& P, int count, cudaStream_t st);
void launch_alg1_child_abar(const Alg1Args& P, int count, cudaStream_t st);
cudaError_t set_alg1_smem(int bytes);
void set_carveout_all();
// latency-optimised CTA-per-node L / L* (narrow.cu)
void set_carveout_narrow();
void launch_L_narrow(const Dev& D, const double* z, double* eta, cudaStream_t st);
void launch_Lt_narrow(const Dev& D, const double* eta, double* z, cudaStream_t st);

}  // namespace spock
