// Streaming dataflow T for wide trees (wide.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "dev.cuh"

namespace spock {

constexpr int kWSpans = 16;  // staged vector operands per item
constexpr int kWMats = 5;    // streamed matrices per item

// base arrays of the staged vector spans (WB_Z / WB_ETA are the launch's inputs)
enum WBase : int {
  WB_Z = 0, WB_ETA, WB_QK, WB_GD, WB_H, WB_G, WB_QKN, WB_GDN, WB_CV, WB_A, WB_LO, WB_HI, WB_RB, WB_AN, WB_LON,
  WB_HIN, WB_COUNT
};

// Per-ticket record, built once on the host (Engine::setup_wide), fetched by a
// 256-byte bulk copy three tickets ahead of use: node metadata, the streamed
// matrices (producer) and the independent vector operands (staged by cp.async
// when the item starts).
struct alignas(16) WRec {
  int32_t kind, node, nch, c0;
  int32_t anc, px, pu, pN;
  int32_t nc, ny, so, s2o;  // so: seg1 offset (non-leaf) / seg3 offset (leaf)
  int32_t yo, nmat, unstaged, nspan;  // unstaged: bit k -> span k is read from global memory
  const double* mp[kWMats];
  int16_t mrows[kWMats];
  int16_t mcols[kWMats];
  int16_t mcc[kWMats];  // columns per ring chunk (even; set for the launch's chunk size)
  int16_t pad0_;
  int32_t voff[kWSpans];
  uint16_t vcnt[kWSpans];
  uint8_t vbase[kWSpans];
  uint8_t pad1_[8];
};
static_assert(sizeof(WRec) == 256, "WRec is one 256-byte bulk copy");

struct WideArgs {
  Dev D;
  const double* z;
  const double* eta;
  double* zo;
  double* eo;
  double alpha;
  int* flagB;   // [nn]  backward item of node i done (T12_i, adj_i, d_i); zeroed before each launch
  int* flagS2;  // [nnl] S2 of parent i done
  int* flagF;   // [nn]  forward (x+, u+) of node i done
  int slots;    // ring slots per warp (power of two)
  int chunk;    // doubles per ring slot (even)
  int warps;    // warps per CTA
  int vecd;     // doubles per per-warp vector buffer (three per warp)
  int vrec;     // doubles of staged vector operands per warp
  int ycap;     // y-block values staged per forward item (larger blocks read from L2)
  int l2_prefetch;  // 1: bulk-prefetch the next ticket's matrices into L2
  const WRec* recs;           // ticket list ([nn + nnl + nn] for a whole T)
  int ntick;                  // number of tickets
  const double* vb[WB_COUNT];  // span bases (WB_Z, WB_ETA unused: taken from z, eta)
  unsigned long long* prof;   // optional [13] cycle counters (SPOCK_WIDE_PROF)
};

// exchange records of the stage-ts nodes of a sharded T (engine.cu shard_*):
// per node [adj (m) | T12 (m) | z_tau | z_s | eta_tau0 | eta_tau1 | eta_s0 | eta_s1]
struct ShardXArgs {
  Dev D;
  const double* z;
  const double* eta;
  const int64_t* xidx;  // 6 indices per stage-ts node: z_tau, z_s, eta_tau0, eta_tau1, eta_s0, eta_s1 (-1: none)
  double* xbuf;         // [G * q * E]
  int bfirst, b0, b1, E;
  int* flagB;           // unpack: set for remote nodes
  int nbound;
  int vec;              // 1: also exchange the z / eta entries (T); 0: adj / T12 only (L*)
};
void launch_shard_pack(const ShardXArgs& X, cudaStream_t st);
void launch_shard_unpack(const ShardXArgs& X, cudaStream_t st);

// standalone L / L* for narrow trees, CTA per node (lop.cu)
int lop_smem_bytes(int rows, int mat_cap, int vec_cap);
cudaError_t lop_configure(int bytes);
void launch_L_lop(const Dev& D, const WideArgs& W, const WRec* lrec, const double* z, double* eta, int rows,
                  int mat_cap, int vec_cap, cudaStream_t st);
void launch_Lt_lop(const Dev& D, const WideArgs& W, const WRec* ltrec, const double* eta, double* z, int rows,
                   int mat_cap, int vec_cap, cudaStream_t st);

int wide_smem_bytes(const WideArgs& A);
int wide_rows(const Dev& D, int max_nc);  // register row groups (template parameter)
cudaError_t wide_configure(int rows, int ctas, int smem_bytes);
const void* wide_kernel_ptr(int rows, int ctas);
cudaError_t launch_T_wide(const WideArgs& A, int rows, int ctas, int grid, cudaStream_t st);

}  // namespace spock
