// Device-side setup kernels (setup_dev.hpp): batched symmetric
// eigendecompositions and the per-block SOC epigraph data of
// soc_data_quadlin (proj/src/problem.cpp:113-161).
//
// Eigendecomposition: one CTA per matrix, a (n2 x n2, n2 = n rounded up to
// even) and the rotation accumulator U (n x n) in shared memory.  Cyclic
// Jacobi in round-robin ("chess tournament") order: each of the n2-1 rounds
// of a sweep rotates n2/2 disjoint index pairs at once, so the column update,
// the row update and the U update of a round are each one fully parallel pass
// over the CTA.  The rotation formula and the negligibility test are the host
// sym_eig's (model.cpp); sweeps stop when a whole sweep applied no rotation.
// The output is canonical like the host's: eigenvalues ascending (stable in
// the diagonal index), each eigenvector's largest-|entry| positive.
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "setup_dev.hpp"

namespace spock {

namespace {

__device__ __forceinline__ void rr_pair(int n2, int round, int k, int& p, int& q) {
  // round-robin: player n2-1 fixed, the others rotate
  const int m = n2 - 1;
  if (k == 0) {
    p = round;
    q = m;
  } else {
    p = (round + k) % m;
    q = (round - k + m) % m;
  }
  if (p > q) {
    const int t = p;
    p = q;
    q = t;
  }
}

__global__ void __launch_bounds__(1024) k_sym_eig(const EigJob* __restrict__ jobs) {
  extern __shared__ __align__(16) double esm[];
  const EigJob J = jobs[blockIdx.x];
  const int n = J.n;
  if (n <= 0) return;
  const int n2 = (n + 1) & ~1, np = n2 / 2;
  double* a = esm;                       // n2 x n2
  double* u = a + size_t(n2) * n2;       // n x n
  double* cs = u + size_t(n) * n;        // np
  double* sn = cs + np;                  // np
  int* act = reinterpret_cast<int*>(sn + np);  // np: pair rotated this round
  __shared__ int any;
  const int tid = threadIdx.x, nt = blockDim.x;
  auto A = [&](int i, int j) -> double& { return a[i + j * n2]; };
  for (int idx = tid; idx < n2 * n2; idx += nt) {
    const int i = idx % n2, j = idx / n2;
    a[idx] = (i < n && j < n) ? 0.5 * (J.M[i + size_t(j) * n] + J.M[j + size_t(i) * n]) : 0.0;
  }
  for (int idx = tid; idx < n * n; idx += nt) u[idx] = (idx % n == idx / n) ? 1.0 : 0.0;
  __syncthreads();
  const double small = DBL_EPSILON * 1e-3;
  for (int sweep = 0; sweep < 100; ++sweep) {
    if (tid == 0) any = 0;
    __syncthreads();
    for (int round = 0; round < n2 - 1; ++round) {
      // 1. rotation of each pair (host formula), or the negligible entry zeroed
      for (int k = tid; k < np; k += nt) {
        int p, q;
        rr_pair(n2, round, k, p, q);
        int on = 0;
        double c = 1.0, s = 0.0;
        if (q < n) {
          const double apq = A(p, q);
          if (apq != 0.0) {
            const double app = A(p, p), aqq = A(q, q);
            if (fabs(apq) <= small * sqrt(fabs(app) * fabs(aqq)) &&
                fabs(apq) <= 1e-300 + small * fmax(fabs(app), fabs(aqq))) {
              A(p, q) = 0.0;
              A(q, p) = 0.0;
            } else {
              const double th = (aqq - app) / (2.0 * apq);
              const double t = fabs(th) > 1e150 ? 0.5 / th : (th >= 0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
              c = 1.0 / sqrt(t * t + 1.0);
              s = t * c;
              on = 1;
            }
          }
        }
        cs[k] = c;
        sn[k] = s;
        act[k] = on;
        if (on) any = 1;
      }
      __syncthreads();
      // 2. columns p, q of a and of U (a <- a J, U <- U J)
      for (int idx = tid; idx < np * n2; idx += nt) {
        const int k = idx / n2, r = idx % n2;
        if (!act[k]) continue;
        int p, q;
        rr_pair(n2, round, k, p, q);
        const double c = cs[k], s = sn[k];
        const double kp = A(r, p), kq = A(r, q);
        A(r, p) = c * kp - s * kq;
        A(r, q) = s * kp + c * kq;
        if (r < n) {
          const double up = u[r + p * n], uq = u[r + q * n];
          u[r + p * n] = c * up - s * uq;
          u[r + q * n] = s * up + c * uq;
        }
      }
      __syncthreads();
      // 3. rows p, q (a <- J' a)
      for (int idx = tid; idx < np * n2; idx += nt) {
        const int k = idx / n2, col = idx % n2;
        if (!act[k]) continue;
        int p, q;
        rr_pair(n2, round, k, p, q);
        const double c = cs[k], s = sn[k];
        const double pk = A(p, col), qk = A(q, col);
        A(p, col) = c * pk - s * qk;
        A(q, col) = s * pk + c * qk;
      }
      __syncthreads();
      for (int k = tid; k < np; k += nt) {
        if (!act[k]) continue;
        int p, q;
        rr_pair(n2, round, k, p, q);
        A(p, q) = 0.0;
        A(q, p) = 0.0;
      }
      __syncthreads();
    }
    const int done = !any;
    __syncthreads();
    if (done) break;
  }
  // ascending, stable in the diagonal index; largest-|entry| positive
  for (int o = tid; o < n; o += nt) {
    const double d = A(o, o);
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const double e = A(j, j);
      rank += (e < d) || (e == d && j < o);
    }
    int im = 0;
    for (int i = 1; i < n; ++i)
      if (fabs(u[i + o * n]) > fabs(u[im + o * n]) * (1.0 + 1e-12)) im = i;
    const double sg = u[im + o * n] < 0 ? -1.0 : 1.0;
    J.W[rank] = d;
    for (int i = 0; i < n; ++i) J.V[i + size_t(rank) * n] = sg * u[i + o * n];
  }
}

// per node: ranks, lambda_max, PSD check, merged order (soc_block, model.cpp)
__global__ void k_soc_rank(const SocRankArgs A) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= A.nb) return;
  const double* wx = A.Wx + size_t(b) * A.nx;
  const double* wu = A.Wu ? A.Wu + size_t(b) * A.nu : nullptr;
  const int nu = wu ? A.nu : 0;
  double lmax = 0.0, lmin = INFINITY;
  for (int k = 0; k < A.nx; ++k) lmax = fmax(lmax, wx[k]), lmin = fmin(lmin, wx[k]);
  for (int k = 0; k < nu; ++k) lmax = fmax(lmax, wu[k]), lmin = fmin(lmin, wu[k]);
  if (!(lmin >= -1e-10 * fmax(lmax, 1.0))) atomicExch(A.err, 1);
  const double th = 1e-10 * lmax;
  // eigenvalues ascending: the kept ones are a suffix
  int px = 0, pu = 0;
  for (int k = 0; k < A.nx; ++k) px += wx[k] > th;
  for (int k = 0; k < nu; ++k) pu += wu[k] > th;
  A.px[b] = px;
  if (A.pu) A.pu[b] = pu;
  A.lmax[b] = lmax;
  int* perm = A.perm + size_t(b) * (A.nx + A.nu);
  int ix = 0, iu = 0, pos = 0;
  const int x0 = A.nx - px, u0 = nu - pu;
  while (ix < px || iu < pu) {
    const bool takex = iu >= pu || (ix < px && wx[x0 + ix] <= wu[u0 + iu]);
    if (takex)
      perm[ix++] = pos++;
    else
      perm[px + iu++] = pos++;
  }
}

// SMS = S' M S with S = V(:, n-p..n): T = M S (n x p) in shared memory, then S'T
__global__ void __launch_bounds__(1024) k_soc_sms(const SocBlockJob* __restrict__ jobs) {
  extern __shared__ __align__(16) double ssm[];
  const SocBlockJob J = jobs[blockIdx.x];
  const int n = J.n, p = J.p, tid = threadIdx.x, nt = blockDim.x;
  if (p <= 0) return;
  const double* S = J.V + size_t(n - p) * n;
  double* T = ssm;
  for (int idx = tid; idx < n * p; idx += nt) {
    const int i = idx % n, k = idx / n;
    double s = 0.0;
    for (int j = 0; j < n; ++j) s = fma(J.M[i + size_t(j) * n], S[j + size_t(k) * n], s);
    T[idx] = s;
  }
  __syncthreads();
  for (int idx = tid; idx < p * p; idx += nt) {
    const int a2 = idx % p, b = idx / p;
    double s = 0.0;
    for (int i = 0; i < n; ++i) s = fma(S[i + size_t(a2) * n], T[i + size_t(b) * n], s);
    J.sms[idx] = s;
  }
}

// sq = U diag(sqrt e) U', isq = U diag(1/sqrt e) U'; H = sq S', qk = v - S S'v,
// w = isq S'v
__global__ void __launch_bounds__(1024) k_soc_build(const SocBlockJob* __restrict__ jobs) {
  extern __shared__ __align__(16) double bsm[];
  const SocBlockJob J = jobs[blockIdx.x];
  const int n = J.n, p = J.p, tid = threadIdx.x, nt = blockDim.x;
  const double* S = J.V + size_t(n - p) * n;
  double* sq = bsm;                 // p x p
  double* isq = sq + size_t(p) * p;  // p x p
  double* sv = isq + size_t(p) * p;  // p
  double* ev = sv + p;               // p (sqrt e)
  for (int k = tid; k < p; k += nt) {
    ev[k] = sqrt(fmax(0.0, J.W2[k]));
    double s = 0.0;
    for (int i = 0; i < n; ++i) s = fma(S[i + size_t(k) * n], J.v[i], s);
    sv[k] = s;
  }
  __syncthreads();
  for (int idx = tid; idx < p * p; idx += nt) {
    const int i = idx % p, j = idx / p;
    double s = 0.0, si = 0.0;
    for (int k = 0; k < p; ++k) {
      const double uu = J.U2[i + size_t(k) * p] * J.U2[j + size_t(k) * p];
      s = fma(uu, ev[k], s);
      si = fma(uu, ev[k] > 0 ? 1.0 / ev[k] : 0.0, si);
    }
    sq[idx] = s;
    isq[idx] = si;
  }
  __syncthreads();
  for (int idx = tid; idx < p * n; idx += nt) {
    const int i = idx % p, j = idx / p;
    double s = 0.0;
    for (int k = 0; k < p; ++k) s = fma(sq[i + k * p], S[j + size_t(k) * n], s);
    J.H[i + size_t(j) * p] = s;
    J.HT[j + size_t(i) * n] = s;
  }
  for (int i = tid; i < n; i += nt) {
    double s = J.v[i];
    for (int k = 0; k < p; ++k) s -= S[i + size_t(k) * n] * sv[k];
    J.qk[i] = s;
  }
  for (int i = tid; i < p; i += nt) {
    double s = 0.0;
    for (int k = 0; k < p; ++k) s = fma(isq[i + k * p], sv[k], s);
    J.w[i] = s;
  }
}

__global__ void k_soc_tail(const SocTailArgs T) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= T.nb) return;
  const int px = T.px[b], pu = T.pu ? T.pu[b] : 0, p = px + pu;
  const double* w = T.w + size_t(b) * (T.nx + T.nu);
  double* a = T.a + T.a_off[b];
  double qn2 = 0.0;
  for (int k = 0; k < px; ++k) {
    a[k] = -0.5 * w[k];
    qn2 += w[k] * w[k];
  }
  for (int k = 0; k < pu; ++k) {
    a[px + k] = -0.5 * w[T.nx + k];
    qn2 += w[T.nx + k] * w[T.nx + k];
  }
  a[p] = -0.125 * qn2 + 0.5;
  a[p + 1] = -0.125 * qn2 - 0.5;
  const double* qk = T.qk + size_t(b) * T.qk_stride;
  double q2 = 0.0;
  for (int k = 0; k < T.qk_stride; ++k) q2 += qk[k] * qk[k];
  T.qk2[b] = q2;
}

__global__ void k_eye(double* P, int64_t count, int n) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= count * n) return;
  const int64_t b = t / n;
  const int k = int(t % n);
  P[size_t(b) * n * n + k + size_t(k) * n] = 1.0;
}

// a Jacobi round updates n2/2 column pairs of n2 entries (then as many rows):
// enough threads that a round is one or two passes
// (n <= 64: the smaller CTAs keep several matrices per SM in flight, measured
// faster on c4's 50 x 50 blocks; n > 64 holds one matrix per SM anyway)
int threads_for(int n) { return n <= 32 ? 64 : (n <= 64 ? 128 : 1024); }

}  // namespace

int eig_smem_bytes(int n) {
  const int n2 = (n + 1) & ~1, np = n2 / 2;
  return int(sizeof(double) * (size_t(n2) * n2 + size_t(n) * n + 2 * np) + sizeof(int) * np + 16);
}

cudaError_t eig_configure(int nmax) {
  const int bytes = eig_smem_bytes(nmax);
  cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(&k_sym_eig),
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return e;
  const int sb = int(sizeof(double) * size_t(nmax) * nmax);
  e = cudaFuncSetAttribute(reinterpret_cast<const void*>(&k_soc_sms), cudaFuncAttributeMaxDynamicSharedMemorySize,
                           sb);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(reinterpret_cast<const void*>(&k_soc_build),
                              cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * sb + int(16 * nmax) + 16);
}

void launch_sym_eig(const EigJob* jobs, int njobs, int nmax, cudaStream_t st) {
  if (njobs > 0) k_sym_eig<<<njobs, threads_for(nmax), eig_smem_bytes(nmax), st>>>(jobs);
}

void launch_soc_rank(const SocRankArgs& a, cudaStream_t st) {
  if (a.nb > 0) k_soc_rank<<<(a.nb + 127) / 128, 128, 0, st>>>(a);
}

void launch_soc_sms(const SocBlockJob* jobs, int njobs, int nmax, cudaStream_t st) {
  if (njobs > 0) k_soc_sms<<<njobs, threads_for(nmax), sizeof(double) * size_t(nmax) * nmax, st>>>(jobs);
}

void launch_soc_build(const SocBlockJob* jobs, int njobs, int nmax, cudaStream_t st) {
  if (njobs > 0)
    k_soc_build<<<njobs, threads_for(nmax), 2 * sizeof(double) * size_t(nmax) * nmax + 16 * nmax + 16, st>>>(jobs);
}

void launch_eye(double* P, int64_t count, int n, cudaStream_t st) {
  if (count <= 0) return;
  cudaMemsetAsync(P, 0, sizeof(double) * size_t(count) * n * n, st);
  const int64_t t = count * n;
  k_eye<<<unsigned((t + 255) / 256), 256, 0, st>>>(P, count, n);
}

void launch_soc_tail(const SocTailArgs& t, cudaStream_t st) {
  if (t.nb > 0) k_soc_tail<<<(t.nb + 127) / 128, 128, 0, st>>>(t);
}

}  // namespace spock
