// Anderson least squares of the SuperMann direction (proj/src/solver.cpp:55-77)
// in double-double arithmetic, shared by the device controller (loop.cu) and the
// host-driven loop (engine.cu).
//
// The reference solves min ||M_d kappa - r|| by Eigen's ColPivHouseholderQR
// with setThreshold(1e-12) (solver.cpp:73-75; the oracle restates it,
// oracle/orc_la.cpp colpiv_qr_solve).  On the device M_d is n_v x m with n_v up
// to 10^7, so the factorisation is taken from the Gram matrix G = M_d'M_d and
// g = M_d'r instead: in exact arithmetic the column-pivoted Cholesky of G is the
// R factor of the column-pivoted QR of M_d (same pivot order, since the
// remaining column norms are the Schur-complement diagonals) and R'c = P'g gives
// c = Q'r.  Forming G in plain double squares the conditioning -- pivots below
// sqrt(eps) relative become unresolvable, where the reference keeps them down
// to 1e-12 relative.  So G and g are accumulated in double-double (error-free
// two-product and two-sum, ~106-bit significands; dd_dots in loop.cu) and the
// pivoted Cholesky, the rank decisions and the triangular solves run in
// double-double too.  The decisions restate Eigen's: the pivot is the first
// largest remaining column norm with the columns physically transposed, the
// "nonzero pivots" cut at |R_kk|^2 < (max_j |a_j| eps)^2 (rows - k) / rows, and
// the solve keeps the pivots above 1e-12 of the largest |R_kk| among them.
#pragma once

#include <cmath>
#include <cstdint>

#ifndef __CUDACC__  // host-only translation units (C-ABI test entry)
#define __host__
#define __device__
#endif

namespace spock {

struct dd {
  double hi, lo;
};

__host__ __device__ inline dd dd_two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
__host__ __device__ inline dd dd_quick(double a, double b) {
  const double s = a + b;
  return {s, b - (s - a)};
}
__host__ __device__ inline dd dd_two_prod(double a, double b) {
  const double p = a * b;
#ifdef __CUDA_ARCH__
  return {p, __fma_rn(a, b, -p)};
#else
  return {p, std::fma(a, b, -p)};
#endif
}
__host__ __device__ inline dd dd_add(dd a, dd b) {
  dd s = dd_two_sum(a.hi, b.hi);
  const dd t = dd_two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = dd_quick(s.hi, s.lo);
  s.lo += t.lo;
  return dd_quick(s.hi, s.lo);
}
__host__ __device__ inline dd dd_neg(dd a) { return {-a.hi, -a.lo}; }
__host__ __device__ inline dd dd_sub(dd a, dd b) { return dd_add(a, dd_neg(b)); }
__host__ __device__ inline dd dd_mul(dd a, dd b) {
  dd p = dd_two_prod(a.hi, b.hi);
  p.lo += a.hi * b.lo + a.lo * b.hi;
  return dd_quick(p.hi, p.lo);
}
// a += x * y (x, y doubles): the accumulation step of the Gram dots
__host__ __device__ inline dd dd_fma(dd a, double x, double y) { return dd_add(a, dd_two_prod(x, y)); }
__host__ __device__ inline dd dd_div(dd a, dd b) {
  const double q1 = a.hi / b.hi;
  dd r = dd_sub(a, dd_mul({q1, 0.0}, b));
  const double q2 = r.hi / b.hi;
  r = dd_sub(r, dd_mul({q2, 0.0}, b));
  const double q3 = r.hi / b.hi;
  return dd_add(dd_quick(q1, q2), {q3, 0.0});
}
__host__ __device__ inline dd dd_sqrt(dd a) {
  if (!(a.hi > 0.0)) return {0.0, 0.0};
  const double x = 1.0 / sqrt(a.hi);
  const double y = a.hi * x;
  const dd y2 = dd_two_prod(y, y);
  const double corr = dd_sub(a, y2).hi * (x * 0.5);
  return dd_two_sum(y, corr);
}
__host__ __device__ inline bool dd_gt(dd a, dd b) { return a.hi > b.hi || (a.hi == b.hi && a.lo > b.lo); }

// kappa (length cols, original column order) from G (cols x cols, column-major,
// both triangles) and g = M_d'r; rows = n_v (Eigen's threshold uses it).
template <int MAXC>
__host__ __device__ inline void aa_kappa_dd(const dd* G, const dd* g, int cols, int64_t rows, double* kap) {
  int piv[MAXC];
  dd W[MAXC * MAXC], Rm[MAXC * MAXC], cv[MAXC];
  for (int a = 0; a < cols; ++a) piv[a] = a;
  for (int e = 0; e < cols * cols; ++e) W[e] = G[e], Rm[e] = {0.0, 0.0};
  for (int a = 0; a < cols; ++a) cv[a] = {0.0, 0.0}, kap[a] = 0.0;
  double maxn2 = 0.0;  // largest squared column norm
  for (int a = 0; a < cols; ++a) maxn2 = fmax(maxn2, G[a + a * cols].hi);
  const double eps = 2.220446049250313e-16;
  const double thr_helper = maxn2 * eps * eps / double(rows);  // (max|a_j| eps)^2 / rows
  int nonzero = cols;
  dd maxpiv = {0.0, 0.0};
  for (int t = 0; t < cols; ++t) {
    int best = t;
    for (int a = t + 1; a < cols; ++a)
      if (dd_gt(W[piv[a] + piv[a] * cols], W[piv[best] + piv[best] * cols])) best = a;
    const dd big_sq = W[piv[best] + piv[best] * cols];
    if (nonzero == cols && big_sq.hi < thr_helper * double(rows - t)) nonzero = t;
    const int tmp = piv[t];
    piv[t] = piv[best];
    piv[best] = tmp;
    const int pt = piv[t];
    const dd rkk = dd_sqrt(W[pt + pt * cols]);
    Rm[t + pt * cols] = rkk;
    if (dd_gt(rkk, maxpiv)) maxpiv = rkk;
    if (!(rkk.hi > 0.0)) continue;  // exactly dependent: row t stays zero
    for (int a = t + 1; a < cols; ++a) Rm[t + piv[a] * cols] = dd_div(W[pt + piv[a] * cols], rkk);
    dd ct = g[pt];
    for (int s = 0; s < t; ++s) ct = dd_sub(ct, dd_mul(Rm[s + pt * cols], cv[s]));
    cv[t] = dd_div(ct, rkk);
    for (int a = t + 1; a < cols; ++a)
      for (int b = t + 1; b < cols; ++b)
        W[piv[a] + piv[b] * cols] =
            dd_sub(W[piv[a] + piv[b] * cols], dd_mul(Rm[t + piv[a] * cols], Rm[t + piv[b] * cols]));
  }
  const double pthr = maxpiv.hi * 1e-12;
  int np = 0;
  for (int t = 0; t < nonzero; ++t) np += (Rm[t + piv[t] * cols].hi > pthr) ? 1 : 0;
  dd kd[MAXC];
  for (int t = np - 1; t >= 0; --t) {
    dd s = cv[t];
    for (int a = t + 1; a < np; ++a) s = dd_sub(s, dd_mul(Rm[t + piv[a] * cols], kd[a]));
    kd[t] = dd_div(s, Rm[t + piv[t] * cols]);
    kap[piv[t]] = kd[t].hi + kd[t].lo;
  }
}

}  // namespace spock
