// TEST INFRASTRUCTURE ONLY -- parity oracle (see orc.hpp).
// Dense LA kit replacing the reference's Eigen call sites, the Philox stream
// (proj/src/rng.cpp) and the fork-join pool (proj/src/parallel.cpp).
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <limits>
#include <mutex>
#include <thread>

#include "orc.hpp"

namespace orc {

Mat matmul(const Mat& A, const Mat& B) {
  Mat C(A.r, B.c);
  for (int j = 0; j < B.c; ++j)
    for (int k = 0; k < A.c; ++k) {
      const double b = B(k, j);
      if (b == 0.0) continue;
      const double* a = A.col(k);
      double* cc = C.col(j);
      for (int i = 0; i < A.r; ++i) cc[i] += a[i] * b;
    }
  return C;
}

Mat matmul_tn(const Mat& A, const Mat& B) {
  Mat C(A.c, B.c);
  for (int j = 0; j < B.c; ++j)
    for (int i = 0; i < A.c; ++i) C(i, j) = dot(A.col(i), B.col(j), A.r);
  return C;
}

Mat transpose(const Mat& A) {
  Mat T(A.c, A.r);
  for (int j = 0; j < A.c; ++j)
    for (int i = 0; i < A.r; ++i) T(j, i) = A(i, j);
  return T;
}

Mat add(const Mat& A, const Mat& B, double sb) {
  Mat C = A;
  for (size_t k = 0; k < C.a.size(); ++k) C.a[k] += sb * B.a[k];
  return C;
}

Vec matvec(const Mat& A, const double* x) {
  Vec y(A.r, 0.0);
  matvec_acc(A, x, y.data());
  return y;
}

void matvec_acc(const Mat& A, const double* x, double* y) {
  for (int j = 0; j < A.c; ++j) {
    const double xj = x[j];
    const double* a = A.col(j);
    for (int i = 0; i < A.r; ++i) y[i] += a[i] * xj;
  }
}

void matvec_t_acc(const Mat& A, const double* x, double* y) {
  for (int j = 0; j < A.c; ++j) y[j] += dot(A.col(j), x, A.r);
}

double dot(const double* a, const double* b, size_t n) {
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

double sqnorm(const Vec& v) { return dot(v.data(), v.data(), v.size()); }

bool cholesky(const Mat& A, Mat& L) {
  const int n = A.r;
  L = Mat(n, n);
  for (int j = 0; j < n; ++j) {
    double d = A(j, j);
    for (int k = 0; k < j; ++k) d -= L(j, k) * L(j, k);
    if (!(d > 0.0)) return false;
    d = std::sqrt(d);
    L(j, j) = d;
    for (int i = j + 1; i < n; ++i) {
      double s = A(i, j);
      for (int k = 0; k < j; ++k) s -= L(i, k) * L(j, k);
      L(i, j) = s / d;
    }
  }
  return true;
}

void chol_solve(const Mat& L, double* b) {
  const int n = L.r;
  for (int i = 0; i < n; ++i) {
    double s = b[i];
    for (int k = 0; k < i; ++k) s -= L(i, k) * b[k];
    b[i] = s / L(i, i);
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = b[i];
    for (int k = i + 1; k < n; ++k) s -= L(k, i) * b[k];
    b[i] = s / L(i, i);
  }
}

void sym_eig(const Mat& A0, Vec& w, Mat& V) {
  const int n = A0.r;
  Mat A(n, n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) A(i, j) = 0.5 * (A0(i, j) + A0(j, i));
  Mat U = Mat::eye(n);
  const double eps = std::numeric_limits<double>::epsilon();
  for (int sweep = 0; sweep < 100; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = A(p, q);
        if (apq == 0.0) continue;
        const double app = A(p, p), aqq = A(q, q);
        if (std::fabs(apq) <= eps * 1e-3 * std::sqrt(std::fabs(app) * std::fabs(aqq)) &&
            std::fabs(apq) <= 1e-300 + eps * 1e-3 * std::max(std::fabs(app), std::fabs(aqq))) {
          A(p, q) = A(q, p) = 0.0;
          continue;
        }
        rotated = true;
        const double theta = (aqq - app) / (2.0 * apq);
        double t;
        if (std::fabs(theta) > 1e150)
          t = 0.5 / theta;
        else
          t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {
          const double akp = A(k, p), akq = A(k, q);
          A(k, p) = c * akp - s * akq;
          A(k, q) = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          const double apk = A(p, k), aqk = A(q, k);
          A(p, k) = c * apk - s * aqk;
          A(q, k) = s * apk + c * aqk;
        }
        A(p, q) = A(q, p) = 0.0;
        for (int k = 0; k < n; ++k) {
          const double ukp = U(k, p), ukq = U(k, q);
          U(k, p) = c * ukp - s * ukq;
          U(k, q) = s * ukp + c * ukq;
        }
      }
    if (!rotated) break;
  }
  std::vector<int> ord(n);
  for (int i = 0; i < n; ++i) ord[i] = i;
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return A(a, a) < A(b, b); });
  w.assign(n, 0.0);
  V = Mat(n, n);
  for (int k = 0; k < n; ++k) {
    w[k] = A(ord[k], ord[k]);
    int imax = 0;
    for (int i = 1; i < n; ++i)
      if (std::fabs(U(i, ord[k])) > std::fabs(U(imax, ord[k])) * (1.0 + 1e-12)) imax = i;
    const double sg = U(imax, ord[k]) < 0 ? -1.0 : 1.0;
    for (int i = 0; i < n; ++i) V(i, k) = sg * U(i, ord[k]);
  }
}

Vec colpiv_qr_solve(const Mat& A0, const Vec& b, double threshold) {
  const int rows = A0.r, cols = A0.c, size = std::min(rows, cols);
  Mat qr = A0;
  Vec hcoef(size, 0.0), normsU(cols), normsD(cols);
  std::vector<int> transp(size);
  for (int k = 0; k < cols; ++k) normsU[k] = normsD[k] = std::sqrt(dot(qr.col(k), qr.col(k), rows));
  double maxn = 0.0;
  for (double v : normsU) maxn = std::max(maxn, v);
  const double eps = std::numeric_limits<double>::epsilon();
  const double thr_helper = (maxn * eps) * (maxn * eps) / rows;
  const double downdate_thr = std::sqrt(eps);
  int nonzero = size;
  double maxpivot = 0.0;
  for (int k = 0; k < size; ++k) {
    int big = k;
    for (int j = k + 1; j < cols; ++j)
      if (normsU[j] > normsU[big]) big = j;
    const double big_sq = normsU[big] * normsU[big];
    if (nonzero == size && big_sq < thr_helper * double(rows - k)) nonzero = k;
    transp[k] = big;
    if (big != k) {
      std::swap_ranges(qr.col(k), qr.col(k) + rows, qr.col(big));
      std::swap(normsU[k], normsU[big]);
      std::swap(normsD[k], normsD[big]);
    }
    // makeHouseholderInPlace on qr.col(k).tail(rows-k)
    double* x = qr.col(k) + k;
    const int len = rows - k;
    const double tail_sq = len == 1 ? 0.0 : dot(x + 1, x + 1, len - 1);
    const double c0 = x[0];
    double tau, beta;
    if (tail_sq <= std::numeric_limits<double>::min()) {
      tau = 0.0;
      beta = c0;
      for (int i = 1; i < len; ++i) x[i] = 0.0;
    } else {
      beta = std::sqrt(c0 * c0 + tail_sq);
      if (c0 >= 0.0) beta = -beta;
      for (int i = 1; i < len; ++i) x[i] /= (c0 - beta);
      tau = (beta - c0) / beta;
    }
    hcoef[k] = tau;
    x[0] = beta;
    if (std::fabs(beta) > maxpivot) maxpivot = std::fabs(beta);
    // applyHouseholderOnTheLeft to bottomRightCorner(rows-k, cols-k-1)
    for (int j = k + 1; j < cols; ++j) {
      double* y = qr.col(j) + k;
      if (len == 1) {
        y[0] *= (1.0 - tau);
      } else if (tau != 0.0) {
        double tmp = y[0];
        for (int i = 1; i < len; ++i) tmp += x[i] * y[i];
        y[0] -= tau * tmp;
        for (int i = 1; i < len; ++i) y[i] -= tau * x[i] * tmp;
      }
    }
    for (int j = k + 1; j < cols; ++j) {
      if (normsU[j] != 0.0) {
        double temp = std::fabs(qr(k, j)) / normsU[j];
        temp = (1.0 + temp) * (1.0 - temp);
        temp = temp < 0.0 ? 0.0 : temp;
        const double r = normsU[j] / normsD[j];
        const double temp2 = temp * r * r;
        if (temp2 <= downdate_thr) {
          normsD[j] = std::sqrt(dot(qr.col(j) + k + 1, qr.col(j) + k + 1, rows - k - 1));
          normsU[j] = normsD[j];
        } else {
          normsU[j] *= std::sqrt(temp);
        }
      }
    }
  }
  std::vector<int> perm(cols);
  for (int i = 0; i < cols; ++i) perm[i] = i;
  for (int k = 0; k < size; ++k) std::swap(perm[k], perm[transp[k]]);
  const double pthr = maxpivot * threshold;
  int np = 0;
  for (int i = 0; i < nonzero; ++i) np += (std::fabs(qr(i, i)) > pthr) ? 1 : 0;
  Vec dst(cols, 0.0);
  if (np == 0) return dst;
  Vec cvec = b;
  for (int k = 0; k < np; ++k) {  // c = Q' b, reflectors 0..np-1
    const double* x = qr.col(k) + k;
    double* y = cvec.data() + k;
    const int len = rows - k;
    const double tau = hcoef[k];
    if (len == 1) {
      y[0] *= (1.0 - tau);
    } else if (tau != 0.0) {
      double tmp = y[0];
      for (int i = 1; i < len; ++i) tmp += x[i] * y[i];
      y[0] -= tau * tmp;
      for (int i = 1; i < len; ++i) y[i] -= tau * x[i] * tmp;
    }
  }
  for (int i = np - 1; i >= 0; --i) {
    double s = cvec[i];
    for (int k = i + 1; k < np; ++k) s -= qr(i, k) * cvec[k];
    cvec[i] = s / qr(i, i);
  }
  for (int i = 0; i < np; ++i) dst[perm[i]] = cvec[i];
  return dst;
}

Mat kernel_projector(const Mat& M) {
  // one-sided Jacobi on X = M' (d x r): columns become V1 * Sigma
  Mat X = transpose(M);
  const int d = X.r, r = X.c;
  const double eps = std::numeric_limits<double>::epsilon();
  for (int sweep = 0; sweep < 100; ++sweep) {
    bool rot = false;
    for (int p = 0; p < r; ++p)
      for (int q = p + 1; q < r; ++q) {
        const double a = dot(X.col(p), X.col(p), d), bq = dot(X.col(q), X.col(q), d);
        const double g = dot(X.col(p), X.col(q), d);
        if (std::fabs(g) <= eps * std::sqrt(a * bq) || g == 0.0) continue;
        rot = true;
        const double zeta = (bq - a) / (2.0 * g);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
        double* xp = X.col(p);
        double* xq = X.col(q);
        for (int i = 0; i < d; ++i) {
          const double u = xp[i], v = xq[i];
          xp[i] = c * u - s * v;
          xq[i] = s * u + c * v;
        }
      }
    if (!rot) break;
  }
  Vec sv(r);
  double smax = 0.0;
  for (int k = 0; k < r; ++k) {
    sv[k] = std::sqrt(dot(X.col(k), X.col(k), d));
    smax = std::max(smax, sv[k]);
  }
  Mat N = Mat::eye(d);
  const double thr = 1e-12 * smax;
  for (int k = 0; k < r; ++k) {
    if (!(sv[k] > thr)) continue;
    const double* x = X.col(k);
    const double inv2 = 1.0 / (sv[k] * sv[k]);
    for (int j = 0; j < d; ++j)
      for (int i = 0; i < d; ++i) N(i, j) -= x[i] * x[j] * inv2;
  }
  return N;
}

// ---------------- Philox4x32-10, proj/src/rng.cpp:10-103 ----------------
namespace {
constexpr uint32_t kM0 = 0xD2511F53u, kM1 = 0xCD9E8D57u, kW0 = 0x9E3779B9u, kW1 = 0xBB67AE85u;
}
Philox::Philox(uint64_t seed, uint64_t stream) {
  key_[0] = uint32_t(seed);
  key_[1] = uint32_t(seed >> 32);
  ctr_[0] = ctr_[1] = 0;
  ctr_[2] = uint32_t(stream);
  ctr_[3] = uint32_t(stream >> 32);
}
void Philox::refill() {
  uint32_t c0 = ctr_[0], c1 = ctr_[1], c2 = ctr_[2], c3 = ctr_[3], k0 = key_[0], k1 = key_[1];
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = uint64_t(kM0) * c0, p1 = uint64_t(kM1) * c2;
    const uint32_t n0 = uint32_t(p1 >> 32) ^ c1 ^ k0, n1 = uint32_t(p1);
    const uint32_t n2 = uint32_t(p0 >> 32) ^ c3 ^ k1, n3 = uint32_t(p0);
    c0 = n0, c1 = n1, c2 = n2, c3 = n3;
    k0 += kW0;
    k1 += kW1;
  }
  blk_[0] = c0, blk_[1] = c1, blk_[2] = c2, blk_[3] = c3;
  if (++ctr_[0] == 0)
    if (++ctr_[1] == 0)
      if (++ctr_[2] == 0) ++ctr_[3];
  pos_ = 0;
}
uint32_t Philox::next_u32() {
  if (pos_ >= 4) refill();
  return blk_[pos_++];
}
uint64_t Philox::next_u64() {
  const uint64_t lo = next_u32();
  const uint64_t hi = next_u32();
  return (hi << 32) | lo;
}
double Philox::uniform() { return double(next_u64() >> 11) * 0x1.0p-53; }
double Philox::normal() {
  if (have_spare_) {
    have_spare_ = false;
    return spare_;
  }
  double u1 = uniform();
  while (u1 <= 0.0) u1 = uniform();
  const double u2 = uniform();
  const double mag = std::sqrt(-2.0 * std::log(u1));
  const double ang = 2.0 * M_PI * u2;
  spare_ = mag * std::sin(ang);
  have_spare_ = true;
  return mag * std::cos(ang);
}

// ---------------- fork-join pool, proj/src/parallel.cpp:20-136 ----------------
namespace {
struct Pool {
  explicit Pool(int n) : nthreads(n) {
    for (int t = 1; t < n; ++t) workers.emplace_back([this, t] { loop(t); });
  }
  ~Pool() {
    {
      std::unique_lock<std::mutex> lk(mtx);
      stop.store(true);
      epoch.fetch_add(1);
    }
    cv.notify_all();
    for (auto& w : workers) w.join();
  }
  void loop(int tid) {
    uint64_t seen = 0;
    for (;;) {
      uint64_t e = epoch.load(std::memory_order_acquire);
      int spins = 0;
      while (e == seen && !stop.load(std::memory_order_acquire)) {
        if (++spins < 20000) {
          std::this_thread::yield();
        } else {
          std::unique_lock<std::mutex> lk(mtx);
          cv.wait(lk, [&] { return epoch.load() != seen || stop.load(); });
        }
        e = epoch.load(std::memory_order_acquire);
      }
      if (stop.load()) return;
      seen = e;
      chunk(tid);
      pending.fetch_sub(1, std::memory_order_acq_rel);
    }
  }
  void chunk(int tid) {
    const int n = jb_end - jb_begin;
    const int per = (n + nthreads - 1) / nthreads;
    const int lo = jb_begin + tid * per, hi = std::min(jb_end, lo + per);
    for (int i = lo; i < hi; ++i) (*job)(i);
  }
  void run(int begin, int end, const std::function<void(int)>& body, uint64_t flops) {
    if (end <= begin) return;
    const uint64_t count = uint64_t(end - begin);
    const bool worth = count >= 256 || count * std::max<uint64_t>(flops, 1) >= 120000;
    if (nthreads == 1 || count == 1 || !worth) {
      for (int i = begin; i < end; ++i) body(i);
      return;
    }
    job = &body;
    jb_begin = begin;
    jb_end = end;
    pending.store(nthreads - 1, std::memory_order_release);
    {
      std::unique_lock<std::mutex> lk(mtx);
      epoch.fetch_add(1, std::memory_order_release);
    }
    cv.notify_all();
    chunk(0);
    while (pending.load(std::memory_order_acquire) != 0) std::this_thread::yield();
    job = nullptr;
  }
  int nthreads;
  std::vector<std::thread> workers;
  std::mutex mtx;
  std::condition_variable cv;
  std::atomic<uint64_t> epoch{0};
  std::atomic<bool> stop{false};
  const std::function<void(int)>* job = nullptr;
  int jb_begin = 0, jb_end = 0;
  std::atomic<int> pending{0};
};
std::unique_ptr<Pool>& pool_slot() {
  static std::unique_ptr<Pool> p;
  return p;
}
Pool& pool() {
  auto& s = pool_slot();
  if (!s) {
    int n = int(std::thread::hardware_concurrency());
    s = std::make_unique<Pool>(n > 0 ? n : 1);
  }
  return *s;
}
}  // namespace

void set_num_threads(int n) {
  pool_slot().reset();
  pool_slot() = std::make_unique<Pool>(n < 1 ? 1 : n);
}
int num_threads() { return pool().nthreads; }
void parallel_for(int begin, int end, const std::function<void(int)>& body, uint64_t flops) {
  pool().run(begin, end, body, flops);
}

}  // namespace orc
