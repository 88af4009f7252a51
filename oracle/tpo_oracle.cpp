// tpo_oracle.cpp -- TEST INFRASTRUCTURE ONLY (see tpo_oracle.h).
//
// Loop-for-loop fp64 restatement of the reference CPU path.  Every function
// cites the reference file:line it follows (paths relative to
// /root/reference/proj).  Eigen is replaced by std::vector; the Eigen GEMMs
// of proj/src/sphere.cpp:130-131,170 become plain loops (same sums, possibly
// different fp64 summation order), and Eigen's complex COD pseudo-inverse
// (proj/src/gtp.cpp:136-139) becomes a complex Householder QR solve (the
// blocks are full column rank, so the pseudo-inverse is unique).
#include "tpo_oracle.h"

#include <algorithm>
#include <array>
#include <cmath>
#include <complex>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

using cd = std::complex<double>;
thread_local std::string g_err;

struct Invalid : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

// -------------------------------------------------------------------------
// wigner.cpp restatement
// -------------------------------------------------------------------------
constexpr double kStructuralZero = 1e-12;  // proj/src/wigner.cpp:17
constexpr double kResidueLimit = 1e-10;    // proj/src/wigner.cpp:19

// proj/src/wigner.cpp:23-31
long double log_factorial(int n) {
  static const std::vector<long double> table = [] {
    std::vector<long double> t(512);
    t[0] = 0.0L;
    for (size_t i = 1; i < t.size(); ++i) t[i] = t[i - 1] + std::log(static_cast<long double>(i));
    return t;
  }();
  return table.at(n);
}

bool triangle(int l1, int l2, int l3) { return l3 >= std::abs(l1 - l2) && l3 <= l1 + l2; }

// Racah closed form, proj/src/wigner.cpp:39-62
double cg_coefficient(int l1, int m1, int l2, int m2, int l3, int m3) {
  if (m1 + m2 != m3 || !triangle(l1, l2, l3)) return 0.0;
  if (std::abs(m1) > l1 || std::abs(m2) > l2 || std::abs(m3) > l3) return 0.0;
  const long double log_pref =
      0.5L * (std::log(2.0L * l3 + 1.0L) + log_factorial(l1 + l2 - l3) +
              log_factorial(l1 - l2 + l3) + log_factorial(-l1 + l2 + l3) -
              log_factorial(l1 + l2 + l3 + 1) + log_factorial(l3 + m3) + log_factorial(l3 - m3) +
              log_factorial(l1 + m1) + log_factorial(l1 - m1) + log_factorial(l2 + m2) +
              log_factorial(l2 - m2));
  const int z_lo = std::max({0, -(l3 - l2 + m1), -(l3 - l1 - m2)});
  const int z_hi = std::min({l1 + l2 - l3, l1 - m1, l2 + m2});
  long double sum = 0.0L;
  for (int z = z_lo; z <= z_hi; ++z) {
    const long double log_den = log_factorial(z) + log_factorial(l1 + l2 - l3 - z) +
                                log_factorial(l1 - m1 - z) + log_factorial(l2 + m2 - z) +
                                log_factorial(l3 - l2 + m1 + z) + log_factorial(l3 - l1 - m2 + z);
    const long double term = std::exp(log_pref - log_den);
    sum += (z % 2 == 0) ? term : -term;
  }
  return static_cast<double>(sum);
}

// complex d x d matrix, row-major
struct CMat {
  int r = 0, c = 0;
  std::vector<cd> a;
  CMat() = default;
  CMat(int r_, int c_) : r(r_), c(c_), a(static_cast<size_t>(r_) * c_) {}
  cd& operator()(int i, int j) { return a[static_cast<size_t>(i) * c + j]; }
  cd operator()(int i, int j) const { return a[static_cast<size_t>(i) * c + j]; }
};

// proj/src/wigner.cpp:249-263
CMat real_basis_change(int l) {
  const int d = 2 * l + 1;
  CMat U(d, d);
  const double inv_sqrt2 = 1.0 / std::sqrt(2.0);
  const cd i_unit(0.0, 1.0);
  U(l, l) = 1.0;
  for (int m = 1; m <= l; ++m) {
    const double sign = (m % 2 == 0) ? 1.0 : -1.0;
    U(l + m, l + m) = sign * inv_sqrt2;
    U(l + m, l - m) = inv_sqrt2;
    U(l - m, l + m) = -i_unit * sign * inv_sqrt2;
    U(l - m, l - m) = i_unit * inv_sqrt2;
  }
  return U;
}

struct CGEntry {
  int m1, m2, m3;
  double value;
};
struct CGTable {
  int l1 = 0, l2 = 0, l3 = 0;
  std::vector<CGEntry> entries;
};

// proj/src/wigner.cpp:234-247
std::vector<double> cg_complex(int l1, int l2, int l3) {
  if (l1 < 0 || l2 < 0 || l3 < 0) throw Invalid("cg_complex: negative degree");
  const int d1 = 2 * l1 + 1, d2 = 2 * l2 + 1, d3 = 2 * l3 + 1;
  std::vector<double> out(static_cast<size_t>(d1) * d2 * d3, 0.0);
  if (!triangle(l1, l2, l3)) return out;
  for (int m1 = -l1; m1 <= l1; ++m1)
    for (int m2 = -l2; m2 <= l2; ++m2) {
      const int m3 = m1 + m2;
      if (std::abs(m3) > l3) continue;
      out[((m1 + l1) * d2 + (m2 + l2)) * d3 + (m3 + l3)] = cg_coefficient(l1, m1, l2, m2, l3, m3);
    }
  return out;
}

// proj/src/wigner.cpp:90-112
CGTable collect_real_table(int l1, int l2, int l3, const std::vector<cd>& dense, const char* what) {
  const int d2 = 2 * l2 + 1, d3 = 2 * l3 + 1;
  const bool odd = (l1 + l2 + l3) % 2 != 0;
  double residue = 0.0;
  CGTable out{l1, l2, l3, {}};
  for (int n1 = -l1; n1 <= l1; ++n1)
    for (int n2 = -l2; n2 <= l2; ++n2)
      for (int n3 = -l3; n3 <= l3; ++n3) {
        const cd v = dense[((n1 + l1) * d2 + (n2 + l2)) * d3 + (n3 + l3)];
        const double keep = odd ? v.imag() : v.real();
        const double drop = odd ? v.real() : v.imag();
        residue = std::max(residue, std::abs(drop));
        if (std::abs(keep) > kStructuralZero) out.entries.push_back({n1, n2, n3, keep});
      }
  if (residue > kResidueLimit)
    throw std::runtime_error(std::string(what) + ": basis change left a mixed table");
  return out;
}

// Scatter over the <=8 real slots n_i = +-|m_i|, proj/src/wigner.cpp:124-149
template <class F>
void scatter_real_slots(int l1, int l2, int l3, int m1, int m2, int m3, const CMat& U1,
                        const CMat& U2, const CMat& U3, F&& emit) {
  for (int n1 : {-std::abs(m1), std::abs(m1)}) {
    const cd u1 = U1(n1 + l1, m1 + l1);
    if (u1 != 0.0) {
      for (int n2 : {-std::abs(m2), std::abs(m2)}) {
        const cd u12 = u1 * U2(n2 + l2, m2 + l2);
        if (u12 != 0.0) {
          for (int n3 : {-std::abs(m3), std::abs(m3)}) {
            const cd u3 = U3(n3 + l3, m3 + l3);
            if (u3 != 0.0) emit(n1, n2, n3, u12, u3);
            if (n3 == 0) break;  // +-0 is one slot
          }
        }
        if (n2 == 0) break;
      }
    }
    if (n1 == 0) break;
  }
}

// proj/src/wigner.cpp:114-151
CGTable build_cg_real(int l1, int l2, int l3) {
  CGTable out{l1, l2, l3, {}};
  if (!triangle(l1, l2, l3)) return out;
  const std::vector<double> cg = cg_complex(l1, l2, l3);
  const CMat U1 = real_basis_change(l1), U2 = real_basis_change(l2), U3 = real_basis_change(l3);
  const int d1 = 2 * l1 + 1, d2 = 2 * l2 + 1, d3 = 2 * l3 + 1;
  std::vector<cd> dense(static_cast<size_t>(d1) * d2 * d3);
  for (int m1 = -l1; m1 <= l1; ++m1)
    for (int m2 = -l2; m2 <= l2; ++m2) {
      const int m3 = m1 + m2;
      if (std::abs(m3) > l3) continue;
      const double c = cg[((m1 + l1) * d2 + (m2 + l2)) * d3 + (m3 + l3)];
      if (c == 0.0) continue;
      scatter_real_slots(l1, l2, l3, m1, m2, m3, U1, U2, U3,
                         [&](int n1, int n2, int n3, cd u12, cd u3) {
                           dense[((n1 + l1) * d2 + (n2 + l2)) * d3 + (n3 + l3)] +=
                               u12 * std::conj(u3) * c;
                         });
    }
  return collect_real_table(l1, l2, l3, dense, "cg_real");
}

// proj/src/wigner.cpp:153-198
CGTable build_gaunt_real(int l1, int l2, int l3) {
  CGTable out{l1, l2, l3, {}};
  if (!triangle(l1, l2, l3) || (l1 + l2 + l3) % 2 != 0) return out;
  const int d1 = 2 * l1 + 1, d2 = 2 * l2 + 1, d3 = 2 * l3 + 1;
  const double pref = std::sqrt((2.0 * l1 + 1) * (2.0 * l2 + 1) / (4.0 * M_PI * (2.0 * l3 + 1)));
  const double c000 = cg_coefficient(l1, 0, l2, 0, l3, 0);
  const CMat U1 = real_basis_change(l1), U2 = real_basis_change(l2), U3 = real_basis_change(l3);
  std::vector<cd> dense(static_cast<size_t>(d1) * d2 * d3);
  for (int m1 = -l1; m1 <= l1; ++m1)
    for (int m2 = -l2; m2 <= l2; ++m2) {
      const int m3 = -(m1 + m2);
      if (std::abs(m3) > l3) continue;
      const double sign = (m3 % 2 == 0) ? 1.0 : -1.0;
      const double g = sign * pref * c000 * cg_coefficient(l1, m1, l2, m2, l3, -m3);
      if (g == 0.0) continue;
      scatter_real_slots(l1, l2, l3, m1, m2, m3, U1, U2, U3,
                         [&](int n1, int n2, int n3, cd u12, cd u3) {
                           dense[((n1 + l1) * d2 + (n2 + l2)) * d3 + (n3 + l3)] += u12 * u3 * g;
                         });
    }
  return collect_real_table(l1, l2, l3, dense, "gaunt_real");
}

// memo caches, proj/src/wigner.cpp:64-81,265-273
using Key3 = std::array<int, 3>;
std::mutex g_cache_mu;
const CGTable& cache_lookup(std::map<Key3, std::unique_ptr<const CGTable>>& cache, int l1, int l2,
                            int l3, CGTable (*build)(int, int, int)) {
  const Key3 key{l1, l2, l3};
  {
    std::lock_guard<std::mutex> lock(g_cache_mu);
    auto it = cache.find(key);
    if (it != cache.end()) return *it->second;
  }
  auto built = std::make_unique<const CGTable>(build(l1, l2, l3));
  std::lock_guard<std::mutex> lock(g_cache_mu);
  auto res = cache.try_emplace(key, std::move(built));
  return *res.first->second;
}
const CGTable& cg_real(int l1, int l2, int l3) {
  static std::map<Key3, std::unique_ptr<const CGTable>> cache;
  return cache_lookup(cache, l1, l2, l3, build_cg_real);
}
const CGTable& gaunt_real(int l1, int l2, int l3) {
  static std::map<Key3, std::unique_ptr<const CGTable>> cache;
  return cache_lookup(cache, l1, l2, l3, build_gaunt_real);
}

// proj/src/wigner.cpp:281-286
void densify_into(const CGTable& t, std::vector<double>& dense) {
  const int d2 = 2 * t.l2 + 1, d3 = 2 * t.l3 + 1;
  dense.assign(static_cast<size_t>(2 * t.l1 + 1) * d2 * d3, 0.0);
  for (const CGEntry& e : t.entries)
    dense[((e.m1 + t.l1) * d2 + (e.m2 + t.l2)) * d3 + (e.m3 + t.l3)] = e.value;
}

// real d x d matrix
struct Mat {
  int r = 0, c = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(int r_, int c_) : r(r_), c(c_), a(static_cast<size_t>(r_) * c_, 0.0) {}
  double& operator()(int i, int j) { return a[static_cast<size_t>(i) * c + j]; }
  double operator()(int i, int j) const { return a[static_cast<size_t>(i) * c + j]; }
};

// proj/src/wigner.cpp:288-312
Mat wigner_d(int l, const double* R) {
  if (l < 0) throw Invalid("wigner_d: negative degree");
  if (l == 0) {
    Mat one(1, 1);
    one(0, 0) = 1.0;
    return one;
  }
  // (y, z, x) component order of the l=1 harmonics
  static const int ax[3] = {1, 2, 0};
  Mat D1(3, 3);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) D1(i, j) = R[ax[i] * 3 + ax[j]];
  if (l == 1) return D1;
  const Mat prev = wigner_d(l - 1, R);
  const CGTable& q = cg_real(1, l - 1, l);
  Mat D(2 * l + 1, 2 * l + 1);
  for (const CGEntry& a : q.entries)
    for (const CGEntry& b : q.entries)
      D(a.m3 + l, b.m3 + l) +=
          a.value * b.value * D1(a.m1 + 1, b.m1 + 1) * prev(a.m2 + l - 1, b.m2 + l - 1);
  return D;
}

// -------------------------------------------------------------------------
// irreps helpers (proj/src/irreps.cpp:9-93): single-copy degree lists
// -------------------------------------------------------------------------
struct Tower {
  std::vector<int> ls;
  std::vector<int> off;
  int dim = 0;
  int lmax = 0;
  Tower(const int* l, int n) {
    if (n < 0 || (n > 0 && !l)) throw Invalid("irreps: bad degree list");
    for (int i = 0; i < n; ++i) {
      if (l[i] < 0) throw Invalid("irreps: degree must be >= 0");  // irreps.cpp:13
      ls.push_back(l[i]);
      off.push_back(dim);
      dim += 2 * l[i] + 1;
      lmax = std::max(lmax, l[i]);
    }
  }
};

inline void count_muls(uint64_t* ops, uint64_t n) {
  if (ops) *ops += n;
}

// -------------------------------------------------------------------------
// sphere.cpp restatement
// -------------------------------------------------------------------------
inline int lidx(int l, int m_abs) { return l * (l + 1) / 2 + m_abs; }  // sphere.hpp:21

// proj/src/sphere.cpp:22-55
Mat legendre_lambda_table(int l_max, const std::vector<double>& cos_theta) {
  const int rows = (l_max + 1) * (l_max + 2) / 2;
  const int n = static_cast<int>(cos_theta.size());
  Mat lam(rows, n);
  const double sqrt2 = std::sqrt(2.0);
  std::vector<double> pbar(rows);
  for (int j = 0; j < n; ++j) {
    const double x = cos_theta[j];
    const double s = std::sqrt(std::max(0.0, 1.0 - x * x));
    pbar[lidx(0, 0)] = std::sqrt(1.0 / (4.0 * M_PI));
    for (int m = 1; m <= l_max; ++m)
      pbar[lidx(m, m)] = pbar[lidx(m - 1, m - 1)] * s * std::sqrt((2.0 * m + 1) / (2.0 * m));
    for (int m = 0; m < l_max; ++m)
      pbar[lidx(m + 1, m)] = x * std::sqrt(2.0 * m + 3) * pbar[lidx(m, m)];
    for (int m = 0; m <= l_max; ++m)
      for (int l = m + 2; l <= l_max; ++l) {
        const double a = std::sqrt((4.0 * l * l - 1) / (static_cast<double>(l) * l - m * m));
        const double a_prev =
            std::sqrt((4.0 * (l - 1.0) * (l - 1) - 1) / (static_cast<double>(l - 1) * (l - 1) - m * m));
        pbar[lidx(l, m)] = a * (x * pbar[lidx(l - 1, m)] - pbar[lidx(l - 2, m)] / a_prev);
      }
    for (int l = 0; l <= l_max; ++l)
      for (int m = 0; m <= l; ++m) lam(lidx(l, m), j) = (m == 0 ? 1.0 : sqrt2) * pbar[lidx(l, m)];
  }
  return lam;
}

// proj/src/sphere.cpp:57-87
void gauss_legendre(int n, std::vector<double>& nodes, std::vector<double>& weights) {
  if (n < 1) throw Invalid("gauss_legendre: need at least one node");
  nodes.assign(n, 0.0);
  weights.assign(n, 0.0);
  for (int i = 0; i < (n + 1) / 2; ++i) {
    double x = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    double dp = 0.0;
    for (int iter = 0; iter < 64; ++iter) {
      double p0 = 1.0, p1 = x;
      for (int k = 2; k <= n; ++k) {
        const double p2 = ((2.0 * k - 1) * x * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      dp = n * (x * p1 - p0) / (x * x - 1.0);
      const double dx = p1 / dp;
      x -= dx;
      if (std::abs(dx) < 1e-15) break;
    }
    const double w = 2.0 / ((1.0 - x * x) * dp * dp);
    nodes[n - 1 - i] = x;
    nodes[i] = -x;
    weights[n - 1 - i] = w;
    weights[i] = w;
  }
  if (n % 2 == 1) nodes[n / 2] = 0.0;
}

struct S2Grid {
  int L_max = 0;
  std::vector<double> nodes, weights;
  int n_phi = 0;
  Mat lambda;  // ((L+1)(L+2)/2) x n_theta
  Mat cs;      // (2L+1) x n_phi
  int n_theta() const { return static_cast<int>(nodes.size()); }
};
using GridPtr = std::shared_ptr<const S2Grid>;

// proj/src/sphere.cpp:89-103
GridPtr make_grid(int L) {
  if (L < 0) throw Invalid("make_grid: L must be >= 0");
  auto g = std::make_shared<S2Grid>();
  g->L_max = L;
  gauss_legendre(L + 1, g->nodes, g->weights);
  g->n_phi = 2 * L + 1;
  g->lambda = legendre_lambda_table(L, g->nodes);
  g->cs = Mat(2 * L + 1, g->n_phi);
  for (int m = -L; m <= L; ++m)
    for (int k = 0; k < g->n_phi; ++k) {
      const double phi = 2.0 * M_PI * k / g->n_phi;
      g->cs(m + L, k) = m < 0 ? std::sin(-m * phi) : (m == 0 ? 1.0 : std::cos(m * phi));
    }
  return g;
}

// proj/src/gtp.cpp:25-32 (product grids are cached per band)
GridPtr product_grid(int L_product) {
  static std::map<int, GridPtr> cache;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  auto res = cache.try_emplace(L_product);
  if (res.second) res.first->second = make_grid(L_product);
  return res.first->second;
}

// proj/src/sphere.cpp:105-134 ; F is n_theta x n_phi
Mat to_sphere(const Tower& x, const double* coeffs, const S2Grid& grid, uint64_t* ops) {
  const int lmax = x.lmax;
  if (lmax > grid.L_max) throw Invalid("to_sphere: grid band limit below input degree");
  const int nt = grid.n_theta();
  const int n_m = 2 * lmax + 1;
  Mat g_m(n_m, nt);
  for (size_t e = 0; e < x.ls.size(); ++e) {
    const int l = x.ls[e];
    const double* c = coeffs + x.off[e];
    for (int m = -l; m <= l; ++m) {
      for (int j = 0; j < nt; ++j) g_m(m + lmax, j) += c[m + l] * grid.lambda(lidx(l, std::abs(m)), j);
      count_muls(ops, nt);
    }
  }
  Mat F(nt, grid.n_phi);
  const int row0 = grid.L_max - lmax;
  for (int j = 0; j < nt; ++j)
    for (int k = 0; k < grid.n_phi; ++k) {
      double acc = 0.0;
      for (int mi = 0; mi < n_m; ++mi) acc += g_m(mi, j) * grid.cs(row0 + mi, k);
      F(j, k) = acc;
    }
  count_muls(ops, static_cast<uint64_t>(n_m) * nt * grid.n_phi);
  return F;
}

// proj/src/sphere.cpp:145-151
Mat pointwise_mul(const Mat& a, const Mat& b, uint64_t* ops) {
  if (a.r != b.r || a.c != b.c) throw Invalid("pointwise_mul: signals live on different grids");
  Mat out(a.r, a.c);
  for (size_t i = 0; i < a.a.size(); ++i) out.a[i] = a.a[i] * b.a[i];
  count_muls(ops, a.a.size());
  return out;
}

// proj/src/sphere.cpp:155-195
std::vector<double> from_sphere_select(const S2Grid& grid, const Mat& F,
                                       const std::vector<int>& degrees, uint64_t* ops) {
  int lmax = 0;
  for (int l : degrees) lmax = std::max(lmax, l);
  if (lmax > grid.L_max) throw Invalid("from_sphere: grid band limit too small for requested degree");
  const int nt = grid.n_theta();
  const int n_m = 2 * lmax + 1;
  const double phi_scale = 2.0 * M_PI / grid.n_phi;
  const int row0 = grid.L_max - lmax;
  Mat h(n_m, nt);
  for (int mi = 0; mi < n_m; ++mi)
    for (int j = 0; j < nt; ++j) {
      double acc = 0.0;
      for (int k = 0; k < grid.n_phi; ++k) acc += grid.cs(row0 + mi, k) * F(j, k);
      h(mi, j) = acc;
    }
  count_muls(ops, static_cast<uint64_t>(n_m) * grid.n_phi * nt);
  for (double& v : h.a) v *= phi_scale;
  count_muls(ops, static_cast<uint64_t>(n_m) * nt);
  for (int mi = 0; mi < n_m; ++mi)
    for (int j = 0; j < nt; ++j) h(mi, j) *= grid.weights[j];
  count_muls(ops, static_cast<uint64_t>(n_m) * nt);
  std::vector<double> out;
  for (int l : degrees) {
    for (int m = -l; m <= l; ++m) {
      double acc = 0.0;
      for (int j = 0; j < nt; ++j) acc += h(m + lmax, j) * grid.lambda(lidx(l, std::abs(m)), j);
      out.push_back(acc);
      count_muls(ops, nt);
    }
  }
  return out;
}

// -------------------------------------------------------------------------
// cgtp.cpp restatement
// -------------------------------------------------------------------------
struct Path {
  int l1, l2, l3;
  bool valid() const { return l1 >= 0 && l2 >= 0 && l3 >= std::abs(l1 - l2) && l3 <= l1 + l2; }
};

// proj/src/cgtp.cpp:91-98
std::vector<Path> valid_paths(int L1, int L2, int L3) {
  std::vector<Path> p;
  for (int l1 = 0; l1 <= L1; ++l1)
    for (int l2 = 0; l2 <= L2; ++l2)
      for (int l3 = std::abs(l1 - l2); l3 <= std::min(L3, l1 + l2); ++l3) p.push_back({l1, l2, l3});
  return p;
}

// proj/src/cgtp.cpp:25-32
int pass_m2(int pass, int m1, int m3) {
  switch (pass) {
    case 0: return m1 + m3;
    case 1: return m1 - m3;
    case 2: return -m1 + m3;
    default: return -m1 - m3;
  }
}

struct PassTables {
  std::array<Mat, 4> t;  // (2l3+1) x (2l1+1)
};

// proj/src/cgtp.cpp:34-69
const PassTables& pass_tables(int l1, int l2, int l3) {
  static std::map<Key3, std::unique_ptr<const PassTables>> cache;
  static std::mutex mu;
  const Key3 key{l1, l2, l3};
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return *it->second;
  }
  const int d1 = 2 * l1 + 1, d2 = 2 * l2 + 1, d3 = 2 * l3 + 1;
  std::vector<double> dense;
  densify_into(cg_real(l1, l2, l3), dense);
  auto at = [&](int m1, int m2, int m3) -> double& {
    return dense[((m1 + l1) * d2 + (m2 + l2)) * d3 + (m3 + l3)];
  };
  auto tables = std::make_unique<PassTables>();
  for (int p = 0; p < 4; ++p) {
    tables->t[p] = Mat(d3, d1);
    for (int m3 = -l3; m3 <= l3; ++m3)
      for (int m1 = -l1; m1 <= l1; ++m1) {
        const int m2 = pass_m2(p, m1, m3);
        if (std::abs(m2) > l2) continue;
        tables->t[p](m3 + l3, m1 + l1) = at(m1, m2, m3);
        at(m1, m2, m3) = 0.0;
      }
  }
  for (double v : dense)
    if (v != 0.0) throw std::logic_error("cgtp: sparse passes failed to cover the table");
  std::lock_guard<std::mutex> lock(mu);
  auto res = cache.try_emplace(key, std::unique_ptr<const PassTables>(tables.release()));
  return *res.first->second;
}

// proj/src/cgtp.cpp:71-76
void check_slices(const Path& p, int nx, int ny, int nout) {
  if (nx != 2 * p.l1 + 1 || ny != 2 * p.l2 + 1 || nout != 2 * p.l3 + 1)
    throw Invalid("cgtp: slice sizes do not match the path degrees");
}

// proj/src/cgtp.cpp:100-118
void cgtp_path_naive(const Path& p, const double* x, const double* y, double* out, uint64_t* ops) {
  const int d3 = 2 * p.l3 + 1;
  std::fill(out, out + d3, 0.0);
  if (!p.valid()) return;
  const int d1 = 2 * p.l1 + 1, d2 = 2 * p.l2 + 1;
  thread_local std::vector<double> scratch;
  densify_into(cg_real(p.l1, p.l2, p.l3), scratch);
  for (int i1 = 0; i1 < d1; ++i1)
    for (int i2 = 0; i2 < d2; ++i2) {
      const double xy = x[i1] * y[i2];
      const double* row = scratch.data() + (static_cast<size_t>(i1) * d2 + i2) * d3;
      for (int i3 = 0; i3 < d3; ++i3) out[i3] += row[i3] * xy;
    }
  count_muls(ops, 2ull * d1 * d2 * d3);
}

// proj/src/cgtp.cpp:120-143
void cgtp_path_sparse(const Path& p, const double* x, const double* y, double* out, uint64_t* ops) {
  const int d3 = 2 * p.l3 + 1;
  std::fill(out, out + d3, 0.0);
  if (!p.valid()) return;
  const PassTables& tabs = pass_tables(p.l1, p.l2, p.l3);
  uint64_t executed = 0;
  for (int pass = 0; pass < 4; ++pass) {
    const Mat& t = tabs.t[pass];
    for (int m3 = -p.l3; m3 <= p.l3; ++m3) {
      double acc = 0.0;
      for (int m1 = -p.l1; m1 <= p.l1; ++m1) {
        const int m2 = pass_m2(pass, m1, m3);
        if (std::abs(m2) > p.l2) continue;
        acc += t(m3 + p.l3, m1 + p.l1) * x[m1 + p.l1] * y[m2 + p.l2];
        executed += 2;
      }
      out[m3 + p.l3] += acc;
    }
  }
  count_muls(ops, executed);
}

// proj/src/cgtp.cpp:145-177 ; returns output dim
int cgtp_mimo(int impl, const Tower& xt, const double* x, const Tower& yt, const double* y,
              double* out, uint64_t* ops) {
  struct Item {
    Path p;
    int i, j;
  };
  std::vector<Item> items;
  int dim = 0;
  for (size_t i = 0; i < xt.ls.size(); ++i)
    for (size_t j = 0; j < yt.ls.size(); ++j) {
      const int l1 = xt.ls[i], l2 = yt.ls[j];
      for (int l3 = std::abs(l1 - l2); l3 <= l1 + l2; ++l3) {
        items.push_back({{l1, l2, l3}, static_cast<int>(i), static_cast<int>(j)});
        dim += 2 * l3 + 1;
      }
    }
  if (!out) return dim;
  int off = 0;
  for (const Item& it : items) {
    const double* xs = x + xt.off[it.i];
    const double* ys = y + yt.off[it.j];
    if (impl == 0)
      cgtp_path_naive(it.p, xs, ys, out + off, ops);
    else
      cgtp_path_sparse(it.p, xs, ys, out + off, ops);
    off += 2 * it.p.l3 + 1;
  }
  return dim;
}

// -------------------------------------------------------------------------
// gtp.cpp restatement
// -------------------------------------------------------------------------
// proj/src/gtp.cpp:228-260
std::vector<double> gtp_grid_select(const Tower& xt, const double* x, const Tower& yt,
                                    const double* y, const std::vector<int>& degrees,
                                    uint64_t* ops) {
  const int band = xt.lmax + yt.lmax;
  const GridPtr grid = product_grid(band);
  const Mat fx = to_sphere(xt, x, *grid, ops);
  const Mat fy = to_sphere(yt, y, *grid, ops);
  const Mat fz = pointwise_mul(fx, fy, ops);
  std::vector<int> inside;
  for (int l : degrees)
    if (l <= band) inside.push_back(l);
  const std::vector<double> low = from_sphere_select(*grid, fz, inside, ops);
  std::vector<double> out;
  size_t off_low = 0;
  for (int l : degrees) {
    for (int m = -l; m <= l; ++m) out.push_back(l <= band ? low[off_low + m + l] : 0.0);
    if (l <= band) off_low += 2 * l + 1;
  }
  return out;
}

struct ModeEntry {
  int u, v;
  cd w;
};
struct FourierTables {
  int L = 0;
  std::vector<std::vector<ModeEntry>> enc;  // l <= L
  std::vector<std::vector<ModeEntry>> dec;  // l <= 2L
};

// Least-squares pseudo-inverse of a full-column-rank complex R x C matrix
// via Householder QR: pinv = R^{-1} Q^H.  Stands in for Eigen's COD
// pseudoInverse (proj/src/gtp.cpp:233-236); identical for full column rank.
CMat pinv_full_column_rank(const CMat& E) {
  const int R = E.r, C = E.c;
  CMat A = E;
  std::vector<std::vector<cd>> vs;
  std::vector<double> betas;
  for (int k = 0; k < C; ++k) {
    double norm2 = 0.0;
    for (int i = k; i < R; ++i) norm2 += std::norm(A(i, k));
    const double norm = std::sqrt(norm2);
    if (norm == 0.0) throw std::runtime_error("fourier_tables: encode block is rank deficient");
    const cd akk = A(k, k);
    const cd phase = std::abs(akk) == 0.0 ? cd(1.0, 0.0) : akk / std::abs(akk);
    const cd alpha = -phase * norm;
    std::vector<cd> v(R, 0.0);
    for (int i = k; i < R; ++i) v[i] = A(i, k);
    v[k] -= alpha;
    double vn2 = 0.0;
    for (int i = k; i < R; ++i) vn2 += std::norm(v[i]);
    const double beta = vn2 == 0.0 ? 0.0 : 2.0 / vn2;
    for (int j = k; j < C; ++j) {
      cd s = 0.0;
      for (int i = k; i < R; ++i) s += std::conj(v[i]) * A(i, j);
      s *= beta;
      for (int i = k; i < R; ++i) A(i, j) -= v[i] * s;
    }
    vs.push_back(std::move(v));
    betas.push_back(beta);
  }
  for (int k = 0; k < C; ++k)
    if (std::abs(A(k, k)) < 1e-12 * std::abs(A(0, 0)))
      throw std::runtime_error("fourier_tables: encode block is rank deficient");
  // Q^H e_r for each r -> columns of Q^H (first C rows needed)
  CMat out(C, R);
  for (int r = 0; r < R; ++r) {
    std::vector<cd> b(R, 0.0);
    b[r] = 1.0;
    for (int k = 0; k < C; ++k) {
      cd s = 0.0;
      for (int i = k; i < R; ++i) s += std::conj(vs[k][i]) * b[i];
      s *= betas[k];
      for (int i = k; i < R; ++i) b[i] -= vs[k][i] * s;
    }
    for (int i = C - 1; i >= 0; --i) {  // back-substitute R x = (Q^H b)[0:C]
      cd s = b[i];
      for (int j = i + 1; j < C; ++j) s -= A(i, j) * out(j, r);
      out(i, r) = s / A(i, i);
    }
  }
  return out;
}

// proj/src/gtp.cpp:147-151
double extended_sh(int l, int m, double phi, const Mat& lambda_cols, int j) {
  const double lam = lambda_cols(lidx(l, std::abs(m)), j);
  const double ang = m < 0 ? std::sin(-m * phi) : (m == 0 ? 1.0 : std::cos(m * phi));
  return lam * ang;
}

// proj/src/gtp.cpp:153-276
FourierTables build_fourier_tables(int L) {
  const int L2 = 2 * L;
  const int n = 4 * L + 2;
  FourierTables tables;
  tables.L = L;
  tables.enc.resize(static_cast<size_t>(L + 1) * (L + 1));
  tables.dec.resize(static_cast<size_t>(L2 + 1) * (L2 + 1));
  std::vector<double> cosines(n), phis(n), thetas(n);
  for (int j = 0; j < n; ++j) {
    const double theta = 2.0 * M_PI * j / n;
    thetas[j] = theta;
    phis[j] = theta;
    cosines[j] = std::cos(theta <= M_PI ? theta : 2.0 * M_PI - theta);
  }
  const Mat lambda_cols = legendre_lambda_table(L2, cosines);
  std::vector<std::vector<ModeEntry>> enc_all(static_cast<size_t>(L2 + 1) * (L2 + 1));
  CMat samples(n, n), by_v(n, n);
  const cd mi(0.0, -1.0);
  for (int l = 0; l <= L2; ++l)
    for (int m = -l; m <= l; ++m) {
      for (int j = 0; j < n; ++j) {
        const bool flip = thetas[j] > M_PI;
        for (int k = 0; k < n; ++k) {
          const double phi = flip ? phis[k] + M_PI : phis[k];
          samples(j, k) = extended_sh(l, m, phi, lambda_cols, j);
        }
      }
      for (int j = 0; j < n; ++j)
        for (int v = -n / 2; v < n - n / 2; ++v) {
          cd acc = 0.0;
          for (int k = 0; k < n; ++k) acc += samples(j, k) * std::exp(mi * (v * phis[k]));
          by_v(j, v + n / 2) = acc / static_cast<double>(n);
        }
      std::vector<ModeEntry>& slot = enc_all[static_cast<size_t>(l) * l + (m + l)];
      for (int v = -n / 2; v < n - n / 2; ++v)
        for (int u = -n / 2; u < n - n / 2; ++u) {
          cd acc = 0.0;
          for (int j = 0; j < n; ++j) acc += by_v(j, v + n / 2) * std::exp(mi * (u * thetas[j]));
          acc /= static_cast<double>(n);
          if (std::abs(acc) < 1e-13) continue;
          if (std::abs(v) != std::abs(m) || std::abs(u) > l)
            throw std::runtime_error("fourier_tables: spectrum outside the expected band");
          slot.push_back({u, v, acc});
        }
    }
  for (int l = 0; l <= L; ++l)
    for (int m = -l; m <= l; ++m)
      tables.enc[static_cast<size_t>(l) * l + (m + l)] = enc_all[static_cast<size_t>(l) * l + (m + l)];

  for (int m_abs = 0; m_abs <= L2; ++m_abs) {
    std::vector<int> cols;
    for (int l = m_abs; l <= L2; ++l) {
      cols.push_back(l * l + (m_abs + l));
      if (m_abs > 0) cols.push_back(l * l + (-m_abs + l));
    }
    std::vector<std::pair<int, int>> rows;
    for (int u = -L2; u <= L2; ++u) {
      rows.emplace_back(u, m_abs);
      if (m_abs > 0) rows.emplace_back(u, -m_abs);
    }
    CMat E(static_cast<int>(rows.size()), static_cast<int>(cols.size()));
    for (size_t c = 0; c < cols.size(); ++c)
      for (const ModeEntry& e : enc_all[cols[c]])
        for (size_t r = 0; r < rows.size(); ++r)
          if (rows[r].first == e.u && rows[r].second == e.v) E(static_cast<int>(r), static_cast<int>(c)) = e.w;
    const CMat pinv = pinv_full_column_rank(E);
    for (size_t c = 0; c < cols.size(); ++c) {
      std::vector<ModeEntry>& slot = tables.dec[cols[c]];
      for (size_t r = 0; r < rows.size(); ++r)
        if (std::abs(pinv(static_cast<int>(c), static_cast<int>(r))) > 1e-13)
          slot.push_back({rows[r].first, rows[r].second, pinv(static_cast<int>(c), static_cast<int>(r))});
    }
  }

  // self-check decode(encode(x)) over the full decode band, gtp.cpp:245-274
  std::mt19937_64 rng(12345);
  std::normal_distribution<double> gauss;
  const int band_dim = (L2 + 1) * (L2 + 1);
  std::vector<double> coeffs(band_dim);
  for (double& c : coeffs) c = gauss(rng);
  const int w = 2 * L2 + 1;
  std::vector<cd> spec(static_cast<size_t>(w) * w);
  for (int l = 0, off = 0; l <= L2; off += 2 * l + 1, ++l)
    for (int m = -l; m <= l; ++m)
      for (const ModeEntry& e : enc_all[static_cast<size_t>(l) * l + (m + l)])
        spec[(e.u + L2) * w + (e.v + L2)] += coeffs[off + m + l] * e.w;
  double err = 0.0;
  for (int l = 0, off = 0; l <= L2; off += 2 * l + 1, ++l)
    for (int m = -l; m <= l; ++m) {
      cd acc = 0.0;
      for (const ModeEntry& e : tables.dec[static_cast<size_t>(l) * l + (m + l)])
        acc += e.w * spec[(e.u + L2) * w + (e.v + L2)];
      err = std::max(err, std::abs(acc - coeffs[off + m + l]));
    }
  if (err > 1e-8) throw std::runtime_error("fourier_tables: encode/decode round trip failed");
  return tables;
}

// proj/src/gtp.cpp:183-195
const FourierTables& fourier_tables(int L) {
  static std::map<int, std::unique_ptr<const FourierTables>> cache;
  static std::mutex mu;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(L);
    if (it != cache.end()) return *it->second;
  }
  auto built = std::make_unique<const FourierTables>(build_fourier_tables(L));
  std::lock_guard<std::mutex> lock(mu);
  auto res = cache.try_emplace(L, std::move(built));
  return *res.first->second;
}

// proj/src/gtp.cpp:262-327
std::vector<double> gtp_fourier_select(const Tower& xt, const double* x, const Tower& yt,
                                       const double* y, const std::vector<int>& degrees,
                                       uint64_t* ops) {
  const int L = std::max(xt.lmax, yt.lmax);
  const FourierTables& tabs = fourier_tables(L);
  const int w = 2 * L + 1;
  auto encode = [&](const Tower& t, const double* v) {
    std::vector<cd> spec(static_cast<size_t>(w) * w);
    for (size_t e = 0; e < t.ls.size(); ++e) {
      const int l = t.ls[e];
      const double* c = v + t.off[e];
      for (int m = -l; m <= l; ++m)
        for (const ModeEntry& me : tabs.enc[static_cast<size_t>(l) * l + (m + l)]) {
          spec[(me.u + L) * w + (me.v + L)] += c[m + l] * me.w;
          count_muls(ops, 2);
        }
    }
    return spec;
  };
  const std::vector<cd> cx = encode(xt, x), cy = encode(yt, y);
  const int wz = 4 * L + 1;
  std::vector<cd> cz(static_cast<size_t>(wz) * wz);
  for (int u1 = -L; u1 <= L; ++u1)
    for (int v1 = -L; v1 <= L; ++v1) {
      const cd a = cx[(u1 + L) * w + (v1 + L)];
      for (int u2 = -L; u2 <= L; ++u2)
        for (int v2 = -L; v2 <= L; ++v2) {
          cz[(u1 + u2 + 2 * L) * wz + (v1 + v2 + 2 * L)] += a * cy[(u2 + L) * w + (v2 + L)];
          count_muls(ops, 4);
        }
    }
  std::vector<double> out;
  for (int l : degrees) {
    for (int m = -l; m <= l; ++m) {
      double val = 0.0;
      if (l <= 2 * L) {
        cd acc = 0.0;
        for (const ModeEntry& me : tabs.dec[static_cast<size_t>(l) * l + (m + l)]) {
          acc += me.w * cz[(me.u + 2 * L) * wz + (me.v + 2 * L)];
          count_muls(ops, 4);
        }
        val = acc.real();
      }
      out.push_back(val);
    }
  }
  return out;
}

// proj/src/gtp.cpp:34-44
std::vector<double> scale_degrees(const Tower& t, const double* x, const double* s, int ns,
                                  uint64_t* ops) {
  std::vector<double> out(x, x + t.dim);
  for (size_t e = 0; e < t.ls.size(); ++e) {
    const int l = t.ls[e];
    if (l >= ns) throw Invalid("weighted_gtp: weight vector shorter than input degrees");
    for (int i = 0; i < 2 * l + 1; ++i) out[t.off[e] + i] *= s[l];
    count_muls(ops, static_cast<uint64_t>(2 * l + 1));
  }
  return out;
}

// -------------------------------------------------------------------------
// mtp.cpp restatement
// -------------------------------------------------------------------------
// proj/src/mtp.cpp:94-97
int mtp_l_tilde(int L1, int L2, int L3) {
  const int m = std::max({L1, L2, L3});
  return (m + 1) / 2;
}

// proj/src/mtp.cpp:20-39 (X is dt x dt row-major)
void embed_one(double* X, int dt, const double* coeffs, int l, int lt, int impl, uint64_t* ops) {
  const CGTable& table = cg_real(lt, lt, l);
  if (impl == 1) {
    for (const CGEntry& e : table.entries) X[(e.m1 + lt) * dt + (e.m2 + lt)] += e.value * coeffs[e.m3 + l];
    count_muls(ops, table.entries.size());
    return;
  }
  thread_local std::vector<double> dense;
  densify_into(table, dense);
  const int d3 = 2 * l + 1;
  for (int i1 = 0; i1 < dt; ++i1)
    for (int i2 = 0; i2 < dt; ++i2) {
      const double* row = dense.data() + (static_cast<size_t>(i1) * dt + i2) * d3;
      double acc = 0.0;
      for (int i3 = 0; i3 < d3; ++i3) acc += row[i3] * coeffs[i3];
      X[i1 * dt + i2] += acc;
    }
  count_muls(ops, static_cast<uint64_t>(dt) * dt * d3);
}

// proj/src/mtp.cpp:48-58
std::vector<double> mtp_embed(const Tower& t, const double* x, int lt, int impl, uint64_t* ops) {
  if (lt < 0) throw Invalid("mtp_embed: l_tilde must be >= 0");
  if (t.lmax > 2 * lt) throw Invalid("mtp_embed: carrier too small for input degrees");
  const int dt = 2 * lt + 1;
  std::vector<double> X(static_cast<size_t>(dt) * dt, 0.0);
  for (size_t e = 0; e < t.ls.size(); ++e) embed_one(X.data(), dt, x + t.off[e], t.ls[e], lt, impl, ops);
  return X;
}

// proj/src/mtp.cpp:119-133
std::vector<double> mtp_matmul(int dt, const double* X, const double* Y, uint64_t* ops) {
  std::vector<double> Z(static_cast<size_t>(dt) * dt, 0.0);
  for (int i = 0; i < dt; ++i)
    for (int k = 0; k < dt; ++k) {
      const double xik = X[i * dt + k];
      for (int j = 0; j < dt; ++j) Z[i * dt + j] += xik * Y[k * dt + j];
    }
  count_muls(ops, static_cast<uint64_t>(dt) * dt * dt);
  return Z;
}

// proj/src/mtp.cpp:60-97
std::vector<double> mtp_extract_select(int dt, const double* Z, const std::vector<int>& degrees,
                                       int lt, int impl, uint64_t* ops) {
  if (dt != 2 * lt + 1) throw Invalid("mtp_extract: matrix does not match the carrier degree");
  int dim = 0;
  for (int l : degrees) dim += 2 * l + 1;
  std::vector<double> out(dim, 0.0);
  int off = 0;
  for (int l3 : degrees) {
    if (l3 <= 2 * lt) {
      const CGTable& table = cg_real(lt, lt, l3);
      const int d3 = 2 * l3 + 1;
      if (impl == 1) {
        for (const CGEntry& e : table.entries)
          out[off + e.m3 + l3] += e.value * Z[(e.m1 + lt) * dt + (e.m2 + lt)];
        count_muls(ops, table.entries.size());
      } else {
        thread_local std::vector<double> dense;
        densify_into(table, dense);
        for (int i1 = 0; i1 < dt; ++i1)
          for (int i2 = 0; i2 < dt; ++i2) {
            const double z = Z[i1 * dt + i2];
            const double* row = dense.data() + (static_cast<size_t>(i1) * dt + i2) * d3;
            for (int i3 = 0; i3 < d3; ++i3) out[off + i3] += row[i3] * z;
          }
        count_muls(ops, static_cast<uint64_t>(dt) * dt * d3);
      }
    }
    off += 2 * l3 + 1;
  }
  return out;
}

// proj/src/mtp.cpp:99-117
std::vector<double> mtp(const Tower& xt, const double* x, const Tower& yt, const double* y, int L3,
                        int impl, int lt_override, uint64_t* ops) {
  if (L3 < 0) throw Invalid("mtp: L3 must be >= 0");
  const int lt_min = mtp_l_tilde(xt.lmax, yt.lmax, L3);
  int lt = lt_min;
  if (lt_override >= 0) {
    if (lt_override < lt_min) throw Invalid("mtp: l_tilde below the minimal carrier degree");
    lt = lt_override;
  }
  const std::vector<double> X = mtp_embed(xt, x, lt, impl, ops);
  const std::vector<double> Y = mtp_embed(yt, y, lt, impl, ops);
  const int dt = 2 * lt + 1;
  const std::vector<double> Z = mtp_matmul(dt, X.data(), Y.data(), ops);
  std::vector<int> degrees(L3 + 1);
  for (int l = 0; l <= L3; ++l) degrees[l] = l;
  return mtp_extract_select(dt, Z.data(), degrees, lt, impl, ops);
}

// proj/src/mtp.cpp:144-180
double mtp_path_weight(int l1, int l2, int l3, int lt) {
  const Path check{l1, l2, l3};
  if (!check.valid() || l1 > 2 * lt || l2 > 2 * lt || l3 > 2 * lt) return 0.0;
  const CGTable& c1 = cg_real(lt, lt, l1);
  const CGTable& c2 = cg_real(lt, lt, l2);
  const CGTable& c3 = cg_real(lt, lt, l3);
  const int dt = 2 * lt + 1;
  std::vector<std::vector<const CGEntry*>> c2_by_row(dt);
  for (const CGEntry& e : c2.entries) c2_by_row[e.m1 + lt].push_back(&e);
  std::vector<std::vector<const CGEntry*>> c3_by_cell(static_cast<size_t>(dt) * dt);
  for (const CGEntry& e : c3.entries) c3_by_cell[(e.m1 + lt) * dt + (e.m2 + lt)].push_back(&e);
  const int d1 = 2 * l1 + 1, d2 = 2 * l2 + 1, d3 = 2 * l3 + 1;
  std::vector<double> K(static_cast<size_t>(d1) * d2 * d3, 0.0);
  for (const CGEntry& e1 : c1.entries)
    for (const CGEntry* e2 : c2_by_row[e1.m2 + lt])
      for (const CGEntry* e3 : c3_by_cell[(e1.m1 + lt) * dt + (e2->m2 + lt)])
        K[((e1.m3 + l1) * d2 + (e2->m3 + l2)) * d3 + (e3->m3 + l3)] += e1.value * e2->value * e3->value;
  const CGTable& c = cg_real(l1, l2, l3);
  double kc = 0.0, cc = 0.0;
  for (const CGEntry& e : c.entries) {
    const double k = K[((e.m1 + l1) * d2 + (e.m2 + l2)) * d3 + (e.m3 + l3)];
    kc += k * e.value;
    cc += e.value * e.value;
  }
  return cc == 0.0 ? 0.0 : kc / cc;
}

// -------------------------------------------------------------------------
// bench.cpp restatement
// -------------------------------------------------------------------------
std::vector<int> tower_degrees(int L) {
  std::vector<int> d(L + 1);
  for (int l = 0; l <= L; ++l) d[l] = l;
  return d;
}

// proj/src/bench.cpp:26-75 (run_once), restricted to one (x, y) pair
void run_once(int kind, int impl, int mode, int L, const Tower& xt, const double* x,
              const Tower& yt, const double* y, double* out, uint64_t* ops) {
  std::vector<double> scratch;
  if (kind == 0) {
    const int ci = impl == 0 ? 0 : 1;
    if (mode == 2) {
      if (!out) {
        scratch.resize(cgtp_mimo(ci, xt, x, yt, y, nullptr, nullptr));
        out = scratch.data();
      }
      cgtp_mimo(ci, xt, x, yt, y, out, ops);
      return;
    }
    const int l3_hi = mode == 1 ? 2 * L : L;
    std::vector<double> seg(2 * l3_hi + 1);
    for (int l3 = (mode == 1 ? 0 : L); l3 <= l3_hi; ++l3) {
      if (ci == 0)
        cgtp_path_naive({L, L, l3}, x, y, seg.data(), ops);
      else
        cgtp_path_sparse({L, L, l3}, x, y, seg.data(), ops);
    }
    return;
  }
  std::vector<int> degrees;
  if (mode == 0)
    degrees = {L};
  else
    degrees = tower_degrees(2 * L);
  if (kind == 1) {
    std::vector<double> r = impl == 2 ? gtp_grid_select(xt, x, yt, y, degrees, ops)
                                      : gtp_fourier_select(xt, x, yt, y, degrees, ops);
    if (out) std::copy(r.begin(), r.end(), out);
    return;
  }
  const int mi = impl == 0 ? 0 : 1;
  const int lt = mode == 0 ? mtp_l_tilde(L, L, L) : mtp_l_tilde(L, L, 2 * L);
  const std::vector<double> X = mtp_embed(xt, x, lt, mi, ops);
  const std::vector<double> Y = mtp_embed(yt, y, lt, mi, ops);
  const int dt = 2 * lt + 1;
  const std::vector<double> Z = mtp_matmul(dt, X.data(), Y.data(), ops);
  std::vector<double> r = mtp_extract_select(dt, Z.data(), degrees, lt, mi, ops);
  if (out) std::copy(r.begin(), r.end(), out);
}

bool impl_applies(int kind, int impl) {  // proj/src/bench.cpp:174-177
  if (kind == 1) return impl == 2 || impl == 3;
  return impl == 0 || impl == 1;
}

template <class Fn>
int guard(Fn&& fn) {
  try {
    return fn();
  } catch (const Invalid& e) {
    g_err = e.what();
    return -ORC_EINVAL;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return -ORC_EINVAL;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return -ORC_ERANGE;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -ORC_ERUNTIME;
  }
}

int copy_table(const CGTable& t, int* m1, int* m2, int* m3, double* v, int cap) {
  const int n = static_cast<int>(t.entries.size());
  if (!m1) return n;
  if (cap < n) {
    g_err = "table buffer too small";
    return -ORC_ECAP;
  }
  for (int i = 0; i < n; ++i) {
    m1[i] = t.entries[i].m1;
    m2[i] = t.entries[i].m2;
    m3[i] = t.entries[i].m3;
    v[i] = t.entries[i].value;
  }
  return n;
}

template <class T>
int batch_impl(int kind, int impl, int L, int64_t B, int C, int y_shared, const T* x, const T* y,
               T* out, int nthreads) {
  if (kind < 0 || kind > 2 || !impl_applies(kind, impl)) throw Invalid("batch: bad kind/impl");
  if (L < 0 || B < 0 || C < 1) throw Invalid("batch: bad sizes");
  const std::vector<int> deg = tower_degrees(L);
  const Tower t(deg.data(), static_cast<int>(deg.size()));
  const int din = t.dim;
  const int dout = kind == 0 ? (L + 1) * (L + 1) * (L + 1) * (L + 1) : (2 * L + 1) * (2 * L + 1);
  // warm the caches once, single-threaded (time_tpo's warmup does the same)
  {
    std::vector<double> z(din, 0.0), o(dout);
    run_once(kind, impl, 2, L, t, z.data(), t, z.data(), o.data(), nullptr);
  }
  const int64_t rows = B * C;
  nthreads = std::max(1, std::min<int>(nthreads, static_cast<int>(std::max<int64_t>(rows, 1))));
  auto work = [&](int64_t r0, int64_t r1) {
    std::vector<double> xs(din), ys(din), os(dout);
    for (int64_t r = r0; r < r1; ++r) {
      const int64_t b = r / C;
      const T* xp = x + r * din;
      const T* yp = y_shared ? y + b * din : y + r * din;
      for (int i = 0; i < din; ++i) {
        xs[i] = static_cast<double>(xp[i]);
        ys[i] = static_cast<double>(yp[i]);
      }
      run_once(kind, impl, 2, L, t, xs.data(), t, ys.data(), os.data(), nullptr);
      T* op = out + r * dout;
      for (int i = 0; i < dout; ++i) op[i] = static_cast<T>(os[i]);
    }
  };
  if (nthreads == 1) {
    work(0, rows);
  } else {
    std::vector<std::thread> th;
    const int64_t chunk = (rows + nthreads - 1) / nthreads;
    for (int i = 0; i < nthreads; ++i) {
      const int64_t r0 = i * chunk, r1 = std::min(rows, r0 + chunk);
      if (r0 < r1) th.emplace_back(work, r0, r1);
    }
    for (auto& h : th) h.join();
  }
  return 0;
}

}  // namespace

// =========================================================================
// C ABI
// =========================================================================
extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

void* orc_rng_new(uint64_t seed) { return new std::mt19937_64(seed); }
void orc_rng_free(void* rng) { delete static_cast<std::mt19937_64*>(rng); }

void orc_rng_irrep_random(void* rng, int dim, double* out) {
  std::normal_distribution<double> gauss;  // fresh per vector, irreps.cpp:79
  auto& g = *static_cast<std::mt19937_64*>(rng);
  for (int i = 0; i < dim; ++i) out[i] = gauss(g);
}

void orc_rng_rotation(void* rng, double* R) {
  // wigner.cpp:219-226: Quaterniond q(gauss, gauss, gauss, gauss) -- g++
  // evaluates the four arguments right-to-left, so z is drawn first.
  std::normal_distribution<double> gauss;
  auto& g = *static_cast<std::mt19937_64*>(rng);
  const double z = gauss(g), y = gauss(g), x = gauss(g), w = gauss(g);
  const double n = std::sqrt(w * w + x * x + y * y + z * z);
  const double qw = w / n, qx = x / n, qy = y / n, qz = z / n;
  // Eigen QuaternionBase::toRotationMatrix
  const double tx = 2 * qx, ty = 2 * qy, tz = 2 * qz;
  const double twx = tx * qw, twy = ty * qw, twz = tz * qw;
  const double txx = tx * qx, txy = ty * qx, txz = tz * qx;
  const double tyy = ty * qy, tyz = tz * qy, tzz = tz * qz;
  R[0] = 1 - (tyy + tzz);
  R[1] = txy - twz;
  R[2] = txz + twy;
  R[3] = txy + twz;
  R[4] = 1 - (txx + tzz);
  R[5] = tyz - twx;
  R[6] = txz - twy;
  R[7] = tyz + twx;
  R[8] = 1 - (txx + tyy);
}

double orc_cg_coefficient(int l1, int m1, int l2, int m2, int l3, int m3) {
  return cg_coefficient(l1, m1, l2, m2, l3, m3);
}

void orc_real_basis_change(int l, double* re, double* im) {
  const CMat U = real_basis_change(l);
  for (size_t i = 0; i < U.a.size(); ++i) {
    re[i] = U.a[i].real();
    im[i] = U.a[i].imag();
  }
}

int orc_cg_real(int l1, int l2, int l3, int* m1, int* m2, int* m3, double* v, int cap) {
  return guard([&] {
    if (l1 < 0 || l2 < 0 || l3 < 0) throw Invalid("cg_real: negative degree");
    return copy_table(cg_real(l1, l2, l3), m1, m2, m3, v, cap);
  });
}

int orc_gaunt_real(int l1, int l2, int l3, int* m1, int* m2, int* m3, double* v, int cap) {
  return guard([&] {
    if (l1 < 0 || l2 < 0 || l3 < 0) throw Invalid("gaunt_real: negative degree");
    return copy_table(gaunt_real(l1, l2, l3), m1, m2, m3, v, cap);
  });
}

int orc_wigner_d(int l, const double* R9, double* D) {
  return guard([&] {
    const Mat d = wigner_d(l, R9);
    std::copy(d.a.begin(), d.a.end(), D);
    return 0;
  });
}

int orc_rotate(const int* ls, int n, const double* x, const double* R9, double* out) {
  return guard([&] {
    const Tower t(ls, n);
    std::map<int, Mat> by_l;  // wigner.cpp:314-325
    for (size_t e = 0; e < t.ls.size(); ++e) {
      const int l = t.ls[e];
      auto it = by_l.find(l);
      if (it == by_l.end()) it = by_l.emplace(l, wigner_d(l, R9)).first;
      const Mat& D = it->second;
      const int d = 2 * l + 1;
      for (int i = 0; i < d; ++i) {
        double acc = 0.0;
        for (int j = 0; j < d; ++j) acc += D(i, j) * x[t.off[e] + j];
        out[t.off[e] + i] = acc;
      }
    }
    return 0;
  });
}

int orc_gauss_legendre(int n, double* nodes, double* weights) {
  return guard([&] {
    std::vector<double> a, b;
    gauss_legendre(n, a, b);
    std::copy(a.begin(), a.end(), nodes);
    std::copy(b.begin(), b.end(), weights);
    return 0;
  });
}

int orc_legendre_lambda(int lmax, const double* cos_theta, int n, double* lam) {
  return guard([&] {
    if (lmax < 0 || n < 0) throw Invalid("legendre: bad sizes");
    const Mat m = legendre_lambda_table(lmax, std::vector<double>(cos_theta, cos_theta + n));
    std::copy(m.a.begin(), m.a.end(), lam);
    return 0;
  });
}

int orc_to_sphere(const int* ls, int n, const double* x, int Lgrid, double* F, uint64_t* ops) {
  return guard([&] {
    const Tower t(ls, n);
    const GridPtr g = make_grid(Lgrid);
    const Mat f = to_sphere(t, x, *g, ops);
    std::copy(f.a.begin(), f.a.end(), F);
    return 0;
  });
}

int orc_from_sphere_select(int Lgrid, const double* F, const int* degrees, int nd, double* out,
                           uint64_t* ops) {
  return guard([&] {
    const GridPtr g = make_grid(Lgrid);
    Mat f(g->n_theta(), g->n_phi);
    std::copy(F, F + f.a.size(), f.a.begin());
    const std::vector<double> r = from_sphere_select(*g, f, std::vector<int>(degrees, degrees + nd), ops);
    std::copy(r.begin(), r.end(), out);
    return static_cast<int>(r.size());
  });
}

int orc_num_paths(int L1, int L2, int L3) {
  return static_cast<int>(valid_paths(L1, L2, L3).size());
}

int orc_valid_paths(int L1, int L2, int L3, int* l1, int* l2, int* l3, int cap) {
  const std::vector<Path> p = valid_paths(L1, L2, L3);
  const int n = static_cast<int>(p.size());
  if (cap < n) return -ORC_ECAP;
  for (int i = 0; i < n; ++i) {
    l1[i] = p[i].l1;
    l2[i] = p[i].l2;
    l3[i] = p[i].l3;
  }
  return n;
}

int orc_cgtp_path(int impl, int l1, int l2, int l3, const double* x, int nx, const double* y,
                  int ny, double* out, int nout, uint64_t* ops) {
  return guard([&] {
    const Path p{l1, l2, l3};
    check_slices(p, nx, ny, nout);
    if (impl == 0)
      cgtp_path_naive(p, x, y, out, ops);
    else
      cgtp_path_sparse(p, x, y, out, ops);
    return 0;
  });
}

int orc_cgtp_mimo(int impl, const int* xls, int nx, const double* x, const int* yls, int ny,
                  const double* y, double* out, uint64_t* ops) {
  return guard([&] {
    const Tower xt(xls, nx), yt(yls, ny);
    return cgtp_mimo(impl, xt, x, yt, y, out, ops);
  });
}

int orc_gtp_grid_select(const int* xls, int nx, const double* x, const int* yls, int ny,
                        const double* y, const int* degrees, int nd, double* out, uint64_t* ops) {
  return guard([&] {
    const Tower xt(xls, nx), yt(yls, ny);
    for (int i = 0; i < nd; ++i)
      if (degrees[i] < 0) throw Invalid("gtp_grid: L3 must be >= 0");
    const std::vector<double> r = gtp_grid_select(xt, x, yt, y, std::vector<int>(degrees, degrees + nd), ops);
    std::copy(r.begin(), r.end(), out);
    return static_cast<int>(r.size());
  });
}

int orc_gtp_fourier_select(const int* xls, int nx, const double* x, const int* yls, int ny,
                           const double* y, const int* degrees, int nd, double* out,
                           uint64_t* ops) {
  return guard([&] {
    const Tower xt(xls, nx), yt(yls, ny);
    for (int i = 0; i < nd; ++i)
      if (degrees[i] < 0) throw Invalid("gtp_fourier: L3 must be >= 0");
    const std::vector<double> r =
        gtp_fourier_select(xt, x, yt, y, std::vector<int>(degrees, degrees + nd), ops);
    std::copy(r.begin(), r.end(), out);
    return static_cast<int>(r.size());
  });
}

int orc_weighted_gtp(const int* xls, int nx, const double* x, const int* yls, int ny,
                     const double* y, const double* a, int na, const double* b, int nb,
                     const double* c, int nc, int L3, double* out, uint64_t* ops) {
  return guard([&] {
    // proj/src/gtp.cpp:206-215
    if (nc != L3 + 1) throw Invalid("weighted_gtp: c must have L3+1 entries");
    const Tower xt(xls, nx), yt(yls, ny);
    const std::vector<double> xs = scale_degrees(xt, x, a, na, ops);
    const std::vector<double> ys = scale_degrees(yt, y, b, nb, ops);
    const std::vector<int> deg = tower_degrees(L3);
    const std::vector<double> z = gtp_grid_select(xt, xs.data(), yt, ys.data(), deg, ops);
    const Tower zt(deg.data(), static_cast<int>(deg.size()));
    const std::vector<double> r = scale_degrees(zt, z.data(), c, nc, ops);
    std::copy(r.begin(), r.end(), out);
    return static_cast<int>(r.size());
  });
}

int orc_fourier_tables(int L, int which, int* counts, int* u, int* v, double* re, double* im,
                       int cap) {
  return guard([&] {
    if (L < 0) throw Invalid("fourier_tables: L must be >= 0");
    const FourierTables& t = fourier_tables(L);
    const auto& modes = which == 0 ? t.enc : t.dec;
    int total = 0;
    for (size_t i = 0; i < modes.size(); ++i) {
      if (counts) counts[i] = static_cast<int>(modes[i].size());
      for (const ModeEntry& e : modes[i]) {
        if (u) {
          if (total >= cap) throw std::runtime_error("fourier table buffer too small");
          u[total] = e.u;
          v[total] = e.v;
          re[total] = e.w.real();
          im[total] = e.w.imag();
        }
        ++total;
      }
    }
    return total;
  });
}

int orc_mtp_l_tilde(int L1, int L2, int L3) { return mtp_l_tilde(L1, L2, L3); }

int orc_mtp_embed(const int* ls, int n, const double* x, int lt, int impl, double* X, uint64_t* ops) {
  return guard([&] {
    const Tower t(ls, n);
    const std::vector<double> r = mtp_embed(t, x, lt, impl, ops);
    std::copy(r.begin(), r.end(), X);
    return 2 * lt + 1;
  });
}

int orc_mtp_matmul(int dt, const double* X, const double* Y, double* Z, uint64_t* ops) {
  return guard([&] {
    if (dt < 1) throw Invalid("mtp_matmul: carriers do not match");
    const std::vector<double> r = mtp_matmul(dt, X, Y, ops);
    std::copy(r.begin(), r.end(), Z);
    return 0;
  });
}

int orc_mtp_extract_select(int dt, const double* Z, const int* degrees, int nd, int lt, int impl,
                           double* out, uint64_t* ops) {
  return guard([&] {
    const std::vector<double> r =
        mtp_extract_select(dt, Z, std::vector<int>(degrees, degrees + nd), lt, impl, ops);
    std::copy(r.begin(), r.end(), out);
    return static_cast<int>(r.size());
  });
}

int orc_mtp(const int* xls, int nx, const double* x, const int* yls, int ny, const double* y,
            int L3, int impl, int lt_override, double* out, uint64_t* ops) {
  return guard([&] {
    const Tower xt(xls, nx), yt(yls, ny);
    const std::vector<double> r = mtp(xt, x, yt, y, L3, impl, lt_override, ops);
    std::copy(r.begin(), r.end(), out);
    return static_cast<int>(r.size());
  });
}

double orc_mtp_path_weight(int l1, int l2, int l3, int lt) { return mtp_path_weight(l1, l2, l3, lt); }

int64_t orc_count_ops(int kind, int impl, int mode, int L) {
  uint64_t ops = 0;
  const int st = guard([&]() -> int {
    // proj/src/bench.cpp:101-112 ; inputs never enter the count
    if (!impl_applies(kind, impl)) throw Invalid("count_ops: implementation does not apply");
    if (L < 0) throw Invalid("count_ops: L must be >= 0");
    std::vector<int> deg = mode == 2 ? tower_degrees(L) : std::vector<int>{L};
    const Tower t(deg.data(), static_cast<int>(deg.size()));
    std::mt19937_64 rng(1);
    std::vector<double> x(t.dim), y(t.dim);
    orc_rng_irrep_random(&rng, t.dim, x.data());
    orc_rng_irrep_random(&rng, t.dim, y.data());
    run_once(kind, impl, mode, L, t, x.data(), t, y.data(), nullptr, &ops);
    return 0;
  });
  return st < 0 ? static_cast<int64_t>(st) : static_cast<int64_t>(ops);
}

long orc_expressivity_count(int kind, int L) {
  // proj/include/tpo/expressivity.hpp:11-16
  if (kind == 0) {
    long n = 0;
    for (int l1 = 0; l1 <= L; ++l1)
      for (int l2 = 0; l2 <= L; ++l2) n += 2 * std::min(l1, l2) + 1;
    return n;
  }
  return 4L * L + 1;
}

int orc_mimo_out_dim(int kind, int L) {
  return kind == 0 ? (L + 1) * (L + 1) * (L + 1) * (L + 1) : (2 * L + 1) * (2 * L + 1);
}

int orc_batch_mimo(int kind, int impl, int L, int64_t B, int C, int y_shared, const double* x,
                   const double* y, double* out, int nthreads) {
  return guard([&] { return batch_impl<double>(kind, impl, L, B, C, y_shared, x, y, out, nthreads); });
}

int orc_batch_mimo_f32(int kind, int impl, int L, int64_t B, int C, int y_shared, const float* x,
                       const float* y, float* out, int nthreads) {
  return guard([&] { return batch_impl<float>(kind, impl, L, B, C, y_shared, x, y, out, nthreads); });
}

}  // extern "C"
