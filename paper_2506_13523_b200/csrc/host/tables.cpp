// Host table builders (fp64).  See tables.hpp for the reference citations.
#include "tables.hpp"

#include <algorithm>
#include <array>
#include <cmath>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>

namespace tpo_b200 {
namespace {

using cd = std::complex<double>;
using cld = std::complex<long double>;

// ln(n!) for n < 512 in long double (the Racah sum cancels; extra mantissa
// bits keep every coefficient at ~1 ulp, as in proj/src/wigner.cpp:21-31).
const std::vector<long double>& lnfact() {
  static const std::vector<long double> t = [] {
    std::vector<long double> v(512, 0.0L);
    for (int i = 1; i < 512; ++i) v[i] = v[i - 1] + std::log(static_cast<long double>(i));
    return v;
  }();
  return t;
}

// <l1 m1 l2 m2 | l3 m3> by Racah's single sum (Condon-Shortley convention).
double racah_cg(int l1, int m1, int l2, int m2, int l3, int m3) {
  if (m1 + m2 != m3) return 0.0;
  if (l3 < std::abs(l1 - l2) || l3 > l1 + l2) return 0.0;
  if (std::abs(m1) > l1 || std::abs(m2) > l2 || std::abs(m3) > l3) return 0.0;
  const auto& f = lnfact();
  const long double half =
      0.5L * (std::log(2.0L * l3 + 1.0L) + f[l1 + l2 - l3] + f[l1 - l2 + l3] + f[l2 + l3 - l1] -
              f[l1 + l2 + l3 + 1] + f[l3 + m3] + f[l3 - m3] + f[l1 + m1] + f[l1 - m1] + f[l2 + m2] +
              f[l2 - m2]);
  const int k0 = std::max({0, l2 - l3 - m1, l1 - l3 + m2});
  const int k1 = std::min({l1 + l2 - l3, l1 - m1, l2 + m2});
  long double s = 0.0L;
  for (int k = k0; k <= k1; ++k) {
    const long double t = std::exp(half - (f[k] + f[l1 + l2 - l3 - k] + f[l1 - m1 - k] + f[l2 + m2 - k] +
                                           f[l3 - l2 + m1 + k] + f[l3 - l1 - m2 + k]));
    s += (k & 1) ? -t : t;
  }
  return static_cast<double>(s);
}

// Complex -> real change of basis U^l (proj/src/wigner.cpp:249-263): row n
// (real index) has nonzeros in columns +-|n| only.  Returned sparsely.
struct URow {
  int col[2];
  cd val[2];
  int n;
};
URow u_row(int l, int n) {
  (void)l;
  const double s = 1.0 / std::sqrt(2.0);
  const cd i(0.0, 1.0);
  URow r{};
  if (n == 0) {
    r.n = 1;
    r.col[0] = 0;
    r.val[0] = 1.0;
    return r;
  }
  const int m = std::abs(n);
  const double sg = (m % 2 == 0) ? 1.0 : -1.0;
  r.n = 2;
  if (n > 0) {  // cos row
    r.col[0] = m;
    r.val[0] = sg * s;
    r.col[1] = -m;
    r.val[1] = s;
  } else {  // sin row
    r.col[0] = m;
    r.val[0] = -i * sg * s;
    r.col[1] = -m;
    r.val[1] = i * s;
  }
  return r;
}

std::vector<CGEntry> build_real_cg(int l1, int l2, int l3) {
  std::vector<CGEntry> out;
  if (l3 < std::abs(l1 - l2) || l3 > l1 + l2) return out;
  const bool odd = ((l1 + l2 + l3) & 1) != 0;
  for (int n1 = -l1; n1 <= l1; ++n1) {
    const URow r1 = u_row(l1, n1);
    for (int n2 = -l2; n2 <= l2; ++n2) {
      const URow r2 = u_row(l2, n2);
      for (int n3 = -l3; n3 <= l3; ++n3) {
        const URow r3 = u_row(l3, n3);
        cd acc = 0.0;
        for (int a = 0; a < r1.n; ++a)
          for (int b = 0; b < r2.n; ++b) {
            const int m3 = r1.col[a] + r2.col[b];
            for (int c = 0; c < r3.n; ++c)
              if (r3.col[c] == m3)
                acc += r1.val[a] * r2.val[b] * std::conj(r3.val[c]) *
                       racah_cg(l1, r1.col[a], l2, r2.col[b], l3, m3);
          }
        const double keep = odd ? acc.imag() : acc.real();
        const double drop = odd ? acc.real() : acc.imag();
        if (std::abs(drop) > 1e-10)
          throw std::runtime_error("real_cg: basis change left a mixed table (" + std::to_string(l1) +
                                   "," + std::to_string(l2) + "," + std::to_string(l3) + ")");
        if (std::abs(keep) > 1e-12) out.push_back({n1, n2, n3, keep});
      }
    }
  }
  return out;
}

void gauss_legendre_impl(int n, std::vector<double>& x, std::vector<double>& w) {
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  for (int i = 0; i < (n + 1) / 2; ++i) {
    double z = std::cos(M_PI * (i + 0.75) / (n + 0.5)), dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = z;
      for (int k = 2; k <= n; ++k) {
        const double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      dp = n * (z * p1 - p0) / (z * z - 1.0);
      const double dz = p1 / dp;
      z -= dz;
      if (std::abs(dz) < 1e-15) break;
    }
    x[n - 1 - i] = z;
    x[i] = -z;
    w[i] = w[n - 1 - i] = 2.0 / ((1.0 - z * z) * dp * dp);
  }
  if (n % 2 == 1) x[n / 2] = 0.0;
}

}  // namespace

double cg_coefficient(int l1, int m1, int l2, int m2, int l3, int m3) { return racah_cg(l1, m1, l2, m2, l3, m3); }

void gauss_legendre(int n, std::vector<double>& nodes, std::vector<double>& weights) {
  gauss_legendre_impl(n, nodes, weights);
}

std::vector<double> legendre_lambda(int lmax, const std::vector<double>& ct) {
  const int n = static_cast<int>(ct.size());
  const int rows = (lmax + 1) * (lmax + 2) / 2;
  std::vector<double> lam(static_cast<size_t>(rows) * n);
  auto id = [](int l, int m) { return l * (l + 1) / 2 + m; };
  std::vector<double> p(rows);
  for (int j = 0; j < n; ++j) {
    const double x = ct[j], s = std::sqrt(std::max(0.0, 1.0 - x * x));
    p[0] = std::sqrt(1.0 / (4.0 * M_PI));
    for (int m = 1; m <= lmax; ++m) p[id(m, m)] = p[id(m - 1, m - 1)] * s * std::sqrt((2.0 * m + 1) / (2.0 * m));
    for (int m = 0; m < lmax; ++m) p[id(m + 1, m)] = x * std::sqrt(2.0 * m + 3) * p[id(m, m)];
    for (int m = 0; m <= lmax; ++m)
      for (int l = m + 2; l <= lmax; ++l) {
        const double a = std::sqrt((4.0 * l * l - 1.0) / (double(l) * l - double(m) * m));
        const double b = std::sqrt((4.0 * (l - 1.0) * (l - 1.0) - 1.0) / (double(l - 1) * (l - 1) - double(m) * m));
        p[id(l, m)] = a * (x * p[id(l - 1, m)] - p[id(l - 2, m)] / b);
      }
    for (int l = 0; l <= lmax; ++l)
      for (int m = 0; m <= l; ++m) lam[static_cast<size_t>(id(l, m)) * n + j] = (m ? std::sqrt(2.0) : 1.0) * p[id(l, m)];
  }
  return lam;
}

const std::vector<CGEntry>& real_cg(int l1, int l2, int l3) {
  static std::mutex mu;
  static std::map<std::array<int, 3>, std::unique_ptr<std::vector<CGEntry>>> cache;
  const std::array<int, 3> key{l1, l2, l3};
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return *it->second;
  }
  auto t = std::make_unique<std::vector<CGEntry>>(build_real_cg(l1, l2, l3));
  std::lock_guard<std::mutex> g(mu);
  return *cache.try_emplace(key, std::move(t)).first->second;
}

const S2Grid& s2_grid(int band) {
  static std::mutex mu;
  static std::map<int, std::unique_ptr<S2Grid>> cache;
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(band);
  if (it != cache.end()) return *it->second;
  auto gr = std::make_unique<S2Grid>();
  gr->band = band;
  gr->n_theta = band + 1;
  gr->n_phi = 2 * band + 1;
  gauss_legendre_impl(band + 1, gr->nodes, gr->weights);
  gr->lam = legendre_lambda(band, gr->nodes);
  gr->cs.resize(static_cast<size_t>(2 * band + 1) * gr->n_phi);
  for (int m = -band; m <= band; ++m)
    for (int k = 0; k < gr->n_phi; ++k) {
      const double phi = 2.0 * M_PI * k / gr->n_phi;
      gr->cs[static_cast<size_t>(m + band) * gr->n_phi + k] =
          m < 0 ? std::sin(-m * phi) : (m == 0 ? 1.0 : std::cos(m * phi));
    }
  return *cache.emplace(band, std::move(gr)).first->second;
}

namespace {

// Spectra of the antipodally extended real harmonics on the 4L+2 torus
// (proj/src/gtp.cpp:143-207).  The phi-DFT of cos/sin(m phi) is analytic
// (v = +-m only), with the antipodal flip contributing (-1)^m for
// theta > pi; the theta-DFT is a direct O(n) sum per u.
std::vector<std::vector<FourierMode>> encode_all(int Lb) {
  const int n = 2 * Lb + 2;  // Lb = 2L decode band, n = 4L+2
  std::vector<double> theta(n), cosv(n);
  for (int j = 0; j < n; ++j) {
    theta[j] = 2.0 * M_PI * j / n;
    cosv[j] = std::cos(theta[j] <= M_PI ? theta[j] : 2.0 * M_PI - theta[j]);
  }
  const std::vector<double> lam = legendre_lambda(Lb, cosv);
  std::vector<std::vector<FourierMode>> all(static_cast<size_t>(Lb + 1) * (Lb + 1));
  for (int l = 0; l <= Lb; ++l)
    for (int m = -l; m <= l; ++m) {
      const int ma = std::abs(m);
      // phi DFT coefficient D(v) for v = +-ma (1/n normalisation included)
      std::vector<std::pair<int, cd>> dv;
      if (m == 0) dv.push_back({0, 1.0});
      else if (m > 0) { dv.push_back({-ma, 0.5}); dv.push_back({ma, 0.5}); }
      else { dv.push_back({-ma, cd(0.0, 0.5)}); dv.push_back({ma, cd(0.0, -0.5)}); }
      auto& slot = all[static_cast<size_t>(l) * l + (m + l)];
      for (const auto& [v, d] : dv) {
        for (int u = -n / 2; u < n - n / 2; ++u) {
          cld acc = 0.0L;
          for (int j = 0; j < n; ++j) {
            const long double sgn = (theta[j] > M_PI && (ma & 1)) ? -1.0L : 1.0L;
            const long double ang = -static_cast<long double>(u) * theta[j];
            acc += sgn * static_cast<long double>(lam[static_cast<size_t>(l * (l + 1) / 2 + ma) * n + j]) *
                   cld(std::cos(ang), std::sin(ang));
          }
          const cd c = cd(static_cast<double>(acc.real()), static_cast<double>(acc.imag())) / double(n) * d;
          if (std::abs(c) < 1e-13) continue;
          if (std::abs(u) > l) throw std::runtime_error("fourier_tables: spectrum outside the expected band");
          slot.push_back({u, v, c});
        }
      }
      // reference order: v outer, u inner (proj/src/gtp.cpp:196-206)
      std::stable_sort(slot.begin(), slot.end(), [](const FourierMode& a, const FourierMode& b) {
        return a.v != b.v ? a.v < b.v : a.u < b.u;
      });
    }
  return all;
}

// Least-squares inverse of a full-column-rank complex block by the normal
// equations in extended precision: pinv = (E^H E)^{-1} E^H (Cholesky).
// Equals Eigen's COD pseudo-inverse (proj/src/gtp.cpp:233-236) for full
// column rank; the blocks are well conditioned (cond <= 5.4 at L=16).
std::vector<cd> pinv_normal(const std::vector<cd>& E, int R, int Cc) {
  std::vector<cld> G(static_cast<size_t>(Cc) * Cc);
  for (int a = 0; a < Cc; ++a)
    for (int b = 0; b < Cc; ++b) {
      cld s = 0.0L;
      for (int r = 0; r < R; ++r) {
        const cd ea = E[static_cast<size_t>(r) * Cc + a], eb = E[static_cast<size_t>(r) * Cc + b];
        s += std::conj(cld(ea.real(), ea.imag())) * cld(eb.real(), eb.imag());
      }
      G[static_cast<size_t>(a) * Cc + b] = s;
    }
  // Cholesky G = L L^H
  std::vector<cld> Lm(static_cast<size_t>(Cc) * Cc, 0.0L);
  for (int i = 0; i < Cc; ++i) {
    for (int j = 0; j <= i; ++j) {
      cld s = G[static_cast<size_t>(i) * Cc + j];
      for (int k = 0; k < j; ++k) s -= Lm[static_cast<size_t>(i) * Cc + k] * std::conj(Lm[static_cast<size_t>(j) * Cc + k]);
      if (i == j) {
        if (s.real() <= 1e-20L) throw std::runtime_error("fourier_tables: encode block is rank deficient");
        Lm[static_cast<size_t>(i) * Cc + i] = std::sqrt(s.real());
      } else {
        Lm[static_cast<size_t>(i) * Cc + j] = s / Lm[static_cast<size_t>(j) * Cc + j].real();
      }
    }
  }
  // solve G X = E^H column by column
  std::vector<cd> P(static_cast<size_t>(Cc) * R);
  std::vector<cld> z(Cc);
  for (int r = 0; r < R; ++r) {
    for (int i = 0; i < Cc; ++i) {  // forward: L z = conj(E[r,:])
      const cd e = E[static_cast<size_t>(r) * Cc + i];
      cld s = std::conj(cld(e.real(), e.imag()));
      for (int k = 0; k < i; ++k) s -= Lm[static_cast<size_t>(i) * Cc + k] * z[k];
      z[i] = s / Lm[static_cast<size_t>(i) * Cc + i].real();
    }
    for (int i = Cc - 1; i >= 0; --i) {  // backward: L^H x = z
      cld s = z[i];
      for (int k = i + 1; k < Cc; ++k) s -= std::conj(Lm[static_cast<size_t>(k) * Cc + i]) * z[k];
      z[i] = s / Lm[static_cast<size_t>(i) * Cc + i].real();
    }
    for (int i = 0; i < Cc; ++i) P[static_cast<size_t>(i) * R + r] = cd(double(z[i].real()), double(z[i].imag()));
  }
  return P;
}

FourierTables build_fourier(int L) {
  const int Lb = 2 * L;
  FourierTables t;
  t.L = L;
  const auto all = encode_all(Lb);
  t.enc.assign(all.begin(), all.begin() + static_cast<long>((L + 1) * (L + 1)));
  t.dec.resize(static_cast<size_t>(Lb + 1) * (Lb + 1));
  for (int ma = 0; ma <= Lb; ++ma) {
    std::vector<int> cols;
    for (int l = ma; l <= Lb; ++l) {
      cols.push_back(l * l + (ma + l));
      if (ma > 0) cols.push_back(l * l + (-ma + l));
    }
    std::vector<std::pair<int, int>> rows;
    for (int u = -Lb; u <= Lb; ++u) {
      rows.push_back({u, ma});
      if (ma > 0) rows.push_back({u, -ma});
    }
    const int R = static_cast<int>(rows.size()), Cc = static_cast<int>(cols.size());
    std::vector<cd> E(static_cast<size_t>(R) * Cc);
    for (int c = 0; c < Cc; ++c)
      for (const FourierMode& e : all[cols[c]])
        for (int r = 0; r < R; ++r)
          if (rows[r].first == e.u && rows[r].second == e.v) E[static_cast<size_t>(r) * Cc + c] = e.w;
    const std::vector<cd> P = pinv_normal(E, R, Cc);
    for (int c = 0; c < Cc; ++c)
      for (int r = 0; r < R; ++r) {
        const cd w = P[static_cast<size_t>(c) * R + r];
        if (std::abs(w) > 1e-13) t.dec[cols[c]].push_back({rows[r].first, rows[r].second, w});
      }
  }
  // decode(encode(e_i)) == e_i over the full decode band (gtp.cpp:245-274)
  double err = 0.0;
  const int w = 2 * Lb + 1;
  for (int l = 0; l <= Lb; ++l)
    for (int m = -l; m <= l; ++m) {
      std::vector<cd> spec(static_cast<size_t>(w) * w);
      for (const FourierMode& e : all[static_cast<size_t>(l) * l + m + l]) spec[(e.u + Lb) * w + (e.v + Lb)] += e.w;
      for (int lp = 0; lp <= Lb; ++lp)
        for (int mp = -lp; mp <= lp; ++mp) {
          cd acc = 0.0;
          for (const FourierMode& d : t.dec[static_cast<size_t>(lp) * lp + mp + lp]) acc += d.w * spec[(d.u + Lb) * w + (d.v + Lb)];
          err = std::max(err, std::abs(acc - ((lp == l && mp == m) ? 1.0 : 0.0)));
        }
    }
  if (err > 1e-8) throw std::runtime_error("fourier_tables: encode/decode round trip failed");
  return t;
}

}  // namespace

const FourierTables& fourier_tables(int L) {
  static std::mutex mu;
  static std::map<int, std::unique_ptr<FourierTables>> cache;
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(L);
    if (it != cache.end()) return *it->second;
  }
  auto t = std::make_unique<FourierTables>(build_fourier(L));
  std::lock_guard<std::mutex> g(mu);
  return *cache.try_emplace(L, std::move(t)).first->second;
}

}  // namespace tpo_b200
