// Host tables of the stage operators and of the analysis
// helpers the reference exposes next to the products (gaunt_real, mtp_path_weights).  Built once in
// fp64; the device copies live in the context (Context::dense_op).
#include <algorithm>
#include <array>
#include <cmath>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>

#include "tables.hpp"

namespace tpo_b200 {
namespace {

inline int flat(int l, int m) { return l * l + m + l; }

// real spherical harmonic Y_lm at grid point (j, k) of an S2Grid (proj/include/tpo/sphere.hpp:11-22)
inline double ylm(const S2Grid& g, int l, int m, int j, int k) { return g.lambda(l, std::abs(m), j) * g.csm(m, k); }

std::vector<CGEntry> build_real_gaunt(int l1, int l2, int l3) {
  std::vector<CGEntry> out;
  if (l3 < std::abs(l1 - l2) || l3 > l1 + l2 || ((l1 + l2 + l3) & 1)) return out;  // selection rules
  // integrand: theta-degree <= l1+l2+l3 <= 2B+1 with B+1 Gauss-Legendre nodes, phi-frequency
  // <= l1+l2+l3 <= 2B with 2B+1 uniform points: the quadrature is exact
  const int B = (l1 + l2 + l3 + 1) / 2;
  const S2Grid& g = s2_grid(B);
  const double phi_w = 2.0 * M_PI / g.n_phi;
  for (int m1 = -l1; m1 <= l1; ++m1)
    for (int m2 = -l2; m2 <= l2; ++m2)
      for (int m3 = -l3; m3 <= l3; ++m3) {
        // real-basis selection: |m3| in {|m1| + |m2|, ||m1| - |m2||}
        const int a1 = std::abs(m1), a2 = std::abs(m2), a3 = std::abs(m3);
        if (a3 != a1 + a2 && a3 != std::abs(a1 - a2)) continue;
        long double acc = 0.0L;
        for (int j = 0; j < g.n_theta; ++j) {
          long double row = 0.0L;
          for (int k = 0; k < g.n_phi; ++k)
            row += static_cast<long double>(g.csm(m1, k)) * g.csm(m2, k) * g.csm(m3, k);
          acc += static_cast<long double>(g.weights[j]) * g.lambda(l1, a1, j) * g.lambda(l2, a2, j) *
                 g.lambda(l3, a3, j) * row;
        }
        const double v = static_cast<double>(acc) * phi_w;
        if (std::abs(v) > 1e-12) out.push_back({m1, m2, m3, v});
      }
  return out;
}

}  // namespace

const std::vector<CGEntry>& real_gaunt(int l1, int l2, int l3) {
  static std::mutex mu;
  static std::map<std::array<int, 3>, std::unique_ptr<std::vector<CGEntry>>> cache;
  const std::array<int, 3> key{l1, l2, l3};
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return *it->second;
  }
  auto t = std::make_unique<std::vector<CGEntry>>(build_real_gaunt(l1, l2, l3));
  std::lock_guard<std::mutex> lk(mu);
  return *cache.try_emplace(key, std::move(t)).first->second;
}

// F(theta_j, phi_k) = sum_(l,m) x_lm Lambda_l|m|(theta_j) cs_m(phi_k) on make_grid(grid_L)
// (proj/src/sphere.cpp:105-134); column g = j * n_phi + k (the reference's row-major F)
std::vector<double> op_to_sphere(int L, int grid_L) {
  const S2Grid& g = s2_grid(grid_L);
  const int din = (L + 1) * (L + 1), G = g.n_theta * g.n_phi;
  std::vector<double> mt(static_cast<size_t>(din) * G);
  for (int l = 0; l <= L; ++l)
    for (int m = -l; m <= l; ++m)
      for (int j = 0; j < g.n_theta; ++j)
        for (int k = 0; k < g.n_phi; ++k)
          mt[static_cast<size_t>(flat(l, m)) * G + j * g.n_phi + k] = ylm(g, l, m, j, k);
  return mt;
}

// x_lm = sum_j w_j Lambda_l|m|(theta_j) (2 pi / n_phi) sum_k F(j,k) cs_m(phi_k), concatenated over
// `degrees` in the given order (proj/src/sphere.cpp:155-195)
std::vector<double> op_from_sphere(int grid_L, const std::vector<int>& degrees) {
  const S2Grid& g = s2_grid(grid_L);
  const int G = g.n_theta * g.n_phi;
  int dsel = 0;
  for (int l : degrees) dsel += 2 * l + 1;
  std::vector<double> mt(static_cast<size_t>(G) * dsel);
  const double phi_scale = 2.0 * M_PI / g.n_phi;
  int off = 0;
  for (int l : degrees) {
    for (int m = -l; m <= l; ++m)
      for (int j = 0; j < g.n_theta; ++j)
        for (int k = 0; k < g.n_phi; ++k)
          mt[static_cast<size_t>(j * g.n_phi + k) * dsel + off + m + l] = g.weights[j] * phi_scale * ylm(g, l, m, j, k);
    off += 2 * l + 1;
  }
  return mt;
}

// X[a][b] = sum_(l,m3) C(lt,lt,l)[a,b,m3] x_(l,m3)  (proj/src/mtp.cpp:20-58), X row-major dt x dt
std::vector<double> op_mtp_embed(int L, int lt) {
  const int din = (L + 1) * (L + 1), dt = 2 * lt + 1;
  std::vector<double> mt(static_cast<size_t>(din) * dt * dt, 0.0);
  for (int l = 0; l <= L; ++l)
    for (const CGEntry& e : real_cg(lt, lt, l))
      mt[static_cast<size_t>(flat(l, e.m3)) * dt * dt + (e.m1 + lt) * dt + (e.m2 + lt)] += e.v;
  return mt;
}

// out_(l3,m3) = sum_(a,b) C(lt,lt,l3)[a,b,m3] Z[a][b] over `degrees`; zero past 2 lt
// (proj/src/mtp.cpp:60-97)
std::vector<double> op_mtp_extract(int lt, const std::vector<int>& degrees) {
  const int dt = 2 * lt + 1;
  int dsel = 0;
  for (int l : degrees) dsel += 2 * l + 1;
  std::vector<double> mt(static_cast<size_t>(dt) * dt * dsel, 0.0);
  int off = 0;
  for (int l3 : degrees) {
    if (l3 <= 2 * lt)
      for (const CGEntry& e : real_cg(lt, lt, l3))
        mt[static_cast<size_t>((e.m1 + lt) * dt + (e.m2 + lt)) * dsel + off + e.m3 + l3] += e.v;
    off += 2 * l3 + 1;
  }
  return mt;
}

// The path kernel K[p][q][r] = sum_{a,k,b} C1[a,k,p] C2[k,b,q] C3[a,b,r] (C_i = cg_real(lt, lt, l_i))
// is evaluated here as dense carrier products: for each (p, q), Z = X_p Y_q with X_p = C1[:,:,p],
// Y_q = C2[:,:,q], then K[p][q][r] = <Z, C3[:,:,r]>_F.  Its projection on the path's CG tensor is the
// weight.
double mtp_path_weight(int l1, int l2, int l3, int lt) {
  const bool valid = l1 >= 0 && l2 >= 0 && l3 >= std::abs(l1 - l2) && l3 <= l1 + l2;
  if (!valid || lt < 0 || l1 > 2 * lt || l2 > 2 * lt || l3 > 2 * lt) return 0.0;
  const int dt = 2 * lt + 1, d1 = 2 * l1 + 1, d2 = 2 * l2 + 1, d3 = 2 * l3 + 1;
  auto dense = [&](int l, int d) {  // [d][dt][dt]
    std::vector<double> c(static_cast<size_t>(d) * dt * dt, 0.0);
    for (const CGEntry& e : real_cg(lt, lt, l))
      c[(static_cast<size_t>(e.m3 + l) * dt + (e.m1 + lt)) * dt + (e.m2 + lt)] = e.v;
    return c;
  };
  const std::vector<double> c1 = dense(l1, d1), c2 = dense(l2, d2), c3 = dense(l3, d3);
  std::vector<double> z(static_cast<size_t>(dt) * dt);
  std::vector<double> K(static_cast<size_t>(d1) * d2 * d3, 0.0);
  for (int p = 0; p < d1; ++p)
    for (int q = 0; q < d2; ++q) {
      const double* X = c1.data() + static_cast<size_t>(p) * dt * dt;
      const double* Y = c2.data() + static_cast<size_t>(q) * dt * dt;
      std::fill(z.begin(), z.end(), 0.0);
      for (int a = 0; a < dt; ++a)
        for (int k = 0; k < dt; ++k) {
          const double xa = X[a * dt + k];
          if (xa == 0.0) continue;
          for (int b = 0; b < dt; ++b) z[a * dt + b] += xa * Y[k * dt + b];
        }
      for (int r = 0; r < d3; ++r) {
        const double* C = c3.data() + static_cast<size_t>(r) * dt * dt;
        double s = 0.0;
        for (int i = 0; i < dt * dt; ++i) s += z[i] * C[i];
        K[(static_cast<size_t>(p) * d2 + q) * d3 + r] = s;
      }
    }
  double kc = 0.0, cc = 0.0;
  for (const CGEntry& e : real_cg(l1, l2, l3)) {
    kc += K[(static_cast<size_t>(e.m1 + l1) * d2 + (e.m2 + l2)) * d3 + (e.m3 + l3)] * e.v;
    cc += e.v * e.v;
  }
  return cc == 0.0 ? 0.0 : kc / cc;
}

}  // namespace tpo_b200
