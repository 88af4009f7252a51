// Drop-in mirror of proj/include/tpo/sphere.hpp (Eigen-free).  The grid tables are host-built once
// per band; to_sphere / from_sphere / pointwise_mul run on the B200 (tpo_to_sphere_f32,
// tpo_from_sphere_f32, tpo_pointwise_mul_f32), fp32-accurate.
#pragma once

#include <memory>
#include <vector>

#include "tpo/irreps.hpp"

namespace tpo {

// proj/include/tpo/sphere.hpp:11-28: Lambda_{l,m}(theta) rows idx(l, m) = l(l+1)/2 + m
struct LegendreCache {
  int l_max = 0;
  Matrix lambda;  // ((l_max+1)(l_max+2)/2) x n_points
  static int idx(int l, int m_abs) { return l * (l + 1) / 2 + m_abs; }
};

Matrix legendre_lambda_table(int l_max, const std::vector<double>& cos_theta);
void gauss_legendre(int n, std::vector<double>& nodes, std::vector<double>& weights);

// proj/include/tpo/sphere.hpp:37-46
struct S2Grid {
  int L_max = 0;
  std::vector<double> theta_nodes;    // cos(theta_j), ascending
  std::vector<double> theta_weights;  // sum 2
  int n_phi = 0;
  LegendreCache leg;
  Matrix cs;  // (2 L_max + 1) x n_phi, row m + L_max
  int n_theta() const { return static_cast<int>(theta_nodes.size()); }
};
using GridPtr = std::shared_ptr<const S2Grid>;

GridPtr make_grid(int L);  // n_theta = L+1, n_phi = 2L+1

struct SphereSignal {
  GridPtr grid;
  Matrix values;  // n_theta x n_phi
};

SphereSignal to_sphere(const IrrepVector& x, const GridPtr& grid, OpCounter* ops = nullptr);
IrrepVector from_sphere(const SphereSignal& f, int L_out, OpCounter* ops = nullptr);
SphereSignal pointwise_mul(const SphereSignal& a, const SphereSignal& b, OpCounter* ops = nullptr);

namespace detail {
IrrepVector from_sphere_select(const SphereSignal& f, const std::vector<int>& degrees, OpCounter* ops = nullptr);
}  // namespace detail

}  // namespace tpo
