// Host-side coefficient / quadrature tables for the device kernels.
//
// These are the product's own builders (the oracle under oracle/ is never
// linked).  They follow the reference table math:
//   real CG           proj/src/wigner.cpp:39-151,249-268
//   S2 grid           proj/src/sphere.cpp:22-103, product band proj/src/gtp.cpp:231-232
//   Fourier tables    proj/src/gtp.cpp:46-179
// and are built once per shape, in fp64, then rounded/split into the
// device formats by context.cpp.
#pragma once

#include <complex>
#include <cstdint>
#include <vector>

namespace tpo_b200 {

struct CGEntry {
  int m1, m2, m3;
  double v;
};

// Real-basis CG table for (l1,l2)->l3, entries sorted (m1, m2, m3) ascending,
// |v| > 1e-12 (proj/src/wigner.cpp:17,105).  Memoized, thread-safe.
const std::vector<CGEntry>& real_cg(int l1, int l2, int l3);

// Gauss-Legendre x uniform-phi grid of band B: n_theta = B+1 nodes
// (ascending cos theta), n_phi = 2B+1; lam rows idx(l,|m|) = l(l+1)/2+|m|
// over n_theta columns; cs rows m+B over n_phi columns.
struct S2Grid {
  int band = 0, n_theta = 0, n_phi = 0;
  std::vector<double> nodes, weights;
  std::vector<double> lam;  // [(B+1)(B+2)/2][n_theta]
  std::vector<double> cs;   // [2B+1][n_phi]
  double lambda(int l, int m_abs, int j) const { return lam[(l * (l + 1) / 2 + m_abs) * n_theta + j]; }
  double csm(int m, int k) const { return cs[(m + band) * n_phi + k]; }
};
const S2Grid& s2_grid(int band);

// Normalized associated Legendre table Lambda_{l,m}(acos x), no CS phase.
std::vector<double> legendre_lambda(int lmax, const std::vector<double>& cos_theta);
// complex-basis <l1 m1 l2 m2 | l3 m3> (Racah, Condon-Shortley), proj/src/wigner.cpp:39-62
double cg_coefficient(int l1, int m1, int l2, int m2, int l3, int m3);
// Gauss-Legendre nodes (ascending in (-1, 1)) and weights (sum 2), proj/src/sphere.cpp:57-87
void gauss_legendre(int n, std::vector<double>& nodes, std::vector<double>& weights);

// ---- stage operators and analysis tables (host/stages.cpp)
// Real Gaunt table (l1,l2)->l3 = integral of Y_l1m1 Y_l2m2 Y_l3m3 over the sphere (the reference's
// gaunt_real, proj/src/wigner.cpp:153-198), entries (m1, m2, m3) ascending, |v| > 1e-12.  Built here
// by exact Gauss-Legendre x uniform-phi quadrature of the real harmonics.  Memoized, thread-safe.
const std::vector<CGEntry>& real_gaunt(int l1, int l2, int l3);
// Dense k-major operators Mt[din][dout] (fp64) of the linear stages:
std::vector<double> op_to_sphere(int L, int grid_L);                            // [(L+1)^2][nt * np]
std::vector<double> op_from_sphere(int grid_L, const std::vector<int>& degrees);  // [nt * np][sum (2l+1)]
std::vector<double> op_mtp_embed(int L, int lt);                                 // [(L+1)^2][dt * dt]
std::vector<double> op_mtp_extract(int lt, const std::vector<int>& degrees);      // [dt * dt][sum (2l+1)]
// MTP path weight w(l1, l2, l3) = <K, C> / <C, C> (proj/src/mtp.cpp:144-180)
double mtp_path_weight(int l1, int l2, int l3, int lt);

struct FourierMode {
  int u, v;
  std::complex<double> w;
};
// enc[(l*l + m + l)] for l <= L, dec[...] for l <= 2L.
struct FourierTables {
  int L = 0;
  std::vector<std::vector<FourierMode>> enc, dec;
};
const FourierTables& fourier_tables(int L);

}  // namespace tpo_b200
