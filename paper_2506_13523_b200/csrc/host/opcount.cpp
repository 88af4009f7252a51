// The reference's OpCounter tallies (proj/include/tpo/opcount.hpp:13-21), computed from shapes.
//
// The GPU kernels do not execute the reference's scalar loops, so the multiply counts the reference
// reports for a call -- the quantity behind `tp bench`'s ops / ops_per_expr columns and count_ops
// (proj/src/bench.cpp:101-112) -- are derived from the same structural rules it applies at each
// count_muls site.  Every count below is a function of the irreps descriptors, the degrees, and the
// sizes of the (shared) CG / Fourier tables, never of the data, exactly as in the reference.
#include "opcount.hpp"

#include <algorithm>
#include <cstdlib>

#include "tables.hpp"

namespace tpo_b200 {
namespace opcount {

// cgtp_path_naive: 2 d1 d2 d3 per valid path (proj/src/cgtp.cpp:100-118)
// cgtp_path_sparse: 2 per (pass, m3, m1) slot whose m2 is in range, structural zeros included
// (proj/src/cgtp.cpp:120-143 with the four m2 patterns of :25-32)
uint64_t cgtp_path(bool naive, int l1, int l2, int l3) {
  if (l1 < 0 || l2 < 0 || l3 < std::abs(l1 - l2) || l3 > l1 + l2) return 0;
  if (naive) return 2ull * (2 * l1 + 1) * (2 * l2 + 1) * (2 * l3 + 1);
  uint64_t slots = 0;
  for (int pass = 0; pass < 4; ++pass)
    for (int m3 = -l3; m3 <= l3; ++m3)
      for (int m1 = -l1; m1 <= l1; ++m1) {
        const int m2 = (pass == 0) ? m1 + m3 : (pass == 1) ? m1 - m3 : (pass == 2) ? -m1 + m3 : -m1 - m3;
        if (std::abs(m2) <= l2) ++slots;
      }
  return 2 * slots;
}

// cgtp_mimo: one path call per (x entry, y entry, l3) (proj/src/cgtp.cpp:145-177)
uint64_t cgtp_mimo(bool naive, const std::vector<int>& xls, const std::vector<int>& yls) {
  uint64_t n = 0;
  for (int l1 : xls)
    for (int l2 : yls)
      for (int l3 = std::abs(l1 - l2); l3 <= l1 + l2; ++l3) n += cgtp_path(naive, l1, l2, l3);
  return n;
}

// to_sphere: nt per (entry copy, m), then the n_m x nt x n_phi expansion (proj/src/sphere.cpp:105-134)
uint64_t to_sphere(const std::vector<Entry>& x, int grid_L) {
  const uint64_t nt = grid_L + 1, np = 2 * grid_L + 1;
  int lmax = 0;
  uint64_t n = 0;
  for (const Entry& e : x) {
    lmax = std::max(lmax, e.l);
    n += static_cast<uint64_t>(e.mul) * (2 * e.l + 1) * nt;
  }
  return n + static_cast<uint64_t>(2 * lmax + 1) * nt * np;
}

uint64_t pointwise_mul(int grid_L) { return static_cast<uint64_t>(grid_L + 1) * (2 * grid_L + 1); }

// from_sphere_select: phi transform n_m n_phi nt, two row scalings n_m nt each, nt per output
// coefficient (proj/src/sphere.cpp:155-195)
uint64_t from_sphere_select(int grid_L, const std::vector<int>& degrees) {
  const uint64_t nt = grid_L + 1, np = 2 * grid_L + 1;
  int lmax = 0;
  uint64_t n = 0;
  for (int l : degrees) {
    lmax = std::max(lmax, l);
    n += static_cast<uint64_t>(2 * l + 1) * nt;
  }
  const uint64_t nm = 2 * lmax + 1;
  return n + nm * np * nt + 2 * nm * nt;
}

// gtp_grid_select: two syntheses on the product grid (band L1 + L2), the pointwise product and the
// analysis of the degrees inside the band (proj/src/gtp.cpp:228-260)
uint64_t gtp_grid_select(const std::vector<Entry>& x, const std::vector<Entry>& y, const std::vector<int>& degrees) {
  int L1 = 0, L2 = 0;
  for (const Entry& e : x) L1 = std::max(L1, e.l);
  for (const Entry& e : y) L2 = std::max(L2, e.l);
  const int band = L1 + L2;
  std::vector<int> inside;
  for (int l : degrees)
    if (l <= band) inside.push_back(l);
  return to_sphere(x, band) + to_sphere(y, band) + pointwise_mul(band) + from_sphere_select(band, inside);
}

// gtp_fourier_select: 2 per encode entry touched (real x complex), 4 per convolution term
// ((2L+1)^4, complex x complex), 4 per decode entry of the requested degrees <= 2L
// (proj/src/gtp.cpp:262-327)
uint64_t gtp_fourier_select(const std::vector<Entry>& x, const std::vector<Entry>& y, const std::vector<int>& degrees) {
  int L = 0;
  for (const Entry& e : x) L = std::max(L, e.l);
  for (const Entry& e : y) L = std::max(L, e.l);
  const FourierTables& t = fourier_tables(L);
  auto encode = [&](const std::vector<Entry>& v) {
    uint64_t n = 0;
    for (const Entry& e : v)
      for (int m = -e.l; m <= e.l; ++m) n += 2ull * e.mul * t.enc[static_cast<size_t>(e.l) * e.l + m + e.l].size();
    return n;
  };
  const uint64_t side = 2 * L + 1;
  uint64_t n = encode(x) + encode(y) + 4 * side * side * side * side;
  for (int l : degrees)
    if (l <= 2 * L)
      for (int m = -l; m <= l; ++m) n += 4ull * t.dec[static_cast<size_t>(l) * l + m + l].size();
  return n;
}

// scale_degrees: mul (2l+1) per entry (proj/src/gtp.cpp:34-44)
uint64_t scale_degrees(const std::vector<Entry>& x) {
  uint64_t n = 0;
  for (const Entry& e : x) n += static_cast<uint64_t>(e.mul) * (2 * e.l + 1);
  return n;
}

// mtp_embed: sparse = nnz(cg_real(lt, lt, l)) per copy, naive = dt^2 (2l+1) (proj/src/mtp.cpp:20-58)
uint64_t mtp_embed(bool naive, const std::vector<Entry>& x, int lt) {
  const uint64_t dt = 2 * lt + 1;
  uint64_t n = 0;
  for (const Entry& e : x)
    n += static_cast<uint64_t>(e.mul) * (naive ? dt * dt * (2 * e.l + 1) : real_cg(lt, lt, e.l).size());
  return n;
}
uint64_t mtp_matmul(int dt) { return static_cast<uint64_t>(dt) * dt * dt; }  // proj/src/mtp.cpp:119-133
// mtp_extract_select: per requested degree <= 2 lt, nnz (sparse) or dt^2 (2l+1) (naive) (:60-97)
uint64_t mtp_extract_select(bool naive, const std::vector<int>& degrees, int lt) {
  const uint64_t dt = 2 * lt + 1;
  uint64_t n = 0;
  for (int l : degrees)
    if (l <= 2 * lt) n += naive ? dt * dt * (2 * l + 1) : real_cg(lt, lt, l).size();
  return n;
}
uint64_t mtp(bool naive, const std::vector<Entry>& x, const std::vector<Entry>& y, int L3, int lt) {
  std::vector<int> deg(L3 + 1);
  for (int l = 0; l <= L3; ++l) deg[l] = l;
  return mtp_embed(naive, x, lt) + mtp_embed(naive, y, lt) + mtp_matmul(2 * lt + 1) + mtp_extract_select(naive, deg, lt);
}

}  // namespace opcount
}  // namespace tpo_b200
