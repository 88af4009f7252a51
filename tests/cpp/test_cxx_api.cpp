// C++ drop-in API test: the tpo:: functions (include/tpo/*.hpp, running on the
// B200 through libtpo_b200.so) against the fp64 oracle (oracle/, test
// infrastructure), in the style of the reference's doctest suites
// (proj/tests/test_{cgtp,gtp,mtp}.cpp).  Exit code 0 = all checks passed.
#include <cmath>
#include <cstdio>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "tpo/cgtp.hpp"
#include "tpo/gtp.hpp"
#include "tpo/mtp.hpp"
#include "tpo_oracle.h"

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    if (cond) {                                                            \
      ++g_pass;                                                            \
    } else {                                                               \
      ++g_fail;                                                            \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                      \
  } while (0)

template <class E, class F>
bool throws_as(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static std::vector<int> degrees_of(const tpo::Irreps& ir) {
  std::vector<int> d;
  for (const auto& e : ir.entries()) d.push_back(e.l);
  return d;
}

// fp32-rounded copy, as the device sees it
static std::vector<double> f32(const std::vector<double>& v) {
  std::vector<double> r;
  for (double d : v) r.push_back(static_cast<double>(static_cast<float>(d)));
  return r;
}

static double normwise(const std::vector<double>& a, const std::vector<double>& b) {
  double num = 0, den = 1e-300;
  for (size_t i = 0; i < a.size(); ++i) {
    num = std::max(num, std::abs(a[i] - b[i]));
    den = std::max(den, std::abs(b[i]));
  }
  return num / den;
}

int main() {
  using namespace tpo;
  std::mt19937_64 rng(20240901);
  const double tol = 1e-5;

  // layout + RNG parity with the reference (proj/README.md:108)
  {
    std::mt19937_64 r(20240901);
    CHECK(IrrepVector::random(Irreps::single_copies(0), r).data[0] == -1.5095082358763112);
    CHECK(Irreps::parse("2x1+1x0").dim() == 7);
    CHECK(Irreps::single_copies(2).str() == "1x0+1x1+1x2");
    CHECK(throws_as<std::invalid_argument>([] { Irreps::parse("not-irreps"); }));
    CHECK((throws_as<std::out_of_range>([] { Irreps::single_copies(1).offset(3); })));
  }
  // CGTP: towers and arbitrary single-copy entry lists
  for (const char* xs : {"1x0+1x1+1x2", "1x1", "1x2+1x0", "1x0+1x1+1x2+1x3"}) {
    for (const char* ys : {"1x0+1x1+1x2", "1x1+1x3"}) {
      const IrrepVector x = IrrepVector::random(Irreps::parse(xs), rng);
      const IrrepVector y = IrrepVector::random(Irreps::parse(ys), rng);
      const IrrepVector z = cgtp_mimo(x, y);
      const std::vector<int> dx = degrees_of(x.irreps), dy = degrees_of(y.irreps);
      const auto xf = f32(x.data), yf = f32(y.data);
      const int n = orc_cgtp_mimo(1, dx.data(), (int)dx.size(), xf.data(), dy.data(), (int)dy.size(), yf.data(),
                                  nullptr, nullptr);
      std::vector<double> ref(n);
      orc_cgtp_mimo(1, dx.data(), (int)dx.size(), xf.data(), dy.data(), (int)dy.size(), yf.data(), ref.data(),
                    nullptr);
      CHECK((int)z.data.size() == n && z.irreps.dim() == n);
      CHECK(normwise(z.data, ref) <= tol);
    }
  }
  CHECK(throws_as<std::invalid_argument>([&] {
    cgtp_mimo(IrrepVector::random(Irreps::parse("2x1"), rng), IrrepVector::random(Irreps::parse("1x1"), rng));
  }));
  // single-path kernels (proj/tests/test_cgtp.cpp:29-79)
  {
    std::vector<double> x(5), y(7), out(9);
    std::normal_distribution<double> g;
    for (double& v : x) v = g(rng);
    for (double& v : y) v = g(rng);
    cgtp_path_sparse({2, 3, 4}, x, y, out);
    std::vector<double> ref(9);
    const auto xf = f32(x), yf = f32(y);
    orc_cgtp_path(1, 2, 3, 4, xf.data(), 5, yf.data(), 7, ref.data(), 9, nullptr);
    CHECK(normwise(out, ref) <= tol);
    std::vector<double> o7(7, 99.0), ones(3, 1.0);
    cgtp_path_naive({1, 1, 3}, ones, ones, o7);
    CHECK(o7[0] == 0.0 && o7[6] == 0.0);
    std::vector<double> bad(5);
    CHECK(throws_as<std::invalid_argument>([&] { cgtp_path_naive({1, 1, 1}, ones, ones, bad); }));
  }
  CHECK(valid_paths(1, 1, 2).paths.size() == 6);
  // GTP grid / Fourier / MTP / weighted
  for (int L = 0; L <= 6; ++L) {
    const IrrepVector x = IrrepVector::random(Irreps::single_copies(L), rng);
    const IrrepVector y = IrrepVector::random(Irreps::single_copies(L), rng);
    const std::vector<int> t = degrees_of(x.irreps);
    const auto xf = f32(x.data), yf = f32(y.data);
    std::vector<int> deg(2 * L + 1);
    for (int l = 0; l <= 2 * L; ++l) deg[l] = l;
    std::vector<double> ref((2 * L + 1) * (2 * L + 1));
    orc_gtp_grid_select(t.data(), L + 1, xf.data(), t.data(), L + 1, yf.data(), deg.data(), 2 * L + 1, ref.data(),
                        nullptr);
    CHECK(normwise(gtp_grid(x, y, 2 * L).data, ref) <= tol);
    orc_gtp_fourier_select(t.data(), L + 1, xf.data(), t.data(), L + 1, yf.data(), deg.data(), 2 * L + 1,
                           ref.data(), nullptr);
    {
      const double e = normwise(gtp_fourier(x, y, 2 * L).data, ref);
      if (!(e <= tol)) std::fprintf(stderr, "gtp_fourier L=%d normwise %.3e\n", L, e);
      CHECK(e <= tol);
    }
    orc_mtp(t.data(), L + 1, xf.data(), t.data(), L + 1, yf.data(), 2 * L, 1, -1, ref.data(), nullptr);
    CHECK(normwise(mtp(x, y, 2 * L).data, ref) <= tol);
  }
  {
    const IrrepVector x = IrrepVector::random(Irreps::single_copies(2), rng);
    const IrrepVector y = IrrepVector::random(Irreps::single_copies(2), rng);
    const IrrepVector a = weighted_gtp(x, y, {1, 1, 1}, {1, 1, 1}, {1, 1, 1, 1, 1}, 4);
    CHECK(normwise(a.data, gtp_grid(x, y, 4).data) <= tol);
    CHECK(throws_as<std::invalid_argument>([&] { weighted_gtp(x, y, {1, 1}, {1, 1, 1}, {1, 1, 1, 1, 1}, 4); }));
    const IrrepVector s = detail::gtp_grid_select(x, y, {3, 1});
    const IrrepVector full = gtp_grid(x, y, 4);
    CHECK(s.irreps.str() == "1x3+1x1");
    CHECK(std::abs(s.data[0] - full.data[9]) <= 1e-6 && std::abs(s.data[7] - full.data[1]) <= 1e-6);
    CHECK(throws_as<std::invalid_argument>([&] { mtp(x, y, 2, MtpImpl::sparse, nullptr, 0); }));
    CHECK(throws_as<std::invalid_argument>([&] { gtp_grid(x, y, -1); }));
  }
  // known answers (proj/tests/test_gtp.cpp:36-43, proj/tests/test_mtp.cpp:73-88)
  {
    IrrepVector x = IrrepVector::zeros(Irreps::single_copies(0)), y = x;
    x.data[0] = 3.0;
    y.data[0] = -2.0;
    CHECK(std::abs(gtp_grid(x, y, 0).data[0] + 6.0 / std::sqrt(4.0 * M_PI)) < 1e-6);
    CHECK(std::abs(mtp(x, y, 0).data[0] + 6.0) < 1e-5);
    CHECK(std::abs(mtp(x, y, 0, MtpImpl::sparse, nullptr, 1).data[0] - 6.0 / std::sqrt(3.0)) < 1e-5);
  }
  std::printf("cxx api: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
