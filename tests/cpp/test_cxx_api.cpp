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

#include "tpo/bench.hpp"
#include "tpo/cgtp.hpp"
#include "tpo/gtp.hpp"
#include "tpo/mtp.hpp"
#include "tpo/sphere.hpp"
#include "tpo/wigner.hpp"
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
  // ---------------------------------------------------------------- round 2: stage / table API
  // OpCounter: the reference's counts per call (proj/include/tpo/opcount.hpp; orc_* count the same loops)
  {
    const IrrepVector x = IrrepVector::random(Irreps::single_copies(3), rng);
    const IrrepVector y = IrrepVector::random(Irreps::single_copies(3), rng);
    const std::vector<int> t = degrees_of(x.irreps);
    const auto xf = f32(x.data), yf = f32(y.data);
    std::vector<double> buf(4096);
    for (int impl = 0; impl <= 1; ++impl) {
      OpCounter c;
      cgtp_mimo(x, y, impl ? CgtpImpl::sparse : CgtpImpl::naive, &c);
      uint64_t r = 0;
      orc_cgtp_mimo(impl, t.data(), 4, xf.data(), t.data(), 4, yf.data(), buf.data(), &r);
      CHECK(c.muls == r);
      OpCounter m;
      mtp(x, y, 6, impl ? MtpImpl::sparse : MtpImpl::naive, &m);
      uint64_t rm = 0;
      orc_mtp(t.data(), 4, xf.data(), t.data(), 4, yf.data(), 6, impl, -1, buf.data(), &rm);
      CHECK(m.muls == rm);
    }
    std::vector<int> deg = {0, 1, 2, 3, 4, 5, 6};
    OpCounter g, f;
    gtp_grid(x, y, 6, &g);
    gtp_fourier(x, y, 6, &f);
    uint64_t rg = 0, rf = 0;
    orc_gtp_grid_select(t.data(), 4, xf.data(), t.data(), 4, yf.data(), deg.data(), 7, buf.data(), &rg);
    orc_gtp_fourier_select(t.data(), 4, xf.data(), t.data(), 4, yf.data(), deg.data(), 7, buf.data(), &rf);
    CHECK(g.muls == rg && f.muls == rf);
    // count_ops relinks (proj/src/bench.cpp:101-112): every kind / impl / mode equals the oracle's
    for (int L = 0; L <= 4; ++L)
      for (int mode = 0; mode < 3; ++mode) {
        const BenchSetting st{static_cast<BenchMode>(mode), L, 1};
        CHECK(count_ops(Kind::cgtp, BenchImpl::naive, st) == static_cast<uint64_t>(orc_count_ops(0, 0, mode, L)));
        CHECK(count_ops(Kind::cgtp, BenchImpl::sparse, st) == static_cast<uint64_t>(orc_count_ops(0, 1, mode, L)));
        CHECK(count_ops(Kind::gtp, BenchImpl::grid, st) == static_cast<uint64_t>(orc_count_ops(1, 2, mode, L)));
        CHECK(count_ops(Kind::gtp, BenchImpl::fourier, st) == static_cast<uint64_t>(orc_count_ops(1, 3, mode, L)));
        CHECK(count_ops(Kind::mtp, BenchImpl::naive, st) == static_cast<uint64_t>(orc_count_ops(2, 0, mode, L)));
        CHECK(count_ops(Kind::mtp, BenchImpl::sparse, st) == static_cast<uint64_t>(orc_count_ops(2, 1, mode, L)));
      }
    CHECK(throws_as<std::invalid_argument>([] { count_ops(Kind::gtp, BenchImpl::naive, {}); }));
  }
  // tables: cg_real / gaunt_real / cg_complex / real_basis_change / fourier_tables / grids
  {
    for (int l1 = 0; l1 <= 4; ++l1)
      for (int l2 = 0; l2 <= 3; ++l2)
        for (int l3 = 0; l3 <= 6; ++l3) {
          for (int gaunt = 0; gaunt <= 1; ++gaunt) {
            const CGTable& tb = gaunt ? gaunt_real(l1, l2, l3) : cg_real(l1, l2, l3);
            std::vector<int> a(512), b(512), c(512);
            std::vector<double> v(512);
            const int n = (gaunt ? orc_gaunt_real : orc_cg_real)(l1, l2, l3, a.data(), b.data(), c.data(), v.data(), 512);
            bool same = n == static_cast<int>(tb.entries.size());
            for (int i = 0; same && i < n; ++i)
              same = tb.entries[i].m1 == a[i] && tb.entries[i].m2 == b[i] && tb.entries[i].m3 == c[i] &&
                     std::abs(tb.entries[i].value - v[i]) < 1e-13;
            CHECK(same);
          }
          const std::vector<double> cc = cg_complex(l1, l2, l3);
          bool ok = true;
          for (int m1 = -l1; m1 <= l1; ++m1)
            for (int m2 = -l2; m2 <= l2; ++m2)
              for (int m3 = -l3; m3 <= l3; ++m3)
                ok = ok && std::abs(cc[((m1 + l1) * (2 * l2 + 1) + (m2 + l2)) * (2 * l3 + 1) + (m3 + l3)] -
                                    orc_cg_coefficient(l1, m1, l2, m2, l3, m3)) < 1e-14;
          CHECK(ok);
        }
    const std::vector<double> dense = densify(cg_real(1, 1, 1));
    // entry (m1, m2, m3) = (0, 1, -1) is -1/sqrt(2) (proj/tests/test_wigner.cpp:69-80)
    CHECK(dense.size() == 27 && std::abs(dense[((0 + 1) * 3 + (1 + 1)) * 3 + (-1 + 1)] + 1.0 / std::sqrt(2.0)) < 1e-15);
    for (int l = 0; l <= 5; ++l) {
      const ComplexMatrix U = real_basis_change(l);
      std::vector<double> re((2 * l + 1) * (2 * l + 1)), im(re.size());
      orc_real_basis_change(l, re.data(), im.data());
      double e = 0.0;
      for (size_t i = 0; i < re.size(); ++i) e = std::max(e, std::abs(U.data[i] - std::complex<double>(re[i], im[i])));
      CHECK(e < 1e-15);
    }
    for (int L = 1; L <= 6; L += 5) {
      const FourierTables& ft = fourier_tables(L);
      std::vector<int> counts((2 * L + 1) * (2 * L + 1)), u(200000), v(200000);
      std::vector<double> re(200000), im(200000);
      const int n = orc_fourier_tables(L, 1, counts.data(), u.data(), v.data(), re.data(), im.data(), 200000);
      int k = 0;
      bool same = static_cast<int>(ft.decode.modes.size()) == (2 * L + 1) * (2 * L + 1);
      for (size_t i = 0; same && i < ft.decode.modes.size(); ++i) {
        double best = 0.0;
        for (const auto& e : ft.decode.modes[i]) {  // every product entry appears in the oracle's list
          double d = 1e300;
          for (int j = k; j < k + counts[i]; ++j)
            if (u[j] == e.u && v[j] == e.v) d = std::abs(e.w - std::complex<double>(re[j], im[j]));
          best = std::max(best, d);
        }
        same = best < 1e-10;
        k += counts[i];
      }
      CHECK(same && k == n);
    }
    const GridPtr g = make_grid(6);
    std::vector<double> nodes(7), w(7);
    orc_gauss_legendre(7, nodes.data(), w.data());
    CHECK(g->n_theta() == 7 && g->n_phi == 13 && std::abs(g->theta_nodes[0] - nodes[0]) < 1e-15 &&
          std::abs(g->theta_weights[3] - w[3]) < 1e-15);
    CHECK(throws_as<std::invalid_argument>([] { make_grid(-1); }));
  }
  // sphere stages on the GPU (proj/src/sphere.cpp) and the round trip (proj/src/verify.cpp:256-309)
  {
    const IrrepVector x = IrrepVector::random(Irreps::parse("1x0+2x1+1x3"), rng);
    const GridPtr g = make_grid(5);
    const SphereSignal F = to_sphere(x, g);
    const std::vector<int> dx = degrees_of(Irreps::single_copies(3));
    std::vector<double> tower(16, 0.0);  // copies summed (linear per entry)
    for (int e = 0; e < x.irreps.num_entries(); ++e)
      for (int c = 0; c < x.irreps.entries()[e].mul; ++c) {
        const int l = x.irreps.l_of(e);
        for (int i = 0; i < 2 * l + 1; ++i) tower[l * l + i] += x.data[x.irreps.offset(e, c) + i];
      }
    std::vector<double> ref(6 * 11);
    const auto tf = f32(tower);
    orc_to_sphere(dx.data(), 4, tf.data(), 5, ref.data(), nullptr);
    CHECK(normwise(F.values.data, ref) <= tol);
    const IrrepVector back = from_sphere(F, 3);
    CHECK(normwise(back.data, tower) <= tol);
    CHECK(throws_as<std::invalid_argument>([&] { to_sphere(x, make_grid(2)); }));
    const SphereSignal P = pointwise_mul(F, F);
    CHECK(std::abs(P.values(2, 3) - F.values(2, 3) * F.values(2, 3)) <= 1e-6 * (1 + std::abs(P.values(2, 3))));
    CHECK(throws_as<std::invalid_argument>([&] { pointwise_mul(F, to_sphere(x, make_grid(6))); }));
  }
  // MTP stages (proj/src/mtp.cpp:20-133) compose to mtp; path weights
  {
    const IrrepVector x = IrrepVector::random(Irreps::single_copies(3), rng);
    const IrrepVector y = IrrepVector::random(Irreps::single_copies(3), rng);
    const int lt = mtp_l_tilde(3, 3, 6);
    const Matrix X = mtp_embed(x, lt), Y = mtp_embed(y, lt);
    const Matrix Z = mtp_matmul(X, Y);
    CHECK(normwise(mtp_extract(Z, 6, lt).data, mtp(x, y, 6).data) <= tol);
    std::vector<double> refX(X.data.size());
    const std::vector<int> t = degrees_of(x.irreps);
    const auto xf = f32(x.data);
    orc_mtp_embed(t.data(), 4, xf.data(), lt, 1, refX.data(), nullptr);
    CHECK(normwise(X.data, refX) <= tol);
    CHECK(throws_as<std::invalid_argument>([&] { mtp_embed(x, 1); }));
    CHECK(throws_as<std::invalid_argument>([&] { mtp_matmul(X, Matrix(3, 3)); }));
    CHECK(mtp_extract_select(Z, {2, 9}, lt).data.size() == 5 + 19);
    for (int l1 = 0; l1 <= 3; ++l1)
      for (int l3 = 0; l3 <= 4; ++l3) CHECK(std::abs(mtp_path_weights(l1, 2, l3, 3) - orc_mtp_path_weight(l1, 2, l3, 3)) < 1e-12);
  }
  // rotations: the reference's draws, Wigner-D and rotate on the GPU (proj/src/wigner.cpp:200-325)
  {
    std::mt19937_64 r1(7);
    void* r2 = orc_rng_new(7);
    const Rotation R = Rotation::random(r1);
    double ref[9];
    orc_rng_rotation(r2, ref);
    orc_rng_free(r2);
    double e = 0.0;
    for (int i = 0; i < 9; ++i) e = std::max(e, std::abs(R.R[i] - ref[i]));
    CHECK(e < 1e-14);
    for (int l = 0; l <= 6; ++l) {
      const Matrix D = wigner_d(l, R);
      std::vector<double> rd((2 * l + 1) * (2 * l + 1));
      orc_wigner_d(l, R.R.data(), rd.data());
      double d = 0.0;
      for (size_t i = 0; i < rd.size(); ++i) d = std::max(d, std::abs(D.data[i] - rd[i]));
      CHECK(d < 1e-10);
    }
    const IrrepVector x = IrrepVector::random(Irreps::parse("2x2+1x0+1x5"), rng);
    const IrrepVector rx = rotate(x, R);
    double worst = 0.0;
    for (int en = 0; en < x.irreps.num_entries(); ++en)
      for (int c = 0; c < x.irreps.entries()[en].mul; ++c) {
        const int l = x.irreps.l_of(en), off = x.irreps.offset(en, c);
        const Matrix D = wigner_d(l, R);
        for (int i = 0; i < 2 * l + 1; ++i) {
          double s = 0.0;
          for (int j = 0; j < 2 * l + 1; ++j) s += D(i, j) * x.data[off + j];
          worst = std::max(worst, std::abs(rx.data[off + i] - s));
        }
      }
    CHECK(worst < 1e-5);
    const Rotation a = Rotation::from_axis_angle({0, 0, 1}, M_PI / 2);
    CHECK(std::abs(a.R[1] + 1.0) < 1e-15 && std::abs(a.R[3] - 1.0) < 1e-15);
    CHECK(throws_as<std::invalid_argument>([] { Rotation::from_axis_angle({0, 0, 0}, 1.0); }));
    CHECK(throws_as<std::invalid_argument>([] { Rotation::from_matrix({2, 0, 0, 0, 1, 0, 0, 0, 1}); }));
    const Rotation ab = a.compose(Rotation::from_matrix(R.R));
    CHECK(std::abs(ab.R[0] - (a.R[0] * R.R[0] + a.R[1] * R.R[3] + a.R[2] * R.R[6])) < 1e-15);
  }
  // Schur linear layer (proj/src/irreps.cpp:95-129)
  {
    LinearLayer layer(Irreps::parse("2x0+1x1"), Irreps::parse("1x1+3x0"));
    CHECK(layer.num_weights() == 2 * 3 + 1);
    CHECK(throws_as<std::invalid_argument>([&] { layer.set_weights({1.0}); }));
    std::mt19937_64 r(3);
    layer.randomize(r);
    const IrrepVector x = IrrepVector::random(layer.in(), rng);
    OpCounter c;
    const IrrepVector y = apply_linear(layer, x, &c);
    std::vector<double> ref(y.data.size(), 0.0);
    uint64_t muls = 0;
    for (size_t i = 0; i < layer.connections().size(); ++i) {
      const auto& cn = layer.connections()[i];
      const int l = layer.in().l_of(cn.in_entry);
      for (int m = 0; m < 2 * l + 1; ++m)
        ref[layer.out().offset(cn.out_entry, cn.out_copy) + m] +=
            layer.weights()[i] * x.data[layer.in().offset(cn.in_entry, cn.in_copy) + m];
      muls += 2 * l + 1;
    }
    CHECK(normwise(y.data, ref) <= tol && c.muls == muls);
    CHECK(throws_as<std::invalid_argument>([&] { apply_linear(layer, IrrepVector::random(Irreps::parse("1x1"), rng)); }));
  }
  std::printf("cxx api: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
