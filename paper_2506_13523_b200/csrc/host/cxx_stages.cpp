// C++ drop-in mirrors of the reference's stage and table API (include/tpo/{wigner,sphere,gtp,mtp,
// bench,irreps}.hpp): one call per reference call, value semantics, the reference's exception types.
// Tables come from the host builders (tables.cpp, stages.cpp); the linear stages and rotations run
// as batch-of-1 launches of the C-ABI stage entry points on the process-wide context.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>

#include "cxx_internal.hpp"
#include "opcount.hpp"
#include "tables.hpp"
#include "tpo/bench.hpp"
#include "tpo/gtp.hpp"
#include "tpo/mtp.hpp"
#include "tpo/sphere.hpp"
#include "tpo/wigner.hpp"
#include "tpo_capi.h"

namespace tpo {
namespace {

using internal::ctx;
using internal::entries_of;
using internal::rethrow;

// one device buffer for the length of a call
template <class T>
struct DevBuf {
  T* p = nullptr;
  explicit DevBuf(size_t n) {
    if (cudaSetDevice(internal::g_dev) != cudaSuccess || cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)) != cudaSuccess)
      throw std::runtime_error("tpo: device allocation failed");
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { cudaFree(p); }
  void put(const std::vector<T>& h) {
    if (!h.empty() && cudaMemcpy(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess)
      throw std::runtime_error("tpo: host -> device copy failed");
  }
  std::vector<T> get(size_t n) const {
    std::vector<T> h(n);
    if (n && cudaMemcpy(h.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost) != cudaSuccess)
      throw std::runtime_error("tpo: device -> host copy failed");
    return h;
  }
};

int max_degree(const Irreps& ir) {
  int m = 0;
  for (const auto& e : ir.entries()) m = std::max(m, e.l);
  return m;
}

// every copy summed into a 0..L tower (the stages are linear per entry)
std::vector<float> tower_of(const IrrepVector& x, int L) {
  if (static_cast<int>(x.data.size()) != x.irreps.dim())
    throw std::invalid_argument("irreps: data length does not match irreps dim");
  std::vector<double> acc(static_cast<size_t>(L + 1) * (L + 1), 0.0);
  for (int e = 0; e < x.irreps.num_entries(); ++e) {
    const int l = x.irreps.l_of(e);
    for (int c = 0; c < x.irreps.entries()[e].mul; ++c) {
      const ConstSlice s = x.slice(e, c);
      for (int i = 0; i < s.size; ++i) acc[static_cast<size_t>(l) * l + i] += s[i];
    }
  }
  return std::vector<float>(acc.begin(), acc.end());
}

IrrepVector single_copies_of(const std::vector<int>& degrees, std::vector<double> data) {
  std::vector<Irreps::Entry> es;
  for (int l : degrees) es.push_back({1, l});
  return {Irreps(std::move(es)), std::move(data)};
}

int dim_of(const std::vector<int>& degrees) {
  int n = 0;
  for (int l : degrees) n += 2 * l + 1;
  return n;
}

std::vector<int> upto(int L) {
  std::vector<int> d(L + 1);
  for (int l = 0; l <= L; ++l) d[l] = l;
  return d;
}

Matrix3 quat_to_matrix(double w, double x, double y, double z) {
  return {1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w),
          2 * (x * y + z * w),     1 - 2 * (x * x + z * z), 2 * (y * z - x * w),
          2 * (x * z - y * w),     2 * (y * z + x * w),     1 - 2 * (x * x + y * y)};
}

}  // namespace

// ------------------------------------------------------------------ rotations (proj/src/wigner.cpp:200-232)
Rotation Rotation::from_axis_angle(const Vector3& axis, double angle) {
  const double n = std::sqrt(axis[0] * axis[0] + axis[1] * axis[1] + axis[2] * axis[2]);
  if (n == 0.0) throw std::invalid_argument("rotation: zero axis");
  const double ux = axis[0] / n, uy = axis[1] / n, uz = axis[2] / n;
  const double c = std::cos(angle), s = std::sin(angle), t = 1.0 - c;
  Rotation r;  // Rodrigues: c I + (1 - c) u u^T + s [u]_x
  r.R = {c + t * ux * ux,      t * ux * uy - s * uz, t * ux * uz + s * uy,
         t * ux * uy + s * uz, c + t * uy * uy,      t * uy * uz - s * ux,
         t * ux * uz - s * uy, t * uy * uz + s * ux, c + t * uz * uz};
  return r;
}

Rotation Rotation::from_matrix(const Matrix3& M) {
  double ortho = 0.0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = 0.0;
      for (int k = 0; k < 3; ++k) s += M[k * 3 + i] * M[k * 3 + j];
      ortho = std::max(ortho, std::abs(s - (i == j ? 1.0 : 0.0)));
    }
  const double det = M[0] * (M[4] * M[8] - M[5] * M[7]) - M[1] * (M[3] * M[8] - M[5] * M[6]) +
                     M[2] * (M[3] * M[7] - M[4] * M[6]);
  if (ortho > 1e-12 || std::abs(det - 1.0) > 1e-12)
    throw std::invalid_argument("rotation: matrix is not a proper rotation");
  Rotation r;
  r.R = M;
  return r;
}

Rotation Rotation::random(std::mt19937_64& rng) {
  std::normal_distribution<double> gauss;
  // Quaterniond(gauss, gauss, gauss, gauss) with g++'s right-to-left argument evaluation:
  // the first draw is z, then y, x, w
  const double z = gauss(rng), y = gauss(rng), x = gauss(rng), w = gauss(rng);
  const double n = std::sqrt(w * w + x * x + y * y + z * z);
  Rotation r;
  r.R = quat_to_matrix(w / n, x / n, y / n, z / n);
  return r;
}

Rotation Rotation::compose(const Rotation& other) const {
  Rotation r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = 0.0;
      for (int k = 0; k < 3; ++k) s += R[i * 3 + k] * other.R[k * 3 + j];
      r.R[i * 3 + j] = s;
    }
  return r;
}

// ------------------------------------------------------------------ tables
std::vector<double> cg_complex(int l1, int l2, int l3) {
  if (l1 < 0 || l2 < 0 || l3 < 0) throw std::invalid_argument("cg_complex: negative degree");
  const int d1 = 2 * l1 + 1, d2 = 2 * l2 + 1, d3 = 2 * l3 + 1;
  std::vector<double> out(static_cast<size_t>(d1) * d2 * d3, 0.0);
  if (l3 < std::abs(l1 - l2) || l3 > l1 + l2) return out;
  for (int m1 = -l1; m1 <= l1; ++m1)
    for (int m2 = -l2; m2 <= l2; ++m2) {
      const int m3 = m1 + m2;
      if (std::abs(m3) <= l3)
        out[(static_cast<size_t>(m1 + l1) * d2 + (m2 + l2)) * d3 + (m3 + l3)] =
            tpo_b200::cg_coefficient(l1, m1, l2, m2, l3, m3);
    }
  return out;
}

ComplexMatrix real_basis_change(int l) {
  // b = conj(U) a (proj/include/tpo/wigner.hpp:51-54): row m > 0 (cos) and m < 0 (sin) mix the +-m
  // columns with 1/sqrt(2) and the Condon-Shortley sign of odd m
  ComplexMatrix U;
  U.rows = U.cols = 2 * l + 1;
  U.data.assign(static_cast<size_t>(U.rows) * U.cols, 0.0);
  auto at = [&](int r, int c) -> std::complex<double>& { return U.data[static_cast<size_t>(r + l) * U.cols + (c + l)]; };
  const double s = 1.0 / std::sqrt(2.0);
  const std::complex<double> i(0.0, 1.0);
  at(0, 0) = 1.0;
  for (int m = 1; m <= l; ++m) {
    const double sg = (m % 2 == 0) ? 1.0 : -1.0;
    at(m, m) = sg * s;
    at(m, -m) = s;
    at(-m, m) = -i * sg * s;
    at(-m, -m) = i * s;
  }
  return U;
}

namespace {
const CGTable& table_cached(int l1, int l2, int l3, bool gaunt) {
  static std::mutex mu;
  static std::map<std::array<int, 4>, std::unique_ptr<CGTable>> cache;
  const std::array<int, 4> key{l1, l2, l3, gaunt ? 1 : 0};
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return *it->second;
  }
  if (l1 < 0 || l2 < 0 || l3 < 0) throw std::invalid_argument(gaunt ? "gaunt_real: negative degree" : "cg_real: negative degree");
  auto t = std::make_unique<CGTable>();
  t->l1 = l1;
  t->l2 = l2;
  t->l3 = l3;
  for (const auto& e : gaunt ? tpo_b200::real_gaunt(l1, l2, l3) : tpo_b200::real_cg(l1, l2, l3))
    t->entries.push_back({e.m1, e.m2, e.m3, e.v});
  std::lock_guard<std::mutex> g(mu);
  return *cache.try_emplace(key, std::move(t)).first->second;
}
}  // namespace

const CGTable& cg_real(int l1, int l2, int l3) { return table_cached(l1, l2, l3, false); }
const CGTable& gaunt_real(int l1, int l2, int l3) { return table_cached(l1, l2, l3, true); }

void densify_into(const CGTable& t, std::vector<double>& dense) {
  const int d2 = t.dim2(), d3 = t.dim3();
  dense.assign(static_cast<size_t>(t.dim1()) * d2 * d3, 0.0);
  for (const CGEntry& e : t.entries)
    dense[(static_cast<size_t>(e.m1 + t.l1) * d2 + (e.m2 + t.l2)) * d3 + (e.m3 + t.l3)] = e.value;
}
std::vector<double> densify(const CGTable& t) {
  std::vector<double> d;
  densify_into(t, d);
  return d;
}

Matrix wigner_d(int l, const Rotation& rot) {
  if (l < 0) throw std::invalid_argument("wigner_d: negative degree");
  tpo_ctx* c = ctx();
  DevBuf<double> R(9), D(static_cast<size_t>(tpo_wigner_d_size(l)));
  R.put(std::vector<double>(rot.R.begin(), rot.R.end()));
  rethrow(tpo_wigner_d_f64(c, l, R.p, D.p, 1, nullptr));
  const std::vector<double> all = D.get(static_cast<size_t>(tpo_wigner_d_size(l)));
  const int d = 2 * l + 1;
  const size_t off = static_cast<size_t>(tpo_wigner_d_size(l) - static_cast<int64_t>(d) * d);
  Matrix M(d, d);
  std::copy(all.begin() + static_cast<long>(off), all.end(), M.data.begin());
  return M;
}

IrrepVector rotate(const IrrepVector& x, const Rotation& rot) {
  if (static_cast<int>(x.data.size()) != x.irreps.dim())
    throw std::invalid_argument("irreps: data length does not match irreps dim");
  // one row per copy, each a tower of the largest degree holding only that copy's block
  const int L = max_degree(x.irreps), dl = (L + 1) * (L + 1);
  std::vector<std::pair<int, int>> copies;  // (degree, offset in x)
  for (int e = 0; e < x.irreps.num_entries(); ++e)
    for (int c = 0; c < x.irreps.entries()[e].mul; ++c) copies.push_back({x.irreps.l_of(e), x.irreps.offset(e, c)});
  IrrepVector out = IrrepVector::zeros(x.irreps);
  if (copies.empty()) return out;
  std::vector<float> rows(copies.size() * dl, 0.f);
  for (size_t r = 0; r < copies.size(); ++r)
    for (int i = 0; i < 2 * copies[r].first + 1; ++i)
      rows[r * dl + copies[r].first * copies[r].first + i] = static_cast<float>(x.data[copies[r].second + i]);
  tpo_ctx* c = ctx();
  DevBuf<double> R(9);
  R.put(std::vector<double>(rot.R.begin(), rot.R.end()));
  DevBuf<float> in(rows.size()), o(rows.size());
  in.put(rows);
  rethrow(tpo_rotate_f32(c, L, R.p, 1, in.p, o.p, static_cast<int64_t>(copies.size()), 1, nullptr));
  const std::vector<float> res = o.get(rows.size());
  for (size_t r = 0; r < copies.size(); ++r)
    for (int i = 0; i < 2 * copies[r].first + 1; ++i)
      out.data[copies[r].second + i] = res[r * dl + copies[r].first * copies[r].first + i];
  return out;
}

// ------------------------------------------------------------------ sphere (proj/src/sphere.cpp)
Matrix legendre_lambda_table(int l_max, const std::vector<double>& cos_theta) {
  if (l_max < 0) throw std::invalid_argument("legendre_lambda_table: l_max must be >= 0");
  const std::vector<double> t = tpo_b200::legendre_lambda(l_max, cos_theta);
  Matrix M((l_max + 1) * (l_max + 2) / 2, static_cast<int>(cos_theta.size()));
  M.data = t;
  return M;
}

void gauss_legendre(int n, std::vector<double>& nodes, std::vector<double>& weights) {
  tpo_b200::gauss_legendre(n, nodes, weights);
}

GridPtr make_grid(int L) {
  if (L < 0) throw std::invalid_argument("make_grid: L must be >= 0");
  const tpo_b200::S2Grid& h = tpo_b200::s2_grid(L);
  auto g = std::make_shared<S2Grid>();
  g->L_max = L;
  g->theta_nodes = h.nodes;
  g->theta_weights = h.weights;
  g->n_phi = h.n_phi;
  g->leg.l_max = L;
  g->leg.lambda = Matrix((L + 1) * (L + 2) / 2, h.n_theta);
  g->leg.lambda.data = h.lam;
  g->cs = Matrix(2 * L + 1, h.n_phi);
  g->cs.data = h.cs;
  return g;
}

SphereSignal to_sphere(const IrrepVector& x, const GridPtr& grid, OpCounter* ops) {
  if (!grid) throw std::invalid_argument("to_sphere: null grid");
  const int lmax = max_degree(x.irreps);
  if (lmax > grid->L_max)
    throw std::invalid_argument("to_sphere: grid band limit " + std::to_string(grid->L_max) + " below input degree " +
                                std::to_string(lmax));
  const std::vector<float> t = tower_of(x, lmax);
  const int G = grid->n_theta() * grid->n_phi;
  DevBuf<float> in(t.size()), F(G);
  in.put(t);
  rethrow(tpo_to_sphere_f32(ctx(), lmax, grid->L_max, in.p, F.p, 1, nullptr));
  const std::vector<float> f = F.get(G);
  SphereSignal s{grid, Matrix(grid->n_theta(), grid->n_phi)};
  s.values.data.assign(f.begin(), f.end());
  count_muls(ops, tpo_b200::opcount::to_sphere(entries_of(x.irreps), grid->L_max));
  return s;
}

SphereSignal pointwise_mul(const SphereSignal& a, const SphereSignal& b, OpCounter* ops) {
  if (!a.grid || !b.grid || a.grid->L_max != b.grid->L_max || a.values.rows != b.values.rows ||
      a.values.cols != b.values.cols)
    throw std::invalid_argument("pointwise_mul: signals live on different grids");
  const size_t n = a.values.data.size();
  DevBuf<float> da(n), db(n), dc(n);
  da.put(std::vector<float>(a.values.data.begin(), a.values.data.end()));
  db.put(std::vector<float>(b.values.data.begin(), b.values.data.end()));
  rethrow(tpo_pointwise_mul_f32(ctx(), da.p, db.p, dc.p, static_cast<int64_t>(n), nullptr));
  const std::vector<float> c = dc.get(n);
  SphereSignal out{a.grid, Matrix(a.values.rows, a.values.cols)};
  out.values.data.assign(c.begin(), c.end());
  count_muls(ops, tpo_b200::opcount::pointwise_mul(a.grid->L_max));
  return out;
}

namespace detail {
IrrepVector from_sphere_select(const SphereSignal& f, const std::vector<int>& degrees, OpCounter* ops) {
  if (!f.grid) throw std::invalid_argument("from_sphere: null grid");
  int lmax = 0;
  for (int l : degrees) lmax = std::max(lmax, l);
  if (lmax > f.grid->L_max) throw std::invalid_argument("from_sphere: grid band limit too small for requested degree");
  const int G = f.grid->n_theta() * f.grid->n_phi, ds = dim_of(degrees);
  DevBuf<float> F(G), out(ds);
  F.put(std::vector<float>(f.values.data.begin(), f.values.data.end()));
  rethrow(tpo_from_sphere_f32(ctx(), f.grid->L_max, degrees.data(), static_cast<int>(degrees.size()), F.p, out.p, 1,
                              nullptr));
  const std::vector<float> o = out.get(ds);
  count_muls(ops, tpo_b200::opcount::from_sphere_select(f.grid->L_max, degrees));
  return single_copies_of(degrees, std::vector<double>(o.begin(), o.end()));
}
}  // namespace detail

IrrepVector from_sphere(const SphereSignal& f, int L_out, OpCounter* ops) {
  if (L_out < 0) throw std::invalid_argument("from_sphere: L_out must be >= 0");
  IrrepVector out = detail::from_sphere_select(f, upto(L_out), ops);
  out.irreps = Irreps::single_copies(L_out);
  return out;
}

// ------------------------------------------------------------------ Fourier tables (proj/src/gtp.cpp:46-195)
const FourierTables& fourier_tables(int L) {
  static std::mutex mu;
  static std::map<int, std::unique_ptr<FourierTables>> cache;
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(L);
    if (it != cache.end()) return *it->second;
  }
  if (L < 0) throw std::invalid_argument("fourier_tables: L must be >= 0");
  const tpo_b200::FourierTables& h = tpo_b200::fourier_tables(L);
  auto t = std::make_unique<FourierTables>();
  t->L = L;
  t->encode.L = L;
  t->decode.L = 2 * L;
  for (const auto& v : h.enc) {
    t->encode.modes.emplace_back();
    for (const auto& e : v) t->encode.modes.back().push_back({e.u, e.v, e.w});
  }
  for (const auto& v : h.dec) {
    t->decode.modes.emplace_back();
    for (const auto& e : v) t->decode.modes.back().push_back({e.u, e.v, e.w});
  }
  std::lock_guard<std::mutex> g(mu);
  return *cache.try_emplace(L, std::move(t)).first->second;
}

// ------------------------------------------------------------------ MTP stages (proj/src/mtp.cpp)
Matrix mtp_embed(const IrrepVector& x, int l_tilde, MtpImpl impl, OpCounter* ops) {
  if (l_tilde < 0) throw std::invalid_argument("mtp_embed: l_tilde must be >= 0");
  const int L = max_degree(x.irreps);
  if (L > 2 * l_tilde) throw std::invalid_argument("mtp_embed: carrier too small for input degrees");
  const int dt = 2 * l_tilde + 1;
  const std::vector<float> t = tower_of(x, L);
  DevBuf<float> in(t.size()), X(static_cast<size_t>(dt) * dt);
  in.put(t);
  rethrow(tpo_mtp_embed_f32(ctx(), L, l_tilde, in.p, X.p, 1, nullptr));
  const std::vector<float> h = X.get(static_cast<size_t>(dt) * dt);
  Matrix M(dt, dt);
  M.data.assign(h.begin(), h.end());
  count_muls(ops, tpo_b200::opcount::mtp_embed(impl == MtpImpl::naive, entries_of(x.irreps), l_tilde));
  return M;
}

Matrix mtp_matmul(const Matrix& X, const Matrix& Y, OpCounter* ops) {
  if (X.rows != X.cols || Y.rows != Y.cols || X.rows != Y.rows)
    throw std::invalid_argument("mtp_matmul: carriers do not match");
  const int dt = X.rows;
  const size_t n = static_cast<size_t>(dt) * dt;
  DevBuf<float> dx(n), dy(n), dz(n);
  dx.put(std::vector<float>(X.data.begin(), X.data.end()));
  dy.put(std::vector<float>(Y.data.begin(), Y.data.end()));
  rethrow(tpo_mtp_matmul_f32(ctx(), dt, dx.p, dy.p, dz.p, 1, nullptr));
  const std::vector<float> z = dz.get(n);
  Matrix Z(dt, dt);
  Z.data.assign(z.begin(), z.end());
  count_muls(ops, tpo_b200::opcount::mtp_matmul(dt));
  return Z;
}

IrrepVector mtp_extract_select(const Matrix& Z, const std::vector<int>& degrees, int l_tilde, MtpImpl impl,
                               OpCounter* ops) {
  const int dt = 2 * l_tilde + 1;
  if (l_tilde < 0 || Z.rows != dt || Z.cols != dt)
    throw std::invalid_argument("mtp_extract: matrix does not match the carrier degree");
  const int ds = dim_of(degrees);
  DevBuf<float> dz(static_cast<size_t>(dt) * dt), out(ds);
  dz.put(std::vector<float>(Z.data.begin(), Z.data.end()));
  rethrow(tpo_mtp_extract_f32(ctx(), l_tilde, degrees.data(), static_cast<int>(degrees.size()), dz.p, out.p, 1, nullptr));
  const std::vector<float> o = out.get(ds);
  count_muls(ops, tpo_b200::opcount::mtp_extract_select(impl == MtpImpl::naive, degrees, l_tilde));
  return single_copies_of(degrees, std::vector<double>(o.begin(), o.end()));
}

IrrepVector mtp_extract(const Matrix& Z, int L3, int l_tilde, MtpImpl impl, OpCounter* ops) {
  if (L3 < 0) throw std::invalid_argument("mtp_extract: L3 must be >= 0");
  IrrepVector out = mtp_extract_select(Z, upto(L3), l_tilde, impl, ops);
  out.irreps = Irreps::single_copies(L3);
  return out;
}

double mtp_path_weights(int l1, int l2, int l3, int l_tilde) { return tpo_b200::mtp_path_weight(l1, l2, l3, l_tilde); }

// ------------------------------------------------------------------ linear layer (proj/src/irreps.cpp:95-129)
LinearLayer::LinearLayer(Irreps in, Irreps out) : in_(std::move(in)), out_(std::move(out)) {
  for (int ei = 0; ei < in_.num_entries(); ++ei)
    for (int ci = 0; ci < in_.entries()[ei].mul; ++ci)
      for (int eo = 0; eo < out_.num_entries(); ++eo) {
        if (out_.l_of(eo) != in_.l_of(ei)) continue;  // Schur: nothing between different degrees
        for (int co = 0; co < out_.entries()[eo].mul; ++co) connections_.push_back({ei, ci, eo, co});
      }
  weights_.assign(connections_.size(), 0.0);
}

void LinearLayer::set_weights(const std::vector<double>& w) {
  if (w.size() != weights_.size())
    throw std::invalid_argument("linear layer: expected " + std::to_string(weights_.size()) + " weights, got " +
                                std::to_string(w.size()));
  weights_ = w;
}

void LinearLayer::randomize(std::mt19937_64& rng) {
  std::normal_distribution<double> gauss;
  for (double& w : weights_) w = gauss(rng);
}

IrrepVector apply_linear(const LinearLayer& layer, const IrrepVector& x, OpCounter* ops) {
  if (!(x.irreps == layer.in())) throw std::invalid_argument("linear layer: input descriptor mismatch");
  if (static_cast<int>(x.data.size()) != x.irreps.dim())
    throw std::invalid_argument("irreps: data length does not match irreps dim");
  std::vector<int> im, il, om, ol;
  for (const auto& e : layer.in().entries()) im.push_back(e.mul), il.push_back(e.l);
  for (const auto& e : layer.out().entries()) om.push_back(e.mul), ol.push_back(e.l);
  IrrepVector out = IrrepVector::zeros(layer.out());
  DevBuf<float> dx(x.data.size()), dy(out.data.size());
  dx.put(std::vector<float>(x.data.begin(), x.data.end()));
  rethrow(tpo_apply_linear_f32(ctx(), im.data(), il.data(), static_cast<int>(im.size()), om.data(), ol.data(),
                               static_cast<int>(om.size()), layer.weights().data(), layer.num_weights(), dx.p, dy.p, 1,
                               nullptr));
  const std::vector<float> y = dy.get(out.data.size());
  out.data.assign(y.begin(), y.end());
  uint64_t n = 0;
  for (const auto& c : layer.connections()) n += 2 * layer.in().l_of(c.in_entry) + 1;
  count_muls(ops, n);
  return out;
}

// ------------------------------------------------------------------ bench counting (proj/src/bench.cpp)
const char* impl_name(BenchImpl i) {
  switch (i) {
    case BenchImpl::naive: return "naive";
    case BenchImpl::sparse: return "sparse";
    case BenchImpl::grid: return "grid";
    default: return "fourier";
  }
}
const char* mode_name(BenchMode m) {
  switch (m) {
    case BenchMode::siso: return "siso";
    case BenchMode::simo: return "simo";
    default: return "mimo";
  }
}
bool impl_applies(Kind kind, BenchImpl impl) {
  if (kind == Kind::gtp) return impl == BenchImpl::grid || impl == BenchImpl::fourier;
  return impl == BenchImpl::naive || impl == BenchImpl::sparse;
}
std::uint64_t count_ops(Kind kind, BenchImpl impl, const BenchSetting& s) {
  if (!impl_applies(kind, impl)) throw std::invalid_argument("count_ops: implementation does not apply to this kind");
  if (s.L < 0) throw std::invalid_argument("count_ops: L must be >= 0");
  const int64_t r = tpo_count_muls(static_cast<int>(kind), static_cast<int>(impl), static_cast<int>(s.mode), s.L);
  if (r < 0) rethrow(static_cast<int>(-r));
  return static_cast<std::uint64_t>(r);
}

}  // namespace tpo
