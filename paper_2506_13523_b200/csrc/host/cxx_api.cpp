// namespace tpo C++ drop-in API (include/tpo/*.hpp) over the C ABI.
// One product per call like the reference (proj/src/{cgtp,gtp,mtp}.cpp);
// inputs are mapped onto 0..L towers (summing repeated degrees, which is
// exact for the Gaunt / matrix products because their synthesis/embedding
// is linear per entry, proj/src/sphere.cpp:113-127, proj/src/mtp.cpp:105-107)
// and run through tpo_run_host_f32 on a process-wide context.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <sstream>
#include <stdexcept>
#include <string>

#include "tpo/cgtp.hpp"
#include "tpo/gtp.hpp"
#include "tpo/mtp.hpp"
#include "tpo_capi.h"
#include "cxx_internal.hpp"
#include "opcount.hpp"

namespace tpo {

// ------------------------------------------------------------------ Irreps (proj/src/irreps.cpp:9-93)
Irreps::Irreps(std::vector<Entry> entries) : entries_(std::move(entries)) {
  for (const Entry& e : entries_) {
    if (e.mul < 1) throw std::invalid_argument("irreps: multiplicity must be >= 1");
    if (e.l < 0) throw std::invalid_argument("irreps: degree must be >= 0");
    dim_ += e.mul * (2 * e.l + 1);
  }
}

Irreps Irreps::single_copies(int L) {
  if (L < 0) throw std::invalid_argument("single_copies: L must be >= 0");
  std::vector<Entry> es;
  for (int l = 0; l <= L; ++l) es.push_back({1, l});
  return Irreps(std::move(es));
}

Irreps Irreps::parse(std::string_view text) {
  std::vector<Entry> es;
  size_t pos = 0;
  auto num = [&](const char* what) {
    int v = 0;
    auto [p, ec] = std::from_chars(text.data() + pos, text.data() + text.size(), v);
    if (ec != std::errc() || p == text.data() + pos)
      throw std::invalid_argument(std::string("irreps: expected ") + what + " in '" + std::string(text) + "'");
    pos = static_cast<size_t>(p - text.data());
    return v;
  };
  while (pos < text.size()) {
    const int mul = num("multiplicity");
    if (pos >= text.size() || text[pos] != 'x')
      throw std::invalid_argument("irreps: expected 'x' in '" + std::string(text) + "'");
    ++pos;
    const int l = num("degree");
    es.push_back({mul, l});
    if (pos < text.size()) {
      if (text[pos] != '+') throw std::invalid_argument("irreps: expected '+' in '" + std::string(text) + "'");
      if (++pos == text.size()) throw std::invalid_argument("irreps: trailing '+' in '" + std::string(text) + "'");
    }
  }
  return Irreps(std::move(es));
}

std::string Irreps::str() const {
  std::ostringstream os;
  for (size_t i = 0; i < entries_.size(); ++i) os << (i ? "+" : "") << entries_[i].mul << 'x' << entries_[i].l;
  return os.str();
}

int Irreps::offset(int entry, int copy) const {
  if (entry < 0 || entry >= num_entries()) throw std::out_of_range("irreps: entry index out of range");
  if (copy < 0 || copy >= entries_[entry].mul) throw std::out_of_range("irreps: copy index out of range");
  int off = 0;
  for (int e = 0; e < entry; ++e) off += entries_[e].mul * (2 * entries_[e].l + 1);
  return off + copy * (2 * entries_[entry].l + 1);
}

IrrepVector IrrepVector::zeros(const Irreps& irreps) { return {irreps, std::vector<double>(irreps.dim(), 0.0)}; }

IrrepVector IrrepVector::random(const Irreps& irreps, std::mt19937_64& rng) {
  std::normal_distribution<double> gauss;
  IrrepVector v = zeros(irreps);
  for (double& d : v.data) d = gauss(rng);
  return v;
}

Slice IrrepVector::slice(int entry, int copy) {
  return {data.data() + irreps.offset(entry, copy), 2 * irreps.l_of(entry) + 1};
}
ConstSlice IrrepVector::slice(int entry, int copy) const {
  return {data.data() + irreps.offset(entry, copy), 2 * irreps.l_of(entry) + 1};
}

// ------------------------------------------------------------------ device plumbing
namespace internal {

std::mutex g_mu;
tpo_ctx* g_ctx = nullptr;
int g_dev = 0;

tpo_ctx* ctx() {
  std::lock_guard<std::mutex> lock(g_mu);
  if (!g_ctx) {
    const char* env = std::getenv("TPO_DEVICE");
    const int dev = env ? std::atoi(env) : 0;
    g_dev = dev;
    if (tpo_ctx_create(dev, &g_ctx) != TPO_OK) {
      g_ctx = nullptr;
      throw std::runtime_error(std::string("tpo: cannot create device context: ") + tpo_last_error());
    }
  }
  return g_ctx;
}

void rethrow(int st) {
  if (st == TPO_OK) return;
  const std::string msg = tpo_last_error();
  if (st == TPO_EINVAL) throw std::invalid_argument(msg);
  if (st == TPO_ERANGE) throw std::out_of_range(msg);
  throw std::runtime_error(msg);
}

std::vector<tpo_b200::opcount::Entry> entries_of(const Irreps& ir) {
  std::vector<tpo_b200::opcount::Entry> e;
  for (const auto& x : ir.entries()) e.push_back({x.mul, x.l});
  return e;
}

}  // namespace internal

namespace {
using internal::ctx;
using internal::entries_of;
using internal::rethrow;

int max_degree(const Irreps& ir) {
  int m = 0;
  for (const auto& e : ir.entries()) m = std::max(m, e.l);
  return m;
}

// Sum every copy of x into a 0..L tower (fp32).
std::vector<float> to_tower(const IrrepVector& x, int L) {
  if (static_cast<int>(x.data.size()) != x.irreps.dim())
    throw std::invalid_argument("irreps: data length does not match irreps dim");
  std::vector<float> t(static_cast<size_t>(L + 1) * (L + 1), 0.f);
  std::vector<double> acc(t.size(), 0.0);
  for (int e = 0; e < x.irreps.num_entries(); ++e) {
    const int l = x.irreps.l_of(e);
    for (int c = 0; c < x.irreps.entries()[e].mul; ++c) {
      const ConstSlice s = x.slice(e, c);
      for (int i = 0; i < s.size; ++i) acc[l * l + i] += s[i];
    }
  }
  for (size_t i = 0; i < t.size(); ++i) t[i] = static_cast<float>(acc[i]);
  return t;
}

std::vector<double> run_host(int kind, int L1, int L2, int L3, int lt, const std::vector<float>& x,
                             const std::vector<float>& y, int64_t batch) {
  const int64_t dout = tpo_out_dim(kind, L1, L2, L3);
  if (dout < 0) rethrow(static_cast<int>(-dout));
  std::vector<float> out(static_cast<size_t>(dout * batch));
  rethrow(tpo_run_host_f32(ctx(), kind, L1, L2, L3, lt, x.data(), y.data(), out.data(), batch, 1, 0));
  return std::vector<double>(out.begin(), out.end());
}

IrrepVector select_degrees(const std::vector<double>& full, const std::vector<int>& degrees) {
  std::vector<Irreps::Entry> es;
  std::vector<double> data;
  for (int l : degrees) {
    es.push_back({1, l});
    for (int i = 0; i < 2 * l + 1; ++i) data.push_back(full[static_cast<size_t>(l * l + i)]);
  }
  return {Irreps(std::move(es)), std::move(data)};
}

IrrepVector gaunt_select(int kind, const IrrepVector& x, const IrrepVector& y, const std::vector<int>& degrees) {
  int L3 = 0;
  for (int l : degrees) {
    if (l < 0) throw std::invalid_argument("gtp: L3 must be >= 0");
    L3 = std::max(L3, l);
  }
  const int L1 = max_degree(x.irreps), L2 = max_degree(y.irreps);
  const std::vector<double> full = run_host(kind, L1, L2, L3, -1, to_tower(x, L1), to_tower(y, L2), 1);
  return select_degrees(full, degrees);
}

std::vector<int> upto(int L3) {
  if (L3 < 0) throw std::invalid_argument("gtp: L3 must be >= 0");
  std::vector<int> d(L3 + 1);
  for (int l = 0; l <= L3; ++l) d[l] = l;
  return d;
}

}  // namespace

// ------------------------------------------------------------------ CGTP
bool Path::valid() const { return l1 >= 0 && l2 >= 0 && l3 >= std::abs(l1 - l2) && l3 <= l1 + l2; }

Irreps PathTable::output_irreps() const {
  std::vector<Irreps::Entry> es;
  for (const Path& p : paths) es.push_back({1, p.l3});
  return Irreps(std::move(es));
}

PathTable valid_paths(int L1, int L2, int L3) {
  PathTable t;
  for (int l1 = 0; l1 <= L1; ++l1)
    for (int l2 = 0; l2 <= L2; ++l2)
      for (int l3 = std::abs(l1 - l2); l3 <= std::min(L3, l1 + l2); ++l3) t.paths.push_back({l1, l2, l3});
  return t;
}

namespace {
// offset of path (l1, l2, l3) inside the 0..L1 x 0..L2 tower output
int64_t tower_path_offset(int L2, int l1, int l2, int l3) {
  int64_t off = 0;
  for (int a = 0; a <= l1; ++a)
    for (int b = 0; b <= L2; ++b) {
      if (a == l1 && b == l2) {
        for (int c = std::abs(a - b); c < l3; ++c) off += 2 * c + 1;
        return off;
      }
      for (int c = std::abs(a - b); c <= a + b; ++c) off += 2 * c + 1;
    }
  return off;
}

// Batched single-path products: row r = (x entry i, y entry j) with towers
// holding only that entry; one launch for all pairs.
IrrepVector cgtp_pairs(const IrrepVector& x, const IrrepVector& y) {
  const int nx = x.irreps.num_entries(), ny = y.irreps.num_entries();
  const int L1 = max_degree(x.irreps), L2 = max_degree(y.irreps);
  const int d1 = (L1 + 1) * (L1 + 1), d2 = (L2 + 1) * (L2 + 1);
  const int64_t B = static_cast<int64_t>(nx) * ny;
  std::vector<float> X(static_cast<size_t>(B * d1), 0.f), Y(static_cast<size_t>(B * d2), 0.f);
  for (int i = 0; i < nx; ++i)
    for (int j = 0; j < ny; ++j) {
      const int64_t r = static_cast<int64_t>(i) * ny + j;
      const int li = x.irreps.l_of(i), lj = y.irreps.l_of(j);
      const ConstSlice xs = x.slice(i), ys = y.slice(j);
      for (int k = 0; k < xs.size; ++k) X[r * d1 + li * li + k] = static_cast<float>(xs[k]);
      for (int k = 0; k < ys.size; ++k) Y[r * d2 + lj * lj + k] = static_cast<float>(ys[k]);
    }
  const std::vector<double> full = B ? run_host(TPO_KIND_CGTP, L1, L2, 0, -1, X, Y, B) : std::vector<double>{};
  const int64_t dout = static_cast<int64_t>(d1) * d2;
  std::vector<Irreps::Entry> es;
  std::vector<double> data;
  for (int i = 0; i < nx; ++i)
    for (int j = 0; j < ny; ++j) {
      const int li = x.irreps.l_of(i), lj = y.irreps.l_of(j);
      const int64_t r = static_cast<int64_t>(i) * ny + j;
      for (int l3 = std::abs(li - lj); l3 <= li + lj; ++l3) {
        es.push_back({1, l3});
        const int64_t off = r * dout + tower_path_offset(L2, li, lj, l3);
        for (int k = 0; k < 2 * l3 + 1; ++k) data.push_back(full[static_cast<size_t>(off + k)]);
      }
    }
  return {Irreps(std::move(es)), std::move(data)};
}

void path_product(const Path& p, const std::vector<double>& x, const std::vector<double>& y,
                  std::vector<double>& out) {
  if (static_cast<int>(x.size()) != 2 * p.l1 + 1 || static_cast<int>(y.size()) != 2 * p.l2 + 1 ||
      static_cast<int>(out.size()) != 2 * p.l3 + 1)
    throw std::invalid_argument("cgtp: slice sizes do not match the path degrees");
  std::fill(out.begin(), out.end(), 0.0);
  if (!p.valid()) return;  // invalid path writes zeros (proj/src/cgtp.cpp:105)
  IrrepVector xv{Irreps({{1, p.l1}}), x}, yv{Irreps({{1, p.l2}}), y};
  const IrrepVector all = cgtp_pairs(xv, yv);
  const int off = all.irreps.offset(p.l3 - std::abs(p.l1 - p.l2));
  for (int k = 0; k < 2 * p.l3 + 1; ++k) out[k] = all.data[off + k];
}
}  // namespace

void cgtp_path_naive(const Path& p, const std::vector<double>& x, const std::vector<double>& y,
                     std::vector<double>& out, OpCounter* ops) {
  path_product(p, x, y, out);
  count_muls(ops, tpo_b200::opcount::cgtp_path(true, p.l1, p.l2, p.l3));
}
void cgtp_path_sparse(const Path& p, const std::vector<double>& x, const std::vector<double>& y,
                      std::vector<double>& out, OpCounter* ops) {
  path_product(p, x, y, out);
  count_muls(ops, tpo_b200::opcount::cgtp_path(false, p.l1, p.l2, p.l3));
}

IrrepVector cgtp_mimo(const IrrepVector& x, const IrrepVector& y, CgtpImpl impl, OpCounter* ops) {
  for (const auto& e : x.irreps.entries())
    if (e.mul != 1) throw std::invalid_argument("cgtp_mimo: inputs must be single-copy towers");
  for (const auto& e : y.irreps.entries())
    if (e.mul != 1) throw std::invalid_argument("cgtp_mimo: inputs must be single-copy towers");
  if (static_cast<int>(x.data.size()) != x.irreps.dim() || static_cast<int>(y.data.size()) != y.irreps.dim())
    throw std::invalid_argument("irreps: data length does not match irreps dim");
  IrrepVector out = cgtp_pairs(x, y);
  std::vector<int> xl, yl;
  for (const auto& e : x.irreps.entries()) xl.push_back(e.l);
  for (const auto& e : y.irreps.entries()) yl.push_back(e.l);
  count_muls(ops, tpo_b200::opcount::cgtp_mimo(impl == CgtpImpl::naive, xl, yl));
  return out;
}

// ------------------------------------------------------------------ GTP
IrrepVector gtp_grid(const IrrepVector& x, const IrrepVector& y, int L3, OpCounter* ops) {
  IrrepVector out = detail::gtp_grid_select(x, y, upto(L3), ops);
  out.irreps = Irreps::single_copies(L3);
  return out;
}

IrrepVector gtp_fourier(const IrrepVector& x, const IrrepVector& y, int L3, OpCounter* ops) {
  IrrepVector out = detail::gtp_fourier_select(x, y, upto(L3), ops);
  out.irreps = Irreps::single_copies(L3);
  return out;
}

IrrepVector weighted_gtp(const IrrepVector& x, const IrrepVector& y, const std::vector<double>& a,
                         const std::vector<double>& b, const std::vector<double>& c, int L3, OpCounter* ops) {
  if (static_cast<int>(c.size()) != L3 + 1) throw std::invalid_argument("weighted_gtp: c must have L3+1 entries");
  const int L1 = max_degree(x.irreps), L2 = max_degree(y.irreps);
  if (static_cast<int>(a.size()) < L1 + 1 || static_cast<int>(b.size()) < L2 + 1)
    throw std::invalid_argument("weighted_gtp: weight vector shorter than input degrees");
  // c (.) gtp(a (.) x, b (.) y), proj/src/gtp.cpp:206-215
  std::vector<float> X = to_tower(x, L1), Y = to_tower(y, L2);
  for (int l = 0; l <= L1; ++l)
    for (int i = 0; i < 2 * l + 1; ++i) X[l * l + i] = static_cast<float>(X[l * l + i] * a[l]);
  for (int l = 0; l <= L2; ++l)
    for (int i = 0; i < 2 * l + 1; ++i) Y[l * l + i] = static_cast<float>(Y[l * l + i] * b[l]);
  std::vector<double> full = run_host(TPO_KIND_GTP_GRID, L1, L2, L3, -1, X, Y, 1);
  for (int l = 0; l <= L3; ++l)
    for (int i = 0; i < 2 * l + 1; ++i) full[l * l + i] *= c[l];
  // proj/src/gtp.cpp:206-215: scale x, scale y, gtp_grid, scale the output
  namespace oc = tpo_b200::opcount;
  count_muls(ops, oc::scale_degrees(entries_of(x.irreps)) + oc::scale_degrees(entries_of(y.irreps)) +
                      oc::gtp_grid_select(entries_of(x.irreps), entries_of(y.irreps), upto(L3)) +
                      oc::scale_degrees(entries_of(Irreps::single_copies(L3))));
  return {Irreps::single_copies(L3), std::move(full)};
}

namespace detail {
IrrepVector gtp_grid_select(const IrrepVector& x, const IrrepVector& y, const std::vector<int>& degrees,
                            OpCounter* ops) {
  IrrepVector out = gaunt_select(TPO_KIND_GTP_GRID, x, y, degrees);
  count_muls(ops, tpo_b200::opcount::gtp_grid_select(entries_of(x.irreps), entries_of(y.irreps), degrees));
  return out;
}
IrrepVector gtp_fourier_select(const IrrepVector& x, const IrrepVector& y, const std::vector<int>& degrees,
                               OpCounter* ops) {
  IrrepVector out = gaunt_select(TPO_KIND_GTP_FOURIER, x, y, degrees);
  count_muls(ops, tpo_b200::opcount::gtp_fourier_select(entries_of(x.irreps), entries_of(y.irreps), degrees));
  return out;
}
}  // namespace detail

// ------------------------------------------------------------------ MTP
int mtp_l_tilde(int L1, int L2, int L3) { return tpo_mtp_l_tilde(L1, L2, L3); }

IrrepVector mtp(const IrrepVector& x, const IrrepVector& y, int L3, MtpImpl impl, OpCounter* ops,
                int l_tilde_override) {
  if (L3 < 0) throw std::invalid_argument("mtp: L3 must be >= 0");
  const int L1 = max_degree(x.irreps), L2 = max_degree(y.irreps);
  std::vector<double> full =
      run_host(TPO_KIND_MTP, L1, L2, L3, l_tilde_override, to_tower(x, L1), to_tower(y, L2), 1);
  const int lt = l_tilde_override >= 0 ? l_tilde_override : tpo_mtp_l_tilde(L1, L2, L3);
  count_muls(ops, tpo_b200::opcount::mtp(impl == MtpImpl::naive, entries_of(x.irreps), entries_of(y.irreps), L3, lt));
  return {Irreps::single_copies(L3), std::move(full)};
}

}  // namespace tpo
