// extern "C" boundary of libtpo_b200.so (declared in include/tpo_capi.h).
#include "tpo_capi.h"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <string>
#include <vector>

#include "host/context.hpp"
#include "host/opcount.hpp"
#include "host/tables.hpp"

using tpo_b200::Context;
using tpo_b200::CudaFailure;
using tpo_b200::InvalidArgument;
using tpo_b200::RowSpec;

struct tpo_ctx {
  explicit tpo_ctx(int dev) : impl(dev) {}
  Context impl;
};

namespace {

constexpr int kMaxL = 32;  // inputs; outputs up to 2 * kMaxL
thread_local std::string g_err;

// restores the caller's current device (recorded by Context::activate) when a C-ABI call returns
struct RestoreDevice {
  ~RestoreDevice() {
    int& prev = tpo_b200::caller_device();
    if (prev >= 0) {
      cudaSetDevice(prev);
      prev = -1;
    }
  }
};

template <class F>
int guarded(F&& f) {
  RestoreDevice restore;
  try {
    f();
    return TPO_OK;
  } catch (const InvalidArgument& e) {
    g_err = e.what();
    return TPO_EINVAL;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return TPO_EINVAL;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return TPO_ERANGE;
  } catch (const CudaFailure& e) {
    g_err = e.what();
    return TPO_ECUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return TPO_ERUNTIME;
  }
}

void check_args(const tpo_ctx* ctx, int L1, int L2, const void* x, const void* y, const void* out,
                int64_t batch, int64_t channels) {
  if (!ctx) throw InvalidArgument("tpo: null context");
  if (L1 < 0 || L2 < 0) throw InvalidArgument("irreps: degree must be >= 0");
  if (L1 > kMaxL || L2 > kMaxL)
    throw InvalidArgument("tpo: input degree above the supported maximum of " + std::to_string(kMaxL));
  if (batch < 0) throw InvalidArgument("tpo: batch must be >= 0");
  if (channels < 1) throw InvalidArgument("tpo: channels must be >= 1");
  if (batch > 0 && (!x || !y || !out)) throw InvalidArgument("tpo: null data pointer");
}

void check_L3(int L3, const char* who) {
  if (L3 < 0) throw InvalidArgument(std::string(who) + ": L3 must be >= 0");
  if (L3 > 2 * kMaxL) throw InvalidArgument(std::string(who) + ": L3 above the supported maximum");
}

RowSpec rows_of(const float* x, const float* y, float* out, int64_t batch, int64_t channels, int y_shared) {
  RowSpec rs{};
  rs.x = x;
  rs.y = y;
  rs.out = out;
  rs.rows = batch * channels;
  rs.channels = channels;
  rs.y_shared = y_shared ? 1 : 0;
  return rs;
}

void launched(tpo_ctx* ctx, cudaError_t e, const char* what) {
  tpo_b200::cuda_check(e, what);
  ctx->impl.launches.fetch_add(1);
}

int min_lt(int L1, int L2, int L3) { return (std::max({L1, L2, L3}) + 1) / 2; }

// optional per-path weights of the CGTP (f2): w[(row / channels) * stride + path]
struct PathWeights {
  const float* w;
  int64_t stride;
  const int* path_of_out;
};

void run_cgtp(tpo_ctx* ctx, int L1, int L2, const RowSpec& rs, cudaStream_t s, const PathWeights* pw = nullptr) {
  const auto& t = ctx->impl.cgtp(L1, L2);
  // kernels without a fused weight: scale the written outputs afterwards
  auto post_scale = [&] {
    if (pw)
      launched(ctx, tpo_b200::launch_path_scale(rs.out, rs.rows, rs.channels, t.dout, pw->path_of_out, pw->w, pw->stride,
                                                ctx->impl.num_sms(), s),
               "cgtp path weights");
  };
  // shared y per edge (config C4): per-edge dense GEMMs on tcgen05 when the shape allows
  const int kp = (t.din1 + 15) / 16 * 16, dout_pad = (t.dout + 15) / 16 * 16;
  const bool aligned = (reinterpret_cast<uintptr_t>(rs.x) % 16 == 0) && (reinterpret_cast<uintptr_t>(rs.out) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(rs.y) % 16 == 0) && t.din2 % 4 == 0;  // x / y rows by TMA
  static const bool edge_tc_on = [] {
    const char* v = std::getenv("TPO_CGTP_EDGE_TC");
    return !(v && *v == '0');
  }();
  if (edge_tc_on && rs.y_shared && rs.channels % 128 == 0 && t.din1 % 4 == 0 && kp <= 64 && t.din2 <= 64 &&
      dout_pad <= 256 && t.dout % 4 == 0 && aligned &&
      tpo_b200::cgtp_edge_tc_smem(t, kp, dout_pad) <= 227 * 1024) {
    tpo_b200::EdgeTcParams p{};
    p.kp = kp;
    p.dout_pad = dout_pad;
    p.tmem_cols = 32;  // two Z buffers of dout_pad rounded to the 32-column store box
    while (p.tmem_cols < 2 * ((dout_pad + 31) / 32 * 32)) p.tmem_cols *= 2;
    tpo_b200::encode_tmap_2d(&p.tm_out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rs.out, static_cast<uint64_t>(t.dout),
                             static_cast<uint64_t>(rs.rows), static_cast<uint64_t>(t.dout) * 4, 32, 128,
                             CU_TENSOR_MAP_SWIZZLE_128B);
    if (pw) {  // fused: the weights scale the edge's M_y columns
      p.path_w = pw->w;
      p.w_stride = pw->stride;
      p.path_of_out = pw->path_of_out;
    }
    launched(ctx, tpo_b200::launch_cgtp_edge_tc(t, p, rs, ctx->impl.num_sms(), s), "cgtp edge tcgen05 kernel");
    return;
  }
  // larger degrees: per-(l1, l2) block GEMMs on tcgen05 (output-write bound)
  static const int tc_min_l = [] {
    const char* v = std::getenv("TPO_CGTP_TC_MINL");
    return v ? std::atoi(v) : 4;  // measured: SIMT wins at L <= 3 (L=4: 0.122 vs 0.147 ms)
  }();
  if (std::max(L1, L2) >= tc_min_l)
    if (const tpo_b200::CgtpTcTables* tc = ctx->impl.cgtp_tc(L1, L2)) {
      launched(ctx, tpo_b200::launch_cgtp_tc(*tc, rs, ctx->impl.num_sms(), s), "cgtp tcgen05 kernel");
      post_scale();
      return;
    }
  launched(ctx, tpo_b200::launch_cgtp(t, rs, ctx->impl.num_sms(), s), "cgtp kernel");
  post_scale();
}

// Inputs wider than the tcgen05 kernel's K limit (L > 12): the product is bilinear,
// so it is the sum over (x degree group, y degree group) of launches on the same
// operators restricted to those columns (Context::dense_split_tc), input windows
// packed by a gather kernel, partial outputs accumulated.  Returns false when a
// part does not fit either.
// Fourier: up to L = 16 (L = 15 / 16 adversarial worst 3.8e-6 / 2.7e-6 after the operand scaling and
// segmented accumulation; 118 / 155 ms per 2^19 shard against 299 / 503 ms on SIMT, profiles/r02i).
// From L = 11 both Gaunt products take the row-quad separable SIMT kernel (grid nodes / the reference
// torus): per 2^19 products 3.5 / 4.5 / 5.8 / 6.7 / 8.1 / 9.0 ms at L = 11..16 against 4.1 / 4.5
// (fused) / 30.8 / 40.1 (degree groups) on tcgen05 for the grid and 4.1 / 8.3 / 30.2 / 42.0 / 111 / 151
// for the Fourier GTP (profiles/r02s); below L = 11 the tcgen05 kernels win (L = 10: 2.0 vs 2.6).
// grid_path "tc" still takes the degree groups up to L = 14 (grid) / 16 (Fourier).
const int kGridSepMinL = [] {
  const char* v = std::getenv("TPO_GRID_SEP_MINL");
  return v ? std::atoi(v) : 11;
}();
const int kFourierSepMinL = [] {
  const char* v = std::getenv("TPO_FOURIER_SEP_MINL");
  return v ? std::atoi(v) : 11;
}();
constexpr int kMaxSplitL = 14;
const int kMaxSplitLFourier = [] {
  const char* v = std::getenv("TPO_FOURIER_SPLIT_MAXL");  // accuracy experiments only
  return v ? std::atoi(v) : 16;
}();
bool run_dense_split(tpo_ctx* ctx, int fourier, int L1, int L2, int L3, const RowSpec& rs, cudaStream_t s) {
  Context& c = ctx->impl;
  static const int kmax = [] {
    const char* v = std::getenv("TPO_GTP_SPLIT_K");
    return v ? std::max(16, std::min(176, std::atoi(v))) : 128;  // 128 vs 176: L=13 24.0 vs 36.6 ms
  }();
  auto groups_of = [](int L) {
    std::vector<std::pair<int, int>> gs;
    for (int a = 0; a <= L;) {
      int b = a;
      while (b + 1 <= L && (b + 2) * (b + 2) - a * a <= kmax) ++b;
      gs.push_back({a, b});
      a = b + 1;
    }
    return gs;
  };
  const auto g1 = groups_of(L1), g2 = groups_of(L2);
  auto fits_all = [&](const std::vector<std::pair<int, int>>& a, const std::vector<std::pair<int, int>>& b) {
    for (const auto& u : a)
      for (const auto& v : b)
        if (!c.dense_split_tc(fourier, L1, L2, L3, u.first, u.second, v.first, v.second).fits) return false;
    return true;
  };
  // (measured and dropped: y whole with x in the widest groups that fit beside it -- the wide K
  // forces narrow grid chunks: L=13 29.2 vs 24.4 ms, L=15 119 vs 86 ms)
  if (!fits_all(g1, g2)) return false;
  const int64_t rows = rs.rows, yrows = rs.y_shared ? rows / rs.channels : rows;
  const int64_t d1 = static_cast<int64_t>(L1 + 1) * (L1 + 1), d2 = static_cast<int64_t>(L2 + 1) * (L2 + 1);
  const int64_t dout = static_cast<int64_t>(L3 + 1) * (L3 + 1);
  auto width = [](const std::pair<int, int>& r) { return (r.second + 1) * (r.second + 1) - r.first * r.first; };
  int w1 = 0, w2 = 0;
  for (const auto& u : g1) w1 = std::max(w1, width(u));
  for (const auto& v : g2) w2 = std::max(w2, width(v));
  float *xw = nullptr, *yw = nullptr, *part = nullptr;
  if (g1.size() > 1) tpo_b200::cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&xw), rows * w1 * sizeof(float), s), "malloc");
  if (g2.size() > 1) tpo_b200::cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&yw), yrows * w2 * sizeof(float), s), "malloc");
  tpo_b200::cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&part), rows * dout * sizeof(float), s), "malloc");
  bool first = true;
  for (const auto& u : g1) {
    const float* xp = rs.x;
    if (g1.size() > 1) {
      launched(ctx, tpo_b200::launch_gather_cols(rs.x, d1, u.first * u.first, width(u), xw, rows, s), "gather x columns");
      xp = xw;
    }
    for (const auto& v : g2) {
      const float* yp = rs.y;
      if (g2.size() > 1) {
        launched(ctx, tpo_b200::launch_gather_cols(rs.y, d2, v.first * v.first, width(v), yw, yrows, s), "gather y columns");
        yp = yw;
      }
      RowSpec r = rs;
      r.x = xp;
      r.y = yp;
      r.out = first ? rs.out : part;
      launched(ctx, tpo_b200::launch_gtp_grid_tc(c.dense_split_tc(fourier, L1, L2, L3, u.first, u.second, v.first, v.second).t,
                                                 r, c.num_sms(), s),
               "gtp tcgen05 kernel (degree groups)");
      if (!first) launched(ctx, tpo_b200::launch_accumulate(part, rs.out, rows * dout, s), "accumulate");
      first = false;
    }
  }
  if (xw) cudaFreeAsync(xw, s);
  if (yw) cudaFreeAsync(yw, s);
  cudaFreeAsync(part, s);
  c.last_grid_path = 1;
  return true;
}

// L1 = L2 = 1 with L3 = 2: the small-degree SIMT kernel beats the 128-row tcgen05 pipeline
// (13.6 vs 19.6 us per 65,536, profiles/r02/grid_small.txt); grid_path "auto" only
bool run_small(tpo_ctx* ctx, int fourier, int L1, int L2, int L3, const RowSpec& rs, cudaStream_t s) {
  Context& c = ctx->impl;
  static const bool on = [] {
    const char* v = std::getenv("TPO_GTP_SMALL");
    return !(v && *v == '0');
  }();
  if (!on || c.grid_path != 0) return false;
  const tpo_b200::GtpSmallOps* o = c.gtp_small(fourier, L1, L2, L3);
  if (!o) return false;

  c.last_grid_path = 3;
  launched(ctx, tpo_b200::launch_gtp_small(*o, rs, c.num_sms(), s), fourier ? "gtp_fourier small kernel" : "gtp_grid small kernel");
  return true;
}

void run_grid(tpo_ctx* ctx, int L1, int L2, int L3, const RowSpec& rs, cudaStream_t s) {
  Context& c = ctx->impl;
  if (run_small(ctx, 0, L1, L2, L3, rs, s)) return;
  const bool sep_auto = c.grid_path == 0 && std::max(L1, L2) >= kGridSepMinL &&
                        tpo_b200::gtp_grid_quad_fits(c.grid_simt(L1, L2, L3));
  if (c.grid_path != 2 && c.grid_path != 3 && !sep_auto) {
    const auto& e = c.grid_tc(L1, L2, L3);
    if (e.fits) {
      c.last_grid_path = 1;
      launched(ctx, tpo_b200::launch_gtp_grid_tc(e.t, rs, c.num_sms(), s), "gtp_grid tcgen05 kernel");
      return;
    }
    if (std::max(L1, L2) > 12 && std::max(L1, L2) <= kMaxSplitL && run_dense_split(ctx, 0, L1, L2, L3, rs, s))
      return;
    if (c.grid_path == 1) throw InvalidArgument("gtp_grid: shape does not fit the tcgen05 tiling");
  }
  c.last_grid_path = 2;
  launched(ctx, tpo_b200::launch_gtp_grid_simt(c.grid_simt(L1, L2, L3), rs, c.num_sms(), s),
           "gtp_grid simt kernel");
}

// Fourier GTP: torus-grid dense operators on the tcgen05 kernel when the shape
// fits (Din <= 128), else the SIMT direct-convolution kernel
void run_fourier(tpo_ctx* ctx, int L1, int L2, int L3, const RowSpec& rs, cudaStream_t s) {
  Context& c = ctx->impl;
  if (run_small(ctx, 1, L1, L2, L3, rs, s)) return;
  if (c.grid_path == 3 || (c.grid_path == 0 && std::max(L1, L2) >= kFourierSepMinL)) {
    const tpo_b200::GridSimtTables* t = c.fourier_sep(L1, L2, L3);
    if (t && tpo_b200::gtp_grid_quad_fits(*t)) {
      c.last_grid_path = 4;
      launched(ctx, tpo_b200::launch_gtp_grid_simt(*t, rs, c.num_sms(), s), "gtp_fourier separable kernel");
      return;
    }
    if (c.grid_path == 3) throw InvalidArgument("gtp_fourier: the separable torus kernel does not take this shape");
  }
  if (c.grid_path != 2) {
    const auto& e = c.fourier_tc(L1, L2, L3);
    if (e.fits) {
      c.last_grid_path = 1;
      launched(ctx, tpo_b200::launch_gtp_grid_tc(e.t, rs, c.num_sms(), s), "gtp_fourier tcgen05 kernel");
      return;
    }
    if (std::max(L1, L2) > 12 && std::max(L1, L2) <= kMaxSplitLFourier && run_dense_split(ctx, 1, L1, L2, L3, rs, s))
      return;
    if (c.grid_path == 1) throw InvalidArgument("gtp_fourier: shape does not fit the tcgen05 tiling");
  }
  c.last_grid_path = 2;
  launched(ctx, tpo_b200::launch_gtp_fourier(c.fourier(L1, L2, L3), rs, c.num_sms(), s), "gtp_fourier kernel");
}

void run_kind(tpo_ctx* ctx, int kind, int L1, int L2, int L3, int lt, const float* x, const float* y,
              float* out, int64_t batch, int64_t channels, int y_shared, cudaStream_t s) {
  check_args(ctx, L1, L2, x, y, out, batch, channels);
  ctx->impl.activate();
  const RowSpec rs = rows_of(x, y, out, batch, channels, y_shared);
  switch (kind) {
    case TPO_KIND_CGTP:
      if (rs.rows > 0) run_cgtp(ctx, L1, L2, rs, s);
      return;
    case TPO_KIND_GTP_GRID:
      check_L3(L3, "gtp_grid");
      if (rs.rows > 0) run_grid(ctx, L1, L2, L3, rs, s);
      return;
    case TPO_KIND_GTP_FOURIER:
      check_L3(L3, "gtp_fourier");
      if (rs.rows > 0) run_fourier(ctx, L1, L2, L3, rs, s);
      return;
    case TPO_KIND_MTP: {
      check_L3(L3, "mtp");
      const int lmin = min_lt(L1, L2, L3);
      int l = lmin;
      if (lt >= 0) {
        if (lt < lmin) throw InvalidArgument("mtp: l_tilde below the minimal carrier degree");
        if (lt > kMaxL) throw InvalidArgument("mtp: l_tilde above the supported maximum");
        l = lt;
      }
      if (rs.rows > 0) {
        if (const tpo_b200::MtpTcTables* tc = ctx->impl.mtp_tc(L1, L2, L3, l))
          launched(ctx, tpo_b200::launch_mtp_tc(*tc, rs, ctx->impl.num_sms(), s), "mtp tcgen05 kernel");
        else
          launched(ctx, tpo_b200::launch_mtp(ctx->impl.mtp(L1, L2, L3, l), rs, ctx->impl.num_sms(), s),
                   "mtp kernel");
      }
      return;
    }
    default:
      throw InvalidArgument("tpo: unknown kind " + std::to_string(kind));
  }
}

int64_t out_dim(int kind, int L1, int L2, int L3) {
  if (L1 < 0 || L2 < 0) throw InvalidArgument("irreps: degree must be >= 0");
  if (kind == TPO_KIND_CGTP) return static_cast<int64_t>(L1 + 1) * (L1 + 1) * (L2 + 1) * (L2 + 1);
  if (kind < 0 || kind > TPO_KIND_MTP) throw InvalidArgument("tpo: unknown kind");
  if (L3 < 0) throw InvalidArgument("tpo: L3 must be >= 0");
  return static_cast<int64_t>(L3 + 1) * (L3 + 1);
}

}  // namespace

extern "C" {

const char* tpo_last_error(void) { return g_err.c_str(); }
const char* tpo_version(void) { return "tpo_b200 0.1 (sm_100a)"; }

int tpo_ctx_create(int device, tpo_ctx** out) {
  return guarded([&] {
    if (!out) throw InvalidArgument("tpo_ctx_create: null out pointer");
    *out = nullptr;
    *out = new tpo_ctx(device);
  });
}

int tpo_ctx_destroy(tpo_ctx* ctx) {
  return guarded([&] { delete ctx; });
}

int64_t tpo_ctx_launches(const tpo_ctx* ctx) { return ctx ? ctx->impl.launches.load() : -TPO_EINVAL; }

int64_t tpo_tower_dim(int L) { return L < 0 ? -TPO_EINVAL : static_cast<int64_t>(L + 1) * (L + 1); }

int64_t tpo_out_dim(int kind, int L1, int L2, int L3) {
  int64_t r = 0;
  const int st = guarded([&] { r = out_dim(kind, L1, L2, L3); });
  return st ? -st : r;
}

int tpo_mtp_l_tilde(int L1, int L2, int L3) { return min_lt(L1, L2, L3); }

int tpo_cgtp_mimo_f32(tpo_ctx* ctx, int L1, int L2, const float* x, const float* y, float* out, int64_t batch,
                      int64_t channels, int y_shared, void* stream) {
  return guarded([&] {
    run_kind(ctx, TPO_KIND_CGTP, L1, L2, 0, -1, x, y, out, batch, channels, y_shared,
             static_cast<cudaStream_t>(stream));
  });
}

int tpo_gtp_grid_f32(tpo_ctx* ctx, int L1, int L2, int L3, const float* x, const float* y, float* out,
                     int64_t batch, int64_t channels, int y_shared, void* stream) {
  return guarded([&] {
    run_kind(ctx, TPO_KIND_GTP_GRID, L1, L2, L3, -1, x, y, out, batch, channels, y_shared,
             static_cast<cudaStream_t>(stream));
  });
}

int tpo_gtp_fourier_f32(tpo_ctx* ctx, int L1, int L2, int L3, const float* x, const float* y, float* out,
                        int64_t batch, int64_t channels, int y_shared, void* stream) {
  return guarded([&] {
    run_kind(ctx, TPO_KIND_GTP_FOURIER, L1, L2, L3, -1, x, y, out, batch, channels, y_shared,
             static_cast<cudaStream_t>(stream));
  });
}

int tpo_mtp_f32(tpo_ctx* ctx, int L1, int L2, int L3, int l_tilde, const float* x, const float* y, float* out,
                int64_t batch, int64_t channels, int y_shared, void* stream) {
  return guarded([&] {
    run_kind(ctx, TPO_KIND_MTP, L1, L2, L3, l_tilde, x, y, out, batch, channels, y_shared,
             static_cast<cudaStream_t>(stream));
  });
}

int tpo_run_f32(tpo_ctx* ctx, int kind, int L1, int L2, int L3, int l_tilde, const float* x, const float* y,
                float* out, int64_t batch, int64_t channels, int y_shared, void* stream) {
  return guarded([&] {
    run_kind(ctx, kind, L1, L2, L3, l_tilde, x, y, out, batch, channels, y_shared,
             static_cast<cudaStream_t>(stream));
  });
}

int tpo_weighted_gtp_f32(tpo_ctx* ctx, int L1, int L2, int L3, const double* a, const double* b, const double* c,
                         const float* x, const float* y, float* out, int64_t batch, int64_t channels, int y_shared,
                         void* stream) {
  return guarded([&] {
    // proj/src/gtp.cpp:206-215: c (.) gtp(a (.) x, b (.) y)
    check_args(ctx, L1, L2, x, y, out, batch, channels);
    check_L3(L3, "weighted_gtp");
    if (!a || !b || !c) throw InvalidArgument("weighted_gtp: weight vector shorter than input degrees");
    ctx->impl.activate();
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t rows = batch * channels;
    if (rows == 0) return;
    // tcgen05 path: the weights ride in the kernel parameters, applied in the input
    // conversion and the epilogue (no extra passes, no temporaries)
    Context& c0 = ctx->impl;
    if (c0.grid_path != 2 && L1 <= 16 && L2 <= 16 && L3 <= 32) {
      const auto& e = c0.grid_tc(L1, L2, L3);
      if (e.fits && e.t.dout_eff <= 448) {  // per-column output weights: wtab_c[448] in the kernel
        tpo_b200::DegreeWeights dw{};
        dw.on = 1;
        for (int i = 0; i <= L1; ++i) dw.a[i] = static_cast<float>(a[i]);
        for (int i = 0; i <= L2; ++i) dw.b[i] = static_cast<float>(b[i]);
        for (int i = 0; i <= L3; ++i) dw.c[i] = static_cast<float>(c[i]);
        c0.last_grid_path = 1;
        launched(ctx, tpo_b200::launch_gtp_grid_tc(e.t, rows_of(x, y, out, batch, channels, y_shared), c0.num_sms(), s,
                                                   &dw),
                 "weighted gtp_grid tcgen05 kernel");
        return;
      }
    }
    const int64_t yrows = y_shared ? batch : rows;
    const int64_t d1 = (L1 + 1) * (L1 + 1), d2 = (L2 + 1) * (L2 + 1);
    float *xs = nullptr, *ys = nullptr, *wd = nullptr;
    const size_t nw = static_cast<size_t>(L1 + 1 + L2 + 1 + L3 + 1);
    tpo_b200::cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&xs), rows * d1 * sizeof(float), s), "malloc");
    tpo_b200::cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&ys), yrows * d2 * sizeof(float), s), "malloc");
    tpo_b200::cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&wd), nw * sizeof(float), s), "malloc");
    std::vector<float> wh;
    for (int i = 0; i <= L1; ++i) wh.push_back(static_cast<float>(a[i]));
    for (int i = 0; i <= L2; ++i) wh.push_back(static_cast<float>(b[i]));
    for (int i = 0; i <= L3; ++i) wh.push_back(static_cast<float>(c[i]));
    tpo_b200::cuda_check(cudaMemcpyAsync(wd, wh.data(), nw * sizeof(float), cudaMemcpyHostToDevice, s), "copy");
    tpo_b200::cuda_check(cudaStreamSynchronize(s), "sync");  // wh is pageable stack memory
    launched(ctx, tpo_b200::launch_scale_degrees(x, xs, rows, L1, wd, s), "scale");
    launched(ctx, tpo_b200::launch_scale_degrees(y, ys, yrows, L2, wd + L1 + 1, s), "scale");
    const RowSpec rs = rows_of(xs, ys, out, batch, channels, y_shared);
    run_grid(ctx, L1, L2, L3, rs, s);
    launched(ctx, tpo_b200::launch_scale_degrees(out, out, rows, L3, wd + L1 + 1 + L2 + 1, s), "scale");
    cudaFreeAsync(xs, s);
    cudaFreeAsync(ys, s);
    cudaFreeAsync(wd, s);
  });
}

namespace {
// grad (tower 0..Lr) = Gaunt contraction of grad_out (tower 0..L3) with the
// other input (tower 0..Lo), on the tcgen05 grid kernel: grad_out's degrees
// (those <= Lr + Lo; higher ones meet no Gaunt triangle) are cut into groups of
// <= 128 columns (the kernel's K limit), each group one launch on its smallest
// exact grid (Context::grid_tc_part), partial results summed.  Shapes the
// kernel cannot take go to the forward path with swapped operands (SIMT).
void gtp_vjp(tpo_ctx* ctx, int Lr, int Lo, int L3, const float* g, const float* other, float* res, int64_t batch,
             int64_t channels, int shared, cudaStream_t s) {
  Context& c = ctx->impl;
  const int64_t rows = batch * channels;
  const int Lg = std::min(L3, Lr + Lo);
  static const int kmax = [] {  // columns per group (the kernel takes K <= 176)
    const char* v = std::getenv("TPO_GTP_BWD_K");
    return v ? std::max(16, std::min(176, std::atoi(v))) : 176;  // 176 vs 128: L=6 0.170 vs 0.357 ms
  }();
  std::vector<std::pair<int, int>> groups;
  for (int a = 0; a <= Lg;) {
    int b = a;
    while (b + 1 <= Lg && (b + 2) * (b + 2) - a * a <= kmax) ++b;
    groups.push_back({a, b});
    a = b + 1;
  }
  // from Lr + Lo = 20 the swapped-operand forward on the row-quad separable kernel beats the degree
  // groups (65,536 products, both gradients: L = 10 1.33 vs 1.42 ms, L = 11 1.66 vs 2.17, L = 12 2.11
  // vs 3.62; L = 8 0.88 vs 0.66; profiles/r02s/bwd_paths.jsonl)
  bool tc = c.grid_path != 2 && !(c.grid_path == 0 && Lr + Lo >= 20);
  for (const auto& gr : groups)
    if (tc && !c.grid_tc_part(gr.first, gr.second, Lo, Lr).fits) tc = false;
  if (!tc || groups.empty()) {
    run_kind(ctx, TPO_KIND_GTP_GRID, L3, Lo, Lr, -1, g, other, res, batch, channels, shared, s);
    return;
  }
  const int64_t dg = static_cast<int64_t>(L3 + 1) * (L3 + 1), dr = static_cast<int64_t>(Lr + 1) * (Lr + 1);
  const bool direct = groups.size() == 1 && Lg == L3;  // grad_out rows are the operand as they are
  float* win = nullptr;
  float* part = nullptr;
  if (!direct) {
    int wmax = 0;
    for (const auto& gr : groups) wmax = std::max(wmax, (gr.second + 1) * (gr.second + 1) - gr.first * gr.first);
    tpo_b200::cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&win), rows * wmax * sizeof(float), s), "malloc");
    if (groups.size() > 1)
      tpo_b200::cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&part), rows * dr * sizeof(float), s), "malloc");
  }
  for (size_t i = 0; i < groups.size(); ++i) {
    const int a = groups[i].first, b = groups[i].second;
    const int64_t w = static_cast<int64_t>(b + 1) * (b + 1) - static_cast<int64_t>(a) * a;
    const float* op = g;
    if (!direct) {  // columns a^2 .. (b+1)^2 - 1 of every grad_out row, packed
      launched(ctx, tpo_b200::launch_gather_cols(g, dg, a * a, static_cast<int>(w), win, rows, s), "gather grad_out columns");
      op = win;
    }
    float* dst = i == 0 ? res : part;
    launched(ctx, tpo_b200::launch_gtp_grid_tc(c.grid_tc_part(a, b, Lo, Lr).t, rows_of(op, other, dst, batch, channels, shared),
                                               c.num_sms(), s),
             "gtp_grid tcgen05 kernel (backward)");
    if (i > 0) launched(ctx, tpo_b200::launch_accumulate(part, res, rows * dr, s), "accumulate");
  }
  if (win) cudaFreeAsync(win, s);
  if (part) cudaFreeAsync(part, s);
}
}  // namespace

namespace {
// MTP backward on the tcgen05 MTP kernel.  With P = (-1)^l per degree,
// grad_x = mtp(g, P y) and grad_y = mtp(P x, g) = P mtp(P g, x); the signs are
// folded into the embed / extract operators (Context::mtp_tc flags) and
// grad_out enters as input 1, cut by degree into groups of <= 64 columns (the
// kernel's K limit); degrees of grad_out above 2 l~ meet zero outputs and are
// skipped.  Returns false (nothing launched) when a shape does not fit.
bool mtp_vjp_tc(tpo_ctx* ctx, int L1, int L2, int L3, int lt, const float* x, const float* y, const float* g,
                float* gx, float* gy, int64_t batch, int64_t channels, int shared, cudaStream_t s) {
  Context& c = ctx->impl;
  const int64_t rows = batch * channels;
  const int Lg = std::min(L3, 2 * lt);
  // (input-2 degree, output degree, flags) per requested gradient
  struct Job { const float* other; int Lo, Lr, flags; float* res; int shared; };
  std::vector<Job> jobs;
  if (gx) jobs.push_back({y, L2, L1, 2, gx, shared});
  if (gy) jobs.push_back({x, L1, L2, 1 | 4, gy, 0});
  // grad_out degree windows as wide as the embed GEMM takes them (112 columns where the kernel's
  // shared memory allows, else 64): fewer launches, gathers and partial accumulations
  std::vector<std::pair<int, int>> groups;
  for (int kmax : {112, 64}) {
    groups.clear();
    for (int a = 0; a <= Lg;) {
      int b = a;
      while (b + 1 <= Lg && (b + 2) * (b + 2) - a * a <= kmax) ++b;
      groups.push_back({a, b});
      a = b + 1;
    }
    bool ok = true;
    for (const Job& j : jobs)
      for (const auto& gr : groups) ok = ok && c.mtp_tc(gr.second, j.Lo, j.Lr, lt, gr.first, j.flags) != nullptr;
    if (ok) break;
    if (kmax == 64) return false;
  }
  const int64_t dg = static_cast<int64_t>(L3 + 1) * (L3 + 1);
  const bool direct = groups.size() == 1 && Lg == L3;
  float* win = nullptr;
  float* part = nullptr;
  int64_t dr_max = 0;
  for (const Job& j : jobs) dr_max = std::max<int64_t>(dr_max, static_cast<int64_t>(j.Lr + 1) * (j.Lr + 1));
  if (!direct) {
    int wmax = 0;
    for (const auto& gr : groups) wmax = std::max(wmax, (gr.second + 1) * (gr.second + 1) - gr.first * gr.first);
    tpo_b200::cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&win), rows * wmax * sizeof(float), s), "malloc");
    if (groups.size() > 1)
      tpo_b200::cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&part), rows * dr_max * sizeof(float), s), "malloc");
  }
  for (size_t i = 0; i < groups.size(); ++i) {
    const int a = groups[i].first, b = groups[i].second;
    const int64_t w = static_cast<int64_t>(b + 1) * (b + 1) - static_cast<int64_t>(a) * a;
    const float* op = g;
    if (!direct) {  // columns a^2 .. (b+1)^2 - 1 of every grad_out row, packed
      launched(ctx, tpo_b200::launch_gather_cols(g, dg, a * a, static_cast<int>(w), win, rows, s), "gather grad_out columns");
      op = win;
    }
    for (const Job& j : jobs) {
      const int64_t dr = static_cast<int64_t>(j.Lr + 1) * (j.Lr + 1);
      float* dst = i == 0 ? j.res : part;
      launched(ctx, tpo_b200::launch_mtp_tc(*c.mtp_tc(b, j.Lo, j.Lr, lt, a, j.flags),
                                            rows_of(op, j.other, dst, batch, channels, j.shared), c.num_sms(), s),
               "mtp tcgen05 kernel (backward)");
      if (i > 0) launched(ctx, tpo_b200::launch_accumulate(part, j.res, rows * dr, s), "accumulate");
    }
  }
  if (win) cudaFreeAsync(win, s);
  if (part) cudaFreeAsync(part, s);
  return true;
}
}  // namespace

// Vector-Jacobian products (backward) of the four products; the reference has
// none (its paper benchmarks backward).
// Every product is bilinear, out_c = sum_ab W_abc x_a y_b, so
// grad_x_a = sum_bc W_abc y_b g_c and grad_y_b = sum_ac W_abc x_a g_c:
//  * GTP (grid / Fourier): W = real Gaunt coefficients, symmetric in (a, b, c),
//    hence grad_x = gtp(g, y; L3, L2 -> L1) and grad_y = gtp(g, x; L3, L1 -> L2)
//    -- the forward kernels on a grid of band L3 + L2 (exact quadrature);
//  * MTP: extract is the adjoint of embed and embed(v)^T = embed(P v) with
//    P = (-1)^l per degree, hence grad_x = mtp(g, P y) and grad_y = mtp(P x, g)
//    (carrier l~ of the forward; degree-parity pass on the other input);
//  * CGTP: transposed real-CG term lists (Context::cgtp_bwd, cgtp_bwd.cu),
//    grad_out swept in shared-memory windows, sums kept in registers.
// grad_x / grad_y may be null (not computed).  With a shared y (one per batch
// entry across channels) grad_y would be a channel reduction: not supported.
int tpo_backward_f32(tpo_ctx* ctx, int kind, int L1, int L2, int L3, int l_tilde, const float* x, const float* y,
                     const float* grad_out, float* grad_x, float* grad_y, int64_t batch, int64_t channels,
                     int y_shared, void* stream) {
  return guarded([&] {
    check_args(ctx, L1, L2, x, y, grad_out, batch, channels);
    if (y_shared && grad_y) throw InvalidArgument("backward: grad_y with a shared y (channel reduction) is not supported");
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t rows = batch * channels;
    ctx->impl.activate();
    Context& c = ctx->impl;
    switch (kind) {
      case TPO_KIND_CGTP: {
        if (rows == 0) return;
        // both gradients in one pass over grad_out on the tensor cores (cgtp_bwd_tc.cu); grad_out is
        // read through a [rows / 4][4 Dout] TMA view, so a ragged tail of < 4 rows and unaligned
        // buffers take the SIMT term-list kernel
        const tpo_b200::CgtpBwdTcTables* tc =
            !y_shared && (reinterpret_cast<uintptr_t>(grad_out) & 15) == 0 ? c.cgtp_bwd_tc(L1, L2) : nullptr;
        const int64_t rows4 = tc ? (rows & ~int64_t{3}) : 0;
        if (rows4 > 0) {
          const int64_t d1 = (L1 + 1) * (L1 + 1), d2 = (L2 + 1) * (L2 + 1), dout = d1 * d2;
          CUtensorMap tm;
          tpo_b200::encode_tmap_2d(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, grad_out, 4 * dout, rows4 / 4, 16 * dout, 36,
                                   32, CU_TENSOR_MAP_SWIZZLE_NONE);
          launched(ctx, tpo_b200::launch_cgtp_bwd_tc(*tc, x, y, grad_out, tm, grad_x, grad_y, rows4, c.num_sms(), s),
                   "cgtp backward tcgen05 kernel");
          if (rows4 == rows) return;
          const int64_t tail = rows - rows4;
          if (grad_x)
            launched(ctx, tpo_b200::launch_cgtp_bwd(c.cgtp_bwd(L1, L2, 0),
                                                    rows_of(grad_out + rows4 * dout, y + rows4 * d2, grad_x + rows4 * d1,
                                                            tail, 1, 0),
                                                    c.num_sms(), s),
                     "cgtp backward kernel");
          if (grad_y)
            launched(ctx, tpo_b200::launch_cgtp_bwd(c.cgtp_bwd(L1, L2, 1),
                                                    rows_of(grad_out + rows4 * dout, x + rows4 * d1, grad_y + rows4 * d2,
                                                            tail, 1, 0),
                                                    c.num_sms(), s),
                     "cgtp backward kernel");
          return;
        }
        if (grad_x)
          launched(ctx, tpo_b200::launch_cgtp_bwd(c.cgtp_bwd(L1, L2, 0), rows_of(grad_out, y, grad_x, batch, channels, y_shared),
                                                  c.num_sms(), s),
                   "cgtp backward kernel");
        if (grad_y)
          launched(ctx, tpo_b200::launch_cgtp_bwd(c.cgtp_bwd(L1, L2, 1), rows_of(grad_out, x, grad_y, batch, channels, 0),
                                                  c.num_sms(), s),
                   "cgtp backward kernel");
        return;
      }
      case TPO_KIND_GTP_GRID:
      case TPO_KIND_GTP_FOURIER: {
        check_L3(L3, "gtp backward");
        if (L3 > kMaxL) throw InvalidArgument("gtp backward: L3 above the supported input maximum");
        if (rows == 0) return;
        if (grad_x) gtp_vjp(ctx, L1, L2, L3, grad_out, y, grad_x, batch, channels, y_shared, s);
        if (grad_y) gtp_vjp(ctx, L2, L1, L3, grad_out, x, grad_y, batch, channels, 0, s);
        return;
      }
      case TPO_KIND_MTP: {
        check_L3(L3, "mtp backward");
        if (L3 > kMaxL) throw InvalidArgument("mtp backward: L3 above the supported input maximum");
        const int lmin = min_lt(L1, L2, L3);
        if (l_tilde >= 0 && l_tilde < lmin) throw InvalidArgument("mtp: l_tilde below the minimal carrier degree");
        const int lt = l_tilde >= 0 ? l_tilde : lmin;
        if (rows == 0) return;
        if (mtp_vjp_tc(ctx, L1, L2, L3, lt, x, y, grad_out, grad_x, grad_y, batch, channels, y_shared, s)) return;
        auto parity = [&](int L) {
          std::vector<double> w(L + 1);
          for (int l = 0; l <= L; ++l) w[l] = (l & 1) ? -1.0 : 1.0;
          return c.degree_weights(w);
        };
        if (grad_x) {
          const int64_t yrows = y_shared ? batch : rows;
          float* py = nullptr;
          tpo_b200::cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&py), std::max<int64_t>(yrows, 1) * (L2 + 1) * (L2 + 1) * sizeof(float), s), "malloc");
          launched(ctx, tpo_b200::launch_scale_degrees(y, py, yrows, L2, parity(L2), s), "parity");
          run_kind(ctx, TPO_KIND_MTP, L3, L2, L1, lt, grad_out, py, grad_x, batch, channels, y_shared, s);
          cudaFreeAsync(py, s);
        }
        if (grad_y) {
          float* px = nullptr;
          tpo_b200::cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&px), rows * (L1 + 1) * (L1 + 1) * sizeof(float), s), "malloc");
          launched(ctx, tpo_b200::launch_scale_degrees(x, px, rows, L1, parity(L1), s), "parity");
          run_kind(ctx, TPO_KIND_MTP, L1, L3, L2, lt, px, grad_out, grad_y, batch, channels, 0, s);
          cudaFreeAsync(px, s);
        }
        return;
      }
      default:
        throw InvalidArgument("backward: unknown kind");
    }
  });
}

namespace {
void cuda_check_s(cudaError_t e, const char* what) { tpo_b200::cuda_check(e, what); }
}  // namespace

namespace {
// Host buffers in, host buffers out, synchronous like the reference's call.  Each
// request's batch is cut into chunks that flow through three streams (copy-in,
// compute, copy-out) and kPipeBufs device buffer sets, so both PCIe directions and
// the kernels overlap (full overlap needs pinned host memory; pageable buffers still
// work, the copies are then staged by the driver).  Consecutive requests share the
// pipeline: it drains once, at the end.
void run_host_requests(tpo_ctx* ctx, const tpo_host_request* reqs, int n) {
  if (n < 0 || (n > 0 && !reqs)) throw InvalidArgument("tpo_run_host_batch: bad request list");
  struct Plan {
    int64_t d1, d2, dout, bc;
  };
  std::vector<Plan> plan(static_cast<size_t>(n));
  static const int64_t chunk_bytes = [] {
    const char* v = std::getenv("TPO_HOST_CHUNK_KB");
    return (v && *v) ? std::atoll(v) * 1024 : (32ll << 20);  // batch of the c2 sweep: 16 MiB 10.18 ms, 32 MiB 9.72 (tools/e2e_batch.py)
  }();
  size_t need_x = 1, need_y = 1, need_z = 1;
  for (int i = 0; i < n; ++i) {
    const tpo_host_request& q = reqs[i];
    check_args(ctx, q.L1, q.L2, q.x, q.y, q.out, q.batch, q.channels);
    // everything run_kind would reject is rejected here, before any chunk is queued
    if (q.kind != TPO_KIND_CGTP) check_L3(q.L3, "tpo_run_host");
    if (q.kind == TPO_KIND_MTP && q.l_tilde >= 0) {
      if (q.l_tilde < min_lt(q.L1, q.L2, q.L3))
        throw InvalidArgument("mtp: l_tilde below the minimal carrier degree");
      if (q.l_tilde > kMaxL) throw InvalidArgument("mtp: l_tilde above the supported maximum");
    }
    Plan& pl = plan[static_cast<size_t>(i)];
    pl.dout = out_dim(q.kind, q.L1, q.L2, q.L3);
    pl.d1 = (q.L1 + 1) * (q.L1 + 1);
    pl.d2 = (q.L2 + 1) * (q.L2 + 1);
    // chunk = whole batch entries (y_shared rows stay with their channels), ~16 MiB of traffic
    const int64_t bytes_per_b =
        4 * q.channels * (pl.d1 + pl.dout + (q.y_shared ? 0 : pl.d2)) + (q.y_shared ? 4 * pl.d2 : 0);
    pl.bc = std::min<int64_t>(std::max<int64_t>(1, chunk_bytes / std::max<int64_t>(bytes_per_b, 1)),
                              std::max<int64_t>(q.batch, 1));
    need_x = std::max(need_x, static_cast<size_t>(pl.bc * q.channels * pl.d1));
    need_y = std::max(need_y, static_cast<size_t>(pl.bc * (q.y_shared ? 1 : q.channels) * pl.d2));
    need_z = std::max(need_z, static_cast<size_t>(pl.bc * q.channels * pl.dout));
  }
  Context& c = ctx->impl;
  c.activate();
  std::lock_guard<std::mutex> lk(c.host_path_mutex());
  const int nb = Context::kPipeBufs;
  float* dx[Context::kPipeBufs];
  float* dy[Context::kPipeBufs];
  float* dz[Context::kPipeBufs];
  for (int b = 0; b < nb; ++b) {
    dx[b] = c.scratch(3 * b + 0, need_x);
    dy[b] = c.scratch(3 * b + 1, need_y);
    dz[b] = c.scratch(3 * b + 2, need_z);
  }
  const cudaStream_t si = c.h2d_stream(), sc = c.host_stream(), so = c.d2h_stream();
  // on any exception below, drain the three pipeline streams before returning: queued async copies
  // must not keep writing into the caller's buffers after the call reports its error
  struct Drain {
    cudaStream_t a, b, c;
    bool armed = true;
    ~Drain() {
      if (armed) {
        cudaStreamSynchronize(a);
        cudaStreamSynchronize(b);
        cudaStreamSynchronize(c);
      }
    }
  } drain{si, sc, so};
  // optional (TPO_HOST_RAMP=1) chunk ramp bc/8 .. bc .. bc/8 to shorten the unoverlapped first
  // copy-in / last copy-out; measured slower than uniform chunks (more per-chunk overhead)
  static const bool ramp = [] {
    const char* v = std::getenv("TPO_HOST_RAMP");
    return v && *v == '1';
  }();
  int64_t k = 0;  // chunk counter over all requests (buffer rotation)
  for (int i = 0; i < n; ++i) {
    const tpo_host_request& q = reqs[i];
    const Plan& pl = plan[static_cast<size_t>(i)];
    const int64_t rows = q.batch * q.channels;
    if (rows == 0) continue;
    const int64_t bc = pl.bc, bmin = std::max<int64_t>(1, bc / 8);
    auto next_chunk = [&](int64_t b0, int64_t kk) {
      const int64_t left = q.batch - b0;
      if (!ramp) return std::min(bc, left);
      int64_t sz = std::min(bc, bmin << std::min<int64_t>(kk, 3));  // ramp up
      if (left <= 2 * sz) sz = std::max(bmin, (left + 1) / 2);      // ramp down
      return std::min(sz, left);
    };
    int64_t kk = 0;
    for (int64_t b0 = 0, nbt = 0; b0 < q.batch; b0 += nbt, ++k, ++kk) {
      const int b = static_cast<int>(k % nb);
      nbt = next_chunk(b0, kk);
      const int64_t r0 = b0 * q.channels, nr = nbt * q.channels;
      const int64_t yr0 = q.y_shared ? b0 : r0, ynr = q.y_shared ? nbt : nr;
      if (k >= nb) cuda_check_s(cudaStreamWaitEvent(si, c.pipe_event(2, b), 0), "wait d2h");
      cuda_check_s(cudaMemcpyAsync(dx[b], q.x + r0 * pl.d1, nr * pl.d1 * sizeof(float), cudaMemcpyHostToDevice, si),
                   "H2D x");
      cuda_check_s(
          cudaMemcpyAsync(dy[b], q.y + yr0 * pl.d2, ynr * pl.d2 * sizeof(float), cudaMemcpyHostToDevice, si),
          "H2D y");
      cuda_check_s(cudaEventRecord(c.pipe_event(0, b), si), "record h2d");
      cuda_check_s(cudaStreamWaitEvent(sc, c.pipe_event(0, b), 0), "wait h2d");
      run_kind(ctx, q.kind, q.L1, q.L2, q.L3, q.l_tilde, dx[b], dy[b], dz[b], nbt, q.channels, q.y_shared, sc);
      cuda_check_s(cudaEventRecord(c.pipe_event(1, b), sc), "record compute");
      cuda_check_s(cudaStreamWaitEvent(so, c.pipe_event(1, b), 0), "wait compute");
      cuda_check_s(cudaMemcpyAsync(q.out + r0 * pl.dout, dz[b], nr * pl.dout * sizeof(float),
                                   cudaMemcpyDeviceToHost, so),
                   "D2H");
      cuda_check_s(cudaEventRecord(c.pipe_event(2, b), so), "record d2h");
    }
  }
  drain.armed = false;
  cuda_check_s(cudaStreamSynchronize(so), "sync");
  cuda_check_s(cudaStreamSynchronize(sc), "sync");
  cuda_check_s(cudaStreamSynchronize(si), "sync");
}
}  // namespace

int tpo_run_host_f32(tpo_ctx* ctx, int kind, int L1, int L2, int L3, int l_tilde, const float* x_host,
                     const float* y_host, float* out_host, int64_t batch, int64_t channels, int y_shared) {
  return guarded([&] {
    tpo_host_request q{};
    q.kind = kind;
    q.L1 = L1;
    q.L2 = L2;
    q.L3 = L3;
    q.l_tilde = l_tilde;
    q.y_shared = y_shared;
    q.batch = batch;
    q.channels = channels;
    q.x = x_host;
    q.y = y_host;
    q.out = out_host;
    run_host_requests(ctx, &q, 1);
  });
}

int tpo_run_host_batch_f32(tpo_ctx* ctx, const tpo_host_request* reqs, int n) {
  return guarded([&] { run_host_requests(ctx, reqs, n); });
}

int tpo_cg_real(int l1, int l2, int l3, int* m1, int* m2, int* m3, double* value, int cap) {
  int n = 0;
  const int st = guarded([&] {
    if (l1 < 0 || l2 < 0 || l3 < 0) throw InvalidArgument("cg_real: negative degree");
    if (l1 + l2 + l3 + 1 > 511) throw InvalidArgument("cg_real: degrees too large");
    const auto& t = tpo_b200::real_cg(l1, l2, l3);
    n = static_cast<int>(t.size());
    if (!m1) return;
    if (cap < n) throw InvalidArgument("cg_real: buffer too small");
    for (int i = 0; i < n; ++i) {
      m1[i] = t[i].m1;
      m2[i] = t[i].m2;
      m3[i] = t[i].m3;
      value[i] = t[i].v;
    }
  });
  return st ? -st : n;
}

int tpo_fourier_table(int L, int which, int* counts, int* u, int* v, double* re, double* im, int cap) {
  int total = 0;
  const int st = guarded([&] {
    if (L < 0 || L > kMaxL) throw InvalidArgument("fourier_tables: L out of range");
    const auto& t = tpo_b200::fourier_tables(L);
    const auto& modes = which == 0 ? t.enc : t.dec;
    for (size_t i = 0; i < modes.size(); ++i) {
      if (counts) counts[i] = static_cast<int>(modes[i].size());
      for (const auto& e : modes[i]) {
        if (u) {
          if (total >= cap) throw InvalidArgument("fourier_tables: buffer too small");
          u[total] = e.u;
          v[total] = e.v;
          re[total] = e.w.real();
          im[total] = e.w.imag();
        }
        ++total;
      }
    }
  });
  return st ? -st : total;
}

int tpo_set_gtp_grid_path(tpo_ctx* ctx, int path) {
  if (!ctx || path < 0 || path > 3) return -TPO_EINVAL;
  return ctx->impl.grid_path.exchange(path);
}

int tpo_last_gtp_grid_path(const tpo_ctx* ctx) { return ctx ? ctx->impl.last_grid_path.load() : -TPO_EINVAL; }

}  // extern "C"

// ------------------------------------------------------------------ stage operators
namespace {
std::vector<int> degree_list(const int* degrees, int n, const char* who) {
  if (n < 0 || (n > 0 && !degrees)) throw InvalidArgument(std::string(who) + ": bad degree list");
  std::vector<int> d(degrees, degrees + n);
  for (int l : d)
    if (l < 0 || l > 2 * kMaxL) throw InvalidArgument(std::string(who) + ": degree out of range");
  return d;
}
std::string key_of(const char* tag, std::initializer_list<int> a, const std::vector<int>& d = {}) {
  std::string k(tag);
  for (int v : a) k += "," + std::to_string(v);
  k += "|";
  for (int v : d) k += std::to_string(v) + ",";
  return k;
}
int dsel_of(const std::vector<int>& d) {
  int n = 0;
  for (int l : d) n += 2 * l + 1;
  return n;
}
void stage_args(const tpo_ctx* ctx, const void* in, const void* out, int64_t batch) {
  if (!ctx) throw InvalidArgument("tpo: null context");
  if (batch < 0) throw InvalidArgument("tpo: batch must be >= 0");
  if (batch > 0 && (!in || !out)) throw InvalidArgument("tpo: null data pointer");
}
}  // namespace

extern "C" {

int tpo_to_sphere_f32(tpo_ctx* ctx, int L, int grid_L, const float* x, float* F, int64_t batch, void* stream) {
  return guarded([&] {
    stage_args(ctx, x, F, batch);
    if (grid_L < 0 || grid_L > 2 * kMaxL) throw InvalidArgument("make_grid: L must be >= 0");
    if (L < 0) throw InvalidArgument("irreps: degree must be >= 0");
    if (L > grid_L)  // proj/src/sphere.cpp:106-110
      throw InvalidArgument("to_sphere: grid band limit " + std::to_string(grid_L) + " below input degree " +
                            std::to_string(L));
    ctx->impl.activate();
    const int din = (L + 1) * (L + 1), G = (grid_L + 1) * (2 * grid_L + 1);
    const float* mt = ctx->impl.dense_op(key_of("to_sphere", {L, grid_L}), [&] { return tpo_b200::op_to_sphere(L, grid_L); });
    launched(ctx, tpo_b200::launch_dense_map(x, din, mt, G, F, batch, static_cast<cudaStream_t>(stream)), "to_sphere");
  });
}

int tpo_from_sphere_f32(tpo_ctx* ctx, int grid_L, const int* degrees, int n_degrees, const float* F, float* out,
                        int64_t batch, void* stream) {
  return guarded([&] {
    stage_args(ctx, F, out, batch);
    if (grid_L < 0 || grid_L > 2 * kMaxL) throw InvalidArgument("make_grid: L must be >= 0");
    const std::vector<int> d = degree_list(degrees, n_degrees, "from_sphere");
    for (int l : d)  // proj/src/sphere.cpp:160-162
      if (l > grid_L) throw InvalidArgument("from_sphere: grid band limit too small for requested degree");
    ctx->impl.activate();
    const int G = (grid_L + 1) * (2 * grid_L + 1), ds = dsel_of(d);
    if (ds == 0) return;
    const float* mt = ctx->impl.dense_op(key_of("from_sphere", {grid_L}, d), [&] { return tpo_b200::op_from_sphere(grid_L, d); });
    launched(ctx, tpo_b200::launch_dense_map(F, G, mt, ds, out, batch, static_cast<cudaStream_t>(stream)), "from_sphere");
  });
}

int tpo_pointwise_mul_f32(tpo_ctx* ctx, const float* a, const float* b, float* out, int64_t n, void* stream) {
  return guarded([&] {
    stage_args(ctx, a, out, n);
    if (n > 0 && !b) throw InvalidArgument("tpo: null data pointer");
    ctx->impl.activate();
    launched(ctx, tpo_b200::launch_pointwise_mul(a, b, out, n, ctx->impl.num_sms(), static_cast<cudaStream_t>(stream)),
             "pointwise_mul");
  });
}

int tpo_mtp_embed_f32(tpo_ctx* ctx, int L, int l_tilde, const float* x, float* X, int64_t batch, void* stream) {
  return guarded([&] {
    stage_args(ctx, x, X, batch);
    if (l_tilde < 0) throw InvalidArgument("mtp_embed: l_tilde must be >= 0");  // proj/src/mtp.cpp:47-51
    if (L < 0) throw InvalidArgument("irreps: degree must be >= 0");
    if (L > 2 * l_tilde) throw InvalidArgument("mtp_embed: carrier too small for input degrees");
    if (l_tilde > kMaxL) throw InvalidArgument("mtp_embed: l_tilde above the supported maximum");
    ctx->impl.activate();
    const int din = (L + 1) * (L + 1), dt = 2 * l_tilde + 1;
    const float* mt = ctx->impl.dense_op(key_of("mtp_embed", {L, l_tilde}), [&] { return tpo_b200::op_mtp_embed(L, l_tilde); });
    launched(ctx, tpo_b200::launch_dense_map(x, din, mt, dt * dt, X, batch, static_cast<cudaStream_t>(stream)), "mtp_embed");
  });
}

int tpo_mtp_matmul_f32(tpo_ctx* ctx, int dt, const float* X, const float* Y, float* Z, int64_t batch, void* stream) {
  return guarded([&] {
    stage_args(ctx, X, Z, batch);
    if (batch > 0 && !Y) throw InvalidArgument("tpo: null data pointer");
    if (dt < 1 || dt > 2 * kMaxL + 1) throw InvalidArgument("mtp_matmul: carriers do not match");
    ctx->impl.activate();
    launched(ctx, tpo_b200::launch_carrier_matmul(X, Y, Z, dt, batch, static_cast<cudaStream_t>(stream)), "mtp_matmul");
  });
}

int tpo_mtp_extract_f32(tpo_ctx* ctx, int l_tilde, const int* degrees, int n_degrees, const float* Z, float* out,
                        int64_t batch, void* stream) {
  return guarded([&] {
    stage_args(ctx, Z, out, batch);
    if (l_tilde < 0 || l_tilde > kMaxL) throw InvalidArgument("mtp_extract: matrix does not match the carrier degree");
    const std::vector<int> d = degree_list(degrees, n_degrees, "mtp_extract");
    ctx->impl.activate();
    const int dt = 2 * l_tilde + 1, ds = dsel_of(d);
    if (ds == 0) return;
    const float* mt = ctx->impl.dense_op(key_of("mtp_extract", {l_tilde}, d), [&] { return tpo_b200::op_mtp_extract(l_tilde, d); });
    launched(ctx, tpo_b200::launch_dense_map(Z, dt * dt, mt, ds, out, batch, static_cast<cudaStream_t>(stream)),
             "mtp_extract");
  });
}

int tpo_apply_linear_f32(tpo_ctx* ctx, const int* in_mul, const int* in_l, int n_in, const int* out_mul,
                         const int* out_l, int n_out, const double* weights, int n_weights, const float* x, float* out,
                         int64_t batch, void* stream) {
  return guarded([&] {
    stage_args(ctx, x, out, batch);
    if (n_in < 0 || n_out < 0 || (n_in && (!in_mul || !in_l)) || (n_out && (!out_mul || !out_l)))
      throw InvalidArgument("linear layer: bad irreps descriptor");
    // proj/src/irreps.cpp:95-104: one weight per (input copy, output copy) of equal degree, in
    // (input entry, input copy, output entry, output copy) order
    std::vector<int> ioff(n_in + 1, 0), ooff(n_out + 1, 0);
    for (int e = 0; e < n_in; ++e) {
      if (in_mul[e] < 1 || in_l[e] < 0) throw InvalidArgument("irreps: bad entry");
      ioff[e + 1] = ioff[e] + in_mul[e] * (2 * in_l[e] + 1);
    }
    for (int e = 0; e < n_out; ++e) {
      if (out_mul[e] < 1 || out_l[e] < 0) throw InvalidArgument("irreps: bad entry");
      ooff[e + 1] = ooff[e] + out_mul[e] * (2 * out_l[e] + 1);
    }
    const int din = ioff[n_in], dout = ooff[n_out];
    std::vector<double> mt(static_cast<size_t>(din) * dout, 0.0);
    int w = 0;
    for (int ei = 0; ei < n_in; ++ei)
      for (int ci = 0; ci < in_mul[ei]; ++ci)
        for (int eo = 0; eo < n_out; ++eo) {
          if (out_l[eo] != in_l[ei]) continue;
          for (int co = 0; co < out_mul[eo]; ++co, ++w) {
            if (w >= n_weights) throw InvalidArgument("linear layer: expected more weights");
            const int d = 2 * in_l[ei] + 1;
            for (int m = 0; m < d; ++m)
              mt[static_cast<size_t>(ioff[ei] + ci * d + m) * dout + ooff[eo] + co * d + m] += weights[w];
          }
        }
    if (w != n_weights)
      throw InvalidArgument("linear layer: expected " + std::to_string(w) + " weights, got " + std::to_string(n_weights));
    ctx->impl.activate();
    if (dout == 0 || batch == 0) return;
    std::vector<float> f(mt.begin(), mt.end());
    float* dm = ctx->impl.scratch(Context::kScratchMisc, f.size());
    tpo_b200::cuda_check(cudaMemcpyAsync(dm, f.data(), f.size() * 4, cudaMemcpyHostToDevice, static_cast<cudaStream_t>(stream)),
             "linear weights");
    tpo_b200::cuda_check(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "linear weights");
    launched(ctx, tpo_b200::launch_dense_map(x, din, dm, dout, out, batch, static_cast<cudaStream_t>(stream)),
             "apply_linear");
  });
}

int tpo_wigner_d_f64(tpo_ctx* ctx, int L, const double* R, double* D, int64_t n, void* stream) {
  return guarded([&] {
    stage_args(ctx, R, D, n);
    if (L < 0) throw InvalidArgument("wigner_d: negative degree");
    if (L > tpo_b200::kWignerMaxL) throw InvalidArgument("wigner_d: degree above the supported maximum");
    ctx->impl.activate();
    const auto& w = ctx->impl.wigner(L);
    launched(ctx, tpo_b200::launch_wigner_d(w, R, D, n, static_cast<cudaStream_t>(stream)), "wigner_d");
  });
}

int64_t tpo_wigner_d_size(int L) {
  if (L < 0) return -TPO_EINVAL;
  int64_t n = 0;
  for (int l = 0; l <= L; ++l) n += static_cast<int64_t>(2 * l + 1) * (2 * l + 1);
  return n;
}

int tpo_rotate_f32(tpo_ctx* ctx, int L, const double* R, int64_t n_rot, const float* x, float* out, int64_t batch,
                   int64_t channels, void* stream) {
  return guarded([&] {
    stage_args(ctx, x, out, batch);
    if (L < 0 || L > tpo_b200::kWignerMaxL) throw InvalidArgument("rotate: degree out of range");
    if (channels < 1) throw InvalidArgument("tpo: channels must be >= 1");
    if (batch > 0 && (n_rot < 1 || n_rot > batch || !R)) throw InvalidArgument("rotate: need 1..batch rotations");
    if (batch == 0) return;
    ctx->impl.activate();
    const auto& w = ctx->impl.wigner(L);
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    double* D = nullptr;
    tpo_b200::cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&D), static_cast<size_t>(n_rot) * w.d_stride * 8, s),
             "rotate scratch");
    launched(ctx, tpo_b200::launch_wigner_d(w, R, D, n_rot, s), "wigner_d");
    launched(ctx, tpo_b200::launch_rotate(w, D, n_rot, x, out, batch, channels, ctx->impl.num_sms(), s), "rotate");
    tpo_b200::cuda_check(cudaFreeAsync(D, s), "rotate scratch");
  });
}

// ------------------------------------------------------------------ host tables
int tpo_gaunt_real(int l1, int l2, int l3, int* m1, int* m2, int* m3, double* value, int cap) {
  int n = 0;
  const int st = guarded([&] {
    if (l1 < 0 || l2 < 0 || l3 < 0) throw InvalidArgument("gaunt_real: negative degree");
    if (l1 + l2 + l3 > 2 * 2 * kMaxL) throw InvalidArgument("gaunt_real: degrees too large");
    const auto& t = tpo_b200::real_gaunt(l1, l2, l3);
    n = static_cast<int>(t.size());
    if (!m1) return;
    if (cap < n) throw InvalidArgument("gaunt_real: buffer too small");
    for (int i = 0; i < n; ++i) {
      m1[i] = t[i].m1;
      m2[i] = t[i].m2;
      m3[i] = t[i].m3;
      value[i] = t[i].v;
    }
  });
  return st ? -st : n;
}

int tpo_s2_grid(int L, double* cos_theta, double* weights) {
  return guarded([&] {
    if (L < 0) throw InvalidArgument("make_grid: L must be >= 0");
    if (L > 4 * kMaxL) throw InvalidArgument("make_grid: L above the supported maximum");
    const auto& g = tpo_b200::s2_grid(L);
    if (cos_theta) std::copy(g.nodes.begin(), g.nodes.end(), cos_theta);
    if (weights) std::copy(g.weights.begin(), g.weights.end(), weights);
  });
}

int tpo_legendre_lambda(int lmax, const double* cos_theta, int n, double* lam) {
  return guarded([&] {
    if (lmax < 0 || n < 0 || (n > 0 && (!cos_theta || !lam))) throw InvalidArgument("legendre_lambda: bad arguments");
    const std::vector<double> t = tpo_b200::legendre_lambda(lmax, std::vector<double>(cos_theta, cos_theta + n));
    std::copy(t.begin(), t.end(), lam);
  });
}

double tpo_mtp_path_weight(int l1, int l2, int l3, int l_tilde) {
  double w = 0.0;
  const int st = guarded([&] {
    if (l_tilde > kMaxL) throw InvalidArgument("mtp_path_weights: l_tilde above the supported maximum");
    w = tpo_b200::mtp_path_weight(l1, l2, l3, l_tilde);
  });
  return st ? std::nan("") : w;
}

int64_t tpo_count_muls(int kind, int impl, int mode, int L) {
  int64_t r = 0;
  const int st = guarded([&] {
    namespace oc = tpo_b200::opcount;
    // proj/src/bench.cpp:18-24,101-112: siso = path [L, L, L]; simo = degree-L inputs, outputs 0..2L;
    // mimo = single_copies(L) inputs, full output band
    if (L < 0) throw InvalidArgument("count_ops: L must be >= 0");
    if (mode < 0 || mode > 2) throw InvalidArgument("unknown mode");
    const bool naive = impl == 0;
    std::vector<oc::Entry> in;
    if (mode == 2)
      for (int l = 0; l <= L; ++l) in.push_back({1, l});
    else
      in.push_back({1, L});
    std::vector<int> ls;
    for (const auto& e : in) ls.push_back(e.l);
    std::vector<int> deg;
    if (mode == 0) deg = {L};
    else
      for (int l = 0; l <= 2 * L; ++l) deg.push_back(l);
    if (kind == 0) {  // cgtp: naive / sparse
      if (impl != 0 && impl != 1) throw InvalidArgument("count_ops: implementation does not apply to this kind");
      if (mode == 2) r = static_cast<int64_t>(oc::cgtp_mimo(naive, ls, ls));
      else
        for (int l3 = (mode == 1 ? 0 : L); l3 <= (mode == 1 ? 2 * L : L); ++l3) r += oc::cgtp_path(naive, L, L, l3);
    } else if (kind == 1) {  // gtp: grid / fourier
      if (impl != 2 && impl != 3) throw InvalidArgument("count_ops: implementation does not apply to this kind");
      r = static_cast<int64_t>(impl == 2 ? oc::gtp_grid_select(in, in, deg) : oc::gtp_fourier_select(in, in, deg));
    } else if (kind == 2) {  // mtp: naive / sparse
      if (impl != 0 && impl != 1) throw InvalidArgument("count_ops: implementation does not apply to this kind");
      const int lt = mode == 0 ? min_lt(L, L, L) : min_lt(L, L, 2 * L);
      r = static_cast<int64_t>(oc::mtp_embed(naive, in, lt) * 2 + oc::mtp_matmul(2 * lt + 1) +
                               oc::mtp_extract_select(naive, deg, lt));
    } else {
      throw InvalidArgument("unknown kind");
    }
  });
  return st ? -st : r;
}

}  // extern "C"

// ------------------------------------------------------------------ per-path weighted CGTP (f2)
namespace {
int num_paths(int L1, int L2) {
  int n = 0;
  for (int l1 = 0; l1 <= L1; ++l1)
    for (int l2 = 0; l2 <= L2; ++l2) n += 2 * std::min(l1, l2) + 1;
  return n;
}
}  // namespace

extern "C" {

int tpo_cgtp_num_paths(int L1, int L2) { return (L1 < 0 || L2 < 0) ? -TPO_EINVAL : num_paths(L1, L2); }

int tpo_cgtp_weighted_f32(tpo_ctx* ctx, int L1, int L2, const float* w, int w_per_edge, const float* x, const float* y,
                          float* out, int64_t batch, int64_t channels, int y_shared, void* stream) {
  return guarded([&] {
    check_args(ctx, L1, L2, x, y, out, batch, channels);
    if (batch > 0 && !w) throw InvalidArgument("cgtp_weighted: null weights");
    ctx->impl.activate();
    if (batch == 0) return;
    const int np = num_paths(L1, L2);
    const int* pof = ctx->impl.int_table("cgtp_path_of_out," + std::to_string(L1) + "," + std::to_string(L2), [&] {
      std::vector<int> v;  // output column -> path index, the reference's path order (proj/src/cgtp.cpp:152-163)
      int p = 0;
      for (int l1 = 0; l1 <= L1; ++l1)
        for (int l2 = 0; l2 <= L2; ++l2)
          for (int l3 = std::abs(l1 - l2); l3 <= l1 + l2; ++l3, ++p)
            for (int m = 0; m < 2 * l3 + 1; ++m) v.push_back(p);
      return v;
    });
    PathWeights pw{w, w_per_edge ? np : 0, pof};
    run_cgtp(ctx, L1, L2, rows_of(x, y, out, batch, channels, y_shared), static_cast<cudaStream_t>(stream), &pw);
  });
}

}  // extern "C"

extern "C" int tpo_set_precision(tpo_ctx* ctx, int mode) {
  if (!ctx || mode < 0 || mode > 1) return -TPO_EINVAL;
  return ctx->impl.precision_mode.exchange(mode);
}
