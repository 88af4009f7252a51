// Device-table construction: turns the fp64 host tables (tables.cpp) into
// the layouts the kernels consume.  See kernels/kernels.hpp for formats.
#include "context.hpp"

#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <complex>
#include <cstring>

#include "../kernels/sm100.cuh"
#include "tables.hpp"

namespace tpo_b200 {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaFailure(std::string(what) + ": " + cudaGetErrorString(e));
}

void encode_tmap_2d(CUtensorMap* m, CUtensorMapDataType dt, const void* base, uint64_t inner, uint64_t outer,
                    uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle sw) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (!encode) throw CudaFailure("cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {row_stride_bytes};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = encode(m, dt, 2, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaFailure("cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
}

namespace {
inline int pad_to(int v, int m) { return (v + m - 1) / m * m; }
inline int flat(int l, int m) { return l * l + m + l; }

void split_half(double v, uint16_t& hi, uint16_t& lo) {
  const __half h = __float2half_rn(static_cast<float>(v));
  const double rem = v - static_cast<double>(__half2float(h));
  const __half l = __float2half_rn(static_cast<float>(rem));
  std::memcpy(&hi, &h, 2);
  std::memcpy(&lo, &l, 2);
}
}  // namespace

Context::Context(int device) : device_(device) {
  int n = 0;
  cuda_check(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
  if (device < 0 || device >= n) throw InvalidArgument("tpo_ctx_create: no such CUDA device");
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  cudaDeviceProp prop{};
  cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
  if (prop.major != 10 || prop.minor != 0)  // the fatbin holds sm_100a SASS only (no PTX, no sm_103)
    throw CudaFailure("device is sm_" + std::to_string(prop.major) + std::to_string(prop.minor) +
                      "; this library is built for sm_100a (B200) only");
  num_sms_ = prop.multiProcessorCount;
  {  // stream-ordered temporaries (backward / weighted / degree-group passes) stay mapped between
     // calls up to 4 GiB (re-mapping them per call cost ~1.3 ms); larger pools shrink at syncs.
     // Note: this is the device's default pool, shared with the rest of the process (e.g. other
     // libraries' cudaMallocAsync), whose release threshold it raises to 4 GiB.
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = 4ull << 30;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  cuda_check(cudaStreamCreateWithFlags(&host_stream_, cudaStreamNonBlocking), "cudaStreamCreate");
  cuda_check(cudaStreamCreateWithFlags(&h2d_stream_, cudaStreamNonBlocking), "cudaStreamCreate");
  cuda_check(cudaStreamCreateWithFlags(&d2h_stream_, cudaStreamNonBlocking), "cudaStreamCreate");
  for (auto& row : pipe_ev_)
    for (auto& e : row) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
}

Context::~Context() {
  cudaSetDevice(device_);
  for (void* p : allocs_) cudaFree(p);
  for (void* p : scratch_)
    if (p) cudaFree(p);
  if (host_stream_) cudaStreamDestroy(host_stream_);
  if (h2d_stream_) cudaStreamDestroy(h2d_stream_);
  if (d2h_stream_) cudaStreamDestroy(d2h_stream_);
  for (auto& row : pipe_ev_)
    for (auto& e : row)
      if (e) cudaEventDestroy(e);
}

int& caller_device() {
  thread_local int dev = -1;
  return dev;
}

void Context::activate() const {
  int& prev = caller_device();
  if (prev < 0) {
    int cur = 0;
    if (cudaGetDevice(&cur) == cudaSuccess) prev = cur;
  }
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
}

void* Context::dev_alloc(size_t bytes) {
  void* p = nullptr;
  cuda_check(cudaMalloc(&p, std::max<size_t>(bytes, 16)), "cudaMalloc(table)");
  allocs_.push_back(p);
  return p;
}

template <class T>
T* Context::upload(const std::vector<T>& v) {
  void* p = dev_alloc(v.size() * sizeof(T));
  if (!v.empty()) {
    cuda_check(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "upload");
    // a pageable H2D cudaMemcpy may return once the data is staged, before the DMA lands, and
    // the kernels run on non-blocking streams that do not order after the legacy stream: wait
    // for the copy here (tables are built once per shape; an intermittent parity failure on
    // the first call of a new shape was traced to this)
    cuda_check(cudaStreamSynchronize(cudaStreamLegacy), "upload sync");
  }
  return static_cast<T*>(p);
}

float* Context::scratch(int slot, size_t floats) {
  const size_t bytes = std::max<size_t>(floats, 4) * sizeof(float);
  if (scratch_cap_[slot] < bytes) {
    if (scratch_[slot]) cudaFree(scratch_[slot]);
    scratch_[slot] = nullptr;
    cuda_check(cudaMalloc(&scratch_[slot], bytes), "cudaMalloc(scratch)");
    scratch_cap_[slot] = bytes;
  }
  return static_cast<float*>(scratch_[slot]);
}

// ------------------------------------------------------------------ CGTP
// Output layout = reference path order (x degree, y degree, l3 ascending),
// proj/src/cgtp.cpp:152-163; term lists from the real CG nonzeros.
namespace {
using TermList = std::vector<std::vector<std::pair<uint32_t, float>>>;  // per output: {i1 | i2 << 16, coef}

// CGTP term lists of every path, in the reference's output order
// (proj/src/cgtp.cpp:152-163): per_out[o] = {(i1, i2, c)} over the real-CG nonzeros
TermList cgtp_terms(int L1, int L2) {
  TermList per_out;
  for (int l1 = 0; l1 <= L1; ++l1)
    for (int l2 = 0; l2 <= L2; ++l2)
      for (int l3 = std::abs(l1 - l2); l3 <= l1 + l2; ++l3) {
        const size_t off = per_out.size();
        per_out.resize(off + 2 * l3 + 1);
        for (const CGEntry& e : real_cg(l1, l2, l3)) {
          const uint32_t i1 = flat(l1, e.m1), i2 = flat(l2, e.m2);
          per_out[off + e.m3 + l3].push_back({i1 | (i2 << 16), static_cast<float>(e.v)});
        }
      }
  return per_out;
}
}  // namespace

// Pack per-output term lists warp-major (kernels.hpp: CgtpTables) and upload.
CgtpTables Context::pack_cgtp(const std::vector<std::vector<std::pair<uint32_t, float>>>& per_out, int din1,
                              int din2) {
  const int dout = static_cast<int>(per_out.size());
  const int nchunks = (dout + kCgtpChunk - 1) / kCgtpChunk;
  const int nwarps = nchunks * kCgtpChunk / 32;
  std::vector<int> off(nwarps), nt(nwarps);
  std::vector<uint2> terms;
  for (int w = 0; w < nwarps; ++w) {
    int tmax = 0;
    for (int i = 0; i < 32; ++i) {
      const int o = w * 32 + i;
      if (o < dout) tmax = std::max<int>(tmax, static_cast<int>(per_out[o].size()));
    }
    off[w] = static_cast<int>(terms.size());
    nt[w] = tmax;
    terms.resize(terms.size() + static_cast<size_t>(tmax) * 32, make_uint2(0u, 0u));  // padding: coef 0
    for (int i = 0; i < 32; ++i) {
      const int o = w * 32 + i;
      if (o >= dout) continue;
      for (size_t k = 0; k < per_out[o].size(); ++k) {
        const float c = per_out[o][k].second;
        uint32_t cb;
        std::memcpy(&cb, &c, 4);
        terms[off[w] + k * 32 + i] = make_uint2(per_out[o][k].first, cb);
      }
    }
  }
  CgtpTables t{};
  t.din1 = din1;
  t.din2 = din2;
  t.dout = dout;
  t.nchunks = nchunks;
  t.terms = upload(terms);
  t.warp_off = upload(off);
  t.warp_nt = upload(nt);
  return t;
}

// Output layout = reference path order (x degree, y degree, l3 ascending),
// proj/src/cgtp.cpp:152-163; term lists from the real CG nonzeros.
const CgtpTables& Context::cgtp(int L1, int L2) {
  std::lock_guard<std::mutex> g(mu_);
  auto it = cgtp_.find({L1, L2});
  if (it != cgtp_.end()) return it->second;
  const CgtpTables t = pack_cgtp(cgtp_terms(L1, L2), (L1 + 1) * (L1 + 1), (L2 + 1) * (L2 + 1));
  return cgtp_.emplace(std::array<int, 2>{L1, L2}, t).first->second;
}

// CGTP backward tables (cgtp_bwd.cu).  With out[o] = sum_t c_t x[i1_t] y[i2_t]:
//   grad_x[a] = sum_{t: i1_t = a} c_t g[o_t] y[i2_t],  grad_y[b] = sum_{t: i2_t = b} c_t g[o_t] x[i1_t].
// Terms are grouped by (virtual output, grad_out window) and packed warp-major.
const CgtpBwdTables& Context::cgtp_bwd(int L1, int L2, int wrt) {
  std::lock_guard<std::mutex> g(mu_);
  auto it = cgtp_bwd_.find({L1, L2, wrt});
  if (it != cgtp_bwd_.end()) return it->second;
  const int din1 = (L1 + 1) * (L1 + 1), din2 = (L2 + 1) * (L2 + 1);
  const int dres = wrt == 0 ? din1 : din2, dother = wrt == 0 ? din2 : din1;
  const TermList fwd = cgtp_terms(L1, L2);
  const int dout = static_cast<int>(fwd.size());
  CgtpBwdTables t{};
  // window: up to 256 columns (tile 36 KB; measured 256 vs 480: L=4 0.66 vs 0.82 ms, L=8 15.7 vs 20.3 ms)
  const char* w_s = std::getenv("TPO_CGTP_BWD_W");  // A/B experiments only
  t.dwin = std::min(dout, w_s ? std::max(16, std::atoi(w_s)) : 256);
  t.nwin = (dout + t.dwin - 1) / t.dwin;
  t.dother = dother;
  t.dres = dres;
  const char* split_s = std::getenv("TPO_CGTP_BWD_SPLIT");  // A/B experiments only
  const int smax = std::max(1, kCgtpChunk / dres);
  t.nsplit = split_s ? std::max(1, std::min(std::atoi(split_s), smax)) : smax;
  const int nvirt = t.nsplit * dres;
  t.nchunks = (nvirt + kCgtpChunk - 1) / kCgtpChunk;
  t.g_stride = dout;
  // per (virtual output, window): {(o - w * dwin) | i_other << 16, c}
  std::vector<std::vector<std::vector<std::pair<uint32_t, float>>>> lists(
      nvirt, std::vector<std::vector<std::pair<uint32_t, float>>>(t.nwin));
  std::vector<int> count(dres, 0);
  for (int o = 0; o < dout; ++o)
    for (const auto& tm : fwd[o]) {
      const uint32_t i1 = tm.first & 0xFFFFu, i2 = tm.first >> 16;
      const int a = static_cast<int>(wrt == 0 ? i1 : i2);
      const uint32_t oth = wrt == 0 ? i2 : i1;
      const int v = (count[a]++ % t.nsplit) * dres + a;
      const int w = o / t.dwin;
      lists[v][w].push_back({static_cast<uint32_t>(o - w * t.dwin) | (oth << 16), tm.second});
    }
  const int nwarps = kCgtpChunk / 32;
  const char* ord_s = std::getenv("TPO_CGTP_BWD_ORDER");  // A/B experiments only
  const bool order_on = !(ord_s && *ord_s == '0');
  std::vector<int> off(static_cast<size_t>(t.nchunks) * t.nwin * nwarps), nt(off.size());
  std::vector<uint2> terms;
  for (int q = 0; q < t.nchunks; ++q)
    for (int w = 0; w < t.nwin; ++w)
      for (int wp = 0; wp < nwarps; ++wp) {
        const size_t idx = (static_cast<size_t>(q) * t.nwin + w) * nwarps + wp;
        int tmax = 0;
        for (int l = 0; l < 32; ++l) {
          const int v = q * kCgtpChunk + wp * 32 + l;
          if (v < nvirt) tmax = std::max<int>(tmax, static_cast<int>(lists[v][w].size()));
        }
        off[idx] = static_cast<int>(terms.size());
        nt[idx] = tmax;
        terms.resize(terms.size() + static_cast<size_t>(tmax) * 32, make_uint2(0u, 0u));  // padding: coef 0
        // step k of the 8 lanes of a quarter warp issue one LDS.128 each into the grad_out tile
        // (row io) and the other input (row iv): rows 4 banks apart, so lanes whose rows agree
        // mod 8 (and differ) conflict.  Greedy per step: each lane takes, among the next 16 of
        // its terms, the one adding the fewest conflicts (same row = broadcast, free)
        std::vector<std::vector<std::pair<uint32_t, float>>> rest(32);
        for (int l = 0; l < 32; ++l) {
          const int v = q * kCgtpChunk + wp * 32 + l;
          if (v < nvirt) rest[l] = lists[v][w];
        }
        for (int k = 0; k < tmax; ++k)
          for (int qq = 0; qq < 4; ++qq) {
            int cio[8] = {}, civ[8] = {};
            std::vector<uint32_t> rio, riv;
            for (int l = qq * 8; l < qq * 8 + 8; ++l) {
              auto& r = rest[l];
              if (r.empty()) continue;
              size_t best = 0;
              int bc = 1 << 30;
              for (size_t c = 0; c < std::min<size_t>(order_on ? 16 : 1, r.size()); ++c) {
                const uint32_t io = r[c].first & 0xFFFFu, iv = r[c].first >> 16;
                const bool sio = std::find(rio.begin(), rio.end(), io) != rio.end();
                const bool siv = std::find(riv.begin(), riv.end(), iv) != riv.end();
                const int cost = (sio ? 0 : cio[io & 7]) + (siv ? 0 : civ[iv & 7]);
                if (cost < bc) { bc = cost; best = c; }
              }
              const auto tm = r[best];
              r.erase(r.begin() + static_cast<long>(best));
              const uint32_t io = tm.first & 0xFFFFu, iv = tm.first >> 16;
              if (std::find(rio.begin(), rio.end(), io) == rio.end()) { rio.push_back(io); ++cio[io & 7]; }
              if (std::find(riv.begin(), riv.end(), iv) == riv.end()) { riv.push_back(iv); ++civ[iv & 7]; }
              uint32_t cb;
              std::memcpy(&cb, &tm.second, 4);
              terms[off[idx] + static_cast<size_t>(k) * 32 + l] = make_uint2(tm.first, cb);
            }
          }
      }
  t.terms = upload(terms);
  t.warp_off = upload(off);
  t.warp_nt = upload(nt);
  return cgtp_bwd_.emplace(std::array<int, 3>{L1, L2, wrt}, t).first->second;
}

// ------------------------------------------------------------------ GTP grid (tcgen05)
namespace {
int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return (v && *v) ? std::atoi(v) : dflt;
}
// tcgen05.mma cycles for one M = 128, K = 16 instruction of width N, as
// measured on B200 (tools/ubench/mma_ubench2.cu): single-thread issue floor
// ~45 cycles, math N / 2 cycles, and operands read from shared memory at
// ~128 B / cycle (A 4 KB + B 32 N bytes for an SS MMA; B only when A is in TMEM).
constexpr int kMaxRingStages = 8;
double mma_ss(int n) { return std::max({45.0, n / 2.0, (4096.0 + 32.0 * n) / 128.0}); }
double mma_ts(int n) { return std::max({45.0, n / 2.0, 32.0 * n / 128.0}); }
// the same per SM for a CTA pair (M = 256, one instruction for both SMs, each
// SM reads its own A and half of B)
double mma_ss_pair(int n) { return std::max({22.5, n / 2.0, (4096.0 + 16.0 * n) / 128.0}); }
double mma_ts_pair(int n) { return std::max({22.5, n / 2.0, 16.0 * n / 128.0}); }
// GEMM 2 N-split of a group of zg outputs (parts of <= 256 rows, multiple of
// 16).  Splitting is kept at 1: narrower MMAs leave too little slack over the
// issue floor to hide the per-stage mbarrier wait (tools/ubench/mma_ubench3.cu).
int parts_for(int zg) {
  int np = 1;
  while (zg / np > 256 || (zg % np) != 0 || ((zg / np) % 16) != 0) ++np;
  return np;
}
}  // namespace

// Dense operators of a "pointwise product" TPO on a point set of G points:
// out = A ((S1 x) .* (S2 y)).  Both the S2-grid GTP (Gauss-Legendre x uniform
// phi product grid) and the Fourier GTP (uniform torus grid, convolution
// theorem) have this form and run through the same tcgen05 kernel.
struct DenseOps {
  int G = 0, din1 = 0, din2 = 0, dout_eff = 0, dout_total = 0;
  bool same_s = false;
  std::vector<double> s1, s2;  // [G][din]
  std::vector<double> a;       // [dout_eff][G]
};

GridTcEntry Context::build_dense_tc(const DenseOps& ops, const char* label, int max_chain) {
  GridTcEntry ent;
  GridTcTables& t = ent.t;
  const int G = ops.G;
  t.din1 = ops.din1;
  t.din2 = ops.din2;
  t.k1p = pad_to(t.din1, 16);
  t.k2p = pad_to(t.din2, 16);
  t.dout_eff = ops.dout_eff;
  t.dout_total = ops.dout_total;
  t.same_s = ops.same_s ? 1 : 0;
  const int max_smem = gtp_grid_tc_max_smem(t.k1p > 128 || t.k2p > 128);
  if (t.k1p > 176 || t.k2p > 176 || max_smem <= 0) {  // SIMT kernels handle these shapes (kKHalfMax)
    ent.fits = false;
    return ent;
  }
  // ---- tiling: choose (output groups, chunk width) minimising estimated MMA cycles per tile
  //   TMEM: zg (Z) + 2 nc (F_x, F_y; P overwrites F_x) <= 512 columns
  const int force_nc = env_int("TPO_GRID_NC", 0), force_groups = env_int("TPO_GRID_GROUPS", 0);
  // CTA pairs are correct but slower inside this kernel (profiles/r01/ubench_summary.md): opt-in
  t.pair = env_int("TPO_GRID_PAIR", 0) && t.k1p <= 128 && t.k2p <= 128 ? 1 : 0;
  auto mss = [&](int n) { return t.pair ? mma_ss_pair(n) : mma_ss(n); };
  auto mts = [&](int n) { return t.pair ? mma_ts_pair(n) : mma_ts(n); };
  double best = 1e300;
  int best_g = 0, best_nc = 0, best_chunks = 0, best_zg = 0;
  for (int ng = 1; ng <= 8; ++ng) {
    if (force_groups && ng != force_groups) continue;
    // a group wider than one MMA (N <= 256) is split into GEMM-2 parts; wide single groups
    // avoid recomputing GEMM 1 per group at the price of narrower grid chunks
    int zg = pad_to((t.dout_eff + ng - 1) / ng, 16);
    if (zg > 256) zg = pad_to(zg, 32);
    if (zg > env_int("TPO_GRID_ZG_MAX", 448)) continue;
    for (int cand = 128; cand >= 16; cand -= 16) {
      if (force_nc && cand != force_nc) continue;
      if (zg + 2 * cand > 512) continue;
      const int nch = (G + cand - 1) / cand;
      const int nc = pad_to((G + nch - 1) / nch, 16);  // rebalance padding over chunks
      const int np = parts_for(zg);
      // in-place operands + two stages of each ring + epilogue staging must fit (K > 128 is tight)
      if (static_cast<int>(512u * (t.k1p + t.k2p) + 2u * 64u * (nc + zg / np) + 8u * 32u * 17u * 4u) > max_smem)
        continue;
      // + ~60 cycles per ring stage for the mbarrier wait when a stage's MMAs lack slack
      const double g1 = 3.0 * ((t.k1p + t.k2p) / 16) * mss(nc) +
                        ((t.k1p + t.k2p) / 16) * std::max(0.0, 60.0 - 3.0 * (mss(nc) - 45.0)) / (t.same_s ? 2 : 1);
      const double g2 = 3.0 * (nc / 16) * np * mts(zg / np);
      const double cost = ng * (nch * (g1 + g2 + 400.0) + 1500.0);
      if (cost < best) {
        best = cost;
        best_g = ng;
        best_nc = nc;
        best_chunks = nch;
        best_zg = zg;
      }
    }
  }
  if (best_g == 0) {
    ent.fits = false;
    return ent;
  }
  const int nc = best_nc;
  t.nc = nc;
  t.nchunks = best_chunks;
  t.nslices = nc / 16;
  t.ngroups = best_g;
  t.zg = best_zg;
  t.nparts = parts_for(t.zg);
  t.zp = t.zg / t.nparts;
  t.safe_war = env_int("TPO_GRID_SAFE_WAR", 1);
  {
    // GEMM-2 accumulation segments of <= ~20 K-steps (60 MMAs): tcgen05 accumulates in fp32 with
    // truncation once per MMA (a per-MMA round-toward-zero model reproduces the measured 1.04e-5 at
    // L = 12 to three digits; tools/precision_model.py), so one accumulator over the whole grid
    // (77 K-steps at L = 12) costs ~1e-5 normwise; segments added in fp32 keep it ~3-4e-6
    // Single accumulation while the chain is short enough for the operator family (max_chain K-steps,
    // measured on adversarial rows, profiles/r02d: grid operators <= 6.8e-6 at L = 10 (54 K-steps);
    // folded torus operators 3.6e-6 at L = 7 (<= 32 K-steps), 7.0e-6 / 9.9e-6 at L = 8 / 10);
    // segments cost a drain of Z per boundary (fp32 reductions in L2), ~25-45%, so they are used
    // only past those limits
    // segment length: 30 K-steps by default (two segments up to 60: torus L = 8-10; three for grid
    // L = 11, Fourier L = 11-12), 20 in strict mode
    const int seg_slices = std::max(1, env_int("TPO_GRID_SEG_SLICES", max_chain <= 20 ? 20 : 30));
    const int total = t.nchunks * t.nslices;
    const int nseg = total > env_int("TPO_GRID_MAX_CHAIN", max_chain) ? (total + seg_slices - 1) / seg_slices : 1;
    t.seg_chunks = std::max(1, (t.nchunks + nseg - 1) / nseg);
    if (t.seg_chunks < t.nchunks) t.pair = 0;  // CTA pairs are an opt-in single-segment experiment
  }
  // input scale: |F(g)| <= ||x||_2 ||S row g||_2, so ||x|| < 2^in_shift keeps P = F_x F_y < 2^14
  {
    auto row_norm_max = [&](const std::vector<double>& S, int din) {
      double m = 0.0;
      for (int gi = 0; gi < G; ++gi) {
        double ss = 0.0;
        for (int k = 0; k < din; ++k) ss += S[static_cast<size_t>(gi) * din + k] * S[static_cast<size_t>(gi) * din + k];
        m = std::max(m, std::sqrt(ss));
      }
      return m;
    };
    const double n1 = row_norm_max(ops.s1, t.din1), n2 = ops.same_s ? n1 : row_norm_max(ops.s2, t.din2);
    t.in_shift = std::max(0, std::min(12, static_cast<int>(std::floor((14.0 - std::log2(std::max(n1 * n2, 1e-30))) / 2))));
  }
  t.dbg = env_int("TPO_GRID_DBG", 0);

  // ---- shared memory: X/Y operands, optional separate raw staging, B ring, epilogue staging
  const uint32_t xy = 512u * (t.k1p + t.k2p);
  const uint32_t raw = static_cast<uint32_t>(pad_to(512 * (t.din1 + t.din2), 1024));
  // epilogue staging per worker warp: 32 x 17 floats
  const uint32_t epi = 8u * 32u * 17u * 4u;
  const int force_inplace = env_int("TPO_GRID_INPLACE", -1), force_stages = env_int("TPO_GRID_STAGES", 0);
  // two B-operand rings; prefer the separate raw staging buffer, then depth
  const int kp = t.pair ? 2 : 1;  // each CTA of a pair streams one row half of every slice
  t.s_stage_bytes = static_cast<uint32_t>(64 * nc / kp);
  t.a_stage_bytes = static_cast<uint32_t>(64 * t.zp / kp);
  auto fixed = [&](int ip) { return static_cast<int>(xy + (ip ? 0u : raw) + epi); };
  int inplace = -1, s_st = 0, a_st = 0;
  int best_score = -1;
  for (int ip = 0; ip <= 1; ++ip) {
    if (force_inplace >= 0 && ip != force_inplace) continue;
    const int room = max_smem - fixed(ip);
    for (int ss = 2; ss <= kMaxRingStages; ++ss)
      for (int sa = 2; sa <= kMaxRingStages; ++sa) {
        if (force_stages && (ss != force_stages || sa != force_stages)) continue;
        if (static_cast<int>(ss * t.s_stage_bytes + sa * t.a_stage_bytes) > room) continue;
        // shallowest ring first; the separate raw buffer (prefetch a whole tile ahead) breaks ties
        const int score = std::min(std::min(ss, sa), 4) * 100 + (ip == 0 ? 50 : 0) + ss + sa;
        if (score > best_score) {
          best_score = score;
          inplace = ip;
          s_st = ss;
          a_st = sa;
        }
      }
  }
  if (inplace < 0) {
    ent.fits = false;
    return ent;
  }
  t.raw_inplace = inplace;
  t.s_stages = s_st;
  t.a_stages = a_st;
  t.off_x = 0;
  t.off_y = 256u * t.k1p * 2u;
  uint32_t o = xy;
  t.off_raw = inplace ? t.off_x : o;
  if (!inplace) o += raw;
  t.off_sring = o;
  o += s_st * t.s_stage_bytes;
  t.off_aring = o;
  o += a_st * t.a_stage_bytes;
  t.off_stage = o;
  o += epi;
  t.smem_bytes = static_cast<int>(o);
  if (env_int("TPO_GRID_VERBOSE", 0))
    std::fprintf(stderr,
                 "[tpo] %s tcgen05 G=%d din=(%d,%d) dout=%d nc=%d chunks=%d groups=%d zg=%d parts=%d s_stages=%d "
                 "a_stages=%d inplace=%d pair=%d smem=%d seg_chunks=%d\n",
                 label, G, t.din1, t.din2, t.dout_eff, nc, t.nchunks, t.ngroups, t.zg, t.nparts, s_st, a_st, inplace,
                 t.pair, t.smem_bytes, t.seg_chunks);

  // ---- operators -> fp16 hi / lo slices in the UMMA canonical layout
  double amax = 0.0;
  for (double v : ops.a) amax = std::max(amax, std::abs(v));
  t.a_shift = amax > 0 ? 12 - (std::ilogb(amax) + 1) : 0;  // max |A| 2^a_shift in [2^11, 2^12)
  const double a_scale = std::ldexp(1.0, t.a_shift);

  // S slices: [chunk][kstep][hi | lo][nc x 16 canonical]
  // one slice = kp row halves, each [hi | lo][(nc / kp) x 16] canonical
  auto build_s = [&](const std::vector<double>& S, int din, int kpad, std::vector<uint16_t>& buf) {
    const int rh = nc / kp;                            // rows per half
    const size_t half = static_cast<size_t>(rh) * 16;  // elements per hi / lo block
    const int nks = kpad / 16;
    buf.assign(static_cast<size_t>(t.nchunks) * nks * 2 * nc * 16, 0);
    for (int c = 0; c < t.nchunks; ++c)
      for (int ks = 0; ks < nks; ++ks)
        for (int hh = 0; hh < kp; ++hh) {
          uint16_t* hi = buf.data() + (static_cast<size_t>(c) * nks + ks) * 2 * nc * 16 + hh * 2 * half;
          uint16_t* lo = hi + half;
          for (int r = 0; r < rh; ++r) {
            const int gidx = c * nc + hh * rh + r;
            for (int kk = 0; kk < 16; ++kk) {
              const int k = ks * 16 + kk;
              const double v = (gidx < G && k < din) ? S[static_cast<size_t>(gidx) * din + k] : 0.0;
              uint16_t hv, lv;
              split_half(v, hv, lv);
              const uint32_t e = sm100::canon_off(r, kk, rh) / 2;
              hi[e] = hv;
              lo[e] = lv;
            }
          }
        }
  };
  std::vector<uint16_t> s1, s2, a;
  build_s(ops.s1, t.din1, t.k1p, s1);
  t.s1_slice_bytes = static_cast<uint32_t>(64 * nc);
  t.s1 = reinterpret_cast<const uint8_t*>(upload(s1));
  if (t.same_s) {
    t.s2 = t.s1;
    t.s2_slice_bytes = t.s1_slice_bytes;
  } else {
    build_s(ops.s2, t.din2, t.k2p, s2);
    t.s2_slice_bytes = static_cast<uint32_t>(64 * nc);
    t.s2 = reinterpret_cast<const uint8_t*>(upload(s2));
  }
  // A slices: [group][chunk][slice][part][hi | lo][zp x 16 canonical]
  {
    const int rh = t.zp / kp;
    const size_t half = static_cast<size_t>(rh) * 16;
    a.assign(static_cast<size_t>(t.ngroups) * t.nchunks * t.nslices * t.nparts * 2 * t.zp * 16, 0);
    for (int gp = 0; gp < t.ngroups; ++gp)
      for (int c = 0; c < t.nchunks; ++c)
        for (int sl = 0; sl < t.nslices; ++sl)
          for (int pt = 0; pt < t.nparts; ++pt)
            for (int hh = 0; hh < kp; ++hh) {
              const size_t blk = ((static_cast<size_t>(gp) * t.nchunks + c) * t.nslices + sl) * t.nparts + pt;
              uint16_t* hi = a.data() + blk * 2 * t.zp * 16 + hh * 2 * half;
              uint16_t* lo = hi + half;
              for (int rr = 0; rr < rh; ++rr) {
                const int row = pt * t.zp + hh * rh + rr;  // output row within the group
                const int o2 = gp * t.zg + row;
                for (int kk = 0; kk < 16; ++kk) {
                  const int gidx = c * nc + sl * 16 + kk;
                  double v = 0.0;
                  if (gidx < G && o2 < t.dout_eff && row < t.zg) v = ops.a[static_cast<size_t>(o2) * G + gidx] * a_scale;
                  uint16_t hv, lv;
                  split_half(v, hv, lv);
                  const uint32_t e = sm100::canon_off(rr, kk, rh) / 2;
                  hi[e] = hv;
                  lo[e] = lv;
                }
              }
            }
    t.a_slice_bytes = static_cast<uint32_t>(64 * t.zp);
    t.a = reinterpret_cast<const uint8_t*>(upload(a));
  }
  if (t.pair) {
    // 2-D TMA views of the tables, [bytes / 64][64 B], one box = one half slice
    // (the cta_group::2 tensor copy signals the pair leader's barrier directly)
    auto make = [&](CUtensorMap* m, const void* base, size_t bytes, uint32_t box_rows) {
      encode_tmap_2d(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, base, 64, bytes / 64, 64, 64, box_rows,
                     CU_TENSOR_MAP_SWIZZLE_NONE);
    };
    make(&t.tm_s1, t.s1, s1.size() * 2, t.s_stage_bytes / 64);
    make(&t.tm_s2, t.s2, (t.same_s ? s1.size() : s2.size()) * 2, t.s_stage_bytes / 64);
    make(&t.tm_a, t.a, a.size() * 2, t.a_stage_bytes / 64);
  }
  ent.fits = true;
  return ent;
}

namespace {
DenseOps make_grid_ops(int L1, int L2, int L3) {
  // dense operators on the reference's product grid (proj/src/sphere.cpp:105-195, gtp.cpp:228-260)
  const int band = L1 + L2;
  const int L3e = std::min(L3, band);
  const S2Grid& gr = s2_grid(band);
  DenseOps ops;
  ops.G = gr.n_theta * gr.n_phi;
  ops.din1 = (L1 + 1) * (L1 + 1);
  ops.din2 = (L2 + 1) * (L2 + 1);
  ops.dout_eff = (L3e + 1) * (L3e + 1);
  ops.dout_total = (L3 + 1) * (L3 + 1);
  ops.same_s = L1 == L2;
  const double phi_scale = 2.0 * M_PI / gr.n_phi;
  auto s_val = [&](int gidx, int k) -> double {  // Lambda_{l|m|}(theta_j) cs_m(phi_k)
    const int j = gidx / gr.n_phi, kk = gidx % gr.n_phi;
    const int l = static_cast<int>(std::sqrt(static_cast<double>(k)) + 1e-9);
    const int m = k - l * l - l;
    return gr.lambda(l, std::abs(m), j) * gr.csm(m, kk);
  };
  ops.s1.resize(static_cast<size_t>(ops.G) * ops.din1);
  for (int gi = 0; gi < ops.G; ++gi)
    for (int k = 0; k < ops.din1; ++k) ops.s1[static_cast<size_t>(gi) * ops.din1 + k] = s_val(gi, k);
  if (!ops.same_s) {
    ops.s2.resize(static_cast<size_t>(ops.G) * ops.din2);
    for (int gi = 0; gi < ops.G; ++gi)
      for (int k = 0; k < ops.din2; ++k) ops.s2[static_cast<size_t>(gi) * ops.din2 + k] = s_val(gi, k);
  }
  ops.a.resize(static_cast<size_t>(ops.dout_eff) * ops.G);
  for (int o = 0; o < ops.dout_eff; ++o)  // quadrature weight w_j * 2 pi / n_phi
    for (int gi = 0; gi < ops.G; ++gi)
      ops.a[static_cast<size_t>(o) * ops.G + gi] = gr.weights[gi / gr.n_phi] * phi_scale * s_val(gi, o);
  return ops;
}
}  // namespace

const GridTcEntry& Context::grid_tc(int L1, int L2, int L3) {
  std::lock_guard<std::mutex> g(mu_);
  const int strict = precision_mode.load();
  auto it = grid_tc_.find({L1, L2, L3, strict});
  if (it != grid_tc_.end()) return it->second;
  return grid_tc_.emplace(std::array<int, 4>{L1, L2, L3, strict},
                          build_dense_tc(make_grid_ops(L1, L2, L3), "gtp_grid", strict ? 20 : 60))
      .first->second;
}

namespace {
DenseOps make_fourier_ops(int L1, int L2, int L3);
}  // namespace

const GtpSmallOps* Context::gtp_small(int fourier, int L1, int L2, int L3) {
  std::lock_guard<std::mutex> g(mu_);
  const std::array<int, 4> key{fourier, L1, L2, L3};
  auto it = gtp_small_.find(key);
  if (it == gtp_small_.end()) {
    SmallEntry e;
    if (L1 == L2 && L3 == L1 + L2 && L1 <= 1) {
      const DenseOps ops = fourier ? make_fourier_ops(L1, L2, L3) : make_grid_ops(L1, L2, L3);
      if (ops.same_s && gtp_small_supported(ops.din1, ops.G, ops.dout_eff)) {
        e.s.assign(ops.s1.begin(), ops.s1.end());
        e.a.assign(ops.a.begin(), ops.a.end());
        e.o.din = ops.din1;
        e.o.G = ops.G;
        e.o.dout_eff = ops.dout_eff;
        e.o.dout_total = ops.dout_total;
        e.ok = true;
      }
      if (std::getenv("TPO_VERBOSE"))
        std::fprintf(stderr, "[tpo] gtp small %s L=%d: din=%d G=%d dout=%d same_s=%d -> %s\n", fourier ? "fourier" : "grid",
                     L1, ops.din1, ops.G, ops.dout_eff, static_cast<int>(ops.same_s), e.ok ? "simt" : "tcgen05");
    }
    it = gtp_small_.emplace(key, std::move(e)).first;
    it->second.o.s = it->second.s.data();
    it->second.o.a = it->second.a.data();
  }
  return it->second.ok ? &it->second.o : nullptr;
}

// Forward GTP (grid or Fourier) with inputs wider than the kernel's K limit: the
// product is bilinear, so it is the sum over degree groups (x degrees [a1, b1],
// y degrees [a2, b2]) of the same operators restricted to those columns.
const GridTcEntry& Context::dense_split_tc(int fourier, int L1, int L2, int L3, int a1, int b1, int a2, int b2) {
  std::lock_guard<std::mutex> g(mu_);
  const std::array<int, 8> key{fourier, L1, L2, L3, a1, b1, a2, b2};
  auto it = dense_split_.find(key);
  if (it != dense_split_.end()) return it->second;
  DenseOps full = fourier ? make_fourier_ops(L1, L2, L3) : make_grid_ops(L1, L2, L3);
  if (full.same_s) full.s2 = full.s1;
  auto cols = [&](const std::vector<double>& S, int din, int a, int b) {
    const int c0 = a * a, w = (b + 1) * (b + 1) - c0;
    std::vector<double> out(static_cast<size_t>(full.G) * w);
    for (int gi = 0; gi < full.G; ++gi)
      for (int k = 0; k < w; ++k) out[static_cast<size_t>(gi) * w + k] = S[static_cast<size_t>(gi) * din + c0 + k];
    return out;
  };
  DenseOps ops = full;
  ops.s1 = cols(full.s1, full.din1, a1, b1);
  ops.s2 = cols(full.s2, full.din2, a2, b2);
  ops.din1 = (b1 + 1) * (b1 + 1) - a1 * a1;
  ops.din2 = (b2 + 1) * (b2 + 1) - a2 * a2;
  ops.same_s = false;
  return dense_split_.emplace(key, build_dense_tc(ops, fourier ? "gtp_fourier split" : "gtp_grid split", 30)).first->second;
}

// Backward operator set of the grid GTP (tpo_backward_f32): input 1 = degrees
// [a, b] of grad_out (its columns a^2 .. (b+1)^2 - 1), input 2 = the tower
// 0..L2 of the other input, output tower 0..Lo.  By the symmetry of the real
// Gaunt coefficients grad = sum_j w_j Y_o(j) G(j) F(j) with G the synthesis of
// those grad_out degrees: the integrand has degree <= Lo + L2 + b, so the
// smallest product grid that integrates it exactly has band
// ceil((Lo + L2 + b) / 2) (GL exact to 2 band + 1 in cos(theta), n_phi = 2 band + 1
// points exact to frequency 2 band) -- the forward's grid when b = Lo + L2.
const GridTcEntry& Context::grid_tc_part(int a, int b, int L2, int Lo) {
  std::lock_guard<std::mutex> g(mu_);
  const std::array<int, 4> key{a, b, L2, Lo};
  auto it = grid_tc_part_.find(key);
  if (it != grid_tc_part_.end()) return it->second;
  const int band = std::max({(Lo + L2 + b + 1) / 2, Lo, L2, b});
  const S2Grid& gr = s2_grid(band);
  DenseOps ops;
  ops.G = gr.n_theta * gr.n_phi;
  ops.din1 = (b + 1) * (b + 1) - a * a;
  ops.din2 = (L2 + 1) * (L2 + 1);
  ops.dout_eff = (Lo + 1) * (Lo + 1);
  ops.dout_total = ops.dout_eff;
  ops.same_s = false;
  const double phi_scale = 2.0 * M_PI / gr.n_phi;
  auto s_val = [&](int gidx, int k) -> double {
    const int j = gidx / gr.n_phi, kk = gidx % gr.n_phi;
    const int l = static_cast<int>(std::sqrt(static_cast<double>(k)) + 1e-9);
    const int m = k - l * l - l;
    return gr.lambda(l, std::abs(m), j) * gr.csm(m, kk);
  };
  ops.s1.resize(static_cast<size_t>(ops.G) * ops.din1);
  for (int gi = 0; gi < ops.G; ++gi)
    for (int k = 0; k < ops.din1; ++k) ops.s1[static_cast<size_t>(gi) * ops.din1 + k] = s_val(gi, a * a + k);
  ops.s2.resize(static_cast<size_t>(ops.G) * ops.din2);
  for (int gi = 0; gi < ops.G; ++gi)
    for (int k = 0; k < ops.din2; ++k) ops.s2[static_cast<size_t>(gi) * ops.din2 + k] = s_val(gi, k);
  ops.a.resize(static_cast<size_t>(ops.dout_eff) * ops.G);
  for (int o = 0; o < ops.dout_eff; ++o)
    for (int gi = 0; gi < ops.G; ++gi)
      ops.a[static_cast<size_t>(o) * ops.G + gi] = gr.weights[gi / gr.n_phi] * phi_scale * s_val(gi, o);
  return grid_tc_part_.emplace(key, build_dense_tc(ops, "gtp_grid backward", 30)).first->second;
}

// Fourier GTP on the tensor cores.  The reference convolves the two torus
// spectra directly (proj/src/gtp.cpp:290-301).  The product spectrum has band
// 2L per axis, so on a uniform N x N torus grid with N = 4L + 1 the
// convolution theorem is exact: cz = DFT_N(IDFT_N(cx) .* IDFT_N(cy)) / N^2.
// Folding encode into the inverse DFT and decode into the forward DFT gives
// two real dense operators (the torus functions of real inputs are real):
//   S[(a,b)][k] = Re sum_{(u,v,w) in enc_k} w w_N^(u a + v b),   w_N = exp(2 pi i / N)
//   A[o][(a,b)] = Re sum_{(U,V,w) in dec_o} w w_N^-(U a + V b) / N^2
namespace {
DenseOps make_fourier_ops(int L1, int L2, int L3) {
  // Torus of N = 4L + 2 points per axis (the reference's n, proj/src/gtp.cpp:58): the
  // product band 4L < N, so the cyclic convolution is exact.  The antipodal extension
  // (proj/src/gtp.cpp:66-74) makes every torus function of a sphere input satisfy
  // g(2 pi - theta, phi + pi) = g(theta, phi); with N even that pairs grid point
  // (a, b) with (N - a, b + N/2) (no fixed points), and the pointwise product keeps the
  // symmetry.  So both dense operators need one point per pair: S rows at the
  // representatives b < N/2, A columns summed over each pair -- G = N^2 / 2.
  const int L = std::max(L1, L2);
  const FourierTables& ft = fourier_tables(L);
  const int N = 4 * L + 2, H = N / 2;
  const int Lz = 2 * L;
  const int L3e = std::min(L3, Lz);
  DenseOps ops;
  ops.G = N * H;
  ops.din1 = (L1 + 1) * (L1 + 1);
  ops.din2 = (L2 + 1) * (L2 + 1);
  ops.dout_eff = (L3e + 1) * (L3e + 1);
  ops.dout_total = (L3 + 1) * (L3 + 1);
  ops.same_s = L1 == L2;
  std::vector<std::complex<double>> wn(N);
  for (int k = 0; k < N; ++k) wn[k] = std::polar(1.0, 2.0 * M_PI * k / N);
  auto modn = [N](long v) { return static_cast<int>(((v % N) + N) % N); };
  auto build_s = [&](int din, std::vector<double>& S) {  // row a * H + b: torus point (a, b), b < N/2
    S.assign(static_cast<size_t>(ops.G) * din, 0.0);
    for (int k = 0; k < din; ++k)
      for (const FourierMode& e : ft.enc[k])
        for (int a = 0; a < N; ++a)
          for (int b = 0; b < H; ++b)
            S[static_cast<size_t>(a * H + b) * din + k] +=
                (e.w * wn[modn(static_cast<long>(e.u) * a + static_cast<long>(e.v) * b)]).real();
  };
  build_s(ops.din1, ops.s1);
  if (!ops.same_s) build_s(ops.din2, ops.s2);
  ops.a.assign(static_cast<size_t>(ops.dout_eff) * ops.G, 0.0);
  const double inv = 1.0 / (static_cast<double>(N) * N);
  for (int o = 0; o < ops.dout_eff; ++o)
    for (const FourierMode& e : ft.dec[o])
      for (int a = 0; a < N; ++a)
        for (int b = 0; b < H; ++b) {
          const int a2 = modn(N - a), b2 = b + H;  // the paired point carries the same product value
          const long ph1 = static_cast<long>(e.u) * a + static_cast<long>(e.v) * b;
          const long ph2 = static_cast<long>(e.u) * a2 + static_cast<long>(e.v) * b2;
          ops.a[static_cast<size_t>(o) * ops.G + a * H + b] +=
              ((e.w * wn[modn(-ph1)]).real() + (e.w * wn[modn(-ph2)]).real()) * inv;
        }
  return ops;
}
}  // namespace

const GridTcEntry& Context::fourier_tc(int L1, int L2, int L3) {
  std::lock_guard<std::mutex> g(mu_);
  const int strict = precision_mode.load();
  auto it = fourier_tc_.find({L1, L2, L3, strict});
  if (it != fourier_tc_.end()) return it->second;
  return fourier_tc_.emplace(std::array<int, 4>{L1, L2, L3, strict},
                             build_dense_tc(make_fourier_ops(L1, L2, L3), "gtp_fourier", strict ? 20 : 36))
      .first->second;
}

// ------------------------------------------------------------------ GTP grid (SIMT separable)
// phi half-period tables and Legendre-analysis items of the row-quad separable kernel
// (gtp_grid_simt.cu) for t.band, t.L3e on an odd azimuth grid of np = 2 band + 1 points
void Context::fill_sep_tables(GridSimtTables& t, int np, const std::function<float(int, int)>& lam1_at,
                              const std::function<float(int, int)>& lam5_at) {
  t.nkp = t.band + 1;
  t.nkpp = (t.nkp + 3) / 4 * 4;
  t.mpad = (t.band + 1 + 3) / 4 * 4;
  std::vector<float> c2c((t.band + 1) * t.nkpp, 0.f), c2s((t.band + 1) * t.nkpp, 0.f), c4c(t.nkp * t.mpad, 0.f),
      c4s(t.nkp * t.mpad, 0.f);
  for (int kp = 0; kp < t.nkp; ++kp) {
    const double phi = 2.0 * M_PI * kp / np;
    for (int m = 0; m <= t.band; ++m) {
      c2c[m * t.nkpp + kp] = c4c[kp * t.mpad + m] = static_cast<float>(m == 0 ? 1.0 : std::cos(m * phi));
      c2s[m * t.nkpp + kp] = static_cast<float>(std::sin(m * phi));
      if (m < t.band) c4s[kp * t.mpad + m] = static_cast<float>(std::sin((m + 1) * phi));
    }
  }
  t.c2c = upload(c2c);
  t.c2s = upload(c2s);
  t.c4c = upload(c4c);
  t.c4s = upload(c4s);
  std::vector<int> it5;
  for (int m = -t.L3e; m <= t.L3e; ++m)
    for (int l0 = std::abs(m); l0 <= t.L3e; ++l0)
      if ((l0 - std::abs(m)) % 4 < 2) it5.push_back(l0 | ((m + t.L3e) << 16));
  t.nitems5 = static_cast<int>(it5.size());
  t.items5 = upload(it5);
  // the analysis weights of both degrees of every item, node-pair-major ([jp][item] float2): one
  // coalesced load per node pair for a warp of items
  const int njp = (t.nt + 1) / 2;
  std::vector<float> w5(static_cast<size_t>(njp) * t.nitems5 * 2, 0.f);
  for (int i = 0; i < t.nitems5; ++i) {
    const int l0 = it5[i] & 0xffff, ma = std::abs((it5[i] >> 16) - t.L3e), l1 = l0 + 2;
    for (int jp = 0; jp < njp; ++jp) {
      w5[(static_cast<size_t>(jp) * t.nitems5 + i) * 2] = lam5_at(l0 * (l0 + 1) / 2 + ma, jp);
      if (l1 <= t.L3e) w5[(static_cast<size_t>(jp) * t.nitems5 + i) * 2 + 1] = lam5_at(l1 * (l1 + 1) / 2 + ma, jp);
    }
  }
  t.lam5t = upload(w5);
  // synthesis values on the first-half nodes, rows padded to a multiple of 4 nodes (float4 loads)
  t.njp4 = (njp + 3) / 4 * 4;
  const int l1max = std::max(t.L1, t.L2), rows1 = (l1max + 1) * (l1max + 2) / 2;
  std::vector<float> w1(static_cast<size_t>(rows1) * t.njp4, 0.f);
  for (int r = 0; r < rows1; ++r)
    for (int jp = 0; jp < njp; ++jp) w1[static_cast<size_t>(r) * t.njp4 + jp] = lam1_at(r, jp);
  t.lam1q = upload(w1);
}

const GridSimtTables& Context::grid_simt(int L1, int L2, int L3) {
  std::lock_guard<std::mutex> g(mu_);
  auto it = grid_simt_.find({L1, L2, L3});
  if (it != grid_simt_.end()) return it->second;
  const int band = L1 + L2;
  const S2Grid& gr = s2_grid(band);
  GridSimtTables t{};
  t.L1 = L1;
  t.L2 = L2;
  t.band = band;
  t.L3e = std::min(L3, band);
  t.dout_total = (L3 + 1) * (L3 + 1);
  t.nt = gr.n_theta;
  t.np = gr.n_phi;
  std::vector<float> lam(gr.lam.begin(), gr.lam.end()), cs(gr.cs.begin(), gr.cs.end()), wq(gr.n_theta);
  for (int j = 0; j < gr.n_theta; ++j) wq[j] = static_cast<float>(gr.weights[j] * 2.0 * M_PI / gr.n_phi);
  t.lam = upload(lam);
  t.cs = upload(cs);
  t.wq = upload(wq);
  t.out_scale = 1.f;
  auto grl = [&](int row, int j) { return static_cast<float>(gr.lam[static_cast<size_t>(row) * t.nt + j]); };
  fill_sep_tables(t, gr.n_phi, grl, grl);
  return grid_simt_.emplace(std::array<int, 3>{L1, L2, L3}, t).first->second;
}

// ------------------------------------------------------------------ GTP Fourier
// Fourier GTP on the row-quad separable kernel.  The reference convolves the encoded torus spectra
// (proj/src/gtp.cpp:262-327) on a torus of N = 4L + 2 points per axis; by the convolution theorem the
// decoded product is out_o = sum_{a,b<N} h(a, b) A_o(a, b), h = f g the product of the torus
// functions f(a, phi) = Re sum_{(u,v,w) in enc} x w w_N^(u a) e^(i v phi) and
// A_o(a, b) = Re sum_{(U,V,w) in dec_o} w w_N^-(U a + V b) / N^2.  Every encode / decode entry of
// order m has |v| = |m|, so in phi both are single harmonics: f = sum_lm x_lm E_lm(a) trig_m(phi) and
// A_o(a, .) = D_o(a) trig_m(.) (trig_m = cos m phi for m >= 0, sin |m| phi for m < 0) -- the grid
// kernel's structure with E in place of Lambda_l|m|(theta_j) and D in place of w_j Lambda.  The phi
// stages run on the kernel's own odd azimuth grid (np = 2 (L1 + L2) + 1 points, exact for the product
// band: factor N / np), and the torus rows a > N/2 fold onto N - a (the antipodal extension,
// proj/src/gtp.cpp:66-74, makes the phi-harmonic m of row N - a (-1)^m times that of row a), leaving
// H + 1 = 2L + 2 rows theta_a = 2 pi a / N in [0, pi], which pair as a <-> H - a (theta <-> pi - theta)
// with parity (-1)^(l+m) as the Gauss-Legendre nodes do.  Every identity is checked on the tables
// (relative 1e-9; tools/fourier_sep_check.py restates the derivation against the oracle) and the
// builder returns nullptr if one fails.
const GridSimtTables* Context::fourier_sep(int L1, int L2, int L3) {
  std::lock_guard<std::mutex> g(mu_);
  auto it = fourier_sep_.find({L1, L2, L3});
  if (it != fourier_sep_.end()) return it->second.get();
  const int L = std::max(L1, L2);
  const FourierTables& ft = fourier_tables(L);
  const int N = 4 * L + 2, H = N / 2, nt = H + 1;
  auto t = std::make_unique<GridSimtTables>();
  t->L1 = L1;
  t->L2 = L2;
  t->band = L1 + L2;
  t->L3e = std::min(L3, t->band);
  t->dout_total = (L3 + 1) * (L3 + 1);
  t->nt = nt;
  t->np = 2 * t->band + 1;
  std::vector<std::complex<double>> wn(N);
  for (int k = 0; k < N; ++k) wn[k] = std::polar(1.0, 2.0 * M_PI * k / N);
  auto modn = [N](long v) { return static_cast<int>(((v % N) + N) % N); };
  bool ok = true;
  double vmax = 0.0, resid = 0.0;
  // one torus row's harmonic of (l, m): sign +1 encode (e^{+i}), -1 decode (e^{-i}, / N^2)
  auto harmonic = [&](const std::vector<FourierMode>& modes, int m, int sign, int a) {
    double cc = 0.0, ss = 0.0;
    for (const FourierMode& e : modes) {
      if (std::abs(e.v) != std::abs(m)) ok = false;
      const std::complex<double> c = e.w * wn[modn(sign * static_cast<long>(e.u) * a)];
      cc += c.real();
      const double im = sign > 0 ? -c.imag() : c.imag();  // sin |m| phi coefficient of the v = +|m| entry
      ss += e.v > 0 ? im : (e.v < 0 ? -im : 0.0);
    }
    resid = std::max(resid, std::abs(m >= 0 ? ss : cc));
    return m >= 0 ? cc : ss;
  };
  std::vector<double> E(static_cast<size_t>(L + 1) * (L + 1) * nt), Dq(static_cast<size_t>(t->L3e + 1) * (t->L3e + 1) * nt);
  for (int k = 0; k < (L + 1) * (L + 1); ++k) {
    const int l = static_cast<int>(std::sqrt(static_cast<double>(k) + 0.5)), m = k - l * l - l;
    for (int a = 0; a < nt; ++a) E[static_cast<size_t>(k) * nt + a] = harmonic(ft.enc[k], m, +1, a);
  }
  const double inv = 1.0 / (static_cast<double>(N) * N), phi_ratio = static_cast<double>(N) / t->np;
  std::vector<double> q(N);
  for (int o = 0; o < (t->L3e + 1) * (t->L3e + 1); ++o) {
    const int l = static_cast<int>(std::sqrt(static_cast<double>(o) + 0.5)), m = o - l * l - l;
    for (int a = 0; a < N; ++a) q[a] = harmonic(ft.dec[o], m, -1, a) * inv;
    const double sg = (std::abs(m) & 1) ? -1.0 : 1.0;
    for (int a = 0; a < nt; ++a)
      Dq[static_cast<size_t>(o) * nt + a] = phi_ratio * (q[a] + (a > 0 && a < H ? sg * q[N - a] : 0.0));
  }
  // pair parity a <-> H - a
  double pres = 0.0;
  auto pair_check = [&](const std::vector<double>& T, int lmax) {
    for (int k = 0; k < (lmax + 1) * (lmax + 1); ++k) {
      const int l = static_cast<int>(std::sqrt(static_cast<double>(k) + 0.5)), m = k - l * l - l;
      const double p = ((l + std::abs(m)) & 1) ? -1.0 : 1.0;
      for (int a = 0; a < nt; ++a) {
        const double v = T[static_cast<size_t>(k) * nt + a];
        vmax = std::max(vmax, std::abs(v));
        pres = std::max(pres, std::abs(T[static_cast<size_t>(k) * nt + (H - a)] - p * v));
      }
    }
  };
  double vE = 0.0;
  pair_check(E, L);
  vE = vmax;
  vmax = 0.0;
  pair_check(Dq, t->L3e);
  if (!ok || resid > 1e-9 * std::max(vE, vmax) * N || pres > 1e-9 * std::max(vE, vmax) * N) {
    fourier_sep_.emplace(std::array<int, 3>{L1, L2, L3}, nullptr);
    return nullptr;
  }
  // the kernel indexes both tables by |m| (row l (l + 1) / 2 + |m|): the cos- and sin-type rows of
  // one degree and |m| must agree
  double sres = 0.0;
  auto by_abs_m = [&](const std::vector<double>& T, int lmax) {
    std::vector<float> v(static_cast<size_t>(lmax + 1) * (lmax + 2) / 2 * nt, 0.f);
    for (int l = 0; l <= lmax; ++l)
      for (int ma = 0; ma <= l; ++ma)
        for (int a = 0; a < nt; ++a) {
          const double p = T[static_cast<size_t>(l * l + l + ma) * nt + a];
          sres = std::max(sres, std::abs(p - T[static_cast<size_t>(l * l + l - ma) * nt + a]));
          v[static_cast<size_t>(l * (l + 1) / 2 + ma) * nt + a] = static_cast<float>(p);
        }
    return v;
  };
  std::vector<float> Ef = by_abs_m(E, L), Df = by_abs_m(Dq, t->L3e), wq(nt, 1.f);
  if (sres > 1e-9 * std::max(vE, vmax) * N) {
    fourier_sep_.emplace(std::array<int, 3>{L1, L2, L3}, nullptr);
    return nullptr;
  }
  t->wq = upload(wq);
  t->lam = nullptr;
  t->cs = nullptr;
  t->out_scale = 1.f;
  fill_sep_tables(*t, t->np, [&](int row, int j) { return Ef[static_cast<size_t>(row) * nt + j]; },
                  [&](int row, int j) { return Df[static_cast<size_t>(row) * nt + j]; });
  return fourier_sep_.emplace(std::array<int, 3>{L1, L2, L3}, std::move(t)).first->second.get();
}

const FourierDevTables& Context::fourier(int L1, int L2, int L3) {
  std::lock_guard<std::mutex> g(mu_);
  auto it = fourier_.find({L1, L2, L3});
  if (it != fourier_.end()) return it->second;
  const int L = std::max(L1, L2);
  const FourierTables& ft = fourier_tables(L);
  const int w = 2 * L + 1, w2 = w * w;
  FourierDevTables t{};
  t.L = L;
  t.L1 = L1;
  t.L2 = L2;
  t.L3 = L3;
  auto enc = [&](int Lx, const int** off_out, const int** idx_out, const float2** w_out, int* n_out) {
    std::vector<std::vector<std::pair<int, float2>>> per_mode(w2);
    for (int l = 0; l <= Lx; ++l)
      for (int m = -l; m <= l; ++m)
        for (const FourierMode& e : ft.enc[flat(l, m)])
          per_mode[(e.u + L) * w + (e.v + L)].push_back(
              {flat(l, m), make_float2(static_cast<float>(e.w.real()), static_cast<float>(e.w.imag()))});
    std::vector<int> off(w2 + 1, 0), idx;
    std::vector<float2> wv;
    for (int md = 0; md < w2; ++md) {
      off[md] = static_cast<int>(idx.size());
      for (auto& p : per_mode[md]) {
        idx.push_back(p.first);
        wv.push_back(p.second);
      }
    }
    off[w2] = static_cast<int>(idx.size());
    *n_out = static_cast<int>(idx.size());
    *off_out = upload(off);
    *idx_out = upload(idx);
    *w_out = upload(wv);
  };
  enc(L1, &t.enc1_off, &t.enc1_idx, &t.enc1_w, &t.nenc1);
  enc(L2, &t.enc2_off, &t.enc2_idx, &t.enc2_w, &t.nenc2);
  // Hermitian half plane of the (4L+1)^2 product spectrum
  const int Lz = 2 * L, wz = 2 * Lz + 1;
  std::vector<int> hid(static_cast<size_t>(wz) * wz, -1);
  std::vector<int2> half;
  for (int V = 0; V <= Lz; ++V)
    for (int U = -Lz; U <= Lz; ++U) {
      if (V == 0 && U < 0) continue;
      hid[(U + Lz) * wz + (V + Lz)] = static_cast<int>(half.size());
      half.push_back(make_int2(U, V));
    }
  t.nhalf = static_cast<int>(half.size());
  t.half_uv = upload(half);
  const int L3e = std::min(L3, Lz);
  t.dout_eff = (L3e + 1) * (L3e + 1);
  t.dout_total = (L3 + 1) * (L3 + 1);
  std::vector<int> doff(t.dout_eff + 1, 0), didx;
  std::vector<float2> dw;
  for (int l = 0; l <= L3e; ++l)
    for (int m = -l; m <= l; ++m) {
      doff[flat(l, m)] = static_cast<int>(didx.size());
      for (const FourierMode& e : ft.dec[flat(l, m)]) {
        int code;
        const int h = hid[(e.u + Lz) * wz + (e.v + Lz)];
        if (h >= 0) {
          code = 2 * h;
        } else {
          code = 2 * hid[(-e.u + Lz) * wz + (-e.v + Lz)] + 1;
        }
        didx.push_back(code);
        dw.push_back(make_float2(static_cast<float>(e.w.real()), static_cast<float>(e.w.imag())));
      }
    }
  doff[t.dout_eff] = static_cast<int>(didx.size());
  t.dec_off = upload(doff);
  t.dec_idx = upload(didx);
  t.dec_w = upload(dw);
  return fourier_.emplace(std::array<int, 3>{L1, L2, L3}, t).first->second;
}

// ------------------------------------------------------------------ MTP
const MtpDevTables& Context::mtp(int L1, int L2, int L3, int lt) {
  std::lock_guard<std::mutex> g(mu_);
  auto it = mtp_.find({L1, L2, L3, lt});
  if (it != mtp_.end()) return it->second;
  const int dt = 2 * lt + 1, dt2 = dt * dt;
  MtpDevTables t{};
  t.lt = lt;
  t.dt = dt;
  t.dtp = (dt + 3) / 4 * 4;
  t.din1 = (L1 + 1) * (L1 + 1);
  t.din2 = (L2 + 1) * (L2 + 1);
  auto term = [](int idx, float c) {
    uint32_t cb;
    std::memcpy(&cb, &c, 4);
    return make_uint2(static_cast<uint32_t>(idx), cb);
  };
  // warp-interleaved term lists (see MtpDevTables): item i -> lane i % 32 of warp i / 32
  auto interleave = [&](const std::vector<std::vector<std::pair<int, float>>>& lists, const int2** idx_out,
                        const uint2** terms_out) {
    std::vector<int2> idx(lists.size());
    std::vector<uint2> terms;
    for (size_t w0 = 0; w0 < lists.size(); w0 += 32) {
      size_t nt = 0;
      for (size_t i = w0; i < std::min(lists.size(), w0 + 32); ++i) nt = std::max(nt, lists[i].size());
      const size_t base = terms.size();
      terms.resize(base + 32 * nt, make_uint2(0u, 0u));
      for (size_t i = w0; i < std::min(lists.size(), w0 + 32); ++i) {
        const size_t first = base + (i - w0);
        idx[i] = make_int2(static_cast<int>(first), static_cast<int>(lists[i].size()));
        for (size_t e = 0; e < lists[i].size(); ++e) terms[first + 32 * e] = term(lists[i][e].first, lists[i][e].second);
      }
    }
    *idx_out = upload(idx);
    *terms_out = upload(terms);
  };
  std::vector<std::vector<std::pair<int, float>>> cells(2 * dt2);
  for (int s2 = 0; s2 < 2; ++s2)
    for (int l = 0; l <= (s2 ? L2 : L1); ++l)  // proj/src/mtp.cpp:20-39
      for (const CGEntry& e : real_cg(lt, lt, l))
        cells[s2 * dt2 + (e.m1 + lt) * dt + (e.m2 + lt)].push_back({flat(l, e.m3), static_cast<float>(e.v)});
  interleave(cells, &t.emb_idx, &t.emb);
  const int L3e = std::min(L3, 2 * lt);  // beyond the carrier band: zero (mtp.cpp:126)
  t.dout_eff = (L3e + 1) * (L3e + 1);
  t.dout_total = (L3 + 1) * (L3 + 1);
  std::vector<std::vector<std::pair<int, float>>> outs(2 * t.dout_eff);
  for (int l3 = 0; l3 <= L3e; ++l3)
    for (const CGEntry& e : real_cg(lt, lt, l3)) {
      const std::pair<int, float> tm{(e.m1 + lt) * t.dtp + (e.m2 + lt), static_cast<float>(e.v)};
      outs[2 * flat(l3, e.m3)].push_back(tm);  // product half 0
      outs[2 * flat(l3, e.m3) + 1].push_back(tm);  // product half 1
    }
  interleave(outs, &t.ext_idx, &t.ext);
  return mtp_.emplace(std::array<int, 4>{L1, L2, L3, lt}, t).first->second;
}

// ------------------------------------------------------------------ CGTP, tcgen05 blocks
// W_{l1 l2}[o][k]: o = position of (l3, m3) inside the block (l3 ascending from
// |l1 - l2|, m3 = -l3..l3, the reference's path order, proj/src/cgtp.cpp:152-163),
// k = (m1 + l1)(2 l2 + 1) + m2 + l2; values = real CG (proj/src/wigner.cpp:114-151).
const CgtpTcTables* Context::cgtp_tc(int L1, int L2) {
  std::lock_guard<std::mutex> g(mu_);
  auto it = cgtp_tc_.find({L1, L2});
  if (it != cgtp_tc_.end()) return it->second.first ? &it->second.second : nullptr;
  auto fail = [&]() -> const CgtpTcTables* {
    cgtp_tc_.emplace(std::array<int, 2>{L1, L2}, std::make_pair(false, CgtpTcTables{}));
    return nullptr;
  };
  const char* env = std::getenv("TPO_CGTP_TC");
  // L <= 16: with the operands scaled into fp16's normal range the block path stays <= 2.6e-6
  // normwise on adversarial rows through L = 15 (profiles/r02i; before: 1.1-1.4e-5 at L = 15)
  static const int max_l = [] {
    const char* v = std::getenv("TPO_CGTP_TC_MAXL");  // A/B and accuracy experiments only
    return v ? std::atoi(v) : 16;
  }();
  if ((env && env[0] == '0') || L1 > std::min(max_l, 16) || L2 > std::min(max_l, 16)) return fail();
  CgtpTcTables t{};
  t.din1 = (L1 + 1) * (L1 + 1);
  t.din2 = (L2 + 1) * (L2 + 1);
  // per-row staging (y row + x_{l1} segment) takes most of shared memory at large L: the W ring
  // needs two stages of 64 * part-width bytes, so the block outputs are cut into narrower N parts
  // when 192-column parts do not fit (L = 16)
  std::vector<CgtpTcUnit> units;
  std::vector<uint16_t> w;
  int out_off = 0, max_npad = 16;
  // large y rows (din2 >= TPO_CGTP_YSEG_MIN, default 196: L2 >= 13) are staged per block instead of per
  // row: the freed shared memory buys 192-column parts and a deeper W ring (cgtp_tc.cu t.yseg)
  static const int yseg_min = [] {
    const char* v = std::getenv("TPO_CGTP_YSEG_MIN");
    return v ? std::atoi(v) : 196;
  }();
  t.yseg = t.din2 >= yseg_min ? 1 : 0;
  t.xy_pitch = t.yseg ? (33 + 8) | 1 : (t.din2 + 33 + 8) | 1;  // [y row |] x_{l1} (reads may run 7 past a y segment)
  const int xy_bytes = 128 * t.xy_pitch * 4 + (t.yseg ? 3 * 128 * 41 * 4 : 0);
  const int budget = 186 * 1024 - xy_bytes;  // the kernel's static staging takes ~35 KB
  int part_cols = kCgtpDCols;
  while (part_cols > 32 && budget / (64 * part_cols) < 2) part_cols -= 32;
  for (int l1 = 0; l1 <= L1; ++l1)
    for (int l2 = 0; l2 <= L2; ++l2) {
      const int n1 = 2 * l1 + 1, n2 = 2 * l2 + 1, n = n1 * n2;
      std::vector<double> W(static_cast<size_t>(n) * n, 0.0);
      int o0 = 0;
      for (int l3 = std::abs(l1 - l2); l3 <= l1 + l2; ++l3) {
        for (const CGEntry& e : real_cg(l1, l2, l3))
          W[static_cast<size_t>(o0 + e.m3 + l3) * n + (e.m1 + l1) * n2 + (e.m2 + l2)] += e.v;
        o0 += 2 * l3 + 1;
      }
      // K order k = m1 * n2p + m2 (n2p = n2 padded to 8; zero columns at the padding)
      const int n2p = pad_to(n2, 8), kw = n1 * n2p;
      const int kpad = pad_to(kw, 16), npad_all = pad_to(n, 16);
      const int parts = (npad_all + part_cols - 1) / part_cols;  // accumulators of <= 192 columns (cgtp_tc.cu kDCols)
      const int np = pad_to((n + parts - 1) / parts, 16);
      for (int p = 0; p < parts; ++p) {
        CgtpTcUnit u{};
        u.l1 = l1;
        u.l2 = l2;
        u.out_off = out_off + p * np;
        u.n_valid = std::min(np, n - p * np);
        u.n_pad = pad_to(u.n_valid, 16);
        u.ksteps = kpad / 16;
        u.w_off = static_cast<int>(w.size() * 2);
        max_npad = std::max(max_npad, u.n_pad);
        const size_t base = w.size();
        w.resize(base + static_cast<size_t>(u.ksteps) * 2 * u.n_pad * 16, 0);
        for (int ks = 0; ks < u.ksteps; ++ks) {
          uint16_t* hi = w.data() + base + static_cast<size_t>(ks) * 2 * u.n_pad * 16;
          uint16_t* lo = hi + u.n_pad * 16;
          for (int r = 0; r < u.n_valid; ++r)
            for (int kk = 0; kk < 16; ++kk) {
              const int k = ks * 16 + kk, m1 = k / n2p, m2 = k % n2p;
              if (k >= kw || m2 >= n2) continue;
              uint16_t hv, lv;
              split_half(std::ldexp(W[static_cast<size_t>(p * np + r) * n + m1 * n2 + m2], kTabShift), hv, lv);
              const uint32_t o = sm100::canon_off(r, kk, u.n_pad) / 2;
              hi[o] = hv;
              lo[o] = lv;
            }
        }
        units.push_back(u);
      }
      out_off += n;
    }
  // super-units: consecutive units packed into one accumulator (kCgtpDCols columns)
  for (size_t i = 0, col = 0; i < units.size(); ++i) {
    if (col + units[i].n_pad > kCgtpDCols) {
      units[i - 1].dcol_last |= 1 << 16;
      col = 0;
    }
    units[i].dcol_last = static_cast<int>(col);
    col += units[i].n_pad;
  }
  units.back().dcol_last |= 1 << 16;
  t.dout = out_off;
  t.nunits = static_cast<int>(units.size());
  t.units = upload(units);
  t.w = reinterpret_cast<const uint8_t*>(upload(w));
  // shared memory: A ring (8 KB stages) | W ring | per-row x | y staging (odd pitch)
  t.b_stage_bytes = 64 * max_npad;
  t.a_stages = kCgtpAStages;  // the P ring lives in TMEM (cgtp_tc.cu kAStagesTmem)
  t.b_stages = std::min(8, budget / t.b_stage_bytes);
  if (t.b_stages < 2) return fail();
  t.off_a = 0;
  t.off_b = 0;
  t.off_xy = t.off_b + t.b_stages * t.b_stage_bytes;
  t.smem_bytes = t.off_xy + xy_bytes;
  if (std::getenv("TPO_VERBOSE"))
    std::fprintf(stderr, "[tpo] cgtp tcgen05 L=(%d,%d) units=%d dout=%d w=%zu B stages a=%d b=%d smem=%d\n", L1, L2,
                 t.nunits, t.dout, w.size() * 2, t.a_stages, t.b_stages, t.smem_bytes);
  return &cgtp_tc_.emplace(std::array<int, 2>{L1, L2}, std::make_pair(true, t)).first->second.second;
}

// CGTP backward blocks (cgtp_bwd_tc.cu): the transposed block W^T[k][o] with k unpadded,
// k = (m1 + l1)(2 l2 + 1) + m2 + l2, o in the forward's path order.  The kernel keeps the row's
// x | y and grad_x | grad_y in shared memory beside the grad_out and W^T rings, which bounds it to
// din1 + din2 <= 128 (L <= 7); shapes whose blocks fit one accumulator hand-off per tile (L1 + L2 <= 4
// or so) are faster on the SIMT kernel.
const CgtpBwdTcTables* Context::cgtp_bwd_tc(int L1, int L2) {
  const char* env = std::getenv("TPO_CGTP_BWD_TC");  // "0": the SIMT kernel (A/B and tests; read per call)
  if (env && env[0] == '0') return nullptr;
  std::lock_guard<std::mutex> g(mu_);
  auto it = cgtp_bwd_tc_.find({L1, L2});
  if (it != cgtp_bwd_tc_.end()) return it->second.first ? &it->second.second : nullptr;
  auto fail = [&]() -> const CgtpBwdTcTables* {
    cgtp_bwd_tc_.emplace(std::array<int, 2>{L1, L2}, std::make_pair(false, CgtpBwdTcTables{}));
    return nullptr;
  };
  if (L1 > 8 || L2 > 8) return fail();
  CgtpBwdTcTables t{};
  t.one_sided = (L1 > 7 || L2 > 7) ? 1 : 0;
  t.din1 = (L1 + 1) * (L1 + 1);
  t.din2 = (L2 + 1) * (L2 + 1);
  t.nblocks = (L1 + 1) * (L2 + 1);
  std::vector<CgtpBwdTcUnit> units;
  std::vector<uint16_t> w;
  int g_off = 0, max_npad = 16;
  for (int l1 = 0; l1 <= L1; ++l1)
    for (int l2 = 0; l2 <= L2; ++l2) {
      const int n1 = 2 * l1 + 1, n2 = 2 * l2 + 1, n = n1 * n2;
      std::vector<double> W(static_cast<size_t>(n) * n, 0.0);  // W[o][k]
      int o0 = 0;
      for (int l3 = std::abs(l1 - l2); l3 <= l1 + l2; ++l3) {
        for (const CGEntry& e : real_cg(l1, l2, l3))
          W[static_cast<size_t>(o0 + e.m3 + l3) * n + (e.m1 + l1) * n2 + (e.m2 + l2)] += e.v;
        o0 += 2 * l3 + 1;
      }
      // N parts of <= 192 accumulator columns made of whole rows m1 of Q (k = m1 n2 + m2)
      const int rpp = std::min(n1, 192 / n2), parts = (n1 + rpp - 1) / rpp;
      for (int p = 0; p < parts; ++p) {
        CgtpBwdTcUnit u{};
        u.l1 = l1;
        u.l2 = l2;
        u.blk = l1 * (L2 + 1) + l2;
        u.g_off = g_off;
        u.n = n;
        u.m1b = p * rpp;
        u.nrows = std::min(rpp, n1 - p * rpp);
        u.k0 = u.m1b * n2;
        u.n_valid = u.nrows * n2;
        u.n_pad = pad_to(u.n_valid, 16);
        u.ksteps = pad_to(n, 16) / 16;
        u.w_off = static_cast<int>(w.size() * 2);
        max_npad = std::max(max_npad, u.n_pad);
        const size_t base = w.size();
        w.resize(base + static_cast<size_t>(u.ksteps) * 2 * u.n_pad * 16, 0);
        for (int ks = 0; ks < u.ksteps; ++ks) {
          uint16_t* hi = w.data() + base + static_cast<size_t>(ks) * 2 * u.n_pad * 16;
          uint16_t* lo = hi + u.n_pad * 16;
          for (int r = 0; r < u.n_valid; ++r)
            for (int kk = 0; kk < 16; ++kk) {
              const int o = ks * 16 + kk;
              if (o >= n) continue;
              uint16_t hv, lv;
              split_half(std::ldexp(W[static_cast<size_t>(o) * n + u.k0 + r], kTabShift), hv, lv);
              const uint32_t off = sm100::canon_off(r, kk, u.n_pad) / 2;
              hi[off] = hv;
              lo[off] = lv;
            }
        }
        units.push_back(u);
      }
      g_off += n;
    }
  int superunits = 1;
  for (size_t i = 0, col = 0; i < units.size(); ++i) {
    if (col + units[i].n_pad > 192) {
      units[i - 1].dcol_last |= 1 << 16;
      col = 0;
      ++superunits;
    }
    units[i].dcol_last = static_cast<int>(col);
    col += units[i].n_pad;
  }
  units.back().dcol_last |= 1 << 16;
  if (superunits < 2) return fail();  // small shapes: the SIMT kernel (cgtp_bwd.cu)
  t.dout = g_off;
  t.nunits = static_cast<int>(units.size());
  // grad_out rows are scaled per row; the kernel reads that exponent per block at L <= 6 (nbp copies,
  // measured faster there) and once per row at L = 7 (shared memory is short)
  t.nbp = (t.din1 > 49 || t.din2 > 49) ? 4 : (t.nblocks + 3) & ~3;
  t.b_stage_bytes = 64 * max_npad;
  constexpr int kSmemMax = 225 * 1024;
  // grad_out ring (HBM) and W^T ring (L2): the W^T ring's depth matters more (measured: L = 6 with
  // 3 / 5 slots 0.395 ms against 4 / 4 0.43), so the deepest grad_out ring leaving >= 6 W^T stages
  t.g_slots = 3;
  for (int gsl : {8, 4})
    if ((kSmemMax - cgtp_bwd_tc_smem(t, 0, gsl)) / t.b_stage_bytes >= 6) {
      t.g_slots = gsl;
      break;
    }
  if (t.din1 > 49 || t.din2 > 49) t.g_slots = 3;  // the L = 7 instantiation (cgtp_bwd_tc.cu WIDE)
  t.b_stages = std::min(8, (kSmemMax - cgtp_bwd_tc_smem(t, 0, t.g_slots)) / t.b_stage_bytes);
  if (const char* v = std::getenv("TPO_BWD_BSTAGES")) t.b_stages = std::min(t.b_stages, std::atoi(v));  // experiments
  if (t.b_stages < 2) return fail();
  t.units = upload(units);
  t.w = reinterpret_cast<const uint8_t*>(upload(w));
  t.off_b = 0;
  t.off_xy = t.b_stages * t.b_stage_bytes;
  t.off_g = t.off_xy + 128 * (((t.din1 + t.din2) | 1) + (t.one_sided ? std::max(t.din1, t.din2) | 1 : (t.din1 + t.din2) | 1)) * 4;
  t.smem_bytes = cgtp_bwd_tc_smem(t, t.b_stages, t.g_slots);
  if (std::getenv("TPO_VERBOSE"))
    std::fprintf(stderr, "[tpo] cgtp bwd tcgen05 L=(%d,%d) units=%d super=%d b_stages=%d g_slots=%d smem=%d\n", L1, L2,
                 t.nunits, superunits, t.b_stages, t.g_slots, t.smem_bytes);
  return &cgtp_bwd_tc_.emplace(std::array<int, 2>{L1, L2}, std::make_pair(true, t)).first->second.second;
}

// ------------------------------------------------------------------ MTP, tcgen05
// Dense embed / extract operators in the TMEM orders of mtp_tc.cu
// (kernels.hpp, MtpTcTables), same CG tables as Context::mtp
// (proj/src/mtp.cpp:20-97).
// a1 > 0: input 1 holds only degrees a1..L1 (columns (l, m) - a1^2; backward
// windows of grad_out).  flags: 1 = (-1)^l on input 1, 2 = on input 2, 4 = on
// the output (the carrier-transpose identities of the MTP backward, capi.cpp).
const MtpTcTables* Context::mtp_tc(int L1, int L2, int L3, int lt, int a1, int flags) {
  std::lock_guard<std::mutex> g(mu_);
  const std::array<int, 6> key{L1, L2, L3, lt, a1, flags};
  auto it = mtp_tc_.find(key);
  if (it != mtp_tc_.end()) return it->second.first ? &it->second.second : nullptr;
  auto fail = [&]() -> const MtpTcTables* {
    mtp_tc_.emplace(key, std::make_pair(false, MtpTcTables{}));
    return nullptr;
  };
  const char* env = std::getenv("TPO_MTP_TC");
  const int dt = 2 * lt + 1;
  if ((env && env[0] == '0') || dt > 13) return fail();
  MtpTcTables t{};
  t.dt = dt;
  t.din1 = (L1 + 1) * (L1 + 1) - a1 * a1;
  t.din2 = (L2 + 1) * (L2 + 1);
  const int L3e = std::min(L3, 2 * lt);
  t.dout_eff = (L3e + 1) * (L3e + 1);
  t.dout_total = (L3 + 1) * (L3 + 1);
  t.n1 = pad_to(dt * dt, 16);
  t.n2 = pad_to(t.dout_eff, 16);
  t.k1 = pad_to(t.din1, 16);
  t.k2 = pad_to(t.din2, 16);
  if (t.k1 > 112 || t.k2 > 64) return fail();  // input 1 wider than 64: backward windows of grad_out
  // per-row matmul split by carrier rows between the two warps of a TMEM lane quarter:
  // Z group 0 = rows i < i1, group 1 (+ tail group 2) = rows i >= i1, cells (i - i0) * dt + j
  const int i1 = (dt + 1) / 2;
  const int size0 = pad_to(i1 * dt, 16), size1 = pad_to((dt - i1) * dt, 16);
  t.kz = size0 + size1;
  t.zgrp_col[0] = 2 * t.n1;
  t.zgrp_size[0] = size0;
  if (t.zgrp_col[0] + size0 > 512) return fail();
  const int room = (512 - (t.zgrp_col[0] + size0)) / 16 * 16;
  t.zgrp_col[1] = t.zgrp_col[0] + size0;
  t.zgrp_size[1] = std::min(size1, room);
  // the tail goes to the Y columns once both halves finished reading them
  t.zgrp_col[2] = t.n1;
  t.zgrp_size[2] = size1 - t.zgrp_size[1];
  t.zgrp_col[3] = 0;
  t.zgrp_size[3] = 0;
  t.y0_reuse = t.zgrp_size[2] > 0;
  if (t.zgrp_size[2] > t.n1) return fail();
  // dense operators (double), rows in TMEM order
  std::vector<double> e1(static_cast<size_t>(t.n1) * t.k1, 0.0), e2(static_cast<size_t>(t.n1) * t.k2, 0.0);
  auto xpos = [&](int i, int k) { return k * dt + i; };
  auto ypos = [&](int k, int j) { return k * dt + j; };
  auto zpos = [&](int i, int j) { return i < i1 ? i * dt + j : size0 + (i - i1) * dt + j; };
  auto sgn = [&](int bit, int l) { return ((flags & bit) && (l & 1)) ? -1.0 : 1.0; };
  for (int l = 0; l <= std::max(L1, L2); ++l)  // proj/src/mtp.cpp:20-39
    for (const CGEntry& e : real_cg(lt, lt, l)) {
      const int a = e.m1 + lt, b = e.m2 + lt, in = flat(l, e.m3);
      if (l >= a1 && l <= L1) e1[static_cast<size_t>(xpos(a, b)) * t.k1 + in - a1 * a1] += sgn(1, l) * e.v;
      if (l <= L2) e2[static_cast<size_t>(ypos(a, b)) * t.k2 + in] += sgn(2, l) * e.v;
    }
  std::vector<double> ex(static_cast<size_t>(t.n2) * t.kz, 0.0);
  for (int l3 = 0; l3 <= L3e; ++l3)  // proj/src/mtp.cpp:60-97
    for (const CGEntry& e : real_cg(lt, lt, l3))
      ex[static_cast<size_t>(flat(l3, e.m3)) * t.kz + zpos(e.m1 + lt, e.m2 + lt)] += sgn(4, l3) * std::ldexp(e.v, kTabShift);
  // per K-step [hi | lo][rows x 16] canonical
  auto tile = [&](const std::vector<double>& m, int rows, int kdim) {
    const int nks = kdim / 16;
    std::vector<uint16_t> buf(static_cast<size_t>(nks) * 2 * rows * 16, 0);
    for (int ks = 0; ks < nks; ++ks) {
      uint16_t* hi = buf.data() + static_cast<size_t>(ks) * 2 * rows * 16;
      uint16_t* lo = hi + rows * 16;
      for (int r = 0; r < rows; ++r)
        for (int kk = 0; kk < 16; ++kk) {
          uint16_t hv, lv;
          split_half(m[static_cast<size_t>(r) * kdim + ks * 16 + kk], hv, lv);
          const uint32_t o = sm100::canon_off(r, kk, rows) / 2;
          hi[o] = hv;
          lo[o] = lv;
        }
    }
    return buf;
  };
  t.e1 = reinterpret_cast<const uint8_t*>(upload(tile(e1, t.n1, t.k1)));
  t.e2 = reinterpret_cast<const uint8_t*>(upload(tile(e2, t.n1, t.k2)));
  t.ext = reinterpret_cast<const uint8_t*>(upload(tile(ex, t.n2, t.kz)));
  // shared memory: ring | X op | Y op | x staging | y staging | epilogue staging
  t.stage_bytes = 64 * t.n1;
  // raw input staging doubles as output half buffer 1; output half buffer 0 doubles as the
  // per-warp staging of the direct-store epilogue
  const int raw_bytes = std::max(128 * (t.din1 + t.din2) * 4, 64 * t.dout_total * 4);
  const int out_bytes = std::max(64 * t.dout_total * 4, 8 * 32 * 17 * 4);
  const int fixed = 128 * t.k1 * 4 + 128 * t.k2 * 4 + raw_bytes + out_bytes;
  const int budget = 220 * 1024;
  t.stages = std::min(8, (budget - fixed) / t.stage_bytes);
  if (t.stages < 2) return fail();
  t.off_xop = t.stages * t.stage_bytes;
  t.off_yop = t.off_xop + 128 * t.k1 * 4;
  t.off_stx = t.off_yop + 128 * t.k2 * 4;
  t.off_sty = t.off_stx + 128 * t.din1 * 4;
  t.off_out = t.off_stx + pad_to(raw_bytes, 128);
  t.smem_bytes = t.off_out + out_bytes + 1024;
  if (std::getenv("TPO_VERBOSE"))
    std::fprintf(stderr, "[tpo] mtp tcgen05 dt=%d n1=%d n2=%d k=(%d,%d) kz=%d zcols=(%d,%d,%d,%d) y0=%d stages=%d smem=%d\n",
                 dt, t.n1, t.n2, t.k1, t.k2, t.kz, t.zgrp_col[0], t.zgrp_col[1], t.zgrp_col[2], t.zgrp_col[3],
                 t.y0_reuse, t.stages, t.smem_bytes);
  return &mtp_tc_.emplace(key, std::make_pair(true, t)).first->second.second;
}

const float* Context::degree_weights(const std::vector<double>& w) {
  std::lock_guard<std::mutex> g(mu_);
  auto it = weights_.find(w);
  if (it != weights_.end()) return it->second;
  std::vector<float> f(w.begin(), w.end());
  const float* d = upload(f);
  weights_.emplace(w, d);
  return d;
}

// ------------------------------------------------------------------ stage operators (stages.cu)
const float* Context::dense_op(const std::string& key, const std::function<std::vector<double>()>& build) {
  {
    std::lock_guard<std::mutex> g(mu_);
    auto it = dense_ops_.find(key);
    if (it != dense_ops_.end()) return it->second;
  }
  const std::vector<double> m = build();
  std::vector<float> f(m.begin(), m.end());
  std::lock_guard<std::mutex> g(mu_);
  auto it = dense_ops_.find(key);
  if (it != dense_ops_.end()) return it->second;
  const float* d = upload(f);
  dense_ops_.emplace(key, d);
  return d;
}

const int* Context::int_table(const std::string& key, const std::function<std::vector<int>()>& build) {
  {
    std::lock_guard<std::mutex> g(mu_);
    auto it = int_tables_.find(key);
    if (it != int_tables_.end()) return it->second;
  }
  const std::vector<int> v = build();
  std::lock_guard<std::mutex> g(mu_);
  auto it = int_tables_.find(key);
  if (it != int_tables_.end()) return it->second;
  const int* d = upload(v);
  int_tables_.emplace(key, d);
  return d;
}

const WignerTables& Context::wigner(int L) {
  std::lock_guard<std::mutex> g(mu_);
  auto it = wigner_.find(L);
  if (it != wigner_.end()) return it->second;
  if (L < 0 || L > kWignerMaxL) throw InvalidArgument("wigner_d: degree out of range");
  WignerTables w{};
  w.L = L;
  std::vector<int> row_off;
  std::vector<WignerEntry> entries;
  int64_t boff = 0;
  for (int l = 0; l <= L; ++l) {
    w.block_off[l] = boff;
    boff += static_cast<int64_t>(2 * l + 1) * (2 * l + 1);
    w.l_off[l] = static_cast<int>(row_off.size());
    w.e_off[l] = static_cast<int>(entries.size());
    if (l < 2) {
      row_off.push_back(0);
      continue;
    }
    // D^l = Q (D^1 (x) D^{l-1}) Q^T with Q = cg_real(1, l-1, l) (proj/src/wigner.cpp:302-311); rows by m3
    std::vector<std::vector<WignerEntry>> by_row(2 * l + 1);
    for (const CGEntry& e : real_cg(1, l - 1, l)) by_row[e.m3 + l].push_back({e.m1 + 1, e.m2 + l - 1, e.v});
    int n = 0;
    for (int i = 0; i <= 2 * l; ++i) {
      row_off.push_back(n);
      for (const WignerEntry& e : by_row[i]) entries.push_back(e);
      n += static_cast<int>(by_row[i].size());
    }
    row_off.push_back(n);
  }
  w.d_stride = boff;
  w.row_off = upload(row_off);
  w.entries = upload(entries);
  std::vector<int64_t> bo(w.block_off, w.block_off + L + 1);
  w.block_off_dev = upload(bo);
  return wigner_.emplace(L, w).first->second;
}

}  // namespace tpo_b200

