// Device-table construction: turns the fp64 host tables (tables.cpp) into
// the layouts the kernels consume.  See kernels/kernels.hpp for formats.
#include "context.hpp"

#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "../kernels/sm100.cuh"
#include "tables.hpp"

namespace tpo_b200 {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaFailure(std::string(what) + ": " + cudaGetErrorString(e));
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
  if (prop.major != 10)
    throw CudaFailure("device is sm_" + std::to_string(prop.major) + std::to_string(prop.minor) +
                      "; this library is built for sm_100a (B200) only");
  num_sms_ = prop.multiProcessorCount;
  cuda_check(cudaStreamCreateWithFlags(&host_stream_, cudaStreamNonBlocking), "cudaStreamCreate");
}

Context::~Context() {
  cudaSetDevice(device_);
  for (void* p : allocs_) cudaFree(p);
  for (void* p : scratch_)
    if (p) cudaFree(p);
  if (host_stream_) cudaStreamDestroy(host_stream_);
}

void Context::activate() const { cuda_check(cudaSetDevice(device_), "cudaSetDevice"); }

void* Context::dev_alloc(size_t bytes) {
  void* p = nullptr;
  cuda_check(cudaMalloc(&p, std::max<size_t>(bytes, 16)), "cudaMalloc(table)");
  allocs_.push_back(p);
  return p;
}

template <class T>
T* Context::upload(const std::vector<T>& v) {
  void* p = dev_alloc(v.size() * sizeof(T));
  if (!v.empty()) cuda_check(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "upload");
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
const CgtpTables& Context::cgtp(int L1, int L2) {
  std::lock_guard<std::mutex> g(mu_);
  auto it = cgtp_.find({L1, L2});
  if (it != cgtp_.end()) return it->second;
  const int din1 = (L1 + 1) * (L1 + 1), din2 = (L2 + 1) * (L2 + 1);
  std::vector<std::vector<std::pair<uint32_t, float>>> per_out;
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
  const int dout = static_cast<int>(per_out.size());
  const int nchunks = (dout + kCgtpChunk - 1) / kCgtpChunk;
  std::vector<int> off(nchunks), nt(nchunks);
  std::vector<uint2> terms;
  for (int q = 0; q < nchunks; ++q) {
    int tmax = 0;
    for (int i = 0; i < kCgtpChunk; ++i) {
      const int o = q * kCgtpChunk + i;
      if (o < dout) tmax = std::max<int>(tmax, static_cast<int>(per_out[o].size()));
    }
    off[q] = static_cast<int>(terms.size());
    nt[q] = tmax;
    terms.resize(terms.size() + static_cast<size_t>(tmax) * kCgtpChunk, make_uint2(0u, 0u));
    for (int i = 0; i < kCgtpChunk; ++i) {
      const int o = q * kCgtpChunk + i;
      if (o >= dout) continue;
      for (size_t t = 0; t < per_out[o].size(); ++t) {
        float c = per_out[o][t].second;
        uint32_t cb;
        std::memcpy(&cb, &c, 4);
        terms[off[q] + t * kCgtpChunk + i] = make_uint2(per_out[o][t].first, cb);
      }
    }
  }
  CgtpTables t{};
  t.din1 = din1;
  t.din2 = din2;
  t.dout = dout;
  t.nchunks = nchunks;
  t.terms = upload(terms);
  t.chunk_off = upload(off);
  t.chunk_nt = upload(nt);
  return cgtp_.emplace(std::array<int, 2>{L1, L2}, t).first->second;
}

// ------------------------------------------------------------------ GTP grid (tcgen05)
const GridTcEntry& Context::grid_tc(int L1, int L2, int L3) {
  std::lock_guard<std::mutex> g(mu_);
  auto it = grid_tc_.find({L1, L2, L3});
  if (it != grid_tc_.end()) return it->second;
  GridTcEntry ent;
  GridTcTables& t = ent.t;
  const int band = L1 + L2;
  const int L3e = std::min(L3, band);
  t.din1 = (L1 + 1) * (L1 + 1);
  t.din2 = (L2 + 1) * (L2 + 1);
  t.k1p = pad_to(t.din1, 16);
  t.k2p = pad_to(t.din2, 16);
  t.dout_eff = (L3e + 1) * (L3e + 1);
  t.dout_total = (L3 + 1) * (L3 + 1);
  t.dout_pad = pad_to(t.dout_eff, 16);
  t.same_s = (L1 == L2) ? 1 : 0;
  const S2Grid& gr = s2_grid(band);
  const int G = gr.n_theta * gr.n_phi;
  const int max_smem = gtp_grid_tc_max_smem();
  auto smem_for = [&](int nc, uint32_t* offs) {
    uint32_t o = 0;
    const uint32_t xy = std::max<uint32_t>(512u * (t.k1p + t.k2p), 128u * 33u * 4u);
    offs[0] = 0;
    offs[1] = 512u * t.k1p;
    o = pad_to(static_cast<int>(xy), 128);
    offs[2] = o;
    o += pad_to(4 * nc * t.k1p, 128);
    offs[3] = o;
    if (!t.same_s) o += pad_to(4 * nc * t.k2p, 128);
    offs[4] = o;
    o += pad_to(512 * nc, 128);
    offs[5] = o;
    o += pad_to(4 * t.dout_pad * nc, 128);
    return static_cast<int>(o);
  };
  int nc = 0;
  uint32_t offs[6] = {};
  if (t.k1p <= 128 && t.k2p <= 128) {
    for (int cand = 128; cand >= 16; cand -= 16)
      if (t.dout_pad + 2 * cand <= 512 && smem_for(cand, offs) <= max_smem) {
        nc = cand;
        break;
      }
  }
  if (nc == 0) {  // does not fit the fused tiling: SIMT separable kernel handles this shape
    ent.fits = false;
    return grid_tc_.emplace(std::array<int, 3>{L1, L2, L3}, ent).first->second;
  }
  t.nchunks = (G + nc - 1) / nc;
  nc = pad_to((G + t.nchunks - 1) / t.nchunks, 16);  // rebalance padding over chunks
  t.nc = nc;
  t.smem_bytes = smem_for(nc, offs);
  t.off_x = offs[0];
  t.off_y = offs[1];
  t.off_s1 = offs[2];
  t.off_s2 = offs[3];
  t.off_p = offs[4];
  t.off_a = offs[5];
  int cols = 32;
  while (cols < t.dout_pad + 2 * nc) cols *= 2;
  t.tmem_cols = cols;

  // dense operators on the product grid (proj/src/sphere.cpp:105-195)
  const double phi_scale = 2.0 * M_PI / gr.n_phi;
  auto s_val = [&](int gidx, int k) -> double {  // S[g][(l,m)]
    const int j = gidx / gr.n_phi, kk = gidx % gr.n_phi;
    const int l = static_cast<int>(std::sqrt(static_cast<double>(k)) + 1e-9);
    const int m = k - l * l - l;
    return gr.lambda(l, std::abs(m), j) * gr.csm(m, kk);
  };
  double amax = 0.0;
  for (int gidx = 0; gidx < G; ++gidx)
    for (int o = 0; o < t.dout_eff; ++o) {
      const int j = gidx / gr.n_phi;
      amax = std::max(amax, std::abs(gr.weights[j] * phi_scale * s_val(gidx, o)));
    }
  t.a_shift = amax > 0 ? -(std::ilogb(amax) + 1) : 0;
  const double a_scale = std::ldexp(1.0, t.a_shift);

  auto build_s = [&](int din, int kp, std::vector<uint16_t>& buf) {
    const size_t half_elems = static_cast<size_t>(nc) * kp;  // per hi / lo block
    buf.assign(static_cast<size_t>(t.nchunks) * 2 * half_elems, 0);
    for (int c = 0; c < t.nchunks; ++c) {
      uint16_t* hi = buf.data() + static_cast<size_t>(c) * 2 * half_elems;
      uint16_t* lo = hi + half_elems;
      for (int r = 0; r < nc; ++r) {
        const int gidx = c * nc + r;
        for (int k = 0; k < kp; ++k) {
          const double v = (gidx < G && k < din) ? s_val(gidx, k) : 0.0;
          uint16_t h, l;
          split_half(v, h, l);
          const uint32_t e = sm100::canon_off(r, k, nc) / 2;
          hi[e] = h;
          lo[e] = l;
        }
      }
    }
  };
  std::vector<uint16_t> s1, s2, a;
  build_s(t.din1, t.k1p, s1);
  t.s1_chunk_bytes = static_cast<uint32_t>(4u * nc * t.k1p);
  t.s1 = reinterpret_cast<const uint8_t*>(upload(s1));
  if (t.same_s) {
    t.s2 = t.s1;
    t.s2_chunk_bytes = t.s1_chunk_bytes;
  } else {
    build_s(t.din2, t.k2p, s2);
    t.s2_chunk_bytes = static_cast<uint32_t>(4u * nc * t.k2p);
    t.s2 = reinterpret_cast<const uint8_t*>(upload(s2));
  }
  {
    const size_t half_elems = static_cast<size_t>(t.dout_pad) * nc;
    a.assign(static_cast<size_t>(t.nchunks) * 2 * half_elems, 0);
    for (int c = 0; c < t.nchunks; ++c) {
      uint16_t* hi = a.data() + static_cast<size_t>(c) * 2 * half_elems;
      uint16_t* lo = hi + half_elems;
      for (int o = 0; o < t.dout_pad; ++o)
        for (int r = 0; r < nc; ++r) {
          const int gidx = c * nc + r;
          double v = 0.0;
          if (gidx < G && o < t.dout_eff) {
            const int j = gidx / gr.n_phi;
            v = gr.weights[j] * phi_scale * s_val(gidx, o) * a_scale;
          }
          uint16_t h, l;
          split_half(v, h, l);
          const uint32_t e = sm100::canon_off(o, r, t.dout_pad) / 2;
          hi[e] = h;
          lo[e] = l;
        }
    }
    t.a_chunk_bytes = static_cast<uint32_t>(4u * t.dout_pad * nc);
    t.a = reinterpret_cast<const uint8_t*>(upload(a));
  }
  ent.fits = true;
  return grid_tc_.emplace(std::array<int, 3>{L1, L2, L3}, ent).first->second;
}

// ------------------------------------------------------------------ GTP grid (SIMT separable)
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
  return grid_simt_.emplace(std::array<int, 3>{L1, L2, L3}, t).first->second;
}

// ------------------------------------------------------------------ GTP Fourier
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
  t.din1 = (L1 + 1) * (L1 + 1);
  t.din2 = (L2 + 1) * (L2 + 1);
  auto emb = [&](int Lx, const int** off_out, const int** idx_out, const float** c_out) {
    std::vector<std::vector<std::pair<int, float>>> cell(dt2);
    for (int l = 0; l <= Lx; ++l)  // proj/src/mtp.cpp:20-39
      for (const CGEntry& e : real_cg(lt, lt, l))
        cell[(e.m1 + lt) * dt + (e.m2 + lt)].push_back({flat(l, e.m3), static_cast<float>(e.v)});
    std::vector<int> off(dt2 + 1), idx;
    std::vector<float> c;
    for (int i = 0; i < dt2; ++i) {
      off[i] = static_cast<int>(idx.size());
      for (auto& p : cell[i]) {
        idx.push_back(p.first);
        c.push_back(p.second);
      }
    }
    off[dt2] = static_cast<int>(idx.size());
    *off_out = upload(off);
    *idx_out = upload(idx);
    *c_out = upload(c);
  };
  emb(L1, &t.emb1_off, &t.emb1_idx, &t.emb1_c);
  emb(L2, &t.emb2_off, &t.emb2_idx, &t.emb2_c);
  const int L3e = std::min(L3, 2 * lt);  // beyond the carrier band: zero (mtp.cpp:126)
  t.dout_eff = (L3e + 1) * (L3e + 1);
  t.dout_total = (L3 + 1) * (L3 + 1);
  std::vector<int> off(t.dout_eff + 1), idx;
  std::vector<float> c;
  for (int l3 = 0; l3 <= L3e; ++l3) {
    std::vector<std::vector<std::pair<int, float>>> per(2 * l3 + 1);
    for (const CGEntry& e : real_cg(lt, lt, l3))
      per[e.m3 + l3].push_back({(e.m1 + lt) * dt + (e.m2 + lt), static_cast<float>(e.v)});
    for (int m3 = -l3; m3 <= l3; ++m3) {
      off[flat(l3, m3)] = static_cast<int>(idx.size());
      for (auto& p : per[m3 + l3]) {
        idx.push_back(p.first);
        c.push_back(p.second);
      }
    }
  }
  off[t.dout_eff] = static_cast<int>(idx.size());
  t.ext_off = upload(off);
  t.ext_idx = upload(idx);
  t.ext_c = upload(c);
  return mtp_.emplace(std::array<int, 4>{L1, L2, L3, lt}, t).first->second;
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

}  // namespace tpo_b200
