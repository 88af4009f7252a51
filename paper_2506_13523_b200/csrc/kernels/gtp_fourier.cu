// Gaunt tensor product in the 2D torus Fourier basis (SIMT).
//
// Reference: tpo::detail::gtp_fourier_select (proj/src/gtp.cpp:262-327):
// sparse encode of both inputs onto (2L+1)^2 torus spectra (:268-287),
// direct 2D spectral convolution to the (4L+1)^2 product spectrum
// (:290-301), sparse decode and real part (:305-326).
// The product of two real functions has a Hermitian spectrum,
// cz(-U,-V) = conj(cz(U,V)), so only the half-plane {V > 0} u {V = 0, U >= 0}
// is convolved (half the complex MACs); decode entries that point into the
// other half read the conjugate.  Per row the two input spectra and the
// half product spectrum live in shared memory.
#include <algorithm>

#include "kernels.hpp"

namespace tpo_b200 {
namespace {

constexpr int kThreads = 256;

__global__ void __launch_bounds__(kThreads)
    fourier_kernel(const __grid_constant__ FourierDevTables t, const __grid_constant__ RowSpec rs, int R) {
  extern __shared__ float sm[];
  const int L = t.L, w = 2 * L + 1, w2 = w * w;
  const int din1 = (t.L1 + 1) * (t.L1 + 1), din2 = (t.L2 + 1) * (t.L2 + 1);
  float* xs = sm;                                             // [R][din1]
  float* ys = xs + R * din1;                                  // [R][din2]
  float2* cx = reinterpret_cast<float2*>(ys + R * din2);      // [R][w2]
  float2* cy = cx + R * w2;                                   // [R][w2]
  float2* cz = cy + R * w2;                                   // [R][nhalf]
  const int64_t ntiles = (rs.rows + R - 1) / R;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row0 = tile * R;
    const int nr = static_cast<int>(std::min<int64_t>(R, rs.rows - row0));
    for (int i = threadIdx.x; i < nr * din1; i += kThreads) xs[i] = __ldg(rs.x + row0 * din1 + i);
    for (int i = threadIdx.x; i < nr * din2; i += kThreads) {
      const int r = i / din2, k = i - r * din2;
      const int64_t g = row0 + r;
      ys[i] = __ldg(rs.y + (rs.y_shared ? g / rs.channels : g) * din2 + k);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nr * w2; i += kThreads) {  // encode (real x complex)
      const int r = i / w2, mode = i - r * w2;
      float2 a = make_float2(0.f, 0.f), b = make_float2(0.f, 0.f);
      for (int e = __ldg(t.enc1_off + mode), e1 = __ldg(t.enc1_off + mode + 1); e < e1; ++e) {
        const float v = xs[r * din1 + __ldg(t.enc1_idx + e)];
        const float2 c = __ldg(t.enc1_w + e);
        a.x = fmaf(v, c.x, a.x);
        a.y = fmaf(v, c.y, a.y);
      }
      for (int e = __ldg(t.enc2_off + mode), e1 = __ldg(t.enc2_off + mode + 1); e < e1; ++e) {
        const float v = ys[r * din2 + __ldg(t.enc2_idx + e)];
        const float2 c = __ldg(t.enc2_w + e);
        b.x = fmaf(v, c.x, b.x);
        b.y = fmaf(v, c.y, b.y);
      }
      cx[i] = a;
      cy[i] = b;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nr * t.nhalf; i += kThreads) {  // 2D convolution, half plane
      const int r = i / t.nhalf, h = i - r * t.nhalf;
      const int2 UV = __ldg(t.half_uv + h);
      const int u_lo = max(-L, UV.x - L), u_hi = min(L, UV.x + L);
      const int v_lo = max(-L, UV.y - L), v_hi = min(L, UV.y + L);
      const float2* X = cx + r * w2;
      const float2* Y = cy + r * w2;
      float re = 0.f, im = 0.f;
      for (int u1 = u_lo; u1 <= u_hi; ++u1) {
        const float2* xrow = X + (u1 + L) * w;
        const float2* yrow = Y + (UV.x - u1 + L) * w;
        for (int v1 = v_lo; v1 <= v_hi; ++v1) {
          const float2 a = xrow[v1 + L];
          const float2 b = yrow[UV.y - v1 + L];
          re = fmaf(a.x, b.x, re);
          re = fmaf(-a.y, b.y, re);
          im = fmaf(a.x, b.y, im);
          im = fmaf(a.y, b.x, im);
        }
      }
      cz[i] = make_float2(re, im);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nr * t.dout_total; i += kThreads) {  // decode, real part
      const int r = i / t.dout_total, o = i - r * t.dout_total;
      float acc = 0.f;
      if (o < t.dout_eff) {
        const float2* Z = cz + r * t.nhalf;
        for (int e = __ldg(t.dec_off + o), e1 = __ldg(t.dec_off + o + 1); e < e1; ++e) {
          const int code = __ldg(t.dec_idx + e);
          const float2 wv = __ldg(t.dec_w + e);
          const float2 z = Z[code >> 1];
          const float zi = (code & 1) ? -z.y : z.y;  // conj for the mirrored half
          acc = fmaf(wv.x, z.x, acc);
          acc = fmaf(-wv.y, zi, acc);
        }
      }
      rs.out[row0 * t.dout_total + i] = acc;
    }
    __syncthreads();
  }
}

}  // namespace

cudaError_t launch_gtp_fourier(const FourierDevTables& t, const RowSpec& rs, int num_sms, cudaStream_t s) {
  if (rs.rows <= 0) return cudaSuccess;
  const int w2 = (2 * t.L + 1) * (2 * t.L + 1);
  const int per_row = (t.L1 + 1) * (t.L1 + 1) + (t.L2 + 1) * (t.L2 + 1) + 4 * w2 + 2 * t.nhalf;
  const int R = std::max(1, std::min(16, (48 * 1024 / 4) / per_row));
  const size_t smem = sizeof(float) * static_cast<size_t>(R) * per_row;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fourier_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fourier_kernel, kThreads, smem);
  const int64_t ntiles = (rs.rows + R - 1) / R;
  const int grid = static_cast<int>(std::min<int64_t>(ntiles, static_cast<int64_t>(num_sms) * std::max(occ, 1)));
  fourier_kernel<<<grid, kThreads, smem, s>>>(t, rs, R);
  return cudaGetLastError();
}

}  // namespace tpo_b200
