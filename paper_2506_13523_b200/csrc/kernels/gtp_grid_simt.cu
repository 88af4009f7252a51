// S2-grid Gaunt tensor product, separable SIMT kernel (large-L path).
//
// Same algorithm as the reference (proj/src/sphere.cpp:105-195): Legendre
// synthesis per m, phi synthesis, pointwise product, phi analysis with the
// quadrature weights folded in, Legendre analysis.  O(L^3) per product
// instead of the dense GEMM formulation's O(L^4); used where the fused
// tcgen05 kernel's TMEM/shared-memory tiling does not fit (output band
// > 448 coefficients or inputs > 128 coefficients, i.e. L > 10) and
// selectable for comparison.  One block per product, persistent over rows;
// all intermediates live in shared memory.
#include <algorithm>

#include "kernels.hpp"

namespace tpo_b200 {
namespace {

constexpr int kThreads = 256;

__global__ void __launch_bounds__(kThreads)
    grid_simt_kernel(const __grid_constant__ GridSimtTables t, const __grid_constant__ RowSpec rs) {
  extern __shared__ float sm[];
  const int nt = t.nt, np = t.np, B = t.band;
  const int din1 = (t.L1 + 1) * (t.L1 + 1), din2 = (t.L2 + 1) * (t.L2 + 1);
  const int nm1 = 2 * t.L1 + 1, nm2 = 2 * t.L2 + 1, nm3 = 2 * t.L3e + 1;
  float* xs = sm;                 // din1
  float* ys = xs + din1;          // din2
  float* gx = ys + din2;          // [nm1][nt]
  float* gy = gx + nm1 * nt;      // [nm2][nt]
  float* P = gy + nm2 * nt;       // [nt][np]
  float* h = P + nt * np;         // [nm3][nt]
  auto lam = [&](int l, int ma, int j) { return __ldg(t.lam + (l * (l + 1) / 2 + ma) * nt + j); };
  auto cs = [&](int m, int k) { return __ldg(t.cs + (m + B) * np + k); };
  for (int64_t row = blockIdx.x; row < rs.rows; row += gridDim.x) {
    const int64_t yr = rs.y_shared ? row / rs.channels : row;
    for (int i = threadIdx.x; i < din1; i += kThreads) xs[i] = __ldg(rs.x + row * din1 + i);
    for (int i = threadIdx.x; i < din2; i += kThreads) ys[i] = __ldg(rs.y + yr * din2 + i);
    __syncthreads();
    // 1. Legendre synthesis g_m(theta_j) = sum_{l>=|m|} x_lm Lambda_l|m|(theta_j)
    for (int i = threadIdx.x; i < (nm1 + nm2) * nt; i += kThreads) {
      const bool isx = i < nm1 * nt;
      const int ii = isx ? i : i - nm1 * nt;
      const int Lx = isx ? t.L1 : t.L2;
      const float* v = isx ? xs : ys;
      const int mi = ii / nt, j = ii - mi * nt, m = mi - Lx, ma = abs(m);
      float acc = 0.f;
      for (int l = ma; l <= Lx; ++l) acc = fmaf(v[l * l + m + l], lam(l, ma, j), acc);
      (isx ? gx : gy)[ii] = acc;
    }
    __syncthreads();
    // 2+3. phi synthesis of both inputs and pointwise product
    for (int i = threadIdx.x; i < nt * np; i += kThreads) {
      const int j = i / np, k = i - j * np;
      float fx = 0.f, fy = 0.f;
      for (int mi = 0; mi < nm1; ++mi) fx = fmaf(gx[mi * nt + j], cs(mi - t.L1, k), fx);
      for (int mi = 0; mi < nm2; ++mi) fy = fmaf(gy[mi * nt + j], cs(mi - t.L2, k), fy);
      P[i] = fx * fy;
    }
    __syncthreads();
    // 4. phi analysis, quadrature weight w_j * 2pi/n_phi folded in
    for (int i = threadIdx.x; i < nm3 * nt; i += kThreads) {
      const int mi = i / nt, j = i - mi * nt, m = mi - t.L3e;
      float acc = 0.f;
      for (int k = 0; k < np; ++k) acc = fmaf(P[j * np + k], cs(m, k), acc);
      h[i] = acc * __ldg(t.wq + j);
    }
    __syncthreads();
    // 5. Legendre analysis; degrees past the band are exactly zero
    for (int o = threadIdx.x; o < t.dout_total; o += kThreads) {
      float acc = 0.f;
      const int l = static_cast<int>(sqrtf(static_cast<float>(o)));
      const int lc = (l + 1) * (l + 1) <= o ? l + 1 : (l * l > o ? l - 1 : l);
      if (lc <= t.L3e) {
        const int m = o - lc * lc - lc, ma = abs(m);
        for (int j = 0; j < nt; ++j) acc = fmaf(h[(m + t.L3e) * nt + j], lam(lc, ma, j), acc);
      }
      rs.out[row * t.dout_total + o] = acc;
    }
    __syncthreads();
  }
}

}  // namespace

cudaError_t launch_gtp_grid_simt(const GridSimtTables& t, const RowSpec& rs, int num_sms, cudaStream_t s) {
  if (rs.rows <= 0) return cudaSuccess;
  const int din1 = (t.L1 + 1) * (t.L1 + 1), din2 = (t.L2 + 1) * (t.L2 + 1);
  const size_t smem = sizeof(float) * (din1 + din2 + (2 * t.L1 + 1 + 2 * t.L2 + 1) * t.nt + t.nt * t.np +
                                       (2 * t.L3e + 1) * t.nt);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(grid_simt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, grid_simt_kernel, kThreads, smem);
  const int grid = static_cast<int>(std::min<int64_t>(rs.rows, static_cast<int64_t>(num_sms) * std::max(occ, 1)));
  grid_simt_kernel<<<grid, kThreads, smem, s>>>(t, rs);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- per-degree scaling
namespace {
__global__ void scale_degrees_kernel(const float* __restrict__ in, float* __restrict__ out, int64_t n,
                                     int dim, int L, const float* __restrict__ w) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int o = static_cast<int>(i % dim);
    int l = static_cast<int>(sqrtf(static_cast<float>(o)));
    if ((l + 1) * (l + 1) <= o) ++l;
    if (l * l > o) --l;
    out[i] = in[i] * __ldg(w + l);
  }
}
}  // namespace

cudaError_t launch_scale_degrees(const float* in, float* out, int64_t rows, int L, const float* w,
                                 cudaStream_t s) {
  const int dim = (L + 1) * (L + 1);
  const int64_t n = rows * dim;
  if (n <= 0) return cudaSuccess;
  const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 32));
  scale_degrees_kernel<<<grid, 256, 0, s>>>(in, out, n, dim, L, w);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- out += in (backward partial sums)
namespace {
__global__ void accumulate_kernel(const float4* __restrict__ in, float4* __restrict__ out, int64_t n4) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float4 a = __ldg(in + i);
    float4 b = out[i];
    b.x += a.x; b.y += a.y; b.z += a.z; b.w += a.w;
    out[i] = b;
  }
}
__global__ void accumulate_tail_kernel(const float* __restrict__ in, float* __restrict__ out, int64_t n) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) out[i] += in[i];
}
}  // namespace

cudaError_t launch_accumulate(const float* in, float* out, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const bool vec = (reinterpret_cast<uintptr_t>(in) % 16 == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0);
  const int64_t n4 = vec ? n / 4 : 0;
  if (n4 > 0) {
    const int grid = static_cast<int>(std::min<int64_t>((n4 + 255) / 256, 148 * 16));
    accumulate_kernel<<<grid, 256, 0, s>>>(reinterpret_cast<const float4*>(in), reinterpret_cast<float4*>(out), n4);
  }
  const int64_t rem = n - 4 * n4;
  if (rem > 0)
    accumulate_tail_kernel<<<static_cast<int>((rem + 255) / 256), 256, 0, s>>>(in + 4 * n4, out + 4 * n4, rem);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- column window gather (backward)
namespace {
__global__ void gather_cols_kernel(const float* __restrict__ src, int64_t stride, int col0, int w,
                                   float* __restrict__ dst, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / w;
    dst[i] = __ldg(src + r * stride + col0 + (i - r * w));
  }
}
}  // namespace

cudaError_t launch_gather_cols(const float* src, int64_t stride, int col0, int w, float* dst, int64_t rows,
                               cudaStream_t s) {
  const int64_t n = rows * w;
  if (n <= 0) return cudaSuccess;
  const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 16));
  gather_cols_kernel<<<grid, 256, 0, s>>>(src, stride, col0, w, dst, n);
  return cudaGetLastError();
}

}  // namespace tpo_b200
