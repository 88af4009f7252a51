// Batched stage operators of the reference's product pipelines, exposed on the C ABI so that a
// caller can run (and time) the stages on their own, as the reference's run_once does
// (proj/src/bench.cpp:58-72):
//   dense_map      out[b] = M in[b] for a fixed linear map M -- to_sphere (proj/src/sphere.cpp:105-134),
//                  from_sphere_select (:155-195), mtp_embed (proj/src/mtp.cpp:20-58),
//                  mtp_extract_select (:60-97), apply_linear (proj/src/irreps.cpp:119-129)
//   carrier_matmul Z[b] = X[b] Y[b], the MTP's classical cubic product (proj/src/mtp.cpp:119-133)
//   pointwise_mul  (proj/src/sphere.cpp:145-151)
//   wigner_d       real Wigner-D blocks of a batch of rotations by the reference's recursion
//                  D^l = Q (D^1 (x) D^{l-1}) Q^T, Q = cg_real(1, l-1, l) (proj/src/wigner.cpp:288-312), fp64
//   rotate         out = blockdiag(D^l) x per row (proj/src/wigner.cpp:314-325)
// The fused product kernels never call these: they are the drop-in surface for the stage API.
#include <algorithm>

#include "kernels.hpp"

namespace tpo_b200 {
namespace {

constexpr int kMapRows = 32;     // rows per block (one warp-width of accumulators per thread)
constexpr int kMapThreads = 256;
constexpr int kMapKChunk = 128;  // input columns staged per pass

// Block = 32 rows x all outputs.  The 32-row input tile is staged transposed ([k][row]) one K
// chunk at a time; thread t owns outputs t, t + 256, ... and keeps 32 row accumulators.  Mt is
// stored k-major ([din][dout]), so a warp's 32 consecutive outputs read one coalesced segment.
__global__ void __launch_bounds__(kMapThreads) dense_map_kernel(const float* __restrict__ in, int din,
                                                                const float* __restrict__ mt, int dout,
                                                                float* __restrict__ out, int64_t rows) {
  __shared__ float4 tile[kMapKChunk][kMapRows / 4];
  const int64_t row0 = static_cast<int64_t>(blockIdx.x) * kMapRows;
  const int nr = static_cast<int>(rows - row0 < kMapRows ? rows - row0 : kMapRows);
  for (int o0 = 0; o0 < dout; o0 += kMapThreads) {
    const int o = o0 + threadIdx.x;
    float acc[kMapRows];
#pragma unroll
    for (int r = 0; r < kMapRows; ++r) acc[r] = 0.f;
    for (int k0 = 0; k0 < din; k0 += kMapKChunk) {
      const int kc = min(kMapKChunk, din - k0);
      __syncthreads();
      float* tf = reinterpret_cast<float*>(tile);
      for (int i = threadIdx.x; i < kMapKChunk * kMapRows; i += kMapThreads) {
        const int r = i / kMapKChunk, k = i % kMapKChunk;  // coalesced along k
        tf[k * kMapRows + r] = (r < nr && k < kc) ? in[(row0 + r) * din + k0 + k] : 0.f;
      }
      __syncthreads();
      if (o < dout) {
        for (int k = 0; k < kc; ++k) {
          const float m = __ldg(mt + static_cast<int64_t>(k0 + k) * dout + o);
#pragma unroll
          for (int r4 = 0; r4 < kMapRows / 4; ++r4) {
            const float4 v = tile[k][r4];  // broadcast
            acc[4 * r4] = fmaf(m, v.x, acc[4 * r4]);
            acc[4 * r4 + 1] = fmaf(m, v.y, acc[4 * r4 + 1]);
            acc[4 * r4 + 2] = fmaf(m, v.z, acc[4 * r4 + 2]);
            acc[4 * r4 + 3] = fmaf(m, v.w, acc[4 * r4 + 3]);
          }
        }
      }
    }
    if (o < dout)
#pragma unroll
      for (int r = 0; r < kMapRows; ++r)
        if (r < nr) out[(row0 + r) * dout + o] = acc[r];
  }
}

// one block per product: X, Y staged in shared memory, thread per output entry
__global__ void __launch_bounds__(256) carrier_matmul_kernel(const float* __restrict__ X, const float* __restrict__ Y,
                                                             float* __restrict__ Z, int dt) {
  extern __shared__ float sm[];
  float* xs = sm;
  float* ys = sm + dt * dt;
  const int64_t b = blockIdx.x;
  const int n = dt * dt;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    xs[i] = X[b * n + i];
    ys[i] = Y[b * n + i];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    const int i = e / dt, j = e % dt;
    float acc = 0.f;
    for (int k = 0; k < dt; ++k) acc = fmaf(xs[i * dt + k], ys[k * dt + j], acc);
    Z[b * n + e] = acc;
  }
}

__global__ void pointwise_mul_kernel(const float* __restrict__ a, const float* __restrict__ b, float* __restrict__ out,
                                     int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = a[i] * b[i];
}

// D^1 in the (y, z, x) component order: D1[i][j] = u_i . R u_j (proj/src/wigner.cpp:292-300)
__device__ __forceinline__ int yzx(int i) { return i == 0 ? 1 : (i == 1 ? 2 : 0); }

// One block per rotation, fp64.  Level l: D^l[i][j] = sum_{a in Q_i} sum_{b in Q_j} a.v b.v D1[a.m1][b.m1]
// D^{l-1}[a.m2][b.m2], Q_i = entries of cg_real(1, l-1, l) with m3 = i (host-grouped), thread per (i, j).
__global__ void __launch_bounds__(256) wigner_d_kernel(WignerTables w, const double* __restrict__ R,
                                                       double* __restrict__ D, int64_t n) {
  extern __shared__ double dsm[];
  const int L = w.L;
  const int dmax = 2 * L + 1;
  double* prev = dsm;               // D^{l-1}
  double* cur = dsm + dmax * dmax;  // D^l
  __shared__ double d1[9];
  const int64_t rot = blockIdx.x;
  const double* Rr = R + rot * 9;
  double* out = D + rot * w.d_stride;
  if (threadIdx.x < 9) {
    const int i = threadIdx.x / 3, j = threadIdx.x % 3;
    d1[threadIdx.x] = Rr[yzx(i) * 3 + yzx(j)];
  }
  if (threadIdx.x == 0) out[0] = 1.0;
  __syncthreads();
  if (L >= 1) {
    for (int e = threadIdx.x; e < 9; e += blockDim.x) {
      prev[e] = d1[e];
      out[1 + e] = d1[e];
    }
  }
  __syncthreads();
  for (int l = 2; l <= L; ++l) {
    const int d = 2 * l + 1, dp = 2 * l - 1;
    const int* off = w.row_off + w.l_off[l];  // [d + 1] offsets into the level's entries
    const WignerEntry* q = w.entries + w.e_off[l];
    for (int e = threadIdx.x; e < d * d; e += blockDim.x) {
      const int i = e / d, j = e % d;
      double acc = 0.0;
      for (int a = off[i]; a < off[i + 1]; ++a)
        for (int b = off[j]; b < off[j + 1]; ++b)
          acc += q[a].v * q[b].v * d1[q[a].m1 * 3 + q[b].m1] * prev[q[a].m2 * dp + q[b].m2];
      cur[e] = acc;
    }
    __syncthreads();
    const int64_t base = w.block_off[l];
    for (int e = threadIdx.x; e < d * d; e += blockDim.x) {
      out[base + e] = cur[e];
      prev[e] = cur[e];
    }
    __syncthreads();
  }
}

// out[row][(l, i)] = sum_j D^l[i][j] x[row][(l, j)], rotation of row = (row / channels) * n_rot / batch
__global__ void rotate_kernel(const double* __restrict__ D, int64_t d_stride, int64_t n_rot, const float* __restrict__ x,
                              float* __restrict__ out, int64_t rows, int64_t channels, int64_t batch, int L,
                              const int64_t* __restrict__ block_off) {
  const int din = (L + 1) * (L + 1);
  const int64_t total = rows * din;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = idx / din;
    const int k = static_cast<int>(idx - row * din);
    const int l = static_cast<int>(sqrtf(static_cast<float>(k) + 0.5f));
    const int i = k - l * l, d = 2 * l + 1;
    const int64_t rot = (row / channels) * n_rot / batch;
    const double* Dl = D + rot * d_stride + block_off[l] + static_cast<int64_t>(i) * d;
    const float* xr = x + row * din + l * l;
    double acc = 0.0;
    for (int j = 0; j < d; ++j) acc += Dl[j] * static_cast<double>(xr[j]);
    out[idx] = static_cast<float>(acc);
  }
}

__global__ void path_scale_kernel(float* __restrict__ out, int64_t rows, int64_t channels, int dout,
                                  const int* __restrict__ path_of_out, const float* __restrict__ w, int64_t w_stride) {
  const int64_t total = rows * dout;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = i / dout;
    const int o = static_cast<int>(i - row * dout);
    out[i] *= __ldg(w + (row / channels) * w_stride + __ldg(path_of_out + o));
  }
}

int grid_for(int64_t work, int per_block, int num_sms) {
  const int64_t b = (work + per_block - 1) / per_block;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(b, static_cast<int64_t>(num_sms) * 8)));
}

}  // namespace

cudaError_t launch_path_scale(float* out, int64_t rows, int64_t channels, int dout, const int* path_of_out,
                              const float* w, int64_t w_stride, int num_sms, cudaStream_t s) {
  if (rows <= 0 || dout <= 0) return cudaSuccess;
  path_scale_kernel<<<grid_for(rows * dout, 256 * 4, num_sms), 256, 0, s>>>(out, rows, channels, dout, path_of_out, w,
                                                                            w_stride);
  return cudaGetLastError();
}

cudaError_t launch_dense_map(const float* in, int din, const float* mt, int dout, float* out, int64_t rows,
                             cudaStream_t s) {
  if (rows <= 0 || dout <= 0) return cudaSuccess;
  const int64_t blocks = (rows + kMapRows - 1) / kMapRows;
  dense_map_kernel<<<static_cast<unsigned>(blocks), kMapThreads, 0, s>>>(in, din, mt, dout, out, rows);
  return cudaGetLastError();
}

cudaError_t launch_carrier_matmul(const float* X, const float* Y, float* Z, int dt, int64_t batch, cudaStream_t s) {
  if (batch <= 0) return cudaSuccess;
  const int smem = 2 * dt * dt * 4;
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(carrier_matmul_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
  }
  carrier_matmul_kernel<<<static_cast<unsigned>(batch), 256, smem, s>>>(X, Y, Z, dt);
  return cudaGetLastError();
}

cudaError_t launch_pointwise_mul(const float* a, const float* b, float* out, int64_t n, int num_sms, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  pointwise_mul_kernel<<<grid_for(n, 256 * 4, num_sms), 256, 0, s>>>(a, b, out, n);
  return cudaGetLastError();
}

cudaError_t launch_wigner_d(const WignerTables& w, const double* R, double* D, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int dmax = 2 * w.L + 1;
  const int smem = 2 * dmax * dmax * 8;
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(wigner_d_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
  }
  wigner_d_kernel<<<static_cast<unsigned>(n), 256, smem, s>>>(w, R, D, n);
  return cudaGetLastError();
}

cudaError_t launch_rotate(const WignerTables& w, const double* D, int64_t n_rot, const float* x, float* out,
                          int64_t batch, int64_t channels, int num_sms, cudaStream_t s) {
  const int64_t rows = batch * channels;
  if (rows <= 0) return cudaSuccess;
  const int64_t work = rows * (w.L + 1) * (w.L + 1);
  rotate_kernel<<<grid_for(work, 256, num_sms), 256, 0, s>>>(D, w.d_stride, n_rot, x, out, rows, channels, batch, w.L,
                                                            w.block_off_dev);
  return cudaGetLastError();
}

}  // namespace tpo_b200
