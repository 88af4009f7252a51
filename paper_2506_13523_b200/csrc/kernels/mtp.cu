// Matrix tensor product (SIMT, batched small matrices).
//
// Reference: tpo::mtp with MtpImpl::sparse (proj/src/mtp.cpp:99-117):
// embed both inputs into (2lt+1)^2 carrier matrices through the real CG
// tables (proj/src/mtp.cpp:20-58), classical cubic matmul Z = X Y
// (:119-133, sub-cubic forbidden by the cost model), extract every output
// degree by the adjoint CG contraction (:60-97).  The embed / extract maps
// are flattened on the host into per-cell and per-output gather lists over
// the CG nonzeros; a block keeps `rows_per_block` products resident in
// shared memory and runs the three phases with all threads.
#include <algorithm>

#include "kernels.hpp"

namespace tpo_b200 {
namespace {

constexpr int kThreads = 256;

__global__ void __launch_bounds__(kThreads)
    mtp_kernel(const __grid_constant__ MtpDevTables t, const __grid_constant__ RowSpec rs, int R) {
  extern __shared__ float sm[];
  const int dt2 = t.dt * t.dt;
  float* xs = sm;                 // [R][din1]
  float* ys = xs + R * t.din1;    // [R][din2]
  float* X = ys + R * t.din2;     // [R][dt2]
  float* Y = X + R * dt2;         // [R][dt2]
  float* Z = Y + R * dt2;         // [R][dt2]
  const int64_t ntiles = (rs.rows + R - 1) / R;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row0 = tile * R;
    const int nr = static_cast<int>(std::min<int64_t>(R, rs.rows - row0));
    // rows are contiguous in global memory: linear, coalesced loads
    for (int i = threadIdx.x; i < nr * t.din1; i += kThreads) xs[i] = __ldg(rs.x + row0 * t.din1 + i);
    for (int i = threadIdx.x; i < nr * t.din2; i += kThreads) {
      const int r = i / t.din2, k = i - r * t.din2;
      const int64_t g = row0 + r;
      ys[i] = __ldg(rs.y + (rs.y_shared ? g / rs.channels : g) * t.din2 + k);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nr * dt2; i += kThreads) {  // embed (sparse CG gather)
      const int r = i / dt2, cell = i - r * dt2;
      float ax = 0.f, ay = 0.f;
      for (int e = __ldg(t.emb1_off + cell), e1 = __ldg(t.emb1_off + cell + 1); e < e1; ++e)
        ax = fmaf(__ldg(t.emb1_c + e), xs[r * t.din1 + __ldg(t.emb1_idx + e)], ax);
      for (int e = __ldg(t.emb2_off + cell), e1 = __ldg(t.emb2_off + cell + 1); e < e1; ++e)
        ay = fmaf(__ldg(t.emb2_c + e), ys[r * t.din2 + __ldg(t.emb2_idx + e)], ay);
      X[i] = ax;
      Y[i] = ay;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nr * dt2; i += kThreads) {  // Z = X Y, classical cubic
      const int r = i / dt2, cell = i - r * dt2;
      const int a = cell / t.dt, b = cell - a * t.dt;
      const float* xr = X + r * dt2 + a * t.dt;
      const float* yc = Y + r * dt2 + b;
      float acc = 0.f;
      for (int k = 0; k < t.dt; ++k) acc = fmaf(xr[k], yc[k * t.dt], acc);
      Z[i] = acc;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nr * t.dout_total; i += kThreads) {  // extract
      const int r = i / t.dout_total, o = i - r * t.dout_total;
      float acc = 0.f;
      if (o < t.dout_eff)
        for (int e = __ldg(t.ext_off + o), e1 = __ldg(t.ext_off + o + 1); e < e1; ++e)
          acc = fmaf(__ldg(t.ext_c + e), Z[r * dt2 + __ldg(t.ext_idx + e)], acc);
      rs.out[row0 * t.dout_total + i] = acc;
    }
    __syncthreads();
  }
}

}  // namespace

cudaError_t launch_mtp(const MtpDevTables& t, const RowSpec& rs, int num_sms, cudaStream_t s) {
  if (rs.rows <= 0) return cudaSuccess;
  const int per_row = t.din1 + t.din2 + 3 * t.dt * t.dt;
  int R = std::max(1, std::min(32, (40 * 1024 / 4) / per_row));
  const size_t smem = sizeof(float) * static_cast<size_t>(R) * per_row;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(mtp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, mtp_kernel, kThreads, smem);
  const int64_t ntiles = (rs.rows + R - 1) / R;
  const int grid = static_cast<int>(std::min<int64_t>(ntiles, static_cast<int64_t>(num_sms) * std::max(occ, 1)));
  mtp_kernel<<<grid, kThreads, smem, s>>>(t, rs, R);
  return cudaGetLastError();
}

}  // namespace tpo_b200
