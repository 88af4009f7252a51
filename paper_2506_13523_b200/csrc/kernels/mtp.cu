// Matrix tensor product (SIMT, batched small matrices).
//
// Reference: tpo::mtp with MtpImpl::sparse (proj/src/mtp.cpp:99-117):
// embed both inputs into (2lt+1)^2 carrier matrices through the real CG
// tables (proj/src/mtp.cpp:20-58), classical cubic matmul Z = X Y
// (:119-133, sub-cubic forbidden by the cost model), extract every output
// degree by the adjoint CG contraction (:60-97).
//
// A block owns a tile of R products with all intermediates in shared memory
// (odd row pitches, so column-wise reads are bank-conflict free).  The embed
// and extract maps are CSR gather lists over the CG nonzeros (host/context.cpp);
// each list entry is fetched once per tile and applied to all R products from
// registers.  The R x dt matmul row tasks keep one output row of Z in
// registers and stream X / Y from shared memory.
#include <algorithm>
#include <cstdlib>

#include "kernels.hpp"

namespace tpo_b200 {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxDt = 33;  // lt <= 16

template <int R, int ZR>
__global__ void __launch_bounds__(kThreads)
    mtp_kernel(const __grid_constant__ MtpDevTables t, const __grid_constant__ RowSpec rs) {
  extern __shared__ float sm[];
  const int dt = t.dt, dt2 = dt * dt;
  const int px = t.din1 | 1, py = t.din2 | 1, pc = dt2 | 1;
  float* xs = sm;             // [R][px]
  float* ys = xs + R * px;    // [R][py]
  float* X = ys + R * py;     // [R][pc]
  float* Y = X + R * pc;      // [R][pc]
  float* Z = Y + R * pc;      // [R][pc]
  const int tid = threadIdx.x;
  const int64_t ntiles = (rs.rows + R - 1) / R;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row0 = tile * R;
    const int64_t left = rs.rows - row0;
    const int nr = left < R ? static_cast<int>(left) : R;
    __syncthreads();
    for (int i = tid; i < R * t.din1; i += kThreads) {
      const int r = i / t.din1, k = i - r * t.din1;
      xs[r * px + k] = r < nr ? __ldg(rs.x + row0 * t.din1 + i) : 0.f;
    }
    for (int i = tid; i < R * t.din2; i += kThreads) {
      const int r = i / t.din2, k = i - r * t.din2;
      const int64_t g = row0 + r;
      const int64_t yr = rs.y_shared ? g / rs.channels : g;
      ys[r * py + k] = r < nr ? __ldg(rs.y + yr * t.din2 + k) : 0.f;
    }
    __syncthreads();
    // ---- embed (proj/src/mtp.cpp:20-58): X[cell] = sum_e c_e x[idx_e]
    for (int cell = tid; cell < 2 * dt2; cell += kThreads) {
      const bool second = cell >= dt2;
      const int cl = second ? cell - dt2 : cell;
      const int* off = second ? t.emb2_off : t.emb1_off;
      const int* idx = second ? t.emb2_idx : t.emb1_idx;
      const float* cf = second ? t.emb2_c : t.emb1_c;
      const float* src = second ? ys : xs;
      const int pitch = second ? py : px;
      float acc[R];
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = 0.f;
      for (int e = __ldg(off + cl), e1 = __ldg(off + cl + 1); e < e1; ++e) {
        const float c = __ldg(cf + e);
        const int k = __ldg(idx + e);
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = fmaf(c, src[r * pitch + k], acc[r]);
      }
      float* dst = (second ? Y : X) + cl;
#pragma unroll
      for (int r = 0; r < R; ++r) dst[r * pc] = acc[r];
    }
    __syncthreads();
    // ---- Z = X Y, classical cubic (proj/src/mtp.cpp:119-133): task = (row r, Z rows i0 .. i0+ZR-1);
    // every Y element loaded from shared memory feeds ZR rows
    const int ntr = (dt + ZR - 1) / ZR;
    for (int task = tid; task < R * ntr; task += kThreads) {
      const int r = task / ntr, i0 = (task - r * ntr) * ZR;
      const float* xr = X + r * pc + i0 * dt;
      const float* yb = Y + r * pc;
      float acc[ZR][kMaxDt];
#pragma unroll
      for (int q = 0; q < ZR; ++q)
#pragma unroll
        for (int j = 0; j < kMaxDt; ++j) acc[q][j] = 0.f;
      for (int k = 0; k < dt; ++k) {
        float a[ZR];
#pragma unroll
        for (int q = 0; q < ZR; ++q) a[q] = i0 + q < dt ? xr[q * dt + k] : 0.f;
        const float* yk = yb + k * dt;
        // 8-wide blocks guarded as a whole: no issue slots spent past dt
#pragma unroll
        for (int j0 = 0; j0 < kMaxDt; j0 += 8) {
          if (j0 < dt) {
#pragma unroll
            for (int jj = 0; jj < 8; ++jj)
              if (j0 + jj < kMaxDt && j0 + jj < dt) {
                const float yv = yk[j0 + jj];
#pragma unroll
                for (int q = 0; q < ZR; ++q) acc[q][j0 + jj] = fmaf(a[q], yv, acc[q][j0 + jj]);
              }
          }
        }
      }
#pragma unroll
      for (int q = 0; q < ZR; ++q) {
        if (i0 + q >= dt) break;
        float* zr = Z + r * pc + (i0 + q) * dt;
#pragma unroll
        for (int j = 0; j < kMaxDt; ++j)
          if (j < dt) zr[j] = acc[q][j];
      }
    }
    __syncthreads();
    // ---- extract (proj/src/mtp.cpp:60-97): out[o] = sum_e c_e Z[cell_e]; zero past the carrier band
    for (int o = tid; o < t.dout_total; o += kThreads) {
      float acc[R];
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = 0.f;
      if (o < t.dout_eff) {
        for (int e = __ldg(t.ext_off + o), e1 = __ldg(t.ext_off + o + 1); e < e1; ++e) {
          const float c = __ldg(t.ext_c + e);
          const int cell = __ldg(t.ext_idx + e);
#pragma unroll
          for (int r = 0; r < R; ++r) acc[r] = fmaf(c, Z[r * pc + cell], acc[r]);
        }
      }
      float* op = rs.out + row0 * t.dout_total + o;
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (r < nr) op[static_cast<int64_t>(r) * t.dout_total] = acc[r];
    }
  }
}

template <int R, int ZR>
cudaError_t launch_rz(const MtpDevTables& t, const RowSpec& rs, int num_sms, cudaStream_t s) {
  const int dt2 = t.dt * t.dt;
  const size_t smem = sizeof(float) * R * ((t.din1 | 1) + (t.din2 | 1) + 3 * (dt2 | 1));
  cudaError_t e = cudaFuncSetAttribute(mtp_kernel<R, ZR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, mtp_kernel<R, ZR>, kThreads, smem);
  const int64_t ntiles = (rs.rows + R - 1) / R;
  const int grid = static_cast<int>(std::min<int64_t>(ntiles, static_cast<int64_t>(num_sms) * std::max(occ, 1)));
  mtp_kernel<R, ZR><<<grid, kThreads, smem, s>>>(t, rs);
  return cudaGetLastError();
}

// Z rows per matmul task: 2 measured fastest at every dt (fewer shared loads per FMA beats the
// lost task parallelism; tools/mtp_simt_timing.py); TPO_MTP_ZR=1|3 for experiments
template <int R>
cudaError_t launch_r(const MtpDevTables& t, const RowSpec& rs, int num_sms, cudaStream_t s) {
  static const int zr = [] {
    const char* v = std::getenv("TPO_MTP_ZR");
    return v ? std::atoi(v) : 2;
  }();
  if (zr == 1) return launch_rz<R, 1>(t, rs, num_sms, s);
  if (zr == 3) return launch_rz<R, 3>(t, rs, num_sms, s);
  return launch_rz<R, 2>(t, rs, num_sms, s);
}

}  // namespace

cudaError_t launch_mtp(const MtpDevTables& t, const RowSpec& rs, int num_sms, cudaStream_t s) {
  if (rs.rows <= 0) return cudaSuccess;
  if (t.dt > kMaxDt) return cudaErrorInvalidValue;
  // rows per tile: as many as keep >= 2 blocks per SM within 227 KB
  const int per_row = ((t.din1 | 1) + (t.din2 | 1) + 3 * ((t.dt * t.dt) | 1)) * 4;
  if (per_row * 32 <= 110 * 1024) return launch_r<32>(t, rs, num_sms, s);
  if (per_row * 16 <= 110 * 1024) return launch_r<16>(t, rs, num_sms, s);
  if (per_row * 8 <= 220 * 1024) return launch_r<8>(t, rs, num_sms, s);
  return launch_r<4>(t, rs, num_sms, s);
}

}  // namespace tpo_b200
