// CGTP backward (vector-Jacobian products), SIMT.
//
// Forward (cgtp.cu, proj/src/cgtp.cpp:120-177): out[o] = sum_t c_t x[i1_t] y[i2_t].
// Backward: grad_x[a] = sum_{t: i1_t = a} c_t g[o_t] y[i2_t] (and likewise
// grad_y), i.e. the same real-CG nonzeros regrouped by input coefficient.
//
// The result has only D_in = (L+1)^2 coefficients per row while grad_out has
// (L+1)^4, so the forward kernel's "one thread per output, whole input row
// staged" layout does not carry over: grad_out rows do not fit in shared
// memory at L >= 6, and D_in outputs would leave most of a 256-thread block
// idle.  Here a block owns kRows = 32 rows, sweeps grad_out in windows of
// dwin columns (staged transposed like the forward tiles), keeps the partial
// sums in registers across windows, and deals each output's term list over
// nsplit virtual outputs; one shared-memory reduction and one store per tile.
// (Measured alternatives, tools/ab_cgtp_bwd.sh: separate launches per window
// accumulating in HBM; per-window thread maps with shared atomics -- 3-5x
// slower at L <= 3, no better at L = 6.)
#include <algorithm>

#include "kernels.hpp"

namespace tpo_b200 {
namespace {

constexpr int kRows = 32;
constexpr int kPitch = kRows + 4;  // as in cgtp.cu: LDS.128 over 4 rows, 4-bank skew per coefficient

template <bool kShared>  // kShared: the other input is one row per edge (tile inside one edge)
__global__ void __launch_bounds__(kCgtpChunk)
    cgtp_bwd_kernel(const __grid_constant__ CgtpBwdTables t, const __grid_constant__ RowSpec rs) {
  extern __shared__ __align__(16) float sm[];
  float* gs = sm;                       // [dwin][kPitch]  grad_out window, transposed
  float* vs = sm + t.dwin * kPitch;     // [dother][kPitch] (kShared: [dother])
  const bool alias = t.dwin * kPitch >= kCgtpChunk * (kRows + 1);
  float* red = alias ? sm : vs + (kShared ? (t.dother + 3) / 4 * 4 : t.dother * kPitch);  // [256][kRows + 1]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t ntiles = (rs.rows + kRows - 1) / kRows;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row0 = tile * kRows;
    const int64_t left = rs.rows - row0;
    const int nr = left < kRows ? static_cast<int>(left) : kRows;
    __syncthreads();  // previous tile's readers (terms, reduction) are done
    if (kShared) {
      for (int k = tid; k < t.dother; k += kCgtpChunk) vs[k] = __ldg(rs.y + (row0 / rs.channels) * t.dother + k);
    } else {
      for (int i = tid; i < kRows * t.dother; i += kCgtpChunk) {
        const int r = i / t.dother, k = i - r * t.dother;
        const int64_t g = row0 + r;
        const int64_t yr = rs.y_shared ? g / rs.channels : g;
        vs[k * kPitch + r] = r < nr ? __ldg(rs.y + yr * t.dother + k) : 0.f;
      }
    }
    for (int q = 0; q < t.nchunks; ++q) {
      float2 acc[kRows / 2];
#pragma unroll
      for (int r = 0; r < kRows / 2; ++r) acc[r] = make_float2(0.f, 0.f);
      for (int w = 0; w < t.nwin; ++w) {
        const int64_t c0 = static_cast<int64_t>(w) * t.dwin;
        const int wc = static_cast<int>(min(static_cast<int64_t>(t.dwin), t.g_stride - c0));
        if (w > 0 || q > 0) __syncthreads();  // readers of the previous window are done
        for (int i = tid; i < kRows * wc; i += kCgtpChunk) {  // coalesced runs of wc floats
          const int r = i / wc, k = i - r * wc;
          gs[k * kPitch + r] = r < nr ? __ldg(rs.x + (row0 + r) * t.g_stride + c0 + k) : 0.f;
        }
        __syncthreads();
        const int wid = (q * t.nwin + w) * (kCgtpChunk / 32) + warp;
        const int nt = __ldg(t.warp_nt + wid);
        const uint2* terms = t.terms + __ldg(t.warp_off + wid) + lane;
        for (int k = 0; k < nt; ++k) {
          const uint2 tm = __ldg(terms + k * 32);
          const int io = static_cast<int>(tm.x & 0xFFFFu), iv = static_cast<int>(tm.x >> 16);
          const float c = __uint_as_float(tm.y);
          const float4* gr = reinterpret_cast<const float4*>(gs + io * kPitch);
          if (kShared) {
            const float cv = c * vs[iv];
            const float2 cv2 = make_float2(cv, cv);
#pragma unroll
            for (int r4 = 0; r4 < kRows / 4; ++r4) {
              const float4 a = gr[r4];
              acc[2 * r4] = __ffma2_rn(cv2, make_float2(a.x, a.y), acc[2 * r4]);
              acc[2 * r4 + 1] = __ffma2_rn(cv2, make_float2(a.z, a.w), acc[2 * r4 + 1]);
            }
          } else {
            const float4* vr = reinterpret_cast<const float4*>(vs + iv * kPitch);
            const float2 c2 = make_float2(c, c);
#pragma unroll
            for (int r4 = 0; r4 < kRows / 4; ++r4) {
              const float4 a = gr[r4], b = vr[r4];
              const float2 p0 = __fmul2_rn(c2, make_float2(a.x, a.y));
              const float2 p1 = __fmul2_rn(c2, make_float2(a.z, a.w));
              acc[2 * r4] = __ffma2_rn(p0, make_float2(b.x, b.y), acc[2 * r4]);
              acc[2 * r4 + 1] = __ffma2_rn(p1, make_float2(b.z, b.w), acc[2 * r4 + 1]);
            }
          }
        }
      }
      if (t.nsplit > 1) {  // single chunk: virtual output tid = p * dres + a
        if (alias) __syncthreads();  // the window tile becomes the reduction buffer
#pragma unroll
        for (int r = 0; r < kRows; ++r) red[tid * (kRows + 1) + r] = (r & 1) ? acc[r >> 1].y : acc[r >> 1].x;
        __syncthreads();
        for (int e = tid; e < nr * t.dres; e += kCgtpChunk) {
          const int r = e / t.dres, a = e - r * t.dres;
          float v = 0.f;
          for (int p = 0; p < t.nsplit; ++p) v += red[(p * t.dres + a) * (kRows + 1) + r];
          rs.out[(row0 + r) * t.dres + a] = v;
        }
      } else {
        const int a = q * kCgtpChunk + tid;
        if (a < t.dres) {
          float* op = rs.out + row0 * t.dres + a;
#pragma unroll
          for (int r = 0; r < kRows; ++r)
            if (r < nr) op[static_cast<int64_t>(r) * t.dres] = (r & 1) ? acc[r >> 1].y : acc[r >> 1].x;
        }
      }
    }
  }
}

}  // namespace

cudaError_t launch_cgtp_bwd(const CgtpBwdTables& t, const RowSpec& rs, int num_sms, cudaStream_t s) {
  if (rs.rows <= 0) return cudaSuccess;
  const bool shared = rs.y_shared && rs.channels % kRows == 0;
  const size_t tile = sizeof(float) * kPitch * t.dwin;
  const size_t other = sizeof(float) * (shared ? (t.dother + 3) / 4 * 4 : static_cast<size_t>(t.dother) * kPitch);
  const size_t red = sizeof(float) * kCgtpChunk * (kRows + 1);
  const size_t smem = tile + other + (t.nsplit > 1 && tile < red ? red : 0);
  auto kern = shared ? cgtp_bwd_kernel<true> : cgtp_bwd_kernel<false>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kCgtpChunk, smem);
  const int64_t ntiles = (rs.rows + kRows - 1) / kRows;
  const int grid = static_cast<int>(std::min<int64_t>(ntiles, static_cast<int64_t>(num_sms) * std::max(occ, 1)));
  kern<<<grid, kCgtpChunk, smem, s>>>(t, rs);
  return cudaGetLastError();
}

}  // namespace tpo_b200
