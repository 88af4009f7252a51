// Path-sparse Clebsch-Gordan tensor product (SIMT).
//
// Reference: tpo::cgtp_mimo with CgtpImpl::sparse (proj/src/cgtp.cpp:145-177,
// 120-143).  The reference walks every path (l1,l2,l3) and contracts its real
// CG table with 4 shifted-diagonal passes.  Here the whole MIMO product is
// flattened into one gather per output coefficient o = (path, m3):
//   out[o] = sum_t c_t * x[i1_t] * y[i2_t]
// over exactly the nonzero real-CG entries (structural zeros are never
// visited).
//
// Layout: a block owns a tile of kRows (sample, channel) rows staged in shared
// memory and sweeps every output pass of kCgtpChunk coefficients over it, so
// the tile is read from HBM once and every term fetch (8 B, coalesced,
// warp-padded) is reused kRows times from registers.  Output stores are whole
// 1 KB row segments per pass (coalesced).  The path is HBM-bound for the
// BASELINE configs (outputs are (L+1)^4 floats per product).
//
// Shared-y mode (config C4: one y per edge, x per channel): when a tile lies
// inside one edge, c_t * y[i2_t] is folded once per term and the inner loop is
// one shared-memory load and one FMA per term-row.
#include <algorithm>

#include "kernels.hpp"

namespace tpo_b200 {
namespace {

constexpr int kRows = 32;  // rows per tile

// Tiles are stored transposed, xs[i][r] (row index fastest, pitch kPitch), so
// one 128-bit shared load fetches a coefficient for 4 rows and the products
// run as packed f32x2 FMAs: per term and 32 rows, 8 LDS.128 + 16 FFMA2
// (shared-y tiles) instead of 32 LDS + 32 FFMA.
constexpr int kPitch = kRows + 4;  // 144 B: consecutive coefficients start 4 banks apart

constexpr int kPf = 8;  // prefetch registers per thread and input (tiles of din <= 64)

template <bool kEdgeTile>
__global__ void __launch_bounds__(kCgtpChunk)
    cgtp_kernel(const __grid_constant__ CgtpTables t, const __grid_constant__ RowSpec rs) {
  extern __shared__ __align__(16) float sm[];
  const int buf_floats = (t.din1 + t.din2) * kPitch;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t ntiles = (rs.rows + kRows - 1) / kRows;
  // element e of a tile is (row e % 32, coefficient e / 32): consecutive lanes take consecutive
  // rows, so the transposed shared-memory stores xs[k][r] hit consecutive banks
  // register prefetch of the next tile for shared-y edge tiles (config C4); other shapes load
  // synchronously with coalesced reads (fewer registers -> more resident blocks)
  const bool prefetch = kEdgeTile && t.din1 * kRows <= kPf * kCgtpChunk;
  float px[kPf];
  auto load_regs = [&](int64_t tile) {
    const int64_t row0 = tile * kRows;
#pragma unroll
    for (int q = 0; q < kPf; ++q) {
      const int e = tid + q * kCgtpChunk;
      const int r = e & (kRows - 1), k = e >> 5;
      const int64_t g = row0 + r;
      px[q] = (k < t.din1 && tile < ntiles && g < rs.rows) ? __ldg(rs.x + g * t.din1 + k) : 0.f;

    }
  };
  int b = 0;
  if (prefetch) load_regs(blockIdx.x);
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, b ^= (prefetch ? 1 : 0)) {
    const int64_t row0 = tile * kRows;
    const int64_t left = rs.rows - row0;
    const int nr = left < kRows ? static_cast<int>(left) : kRows;
    float* xs = sm + b * buf_floats;       // [din1][kPitch]
    float* ys = xs + t.din1 * kPitch;      // [din2][kPitch] (edge tiles: [din2])
    if (prefetch) {
      // double-buffered tiles: the readers of buffer b finished before the previous barrier
#pragma unroll
      for (int q = 0; q < kPf; ++q) {
        const int e = tid + q * kCgtpChunk;
        const int r = e & (kRows - 1), k = e >> 5;
        if (k < t.din1) xs[k * kPitch + r] = px[q];
      }
    } else {
      __syncthreads();  // single buffer: previous tile's readers are done
      for (int i = tid; i < kRows * t.din1; i += kCgtpChunk) {  // coalesced rows
        const int r = i / t.din1, k = i - r * t.din1;
        xs[k * kPitch + r] = r < nr ? __ldg(rs.x + row0 * t.din1 + i) : 0.f;
      }
      if (!kEdgeTile)
        for (int i = tid; i < kRows * t.din2; i += kCgtpChunk) {
          const int r = i / t.din2, k = i - r * t.din2;
          const int64_t g = row0 + r;
          const int64_t yr = rs.y_shared ? g / rs.channels : g;
          ys[k * kPitch + r] = r < nr ? __ldg(rs.y + yr * t.din2 + k) : 0.f;
        }
    }
    if (kEdgeTile)
      for (int k = tid; k < t.din2; k += kCgtpChunk) ys[k] = __ldg(rs.y + (row0 / rs.channels) * t.din2 + k);
    __syncthreads();
    if (prefetch) load_regs(tile + gridDim.x);  // in flight during this tile's compute
    for (int q = 0; q < t.nchunks; ++q) {
      const int o = q * kCgtpChunk + tid;
      const int wid = q * (kCgtpChunk / 32) + warp;
      const int nt = __ldg(t.warp_nt + wid);
      const uint2* terms = t.terms + __ldg(t.warp_off + wid) + lane;
      float2 acc[kRows / 2];
#pragma unroll
      for (int r = 0; r < kRows / 2; ++r) acc[r] = make_float2(0.f, 0.f);
      for (int k = 0; k < nt; ++k) {
        const uint2 w = __ldg(terms + k * 32);
        const int i1 = static_cast<int>(w.x & 0xFFFFu), i2 = static_cast<int>(w.x >> 16);
        const float c = __uint_as_float(w.y);
        const float4* xr = reinterpret_cast<const float4*>(xs + i1 * kPitch);
        if (kEdgeTile) {
          const float cy = c * ys[i2];
          const float2 cy2 = make_float2(cy, cy);
#pragma unroll
          for (int r4 = 0; r4 < kRows / 4; ++r4) {
            const float4 v = xr[r4];
            acc[2 * r4] = __ffma2_rn(cy2, make_float2(v.x, v.y), acc[2 * r4]);
            acc[2 * r4 + 1] = __ffma2_rn(cy2, make_float2(v.z, v.w), acc[2 * r4 + 1]);
          }
        } else {
          const float4* yr = reinterpret_cast<const float4*>(ys + i2 * kPitch);
          const float2 c2 = make_float2(c, c);
#pragma unroll
          for (int r4 = 0; r4 < kRows / 4; ++r4) {
            const float4 v = xr[r4], u = yr[r4];
            const float2 p0 = __fmul2_rn(c2, make_float2(v.x, v.y));
            const float2 p1 = __fmul2_rn(c2, make_float2(v.z, v.w));
            acc[2 * r4] = __ffma2_rn(p0, make_float2(u.x, u.y), acc[2 * r4]);
            acc[2 * r4 + 1] = __ffma2_rn(p1, make_float2(u.z, u.w), acc[2 * r4 + 1]);
          }
        }
      }
      if (o < t.dout) {
        float* op = rs.out + row0 * t.dout + o;
#pragma unroll
        for (int r = 0; r < kRows; ++r)
          if (r < nr) op[static_cast<int64_t>(r) * t.dout] = (r & 1) ? acc[r >> 1].y : acc[r >> 1].x;
      }
    }
  }
}

}  // namespace

cudaError_t launch_cgtp(const CgtpTables& t, const RowSpec& rs, int num_sms, cudaStream_t s) {
  if (rs.rows <= 0) return cudaSuccess;
  // every tile inside one edge: channels a multiple of the tile height
  const bool edge = rs.y_shared && rs.channels % kRows == 0;
  // edge tiles with register prefetch use a double-buffered tile
  const bool dbl = edge && t.din1 * kRows <= kPf * kCgtpChunk;
  const size_t smem = (dbl ? 2 : 1) * sizeof(float) * kPitch * (t.din1 + t.din2);
  auto kern = edge ? cgtp_kernel<true> : cgtp_kernel<false>;
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
