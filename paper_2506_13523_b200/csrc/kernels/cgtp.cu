// Path-sparse Clebsch-Gordan tensor product (SIMT).
//
// Reference: tpo::cgtp_mimo with CgtpImpl::sparse (proj/src/cgtp.cpp:145-177,
// 120-143).  The reference walks every path (l1,l2,l3) and contracts its real
// CG table with 4 shifted-diagonal passes.  Here the whole MIMO product is
// flattened into one gather per output coefficient o = (path, m3):
//   out[o] = sum_t c_t * x[i1_t] * y[i2_t]
// over exactly the nonzero real-CG entries (structural zeros are never
// visited).  Term lists are padded per 128-output chunk and stored
// term-major so a warp reads them coalesced; each thread owns one output
// column and sweeps a 16-row tile of (sample, channel) rows staged in shared
// memory, so one term fetch is reused 16 times and the output stores of a
// warp are 128 contiguous bytes.
#include <algorithm>

#include "kernels.hpp"

namespace tpo_b200 {
namespace {

constexpr int kRows = 16;  // rows per tile

__global__ void __launch_bounds__(kCgtpChunk)
    cgtp_kernel(const __grid_constant__ CgtpTables t, const __grid_constant__ RowSpec rs) {
  extern __shared__ float sm[];
  float* xs = sm;                       // [kRows][din1]
  float* ys = sm + kRows * t.din1;      // [kRows][din2]
  // linear block id = tile * nchunks + chunk: the chunks of one row tile run
  // back to back, so the tile's x/y rows and the term table stay L2-resident
  const int q = static_cast<int>(blockIdx.x % static_cast<unsigned>(t.nchunks));  // output chunk
  const int64_t tile = blockIdx.x / static_cast<unsigned>(t.nchunks);
  const int o = q * kCgtpChunk + threadIdx.x;
  const int nt = t.chunk_nt[q];
  const uint2* terms = t.terms + t.chunk_off[q] + threadIdx.x;
  const int64_t row0 = tile * kRows;

  for (int i = threadIdx.x; i < kRows * t.din1; i += blockDim.x) {
    const int r = i / t.din1, k = i - r * t.din1;
    const int64_t g = row0 + r;
    xs[i] = g < rs.rows ? __ldg(rs.x + g * t.din1 + k) : 0.f;
  }
  for (int i = threadIdx.x; i < kRows * t.din2; i += blockDim.x) {
    const int r = i / t.din2, k = i - r * t.din2;
    const int64_t g = row0 + r;
    const int64_t yr = rs.y_shared ? g / rs.channels : g;
    ys[i] = g < rs.rows ? __ldg(rs.y + yr * t.din2 + k) : 0.f;
  }
  __syncthreads();

  float acc[kRows];
#pragma unroll
  for (int r = 0; r < kRows; ++r) acc[r] = 0.f;
  for (int tt = 0; tt < nt; ++tt) {
    const uint2 w = __ldg(terms + static_cast<size_t>(tt) * kCgtpChunk);
    const int i1 = static_cast<int>(w.x & 0xFFFFu), i2 = static_cast<int>(w.x >> 16);
    const float c = __uint_as_float(w.y);
#pragma unroll
    for (int r = 0; r < kRows; ++r) acc[r] = fmaf(c * xs[r * t.din1 + i1], ys[r * t.din2 + i2], acc[r]);
  }
  if (o < t.dout) {
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      const int64_t g = row0 + r;
      if (g < rs.rows) rs.out[g * t.dout + o] = acc[r];
    }
  }
}

}  // namespace

cudaError_t launch_cgtp(const CgtpTables& t, const RowSpec& rs, cudaStream_t s) {
  if (rs.rows <= 0) return cudaSuccess;
  const int64_t tiles = (rs.rows + kRows - 1) / kRows;
  const size_t smem = sizeof(float) * kRows * (t.din1 + t.din2);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(cgtp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  const int64_t nblocks = tiles * t.nchunks;
  if (nblocks > 2147483647LL) return cudaErrorInvalidConfiguration;  // caller chunks the batch
  cgtp_kernel<<<static_cast<unsigned>(nblocks), kCgtpChunk, smem, s>>>(t, rs);
  return cudaGetLastError();
}

}  // namespace tpo_b200
