// Matrix tensor product (SIMT, batched small matrices) -- the path for carriers the tcgen05 kernel
// does not hold (dt = 2 lt + 1 > 13, i.e. L >= 7 at L3 = 2L, and any l_tilde override past that).
//
// Reference: tpo::mtp with MtpImpl::sparse (proj/src/mtp.cpp:99-117): embed both inputs into
// (2lt+1)^2 carrier matrices through the real CG tables (proj/src/mtp.cpp:20-58), classical cubic
// matmul Z = X Y (:119-133, sub-cubic forbidden by the cost model), extract every output degree by
// the adjoint CG contraction (:60-97).
//
// A block of 512 threads owns a tile of R products (R = 4..32, a multiple of 4) with every
// intermediate in shared memory, stored product-minor: element e of product r at [e][r].  One
// 128-bit shared load then feeds the same term to 4 products:
//   embed    item = (carrier cell, up to 16 products): per CSR term one coefficient fetch and
//            16 FMAs fed by 4 LDS.128 (host/context.cpp builds the per-cell lists over the CG nonzeros)
//   matmul   item = (4 x 4 block of Z, 4 products): per k, 8 LDS.128 and 64 FMAs; carriers are
//            padded to dtp = dt rounded up to 4 with zero rows / columns, so blocks need no guards;
//            Z overwrites X once every block has its sums in registers
//   extract  item = (output coefficient, up to 16 products): per CSR term 4 LDS.128, 16 FMAs;
//            outputs past the carrier band are exactly zero
#include <algorithm>

#include "kernels.hpp"

namespace tpo_b200 {
namespace {

constexpr int kThreads = 512;

// acc[q] += c_e * src[idx_e * G + q] over the CSR terms [e0, e1) of one item (PI products, G float4
// groups per element); terms are {index, coefficient bits}, loaded four at a time so the L2 latency
// of the lists overlaps
template <int PI, int G>
__device__ __forceinline__ void accumulate_terms_g(const uint2* __restrict__ terms, int e0, int e1, const float4* src,
                                                   float4 (&acc)[PI / 4]) {
  auto one = [&](uint2 tm) {
    const float c = __uint_as_float(tm.y);
    const float4* sv = src + static_cast<int>(tm.x) * G;
#pragma unroll
    for (int q = 0; q < PI / 4; ++q) {
      const float4 v = sv[q];
      acc[q].x = fmaf(c, v.x, acc[q].x);
      acc[q].y = fmaf(c, v.y, acc[q].y);
      acc[q].z = fmaf(c, v.z, acc[q].z);
      acc[q].w = fmaf(c, v.w, acc[q].w);
    }
  };
  int e = e0;
  for (; e + 4 <= e1; e += 4) {
    const uint2 a = __ldg(terms + e), b = __ldg(terms + e + 1), c = __ldg(terms + e + 2), d = __ldg(terms + e + 3);
    one(a);
    one(b);
    one(c);
    one(d);
  }
  for (; e < e1; ++e) one(__ldg(terms + e));
}

template <int R>
__global__ void __launch_bounds__(kThreads, 1)
    mtp_kernel(const __grid_constant__ MtpDevTables t, const __grid_constant__ RowSpec rs) {
  extern __shared__ float4 sm4[];
  constexpr int G = R / 4;              // float4 groups per element
  constexpr int EP = G > 1 ? G + 1 : 1;  // element pitch in float4: +1 spreads elements over the banks
  constexpr int PI = R < 16 ? R : 16;   // products per embed / extract item
  constexpr int GI = R / PI;            // items per cell / output
  const int dt = t.dt, dtp = t.dtp, dt2 = dt * dt, cells = dtp * dtp;
  float4* xs = sm4;                 // [din1][EP]
  float4* ys = xs + t.din1 * EP;    // [din2][EP]
  float4* X = ys + t.din2 * EP;     // [dtp * dtp][EP], i * dtp + k; Z after the matmul
  float4* Y = X + cells * EP;       // [dtp * dtp][EP], k * dtp + j
  const int tid = threadIdx.x;
  for (int i = tid; i < 2 * cells * EP; i += kThreads) X[i] = make_float4(0.f, 0.f, 0.f, 0.f);  // padding stays 0
  const int nb = dtp / 4;
  const int64_t ntiles = (rs.rows + R - 1) / R;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row0 = tile * R;
    const int nr = static_cast<int>(rs.rows - row0 < R ? rs.rows - row0 : R);
    __syncthreads();  // previous tile's extract has read Z
    {  // stage inputs product-minor (coalesced global reads)
      float* xf = reinterpret_cast<float*>(xs);
      float* yf = reinterpret_cast<float*>(ys);
      for (int i = tid; i < R * t.din1; i += kThreads) {
        const int r = i / t.din1, k = i - r * t.din1;
        xf[k * EP * 4 + r] = r < nr ? __ldg(rs.x + row0 * t.din1 + i) : 0.f;
      }
      for (int i = tid; i < R * t.din2; i += kThreads) {
        const int r = i / t.din2, k = i - r * t.din2;
        const int64_t gr = row0 + r;
        const int64_t yr = rs.y_shared ? gr / rs.channels : gr;
        yf[k * EP * 4 + r] = r < nr ? __ldg(rs.y + yr * t.din2 + k) : 0.f;
      }
    }
    __syncthreads();
    // ---- embed (proj/src/mtp.cpp:20-58): X[a][b] = sum_e c_e x[idx_e], Y likewise.  An item is
    // (cell, PI products): each CSR term (coefficient + index, from L1) feeds PI FMAs
    for (int item = tid; item < 2 * dt2 * GI; item += kThreads) {
      const bool second = item >= dt2 * GI;
      const int it = second ? item - dt2 * GI : item;
      const int cell = it / GI, g0 = (it - cell * GI) * (PI / 4);
      const int* off = second ? t.emb2_off : t.emb1_off;
      const uint2* terms = second ? t.emb2 : t.emb1;
      const float4* src = (second ? ys : xs) + g0;
      float4 acc[PI / 4];
#pragma unroll
      for (int q = 0; q < PI / 4; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      // the term list lives in L2: four independent term loads in flight per step
      accumulate_terms_g<PI, EP>(terms, __ldg(off + cell), __ldg(off + cell + 1), src, acc);
      const int a = cell / dt, b = cell - a * dt;
      float4* dst = (second ? Y : X) + (a * dtp + b) * EP + g0;
#pragma unroll
      for (int q = 0; q < PI / 4; ++q) dst[q] = acc[q];
    }
    __syncthreads();
    // ---- Z = X Y, classical cubic (proj/src/mtp.cpp:119-133): one 4 x 4 block of 4 products per thread
    const int ntask = nb * nb * G;
    const bool has = tid < ntask;
    const int g = tid % G, blk = tid / G, i0 = (blk / nb) * 4, j0 = (blk % nb) * 4;
    float4 acc[4][4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int p = 0; p < 4; ++p) acc[q][p] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (has) {
      for (int k = 0; k < dt; ++k) {
        float4 a[4], b[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) a[q] = X[((i0 + q) * dtp + k) * EP + g];
#pragma unroll
        for (int p = 0; p < 4; ++p) b[p] = Y[(k * dtp + j0 + p) * EP + g];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            acc[q][p].x = fmaf(a[q].x, b[p].x, acc[q][p].x);
            acc[q][p].y = fmaf(a[q].y, b[p].y, acc[q][p].y);
            acc[q][p].z = fmaf(a[q].z, b[p].z, acc[q][p].z);
            acc[q][p].w = fmaf(a[q].w, b[p].w, acc[q][p].w);
          }
      }
    }
    __syncthreads();  // every block read X: Z may overwrite it
    if (has)
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int p = 0; p < 4; ++p) X[((i0 + q) * dtp + j0 + p) * EP + g] = acc[q][p];
    __syncthreads();
    // ---- extract (proj/src/mtp.cpp:60-97): out[o] = sum_e c_e Z[cell_e]; zero past the carrier band.
    // item = (output coefficient, PI products)
    for (int item = tid; item < t.dout_total * GI; item += kThreads) {
      const int o = item / GI, g0 = (item - o * GI) * (PI / 4);
      float4 acc4[PI / 4];
#pragma unroll
      for (int q = 0; q < PI / 4; ++q) acc4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (o < t.dout_eff) accumulate_terms_g<PI, EP>(t.ext, __ldg(t.ext_off + o), __ldg(t.ext_off + o + 1), X + g0, acc4);
#pragma unroll
      for (int q = 0; q < PI / 4; ++q) {
        const int r = 4 * (g0 + q);
        float* op = rs.out + (row0 + r) * t.dout_total + o;
        if (r < nr) op[0] = acc4[q].x;
        if (r + 1 < nr) op[t.dout_total] = acc4[q].y;
        if (r + 2 < nr) op[2 * static_cast<int64_t>(t.dout_total)] = acc4[q].z;
        if (r + 3 < nr) op[3 * static_cast<int64_t>(t.dout_total)] = acc4[q].w;
      }
    }
  }
}

template <int R>
size_t smem_for(const MtpDevTables& t) {
  constexpr int EP = R / 4 > 1 ? R / 4 + 1 : 1;
  return sizeof(float) * 4 * EP * (t.din1 + t.din2 + 2 * t.dtp * t.dtp);
}

template <int R>
cudaError_t launch_r(const MtpDevTables& t, const RowSpec& rs, int num_sms, cudaStream_t s) {
  const size_t smem = smem_for<R>(t);
  cudaError_t e = cudaFuncSetAttribute(mtp_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const int64_t ntiles = (rs.rows + R - 1) / R;
  const int grid = static_cast<int>(std::min<int64_t>(ntiles, num_sms));
  mtp_kernel<R><<<grid, kThreads, smem, s>>>(t, rs);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_mtp(const MtpDevTables& t, const RowSpec& rs, int num_sms, cudaStream_t s) {
  if (rs.rows <= 0) return cudaSuccess;
  // the largest tile whose intermediates fit in shared memory and whose matmul blocks fit the block
  const int nb = t.dtp / 4;
  auto fits = [&](size_t smem, int R) { return smem <= 220u * 1024u && nb * nb * (R / 4) <= kThreads; };
  if (fits(smem_for<32>(t), 32)) return launch_r<32>(t, rs, num_sms, s);
  if (fits(smem_for<16>(t), 16)) return launch_r<16>(t, rs, num_sms, s);
  if (fits(smem_for<8>(t), 8)) return launch_r<8>(t, rs, num_sms, s);
  if (fits(smem_for<4>(t), 4)) return launch_r<4>(t, rs, num_sms, s);
  return cudaErrorInvalidValue;
}

}  // namespace tpo_b200
