// Fused S2-grid Gaunt tensor product on the 5th-generation tensor cores.
//
// Reference path: tpo::detail::gtp_grid_select (proj/src/gtp.cpp:228-260) =
// to_sphere (proj/src/sphere.cpp:105-134) x2, pointwise_mul (:145-151),
// from_sphere_select (:155-195).  Per tile of 128 samples this kernel does
//   F_x = X S1^T,  F_y = Y S2^T        (SH -> grid, GEMM 1, TMEM accumulators)
//   P   = F_x (.) F_y                  (pointwise product, registers)
//   Z  += P A^T                        (grid -> SH quadrature, GEMM 2, TMEM)
// chunk by chunk over the grid points, so grid values never leave the SM.
// S[g][(l,m)] = Lambda_{l|m|}(theta_j) cs_m(phi_k) and
// A[(l,m)][g] = w_j (2 pi / n_phi) Lambda_{l|m|}(theta_j) cs_m(phi_k) are
// built by host/context.cpp on the reference's product grid (band L1+L2).
//
// Precision: "3xFP16".  Every fp32 operand v is split v = hi + lo with hi, lo
// fp16 (11 significant bits each) and products use hi*hi + hi*lo + lo*hi on
// kind::f16 tcgen05.mma with fp32 accumulation (dropped lo*lo ~ 2^-22 rel).
// fp16's exponent range is made safe by power-of-two normalisation: each
// input row is scaled by 2^-e so that ||x||_2 in [0.5, 1) (|F| is then
// bounded by (L+1)/sqrt(4 pi) by the addition theorem), the A table by
// 2^a_shift, and the output is rescaled by 2^(ex + ey - a_shift) exactly.
//
// Data movement: operands for one grid chunk are pre-tiled on the host in
// the UMMA canonical K-major (SWIZZLE_NONE) layout and streamed into shared
// memory with one 1D TMA bulk copy each (cp.async.bulk -> UBLKCP), tracked
// by mbarrier transaction counts.  X/Y tiles stay resident for the whole
// chunk loop.  One elected thread issues all tcgen05.mma; completion is
// signalled through tcgen05.commit -> mbarrier.
#include <algorithm>

#include "kernels.hpp"
#include "sm100.cuh"

namespace tpo_b200 {
using namespace sm100;

namespace {

constexpr int BM = 128;          // samples per tile == TMEM lanes == threads
constexpr int kStageStride = 33; // epilogue staging row pitch (floats)

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Load a 128-row tile of one input, normalise each row by a power of two
// (||row||_2 -> [0.5, 1)), split into fp16 hi/lo and store both in the
// canonical K-major layout (R = 128, K = kp).  Warp w handles rows
// [32w, 32w+32); lanes walk k so global loads are coalesced.
__device__ __forceinline__ void load_split_tile(const float* __restrict__ src, int64_t row0,
                                                const RowSpec& rs, bool is_y, int din, int kp,
                                                uint8_t* hi, uint8_t* lo, int* e_out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int rr = 0; rr < 32; ++rr) {
    const int r = warp * 32 + rr;
    const int64_t g = row0 + r;
    const bool valid = g < rs.rows;
    const int64_t srow = (is_y && rs.y_shared) ? g / rs.channels : g;
    const float* p = src + (valid ? srow : 0) * din;
    float v[4];
    float ss = 0.f;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k = lane + 32 * q;
      v[q] = (valid && k < din) ? __ldg(p + k) : 0.f;
      ss = fmaf(v[q], v[q], ss);
    }
    ss = warp_sum(ss);
    int e = 0;
    if (ss > 0.f && ss < 3.0e38f) e = ilogbf(sqrtf(ss)) + 1;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k = lane + 32 * q;
      if (k < kp) {
        const float xs = scalbnf(v[q], -e);
        const __half h = __float2half_rn(xs);
        const __half l = __float2half_rn(xs - __half2float(h));
        const uint32_t off = canon_off(r, k, BM);
        *reinterpret_cast<__half*>(hi + off) = h;
        *reinterpret_cast<__half*>(lo + off) = l;
      }
    }
    if (lane == 0) e_out[r] = e;
  }
}

// D(128 x N) (+)= A(128 x K) B(N x K)^T in 3xFP16: hi*hi + hi*lo + lo*hi.
// Operands are canonical K-major with row-group stride 128 B and K-core
// stride a_lbo / b_lbo.  Issued by one thread.
__device__ __forceinline__ void gemm3x(uint32_t d, uint32_t a_hi, uint32_t a_lo, uint32_t a_lbo,
                                       uint32_t b_hi, uint32_t b_lo, uint32_t b_lbo, int K,
                                       uint32_t idesc, bool zero_first) {
  for (int ks = 0; ks < K / 16; ++ks) {
    const uint32_t ao = ks * 2 * a_lbo, bo = ks * 2 * b_lbo;
    const uint64_t ah = make_sdesc(a_hi + ao, a_lbo, 128), al = make_sdesc(a_lo + ao, a_lbo, 128);
    const uint64_t bh = make_sdesc(b_hi + bo, b_lbo, 128), bl = make_sdesc(b_lo + bo, b_lbo, 128);
    mma_f16_ss(d, ah, bh, idesc, (zero_first && ks == 0) ? 0u : 1u);
    mma_f16_ss(d, ah, bl, idesc, 1u);
    mma_f16_ss(d, al, bh, idesc, 1u);
  }
}

__device__ __forceinline__ uint32_t pack_half2(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

__global__ void __launch_bounds__(BM, 1)
    gtp_grid_tc_kernel(const __grid_constant__ GridTcTables t, const __grid_constant__ RowSpec rs) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[4];
  __shared__ uint32_t tmem_sh;
  __shared__ int ex_sh[BM], ey_sh[BM];
  uint64_t* bar_s = &bars[0];   // S chunk landed (TMA)
  uint64_t* bar_a = &bars[1];   // A chunk landed (TMA)
  uint64_t* bar_g1 = &bars[2];  // GEMM 1 of the chunk retired
  uint64_t* bar_g2 = &bars[3];  // GEMM 2 of the chunk retired

  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    tmem_alloc(&tmem_sh, t.tmem_cols);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_sh;
  const uint32_t lane_base = tmem + (static_cast<uint32_t>(warp * 32) << 16);
  const int fx0 = t.dout_pad, fy0 = t.dout_pad + t.nc;

  uint8_t* xh = smem + t.off_x;
  uint8_t* xl = xh + BM * t.k1p * 2;
  uint8_t* yh = smem + t.off_y;
  uint8_t* yl = yh + BM * t.k2p * 2;
  uint8_t* s1 = smem + t.off_s1;
  uint8_t* s2 = t.same_s ? s1 : smem + t.off_s2;
  uint8_t* pb = smem + t.off_p;
  uint8_t* ab = smem + t.off_a;
  const uint32_t p_half = BM * t.nc * 2;
  const uint32_t s1_half = t.nc * t.k1p * 2, s2_half = t.nc * t.k2p * 2;
  const uint32_t a_half = t.dout_pad * t.nc * 2;
  const uint32_t lbo_m = (BM / 8) * 128;          // X, Y, P (R = 128)
  const uint32_t lbo_s = (t.nc / 8) * 128;        // S chunk (R = nc)
  const uint32_t lbo_a = (t.dout_pad / 8) * 128;  // A chunk (R = dout_pad)
  const uint32_t id1 = idesc_f16(BM, t.nc);

  uint32_t ph_s = 0, ph_a = 0, ph_g1 = 0, ph_g2 = 0;
  const int64_t ntiles = (rs.rows + BM - 1) / BM;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row0 = tile * BM;
    if (tid == 0) {  // chunk 0 operands; every MMA of the previous tile has retired
      mbar_arrive_expect_tx(bar_s, t.s1_chunk_bytes + (t.same_s ? 0u : t.s2_chunk_bytes));
      bulk_g2s(s1, t.s1, t.s1_chunk_bytes, bar_s);
      if (!t.same_s) bulk_g2s(s2, t.s2, t.s2_chunk_bytes, bar_s);
      mbar_arrive_expect_tx(bar_a, t.a_chunk_bytes);
      bulk_g2s(ab, t.a, t.a_chunk_bytes, bar_a);
    }
    load_split_tile(rs.x, row0, rs, false, t.din1, t.k1p, xh, xl, ex_sh);
    load_split_tile(rs.y, row0, rs, true, t.din2, t.k2p, yh, yl, ey_sh);
    fence_proxy_async_smem();
    __syncthreads();

    for (int c = 0; c < t.nchunks; ++c) {
      if (tid == 0) {
        mbar_wait(bar_s, ph_s);
        tc_fence_after();
        gemm3x(tmem + fx0, smem_u32(xh), smem_u32(xl), lbo_m, smem_u32(s1), smem_u32(s1) + s1_half, lbo_s,
               t.k1p, id1, true);
        gemm3x(tmem + fy0, smem_u32(yh), smem_u32(yl), lbo_m, smem_u32(s2), smem_u32(s2) + s2_half, lbo_s,
               t.k2p, id1, true);
        tc_commit(bar_g1);
      }
      ph_s ^= 1;
      if (c > 0) {
        if (tid == 0) {  // GEMM 2 of chunk c-1 retired: A buffer free -> prefetch A[c]
          mbar_wait(bar_g2, ph_g2);
          mbar_arrive_expect_tx(bar_a, t.a_chunk_bytes);
          bulk_g2s(ab, t.a + static_cast<size_t>(c) * t.a_chunk_bytes, t.a_chunk_bytes, bar_a);
        }
        ph_g2 ^= 1;
      }
      mbar_wait(bar_g1, ph_g1);
      ph_g1 ^= 1;
      tc_fence_after();
      if (tid == 0 && c + 1 < t.nchunks) {  // S buffer free -> prefetch S[c+1]
        mbar_arrive_expect_tx(bar_s, t.s1_chunk_bytes + (t.same_s ? 0u : t.s2_chunk_bytes));
        bulk_g2s(s1, t.s1 + static_cast<size_t>(c + 1) * t.s1_chunk_bytes, t.s1_chunk_bytes, bar_s);
        if (!t.same_s)
          bulk_g2s(s2, t.s2 + static_cast<size_t>(c + 1) * t.s2_chunk_bytes, t.s2_chunk_bytes, bar_s);
      }
      // pointwise product on the grid chunk, split to fp16 hi/lo -> P (A operand of GEMM 2)
      for (int j0 = 0; j0 < t.nc; j0 += 16) {
        uint32_t fx[16], fy[16];
        tmem_ld16(lane_base + fx0 + j0, fx);
        tmem_ld16(lane_base + fy0 + j0, fy);
        tmem_wait_ld();
        uint32_t hw[8], lw[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float a0 = __uint_as_float(fx[2 * q]) * __uint_as_float(fy[2 * q]);
          const float a1 = __uint_as_float(fx[2 * q + 1]) * __uint_as_float(fy[2 * q + 1]);
          const __half2 h = __floats2half2_rn(a0, a1);
          const float2 hf = __half22float2(h);
          hw[q] = *reinterpret_cast<const uint32_t*>(&h);
          lw[q] = pack_half2(a0 - hf.x, a1 - hf.y);
        }
        const uint32_t o0 = canon_off(tid, j0, BM), o1 = canon_off(tid, j0 + 8, BM);
        *reinterpret_cast<uint4*>(pb + o0) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        *reinterpret_cast<uint4*>(pb + o1) = make_uint4(hw[4], hw[5], hw[6], hw[7]);
        *reinterpret_cast<uint4*>(pb + p_half + o0) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
        *reinterpret_cast<uint4*>(pb + p_half + o1) = make_uint4(lw[4], lw[5], lw[6], lw[7]);
      }
      tc_fence_before();
      fence_proxy_async_smem();
      __syncthreads();
      if (tid == 0) {
        mbar_wait(bar_a, ph_a);
        tc_fence_after();
        for (int n0 = 0; n0 < t.dout_pad; n0 += 256) {
          const int nn = min(256, t.dout_pad - n0);
          const uint32_t bo = (n0 / 8) * 128;
          gemm3x(tmem + n0, smem_u32(pb), smem_u32(pb) + p_half, lbo_m, smem_u32(ab) + bo,
                 smem_u32(ab) + a_half + bo, lbo_a, t.nc, idesc_f16(BM, nn), c == 0);
        }
        tc_commit(bar_g2);
      }
      ph_a ^= 1;
    }

    // ---- epilogue: TMEM -> registers -> rescale -> smem stage -> coalesced stores
    mbar_wait(bar_g2, ph_g2);
    ph_g2 ^= 1;
    tc_fence_after();
    float* stage = reinterpret_cast<float*>(smem + t.off_x);
    const int e_row = ex_sh[tid] + ey_sh[tid] - t.a_shift;
    for (int c0 = 0; c0 < t.dout_total; c0 += 32) {
      uint32_t r0[16], r1[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) r0[q] = r1[q] = 0u;
      if (c0 < t.dout_pad) tmem_ld16(lane_base + c0, r0);
      if (c0 + 16 < t.dout_pad) tmem_ld16(lane_base + c0 + 16, r1);
      tmem_wait_ld();
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        stage[tid * kStageStride + q] = (c0 + q < t.dout_eff) ? scalbnf(__uint_as_float(r0[q]), e_row) : 0.f;
        stage[tid * kStageStride + 16 + q] =
            (c0 + 16 + q < t.dout_eff) ? scalbnf(__uint_as_float(r1[q]), e_row) : 0.f;
      }
      __syncthreads();
      for (int i = tid; i < BM * 32; i += BM) {
        const int r = i >> 5, cc = i & 31;
        const int64_t g = row0 + r;
        const int col = c0 + cc;
        if (g < rs.rows && col < t.dout_total) rs.out[g * t.dout_total + col] = stage[r * kStageStride + cc];
      }
      tc_fence_before();
      __syncthreads();
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, t.tmem_cols);
}

}  // namespace

int gtp_grid_tc_max_smem() {
  // 227 KB opt-in minus the kernel's static shared memory
  return 232448 - static_cast<int>(4 * 8 + 4 + 2 * BM * 4) - 64;
}

cudaError_t launch_gtp_grid_tc(const GridTcTables& t, const RowSpec& rs, int num_sms, cudaStream_t s) {
  if (rs.rows <= 0) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(gtp_grid_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       t.smem_bytes);
  if (e != cudaSuccess) return e;
  int occ = 1;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gtp_grid_tc_kernel, BM, t.smem_bytes);
  if (e != cudaSuccess) return e;
  occ = std::max(1, std::min(occ, 512 / t.tmem_cols));  // TMEM columns per SM
  const int64_t ntiles = (rs.rows + BM - 1) / BM;
  const int grid = static_cast<int>(std::min<int64_t>(ntiles, static_cast<int64_t>(num_sms) * occ));
  gtp_grid_tc_kernel<<<grid, BM, t.smem_bytes, s>>>(t, rs);
  return cudaGetLastError();
}

}  // namespace tpo_b200
