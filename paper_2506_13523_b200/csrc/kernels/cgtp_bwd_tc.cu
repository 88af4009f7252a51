// CGTP backward (vector-Jacobian products) on tcgen05, per (l1, l2) block.
//
// The forward block product is out_block = W . (x_{l1} (x) y_{l2}) (cgtp_tc.cu, the reference's
// path order proj/src/cgtp.cpp:152-163).  Its VJP with grad_out block g is
//   Q = W^T g_block          (Q[m1 n2 + m2] = sum_o W[o][m1 n2 + m2] g[o])
//   grad_x_{l1}[m1] += sum_m2 Q[m1, m2] y_{l2}[m2],   grad_y_{l2}[m2] += sum_m1 Q[m1, m2] x_{l1}[m1]
// so per 128-row tile and block, Q is one dense GEMM on the tensor cores (3xFP16, grad_out rows
// scaled by exact powers of two) and the two small contractions run in the epilogue
// straight from TMEM.  grad_out -- (L+1)^4 floats per row, the dominant traffic -- feeds both
// gradients.
//
// Two kernels:
//   cgtp_bwd_scale_kernel  one warp per row: max |g| -> int8 exponent (coalesced)
//   cgtp_bwd_tc_kernel     warp 0 TMA producer of the W^T ring, warp 1 MMA issuer, warps 2-9 A
//                          builders (grad_out K-steps through a cp.async ring in shared memory ->
//                          fp16 hi / lo in a TMEM ring; two threads per row), warps 10-17 epilogue
//                          (per TMEM lane quarter one warp for grad_x, one for grad_y)
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kernels.hpp"
#include "sm100.cuh"

namespace tpo_b200 {
using namespace sm100;

namespace {

constexpr int BM = 128;
constexpr int kThreads = 608;  // 19 warps
constexpr int kGWarp = 18;     // grad_out ring producer
constexpr int kMaxStages = 8;
constexpr int kKps = 2;        // K-steps per A stage
constexpr int kDCols = 192;    // TMEM: two accumulators [0, 192), [192, 384) and the A ring [384, 512)
constexpr int kARing = 384;
constexpr int kAStagesTmem = 4;
constexpr int kBoxW = 36;                 // grad_out TMA box: [32 lines][36 floats] (a 16B-aligned window
constexpr int kBox = 32 * kBoxW;           // around the stage's 32 columns: TMA box starts must be 16B aligned)
constexpr int kGSlotBox = 4 * kBox;        // grad_out ring slot: four boxes (18 KB)
constexpr int B_AF = 0, B_AE = 8, B_BF = 16, B_BE = 24, B_DF = 32, B_DE = 34, B_EF = 36, B_GF = 38, B_GE = 46,
              kBars = 54;

// 2-D tensor TMA into this CTA's shared memory, completion as tx bytes on `bar`
__device__ __forceinline__ void tma2d_load(void* dst, const CUtensorMap* tmap, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// mbarrier wait that lets the warp sleep in try_wait instead of spinning on issue slots
__device__ __forceinline__ void mbar_wait_s(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 10000000;\n\t"
      "@!p bra WAITS_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// e[row][b] = exponent with max |g_row| 2^-e in [2^6, 2^7) for every block b: grad_out rows are scaled
// per row, as the forward scales its input rows (row_scale_exp).  One warp per row, coalesced, eight
// loads per lane in flight.
__global__ void __launch_bounds__(256) cgtp_bwd_scale_kernel(const __grid_constant__ CgtpBwdTcTables t,
                                                             const float* __restrict__ g, int64_t rows,
                                                             int8_t* __restrict__ e) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int dout = t.dout, nbp = t.nbp;
  for (int64_t row = wid; row < rows; row += nw) {
    const float* gr = g + row * dout;
    float m = 0.f;
    for (int i0 = 0; i0 < dout; i0 += 256) {
      float v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int i = i0 + 32 * k + lane;
        v[k] = i < dout ? __ldg(gr + i) : 0.f;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) m = fmaxf(m, fabsf(v[k]));
    }
    const float mx = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(m)));
    const int8_t ev = static_cast<int8_t>(row_scale_exp(mx, 1) - kInShift);
    for (int b = lane; b < nbp; b += 32) e[row * nbp + b] = ev;
  }
}

__device__ unsigned long long* g_bwd_prof;  // TPO_CGTP_BWD_PROF=1: per-CTA role timings (clock64)
constexpr int kProfSlots = 16;

// One block's share of the row's gradients from its Q columns in TMEM (k = m1 N2 + m2, from column
// cb): grad_x[ix0 + m1] += s sum_m2 Q y[iy0 + m2] (GX) or grad_y[iy0 + m2] += s sum_m1 Q x[ix0 + m1].
// A 16-column load covers 16 / N2 rows m1 of Q (two loads per row past 16 columns).
template <int N2, bool GX>
__device__ __forceinline__ void epi_unit(uint32_t cb, int n1, const float* xr, float* ar, int ix0, int iy0, float s) {
  constexpr int NL = N2 > 16 ? 2 : 1;             // 16-column TMEM loads per step
  constexpr int RPL = N2 > 16 ? 1 : 16 / N2;      // rows m1 of Q per step
  float yv[N2], gy[N2];
#pragma unroll
  for (int m2 = 0; m2 < N2; ++m2) {
    yv[m2] = GX ? xr[iy0 + m2] : 0.f;
    gy[m2] = 0.f;
  }
  for (int m0 = 0; m0 < n1; m0 += RPL) {
    uint32_t v[16 * NL];
    tmem_ld16(cb + m0 * N2, *reinterpret_cast<uint32_t(*)[16]>(v));  // columns past the block: ignored
    if (NL == 2) tmem_ld16(cb + m0 * N2 + 16, *reinterpret_cast<uint32_t(*)[16]>(v + 16 * (NL - 1)));
    tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < RPL; ++j) {
      if (m0 + j >= n1) break;  // warp-uniform
      if (GX) {
        float a = 0.f;
#pragma unroll
        for (int m2 = 0; m2 < N2; ++m2) a = fmaf(__uint_as_float(v[j * N2 + m2]), yv[m2], a);
        ar[ix0 + m0 + j] = fmaf(a, s, ar[ix0 + m0 + j]);
      } else {
        const float xv = xr[ix0 + m0 + j];
#pragma unroll
        for (int m2 = 0; m2 < N2; ++m2) gy[m2] = fmaf(__uint_as_float(v[j * N2 + m2]), xv, gy[m2]);
      }
    }
  }
  if (!GX)
#pragma unroll
    for (int m2 = 0; m2 < N2; ++m2) ar[iy0 + m2] = fmaf(gy[m2], s, ar[iy0 + m2]);
}

// G: grad_out ring slots; WIDE: blocks with 2 l2 + 1 = 15 (L = 7; a separate instantiation keeps the
// L <= 6 epilogue free of the wider register arrays)
// SIDE: 0 both gradients; 1 grad_x only, 2 grad_y only (L = 8: the row's accumulator then holds one
// side, and one launch per gradient reads grad_out)
template <int G, bool PROF, bool WIDE, int SIDE = 0>
__global__ void __launch_bounds__(kThreads, 1)
    cgtp_bwd_tc_kernel(const __grid_constant__ CgtpBwdTcTables t, const float* __restrict__ x,
                       const float* __restrict__ y, const int8_t* __restrict__ eg, float* __restrict__ gx, float* __restrict__ gy, int64_t rows) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[kBars];
  __shared__ uint32_t tmem_sh;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t ntiles = (rows + BM - 1) / BM;
  const int dxy = t.din1 + t.din2, pitch = dxy | 1;  // odd pitch: per-row arrays are bank-conflict free
  const int nbp = t.nbp;
  uint8_t* ring_b = smem + t.off_b;
  float* rowbuf = reinterpret_cast<float*>(smem + t.off_xy);     // [128][pitch] x | y of the row
  const int apitch = SIDE == 0 ? pitch : (SIDE == 1 ? t.din1 : t.din2) | 1;
  float* acc = rowbuf + BM * pitch;                                // [128][apitch] grad_x | grad_y
  float* gring = reinterpret_cast<float*>(smem + t.off_g + ((128u - (smem_u32(smem + t.off_g) & 127u)) & 127u));
  // ^ [G][4][32][36] floats, 128B aligned (the host reserves the slack)
  int8_t* eslot = reinterpret_cast<int8_t*>(gring + G * kGSlotBox);  // [2][128][nbp]

  if (tid == 0) {
    for (int i = 0; i < kMaxStages; ++i) {
      mbar_init(&bars[B_AF + i], 2 * BM);
      mbar_init(&bars[B_AE + i], 1);
      mbar_init(&bars[B_BF + i], 1);
      mbar_init(&bars[B_BE + i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars[B_DF + i], 1);
      mbar_init(&bars[B_DE + i], 2 * BM);
      mbar_init(&bars[B_EF + i], 2 * BM);
    }
    for (int i = 0; i < G; ++i) {
      mbar_init(&bars[B_GF + i], 1);
      mbar_init(&bars[B_GE + i], 2 * BM);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc(&tmem_sh, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_sh;
  long long pc[kProfSlots] = {};
  const long long t_begin = clock64();
  auto timed = [&](int k, auto&& fn) {
    if (PROF) {
      const long long t0 = clock64();
      fn();
      pc[k] += clock64() - t0;
    } else {
      fn();
    }
  };
  auto flush_prof = [&](int k0, int k1, int ktot) {
    if (PROF && lane == 0) {
      pc[ktot] = clock64() - t_begin;
      for (int k = k0; k < k1; ++k) g_bwd_prof[blockIdx.x * kProfSlots + k] = pc[k];
      g_bwd_prof[blockIdx.x * kProfSlots + ktot] = pc[ktot];
    }
  };

  if (warp == 0) {
    // ============================================= W^T ring producer
    if (lane == 0) {
      int nb = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
        for (int u = 0; u < t.nunits; ++u) {
          const CgtpBwdTcUnit un = t.units[u];
          const uint32_t bytes = 64u * un.n_pad;
          for (int ks = 0; ks < un.ksteps; ++ks, ++nb) {
            const int s = nb % t.b_stages;
            if (nb >= t.b_stages) timed(0, [&] { mbar_wait_s(&bars[B_BE + s], ((nb / t.b_stages) - 1) & 1); });
            mbar_arrive_expect_tx(&bars[B_BF + s], bytes);
            bulk_g2s(ring_b + s * t.b_stage_bytes, t.w + un.w_off + static_cast<size_t>(ks) * bytes, bytes,
                     &bars[B_BF + s]);
          }
        }
      flush_prof(0, 1, 1);
    }
  } else if (warp == kGWarp) {
    // ============================================= grad_out ring producer
    // stage (tile, unit, s): rows 4 i + k of the tile, columns o = 32 s .. of the block, as four boxes
    // [32 lines][36 floats] of the 4-rows-per-line view (box k = TMEM lane quarter k), each starting
    // at the 16B-aligned column at or below the stage's first
    if (lane == 0) {
      int ng = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
        for (int u = 0; u < t.nunits; ++u) {
          const CgtpBwdTcUnit un = t.units[u];
          for (int ks = 0; ks < un.ksteps; ks += 2, ++ng) {
            const int gsl = ng % G;
            if (ng >= G) timed(14, [&] { mbar_wait_s(&bars[B_GE + gsl], ((ng / G) - 1) & 1); });
            mbar_arrive_expect_tx(&bars[B_GF + gsl], 4u * kGSlotBox);
            for (int k = 0; k < 4; ++k)
              tma2d_load(gring + gsl * kGSlotBox + k * kBox, &t.tm_g, (k * t.dout + un.g_off + 16 * ks) & ~3,
                         static_cast<int>(tile * (BM / 4)), &bars[B_GF + gsl]);
          }
        }
      flush_prof(14, 15, 15);
    }
  } else if (warp == 1) {
    // ============================================= MMA issuer (as the forward block kernel)
    const bool el = elect_one_sync();
    int sa = 0, pa = 0, sb = 0, pb = 0, gs = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
      for (int u = 0; u < t.nunits; ++u) {
        const CgtpBwdTcUnit un = t.units[u];
        const int d = gs & 1;
        const int dcol = un.dcol_last & 0xFFFF;
        if (dcol == 0 && gs >= 2) {
          timed(2, [&] { mbar_wait_s(&bars[B_DE + d], ((gs >> 1) - 1) & 1); });
          tc_fence_after();
        }
        const uint32_t id = idesc_f16(BM, un.n_pad);
        const uint32_t lbo_b = (un.n_pad / 8) * 128, half_b = 32u * un.n_pad;
        for (int ks = 0; ks < un.ksteps; ++ks) {
          const int j = ks & (kKps - 1);
          if (j == 0) timed(3, [&] { mbar_wait_s(&bars[B_AF + sa], pa); });
          timed(4, [&] { mbar_wait_s(&bars[B_BF + sb], pb); });
          tc_fence_after();
          const uint32_t ah = tmem + kARing + 32u * sa + 16u * j, al = ah + 8u;
          const uint32_t b0 = smem_u32(ring_b + sb * t.b_stage_bytes);
          const uint64_t bh = make_sdesc(b0, lbo_b, 128), bl = make_sdesc(b0 + half_b, lbo_b, 128);
          const uint32_t dc = tmem + static_cast<uint32_t>(kDCols) * d + dcol;
          if (el) mma_f16_ts(dc, ah, bh, id, ks > 0 ? 1u : 0u);
          if (el) mma_f16_ts(dc, ah, bl, id, 1u);
          if (el) mma_f16_ts(dc, al, bh, id, 1u);
          if (el) tc_commit(&bars[B_BE + sb]);
          if (j == kKps - 1 || ks + 1 == un.ksteps) {
            if (el) tc_commit(&bars[B_AE + sa]);
            if (++sa == kAStagesTmem) {
              sa = 0;
              pa ^= 1;
            }
          }
          __syncwarp();
          if (++sb == t.b_stages) {
            sb = 0;
            pb ^= 1;
          }
        }
        if (un.dcol_last >> 16) {
          if (el) tc_commit(&bars[B_DF + d]);
          __syncwarp();
          ++gs;
        }
      }
    flush_prof(2, 5, 5);
  } else if (warp < 10) {
    // ============================================= A builders: grad_out stages of the block
    // TMEM lane r holds tile row 4 (r % 32) + r / 32 (the grad_out boxes' row order; the MMA does
    // not care).  Thread (r, h) converts K-step h of each stage (16 floats of line r % 32 of box
    // r / 32, starting `shift` floats into the 16B-aligned window) into the TMEM A ring.
    const int r = 32 * (warp & 3) + lane, h = (warp - 2) >> 2;
    const int rt = 4 * (r & 31) + (r >> 5);  // tile row
    const int qb = r >> 5;                   // box (warp-uniform)
    const uint32_t lbw = tmem + (static_cast<uint32_t>(32 * (warp & 3)) << 16);
    const float* mybox = gring + qb * kBox + (r & 31) * kBoxW + 16 * h;
    int sa = 0, pa = 0, na = 0, it = 0, cj = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int64_t row = tile * BM + rt;
      const bool ok = row < rows;
      int8_t* es = eslot + (it & 1) * BM * nbp + r * nbp;
      if (it >= 2) timed(7, [&] { mbar_wait_s(&bars[B_EF + (it & 1)], ((it >> 1) - 1) & 1); });  // epilogue done with the slot
      // the row's exponent (grad_out rows are scaled per row): a register here, a shared copy for the
      // epilogue written by one of the row's two threads
      const float sc = pow2i(ok ? -static_cast<int>(__ldg(eg + row * nbp)) : 0);
      if (h == 0)
        for (int b = 0; b < nbp; b += 4)
          *reinterpret_cast<int*>(es + b) = ok ? __ldg(reinterpret_cast<const int*>(eg + row * nbp + b)) : 0;
      for (int u = 0; u < t.nunits; ++u) {
        const CgtpBwdTcUnit un = t.units[u];
        const int shift = (qb * t.dout + un.g_off) & 3;  // block start inside this box's aligned window
        for (int ks0 = 0; ks0 < un.ksteps; ks0 += kKps) {
          if (na++ >= kAStagesTmem) {
            timed(8, [&] { mbar_wait_s(&bars[B_AE + sa], pa ^ 1); });
            tc_fence_after();
          }
          const int slot = cj % G;
          timed(9, [&] { mbar_wait_s(&bars[B_GF + slot], (cj / G) & 1); });
          const int o0 = 16 * (ks0 + h);
          const float4* sv = reinterpret_cast<const float4*>(mybox + slot * kGSlotBox);
          float w[20], v[16];
#pragma unroll
          for (int c4 = 0; c4 < 5; ++c4) {
            const float4 f = sv[c4];
            w[4 * c4] = f.x;
            w[4 * c4 + 1] = f.y;
            w[4 * c4 + 2] = f.z;
            w[4 * c4 + 3] = f.w;
          }
          switch (shift) {  // warp-uniform
#define TPO_SHIFT_CASE(S) \
  case S:                 \
    _Pragma("unroll") for (int c = 0; c < 16; ++c) v[c] = w[c + S]; break;
            TPO_SHIFT_CASE(0)
            TPO_SHIFT_CASE(1)
            TPO_SHIFT_CASE(2)
            default:
              TPO_SHIFT_CASE(3)
#undef TPO_SHIFT_CASE
          }
          mbar_arrive_warp(&bars[B_GE + slot]);
          ++cj;
          if (ks0 + h < un.ksteps) {  // (the odd tail K-step of a unit is never issued)
            // rows past the batch are zeros (TMA out-of-bounds fill, scale 1); columns past the
            // block belong to the next one and are masked (warp-uniform: the block's last K-step)
            if (o0 + 16 > un.n) {
#pragma unroll
              for (int c = 0; c < 16; ++c)
                if (o0 + c >= un.n) v[c] = 0.f;
            }
            uint32_t hw[8], lw[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float a0 = v[2 * q] * sc;
              const float a1 = v[2 * q + 1] * sc;
              const __half2 hh = __floats2half2_rn(a0, a1);
              const float2 hf = __half22float2(hh);
              hw[q] = *reinterpret_cast<const uint32_t*>(&hh);
              lw[q] = pack_half2(a0 - hf.x, a1 - hf.y);
            }
            const uint32_t col = kARing + 32u * sa + 16u * h;
            tmem_st8(lbw + col, hw);
            tmem_st8(lbw + col + 8u, lw);
          }
          timed(13, [&] { tmem_wait_st(); });
          tc_fence_before();
          mbar_arrive_warp(&bars[B_AF + sa]);
          if (++sa == kAStagesTmem) {
            sa = 0;
            pa ^= 1;
          }
        }
      }
    }
    if (warp == 2) flush_prof(6, 10, 10);
    if (warp == 2) flush_prof(13, 14, 10);
  } else {
    // ============================================= epilogue: Q from TMEM -> the row's gradients
    // per unit (block l1, l2; n1 x n2 columns, k = m1 n2 + m2) one 16-column TMEM load per m1 row
    // gives Q[m1, 0 .. n2).  The quarter's first warp owns grad_x (summed in a register over m2,
    // one shared-memory update per m1), the second grad_y (a register array over m2, one update per
    // block): disjoint parts of the row's accumulator, so no partial sums to merge
    const int q = warp & 3, eh = (warp - 10) >> 2;
    const int r = q * 32 + lane;
    const int rt = 4 * lane + q;  // tile row of TMEM lane r (see the builders)
    const uint32_t lb = tmem + (static_cast<uint32_t>(q * 32) << 16);
    float* xr = rowbuf + r * pitch;  // x row | y row (true values)
    // grad_x | grad_y of the row (one-sided: grad_y indices din1 + .. land at the row's start)
    float* ar = acc + r * apitch - (SIDE == 2 ? t.din1 : 0);
    const bool active = SIDE == 0 || (SIDE == 1) == (eh == 0);  // this warp's side is computed
    int gs = 0, it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int64_t row = tile * BM + rt;
      const bool ok = row < rows;
      const int8_t* es = eslot + (it & 1) * BM * nbp + r * nbp;
      if (eh == 0) {
        if (ok) {
          for (int k = 0; k < t.din1; ++k) cp_async4(xr + k, x + row * t.din1 + k);
          for (int k = 0; k < t.din2; ++k) cp_async4(xr + t.din1 + k, y + row * t.din2 + k);
          cp_async_wait_all();
        } else {
          for (int k = 0; k < dxy; ++k) xr[k] = 0.f;
        }
        if (active)
          for (int k = 0; k < t.din1; ++k) ar[k] = 0.f;
      } else if (active) {
        for (int k = t.din1; k < dxy; ++k) ar[k] = 0.f;
      }
      named_bar_sync(2 + q, 64);  // the row's x / y staged
      for (int u0 = 0; u0 < t.nunits; ++gs) {
        int u1 = u0;
        while (!(t.units[u1].dcol_last >> 16)) ++u1;
        const int d = gs & 1;
        timed(11, [&] { mbar_wait_s(&bars[B_DF + d], (gs >> 1) & 1); });
        tc_fence_after();
        const uint32_t dbase = lb + static_cast<uint32_t>(kDCols) * d;
        for (int u = u0; u <= u1; ++u) {
          const CgtpBwdTcUnit un = t.units[u];
          // the unit covers rows m1 = m1b .. m1b + nrows of Q (N parts of whole rows at L = 7; one
          // part, all 2 l1 + 1 rows, below)
          const int n2 = 2 * un.l2 + 1, n1 = WIDE ? un.nrows : 2 * un.l1 + 1;
          const int ix0 = un.l1 * un.l1 + (WIDE ? un.m1b : 0), iy0 = t.din1 + un.l2 * un.l2;
          const float s = pow2i(static_cast<int>(es[WIDE ? 0 : un.blk]) - kTabShift);
          const uint32_t cb = dbase + (un.dcol_last & 0xFFFF);
          if (!active) continue;
          switch (n2) {  // warp-uniform
#define TPO_EPI(N2)                                                    \
  case N2:                                                             \
    if (eh == 0)                                                       \
      epi_unit<N2, true>(cb, n1, xr, ar, ix0, iy0, s);                 \
    else                                                               \
      epi_unit<N2, false>(cb, n1, xr, ar, ix0, iy0, s);                \
    break;
            TPO_EPI(1) TPO_EPI(3) TPO_EPI(5) TPO_EPI(7) TPO_EPI(9) TPO_EPI(11)
            default:
              if constexpr (WIDE) {
                if (n2 == 15) {
                  if (eh == 0)
                    epi_unit<15, true>(cb, n1, xr, ar, ix0, iy0, s);
                  else
                    epi_unit<15, false>(cb, n1, xr, ar, ix0, iy0, s);
                  break;
                }
                if (n2 == 17) {
                  if (eh == 0)
                    epi_unit<17, true>(cb, n1, xr, ar, ix0, iy0, s);
                  else
                    epi_unit<17, false>(cb, n1, xr, ar, ix0, iy0, s);
                  break;
                }
              }
              TPO_EPI(13)
#undef TPO_EPI
          }
        }
        tc_fence_before();
        mbar_arrive_warp(&bars[B_DE + d]);
        u0 = u1 + 1;
      }
      mbar_arrive_warp(&bars[B_EF + (it & 1)]);  // this tile's exponents are no longer read
      if (ok && active) {
        if (eh == 0 && gx)
          for (int k = 0; k < t.din1; ++k) gx[row * t.din1 + k] = ar[k];
        if (eh == 1 && gy)
          for (int k = 0; k < t.din2; ++k) gy[row * t.din2 + k] = ar[t.din1 + k];
      }
      named_bar_sync(2 + q, 64);  // rowbuf free for the next tile's x / y
    }
    if (warp == 10) flush_prof(11, 12, 12);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

}  // namespace

int cgtp_bwd_tc_smem(const CgtpBwdTcTables& t, int b_stages, int g_slots) {
  const int pitch = (t.din1 + t.din2) | 1;
  const int apitch = t.one_sided ? std::max(t.din1, t.din2) | 1 : pitch;
  const int off_g = b_stages * t.b_stage_bytes + BM * (pitch + apitch) * 4;
  return off_g + 1024 + g_slots * kGSlotBox * 4 + 2 * BM * t.nbp;
}

cudaError_t launch_cgtp_bwd_tc(const CgtpBwdTcTables& t, const float* x, const float* y, const float* g,
                               const CUtensorMap& tm_g, float* gx, float* gy, int64_t rows, int num_sms,
                               cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  static const bool prof = [] {
    const char* v = std::getenv("TPO_CGTP_BWD_PROF");  // timing experiments only
    return v && *v == '1';
  }();
  const bool wide = t.din1 > 49 || t.din2 > 49;  // L >= 7 (always three grad_out slots there)
  auto kern = wide                 ? cgtp_bwd_tc_kernel<3, false, true>
              : t.g_slots == 8     ? cgtp_bwd_tc_kernel<8, false, false>
              : t.g_slots == 4     ? (prof ? cgtp_bwd_tc_kernel<4, true, false> : cgtp_bwd_tc_kernel<4, false, false>)
                                   : cgtp_bwd_tc_kernel<3, false, false>;
  auto kx = cgtp_bwd_tc_kernel<3, false, true, 1>, ky = cgtp_bwd_tc_kernel<3, false, true, 2>;
  cudaError_t e = cudaSuccess;
  for (auto k : {kern, kx, ky})
    if ((e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, t.smem_bytes)) != cudaSuccess) return e;
  int8_t* eg = nullptr;
  if ((e = cudaMallocAsync(reinterpret_cast<void**>(&eg), static_cast<size_t>(rows) * t.nbp, s)) != cudaSuccess) return e;
  const int64_t ntiles = (rows + BM - 1) / BM;
  const int sgrid = static_cast<int>(std::min<int64_t>((rows + 7) / 8, 8 * num_sms));
  cgtp_bwd_scale_kernel<<<sgrid, 256, 0, s>>>(t, g, rows, eg);
  const int grid = static_cast<int>(std::min<int64_t>(ntiles, num_sms));
  unsigned long long* buf = nullptr;
  if (prof) {
    cudaMalloc(&buf, sizeof(unsigned long long) * kProfSlots * grid);
    cudaMemset(buf, 0, sizeof(unsigned long long) * kProfSlots * grid);
    cudaMemcpyToSymbol(g_bwd_prof, &buf, sizeof(buf));
  }
  CgtpBwdTcTables tt = t;
  tt.tm_g = tm_g;
  if (t.one_sided) {  // one launch per requested gradient (L = 8)
    if (gx) kx<<<grid, kThreads, t.smem_bytes, s>>>(tt, x, y, eg, gx, nullptr, rows);
    if (gy) ky<<<grid, kThreads, t.smem_bytes, s>>>(tt, x, y, eg, nullptr, gy, rows);
  } else {
    kern<<<grid, kThreads, t.smem_bytes, s>>>(tt, x, y, eg, gx, gy, rows);
  }
  if (prof) {
    std::vector<unsigned long long> h(static_cast<size_t>(kProfSlots) * grid);
    cudaStreamSynchronize(s);
    cudaMemcpy(h.data(), buf, h.size() * sizeof(h[0]), cudaMemcpyDeviceToHost);
    const char* names[kProfSlots] = {"w:BE", "w:tot", "mma:DE", "mma:AF", "mma:BF", "mma:tot", "bld:GE", "bld:EF",
                                     "bld:AE", "bld:GF", "bld:tot", "epi:DF", "epi:tot", "bld:wst", "g:GE", "g:tot"};
    std::fprintf(stderr, "[cgtp bwd prof] mean cycles per CTA:");
    for (int k = 0; k < 16; ++k) {
      double m = 0;
      for (int b = 0; b < grid; ++b) m += static_cast<double>(h[b * kProfSlots + k]);
      std::fprintf(stderr, " %s=%.0f", names[k], m / grid);
    }
    std::fprintf(stderr, "\n");
    cudaFree(buf);
  }
  e = cudaGetLastError();
  cudaFreeAsync(eg, s);
  return e;
}

}  // namespace tpo_b200
