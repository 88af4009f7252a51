// Channel-wise CGTP with one y per edge (config C4) on the tensor cores.
//
// Reference: tpo::cgtp_mimo applied per (edge, channel) with the edge's y
// (proj/src/cgtp.cpp:145-177; SURVEY.md a11 defines the channel-wise form).
// For a fixed y the product is linear in x:
//   out[c][o] = sum_t c_t x[c][i1_t] y[i2_t] = sum_i1 x[c][i1] M_y[i1][o],
//   M_y[i1][o] = sum_{t in terms(o), i1_t = i1} c_t y[i2_t]
// so each (edge, block of 128 channels) is one dense GEMM
//   D[128 x Dout] = X[128 x Din1] . M_y[Din1 x Dout]
// on tcgen05 (3xFP16 as in the grid kernel: hi*hi + hi*lo + lo*hi, fp32
// accumulation in TMEM, exact power-of-two scaling of every x row and of y).
// The kernel is bound by the output write (Dout floats per channel): the
// epilogue stages 32-column boxes in 128B-swizzled shared memory (conflict
// free) and writes them with TMA tensor stores that drain while the next unit
// is computed.
#include <algorithm>

#include "kernels.hpp"
#include "sm100.cuh"

namespace tpo_b200 {
using namespace sm100;

namespace {

constexpr int BM = 128;        // channels per unit == TMEM lanes
constexpr int kThreads = 256;  // 8 warps: 2 per TMEM lane quarter
constexpr int kBoxCols = 32;   // epilogue TMA store box: 128 rows x 32 fp32 (128 B rows, 128B swizzle)
constexpr int kBoxBytes = BM * kBoxCols * 4;
constexpr int kBoxBufs = 8;


__device__ __forceinline__ void tma_store_2d(const void* tmap, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(tmap)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Warp roles: warps 4-7 ("prep", thread = channel row) convert X, build M_y
// and (elected lane) issue the MMA into TMEM buffer i & 1; warps 0-3
// ("epilogue", one per TMEM lane quarter) drain the other buffer through
// swizzled boxes and TMA tensor stores.  X / M / row scales are double
// buffered by unit parity; the raw x tile is prefetched two units ahead.
__global__ void __launch_bounds__(kThreads, 1)
    cgtp_edge_tc_kernel(const __grid_constant__ CgtpTables t, const __grid_constant__ EdgeTcParams p,
                        const __grid_constant__ RowSpec rs) {
  extern __shared__ __align__(1024) uint8_t smem[];
  // 0,1 raw x landed; 2,3 Z buffer full (MMA done); 4,5 Z buffer drained (epilogue)
  __shared__ __align__(8) uint64_t bars[6];
  __shared__ uint32_t tmem_sh;
  __shared__ int ex_sh[2][BM];
  __shared__ __align__(16) float ys_sh[2][64];  // the edge's y, prefetched with the x tile (by unit parity)
  __shared__ int ey_sh[2];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kp = p.kp;
  const int zb_cols = (p.dout_pad + kBoxCols - 1) / kBoxCols * kBoxCols;  // one Z buffer (whole store boxes)
  uint8_t* box = smem;                                                 // [kBoxBufs][128 x 128 B] swizzled
  float* raw = reinterpret_cast<float*>(smem + kBoxBufs * kBoxBytes);  // [2][128 x din1]
  uint8_t* ops = reinterpret_cast<uint8_t*>(raw + 2 * BM * t.din1);
  ops = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(ops) + 127) & ~uintptr_t(127));
  const uint32_t xbuf = 2 * BM * kp * 2, mbuf = 2 * p.dout_pad * kp * 2;  // hi + lo
  auto xh_of = [&](int b) { return ops + b * (xbuf + mbuf); };
  auto mh_of = [&](int b) { return ops + b * (xbuf + mbuf) + xbuf; };
  float* mrow = reinterpret_cast<float*>(ops + 2 * (xbuf + mbuf));     // [dout_pad][kp + 1] fp32 scratch

  if (tid == 0) {
    for (int i = 0; i < 6; ++i) mbar_init(&bars[i], i >= 4 ? BM : 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    tmem_alloc(&tmem_sh, p.tmem_cols);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_sh;

  const int64_t blocks_per_edge = rs.channels / BM;
  const int64_t nunits = (rs.rows / rs.channels) * blocks_per_edge;
  const uint32_t xbytes = BM * t.din1 * 4;

  if (warp >= 4) {
    // ===================================================== prep + MMA
    const int r = tid - 128;  // channel row of the unit
    const bool el = (warp == 4) && elect_one_sync();
    // x tile and the edge's y row (din2 floats; 16 B multiple on this path) land on one barrier
    const uint32_t ybytes = static_cast<uint32_t>(t.din2) * 4u;
    auto issue_x = [&](int64_t u, int b) {
      mbar_arrive_expect_tx(&bars[b], xbytes + ybytes);
      bulk_g2s(raw + b * BM * t.din1, rs.x + u * BM * t.din1, xbytes, &bars[b]);
      bulk_g2s(ys_sh[b], rs.y + (u / blocks_per_edge) * t.din2, ybytes, &bars[b]);
    };
    if (r == 0) {
      if (blockIdx.x < nunits) issue_x(blockIdx.x, 0);
      if (blockIdx.x + gridDim.x < nunits) issue_x(blockIdx.x + gridDim.x, 1);
    }
    int it = 0;
    for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x, ++it) {
      const int b = it & 1;
      // buffers of parity b (X/M operands, row scales, Z) were last used by unit it - 2
      if (it >= 2) mbar_wait(&bars[4 + b], ((it >> 1) - 1) & 1);
      tc_fence_after();
      // ---- x tile and y row landed (prefetched two units ahead)
      mbar_wait(&bars[b], (it >> 1) & 1);
      const float* ysb = ys_sh[b];
      if (warp == 4) {
        float mx = 0.f;
        for (int k = lane; k < t.din2; k += 32) mx = fmaxf(mx, fabsf(ysb[k]));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane == 0) ey_sh[b] = row_scale_exp(mx, 1) - kInShift;  // max|y| < 2^7: |M_y| < 2^7 sum|c|
      }
      // ---- x row r: norm pass and split pass over shared memory (din1 % 4 == 0 on this path)
      const float4* rx4 = reinterpret_cast<const float4*>(raw + b * BM * t.din1 + r * t.din1);
      float mx = 0.f;
      for (int k4 = 0; k4 < t.din1 / 4; ++k4) {
        const float4 a = rx4[k4];
        mx = fmaxf(fmaxf(mx, fabsf(a.x)), fmaxf(fabsf(a.y), fmaxf(fabsf(a.z), fabsf(a.w))));
      }
      const int e = row_scale_exp(mx, 1) - kInShift;
      const float sc = pow2i(-e);
      uint8_t* xh = xh_of(b);
      uint8_t* xl = xh + BM * kp * 2;
      for (int j0 = 0; j0 < kp; j0 += 8) {
        float v[8];
#pragma unroll
        for (int qq = 0; qq < 2; ++qq) {
          const float4 a = (j0 + 4 * qq < t.din1) ? rx4[(j0 >> 2) + qq] : make_float4(0.f, 0.f, 0.f, 0.f);
          v[4 * qq] = a.x * sc; v[4 * qq + 1] = a.y * sc; v[4 * qq + 2] = a.z * sc; v[4 * qq + 3] = a.w * sc;
        }
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
          const __half2 h2 = __floats2half2_rn(v[2 * qq], v[2 * qq + 1]);
          const float2 hf = __half22float2(h2);
          hw[qq] = *reinterpret_cast<const uint32_t*>(&h2);
          lw[qq] = pack_half2(v[2 * qq] - hf.x, v[2 * qq + 1] - hf.y);
        }
        const uint32_t off = canon_off(r, j0, BM);
        *reinterpret_cast<uint4*>(xh + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        *reinterpret_cast<uint4*>(xl + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
      }
      ex_sh[b][r] = e;
      named_bar_sync(1, 128);  // raw buffer b consumed; ey known
      // ---- M_y^T (B operand, row o, K = i1): thread sums c_t y[i2_t] over the CG terms of its outputs
      const float ysc = pow2i(-ey_sh[b]);
      uint8_t* mh = mh_of(b);
      uint8_t* ml = mh + p.dout_pad * kp * 2;
      const int64_t edge = u / blocks_per_edge;
      for (int o = r; o < p.dout_pad; o += 128) {
        float* row = mrow + o * (kp + 1);  // owned by this thread
        for (int k = 0; k < kp; ++k) row[k] = 0.f;
        if (o < t.dout) {
          const int w = o >> 5, ln = o & 31;
          const int nt = __ldg(t.warp_nt + w);
          const uint2* terms = t.terms + __ldg(t.warp_off + w) + ln;
          // per-path weight of this output column, folded into M_y (f2)
          const float yso = p.path_w ? ysc * __ldg(p.path_w + edge * p.w_stride + __ldg(p.path_of_out + o)) : ysc;
          for (int k = 0; k < nt; ++k) {
            const uint2 tw = __ldg(terms + k * 32);
            const int i1 = static_cast<int>(tw.x & 0xFFFFu), i2 = static_cast<int>(tw.x >> 16);
            row[i1] += __uint_as_float(tw.y) * ysb[i2] * yso;  // padding terms: coefficient 0
          }
        }
        for (int j0 = 0; j0 < kp; j0 += 8) {
          uint32_t hw[4], lw[4];
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {
            const float a0 = row[j0 + 2 * qq], a1 = row[j0 + 2 * qq + 1];
            const __half2 h2 = __floats2half2_rn(a0, a1);
            const float2 hf = __half22float2(h2);
            hw[qq] = *reinterpret_cast<const uint32_t*>(&h2);
            lw[qq] = pack_half2(a0 - hf.x, a1 - hf.y);
          }
          const uint32_t off = canon_off(o, j0, p.dout_pad);
          *reinterpret_cast<uint4*>(mh + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
          *reinterpret_cast<uint4*>(ml + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      named_bar_sync(1, 128);
      // raw x and y of buffer b are consumed (y by the M_y build above): prefetch unit u + 2
      if (r == 0 && u + 2 * gridDim.x < nunits) issue_x(u + 2 * gridDim.x, b);
      // ---- D[b] = X . M_y (3xFP16), N split into <= 256-column MMAs
      if (warp == 4) {
        tc_fence_after();
        const uint32_t lbo_x = (BM / 8) * 128, lbo_m = (p.dout_pad / 8) * 128;
        const uint32_t zcol = static_cast<uint32_t>(b * zb_cols);
        for (int ks = 0; ks < kp / 16; ++ks) {
          const uint64_t ah = make_sdesc(smem_u32(xh) + ks * 2 * lbo_x, lbo_x, 128);
          const uint64_t al = make_sdesc(smem_u32(xl) + ks * 2 * lbo_x, lbo_x, 128);
          for (int n0 = 0; n0 < p.dout_pad; n0 += 256) {
            const int nn = min(256, p.dout_pad - n0);
            const uint32_t bo = (n0 / 8) * 128 + ks * 2 * lbo_m;
            const uint64_t bh = make_sdesc(smem_u32(mh) + bo, lbo_m, 128);
            const uint64_t bl = make_sdesc(smem_u32(ml) + bo, lbo_m, 128);
            const uint32_t id = idesc_f16(BM, nn);
            if (el) mma_f16_ss(tmem + zcol + n0, ah, bh, id, ks > 0 ? 1u : 0u);
            if (el) mma_f16_ss(tmem + zcol + n0, ah, bl, id, 1u);
            if (el) mma_f16_ss(tmem + zcol + n0, al, bh, id, 1u);
          }
        }
        if (el) tc_commit(&bars[2 + b]);
        __syncwarp();
      }
    }
  } else {
    // ===================================================== epilogue (warp = TMEM lane quarter)
    const int et = tid;  // 0..127 == tile row
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    const int nbox = (t.dout + kBoxCols - 1) / kBoxCols;
    int it = 0, nstores = 0;
    for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x, ++it) {
      const int b = it & 1;
      mbar_wait(&bars[2 + b], (it >> 1) & 1);
      tc_fence_after();
      const int es = ex_sh[b][et] + ey_sh[b];
      const float s_lo = pow2i(es >> 1), s_hi = pow2i(es - (es >> 1));
      const int64_t row0 = u * BM;
      for (int bx = 0; bx < nbox; ++bx, ++nstores) {
        uint8_t* bb = box + (nstores % kBoxBufs) * kBoxBytes;
        // at most kBoxBufs - 1 stores in flight: the one that used this buffer has been read out
        if (et == 0) bulk_wait_read<kBoxBufs - 1>();
        named_bar_sync(2, 128);
        uint32_t v0[16], v1[16];
        tmem_ld16(lane_base + b * zb_cols + bx * kBoxCols, v0);
        tmem_ld16(lane_base + b * zb_cols + bx * kBoxCols + 16, v1);
        tmem_wait_ld();
        // 128B swizzle: 16-byte chunk j of row et lives at chunk j ^ (et & 7)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t* src = j < 4 ? v0 + 4 * j : v1 + 4 * (j - 4);
          *reinterpret_cast<float4*>(bb + et * 128 + ((j ^ (et & 7)) << 4)) =
              make_float4(__uint_as_float(src[0]) * s_lo * s_hi, __uint_as_float(src[1]) * s_lo * s_hi,
                          __uint_as_float(src[2]) * s_lo * s_hi, __uint_as_float(src[3]) * s_lo * s_hi);
        }
        fence_proxy_async_smem();
        named_bar_sync(2, 128);
        if (et == 0) {
          tma_store_2d(&p.tm_out, bb, bx * kBoxCols, static_cast<int>(row0));
          bulk_commit();
        }
      }
      tc_fence_before();
      mbar_arrive_warp(&bars[4 + b]);
    }
    if (et == 0) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, p.tmem_cols);
}

}  // namespace

int cgtp_edge_tc_smem(const CgtpTables& t, int kp, int dout_pad) {
  return kBoxBufs * kBoxBytes + 2 * BM * t.din1 * 4 + 128 + 2 * (2 * BM * kp * 2 + 2 * dout_pad * kp * 2) +
         dout_pad * (kp + 1) * 4;
}

cudaError_t launch_cgtp_edge_tc(const CgtpTables& t, const EdgeTcParams& p, const RowSpec& rs, int num_sms,
                                cudaStream_t s) {
  if (rs.rows <= 0) return cudaSuccess;
  const int smem = cgtp_edge_tc_smem(t, p.kp, p.dout_pad);
  cudaError_t e = cudaFuncSetAttribute(cgtp_edge_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int64_t nunits = rs.rows / BM;
  const int grid = static_cast<int>(std::min<int64_t>(nunits, num_sms));
  cgtp_edge_tc_kernel<<<grid, kThreads, smem, s>>>(t, p, rs);
  return cudaGetLastError();
}

}  // namespace tpo_b200
