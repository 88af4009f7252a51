// Matrix tensor product on tcgen05 (carrier dt = 2 lt + 1 <= 13).
//
// Reference: tpo::mtp with MtpImpl::sparse (proj/src/mtp.cpp:99-117): embed
// both inputs into dt x dt carrier matrices through the real CG tables
// (:20-58), classical cubic matmul Z = X Y (:119-133), extract every output
// degree by the adjoint CG contraction (:60-97).
//
// Embed and extract are linear maps with fixed coefficients, so per 128-row
// tile they are dense GEMMs on the tensor cores (3xFP16: hi*hi + hi*lo + lo*hi,
// fp32 accumulation in TMEM, rows scaled by exact powers of two):
//   GEMM 1:  X^T-ordered carrier  [128 x n1] = x[128 x k1] . E1^T,  Y likewise
//   middle:  Z = X Y per row on SIMT, thread = TMEM lane, operands read with
//            tcgen05.ld, Z written back to TMEM as fp16 hi/lo K-steps
//   GEMM 2:  out [128 x n2] = Z[128 x kz] . Ext^T   (A operand from TMEM)
// The carrier matrices never leave the SM; HBM traffic is the inputs and the
// output (the MTP roofline is HBM for the BASELINE shapes).
//
// Warps: 0-3 input staging / conversion and epilogue (thread = tile row),
// 4-7 middle (thread = TMEM lane), 8 TMA producer of the B-operand ring
// (E2, E1, Ext K-steps in consumption order), 9 TMEM owner + MMA issuer.
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
constexpr int kThreads = 320;
constexpr int kMaxStages = 8;
constexpr int kStageStride = 17;
// barriers: ring full [8], ring empty [8], then
constexpr int B_OPS_READY = 2 * kMaxStages;  // X/Y operands of the next tile converted (128 arrivals)
constexpr int B_G1_DONE = B_OPS_READY + 1;   // GEMM 1 retired (commit)
constexpr int B_Z_READY = B_G1_DONE + 1;     // Z written to TMEM (128 arrivals)
constexpr int B_G2_DONE = B_Z_READY + 1;     // GEMM 2 retired (commit)
constexpr int B_D_FREE = B_G2_DONE + 1;      // epilogue read the output columns (256 arrivals)
constexpr int B_STAGE_FULL = B_D_FREE + 1;   // TMA staging of a tile's raw inputs landed
constexpr int B_YREAD = B_STAGE_FULL + 1;     // [4] per lane quarter: both row halves finished reading Y (64 arrivals)
constexpr int kBars = B_YREAD + 4;

__device__ __forceinline__ void tmem_ld8p(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
// wait for this thread's outstanding TMEM loads; the loaded registers pass through the
// asm so no use of them can be scheduled above the wait

__device__ __forceinline__ void tmem_wait_ld_bind24(uint32_t (&a)[24]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4]), "+r"(a[5]), "+r"(a[6]), "+r"(a[7]),
                 "+r"(a[8]), "+r"(a[9]), "+r"(a[10]), "+r"(a[11]), "+r"(a[12]), "+r"(a[13]), "+r"(a[14]),
                 "+r"(a[15]), "+r"(a[16]), "+r"(a[17]), "+r"(a[18]), "+r"(a[19]), "+r"(a[20]), "+r"(a[21]),
                 "+r"(a[22]), "+r"(a[23])
               :
               : "memory");
}
__device__ __forceinline__ void tmem_ld16p(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

template <int DT>
struct Carrier {
  static constexpr int N1 = (DT * DT + 15) / 16 * 16;
  static constexpr int J1 = (DT + 1) / 2;  // Y column block 0: j < J1
  static constexpr int IA = (DT + 1) / 2;  // carrier rows of warp half 0: i < IA
};

// Row half H of the per-row matmul
//   Z[i][j] = sum_k X[i][k] Y[k][j],  i in half H (i < IA or i >= IA), all j,
// accumulated in registers (packed f32x2 FMAs along j).  Each k step is one x8 TMEM
// load of X column k (rows of this half) and one x16 load of Y row k, both at
// unaligned column starts (extra columns ignored); loads of step k + 1 fly while
// step k computes.  Written to TMEM as fp16 hi / lo K-steps (cells (i - i0) * DT + j,
// padded to 16 with zeros): K-steps b < nb1 at column zc1 + 16 b, the rest at
// zc2 + 16 (b - nb1) after `sync` (the other half of the quarter finished reading Y).
// The two halves of a lane quarter meet on an mbarrier (64 arrivals, one phase per tile): they reach
// it from different code (the two instantiations), which a counted bar.sync also allows but
// compute-sanitizer synccheck reports as divergence.
__device__ __forceinline__ void halves_meet(uint64_t* bar, uint32_t phase) {
  mbar_arrive(bar);
  mbar_wait(bar, phase);
}

template <int DT, int H>
__device__ __forceinline__ void middle_half(uint32_t lb, uint32_t zc1, int nb1, uint32_t zc2, bool sync2, uint64_t* ybar,
                                            uint32_t yphase) {
  constexpr int N1 = Carrier<DT>::N1, IA = Carrier<DT>::IA;
  constexpr int I0 = H ? IA : 0, NI = H ? DT - IA : IA;
  constexpr int NJ = DT, NP = NJ / 2;  // packed pairs along j, plus one scalar column (DT odd)
  if constexpr (NI > 0) {
    float2 acc[NI][NP > 0 ? NP : 1];
    float acc1[NI];
#pragma unroll
    for (int i = 0; i < NI; ++i) {
#pragma unroll
      for (int j = 0; j < NP; ++j) acc[i][j] = make_float2(0.f, 0.f);
      acc1[i] = 0.f;
    }
    uint32_t cur[24], nxt[24];  // [X column k rows (x8) | Y row k (x16)]
#pragma unroll
    for (int e = 0; e < 24; ++e) cur[e] = nxt[e] = 0u;
    auto issue = [&](int k, uint32_t* d) {
      tmem_ld8p(lb + k * DT + I0, d);
      tmem_ld16p(lb + N1 + k * DT, d + 8);
    };
    auto step = [&](const uint32_t* v) {
      float2 yp[NP > 0 ? NP : 1];
#pragma unroll
      for (int j = 0; j < NP; ++j) yp[j] = make_float2(__uint_as_float(v[8 + 2 * j]), __uint_as_float(v[9 + 2 * j]));
      const float ylast = __uint_as_float(v[8 + NJ - 1]);
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        const float xv = __uint_as_float(v[i]);
        const float2 x2 = make_float2(xv, xv);
#pragma unroll
        for (int j = 0; j < NP; ++j) acc[i][j] = __ffma2_rn(x2, yp[j], acc[i][j]);
        acc1[i] = fmaf(xv, ylast, acc1[i]);
      }
    };
    // runtime k loop (small code: a fully unrolled form missed in the instruction cache)
    issue(0, cur);
    tmem_wait_ld_bind24(cur);
#pragma unroll 1
    for (int k = 0; k < DT; k += 2) {
      if (k + 1 < DT) issue(k + 1, nxt);
      step(cur);
      if (k + 1 < DT) {
        tmem_wait_ld_bind24(nxt);
        if (k + 2 < DT) issue(k + 2, cur);
        step(nxt);
        if (k + 2 < DT) tmem_wait_ld_bind24(cur);
      }
    }
    if (sync2) halves_meet(ybar, yphase);  // both halves done reading: part 2 may overwrite Y
    constexpr int NC = NI * NJ;
#pragma unroll
    for (int b = 0; b < (NC + 15) / 16; ++b) {
      uint32_t hw[8], lw[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        auto z = [&](int c) {
          const int i = c / NJ, j = c % NJ;
          if (c >= NC) return 0.f;
          if (j == NJ - 1) return acc1[i];
          return (j & 1) ? acc[i][j >> 1].y : acc[i][j >> 1].x;
        };
        const float a0 = z(b * 16 + 2 * q), a1 = z(b * 16 + 2 * q + 1);
        const __half2 hh = __floats2half2_rn(a0, a1);
        const float2 hf = __half22float2(hh);
        hw[q] = *reinterpret_cast<const uint32_t*>(&hh);
        lw[q] = pack_half2(a0 - hf.x, a1 - hf.y);
      }
      const uint32_t zc = b < nb1 ? zc1 + 16 * b : zc2 + 16 * (b - nb1);
      tmem_st8(lb + zc, hw);
      tmem_st8(lb + zc + 8, lw);
    }
  } else {
    if (sync2) halves_meet(ybar, yphase);
  }
}

// Row r of the tile from the staging buffer (dense rows, as the TMA bulk copy lands them) -> fp16 hi / lo in the
// canonical K-major layout (K padded to kp with zeros); returns the exponent e of
// the exact scale 2^-e.
__device__ __forceinline__ int convert_row(const float* st, int din, int kp, uint8_t* hi, uint8_t* lo, int r) {
  const float* src = st + r * din;
  float m0 = 0.f, m1 = 0.f, m2 = 0.f, m3 = 0.f;
  int k = 0;
  for (; k + 4 <= din; k += 4) {
    m0 = fmaxf(m0, fabsf(src[k])); m1 = fmaxf(m1, fabsf(src[k + 1]));
    m2 = fmaxf(m2, fabsf(src[k + 2])); m3 = fmaxf(m3, fabsf(src[k + 3]));
  }
  for (; k < din; ++k) m0 = fmaxf(m0, fabsf(src[k]));
  const int e = row_scale_exp(fmaxf(fmaxf(m0, m1), fmaxf(m2, m3)), din) - kInShift;  // ||x|| < 2^7: |Z| < 2^14
  const float sc = pow2i(-e);
#pragma unroll 2
  for (int k0 = 0; k0 < kp; k0 += 8) {
    float v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = k0 + q < din ? src[k0 + q] * sc : 0.f;
    uint32_t hw[4], lw[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const __half2 hh = __floats2half2_rn(v[2 * q], v[2 * q + 1]);
      const float2 hf = __half22float2(hh);
      hw[q] = *reinterpret_cast<const uint32_t*>(&hh);
      lw[q] = pack_half2(v[2 * q] - hf.x, v[2 * q + 1] - hf.y);
    }
    const uint32_t off = canon_off(r, k0, BM);
    *reinterpret_cast<uint4*>(hi + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
    *reinterpret_cast<uint4*>(lo + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
  }
  return e;
}

// optional in-kernel cycle accounting (env TPO_MTP_PROF=1), kProfSlots per CTA:
// half A: 0 total, 1 staging, 2 wait G1, 15 middle, 3 convert, 4 wait G2, 5 epilogue | half B: 6 wait G1,
// 7 middle, 8 convert | 9 MMA wait ops, 10 GEMM 1 issue, 11 wait D free, 12 wait Z, 13 GEMM 2 issue, 14 MMA total
constexpr int kProfSlots = 16;
__device__ unsigned long long* g_mtp_prof = nullptr;
__device__ __forceinline__ long long now() { return clock64(); }

template <int DT, bool PROF>
__global__ void __launch_bounds__(kThreads, 1)
    mtp_tc_kernel(const __grid_constant__ MtpTcTables t, const __grid_constant__ RowSpec rs) {
  // used directly (no pointer re-alignment): every access stays in the shared space (LDS / STS);
  // the SWIZZLE_NONE operand layouts need 16 B alignment only
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[kBars];
  __shared__ uint32_t tmem_sh;
  __shared__ int ex_sh[2][BM], ey_sh[2][BM];  // row scale exponents of x / y by tile parity

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t ntiles = (rs.rows + BM - 1) / BM;
  uint8_t* ring = smem;
  uint8_t* xop = smem + t.off_xop;  // [hi | lo] 128 x k1 canonical
  uint8_t* yop = smem + t.off_yop;
  float* stx = reinterpret_cast<float*>(smem + t.off_stx);
  float* sty = reinterpret_cast<float*>(smem + t.off_sty);
  float* outb = reinterpret_cast<float*>(smem + t.off_out);  // rows 0-63 of a tile's output (row-major)
  float* epi = outb;  // per-warp [32][17] staging of the direct-store epilogue (ragged tiles) aliases it

  if (tid == 0) {
    for (int i = 0; i < kMaxStages; ++i) {
      mbar_init(&bars[i], 1);
      mbar_init(&bars[kMaxStages + i], 1);
    }
    mbar_init(&bars[B_OPS_READY], 2 * BM);
    mbar_init(&bars[B_G1_DONE], 1);
    mbar_init(&bars[B_Z_READY], 2 * BM);
    mbar_init(&bars[B_G2_DONE], 1);
    mbar_init(&bars[B_D_FREE], 2 * BM);
    mbar_init(&bars[B_STAGE_FULL], 1);
    for (int i = 0; i < 4; ++i) mbar_init(&bars[B_YREAD + i], 64);
    fence_mbar_init();
  }
  if (warp == 9) {
    tmem_alloc(&tmem_sh, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_sh;
  long long pc[kProfSlots] = {};
  auto tick = [&](int slot, long long t0) {
    if (PROF) pc[slot] += now() - t0;
  };

  const int half_lane = lane >> 4, cl = lane & 15;
  float* st = epi + warp * 32 * kStageStride;
  // half of the output column blocks (cb = cb0, cb0 + 2, ...) of this warp's 32 rows:
  // TMEM -> rescale -> staging -> two 64 B row segments per store instruction
  auto epilogue_part = [&](uint32_t lb, int e_row, int64_t row0, int cb0) {
    for (int cb = cb0; cb < t.n2 / 16; cb += 2) {
      uint32_t v[16];
      tmem_ld16(lb + cb * 16, v);
      tmem_wait_ld();
#pragma unroll
      for (int q = 0; q < 16; ++q) st[lane * kStageStride + q] = mul_pow2(__uint_as_float(v[q]), e_row);
      __syncwarp();
      const int col = cb * 16 + cl;
      if (col < t.dout_eff) {
        float* op = rs.out + (row0 + half_lane) * t.dout_total + col;
        const int64_t rows_left = rs.rows - row0 - half_lane;
#pragma unroll 4
        for (int rr = 0; rr < 32; rr += 2)
          if (rr < rows_left) op[static_cast<int64_t>(rr) * t.dout_total] = st[(rr + half_lane) * kStageStride + cl];
      }
      __syncwarp();
    }
  };

  // whole tiles: quarter q stages its 32 rows (all dout_total columns, zeros past the carrier band)
  // into half buffer q >> 1 (rows 0-63: outb, rows 64-127: the raw input staging, free by now), and
  // one thread per half writes the 64 contiguous output rows with a single bulk copy
  const bool out_al = (reinterpret_cast<uintptr_t>(rs.out) & 15) == 0;
  auto bulk_ok = [&](int64_t tl) { return out_al && (tl + 1) * BM <= rs.rows; };
  auto epilogue_bulk = [&](uint32_t lb, int e_row, int64_t tile, int q, int cb0) {
    const int h = q >> 1;
    float* ob = h ? stx : outb;
    named_bar_sync(2 + h, 2 * 64);  // the half buffer is free (previous store read, raw inputs converted)
    const int lr = (q & 1) * 32 + lane;
    const int ncb = (t.dout_total + 15) / 16;
    for (int cb = cb0; cb < ncb; cb += 2) {
      float v[16];
      if (cb < t.n2 / 16) {
        uint32_t u[16];
        tmem_ld16(lb + cb * 16, u);
        tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = mul_pow2(__uint_as_float(u[k]), e_row);
      } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = 0.f;
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int c = cb * 16 + k;
        if (c < t.dout_total) ob[lr * t.dout_total + c] = c < t.dout_eff ? v[k] : 0.f;
      }
    }
    tc_fence_before();
    mbar_arrive_warp(&bars[B_D_FREE]);
    fence_proxy_async_smem();
    named_bar_sync(2 + h, 2 * 64);
    if (tid == 64 * h) {
      bulk_s2g(rs.out + (tile * BM + 64 * h) * t.dout_total, ob, 64u * t.dout_total * 4u);
      bulk_wait_read_all();
    }
  };

  if (warp < 8) {
    // ============================================= workers: warp half hw of lane quarter q (thread = tile row)
    // hw 0: middle rows i < IA, converts x; hw 1: middle rows i >= IA, converts y; both drain
    // half of the output column blocks
    const int q = warp & 3, hw = warp >> 2;
    const int r = q * 32 + lane;
    const uint32_t lb = tmem + (static_cast<uint32_t>(q * 32) << 16);
    // whole tiles of 16 B aligned inputs are staged by TMA bulk copies one tile ahead
    const bool aligned =
        ((reinterpret_cast<uintptr_t>(rs.x) | (rs.y_shared ? 0 : reinterpret_cast<uintptr_t>(rs.y))) & 15) == 0;
    auto tma_x = [&](int64_t tl) { return aligned && (tl + 1) * BM <= rs.rows; };
    auto tma_y = [&](int64_t tl) { return tma_x(tl) && !rs.y_shared; };
    auto issue_stage = [&](int64_t tl) {  // one thread
      if (!tma_x(tl)) return;
      const uint32_t bx = BM * t.din1 * 4, by = tma_y(tl) ? BM * t.din2 * 4 : 0;
      mbar_arrive_expect_tx(&bars[B_STAGE_FULL], bx + by);
      bulk_g2s(stx, rs.x + tl * BM * t.din1, bx, &bars[B_STAGE_FULL]);
      if (by) bulk_g2s(sty, rs.y + tl * BM * t.din2, by, &bars[B_STAGE_FULL]);
    };
    // the rest (ragged tile, shared y): this quarter's 32 rows of one input, 16 rows per
    // batch with all loads in flight before the first store
    auto stage_rows = [&](int64_t tile, bool is_y) {
      const int din = is_y ? t.din2 : t.din1;
      float* dst = is_y ? sty : stx;
      constexpr int kRB = 8, kC = 4;  // din <= 128 (backward windows of grad_out up to 112 columns)
#pragma unroll 1
      for (int r0 = 0; r0 < 32; r0 += kRB) {
        float v[kRB][kC];
#pragma unroll
        for (int rr = 0; rr < kRB; ++rr) {
          const int64_t g = tile * BM + q * 32 + r0 + rr;
          const bool ok = g < rs.rows;
          const float* src = is_y ? rs.y + (ok ? (rs.y_shared ? g / rs.channels : g) : 0) * t.din2
                                  : rs.x + (ok ? g : 0) * t.din1;
#pragma unroll
          for (int c = 0; c < kC; ++c) {
            const int k = lane + 32 * c;
            v[rr][c] = (ok && k < din) ? __ldg(src + k) : 0.f;
          }
        }
#pragma unroll
        for (int rr = 0; rr < kRB; ++rr)
#pragma unroll
          for (int c = 0; c < kC; ++c) {
            const int k = lane + 32 * c;
            if (k < din) dst[(q * 32 + r0 + rr) * din + k] = v[rr][c];
          }
      }
      __syncwarp();
    };
    int ns = 0;  // TMA stagings consumed (B_STAGE_FULL phase)
    auto land = [&](int64_t tl) {
      if (tma_x(tl)) {
        mbar_wait(&bars[B_STAGE_FULL], ns & 1);
        ++ns;
      }
      if (hw == 0 && !tma_x(tl)) stage_rows(tl, false);
      if (hw == 1 && !tma_y(tl)) stage_rows(tl, true);
    };
    auto convert_mine = [&](int slot) {
      if (hw == 0) ex_sh[slot][r] = convert_row(stx, t.din1, t.k1, xop, xop + BM * t.k1 * 2, r);
      else ey_sh[slot][r] = convert_row(sty, t.din2, t.k2, yop, yop + BM * t.k2 * 2, r);
      fence_proxy_async_smem();
      mbar_arrive_warp(&bars[B_OPS_READY]);
    };
    int ny = 0;  // Y-read meetings so far (phase of bars[B_YREAD + q])
    auto middle_mine = [&]() {
      // half 0: Z group 0 in one piece; half 1: group 1, its tail (if any) in the Y columns
      const uint32_t yphase = static_cast<uint32_t>(ny & 1);
      if (hw == 0)
        middle_half<DT, 0>(lb, static_cast<uint32_t>(t.zgrp_col[0]), 64, 0u, t.y0_reuse != 0, &bars[B_YREAD + q], yphase);
      else
        middle_half<DT, 1>(lb, static_cast<uint32_t>(t.zgrp_col[1]), t.zgrp_size[1] / 16,
                           static_cast<uint32_t>(t.zgrp_col[2]), t.y0_reuse != 0, &bars[B_YREAD + q], yphase);
      if (t.y0_reuse) ++ny;
    };
    int it = 0;
    int64_t tile = blockIdx.x;
    const long long tstart = now();
    if (tile < ntiles) {
      if (tid == 0) issue_stage(tile);
      land(tile);
      convert_mine(0);
      named_bar_sync(1, 2 * BM);  // staging consumed
      if (tid == 0 && tile + gridDim.x < ntiles) issue_stage(tile + gridDim.x);
    }
    for (; tile < ntiles; tile += gridDim.x, ++it) {
      const int64_t nxt = tile + gridDim.x;
      long long t0 = now();
      mbar_wait(&bars[B_G1_DONE], it & 1);
      tc_fence_after();
      tick(hw ? 6 : 2, t0);
      t0 = now();
      middle_mine();
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive_warp(&bars[B_Z_READY]);
      tick(hw ? 7 : 15, t0);
      t0 = now();
      if (nxt < ntiles) land(nxt);  // the TMA had the whole middle to land
      if (!hw) tick(1, t0);
      t0 = now();
      if (nxt < ntiles) convert_mine((it + 1) & 1);
      named_bar_sync(1, 2 * BM);  // raw staging consumed: it may now hold output rows 64-127
      tick(hw ? 8 : 3, t0);
      t0 = now();
      mbar_wait(&bars[B_G2_DONE], it & 1);
      tc_fence_after();
      if (!hw) tick(4, t0);
      t0 = now();
      const int e_row = ex_sh[it & 1][r] + ey_sh[it & 1][r] - kTabShift;  // Ext is stored times 2^kTabShift
      const bool bulk = bulk_ok(tile);
      if (bulk) {
        epilogue_bulk(lb, e_row, tile, q, hw);
      } else {
        epilogue_part(lb, e_row, tile * BM + q * 32, hw);
        tc_fence_before();
        mbar_arrive_warp(&bars[B_D_FREE]);
      }
      // raw inputs of the tile after next (the staging buffer was output half buffer 1)
      if (tid == 64 && nxt + gridDim.x < ntiles) issue_stage(nxt + gridDim.x);
      // degrees past the carrier band are exactly zero (proj/src/mtp.cpp:126)
      if (!bulk && hw == 0 && t.dout_total > t.dout_eff)
        for (int rr = 0; rr < 32; ++rr) {
          const int64_t g = tile * BM + q * 32 + rr;
          if (g >= rs.rows) break;
          for (int col = t.dout_eff + lane; col < t.dout_total; col += 32) rs.out[g * t.dout_total + col] = 0.f;
        }
      if (!hw) tick(5, t0);
    }
    if (!hw) tick(0, tstart);
    if (PROF && tid == 0)
      for (int k : {0, 1, 2, 3, 4, 5, 15}) g_mtp_prof[blockIdx.x * kProfSlots + k] = pc[k];
    if (PROF && tid == 128)
      for (int k = 6; k < 9; ++k) g_mtp_prof[blockIdx.x * kProfSlots + k] = pc[k];
  } else if (warp == 8) {
    // ============================================= TMA producer: E2, E1, Ext K-steps per tile
    if (lane == 0) {
      const uint32_t b1 = 64u * t.n1, b2 = 64u * t.n2;
      int n = 0;
      auto push = [&](const uint8_t* src, uint32_t bytes) {
        const int s = n % t.stages;
        if (n >= t.stages) mbar_wait(&bars[kMaxStages + s], ((n / t.stages) - 1) & 1);
        mbar_arrive_expect_tx(&bars[s], bytes);
        bulk_g2s(ring + s * t.stage_bytes, src, bytes, &bars[s]);
        ++n;
      };
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        for (int ks = 0; ks < t.k2 / 16; ++ks) push(t.e2 + ks * b1, b1);
        for (int ks = 0; ks < t.k1 / 16; ++ks) push(t.e1 + ks * b1, b1);
        for (int ks = 0; ks < t.kz / 16; ++ks) push(t.ext + ks * b2, b2);
      }
    }
  } else {
    // ============================================= MMA issuer (converged warp, elected lane)
    const bool el = elect_one_sync();
    const uint32_t lbo_op = (BM / 8) * 128, lbo1 = (t.n1 / 8) * 128, lbo2 = (t.n2 / 8) * 128;
    const uint32_t half1 = 32u * t.n1, half2 = 32u * t.n2;  // bytes of the hi block of a stage
    const uint32_t id1 = idesc_f16(BM, t.n1), id2 = idesc_f16(BM, t.n2);
    int n = 0;
    auto take = [&]() {
      const int s = n % t.stages;
      mbar_wait(&bars[s], (n / t.stages) & 1);
      tc_fence_after();
      ++n;
      return s;
    };
    auto gemm1 = [&](const uint8_t* op, int kp, uint32_t dcol) {
      const uint8_t* lo = op + BM * kp * 2;
      for (int ks = 0; ks < kp / 16; ++ks) {
        const int s = take();
        const uint32_t sb = smem_u32(ring + s * t.stage_bytes);
        const uint64_t ah = make_sdesc(smem_u32(op) + ks * 2 * lbo_op, lbo_op, 128);
        const uint64_t al = make_sdesc(smem_u32(lo) + ks * 2 * lbo_op, lbo_op, 128);
        const uint64_t bh = make_sdesc(sb, lbo1, 128), bl = make_sdesc(sb + half1, lbo1, 128);
        if (el) mma_f16_ss(tmem + dcol, ah, bh, id1, ks > 0 ? 1u : 0u);
        if (el) mma_f16_ss(tmem + dcol, ah, bl, id1, 1u);
        if (el) mma_f16_ss(tmem + dcol, al, bh, id1, 1u);
        if (el) tc_commit(&bars[kMaxStages + s]);
        __syncwarp();
      }
    };
    int it = 0;
    const long long tstart = now();
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      long long t0 = now();
      mbar_wait(&bars[B_OPS_READY], it & 1);
      tc_fence_after();
      tick(9, t0);
      t0 = now();
      gemm1(yop, t.k2, static_cast<uint32_t>(t.n1));  // Y block: free once the previous GEMM 2 issued
      tick(10, t0);
      if (it > 0) {
        t0 = now();
        mbar_wait(&bars[B_D_FREE], (it - 1) & 1);  // previous epilogue drained columns [0, n2)
        tc_fence_after();
        tick(11, t0);
      }
      t0 = now();
      gemm1(xop, t.k1, 0u);
      if (el) tc_commit(&bars[B_G1_DONE]);
      __syncwarp();
      tick(10, t0);
      t0 = now();
      mbar_wait(&bars[B_Z_READY], it & 1);
      tc_fence_after();
      tick(12, t0);
      t0 = now();
      int ks = 0;
      for (int g = 0; g < 4; ++g)  // Z groups in K order: (block 0, half 0), (0, 1), (1, 0), (1, 1)
        for (int c = 0; c < t.zgrp_size[g]; c += 16, ++ks) {
          const int s = take();
          const uint32_t sb = smem_u32(ring + s * t.stage_bytes);
          const uint32_t zh = tmem + static_cast<uint32_t>(t.zgrp_col[g] + c);
          const uint64_t bh = make_sdesc(sb, lbo2, 128), bl = make_sdesc(sb + half2, lbo2, 128);
          if (el) mma_f16_ts(tmem, zh, bh, id2, ks > 0 ? 1u : 0u);
          if (el) mma_f16_ts(tmem, zh, bl, id2, 1u);
          if (el) mma_f16_ts(tmem, zh + 8, bh, id2, 1u);
          if (el) tc_commit(&bars[kMaxStages + s]);
          __syncwarp();
        }
      if (el) tc_commit(&bars[B_G2_DONE]);
      __syncwarp();
      tick(13, t0);
    }
    tick(14, tstart);
    if (PROF && lane == 0)
      for (int k = 9; k < 15; ++k) g_mtp_prof[blockIdx.x * kProfSlots + k] = pc[k];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 9) tmem_dealloc(tmem, 512);
}

template <int DT>
cudaError_t launch_dt(const MtpTcTables& t, const RowSpec& rs, int num_sms, cudaStream_t s) {
  static const bool prof = [] {
    const char* v = std::getenv("TPO_MTP_PROF");
    return v && *v == '1';
  }();
  auto kern = prof ? mtp_tc_kernel<DT, true> : mtp_tc_kernel<DT, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, t.smem_bytes);
  if (e != cudaSuccess) return e;
  const int64_t ntiles = (rs.rows + BM - 1) / BM;
  const int grid = static_cast<int>(std::min<int64_t>(ntiles, num_sms));
  unsigned long long* buf = nullptr;
  if (prof) {
    cudaMalloc(&buf, sizeof(unsigned long long) * kProfSlots * grid);
    cudaMemset(buf, 0, sizeof(unsigned long long) * kProfSlots * grid);
    cudaMemcpyToSymbol(g_mtp_prof, &buf, sizeof(buf));
  }
  kern<<<grid, kThreads, t.smem_bytes, s>>>(t, rs);
  e = cudaGetLastError();
  if (prof && e == cudaSuccess) {
    std::vector<unsigned long long> h(kProfSlots * grid);
    cudaStreamSynchronize(s);
    cudaMemcpy(h.data(), buf, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    double avg[kProfSlots] = {};
    for (int b = 0; b < grid; ++b)
      for (int k = 0; k < kProfSlots; ++k) avg[k] += static_cast<double>(h[b * kProfSlots + k]) / grid;
    std::fprintf(stderr,
                 "[tpo-prof] mtp dt=%d tiles=%lld grid=%d | conv: total %.0f stage %.0f wait_g1 %.0f convert %.0f "
                 "wait_g2 %.0f epilogue %.0f | middle: wait_g1 %.0f pass0 %.0f pass1 %.0f | mma: wait_ops %.0f "
                 "gemm1 %.0f wait_dfree %.0f wait_z %.0f gemm2 %.0f total %.0f\n",
                 t.dt, static_cast<long long>(ntiles), grid, avg[0], avg[1], avg[2], avg[3], avg[4], avg[5], avg[6],
                 avg[7], avg[8], avg[9], avg[10], avg[11], avg[12], avg[13], avg[14]);
    cudaFree(buf);
  }
  return e;
}

}  // namespace

cudaError_t launch_mtp_tc(const MtpTcTables& t, const RowSpec& rs, int num_sms, cudaStream_t s) {
  if (rs.rows <= 0) return cudaSuccess;
  switch (t.dt) {
    case 1: return launch_dt<1>(t, rs, num_sms, s);
    case 3: return launch_dt<3>(t, rs, num_sms, s);
    case 5: return launch_dt<5>(t, rs, num_sms, s);
    case 7: return launch_dt<7>(t, rs, num_sms, s);
    case 9: return launch_dt<9>(t, rs, num_sms, s);
    case 11: return launch_dt<11>(t, rs, num_sms, s);
    case 13: return launch_dt<13>(t, rs, num_sms, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace tpo_b200
