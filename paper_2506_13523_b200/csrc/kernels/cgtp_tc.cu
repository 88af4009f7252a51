// Clebsch-Gordan tensor product on tcgen05, per (l1, l2) block.
//
// Reference: tpo::cgtp_mimo (proj/src/cgtp.cpp:145-177) walks the paths
// (l1, l2, l3) in lexicographic order and contracts each real CG table
// (proj/src/cgtp.cpp:120-143).  For fixed (l1, l2) the outputs of all l3 form
// one contiguous block of (2 l1 + 1)(2 l2 + 1) coefficients, and
//   out_block = W_{l1 l2} . (x_{l1} (x) y_{l2})
// where W is the square real-CG change of basis and x (x) y the outer product.
// Per 128-row tile and block that is one dense GEMM
//   D[128 x n] = P[128 x n] . W^T,   P[r][m1 * (2 l2 + 1) + m2] = x_r[l1, m1] y_r[l2, m2]
// on the tensor cores (3xFP16: hi*hi + hi*lo + lo*hi, fp32 accumulation in
// TMEM, rows scaled by exact powers of two).  The dense W spends ~n/4 more
// multiplies than the CG nonzeros, which the tensor pipe absorbs: the kernel is
// bound by the output write ((L+1)^4 floats per product).
//
// Warps: 0 TMA producer of the W ring, 1 MMA issuer (converged, elected lane),
// 2-9 P builders (two threads per tile row, 8 products of each K-step each ->
// fp16 hi/lo canonical A stages), 10-17 epilogue (two warps per TMEM lane
// quarter on alternating 32-column blocks; two 256-column accumulators
// alternate, so one super-unit of consecutive blocks drains while the next
// computes).
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
constexpr int kWarps = kThreads / 32;
constexpr int kMaxStages = 8;
constexpr int kStageStride = 33;  // epilogue staging row pitch (32-column blocks)
constexpr int kKps = 2;      // K-steps per A stage
constexpr int kDCols = kCgtpDCols;  // TMEM: two accumulators [0, 192), [192, 384) ...
constexpr int kARing = 2 * kDCols;  // ... and the A ring [384, 512): stage sa, K-step j: hi at 32 sa + 16 j, lo + 8
constexpr int kAStagesTmem = kCgtpAStages;
constexpr int kXSeg = 33;  // staged x_{l1} segment: 2 l1 + 1 <= 33 (l1 <= 16)
constexpr int kYSeg = 40;  // staged y_{l2} segment (t.yseg): 2 l2 + 1 <= 33, read up to 8 cpr <= 40
constexpr int kYSegPitch = kYSeg + 1;
// barriers: A full [8], A empty [8], B full [8], B empty [8], D full [2], D empty [2]
constexpr int B_AF = 0, B_AE = 8, B_BF = 16, B_BE = 24, B_DF = 32, B_DE = 34, kBars = 36;

__device__ __forceinline__ void tmem_st4(uint32_t taddr, const uint32_t (&r)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(r[0]), "r"(r[1]),
               "r"(r[2]), "r"(r[3])
               : "memory");
}

// optional in-kernel cycle accounting (env TPO_CGTP_PROF=1), kProfSlots per CTA:
// 0 producer total, 1 producer ring waits | 2 MMA total, 3 A waits, 4 B waits, 5 D-empty waits |
// 6 builder total, 7 staging, 8 A-empty waits | 9 epilogue total, 10 D-full waits
constexpr int kProfSlots = 12;
__device__ unsigned long long* g_cgtp_prof = nullptr;

template <bool PROF>
__global__ void __launch_bounds__(kThreads, 1)
    cgtp_tc_kernel(const __grid_constant__ CgtpTcTables t, const __grid_constant__ RowSpec rs) {
  extern __shared__ __align__(128) uint8_t smem[];  // used directly: accesses stay in the shared space
  __shared__ __align__(8) uint64_t bars[kBars];
  __shared__ uint32_t tmem_sh;
  __shared__ int e_sh[2][BM];  // row scale exponent (x + y) by tile parity
  __shared__ int ex_sh[BM], ey_sh[BM];
  __shared__ float epi[8 * 32 * kStageStride];  // epilogue staging per epilogue warp

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t ntiles = (rs.rows + BM - 1) / BM;
  uint8_t* ring_b = smem + t.off_b;
  float* rowbuf = reinterpret_cast<float*>(smem + t.off_xy);  // [128][pitch]: y row | x_{l1} (odd pitch)
  float* yseg = rowbuf + BM * t.xy_pitch;  // t.yseg: [3][128][kYSegPitch] y_{l2} segments by block sequence

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
  auto now = [] { return clock64(); };
  auto tick = [&](int k, long long t0) {
    if (PROF) pc[k] += clock64() - t0;
  };
  const long long t_begin = clock64();

  if (warp == 0 || warp == kWarps - 1) {
    // ============================================= W ring producers
    // two issuing threads in different warps take alternate ring stages: one thread's bulk-copy
    // issue (~250 cycles per copy) would limit the W stream at large L
    if (lane == 0) {
      const int pid = warp == 0 ? 0 : 1;
      int nb = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
        for (int u = 0; u < t.nunits; ++u) {
          const CgtpTcUnit un = t.units[u];
          const uint32_t bytes = 64u * un.n_pad;
          for (int ks = 0; ks < un.ksteps; ++ks, ++nb) {
            if ((nb & 1) != pid) continue;
            const int s = nb % t.b_stages;
            const long long t0 = now();
            if (nb >= t.b_stages) mbar_wait(&bars[B_BE + s], ((nb / t.b_stages) - 1) & 1);
            tick(1, t0);
            mbar_arrive_expect_tx(&bars[B_BF + s], bytes);
            bulk_g2s(ring_b + s * t.b_stage_bytes, t.w + un.w_off + static_cast<size_t>(ks) * bytes, bytes,
                     &bars[B_BF + s]);
          }
        }
      tick(0, t_begin);
      if (PROF && pid == 0) for (int k = 0; k < 2; ++k) g_cgtp_prof[blockIdx.x * kProfSlots + k] = pc[k];
    }
  } else if (warp == 1) {
    // ============================================= MMA issuer
    const bool el = elect_one_sync();
    const uint32_t lbo_a = (BM / 8) * 128;
    int sa = 0, pa = 0, sb = 0, pb = 0, gs = 0;  // ring slots / phases, super-units issued
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
      for (int u = 0; u < t.nunits; ++u) {
        const CgtpTcUnit un = t.units[u];
        const int d = gs & 1;
        const int dcol = un.dcol_last & 0xFFFF;
        if (dcol == 0 && gs >= 2) {  // first unit of a super-unit: its accumulator was drained
          const long long t0 = now();
          mbar_wait(&bars[B_DE + d], ((gs >> 1) - 1) & 1);
          tc_fence_after();
          tick(5, t0);
        }
        const uint32_t id = idesc_f16(BM, un.n_pad);
        const uint32_t lbo_b = (un.n_pad / 8) * 128, half_b = 32u * un.n_pad;
        for (int ks = 0; ks < un.ksteps; ++ks) {
          const int j = ks & (kKps - 1);  // K-step inside the A stage (units start a new stage)
          long long t0 = now();
          if (j == 0) mbar_wait(&bars[B_AF + sa], pa);
          tick(3, t0);
          t0 = now();
          mbar_wait(&bars[B_BF + sb], pb);
          tick(4, t0);
          tc_fence_after();
          const uint32_t ah = tmem + kARing + 32u * sa + 16u * j, al = ah + 8u;  // P in TMEM (TS mode)
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
        if (un.dcol_last >> 16) {  // last unit of the super-unit
          if (el) tc_commit(&bars[B_DF + d]);
          __syncwarp();
          ++gs;
        }
      }
    tick(2, t_begin);
    if (PROF && lane == 0) for (int k = 2; k < 6; ++k) g_cgtp_prof[blockIdx.x * kProfSlots + k] = pc[k];
  } else if (warp < 10) {
    // ============================================= P builders (two threads per tile row)
    // K order inside a block: k = m1 * n2p + m2 with n2p = 2 l2 + 1 padded to 8, so each
    // thread's 8-product chunk (chunk 2 ks + h of the block) is one x value times 8
    // consecutive y values (W has zero columns at the padding).
    // TMEM lane access: warp w reaches lanes 32 (w % 4) ..; two warps per quarter split the K-step
    const int r = 32 * (warp & 3) + lane, h = (warp - 2) >> 2, pt = h * BM + r;
    const uint32_t lbw = tmem + (static_cast<uint32_t>(32 * (warp & 3)) << 16);
    float* row = rowbuf + r * t.xy_pitch;  // y row (scaled) at [0, din2), x_{l1} (scaled) at [din2, din2 + kXSeg)
    int sa = 0, pa = 0, na = 0, it = 0;    // A ring slot / phase / stages produced
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int64_t g = tile * BM + r;
      const bool ok = g < rs.rows;
      const float* xr = rs.x + (ok ? g : 0) * t.din1;
      const long long ts0 = now();
      named_bar_sync(1, 2 * BM);  // both halves are done with the previous tile's row
      if (h == 1 && t.yseg) {  // y segments are staged per block below: only the row scale here
        const float* yr = rs.y + (rs.y_shared ? g / rs.channels : g) * t.din2;
        float m0 = 0.f, m1 = 0.f, m2 = 0.f, m3 = 0.f;
        if (ok) {
          int k = 0;
          for (; k + 4 <= t.din2; k += 4) {
            m0 = fmaxf(m0, fabsf(__ldg(yr + k))); m1 = fmaxf(m1, fabsf(__ldg(yr + k + 1)));
            m2 = fmaxf(m2, fabsf(__ldg(yr + k + 2))); m3 = fmaxf(m3, fabsf(__ldg(yr + k + 3)));
          }
          for (; k < t.din2; ++k) m0 = fmaxf(m0, fabsf(__ldg(yr + k)));
        }
        ey_sh[r] = row_scale_exp(fmaxf(fmaxf(m0, m1), fmaxf(m2, m3)), 1) - kInShift;
      } else if (h == 1) {  // stage the y row: every load in flight at once
        if (ok) {
          const float* yr = rs.y + (rs.y_shared ? g / rs.channels : g) * t.din2;
          for (int k = 0; k < t.din2; ++k) cp_async4(row + k, yr + k);
          cp_async_wait_all();
        } else {
          for (int k = 0; k < t.din2; ++k) row[k] = 0.f;
        }
        float m0 = 0.f, m1 = 0.f;
        int k = 0;
        for (; k + 2 <= t.din2; k += 2) {
          m0 = fmaxf(m0, fabsf(row[k]));
          m1 = fmaxf(m1, fabsf(row[k + 1]));
        }
        if (k < t.din2) m0 = fmaxf(m0, fabsf(row[k]));
        const int ey = row_scale_exp(fmaxf(m0, m1), 1) - kInShift;  // max|y| 2^-ey in [2^6, 2^7)
        const float sy = pow2i(-ey);
        for (k = 0; k < t.din2; ++k) row[k] *= sy;
        ey_sh[r] = ey;
      } else {  // x row norm (its degree segments are staged per l1 below)
        float m0 = 0.f, m1 = 0.f, m2 = 0.f, m3 = 0.f;
        if (ok) {
          int k = 0;
          for (; k + 4 <= t.din1; k += 4) {
            m0 = fmaxf(m0, fabsf(__ldg(xr + k))); m1 = fmaxf(m1, fabsf(__ldg(xr + k + 1)));
            m2 = fmaxf(m2, fabsf(__ldg(xr + k + 2))); m3 = fmaxf(m3, fabsf(__ldg(xr + k + 3)));
          }
          for (; k < t.din1; ++k) m0 = fmaxf(m0, fabsf(__ldg(xr + k)));
        }
        ex_sh[r] = row_scale_exp(fmaxf(fmaxf(m0, m1), fmaxf(m2, m3)), 1) - kInShift;
      }
      named_bar_sync(1, 2 * BM);
      const int ex = ex_sh[r];
      if (h == 0) e_sh[it & 1][r] = ex + ey_sh[r] - kTabShift;  // W is stored times 2^kTabShift
      // with per-block y segments the raw y values are staged and y's scale rides on x
      const float sx = t.yseg ? pow2i(-ex - ey_sh[r]) : pow2i(-ex);
      tick(7, ts0);
      int cur_l1 = -1;
      // per-block y segments (t.yseg, large din2): the h = 1 thread of each row copies the segment
      // of the next block with cp.async while this block is built (zero-filled past 2 l2 + 1), three
      // buffers by block sequence: the one refilled was last read two blocks ago
      const float* yrow = rs.y + (ok ? (rs.y_shared ? g / rs.channels : g) : 0) * t.din2;
      auto stage_seg = [&](int uu, int buf) {
        if (h == 1 && uu < t.nunits) {
          const int l2 = t.units[uu].l2, n2 = 2 * l2 + 1;
          float* dst = yseg + (buf * BM + r) * kYSegPitch;
          for (int j = 0; j < kYSeg; ++j) {
            const bool v = ok && j < n2;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst + j)),
                         "l"(yrow + (v ? l2 * l2 + j : 0)), "r"(v ? 4 : 0)
                         : "memory");
          }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      };
      int bs = -1;  // block sequence number inside the tile (t.yseg)
      if (t.yseg) {
        named_bar_sync(1, 2 * BM);  // both halves are past the previous tile's segments
        stage_seg(0, 0);
      }
      for (int u = 0; u < t.nunits; ++u) {
        const CgtpTcUnit un = t.units[u];
        const int n1 = 2 * un.l1 + 1, n2p = (2 * un.l2 + 1 + 7) & ~7, cpr = n2p >> 3;
        if (t.yseg && (u == 0 || t.units[u - 1].l2 != un.l2 || t.units[u - 1].l1 != un.l1)) {
          ++bs;
          int nu = u + 1;  // first unit of the next block
          while (nu < t.nunits && t.units[nu].l1 == un.l1 && t.units[nu].l2 == un.l2) ++nu;
          stage_seg(nu, (bs + 1) % 3);
          asm volatile("cp.async.wait_group 1;" ::: "memory");  // this block's segment landed
          named_bar_sync(1, 2 * BM);                              // ... in every row
        }
        if (un.l1 != cur_l1) {  // restage x_{l1} (both halves are past the previous block)
          named_bar_sync(1, 2 * BM);
          if (h == 0)
            for (int j = 0; j < kXSeg; ++j)  // zeros past n1: y reads may run into this segment (times 0 in W)
              row[(t.yseg ? 0 : t.din2) + j] = (ok && j < n1) ? __ldg(xr + un.l1 * un.l1 + j) * sx : 0.f;
          named_bar_sync(1, 2 * BM);
          cur_l1 = un.l1;
        }
        const float* xs = row + (t.yseg ? 0 : t.din2);
        const float* ys = t.yseg ? yseg + ((bs % 3) * BM + r) * kYSegPitch : row + un.l2 * un.l2;
        // chunk c = h + 2 k of this thread (8 products: x index m1 = c / cpr, y offset 8 (c % cpr)),
        // advanced incrementally: every K-step moves c by 2
        int m1 = cpr == 1 ? h : 0, rem = cpr == 1 ? 0 : h;
        for (int ks0 = 0; ks0 < un.ksteps; ks0 += kKps) {  // one A stage = kKps K-steps
          const long long t0 = now();
          if (na++ >= kAStagesTmem) {
            mbar_wait(&bars[B_AE + sa], pa ^ 1);
            tc_fence_after();
          }
          tick(8, t0);
#pragma unroll
          for (int j = 0; j < kKps; ++j) {  // (tail sub-steps past the unit are built but never issued)
            const float xv = m1 < n1 ? xs[m1] : 0.f;
            const float* yp = ys + 8 * rem;
            uint32_t hw[4], lw[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float p0 = xv * yp[2 * q], p1 = xv * yp[2 * q + 1];
              const __half2 hh = __floats2half2_rn(p0, p1);
              const float2 hf = __half22float2(hh);
              hw[q] = *reinterpret_cast<const uint32_t*>(&hh);
              lw[q] = pack_half2(p0 - hf.x, p1 - hf.y);
            }
            // this thread's 8 products = 4 packed columns of the K-step's hi and lo blocks
            const uint32_t col = kARing + 32u * sa + 16u * j + 4u * h;
            tmem_st4(lbw + col, hw);
            tmem_st4(lbw + col + 8u, lw);
            rem += 2;  // next chunk of this thread: c + 2
            if (rem >= cpr) {
              rem -= cpr;
              ++m1;
            }
            if (rem >= cpr) {
              rem -= cpr;
              ++m1;
            }
          }
          const long long tf = now();
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive_warp(&bars[B_AF + sa]);
          tick(11, tf);
          if (++sa == kAStagesTmem) {
            sa = 0;
            pa ^= 1;
          }
        }
      }
    }
    tick(6, t_begin);
    if (PROF && pt == 0) for (int k : {6, 7, 8, 11}) g_cgtp_prof[blockIdx.x * kProfSlots + k] = pc[k];
  } else if (warp < kWarps - 1) {
    // ============================================= epilogue (thread = TMEM lane)
    const int q = warp & 3, eh = (warp - 10) >> 2;  // lane quarter, which of its two warps
    const uint32_t lb = tmem + (static_cast<uint32_t>(q * 32) << 16);
    float* st = epi + (warp - 10) * 32 * kStageStride;
    const int64_t stride = t.dout;
    int gs = 0, it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int64_t row0 = tile * BM + q * 32;
      const int64_t left = rs.rows - row0;
      const int nr = left >= 32 ? 32 : (left > 0 ? static_cast<int>(left) : 0);
      for (int u0 = 0; u0 < t.nunits; ++gs) {
        int u1 = u0;  // units [u0, u1] form this super-unit
        while (!(t.units[u1].dcol_last >> 16)) ++u1;
        const CgtpTcUnit ul = t.units[u1];
        const int ncols = (ul.dcol_last & 0xFFFF) + ul.n_pad;  // multiple of 16
        const int d = gs & 1;
        const long long t0 = now();
        mbar_wait(&bars[B_DF + d], (gs >> 1) & 1);
        tc_fence_after();
        tick(10, t0);
        const int e_row = e_sh[it & 1][q * 32 + lane];
        const float s_lo = pow2i(e_row >> 1), s_hi = pow2i(e_row - (e_row >> 1));  // exact, split for range
        const uint32_t dbase = lb + static_cast<uint32_t>(kDCols) * d;
        int uu = u0;
        // 32-column blocks (the last may be 16 wide), alternating between the quarter's two warps
        for (int c0 = 32 * eh; c0 < ncols; c0 += 64) {
          uint32_t v[32];
          tmem_ld16(dbase + c0, *reinterpret_cast<uint32_t(*)[16]>(v));
          if (c0 + 16 < ncols) tmem_ld16(dbase + c0 + 16, *reinterpret_cast<uint32_t(*)[16]>(v + 16));
          tmem_wait_ld();
#pragma unroll
          for (int k = 0; k < 32; ++k) st[lane * kStageStride + k] = __uint_as_float(v[k]) * s_lo * s_hi;
          __syncwarp();
          // column c0 + lane of the accumulator -> unit -> output column
          const int c = c0 + lane;
          while (uu < u1 && (t.units[uu].dcol_last & 0xFFFF) + t.units[uu].n_pad <= c0) ++uu;
          int um = uu;
          while (um < u1 && (t.units[um].dcol_last & 0xFFFF) + t.units[um].n_pad <= c) ++um;
          const CgtpTcUnit un = t.units[um];
          const int col = c - (un.dcol_last & 0xFFFF);
          if (c < ncols && col < un.n_valid) {
            float* op = rs.out + row0 * stride + un.out_off + col;
            const float* sp = st + lane;
#pragma unroll 8
            for (int rr = 0; rr < 32; ++rr, op += stride, sp += kStageStride)
              if (rr < nr) *op = *sp;
          }
          __syncwarp();
        }
        tc_fence_before();
        mbar_arrive_warp(&bars[B_DE + d]);
        u0 = u1 + 1;
      }
    }
    tick(9, t_begin);
    if (PROF && warp == 10 && lane == 0) for (int k = 9; k < 11; ++k) g_cgtp_prof[blockIdx.x * kProfSlots + k] = pc[k];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

}  // namespace

cudaError_t launch_cgtp_tc(const CgtpTcTables& t, const RowSpec& rs, int num_sms, cudaStream_t s) {
  if (rs.rows <= 0) return cudaSuccess;
  static const bool prof = [] {
    const char* v = std::getenv("TPO_CGTP_PROF");
    return v && *v == '1';
  }();
  auto kern = prof ? cgtp_tc_kernel<true> : cgtp_tc_kernel<false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, t.smem_bytes);
  if (e != cudaSuccess) return e;
  const int64_t ntiles = (rs.rows + BM - 1) / BM;
  const int grid = static_cast<int>(std::min<int64_t>(ntiles, num_sms));
  unsigned long long* buf = nullptr;
  if (prof) {
    cudaMalloc(&buf, sizeof(unsigned long long) * kProfSlots * grid);
    cudaMemset(buf, 0, sizeof(unsigned long long) * kProfSlots * grid);
    cudaMemcpyToSymbol(g_cgtp_prof, &buf, sizeof(buf));
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
                 "[tpo-prof] cgtp tiles=%lld | producer %.0f ring %.0f | mma %.0f a_wait %.0f b_wait %.0f d_empty %.0f | "
                 "builder %.0f staging %.0f a_empty %.0f fence %.0f | epilogue %.0f d_full %.0f\n",
                 static_cast<long long>(ntiles), avg[0], avg[1], avg[2], avg[3], avg[4], avg[5], avg[6], avg[7], avg[8],
                 avg[11], avg[9], avg[10]);
    cudaFree(buf);
  }
  return e;
}

}  // namespace tpo_b200
