// Fused S2-grid Gaunt tensor product on the 5th-generation tensor cores.
//
// Reference path: tpo::detail::gtp_grid_select (proj/src/gtp.cpp:228-260) =
// to_sphere (proj/src/sphere.cpp:105-134) x2, pointwise_mul (:145-151),
// from_sphere_select (:155-195).  Per 128-row tile and output group g:
//   F_x = X S1^T,  F_y = Y S2^T     (SH -> grid, GEMM 1, TMEM accumulators)
//   P   = F_x (.) F_y               (pointwise product, written back to TMEM)
//   Z_g += P A_g^T                  (grid -> SH quadrature, GEMM 2, A from TMEM)
// chunk by chunk (nc grid points) over the product grid, so grid values never
// leave the SM.  S[g][(l,m)] = Lambda_{l|m|}(theta_j) cs_m(phi_k) and
// A[(l,m)][g] = w_j (2 pi / n_phi) Lambda_{l|m|}(theta_j) cs_m(phi_k) are built
// by host/context.cpp on the reference's product grid (band L1+L2).
//
// Precision: "3xFP16".  Every fp32 operand v is split v = hi + lo (fp16 each)
// and products use hi*hi + hi*lo + lo*hi with fp32 accumulation.  fp16's
// range is made safe by exact power-of-two scaling: each input row is scaled
// so that ||x||_2 in [0.5, 1) (|F| <= (L+1)/sqrt(4 pi) by the addition
// theorem), the A table by 2^a_shift; the epilogue rescales exactly.
//
// Warp roles (one persistent CTA per SM, 10 warps):
//   warp 0     TMA producer: B-operand slices (S / A tables, one K-step each)
//              through an mbarrier ring; raw input tiles (1D bulk copies).
//   warp 1     MMA issuer (one thread) + TMEM owner.
//   warps 2-9  workers: input conversion (norm, split, canonical layout),
//              pointwise product TMEM -> TMEM, epilogue TMEM -> HBM.
// MMA shapes are M = 128 and N >= 96 wherever possible: the tcgen05 issue
// floor measured on B200 is ~45 cycles per instruction (tools/ubench), so
// narrow MMAs would be issue-bound.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kernels.hpp"
#include "sm100.cuh"

namespace tpo_b200 {
using namespace sm100;

namespace {

constexpr int BM = 128;            // rows per tile == TMEM lanes
constexpr int kWorkerWarps = 8;
constexpr int kWorkers = kWorkerWarps * 32;
constexpr int kThreads = 96 + kWorkers;  // + producer A warp (warp 10)
constexpr int kKHalfMax = 88;      // input K (padded) <= 176 (L <= 12), split over 2 threads per row
constexpr int kKHalfStd = 64;      // K <= 128 (L <= 10): the default instantiation (no spills at 168 registers)
constexpr int kStageStride = 17;   // epilogue staging row pitch (floats)
constexpr int kMaxStages = 8;
constexpr int kMaxSlices = 8;      // nc <= 128

// barrier slots: two B-operand rings (S table for GEMM 1, A table for GEMM 2),
// each fed by its own producer warp -- a single thread issues at most one
// bulk copy per ~250 cycles (tools/ubench/tma_ubench.cu)
constexpr int B_SFULL = 0;
constexpr int B_SEMPTY = B_SFULL + kMaxStages;
constexpr int B_AFULL = B_SEMPTY + kMaxStages;
constexpr int B_AEMPTY = B_AFULL + kMaxStages;
constexpr int B_RAW_FULL = B_AEMPTY + kMaxStages;
constexpr int B_RAW_FREE = B_RAW_FULL + 1;
constexpr int B_XY_FREE = B_RAW_FREE + 1;
constexpr int B_XY_READY = B_XY_FREE + 1;
constexpr int B_F_FULL = B_XY_READY + 1;
constexpr int B_P_READY = B_F_FULL + 1;
constexpr int B_G2_DONE = B_P_READY + kMaxSlices;
constexpr int B_Z_FULL = B_G2_DONE + 1;
constexpr int B_Z_EMPTY = B_Z_FULL + 1;
constexpr int kNumBars = B_Z_EMPTY + 1;

struct Unit {
  int64_t tile;
  int g;
};

__device__ __forceinline__ Unit unit_of(int64_t u, int ngroups) {
  return Unit{u / ngroups, static_cast<int>(u % ngroups)};
}

// worker idx of cnt owns the contiguous unit range [u_begin, u_end):
// consecutive units are the output groups of one tile, which then reuses its
// resident X / Y
__device__ __forceinline__ void unit_range(int64_t nunits, int64_t idx, int64_t cnt, int64_t& u_begin,
                                           int64_t& u_end) {
  u_begin = nunits * idx / cnt;
  u_end = nunits * (idx + 1) / cnt;
}

// arrive `count` on a barrier of the MMA-issuing CTA (the pair leader, rank 0).
// kTmemOnly: the dependency is TMEM traffic already completed and fenced
// (tcgen05.wait + fence::before_thread_sync), so the remote arrive can be
// relaxed and does not wait for this thread's outstanding global stores.
template <bool PAIR, bool kTmemOnly = false>
__device__ __forceinline__ void arrive_leader(uint64_t* bar, uint32_t count, uint32_t rank) {
  if (PAIR && rank != 0) {
    if (kTmemOnly) mbar_arrive_cluster_relaxed(mapa_shared(smem_u32(bar), 0), count);
    else mbar_arrive_cluster(mapa_shared(smem_u32(bar), 0), count);
  } else {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  }
}
template <bool PAIR>
__device__ __forceinline__ void wait_leader(uint64_t* bar, uint32_t parity) {
  if (PAIR) mbar_wait_cluster(bar, parity);
  else mbar_wait(bar, parity);
}

// a tile whose x / y rows are one contiguous, 16-byte aligned block can be
// fetched with two bulk copies; anything else (tail tile, shared y, odd base
// pointer) is gathered by the workers
__device__ __forceinline__ bool tile_tma_ok(const RowSpec& rs, int64_t tile) {
  return !rs.y_shared && (tile + 1) * BM <= rs.rows && ((reinterpret_cast<uintptr_t>(rs.x) & 15) == 0) &&
         ((reinterpret_cast<uintptr_t>(rs.y) & 15) == 0);
}

// degree of flat index k = l^2 + m + l (exact for k < 2^20)
__device__ __forceinline__ int degree_of(int k) { return __float2int_rd(sqrtf(static_cast<float>(k) + 0.5f)); }

// Convert one input of the tile: raw fp32 rows [128][din] in shared memory ->
// fp16 hi / lo in the canonical K-major layout (R = 128, K = kp), each row
// scaled by 2^-e with ||row||_2 * 2^-e < 1 (row_scale_exp).  Thread (r, h) owns half
// h of row r.  Two phases separated by a worker barrier, so the raw rows may
// alias the destination (in-place mode).
// in-place staging (raw rows share the operand buffers): every value is read into registers
// before the barrier, so no thread overwrites a raw value another thread has yet to read
template <int KH>
__device__ __noinline__ void convert_input_regs(const float* raw, const float* wdeg, int din, int kp, int in_shift,
                                                   uint8_t* dst_hi, uint8_t* dst_lo, float* part, int16_t* e_out, int r,
                                                   int h, bool wait_free, uint64_t* xy_free, uint32_t xy_free_par) {
  const int kh = kp >> 1;  // multiple of 8
  const int k0 = h * kh;
  const float* src = raw + r * din + k0;
  const int nv = min(kh, din - k0);  // valid raw values of this half (may be <= 0)
  float v[KH];
  float mx = 0.f;
  if ((din & 3) == 0) {
    // rows of a multiple of 4 floats sit a multiple of 16 B apart: 128-bit reads (a scalar
    // read of the same k by 32 rows would hit one bank 32 / gcd-fold, e.g. 32-way at din = 64)
    const float4* src4 = reinterpret_cast<const float4*>(src);
#pragma unroll
    for (int j0 = 0; j0 < KH; j0 += 4) {
      if (j0 < kh) {
        const float4 a = (j0 < nv) ? src4[j0 >> 2] : make_float4(0.f, 0.f, 0.f, 0.f);
        v[j0] = a.x; v[j0 + 1] = a.y; v[j0 + 2] = a.z; v[j0 + 3] = a.w;
      }
    }
  } else {
#pragma unroll
    for (int j0 = 0; j0 < KH; j0 += 8) {
      if (j0 < kh) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          v[j0 + q] = (j0 + q < nv) ? src[j0 + q] : 0.f;
        }
      }
    }
  }
  if (wdeg) {  // fused per-degree input weights (weighted GTP)
#pragma unroll
    for (int j = 0; j < KH; ++j)
      if (j < kh) v[j] *= wdeg[k0 + j];
  }
#pragma unroll
  for (int j = 0; j < KH; ++j)
    if (j < kh) mx = fmaxf(mx, fabsf(v[j]));
  part[h * BM + r] = mx;
  named_bar_sync(1, kWorkers);
  if (wait_free) mbar_wait(xy_free, xy_free_par);  // the previous unit's GEMM 1 has retired
  // ||x||_2 2^-e < 2^in_shift: the products F_x F_y stay below 2^14 (host bound), far from fp16's
  // subnormal range for all but negligible values
  const int e = row_scale_exp(fmaxf(part[r], part[BM + r]), din) - in_shift;
  const float sc = pow2i(-e);
#pragma unroll
  for (int j0 = 0; j0 < KH; j0 += 8) {
    if (j0 < kh) {
      uint32_t hw[4], lw[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float a0 = v[j0 + 2 * q] * sc, a1 = v[j0 + 2 * q + 1] * sc;
        const __half2 hh = __floats2half2_rn(a0, a1);
        const float2 hf = __half22float2(hh);
        hw[q] = *reinterpret_cast<const uint32_t*>(&hh);
        lw[q] = pack_half2(a0 - hf.x, a1 - hf.y);
      }
      const uint32_t off = canon_off(r, k0 + j0, BM);
      *reinterpret_cast<uint4*>(dst_hi + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
      *reinterpret_cast<uint4*>(dst_lo + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
  }
  e_out[h * BM + r] = static_cast<int16_t>(e);  // one copy per worker half: (r, h) reads its own in the epilogue
}

__device__ __noinline__ void convert_input(const float* raw, const float* wdeg, int din, int kp, int in_shift,
                                              uint8_t* dst_hi, uint8_t* dst_lo, float* part, int16_t* e_out, int r, int h,
                                              bool wait_free, uint64_t* xy_free, uint32_t xy_free_par) {
  // two short passes over the staged row (norm, then scale + split): small code, which
  // matters because this runs once per tile and is otherwise cold in the instruction cache
  const int kh = kp >> 1;  // multiple of 8
  const int k0 = h * kh;
  const float* src = raw + r * din + k0;
  const int nv = min(kh, din - k0);  // valid raw values of this half (may be <= 0)
  // rows of a multiple of 4 floats sit a multiple of 16 B apart: 128-bit reads (a scalar read of
  // the same k by 32 rows would hit one bank up to 32-fold, e.g. din = 64)
  const bool vec = (din & 3) == 0;
  auto load8 = [&](int j0, float (&v)[8]) {
    if (vec) {
      const float4* s4 = reinterpret_cast<const float4*>(src + j0);
      const float4 a = j0 < nv ? s4[0] : make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 b = j0 + 4 < nv ? s4[1] : make_float4(0.f, 0.f, 0.f, 0.f);
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = j0 + q < nv ? src[j0 + q] : 0.f;
    }
    if (wdeg) {  // fused per-degree input weights (weighted GTP)
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] *= wdeg[k0 + j0 + q];
    }
  };
  float mx0 = 0.f, mx1 = 0.f;
#pragma unroll 1
  for (int j0 = 0; j0 < kh; j0 += 8) {
    float v[8];
    load8(j0, v);
#pragma unroll
    for (int q = 0; q < 8; q += 2) {
      mx0 = fmaxf(mx0, fabsf(v[q]));
      mx1 = fmaxf(mx1, fabsf(v[q + 1]));
    }
  }
  part[h * BM + r] = fmaxf(mx0, mx1);
  named_bar_sync(1, kWorkers);
  if (wait_free) mbar_wait(xy_free, xy_free_par);  // the previous unit's GEMM 1 has retired
  // ||x||_2 2^-e < 2^in_shift: the products F_x F_y stay below 2^14 (host bound), far from fp16's
  // subnormal range for all but negligible values
  const int e = row_scale_exp(fmaxf(part[r], part[BM + r]), din) - in_shift;
  const float sc = pow2i(-e);
#pragma unroll 1
  for (int j0 = 0; j0 < kh; j0 += 8) {
    float v[8];
    load8(j0, v);
    uint32_t hw[4], lw[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float a0 = v[2 * q] * sc, a1 = v[2 * q + 1] * sc;
      const __half2 hh = __floats2half2_rn(a0, a1);
      const float2 hf = __half22float2(hh);
      hw[q] = *reinterpret_cast<const uint32_t*>(&hh);
      lw[q] = pack_half2(a0 - hf.x, a1 - hf.y);
    }
    const uint32_t off = canon_off(r, k0 + j0, BM);
    *reinterpret_cast<uint4*>(dst_hi + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
    *reinterpret_cast<uint4*>(dst_lo + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
  }
  e_out[h * BM + r] = static_cast<int16_t>(e);  // one copy per worker half: (r, h) reads its own in the epilogue
}

// Optional per-role cycle accounting (PROF = true; debugging aid, env
// TPO_GRID_PROF=1): slot layout per CTA in `g_prof` (unsigned long long):
//   MMA thread : 0 total, 1 wait xy_ready, 2 wait S ring, 3 wait p_ready, 4 wait z_empty, 5 wait g2_done,
//                6 wait A ring
//   worker w2  : 8 total, 9 wait f_full, 10 product, 11 convert, 12 wait z_full, 13 epilogue
constexpr int kProfSlots = 16;
__device__ unsigned long long* g_prof = nullptr;

// PAIR: CTA pairs (cluster of 2) run tcgen05.mma.cta_group::2 with M = 256:
// each CTA owns 128 rows (its own X / Y, TMEM lanes, epilogue) and streams
// only its half of every B operand (S / A slice halves), halving the shared
// memory read traffic of GEMM 1, the ring TMA writes per SM and -- most
// important -- the number of MMA instructions per unit of work.  Rank 0
// issues every MMA; its commits multicast to both CTAs; the rank-1 MMA warp
// forwards "my half landed" to rank 0's ring slots; workers signal rank 0.
// SEG: GEMM 2 runs in several accumulation segments (t.seg_chunks < t.nchunks); the single-segment
// instantiation compiles without the segment hand-offs and the L2 reductions.
template <bool PROF, bool PAIR, int KH = kKHalfStd, bool SEG = false>
__global__ void __launch_bounds__(kThreads, 1)
    gtp_grid_tc_kernel(const __grid_constant__ GridTcTables t, const __grid_constant__ RowSpec rs,
                       const __grid_constant__ DegreeWeights dw) {
  unsigned long long pc[kProfSlots];
#pragma unroll
  for (int k = 0; k < kProfSlots; ++k) pc[k] = 0;
  auto now = []() -> unsigned long long { return PROF ? clock64() : 0ull; };
  const unsigned long long t_start = now();
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[kNumBars];
  __shared__ uint32_t tmem_sh;
  __shared__ int16_t ex_sh[2][2 * BM], ey_sh[2][2 * BM];  // [tile parity][worker half][row] (same bytes as int [2][BM])
  __shared__ float part_sh[2 * BM];
  // weighted GTP: per-column weights (flat (l,m) index -> weight of degree l), filled once
  __shared__ float wtab_x[2 * KH], wtab_y[2 * KH], wtab_c[448];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  constexpr int kPair = PAIR ? 2 : 1;
  if (tid == 0) {
    for (int i = 0; i < kNumBars; ++i) {
      uint32_t cnt = 1;
      if (i == B_RAW_FREE) cnt = kWorkers;
      if (i == B_XY_READY || i == B_Z_EMPTY) cnt = kWorkers * kPair;
      if (i >= B_P_READY && i < B_P_READY + kMaxSlices) cnt = BM * kPair;
      mbar_init(&bars[i], cnt);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    if (PAIR) {
      tmem_alloc_pair(&tmem_sh, 512);
      tmem_relinquish_pair();
    } else {
      tmem_alloc(&tmem_sh, 512);
      tmem_relinquish();
    }
  }
  tc_fence_before();
  if (PAIR) cluster_sync_all();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_sh;

  // a unit tile is kPair x 128 rows; this CTA owns the 128 rows of tile ut * kPair + rank
  const int64_t ntiles = (rs.rows + BM * kPair - 1) / (BM * kPair);
  const int64_t nunits = ntiles * t.ngroups;
  int64_t u_begin, u_end;
  unit_range(nunits, blockIdx.x / kPair, gridDim.x / kPair, u_begin, u_end);
  auto my_tile = [&](int64_t ut) { return ut * kPair + rank; };
  uint8_t* xh = smem + t.off_x;
  uint8_t* xl = xh + BM * t.k1p * 2;
  uint8_t* yh = smem + t.off_y;
  uint8_t* yl = yh + BM * t.k2p * 2;
  float* raw_x = reinterpret_cast<float*>(smem + t.off_raw);
  float* raw_y = t.raw_inplace ? reinterpret_cast<float*>(smem + t.off_y) : raw_x + BM * t.din1;
  uint8_t* sring = smem + t.off_sring;
  uint8_t* aring = smem + t.off_aring;
  const uint32_t zc = static_cast<uint32_t>(t.zg);   // TMEM: Z [0, zg), F_x [zc, zc+nc), F_y [zc+nc, zc+2nc)
  const uint32_t fx = zc, fy = zc + t.nc;

  if (warp == 0) {
    // ===================================================== TMA producer
    // converged warp, elected lane issues (as for the MMA issuer)
    const bool pl = elect_one_sync();
    {
      int stage = 0;
      uint32_t ph = 0;
      auto push = [&](const uint8_t* src, uint32_t bytes, bool second) {
        mbar_wait(&bars[B_SEMPTY + stage], ph ^ 1);
        if (PAIR) {
          // both CTAs' halves complete on the leader's slot barrier (tensor TMA, cta_group::2)
          if (pl && leader) mbar_arrive_expect_tx(&bars[B_SFULL + stage], 2 * t.s_stage_bytes);
          const CUtensorMap* tm = second ? &t.tm_s2 : &t.tm_s1;
          const uint8_t* base = second ? t.s2 : t.s1;
          const int row = static_cast<int>((src - base + rank * t.s_stage_bytes) / 64);
          if (pl) tma2d_load_pair(sring + stage * t.s_stage_bytes, tm, 0, row, &bars[B_SFULL + stage]);
        } else {
          if (pl) mbar_arrive_expect_tx(&bars[B_SFULL + stage], t.s_stage_bytes);
          if (pl) bulk_g2s(sring + stage * t.s_stage_bytes, src, t.s_stage_bytes, &bars[B_SFULL + stage]);
        }
        if (++stage == t.s_stages) {
          stage = 0;
          ph ^= 1;
        }
      };
      // raw tile number v of this CTA: the destination must be free, i.e. tile
      // v-1's last GEMM 1 retired (in-place: raw lands in the X/Y operand
      // buffers) or the workers finished reading raw tile v-1 (separate buffer)
      auto issue_raw = [&](int64_t tile, int64_t v) {
        if (v > 0) mbar_wait(&bars[t.raw_inplace ? B_XY_FREE : B_RAW_FREE], static_cast<uint32_t>((v - 1) & 1));
        const uint32_t bx = BM * t.din1 * 4, by = BM * t.din2 * 4;
        if (pl) mbar_arrive_expect_tx(&bars[B_RAW_FULL], bx + by);
        if (pl) bulk_g2s(raw_x, rs.x + tile * BM * t.din1, bx, &bars[B_RAW_FULL]);
        if (pl) bulk_g2s(raw_y, rs.y + tile * BM * t.din2, by, &bars[B_RAW_FULL]);
      };
      int64_t v = 0;  // tile sequence number
      if (u_begin < u_end) {
        const Unit u0 = unit_of(u_begin, t.ngroups);
        if (tile_tma_ok(rs, my_tile(u0.tile))) issue_raw(my_tile(u0.tile), 0);
      }
      for (int64_t u = u_begin; u < u_end; ++u) {
        const Unit cu = unit_of(u, t.ngroups);
        const bool first_of_tile = (u == u_begin) || unit_of(u - 1, t.ngroups).tile != cu.tile;
        const bool last_of_tile = (u + 1 == u_end) || unit_of(u + 1, t.ngroups).tile != cu.tile;
        // the next tile of this CTA starts right after this tile's units
        const int64_t next_u = u + (t.ngroups - cu.g);
        const bool has_next = next_u < u_end;
        for (int c = 0; c < t.nchunks; ++c) {
          for (int ks = 0; ks < t.k1p / 16; ++ks)
            push(t.s1 + static_cast<size_t>(c * (t.k1p / 16) + ks) * t.s1_slice_bytes, t.s1_slice_bytes, false);
          if (!t.same_s)
            for (int ks = 0; ks < t.k2p / 16; ++ks)
              push(t.s2 + static_cast<size_t>(c * (t.k2p / 16) + ks) * t.s2_slice_bytes, t.s2_slice_bytes, true);
          const bool raw_point = t.raw_inplace ? (last_of_tile && c == t.nchunks - 1) : (first_of_tile && c == 0);
          if (raw_point && has_next) {
            const Unit nu = unit_of(next_u, t.ngroups);
            if (tile_tma_ok(rs, my_tile(nu.tile))) issue_raw(my_tile(nu.tile), v + 1);
          }
        }
        if (last_of_tile) ++v;
      }
    }
  } else if (warp == 10) {
    // ===================================================== TMA producer, A table (GEMM 2)
    const bool pl = elect_one_sync();
    {
      int stage = 0;
      uint32_t ph = 0;
      for (int64_t u = u_begin; u < u_end; ++u) {
        const Unit cu = unit_of(u, t.ngroups);
        const size_t abase = static_cast<size_t>(cu.g) * t.nchunks * t.nslices * t.nparts;
        const int n = t.nchunks * t.nslices * t.nparts;
        for (int k = 0; k < n; ++k) {
          mbar_wait(&bars[B_AEMPTY + stage], ph ^ 1);
          if (PAIR) {
            if (pl && leader) mbar_arrive_expect_tx(&bars[B_AFULL + stage], 2 * t.a_stage_bytes);
            const int row = static_cast<int>(((abase + k) * t.a_slice_bytes + rank * t.a_stage_bytes) / 64);
            if (pl) tma2d_load_pair(aring + stage * t.a_stage_bytes, &t.tm_a, 0, row, &bars[B_AFULL + stage]);
          } else {
            if (pl) mbar_arrive_expect_tx(&bars[B_AFULL + stage], t.a_stage_bytes);
            if (pl)
              bulk_g2s(aring + stage * t.a_stage_bytes, t.a + (abase + k) * t.a_slice_bytes, t.a_stage_bytes,
                       &bars[B_AFULL + stage]);
          }
          if (++stage == t.a_stages) {
            stage = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================================================== MMA issuer
    // The whole (converged) warp runs the loop and waits; one elected lane
    // issues each tcgen05 instruction.  Keeping the warp converged lets the
    // descriptors live in uniform registers without a divergent waterfall per
    // MMA, which lowers the per-instruction issue cost of the single issuer.
    const bool leader_lane = elect_one_sync();
    if (PAIR && !leader) {
      // rank 1: nothing to issue -- its TMA halves complete on the leader's barriers
    } else {
      int s_stage = 0, a_stage = 0;
      uint32_t s_ph = 0, a_ph = 0;
      // next slice of a ring: wait until it landed, return its shared-memory address
      auto take_s = [&](uint32_t& slot) -> uint32_t {
        slot = B_SEMPTY + s_stage;
        const auto t0 = now();
        wait_leader<PAIR>(&bars[B_SFULL + s_stage], s_ph);
        pc[2] += now() - t0;
        tc_fence_after();
        const uint32_t a = smem_u32(sring + s_stage * t.s_stage_bytes);
        if (++s_stage == t.s_stages) {
          s_stage = 0;
          s_ph ^= 1;
        }
        return a;
      };
      auto take_a = [&](uint32_t& slot) -> uint32_t {
        slot = B_AEMPTY + a_stage;
        const auto t0 = now();
        wait_leader<PAIR>(&bars[B_AFULL + a_stage], a_ph);
        pc[6] += now() - t0;
        tc_fence_after();
        const uint32_t a = smem_u32(aring + a_stage * t.a_stage_bytes);
        if (++a_stage == t.a_stages) {
          a_stage = 0;
          a_ph ^= 1;
        }
        return a;
      };
      // pair: M = 256 and each CTA's B tile is its row half (nc / 2 or zp / 2 rows)
      const uint32_t id1 = idesc_f16(BM * kPair, t.nc), id2 = idesc_f16(BM * kPair, t.zp);
      const uint32_t lbo_x = (BM / 8) * 128;
      const uint32_t bn_s = t.nc / kPair, bn_a = t.zp / kPair;
      const uint32_t lbo_s = (bn_s / 8) * 128, lbo_a = (bn_a / 8) * 128;
      const uint32_t s_half = bn_s * 32, a_half = bn_a * 32;  // lo block offset inside a stage
      const uint64_t dx_hi = make_sdesc(smem_u32(xh), lbo_x, 128), dx_lo = make_sdesc(smem_u32(xl), lbo_x, 128);
      const uint64_t dy_hi = make_sdesc(smem_u32(yh), lbo_x, 128), dy_lo = make_sdesc(smem_u32(yl), lbo_x, 128);
      const uint64_t kstep_x = (2 * lbo_x) >> 4;  // descriptor advance per K-step of X/Y
      int64_t j = 0;  // chunk counter
      int64_t i = 0;  // unit counter
      int64_t v = 0;  // tile sequence number
      int64_t d = 0;  // Z hand-offs to the epilogue (one per accumulation segment)
      for (int64_t u = u_begin; u < u_end; ++u, ++i) {
        const Unit cu = unit_of(u, t.ngroups);
        const bool first_of_tile = (u == u_begin) || unit_of(u - 1, t.ngroups).tile != cu.tile;
        const bool last_of_tile = (u + 1 == u_end) || unit_of(u + 1, t.ngroups).tile != cu.tile;
        if (first_of_tile) {
          const auto t0 = now();
          wait_leader<PAIR>(&bars[B_XY_READY], static_cast<uint32_t>(v & 1));
          pc[1] += now() - t0;
          tc_fence_after();
        }
        for (int c = 0; c < t.nchunks; ++c, ++j) {
          if (j > 0 && t.safe_war) {  // P of the previous chunk (in F_x) consumed
            const auto t0 = now();
            mbar_wait(&bars[B_G2_DONE], static_cast<uint32_t>((j - 1) & 1));
            pc[5] += now() - t0;
            tc_fence_after();
          }
          // ---- GEMM 1: F_x = X S1^T, F_y = Y S2^T (3xFP16)
          const int ks1 = t.k1p / 16;
          for (int ks = 0; ks < ks1; ++ks) {
            uint32_t slot;
            const uint32_t sb = take_s(slot);
            const uint64_t bh = make_sdesc(sb, lbo_s, 128), bl = make_sdesc(sb + s_half, lbo_s, 128);
            const uint64_t ah = dx_hi + ks * kstep_x, al = dx_lo + ks * kstep_x;
            const uint32_t acc = ks > 0 ? 1u : 0u;
            if (leader_lane) (PAIR ? mma_f16_ss_pair : mma_f16_ss)(tmem + fx, ah, bh, id1, acc);
            if (leader_lane) (PAIR ? mma_f16_ss_pair : mma_f16_ss)(tmem + fx, ah, bl, id1, 1u);
            if (leader_lane) (PAIR ? mma_f16_ss_pair : mma_f16_ss)(tmem + fx, al, bh, id1, 1u);
            if (t.same_s) {
              const uint64_t yh_ = dy_hi + ks * kstep_x, yl_ = dy_lo + ks * kstep_x;
              if (leader_lane) (PAIR ? mma_f16_ss_pair : mma_f16_ss)(tmem + fy, yh_, bh, id1, acc);
              if (leader_lane) (PAIR ? mma_f16_ss_pair : mma_f16_ss)(tmem + fy, yh_, bl, id1, 1u);
              if (leader_lane) (PAIR ? mma_f16_ss_pair : mma_f16_ss)(tmem + fy, yl_, bh, id1, 1u);
            }
            if (leader_lane) (PAIR ? tc_commit_pair : tc_commit)(&bars[slot]);
          }
          if (!t.same_s) {
            for (int ks = 0; ks < t.k2p / 16; ++ks) {
              uint32_t slot;
              const uint32_t sb = take_s(slot);
              const uint32_t s2_half = s_half;
              const uint64_t bh = make_sdesc(sb, lbo_s, 128), bl = make_sdesc(sb + s2_half, lbo_s, 128);
              const uint64_t ah = dy_hi + ks * kstep_x, al = dy_lo + ks * kstep_x;
              const uint32_t acc = ks > 0 ? 1u : 0u;
              if (leader_lane) (PAIR ? mma_f16_ss_pair : mma_f16_ss)(tmem + fy, ah, bh, id1, acc);
              if (leader_lane) (PAIR ? mma_f16_ss_pair : mma_f16_ss)(tmem + fy, ah, bl, id1, 1u);
              if (leader_lane) (PAIR ? mma_f16_ss_pair : mma_f16_ss)(tmem + fy, al, bh, id1, 1u);
              if (leader_lane) (PAIR ? tc_commit_pair : tc_commit)(&bars[slot]);
            }
          }
          if (leader_lane) (PAIR ? tc_commit_pair : tc_commit)(&bars[B_F_FULL]);
          if (c == t.nchunks - 1 && last_of_tile) if (leader_lane) (PAIR ? tc_commit_pair : tc_commit)(&bars[B_XY_FREE]);
          // ---- GEMM 2: Z += P A^T, P (hi/lo fp16) read from TMEM in place of F_x; a new
          // accumulation segment starts a fresh Z once the epilogue has drained the last one
          const bool seg_start = SEG ? (c % t.seg_chunks) == 0 : c == 0;
          if (seg_start && d > 0) {
            const auto t0 = now();
            wait_leader<PAIR>(&bars[B_Z_EMPTY], static_cast<uint32_t>((d - 1) & 1));
            pc[4] += now() - t0;
            tc_fence_after();
          }
          for (int s = 0; s < t.nslices; ++s) {
            {
              const auto t0 = now();
              wait_leader<PAIR>(&bars[B_P_READY + s], static_cast<uint32_t>(j & 1));
              pc[3] += now() - t0;
            }
            const uint32_t p_hi = tmem + fx + 16 * s, p_lo = p_hi + 8;
            for (int pt = 0; pt < t.nparts; ++pt) {
              uint32_t slot;
              const uint32_t sb = take_a(slot);
              const uint64_t bh = make_sdesc(sb, lbo_a, 128), bl = make_sdesc(sb + a_half, lbo_a, 128);
              const uint32_t zd = tmem + pt * t.zp;
              if (leader_lane) (PAIR ? mma_f16_ts_pair : mma_f16_ts)(zd, p_hi, bh, id2, (seg_start && s == 0) ? 0u : 1u);
              if (leader_lane) (PAIR ? mma_f16_ts_pair : mma_f16_ts)(zd, p_hi, bl, id2, 1u);
              if (leader_lane) (PAIR ? mma_f16_ts_pair : mma_f16_ts)(zd, p_lo, bh, id2, 1u);
              if (leader_lane) (PAIR ? tc_commit_pair : tc_commit)(&bars[slot]);
            }
          }
          if (leader_lane) (PAIR ? tc_commit_pair : tc_commit)(&bars[B_G2_DONE]);
          if (SEG ? ((c + 1) % t.seg_chunks == 0 || c + 1 == t.nchunks) : c + 1 == t.nchunks) {
            if (leader_lane) (PAIR ? tc_commit_pair : tc_commit)(&bars[B_Z_FULL]);
            ++d;
          }
        }
        if (last_of_tile) ++v;
      }
      pc[0] = now() - t_start;
      if (PROF && lane == 0) for (int k = 0; k < 8; ++k) g_prof[blockIdx.x * kProfSlots + k] = pc[k];
    }
  } else {
    // ===================================================== workers
    const int q = warp & 3;                // TMEM lane quarter of this warp
    const int h = (warp - 2) >> 2;         // worker half: 0 (warps 2-5) or 1 (warps 6-9)
    const int r = q * 32 + lane;           // tile row == TMEM lane
    const int wt = tid - 64;               // 0..255
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(q * 32) << 16);
    float* stage = reinterpret_cast<float*>(smem + t.off_stage) + (warp - 2) * 32 * kStageStride;
    uint32_t n_raw = 0;
    int64_t j = 0;

    // worker -> MMA-issuer signals: per thread locally, per warp (count 32) to the pair leader
    // warp-aggregated: the warp's threads order their writes with __syncwarp and one lane arrives
    // for all 32 (a per-thread arrive serialises 128-256 mbarrier updates per signal)
    auto signal_leader = [&](uint64_t* bar, bool tmem_only) {
      __syncwarp();
      if (lane == 0) {
        if (PAIR && tmem_only) arrive_leader<PAIR, true>(bar, 32, rank);
        else arrive_leader<PAIR>(bar, 32, rank);
      }
    };
    if (dw.on) {  // fused per-degree weights (weighted GTP): per-column tables, broadcast reads
      for (int k = wt; k < 448; k += kWorkers) {
        if (k < 2 * KH) {
          wtab_x[k] = dw.a[min(degree_of(k), 16)];
          wtab_y[k] = dw.b[min(degree_of(k), 16)];
        }
        wtab_c[k] = dw.c[min(degree_of(k), 32)];
      }
      named_bar_sync(1, kWorkers);
    }
    const float* wx = dw.on ? wtab_x : nullptr;
    const float* wy = dw.on ? wtab_y : nullptr;
    auto convert = [&](int64_t u, int64_t iu) {
      const Unit cu = unit_of(u, t.ngroups);
      const int buf = static_cast<int>(iu & 1);
      const int64_t tile = my_tile(cu.tile);
      const bool tma = tile_tma_ok(rs, tile);
      named_bar_sync(1, kWorkers);  // part_sh / raw of the previous conversion fully consumed
      if (tma) {
        mbar_wait(&bars[B_RAW_FULL], n_raw & 1);
        ++n_raw;
      } else {
        // gather path: the raw region must be free (in-place: previous GEMM 1 retired)
        if (t.raw_inplace && iu > 0) mbar_wait(&bars[B_XY_FREE], static_cast<uint32_t>((iu - 1) & 1));
        const int64_t row0 = tile * BM;
        for (int idx = wt; idx < BM * t.din1; idx += kWorkers) {
          const int rr = idx / t.din1;
          raw_x[idx] = (row0 + rr < rs.rows) ? __ldg(rs.x + row0 * t.din1 + idx) : 0.f;
        }
        for (int idx = wt; idx < BM * t.din2; idx += kWorkers) {
          const int rr = idx / t.din2, kk = idx - rr * t.din2;
          const int64_t g = row0 + rr;
          const int64_t yr = rs.y_shared ? g / rs.channels : g;
          raw_y[idx] = (g < rs.rows) ? __ldg(rs.y + yr * t.din2 + kk) : 0.f;
        }
        named_bar_sync(1, kWorkers);
      }
      const bool wait_free = iu > 0;
      const uint32_t par = static_cast<uint32_t>((iu - 1) & 1);
      if (t.dbg & 4) {
        if (wait_free) mbar_wait(&bars[B_XY_FREE], par);
        if (!t.raw_inplace) mbar_arrive(&bars[B_RAW_FREE]);
      } else if (t.raw_inplace) {
        convert_input_regs<KH>(raw_x, wx, t.din1, t.k1p, t.in_shift, xh, xl, part_sh, ex_sh[buf], r, h, wait_free,
                               &bars[B_XY_FREE], par);
        named_bar_sync(1, kWorkers);
        convert_input_regs<KH>(raw_y, wy, t.din2, t.k2p, t.in_shift, yh, yl, part_sh, ey_sh[buf], r, h, false,
                               &bars[B_XY_FREE], par);
      } else {
        // both inputs are read before the raw buffer is handed back to the producer
        convert_input(raw_x, wx, t.din1, t.k1p, t.in_shift, xh, xl, part_sh, ex_sh[buf], r, h, wait_free,
                      &bars[B_XY_FREE], par);
        named_bar_sync(1, kWorkers);
        convert_input(raw_y, wy, t.din2, t.k2p, t.in_shift, yh, yl, part_sh, ey_sh[buf], r, h, false,
                      &bars[B_XY_FREE], par);
        mbar_arrive(&bars[B_RAW_FREE]);
      }
      fence_proxy_async_smem();
      signal_leader(&bars[B_XY_READY], false);
    };

    int64_t i = 0;  // unit counter
    int64_t v = 0;  // tile sequence number
    int64_t d = 0;  // Z hand-offs received (one per accumulation segment)
    // ---- epilogue of one accumulation segment: Z -> registers -> rescale -> staging -> coalesced
    // row-segment stores; segments after the first add their partial sum to the stored one with
    // fp32 reductions in L2 (round to nearest; only the lane that stored an element adds to it, in
    // program order, so the result is deterministic)
    auto drain = [&](const Unit& cu, int buf, bool add, bool final_seg) {
      { const auto t0 = now(); mbar_wait(&bars[B_Z_FULL], static_cast<uint32_t>(d & 1)); pc[12] += now() - t0; }
      ++d;
      const auto te0 = now();
      tc_fence_after();
      const int e_row = ex_sh[buf][h * BM + r] + ey_sh[buf][h * BM + r] - t.a_shift;
      const int64_t row0 = my_tile(cu.tile) * BM + q * 32;
      const int col0 = cu.g * t.zg;
      const int col_end = min(col0 + t.zg, t.dout_eff);
      const int nblk = t.zg / 16;
      const int half_lane = lane >> 4, cl = lane & 15;
      const float s_lo = pow2i(e_row >> 1), s_hi = pow2i(e_row - (e_row >> 1));  // exact 2^e_row, split for range
      const int64_t stride2 = 2 * static_cast<int64_t>(t.dout_total);
      const int64_t left = rs.rows - row0 - half_lane;  // rows of this half-lane in the quarter
      const bool full = left >= 32;
      const float* sp0 = stage + half_lane * kStageStride + cl;
      float* op0 = rs.out + (row0 + half_lane) * t.dout_total + col0 + cl;
      for (int cb = h; cb < ((t.dbg & 2) ? 0 : nblk); cb += 2) {
        uint32_t v0[16];
        tmem_ld16(lane_base + cb * 16, v0);
        tmem_wait_ld();
#pragma unroll
        for (int qq = 0; qq < 16; ++qq) stage[lane * kStageStride + qq] = __uint_as_float(v0[qq]) * s_lo * s_hi;
        __syncwarp();
        // two rows per store instruction: lanes 0-15 row rr, lanes 16-31 row rr + 1
        if (col0 + cb * 16 + cl < col_end) {
          float* op = op0 + cb * 16;
          const float* sp = sp0;
          const float wc = dw.on ? wtab_c[col0 + cb * 16 + cl] : 1.f;  // fused output weights (weighted GTP)
          if (SEG && add && !(t.dbg & 8)) {  // later segments: fire-and-forget fp32 reductions in L2 (red.global.add, round to nearest)
            for (int rr = 0; rr < (full ? 32 : left); rr += 2, op += stride2, sp += 2 * kStageStride)
              atomicAdd(op, *sp * wc);
          } else if (full) {
#pragma unroll
            for (int rr = 0; rr < 32; rr += 2, op += stride2, sp += 2 * kStageStride) *op = *sp * wc;
          } else {
            for (int rr = 0; rr < left; rr += 2, op += stride2, sp += 2 * kStageStride) *op = *sp * wc;
          }
        }
        __syncwarp();
      }
      tc_fence_before();
      signal_leader(&bars[B_Z_EMPTY], true);
      pc[13] += now() - te0;
      // degrees past the product band are exactly zero (proj/src/gtp.cpp:237-258)
      if (final_seg && cu.g == t.ngroups - 1 && t.dout_total > t.dout_eff && h == 0) {
        for (int rr = 0; rr < 32; ++rr) {
          const int64_t g = row0 + rr;
          if (g >= rs.rows) break;
          for (int col = t.dout_eff + lane; col < t.dout_total; col += 32) rs.out[g * t.dout_total + col] = 0.f;
        }
      }
    };
    { const auto t0 = now(); if (u_begin < u_end) convert(u_begin, 0); pc[11] += now() - t0; }
    for (int64_t u = u_begin; u < u_end; ++u, ++i) {
      const Unit cu = unit_of(u, t.ngroups);
      const bool last_of_tile = (u + 1 == u_end) || unit_of(u + 1, t.ngroups).tile != cu.tile;
      const int buf = static_cast<int>(v & 1);  // ex/ey of this unit's tile
      // ---- pointwise product, chunk by chunk; P overwrites F_x slice by slice
      for (int c = 0; c < t.nchunks; ++c, ++j) {
        { const auto t0 = now(); mbar_wait(&bars[B_F_FULL], static_cast<uint32_t>(j & 1)); pc[9] += now() - t0; }
        tc_fence_after();
        const auto tp0 = now();
        for (int s = h; s < t.nslices; s += 2) {
          if (t.dbg & 1) {
            signal_leader(&bars[B_P_READY + s], true);
            continue;
          }
          uint32_t vx[16], vy[16];
          tmem_ld16(lane_base + fx + 16 * s, vx);
          tmem_ld16(lane_base + fy + 16 * s, vy);
          tmem_wait_ld();
          uint32_t hw[8], lw[8];
#pragma unroll
          for (int qq = 0; qq < 8; ++qq) {
            const float a0 = __uint_as_float(vx[2 * qq]) * __uint_as_float(vy[2 * qq]);
            const float a1 = __uint_as_float(vx[2 * qq + 1]) * __uint_as_float(vy[2 * qq + 1]);
            const __half2 hh = __floats2half2_rn(a0, a1);
            const float2 hf = __half22float2(hh);
            hw[qq] = *reinterpret_cast<const uint32_t*>(&hh);
            lw[qq] = pack_half2(a0 - hf.x, a1 - hf.y);
          }
          tmem_st8(lane_base + fx + 16 * s, hw);
          tmem_st8(lane_base + fx + 16 * s + 8, lw);
          tmem_wait_st();
          tc_fence_before();
          signal_leader(&bars[B_P_READY + s], true);
        }
        pc[10] += now() - tp0;
        // ---- an accumulation segment ends before the unit's last chunk: drain its partial sum
        // (overlaps the next chunk's GEMM 1)
        if (SEG && (c + 1) % t.seg_chunks == 0 && c + 1 < t.nchunks) drain(cu, buf, c + 1 > t.seg_chunks, false);
      }
      // ---- next unit's inputs (overlaps this unit's last GEMM 2)
      if (last_of_tile && u + 1 < u_end) {
        const auto t0 = now();
        convert(u + 1, v + 1);
        pc[11] += now() - t0;
      }
      drain(cu, buf, SEG && t.nchunks > t.seg_chunks, true);
      if (last_of_tile) ++v;
    }
    pc[8] = now() - t_start;
    if (PROF && warp == 2 && lane == 0)
      for (int k = 8; k < kProfSlots; ++k) g_prof[blockIdx.x * kProfSlots + k] = pc[k];
  }
  tc_fence_before();
  if (PAIR) cluster_sync_all();
  else __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    if (PAIR) tmem_dealloc_pair(tmem, 512);
    else tmem_dealloc(tmem, 512);
  }
}

}  // namespace

int gtp_grid_tc_max_smem(bool big_k) {
  cudaFuncAttributes a{};
  if (cudaFuncGetAttributes(&a, big_k ? gtp_grid_tc_kernel<false, false, kKHalfMax> : gtp_grid_tc_kernel<false, true>) !=
      cudaSuccess)
    return 0;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) return 0;
  return optin - static_cast<int>(a.sharedSizeBytes) - 1024;  // slack for the 1 KB dynamic alignment
}

cudaError_t launch_gtp_grid_tc(const GridTcTables& t, const RowSpec& rs, int num_sms, cudaStream_t s,
                               const DegreeWeights* w) {
  DegreeWeights dw{};
  if (w) dw = *w;
  if (rs.rows <= 0) return cudaSuccess;
  static const bool prof_env = [] {
    const char* v = std::getenv("TPO_GRID_PROF");
    return v && *v == '1';
  }();
  const bool prof = prof_env && t.seg_chunks >= t.nchunks;
  // K > 128 (L = 11, 12): a separate instantiation with the wider register conversion, so the
  // default one keeps its register budget (the wide one spills ~100 B in cold code)
  const bool big = t.k1p > 2 * kKHalfStd || t.k2p > 2 * kKHalfStd;
  if (big && t.pair) return cudaErrorInvalidValue;  // planner never pairs K > 128
  const bool seg = t.seg_chunks < t.nchunks;
  if (seg && t.pair) return cudaErrorInvalidValue;  // the planner never pairs segmented shapes
  auto kern = big ? (seg ? gtp_grid_tc_kernel<false, false, kKHalfMax, true> : gtp_grid_tc_kernel<false, false, kKHalfMax>)
              : seg ? gtp_grid_tc_kernel<false, false, kKHalfStd, true>  // (no cycle accounting variant)
              : t.pair ? (prof ? gtp_grid_tc_kernel<true, true> : gtp_grid_tc_kernel<false, true>)
                       : (prof ? gtp_grid_tc_kernel<true, false> : gtp_grid_tc_kernel<false, false>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, t.smem_bytes);
  if (e != cudaSuccess) return e;
  const int kp = t.pair ? 2 : 1;
  const int64_t units = ((rs.rows + BM * kp - 1) / (BM * kp)) * t.ngroups;
  const int grid = kp * static_cast<int>(std::min<int64_t>(units, num_sms / kp));
  unsigned long long* buf = nullptr;
  if (prof) {
    cudaMalloc(&buf, sizeof(unsigned long long) * kProfSlots * grid);
    cudaMemset(buf, 0, sizeof(unsigned long long) * kProfSlots * grid);
    cudaMemcpyToSymbol(g_prof, &buf, sizeof(buf));
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = t.smem_bytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kp;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, t, rs, dw);
  if (prof && e == cudaSuccess) {
    std::vector<unsigned long long> h(kProfSlots * grid);
    cudaStreamSynchronize(s);
    cudaMemcpy(h.data(), buf, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    // MMA slots averaged over the MMA-issuing CTAs (pair leaders), worker slots over all
    double avg[kProfSlots] = {};
    int n_mma = 0;
    for (int b = 0; b < grid; ++b) n_mma += h[b * kProfSlots] != 0;
    for (int b = 0; b < grid; ++b)
      for (int k = 0; k < kProfSlots; ++k)
        avg[k] += static_cast<double>(h[b * kProfSlots + k]) / (k < 8 ? std::max(n_mma, 1) : grid);
    std::fprintf(stderr,
                 "[tpo-prof] units=%lld grid=%d MMA: total %.0f xy_ready %.0f s_ring %.0f p_ready %.0f z_empty %.0f "
                 "g2_done %.0f a_ring %.0f | worker: total %.0f f_full %.0f product %.0f convert %.0f z_full %.0f epilogue %.0f\n",
                 static_cast<long long>(units), grid, avg[0], avg[1], avg[2], avg[3], avg[4], avg[5], avg[6], avg[8], avg[9],
                 avg[10], avg[11], avg[12], avg[13]);
    cudaFree(buf);
  }
  return e;
}

}  // namespace tpo_b200
