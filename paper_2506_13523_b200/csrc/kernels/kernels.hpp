// Device-table descriptors and launchers for the four TPO kernels.
// Tables are built on the host (host/context.cpp) and live in device memory
// owned by the tpo_ctx; launchers are asynchronous on the given stream.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace tpo_b200 {

// Row indexing shared by all kernels: row r in [0, rows) is (b, c) with
// rows = batch * channels; x row = r, y row = y_shared ? r / channels : r.
struct RowSpec {
  const float* x;
  const float* y;
  float* out;
  int64_t rows;
  int64_t channels;
  int y_shared;
};

// ---------------------------------------------------------------- 3xFP16 scaling
// Exact power-of-two scales that keep the fp16 hi / lo parts of every GEMM operand well inside
// fp16's normal range (its subnormals carry only absolute precision 2^-24, which was the
// dominant error for small rows when values sat near 1):
//   kInShift   input rows are scaled so that max|x| < 2^kInShift (CGTP blocks, edge kernel) or
//              ||x||_2 < 2^kInShift (MTP, whose carrier matrices are isometric in x), so products
//              of two scaled values stay below 2^14;
//   kTabShift  constant operator tables with entries <= 1 (real CG blocks, MTP extract) are
//              stored times 2^kTabShift; the epilogue divides both back out exactly.
constexpr int kInShift = 7;
constexpr int kTabShift = 11;

// ---------------------------------------------------------------- CGTP
// Output coefficient o is owned by thread o % kCgtpChunk of output pass
// o / kCgtpChunk.  Terms {i1 | i2 << 16, coef bits} are stored term-major per
// warp (32 outputs), padded to that warp's longest list:
//   term t of output o: terms[warp_off[o / 32] + t * 32 + o % 32], t < warp_nt[o / 32].
constexpr int kCgtpChunk = 256;
struct CgtpTables {
  int din1, din2, dout, nchunks;
  const uint2* terms;
  const int* warp_off;  // [nchunks * kCgtpChunk / 32]
  const int* warp_nt;   // [nchunks * kCgtpChunk / 32]
};
cudaError_t launch_cgtp(const CgtpTables& t, const RowSpec& rs, int num_sms, cudaStream_t s);

// CGTP backward (cgtp_bwd.cu): grad[a] = sum_t c_t g[o_t] v[i_t] over the
// transposed term lists (a = coefficient of the input the gradient is for,
// v = the other input, g = grad_out).  A block owns 32 rows and sweeps grad_out
// in windows of dwin columns staged in shared memory, accumulating in
// registers; the term list of output a is dealt over nsplit virtual outputs
// p * dres + a (nsplit * dres <= kCgtpChunk) reduced through shared memory.
//   term t of virtual output v, window w: terms[warp_off[(q * nwin + w) * 8 + (v % 256) / 32] + t * 32 + v % 32],
//   q = v / 256, t < warp_nt[same index]; term.x = (o - w * dwin) | i << 16.
struct CgtpBwdTables {
  int dwin, nwin, dother, dres, nsplit, nchunks;
  int64_t g_stride;  // grad_out row length (forward Dout)
  const uint2* terms;
  const int* warp_off;
  const int* warp_nt;
};
cudaError_t launch_cgtp_bwd(const CgtpBwdTables& t, const RowSpec& rs, int num_sms, cudaStream_t s);

// Shared-y CGTP (one y per edge, channels a multiple of 128) as per-edge dense
// GEMMs on tcgen05: out[c] = x[c] . M_y (cgtp_edge_tc.cu).  tm_out: 2-D TMA
// view of out [rows][dout] fp32, box 32 x 128, 128B swizzle (built per call).
struct EdgeTcParams {
  int kp;        // Din1 padded to 16 (<= 64)
  int dout_pad;  // Dout padded to 16 (<= 256: two TMEM accumulators)
  int tmem_cols;
  // optional per-path weights (MACE "uvu"): output o of edge e is scaled by
  // path_w[e * w_stride + path_of_out[o]] (w_stride 0: one weight vector for every edge); folded
  // into the edge's M_y columns, so the weighted product costs nothing extra
  const float* path_w;
  int64_t w_stride;
  const int* path_of_out;
  alignas(64) CUtensorMap tm_out;
};
int cgtp_edge_tc_smem(const CgtpTables& t, int kp, int dout_pad);
cudaError_t launch_cgtp_edge_tc(const CgtpTables& t, const EdgeTcParams& p, const RowSpec& rs, int num_sms,
                                cudaStream_t s);

// General CGTP on tcgen05 (cgtp_tc.cu): per (l1, l2) block one dense GEMM
// out_block = (x_{l1} (x) y_{l2}) . W^T with the square real-CG block W.  A unit is
// (block, N part of <= 256 outputs); consecutive units share one accumulator
// ("super-unit", <= 256 columns, one hand-off to the epilogue); w holds per unit and K-step
// [hi | lo][n_pad rows (block outputs)][16 (k = m1 (2 l2 + 1) + m2)] canonical.
struct CgtpTcUnit {
  int l1, l2, out_off, n_valid, n_pad, ksteps, w_off;
  int dcol_last;  // column inside the 256-column accumulator | (last unit of its super-unit) << 16
};
// TMEM plan of the CGTP block kernel: two accumulators of kCgtpDCols columns and an fp16 hi/lo P ring
// of kCgtpAStages stages x 2 K-steps (32 columns each) -- 2 * kCgtpDCols + 32 * kCgtpAStages = 512
#ifndef TPO_CGTP_DCOLS
#define TPO_CGTP_DCOLS 192
#endif
constexpr int kCgtpDCols = TPO_CGTP_DCOLS;
constexpr int kCgtpAStages = (512 - 2 * kCgtpDCols) / 32;
struct CgtpTcTables {
  int din1, din2, dout, nunits;
  int a_stages, b_stages, b_stage_bytes, smem_bytes;
  int off_a, off_b, off_xy, xy_pitch;  // xy: per-row staging [128][xy_pitch], x row | y row
  int yseg;  // 1: y staged per block ([3][128][41] after xy) instead of the whole row (large din2)
  const CgtpTcUnit* units;
  const uint8_t* w;
};
cudaError_t launch_cgtp_tc(const CgtpTcTables& t, const RowSpec& rs, int num_sms, cudaStream_t s);

// CGTP backward on tcgen05 (cgtp_bwd_tc.cu): per (l1, l2) block Q = W^T g_block as a dense GEMM
// (A = grad_out block, K = block outputs o; N = k = (m1 + l1)(2 l2 + 1) + m2 + l2), contracted with
// y / x in the epilogue.  A unit is one block (n <= 169 columns: L <= 6, a single N part); w holds per unit and K-step
// [hi | lo][n_pad rows (k)][16 (o)] canonical, times 2^kTabShift.
struct CgtpBwdTcUnit {
  int l1, l2, blk, g_off, n, k0, n_valid, n_pad, ksteps, w_off;
  int dcol_last;  // as CgtpTcUnit
  int m1b, nrows;  // the part's rows m1 of Q: [m1b, m1b + nrows) (k0 = m1b n2, n_valid = nrows n2)
};
struct CgtpBwdTcTables {
  int din1, din2, dout, nunits, nblocks, nbp;  // nbp: nblocks rounded up to 4 (exponent rows)
  int b_stages, b_stage_bytes, g_slots, smem_bytes, off_b, off_xy, off_g;
  int one_sided;  // 1 (L = 8): the row accumulator holds one gradient, one launch per gradient
  const CgtpBwdTcUnit* units;
  const uint8_t* w;
  alignas(64) CUtensorMap tm_g;  // set per call by the launcher
};
int cgtp_bwd_tc_smem(const CgtpBwdTcTables& t, int b_stages, int g_slots);
// tm_g: grad_out viewed as [rows / 4][4 Dout] fp32 (rows a multiple of 4), box 36 x 32, no swizzle
cudaError_t launch_cgtp_bwd_tc(const CgtpBwdTcTables& t, const float* x, const float* y, const float* g,
                               const CUtensorMap& tm_g, float* gx, float* gy, int64_t rows, int num_sms,
                               cudaStream_t s);

// Grid / Fourier GTP at small degree on SIMT (gtp_small.cu): the dense operators of the tcgen05
// kernel (out = A ((S x) .* (S y)), L1 = L2, same S) as fp32 host arrays, copied into the kernel's
// parameter space per launch.  Shapes: gtp_small_supported.
struct GtpSmallOps {
  int din = 0, G = 0, dout_eff = 0, dout_total = 0;
  const float* s = nullptr;  // host [G][din]
  const float* a = nullptr;  // host [dout_eff][G]
};
bool gtp_small_supported(int din, int G, int dout);
cudaError_t launch_gtp_small(const GtpSmallOps& o, const RowSpec& rs, int num_sms, cudaStream_t s);

// ---------------------------------------------------------------- GTP grid, tcgen05
// Dense operators of the reference's product grid, pre-split into fp16 hi/lo
// and pre-tiled on the host in the UMMA canonical K-major layout, one
// contiguous block per MMA K-step ("slice") so that every ring stage of the
// kernel is a single 1D TMA bulk copy:
//   s1[c][ks] : [hi | lo] x [nc rows (grid points of chunk c)][16 (K = (l,m) 16ks..)]
//   a[g][c][s][p]: [hi | lo] x [zp rows (outputs p*zp.. of group g)][16 (K = grid points 16s..)]
// Work unit = (128-row tile, output group g); the grid is swept in chunks of
// nc points (N of GEMM 1, K of GEMM 2).
struct GridTcTables {
  int din1, din2, k1p, k2p;  // input dims, K padded to 16
  int nc, nchunks, nslices;  // grid points per chunk (multiple of 16), chunks, nc / 16
  int ngroups, zg;           // output groups, outputs per group (padded to 16, <= 256)
  int nparts, zp;            // GEMM 2 N-split: zg = nparts * zp, zp <= 128 (keeps ring stages small)
  int dout_eff;              // outputs computed (degrees <= min(L3, band))
  int dout_total;            // (L3+1)^2 written (zeros past the band)
  int a_shift;               // device A = A * 2^a_shift (max |A| in [2^12, 2^13))
  int in_shift;              // input rows scaled to ||x||_2 < 2^in_shift: the largest scale keeping every
                             // P = F_x F_y below 2^14 (|F(g)| <= ||x|| ||S row g||), so the fp16 hi / lo
                             // parts of inputs and products stay clear of fp16's subnormal range
  int same_s;                // s2 == s1 (L1 == L2)
  int s_stages, a_stages;    // B-operand rings (S table -> GEMM 1, A table -> GEMM 2), one producer warp each
  uint32_t s_stage_bytes, a_stage_bytes;
  int raw_inplace;           // raw input tiles land in the X/Y operand buffers
  int safe_war;              // wait for GEMM 2 of chunk c before GEMM 1 of chunk c+1
  int seg_chunks;            // GEMM-2 accumulation segment (chunks): the tensor pipe's fp32 accumulation
                             // truncates (round toward zero) once per MMA, so the error grows with the
                             // number of MMAs into one accumulator; each segment starts a fresh Z and its
                             // partial sum is added in fp32 (round to nearest) into the output row
  int pair;                  // CTA pairs, tcgen05 cta_group::2 (M = 256); slices stored as two row halves
  int dbg;                   // timing experiments only (results invalid): 1 no product, 2 no epilogue, 4 no convert,
                             // 8 plain stores instead of reductions for segment sums
  int smem_bytes;
  uint32_t off_x, off_y, off_raw, off_sring, off_aring, off_stage;  // dynamic shared-memory carve-up
  const uint8_t* s1;
  const uint8_t* s2;
  const uint8_t* a;
  uint32_t s1_slice_bytes, s2_slice_bytes, a_slice_bytes;
  // pair mode: 2-D TMA views [bytes / 64][64 B] of the tables, box = one half slice
  alignas(64) CUtensorMap tm_s1;
  alignas(64) CUtensorMap tm_s2;
  alignas(64) CUtensorMap tm_a;
};
// Per-degree weights fused into the grid kernel (weighted GTP, proj/src/gtp.cpp:206-215):
// x[l,m] *= a[l], y[l,m] *= b[l] in the input conversion, out[l,m] *= c[l] in the epilogue.
struct DegreeWeights {
  int on;
  float a[17], b[17], c[33];
};
cudaError_t launch_gtp_grid_tc(const GridTcTables& t, const RowSpec& rs, int num_sms, cudaStream_t s,
                               const DegreeWeights* w = nullptr);
int gtp_grid_tc_max_smem(bool big_k = false);  // big_k: the K > 128 instantiation

// ---------------------------------------------------------------- GTP grid, SIMT separable
struct GridSimtTables {
  int L1, L2, band, L3e, dout_total;  // L3e = min(L3, band)
  int nt, np;
  const float* lam;   // [(band+1)(band+2)/2][nt]
  const float* cs;    // [2*band+1][np]
  const float* wq;    // [nt] = w_j * 2pi/np
  float out_scale;    // 1
  // symmetric (row-quad) kernel: phi_{np-k} = 2pi - phi_k and theta_{nt-1-j} = pi - theta_j fold
  // both transforms in half; tables over the half-period kp = 0..band
  int nkp, nkpp, mpad;    // band + 1, nkp rounded up to 4, (band + 1) rounded up to 4
  const float* c2c;       // [band + 1][nkpp]  cos(m phi_kp)     (phi synthesis, m >= 0)
  const float* c2s;       // [band + 1][nkpp]  sin(m phi_kp)     (phi synthesis, m < 0)
  const float* c4c;       // [nkp][mpad]       cos(m phi_kp)     (phi analysis, m >= 0)
  const float* c4s;       // [nkp][mpad]       sin((m+1) phi_kp) (phi analysis, m < 0)
  const int* items5;      // Legendre analysis items: l0 | (m + L3e) << 16, l1 = l0 + 2 of the same parity
  int nitems5;
  // theta tables of the row-quad kernel by (l, |m|) (row l (l + 1) / 2 + |m|): synthesis values at
  // the nodes (l <= max(L1, L2)) and analysis weights (l <= L3e).  Grid: Lambda_l|m|(theta_j) for
  // both (w_j in wq); Fourier: the reference torus's encode / decode spectra summed at the torus rows
  // (Context::fourier_sep).  By |m|: signed-order tables did not fit in L1 beside the shared memory
  // at L = 13..15 (+15-20%).
  const float* lam5t;  // [njp][nitems5] float2: lam5 of an item's two degrees, node-pair-major
  const float* lam1q;  // [l (l + 1) / 2 + |m|][njp4]: lam1 on the first-half nodes, rows of 4-node quads
  int njp4;
};
cudaError_t launch_gtp_grid_simt(const GridSimtTables& t, const RowSpec& rs, int num_sms, cudaStream_t s);
bool gtp_grid_quad_fits(const GridSimtTables& t);  // the row-quad kernel's shared memory fits

// ---------------------------------------------------------------- GTP Fourier
// Encode gather lists per spectrum mode (u,v) of the (2L+1)^2 input spectra,
// direct 2D convolution on the Hermitian half-plane of the (4L+1)^2 product
// spectrum, decode gather lists per output coefficient.
struct FourierDevTables {
  int L, L1, L2, L3, dout_total, dout_eff;
  int nenc1, nenc2;        // entries in the encode lists for x / y
  const int* enc1_off;     // [(2L+1)^2 + 1] CSR over modes, entries (input idx, w)
  const int* enc1_idx;
  const float2* enc1_w;
  const int* enc2_off;
  const int* enc2_idx;
  const float2* enc2_w;
  const int* dec_off;      // [dout_eff + 1] CSR, entries (half-plane mode idx, w, conj flag in idx sign)
  const int* dec_idx;
  const float2* dec_w;
  int nhalf;               // number of half-plane product modes
  const int2* half_uv;     // [nhalf] (U, V)
};
cudaError_t launch_gtp_fourier(const FourierDevTables& t, const RowSpec& rs, int num_sms, cudaStream_t s);

// ---------------------------------------------------------------- MTP
struct MtpDevTables {
  int lt, dt, din1, din2, dout_total, dout_eff;
  int dtp;  // dt rounded up to 4: the kernel's padded carrier pitch
  // Term lists {index, coef bits} stored warp-interleaved: item i (handled by lane i % 32) has
  // idx[i] = {first, count} and its e-th term at first + 32 e, so a warp's term loads are coalesced.
  // embed items: the dt*dt cells of X (index = x coefficient), then those of Y (index = y coefficient)
  const int2* emb_idx;  // [2 dt*dt]
  const uint2* emb;
  // extract items: (output coefficient o < dout_eff, product half g) = 2 o + g (index = padded cell
  // a * dtp + b)
  const int2* ext_idx;  // [2 dout_eff]
  const uint2* ext;
};
cudaError_t launch_mtp(const MtpDevTables& t, const RowSpec& rs, int num_sms, cudaStream_t s);

// MTP on tcgen05 (mtp_tc.cu), carrier dt = 2 lt + 1 <= 13.  Embed and extract
// are dense 3xFP16 GEMMs whose B operands are streamed per K-step through a
// TMA ring; the dt x dt per-product matmul runs on SIMT straight from TMEM.
// TMEM columns (512 per CTA): X^T at [0, n1) (X[i][k] at k*dt + i), Y at
// [n1, 2 n1) (Y[k][j] at k*dt + j), Z of carrier rows i < i1 = (dt+1)/2 (group 0)
// and i >= i1 (group 1, its tail in group 2 = the Y columns once read) as fp16
// hi/lo K-steps, cells (i - i0) * dt + j, K order g = 0..3; GEMM-2 output at [0, n2).
//   e1[ks] / e2[ks]: [hi | lo] x [n1 rows (X / Y position)][16 (input idx 16ks..)] canonical
//   ext[ks]        : [hi | lo] x [n2 rows (output)][16 (Z position 16ks..)] canonical
struct MtpTcTables {
  int dt, n1, n2, k1, k2, kz;  // padded GEMM dims
  int din1, din2, dout_eff, dout_total;
  int zgrp_col[4], zgrp_size[4];  // Z groups in K order: TMEM column, K extent
  int y0_reuse;                   // group 2 lives in the Y columns (row halves sync before writing it)
  int stages, stage_bytes, smem_bytes;
  int off_xop, off_yop, off_stx, off_sty, off_out;  // dynamic shared memory layout
  const uint8_t* e1;
  const uint8_t* e2;
  const uint8_t* ext;
};
cudaError_t launch_mtp_tc(const MtpTcTables& t, const RowSpec& rs, int num_sms, cudaStream_t s);

// ---------------------------------------------------------------- weighted epilogue helpers
// x[r][(l,m)] *= w[l] (per-degree scaling, proj/src/gtp.cpp:34-44)
cudaError_t launch_scale_degrees(const float* in, float* out, int64_t rows, int L, const float* w,
                                 cudaStream_t s);
// out[i] += in[i], i < n (backward partial sums)
cudaError_t launch_accumulate(const float* in, float* out, int64_t n, cudaStream_t s);
// dst[r][k] = src[r * stride + col0 + k], k < w (backward: a window of grad_out columns, packed)
cudaError_t launch_gather_cols(const float* src, int64_t stride, int col0, int w, float* dst, int64_t rows,
                               cudaStream_t s);

// ---------------------------------------------------------------- per-path weights (stages.cu)
// out[row][o] *= w[(row / channels) * w_stride + path_of_out[o]]
cudaError_t launch_path_scale(float* out, int64_t rows, int64_t channels, int dout, const int* path_of_out,
                              const float* w, int64_t w_stride, int num_sms, cudaStream_t s);

// ---------------------------------------------------------------- stage operators (stages.cu)
// out[b][o] = sum_k mt[k][o] in[b][k]  (mt k-major [din][dout], fp32)
cudaError_t launch_dense_map(const float* in, int din, const float* mt, int dout, float* out, int64_t rows,
                             cudaStream_t s);
// Z[b] = X[b] Y[b], dt x dt row-major carriers
cudaError_t launch_carrier_matmul(const float* X, const float* Y, float* Z, int dt, int64_t batch, cudaStream_t s);
cudaError_t launch_pointwise_mul(const float* a, const float* b, float* out, int64_t n, int num_sms, cudaStream_t s);
// Wigner-D recursion tables: level l's entries of cg_real(1, l-1, l) grouped by m3, with m1 as an index
// into D^1 (m1 + 1) and m2 into D^{l-1} (m2 + l - 1)
struct WignerEntry {
  int m1, m2;
  double v;
};
constexpr int kWignerMaxL = 64;
struct WignerTables {
  int L;
  int64_t d_stride;                    // sum_{l <= L} (2l+1)^2 doubles per rotation
  int64_t block_off[kWignerMaxL + 1];  // offset of D^l in a rotation's blocks
  int l_off[kWignerMaxL + 1];          // level l's row offsets start at row_off[l_off[l]]
  int e_off[kWignerMaxL + 1];          // level l's entries start at entries[e_off[l]]
  const int* row_off;
  const WignerEntry* entries;
  const int64_t* block_off_dev;
};
cudaError_t launch_wigner_d(const WignerTables& w, const double* R, double* D, int64_t n, cudaStream_t s);
cudaError_t launch_rotate(const WignerTables& w, const double* D, int64_t n_rot, const float* x, float* out,
                          int64_t batch, int64_t channels, int num_sms, cudaStream_t s);

}  // namespace tpo_b200
