// Grid / Fourier GTP at L1 = L2 = 1, L3 = 2 on SIMT (one lane per product).
//
// Both GTPs are out = A ((S x) .* (S y)) with small dense operators (proj/src/gtp.cpp:228-260 for the
// product grid, :290-301 for the torus convolution, as Context::grid_tc / fourier_tc build them); at
// L = 1 they hold <= 234 coefficients, so they travel as a __grid_constant__ kernel parameter and
// every multiply-add takes its coefficient straight from the constant bank (warp-uniform), fully
// unrolled over the compile-time shape: G (2 Din + 1 + Dout) FFMAs per product and no tile pipeline,
// which is what the 128-row tcgen05 kernel costs at these sizes (its prologue and per-tile chain
// dominate: ~20 us per 65,536 products at L = 1 for 4.5 MB of traffic).  A block owns 32 products
// (one per lane); its four warps split the points and their partial outputs are summed in shared
// memory, which gives four times the warps of a thread-per-product mapping.  fp32 throughout.
#include <algorithm>

#include "kernels.hpp"

namespace tpo_b200 {

namespace {

constexpr int kRows = 32;   // products per block (one per lane)
constexpr int kSplit = 4;   // warps per block: each sums a quarter of the points for the 32 products

template <int DIN, int G, int DOUT>
struct SmallOps {
  float s[G * DIN];   // S[g][k]
  float a[DOUT * G];  // A[o][g]
};

// acc[o] += sum_{g in [G0, G1)} A[o][g] (S[g] . x) (S[g] . y); coefficients warp-uniform
template <int DIN, int G, int DOUT, int G0, int G1>
__device__ __forceinline__ void accumulate_points(const SmallOps<DIN, G, DOUT>& op, const float (&x)[DIN],
                                                  const float (&y)[DIN], float (&acc)[DOUT]) {
#pragma unroll
  for (int g = G0; g < G1; ++g) {
    float fx = 0.f, fy = 0.f;
#pragma unroll
    for (int k = 0; k < DIN; ++k) {
      fx = fmaf(op.s[g * DIN + k], x[k], fx);
      fy = fmaf(op.s[g * DIN + k], y[k], fy);
    }
    const float p = fx * fy;
#pragma unroll
    for (int o = 0; o < DOUT; ++o) acc[o] = fmaf(op.a[o * G + g], p, acc[o]);
  }
}

template <int DIN, int G, int DOUT>
__global__ void __launch_bounds__(kRows * kSplit) gtp_small_kernel(const __grid_constant__ SmallOps<DIN, G, DOUT> op,
                                                                   const __grid_constant__ RowSpec rs, int dout_total) {
  constexpr int PI = DIN | 1;   // odd row pitches: per-lane rows are bank-conflict free
  constexpr int PO = DOUT | 1;
  __shared__ float xs[kRows * PI], ys[kRows * PI], part[kSplit][kRows * PO];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int64_t ntiles = (rs.rows + kRows - 1) / kRows;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row0 = tile * kRows;
    const int nr = static_cast<int>(rs.rows - row0 < kRows ? rs.rows - row0 : kRows);
    __syncthreads();  // the previous tile's partial sums were read
    for (int i = t; i < nr * DIN; i += kRows * kSplit) {  // coalesced staging
      const int r = i / DIN, k = i - r * DIN;
      xs[r * PI + k] = __ldg(rs.x + row0 * DIN + i);
      const int64_t yr = rs.y_shared ? (row0 + r) / rs.channels : row0 + r;
      ys[r * PI + k] = __ldg(rs.y + yr * DIN + k);
    }
    __syncthreads();
    {
      float x[DIN], y[DIN], acc[DOUT];
#pragma unroll
      for (int k = 0; k < DIN; ++k) {
        x[k] = xs[lane * PI + k];
        y[k] = ys[lane * PI + k];
      }
#pragma unroll
      for (int o = 0; o < DOUT; ++o) acc[o] = 0.f;
      constexpr int Q = (G + kSplit - 1) / kSplit;
      switch (w) {  // warp-uniform: warp w sums points [w Q, (w + 1) Q)
        case 0: accumulate_points<DIN, G, DOUT, 0, Q>(op, x, y, acc); break;
        case 1: accumulate_points<DIN, G, DOUT, Q, 2 * Q>(op, x, y, acc); break;
        case 2: accumulate_points<DIN, G, DOUT, 2 * Q, 3 * Q>(op, x, y, acc); break;
        default: accumulate_points<DIN, G, DOUT, 3 * Q, G>(op, x, y, acc); break;
      }
#pragma unroll
      for (int o = 0; o < DOUT; ++o) part[w][lane * PO + o] = acc[o];
    }
    __syncthreads();
    for (int i = t; i < nr * dout_total; i += kRows * kSplit) {  // coalesced; degrees past the band are zero
      const int r = i / dout_total, o = i - r * dout_total;
      float v = 0.f;
      if (o < DOUT) {
#pragma unroll
        for (int q = 0; q < kSplit; ++q) v += part[q][r * PO + o];
      }
      rs.out[row0 * dout_total + i] = v;
    }
  }
}

template <int DIN, int G, int DOUT>
cudaError_t launch_t(const float* s, const float* a, const RowSpec& rs, int dout_total, int num_sms, cudaStream_t st) {
  static_assert(sizeof(SmallOps<DIN, G, DOUT>) <= 32000, "operators must fit the kernel parameter space");
  SmallOps<DIN, G, DOUT> op;
  std::copy(s, s + G * DIN, op.s);
  std::copy(a, a + DOUT * G, op.a);
  const int64_t ntiles = (rs.rows + kRows - 1) / kRows;
  const int grid = static_cast<int>(std::min<int64_t>(ntiles, 16 * static_cast<int64_t>(num_sms)));
  gtp_small_kernel<DIN, G, DOUT><<<grid, kRows * kSplit, 0, st>>>(op, rs, dout_total);
  return cudaGetLastError();
}

}  // namespace

// L = 1 only: at L = 2 / 3 the fully unrolled kernels (2.5 k / 7.5 k FFMAs per product) thrash the
// instruction cache and lose to the tcgen05 kernel (profiles/r02/grid_small.txt)
bool gtp_small_supported(int din, int G, int dout) { return din == 4 && dout == 9 && (G == 15 || G == 18); }

cudaError_t launch_gtp_small(const GtpSmallOps& o, const RowSpec& rs, int num_sms, cudaStream_t s) {
  if (rs.rows <= 0) return cudaSuccess;
#define TPO_SMALL(D_, G_, O_) \
  if (o.din == D_ && o.G == G_ && o.dout_eff == O_) return launch_t<D_, G_, O_>(o.s, o.a, rs, o.dout_total, num_sms, s);
  TPO_SMALL(4, 15, 9)
  TPO_SMALL(4, 18, 9)
#undef TPO_SMALL
  return cudaErrorInvalidValue;
}

}  // namespace tpo_b200
