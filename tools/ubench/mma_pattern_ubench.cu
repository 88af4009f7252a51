// The grid kernel's MMA pattern without any synchronisation: per "chunk"
// GEMM 1 = 8 K-steps x (3 SS MMAs into F_x + 3 into F_y), N = NC, then
// GEMM 2 = NC/16 K-steps x 3 TS MMAs (A = P from TMEM) into Z, N = 224.
// VAR 0: P lives inside F_x (as in the kernel: WAR between G2 and next G1)
// VAR 1: P in a separate TMEM region (no overlap with F)
// VAR 2: only GEMM 1; VAR 3: only GEMM 2
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2506_13523_b200/csrc/kernels/sm100.cuh"
using namespace tpo_b200::sm100;

template <int NC, int VAR, int TMA>
__global__ void __launch_bounds__(128, 1) k(int reps, long long* out, const uint8_t* tab) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t tbar[4];
  __shared__ __align__(8) uint64_t dbar[3];
  __shared__ volatile int done;
  __shared__ uint32_t tm;
  const int tid = threadIdx.x;
  for (int i = tid; i < 224 * 1024 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (tid == 0) { mbar_init(&bar, 1); for (int i = 0; i < 4; ++i) mbar_init(&tbar[i], 1); for (int i = 0; i < 3; ++i) mbar_init(&dbar[i], 1); done = 0; fence_mbar_init(); }
  fence_proxy_async_smem();
  if (tid < 32) { tmem_alloc(&tm, 512); tmem_relinquish(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t t = tm;
  if (tid == 0) {
    const uint32_t xa = smem_u32(smem), sb = smem_u32(smem + 128 * 1024), ab = smem_u32(smem + 160 * 1024);
    constexpr uint32_t id1 = idesc_f16(128, NC), id2 = idesc_f16(128, 224);
    constexpr uint32_t lbo_x = 16 * 128, lbo_s = (NC / 8) * 128, lbo_a = (224 / 8) * 128;
    const uint64_t dx = make_sdesc(xa, lbo_x, 128), ds = make_sdesc(sb, lbo_s, 128), da = make_sdesc(ab, lbo_a, 128);
    constexpr uint32_t zc = 224, fx = zc, fy = zc + NC;
    constexpr uint32_t pbase = VAR == 1 ? 512 - NC : fx;  // P region
    long long c0 = clock64();
    int n = 0;
    uint32_t ph[3] = {0, 0, 0};
    auto g1 = [&](uint32_t fxo, uint32_t fyo) {
#pragma unroll 1
      for (int ks = 0; ks < 8; ++ks) {
        const uint64_t xh = dx + ((ks * 2 * lbo_x) >> 4);
        const uint64_t xl = xh + (32768u >> 4), yh = xh + (65536u >> 4), yl = xh + (98304u >> 4);
        const uint64_t bh = ds + (((ks & 3) * 2 * lbo_s) >> 4), bl = bh + ((NC * 32u) >> 4);
        mma_f16_ss(t + fxo, xh, bh, id1, ks > 0); mma_f16_ss(t + fxo, xh, bl, id1, 1); mma_f16_ss(t + fxo, xl, bh, id1, 1);
        mma_f16_ss(t + fyo, yh, bh, id1, ks > 0); mma_f16_ss(t + fyo, yh, bl, id1, 1); mma_f16_ss(t + fyo, yl, bh, id1, 1);
        n += 6;
      }
    };
    auto g2 = [&](uint32_t pb) {
#pragma unroll 1
      for (int s = 0; s < NC / 16; ++s) {
        const uint32_t p = t + pb + 16 * s;
        mma_f16_ts(t, p, da, id2, 1); mma_f16_ts(t, p, da, id2, 1); mma_f16_ts(t, p + 8, da, id2, 1);
        n += 3;
      }
    };
    auto drain = [&](int b) { tc_commit(&dbar[b]); mbar_wait(&dbar[b], ph[b]); ph[b] ^= 1; };
    if (VAR == 5) {
      for (int r = 0; r < reps; ++r) { g1(fx, fy); drain(0); g2(fx); drain(1); }
    } else if (VAR == 6) {  // two F buffers (nc <= 64 so they fit next to Z = 224 columns)
      const uint32_t f0 = 224, f1 = 224 + 2 * NC;
      g1(f0, f0 + NC);
      for (int r = 0; r < reps; ++r) {
        const uint32_t cur = (r & 1) ? f1 : f0, nxt = (r & 1) ? f0 : f1;
        tc_commit(&dbar[r & 1]);                     // G1(r) done -> "products" may start
        g1(nxt, nxt + NC);                           // G1(r + 1) queued behind
        mbar_wait(&dbar[r & 1], ph[r & 1]); ph[r & 1] ^= 1;  // products(r) done (immediate)
        g2(cur);
      }
    } else {
    for (int r = 0; r < reps; ++r) {
      if (VAR != 3) {
#pragma unroll 1
        for (int ks = 0; ks < 8; ++ks) {
          // X_hi, X_lo, Y_hi, Y_lo: 4 distinct 128 x 128 fp16 tiles (32 KB each) as in the kernel
          const uint64_t xh = dx + ((ks * 2 * lbo_x) >> 4);
          const uint64_t xl = xh + ((VAR >= 4 ? 0u : 32768u) >> 4);
          const uint64_t yh = xh + ((VAR >= 4 ? 0u : 65536u) >> 4), yl = xh + ((VAR >= 4 ? 0u : 98304u) >> 4);
          const uint64_t bh = ds + (((ks & 3) * 2 * lbo_s) >> 4), bl = bh + ((NC * 32u) >> 4);
          mma_f16_ss(t + fx, xh, bh, id1, ks > 0); mma_f16_ss(t + fx, xh, bl, id1, 1); mma_f16_ss(t + fx, xl, bh, id1, 1);
          mma_f16_ss(t + fy, yh, bh, id1, ks > 0); mma_f16_ss(t + fy, yh, bl, id1, 1); mma_f16_ss(t + fy, yl, bh, id1, 1);
          n += 6;
        }
      }
      if (VAR != 2) {
#pragma unroll 1
        for (int s = 0; s < NC / 16; ++s) {
          const uint32_t p = t + pbase + (VAR == 1 ? 8 * s : 16 * s);
          mma_f16_ts(t, p, da, id2, 1); mma_f16_ts(t, p, da, id2, 1); mma_f16_ts(t, p + 8, da, id2, 1);
          n += 3;
        }
      }
    }
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    out[blockIdx.x] = (clock64() - c0) * 1000 / n;
    done = 1;
  }
  if (TMA && tid == 32) {  // concurrent ring refills into a separate smem region
    int uses[4] = {0, 0, 0, 0};
    size_t src = (blockIdx.x * 65536u) % (1u << 20);
    for (int it = 0; !done && it < 200000; ++it) {
      const int st = it & 3;
      if (uses[st] > 0) mbar_wait(&tbar[st], (uses[st] - 1) & 1);
      mbar_arrive_expect_tx(&tbar[st], TMA);
      bulk_g2s(smem + 192 * 1024 + st * 8192, tab + src, TMA, &tbar[st]);
      ++uses[st];
      src = (src + TMA) % (1u << 20);
    }
    for (int st = 0; st < 4; ++st)
      if (uses[st] > 0) mbar_wait(&tbar[st], (uses[st] - 1) & 1);
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (tid < 32) tmem_dealloc(t, 512);
}

template <int NC, int VAR, int TMA>
void run(long long* d, const uint8_t* tab) {
  auto kk = k<NC, VAR, TMA>;
  cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024);
  for (int it = 0; it < 2; ++it) kk<<<148, 128, 224 * 1024>>>(32, d, tab);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
  long long h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double s = 0; for (int i = 0; i < 148; ++i) s += h[i];
  // ideal: G1 48 x max(45, NC/2, (4096+32NC)/128); G2 3NC/16 x 112
  const double g1 = 48 * fmax(fmax(45.0, NC / 2.0), (4096.0 + 32.0 * NC) / 128.0), g2 = 3.0 * NC / 16 * 112;
  const double nm = (VAR == 2 ? 48 : VAR == 3 ? 3 * NC / 16 : 48 + 3 * NC / 16);  // VAR 4: like 0 with one A tile
  const double ideal = (VAR == 2 ? g1 : VAR == 3 ? g2 : g1 + g2) / nm;
  printf("{\"NC\": %d, \"tma_bytes\": %d, \"var\": %d, \"cyc_per_mma\": %.1f, \"model\": %.1f}\n", NC, TMA, VAR, s / 148 / 1000, ideal);
}
int main() {
  long long* d; cudaMalloc(&d, 148 * 8);
  uint8_t* tab; cudaMalloc(&tab, 2 << 20); cudaMemset(tab, 0, 2 << 20);
  run<128, 0, 0>(d, tab); run<128, 5, 0>(d, tab); run<64, 0, 0>(d, tab); run<64, 5, 0>(d, tab); run<64, 6, 0>(d, tab);
  return 0;
}
