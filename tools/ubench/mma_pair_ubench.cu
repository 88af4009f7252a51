// tcgen05.mma.cta_group::2 (M=256 over a CTA pair) issue/throughput vs N,
// SS and TS, groups of 3 MMAs with and without a per-group mbarrier wait.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2506_13523_b200/csrc/kernels/sm100.cuh"
using namespace tpo_b200::sm100;

template <int N, int MODE, int WAIT>  // MODE 0 SS, 1 TS
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k(int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ uint32_t tm;
  const int tid = threadIdx.x;
  const uint32_t rank = cluster_ctarank();
  for (int i = tid; i < 96 * 1024 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (tid == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); fence_mbar_init(); }
  fence_proxy_async_smem();
  if (tid < 32) { tmem_alloc_pair(&tm, 512); tmem_relinquish_pair(); }
  tc_fence_before(); cluster_sync_all(); tc_fence_after();
  const uint32_t t = tm;
  if (rank == 0 && tid == 0) {
    mbar_arrive(&bar[1]);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32 * 1024);
    constexpr uint32_t idesc = idesc_f16(256, N);
    constexpr uint32_t lbo_a = 16 * 128, lbo_b = (N / 2 / 8) * 128;
    const uint64_t ad0 = make_sdesc(a, lbo_a, 128), bd0 = make_sdesc(b, lbo_b, 128);
    long long c0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        if (WAIT == 1) { mbar_wait(&bar[1], 0); tc_fence_after(); }
        if (WAIT == 2) { mbar_wait_cluster(&bar[1], 0); tc_fence_after(); }
        if (WAIT == 3) { mbar_wait_cluster(&bar[1], 0); mbar_wait_cluster(&bar[1], 0); tc_fence_after(); }
        const uint64_t bd = bd0 + ((kk * 2 * lbo_b) >> 4);
        if (MODE == 0) {
          const uint64_t ad = ad0 + ((kk * 2 * lbo_a) >> 4);
          mma_f16_ss_pair(t, ad, bd, idesc, 1u); mma_f16_ss_pair(t, ad, bd, idesc, 1u); mma_f16_ss_pair(t, ad, bd, idesc, 1u);
        } else {
          mma_f16_ts_pair(t, t + 256 + kk * 8, bd, idesc, 1u); mma_f16_ts_pair(t, t + 256, bd, idesc, 1u); mma_f16_ts_pair(t, t + 264, bd, idesc, 1u);
        }
      }
    }
    tc_commit_pair(&bar[0]);
    mbar_wait(&bar[0], 0);
    out[blockIdx.x / 2] = clock64() - c0;
  }
  if (rank == 1 && tid == 0) mbar_wait(&bar[0], 0);
  tc_fence_before(); cluster_sync_all(); tc_fence_after();
  if (tid < 32) tmem_dealloc_pair(t, 512);
}

template <int N, int MODE, int WAIT>
void run(long long* d) {
  auto kk = k<N, MODE, WAIT>;
  cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  const int reps = 64;
  for (int it = 0; it < 2; ++it) kk<<<148, 128, 96 * 1024>>>(reps, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
  long long h[74]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double s = 0; for (int i = 0; i < 74; ++i) s += h[i];
  printf("{\"pair\": 1, \"mode\": \"%s\", \"N\": %d, \"wait\": %d, \"cyc_per_mma\": %.1f, \"ideal_M128_equiv\": %.1f}\n",
         MODE ? "TS" : "SS", N, WAIT, s / 74 / (reps * 24), N / 2.0);
}
int main() {
  long long* d; cudaMalloc(&d, 74 * 8);
  run<128, 0, 1>(d); run<128, 0, 2>(d); run<128, 0, 3>(d);
  run<224, 1, 1>(d); run<224, 1, 2>(d); run<224, 1, 3>(d);
  return 0;
}
