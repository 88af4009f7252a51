// Per-MMA cost of the grid kernel's issue pattern: groups of 3 SS MMAs
// (M=128, N, K=16) with optional tcgen05.commit and mbarrier wait + fence per group.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2506_13523_b200/csrc/kernels/sm100.cuh"
using namespace tpo_b200::sm100;

template <int N, int VAR>
__global__ void __launch_bounds__(128, 1) k(int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar[10];
  __shared__ uint32_t tm;
  const int tid = threadIdx.x;
  for (int i = tid; i < 160 * 1024 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (tid == 0) { for (int i = 0; i < 10; ++i) mbar_init(&bar[i], 1); fence_mbar_init(); }
  if (tid < 32) { tmem_alloc(&tm, 512); tmem_relinquish(); }
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t t = tm;
  if (tid == 0) {
    // "ready" barrier: complete phase 0 once
    mbar_arrive(&bar[8]);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 64 * 1024);
    constexpr uint32_t idesc = idesc_f16(128, N);
    constexpr uint32_t lbo_a = 16 * 128, lbo_b = (N / 8) * 128;
    long long c0 = clock64();
    int stage = 0;
    for (int r = 0; r < reps; ++r) {
      for (int k = 0; k < 8; ++k) {
        if (VAR == 2) { mbar_wait(&bar[8], 0); tc_fence_after(); }
        if (VAR == 3) { mbar_wait(&bar[8], 0); }
        if (VAR == 4) { tc_fence_after(); }
        if (VAR == 5 && (k & 1) == 0) { mbar_wait(&bar[8], 0); tc_fence_after(); }
        if (VAR == 6) { uint32_t ok; asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.b32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(&bar[8])) : "memory"); if (!ok) mbar_wait(&bar[8], 0); tc_fence_after(); }
        const uint64_t ad = make_sdesc(a + k * 2 * lbo_a, lbo_a, 128);
        const uint64_t bh = make_sdesc(b + stage * 8192, lbo_b, 128), bl = make_sdesc(b + stage * 8192 + N * 32, lbo_b, 128);
        mma_f16_ss(t, ad, bh, idesc, 1u);
        mma_f16_ss(t, ad, bl, idesc, 1u);
        mma_f16_ss(t, ad + 1, bh, idesc, 1u);
        if (VAR >= 1) tc_commit(&bar[stage]);
        if (++stage == 8) stage = 0;
      }
    }
    tc_commit(&bar[9]);
    mbar_wait(&bar[9], 0);
    long long c1 = clock64();
    out[blockIdx.x] = c1 - c0;
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (tid < 32) tmem_dealloc(t, 512);
}

template <int N, int VAR>
void run(long long* d) {
  auto kk = k<N, VAR>;
  cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  const int reps = 128;
  for (int it = 0; it < 2; ++it) kk<<<148, 128, 160 * 1024>>>(reps, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
  long long h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  long long s = 0; for (int i = 0; i < 148; ++i) s += h[i];
  printf("{\"N\": %d, \"variant\": %d, \"cyc_per_mma\": %.1f}\n", N, VAR, double(s) / 148 / (reps * 24));
}
int main() {
  long long* d; cudaMalloc(&d, 148 * 8);
  run<128, 1>(d); run<128, 2>(d); run<128, 3>(d); run<128, 4>(d); run<128, 5>(d); run<128, 6>(d);
  run<224, 1>(d); run<224, 2>(d); run<224, 3>(d);
  return 0;
}
