// Microbenchmark: tcgen05.mma (kind::f16, M=128, K=16) issue/throughput vs N
// for A from shared memory (SS) and A from TMEM (TS), and tcgen05.ld
// throughput.  One CTA per SM, all SMs busy.  Prints cycles per MMA.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2506_13523_b200/csrc/kernels/sm100.cuh"
using namespace tpo_b200::sm100;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
               :: "r"(d), "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc) : "memory");
}

template <int MODE>  // 0 = SS, 1 = TS
__global__ void __launch_bounds__(128, 1) k_mma(int N, int reps, int kdepth, int nacc, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tm;
  const int tid = threadIdx.x;
  for (int i = tid; i < 128 * 1024 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (tid < 32) { tmem_alloc(&tm, 512); tmem_relinquish(); }
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t t = tm;
  long long c0 = 0, c1 = 0;
  if (tid == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32 * 1024);
    const uint32_t idesc = idesc_f16(128, N);
    // A: R=128 rows, K=16*kdepth; B: R=N rows
    const uint32_t lbo_a = 16 * 128, lbo_b = (N / 8) * 128;
    c0 = clock64();
    for (int r = 0; r < reps; ++r)
      for (int k = 0; k < kdepth; ++k) {
        const uint64_t bd = make_sdesc(b + k * 2 * lbo_b, lbo_b, 128);
        if (MODE == 0) {
          const uint64_t ad = make_sdesc(a + k * 2 * lbo_a, lbo_a, 128);
          mma_f16_ss(t + (k % nacc) * N, ad, bd, idesc, 1u);
        } else {
          mma_ts(t + (k % nacc) * N, t + 448 + (k & 7) * 8, bd, idesc, 1u);
        }
      }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    c1 = clock64();
    out[blockIdx.x] = c1 - c0;
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (tid < 32) tmem_dealloc(t, 512);
}

__global__ void __launch_bounds__(128, 1) k_ld(int reps, long long* out) {
  __shared__ uint32_t tm;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid < 32) { tmem_alloc(&tm, 512); tmem_relinquish(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t t = tm + ((warp * 32) << 16);
  uint32_t acc = 0;
  long long c0 = clock64();
  for (int r = 0; r < reps; ++r) {
    uint32_t v[16];
    tmem_ld16(t + (r & 31) * 16, v);
    tmem_wait_ld();
#pragma unroll
    for (int q = 0; q < 16; ++q) acc += v[q];
  }
  long long c1 = clock64();
  if (tid == 0) out[blockIdx.x] = c1 - c0;
  if (acc == 0x12345678) out[0] = 0;
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (tid < 32) tmem_dealloc(tm, 512);
}

int main() {
  int nsm = 148;
  long long* d; cudaMalloc(&d, 1024 * 8);
  long long h[1024];
  cudaFuncSetAttribute(k_mma<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
  cudaFuncSetAttribute(k_mma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
  const int reps = 512;
  for (int mode = 0; mode < 2; ++mode)
    for (int N : {16, 32, 64, 128, 192, 256})
     for (int nacc : {1, 2, 4}) {
      if (nacc * N > 448 || (mode == 1 && nacc * N > 448)) continue;
      const int kd = 8;
      for (int it = 0; it < 2; ++it) {
        if (mode == 0) k_mma<0><<<nsm, 128, 128 * 1024>>>(N, reps, kd, nacc, d);
        else k_mma<1><<<nsm, 128, 128 * 1024>>>(N, reps, kd, nacc, d);
      }
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, d, nsm * 8, cudaMemcpyDeviceToHost);
      long long mx = 0, sum = 0;
      for (int i = 0; i < nsm; ++i) { mx = h[i] > mx ? h[i] : mx; sum += h[i]; }
      const double per = double(sum) / nsm / (reps * kd);
      const double ideal = 128.0 * N / 256.0;
      printf("{\"mode\": \"%s\", \"nacc\": %d, \"N\": %d, \"cyc_per_mma\": %.2f, \"ideal\": %.1f, \"eff\": %.3f, \"max_cyc\": %lld}\n",
             mode ? "TS" : "SS", nacc, N, per, ideal, ideal / per, mx);
    }
  for (int it = 0; it < 2; ++it) k_ld<<<nsm, 128>>>(4096, d);
  cudaDeviceSynchronize();
  cudaMemcpy(h, d, nsm * 8, cudaMemcpyDeviceToHost);
  long long sum = 0; for (int i = 0; i < nsm; ++i) sum += h[i];
  printf("{\"tmem_ld_32x32b_x16\": {\"cyc_per_ld_per_warp\": %.2f, \"bytes_per_cyc_per_sm\": %.1f}}\n",
         double(sum) / nsm / 4096, 4 * 32 * 16 * 4 / (double(sum) / nsm / 4096));
  return 0;
}
