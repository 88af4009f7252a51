// Microbenchmark v2: tcgen05.mma issue floor with precomputed descriptors
// (no per-MMA descriptor arithmetic beyond a 64-bit add), fully unrolled.
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

__device__ __forceinline__ uint32_t elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P1;\n\telect.sync _|P1, 0xffffffff;\n\tselp.b32 %0, 1, 0, P1;\n\t}" : "=r"(pred));
  return pred;
}
__device__ __forceinline__ void mma4_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint64_t da, uint64_t db) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
               ".reg .b64 a1, a2, a3, b1, b2, b3;\n\t"
               "add.s64 a1, %1, %4;\n\tadd.s64 a2, a1, %4;\n\tadd.s64 a3, a2, %4;\n\t"
               "add.s64 b1, %2, %5;\n\tadd.s64 b2, b1, %5;\n\tadd.s64 b3, b2, %5;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, p;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, p;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, p;\n\t}"
               :: "r"(d), "l"(a), "l"(b), "r"(idesc), "l"(da), "l"(db) : "memory");
}
template <int MODE, int N, int NACC>
__global__ void __launch_bounds__(128, 1) k_mma(int reps, long long* out) {
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
  if ((MODE == 2 && tid < 32) || (MODE != 2 && tid == 0)) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32 * 1024);
    constexpr uint32_t idesc = idesc_f16(128, N);
    constexpr uint32_t lbo_a = 16 * 128, lbo_b = (N / 8) * 128;
    const uint64_t ad0 = make_sdesc(a, lbo_a, 128), bd0 = make_sdesc(b, lbo_b, 128);
    long long c0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint64_t bd = bd0 + ((k * 2 * lbo_b) >> 4);
        if (MODE == 2) { if (elect_one()) mma_f16_ss(t + (k % NACC) * N, ad0 + ((k * 2 * lbo_a) >> 4), bd, idesc, 1u); __syncwarp(); }
        else if (MODE == 3) { if ((k & 3) == 0) mma4_ss(t, ad0 + ((k * 2 * lbo_a) >> 4), bd, idesc, (2 * lbo_a) >> 4, (2 * lbo_b) >> 4); }
        else if (MODE == 0) mma_f16_ss(t + (k % NACC) * N, ad0 + ((k * 2 * lbo_a) >> 4), bd, idesc, 1u);
        else mma_ts(t + (k % NACC) * N, t + 448 + k * 8, bd, idesc, 1u);
      }
    }
    if (MODE != 2 || elect_one()) tc_commit(&bar);
    __syncwarp(MODE == 2 ? 0xffffffffu : 1u);
    mbar_wait(&bar, 0);
    long long c1 = clock64();
    if (tid == 0) out[blockIdx.x] = c1 - c0;
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (tid < 32) tmem_dealloc(t, 512);
}

template <int MODE, int N, int NACC>
void run(long long* d, int nsm) {
  auto k = k_mma<MODE, N, NACC>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
  const int reps = 256;
  for (int it = 0; it < 2; ++it) k<<<nsm, 128, 128 * 1024>>>(reps, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
  long long h[1024];
  cudaMemcpy(h, d, nsm * 8, cudaMemcpyDeviceToHost);
  long long sum = 0; for (int i = 0; i < nsm; ++i) sum += h[i];
  const double per = double(sum) / nsm / (reps * 8);
  const double ideal = 128.0 * N / 256.0;
  printf("{\"mode\": \"%s\", \"nacc\": %d, \"N\": %d, \"cyc_per_mma\": %.2f, \"ideal\": %.1f, \"eff\": %.3f}\n",
         MODE == 1 ? "TS" : MODE == 2 ? "SS-warp-elect" : MODE == 3 ? "SS-asm4" : "SS", NACC, N, per, ideal, ideal / per);
}

int main(int argc, char** argv) {
  int nsm = argc > 1 ? atoi(argv[1]) : 148;
  long long* d; cudaMalloc(&d, 1024 * 8);
  run<0, 16, 1>(d, nsm); run<0, 16, 4>(d, nsm);
  run<0, 32, 1>(d, nsm); run<0, 32, 4>(d, nsm);
  run<0, 64, 1>(d, nsm); run<0, 64, 4>(d, nsm);
  run<0, 128, 1>(d, nsm); run<0, 128, 2>(d, nsm);
  run<0, 256, 1>(d, nsm);
  run<2, 16, 1>(d, nsm); run<2, 32, 1>(d, nsm); run<2, 64, 1>(d, nsm); run<2, 128, 1>(d, nsm);
  run<3, 16, 1>(d, nsm); run<3, 32, 1>(d, nsm); run<3, 64, 1>(d, nsm); run<3, 128, 1>(d, nsm);
  if (nsm < 0) run<1, 16, 1>(d, nsm); run<1, 16, 4>(d, nsm);
  run<1, 32, 1>(d, nsm); run<1, 32, 4>(d, nsm);
  run<1, 64, 1>(d, nsm); run<1, 64, 4>(d, nsm);
  run<1, 128, 1>(d, nsm); run<1, 128, 2>(d, nsm);
  run<1, 256, 1>(d, nsm);
  return 0;
}
