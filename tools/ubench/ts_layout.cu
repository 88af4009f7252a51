// Correctness probe: tcgen05.mma kind::f16 with A from TMEM (M=128, N=16, K=16).
// Writes A via tcgen05.st assuming lane = row, 32-bit column j = (A[r][2j], A[r][2j+1]),
// B in smem canonical K-major, compares D against a CPU reference.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include "../../paper_2506_13523_b200/csrc/kernels/sm100.cuh"
using namespace tpo_b200::sm100;

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
               :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]) : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
               :: "r"(d), "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc) : "memory");
}
__global__ void k(const float* A, const float* B, float* D) {  // A [128][16], B [16][16] (n,k)
  __shared__ __align__(128) uint8_t bs[16 * 16 * 2];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tm;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 256; i += 128) {
    const int n = i / 16, kk = i % 16;
    *reinterpret_cast<__half*>(bs + canon_off(n, kk, 16)) = __float2half(B[i]);
  }
  if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) { tmem_alloc(&tm, 64); tmem_relinquish(); }
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t t = tm, lane_base = t + ((warp * 32) << 16);
  uint32_t w[8];
  for (int j = 0; j < 8; ++j) {
    __half2 h = __floats2half2_rn(A[tid * 16 + 2 * j], A[tid * 16 + 2 * j + 1]);
    w[j] = *reinterpret_cast<uint32_t*>(&h);
  }
  tmem_st8(lane_base + 32, w);
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (tid == 0) {
    mma_ts(t, t + 32, make_sdesc(smem_u32(bs), 16 * 16, 128), idesc_f16(128, 16), 0u);
    tc_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t r[16];
  tmem_ld16(lane_base, r);
  tmem_wait_ld();
  for (int n = 0; n < 16; ++n) D[tid * 16 + n] = __uint_as_float(r[n]);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == 0) tmem_dealloc(t, 64);
}
int main() {
  float hA[128 * 16], hB[256], hD[128 * 16];
  for (int i = 0; i < 128 * 16; ++i) hA[i] = (float)((i * 7) % 13 - 6);
  for (int i = 0; i < 256; ++i) hB[i] = (float)((i * 5) % 11 - 5);
  float *A, *B, *D; cudaMalloc(&A, sizeof hA); cudaMalloc(&B, sizeof hB); cudaMalloc(&D, sizeof hD);
  cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice); cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
  k<<<1, 128>>>(A, B, D);
  cudaError_t e = cudaDeviceSynchronize();
  if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
  cudaMemcpy(hD, D, sizeof hD, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  for (int m = 0; m < 128; ++m) for (int n = 0; n < 16; ++n) {
    double ref = 0; for (int kk = 0; kk < 16; ++kk) ref += hA[m * 16 + kk] * hB[n * 16 + kk];
    maxerr = fmax(maxerr, fabs(ref - hD[m * 16 + n]));
  }
  printf("{\"ts_layout_maxerr\": %g, \"D00\": %g}\n", maxerr, hD[0]);
  return 0;
}
