// TMA (cp.async.bulk) streaming rate from an L2-resident table into a
// shared-memory ring, all SMs busy: producer thread issues slices, consumer
// thread waits for each and releases it immediately.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2506_13523_b200/csrc/kernels/sm100.cuh"
using namespace tpo_b200::sm100;

template <int VAR>
__global__ void __launch_bounds__(128, 1) k(const uint8_t* tab, size_t tab_bytes, int slice, int depth, int nslices,
                                           long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[16], empty[16];
  const int tid = threadIdx.x;
  if (tid == 0) { for (int i = 0; i < 16; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); } fence_mbar_init(); }
  __syncthreads();
  long long c0 = clock64();
  if (VAR == 2 && (tid == 0 || tid == 64)) {
    const int base = tid == 0 ? 0 : 8;
    size_t src = (size_t(blockIdx.x) * 7919 * slice + base * slice) % tab_bytes;
    const int ns = nslices / 2;
    for (int n = 0; n < ns; ++n) {
      const int st = n % depth;
      if (n >= depth) mbar_wait(&full[base + st], ((n / depth) - 1) & 1);
      mbar_arrive_expect_tx(&full[base + st], slice);
      bulk_g2s(smem + (base / 8) * 100 * 1024 + st * slice, tab + src, slice, &full[base + st]);
      src += slice;
      if (src + slice > tab_bytes) src = 0;
    }
    for (int st = 0; st < depth && st < ns; ++st) {
      const int last = ((ns - 1 - st) / depth) * depth + st;
      mbar_wait(&full[base + st], (last / depth) & 1);
    }
    if (tid == 0) out[blockIdx.x] = clock64() - c0;
  } else if (VAR != 2 && tid == 0) {
    size_t src = (size_t(blockIdx.x) * 7919 * slice) % tab_bytes;
    for (int n = 0; n < nslices; ++n) {
      const int st = n % depth;
      if (VAR == 0 && n >= depth) mbar_wait(&empty[st], ((n / depth) - 1) & 1);
      if (VAR == 1 && n >= depth) mbar_wait(&full[st], ((n / depth) - 1) & 1);  // own completion, no consumer
      mbar_arrive_expect_tx(&full[st], slice);
      bulk_g2s(smem + st * slice, tab + src, slice, &full[st]);
      src += slice;
      if (src + slice > tab_bytes) src = 0;
    }
    if (VAR == 1) {
      for (int st = 0; st < depth && st < nslices; ++st) {
        const int last = ((nslices - 1 - st) / depth) * depth + st;
        mbar_wait(&full[st], (last / depth) & 1);
      }
      out[blockIdx.x] = clock64() - c0;
    }
  } else if (tid == 32 && VAR == 0) {
    for (int n = 0; n < nslices; ++n) {
      const int st = n % depth;
      mbar_wait(&full[st], (n / depth) & 1);
      mbar_arrive(&empty[st]);
    }
    out[blockIdx.x] = clock64() - c0;
  }
}

int main() {
  const size_t tab_bytes = 1200 * 1024;
  uint8_t* tab; cudaMalloc(&tab, tab_bytes); cudaMemset(tab, 1, tab_bytes);
  long long* d; cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int var : {1, 2})
  for (int slice : {4096, 8192, 12288})
    for (int depth : {4, 8}) {
      if (var == 2 && slice * depth > 100 * 1024) continue;
      if (slice * depth > 200 * 1024) continue;
      const int ns = 2000;
      for (int it = 0; it < 2; ++it) {
        if (var == 0) k<0><<<148, 128, 200 * 1024>>>(tab, tab_bytes, slice, depth, ns, d);
        else if (var == 1) k<1><<<148, 128, 200 * 1024>>>(tab, tab_bytes, slice, depth, ns, d);
        else k<2><<<148, 128, 200 * 1024>>>(tab, tab_bytes, slice, depth, ns, d);
      }
      cudaError_t e = cudaDeviceSynchronize();
      if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      long long h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
      double s = 0; for (int i = 0; i < 148; ++i) s += h[i];
      s /= 148;
      printf("{\"var\": %d, \"slice\": %d, \"depth\": %d, \"bytes_per_cyc_per_sm\": %.1f, \"cyc_per_slice\": %.0f}\n", var, slice, depth,
             double(slice) * ns / s, s / ns);
    }
  return 0;
}
