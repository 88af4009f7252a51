// Minimal 2-D TMA load check (param-space tensor map, plain CTA launch).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

struct P { int a; alignas(64) CUtensorMap tm; };

__global__ void k(const __grid_constant__ P p, const CUtensorMap* gmap, float* out, int variant) {
  extern __shared__ __align__(1024) float sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(4096));
    const CUtensorMap* tm = variant == 3 ? gmap : &p.tm;
    if (variant != 1)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(su32(sm)), "l"(reinterpret_cast<uint64_t>(tm)), "r"(variant >= 10 ? variant - 10 : 5), "r"(0), "r"(su32(&bar)) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(su32(sm)), "l"(reinterpret_cast<uint64_t>(&p.tm)), "r"(variant >= 10 ? variant - 10 : 5), "r"(0), "r"(su32(&bar)) : "memory");
  }
  asm volatile("{\n\t.reg .pred q;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%0], 0;\n\t@!q bra W;\n\t}" ::"r"(su32(&bar)));
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = sm[i];
}

int main(int argc, char** argv) {
  const int only = argc > 1 ? atoi(argv[1]) : 0;
  const int inner = 1024, outer = 64;
  float* g; cudaMalloc(&g, inner * outer * 4);
  float* h = new float[inner * outer];
  for (int i = 0; i < inner * outer; ++i) h[i] = i;
  cudaMemcpy(g, h, inner * outer * 4, cudaMemcpyHostToDevice);
  float* out; cudaMalloc(&out, 4096);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q{};
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  for (int variant = only; variant <= only; ++variant)
    for (int sw = 0; sw < 2; ++sw) {
      P p{};
      const cuuint64_t dims[2] = {inner, outer};
      const cuuint64_t strides[1] = {inner * 4};
      const cuuint32_t box[2] = {32, 32};
      const cuuint32_t es[2] = {1, 1};
      CUresult r = enc(&p.tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       sw ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
      CUtensorMap* gm; cudaMalloc(&gm, sizeof(CUtensorMap));
      cudaMemcpy(gm, &p.tm, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
      if (variant == 2) {
        cudaLaunchConfig_t cfg{}; cfg.gridDim = 1; cfg.blockDim = 128; cfg.dynamicSmemBytes = 8192;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, k, p, (const CUtensorMap*)gm, out, variant);
      } else {
        k<<<1, 128, 8192>>>(p, gm, out, variant);
      }
      cudaError_t e = cudaDeviceSynchronize();
      float o[4] = {};
      cudaMemcpy(o, out, 16, cudaMemcpyDeviceToHost);
      std::printf("variant %d swizzle %d encode %d -> %s  out[0..3] = %g %g %g %g\n", variant, sw, (int)r,
                  cudaGetErrorString(e), o[0], o[1], o[2], o[3]);
      if (e != cudaSuccess) return 1;
    }
  return 0;
}
