// Standalone probe of TMA tensor loads (debug aid): ./tma_probe <variant>
//  0: 3-D map as __grid_constant__ param   1: 2-D map as __grid_constant__ param
//  2: 3-D map in global memory              3: 3-D map, box inner 32 floats
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int DIM>
__global__ void k(const __grid_constant__ CUtensorMap tm, const CUtensorMap* gtm, float* out, int bx, int by, int bz,
                  unsigned bytes) {
  extern __shared__ __align__(128) float sm[];
  __shared__ __align__(8) unsigned long long bar;
  const CUtensorMap* map = gtm ? gtm : &tm;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(bytes) : "memory");
    if (DIM == 3 && bytes == 7392u + 1u) {
      // never
    } else if (DIM == 3 && gtm == (const CUtensorMap*)1) {
    } else if (DIM == 3 && bz == 7) {  // 1-D bulk copy sanity
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su32(sm)), "l"(out), "r"(bytes), "r"(su32(&bar)) : "memory");
    } else if (DIM == 3 && bz == 8) {  // no .tile
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
          ::"r"(su32(sm)), "l"(reinterpret_cast<unsigned long long>(map)), "r"(bx), "r"(by), "r"(1), "r"(su32(&bar))
          : "memory");
    } else if (DIM == 3)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
          ::"r"(su32(sm)), "l"(reinterpret_cast<unsigned long long>(map)), "r"(bx), "r"(by), "r"(bz), "r"(su32(&bar))
          : "memory");
    else
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
          ::"r"(su32(sm)), "l"(reinterpret_cast<unsigned long long>(map)), "r"(bx), "r"(by), "r"(su32(&bar))
          : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(su32(&bar))
               : "memory");
  for (unsigned i = threadIdx.x; i < bytes / 4; i += blockDim.x) out[i] = sm[i];
}

int main(int argc, char** argv) {
  const int v = argc > 1 ? atoi(argv[1]) : 0;
  const int W = 128, H = 96, C = 3;
  float* img;
  cudaMalloc(&img, sizeof(float) * W * H * C);
  float* h = (float*)malloc(sizeof(float) * W * H * C);
  for (int i = 0; i < W * H * C; ++i) h[i] = (float)i;
  cudaMemcpy(img, h, sizeof(float) * W * H * C, cudaMemcpyHostToDevice);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = (CUresult(*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill))p;
  CUtensorMap tm;
  memset(&tm, 0, sizeof tm);
  const int bw = v == 3 ? 32 : (v == 7 ? 48 : 44), bh = 42;
  CUresult r;
  if (v == 1) {
    cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)H * C}, str[1] = {(cuuint64_t)W * 4};
    cuuint32_t box[2] = {(cuuint32_t)bw, (cuuint32_t)bh}, es[2] = {1, 1};
    r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, img, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)C}, str[2] = {(cuuint64_t)W * 4, (cuuint64_t)W * H * 4};
    cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, 1}, es[3] = {1, 1, 1};
    r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, img, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  printf("variant %d: entry %d encode %d\n", v, (int)q, (int)r);
  CUtensorMap* g = nullptr;
  if (v == 2) {
    cudaMalloc(&g, sizeof tm);
    cudaMemcpy(g, &tm, sizeof tm, cudaMemcpyHostToDevice);
  }
  float* out;
  const unsigned bytes = bw * bh * 4;
  cudaMalloc(&out, bytes);
  cudaFuncSetAttribute(k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  if (v == 1) k<2><<<1, 128, 16384>>>(tm, nullptr, out, -5, 96 + 10, 0, bytes);
  else if (v == 4) k<3><<<1, 128, 16384>>>(tm, g, out, -5, 10, 7, bytes);
  else if (v == 5) k<3><<<1, 128, 16384>>>(tm, g, out, -5, 10, 8, bytes);
  else if (v == 6) k<3><<<1, 128, 16384>>>(tm, g, out, 0, 0, 1, bytes);
  else if (v == 7) k<3><<<1, 128, 16384>>>(tm, g, out, -8, -5, 1, bytes);
  else k<3><<<1, 128, 16384>>>(tm, g, out, -5, 10, 1, bytes);
  cudaError_t e = cudaDeviceSynchronize();
  float* ho = (float*)malloc(bytes);
  cudaMemcpy(ho, out, bytes, cudaMemcpyDeviceToHost);
  if (v == 7) printf("v7: out[0]=%g (want 0) out[5*48+8]=%g (want %g) out[6*48+10]=%g (want %g)\n", ho[0], ho[5*48+8], (float)(W*H), ho[6*48+10], (float)(W*H + W + 2));
  printf("variant %d: %s; out[0..2] = %g %g %g (row0 col5 = %g, want %g)\n", v, cudaGetErrorString(e), ho[0], ho[1],
         ho[2], ho[5], (float)(1 * W * H + 10 * W + 0));
  return e == cudaSuccess ? 0 : 1;
}
