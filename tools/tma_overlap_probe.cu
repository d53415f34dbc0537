// Probe: does cuTensorMapEncodeTiled accept a 2-D view whose row stride (256 B) is smaller
// than its inner extent (384 B), and does TMA read the overlapping windows correctly?
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void k(const __grid_constant__ CUtensorMap m, int c0, int r0, uint8_t* out) {
  __shared__ alignas(1024) uint8_t s[128 * 8];
  __shared__ alignas(8) uint64_t bar;
  uint32_t sb = (uint32_t)__cvta_generic_to_shared(&bar), sd = (uint32_t)__cvta_generic_to_shared(s);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(128 * 8));
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(sd), "l"(&m), "r"(c0), "r"(r0), "r"(sb) : "memory");
    uint32_t ok = 0;
    while (!ok) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(sb));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 128 * 8; i += blockDim.x) out[i] = s[i];
}

int main() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  Enc enc = (Enc)p;
  const int L = 4096 + 512;
  std::vector<uint8_t> h(L);
  for (int i = 0; i < L; ++i) h[i] = (uint8_t)(i * 7 + (i >> 8));
  uint8_t *d, *o;
  cudaMalloc(&d, L); cudaMalloc(&o, 1024);
  cudaMemcpy(d, h.data(), L, cudaMemcpyHostToDevice);
  CUtensorMap m;
  cuuint64_t dims[2] = {384, 16};
  cuuint64_t strides[1] = {256};
  cuuint32_t box[2] = {128, 8};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode overlapping (dim0=384, stride=256): %d\n", (int)r);
  if (r != CUDA_SUCCESS) return 0;
  int bad = 0;
  for (int c0 : {0, 16, 128, 208, 240, 256}) {
    k<<<1, 128>>>(m, c0, 3, o);
    std::vector<uint8_t> g(1024);
    cudaMemcpy(g.data(), o, 1024, cudaMemcpyDeviceToHost);
    for (int row = 0; row < 8; ++row)
      for (int i = 0; i < 128; ++i) {
        int src = (3 + row) * 256 + c0 + i;
        uint8_t want = (c0 + i < 384) ? h[src] : 0;
        if (g[row * 128 + i] != want) ++bad;
      }
    printf("c0=%d err=%s\n", c0, cudaGetErrorString(cudaDeviceSynchronize()));
  }
  printf("mismatches: %d\n", bad);
  return 0;
}
