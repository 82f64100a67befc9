// TMA latency / throughput probe: one CTA loads k boxes (64 x R rows bf16,
// SWIZZLE_128B) from a (rows x 512) bf16 tensor and waits; clock64.
#include <cstdio>
#include <cstdint>
#include <cudaTypedefs.h>
#include <cuda.h>
#include "../../../paper_2602_10016_b200/csrc/tc_common.cuh"
using namespace kl::tc;
__global__ void probe(const __grid_constant__ CUtensorMap m, int k, int rows, int rep, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1); fence_barrier_init();
    prefetch_tmap(&m);
    long long tot = 0, first = 0;
    for (int r = 0; r < rep; ++r) {
      long long c0 = clock64();
      mbar_arrive_expect_tx(&bar, k * rows * 128);
      for (int i = 0; i < k; ++i)
        tma_load_3d(s + i * rows * 128, &m, &bar, (i % 8) * 64, ((blockIdx.x * 97 + r * 13 + i / 8) * rows) % 65536, 0);
      mbar_wait(&bar, r & 1);
      long long c1 = clock64();
      if (r == 0) first = c1 - c0; else tot += c1 - c0;
    }
    out[blockIdx.x * 2] = first; out[blockIdx.x * 2 + 1] = tot / (rep - 1);
  }
}
int main() {
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  const long long R = 65536 + 128, C = 512;
  void* buf; cudaMalloc(&buf, R * C * 2); cudaMemset(buf, 0, R * C * 2);
  long long* d; cudaMalloc(&d, 148 * 16);
  for (int rows : {64, 128}) {
    CUtensorMap m;
    cuuint64_t dims[3] = {(cuuint64_t)C, (cuuint64_t)R, 1};
    cuuint64_t str[2] = {(cuuint64_t)(C * 2), (cuuint64_t)(C * 2 * R)};
    cuuint32_t box[3] = {64, (cuuint32_t)rows, 1}, es[3] = {1, 1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int grid : {1, 148})
      for (int k : {1, 4, 8, 16}) {
        if (k * rows * 128 > 200000) continue;
        cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 210000);
        probe<<<grid, 32, 210000>>>(m, k, rows, 20, d);
        cudaDeviceSynchronize();
        long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("grid %3d box 64x%3d k=%2d (%6d B): first %6lld clk, steady %6lld clk -> %.1f B/clk/SM  %s\n", grid, rows, k,
               k * rows * 128, h[0], h[1], (double)k * rows * 128 / h[1], cudaGetErrorString(cudaGetLastError()));
      }
  }
  return 0;
}
