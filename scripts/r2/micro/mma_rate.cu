// tcgen05.mma throughput probe: one thread issues R MMAs (M=128, N in {32..256},
// K=16, bf16, SS or TS operands) into one TMEM accumulator; clock64 around
// issue + commit-wait.
#include <cstdio>
#include <cstdint>
#include "../../../paper_2602_10016_b200/csrc/tc_common.cuh"
using namespace kl::tc;
template <int N, bool TS>
__global__ void probe(int R, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) ((uint32_t*)s)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc(&tslot, 512);
  fence_async_smem();
  fence_before(); __syncthreads(); fence_after();
  uint32_t t = tslot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(s), b = smem_u32(s + 32768);
    const uint32_t idesc = idesc_bf16(128, N, 0, 0);
    long long c0 = clock64();
    for (int r = 0; r < R; ++r) {
      if (TS) mma_bf16_ts(t, t + 256 + (r & 3) * 8, sdesc(b + (r & 3) * 32, 16, 1024), idesc, 1u);
      else mma_bf16(t, sdesc(a + (r & 3) * 32, 16, 1024), sdesc(b + (r & 3) * 32, 16, 1024), idesc, 1u);
    }
    long long c1 = clock64();
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long c2 = clock64();
    out[0] = c1 - c0; out[1] = c2 - c0;
  }
  fence_before(); __syncthreads(); fence_after();
  if (threadIdx.x < 32) tmem_dealloc(t, 512);
}
template <int N, bool TS> void run(long long* d) {
  const int R = 1024;
  cudaFuncSetAttribute(probe<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  probe<N, TS><<<1, 128, 70000>>>(R, d);
  cudaDeviceSynchronize();
  long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  double macs = 128.0 * N * 16 * R;
  printf("N=%3d %s: issue %lld clk, done %lld clk -> %.1f clk/MMA, %.0f MAC/clk (%s)\n", N, TS ? "TS" : "SS", h[0], h[1],
         (double)h[1] / R, macs / h[1], cudaGetErrorString(cudaGetLastError()));
}
int main() {
  long long* d; cudaMalloc(&d, 64);
  run<32, false>(d); run<64, false>(d); run<128, false>(d); run<256, false>(d);
  run<64, true>(d); run<128, true>(d); run<256, true>(d);
  return 0;
}
