// TMEM read bandwidth probe: W warps (W<=8) each read their sub-partition's
// 32 lanes x 256 columns with tcgen05.ld 32x32b.x32, R times; clock64 per warp.
#include <cstdio>
#include <cstdint>
#include "../../../paper_2602_10016_b200/csrc/tc_common.cuh"
using namespace kl::tc;
template <int MODE> __global__ void probe(int R, long long* out, float* sink) {
  __shared__ uint32_t taddr_s;
  int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc(&taddr_s, 512);
  fence_before(); __syncthreads(); fence_after();
  uint32_t t = taddr_s;
  uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
  float acc = 0.f;
  __syncthreads();
  long long c0 = clock64();
  for (int r = 0; r < R; ++r) {
    if (MODE == 0) {
    for (int c = 0; c < 256; c += 32) {
      float v[32];
      tmem_ld32(t + lane_base + c + (warp >> 2) * 256, v);
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += v[i];
    }
    } else {
    for (int c = 0; c < 256; c += 128) {
      uint32_t v[128];
#pragma unroll
      for (int j = 0; j < 4; ++j) tmem_ld32_nowait(t + lane_base + c + j * 32 + (warp >> 2) * 256, v + 32 * j);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 128; ++i) acc += __uint_as_float(v[i]);
    }
    }
  }
  long long c1 = clock64();
  if ((threadIdx.x & 31) == 0) out[blockIdx.x * 8 + warp] = c1 - c0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  fence_before(); __syncthreads(); fence_after();
  if (warp == 0) tmem_dealloc(t, 512);
}
int main() {
  long long* d; float* s; cudaMalloc(&d, 8 * 148 * 8); cudaMalloc(&s, 148 * 256 * 4);
  for (int mode = 0; mode < 2; ++mode)
  for (int W : {1, 2, 4, 8}) {
    int R = 200;
    if (mode == 0) probe<0><<<1, 32 * W>>>(R, d, s); else probe<1><<<1, 32 * W>>>(R, d, s);
    cudaDeviceSynchronize();
    long long h[8]; cudaMemcpy(h, d, 8 * 8, cudaMemcpyDeviceToHost);
    long long mx = 0; for (int i = 0; i < W; ++i) mx = h[i] > mx ? h[i] : mx;
    double bytes = (double)W * R * 256 * 32 * 4;
    printf("mode %d warps %d: %lld clk, %.1f B/clk per SM (%.1f per warp)  err=%s\n", mode, W, mx, bytes / mx, bytes / mx / W,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
