// Shared device helpers for libkunlun_sm100a (B200, sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <utility>

#include "../../include/kunlun_capi.h"

namespace kl {

typedef __nv_bfloat16 bf16;

// ---- error plumbing (host) -------------------------------------------------
void set_error(const char* fmt, ...);
int launch_check(const char* what);
void count_launch(unsigned n = 1);
void count_path(int path, unsigned n = 1);  // KL_PATH_* kernel-family counters
bool pdl_enabled();
void bind_device(cudaStream_t s);

// ---- launches: programmatic dependent launch (PDL) --------------------------
// Every kernel of the library calls KL_PDL_ENTRY() before its first global
// memory access and, when PDL is on (default; kl_set_pdl / KL_PDL=0 turns it
// off), is launched with programmatic stream serialization: it lets the next
// kernel in the
// stream be scheduled while this one drains, and waits (griddepcontrol.wait)
// for the full completion + memory flush of its predecessor before touching
// global memory.  Inside a captured CUDA graph the launch becomes a
// programmatic edge, hiding most of the per-kernel launch gap.
#define KL_PDL_ENTRY()                                             \
  do {                                                             \
    asm volatile("griddepcontrol.wait;" ::: "memory");             \
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); \
  } while (0)

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ---- typed load / store -----------------------------------------------------
__device__ __forceinline__ float ldf(const float* p) { return *p; }
__device__ __forceinline__ float ldf(const bf16* p) { return __bfloat162float(*p); }
__device__ __forceinline__ void stf(float* p, float v) { *p = v; }
__device__ __forceinline__ void stf(bf16* p, float v) { *p = __float2bfloat16(v); }
// value as stored in T (round-trip through the storage type)
__device__ __forceinline__ float rtf(float v, const float*) { return v; }
__device__ __forceinline__ float rtf(float v, const bf16*) { return __bfloat162float(__float2bfloat16(v)); }

// ---- activation table (tensor.py:431-440), accurate fp32 libm -------------
__device__ __forceinline__ float sigmoidf_(float x) {
  if (x >= 0.f) return 1.f / (1.f + expf(-x));
  float e = expf(x);
  return e / (1.f + e);
}

__device__ __forceinline__ float act_apply(int code, float x) {
  switch (code) {
    case KL_ACT_RELU: return x > 0.f ? x : 0.f;
    case KL_ACT_SILU: return x * sigmoidf_(x);
    case KL_ACT_TANH: return tanhf(x);
    case KL_ACT_SIGMOID: return sigmoidf_(x);
    case KL_ACT_EXP: return expf(x);
    case KL_ACT_SQRT: return sqrtf(x);
    case KL_ACT_LOG: return logf(x);
    default: return x;
  }
}

// dfn(x, y) of tensor.py:425-440, with y = act(x) recomputed.
__device__ __forceinline__ float act_deriv(int code, float x) {
  switch (code) {
    case KL_ACT_RELU: return x > 0.f ? 1.f : 0.f;
    case KL_ACT_SILU: {
      float s = sigmoidf_(x);
      return s * (1.f + x * (1.f - s));
    }
    case KL_ACT_TANH: {
      float y = tanhf(x);
      return 1.f - y * y;
    }
    case KL_ACT_SIGMOID: {
      float y = sigmoidf_(x);
      return y * (1.f - y);
    }
    case KL_ACT_EXP: return expf(x);
    case KL_ACT_SQRT: return 0.5f / sqrtf(x);
    case KL_ACT_LOG: return 1.f / x;
    default: return 1.f;
  }
}

// Epilogue parameters shared by the SIMT and tcgen05 GEMMs.
struct Epi {
  float alpha, beta;
  const float* bias;
  const int* row_limit;
  int aux_mode;
  int n_act, act_group;
  int act_codes[KL_MAX_ACT_GROUPS];
};

__device__ __forceinline__ int epi_code(const Epi& e, int n) {
  if (e.n_act == 0) return KL_ACT_IDENTITY;
  if (e.n_act == 1) return e.act_codes[0];
  return e.act_codes[(n / e.act_group) % e.n_act];
}

}  // namespace kl
