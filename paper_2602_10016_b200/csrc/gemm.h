// Internal GEMM descriptor + the shared epilogue (SIMT and tcgen05 paths).
#pragma once

#include "common.cuh"

namespace kl {

struct GemmDesc {
  int M, N, K;
  int nb1, nb2, red1, red2;
  int ab_dtype, c_dtype;
  const void* A;
  long long a_rs, a_cs, a_s1, a_s2;
  const void* B;
  long long b_rs, b_cs, b_s1, b_s2;
  void* C;
  long long c_rs, c_cs, c_s1, c_s2;
  const void* R;
  long long r_rs, r_cs, r_s1, r_s2;
  void* aux;
  float* ws;  // split-K scratch (fp32) or NULL
  long long ws_bytes;
};

// out = act(alpha*acc [* act'(aux)] + bias) [pre-act -> aux] + beta*C + R;
// rows at or beyond the per-batch row limit are written as exact zeros.
// With aux_mode == 2 the codes select the derivative and no forward
// activation is applied (dact epilogue of a dgrad GEMM).
template <typename TC>
__device__ __forceinline__ void epilogue_store(const Epi& e, TC* C, const TC* R, TC* X, long long off,
                                               long long roff, int m, int n, int lim, float acc) {
  if (m >= lim) {
    if (X && e.aux_mode == 1) stf(X + off, 0.f);
    stf(C + off, 0.f);
    return;
  }
  float v = e.alpha * acc;
  const int code = epi_code(e, n);
  if (e.aux_mode == 2) v *= act_deriv(code, ldf(X + off));
  if (e.bias) v += e.bias[n];
  if (e.aux_mode == 1) stf(X + off, v);
  if (e.aux_mode != 2) v = act_apply(code, v);
  if (e.beta != 0.f) v += e.beta * ldf(C + off);
  if (R) v += ldf(R + roff);
  stf(C + off, v);
}

int gemm_simt(const GemmDesc& g, const Epi& e, cudaStream_t s);
// Sums split-K partials ws[split][out batch][M][N] (fp32) and applies the
// full epilogue.
int splitk_reduce(const GemmDesc& g, const Epi& e, const float* ws, int splits, int n_out, cudaStream_t s);
// Returns KL_EUNSUPPORTED (without error text) when the shape/layout is not
// one the tcgen05 kernel takes; the caller then uses the SIMT kernel.
int gemm_tc(const GemmDesc& g, const Epi& e, cudaStream_t s);

}  // namespace kl
