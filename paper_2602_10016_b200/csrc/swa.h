// Internal sliding-window attention descriptor.
#pragma once

#include "common.cuh"

namespace kl {

struct SwaP {
  int B, T, H, d_h, w, causal, dtype;
  float scale;
  const int* lengths;
  const void* QKV;
  long long ld_qkv, bs_qkv;
  void* O;
  long long ld_o, bs_o;
  float* LSE;
  const void* dO;
  void* dQKV;
  float* Dbuf;
  unsigned long long* trace = nullptr;  // debug: CTA 0's pipeline clock stamps (KL_SWA_TRACE), dK / dV kernel
  int dq_rowdot = 0;  // dQ v3 kernel: form D = rowsum(dO * O) itself (O tiles by TMA) and write Dbuf
};

int swa_fwd_simt(const SwaP& p, cudaStream_t s);
int swa_bwd_simt(const SwaP& p, cudaStream_t s);
int swa_support(const SwaP& p, int* support, cudaStream_t s);
// tcgen05 path (bf16, d_h in {16,32,64,128}); KL_EUNSUPPORTED -> caller falls back.
int swa_fwd_tc(const SwaP& p, cudaStream_t s);
int swa_bwd_tc(const SwaP& p, cudaStream_t s);

}  // namespace kl
