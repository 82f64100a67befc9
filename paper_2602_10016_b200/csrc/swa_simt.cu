// Sliding-window multi-head attention, SIMT flash kernels (fp32 parity path
// and generic fallback).  Reference semantics: attention.py:69-129 with
// band_mask / _length_mask (attention.py:96-112) and masked_softmax_lastdim
// (tensor.py:485-505: fully-masked rows -> 0).  Out-of-band key tiles are
// never loaded: each 64-query tile visits keys [q0-w, q0+63+w] only.
#include "common.cuh"
#include "swa.h"

namespace kl {

namespace {

constexpr int TQ = 64;  // query / key tile

__device__ __forceinline__ bool key_ok(int qi, int kj, int len, int hi, int w, int causal) {
  if (qi >= len || kj > hi) return false;
  int dd = qi - kj;
  if (dd > w || -dd > w) return false;
  if (causal && kj > qi) return false;
  return true;
}

template <typename T, int DH>
__global__ void __launch_bounds__(256) swa_fwd_kernel(SwaP p) {
  KL_PDL_ENTRY();
  extern __shared__ float sm[];
  constexpr int LD = DH + 1;
  float* Qs = sm;
  float* Ks = Qs + TQ * LD;
  float* Vs = Ks + TQ * LD;
  float* Ps = Vs + TQ * LD;  // [TQ][TQ+1]
  const int b = blockIdx.z, h = blockIdx.y, q0 = blockIdx.x * TQ;
  const int len = p.lengths[b];
  const int tid = threadIdx.x, r = tid >> 2, sub = tid & 3;
  const T* qkv = (const T*)p.QKV + (long long)b * p.bs_qkv;
  const int HD = p.H * DH;
  for (int e = tid; e < TQ * DH; e += 256) {
    int rr = e / DH, c = e % DH, t = q0 + rr;
    Qs[rr * LD + c] = (t < len) ? ldf(qkv + (long long)t * p.ld_qkv + h * DH + c) : 0.f;
  }
  const int qi = q0 + r;
  float m_i = -INFINITY, l_i = 0.f;
  float o[DH / 4];
#pragma unroll
  for (int c = 0; c < DH / 4; ++c) o[c] = 0.f;
  const int lo = max(0, q0 - p.w);
  int hi = min(len - 1, q0 + TQ - 1 + p.w);
  if (p.causal) hi = min(hi, q0 + TQ - 1);
  for (int k0 = lo; k0 <= hi; k0 += TQ) {
    __syncthreads();
    for (int e = tid; e < TQ * DH; e += 256) {
      int rr = e / DH, c = e % DH, t = k0 + rr;
      bool v = t <= hi;
      Ks[rr * LD + c] = v ? ldf(qkv + (long long)t * p.ld_qkv + HD + h * DH + c) : 0.f;
      Vs[rr * LD + c] = v ? ldf(qkv + (long long)t * p.ld_qkv + 2 * HD + h * DH + c) : 0.f;
    }
    __syncthreads();
    float s[TQ / 4];
    float mloc = -INFINITY;
#pragma unroll
    for (int j = 0; j < TQ / 4; ++j) {
      const int kk = sub + 4 * j;
      float acc = 0.f;
#pragma unroll
      for (int c = 0; c < DH; ++c) acc = fmaf(Qs[r * LD + c], Ks[kk * LD + c], acc);
      bool ok = key_ok(qi, k0 + kk, len, hi, p.w, p.causal);
      s[j] = ok ? acc * p.scale : -INFINITY;
      mloc = fmaxf(mloc, s[j]);
    }
    mloc = fmaxf(mloc, __shfl_xor_sync(0xffffffffu, mloc, 1));
    mloc = fmaxf(mloc, __shfl_xor_sync(0xffffffffu, mloc, 2));
    const float m_new = fmaxf(m_i, mloc);
    float alpha = 1.f, lsum = 0.f;
    if (m_new != -INFINITY) alpha = (m_i == -INFINITY) ? 0.f : expf(m_i - m_new);
#pragma unroll
    for (int j = 0; j < TQ / 4; ++j) {
      float pj = (s[j] == -INFINITY) ? 0.f : expf(s[j] - m_new);
      Ps[r * (TQ + 1) + sub + 4 * j] = pj;
      lsum += pj;
    }
    lsum += __shfl_xor_sync(0xffffffffu, lsum, 1);
    lsum += __shfl_xor_sync(0xffffffffu, lsum, 2);
    l_i = l_i * alpha + lsum;
    m_i = m_new;
#pragma unroll
    for (int c = 0; c < DH / 4; ++c) o[c] *= alpha;
    __syncwarp();
    for (int kk = 0; kk < TQ; ++kk) {
      float pv = Ps[r * (TQ + 1) + kk];
#pragma unroll
      for (int c = 0; c < DH / 4; ++c) o[c] = fmaf(pv, Vs[kk * LD + sub + 4 * c], o[c]);
    }
  }
  if (qi < p.T) {
    T* O = (T*)p.O + (long long)b * p.bs_o + (long long)qi * p.ld_o + h * DH;
    const float inv = l_i > 0.f ? 1.f / l_i : 0.f;
#pragma unroll
    for (int c = 0; c < DH / 4; ++c) stf(O + sub + 4 * c, o[c] * inv);
    if (sub == 0) p.LSE[((long long)b * p.H + h) * p.T + qi] = l_i > 0.f ? m_i + logf(l_i) : INFINITY;
  }
}

template <typename T, int DH>
__global__ void swa_rowdot_kernel(SwaP p) {
  KL_PDL_ENTRY();
  // D[b,h,t] = sum_c dO * O (the softmax-VJP inner product, tensor.py:501-503)
  long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long total = (long long)p.B * p.H * p.T;
  if (idx >= total) return;
  int t = idx % p.T;
  int h = (idx / p.T) % p.H;
  int b = idx / ((long long)p.T * p.H);
  const T* o = (const T*)p.O + (long long)b * p.bs_o + (long long)t * p.ld_o + h * DH;
  const T* g = (const T*)p.dO + (long long)b * p.bs_o + (long long)t * p.ld_o + h * DH;
  float acc = 0.f;
#pragma unroll 8
  for (int c = 0; c < DH; ++c) acc = fmaf(ldf(o + c), ldf(g + c), acc);
  p.Dbuf[idx] = acc;
}

template <typename T, int DH>
__global__ void __launch_bounds__(256) swa_bwd_dkv_kernel(SwaP p) {
  KL_PDL_ENTRY();
  extern __shared__ float sm[];
  constexpr int LD = DH + 1;
  float* Ks = sm;
  float* Vs = Ks + TQ * LD;
  float* Qs = Vs + TQ * LD;
  float* Gs = Qs + TQ * LD;
  float* Ps = Gs + TQ * LD;     // [TQ][TQ+1]
  float* Ds = Ps + TQ * (TQ + 1);  // [TQ][TQ+1]
  float* lse = Ds + TQ * (TQ + 1);
  float* dd = lse + TQ;
  const int b = blockIdx.z, h = blockIdx.y, k0 = blockIdx.x * TQ;
  const int len = p.lengths[b];
  const int tid = threadIdx.x, r = tid >> 2, sub = tid & 3;
  const T* qkv = (const T*)p.QKV + (long long)b * p.bs_qkv;
  const T* dO = (const T*)p.dO + (long long)b * p.bs_o;
  const int HD = p.H * DH;
  const float* LSE = p.LSE + ((long long)b * p.H + h) * p.T;
  const float* Dv = p.Dbuf + ((long long)b * p.H + h) * p.T;
  for (int e = tid; e < TQ * DH; e += 256) {
    int rr = e / DH, c = e % DH, t = k0 + rr;
    bool v = t < len;
    Ks[rr * LD + c] = v ? ldf(qkv + (long long)t * p.ld_qkv + HD + h * DH + c) : 0.f;
    Vs[rr * LD + c] = v ? ldf(qkv + (long long)t * p.ld_qkv + 2 * HD + h * DH + c) : 0.f;
  }
  const int kj = k0 + r;
  float dk[DH / 4], dv[DH / 4];
#pragma unroll
  for (int c = 0; c < DH / 4; ++c) dk[c] = dv[c] = 0.f;
  int qlo = max(0, k0 - p.w);
  if (p.causal) qlo = max(qlo, k0);
  const int qhi = min(len - 1, k0 + TQ - 1 + p.w);
  for (int q0 = qlo; q0 <= qhi; q0 += TQ) {
    __syncthreads();
    for (int e = tid; e < TQ * DH; e += 256) {
      int rr = e / DH, c = e % DH, t = q0 + rr;
      bool v = t <= qhi;
      Qs[rr * LD + c] = v ? ldf(qkv + (long long)t * p.ld_qkv + h * DH + c) : 0.f;
      Gs[rr * LD + c] = v ? ldf(dO + (long long)t * p.ld_o + h * DH + c) : 0.f;
    }
    if (tid < TQ) {
      int t = q0 + tid;
      lse[tid] = t <= qhi ? LSE[t] : INFINITY;
      dd[tid] = t <= qhi ? Dv[t] : 0.f;
    }
    __syncthreads();
#pragma unroll 4
    for (int j = 0; j < TQ / 4; ++j) {
      const int qq = sub + 4 * j, qi = q0 + qq;
      // key j is visible to query i iff the forward mask admitted (i, j)
      const int fhi_q0 = (qi / TQ) * TQ;  // forward tile of query qi
      int fhi = min(len - 1, fhi_q0 + TQ - 1 + p.w);
      if (p.causal) fhi = min(fhi, fhi_q0 + TQ - 1);
      bool ok = (kj < len) && qi <= qhi && key_ok(qi, kj, len, fhi, p.w, p.causal);
      float pr = 0.f, ds = 0.f;
      if (ok) {
        float s = 0.f, dp = 0.f;
#pragma unroll
        for (int c = 0; c < DH; ++c) {
          s = fmaf(Ks[r * LD + c], Qs[qq * LD + c], s);
          dp = fmaf(Vs[r * LD + c], Gs[qq * LD + c], dp);
        }
        pr = expf(s * p.scale - lse[qq]);
        ds = pr * (dp - dd[qq]);
      }
      Ps[r * (TQ + 1) + qq] = pr;
      Ds[r * (TQ + 1) + qq] = ds;
    }
    __syncwarp();
    for (int qq = 0; qq < TQ; ++qq) {
      float pr = Ps[r * (TQ + 1) + qq], ds = Ds[r * (TQ + 1) + qq];
#pragma unroll
      for (int c = 0; c < DH / 4; ++c) {
        dv[c] = fmaf(pr, Gs[qq * LD + sub + 4 * c], dv[c]);
        dk[c] = fmaf(ds, Qs[qq * LD + sub + 4 * c], dk[c]);
      }
    }
  }
  if (kj < p.T) {
    T* out = (T*)p.dQKV + (long long)b * p.bs_qkv + (long long)kj * p.ld_qkv;
#pragma unroll
    for (int c = 0; c < DH / 4; ++c) {
      stf(out + HD + h * DH + sub + 4 * c, dk[c] * p.scale);
      stf(out + 2 * HD + h * DH + sub + 4 * c, dv[c]);
    }
  }
}

template <typename T, int DH>
__global__ void __launch_bounds__(256) swa_bwd_dq_kernel(SwaP p) {
  KL_PDL_ENTRY();
  extern __shared__ float sm[];
  constexpr int LD = DH + 1;
  float* Qs = sm;
  float* Gs = Qs + TQ * LD;
  float* Ks = Gs + TQ * LD;
  float* Vs = Ks + TQ * LD;
  float* Ds = Vs + TQ * LD;  // [TQ][TQ+1]
  const int b = blockIdx.z, h = blockIdx.y, q0 = blockIdx.x * TQ;
  const int len = p.lengths[b];
  const int tid = threadIdx.x, r = tid >> 2, sub = tid & 3;
  const T* qkv = (const T*)p.QKV + (long long)b * p.bs_qkv;
  const T* dO = (const T*)p.dO + (long long)b * p.bs_o;
  const int HD = p.H * DH;
  for (int e = tid; e < TQ * DH; e += 256) {
    int rr = e / DH, c = e % DH, t = q0 + rr;
    bool v = t < len;
    Qs[rr * LD + c] = v ? ldf(qkv + (long long)t * p.ld_qkv + h * DH + c) : 0.f;
    Gs[rr * LD + c] = v ? ldf(dO + (long long)t * p.ld_o + h * DH + c) : 0.f;
  }
  const int qi = q0 + r;
  const float lse_r = qi < len ? p.LSE[((long long)b * p.H + h) * p.T + qi] : INFINITY;
  const float d_r = qi < len ? p.Dbuf[((long long)b * p.H + h) * p.T + qi] : 0.f;
  float dq[DH / 4];
#pragma unroll
  for (int c = 0; c < DH / 4; ++c) dq[c] = 0.f;
  const int lo = max(0, q0 - p.w);
  int hi = min(len - 1, q0 + TQ - 1 + p.w);
  if (p.causal) hi = min(hi, q0 + TQ - 1);
  for (int k0 = lo; k0 <= hi; k0 += TQ) {
    __syncthreads();
    for (int e = tid; e < TQ * DH; e += 256) {
      int rr = e / DH, c = e % DH, t = k0 + rr;
      bool v = t <= hi;
      Ks[rr * LD + c] = v ? ldf(qkv + (long long)t * p.ld_qkv + HD + h * DH + c) : 0.f;
      Vs[rr * LD + c] = v ? ldf(qkv + (long long)t * p.ld_qkv + 2 * HD + h * DH + c) : 0.f;
    }
    __syncthreads();
#pragma unroll 4
    for (int j = 0; j < TQ / 4; ++j) {
      const int kk = sub + 4 * j;
      float ds = 0.f;
      if (key_ok(qi, k0 + kk, len, hi, p.w, p.causal)) {
        float s = 0.f, dp = 0.f;
#pragma unroll
        for (int c = 0; c < DH; ++c) {
          s = fmaf(Qs[r * LD + c], Ks[kk * LD + c], s);
          dp = fmaf(Gs[r * LD + c], Vs[kk * LD + c], dp);
        }
        float pr = expf(s * p.scale - lse_r);
        ds = pr * (dp - d_r);
      }
      Ds[r * (TQ + 1) + kk] = ds;
    }
    __syncwarp();
    for (int kk = 0; kk < TQ; ++kk) {
      float ds = Ds[r * (TQ + 1) + kk];
#pragma unroll
      for (int c = 0; c < DH / 4; ++c) dq[c] = fmaf(ds, Ks[kk * LD + sub + 4 * c], dq[c]);
    }
  }
  if (qi < p.T) {
    T* out = (T*)p.dQKV + (long long)b * p.bs_qkv + (long long)qi * p.ld_qkv + h * DH;
#pragma unroll
    for (int c = 0; c < DH / 4; ++c) stf(out + sub + 4 * c, dq[c] * p.scale);
  }
}

__global__ void swa_support_kernel(SwaP p, int* support) {
  KL_PDL_ENTRY();
  long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)p.B * p.T) return;
  const int b = idx / p.T, qi = idx % p.T;
  const int len = p.lengths[b];
  const int q0 = (qi / TQ) * TQ;
  const int lo = max(0, q0 - p.w);
  int hi = min(len - 1, q0 + TQ - 1 + p.w);
  if (p.causal) hi = min(hi, q0 + TQ - 1);
  int cnt = 0;
  for (int k0 = lo; k0 <= hi; k0 += TQ)
    for (int kk = 0; kk < TQ; ++kk) cnt += key_ok(qi, k0 + kk, len, hi, p.w, p.causal) ? 1 : 0;
  support[idx] = cnt;
}

template <typename T, int DH>
int launch_fwd(const SwaP& p, cudaStream_t s) {
  const size_t smem = (3 * TQ * (DH + 1) + TQ * (TQ + 1)) * sizeof(float);
  cudaFuncSetAttribute(swa_fwd_kernel<T, DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid((p.T + TQ - 1) / TQ, p.H, p.B);
  launch_k(swa_fwd_kernel<T, DH>, grid, 256, smem, s, p);
  count_launch();
  count_path(KL_PATH_SWA_FWD_SIMT);
  return launch_check("swa_fwd_simt");
}

template <typename T, int DH>
int launch_bwd(const SwaP& p, cudaStream_t s) {
  long long total = (long long)p.B * p.H * p.T;
  launch_k(swa_rowdot_kernel<T, DH>, (unsigned)((total + 255) / 256), 256, 0, s, p);
  const size_t smem1 = (4 * TQ * (DH + 1) + 2 * TQ * (TQ + 1) + 2 * TQ) * sizeof(float);
  cudaFuncSetAttribute(swa_bwd_dkv_kernel<T, DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1);
  dim3 grid((p.T + TQ - 1) / TQ, p.H, p.B);
  launch_k(swa_bwd_dkv_kernel<T, DH>, grid, 256, smem1, s, p);
  const size_t smem2 = (4 * TQ * (DH + 1) + TQ * (TQ + 1)) * sizeof(float);
  cudaFuncSetAttribute(swa_bwd_dq_kernel<T, DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
  launch_k(swa_bwd_dq_kernel<T, DH>, grid, 256, smem2, s, p);
  count_launch(3);
  count_path(KL_PATH_SWA_BWD_SIMT);
  return launch_check("swa_bwd_simt");
}

template <typename T>
int fwd_dh(const SwaP& p, cudaStream_t s) {
  switch (p.d_h) {
    case 4: return launch_fwd<T, 4>(p, s);
    case 8: return launch_fwd<T, 8>(p, s);
    case 16: return launch_fwd<T, 16>(p, s);
    case 32: return launch_fwd<T, 32>(p, s);
    case 64: return launch_fwd<T, 64>(p, s);
    case 128: return launch_fwd<T, 128>(p, s);
  }
  set_error("kl_swa_fwd: head dim %d unsupported (4/8/16/32/64/128)", p.d_h);
  return KL_EUNSUPPORTED;
}

template <typename T>
int bwd_dh(const SwaP& p, cudaStream_t s) {
  switch (p.d_h) {
    case 4: return launch_bwd<T, 4>(p, s);
    case 8: return launch_bwd<T, 8>(p, s);
    case 16: return launch_bwd<T, 16>(p, s);
    case 32: return launch_bwd<T, 32>(p, s);
    case 64: return launch_bwd<T, 64>(p, s);
    case 128: return launch_bwd<T, 128>(p, s);
  }
  set_error("kl_swa_bwd: head dim %d unsupported (4/8/16/32/64/128)", p.d_h);
  return KL_EUNSUPPORTED;
}

}  // namespace

int swa_fwd_simt(const SwaP& p, cudaStream_t s) {
  return p.dtype == KL_F32 ? fwd_dh<float>(p, s) : fwd_dh<bf16>(p, s);
}

int swa_bwd_simt(const SwaP& p, cudaStream_t s) {
  return p.dtype == KL_F32 ? bwd_dh<float>(p, s) : bwd_dh<bf16>(p, s);
}

int swa_support(const SwaP& p, int* support, cudaStream_t s) {
  long long total = (long long)p.B * p.T;
  launch_k(swa_support_kernel, (unsigned)((total + 255) / 256), 256, 0, s, p, support);
  count_launch();
  return launch_check("swa_support");
}

}  // namespace kl

namespace kl {
// D[b,h,t] = rowsum(dO * O) for the tcgen05 backward kernels.
// Warp per (b, t) row of a bf16 (B, T, H*64) pair: each lane owns 8 contiguous
// elements (16-byte loads, the warp reads the row's 512 B... H*128 B), the 8 lanes
// of a head reduce with shuffles.  Coalesced; one pass over O and dO.
__global__ void swa_rowdot_bf16_h64(SwaP p) {
  KL_PDL_ENTRY();
  const long long row = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= (long long)p.B * p.T) return;
  const int lane = threadIdx.x & 31;
  const int b = row / p.T, t = row % p.T;
  const bf16* o = (const bf16*)p.O + (long long)b * p.bs_o + (long long)t * p.ld_o;
  const bf16* g = (const bf16*)p.dO + (long long)b * p.bs_o + (long long)t * p.ld_o;
  const int HD = p.H * 64;
  for (int c0 = lane * 8; c0 < HD; c0 += 256) {
    const uint4 a = *reinterpret_cast<const uint4*>(o + c0);
    const uint4 d = *reinterpret_cast<const uint4*>(g + c0);
    const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
    const __nv_bfloat162* d2 = reinterpret_cast<const __nv_bfloat162*>(&d);
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 x = __bfloat1622float2(a2[i]), y = __bfloat1622float2(d2[i]);
      acc = fmaf(x.x, y.x, fmaf(x.y, y.y, acc));
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    acc += __shfl_xor_sync(0xffffffffu, acc, 4);
    if ((lane & 7) == 0) {
      const int h = c0 / 64;
      p.Dbuf[((long long)b * p.H + h) * p.T + t] = acc;
    }
  }
}

int swa_rowdot(const SwaP& p, cudaStream_t s) {
  long long total = (long long)p.B * p.H * p.T;
  unsigned g = (unsigned)((total + 255) / 256);
  const bool vec = p.dtype == KL_BF16 && p.d_h == 64 && p.ld_o % 8 == 0 && p.bs_o % 8 == 0 &&
                   ((uintptr_t)p.O & 15) == 0 && ((uintptr_t)p.dO & 15) == 0;
  if (vec) {
    const long long rows = (long long)p.B * p.T;
    launch_k(swa_rowdot_bf16_h64, (unsigned)((rows + 7) / 8), 256, 0, s, p);
  } else if (p.dtype == KL_BF16 && p.d_h == 64) {
    launch_k(swa_rowdot_kernel<bf16, 64>, g, 256, 0, s, p);
  } else if (p.dtype == KL_F32 && p.d_h == 64) {
    launch_k(swa_rowdot_kernel<float, 64>, g, 256, 0, s, p);
  } else {
    set_error("swa_rowdot: unsupported head dim %d", p.d_h);
    return KL_EUNSUPPORTED;
  }
  count_launch();
  return launch_check("swa_rowdot");
}
}  // namespace kl
