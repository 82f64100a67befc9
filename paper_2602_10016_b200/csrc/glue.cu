// Small-dimension glue kernels of the Kunlun layer (HBM / latency bound):
// column softmax for HSP/PMA pooling, RMSNorm, recent rows, Wukong
// pairwise-dot (gram + triu), gated expert residual, BCE, casts, activation,
// non-finite scan.  Each cites the reference op it reproduces.
#include <algorithm>

#include "common.cuh"

namespace kl {

int tc_num_sms();  // cached cudaDevAttrMultiProcessorCount (gemm_tc.cu)

namespace {

// ---------------------------------------------------------------------------
// Column softmax over rows t < len (queries are columns):
// masked_softmax_lastdim (tensor.py:485-505) applied to the transposed HSP/PMA
// score block of multi_head_attention (attention.py:89-91).
// Block = 32 columns x 8 row groups; each thread keeps CS_U independent
// online (max, sum) pairs so CS_U row loads are in flight at once (the kernels
// are HBM/L2 bound: one stats pass + one write pass over the score block).
constexpr int CS_U = 8;

template <typename TI, typename TO>
__global__ void __launch_bounds__(256) colsoftmax_fwd_kernel(kl_colsoftmax_args a) {
  KL_PDL_ENTRY();
  __shared__ float redm[8][33], reds[8][33];
  const int b = blockIdx.y;
  const int cl = threadIdx.x & 31, rg = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + cl;
  const int len = a.lengths[b];
  const TI* X = (const TI*)a.X + (long long)b * a.x_bs + c;
  TO* P = (TO*)a.P + (long long)b * a.p_bs + c;
  float m[CS_U], sm[CS_U];
#pragma unroll
  for (int u = 0; u < CS_U; ++u) {
    m[u] = -INFINITY;
    sm[u] = 0.f;
  }
  if (c < a.C) {
    for (int t0 = rg; t0 < len; t0 += 8 * CS_U) {
      float v[CS_U];
#pragma unroll
      for (int u = 0; u < CS_U; ++u) {
        const int t = t0 + 8 * u;
        v[u] = t < len ? ldf(X + (long long)t * a.x_rs) : -INFINITY;
      }
#pragma unroll
      for (int u = 0; u < CS_U; ++u) {
        if (v[u] == -INFINITY) continue;
        const float mn = fmaxf(m[u], v[u]);
        sm[u] = sm[u] * __expf(m[u] - mn) + __expf(v[u] - mn);
        m[u] = mn;
      }
    }
  }
  float mt = m[0];
#pragma unroll
  for (int u = 1; u < CS_U; ++u) mt = fmaxf(mt, m[u]);
  float st = 0.f;
#pragma unroll
  for (int u = 0; u < CS_U; ++u) st += m[u] == -INFINITY ? 0.f : sm[u] * __expf(m[u] - mt);
  redm[rg][cl] = mt;
  reds[rg][cl] = st;
  __syncthreads();
  float mx = redm[0][cl];
#pragma unroll
  for (int i = 1; i < 8; ++i) mx = fmaxf(mx, redm[i][cl]);
  float ssum = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) ssum += redm[i][cl] == -INFINITY ? 0.f : reds[i][cl] * __expf(redm[i][cl] - mx);
  if (c >= a.C) return;
  const float inv = ssum > 0.f ? 1.f / ssum : 0.f;
  for (int t0 = rg; t0 < a.T; t0 += 8 * CS_U) {
    float v[CS_U];
#pragma unroll
    for (int u = 0; u < CS_U; ++u) {
      const int t = t0 + 8 * u;
      v[u] = t < len ? ldf(X + (long long)t * a.x_rs) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < CS_U; ++u) {
      const int t = t0 + 8 * u;
      if (t < a.T) stf(P + (long long)t * a.p_rs, t < len ? expf(v[u] - mx) * inv : 0.f);
    }
  }
  if (rg == 0 && a.LSE) a.LSE[(long long)b * a.C + c] = len > 0 ? mx + logf(ssum) : INFINITY;
}

// dX = P * (dP - sum_t P dP)   (tensor.py:501-503); P in TP, dP in TG, dX in TO.
// RECOMP: P = exp(X - LSE[c]) recomputed in fp32 from the fp32 scores X and
// the forward's log-sum-exp (no bf16 rounding of P in the score gradient).
template <typename TP, typename TG, typename TO, bool RECOMP = false>
__global__ void __launch_bounds__(256) colsoftmax_bwd_kernel(kl_colsoftmax_args a) {
  KL_PDL_ENTRY();
  __shared__ float red[8][33];
  const int b = blockIdx.y;
  const int cl = threadIdx.x & 31, rg = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + cl;
  const int len = a.lengths[b];
  const TP* P = RECOMP ? (const TP*)a.X + (long long)b * a.x_bs + c : (const TP*)a.P + (long long)b * a.p_bs + c;
  const long long p_rs = RECOMP ? a.x_rs : a.p_rs;
  const float lse = (RECOMP && c < a.C && len > 0) ? a.LSE[(long long)b * a.C + c] : 0.f;
  auto ldp = [&](long long t) { return RECOMP ? expf(ldf(P + t * p_rs) - lse) : ldf(P + t * p_rs); };
  const TG* G = (const TG*)a.dP + (long long)b * a.dp_bs + c;
  TO* D = (TO*)a.dX + (long long)b * a.dx_bs + c;
  TO* L = a.dX_lo ? (TO*)a.dX_lo + (long long)b * a.dx_bs + c : nullptr;
  float acc[CS_U];
#pragma unroll
  for (int u = 0; u < CS_U; ++u) acc[u] = 0.f;
  if (c < a.C && !a.Dcol)
    for (int t0 = rg; t0 < len; t0 += 8 * CS_U) {
#pragma unroll
      for (int u = 0; u < CS_U; ++u) {
        const int t = t0 + 8 * u;
        if (t < len) acc[u] += ldp(t) * ldf(G + (long long)t * a.dp_rs);
      }
    }
  float at = 0.f;
#pragma unroll
  for (int u = 0; u < CS_U; ++u) at += acc[u];
  red[rg][cl] = at;
  __syncthreads();
  float dsum = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) dsum += red[i][cl];
  if (c >= a.C) return;
  if (a.Dcol) dsum = a.Dcol[(long long)b * a.C + c];
  for (int t0 = rg; t0 < a.T; t0 += 8 * CS_U) {
    float pv[CS_U], gv[CS_U];
#pragma unroll
    for (int u = 0; u < CS_U; ++u) {
      const int t = t0 + 8 * u;
      pv[u] = t < len ? ldp(t) : 0.f;
      gv[u] = t < len ? ldf(G + (long long)t * a.dp_rs) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < CS_U; ++u) {
      const int t = t0 + 8 * u;
      if (t >= a.T) continue;
      const float v = t < len ? pv[u] * (gv[u] - dsum) : 0.f;
      stf(D + (long long)t * a.dx_rs, v);
      if (L) {
        // bf16 residual of the rounded value: hi + lo carries ~16 mantissa bits
        // into the cancellation-heavy reduction dQ = sum_t dX S (seqsum VJP)
        stf(L + (long long)t * a.dx_rs, v - rtf(v, D));
      }
    }
  }
}

// ---------------------------------------------------------------------------
__device__ float block_sum(float v, float* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  float t = 0.f;
  const int nw = blockDim.x >> 5;
  for (int i = 0; i < nw; ++i) t += sh[i];
  return t;
}

__device__ double block_sum_d(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  const int nw = blockDim.x >> 5;
  for (int i = 0; i < nw; ++i) t += sh[i];
  return t;
}

// rms_norm (tensor.py:552-556): one block per row.
__global__ void rmsnorm_fwd_kernel(int d, float eps, const float* x, const float* gain, float* y, long long x_bs,
                                   long long g_bs, long long y_bs) {
  KL_PDL_ENTRY();
  x += blockIdx.y * x_bs;
  gain += blockIdx.y * g_bs;
  y += blockIdx.y * y_bs;
  __shared__ float sh[32];
  const float* xr = x + (long long)blockIdx.x * d;
  float ss = 0.f;
  for (int c = threadIdx.x; c < d; c += blockDim.x) ss += xr[c] * xr[c];
  ss = block_sum(ss, sh);
  const float s = 1.f / sqrtf(ss / d + eps);
  for (int c = threadIdx.x; c < d; c += blockDim.x) y[(long long)blockIdx.x * d + c] = xr[c] * s * gain[c];
}

// Single block: dx = s*gg - s^3/d * x * sum(gg*x), gg = dy*gain; dgain = sum_rows dy*x*s.
// Phase 1: one warp per row computes s and k = s^3/d * sum(gg*x) into smem;
// phase 2: one thread per column writes dx for every row and accumulates
// dgain in fp64.
__global__ void __launch_bounds__(256) rmsnorm_bwd_kernel(int rows, int d, float eps, const float* x,
                                                         const float* gain, const float* dy, float* dx,
                                                         float* dgain, long long x_bs, long long g_bs,
                                                         long long dy_bs, long long dx_bs, long long dg_bs,
                                                         int acc) {
  KL_PDL_ENTRY();
  x += blockIdx.x * x_bs;
  gain += blockIdx.x * g_bs;
  dy += blockIdx.x * dy_bs;
  dx += blockIdx.x * dx_bs;
  dgain += blockIdx.x * dg_bs;
  extern __shared__ float rs[];  // s[rows], k[rows]
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int r = w; r < rows; r += blockDim.x >> 5) {
    const float* xr = x + (long long)r * d;
    const float* gr = dy + (long long)r * d;
    float ss = 0.f, gx = 0.f;
    for (int c = l; c < d; c += 32) {
      const float xv = xr[c];
      ss += xv * xv;
      gx += gr[c] * gain[c] * xv;
    }
    for (int o = 16; o > 0; o >>= 1) {
      ss += __shfl_xor_sync(0xffffffffu, ss, o);
      gx += __shfl_xor_sync(0xffffffffu, gx, o);
    }
    if (l == 0) {
      const float sv = 1.f / sqrtf(ss / d + eps);
      rs[r] = sv;
      rs[rows + r] = sv * sv * sv / d * gx;
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    double dg = 0.0;
    const float gc = gain[c];
    for (int r = 0; r < rows; ++r) {
      const float xv = x[(long long)r * d + c], gv = dy[(long long)r * d + c];
      const float v = rs[r] * gv * gc - rs[rows + r] * xv;
      dx[(long long)r * d + c] = acc ? dx[(long long)r * d + c] + v : v;
      dg += (double)gv * (double)xv * (double)rs[r];
    }
    dgain[c] = acc ? dgain[c] + (float)dg : (float)dg;
  }
}

// ---------------------------------------------------------------------------
// recent_rows (seqsum.py:186-196)
template <typename T>
__global__ void recent_fwd_kernel(int B, int T_, int d, int n, const T* S, long long s_bs, const int* lengths,
                                  T* out, long long o_bs) {
  KL_PDL_ENTRY();
  long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)B * n * d) return;
  int c = idx % d, r = (idx / d) % n, b = idx / ((long long)d * n);
  int t = lengths[b] - n + r;
  float v = t >= 0 ? ldf(S + (long long)b * s_bs + (long long)t * d + c) : 0.f;
  stf(out + (long long)b * o_bs + (long long)r * d + c, v);
}

template <typename T>
__global__ void recent_bwd_kernel(int B, int T_, int d, int n, const T* dout, long long o_bs, const int* lengths,
                                  T* dS, long long s_bs) {
  KL_PDL_ENTRY();
  long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)B * n * d) return;
  int c = idx % d, r = (idx / d) % n, b = idx / ((long long)d * n);
  int t = lengths[b] - n + r;
  if (t < 0) return;
  T* p = dS + (long long)b * s_bs + (long long)t * d + c;
  stf(p, ldf(p) + ldf(dout + (long long)b * o_bs + (long long)r * d + c));
}

// ---------------------------------------------------------------------------
// triu_flatten(x x^T) (interaction.py:63-76, 117): np.triu_indices row-major.
__device__ __forceinline__ int triu_index(int r, int c, int n) { return r * n - r * (r - 1) / 2 + (c - r); }

// One block per sample: x[b] (n x d) staged in smem as fp32 (rows padded by 4
// floats); one warp per pair (lanes split the d-length dot product).  With
// VEC the rows are read as 16-byte vectors, all of a thread's loads issued
// before any smem store (the scalar staging loop serialised one global-load
// latency per element).
template <typename T>
__device__ __forceinline__ void ld8(const T* p, float* o);
template <>
__device__ __forceinline__ void ld8<float>(const float* p, float* o) {
  float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
  o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w; o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
}
template <>
__device__ __forceinline__ void ld8<bf16>(const bf16* p, float* o) {
  uint4 u = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __bfloat1622float2(h[i]);
    o[2 * i] = f.x;
    o[2 * i + 1] = f.y;
  }
}
template <typename T>
__device__ __forceinline__ void st8(T* p, const float* v);
template <>
__device__ __forceinline__ void st8<float>(float* p, const float* v) {
  *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  *reinterpret_cast<float4*>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
}
template <>
__device__ __forceinline__ void st8<bf16>(bf16* p, const float* v) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
  *reinterpret_cast<uint4*>(p) = u;
}

// stage x[b] (n x d, row stride x_rs) into xs (row stride ld = d + 4) as fp32
template <typename T, bool VEC>
__device__ __forceinline__ void stage_rows(const T* xb, long long x_rs, int n, int d, float* xs, int ld) {
  if constexpr (VEC) {
    const int dv = d >> 3, nv = n * dv;
    for (int i0 = threadIdx.x; i0 < nv; i0 += 4 * blockDim.x) {
      float v[4][8];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * blockDim.x;
        if (i < nv) ld8(xb + (long long)(i / dv) * x_rs + (i % dv) * 8, v[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * blockDim.x;
        if (i < nv) {
          float* q = xs + (i / dv) * ld + (i % dv) * 8;
          *reinterpret_cast<float4*>(q) = make_float4(v[u][0], v[u][1], v[u][2], v[u][3]);
          *reinterpret_cast<float4*>(q + 4) = make_float4(v[u][4], v[u][5], v[u][6], v[u][7]);
        }
      }
    }
  } else {
    for (int i = threadIdx.x; i < n * d; i += blockDim.x) xs[(i / d) * ld + i % d] = ldf(xb + (long long)(i / d) * x_rs + i % d);
  }
}

template <typename T, bool VEC>
__global__ void __launch_bounds__(256) gram_triu_fwd_kernel(int n, int d, const T* x, long long x_rs,
                                                           long long x_bs, T* tri, long long t_bs) {
  KL_PDL_ENTRY();
  extern __shared__ float xs[];
  const int b = blockIdx.x, ld = d + 4;
  stage_rows<T, VEC>(x + (long long)b * x_bs, x_rs, n, d, xs, ld);
  __syncthreads();
  const int np_ = n * (n + 1) / 2;
  // blockIdx.y splits the pairs: more CTAs per sample, shorter warp chains
  const int l = threadIdx.x & 31, nw = (blockDim.x >> 5) * gridDim.y;
  const int w = blockIdx.y * (blockDim.x >> 5) + (threadIdx.x >> 5);
  int r = 0, rbase = 0;  // pair p = rbase + (c - r) for row r
  for (int p = w; p < np_; p += nw) {
    while (p >= rbase + (n - r)) {
      rbase += n - r;
      ++r;
    }
    const int c = r + (p - rbase);
    const float* xr = xs + r * ld;
    const float* xc = xs + c * ld;
    float acc = 0.f;
    if (VEC) {
      for (int k = 4 * l; k < d; k += 128) {
        const float4 a = *reinterpret_cast<const float4*>(xr + k), bb = *reinterpret_cast<const float4*>(xc + k);
        acc = fmaf(a.x, bb.x, fmaf(a.y, bb.y, fmaf(a.z, bb.z, fmaf(a.w, bb.w, acc))));
      }
    } else {
      for (int k = l; k < d; k += 32) acc = fmaf(xr[k], xc[k], acc);
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (l == 0) stf(tri + (long long)b * t_bs + p, acc);
  }
  // zero padding columns [np, t_bs) of a contiguous (B, t_bs) tri
  if (blockIdx.y == 0)
    for (int p = np_ + threadIdx.x; p < t_bs; p += blockDim.x) stf(tri + (long long)b * t_bs + p, 0.f);
}

// dx[b, r, k] += sum_j W[r][j] x[b, j, k], W symmetric from dtri (diagonal x2).
// VEC: thread = (row, 8 columns); the dx read-modify-write is one 16-byte
// vector each way.
template <typename T, bool VEC>
__global__ void __launch_bounds__(256) gram_triu_bwd_kernel(int n, int d, const T* x, long long x_rs,
                                                           long long x_bs, const T* dtri, long long t_bs, T* dx,
                                                           long long dx_rs, long long dx_bs) {
  KL_PDL_ENTRY();
  extern __shared__ float sm[];
  const int ld = d + 4;
  float* xs = sm;           // n x ld
  float* W = sm + n * ld;   // n x n
  const int b = blockIdx.x;
  const T* db = dtri + (long long)b * t_bs;
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) {
    const int r = i / n, j = i % n, lo = min(r, j), hi = max(r, j);
    W[i] = ldf(db + triu_index(lo, hi, n)) * (r == j ? 2.f : 1.f);
  }
  stage_rows<T, VEC>(x + (long long)b * x_bs, x_rs, n, d, xs, ld);
  __syncthreads();
  T* dxb = dx + (long long)b * dx_bs;
  if constexpr (VEC) {
    const int dv = d >> 3;  // blockIdx.y splits the (row, 8-column) items
    for (int i = blockIdx.y * blockDim.x + threadIdx.x; i < n * dv; i += blockDim.x * gridDim.y) {
      const int r = i / dv, k = (i % dv) * 8;
      T* p = dxb + (long long)r * dx_rs + k;
      float acc[8];
      ld8(p, acc);
      const float* wr = W + r * n;
      for (int j = 0; j < n; ++j) {
        const float wj = wr[j];
        const float4 a = *reinterpret_cast<const float4*>(xs + j * ld + k);
        const float4 c = *reinterpret_cast<const float4*>(xs + j * ld + k + 4);
        acc[0] = fmaf(wj, a.x, acc[0]); acc[1] = fmaf(wj, a.y, acc[1]);
        acc[2] = fmaf(wj, a.z, acc[2]); acc[3] = fmaf(wj, a.w, acc[3]);
        acc[4] = fmaf(wj, c.x, acc[4]); acc[5] = fmaf(wj, c.y, acc[5]);
        acc[6] = fmaf(wj, c.z, acc[6]); acc[7] = fmaf(wj, c.w, acc[7]);
      }
      st8(p, acc);
    }
  } else {
    for (int i = blockIdx.y * blockDim.x + threadIdx.x; i < n * d; i += blockDim.x * gridDim.y) {
      const int r = i / d, k = i % d;
      float acc = 0.f;
      for (int j = 0; j < n; ++j) acc = fmaf(W[r * n + j], xs[j * ld + k], acc);
      T* p = dxb + (long long)r * dx_rs + k;
      stf(p, ldf(p) + acc);
    }
  }
}

// ---------------------------------------------------------------------------
// wukong_expert residual: x + gate_deep*deep + gate_dot*dot (interaction.py:121)
template <typename T>
__global__ void gated_fwd_kernel(int rows, int d, const T* x, long long x_rs, const T* deep, const T* dot,
                                 const float* gd, const float* gt, T* out, long long o_rs) {
  KL_PDL_ENTRY();
  long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)rows * d) return;
  int c = idx % d;
  long long r = idx / d;
  float v = ldf(x + r * x_rs + c) + gd[0] * ldf(deep + idx) + gt[0] * ldf(dot + idx);
  stf(out + r * o_rs + c, v);
}

template <typename T>
__global__ void __launch_bounds__(256) gated_bwd_kernel(int rows, int d, const T* g, long long g_rs, const T* deep,
                                                        const T* dot, const float* gd, const float* gt, T* ddeep,
                                                        T* ddot, double* partial) {
  KL_PDL_ENTRY();
  __shared__ double shd[32];
  double a = 0.0, b = 0.0;
  const long long total = (long long)rows * d;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    int c = idx % d;
    long long r = idx / d;
    float gv = ldf(g + r * g_rs + c);
    a += (double)gv * (double)ldf(deep + idx);
    b += (double)gv * (double)ldf(dot + idx);
    stf(ddeep + idx, gv * gd[0]);
    stf(ddot + idx, gv * gt[0]);
  }
  a = block_sum_d(a, shd);
  b = block_sum_d(b, shd);
  if (threadIdx.x == 0) {
    partial[2 * blockIdx.x] = a;
    partial[2 * blockIdx.x + 1] = b;
  }
}

__global__ void reduce_pairs_kernel(int nblk, const double* partial, float* o0, float* o1) {
  KL_PDL_ENTRY();
  __shared__ double sh[32];
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) {
    a += partial[2 * i];
    b += partial[2 * i + 1];
  }
  a = block_sum_d(a, sh);
  b = block_sum_d(b, sh);
  if (threadIdx.x == 0) {  // accumulate into the gate gradients
    o0[0] += (float)a;
    o1[0] += (float)b;
  }
}

// ---------------------------------------------------------------------------
// bce_with_logits (tensor.py:535-549)
__global__ void bce_kernel(int n, const float* z, const float* y, float* loss, float* dz) {
  KL_PDL_ENTRY();
  __shared__ float sh[32];
  float acc = 0.f;
  const float inv = 1.f / (float)max(n, 1);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    float zi = z[i], yi = y[i];
    acc += fmaxf(zi, 0.f) - yi * zi + log1pf(expf(-fabsf(zi)));
    dz[i] = (sigmoidf_(zi) - yi) * inv;
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) loss[0] = acc * inv;
}

// Normalized entropy (PAPER.md:438-446 Eq. A1-A2): one block,
// fp64 accumulation.  kind 0: p = probabilities clipped to [1e-12, 1 - 1e-12];
// kind 1: p = logits, log(sigmoid) evaluated stably.  out = {cross_entropy,
// background_entropy, ne, ctr}; a degenerate background (ctr 0 or 1) gives ne = NaN.
__global__ void ne_kernel(int n, int kind, const float* p, const float* y, double* out) {
  KL_PDL_ENTRY();
  __shared__ double sh[32];
  double ce = 0.0, ys = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double yi = y[i], pi = p[i];
    double lp, lq;  // log(p), log(1 - p)
    if (kind == 1) {
      lp = -log1p(exp(-fabs(pi))) + fmin(pi, 0.0);
      lq = -log1p(exp(-fabs(pi))) - fmax(pi, 0.0);
    } else {
      const double c = fmin(fmax(pi, 1e-12), 1.0 - 1e-12);
      lp = log(c);
      lq = log1p(-c);
    }
    ce -= yi * lp + (1.0 - yi) * lq;
    ys += yi;
  }
  ce = block_sum_d(ce, sh);
  ys = block_sum_d(ys, sh);
  if (threadIdx.x == 0) {
    const double inv = 1.0 / (double)max(n, 1), ctr = ys * inv;
    const double h = (ctr > 0.0 && ctr < 1.0) ? -ctr * log(ctr) - (1.0 - ctr) * log1p(-ctr) : 0.0;
    out[0] = ce * inv;
    out[1] = h;
    out[2] = h > 0.0 ? ce * inv / h : nan("");
    out[3] = ctr;
  }
}

// ROTE (preproc.py:187-199; rotate_pairs tensor.py:508-532): thread = one
// (sample, row, column pair), grid-stride; angles in fp64, reduced to
// [-1/2, 1/2] turns, then fp32 sincospi (no Payne-Hanek path, no fp64 divide).
template <typename T>
__global__ void rote_kernel(kl_rote_args a) {
  KL_PDL_ENTRY();
  const int half = a.d >> 1;
  const long long total = (long long)a.B * a.T * half;
  const T* x = (const T*)a.x;
  T* y = (T*)a.y;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx % half);
    const long long bt = idx / half;
    const int t = (int)(bt % a.T), b = (int)(bt / a.T);
    const T* xp = x + (long long)b * a.x_bs + (long long)t * a.x_rs + 2 * i;
    T* yp = y + (long long)b * a.y_bs + (long long)t * a.y_rs + 2 * i;
    const float x0 = ldf(xp), x1 = ldf(xp + 1);
    const int len = a.lengths ? min(max(a.lengths[b], 0), a.T) : a.T;  // clamped: never read past the sample
    if (t >= len) {
      stf(yp, x0);
      stf(yp + 1, x1);
      continue;
    }
    double ang = (double)t * a.pos_freqs[i];
    if (a.timestamps) {
      const double* ts = a.timestamps + (long long)b * a.ts_bs;
      const double gap = a.gap_mode == 0 ? (t > 0 ? ts[t] - ts[t - 1] : 0.0) : ts[len - 1] - ts[t];
      ang += log1p(fmax(gap, 0.0) / a.tau_scale) * a.temp_freqs[i];
    }
    double u = ang * 0.15915494309189533577;  // turns
    u -= rint(u);
    float sn, cs;
    sincospif((float)(2.0 * u), &sn, &cs);
    if (a.inverse) sn = -sn;
    stf(yp, x0 * cs - x1 * sn);
    stf(yp + 1, x0 * sn + x1 * cs);
  }
}

// Vector ROTE: thread = 4 consecutive column pairs (16 B of bf16) of one row,
// 32-bit indexing, one log1p per thread instead of one per pair, the pair
// frequencies held in registers across grid-stride iterations; sin/cos by
// MUFU on the turn-reduced angle.  Needs d % 8 == 0, 8-element-aligned strides and 16 B-aligned bases.
template <typename T>
struct RoteVec;
template <>
struct RoteVec<bf16> {
  static __device__ __forceinline__ void load(const bf16* p, float* v) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 f = __bfloat1622float2(h[k]);
      v[2 * k] = f.x;
      v[2 * k + 1] = f.y;
    }
  }
  static __device__ __forceinline__ void store(bf16* p, const float* v) {
    uint4 u;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int k = 0; k < 4; ++k) h[k] = __floats2bfloat162_rn(v[2 * k], v[2 * k + 1]);
    *reinterpret_cast<uint4*>(p) = u;
  }
};
template <>
struct RoteVec<float> {
  static __device__ __forceinline__ void load(const float* p, float* v) {
    const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
    v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w, v[4] = b.x, v[5] = b.y, v[6] = b.z, v[7] = b.w;
  }
  static __device__ __forceinline__ void store(float* p, const float* v) {
    reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
};

template <typename T>
__global__ void __launch_bounds__(256, 4) rote_vec_kernel(kl_rote_args a) {
  KL_PDL_ENTRY();
  const int cpr = a.d >> 3;  // 4-pair chunks per row
  const unsigned total = (unsigned)a.B * (unsigned)a.T * (unsigned)cpr;
  const T* x = (const T*)a.x;
  T* y = (T*)a.y;
  const double inv_tau = 1.0 / a.tau_scale;
  // The launcher makes the grid stride a multiple of cpr: each thread keeps one
  // column chunk c (frequencies in registers) and walks rows (b, t) by a fixed
  // step with no division in the loop.
  const unsigned idx0 = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx0 >= total) return;
  const unsigned c = idx0 % (unsigned)cpr, r0 = idx0 / (unsigned)cpr;
  const unsigned rstep = gridDim.x * blockDim.x / (unsigned)cpr;
  const int db = (int)(rstep / (unsigned)a.T), dt = (int)(rstep % (unsigned)a.T);
  double pf[4], tf[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    pf[k] = __ldg(a.pos_freqs + 4 * c + k);
    tf[k] = __ldg(a.temp_freqs + 4 * c + k);
  }
  int b = (int)(r0 / (unsigned)a.T), t = (int)(r0 % (unsigned)a.T);
  for (; b < a.B; b += db, t += dt) {
    if (t >= a.T) t -= a.T, ++b;
    if (b >= a.B) break;
    const T* xp = x + (long long)b * a.x_bs + (long long)t * a.x_rs + 8 * c;
    T* yp = y + (long long)b * a.y_bs + (long long)t * a.y_rs + 8 * c;
    float v[8];
    RoteVec<T>::load(xp, v);
    const int len = a.lengths ? min(max(__ldg(a.lengths + b), 0), a.T) : a.T;  // clamped: never read past the sample
    if (t < len) {
      double g = 0.0;
      if (a.timestamps) {
        const double* ts = a.timestamps + (long long)b * a.ts_bs;
        const double gap = a.gap_mode == 0 ? (t > 0 ? __ldg(ts + t) - __ldg(ts + t - 1) : 0.0)
                                           : __ldg(ts + len - 1) - __ldg(ts + t);
        g = log1p(fmax(gap, 0.0) * inv_tau);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        double u = fma(g, tf[k], (double)t * pf[k]) * 0.15915494309189533577;  // turns
        u -= rint(u);
        // |2 pi u| <= pi: MUFU sin/cos, |abs err| <= 2^-21 on this range
        float sn, cs;
        __sincosf((float)(6.283185307179586477 * u), &sn, &cs);
        if (a.inverse) sn = -sn;
        const float x0 = v[2 * k], x1 = v[2 * k + 1];
        v[2 * k] = x0 * cs - x1 * sn;
        v[2 * k + 1] = x0 * sn + x1 * cs;
      }
    }
    RoteVec<T>::store(yp, v);
  }
}

template <typename TI, typename TO>
__global__ void cast_kernel(long long n, const TI* x, TO* y) {
  KL_PDL_ENTRY();
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    stf(y + i, ldf(x + i));
}

struct ActCodes {
  int n_act, group;
  int codes[KL_MAX_ACT_GROUPS];
};

template <typename T>
__global__ void act_kernel(int rows, int cols, const T* x, long long ld, T* y, long long ld_y, ActCodes ac) {
  KL_PDL_ENTRY();
  long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)rows * cols) return;
  int c = idx % cols;
  long long r = idx / cols;
  int code = ac.n_act == 0 ? 0 : ac.codes[(c / ac.group) % ac.n_act];
  stf(y + r * ld_y + c, act_apply(code, ldf(x + r * ld + c)));
}

template <typename T>
__global__ void act_bwd_kernel(int rows, int cols, const T* g, long long ldg, const T* x, long long ldx, T* y,
                               long long ld_y, ActCodes ac) {
  KL_PDL_ENTRY();
  long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)rows * cols) return;
  int c = idx % cols;
  long long r = idx / cols;
  int code = ac.n_act == 0 ? 0 : ac.codes[(c / ac.group) % ac.n_act];
  stf(y + r * ld_y + c, ldf(g + r * ldg + c) * act_deriv(code, ldf(x + r * ldx + c)));
}

template <typename T>
__global__ void finite_kernel(long long n, const T* x, unsigned int* flag) {
  KL_PDL_ENTRY();
  bool bad = false;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    bad |= !isfinite(ldf(x + i));
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

inline unsigned nblk(long long n, int t = 256) { return (unsigned)((n + t - 1) / t); }

}  // namespace

}  // namespace kl

using namespace kl;

extern "C" int kl_colsoftmax_fwd(const kl_colsoftmax_args* a, void* stream) {
  if (!a || a->Bn < 0 || a->T < 0 || a->C < 0) { set_error("kl_colsoftmax_fwd: bad args"); return KL_EBADSHAPE; }
  if (a->Bn == 0 || a->C == 0 || a->T == 0) return KL_OK;
  cudaStream_t s = (cudaStream_t)stream;
  dim3 grid((a->C + 31) / 32, a->Bn);
  if (a->dtype_in == KL_F32 && a->dtype_out == KL_F32) launch_k(colsoftmax_fwd_kernel<float, float>, grid, 256, 0, s, *a);
  else if (a->dtype_in == KL_F32) launch_k(colsoftmax_fwd_kernel<float, bf16>, grid, 256, 0, s, *a);
  else if (a->dtype_out == KL_F32) launch_k(colsoftmax_fwd_kernel<bf16, float>, grid, 256, 0, s, *a);
  else launch_k(colsoftmax_fwd_kernel<bf16, bf16>, grid, 256, 0, s, *a);
  count_launch();
  count_path(KL_PATH_COLSOFTMAX);
  return launch_check("colsoftmax_fwd");
}

extern "C" int kl_colsoftmax_bwd(const kl_colsoftmax_args* a, void* stream) {
  if (!a) { set_error("kl_colsoftmax_bwd: null args"); return KL_EBADSHAPE; }
  if (a->Bn == 0 || a->C == 0 || a->T == 0) return KL_OK;
  cudaStream_t s = (cudaStream_t)stream;
  dim3 grid((a->C + 31) / 32, a->Bn);
  // P in dtype_out, dP in dtype_dp, dX (and dX_lo) in dtype_in
  const int tp = a->dtype_out, tg = a->dtype_dp, to = a->dtype_in;
  if (a->X && a->LSE) {  // P recomputed from fp32 scores + LSE
    if (tg != KL_F32) { set_error("kl_colsoftmax_bwd: recompute mode needs fp32 dP"); return KL_EUNSUPPORTED; }
    if (to == KL_F32) launch_k(colsoftmax_bwd_kernel<float, float, float, true>, grid, 256, 0, s, *a);
    else launch_k(colsoftmax_bwd_kernel<float, float, bf16, true>, grid, 256, 0, s, *a);
  } else if (tp == KL_F32 && tg == KL_F32 && to == KL_F32) launch_k(colsoftmax_bwd_kernel<float, float, float>, grid, 256, 0, s, *a);
  else if (tp == KL_F32 && tg == KL_F32) launch_k(colsoftmax_bwd_kernel<float, float, bf16>, grid, 256, 0, s, *a);
  else if (tp == KL_BF16 && tg == KL_F32 && to == KL_BF16) launch_k(colsoftmax_bwd_kernel<bf16, float, bf16>, grid, 256, 0, s, *a);
  else if (tp == KL_BF16 && tg == KL_F32) launch_k(colsoftmax_bwd_kernel<bf16, float, float>, grid, 256, 0, s, *a);
  else if (tp == KL_BF16 && tg == KL_BF16 && to == KL_BF16) launch_k(colsoftmax_bwd_kernel<bf16, bf16, bf16>, grid, 256, 0, s, *a);
  else {
    set_error("kl_colsoftmax_bwd: unsupported dtype combination (P %d, dP %d, dX %d)", tp, tg, to);
    return KL_EUNSUPPORTED;
  }
  count_launch();
  return launch_check("colsoftmax_bwd");
}

extern "C" int kl_rmsnorm_fwd(int rows, int d, float eps, const float* x, const float* gain, float* y, void* stream) {
  return kl_rmsnorm_fwd_b(1, rows, d, eps, x, 0, gain, 0, y, 0, stream);
}

extern "C" int kl_rmsnorm_fwd_b(int nb, int rows, int d, float eps, const float* x, long long x_bs, const float* gain,
                                long long g_bs, float* y, long long y_bs, void* stream) {
  if (nb <= 0 || rows <= 0 || d <= 0) return KL_OK;
  launch_k(rmsnorm_fwd_kernel, dim3(rows, nb), 256, 0, (cudaStream_t)stream, d, eps, x, gain, y, x_bs, g_bs, y_bs);
  count_launch();
  return launch_check("rmsnorm_fwd");
}

extern "C" int kl_rmsnorm_bwd(int rows, int d, float eps, const float* x, const float* gain, const float* dy,
                              float* dx, float* dgain, void* stream) {
  return kl_rmsnorm_bwd_b(1, rows, d, eps, x, 0, gain, 0, dy, 0, dx, 0, dgain, 0, 0, stream);
}

extern "C" int kl_rmsnorm_bwd_b(int nb, int rows, int d, float eps, const float* x, long long x_bs, const float* gain,
                                long long g_bs, const float* dy, long long dy_bs, float* dx, long long dx_bs,
                                float* dgain, long long dg_bs, int accumulate, void* stream) {
  if (nb <= 0 || d <= 0) return KL_OK;
  if (rows > 8192) { set_error("kl_rmsnorm_bwd: rows %d > 8192", rows); return KL_EUNSUPPORTED; }
  const size_t sm = 2 * (size_t)std::max(rows, 1) * sizeof(float);
  if (sm > 48 * 1024) cudaFuncSetAttribute(rmsnorm_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  launch_k(rmsnorm_bwd_kernel, nb, 256, sm, (cudaStream_t)stream, rows, d, eps, x, gain, dy, dx, dgain, x_bs, g_bs,
           dy_bs, dx_bs, dg_bs, accumulate);
  count_launch();
  return launch_check("rmsnorm_bwd");
}

extern "C" int kl_recent_rows_fwd(int B, int T, int d, int n, int dtype, const void* S, long long s_bs,
                                  const int* lengths, void* out, long long o_bs, void* stream) {
  long long tot = (long long)B * n * d;
  if (tot == 0) return KL_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == KL_F32) launch_k(recent_fwd_kernel<float>, nblk(tot), 256, 0, s, B, T, d, n, (const float*)S, s_bs, lengths, (float*)out, o_bs);
  else launch_k(recent_fwd_kernel<bf16>, nblk(tot), 256, 0, s, B, T, d, n, (const bf16*)S, s_bs, lengths, (bf16*)out, o_bs);
  count_launch();
  return launch_check("recent_rows_fwd");
}

extern "C" int kl_recent_rows_bwd(int B, int T, int d, int n, int dtype, const void* dout, long long o_bs,
                                  const int* lengths, void* dS, long long s_bs, void* stream) {
  long long tot = (long long)B * n * d;
  if (tot == 0) return KL_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == KL_F32) launch_k(recent_bwd_kernel<float>, nblk(tot), 256, 0, s, B, T, d, n, (const float*)dout, o_bs, lengths, (float*)dS, s_bs);
  else launch_k(recent_bwd_kernel<bf16>, nblk(tot), 256, 0, s, B, T, d, n, (const bf16*)dout, o_bs, lengths, (bf16*)dS, s_bs);
  count_launch();
  return launch_check("recent_rows_bwd");
}

static inline bool vec8_ok(const void* p, long long rs, int d) {
  return d % 8 == 0 && rs % 8 == 0 && ((uintptr_t)p & 15) == 0;
}

// CTAs per sample: enough that each warp / thread gets a few work items
static inline unsigned gram_split(int items, int per_cta) {
  int s = (items + 4 * per_cta - 1) / (4 * per_cta);
  return (unsigned)std::max(1, std::min(s, 8));
}

template <typename T>
static void gram_fwd_launch(int B, int n, int d, const T* x, long long x_rs, long long x_bs, T* tri, long long t_bs,
                            size_t sm, cudaStream_t s) {
  if (vec8_ok(x, x_rs, d) && x_bs % 8 == 0) {
    cudaFuncSetAttribute(gram_triu_fwd_kernel<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    launch_k(gram_triu_fwd_kernel<T, true>, dim3(B, gram_split(n * (n + 1) / 2, 8)), 256, sm, s, n, d, x, x_rs, x_bs, tri, t_bs);
  } else {
    cudaFuncSetAttribute(gram_triu_fwd_kernel<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    launch_k(gram_triu_fwd_kernel<T, false>, dim3(B, gram_split(n * (n + 1) / 2, 8)), 256, sm, s, n, d, x, x_rs, x_bs, tri, t_bs);
  }
}

extern "C" int kl_gram_triu_fwd(int B, int n, int d, int dtype, const void* x, long long x_rs, long long x_bs,
                                void* tri, long long t_bs, void* stream) {
  if ((long long)B * n == 0) return KL_OK;
  const size_t sm = (size_t)n * (d + 4) * sizeof(float);
  if (sm > 200 * 1024) { set_error("kl_gram_triu_fwd: n*d = %d too large", n * d); return KL_EUNSUPPORTED; }
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == KL_F32)
    gram_fwd_launch(B, n, d, (const float*)x, x_rs, x_bs, (float*)tri, t_bs, sm, s);
  else
    gram_fwd_launch(B, n, d, (const bf16*)x, x_rs, x_bs, (bf16*)tri, t_bs, sm, s);
  count_launch();
  return launch_check("gram_triu_fwd");
}

template <typename T>
static void gram_bwd_launch(int B, int n, int d, const T* x, long long x_rs, long long x_bs, const T* dtri,
                            long long t_bs, T* dx, long long dx_rs, long long dx_bs, size_t sm, cudaStream_t s) {
  if (vec8_ok(x, x_rs, d) && x_bs % 8 == 0 && vec8_ok(dx, dx_rs, d) && dx_bs % 8 == 0) {
    cudaFuncSetAttribute(gram_triu_bwd_kernel<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    launch_k(gram_triu_bwd_kernel<T, true>, dim3(B, gram_split(n * d / 8, 64)), 256, sm, s, n, d, x, x_rs, x_bs, dtri, t_bs, dx, dx_rs, dx_bs);
  } else {
    cudaFuncSetAttribute(gram_triu_bwd_kernel<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    launch_k(gram_triu_bwd_kernel<T, false>, dim3(B, gram_split(n * d, 512)), 256, sm, s, n, d, x, x_rs, x_bs, dtri, t_bs, dx, dx_rs, dx_bs);
  }
}

extern "C" int kl_gram_triu_bwd(int B, int n, int d, int dtype, const void* x, long long x_rs, long long x_bs,
                                const void* dtri, long long t_bs, void* dx, long long dx_rs, long long dx_bs,
                                void* stream) {
  if ((long long)B * n * d == 0) return KL_OK;
  const size_t sm = ((size_t)n * (d + 4) + (size_t)n * n) * sizeof(float);
  if (sm > 200 * 1024) { set_error("kl_gram_triu_bwd: n*d = %d too large", n * d); return KL_EUNSUPPORTED; }
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == KL_F32)
    gram_bwd_launch(B, n, d, (const float*)x, x_rs, x_bs, (const float*)dtri, t_bs, (float*)dx, dx_rs, dx_bs, sm, s);
  else
    gram_bwd_launch(B, n, d, (const bf16*)x, x_rs, x_bs, (const bf16*)dtri, t_bs, (bf16*)dx, dx_rs, dx_bs, sm, s);
  count_launch();
  return launch_check("gram_triu_bwd");
}

extern "C" int kl_gated_sum_fwd(int rows, int d, int dtype, const void* x, long long x_rs, const void* deep,
                                const void* dot, const float* gd, const float* gt, void* out, long long o_rs,
                                void* stream) {
  long long tot = (long long)rows * d;
  if (tot == 0) return KL_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == KL_F32)
    launch_k(gated_fwd_kernel<float>, nblk(tot), 256, 0, s, rows, d, (const float*)x, x_rs, (const float*)deep, (const float*)dot, gd, gt, (float*)out, o_rs);
  else
    launch_k(gated_fwd_kernel<bf16>, nblk(tot), 256, 0, s, rows, d, (const bf16*)x, x_rs, (const bf16*)deep, (const bf16*)dot, gd, gt, (bf16*)out, o_rs);
  count_launch();
  return launch_check("gated_sum_fwd");
}

extern "C" int kl_gated_sum_bwd(int rows, int d, int dtype, const void* g, long long g_rs, const void* deep,
                                const void* dot, const float* gd, const float* gt, void* ddeep, void* ddot,
                                float* dgd, float* dgt, float* scratch, void* stream) {
  long long tot = (long long)rows * d;
  cudaStream_t s = (cudaStream_t)stream;
  int nb = (int)std::min<long long>(512, (tot + 255) / 256);
  if (nb < 1) nb = 1;
  if (dtype == KL_F32)
    launch_k(gated_bwd_kernel<float>, nb, 256, 0, s, rows, d, (const float*)g, g_rs, (const float*)deep, (const float*)dot, gd, gt, (float*)ddeep, (float*)ddot, (double*)scratch);
  else
    launch_k(gated_bwd_kernel<bf16>, nb, 256, 0, s, rows, d, (const bf16*)g, g_rs, (const bf16*)deep, (const bf16*)dot, gd, gt, (bf16*)ddeep, (bf16*)ddot, (double*)scratch);
  launch_k(reduce_pairs_kernel, 1, 256, 0, s, nb, (const double*)scratch, dgd, dgt);
  count_launch(2);
  return launch_check("gated_sum_bwd");
}

extern "C" int kl_rote(const kl_rote_args* a, void* stream) {
  if (!a || a->B < 0 || a->T < 0 || a->d < 2 || (a->d & 1) || (a->dtype != KL_F32 && a->dtype != KL_BF16) ||
      !a->pos_freqs || !a->temp_freqs || !(a->tau_scale > 0.0) || (a->gap_mode != 0 && a->gap_mode != 1) ||
      (a->x == a->y && (long long)a->B * a->T > 0)) {
    set_error("kl_rote: bad args (d even >= 2, tau_scale > 0, gap_mode 0/1, y != x)");
    return KL_EBADSHAPE;
  }
  const long long total = (long long)a->B * a->T * (a->d / 2);
  if (total == 0) return 0;
  const auto al16 = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
  const bool vec = a->d % 8 == 0 && a->x_rs % 8 == 0 && a->x_bs % 8 == 0 && a->y_rs % 8 == 0 &&
                   a->y_bs % 8 == 0 && al16(a->x) && al16(a->y) && total / 4 < (1LL << 31);
  if (vec) {
    const long long cpr = a->d / 8;
    // persistent: one wave of 4 blocks/SM (148*4*256 = 2^11*74 threads on a
    // B200 divide any power-of-two cpr <= 2048); otherwise the grid is rounded
    // to a multiple of cpr
    long long grid = std::min<long long>((total / 4 + 255) / 256, (long long)tc_num_sms() * 4);
    if ((grid * 256) % cpr) grid = (grid + cpr - 1) / cpr * cpr;
    if (a->dtype == KL_BF16)
      launch_k(rote_vec_kernel<bf16>, (int)grid, 256, 0, (cudaStream_t)stream, *a);
    else
      launch_k(rote_vec_kernel<float>, (int)grid, 256, 0, (cudaStream_t)stream, *a);
    return launch_check("rote");
  }
  const int grid = (int)std::min<long long>((total + 255) / 256, (long long)tc_num_sms() * 16);
  if (a->dtype == KL_BF16)
    launch_k(rote_kernel<bf16>, grid, 256, 0, (cudaStream_t)stream, *a);
  else
    launch_k(rote_kernel<float>, grid, 256, 0, (cudaStream_t)stream, *a);
  return launch_check("rote");
}

extern "C" int kl_ne(int n, int kind, const float* p, const float* y, double* out, void* stream) {
  if (n < 1 || (kind != 0 && kind != 1)) {
    set_error("kl_ne: needs n >= 1 and kind 0 (probabilities) or 1 (logits)");
    return KL_EBADSHAPE;
  }
  launch_k(ne_kernel, 1, 256, 0, (cudaStream_t)stream, n, kind, p, y, out);
  return launch_check("ne");
}

extern "C" int kl_bce_fwd_bwd(int n, const float* z, const float* y, float* loss, float* dz, void* stream) {
  launch_k(bce_kernel, 1, 256, 0, (cudaStream_t)stream, n, z, y, loss, dz);
  count_launch();
  return launch_check("bce");
}

extern "C" int kl_cast(long long n, int dtype_in, const void* x, int dtype_out, void* y, void* stream) {
  if (n == 0) return KL_OK;
  cudaStream_t s = (cudaStream_t)stream;
  unsigned g = (unsigned)std::min<long long>((n + 255) / 256, (long long)tc_num_sms() * 16);
  if (dtype_in == KL_F32 && dtype_out == KL_BF16) launch_k(cast_kernel<float, bf16>, g, 256, 0, s, n, (const float*)x, (bf16*)y);
  else if (dtype_in == KL_BF16 && dtype_out == KL_F32) launch_k(cast_kernel<bf16, float>, g, 256, 0, s, n, (const bf16*)x, (float*)y);
  else if (dtype_in == KL_F32) launch_k(cast_kernel<float, float>, g, 256, 0, s, n, (const float*)x, (float*)y);
  else launch_k(cast_kernel<bf16, bf16>, g, 256, 0, s, n, (const bf16*)x, (bf16*)y);
  count_launch();
  return launch_check("cast");
}

extern "C" int kl_act_fwd(int rows, int cols, int dtype, const void* x, long long ld, void* y, long long ld_y,
                          int n_act, int act_group, const int* codes, void* stream) {
  long long tot = (long long)rows * cols;
  if (tot == 0) return KL_OK;
  if (n_act < 0 || n_act > KL_MAX_ACT_GROUPS) { set_error("kl_act_fwd: n_act %d", n_act); return KL_EBADSHAPE; }
  ActCodes ac{};
  ac.n_act = n_act;
  ac.group = act_group > 0 ? act_group : 1;
  for (int i = 0; i < n_act; ++i) ac.codes[i] = codes[i];
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == KL_F32) launch_k(act_kernel<float>, nblk(tot), 256, 0, s, rows, cols, (const float*)x, ld, (float*)y, ld_y, ac);
  else launch_k(act_kernel<bf16>, nblk(tot), 256, 0, s, rows, cols, (const bf16*)x, ld, (bf16*)y, ld_y, ac);
  count_launch();
  return launch_check("act_fwd");
}

extern "C" int kl_act_bwd(int rows, int cols, int dtype, const void* g, long long ldg, const void* x, long long ldx,
                          void* y, long long ld_y, int n_act, int act_group, const int* codes, void* stream) {
  long long tot = (long long)rows * cols;
  if (tot == 0) return KL_OK;
  if (n_act < 0 || n_act > KL_MAX_ACT_GROUPS) { set_error("kl_act_bwd: n_act %d", n_act); return KL_EBADSHAPE; }
  ActCodes ac{};
  ac.n_act = n_act;
  ac.group = act_group > 0 ? act_group : 1;
  for (int i = 0; i < n_act; ++i) ac.codes[i] = codes[i];
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == KL_F32) launch_k(act_bwd_kernel<float>, nblk(tot), 256, 0, s, rows, cols, (const float*)g, ldg, (const float*)x, ldx, (float*)y, ld_y, ac);
  else launch_k(act_bwd_kernel<bf16>, nblk(tot), 256, 0, s, rows, cols, (const bf16*)g, ldg, (const bf16*)x, ldx, (bf16*)y, ld_y, ac);
  count_launch();
  return launch_check("act_bwd");
}

extern "C" int kl_check_finite(long long n, int dtype, const void* x, unsigned int* flag, void* stream) {
  if (n == 0) return KL_OK;
  cudaStream_t s = (cudaStream_t)stream;
  unsigned g = (unsigned)std::min<long long>((n + 255) / 256, (long long)tc_num_sms() * 8);
  if (dtype == KL_F32) launch_k(finite_kernel<float>, g, 256, 0, s, n, (const float*)x, flag);
  else launch_k(finite_kernel<bf16>, g, 256, 0, s, n, (const bf16*)x, flag);
  count_launch();
  return launch_check("check_finite");
}

// ---------------------------------------------------------------------------
// Fused Adam over the flat fp32 parameter buffer (SPEC.md:672-675 trainer
// default: beta1 .9, beta2 .999, eps 1e-8), writing the bf16 compute mirror in
// the same pass so no separate cast kernel runs before the next forward.
namespace kl {
namespace {
// float4-vectorised; the step count may live on the device (graph replay):
// the bias corrections are computed per block from *step_dev.
__global__ void adam_kernel(long long n, float lr, float b1, float b2, float eps, int step, const int* step_dev,
                            float* w, const float* g, float* m, float* v, bf16* wc) {
  KL_PDL_ENTRY();
  const int t = step_dev ? *step_dev : step;
  const float c1 = 1.f / (1.f - powf(b1, (float)t));
  const float c2 = 1.f / (1.f - powf(b2, (float)t));
  const long long n4 = n / 4;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    const float4 gi = reinterpret_cast<const float4*>(g)[i];
    float4 mi = reinterpret_cast<float4*>(m)[i], vi = reinterpret_cast<float4*>(v)[i];
    float4 wi = reinterpret_cast<float4*>(w)[i];
    float* mp = &mi.x;
    float* vp = &vi.x;
    float* wp = &wi.x;
    const float* gp = &gi.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      mp[k] = b1 * mp[k] + (1.f - b1) * gp[k];
      vp[k] = b2 * vp[k] + (1.f - b2) * gp[k] * gp[k];
      wp[k] = wp[k] - lr * (mp[k] * c1) / (sqrtf(vp[k] * c2) + eps);
    }
    reinterpret_cast<float4*>(m)[i] = mi;
    reinterpret_cast<float4*>(v)[i] = vi;
    reinterpret_cast<float4*>(w)[i] = wi;
    if (wc) {
      reinterpret_cast<__nv_bfloat162*>(wc)[2 * i] = __floats2bfloat162_rn(wi.x, wi.y);
      reinterpret_cast<__nv_bfloat162*>(wc)[2 * i + 1] = __floats2bfloat162_rn(wi.z, wi.w);
    }
  }
  for (long long i = n4 * 4 + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const float gi = g[i];
    const float mi = b1 * m[i] + (1.f - b1) * gi;
    const float vi = b2 * v[i] + (1.f - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    const float wi = w[i] - lr * (mi * c1) / (sqrtf(vi * c2) + eps);
    w[i] = wi;
    if (wc) wc[i] = __float2bfloat16(wi);
  }
}

__global__ void tick_kernel(int* step_dev) {
  KL_PDL_ENTRY(); *step_dev += 1; }
}  // namespace
}  // namespace kl

extern "C" int kl_adam_step(long long n, float lr, float beta1, float beta2, float eps, int step, int* step_dev,
                            float* w, const float* g, float* m, float* v, void* w_bf16, void* stream) {
  if (n == 0) return KL_OK;
  if (!step_dev && step < 1) { set_error("kl_adam_step: step must be >= 1"); return KL_EBADSHAPE; }
  if (step_dev && step != 0 && step != -1) { set_error("kl_adam_step: step must be 0 or -1 with step_dev"); return KL_EBADSHAPE; }
  if (((uintptr_t)w | (uintptr_t)g | (uintptr_t)m | (uintptr_t)v) & 15) {
    set_error("kl_adam_step: buffers must be 16-byte aligned");
    return KL_EBADSHAPE;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const bool tick = step_dev && step != -1;
  if (tick) launch_k(tick_kernel, 1, 1, 0, s, step_dev);
  unsigned grid = (unsigned)std::min<long long>((n / 4 + 255) / 256 + 1, (long long)tc_num_sms() * 8);
  launch_k(adam_kernel, grid, 256, 0, s, n, lr, beta1, beta2, eps, step, step_dev, w, g, m, v, (bf16*)w_bf16);
  count_launch(tick ? 2 : 1);
  return launch_check("adam_step");
}

extern "C" int kl_adam_tick(int* step_dev, void* stream) {
  launch_k(tick_kernel, 1, 1, 0, (cudaStream_t)stream, step_dev);
  count_launch();
  return launch_check("adam_tick");
}

namespace kl {
namespace {
// out[r] = sum_k a[r, k] * b[r, k] (fp32 accumulation): one warp per row,
// 16-byte loads when rows are 16-byte aligned (the softmax-VJP row term
// rowsum(dO * O) of the pooling backward).
template <typename T, bool VEC>
__global__ void __launch_bounds__(256) rowdot_kernel(int rows, int d, const T* a, long long a_rs, const T* b,
                                                     long long b_rs, float* out) {
  KL_PDL_ENTRY();
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= rows) return;
  const T* ar = a + (long long)r * a_rs;
  const T* br = b + (long long)r * b_rs;
  float acc = 0.f;
  if (VEC) {
    for (int k = lane * 8; k < d; k += 256) {
      float x[8], y[8];
      ld8(ar + k, x);
      ld8(br + k, y);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc = fmaf(x[i], y[i], acc);
    }
  } else {
    for (int k = lane; k < d; k += 32) acc = fmaf(ldf(ar + k), ldf(br + k), acc);
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) out[r] = acc;
}
}  // namespace
}  // namespace kl

extern "C" int kl_rowdot(int rows, int d, int dtype, const void* a, long long a_rs, const void* b, long long b_rs,
                         float* out, void* stream) {
  using namespace kl;
  if (rows <= 0) return KL_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned grid = (unsigned)((rows + 7) / 8);
  const bool vec = vec8_ok(a, a_rs, d) && vec8_ok(b, b_rs, d);
  if (dtype == KL_F32) {
    if (vec) launch_k(rowdot_kernel<float, true>, grid, 256, 0, s, rows, d, (const float*)a, a_rs, (const float*)b, b_rs, out);
    else launch_k(rowdot_kernel<float, false>, grid, 256, 0, s, rows, d, (const float*)a, a_rs, (const float*)b, b_rs, out);
  } else {
    if (vec) launch_k(rowdot_kernel<bf16, true>, grid, 256, 0, s, rows, d, (const bf16*)a, a_rs, (const bf16*)b, b_rs, out);
    else launch_k(rowdot_kernel<bf16, false>, grid, 256, 0, s, rows, d, (const bf16*)a, a_rs, (const bf16*)b, b_rs, out);
  }
  count_launch();
  return launch_check("rowdot");
}

// ---------------------------------------------------------------------------
// Non-sequence embedding (preproc.py:103-136: embed_dense, embed_sparse,
// assemble_nonseq) fused into one pass: out[b, 0] = proj x_dense[b] (m small:
// per-thread dot products), out[b, 1 + i] = table[offset_i + ids[b, i]] (row
// gathers of the stacked per-feature tables).  One block per sample row
// (b, i), threads over d.  HBM-bound: one read of each gathered row, one write.
namespace kl {
namespace emb {
template <typename T>
__global__ void __launch_bounds__(128) embed_fwd_kernel(int n_sparse, int d, int m, const float* xd, const T* proj,
                                                        const T* table, const long long* offsets,
                                                        const long long* ids, long long vocab_tot, T* out) {
  KL_PDL_ENTRY();
  const int b = blockIdx.y, i = blockIdx.x;  // i = 0: dense row, i >= 1: sparse feature i - 1
  T* o = out + ((long long)b * (n_sparse + 1) + i) * d;
  if (i == 0) {
    const float* x = xd + (long long)b * m;
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
      float acc = 0.f;
      for (int k = 0; k < m; ++k) acc = fmaf(ldf(proj + (long long)c * m + k), __ldg(x + k), acc);
      stf(o + c, acc);
    }
    return;
  }
  long long row = offsets[i - 1] + ids[(long long)b * n_sparse + (i - 1)];
  row = row < 0 ? 0 : (row >= vocab_tot ? vocab_tot - 1 : row);  // host-validated; clamped for memory safety
  const T* src = table + row * d;
  for (int c = threadIdx.x; c < d; c += blockDim.x) o[c] = src[c];
}

// VJP: dtable[row] += dout[b, 1 + i] (fp32 atomics: several samples can pick
// one id), dproj[c, k] += sum_b dout[b, 0, c] x_dense[b, k].
template <typename T>
__global__ void __launch_bounds__(128) embed_bwd_kernel(int B, int n_sparse, int d, int m, const float* xd,
                                                        const T* dout, const long long* offsets, const long long* ids,
                                                        long long vocab_tot, float* dtable, float* dproj) {
  KL_PDL_ENTRY();
  const int i = blockIdx.x;
  if (i == 0) {  // dense projection gradient: block per (c chunk); loops over the batch
    for (int c = threadIdx.x + blockIdx.y * blockDim.x; c < d; c += blockDim.x * gridDim.y)
      for (int k = 0; k < m; ++k) {
        float acc = 0.f;
        for (int b = 0; b < B; ++b)
          acc = fmaf(ldf(dout + (long long)b * (n_sparse + 1) * d + c), __ldg(xd + (long long)b * m + k), acc);
        dproj[(long long)c * m + k] += acc;
      }
    return;
  }
  for (int b = blockIdx.y; b < B; b += gridDim.y) {
    long long row = offsets[i - 1] + ids[(long long)b * n_sparse + (i - 1)];
    if (row < 0 || row >= vocab_tot) continue;
    const T* g = dout + ((long long)b * (n_sparse + 1) + i) * d;
    float* dst = dtable + row * d;
    for (int c = threadIdx.x; c < d; c += blockDim.x) atomicAdd(dst + c, ldf(g + c));
  }
}
}  // namespace emb
}  // namespace kl

extern "C" int kl_embed_nonseq_fwd(int B, int n_sparse, int d, int m, int dtype, const float* x_dense,
                                   const void* proj, const void* table, const long long* offsets,
                                   const long long* ids, long long vocab_tot, void* out, void* stream) {
  if (B < 0 || n_sparse < 0 || d < 1 || m < 0) { set_error("kl_embed_nonseq_fwd: bad extents"); return KL_EBADSHAPE; }
  if (B == 0) return KL_OK;
  dim3 grid(n_sparse + 1, B);
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == KL_F32)
    launch_k(kl::emb::embed_fwd_kernel<float>, grid, 128, 0, s, n_sparse, d, m, x_dense, (const float*)proj,
             (const float*)table, offsets, ids, vocab_tot, (float*)out);
  else
    launch_k(kl::emb::embed_fwd_kernel<bf16>, grid, 128, 0, s, n_sparse, d, m, x_dense, (const bf16*)proj, (const bf16*)table,
             offsets, ids, vocab_tot, (bf16*)out);
  count_launch();
  return launch_check("embed_nonseq_fwd");
}

extern "C" int kl_embed_nonseq_bwd(int B, int n_sparse, int d, int m, int dtype, const float* x_dense,
                                   const void* dout, const long long* offsets, const long long* ids,
                                   long long vocab_tot, float* dtable, float* dproj, void* stream) {
  if (B < 0 || n_sparse < 0 || d < 1 || m < 0) { set_error("kl_embed_nonseq_bwd: bad extents"); return KL_EBADSHAPE; }
  if (B == 0) return KL_OK;
  dim3 grid(n_sparse + 1, std::min(B, 64));
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == KL_F32)
    launch_k(kl::emb::embed_bwd_kernel<float>, grid, 128, 0, s, B, n_sparse, d, m, x_dense, (const float*)dout, offsets, ids,
             vocab_tot, dtable, dproj);
  else
    launch_k(kl::emb::embed_bwd_kernel<bf16>, grid, 128, 0, s, B, n_sparse, d, m, x_dense, (const bf16*)dout, offsets, ids,
             vocab_tot, dtable, dproj);
  count_launch();
  return launch_check("embed_nonseq_bwd");
}

// ---------------------------------------------------------------------------
// masked_softmax_lastdim (tensor.py:485-505) with an explicit boolean mask:
// one warp per row of n columns; fully-masked rows give 0.  The mask is
// (rows / mask_div) x n, so one (n_q, n_k) mask serves every (batch, head).
namespace kl {
namespace msm {
__global__ void __launch_bounds__(256) masked_softmax_fwd_kernel(long long rows, int n, const float* x,
                                                                 const unsigned char* mask, long long mask_div,
                                                                 float* y) {
  KL_PDL_ENTRY();
  const long long row = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float* xr = x + row * n;
  const unsigned char* mr = mask + (row % mask_div) * n;
  float mx = -INFINITY;
  for (int c = lane; c < n; c += 32)
    if (mr[c]) mx = fmaxf(mx, xr[c]);
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float s = 0.f;
  for (int c = lane; c < n; c += 32)
    if (mr[c]) s += expf(xr[c] - mx);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float inv = s > 0.f ? 1.f / s : 0.f;
  for (int c = lane; c < n; c += 32) y[row * n + c] = mr[c] ? expf(xr[c] - mx) * inv : 0.f;
}
// dx = y * (g - sum(g * y))   (tensor.py:501-503)
__global__ void __launch_bounds__(256) masked_softmax_bwd_kernel(long long rows, int n, const float* y, const float* g,
                                                                 float* dx) {
  KL_PDL_ENTRY();
  const long long row = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float* yr = y + row * n;
  const float* gr = g + row * n;
  float acc = 0.f;
  for (int c = lane; c < n; c += 32) acc = fmaf(yr[c], gr[c], acc);
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  for (int c = lane; c < n; c += 32) dx[row * n + c] = yr[c] * (gr[c] - acc);
}
}  // namespace msm
}  // namespace kl

extern "C" int kl_masked_softmax_fwd(long long rows, int n, const float* x, const unsigned char* mask,
                                     long long mask_rows, float* y, void* stream) {
  if (rows < 0 || n < 0 || mask_rows < 1) { set_error("kl_masked_softmax_fwd: bad extents"); return KL_EBADSHAPE; }
  if (rows == 0 || n == 0) return KL_OK;
  launch_k(kl::msm::masked_softmax_fwd_kernel, (unsigned)((rows + 7) / 8), 256, 0, (cudaStream_t)stream, rows, n, x,
           mask, mask_rows, y);
  count_launch();
  return launch_check("masked_softmax_fwd");
}

extern "C" int kl_masked_softmax_bwd(long long rows, int n, const float* y, const float* g, float* dx, void* stream) {
  if (rows < 0 || n < 0) { set_error("kl_masked_softmax_bwd: bad extents"); return KL_EBADSHAPE; }
  if (rows == 0 || n == 0) return KL_OK;
  launch_k(kl::msm::masked_softmax_bwd_kernel, (unsigned)((rows + 7) / 8), 256, 0, (cudaStream_t)stream, rows, n, y,
           g, dx);
  count_launch();
  return launch_check("masked_softmax_bwd");
}

// ---------------------------------------------------------------------------
// Row regrouping (the token-axis concatenations / splits of the layer:
// SummaryBundle [CLS | seeds | recent] rows (seqsum.py:148-162), the expert
// slices of [X | summaries] and their re-concatenation (interaction.py:
// 144-157), the pooled-row gradients of the HSP backward): every destination
// row is one source row (or zeros), all segments of all samples in ONE launch.
// HBM-bound: one read and one write of each row, 16-byte vectors when the
// rows allow.  A block per (destination row, sample).
namespace kl {
namespace rg {
struct Segs {
  int n_seg, d, esz;
  int row0[KL_MAX_SEGS + 1];  // destination-row prefix of the segments
  kl_regroup_seg seg[KL_MAX_SEGS];
};

template <int VB>  // bytes per vector access (16 or the element size)
__global__ void __launch_bounds__(128) regroup_kernel(Segs sg) {
  KL_PDL_ENTRY();
  const int r = blockIdx.x, b = blockIdx.y;
  int s = 0;
  while (s + 1 < sg.n_seg && r >= sg.row0[s + 1]) ++s;
  const kl_regroup_seg& g = sg.seg[s];
  const int i = r - sg.row0[s];
  const long long rb = (long long)sg.d * sg.esz;  // row bytes
  char* dst = (char*)g.dst + ((long long)b * g.dst_bs + (long long)i * g.dst_rs) * sg.esz;
  if (g.src == nullptr) {
    for (long long o = (long long)threadIdx.x * VB; o < rb; o += 128 * VB) {
      if (VB == 16) *reinterpret_cast<uint4*>(dst + o) = make_uint4(0u, 0u, 0u, 0u);
      else if (VB == 4) *reinterpret_cast<uint32_t*>(dst + o) = 0u;
      else *reinterpret_cast<uint16_t*>(dst + o) = 0;
    }
    return;
  }
  const char* src = (const char*)g.src + ((long long)b * g.src_bs + (long long)i * g.src_rs) * sg.esz;
  for (long long o = (long long)threadIdx.x * VB; o < rb; o += 128 * VB) {
    if (VB == 16) *reinterpret_cast<uint4*>(dst + o) = *reinterpret_cast<const uint4*>(src + o);
    else if (VB == 4) *reinterpret_cast<uint32_t*>(dst + o) = *reinterpret_cast<const uint32_t*>(src + o);
    else *reinterpret_cast<uint16_t*>(dst + o) = *reinterpret_cast<const uint16_t*>(src + o);
  }
}

// out[b * out_bs + i] = sum_k a[b, i, k] * b[b, i, k] for i < n (rows of a
// (B, n, d) strided tensor pair): the softmax-VJP row term of one pooled part.
template <typename T, bool VEC>
__global__ void __launch_bounds__(256) rowdot3_kernel(int B, int n, int d, const T* a, long long a_bs,
                                                      long long a_rs, const T* b, long long b_bs, long long b_rs,
                                                      float* out, long long out_bs) {
  KL_PDL_ENTRY();
  const long long r = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= (long long)B * n) return;
  const int bb = (int)(r / n), i = (int)(r % n);
  const T* ar = a + bb * a_bs + i * a_rs;
  const T* br = b + bb * b_bs + i * b_rs;
  float acc = 0.f;
  if (VEC) {
    for (int k = lane * 8; k < d; k += 256) {
      float x[8], y[8];
      ld8(ar + k, x);
      ld8(br + k, y);
#pragma unroll
      for (int u = 0; u < 8; ++u) acc = fmaf(x[u], y[u], acc);
    }
  } else {
    for (int k = lane; k < d; k += 32) acc = fmaf(ldf(ar + k), ldf(br + k), acc);
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) out[bb * out_bs + i] = acc;
}
}  // namespace rg
}  // namespace kl

extern "C" int kl_regroup(const kl_regroup_args* a, void* stream) {
  using namespace kl;
  if (!a || a->B < 0 || a->d < 1 || a->n_seg < 1 || a->n_seg > KL_MAX_SEGS ||
      (a->dtype != KL_BF16 && a->dtype != KL_F32)) {
    set_error("kl_regroup: bad extents (B >= 0, d >= 1, 1..%d segments, bf16 / fp32)", KL_MAX_SEGS);
    return KL_EBADSHAPE;
  }
  rg::Segs sg{};
  sg.n_seg = a->n_seg;
  sg.d = a->d;
  sg.esz = a->dtype == KL_F32 ? 4 : 2;
  bool vec = (a->d * sg.esz) % 16 == 0;
  int rows = 0;
  for (int s = 0; s < a->n_seg; ++s) {
    const kl_regroup_seg& g = a->seg[s];
    if (g.rows < 0 || !g.dst) {
      set_error("kl_regroup: segment %d has no destination or negative rows", s);
      return KL_EBADSHAPE;
    }
    sg.row0[s] = rows;
    sg.seg[s] = g;
    rows += g.rows;
    auto al = [&](const void* p, long long bs, long long rs) {
      return ((uintptr_t)p & 15) == 0 && (bs * sg.esz) % 16 == 0 && (rs * sg.esz) % 16 == 0;
    };
    vec = vec && al(g.dst, g.dst_bs, g.dst_rs) && (!g.src || al(g.src, g.src_bs, g.src_rs));
  }
  sg.row0[a->n_seg] = rows;
  if (rows == 0 || a->B == 0) return KL_OK;
  cudaStream_t s = (cudaStream_t)stream;
  dim3 grid((unsigned)rows, (unsigned)a->B);
  if (vec) launch_k(rg::regroup_kernel<16>, grid, 128, 0, s, sg);
  else if (sg.esz == 4) launch_k(rg::regroup_kernel<4>, grid, 128, 0, s, sg);
  else launch_k(rg::regroup_kernel<2>, grid, 128, 0, s, sg);
  count_launch();
  return launch_check("regroup");
}

extern "C" int kl_rowdot3(int B, int n, int d, int dtype, const void* a, long long a_bs, long long a_rs, const void* b,
                          long long b_bs, long long b_rs, float* out, long long out_bs, void* stream) {
  using namespace kl;
  if (B < 0 || n < 0 || d < 1) { set_error("kl_rowdot3: bad extents"); return KL_EBADSHAPE; }
  if ((long long)B * n == 0) return KL_OK;
  const unsigned grid = (unsigned)(((long long)B * n + 7) / 8);
  cudaStream_t s = (cudaStream_t)stream;
  const bool vec = vec8_ok(a, a_rs, d) && vec8_ok(b, b_rs, d) && a_bs % 8 == 0 && b_bs % 8 == 0;
  if (dtype == KL_F32) {
    if (vec)
      launch_k(rg::rowdot3_kernel<float, true>, grid, 256, 0, s, B, n, d, (const float*)a, a_bs, a_rs,
               (const float*)b, b_bs, b_rs, out, out_bs);
    else
      launch_k(rg::rowdot3_kernel<float, false>, grid, 256, 0, s, B, n, d, (const float*)a, a_bs, a_rs,
               (const float*)b, b_bs, b_rs, out, out_bs);
  } else {
    if (vec)
      launch_k(rg::rowdot3_kernel<bf16, true>, grid, 256, 0, s, B, n, d, (const bf16*)a, a_bs, a_rs, (const bf16*)b,
               b_bs, b_rs, out, out_bs);
    else
      launch_k(rg::rowdot3_kernel<bf16, false>, grid, 256, 0, s, B, n, d, (const bf16*)a, a_bs, a_rs,
               (const bf16*)b, b_bs, b_rs, out, out_bs);
  }
  count_launch();
  return launch_check("rowdot3");
}

extern "C" int kl_memset(void* p, long long bytes, void* stream) {
  if (bytes < 0 || (bytes > 0 && !p)) { kl::set_error("kl_memset: bad buffer"); return KL_EBADSHAPE; }
  if (bytes == 0) return KL_OK;
  cudaMemsetAsync(p, 0, (size_t)bytes, (cudaStream_t)stream);
  return kl::launch_check("memset");
}
