#include <cstdio>
// Persistent, warp-specialized tcgen05 GEMM for sm_100a (bf16 x bf16 -> fp32
// in TMEM) with the generic kl_gemm epilogue.
//
//   warp 0      TMA producer: A/B tiles -> SWIZZLE_128B smem ring (mbarriers)
//   warp 1      MMA issuer: one thread issues tcgen05.mma (M=128, N=BN, K=16)
//   warps 2..5  epilogue: tcgen05.ld TMEM -> registers -> epilogue -> global
//
// Two TMEM accumulators (double buffer) let the epilogue of tile t overlap the
// MMAs of tile t+1.  Operands may be K-major or MN-major (the UMMA descriptor
// major bits), batched over two strided dims (TMA tensor dims 2-3), and a
// batch dim may be reduced (its tiles accumulate into one TMEM tile).
#include <cudaTypedefs.h>

#include <stdlib.h>

#include <algorithm>

#include "gemm.h"
#include "tc_common.cuh"

namespace kl {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int NTHREADS = 192;
constexpr int NTHREADS_WIDE = 320;  // wide tiles: 8 epilogue warps (2 column halves per TMEM lane quarter)

struct TcParams {
  int M, N, K, BN;
  int tiles_m, tiles_n, n_out;
  int nb1, nb2, red1, red2;
  int kblocks;
  int a_mn, b_mn;
  int a_has1, a_has2, b_has1, b_has2;
  int b_boxes;
  int stages;
  uint32_t a_stage_bytes, b_stage_bytes;
  uint32_t acc_stride;
  uint32_t tmem_cols;
  int splits;  // split-K over the (reduced batch x k-block) iterations; >1 -> fp32 atomics
  void* C;
  long long c_rs, c_cs, c_s1, c_s2;
  const void* R;
  long long r_rs, r_cs, r_s1, r_s2;
  void* aux;
  int vec_c;  // C rows admit paired (4 B bf16 / 8 B fp32) stores at even columns
  int vec_r;  // same for the residual
  int r_boxes;  // >0: residual tile staged by TMA in r_boxes 64-column boxes
  int r_has1, r_has2;
  float* ws;    // split-K partials [split][out batch][M][N] (fp32) or NULL (atomics)
  int c_has1, c_has2;  // MODE 2: C tensor-map batch dims present
  int reduce_c;        // MODE 2: TMA reduce-add into C (fp32 accumulate / split-K)
  int x_tma;           // MODE 3, aux_mode 1: pre-activation stored by TMA (tmX, C's layout)
  int r_bufs;          // residual tile buffers (2; 1 for 256-wide tiles with a long reduction)
  int n_fast;          // tile order: N tiles of one M block adjacent (A read once from HBM)
  int wide;            // PAIR: 256 x 512 tiles — two N = 256 products per k step into one 512-column
                       // accumulator (no double buffer); each CTA stages 2 x 128 B columns
  int r_glob;          // wide tiles with a residual: the epilogue warps read it from global memory,
                       // coalesced, into their staging boxes (no producer-staged residual tiles)
  int epi_regs_off;    // KL_GEMM_EPI_REGS=0: wide bf16 tiles drain TMEM through epi_tma (A/B testing)
};

constexpr int SLD = 66;  // epilogue staging row stride (floats): 64 columns + pad, 8-byte aligned

__device__ __forceinline__ void st2(bf16* p, float a, float b) {
  *reinterpret_cast<__nv_bfloat162*>(p) = __floats2bfloat162_rn(a, b);
}
__device__ __forceinline__ void st2(float* p, float a, float b) { *reinterpret_cast<float2*>(p) = make_float2(a, b); }

template <typename TC>
__device__ __forceinline__ void store_pair(TC* p, long long cs, float a, float b, bool ok0, bool ok1, int vec) {
  if (vec && ok0 && ok1) {
    st2(p, a, b);
  } else {
    if (ok0) stf(p, a);
    if (ok1) stf(p + cs, b);
  }
}

template <typename TC>
__device__ __forceinline__ void ld_pair(const TC* p, long long cs, bool ok0, bool ok1, int vec, float& a, float& b) {
  if (vec && ok0 && ok1) {
    if constexpr (sizeof(TC) == 2) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(p));
      a = f.x;
      b = f.y;
    } else {
      const float2 f = *reinterpret_cast<const float2*>(p);
      a = f.x;
      b = f.y;
    }
  } else {
    a = ok0 ? ldf(p) : 0.f;
    b = ok1 ? ldf(p + cs) : 0.f;
  }
}

// Activation / derivative over 8 values of one column: the tag switch is hoisted
// out of the row loop (one branch per 8 rows).  bf16-path intrinsics (__expf,
// __fdividef): the result is rounded to bf16.
__device__ __forceinline__ float fsig(float x) { return __fdividef(1.f, 1.f + __expf(-x)); }

__device__ __forceinline__ void act8(int code, float* v) {
  switch (code) {
    case KL_ACT_RELU:
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = fmaxf(v[i], 0.f);
      break;
    case KL_ACT_SILU:
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = v[i] * fsig(v[i]);
      break;
    case KL_ACT_TANH:
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = tanhf(v[i]);
      break;
    case KL_ACT_SIGMOID:
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = fsig(v[i]);
      break;
    case KL_ACT_EXP:
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = __expf(v[i]);
      break;
    case KL_ACT_SQRT:
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = sqrtf(v[i]);
      break;
    case KL_ACT_LOG:
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = __logf(v[i]);
      break;
    default:
      break;
  }
}

__device__ __forceinline__ void dact8(int code, float* v, const float* x) {
  switch (code) {
    case KL_ACT_RELU:
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = x[i] > 0.f ? v[i] : 0.f;
      break;
    case KL_ACT_SILU:
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float s = fsig(x[i]);
        v[i] *= s * (1.f + x[i] * (1.f - s));
      }
      break;
    case KL_ACT_TANH:
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float y = tanhf(x[i]);
        v[i] *= 1.f - y * y;
      }
      break;
    case KL_ACT_SIGMOID:
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float y = fsig(x[i]);
        v[i] *= y * (1.f - y);
      }
      break;
    case KL_ACT_EXP:
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] *= __expf(x[i]);
      break;
    case KL_ACT_SQRT:
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] *= __fdividef(0.5f, sqrtf(x[i]));
      break;
    case KL_ACT_LOG:
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] *= __fdividef(1.f, x[i]);
      break;
    default:
      break;
  }
}

// Generic epilogue over a lane's column pair, eight rows at a time.  Every
// optional feature is a warp-uniform branch around its own unrolled 8-row
// loop, so its 16 loads are in flight together and disabled features cost one
// branch per 8 rows.
template <typename TC>
__device__ __forceinline__ void epi_generic(const TcParams& p, const Epi& e, const float* stg, TC* C, const TC* R,
                                            TC* X, int m0, int rows, int n, bool ok0, bool ok1, int lim,
                                            const bf16* Rs, int rrow0, int rcol) {
  const int lane = threadIdx.x & 31;
  const int code0 = epi_code(e, n), code1 = epi_code(e, n + 1);
  const float b0 = (e.bias && ok0) ? e.bias[n] : 0.f, b1 = (e.bias && ok1) ? e.bias[n + 1] : 0.f;
  const long long cbase = (long long)m0 * p.c_rs + (long long)n * p.c_cs;
  const long long rbase = (long long)m0 * p.r_rs + (long long)n * p.r_cs;
  for (int r0 = 0; r0 < rows; r0 += 8) {
    float v0[8], v1[8];
    bool in[8], live[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float2 a = *reinterpret_cast<const float2*>(&stg[(r0 + i) * SLD + 2 * lane]);
      in[i] = (r0 + i < rows);
      live[i] = (m0 + r0 + i < lim);
      v0[i] = e.alpha * a.x + b0;
      v1[i] = e.alpha * a.y + b1;
    }
    if (e.aux_mode == 2) {  // dgrad of an activation: acc * act'(pre), bias (if any) after
      float x0[8], x1[8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
        ld_pair(X + cbase + (long long)(r0 + i) * p.c_rs, p.c_cs, ok0 && in[i], ok1 && in[i], p.vec_c, x0[i], x1[i]);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        v0[i] -= b0;
        v1[i] -= b1;
      }
      dact8(code0, v0, x0);
      dact8(code1, v1, x1);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        v0[i] += b0;
        v1[i] += b1;
      }
    }
    if (e.row_limit) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (!live[i]) v0[i] = v1[i] = 0.f;
    }
    if (e.aux_mode == 1) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (in[i]) store_pair(X + cbase + (long long)(r0 + i) * p.c_rs, p.c_cs, v0[i], v1[i], ok0, ok1, p.vec_c);
    }
    if (e.aux_mode != 2 && e.n_act) {
      act8(code0, v0);
      act8(code1, v1);
      if (e.row_limit) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (!live[i]) v0[i] = v1[i] = 0.f;
      }
    }
    if (e.beta != 0.f) {
      float c0[8], c1[8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
        ld_pair(C + cbase + (long long)(r0 + i) * p.c_rs, p.c_cs, ok0 && in[i], ok1 && in[i], p.vec_c, c0[i], c1[i]);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        v0[i] += e.beta * c0[i];
        v1[i] += e.beta * c1[i];
      }
    }
    if (Rs) {
      // residual tile staged in smem by the TMA producer (row-major 64-col boxes)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int rr = rrow0 + r0 + i;
        const float2 f = __bfloat1622float2(
            *reinterpret_cast<const __nv_bfloat162*>(Rs + (rcol >> 6) * (128 * 64) + rr * 64 + (rcol & 63)));
        v0[i] += f.x;
        v1[i] += f.y;
      }
    } else if (R) {
      float q0[8], q1[8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
        ld_pair(R + rbase + (long long)(r0 + i) * p.r_rs, p.r_cs, ok0 && in[i], ok1 && in[i], p.vec_r, q0[i], q1[i]);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        v0[i] += q0[i];
        v1[i] += q1[i];
      }
    }
    if (e.row_limit && (e.beta != 0.f || R || Rs)) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (!live[i]) v0[i] = v1[i] = 0.f;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (in[i]) store_pair(C + cbase + (long long)(r0 + i) * p.c_rs, p.c_cs, v0[i], v1[i], ok0, ok1, p.vec_c);
  }
}

// MODE 2 epilogue: thread = output row.  Each 32-column TMEM slab gets the
// epilogue in registers (alpha, bias, activation, row limit, residual from the
// TMA-staged SWIZZLE_128B tile) and is written as swizzled 16-byte chunks into
// one of the warp's two 32-row x 128-byte staging boxes, which a single TMA
// store (or fp32 reduce-add, for accumulate-into-C and split-K) writes out.
// Activation of a 32-column slab sharing one code (MODE 3; bf16-operand
// GEMMs, hardware approximations: ex2/rcp/tanh.approx, rel. err <= 2^-11).
__device__ __forceinline__ float tanh_apx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_apx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// The TMA-store epilogue instantiates only the activations the model's
// GEMM epilogues use (identity, relu, silu, tanh; host-checked, others take
// the generic epilogue): every case is a 32-wide unrolled loop, and each extra
// case grows the epilogue warps' code (instruction-cache pressure).
template <int N>
__device__ __forceinline__ void act_n(int code, float* v) {
  if (code == KL_ACT_RELU) {
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = fmaxf(v[i], 0.f);
  } else if (code == KL_ACT_SILU) {
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = v[i] * rcp_apx(1.f + __expf(-v[i]));
  } else if (code == KL_ACT_TANH) {
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = tanh_apx(v[i]);
  }
}
// v *= act'(a) for the same four codes (x = pre-activation), fp32 accurate
template <int N>
__device__ __forceinline__ void dact_n(int code, float* v, const float* a) {
  if (code == KL_ACT_RELU) {
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = a[i] > 0.f ? v[i] : 0.f;
  } else if (code == KL_ACT_SILU) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const float sg = 1.f / (1.f + expf(-a[i]));
      v[i] *= sg * (1.f + a[i] * (1.f - sg));
    }
  } else if (code == KL_ACT_TANH) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const float y = tanhf(a[i]);
      v[i] *= 1.f - y * y;
    }
  }
}
// A 32-column slab: activation groups are multiples of 16 columns (host-
// checked), so each 16-column half has one code (e.g. GDPA's per-head runs
// of n_kv = 16 generated rows).
__device__ __forceinline__ void act32(const Epi& e, int n0, float* v) {
  const int c0 = epi_code(e, n0), c1 = epi_code(e, n0 + 16);
  if (c0 == c1) {
    act_n<32>(c0, v);
  } else {
    act_n<16>(c0, v);
    act_n<16>(c1, v + 16);
  }
}
__device__ __forceinline__ void dact32(const Epi& e, int n0, float* v, const float* a) {
  const int c0 = epi_code(e, n0), c1 = epi_code(e, n0 + 16);
  if (c0 == c1) {
    dact_n<32>(c0, v, a);
  } else {
    dact_n<16>(c0, v, a);
    dact_n<16>(c1, v + 16, a + 16);
  }
}

__device__ __forceinline__ void ld8_row(const float* p, float* o) {
  const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
  o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w; o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
}
__device__ __forceinline__ void ld8_row(const bf16* p, float* o) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[k]));
    o[2 * k] = f.x;
    o[2 * k + 1] = f.y;
  }
}
__device__ __forceinline__ void st8_row(float* p, const float* v, bool live) {
  *reinterpret_cast<float4*>(p) = live ? make_float4(v[0], v[1], v[2], v[3]) : make_float4(0.f, 0.f, 0.f, 0.f);
  *reinterpret_cast<float4*>(p + 4) = live ? make_float4(v[4], v[5], v[6], v[7]) : make_float4(0.f, 0.f, 0.f, 0.f);
}
__device__ __forceinline__ void st8_row(bf16* p, const float* v, bool live) {
  uint4 u = make_uint4(0u, 0u, 0u, 0u);
  if (live) {
    u.x = tc::pack_bf16(v[0], v[1]);
    u.y = tc::pack_bf16(v[2], v[3]);
    u.z = tc::pack_bf16(v[4], v[5]);
    u.w = tc::pack_bf16(v[6], v[7]);
  }
  *reinterpret_cast<uint4*>(p) = u;
}

template <typename TC, bool FULL>
__device__ __forceinline__ void epi_tma(const TcParams& p, const Epi& e, const CUtensorMap* tmC,
                                        const CUtensorMap* tmX, uint32_t tbase, uint8_t* stg, float* bsm, int mb,
                                        int nb, int zc2, int zc1, int lane_base, int lim, const uint8_t* Rs,
                                        int& nbox, TC* X, int c_lo, int c_hi, const TC* Rg) {
  // aux_mode 1 with a tensor map: the pre-activation is staged in the warp's
  // second box and TMA-stored beside C (one box pair in flight)
  const bool xtma = FULL && e.aux_mode == 1 && p.x_tma;
  const int lane = threadIdx.x & 31;
  constexpr int SPB = 128 / (int)sizeof(TC) / 32;  // 32-column slabs per 128-byte box row: 2 bf16, 1 fp32
  const int row = lane_base + lane;
  const bool live = mb * BM + row < lim;
  // (FULL: the caller staged this tile's bias in bsm before the accumulator wait)
  uint8_t* buf = stg;
  // Rg (bf16 C only): the residual of each 64-column box, loaded coalesced
  // (8 rows x 128 B per warp instruction) one box ahead into registers, then
  // put into the box's staging buffer, where each row thread adds it before
  // writing its result over it
  uint4 rnext[8];
  auto r_load = [&](int cb) {
    const int cc = lane & 7;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int R = (lane >> 3) + 4 * i, row = mb * BM + lane_base + R;
      rnext[i] = row < p.M ? __ldg(reinterpret_cast<const uint4*>(Rg + (long long)row * p.r_rs + nb * p.BN + cb + 8 * cc))
                           : make_uint4(0u, 0u, 0u, 0u);
    }
  };
  if constexpr (sizeof(TC) == 2) {
    if (Rg) r_load(c_lo);
  }
#pragma unroll 1
  for (int c = c_lo; c < c_hi; c += 32) {
    const int hb = (c >> 5) % SPB;
    if (hb == 0) {
      buf = xtma ? stg : stg + (nbox & 1) * 4096;
      if (lane == 0) {
        if (xtma)
          tc::bulk_wait_read0();
        else
          tc::bulk_wait_read1();
      }
      __syncwarp();
      if constexpr (sizeof(TC) == 2) {
        if (Rg) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int R = (lane >> 3) + 4 * i, cc = lane & 7;
            *reinterpret_cast<uint4*>(buf + R * 128 + ((cc ^ (R & 7)) << 4)) = rnext[i];
          }
          __syncwarp();
          if (c + 64 < c_hi) r_load(c + 64);
        }
      }
    }
    float v[32];
    tc::tmem_ld32(tbase + c, v);
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] *= e.alpha;
    // aux (pre-activation) row segment of this slab: thread = row, 32 columns
    const int m_row = mb * BM + row, n0 = nb * p.BN + c;
    TC* xrow = (FULL && e.aux_mode && m_row < p.M) ? X + (long long)m_row * p.c_rs + n0 : nullptr;
    if (FULL && e.aux_mode == 2 && xrow) {  // backward: v *= act'(pre-activation)
      float a[32];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (n0 + 8 * q + 8 <= p.N) {
          ld8_row(xrow + 8 * q, a + 8 * q);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) a[8 * q + i] = n0 + 8 * q + i < p.N ? ldf(xrow + 8 * q + i) : 0.f;
        }
      }
      dact32(e, n0, v, a);
    }
    if (FULL) {
      if (e.bias) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 b4 = *reinterpret_cast<const float4*>(bsm + c + 4 * q);
          v[4 * q] += b4.x;
          v[4 * q + 1] += b4.y;
          v[4 * q + 2] += b4.z;
          v[4 * q + 3] += b4.w;
        }
      }
      if (xtma) {  // forward: pre-activation -> the aux staging box (same swizzle as C)
        uint8_t* xr = stg + 4096 + lane * 128;
        if constexpr (sizeof(TC) == 2) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int chunk = hb * 4 + q;
            uint4 u = make_uint4(0u, 0u, 0u, 0u);
            if (live) {
              u.x = tc::pack_bf16(v[8 * q], v[8 * q + 1]);
              u.y = tc::pack_bf16(v[8 * q + 2], v[8 * q + 3]);
              u.z = tc::pack_bf16(v[8 * q + 4], v[8 * q + 5]);
              u.w = tc::pack_bf16(v[8 * q + 6], v[8 * q + 7]);
            }
            *reinterpret_cast<uint4*>(xr + ((chunk ^ (lane & 7)) << 4)) = u;
          }
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const uint4 u = live ? make_uint4(__float_as_uint(v[4 * q]), __float_as_uint(v[4 * q + 1]),
                                              __float_as_uint(v[4 * q + 2]), __float_as_uint(v[4 * q + 3]))
                                 : make_uint4(0u, 0u, 0u, 0u);
            *reinterpret_cast<uint4*>(xr + ((q ^ (lane & 7)) << 4)) = u;
          }
        }
      } else if (e.aux_mode == 1 && xrow) {  // forward: keep the pre-activation for the backward
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (n0 + 8 * q + 8 <= p.N) {
            st8_row(xrow + 8 * q, v + 8 * q, live);
          } else {
#pragma unroll
            for (int i = 0; i < 8; ++i)
              if (n0 + 8 * q + i < p.N) stf(xrow + 8 * q + i, live ? v[8 * q + i] : 0.f);
          }
        }
      }
      if (e.n_act && e.aux_mode != 2) act32(e, nb * p.BN + c, v);  // 16-column-uniform (host-checked)
    }
    if (Rs) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int cc = c + 8 * q;
        const uint4 u = *reinterpret_cast<const uint4*>(Rs + (cc >> 6) * 16384 + tc::sw128_off(row, cc & 63, BM));
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[k]));
          v[8 * q + 2 * k] += f.x;
          v[8 * q + 2 * k + 1] += f.y;
        }
      }
    }
    uint8_t* rowp = buf + lane * 128;
    if constexpr (sizeof(TC) == 2) {
      if (Rg) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint4 u = *reinterpret_cast<const uint4*>(rowp + (((hb * 4 + q) ^ (lane & 7)) << 4));
          const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[k]));
            v[8 * q + 2 * k] += f.x;
            v[8 * q + 2 * k + 1] += f.y;
          }
        }
      }
    }
    if (!live) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = 0.f;
    }
    if constexpr (sizeof(TC) == 2) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int chunk = hb * 4 + q;
        uint4 u;
        u.x = tc::pack_bf16(v[8 * q], v[8 * q + 1]);
        u.y = tc::pack_bf16(v[8 * q + 2], v[8 * q + 3]);
        u.z = tc::pack_bf16(v[8 * q + 4], v[8 * q + 5]);
        u.w = tc::pack_bf16(v[8 * q + 6], v[8 * q + 7]);
        *reinterpret_cast<uint4*>(rowp + ((chunk ^ (lane & 7)) << 4)) = u;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint4 u = make_uint4(__float_as_uint(v[4 * q]), __float_as_uint(v[4 * q + 1]),
                                   __float_as_uint(v[4 * q + 2]), __float_as_uint(v[4 * q + 3]));
        *reinterpret_cast<uint4*>(rowp + ((q ^ (lane & 7)) << 4)) = u;
      }
    }
    if (hb == SPB - 1 || c + 32 >= c_hi) {
      tc::fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        const int gc = nb * p.BN + c - 32 * hb, gr = mb * BM + lane_base;
        if (p.reduce_c)
          tc::tma_reduce_add_4d(tmC, buf, gc, gr, zc2, zc1);
        else
          tc::tma_store_4d(tmC, buf, gc, gr, zc2, zc1);
        if (xtma) tc::tma_store_4d(tmX, stg + 4096, gc, gr, zc2, zc1);
        tc::bulk_commit();
      }
      ++nbox;
    }
  }
  if (FULL && e.bias) __syncwarp();  // bsm rewritten for the next tile
}

// Wide tiles, bf16 C without bias / activation / residual: the accumulator
// is released BEFORE the TMA stores, so the next tile's MMAs overlap this
// tile's stores (a wide tile's 512 columns fill TMEM: there is no second
// accumulator to overlap with).  The warp's 256 columns: the first 128 are
// packed straight into its two staging boxes, the last 128 into 64 registers
// (10 warps cap a thread at 168 registers); then the accumulator barrier,
// then four box stores.
template <typename TC>
__device__ __forceinline__ void epi_wide_regs(const TcParams& p, const Epi& e, const CUtensorMap* tmC, uint32_t tbase,
                                              uint8_t* stg, int mb, int nb, int zc2, int zc1, int lane_base, int lim,
                                              int& nbox, int c_lo, uint32_t tempty_leader) {
  const int lane = threadIdx.x & 31;
  const bool live = mb * BM + lane_base + lane < lim;
  if (lane == 0) tc::bulk_wait_read0();  // the previous tile's boxes
  __syncwarp();
  uint32_t pk[64];
  auto put = [&](int s, const uint32_t* r) {
    uint32_t w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      w[i] = live ? tc::pack_bf16(__uint_as_float(r[2 * i]) * e.alpha, __uint_as_float(r[2 * i + 1]) * e.alpha) : 0u;
    if (s < 8) {
      uint8_t* row = stg + (s >> 2) * 4096 + lane * 128;
#pragma unroll
      for (int q = 0; q < 2; ++q)
        *reinterpret_cast<uint4*>(row + ((((s & 3) * 2 + q) ^ (lane & 7)) << 4)) =
            make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) pk[8 * (s - 8) + i] = w[i];
    }
  };
#pragma unroll
  for (int s = 0; s < 16; s += 2) {  // 16-column loads, two in flight per wait
    uint32_t r0[16], r1[16];
    tc::tmem_ld16_nowait(tbase + c_lo + 16 * s, r0);
    tc::tmem_ld16_nowait(tbase + c_lo + 16 * s + 16, r1);
    tc::tmem_wait_ld();
    tc::reg_fence<16>(r0);
    tc::reg_fence<16>(r1);
    put(s, r0);
    put(s + 1, r1);
  }
  tc::fence_before();
  tc::fence_async_smem();
  __syncwarp();
  const int gr = mb * BM + lane_base, gc = nb * p.BN + c_lo;
  if (lane == 0) {
    tc::mbar_arrive_cluster(tempty_leader);
    tc::tma_store_4d(tmC, stg, gc, gr, zc2, zc1);
    tc::bulk_commit();
    tc::tma_store_4d(tmC, stg + 4096, gc + 64, gr, zc2, zc1);
    tc::bulk_commit();
  }
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    uint8_t* buf = stg + b * 4096;
    if (lane == 0) tc::bulk_wait_read1();
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 8; ++q)
      *reinterpret_cast<uint4*>(buf + lane * 128 + ((q ^ (lane & 7)) << 4)) =
          make_uint4(pk[32 * b + 4 * q], pk[32 * b + 4 * q + 1], pk[32 * b + 4 * q + 2], pk[32 * b + 4 * q + 3]);
    tc::fence_async_smem();
    __syncwarp();
    if (lane == 0) {
      tc::tma_store_4d(tmC, buf, gc + 128 + 64 * b, gr, zc2, zc1);
      tc::bulk_commit();
    }
  }
  nbox += 4;
}

// MODE 0: plain store, 1: generic epilogue (lane = column pair), 2/3: TMA-store
// epilogue (thread = row; see epi_tma) without / with bias and activations.
// PAIR: a CTA pair (cluster of 2, cta_group::2) computes a 256 x BN tile —
// each CTA loads its 128 A rows and half of the tile's B columns, the leader
// issues M = 256 MMAs over both CTAs' shared memory, each CTA's TMEM holds its
// 128 rows.  Half the B operand bytes per CTA and half the MMA instructions
// per output (the single-CTA kernel is bound by L2 -> SM operand traffic at
// ~10 TB/s: ncu, c4 projections).
template <typename TC, int MODE, bool PAIR = false>
__global__ void __launch_bounds__(NTHREADS_WIDE, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmR, const __grid_constant__ CUtensorMap tmC,
                   const __grid_constant__ CUtensorMap tmX, TcParams p,
                   Epi e) {
  constexpr bool PLAIN = MODE == 0;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = sA + p.stages * p.a_stage_bytes;
  uint8_t* sR = sB + p.stages * p.b_stage_bytes;  // 2 x r_boxes x 16 KB residual tiles (TMA)
  // epilogue staging: MODE 0/1 transpose (one 32 x 64 fp32 slab per warp);
  // MODE 2 two 4 KB swizzled TMA boxes per warp
  __shared__ __align__(1024) float stage_s[4 * 32 * SLD];
  uint64_t* full = (uint64_t*)(sR + (p.r_boxes ? p.r_bufs * p.r_boxes * 16384 : 0));
  uint64_t* empty = full + p.stages;
  uint64_t* tfull = empty + p.stages;
  uint64_t* tempty = tfull + 2;
  uint64_t* rfull = tempty + 2;
  uint64_t* rempty = rfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(rempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_epi = (int)(blockDim.x >> 5) - 2;  // 4, or 8 for wide tiles
  // wide tiles: staging boxes of epilogue warps 6..9 (dynamic, 1 KB aligned, after the bias rows)
  uint8_t* sX = (uint8_t*)((((uintptr_t)(reinterpret_cast<float*>(rempty + 2 + 2) + 4 * 512)) + 1023) & ~(uintptr_t)1023);
  const uint32_t rank = PAIR ? tc::cluster_ctarank() : 0u;
  const int unit0 = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int ustep = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tmA);
    tc::prefetch_tmap(&tmB);
    if (p.r_boxes) tc::prefetch_tmap(&tmR);
    if (MODE >= 2) tc::prefetch_tmap(&tmC);
    if (MODE == 3 && p.x_tma) tc::prefetch_tmap(&tmX);
    for (int s = 0; s < p.stages; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&tfull[i], 1);
      tc::mbar_init(&tempty[i], (PAIR ? 2 : 1) * n_epi);  // pair: both CTAs' epilogue warps drain the leader's MMAs
      tc::mbar_init(&rfull[i], 1);
      tc::mbar_init(&rempty[i], 4);
    }
    tc::fence_barrier_init();
  }
  if (warp == 1) {
    if (PAIR)
      tc::tmem_alloc_pair(tmem_slot, p.tmem_cols);
    else
      tc::tmem_alloc(tmem_slot, p.tmem_cols);
  }
  tc::fence_before();
  __syncthreads();
  if (PAIR) tc::cluster_sync();  // the peer's barriers exist before any remote arrive / TMA signal
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  // PDL: the prologue above (barrier init, TMEM alloc, tensor-map prefetch)
  // overlaps the previous kernel; global memory is touched only after this
  KL_PDL_ENTRY();

  const int n_red = (p.red1 ? p.nb1 : 1) * (p.red2 ? p.nb2 : 1);
  const int iters = n_red * p.kblocks;
  const int total = p.tiles_m * p.tiles_n * p.n_out * p.splits;
  const int nb2o = p.red2 ? 1 : p.nb2;
  const int r2n = p.red2 ? p.nb2 : 1;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t tx = p.a_stage_bytes + p.b_stage_bytes;
      int t = 0;
      for (int unit = unit0; unit < total; unit += ustep, ++t) {
        const int tile = unit / p.splits, sp = unit % p.splits;
        const int it0 = (int)((long long)iters * sp / p.splits), it1 = (int)((long long)iters * (sp + 1) / p.splits);
        const int mbt = p.n_fast ? (tile / p.tiles_n) % p.tiles_m : tile % p.tiles_m;
        const int mb = PAIR ? 2 * mbt + (int)rank : mbt;  // this CTA's 128-row block
        const int nb = p.n_fast ? tile % p.tiles_n : (tile / p.tiles_m) % p.tiles_n;
        const int zo = tile / (p.tiles_m * p.tiles_n);
        const int z1o = p.red1 ? 0 : zo / nb2o, z2o = p.red2 ? 0 : zo % nb2o;
        // residual tile for this output tile: double-buffered against the
        // epilogue and issued before the tile's operand loads; single-buffered
        // (r_bufs == 1) it is issued after them, so waiting for the previous
        // tile's epilogue never holds back this tile's mainloop
        auto load_r = [&]() {
          const int rb = t % p.r_bufs;
          tc::mbar_wait(&rempty[rb], ((t / p.r_bufs) & 1) ^ 1);
          tc::mbar_arrive_expect_tx(&rfull[rb], p.r_boxes * 16384);
          for (int j = 0; j < p.r_boxes; ++j)
            tc::tma_load_4d(sR + (rb * p.r_boxes + j) * 16384, &tmR, &rfull[rb], nb * p.BN + j * 64, mb * BM,
                            p.r_has2 ? z2o : 0, p.r_has1 ? z1o : 0);
        };
        if (p.r_boxes && p.r_bufs == 2) load_r();
        for (int it = it0; it < it1; ++it) {
          const int r = it / p.kblocks, kb = it % p.kblocks;
          const int z1 = p.red1 ? r / r2n : z1o;
          const int z2 = p.red2 ? r % r2n : z2o;
          const int a1 = p.a_has1 ? z1 : 0, a2 = p.a_has2 ? z2 : 0;
          const int b1 = p.b_has1 ? z1 : 0, b2 = p.b_has2 ? z2 : 0;
          {
            tc::mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* da = sA + stage * p.a_stage_bytes;
            uint8_t* db = sB + stage * p.b_stage_bytes;
            if constexpr (PAIR) {
              // both CTAs' operand halves complete on the leader's full barrier
              if (rank == 0) tc::mbar_arrive_expect_tx(&full[stage], 2 * tx);
              const uint32_t fb = tc::mapa(&full[stage], 0);
              const int n0 = nb * p.BN + (int)rank * (p.BN / 2);
              if (!p.a_mn) {
                tc::tma_load_4d_pair(da, &tmA, fb, kb * BK, mb * BM, a2, a1);
              } else {
                tc::tma_load_4d_pair(da, &tmA, fb, mb * BM, kb * BK, a2, a1);
                tc::tma_load_4d_pair(da + 8192, &tmA, fb, mb * BM + 64, kb * BK, a2, a1);
              }
              if (p.wide) {  // columns [256 h + 128 rank, +128) of each 256-column product h
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                  const int nh = nb * p.BN + h * 256 + (int)rank * 128;
                  if (!p.b_mn) {
                    tc::tma_load_4d_pair(db + h * 16384, &tmB, fb, kb * BK, nh, b2, b1);
                  } else {
                    tc::tma_load_4d_pair(db + h * 16384, &tmB, fb, nh, kb * BK, b2, b1);
                    tc::tma_load_4d_pair(db + h * 16384 + 8192, &tmB, fb, nh + 64, kb * BK, b2, b1);
                  }
                }
              } else if (!p.b_mn) {
                tc::tma_load_4d_pair(db, &tmB, fb, kb * BK, n0, b2, b1);
              } else {
                for (int j = 0; j < p.b_boxes; ++j)
                  tc::tma_load_4d_pair(db + j * 8192, &tmB, fb, n0 + j * 64, kb * BK, b2, b1);
              }
            } else {
            tc::mbar_arrive_expect_tx(&full[stage], tx);
            if (!p.a_mn) {
              tc::tma_load_4d(da, &tmA, &full[stage], kb * BK, mb * BM, a2, a1);
            } else {
              tc::tma_load_4d(da, &tmA, &full[stage], mb * BM, kb * BK, a2, a1);
              tc::tma_load_4d(da + 8192, &tmA, &full[stage], mb * BM + 64, kb * BK, a2, a1);
            }
            if (!p.b_mn) {
              tc::tma_load_4d(db, &tmB, &full[stage], kb * BK, nb * p.BN, b2, b1);
            } else {
              for (int j = 0; j < p.b_boxes; ++j)
                tc::tma_load_4d(db + j * 8192, &tmB, &full[stage], nb * p.BN + j * 64, kb * BK, b2, b1);
            }
            }
            if (++stage == p.stages) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
        if (p.r_boxes && p.r_bufs == 1) load_r();
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // (pair: the leader issues for both CTAs)
      const uint32_t idesc = tc::idesc_bf16(PAIR ? 2 * BM : BM, p.wide ? 256 : p.BN, p.a_mn, p.b_mn);
      int stage = 0;
      uint32_t phase = 0;
      int t = 0;
      for (int unit = unit0; unit < total; unit += ustep, ++t) {
        const int sp = unit % p.splits;
        const int it0 = (int)((long long)iters * sp / p.splits), it1 = (int)((long long)iters * (sp + 1) / p.splits);
        const int acc = p.wide ? 0 : t & 1;
        const uint32_t acc_phase = p.wide ? t & 1 : (t >> 1) & 1;
        tc::mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc::fence_after();
        const uint32_t d = tmem + acc * p.acc_stride;
        for (int it = it0; it < it1; ++it) {
          tc::mbar_wait(&full[stage], phase);
          tc::fence_after();
          const uint32_t a0 = tc::smem_u32(sA + stage * p.a_stage_bytes);
          const uint32_t b0 = tc::smem_u32(sB + stage * p.b_stage_bytes);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = p.a_mn ? tc::sdesc(a0 + k * 2048, 8192, 1024) : tc::sdesc(a0 + k * 32, 16, 1024);
            const uint64_t bd = p.b_mn ? tc::sdesc(b0 + k * 2048, 8192, 1024) : tc::sdesc(b0 + k * 32, 16, 1024);
            if constexpr (PAIR) {
              tc::mma_bf16_pair(d, ad, bd, idesc, (it > it0 || k > 0) ? 1u : 0u);
              if (p.wide)
                tc::mma_bf16_pair(d + 256, ad, bd + (16384 >> 4), idesc, (it > it0 || k > 0) ? 1u : 0u);
            } else
              tc::mma_bf16(d, ad, bd, idesc, (it > it0 || k > 0) ? 1u : 0u);
          }
          if constexpr (PAIR)
            tc::mma_commit_pair(&empty[stage], 3);  // frees the stage in both CTAs
          else
            tc::mma_commit(&empty[stage]);
          if (++stage == p.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if constexpr (PAIR)
          tc::mma_commit_pair(&tfull[acc], 3);
        else
          tc::mma_commit(&tfull[acc]);
      }
    }
  } else {
    const int lane_base = (warp & 3) * 32;
    int t = 0, nbox = 0;
    for (int unit = unit0; unit < total; unit += ustep, ++t) {
      const int tile = unit / p.splits;
      const int acc = p.wide ? 0 : t & 1;
      const uint32_t acc_phase = p.wide ? t & 1 : (t >> 1) & 1;
      const int mbt = p.n_fast ? (tile / p.tiles_n) % p.tiles_m : tile % p.tiles_m;
      const int mb = PAIR ? 2 * mbt + (int)rank : mbt;
      const int nb = p.n_fast ? tile % p.tiles_n : (tile / p.tiles_m) % p.tiles_n;
      const int zo = tile / (p.tiles_m * p.tiles_n);
      const int z1o = p.red1 ? 0 : zo / nb2o, z2o = p.red2 ? 0 : zo % nb2o;
      TC* C = (TC*)p.C + (long long)z1o * (p.red1 ? 0 : p.c_s1) + (long long)z2o * (p.red2 ? 0 : p.c_s2);
      const TC* R = p.R ? (const TC*)p.R + (long long)z1o * (p.red1 ? 0 : p.r_s1) + (long long)z2o * (p.red2 ? 0 : p.r_s2)
                        : nullptr;
      TC* X = p.aux ? (TC*)p.aux + (long long)z1o * (p.red1 ? 0 : p.c_s1) + (long long)z2o * (p.red2 ? 0 : p.c_s2)
                    : nullptr;
      const int lim = e.row_limit ? e.row_limit[zo] : 0x7fffffff;
      const int m0 = mb * BM + lane_base;
      float* stg = stage_s + (warp - 2) * (32 * SLD);
      // this warp's columns of the tile (wide tiles: one half per 4 warps) and its bias row
      const int ch = (warp - 2) >> 2, cw = p.BN / (n_epi >> 2), c_lo = ch * cw;
      float* bsm = reinterpret_cast<float*>(rempty + 2 + 2) + (warp - 2) * (n_epi == 8 ? 256 : 512);
      if (MODE == 3 && e.bias) {
        // this tile's bias -> the warp's smem row, while the tile's MMAs run
        // (read back as broadcasts by epi_tma)
        for (int c = c_lo + lane; c < c_lo + cw; c += 32) {
          const int n = nb * p.BN + c;
          bsm[c - c_lo] = n < p.N ? __ldg(&e.bias[n]) : 0.f;
        }
        __syncwarp();
      }
      tc::mbar_wait(&tfull[acc], acc_phase);
      tc::fence_after();
      const uint32_t tbase = tmem + acc * p.acc_stride + ((uint32_t)lane_base << 16);
      const int rows = min(32, p.M - m0);
      if constexpr (MODE >= 2) {
        const uint8_t* Rs = nullptr;
        if (p.r_boxes) {
          tc::mbar_wait(&rfull[t % p.r_bufs], (t / p.r_bufs) & 1);
          Rs = sR + (t % p.r_bufs) * p.r_boxes * 16384;
        }
        // 8 epilogue warps (wide tiles): warps 6..9 take the upper column half,
        // staged in dynamic shared memory after the operand ring
        uint8_t* ebuf = ch == 0 ? reinterpret_cast<uint8_t*>(stage_s) + (warp - 2) * 8192
                                : sX + (warp - 6) * 8192;
        if (MODE == 2 && PAIR && sizeof(TC) == 2 && p.wide && !p.reduce_c && !Rs && !p.r_glob && !p.epi_regs_off) {
          epi_wide_regs<TC>(p, e, &tmC, tbase, ebuf, mb, nb, p.c_has2 ? z2o : 0, p.c_has1 ? z1o : 0, lane_base,
                            lim, nbox, ch * cw, tc::mapa(&tempty[acc], 0));
          continue;  // accumulator already released
        }
        epi_tma<TC, MODE == 3>(p, e, &tmC, &tmX, tbase, ebuf, bsm - c_lo, mb, nb,
                    p.c_has2 ? z2o : 0, p.c_has1 ? z1o : 0, lane_base, lim, Rs, nbox, X, ch * cw, ch * cw + cw,
                    p.r_glob ? R : nullptr);
      } else
      for (int c0 = 0; c0 < p.BN; c0 += 64) {
        // TMEM (thread = row) -> smem transpose -> each lane owns a column
        // pair and walks the warp's 32 rows: every global access of a warp is
        // one contiguous 128 B (bf16) / 256 B (fp32) row segment.
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          if (c0 + 16 * q4 < p.BN) {
            float v[16];
            tc::tmem_ld16(tbase + c0 + 16 * q4, v);
#pragma unroll
            for (int j = 0; j < 16; j += 2)
              *reinterpret_cast<float2*>(&stg[lane * SLD + 16 * q4 + j]) = make_float2(v[j], v[j + 1]);
          }
        }
        __syncwarp();
        const int cl = c0 + 2 * lane;
        const int n = nb * p.BN + cl;
        const bool ok0 = cl < p.BN && n < p.N, ok1 = cl + 1 < p.BN && n + 1 < p.N;
        if (p.splits > 1 && p.ws) {
          // split-K partial tile -> workspace; a second pass reduces + applies the epilogue
          float* wp = p.ws + ((long long)(unit % p.splits) * p.n_out + zo) * p.M * p.N + (long long)m0 * p.N + n;
          for (int r = 0; r < rows; ++r) {
            const float2 a = *reinterpret_cast<const float2*>(&stg[r * SLD + 2 * lane]);
            store_pair(wp + (long long)r * p.N, 1, a.x, a.y, ok0, ok1, (p.N % 2) == 0);
          }
        } else if (p.splits > 1) {
          // split-K partial: C += alpha * partial (fp32, beta == 1 accumulate)
          float* cp = (float*)C + (long long)m0 * p.c_rs + (long long)n * p.c_cs;
          for (int r = 0; r < rows; ++r) {
            const float2 a = *reinterpret_cast<const float2*>(&stg[r * SLD + 2 * lane]);
            if (ok0) atomicAdd(cp + (long long)r * p.c_rs, e.alpha * a.x);
            if (ok1) atomicAdd(cp + (long long)r * p.c_rs + p.c_cs, e.alpha * a.y);
          }
        } else if (PLAIN) {
          TC* cp = C + (long long)m0 * p.c_rs + (long long)n * p.c_cs;
#pragma unroll 4
          for (int r = 0; r < rows; ++r) {
            const float2 a = *reinterpret_cast<const float2*>(&stg[r * SLD + 2 * lane]);
            store_pair(cp + (long long)r * p.c_rs, p.c_cs, a.x, a.y, ok0, ok1, p.vec_c);
          }
        } else {
          const bf16* Rs = nullptr;
          if (p.r_boxes) {
            if (c0 == 0) tc::mbar_wait(&rfull[t % p.r_bufs], (t / p.r_bufs) & 1);
            Rs = reinterpret_cast<const bf16*>(sR + (t % p.r_bufs) * p.r_boxes * 16384);
          }
          epi_generic(p, e, stg, C, R, X, m0, rows, n, ok0, ok1, lim, Rs, lane_base, cl);
        }
        __syncwarp();
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR)
          tc::mbar_arrive_cluster(tc::mapa(&tempty[acc], 0));  // the leader's accumulator barrier
        else
          tc::mbar_arrive(&tempty[acc]);
        if (p.r_boxes) tc::mbar_arrive(&rempty[t % p.r_bufs]);
      }
    }
    if (MODE >= 2 && lane == 0) tc::bulk_wait0();
  }
  __syncthreads();
  if (PAIR) {
    tc::cluster_sync();  // no remote arrive / operand read of the peer is still in flight
    if (warp == 1) tc::tmem_dealloc_pair(tmem, p.tmem_cols);
  } else if (warp == 1) {
    tc::tmem_dealloc(tmem, p.tmem_cols);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

// 4-D bf16 tensor map: dims (inner, outer, b2, b1), element strides; a batch
// dim with stride 0 (broadcast) becomes extent 1.
bool make_map(CUtensorMap* m, const void* ptr, long long inner, long long outer, long long s_outer, int nb2,
              long long s2, int nb1, long long s1, uint32_t box_inner, uint32_t box_outer, int* has2, int* has1,
              bool swizzle = true, int esz = 2) {
  auto fn = encode_fn();
  if (!fn) return false;
  *has2 = (s2 != 0 && nb2 > 1);
  *has1 = (s1 != 0 && nb1 > 1);
  cuuint64_t dims[4] = {(cuuint64_t)inner, (cuuint64_t)outer, (cuuint64_t)(*has2 ? nb2 : 1),
                        (cuuint64_t)(*has1 ? nb1 : 1)};
  long long so = s_outer * esz;
  long long b2 = *has2 ? s2 * esz : std::max<long long>(so * outer, 16);
  long long b1 = *has1 ? s1 * esz : std::max<long long>(b2 * (long long)dims[2], 16);
  auto bad = [](long long s) { return s <= 0 || (s % 16) != 0 || s >= (1ll << 40); };
  if (bad(so) || bad(b2) || bad(b1)) return false;
  b2 = (b2 + 15) / 16 * 16;
  b1 = (b1 + 15) / 16 * 16;
  cuuint64_t strides[3] = {(cuuint64_t)so, (cuuint64_t)b2, (cuuint64_t)b1};
  cuuint32_t box[4] = {box_inner, box_outer, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(m, esz == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4,
                  const_cast<void*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace

int gemm_path();

// KL_GEMM_PAIR=0 keeps every GEMM on single CTAs (A/B testing).
static bool getenv_flag_nopair() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("KL_GEMM_PAIR");
    v = (e && e[0] == '0') ? 1 : 0;
  }
  return v == 1;
}
// KL_GEMM_EPI1=1 forces the MODE 0/1 epilogues (A/B testing).
static bool getenv_flag_epi1() {
  static int v = -1;
  if (v < 0) v = getenv("KL_GEMM_EPI1") ? 1 : 0;
  return v == 1;
}

static int r_wide_kb() {  // KL_GEMM_RWIDE_KB: min k-blocks for 256-wide residual tiles (A/B)
  static int v = -1;
  if (v < 0) v = getenv("KL_GEMM_RWIDE_KB") ? atoi(getenv("KL_GEMM_RWIDE_KB")) : 4;
  return v;
}

static double ws_penalty() {  // KL_GEMM_WS_PENALTY: cost (clk) of the split-K reduce pass's extra launch (A/B)
  static double v = -1.0;
  if (v < 0) v = getenv("KL_GEMM_WS_PENALTY") ? atof(getenv("KL_GEMM_WS_PENALTY")) : 2000.0;
  return v;
}

static int wide_min_k() {  // KL_GEMM_WIDE_K: shortest reduction of a stored-output wide GEMM (A/B)
  static int v = -1;
  if (v < 0) v = getenv("KL_GEMM_WIDE_K") ? atoi(getenv("KL_GEMM_WIDE_K")) : 512;
  return v;
}

int gemm_tc(const GemmDesc& g0, const Epi& e0, cudaStream_t s) {
  if (g0.ab_dtype != KL_BF16) return KL_EUNSUPPORTED;
  if (!kl_tcgen05_available()) return KL_EUNSUPPORTED;
  // small problems go to the SIMT kernel unless forced
  // (counting every batch: a batch of small products fills the SMs with tiles)
  if (gemm_path() != 2 && (long long)g0.M * g0.N * g0.K * g0.nb1 * g0.nb2 < (1ll << 18)) return KL_EUNSUPPORTED;
  GemmDesc g = g0;
  Epi e = e0;
  // column-major C with an element-wise-free epilogue: compute C^T = B^T A^T
  // instead, so C rows are contiguous for the TMA-store epilogue (operand
  // majors swap roles; the kernel takes either major for A and B)
  if (g.c_cs != 1 && g.c_rs == 1 && !e.bias && !e.aux_mode && e.n_act == 0 && !e.row_limit && !g.R) {
    std::swap(g.M, g.N);
    std::swap(g.A, g.B);
    const long long ars = g.a_rs, acs = g.a_cs, as1 = g.a_s1, as2 = g.a_s2;
    g.a_rs = g.b_cs;
    g.a_cs = g.b_rs;
    g.a_s1 = g.b_s1;
    g.a_s2 = g.b_s2;
    g.b_rs = acs;
    g.b_cs = ars;
    g.b_s1 = as1;
    g.b_s2 = as2;
    std::swap(g.c_rs, g.c_cs);
  }
  // C += ... on a bf16 output is the residual epilogue with R = C
  if (g.c_dtype == KL_BF16 && e.beta == 1.f && !g.R) {
    g.R = g.C;
    g.r_rs = g.c_rs;
    g.r_cs = g.c_cs;
    g.r_s1 = g.red1 ? 0 : g.c_s1;
    g.r_s2 = g.red2 ? 0 : g.c_s2;
    e.beta = 0.f;
  }
  const bool a_k = (g.a_cs == 1), a_m = (g.a_rs == 1) && !a_k;
  const bool b_k = (g.b_rs == 1), b_n = (g.b_cs == 1) && !b_k;
  if (!(a_k || a_m) || !(b_k || b_n)) return KL_EUNSUPPORTED;
  if (((uintptr_t)g.A & 15) || ((uintptr_t)g.B & 15)) return KL_EUNSUPPORTED;

  TcParams p{};
  p.M = g.M;
  p.N = g.N;
  p.K = g.K;
  // residual tiles arrive by TMA when their layout allows (bf16, unit column
  // stride, 16-byte aligned rows); those GEMMs use N tiles of <= 128 so the
  // double-buffered residual fits next to the operand ring.
  CUtensorMap tr;
  bool use_r = g.R && g.c_dtype == KL_BF16 && g.r_cs == 1 && !g.red1 && !g.red2;
  // residual tiles are double-buffered next to the operand ring with N tiles
  // of <= 128; a reduction of >= 4 k-blocks (the epilogue of one tile has a
  // mainloop to finish before the next residual tile is needed) may take
  // 256-wide tiles with a single residual buffer (measured: out-projection
  // 47 -> 40 us, QKV dX 105 -> 80 us at c2)
  const bool r_wide = use_r && (g.K + BK - 1) / BK >= r_wide_kb();
  const int bn_max = use_r && !r_wide ? 128 : 256;
  const int n_out0 = (g.red1 ? 1 : g.nb1) * (g.red2 ? 1 : g.nb2);
  const long long k_tot = (long long)((g.red1 ? g.nb1 : 1) * (g.red2 ? g.nb2 : 1)) * g.K;
  // N tiles are whole TMA-store boxes: 128-byte rows, i.e. 64 bf16 or 32 fp32
  // columns.  (A 96-column bf16 tile would store its last half-filled
  // 64-column box over the neighbouring tile's first 32 columns.)
  const int box_cols = g.c_dtype == KL_BF16 ? 64 : 32;
  auto split_n = [&](int cap) {
    int tn = (g.N + cap - 1) / cap;
    int b = (g.N + tn - 1) / tn;
    b = (b + box_cols - 1) / box_cols * box_cols;
    return std::min(b, std::max(cap, box_cols));
  };
  int bn = split_n(bn_max);
  // Split-K plan for a tile count: weight-gradient shapes (few output tiles,
  // a long reduction) spread the reduction over the SMs; with an fp32
  // accumulate-only epilogue the partial tiles add with fp32 atomics, any
  // other epilogue goes through fp32 partials in the workspace + one reduce /
  // epilogue pass.  Returns the split count; *ws_path tells which.
  const bool accum_only = g.c_dtype == KL_F32 && e.beta == 1.f && !e.bias && !e.row_limit && !e.aux_mode &&
                          e.n_act == 0 && !g.R;
  const int kblocks0 = (g.K + BK - 1) / BK;
  const int iters0 = ((g.red1 ? g.nb1 : 1) * (g.red2 ? g.nb2 : 1)) * kblocks0;
  auto plan_splits = [&](long long tiles, bool* ws_path) {
    *ws_path = false;
    if (accum_only && tiles < num_sms() && iters0 >= 8)
      return (int)std::max<long long>(1, std::min<long long>(num_sms() / tiles, iters0 / 4));
    if (!accum_only && g.ws && tiles * 2 <= num_sms() && iters0 >= 8 && !use_r) {
      int sp = (int)std::max<long long>(1, std::min<long long>(num_sms() / tiles, iters0 / 4));
      const long long per = (long long)n_out0 * g.M * g.N * 4;
      while (sp > 1 && per * sp > g.ws_bytes) --sp;
      if (sp > 1) {
        *ws_path = true;
        return sp;
      }
    }
    return 1;
  };
  {
    // Tile width from a cycle model of one SM: a 128 x BN tile streams
    // (128 + BN) bf16 operand columns per k (~64 B/clk of L2 bandwidth per SM)
    // and issues 128*BN MACs per k (~2780 MAC/clk dense bf16), plus a fixed
    // pipeline fill and a BN-wide epilogue; total = waves x tile cost (+ the
    // workspace split-K reduce).  Few M tiles -> narrower N tiles or split-K
    // instead of idle SMs.
    const int tiles_m0 = (g.M + BM - 1) / BM;
    double best = -1.0;
    const int caps[4] = {256, 128, 64, 32};
    for (int ci = 0; ci < 4; ++ci) {
      const int cap = caps[ci];
      if (cap > bn_max) continue;
      // MN-major B is staged in 64-column boxes; bf16 C is stored in 64-column
      // TMA boxes: neither may be split below 64 columns
      if (cap < 64 && (!b_k || g.c_dtype == KL_BF16)) continue;
      const int b = split_n(cap);
      const long long tiles = (long long)tiles_m0 * ((g.N + b - 1) / b) * n_out0;
      bool wsp = false;
      const int sp = plan_splits(tiles, &wsp);
      const long long waves = (tiles * sp + num_sms() - 1) / num_sms();
      const double per_k = std::max(128.0 * b / 2780.0, (128.0 + b) * 2.0 / 64.0);
      double cost = (double)waves * ((double)k_tot / sp * per_k + 500.0 + 4.0 * b);
      if (wsp) cost += (double)n_out0 * g.M * g.N * 4.0 * (sp + 1) / 3100.0 + ws_penalty();
      if (best < 0 || cost < best * 0.97) {  // ties -> the wider tile
        best = cost;
        bn = b;
      }
    }
    static int force = -1;
    if (force < 0) {
      const char* v = getenv("KL_GEMM_BN");
      force = v ? atoi(v) : 0;
    }
    if (force >= 16) bn = std::min(split_n(bn_max), (force + box_cols - 1) / box_cols * box_cols);
  }
  p.BN = bn;
  p.tiles_n = (g.N + bn - 1) / bn;
  p.tiles_m = (g.M + BM - 1) / BM;
  // Tile order.  M-adjacent (default): the CTAs of one wave share an N tile,
  // so B is read once and A streams.  When A (M x K per output batch) is
  // larger than the L2 can keep across the N passes and the larger operand,
  // M-adjacent re-reads A from HBM once per N tile (ncu, c4 QKV projection:
  // 803 MB DRAM reads for a 134 MB A); N-adjacent makes the tiles_n CTAs that
  // share an A block run in the same wave.
  {
    const long long a_bytes = (long long)g.M * g.K * 2, b_bytes = (long long)g.N * g.K * 2;
    int nf = p.tiles_n > 1 && a_bytes > b_bytes && a_bytes > (48LL << 20) ? 1 : 0;
    if (const char* v = getenv("KL_GEMM_NFAST")) nf = atoi(v);  // A/B testing
    p.n_fast = nf;
  }
  p.nb1 = g.nb1;
  p.nb2 = g.nb2;
  p.red1 = g.red1;
  p.red2 = g.red2;
  p.n_out = (g.red1 ? 1 : g.nb1) * (g.red2 ? 1 : g.nb2);
  p.kblocks = (g.K + BK - 1) / BK;
  p.a_mn = a_m ? 1 : 0;
  p.b_mn = b_n ? 1 : 0;
  p.b_boxes = b_n ? (bn + 63) / 64 : 1;
  p.a_stage_bytes = BM * BK * 2;
  p.b_stage_bytes = b_n ? p.b_boxes * 64 * BK * 2 : bn * BK * 2;
  const uint32_t stage = p.a_stage_bytes + p.b_stage_bytes;
  // MODE 2 (TMA-store epilogue): contiguous, 16-byte aligned C rows (and aux
  // rows, written / read per thread-row beside the TMA store), N tiles in
  // 32-column slabs; fp32 C only plain (beta 0) or
  // accumulate-only (beta 1 -> TMA reduce-add).
  const int esz_c = g.c_dtype == KL_BF16 ? 2 : 4;
  const bool accum_only0 = g.c_dtype == KL_F32 && e.beta == 1.f && !e.bias && !e.row_limit && !e.aux_mode &&
                           e.n_act == 0 && !g.R;
  bool mode2 = !getenv_flag_epi1() && g.c_cs == 1 && ((uintptr_t)g.C & 15) == 0 && (g.c_rs * esz_c) % 16 == 0 &&
               (g.c_s1 * esz_c) % 16 == 0 && (g.c_s2 * esz_c) % 16 == 0 &&
               (!e.aux_mode || (g.aux && ((uintptr_t)g.aux & 15) == 0)) && bn % 32 == 0 &&
               (g.c_dtype == KL_BF16 ? e.beta == 0.f : (e.beta == 0.f && !g.R) || accum_only0) &&
               (!g.R || use_r) && (e.n_act <= 1 || (e.act_group > 0 && e.act_group % 16 == 0));
  for (int i = 0; i < e.n_act && mode2; ++i) {
    const int c = e.act_codes[i];
    mode2 = c == KL_ACT_IDENTITY || c == KL_ACT_RELU || c == KL_ACT_SILU || c == KL_ACT_TANH;
  }
  if (use_r) {
    int h2 = 0, h1 = 0;
    use_r = ((uintptr_t)g.R & 15) == 0 &&
            make_map(&tr, g.R, g.N, g.M, g.r_rs, g.nb2, g.r_s2, g.nb1, g.r_s1, 64, BM, &h2, &h1, mode2);
    p.r_has2 = h2;
    p.r_has1 = h1;
    if (!use_r) mode2 = false;
  }
  CUtensorMap tc_map;
  if (mode2) {
    int h2 = 0, h1 = 0;
    const long long s1c = g.red1 ? 0 : g.c_s1, s2c = g.red2 ? 0 : g.c_s2;
    mode2 = make_map(&tc_map, g.C, g.N, g.M, g.c_rs, g.red2 ? 1 : g.nb2, s2c, g.red1 ? 1 : g.nb1, s1c,
                     128 / esz_c, 32, &h2, &h1, true, esz_c);
    p.c_has2 = h2;
    p.c_has1 = h1;
    p.reduce_c = accum_only0 ? 1 : 0;
  }
  CUtensorMap tx_map;
  p.x_tma = 0;
  if (mode2 && e.aux_mode == 1 && g.aux && ((uintptr_t)g.aux & 15) == 0) {
    int h2 = 0, h1 = 0;
    const long long s1c = g.red1 ? 0 : g.c_s1, s2c = g.red2 ? 0 : g.c_s2;
    p.x_tma = make_map(&tx_map, g.aux, g.N, g.M, g.c_rs, g.red2 ? 1 : g.nb2, s2c, g.red1 ? 1 : g.nb1, s1c,
                       128 / esz_c, 32, &h2, &h1, true, esz_c) && h2 == p.c_has2 && h1 == p.c_has1;
  }
  // CTA pairs (cta_group::2) for the TMA-store epilogues on N tiles of 128 /
  // 256 with at least two 128-row blocks; the workspace split-K path and the
  // MODE 0/1 epilogues stay single-CTA.
  // Only for long mainloops (K >= 512) over at least two waves of tiles: a
  // pair needs both SMs of a TPC free at once, which costs overlap with the
  // concurrent graph branches on short GEMMs (measured: c2, K = 256, step
  // 6.20 -> 6.37 ms with pairs everywhere; c4 29.9 -> 29.4 ms).
  const long long tiles128 = (long long)((g.M + BM - 1) / BM) * ((g.N + bn - 1) / bn) * n_out0;
  bool pair = mode2 && bn % 128 == 0 && (g.M + BM - 1) / BM >= 2 && k_tot >= 512 && tiles128 >= 2LL * num_sms() &&
              !getenv_flag_nopair();
  if (pair) {  // the split plan the launch below makes for the pair tile count must not use the workspace
    bool wsp = false;
    const long long tiles2 = (long long)((g.M + 2 * BM - 1) / (2 * BM)) * p.tiles_n * p.n_out;
    if (plan_splits(tiles2, &wsp) > 1 && wsp) pair = false;
  }
  // Wide CTA pairs for the weight-gradient shapes (fp32 accumulate-only, a
  // long reduction split over the SMs, N a multiple of 512): 256 x 512 tiles
  // stage 48 KB of operands per 2 x 128 x 256 x 64 MACs per CTA (47 B/clk at
  // the MMA rate) where single-CTA 128 x 256 tiles need 94 B/clk — above the
  // ~60 B/clk/SM the TMA delivers with every SM loading (measured,
  // scripts/r2/micro/tma_lat.cu).  One 512-column accumulator: the epilogue
  // (once per long split) is not overlapped.
  // Stored outputs (bf16 / plain fp32): the 512-column epilogue is not
  // overlapped with the next tile's mainloop, so it runs on 8 warps (two
  // column halves per TMEM lane quarter); with 4 warps a K = 512 tile lost
  // more than the operand bytes saved (QKV projection 199 -> 219 us), with 8:
  // QKV projection 208 -> 204 us, HSP dS (K = 640) 102 -> 86 us, QKV dX
  // (K = 1536) 188 -> 164 us, 8192^3 936 -> 700 us.
  // a residual (bf16 C, unit column stride, 16-byte rows: what use_r checked) is read by the wide
  // epilogue itself (TcParams::r_glob) instead of producer-staged 128 KB tiles
  // (the extra residual reads of the un-overlapped epilogue pay off only for long reductions:
  // QKV dX, K = 1536, 211 -> 191 us; K = 512 / 640: 102 -> 116 / 112 -> 125 us)
  const bool r_ok = !use_r || (g.r_cs == 1 && (g.r_rs % 8) == 0 && ((uintptr_t)g.R & 15) == 0 && k_tot >= 1536 &&
                               !getenv("KL_GEMM_NOWIDE_R"));
  const bool wide = mode2 && r_ok && g.N % 512 == 0 && (g.M + BM - 1) / BM >= 2 && !getenv_flag_nopair() &&
                    !getenv("KL_GEMM_NOWIDE") &&
                    ((accum_only0 && !pair && k_tot >= 8192) ||
                     (!accum_only0 && k_tot >= wide_min_k() &&
                      (long long)((g.M + 2 * BM - 1) / (2 * BM)) * (g.N / 512) * n_out0 >= num_sms() / 2));
  if (wide) {
    pair = true;
    bn = 512;
    p.BN = 512;
    p.tiles_n = g.N / 512;
    if (use_r) {
      p.r_glob = 1;
      use_r = false;
    }
  }
  p.wide = wide ? 1 : 0;
  if (pair) {
    p.tiles_m = (g.M + 2 * BM - 1) / (2 * BM);
    p.b_boxes = wide ? 4 : (b_n ? (bn / 2 + 63) / 64 : 1);
    p.b_stage_bytes = wide ? 2 * 128 * BK * 2 : (b_n ? p.b_boxes * 64 * BK * 2 : (bn / 2) * BK * 2);
  }
  const uint32_t stage_p = p.a_stage_bytes + p.b_stage_bytes;
  p.r_boxes = use_r ? (bn + 63) / 64 : 0;
  p.r_bufs = bn > 128 ? 1 : 2;
  const uint32_t rbytes = (uint32_t)p.r_bufs * p.r_boxes * 16384;
  // dynamic smem budget: 227 KB minus the 33 KB static epilogue staging
  p.stages = std::min<int>(8, (int)((188 * 1024 - rbytes) / stage_p));
  if (p.stages < 2) return KL_EUNSUPPORTED;
  p.acc_stride = bn > 128 ? 256 : (bn > 64 ? 128 : (bn > 32 ? 64 : 32));
  p.tmem_cols = 2 * p.acc_stride;
  if (wide) {
    p.acc_stride = 0;
    p.tmem_cols = 512;
  }
  if (p.tmem_cols < 32) p.tmem_cols = 32;

  CUtensorMap ta, tb;
  if (a_k) {
    if (!make_map(&ta, g.A, g.K, g.M, g.a_rs, g.nb2, g.a_s2, g.nb1, g.a_s1, BK, BM, &p.a_has2, &p.a_has1))
      return KL_EUNSUPPORTED;
  } else {
    if (!make_map(&ta, g.A, g.M, g.K, g.a_cs, g.nb2, g.a_s2, g.nb1, g.a_s1, 64, BK, &p.a_has2, &p.a_has1))
      return KL_EUNSUPPORTED;
  }
  if (b_k) {
    if (!make_map(&tb, g.B, g.K, g.N, g.b_cs, g.nb2, g.b_s2, g.nb1, g.b_s1, BK, wide ? 128 : (pair ? bn / 2 : bn),
                  &p.b_has2, &p.b_has1))
      return KL_EUNSUPPORTED;
  } else {
    if (!make_map(&tb, g.B, g.N, g.K, g.b_rs, g.nb2, g.b_s2, g.nb1, g.b_s1, 64, BK, &p.b_has2, &p.b_has1))
      return KL_EUNSUPPORTED;
  }
  p.C = g.C;
  p.c_rs = g.c_rs;
  p.c_cs = g.c_cs;
  p.c_s1 = g.c_s1;
  p.c_s2 = g.c_s2;
  p.R = g.R;
  p.r_rs = g.r_rs;
  p.r_cs = g.r_cs;
  p.r_s1 = g.r_s1;
  p.r_s2 = g.r_s2;
  p.aux = g.aux;
  {
    const int esz = g.c_dtype == KL_BF16 ? 2 : 4;
    auto al = [&](const void* q) { return ((uintptr_t)q % (2 * esz)) == 0; };
    p.vec_c = g.c_cs == 1 && g.c_rs % 2 == 0 && (g.c_s1 % 2 == 0) && (g.c_s2 % 2 == 0) && al(g.C) &&
              (!g.aux || al(g.aux));
    p.vec_r = g.R && g.r_cs == 1 && g.r_rs % 2 == 0 && (g.r_s1 % 2 == 0) && (g.r_s2 % 2 == 0) && al(g.R);
  }

  const size_t smem = 1024 + (size_t)p.stages * stage_p + rbytes + (2 * p.stages + 8) * 8 + 16 + 4 * 512 * 4 +
                      (wide ? 1024 + 4 * 8192 : 0);
  const int nthreads = wide ? NTHREADS_WIDE : NTHREADS;
  const int tiles = p.tiles_m * p.tiles_n * p.n_out;
  const int iters = ((g.red1 ? g.nb1 : 1) * (g.red2 ? g.nb2 : 1)) * p.kblocks;
  p.ws = nullptr;
  {
    bool wsp = false;
    p.splits = plan_splits(tiles, &wsp);
    if (wsp) p.ws = g.ws;
    if (wide) {  // units are CTA pairs: one wave of num_sms / 2 pairs; stored outputs are not split
      p.ws = nullptr;
      p.splits = accum_only0 ? std::max(1, std::min(num_sms() / 2 / std::max(tiles, 1), iters / 4)) : 1;
    }
  }
  {
    static int off = -1;
    if (off < 0) off = (getenv("KL_GEMM_EPI_REGS") && getenv("KL_GEMM_EPI_REGS")[0] == '0') ? 1 : 0;
    p.epi_regs_off = off;
  }
  const int total = tiles * p.splits;
  const int grid = pair ? 2 * std::min(total, num_sms() / 2) : std::min(total, num_sms());
  const bool plain = e.alpha == 1.f && e.beta == 0.f && !e.bias && !e.row_limit && !e.aux_mode && e.n_act == 0 &&
                     !g.R;
  {
    static int trace = -1;
    if (trace < 0) trace = getenv("KL_GEMM_TRACE") ? 1 : 0;
    if (trace)
      fprintf(stderr, "gemm_tc M=%d N=%d K=%d nb=%dx%d red=%d%d c=%s beta=%g bias=%d aux=%d act=%d/%d R=%d lim=%d "
              "mode2=%d bn=%d splits=%d ws=%d pair=%d wide=%d stages=%d\n", g.M, g.N, g.K, g.nb1, g.nb2, g.red1, g.red2,
              g.c_dtype == KL_BF16 ? "bf16" : "f32", e.beta, e.bias != nullptr, e.aux_mode, e.n_act, e.act_group,
              g.R != nullptr, e.row_limit != nullptr, (int)mode2, bn, p.splits, p.ws != nullptr, (int)(pair && !p.ws),
              p.wide, p.stages);
  }
  auto launch = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_k(kern, grid, nthreads, smem, s, ta, tb, use_r ? tr : ta, mode2 ? tc_map : ta, p.x_tma ? tx_map : ta, p,
             e);
  };
  auto launch_pair = [&](auto kern) {  // clusters of 2 CTAs (a TPC's two SMs)
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(nthreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    cudaLaunchKernelEx(&cfg, kern, ta, tb, use_r ? tr : ta, mode2 ? tc_map : ta, p.x_tma ? tx_map : ta, p, e);
  };
  if (pair && !p.ws) {
    const bool full = e.bias || e.n_act || e.aux_mode;
    if (g.c_dtype == KL_BF16)
      full ? launch_pair(gemm_tc_kernel<bf16, 3, true>) : launch_pair(gemm_tc_kernel<bf16, 2, true>);
    else
      full ? launch_pair(gemm_tc_kernel<float, 3, true>) : launch_pair(gemm_tc_kernel<float, 2, true>);
  } else if (mode2 && !p.ws) {
    const bool full = e.bias || e.n_act || e.aux_mode;
    if (g.c_dtype == KL_BF16) full ? launch(gemm_tc_kernel<bf16, 3>) : launch(gemm_tc_kernel<bf16, 2>);
    else full ? launch(gemm_tc_kernel<float, 3>) : launch(gemm_tc_kernel<float, 2>);
  } else if (g.c_dtype == KL_BF16) {
    if (plain) launch(gemm_tc_kernel<bf16, 0>);
    else launch(gemm_tc_kernel<bf16, 1>);
  } else {
    if (plain) launch(gemm_tc_kernel<float, 0>);
    else launch(gemm_tc_kernel<float, 1>);
  }
  count_launch();
  count_path(KL_PATH_GEMM_TC);
  if (wide) count_path(KL_PATH_GEMM_WIDE);
  int rc = launch_check("gemm_tc");
  if (rc || !p.ws) return rc;
  return splitk_reduce(g, e, p.ws, p.splits, p.n_out, s);
}

}  // namespace kl

namespace kl {
PFN_cuTensorMapEncodeTiled_v12000 tc_encode_fn() { return encode_fn(); }
int tc_num_sms() { return num_sms(); }
}  // namespace kl

namespace kl {
// Sum the split-K partials and apply the full epilogue (element-wise).
template <typename TC>
__global__ void __launch_bounds__(256) splitk_reduce_kernel(GemmDesc g, Epi e, const float* ws, int splits, int n_out) {
  KL_PDL_ENTRY();
  const long long MN = (long long)g.M * g.N, total = MN * n_out;
  const int nb2o = g.red2 ? 1 : g.nb2;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int zo = (int)(i / MN);
    const long long mn = i % MN;
    const int m = (int)(mn / g.N), n = (int)(mn % g.N);
    // independent partial sums: the split loads are issued back to back
    // instead of one dependent L2 round trip per split
    float a4[4] = {0.f, 0.f, 0.f, 0.f};
    int s = 0;
    for (; s + 4 <= splits; s += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) a4[u] += ws[(long long)(s + u) * total + i];
    }
    for (; s < splits; ++s) a4[0] += ws[(long long)s * total + i];
    const float acc = (a4[0] + a4[1]) + (a4[2] + a4[3]);
    const int z1o = g.red1 ? 0 : zo / nb2o, z2o = g.red2 ? 0 : zo % nb2o;
    TC* C = (TC*)g.C + (long long)z1o * (g.red1 ? 0 : g.c_s1) + (long long)z2o * (g.red2 ? 0 : g.c_s2);
    const TC* R = g.R ? (const TC*)g.R + (long long)z1o * (g.red1 ? 0 : g.r_s1) + (long long)z2o * (g.red2 ? 0 : g.r_s2)
                      : nullptr;
    TC* X = g.aux ? (TC*)g.aux + (long long)z1o * (g.red1 ? 0 : g.c_s1) + (long long)z2o * (g.red2 ? 0 : g.c_s2)
                  : nullptr;
    const int lim = e.row_limit ? e.row_limit[zo] : 0x7fffffff;
    epilogue_store(e, C, R, X, (long long)m * g.c_rs + (long long)n * g.c_cs,
                   (long long)m * g.r_rs + (long long)n * g.r_cs, m, n, lim, acc);
  }
}


int splitk_reduce(const GemmDesc& g, const Epi& e, const float* ws, int splits, int n_out, cudaStream_t s) {
  const long long total_el = (long long)n_out * g.M * g.N;
  const unsigned rg = (unsigned)std::min<long long>((total_el + 255) / 256, 148 * 16);
  if (g.c_dtype == KL_BF16)
    launch_k(splitk_reduce_kernel<bf16>, rg, 256, 0, s, g, e, ws, splits, n_out);
  else
    launch_k(splitk_reduce_kernel<float>, rg, 256, 0, s, g, e, ws, splits, n_out);
  count_launch();
  return launch_check("gemm_splitk_reduce");
}
}  // namespace kl
