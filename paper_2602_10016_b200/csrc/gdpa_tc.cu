// Fused GDPA core on tcgen05/TMEM, fed by TMA (SURVEY.md §8(a) row "GDPA").
//
// The folded personalized FFN of one sample (gdpa.py:120-187 with the
// per-sample fold Kt = K W_q, Vt = V W_out^T of SURVEY.md Appendix C):
//     Z = S Kt^T * inv_tau   (T x HK),   A = Act_h(Z)  (per n_kv column block)
//     Y = S + A Vt           (T x d);    rows >= length pass through.
// and its VJP
//     dZ = (dY Vt^T) * Act'(Z) * inv_tau,  dS = dY + dZ Kt,
//     dKt = dZ^T S,                         dVt = A^T dY.
//
// Forward, one persistent CTA per SM over (sample, 128-row tile) items:
//   warp 0  TMA producer: Kt/Vt of the current sample (once per sample) and a
//           2-slot ring of S tiles (128 x d bf16, SWIZZLE_128B atoms of 64 cols)
//   warp 1  MMA issuer: Z = S Kt^T into a double-buffered TMEM accumulator
//           (HK = 64 columns), then Y = A Vt (N = d <= 256) into TMEM
//   warps 2-9  epilogue: Z -> Act -> bf16 A tile in smem (operand of the
//           second MMA), then Y + S (residual read from the S tile in smem)
//           written back INTO the S slot, then copied out with coalesced
//           16-byte stores (one 512 B row per warp instruction) and the
//           slot released.
// Z and A never touch HBM: per tile the kernel reads S once and writes Y once
// (algorithmic traffic 4*d bytes per row).
//
// Backward, one CTA per sample (dKt/dVt accumulate over the sample's tiles in
// TMEM: 2 x (d/128) x 64 columns):
//   MMA  dA = dY Vt^T, Z = S Kt^T            (TMEM cols [0,64), [64,128))
//   epi  dZ, A -> bf16 tiles in smem
//   MMA  dS = dZ Kt (TMEM [0,d)), dKt^T += S^T dZ, dVt^T += dY^T A
//        (S^T / dY^T are the same smem tiles read as MN-major operands)
//   epi  dS + dY -> written into the dY tile, copied out to dS
//   end of sample: dKt, dVt (bf16) from TMEM.
// Traffic per row: read S, dY; write dS (6*d bytes) + 2*HK*d*2 per sample.
#include <cudaTypedefs.h>

#include <stdlib.h>

#include <algorithm>

#include "common.cuh"
#include "tc_common.cuh"

namespace kl {

PFN_cuTensorMapEncodeTiled_v12000 tc_encode_fn();
int tc_num_sms();

namespace gdpa {

constexpr int TB = 128;                  // rows per tile
constexpr int HK = 64;                   // H * n_kv columns of Z
constexpr int NT = 352;                  // 11 warps
constexpr uint32_t ATOM_S = TB * 128;    // 128 rows x 64 bf16
constexpr uint32_t ATOM_KV = HK * 128;   // 64 rows x 64 bf16

struct P {
  int B, T;
  bf16* out;               // Y (fwd) or dS (bwd): (B, T, D), rows o_rs apart
  long long o_rs, o_bs;
  float inv_tau;
  const int* lengths;
  unsigned char code[HK];  // activation code per Z column
  int uniform16;           // every 16-column group shares one code
  unsigned long long* trace;  // debug: per-tile clock64 stamps of CTA 0, or NULL
  bf16* dKt;               // (B, HK, D) bf16, backward
  bf16* dVt;
};

// K-major operand whose K extent is split in 64-column atoms `atom` bytes apart.
__device__ __forceinline__ uint64_t dk(uint32_t base, int kk, uint32_t atom) {
  return tc::sdesc(base + (kk >> 2) * atom + (kk & 3) * 32, 16, 1024);
}
// MN-major operand: 64-element MN chunks `lbo` bytes apart, 16 K-rows per step.
__device__ __forceinline__ uint64_t dmn(uint32_t base, int kk, uint32_t lbo) {
  return tc::sdesc(base + kk * 2048, lbo, 1024);
}

#define TR(c, slot)                                                    \
  do {                                                                 \
    if (p.trace && blockIdx.x == 0 && (c) < 32) p.trace[(c) * 16 + (slot)] = clock64(); \
  } while (0)

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n)); }

// 8 packed bf16 pairs (16 columns) into a K-major SW128 tile of TB rows.
__device__ __forceinline__ void store_sw16(uint8_t* blk, int r, int c0, const uint32_t* pk) {
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    uint4 u = make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
    *reinterpret_cast<uint4*>(blk + tc::sw128_off(r, c0 + 8 * c, TB)) = u;
  }
}

// Activation over a run of N columns sharing one code (the per-head column
// block): y = Act(z*s) and, for the VJP, dy = g * Act'(z*s) * s.  Hardware
// approximations (ex2/rcp/tanh.approx, rel. err <= 2^-11) — A and dZ are
// rounded to bf16 (2^-9) right after.  Codes as tensor.py:431-440.
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_fast(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sigm_fast(float x) { return rcp_fast(1.f + __expf(-x)); }

template <int N, bool BWD>
__device__ __forceinline__ void act_run(int code, const float* z, const float* g, float s, float* y, float* dy) {
  switch (code) {
    case KL_ACT_RELU:
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const float x = z[i] * s;
        y[i] = fmaxf(x, 0.f);
        if (BWD) dy[i] = x > 0.f ? g[i] * s : 0.f;
      }
      break;
    case KL_ACT_SILU:
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const float x = z[i] * s, sg = sigm_fast(x);
        y[i] = x * sg;
        if (BWD) dy[i] = g[i] * s * sg * (1.f + x * (1.f - sg));
      }
      break;
    case KL_ACT_TANH:
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const float t = tanh_fast(z[i] * s);
        y[i] = t;
        if (BWD) dy[i] = g[i] * s * (1.f - t * t);
      }
      break;
    default:
#pragma unroll
      for (int i = 0; i < N; ++i) {
        y[i] = z[i] * s;
        if (BWD) dy[i] = g[i] * s;
      }
  }
}

// This thread's 32 Z columns [c0, c0+32): two per-head runs of 16 (every
// 16-column group shares one code: n_kv % 16 == 0, host-checked).  The fused
// kernels take the reference's default activation cycle (identity, relu,
// silu, tanh; gdpa.py:31); other tags run the GEMM composition.  Each extra
// unrolled case grows the kernels' code (instruction-cache pressure).
template <bool BWD>
__device__ __forceinline__ void act_cols32(const unsigned char* code, int c0, bool, const float* z, const float* g,
                                           float s, float* y, float* dy) {
  act_run<16, BWD>(code[c0], z, g, s, y, dy);
  act_run<16, BWD>(code[c0 + 16], z + 16, g + 16, s, y + 16, dy + 16);
}

// In-place: tile(r, c0..c0+31) = bf16(acc[0..31] + tile(r, c0..c0+31)).
__device__ __forceinline__ void add_residual32(uint8_t* tile, int r, int c0, const float* acc) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint4* ptr = reinterpret_cast<uint4*>(tile + tc::sw128_off(r, c0 + 8 * c, TB));
    uint4 u = *ptr;
    uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat162 h = *reinterpret_cast<__nv_bfloat162*>(&w[i]);
      const float2 f = __bfloat1622float2(h);
      w[i] = tc::pack_bf16(acc[8 * c + 2 * i] + f.x, acc[8 * c + 2 * i + 1] + f.y);
    }
    *ptr = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// The 8 epilogue warps (256 threads, named barrier 1) copy a finished
// swizzled 128 x D tile to global rows q0.. (< T): one warp writes 512
// contiguous bytes per instruction.
template <int D>
__device__ __forceinline__ void copy_out(const uint8_t* tile, bf16* out, long long rs, int q0, int T, int tid) {
  constexpr int CPR = D / 8;  // 16-byte chunks per row
#pragma unroll 4
  for (int q = tid; q < TB * CPR; q += 256) {
    const int row = q / CPR, col = (q % CPR) * 8;
    const uint4 v = *reinterpret_cast<const uint4*>(tile + tc::sw128_off(row, col, TB));
    if (q0 + row < T) *reinterpret_cast<uint4*>(out + (long long)(q0 + row) * rs + col) = v;
  }
}

__device__ __forceinline__ uint8_t* align1k(uint8_t* p) {
  return (uint8_t*)(((uintptr_t)p + 1023) & ~(uintptr_t)1023);
}

template <int D>
constexpr size_t fwd_smem() {
  return 1024 + 2 * (D / 64) * ATOM_S + 2 * (D / 64) * ATOM_KV + ATOM_S + 256;
}
template <int D>
constexpr size_t bwd_smem() {
  return 1024 + 2 * (D / 64) * ATOM_S + 2 * (D / 64) * ATOM_KV + 2 * ATOM_S + 256;
}

// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(NT, 1)
    gdpa_fwd_kernel(const __grid_constant__ CUtensorMap ts, const __grid_constant__ CUtensorMap tk,
                    const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap ty, const P p) {
  constexpr int NA = D / 64;
  constexpr uint32_t SLOT = NA * ATOM_S;
  constexpr uint32_t IDESC_Z = tc::idesc_bf16(TB, HK, 0, 0);
  constexpr uint32_t IDESC_Y = tc::idesc_bf16(TB, D, 0, 1);
  constexpr uint32_t T_Y = 256;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sS = align1k(smem_raw);       // 2 slots
  uint8_t* sK = sS + 2 * SLOT;
  uint8_t* sV = sK + NA * ATOM_KV;
  uint8_t* sA = sV + NA * ATOM_KV;
  uint64_t* bar = (uint64_t*)(sA + ATOM_S);
  uint64_t* s_full = bar;        // [2]
  uint64_t* s_empty = bar + 2;   // [2]
  uint64_t* kv_full = bar + 4;
  uint64_t* kv_empty = bar + 5;
  uint64_t* z_full = bar + 6;    // [2]
  uint64_t* z_empty = bar + 8;   // [2]
  uint64_t* a_full = bar + 10;
  uint64_t* a_empty = bar + 11;
  uint64_t* y_full = bar + 12;
  uint64_t* y_empty = bar + 13;
  uint64_t* st_full = bar + 14;  // [2]
  uint32_t* tslot = (uint32_t*)(bar + 16);

  const int nT = (p.T + TB - 1) / TB;
  const int W = p.B * nT;
  const int i0 = (int)((long long)W * blockIdx.x / gridDim.x);
  const int i1 = (int)((long long)W * (blockIdx.x + 1) / gridDim.x);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ unsigned char code[HK];
  if (threadIdx.x < HK) code[threadIdx.x] = p.code[threadIdx.x];

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&ts);
    tc::prefetch_tmap(&tk);
    tc::prefetch_tmap(&tv);
    tc::prefetch_tmap(&ty);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&s_full[i], 1);
      tc::mbar_init(&s_empty[i], 1);
      tc::mbar_init(&z_full[i], 1);
      tc::mbar_init(&z_empty[i], 8);
      tc::mbar_init(&st_full[i], 8);
    }
    tc::mbar_init(kv_full, 1);
    tc::mbar_init(kv_empty, 1);
    tc::mbar_init(a_full, 8);
    tc::mbar_init(a_empty, 1);
    tc::mbar_init(y_full, 1);
    tc::mbar_init(y_empty, 8);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tslot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  // PDL: the prologue above (barrier init, TMEM alloc, tensor-map prefetch)
  // overlaps the previous kernel; global memory is touched only after this
  KL_PDL_ENTRY();

  if (warp == 0) {
    if (lane == 0) {
      int cur_b = -1, ns = 0;
      for (int k = i0, c = 0; k < i1; ++k, ++c) {
        const int b = k / nT, q0 = (k % nT) * TB;
        if (b != cur_b) {
          tc::mbar_wait(kv_empty, (ns & 1) ^ 1);
          tc::mbar_arrive_expect_tx(kv_full, 2 * NA * ATOM_KV);
#pragma unroll
          for (int a = 0; a < NA; ++a) {
            tc::tma_load_3d(sK + a * ATOM_KV, &tk, kv_full, a * 64, 0, b);
            tc::tma_load_3d(sV + a * ATOM_KV, &tv, kv_full, a * 64, 0, b);
          }
          cur_b = b;
          ++ns;
        }
        const int sl = c & 1;
        tc::mbar_wait(&s_empty[sl], ((c >> 1) & 1) ^ 1);
        TR(c, 0);
        tc::mbar_arrive_expect_tx(&s_full[sl], SLOT);
#pragma unroll
        for (int a = 0; a < NA; ++a) tc::tma_load_3d(sS + sl * SLOT + a * ATOM_S, &ts, &s_full[sl], a * 64, q0, b);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int ns = 0;
      auto mma1 = [&](int k, int c) {
        const int sl = c & 1;
        if (k == i0 || k % nT == 0) {  // first tile of a sample in this CTA
          tc::mbar_wait(kv_full, ns & 1);
          ++ns;
        }
        tc::mbar_wait(&s_full[sl], (c >> 1) & 1);
        TR(c, 1);
        tc::mbar_wait(&z_empty[sl], ((c >> 1) & 1) ^ 1);
        tc::fence_after();
        const uint32_t sa = tc::smem_u32(sS + sl * SLOT), ka = tc::smem_u32(sK);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          tc::mma_bf16(tmem + sl * HK, dk(sa, kk, ATOM_S), dk(ka, kk, ATOM_KV), IDESC_Z, kk > 0);
        tc::mma_commit(&z_full[sl]);
      };
      if (i0 < i1) mma1(i0, 0);
      for (int k = i0, c = 0; k < i1; ++k, ++c) {
        const bool last_of_sample = (k + 1 == i1) || ((k + 1) % nT == 0);
        tc::mbar_wait(a_full, c & 1);
        TR(c, 2);
        tc::mbar_wait(y_empty, (c & 1) ^ 1);
        TR(c, 3);
        tc::fence_after();
        const uint32_t aa = tc::smem_u32(sA), va = tc::smem_u32(sV);
#pragma unroll
        for (int kk = 0; kk < HK / 16; ++kk) tc::mma_bf16(tmem + T_Y, dk(aa, kk, ATOM_S), dmn(va, kk, ATOM_KV), IDESC_Y, kk > 0);
        tc::mma_commit(y_full);
        tc::mma_commit(a_empty);
        if (last_of_sample) tc::mma_commit(kv_empty);
        // the next tile's Z runs while this tile's Y epilogue drains
        if (k + 1 < i1) mma1(k + 1, c + 1);
      }
    }
  } else if (warp < 10) {
    const int qtr = warp & 3, hf = (warp - 2) >> 2;
    const int r = qtr * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(qtr * 32) << 16);
    for (int k = i0, c = 0; k < i1; ++k, ++c) {
      const int b = k / nT, q0 = (k % nT) * TB;
      int len = __ldg(&p.lengths[b]);
      asm volatile("" : "+r"(len));  // materialise before the barrier wait
      const bool live = q0 + r < len;
      const int sl = c & 1;
      // ---- A = Act(Z) (this half's 32 columns) -> sA
      tc::mbar_wait(&z_full[sl], (c >> 1) & 1);
      if (warp == 2 && lane == 0) TR(c, 4);
      tc::fence_after();
      float v[32];
      tc::tmem_ld32(trow + sl * HK + hf * 32, v);
      if (warp == 2 && lane == 0) TR(c, 9);
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&z_empty[sl]);
      uint32_t pk[16];
      {
        float y[32];
        act_cols32<false>(code, hf * 32, p.uniform16, v, nullptr, p.inv_tau, y, nullptr);
#pragma unroll
        for (int i = 0; i < 32; i += 2) pk[i >> 1] = live ? tc::pack_bf16(y[i], y[i + 1]) : 0u;
      }
      if (warp == 2 && lane == 0) TR(c, 10);
      tc::mbar_wait(a_empty, (c & 1) ^ 1);
      if (warp == 2 && lane == 0) TR(c, 5);
      store_sw16(sA, r, hf * 32, pk);
      store_sw16(sA, r, hf * 32 + 16, pk + 8);
      tc::fence_async_smem();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(a_full);
      // ---- Y = acc + S, in place in the S slot
      tc::mbar_wait(y_full, c & 1);
      if (warp == 2 && lane == 0) TR(c, 6);
      tc::fence_after();
      uint8_t* tile = sS + sl * SLOT;
#pragma unroll 1
      for (int cc = hf * (D / 2); cc < (hf + 1) * (D / 2); cc += 64) {
        uint32_t u[64];
        tc::tmem_ld32_nowait(trow + T_Y + cc, u);
        tc::tmem_ld32_nowait(trow + T_Y + cc + 32, u + 32);
        tc::tmem_wait_ld();
        tc::reg_fence<64>(u);
        add_residual32(tile, r, cc, reinterpret_cast<const float*>(u));
        add_residual32(tile, r, cc + 32, reinterpret_cast<const float*>(u + 32));
      }
      if (warp == 2 && lane == 0) TR(c, 7);
      tc::fence_before();
      tc::fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        tc::mbar_arrive(y_empty);
        tc::mbar_arrive(&st_full[sl]);
      }
    }
  } else if (lane == 0) {  // warp 10: TMA store of finished slots
    for (int k = i0, c = 0; k < i1; ++k, ++c) {
      const int b = k / nT, q0 = (k % nT) * TB, sl = c & 1;
      tc::mbar_wait(&st_full[sl], (c >> 1) & 1);
#pragma unroll
      for (int a = 0; a < NA; ++a) tc::tma_store_3d(&ty, sS + sl * SLOT + a * ATOM_S, a * 64, q0, b);
      tc::bulk_commit();
      tc::bulk_wait_read0();
      TR(c, 8);
      tc::mbar_arrive(&s_empty[sl]);
    }
    tc::bulk_wait0();
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(NT, 1)
    gdpa_bwd_kernel(const __grid_constant__ CUtensorMap ts, const __grid_constant__ CUtensorMap tg,
                    const __grid_constant__ CUtensorMap tk, const __grid_constant__ CUtensorMap tv,
                    const __grid_constant__ CUtensorMap tds, const P p) {
  constexpr int NA = D / 64, NM = D / 128;
  constexpr uint32_t SLOT = NA * ATOM_S;
  constexpr uint32_t IDESC_Z = tc::idesc_bf16(TB, HK, 0, 0);
  constexpr uint32_t IDESC_DS = tc::idesc_bf16(TB, D, 0, 1);
  constexpr uint32_t IDESC_W = tc::idesc_bf16(TB, HK, 1, 1);
  constexpr uint32_t T_DK = 256, T_DV = 384;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sS = align1k(smem_raw);
  uint8_t* sG = sS + SLOT;
  uint8_t* sK = sG + SLOT;
  uint8_t* sV = sK + NA * ATOM_KV;
  uint8_t* sDZ = sV + NA * ATOM_KV;
  uint8_t* sA = sDZ + ATOM_S;
  uint64_t* bar = (uint64_t*)(sA + ATOM_S);
  uint64_t* sg_full = bar;
  uint64_t* sg_empty = bar + 1;
  uint64_t* kv_full = bar + 2;
  uint64_t* kv_empty = bar + 3;
  uint64_t* zz_full = bar + 4;
  uint64_t* dz_full = bar + 5;
  uint64_t* ds_full = bar + 6;
  uint64_t* acc_full = bar + 7;
  uint64_t* acc_empty = bar + 8;
  uint64_t* st_full = bar + 9;
  uint32_t* tslot = (uint32_t*)(bar + 10);

  const int nT = (p.T + TB - 1) / TB;
  const int b0 = (int)((long long)p.B * blockIdx.x / gridDim.x);
  const int b1 = (int)((long long)p.B * (blockIdx.x + 1) / gridDim.x);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ unsigned char code[HK];
  if (threadIdx.x < HK) code[threadIdx.x] = p.code[threadIdx.x];

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&ts);
    tc::prefetch_tmap(&tg);
    tc::prefetch_tmap(&tk);
    tc::prefetch_tmap(&tv);
    tc::mbar_init(sg_full, 1);
    tc::prefetch_tmap(&tds);
    tc::mbar_init(sg_empty, 1);
    tc::mbar_init(st_full, 8);
    tc::mbar_init(kv_full, 1);
    tc::mbar_init(kv_empty, 1);
    tc::mbar_init(zz_full, 1);
    tc::mbar_init(dz_full, 8);
    tc::mbar_init(ds_full, 1);
    tc::mbar_init(acc_full, 1);
    tc::mbar_init(acc_empty, 8);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tslot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  // PDL: the prologue above (barrier init, TMEM alloc, tensor-map prefetch)
  // overlaps the previous kernel; global memory is touched only after this
  KL_PDL_ENTRY();

  if (warp == 0) {
    if (lane == 0) {
      int c = 0, ns = 0;
      for (int b = b0; b < b1; ++b, ++ns) {
        tc::mbar_wait(kv_empty, (ns & 1) ^ 1);
        tc::mbar_arrive_expect_tx(kv_full, 2 * NA * ATOM_KV);
#pragma unroll
        for (int a = 0; a < NA; ++a) {
          tc::tma_load_3d(sK + a * ATOM_KV, &tk, kv_full, a * 64, 0, b);
          tc::tma_load_3d(sV + a * ATOM_KV, &tv, kv_full, a * 64, 0, b);
        }
        for (int t = 0; t < nT; ++t, ++c) {
          tc::mbar_wait(sg_empty, (c & 1) ^ 1);
          TR(c, 0);
          tc::mbar_arrive_expect_tx(sg_full, 2 * SLOT);
#pragma unroll
          for (int a = 0; a < NA; ++a) {
            tc::tma_load_3d(sS + a * ATOM_S, &ts, sg_full, a * 64, t * TB, b);
            tc::tma_load_3d(sG + a * ATOM_S, &tg, sg_full, a * 64, t * TB, b);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int c = 0, ns = 0;
      const uint32_t ua = tc::smem_u32(sS), ga = tc::smem_u32(sG), ka = tc::smem_u32(sK), va = tc::smem_u32(sV);
      const uint32_t dza = tc::smem_u32(sDZ), aa = tc::smem_u32(sA);
      for (int b = b0; b < b1; ++b, ++ns) {
        tc::mbar_wait(kv_full, ns & 1);
        for (int t = 0; t < nT; ++t, ++c) {
          tc::mbar_wait(sg_full, c & 1);
          TR(c, 1);
          tc::fence_after();
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            tc::mma_bf16(tmem, dk(ga, kk, ATOM_S), dk(va, kk, ATOM_KV), IDESC_Z, kk > 0);
            tc::mma_bf16(tmem + HK, dk(ua, kk, ATOM_S), dk(ka, kk, ATOM_KV), IDESC_Z, kk > 0);
          }
          tc::mma_commit(zz_full);
          tc::mbar_wait(dz_full, c & 1);
          TR(c, 2);
          if (t == 0) tc::mbar_wait(acc_empty, (ns & 1) ^ 1);
          tc::fence_after();
#pragma unroll
          for (int kk = 0; kk < HK / 16; ++kk) tc::mma_bf16(tmem, dk(dza, kk, ATOM_S), dmn(ka, kk, ATOM_KV), IDESC_DS, kk > 0);
#pragma unroll
          for (int mh = 0; mh < NM; ++mh) {
#pragma unroll
            for (int kk = 0; kk < TB / 16; ++kk) {
              const uint32_t acc = (t > 0 || kk > 0) ? 1u : 0u;
              tc::mma_bf16(tmem + T_DK + mh * HK, dmn(ua + 2 * mh * ATOM_S, kk, ATOM_S), dmn(dza, kk, ATOM_S),
                           IDESC_W, acc);
              tc::mma_bf16(tmem + T_DV + mh * HK, dmn(ga + 2 * mh * ATOM_S, kk, ATOM_S), dmn(aa, kk, ATOM_S),
                           IDESC_W, acc);
            }
          }
          tc::mma_commit(ds_full);
          TR(c, 3);
        }
        tc::mma_commit(acc_full);
        tc::mma_commit(kv_empty);
      }
    }
  } else if (warp < 10) {
    const int qtr = warp & 3, hf = (warp - 2) >> 2;
    const int r = qtr * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(qtr * 32) << 16);
    int c = 0, ns = 0;
    for (int b = b0; b < b1; ++b, ++ns) {
      const int len = __ldg(&p.lengths[b]);
      for (int t = 0; t < nT; ++t, ++c) {
        const bool live = t * TB + r < len;
        // ---- dZ = dA * Act'(Z) * inv_tau, A = Act(Z) -> smem operand tiles
        tc::mbar_wait(zz_full, c & 1);
        if (warp == 2 && lane == 0) TR(c, 4);
        tc::fence_after();
        float da[32], z[32];
        tc::tmem_ld32_nowait(trow + hf * 32, reinterpret_cast<uint32_t*>(da));
        tc::tmem_ld32_nowait(trow + HK + hf * 32, reinterpret_cast<uint32_t*>(z));
        tc::tmem_wait_ld();
        tc::reg_fence<32>(reinterpret_cast<uint32_t*>(da));
        tc::reg_fence<32>(reinterpret_cast<uint32_t*>(z));
        uint32_t pdz[16], pa[16];
        {
          float y[32], dy[32];
          act_cols32<true>(code, hf * 32, p.uniform16, z, da, p.inv_tau, y, dy);
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            pdz[i >> 1] = live ? tc::pack_bf16(dy[i], dy[i + 1]) : 0u;
            pa[i >> 1] = live ? tc::pack_bf16(y[i], y[i + 1]) : 0u;
          }
        }
        store_sw16(sDZ, r, hf * 32, pdz);
        store_sw16(sDZ, r, hf * 32 + 16, pdz + 8);
        store_sw16(sA, r, hf * 32, pa);
        store_sw16(sA, r, hf * 32 + 16, pa + 8);
        tc::fence_before();
        tc::fence_async_smem();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(dz_full);
        // ---- dS = acc + dY, in place in the dY tile
        tc::mbar_wait(ds_full, c & 1);
        if (warp == 2 && lane == 0) TR(c, 6);
        tc::fence_after();
#pragma unroll 1
        for (int cc = hf * (D / 2); cc < (hf + 1) * (D / 2); cc += 64) {
          uint32_t u[64];
          tc::tmem_ld32_nowait(trow + cc, u);
          tc::tmem_ld32_nowait(trow + cc + 32, u + 32);
          tc::tmem_wait_ld();
          tc::reg_fence<64>(u);
          add_residual32(sG, r, cc, reinterpret_cast<const float*>(u));
          add_residual32(sG, r, cc + 32, reinterpret_cast<const float*>(u + 32));
        }
        if (warp == 2 && lane == 0) TR(c, 7);
        tc::fence_before();
        tc::fence_async_smem();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(st_full);
      }
      // ---- dKt, dVt of this sample: TMEM lane = feature column c
      tc::mbar_wait(acc_full, ns & 1);
      tc::fence_after();
      if (hf < NM) {
        const int col = hf * 128 + r;
        bf16* dk_out = p.dKt + (long long)b * HK * D + col;
        bf16* dv_out = p.dVt + (long long)b * HK * D + col;
#pragma unroll
        for (int h = 0; h < HK; h += 32) {
          float v[32];
          tc::tmem_ld32(trow + T_DK + hf * HK + h, v);
#pragma unroll
          for (int i = 0; i < 32; ++i) dk_out[(long long)(h + i) * D] = __float2bfloat16(v[i]);
          tc::tmem_ld32(trow + T_DV + hf * HK + h, v);
#pragma unroll
          for (int i = 0; i < 32; ++i) dv_out[(long long)(h + i) * D] = __float2bfloat16(v[i]);
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(acc_empty);
    }
  } else if (lane == 0) {  // warp 10: TMA store of dS tiles
    int c = 0;
    for (int b = b0; b < b1; ++b) {
      for (int t = 0; t < nT; ++t, ++c) {
        tc::mbar_wait(st_full, c & 1);
#pragma unroll
        for (int a = 0; a < NA; ++a) tc::tma_store_3d(&tds, sG + a * ATOM_S, a * 64, t * TB, b);
        tc::bulk_commit();
        tc::bulk_wait_read0();
        TR(c, 8);
        tc::mbar_arrive(sg_empty);
      }
    }
    tc::bulk_wait0();
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------------------
// d = 512 (the c4 shape, H*n_kv = HK2 = 128).  A resident 128 x 512 S tile
// plus the 128 x 512 Kt / Vt of a sample would need ~384 KB of shared
// memory, and a 128 x 512 fp32 output accumulator fills TMEM, so these
// kernels stream the K = d contractions in 64-column atoms and produce the
// d-wide results in two 256-column halves:
//
// Forward, persistent CTAs over (sample, 128-row tile) items:
//   warp 0     TMA: 8 (S atom, Kt atom) stages per tile into a 4-slot ring,
//              then each half of Vt (4 atoms, MN-major B operand) into a slot
//   warp 1     MMA: Z = sum_a S_a Kt_a^T (double-buffered, 2 x 128 TMEM
//              columns), Y_h = A Vt[:, h] (N = 256, TMEM [256, 512))
//   warps 2-9  Z -> Act (per 16-column head group) -> bf16 A tile in smem;
//              Y_h + S[:, h] (residual read from global / L2) -> bf16 rows.
// Backward, persistent CTAs over the same items:
//   MMA   dA = sum_a dY_a Vt_a^T, Z = sum_a S_a Kt_a^T (one 2-slot ring of
//         (dY, Vt, S, Kt) atoms); dS_h = dZ Kt[:, h] (N = 256)
//   warps dZ = dA Act'(Z) / tau, A = Act(Z): both to HBM (the caller's
//         dKt = dZ^T S and dVt = A^T dY GEMMs), dZ also to smem; dS_h + dY
//         -> bf16 rows.
constexpr int HK2 = 128;
constexpr int NT5 = 320;                       // warp 0 TMA, 1 MMA, 2-9 epilogue
constexpr int NT6 = 352;                       // + warp 10: the second operand loader (d = 512)
constexpr int RST = 3;                         // forward ring stages (+ 16 KB epilogue staging)
constexpr uint32_t FSTAGE = 2 * ATOM_S;        // S atom | Kt atom (128 rows x 64)
constexpr uint32_t BSTAGE = 4 * ATOM_S;        // dY | Vt | S | Kt atoms

struct P5 {
  int B, T;
  bf16* out;            // Y (fwd) or dS (bwd): (B, T, 512), rows o_rs apart
  long long o_rs, o_bs;
  const bf16* res;      // residual: S (fwd) or dY (bwd), same layout
  long long r_rs, r_bs;
  float inv_tau;
  const int* lengths;
  unsigned char code[HK2];
  bf16* dZ;             // bwd: (B, T, HK2)
  bf16* A;
  unsigned long long* trace;  // debug: per-tile clock64 stamps of CTA 0 ([tile < 32][event < 16]), or NULL
};
#define T5(c, slot)                                                                          \
  do {                                                                                       \
    if (p.trace && blockIdx.x == 0 && (c) < 32) p.trace[(c) * 16 + (slot)] = clock64();      \
  } while (0)

// Act over this thread's 64 Z columns [c0, c0 + 64): four 16-column head groups.
template <bool BWD>
__device__ __forceinline__ void act_cols64(const unsigned char* code, int c0, const float* z, const float* g,
                                           float s, float* y, float* dy) {
#pragma unroll
  for (int q = 0; q < 4; ++q)
    act_run<16, BWD>(code[c0 + 16 * q], z + 16 * q, BWD ? g + 16 * q : nullptr, s, y + 16 * q,
                     BWD ? dy + 16 * q : nullptr);
}

// 32 fp32 accumulator columns + 32 bf16 residual columns (4 prefetched
// 16-byte chunks) -> 32 bf16 outputs.
__device__ __forceinline__ void add_res_store32(const float* v, const uint4* rp, bf16* out) {
  uint4* op = reinterpret_cast<uint4*>(out);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint4 u = rp[c];
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
    uint32_t o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[i]));
      o[i] = tc::pack_bf16(v[8 * c + 2 * i] + f.x, v[8 * c + 2 * i + 1] + f.y);
    }
    op[c] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// This thread's 128 residual columns of one output half, loaded before the
// accumulator wait (the global / L2 latency hides behind the MMAs).
__device__ __forceinline__ void prefetch_res128(const bf16* src, bool ok, uint4* r) {
  const uint4* p = reinterpret_cast<const uint4*>(src);
#pragma unroll
  for (int c = 0; c < 16; ++c) r[c] = ok ? __ldg(p + c) : make_uint4(0u, 0u, 0u, 0u);
}

// Coalesced epilogue I/O of one warp's 32 rows x 32 bf16 columns.  With
// thread = row (the TMEM lane layout) a 16-byte access per thread touches 32
// different 128-byte lines per warp instruction; going through a 2 KB
// per-warp staging tile, every warp instruction covers 8 rows x 64 B (4x
// fewer L1 wavefronts: clock-stamp trace of the d = 512 GDPA forward, one
// 128 x 256 output half took 6-8 k clk in its row-per-thread stores and
// residual loads).  Staging row R, 16-byte chunk c lives at R*64 + (c ^ (R>>1 & 3))*16
// (conflict-free for both the row-per-thread and the lane-per-chunk pattern).
__device__ __forceinline__ uint32_t stg_off(int R, int c) { return R * 64 + ((c ^ ((R >> 1) & 3)) << 4); }

// lane's 4 coalesced 16-byte residual chunks: rows row0 + (lane >> 2) + 8 i, chunk lane & 3
__device__ __forceinline__ void res_load_co(const bf16* base, long long rs, int row0, int nvalid, int col0,
                                            uint4* r4) {
  const int lane = threadIdx.x & 31, c = lane & 3;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int R = (lane >> 2) + 8 * i;
    r4[i] = R < nvalid ? __ldg(reinterpret_cast<const uint4*>(base + (long long)(row0 + R) * rs + col0 + 8 * c))
                       : make_uint4(0u, 0u, 0u, 0u);
  }
}

// out[row0 + lane, col0 .. col0 + 32) = acc (this thread's row) + residual
// (r4: res_load_co chunks), stored coalesced; stg: the warp's 2 KB staging tile.
__device__ __forceinline__ void res_add_store_co(uint8_t* stg, const uint4* r4, const float* acc, bf16* obase,
                                                 long long os, int row0, int nvalid, int col0) {
  const int lane = threadIdx.x & 31, c = lane & 3;
#pragma unroll
  for (int i = 0; i < 4; ++i) *reinterpret_cast<uint4*>(stg + stg_off((lane >> 2) + 8 * i, c)) = r4[i];
  __syncwarp();
  uint4 o[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint4 u = *reinterpret_cast<const uint4*>(stg + stg_off(lane, q));
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
    uint32_t v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[i]));
      v[i] = tc::pack_bf16(acc[8 * q + 2 * i] + f.x, acc[8 * q + 2 * i + 1] + f.y);
    }
    o[q] = make_uint4(v[0], v[1], v[2], v[3]);
  }
  __syncwarp();
#pragma unroll
  for (int q = 0; q < 4; ++q) *reinterpret_cast<uint4*>(stg + stg_off(lane, q)) = o[q];
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int R = (lane >> 2) + 8 * i;
    if (R < nvalid)
      *reinterpret_cast<uint4*>(obase + (long long)(row0 + R) * os + col0 + 8 * c) =
          *reinterpret_cast<const uint4*>(stg + stg_off(R, c));
  }
  __syncwarp();
}

__global__ void __launch_bounds__(NT6, 1)
    gdpa_fwd512_kernel(const __grid_constant__ CUtensorMap ts, const __grid_constant__ CUtensorMap tk,
                       const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tr32,
                       const __grid_constant__ CUtensorMap to32, const P5 p) {
  constexpr uint32_t IDESC_Z = tc::idesc_bf16(TB, HK2, 0, 0);
  constexpr uint32_t IDESC_Y = tc::idesc_bf16(TB, 256, 0, 1);
  constexpr uint32_t T_Y = 256;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sR = align1k(smem_raw);          // RST x (S atom | Kt atom)
  uint8_t* sV = sR + RST * FSTAGE;          // Vt half: 4 atoms
  uint8_t* sA = sV + 4 * ATOM_S;            // 128 x 128 bf16 (2 atoms)
  uint8_t* sStg = sA + 2 * ATOM_S;          // 8 x 4 KB per-warp epilogue tiles (32 rows x 64 cols, SW128)
  uint64_t* bar = (uint64_t*)(sStg + 8 * 4096);
  uint64_t* rs_full = bar;                  // [RST]
  uint64_t* rs_empty = bar + RST;           // [RST]
  uint64_t* vs_full = bar + 2 * RST;
  uint64_t* vs_empty = vs_full + 1;
  uint64_t* z_full = vs_full + 2;           // [2]
  uint64_t* z_empty = vs_full + 4;          // [2]
  uint64_t* a_full = vs_full + 6;
  uint64_t* a_empty = vs_full + 7;
  uint64_t* y_full = vs_full + 8;
  uint64_t* y_empty = vs_full + 9;
  uint64_t* rbar = vs_full + 10;            // [8] per-warp residual tile landed
  uint32_t* tslot = (uint32_t*)(vs_full + 18);

  const int nT = (p.T + TB - 1) / TB;
  const int W = p.B * nT;
  const int i0 = (int)((long long)W * blockIdx.x / gridDim.x);
  const int i1 = (int)((long long)W * (blockIdx.x + 1) / gridDim.x);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ unsigned char code[HK2];
  if (threadIdx.x < HK2) code[threadIdx.x] = p.code[threadIdx.x];

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&ts);
    tc::prefetch_tmap(&tk);
    tc::prefetch_tmap(&tv);
    for (int i = 0; i < RST; ++i) {
      tc::mbar_init(&rs_full[i], 1);
      tc::mbar_init(&rs_empty[i], 1);
    }
    tc::mbar_init(vs_full, 1);
    tc::mbar_init(vs_empty, 1);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&z_full[i], 1);
      tc::mbar_init(&z_empty[i], 8);
    }
    tc::mbar_init(a_full, 8);
    tc::mbar_init(a_empty, 1);
    tc::mbar_init(y_full, 1);
    tc::mbar_init(y_empty, 8);
    for (int i = 0; i < 8; ++i) tc::mbar_init(&rbar[i], 1);
    tc::prefetch_tmap(&tr32);
    tc::prefetch_tmap(&to32);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tslot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  KL_PDL_ENTRY();

  if (warp == 0) {
    if (lane == 0) {
      // Z operand stages (S atom | Kt atom) only; the Vt halves come from
      // warp 10, so the Z stream never waits behind the single Vt buffer's
      // release by a Y product
      int rc = 0;
      auto load_z = [&](int k) {
        const int b = k / nT, q0 = (k % nT) * TB;
#pragma unroll 1
        for (int a = 0; a < 8; ++a, ++rc) {
          const int st = rc % RST;
          tc::mbar_wait(&rs_empty[st], ((rc / RST) & 1) ^ 1);
          tc::mbar_arrive_expect_tx(&rs_full[st], FSTAGE);
          tc::tma_load_3d(sR + st * FSTAGE, &ts, &rs_full[st], a * 64, q0, b);
          tc::tma_load_3d(sR + st * FSTAGE + ATOM_S, &tk, &rs_full[st], a * 64, 0, b);
        }
      };
      for (int k = i0; k < i1; ++k) {
        T5(k - i0, 0);
        load_z(k);
        T5(k - i0, 2);
      }
    }
  } else if (warp == 10) {
    if (lane == 0) {
      int vc = 0;
      for (int k = i0; k < i1; ++k)
        for (int h = 0; h < 2; ++h, ++vc) {
          const int b = k / nT;
          tc::mbar_wait(vs_empty, (vc & 1) ^ 1);
          tc::mbar_arrive_expect_tx(vs_full, 4 * ATOM_S);
#pragma unroll
          for (int a = 0; a < 4; ++a) tc::tma_load_3d(sV + a * ATOM_S, &tv, vs_full, (4 * h + a) * 64, 0, b);
        }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // Polling issue loop: the Y halves of tile k (latency-critical: the
      // epilogue waits on them) go out as soon as A(k), the accumulator and
      // the Vt half are ready, the next tile's Z atoms whenever a ring stage
      // has landed — neither waits behind the other in program order (the
      // in-order form issued Y0(k) only after all of Z(k+1)'s operand stream:
      // clock-stamp trace, ~10 k clk per tile).
      int rc = 0, zc = 0, vc = 0, yc = 0, ac = 0;
      int zt = i0, za = 0, yt = i0, yh = 0;
      bool zbuf = false, a_ok = false;
      const uint32_t r0 = tc::smem_u32(sR), va = tc::smem_u32(sV), aa = tc::smem_u32(sA);
      while (yt < i1) {
        if (yt < zt) {  // Z(yt) is issued: its Y halves
          if (!a_ok) a_ok = tc::mbar_try(a_full, ac & 1);
          if (a_ok && tc::mbar_try(y_empty, (yc & 1) ^ 1) && tc::mbar_try(vs_full, vc & 1)) {
            if (yh == 0) T5(yt - i0, 6);
            T5(yt - i0, 7 + yh);
            tc::fence_after();
#pragma unroll
            for (int kk = 0; kk < HK2 / 16; ++kk)
              tc::mma_bf16(tmem + T_Y, dk(aa, kk, ATOM_S), dmn(va, kk, ATOM_S), IDESC_Y, kk > 0 ? 1u : 0u);
            tc::mma_commit(y_full);
            tc::mma_commit(vs_empty);
            ++yc;
            ++vc;
            if (++yh == 2) {
              tc::mma_commit(a_empty);
              ++ac;
              a_ok = false;
              yh = 0;
              ++yt;
            }
          }
        }
        if (zt < i1 && zt <= yt + 1) {  // Z at most one tile ahead of Y
          const int z = zc & 1;
          if (!zbuf) {
            zbuf = tc::mbar_try(&z_empty[z], ((zc >> 1) & 1) ^ 1);
            if (zbuf) T5(zt - i0, 4);
          }
          const int st = rc % RST;
          if (zbuf && tc::mbar_try(&rs_full[st], (rc / RST) & 1)) {
            tc::fence_after();
            const uint32_t sa = r0 + st * FSTAGE, ka = sa + ATOM_S;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              tc::mma_bf16(tmem + z * HK2, dk(sa, kk, ATOM_S), dk(ka, kk, ATOM_S), IDESC_Z, (za | kk) > 0 ? 1u : 0u);
            tc::mma_commit(&rs_empty[st]);
            ++rc;
            if (++za == 8) {
              tc::mma_commit(&z_full[z]);
              T5(zt - i0, 5);
              ++zc;
              ++zt;
              za = 0;
              zbuf = false;
            }
          }
        }
      }
    }
  } else {
    const int qtr = warp & 3, hf = (warp - 2) >> 2;
    const int r = qtr * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(qtr * 32) << 16);
    int zc = 0, yc = 0, ac = 0, rph = 0;
    for (int k = i0; k < i1; ++k) {
      const int b = k / nT, q0 = (k % nT) * TB;
      int len = __ldg(&p.lengths[b]);
      asm volatile("" : "+r"(len));
      const bool live = q0 + r < len;
      const int z = zc & 1;
      tc::mbar_wait(&z_full[z], (zc >> 1) & 1);
      if (threadIdx.x == 64) T5(k - i0, 9);
      tc::fence_after();
      float v[64];
      tc::tmem_ld32(trow + z * HK2 + hf * 64, v);
      tc::tmem_ld32(trow + z * HK2 + hf * 64 + 32, v + 32);
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&z_empty[z]);
      ++zc;
      uint32_t pk[32];
      {
        float y[64];
        act_cols64<false>(code, hf * 64, v, nullptr, p.inv_tau, y, nullptr);
#pragma unroll
        for (int i = 0; i < 64; i += 2) pk[i >> 1] = live ? tc::pack_bf16(y[i], y[i + 1]) : 0u;
      }
      tc::mbar_wait(a_empty, (ac & 1) ^ 1);
#pragma unroll
      for (int g = 0; g < 4; ++g) store_sw16(sA, r, hf * 64 + 16 * g, pk + 8 * g);
      tc::fence_async_smem();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(a_full);
      if (threadIdx.x == 64) T5(k - i0, 10);
      ++ac;
      // Y_h + S[:, h] -> Y: per warp two 32-row x 64-column tiles per half, the
      // residual TMA-loaded into the warp's SW128 staging tile, the sum written
      // back in place by the row threads and TMA-stored (no per-thread global
      // accesses: a row-per-thread 16-byte store touches 32 lines per warp
      // instruction — clock-stamp trace, ~5 k clk per output half)
      const int row0 = q0 + qtr * 32;
      uint8_t* stg = sStg + (warp - 2) * 4096;
      uint64_t* rb = &rbar[warp - 2];
      auto res_issue = [&](int col0) {
        if (lane == 0) {
          tc::bulk_wait_read0();  // the previous tile's TMA store has read the staging tile
          tc::mbar_arrive_expect_tx(rb, 4096);
          tc::tma_load_3d(stg, &tr32, rb, col0, row0, b);
        }
      };
      for (int h = 0; h < 2; ++h, ++yc) {
        res_issue(h * 256 + hf * 128);  // lands while the Y half's MMAs run
        tc::mbar_wait(y_full, yc & 1);
        if (threadIdx.x == 64) T5(k - i0, 11 + 2 * h);
        tc::fence_after();
#pragma unroll 1
        for (int cc = 0; cc < 2; ++cc) {
          const int col0 = h * 256 + hf * 128 + cc * 64;
          float acc[64];
          tc::tmem_ld32x2(trow + T_Y + hf * 128 + 64 * cc, acc, trow + T_Y + hf * 128 + 64 * cc + 32, acc + 32);
          if (cc == 1) {
            tc::fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(y_empty);
            res_issue(col0);
          }
          tc::mbar_wait(rb, rph & 1);
          ++rph;
          uint8_t* rowp = stg + lane * 128;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            uint4* cp = reinterpret_cast<uint4*>(rowp + ((q ^ (lane & 7)) << 4));
            const uint4 u = *cp;
            const uint32_t w[4] = {u.x, u.y, u.z, u.w};
            uint32_t o[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[i]));
              o[i] = tc::pack_bf16(acc[8 * q + 2 * i] + f.x, acc[8 * q + 2 * i + 1] + f.y);
            }
            *cp = make_uint4(o[0], o[1], o[2], o[3]);
          }
          tc::fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            tc::tma_store_3d(&to32, stg, col0, row0, b);
            tc::bulk_commit();
          }
        }
        if (threadIdx.x == 64) T5(k - i0, 12 + 2 * h);
      }
    }
    if (lane == 0) tc::bulk_wait0();
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

size_t fwd512_smem() { return 1024 + RST * FSTAGE + 4 * ATOM_S + 2 * ATOM_S + 8 * 4096 + (2 * RST + 18) * 8 + 16; }

// Backward (d = 512), persistent CTAs over (sample, 128-row tile) items:
//   warp 0     TMA: per tile 8 (dY | Vt | S | Kt) atom stages (2-slot ring),
//              then the 4 Kt column quarters (128 x 128, MN-major B of dS)
//   warp 1     MMA: dA = sum_a dY_a Vt_a^T, Z = sum_a S_a Kt_a^T;
//              dS_q = dZ Kt[:, q] (N = 128) into a double-buffered TMEM pair
//   warps 2-9  dZ = dA Act'(Z) / tau, A = Act(Z) -> dZ to smem (the dS
//              products' A operand) and, with A, to HBM by TMA store (the
//              caller's dKt / dVt GEMMs); dS_q + dY -> dS: per warp a 32-row x
//              64-column tile, residual TMA-loaded into and the sum TMA-stored
//              from its staging tile.  (Row-per-thread 16-byte global accesses
//              touch 32 lines per warp instruction; quarter-width dS products
//              free the shared memory for the staging tiles and let the next
//              quarter's product overlap this quarter's epilogue.)
__global__ void __launch_bounds__(NT6, 1)
    gdpa_bwd512_kernel(const __grid_constant__ CUtensorMap ts, const __grid_constant__ CUtensorMap tg,
                       const __grid_constant__ CUtensorMap tk, const __grid_constant__ CUtensorMap tv,
                       const __grid_constant__ CUtensorMap tkq, const __grid_constant__ CUtensorMap tg32,
                       const __grid_constant__ CUtensorMap to32, const __grid_constant__ CUtensorMap tz32,
                       const __grid_constant__ CUtensorMap ta32, const P5 p) {
  constexpr uint32_t IDESC_Z = tc::idesc_bf16(TB, HK2, 0, 0);
  constexpr uint32_t IDESC_DS = tc::idesc_bf16(TB, 128, 0, 1);
  constexpr uint32_t T_DA = 0, T_Z = 128, T_DS = 256;  // dS: 2 x 128 columns
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sR = align1k(smem_raw);          // 2 x (dY | Vt | S | Kt atoms)
  uint8_t* sK = sR + 2 * BSTAGE;            // Kt quarter: 2 atoms (128 x 128, MN-major B of dS_q)
  uint8_t* sD = sK + 2 * ATOM_S;            // dZ tile 128 x 128 bf16
  uint8_t* sStg = sD + 2 * ATOM_S;          // 8 x 4 KB per-warp epilogue tiles
  uint64_t* bar = (uint64_t*)(sStg + 8 * 4096);
  uint64_t* rs_full = bar;                  // [2]
  uint64_t* rs_empty = bar + 2;             // [2]
  uint64_t* ks_full = bar + 4;
  uint64_t* ks_empty = bar + 5;
  uint64_t* zz_full = bar + 6;
  uint64_t* zz_empty = bar + 7;
  uint64_t* d_full = bar + 8;
  uint64_t* d_empty = bar + 9;
  uint64_t* s_full = bar + 10;              // [2]
  uint64_t* s_empty = bar + 12;             // [2]
  uint64_t* rbar = bar + 14;                // [8]
  uint32_t* tslot = (uint32_t*)(bar + 22);

  const int nT = (p.T + TB - 1) / TB;
  const int W = p.B * nT;
  const int i0 = (int)((long long)W * blockIdx.x / gridDim.x);
  const int i1 = (int)((long long)W * (blockIdx.x + 1) / gridDim.x);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ unsigned char code[HK2];
  if (threadIdx.x < HK2) code[threadIdx.x] = p.code[threadIdx.x];

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&ts);
    tc::prefetch_tmap(&tg);
    tc::prefetch_tmap(&tk);
    tc::prefetch_tmap(&tv);
    tc::prefetch_tmap(&tkq);
    tc::prefetch_tmap(&tg32);
    tc::prefetch_tmap(&to32);
    tc::prefetch_tmap(&tz32);
    tc::prefetch_tmap(&ta32);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&rs_full[i], 1);
      tc::mbar_init(&rs_empty[i], 1);
      tc::mbar_init(&s_full[i], 1);
      tc::mbar_init(&s_empty[i], 8);
    }
    tc::mbar_init(ks_full, 1);
    tc::mbar_init(ks_empty, 1);
    tc::mbar_init(zz_full, 1);
    tc::mbar_init(zz_empty, 8);
    tc::mbar_init(d_full, 8);
    tc::mbar_init(d_empty, 1);
    for (int i = 0; i < 8; ++i) tc::mbar_init(&rbar[i], 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tslot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  KL_PDL_ENTRY();

  if (warp == 0) {
    if (lane == 0) {
      int rc = 0;
      for (int k = i0; k < i1; ++k) {
        const int b = k / nT, q0 = (k % nT) * TB;
#pragma unroll 1
        for (int a = 0; a < 8; ++a, ++rc) {
          const int st = rc & 1;
          tc::mbar_wait(&rs_empty[st], ((rc >> 1) & 1) ^ 1);
          uint8_t* d = sR + st * BSTAGE;
          tc::mbar_arrive_expect_tx(&rs_full[st], BSTAGE);
          tc::tma_load_3d(d, &tg, &rs_full[st], a * 64, q0, b);
          tc::tma_load_3d(d + ATOM_S, &tv, &rs_full[st], a * 64, 0, b);
          tc::tma_load_3d(d + 2 * ATOM_S, &ts, &rs_full[st], a * 64, q0, b);
          tc::tma_load_3d(d + 3 * ATOM_S, &tk, &rs_full[st], a * 64, 0, b);
        }
      }
    }
  } else if (warp == 10) {
    // the Kt column quarters (dS products' B operand): their own loader, so
    // the next tile's (dY | Vt | S | Kt) stages never wait behind them
    if (lane == 0) {
      int kc = 0;
      for (int k = i0; k < i1; ++k) {
        const int b = k / nT;
        for (int q = 0; q < 4; ++q, ++kc) {
          tc::mbar_wait(ks_empty, (kc & 1) ^ 1);
          tc::mbar_arrive_expect_tx(ks_full, 2 * ATOM_S);
#pragma unroll
          for (int a = 0; a < 2; ++a) tc::tma_load_3d(sK + a * ATOM_S, &tkq, ks_full, (2 * q + a) * 64, 0, b);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int rc = 0, kc = 0, sc = 0, c = 0;
      const uint32_t r0 = tc::smem_u32(sR), ka0 = tc::smem_u32(sK), da = tc::smem_u32(sD);
      for (int k = i0; k < i1; ++k, ++c) {
        tc::mbar_wait(zz_empty, (c & 1) ^ 1);
        tc::fence_after();
#pragma unroll 1
        for (int a = 0; a < 8; ++a, ++rc) {
          const int st = rc & 1;
          tc::mbar_wait(&rs_full[st], (rc >> 1) & 1);
          tc::fence_after();
          const uint32_t ga = r0 + st * BSTAGE, vva = ga + ATOM_S, sa = ga + 2 * ATOM_S, kta = ga + 3 * ATOM_S;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint32_t acc = (a | kk) > 0 ? 1u : 0u;
            tc::mma_bf16(tmem + T_DA, dk(ga, kk, ATOM_S), dk(vva, kk, ATOM_S), IDESC_Z, acc);
            tc::mma_bf16(tmem + T_Z, dk(sa, kk, ATOM_S), dk(kta, kk, ATOM_S), IDESC_Z, acc);
          }
          tc::mma_commit(&rs_empty[st]);
        }
        tc::mma_commit(zz_full);
        tc::mbar_wait(d_full, c & 1);
        for (int q = 0; q < 4; ++q, ++sc, ++kc) {
          const int sb = sc & 1;
          tc::mbar_wait(&s_empty[sb], ((sc >> 1) & 1) ^ 1);
          tc::mbar_wait(ks_full, kc & 1);
          tc::fence_after();
#pragma unroll
          for (int kk = 0; kk < HK2 / 16; ++kk)
            tc::mma_bf16(tmem + T_DS + sb * 128, dk(da, kk, ATOM_S), dmn(ka0, kk, ATOM_S), IDESC_DS,
                         kk > 0 ? 1u : 0u);
          tc::mma_commit(&s_full[sb]);
          tc::mma_commit(ks_empty);
        }
        tc::mma_commit(d_empty);
      }
    }
  } else {
    const int qtr = warp & 3, hf = (warp - 2) >> 2;
    const int r = qtr * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(qtr * 32) << 16);
    uint8_t* stg = sStg + (warp - 2) * 4096;
    uint64_t* rb = &rbar[warp - 2];
    int c = 0, sc = 0, rph = 0;
    for (int k = i0; k < i1; ++k, ++c) {
      const int b = k / nT, q0 = (k % nT) * TB;
      int len = __ldg(&p.lengths[b]);
      asm volatile("" : "+r"(len));
      const bool live = q0 + r < len;
      const int row0 = q0 + qtr * 32;
      const long long zrow0 = (long long)b * p.T + row0;  // row of the flat (B*T, 128) dZ / A
      tc::mbar_wait(zz_full, c & 1);
      tc::fence_after();
      uint32_t pdz[32], pa[32];
#pragma unroll
      for (int hc = 0; hc < 2; ++hc) {  // two 32-column chunks (two head groups each)
        float da[32], z[32], y[32], dy[32];
        tc::tmem_ld32x2(trow + T_DA + hf * 64 + 32 * hc, da, trow + T_Z + hf * 64 + 32 * hc, z);
        act_cols32<true>(code, hf * 64 + 32 * hc, true, z, da, p.inv_tau, y, dy);
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          pdz[16 * hc + (i >> 1)] = live ? tc::pack_bf16(dy[i], dy[i + 1]) : 0u;
          pa[16 * hc + (i >> 1)] = live ? tc::pack_bf16(y[i], y[i + 1]) : 0u;
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(zz_empty);
      // A -> this warp's staging tile (SW128, 32 rows x 64 columns) -> HBM
      if (lane == 0) tc::bulk_wait_read0();  // the previous TMA store has read the tile
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 8; ++q)
        *reinterpret_cast<uint4*>(stg + lane * 128 + ((q ^ (lane & 7)) << 4)) =
            make_uint4(pa[4 * q], pa[4 * q + 1], pa[4 * q + 2], pa[4 * q + 3]);
      tc::mbar_wait(d_empty, (c & 1) ^ 1);
#pragma unroll
      for (int g = 0; g < 4; ++g) store_sw16(sD, r, hf * 64 + 16 * g, pdz + 8 * g);
      tc::fence_async_smem();
      __syncwarp();
      const bool full_box = row0 + 32 <= p.T;  // the flat (B*T, 128) rows past T belong to the next sample
      if (lane == 0) {
        tc::mbar_arrive(d_full);
        if (full_box) {
          // dZ rows straight from the operand tile (atom hf, rows [32 qtr, +32): a SW128 box), A from staging
          tc::tma_store_3d(&tz32, sD + hf * ATOM_S + qtr * 4096, hf * 64, (int)zrow0, 0);
          tc::tma_store_3d(&ta32, stg, hf * 64, (int)zrow0, 0);
        }
        tc::bulk_commit();
      }
      if (!full_box && q0 + r < p.T) {  // sequence tail: this thread's row
        uint4* zo = reinterpret_cast<uint4*>(p.dZ + (zrow0 + lane) * HK2 + hf * 64);
        uint4* ao = reinterpret_cast<uint4*>(p.A + (zrow0 + lane) * HK2 + hf * 64);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          zo[q] = make_uint4(pdz[4 * q], pdz[4 * q + 1], pdz[4 * q + 2], pdz[4 * q + 3]);
          ao[q] = make_uint4(pa[4 * q], pa[4 * q + 1], pa[4 * q + 2], pa[4 * q + 3]);
        }
      }
      // dS_q + dY -> dS, quarter q: this warp's 32 rows x columns [128 q + 64 hf, +64)
      auto res_issue = [&](int col0) {
        if (lane == 0) {
          tc::bulk_wait_read0();
          tc::mbar_arrive_expect_tx(rb, 4096);
          tc::tma_load_3d(stg, &tg32, rb, col0, row0, b);
        }
      };
      res_issue(hf * 64);
      for (int q = 0; q < 4; ++q, ++sc) {
        const int sb = sc & 1;
        const int col0 = q * 128 + hf * 64;
        tc::mbar_wait(&s_full[sb], (sc >> 1) & 1);
        tc::fence_after();
        float acc[64];
        tc::tmem_ld32x2(trow + T_DS + sb * 128 + hf * 64, acc, trow + T_DS + sb * 128 + hf * 64 + 32, acc + 32);
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&s_empty[sb]);
        tc::mbar_wait(rb, rph & 1);
        ++rph;
        uint8_t* rowp = stg + lane * 128;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          uint4* cp = reinterpret_cast<uint4*>(rowp + ((u ^ (lane & 7)) << 4));
          const uint4 v4 = *cp;
          const uint32_t w[4] = {v4.x, v4.y, v4.z, v4.w};
          uint32_t o[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[i]));
            o[i] = tc::pack_bf16(acc[8 * u + 2 * i] + f.x, acc[8 * u + 2 * i + 1] + f.y);
          }
          *cp = make_uint4(o[0], o[1], o[2], o[3]);
        }
        tc::fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          tc::tma_store_3d(&to32, stg, col0, row0, b);
          tc::bulk_commit();
        }
        if (q + 1 < 4) res_issue(col0 + 128);
      }
    }
    if (lane == 0) tc::bulk_wait0();
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

size_t bwd512_smem() { return 1024 + 2 * BSTAGE + 2 * ATOM_S + 2 * ATOM_S + 8 * 4096 + 22 * 8 + 16; }

static int last_rc = 0;
bool map3(CUtensorMap* m, const void* ptr, long long inner, long long rows, long long B, long long ld, long long bs,
          int box_rows) {
  auto fn = tc_encode_fn();
  last_rc = -1;
  if (!fn) return false;
  last_rc = -2;
  if (((uintptr_t)ptr & 15) || (ld * 2) % 16 || (bs * 2) % 16) return false;
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)rows, (cuuint64_t)B};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * 2), (cuuint64_t)(bs * 2)};
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  last_rc = (int)fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return last_rc == (int)CUDA_SUCCESS;
}

}  // namespace gdpa
}  // namespace kl

// ---------------------------------------------------------------------------
// C ABI
using namespace kl;

static int gdpa_prepare(const kl_gdpa_args* a, const char* who, gdpa::P& p, void* stream) {
  bind_device((cudaStream_t)stream);
  if (!a || a->B < 0 || a->T < 0 || a->d < 1 || a->HK < 1 || a->n_kv < 1) {
    set_error("%s: bad extents", who);
    return KL_EBADSHAPE;
  }
  if (a->HK % a->n_kv) {
    set_error("%s: HK=%d is not a multiple of n_kv=%d", who, a->HK, a->n_kv);
    return KL_EBADSHAPE;
  }
  if (!a->lengths || !a->S || !a->Kt || !a->Vt) {
    set_error("%s: lengths, S, Kt and Vt are required", who);
    return KL_EBADSHAPE;
  }
  const bool shape_ok = (a->HK == gdpa::HK && (a->d == 128 || a->d == 256)) || (a->HK == gdpa::HK2 && a->d == 512);
  if (a->dtype != KL_BF16 || !shape_ok || !kl_tcgen05_available()) {
    set_error("%s: fused path takes bf16 with (HK=64, d in {128,256}) or (HK=128, d=512) on sm_100 "
              "(got dtype=%d HK=%d d=%d)", who, a->dtype, a->HK, a->d);
    return KL_EUNSUPPORTED;
  }
  if (a->n_act < 0 || a->n_act > KL_MAX_ACT_GROUPS) {
    set_error("%s: bad n_act %d", who, a->n_act);
    return KL_EBADSHAPE;
  }
  p.B = a->B;
  p.T = a->T;
  p.inv_tau = a->inv_tau;
  p.lengths = a->lengths;
  unsigned char codes[gdpa::HK2];
  for (int j = 0; j < a->HK; ++j) {
    const int h = j / a->n_kv;
    codes[j] = (unsigned char)(a->n_act ? a->act_codes[h % a->n_act] : KL_ACT_IDENTITY);
    if (j < gdpa::HK) p.code[j] = codes[j];
  }
  p.uniform16 = 1;
  for (int j = 0; j < a->HK; ++j) {
    if (codes[j] != codes[j & ~15]) p.uniform16 = 0;
    const int c = codes[j];
    if (c != KL_ACT_IDENTITY && c != KL_ACT_RELU && c != KL_ACT_SILU && c != KL_ACT_TANH) {
      set_error("%s: fused path takes identity/relu/silu/tanh heads (got code %d)", who, c);
      return KL_EUNSUPPORTED;
    }
  }
  if (!p.uniform16) {
    set_error("%s: fused path needs n_kv %% 16 == 0 (got %d)", who, a->n_kv);
    return KL_EUNSUPPORTED;
  }
  p.o_rs = a->s_rs;
  p.o_bs = a->s_bs;
  p.trace = (unsigned long long*)a->trace;
  p.dKt = (bf16*)a->dKt;
  p.dVt = (bf16*)a->dVt;
  return KL_OK;
}

template <int D>
static int gdpa_fwd_launch(const kl_gdpa_args* a, const gdpa::P& p, cudaStream_t s) {
  CUtensorMap ts, tk, tv, ty;
  const long long kvbs = (long long)gdpa::HK * D;
  if (!gdpa::map3(&ts, a->S, D, a->T, a->B, a->s_rs, a->s_bs, gdpa::TB) ||
      !gdpa::map3(&ty, a->Y, D, a->T, a->B, a->s_rs, a->s_bs, gdpa::TB) ||
      !gdpa::map3(&tk, a->Kt, D, gdpa::HK, a->B, D, kvbs, gdpa::HK) ||
      !gdpa::map3(&tv, a->Vt, D, gdpa::HK, a->B, D, kvbs, gdpa::HK)) {
    set_error("kl_gdpa_fwd: tensor map encode failed (alignment?)");
    return KL_EUNSUPPORTED;
  }
  const size_t smem = gdpa::fwd_smem<D>();
  cudaFuncSetAttribute(gdpa::gdpa_fwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int W = a->B * ((a->T + gdpa::TB - 1) / gdpa::TB);
  const int grid = std::min(W, tc_num_sms());
  gdpa::P q = p;
  q.out = (bf16*)a->Y;
  launch_k(gdpa::gdpa_fwd_kernel<D>, grid, gdpa::NT, smem, s, ts, tk, tv, ty, q);
  count_launch();
  count_path(KL_PATH_GDPA_FWD_TC);
  return launch_check("gdpa_fwd_tc");
}

template <int D>
static int gdpa_bwd_launch(const kl_gdpa_args* a, const gdpa::P& p, cudaStream_t s) {
  CUtensorMap ts, tg, tk, tv, tds;
  const long long kvbs = (long long)gdpa::HK * D;
  const int ok = (gdpa::map3(&ts, a->S, D, a->T, a->B, a->s_rs, a->s_bs, gdpa::TB) ? 1 : 0) |
                 (gdpa::map3(&tg, a->dY, D, a->T, a->B, a->s_rs, a->s_bs, gdpa::TB) ? 2 : 0) |
                 (gdpa::map3(&tds, a->dS, D, a->T, a->B, a->s_rs, a->s_bs, gdpa::TB) ? 4 : 0) |
                 (gdpa::map3(&tk, a->Kt, D, gdpa::HK, a->B, D, kvbs, gdpa::HK) ? 8 : 0) |
                 (gdpa::map3(&tv, a->Vt, D, gdpa::HK, a->B, D, kvbs, gdpa::HK) ? 16 : 0);
  if (ok != 31) {
    set_error("kl_gdpa_bwd: tensor map encode failed (alignment?) rc=%d mask=%d S=%p dY=%p dS=%p Kt=%p Vt=%p rs=%lld bs=%lld",
              gdpa::last_rc, ok, a->S, a->dY, a->dS, a->Kt, a->Vt, a->s_rs, a->s_bs);
    return KL_EUNSUPPORTED;
  }
  const size_t smem = gdpa::bwd_smem<D>();
  cudaFuncSetAttribute(gdpa::gdpa_bwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = std::min(a->B, tc_num_sms());
  gdpa::P q = p;
  q.out = (bf16*)a->dS;
  launch_k(gdpa::gdpa_bwd_kernel<D>, grid, gdpa::NT, smem, s, ts, tg, tk, tv, tds, q);
  count_launch();
  count_path(KL_PATH_GDPA_BWD_TC);
  return launch_check("gdpa_bwd_tc");
}

static gdpa::P5 p5_of(const kl_gdpa_args* a, const gdpa::P& p) {
  gdpa::P5 q{};
  q.B = a->B;
  q.T = a->T;
  q.inv_tau = a->inv_tau;
  q.lengths = a->lengths;
  for (int j = 0; j < gdpa::HK2; ++j) {
    const int h = j / a->n_kv;
    q.code[j] = (unsigned char)(a->n_act ? a->act_codes[h % a->n_act] : KL_ACT_IDENTITY);
  }
  q.o_rs = q.r_rs = a->s_rs;
  q.o_bs = q.r_bs = a->s_bs;
  return q;
}

static int gdpa_fwd512_launch(const kl_gdpa_args* a, const gdpa::P& p, cudaStream_t s) {
  CUtensorMap ts, tk, tv;
  const long long kvbs = (long long)gdpa::HK2 * 512;
  if (!gdpa::map3(&ts, a->S, 512, a->T, a->B, a->s_rs, a->s_bs, gdpa::TB) ||
      !gdpa::map3(&tk, a->Kt, 512, gdpa::HK2, a->B, 512, kvbs, gdpa::HK2) ||
      !gdpa::map3(&tv, a->Vt, 512, gdpa::HK2, a->B, 512, kvbs, gdpa::HK2)) {
    set_error("kl_gdpa_fwd: tensor map encode failed (alignment?)");
    return KL_EUNSUPPORTED;
  }
  if ((a->s_rs % 8) || (a->s_bs % 8) || ((uintptr_t)a->S & 15) || ((uintptr_t)a->Y & 15)) {
    set_error("kl_gdpa_fwd: S / Y rows must be 16-byte aligned");
    return KL_EUNSUPPORTED;
  }
  CUtensorMap tr32, to32;  // 32-row residual / output tiles of the epilogue
  if (!gdpa::map3(&tr32, a->S, 512, a->T, a->B, a->s_rs, a->s_bs, 32) ||
      !gdpa::map3(&to32, a->Y, 512, a->T, a->B, a->s_rs, a->s_bs, 32)) {
    set_error("kl_gdpa_fwd: tensor map encode failed (alignment?)");
    return KL_EUNSUPPORTED;
  }
  gdpa::P5 q = p5_of(a, p);
  q.trace = (unsigned long long*)a->trace;
  q.out = (bf16*)a->Y;
  q.res = (const bf16*)a->S;
  const size_t smem = gdpa::fwd512_smem();
  cudaFuncSetAttribute(gdpa::gdpa_fwd512_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int W = a->B * ((a->T + gdpa::TB - 1) / gdpa::TB);
  int grid = std::min(W, tc_num_sms());
  if (const char* g = getenv("KL_GDPA_GRID")) grid = std::max(1, std::min(grid, atoi(g)));  // testing: multi-tile CTAs
  launch_k(gdpa::gdpa_fwd512_kernel, grid, gdpa::NT6, smem, s, ts, tk, tv, tr32, to32, q);
  count_launch();
  count_path(KL_PATH_GDPA_FWD_TC512);
  return launch_check("gdpa_fwd512_tc");
}

static int gdpa_bwd512_launch(const kl_gdpa_args* a, const gdpa::P& p, cudaStream_t s) {
  if (!a->dZ_out || !a->A_out) {
    set_error("kl_gdpa_bwd: d = 512 needs dZ_out and A_out (B, T, 128) scratch");
    return KL_EBADSHAPE;
  }
  CUtensorMap ts, tg, tk, tv;
  const long long kvbs = (long long)gdpa::HK2 * 512;
  if (!gdpa::map3(&ts, a->S, 512, a->T, a->B, a->s_rs, a->s_bs, gdpa::TB) ||
      !gdpa::map3(&tg, a->dY, 512, a->T, a->B, a->s_rs, a->s_bs, gdpa::TB) ||
      !gdpa::map3(&tk, a->Kt, 512, gdpa::HK2, a->B, 512, kvbs, gdpa::HK2) ||
      !gdpa::map3(&tv, a->Vt, 512, gdpa::HK2, a->B, 512, kvbs, gdpa::HK2)) {
    set_error("kl_gdpa_bwd: tensor map encode failed (alignment?)");
    return KL_EUNSUPPORTED;
  }
  if ((a->s_rs % 8) || (a->s_bs % 8) || ((uintptr_t)a->dY & 15) || ((uintptr_t)a->dS & 15) ||
      ((uintptr_t)a->dZ_out & 15) || ((uintptr_t)a->A_out & 15)) {
    set_error("kl_gdpa_bwd: dY / dS / dZ / A rows must be 16-byte aligned");
    return KL_EUNSUPPORTED;
  }
  // Kt column quarters (128 rows x 2 boxes) and the epilogue's 32-row tiles:
  // dY residual, dS output, dZ / A rows of the flat (B*T, 128) buffers
  CUtensorMap tkq, tg32, to32, tz32, ta32;
  if (!gdpa::map3(&tkq, a->Kt, 512, gdpa::HK2, a->B, 512, kvbs, gdpa::HK2) ||
      !gdpa::map3(&tg32, a->dY, 512, a->T, a->B, a->s_rs, a->s_bs, 32) ||
      !gdpa::map3(&to32, a->dS, 512, a->T, a->B, a->s_rs, a->s_bs, 32) ||
      !gdpa::map3(&tz32, a->dZ_out, gdpa::HK2, (long long)a->B * a->T, 1, gdpa::HK2,
                  (long long)a->B * a->T * gdpa::HK2, 32) ||
      !gdpa::map3(&ta32, a->A_out, gdpa::HK2, (long long)a->B * a->T, 1, gdpa::HK2,
                  (long long)a->B * a->T * gdpa::HK2, 32)) {
    set_error("kl_gdpa_bwd: tensor map encode failed (alignment?)");
    return KL_EUNSUPPORTED;
  }
  gdpa::P5 q = p5_of(a, p);
  q.out = (bf16*)a->dS;
  q.res = (const bf16*)a->dY;
  q.dZ = (bf16*)a->dZ_out;
  q.A = (bf16*)a->A_out;
  const size_t smem = gdpa::bwd512_smem();
  cudaFuncSetAttribute(gdpa::gdpa_bwd512_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int W = a->B * ((a->T + gdpa::TB - 1) / gdpa::TB);
  int grid = std::min(W, tc_num_sms());
  if (const char* g = getenv("KL_GDPA_GRID")) grid = std::max(1, std::min(grid, atoi(g)));  // testing: multi-tile CTAs
  launch_k(gdpa::gdpa_bwd512_kernel, grid, gdpa::NT6, smem, s, ts, tg, tk, tv, tkq, tg32, to32, tz32, ta32, q);
  count_launch();
  count_path(KL_PATH_GDPA_BWD_TC512);
  return launch_check("gdpa_bwd512_tc");
}

extern "C" int kl_gdpa_fwd(const kl_gdpa_args* a, void* stream) {
  gdpa::P p;
  int rc = gdpa_prepare(a, "kl_gdpa_fwd", p, stream);
  if (rc) return rc;
  if (!a->Y) {
    set_error("kl_gdpa_fwd: Y is required");
    return KL_EBADSHAPE;
  }
  if (a->B == 0 || a->T == 0) return KL_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (a->d == 512) return gdpa_fwd512_launch(a, p, s);
  return a->d == 256 ? gdpa_fwd_launch<256>(a, p, s) : gdpa_fwd_launch<128>(a, p, s);
}

extern "C" int kl_gdpa_bwd(const kl_gdpa_args* a, void* stream) {
  gdpa::P p;
  int rc = gdpa_prepare(a, "kl_gdpa_bwd", p, stream);
  if (rc) return rc;
  if (!a->dY || !a->dS || (a->d != 512 && (!a->dKt || !a->dVt))) {
    set_error("kl_gdpa_bwd: dY, dS and (d < 512) dKt, dVt are required");
    return KL_EBADSHAPE;
  }
  if (a->B == 0) return KL_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (a->d == 512) return a->T == 0 ? KL_OK : gdpa_bwd512_launch(a, p, s);
  if (a->T == 0) {
    cudaMemsetAsync(a->dKt, 0, (size_t)a->B * a->HK * a->d * 2, s);
    cudaMemsetAsync(a->dVt, 0, (size_t)a->B * a->HK * a->d * 2, s);
    return launch_check("gdpa_bwd_tc");
  }
  return a->d == 256 ? gdpa_bwd_launch<256>(a, p, s) : gdpa_bwd_launch<128>(a, p, s);
}
