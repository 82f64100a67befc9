// Sliding-window multi-head attention on tcgen05 (sm_100a), head dim 64.
//
// Reference semantics: attention.py:69-129 (band |i-j| <= w, optional causal,
// length mask; fully-masked rows -> 0 via masked_softmax_lastdim,
// tensor.py:485-505), scale 1/sqrt(d_h) (attention.py:83).
//
// One CTA per (sample, head, 128-row block).  With w <= 128 a 128-query block
// sees at most three 128-key blocks, so every score block of a tile fits in
// TMEM at once (3 x 128 columns + the 64-column O accumulator): the softmax is
// computed exactly (row max over all visible keys first, then exp / sum), no
// online rescaling, and P never leaves the SM.  Key blocks outside the band are
// never loaded.
//
//   warp 0      TMA: Q / K / V (/ dO) blocks, 128 x 64 bf16, SWIZZLE_128B
//   warp 1      single-thread tcgen05.mma issue
//   warps 2..5  softmax / gradient math, thread = TMEM lane = row
//
// Backward (FA2 structure): a KV-major kernel accumulates dK, dV in TMEM over
// the <= 3 query blocks that see the key block; a Q-major kernel accumulates
// dQ over the <= 3 key blocks; probabilities are recomputed from the forward
// log-sum-exp.  No atomics.
#include <cudaTypedefs.h>
#include <stdlib.h>

#include <algorithm>

#include "swa.h"
#include "tc_common.cuh"

namespace kl {

PFN_cuTensorMapEncodeTiled_v12000 tc_encode_fn();
int tc_num_sms();

namespace {

constexpr int TB = 128;                 // query / key block
constexpr int DH = 64;                  // head dim handled here
constexpr int TILE = TB * DH * 2;       // 16 KB: a 128 x 64 bf16 block
constexpr int PBLK = TB * TB * 2;       // 32 KB: a 128 x 128 bf16 P / dS block
constexpr int NT = 192;

constexpr uint32_t IDESC_S = tc::idesc_bf16(128, 128, 0, 0);   // S = X Y^T, both K-major
constexpr uint32_t IDESC_PV = tc::idesc_bf16(128, 64, 0, 1);   // O += P V, V MN-major

__device__ __forceinline__ uint64_t d_kmaj64(uint32_t base, int kk) { return tc::sdesc(base + kk * 32, 16, 1024); }
__device__ __forceinline__ uint64_t d_p(uint32_t base, int kk) {
  return tc::sdesc(base + (kk >> 2) * (TB * 128) + (kk & 3) * 32, 16, 1024);
}
__device__ __forceinline__ uint64_t d_mn(uint32_t base, int kk) { return tc::sdesc(base + kk * 2048, 8192, 1024); }

__device__ __forceinline__ bool valid(int q, int k, int len, int w, int causal) {
  if (q >= len || k >= len || k < 0) return false;
  const int dd = q - k;
  if (dd > w || -dd > w) return false;
  return !(causal && k > q);
}

struct Band {
  int lo, n;
};
// 128-blocks of keys seen by queries [q0, q0+128) (forward / dQ).
__device__ __forceinline__ Band key_band(int q0, int len, int w, int causal) {
  int lo = max(0, q0 - w);
  int hi = min(len - 1, q0 + TB - 1 + w);
  if (causal) hi = min(hi, q0 + TB - 1);
  return {lo / TB, hi / TB - lo / TB + 1};
}
// 128-blocks of queries that see keys [k0, k0+128) (dK / dV).
__device__ __forceinline__ Band query_band(int k0, int len, int w, int causal) {
  int lo = max(0, k0 - w);
  if (causal) lo = max(lo, k0);
  int hi = min(len - 1, k0 + TB - 1 + w);
  return {lo / TB, hi / TB - lo / TB + 1};
}

// Store a 64-wide fp32 TMEM row (two tcgen05.ld.x32) as bf16, scaled.  The
// TMEM loads are warp-collective (.sync.aligned): every lane executes them and
// only the global store is predicated on `ok`.
__device__ __forceinline__ void store_row64(bf16* dst, uint32_t taddr, float scale, bool ok) {
  float v[32];
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    tc::tmem_ld32(taddr + half * 32, v);
    if (!ok) continue;
    uint4* o = reinterpret_cast<uint4*>(dst + half * 32);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint4 u;
      u.x = tc::pack_bf16(v[8 * c + 0] * scale, v[8 * c + 1] * scale);
      u.y = tc::pack_bf16(v[8 * c + 2] * scale, v[8 * c + 3] * scale);
      u.z = tc::pack_bf16(v[8 * c + 4] * scale, v[8 * c + 5] * scale);
      u.w = tc::pack_bf16(v[8 * c + 6] * scale, v[8 * c + 7] * scale);
      o[c] = u;
    }
  }
}


// Coalesced store of one warp's 32 rows x 64 bf16 columns (thread = row; pk =
// the row's 32 packed pairs) through a 4 KB staging region: each store
// instruction covers 4 rows x 128 B, where a row-per-thread 16-byte store
// touches 32 lines per warp instruction (4-8x the L1 wavefronts).
__device__ __forceinline__ void store_rows64_co(uint8_t* stg, const uint32_t* pk, bf16* base, long long ld, int row0,
                                                int nvalid) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int c = 0; c < 8; ++c)
    *reinterpret_cast<uint4*>(stg + lane * 128 + ((c ^ (lane & 7)) << 4)) =
        make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
  __syncwarp();
  const int c = lane & 7;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int R = (lane >> 3) + 4 * i;
    if (R < nvalid)
      *reinterpret_cast<uint4*>(base + (long long)(row0 + R) * ld + 8 * c) =
          *reinterpret_cast<const uint4*>(stg + R * 128 + ((c ^ (R & 7)) << 4));
  }
  __syncwarp();
}

// Write 32 bf16 (one tcgen05.ld.x32 worth) of row r, columns [c0, c0+32), into
// a K-major SWIZZLE_128B 128 x 128 block.
__device__ __forceinline__ void store_sw(uint8_t* blk, int r, int c0, const uint32_t* pk) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint4 u = make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
    *reinterpret_cast<uint4*>(blk + tc::sw128_off(r, c0 + 8 * c, TB)) = u;
  }
}

__device__ __forceinline__ void zero_rows(bf16* base, long long ld, int r0, int rows, int T, int tid, int nthr) {
  for (int i = tid; i < rows * DH; i += nthr) {
    const int r = r0 + i / DH;
    if (r < T) base[(long long)r * ld + i % DH] = __float2bfloat16(0.f);
  }
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(NT, 1) swa_fwd_tc_kernel(const __grid_constant__ CUtensorMap tq, SwaP p) {
  KL_PDL_ENTRY();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sQ = sm;
  uint8_t* sK = sQ + TILE;
  uint8_t* sV = sK + 3 * TILE;
  uint8_t* sP = sV + 3 * TILE;
  uint64_t* bar = (uint64_t*)(sP + 3 * PBLK);  // qk, v, s, p, o
  uint32_t* tslot = (uint32_t*)(bar + 8);

  const int b = blockIdx.z, h = blockIdx.y, q0 = blockIdx.x * TB;
  const int len = p.lengths[b];
  const int HD = p.H * DH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  bf16* O = (bf16*)p.O + (long long)b * p.bs_o + h * DH;
  if (q0 >= len) {  // padding-only tile: O = 0, LSE = +inf
    zero_rows(O, p.ld_o, q0, TB, p.T, threadIdx.x, NT);
    for (int r = threadIdx.x; r < TB; r += NT)
      if (q0 + r < p.T) p.LSE[((long long)b * p.H + h) * p.T + q0 + r] = INFINITY;
    return;
  }
  const Band kb = key_band(q0, len, p.w, p.causal);
  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tq);
    tc::mbar_init(&bar[0], 1);
    tc::mbar_init(&bar[1], 1);
    tc::mbar_init(&bar[2], 1);
    tc::mbar_init(&bar[3], 4);
    tc::mbar_init(&bar[4], 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tslot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (lane == 0) {
      tc::mbar_arrive_expect_tx(&bar[0], (1 + kb.n) * TILE);
      tc::tma_load_3d(sQ, &tq, &bar[0], h * DH, q0, b);
      for (int j = 0; j < kb.n; ++j) tc::tma_load_3d(sK + j * TILE, &tq, &bar[0], HD + h * DH, (kb.lo + j) * TB, b);
      tc::mbar_arrive_expect_tx(&bar[1], kb.n * TILE);
      for (int j = 0; j < kb.n; ++j)
        tc::tma_load_3d(sV + j * TILE, &tq, &bar[1], 2 * HD + h * DH, (kb.lo + j) * TB, b);
    }
  } else if (warp == 1) {
    if (lane == 0) {
      tc::mbar_wait(&bar[0], 0);
      tc::fence_after();
      const uint32_t q = tc::smem_u32(sQ);
      for (int j = 0; j < kb.n; ++j) {
        const uint32_t k = tc::smem_u32(sK + j * TILE);
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk)
          tc::mma_bf16(tmem + j * TB, d_kmaj64(q, kk), d_kmaj64(k, kk), IDESC_S, kk > 0);
      }
      tc::mma_commit(&bar[2]);
      tc::mbar_wait(&bar[3], 0);
      tc::mbar_wait(&bar[1], 0);
      tc::fence_after();
      for (int j = 0; j < kb.n; ++j) {
        const uint32_t pp = tc::smem_u32(sP + j * PBLK), v = tc::smem_u32(sV + j * TILE);
#pragma unroll
        for (int kk = 0; kk < TB / 16; ++kk) tc::mma_bf16(tmem + 384, d_p(pp, kk), d_mn(v, kk), IDESC_PV, (j | kk) > 0);
      }
      tc::mma_commit(&bar[4]);
    }
  } else {
    const int lb = (warp & 3) * 32, r = lb + lane, q = q0 + r;
    const uint32_t trow = tmem + ((uint32_t)lb << 16);
    const float sc = p.scale;
    tc::mbar_wait(&bar[2], 0);
    tc::fence_after();
    float m = -INFINITY;
    for (int j = 0; j < kb.n; ++j) {
      for (int c0 = 0; c0 < TB; c0 += 32) {
        float v[32];
        tc::tmem_ld32(trow + j * TB + c0, v);
        const int k0 = (kb.lo + j) * TB + c0;
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (valid(q, k0 + i, len, p.w, p.causal)) m = fmaxf(m, v[i] * sc);
      }
    }
    float l = 0.f;
    for (int j = 0; j < kb.n; ++j) {
      for (int c0 = 0; c0 < TB; c0 += 32) {
        float v[32];
        uint32_t pk[16];
        tc::tmem_ld32(trow + j * TB + c0, v);
        const int k0 = (kb.lo + j) * TB + c0;
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float a = valid(q, k0 + i, len, p.w, p.causal) ? __expf(v[i] * sc - m) : 0.f;
          const float bb = valid(q, k0 + i + 1, len, p.w, p.causal) ? __expf(v[i + 1] * sc - m) : 0.f;
          l += a + bb;
          pk[i >> 1] = tc::pack_bf16(a, bb);
        }
        store_sw(sP + j * PBLK, r, c0, pk);
      }
    }
    tc::fence_async_smem();
    tc::fence_before();
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(&bar[3]);
    tc::mbar_wait(&bar[4], 0);
    tc::fence_after();
    store_row64(O + (long long)q * p.ld_o, trow + 384, l > 0.f ? 1.f / l : 0.f, q < p.T);
    if (q < p.T) p.LSE[((long long)b * p.H + h) * p.T + q] = l > 0.f ? m + logf(l) : INFINITY;
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------------------
// dK, dV for one 128-key block.
__global__ void __launch_bounds__(NT, 1)
    swa_bwd_dkv_tc_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tdo, SwaP p) {
  KL_PDL_ENTRY();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sK = sm;
  uint8_t* sV = sK + TILE;
  uint8_t* sQ = sV + TILE;
  uint8_t* sG = sQ + 3 * TILE;
  uint8_t* sPT = sG + 3 * TILE;
  uint8_t* sDT = sPT + PBLK;
  float* lse = (float*)(sDT + PBLK);
  float* dd = lse + 3 * TB;
  uint64_t* bar = (uint64_t*)(dd + 3 * TB);  // ld, sdp, pds, mm
  uint32_t* tslot = (uint32_t*)(bar + 8);

  const int b = blockIdx.z, h = blockIdx.y, k0 = blockIdx.x * TB;
  const int len = p.lengths[b];
  const int HD = p.H * DH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  bf16* dqkv = (bf16*)p.dQKV + (long long)b * p.bs_qkv;
  if (k0 >= len) {
    zero_rows(dqkv + HD + h * DH, p.ld_qkv, k0, TB, p.T, threadIdx.x, NT);
    zero_rows(dqkv + 2 * HD + h * DH, p.ld_qkv, k0, TB, p.T, threadIdx.x, NT);
    return;
  }
  const Band qb = query_band(k0, len, p.w, p.causal);
  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tq);
    tc::prefetch_tmap(&tdo);
    tc::mbar_init(&bar[0], 1);
    tc::mbar_init(&bar[1], 1);
    tc::mbar_init(&bar[2], 4);
    tc::mbar_init(&bar[3], 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tslot, 512);
  if (warp >= 2) {  // stage LSE / D of the query blocks
    const float* LSE = p.LSE + ((long long)b * p.H + h) * p.T;
    const float* D = p.Dbuf + ((long long)b * p.H + h) * p.T;
    for (int i = threadIdx.x - 64; i < qb.n * TB; i += 128) {
      const int q = qb.lo * TB + i;
      lse[i] = q < len ? LSE[q] : INFINITY;
      dd[i] = q < len ? D[q] : 0.f;
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t T_S = 0, T_DP = 128, T_DV = 256, T_DK = 320;

  if (warp == 0) {
    if (lane == 0) {
      tc::mbar_arrive_expect_tx(&bar[0], (2 + 2 * qb.n) * TILE);
      tc::tma_load_3d(sK, &tq, &bar[0], HD + h * DH, k0, b);
      tc::tma_load_3d(sV, &tq, &bar[0], 2 * HD + h * DH, k0, b);
      for (int i = 0; i < qb.n; ++i) {
        tc::tma_load_3d(sQ + i * TILE, &tq, &bar[0], h * DH, (qb.lo + i) * TB, b);
        tc::tma_load_3d(sG + i * TILE, &tdo, &bar[0], h * DH, (qb.lo + i) * TB, b);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      tc::mbar_wait(&bar[0], 0);
      const uint32_t k = tc::smem_u32(sK), v = tc::smem_u32(sV);
      const uint32_t pt = tc::smem_u32(sPT), dt = tc::smem_u32(sDT);
      for (int i = 0; i < qb.n; ++i) {
        tc::fence_after();
        const uint32_t q = tc::smem_u32(sQ + i * TILE), g = tc::smem_u32(sG + i * TILE);
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) tc::mma_bf16(tmem + T_S, d_kmaj64(k, kk), d_kmaj64(q, kk), IDESC_S, kk > 0);
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) tc::mma_bf16(tmem + T_DP, d_kmaj64(v, kk), d_kmaj64(g, kk), IDESC_S, kk > 0);
        tc::mma_commit(&bar[1]);
        tc::mbar_wait(&bar[2], i & 1);
        tc::fence_after();
#pragma unroll
        for (int kk = 0; kk < TB / 16; ++kk)
          tc::mma_bf16(tmem + T_DV, d_p(pt, kk), d_mn(g, kk), IDESC_PV, (i | kk) > 0);
#pragma unroll
        for (int kk = 0; kk < TB / 16; ++kk)
          tc::mma_bf16(tmem + T_DK, d_p(dt, kk), d_mn(q, kk), IDESC_PV, (i | kk) > 0);
        tc::mma_commit(&bar[3]);
      }
    }
  } else {
    const int lb = (warp & 3) * 32, r = lb + lane, key = k0 + r;
    const uint32_t trow = tmem + ((uint32_t)lb << 16);
    const float sc = p.scale;
    for (int i = 0; i < qb.n; ++i) {
      tc::mbar_wait(&bar[1], i & 1);
      if (i > 0) tc::mbar_wait(&bar[3], (i - 1) & 1);  // previous MMAs done with sPT / sDT
      tc::fence_after();
      const int qbase = (qb.lo + i) * TB;
      for (int c0 = 0; c0 < TB; c0 += 32) {
        float s[32], dp[32];
        uint32_t pp[16], pd[16];
        tc::tmem_ld32(trow + T_S + c0, s);
        tc::tmem_ld32(trow + T_DP + c0, dp);
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          float pr[2], ds[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int qi = qbase + c0 + j + u;
            const int li = i * TB + c0 + j + u;
            pr[u] = valid(qi, key, len, p.w, p.causal) ? __expf(s[j + u] * sc - lse[li]) : 0.f;
            ds[u] = pr[u] * (dp[j + u] - dd[li]);
          }
          pp[j >> 1] = tc::pack_bf16(pr[0], pr[1]);
          pd[j >> 1] = tc::pack_bf16(ds[0], ds[1]);
        }
        store_sw(sPT, r, c0, pp);
        store_sw(sDT, r, c0, pd);
      }
      tc::fence_async_smem();
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&bar[2]);
    }
    tc::mbar_wait(&bar[3], (qb.n - 1) & 1);
    tc::fence_after();
    store_row64(dqkv + (long long)key * p.ld_qkv + HD + h * DH, trow + T_DK, sc, key < p.T);
    store_row64(dqkv + (long long)key * p.ld_qkv + 2 * HD + h * DH, trow + T_DV, 1.f, key < p.T);
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------------------
// dQ for one 128-query block.
__global__ void __launch_bounds__(NT, 1)
    swa_bwd_dq_tc_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tdo, SwaP p) {
  KL_PDL_ENTRY();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sQ = sm;
  uint8_t* sG = sQ + TILE;
  uint8_t* sK = sG + TILE;
  uint8_t* sV = sK + 3 * TILE;
  uint8_t* sDS = sV + 3 * TILE;
  uint64_t* bar = (uint64_t*)(sDS + PBLK);  // ld, sdp, ds, mm
  uint32_t* tslot = (uint32_t*)(bar + 8);

  const int b = blockIdx.z, h = blockIdx.y, q0 = blockIdx.x * TB;
  const int len = p.lengths[b];
  const int HD = p.H * DH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  bf16* dqkv = (bf16*)p.dQKV + (long long)b * p.bs_qkv;
  if (q0 >= len) {
    zero_rows(dqkv + h * DH, p.ld_qkv, q0, TB, p.T, threadIdx.x, NT);
    return;
  }
  const Band kb = key_band(q0, len, p.w, p.causal);
  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tq);
    tc::prefetch_tmap(&tdo);
    tc::mbar_init(&bar[0], 1);
    tc::mbar_init(&bar[1], 1);
    tc::mbar_init(&bar[2], 4);
    tc::mbar_init(&bar[3], 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tslot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t T_S = 0, T_DP = 128, T_DQ = 256;

  if (warp == 0) {
    if (lane == 0) {
      tc::mbar_arrive_expect_tx(&bar[0], (2 + 2 * kb.n) * TILE);
      tc::tma_load_3d(sQ, &tq, &bar[0], h * DH, q0, b);
      tc::tma_load_3d(sG, &tdo, &bar[0], h * DH, q0, b);
      for (int j = 0; j < kb.n; ++j) {
        tc::tma_load_3d(sK + j * TILE, &tq, &bar[0], HD + h * DH, (kb.lo + j) * TB, b);
        tc::tma_load_3d(sV + j * TILE, &tq, &bar[0], 2 * HD + h * DH, (kb.lo + j) * TB, b);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      tc::mbar_wait(&bar[0], 0);
      const uint32_t q = tc::smem_u32(sQ), g = tc::smem_u32(sG), ds = tc::smem_u32(sDS);
      for (int j = 0; j < kb.n; ++j) {
        tc::fence_after();
        const uint32_t k = tc::smem_u32(sK + j * TILE), v = tc::smem_u32(sV + j * TILE);
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) tc::mma_bf16(tmem + T_S, d_kmaj64(q, kk), d_kmaj64(k, kk), IDESC_S, kk > 0);
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) tc::mma_bf16(tmem + T_DP, d_kmaj64(g, kk), d_kmaj64(v, kk), IDESC_S, kk > 0);
        tc::mma_commit(&bar[1]);
        tc::mbar_wait(&bar[2], j & 1);
        tc::fence_after();
#pragma unroll
        for (int kk = 0; kk < TB / 16; ++kk)
          tc::mma_bf16(tmem + T_DQ, d_p(ds, kk), d_mn(k, kk), IDESC_PV, (j | kk) > 0);
        tc::mma_commit(&bar[3]);
      }
    }
  } else {
    const int lb = (warp & 3) * 32, r = lb + lane, q = q0 + r;
    const uint32_t trow = tmem + ((uint32_t)lb << 16);
    const float sc = p.scale;
    const float lse_r = q < len ? p.LSE[((long long)b * p.H + h) * p.T + q] : INFINITY;
    const float d_r = q < len ? p.Dbuf[((long long)b * p.H + h) * p.T + q] : 0.f;
    for (int j = 0; j < kb.n; ++j) {
      tc::mbar_wait(&bar[1], j & 1);
      if (j > 0) tc::mbar_wait(&bar[3], (j - 1) & 1);
      tc::fence_after();
      const int kbase = (kb.lo + j) * TB;
      for (int c0 = 0; c0 < TB; c0 += 32) {
        float s[32], dp[32];
        uint32_t pd[16];
        tc::tmem_ld32(trow + T_S + c0, s);
        tc::tmem_ld32(trow + T_DP + c0, dp);
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          float ds[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const float pr = valid(q, kbase + c0 + i + u, len, p.w, p.causal) ? __expf(s[i + u] * sc - lse_r) : 0.f;
            ds[u] = pr * (dp[i + u] - d_r);
          }
          pd[i >> 1] = tc::pack_bf16(ds[0], ds[1]);
        }
        store_sw(sDS, r, c0, pd);
      }
      tc::fence_async_smem();
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&bar[2]);
    }
    tc::mbar_wait(&bar[3], (kb.n - 1) & 1);
    tc::fence_after();
    store_row64(dqkv + (long long)q * p.ld_qkv + h * DH, trow + T_DQ, sc, q < p.T);
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

// ===========================================================================
// Forward v2: persistent, pipelined.
//
// Each CTA owns a contiguous range of (sample, head, 128-row block) work items
// in sequence order, so consecutive items are consecutive query blocks of one
// sequence: a key/value block is loaded once and reused by the (<= 3) query
// blocks that see it (3-slot ring, block j in slot j % 3).  Roles overlap
// across items: TMA prefetches the next Q / K / V while the MMA warp computes
// the next tile's scores as soon as the softmax warps have drained the current
// ones, and P V of a tile streams block by block through a 2-slot P ring.
// Eight softmax warps: warps q and q+4 share TMEM lane quarter q (rows) and
// split each 128-key block into two 64-key halves; row max / sum are combined
// through shared memory with one named barrier each.
// ===========================================================================
namespace v2 {

constexpr int NT2 = 320;  // warp 0 TMA, warp 1 MMA, warps 2..9 softmax
constexpr int KVS = 3;    // key/value ring slots

struct Item {
  int b, h, q0, len, lo, n;
  bool real;
};

__device__ __forceinline__ Item decode(const SwaP& p, int idx, int nT) {
  Item it;
  const int qt = idx % nT, bh = idx / nT;
  it.h = bh % p.H;
  it.b = bh / p.H;
  it.q0 = qt * TB;
  it.len = p.lengths[it.b];
  it.real = it.q0 < it.len;
  if (it.real) {
    const Band kb = key_band(it.q0, it.len, p.w, p.causal);
    it.lo = kb.lo;
    it.n = kb.n;
  } else {
    it.lo = 0;
    it.n = 0;
  }
  return it;
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n)); }

__global__ void __launch_bounds__(NT2, 1) swa_fwd_tc2_kernel(const __grid_constant__ CUtensorMap tq, SwaP p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sQ = sm;                       // 2 x 16 KB
  uint8_t* sKV = sQ + 2 * TILE;           // KVS x (K 16 KB | V 16 KB)
  uint8_t* sP = sKV + KVS * 2 * TILE;     // 2 x 32 KB
  // [2 halves][128 rows] max, then sum: a static array so the compiler emits
  // LDS/STS (pointers derived from the aligned dynamic base are generic)
  __shared__ float red[2 * TB];
  uint64_t* bar = (uint64_t*)(sP + 2 * PBLK);
  uint64_t* q_full = bar;        // [2]
  uint64_t* q_empty = bar + 2;   // [2]
  uint64_t* kv_full = bar + 4;   // [3]
  uint64_t* kv_empty = bar + 7;  // [3]
  uint64_t* p_full = bar + 10;   // [2]
  uint64_t* p_empty = bar + 12;  // [2]
  uint64_t* s_full = bar + 14;
  uint64_t* s_empty = bar + 15;
  uint64_t* o_full = bar + 16;
  uint64_t* o_empty = bar + 17;
  uint32_t* tslot = (uint32_t*)(bar + 18);

  const int nT = (p.T + TB - 1) / TB;
  const int W = p.B * p.H * nT;
  const int i0 = (int)((long long)W * blockIdx.x / gridDim.x);
  const int i1 = (int)((long long)W * (blockIdx.x + 1) / gridDim.x);
  const int HD = p.H * DH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tq);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&q_full[i], 1);
      tc::mbar_init(&q_empty[i], 1);
      tc::mbar_init(&p_full[i], 8);
      tc::mbar_init(&p_empty[i], 1);
    }
    for (int i = 0; i < KVS; ++i) {
      tc::mbar_init(&kv_full[i], 1);
      tc::mbar_init(&kv_empty[i], 1);
    }
    tc::mbar_init(s_full, 1);
    tc::mbar_init(s_empty, 8);
    tc::mbar_init(o_full, 1);
    tc::mbar_init(o_empty, 8);
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
  const uint32_t T_O = 384;

  if (warp == 0) {
    if (lane == 0) {
      int qcount = 0, cur_bh = -1, hi_loaded = -1;
      int kv_use[KVS] = {0, 0, 0};
      for (int idx = i0; idx < i1; ++idx) {
        const Item it = decode(p, idx, nT);
        if (!it.real) continue;
        const int bh = idx / nT;
        if (bh != cur_bh) {
          cur_bh = bh;
          hi_loaded = -1;
        }
        const int qs = qcount & 1;
        tc::mbar_wait(&q_empty[qs], ((qcount >> 1) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&q_full[qs], TILE);
        tc::tma_load_3d(sQ + qs * TILE, &tq, &q_full[qs], it.h * DH, it.q0, it.b);
        ++qcount;
        for (int j = it.lo; j < it.lo + it.n; ++j) {
          if (j <= hi_loaded) continue;
          const int s = j % KVS;
          tc::mbar_wait(&kv_empty[s], (kv_use[s] & 1) ^ 1);
          tc::mbar_arrive_expect_tx(&kv_full[s], 2 * TILE);
          tc::tma_load_3d(sKV + s * 2 * TILE, &tq, &kv_full[s], HD + it.h * DH, j * TB, it.b);
          tc::tma_load_3d(sKV + s * 2 * TILE + TILE, &tq, &kv_full[s], 2 * HD + it.h * DH, j * TB, it.b);
          ++kv_use[s];
          hi_loaded = j;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int qcount = 0, cur_bh = -1, hi_seen = -1, t = 0, pcount = 0;
      int kv_use[KVS] = {0, 0, 0};
      for (int idx = i0; idx < i1; ++idx) {
        const Item it = decode(p, idx, nT);
        if (!it.real) continue;
        const int bh = idx / nT;
        if (bh != cur_bh) {
          cur_bh = bh;
          hi_seen = -1;
        }
        const int qs = qcount & 1;
        tc::mbar_wait(&q_full[qs], (qcount >> 1) & 1);
        tc::mbar_wait(s_empty, (t & 1) ^ 1);  // softmax has drained the previous tile's scores
        const uint32_t qa = tc::smem_u32(sQ + qs * TILE);
        for (int jj = 0; jj < it.n; ++jj) {
          const int j = it.lo + jj, s = j % KVS;
          if (j > hi_seen) {
            tc::mbar_wait(&kv_full[s], kv_use[s] & 1);
            ++kv_use[s];
            hi_seen = j;
          }
          tc::fence_after();
          const uint32_t ka = tc::smem_u32(sKV + s * 2 * TILE);
#pragma unroll
          for (int kk = 0; kk < DH / 16; ++kk)
            tc::mma_bf16(tmem + jj * TB, d_kmaj64(qa, kk), d_kmaj64(ka, kk), IDESC_S, kk > 0);
        }
        tc::mma_commit(s_full);
        tc::mma_commit(&q_empty[qs]);
        ++qcount;
        tc::mbar_wait(o_empty, (t & 1) ^ 1);  // epilogue has read the previous O
        for (int jj = 0; jj < it.n; ++jj) {
          const int ps = pcount & 1;
          tc::mbar_wait(&p_full[ps], (pcount >> 1) & 1);
          tc::fence_after();
          const uint32_t pa = tc::smem_u32(sP + ps * PBLK);
          const uint32_t va = tc::smem_u32(sKV + ((it.lo + jj) % KVS) * 2 * TILE + TILE);
#pragma unroll
          for (int kk = 0; kk < TB / 16; ++kk) tc::mma_bf16(tmem + T_O, d_p(pa, kk), d_mn(va, kk), IDESC_PV, (jj | kk) > 0);
          tc::mma_commit(&p_empty[ps]);
          ++pcount;
        }
        tc::mma_commit(o_full);
        // release the key/value blocks the next item of this sequence no longer needs
        int keep_lo = it.lo + it.n;  // default: sequence ends here, release all
        if (idx + 1 < i1 && (idx + 1) / nT == bh) {
          const Item nx = decode(p, idx + 1, nT);
          if (nx.real) keep_lo = nx.lo;
        }
        for (int j = it.lo; j < it.lo + it.n && j < keep_lo; ++j) tc::mma_commit(&kv_empty[j % KVS]);
        ++t;
      }
    }
  } else {
    const int qtr = warp & 3, hf = (warp - 2) >> 2;
    const int r = qtr * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(qtr * 32) << 16);
    const float c2 = p.scale * 1.4426950408889634f;  // scores in log2 units
    int t = 0, pcount = 0;
    bf16* Obase = (bf16*)p.O;
    for (int idx = i0; idx < i1; ++idx) {
      const Item it = decode(p, idx, nT);
      bf16* O = Obase + (long long)it.b * p.bs_o + it.h * DH;
      if (!it.real) {  // padding-only tile
        const int tid = threadIdx.x - 64;
        zero_rows(O, p.ld_o, it.q0, TB, p.T, tid, 256);
        for (int rr = tid; rr < TB; rr += 256)
          if (it.q0 + rr < p.T) p.LSE[((long long)it.b * p.H + it.h) * p.T + it.q0 + rr] = INFINITY;
        continue;
      }
      const int q = it.q0 + r;
      int klo = max(0, q - p.w), khi = min(it.len - 1, q + p.w);
      if (p.causal) khi = min(khi, q);
      if (q >= it.len) khi = -1;  // padding row: nothing visible
      tc::mbar_wait(s_full, t & 1);
      tc::fence_after();
      // pass 1: row max over this half's columns
      float m = -INFINITY;
      for (int jj = 0; jj < it.n; ++jj) {
#pragma unroll
        for (int c = 0; c < 64; c += 32) {
          const int col = hf * 64 + c;
          const int k0 = (it.lo + jj) * TB + col;
          float v[32];
          tc::tmem_ld32(trow + jj * TB + col, v);
          if (k0 >= klo && k0 + 31 <= khi) {
#pragma unroll
            for (int i = 0; i < 32; ++i) m = fmaxf(m, v[i]);
          } else if (k0 <= khi && k0 + 31 >= klo) {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (k0 + i >= klo && k0 + i <= khi) m = fmaxf(m, v[i]);
          }
        }
      }
      red[hf * TB + r] = m;
      named_bar(1, 256);
      m = fmaxf(red[r], red[TB + r]);
      const float mb = (m == -INFINITY) ? 0.f : m * c2;
      // pass 2: P = exp2(s*c2 - m*c2) into the P ring, partial row sums
      float l = 0.f;
      for (int jj = 0; jj < it.n; ++jj) {
        const int ps = pcount & 1;
        tc::mbar_wait(&p_empty[ps], ((pcount >> 1) & 1) ^ 1);
        uint8_t* pblk = sP + ps * PBLK;
#pragma unroll
        for (int c = 0; c < 64; c += 32) {
          const int col = hf * 64 + c;
          const int k0 = (it.lo + jj) * TB + col;
          uint32_t pk[16];
          float v[32];
          tc::tmem_ld32(trow + jj * TB + col, v);  // warp-collective: every lane loads
          if (k0 > khi || k0 + 31 < klo) {
#pragma unroll
            for (int i = 0; i < 16; ++i) pk[i] = 0u;
          } else {
            if (k0 >= klo && k0 + 31 <= khi) {
#pragma unroll
              for (int i = 0; i < 32; i += 2) {
                const float a = ex2(fmaf(v[i], c2, -mb)), bq = ex2(fmaf(v[i + 1], c2, -mb));
                l += a + bq;
                pk[i >> 1] = tc::pack_bf16(a, bq);
              }
            } else {
#pragma unroll
              for (int i = 0; i < 32; i += 2) {
                const bool ok0 = k0 + i >= klo && k0 + i <= khi, ok1 = k0 + i + 1 >= klo && k0 + i + 1 <= khi;
                const float a = ok0 ? ex2(fmaf(v[i], c2, -mb)) : 0.f;
                const float bq = ok1 ? ex2(fmaf(v[i + 1], c2, -mb)) : 0.f;
                l += a + bq;
                pk[i >> 1] = tc::pack_bf16(a, bq);
              }
            }
          }
          store_sw(pblk, r, col, pk);
        }
        tc::fence_async_smem();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&p_full[ps]);
        ++pcount;
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(s_empty);
      red[hf * TB + r] = l;
      named_bar(1, 256);
      l = red[r] + red[TB + r];
      named_bar(1, 256);  // red reused by the next tile's max
      // epilogue: O (this half's 32 columns) / l -> bf16
      tc::mbar_wait(o_full, t & 1);
      tc::fence_after();
      {
        float v[32];
        tc::tmem_ld32(trow + T_O + hf * 32, v);
        if (q < p.T) {
          const float inv = l > 0.f ? 1.f / l : 0.f;
          uint4* o = reinterpret_cast<uint4*>(O + (long long)q * p.ld_o + hf * 32);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint4 u;
            u.x = tc::pack_bf16(v[8 * c + 0] * inv, v[8 * c + 1] * inv);
            u.y = tc::pack_bf16(v[8 * c + 2] * inv, v[8 * c + 3] * inv);
            u.z = tc::pack_bf16(v[8 * c + 4] * inv, v[8 * c + 5] * inv);
            u.w = tc::pack_bf16(v[8 * c + 6] * inv, v[8 * c + 7] * inv);
            o[c] = u;
          }
          if (hf == 0)
            p.LSE[((long long)it.b * p.H + it.h) * p.T + q] =
                l > 0.f ? (mb + __log2f(l)) * 0.6931471805599453f : INFINITY;
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(o_empty);
      ++t;
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

size_t smem_bytes() { return 1024 + 2 * TILE + KVS * 2 * TILE + 2 * PBLK + 18 * 8 + 16; }

// ---------------------------------------------------------------------------
// dQ v2: persistent over query blocks (same item order and K/V ring as the
// forward).  Per key block j: S = Q K_j^T and dP = dO V_j^T land in TMEM
// (single buffer; the next block's pair is issued as soon as the compute warps
// have read the current one), the compute warps write dS = P (dP - D) (bf16)
// into a 2-slot ring, and dQ += dS K_j accumulates in TMEM.
__global__ void __launch_bounds__(NT2, 1)
    swa_bwd_dq_tc2_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tdo, SwaP p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sQG = sm;                      // 2 x (Q 16 KB | dO 16 KB)
  uint8_t* sKV = sQG + 2 * 2 * TILE;      // KVS x (K | V)
  uint8_t* sDS = sKV + KVS * 2 * TILE;    // 2 x 32 KB
  uint64_t* bar = (uint64_t*)(sDS + 2 * PBLK);
  uint64_t* qg_full = bar;       // [2]
  uint64_t* qg_empty = bar + 2;  // [2]
  uint64_t* kv_full = bar + 4;   // [3]
  uint64_t* kv_empty = bar + 7;  // [3]
  uint64_t* ds_full = bar + 10;  // [2]
  uint64_t* ds_empty = bar + 12; // [2]
  uint64_t* sdp_full = bar + 14;
  uint64_t* sdp_empty = bar + 15;
  uint64_t* dq_full = bar + 16;
  uint64_t* dq_empty = bar + 17;
  uint32_t* tslot = (uint32_t*)(bar + 18);

  const int nT = (p.T + TB - 1) / TB;
  const int W = p.B * p.H * nT;
  const int i0 = (int)((long long)W * blockIdx.x / gridDim.x);
  const int i1 = (int)((long long)W * (blockIdx.x + 1) / gridDim.x);
  const int HD = p.H * DH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tq);
    tc::prefetch_tmap(&tdo);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&qg_full[i], 1);
      tc::mbar_init(&qg_empty[i], 1);
      tc::mbar_init(&ds_full[i], 8);
      tc::mbar_init(&ds_empty[i], 1);
    }
    for (int i = 0; i < KVS; ++i) {
      tc::mbar_init(&kv_full[i], 1);
      tc::mbar_init(&kv_empty[i], 1);
    }
    tc::mbar_init(sdp_full, 1);
    tc::mbar_init(sdp_empty, 8);
    tc::mbar_init(dq_full, 1);
    tc::mbar_init(dq_empty, 8);
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
  const uint32_t T_S = 0, T_DP = 128, T_DQ = 256;

  if (warp == 0) {
    if (lane == 0) {
      int qcount = 0, cur_bh = -1, hi_loaded = -1;
      int kv_use[KVS] = {0, 0, 0};
      for (int idx = i0; idx < i1; ++idx) {
        const Item it = decode(p, idx, nT);
        if (!it.real) continue;
        const int bh = idx / nT;
        if (bh != cur_bh) {
          cur_bh = bh;
          hi_loaded = -1;
        }
        const int qs = qcount & 1;
        tc::mbar_wait(&qg_empty[qs], ((qcount >> 1) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&qg_full[qs], 2 * TILE);
        tc::tma_load_3d(sQG + qs * 2 * TILE, &tq, &qg_full[qs], it.h * DH, it.q0, it.b);
        tc::tma_load_3d(sQG + qs * 2 * TILE + TILE, &tdo, &qg_full[qs], it.h * DH, it.q0, it.b);
        ++qcount;
        for (int j = it.lo; j < it.lo + it.n; ++j) {
          if (j <= hi_loaded) continue;
          const int s = j % KVS;
          tc::mbar_wait(&kv_empty[s], (kv_use[s] & 1) ^ 1);
          tc::mbar_arrive_expect_tx(&kv_full[s], 2 * TILE);
          tc::tma_load_3d(sKV + s * 2 * TILE, &tq, &kv_full[s], HD + it.h * DH, j * TB, it.b);
          tc::tma_load_3d(sKV + s * 2 * TILE + TILE, &tq, &kv_full[s], 2 * HD + it.h * DH, j * TB, it.b);
          ++kv_use[s];
          hi_loaded = j;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int qcount = 0, cur_bh = -1, hi_seen = -1, t = 0, sdp = 0, dsc = 0;
      int kv_use[KVS] = {0, 0, 0};
      auto score = [&](uint32_t qa, uint32_t ga, int j) {
        const uint32_t ka = tc::smem_u32(sKV + (j % KVS) * 2 * TILE), va = ka + TILE;
        tc::mbar_wait(sdp_empty, (sdp & 1) ^ 1);
        tc::fence_after();
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) tc::mma_bf16(tmem + T_S, d_kmaj64(qa, kk), d_kmaj64(ka, kk), IDESC_S, kk > 0);
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) tc::mma_bf16(tmem + T_DP, d_kmaj64(ga, kk), d_kmaj64(va, kk), IDESC_S, kk > 0);
        tc::mma_commit(sdp_full);
        ++sdp;
      };
      for (int idx = i0; idx < i1; ++idx) {
        const Item it = decode(p, idx, nT);
        if (!it.real) continue;
        const int bh = idx / nT;
        if (bh != cur_bh) {
          cur_bh = bh;
          hi_seen = -1;
        }
        const int qs = qcount & 1;
        tc::mbar_wait(&qg_full[qs], (qcount >> 1) & 1);
        const uint32_t qa = tc::smem_u32(sQG + qs * 2 * TILE), ga = qa + TILE;
        for (int jj = 0; jj < it.n; ++jj) {
          const int j = it.lo + jj, s = j % KVS;
          if (j > hi_seen) {
            tc::mbar_wait(&kv_full[s], kv_use[s] & 1);
            ++kv_use[s];
            hi_seen = j;
          }
        }
        score(qa, ga, it.lo);
        tc::mbar_wait(dq_empty, (t & 1) ^ 1);
        for (int jj = 0; jj < it.n; ++jj) {
          if (jj + 1 < it.n) score(qa, ga, it.lo + jj + 1);  // waits until block jj's S/dP were read
          else tc::mma_commit(&qg_empty[qs]);
          const int ds = dsc & 1;
          tc::mbar_wait(&ds_full[ds], (dsc >> 1) & 1);
          tc::fence_after();
          const uint32_t da = tc::smem_u32(sDS + ds * PBLK);
          const uint32_t ka = tc::smem_u32(sKV + ((it.lo + jj) % KVS) * 2 * TILE);
#pragma unroll
          for (int kk = 0; kk < TB / 16; ++kk) tc::mma_bf16(tmem + T_DQ, d_p(da, kk), d_mn(ka, kk), IDESC_PV, (jj | kk) > 0);
          tc::mma_commit(&ds_empty[ds]);
          ++dsc;
        }
        tc::mma_commit(dq_full);
        ++qcount;
        int keep_lo = it.lo + it.n;
        if (idx + 1 < i1 && (idx + 1) / nT == bh) {
          const Item nx = decode(p, idx + 1, nT);
          if (nx.real) keep_lo = nx.lo;
        }
        for (int j = it.lo; j < it.lo + it.n && j < keep_lo; ++j) tc::mma_commit(&kv_empty[j % KVS]);
        ++t;
      }
    }
  } else {
    const int qtr = warp & 3, hf = (warp - 2) >> 2;
    const int r = qtr * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(qtr * 32) << 16);
    const float c2 = p.scale * 1.4426950408889634f;
    int t = 0, sdp = 0, dsc = 0;
    bf16* dq = (bf16*)p.dQKV;
    for (int idx = i0; idx < i1; ++idx) {
      const Item it = decode(p, idx, nT);
      bf16* out = dq + (long long)it.b * p.bs_qkv + it.h * DH;
      if (!it.real) {
        zero_rows(out, p.ld_qkv, it.q0, TB, p.T, threadIdx.x - 64, 256);
        continue;
      }
      const int q = it.q0 + r;
      int klo = max(0, q - p.w), khi = min(it.len - 1, q + p.w);
      if (p.causal) khi = min(khi, q);
      float lse2 = 0.f, dr = 0.f;
      if (q < it.len) {
        lse2 = p.LSE[((long long)it.b * p.H + it.h) * p.T + q] * 1.4426950408889634f;
        dr = p.Dbuf[((long long)it.b * p.H + it.h) * p.T + q];
      } else {
        khi = -1;
      }
      for (int jj = 0; jj < it.n; ++jj) {
        tc::mbar_wait(sdp_full, sdp & 1);
        const int ds = dsc & 1;
        tc::mbar_wait(&ds_empty[ds], ((dsc >> 1) & 1) ^ 1);
        tc::fence_after();
        uint8_t* dblk = sDS + ds * PBLK;
#pragma unroll
        for (int c = 0; c < 64; c += 32) {
          const int col = hf * 64 + c;
          const int k0 = (it.lo + jj) * TB + col;
          float s[32], g[32];
          uint32_t pk[16];
          tc::tmem_ld32(trow + T_S + col, s);
          tc::tmem_ld32(trow + T_DP + col, g);
          if (k0 > khi || k0 + 31 < klo) {
#pragma unroll
            for (int i = 0; i < 16; ++i) pk[i] = 0u;
          } else if (k0 >= klo && k0 + 31 <= khi) {
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              const float a = ex2(fmaf(s[i], c2, -lse2)) * (g[i] - dr);
              const float bq = ex2(fmaf(s[i + 1], c2, -lse2)) * (g[i + 1] - dr);
              pk[i >> 1] = tc::pack_bf16(a, bq);
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              const bool ok0 = k0 + i >= klo && k0 + i <= khi, ok1 = k0 + i + 1 >= klo && k0 + i + 1 <= khi;
              const float a = ok0 ? ex2(fmaf(s[i], c2, -lse2)) * (g[i] - dr) : 0.f;
              const float bq = ok1 ? ex2(fmaf(s[i + 1], c2, -lse2)) * (g[i + 1] - dr) : 0.f;
              pk[i >> 1] = tc::pack_bf16(a, bq);
            }
          }
          store_sw(dblk, r, col, pk);
        }
        tc::fence_before();
        tc::fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          tc::mbar_arrive(sdp_empty);
          tc::mbar_arrive(&ds_full[ds]);
        }
        ++sdp;
        ++dsc;
      }
      tc::mbar_wait(dq_full, t & 1);
      tc::fence_after();
      {
        float v[32];
        tc::tmem_ld32(trow + T_DQ + hf * 32, v);
        if (q < p.T) {
          uint4* o = reinterpret_cast<uint4*>(out + (long long)q * p.ld_qkv + hf * 32);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint4 u;
            u.x = tc::pack_bf16(v[8 * c + 0] * p.scale, v[8 * c + 1] * p.scale);
            u.y = tc::pack_bf16(v[8 * c + 2] * p.scale, v[8 * c + 3] * p.scale);
            u.z = tc::pack_bf16(v[8 * c + 4] * p.scale, v[8 * c + 5] * p.scale);
            u.w = tc::pack_bf16(v[8 * c + 6] * p.scale, v[8 * c + 7] * p.scale);
            o[c] = u;
          }
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(dq_empty);
      ++t;
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

size_t dq_smem_bytes() { return 1024 + 4 * TILE + KVS * 2 * TILE + 2 * PBLK + 18 * 8 + 16; }

// ---------------------------------------------------------------------------
// dK, dV v2: persistent over key blocks in sequence order; the (<= 3) query
// blocks a key block sees come from a 3-slot Q / dO ring reused across
// consecutive key blocks.  Per query block i: S^T = K Q_i^T, dP^T = V dO_i^T
// (TMEM), compute warps write P^T and dS^T (bf16, smem), then
// dV += P^T dO_i and dK += dS^T Q_i accumulate in TMEM.  LSE / D of the query
// block are staged in smem by the compute warps.
__global__ void __launch_bounds__(NT2, 1)
    swa_bwd_dkv_tc2_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tdo, SwaP p) {
  KL_PDL_ENTRY();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sKVb = sm;                      // K 16 KB | V 16 KB
  uint8_t* sQG = sKVb + 2 * TILE;          // KVS x (Q | dO)
  uint8_t* sPT = sQG + KVS * 2 * TILE;     // 32 KB
  uint8_t* sDT = sPT + PBLK;               // 32 KB
  __shared__ __align__(16) float sLD[4 * TB];  // 2 x (lse[128] | D[128]), static: LDS.128 broadcasts
  uint64_t* bar = (uint64_t*)(sDT + PBLK);
  uint64_t* kv_full = bar;
  uint64_t* kv_empty = bar + 1;
  uint64_t* qg_full = bar + 2;   // [3]
  uint64_t* qg_empty = bar + 5;  // [3]
  uint64_t* sdp_full = bar + 8;
  uint64_t* sdp_empty = bar + 9;
  uint64_t* pd_full = bar + 10;
  uint64_t* pd_empty = bar + 11;
  uint64_t* acc_full = bar + 12;
  uint64_t* acc_empty = bar + 13;
  uint32_t* tslot = (uint32_t*)(bar + 14);

  const int nT = (p.T + TB - 1) / TB;
  const int W = p.B * p.H * nT;
  const int i0 = (int)((long long)W * blockIdx.x / gridDim.x);
  const int i1 = (int)((long long)W * (blockIdx.x + 1) / gridDim.x);
  const int HD = p.H * DH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto qband = [&](int idx, int& b, int& h, int& k0, int& len, int& lo, int& n) {
    const int kt = idx % nT, bh = idx / nT;
    h = bh % p.H;
    b = bh / p.H;
    k0 = kt * TB;
    len = p.lengths[b];
    if (k0 >= len) {
      lo = n = 0;
      return false;
    }
    const Band qb = query_band(k0, len, p.w, p.causal);
    lo = qb.lo;
    n = qb.n;
    return true;
  };
  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tq);
    tc::prefetch_tmap(&tdo);
    tc::mbar_init(kv_full, 1);
    tc::mbar_init(kv_empty, 1);
    for (int i = 0; i < KVS; ++i) {
      tc::mbar_init(&qg_full[i], 1);
      tc::mbar_init(&qg_empty[i], 1);
    }
    tc::mbar_init(sdp_full, 1);
    tc::mbar_init(sdp_empty, 8);
    tc::mbar_init(pd_full, 8);
    tc::mbar_init(pd_empty, 1);
    tc::mbar_init(acc_full, 1);
    tc::mbar_init(acc_empty, 8);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tslot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t T_S = 0, T_DP = 128, T_DV = 256, T_DK = 320;

  if (warp == 0) {
    if (lane == 0) {
      int t = 0, cur_bh = -1, hi_loaded = -1;
      int qg_use[KVS] = {0, 0, 0};
      for (int idx = i0; idx < i1; ++idx) {
        int b, h, k0, len, lo, n;
        if (!qband(idx, b, h, k0, len, lo, n)) continue;
        const int bh = idx / nT;
        if (bh != cur_bh) {
          cur_bh = bh;
          hi_loaded = -1;
        }
        tc::mbar_wait(kv_empty, (t & 1) ^ 1);
        tc::mbar_arrive_expect_tx(kv_full, 2 * TILE);
        tc::tma_load_3d(sKVb, &tq, kv_full, HD + h * DH, k0, b);
        tc::tma_load_3d(sKVb + TILE, &tq, kv_full, 2 * HD + h * DH, k0, b);
        for (int i = lo; i < lo + n; ++i) {
          if (i <= hi_loaded) continue;
          const int s = i % KVS;
          tc::mbar_wait(&qg_empty[s], (qg_use[s] & 1) ^ 1);
          tc::mbar_arrive_expect_tx(&qg_full[s], 2 * TILE);
          tc::tma_load_3d(sQG + s * 2 * TILE, &tq, &qg_full[s], h * DH, i * TB, b);
          tc::tma_load_3d(sQG + s * 2 * TILE + TILE, &tdo, &qg_full[s], h * DH, i * TB, b);
          ++qg_use[s];
          hi_loaded = i;
        }
        ++t;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int t = 0, cur_bh = -1, hi_seen = -1, sdp = 0, pdc = 0;
      int qg_use[KVS] = {0, 0, 0};
      const uint32_t ka = tc::smem_u32(sKVb), va = ka + TILE;
      const uint32_t pt = tc::smem_u32(sPT), dt = tc::smem_u32(sDT);
      for (int idx = i0; idx < i1; ++idx) {
        int b, h, k0, len, lo, n;
        if (!qband(idx, b, h, k0, len, lo, n)) continue;
        const int bh = idx / nT;
        if (bh != cur_bh) {
          cur_bh = bh;
          hi_seen = -1;
        }
        tc::mbar_wait(kv_full, t & 1);
        for (int i = lo; i < lo + n; ++i) {
          if (i <= hi_seen) continue;
          const int s = i % KVS;
          tc::mbar_wait(&qg_full[s], qg_use[s] & 1);
          ++qg_use[s];
          hi_seen = i;
        }
        auto score = [&](int i) {
          const uint32_t qa = tc::smem_u32(sQG + (i % KVS) * 2 * TILE), ga = qa + TILE;
          tc::mbar_wait(sdp_empty, (sdp & 1) ^ 1);
          tc::fence_after();
#pragma unroll
          for (int kk = 0; kk < DH / 16; ++kk) tc::mma_bf16(tmem + T_S, d_kmaj64(ka, kk), d_kmaj64(qa, kk), IDESC_S, kk > 0);
#pragma unroll
          for (int kk = 0; kk < DH / 16; ++kk) tc::mma_bf16(tmem + T_DP, d_kmaj64(va, kk), d_kmaj64(ga, kk), IDESC_S, kk > 0);
          tc::mma_commit(sdp_full);
          ++sdp;
        };
        score(lo);
        tc::mbar_wait(acc_empty, (t & 1) ^ 1);
        for (int ii = 0; ii < n; ++ii) {
          const int i = lo + ii;
          if (ii + 1 < n) score(i + 1);
          else tc::mma_commit(kv_empty);  // K / V of this block no longer read
          tc::mbar_wait(pd_full, pdc & 1);
          tc::fence_after();
          const uint32_t qa = tc::smem_u32(sQG + (i % KVS) * 2 * TILE), ga = qa + TILE;
#pragma unroll
          for (int kk = 0; kk < TB / 16; ++kk) tc::mma_bf16(tmem + T_DV, d_p(pt, kk), d_mn(ga, kk), IDESC_PV, (ii | kk) > 0);
#pragma unroll
          for (int kk = 0; kk < TB / 16; ++kk) tc::mma_bf16(tmem + T_DK, d_p(dt, kk), d_mn(qa, kk), IDESC_PV, (ii | kk) > 0);
          tc::mma_commit(pd_empty);
          ++pdc;
        }
        tc::mma_commit(acc_full);
        int keep_lo = lo + n;
        if (idx + 1 < i1 && (idx + 1) / nT == bh) {
          int b2, h2, k02, len2, lo2, n2;
          if (qband(idx + 1, b2, h2, k02, len2, lo2, n2)) keep_lo = lo2;
        }
        for (int i = lo; i < lo + n && i < keep_lo; ++i) tc::mma_commit(&qg_empty[i % KVS]);
        ++t;
      }
    }
  } else {
    const int qtr = warp & 3, hf = (warp - 2) >> 2;
    const int r = qtr * 32 + lane;
    const int ctid = threadIdx.x - 64;
    const uint32_t trow = tmem + ((uint32_t)(qtr * 32) << 16);
    const float c2 = p.scale * 1.4426950408889634f;
    int t = 0, sdp = 0, pdc = 0;
    bf16* dqkv = (bf16*)p.dQKV;
    for (int idx = i0; idx < i1; ++idx) {
      int b, h, k0, len, lo, n;
      const bool real = qband(idx, b, h, k0, len, lo, n);
      bf16* out = dqkv + (long long)b * p.bs_qkv + h * DH;
      if (!real) {
        zero_rows(out + HD, p.ld_qkv, k0, TB, p.T, ctid, 256);
        zero_rows(out + 2 * HD, p.ld_qkv, k0, TB, p.T, ctid, 256);
        continue;
      }
      const int key = k0 + r;
      int qlo = max(0, key - p.w), qhi = min(len - 1, key + p.w);
      if (p.causal) qlo = max(qlo, key);
      if (key >= len) qhi = -1;
      const float* LSE = p.LSE + ((long long)b * p.H + h) * p.T;
      const float* D = p.Dbuf + ((long long)b * p.H + h) * p.T;
      // thread ctid < 128 stages LSE (log2 units), the others D, of one query
      // row; the next block's value is loaded while this block is processed
      auto ld_ld = [&](int ii) {
        const int q = (lo + ii) * TB + (ctid & (TB - 1));
        if (ctid < TB) return q < len ? LSE[q] * 1.4426950408889634f : INFINITY;
        return q < len ? D[q] : 0.f;
      };
      float nxt = ld_ld(0);
      for (int ii = 0; ii < n; ++ii) {
        const int qb0 = (lo + ii) * TB;
        float* ls = sLD + (pdc & 1) * 2 * TB;
        float* dd = ls + TB;
        ls[ctid] = nxt;  // ctid >= TB lands in dd
        named_bar(1, 256);
        if (ii + 1 < n) nxt = ld_ld(ii + 1);
        tc::mbar_wait(sdp_full, sdp & 1);
        tc::mbar_wait(pd_empty, (pdc & 1) ^ 1);
        tc::fence_after();
#pragma unroll
        for (int c = 0; c < 64; c += 32) {
          const int col = hf * 64 + c;
          const int q0c = qb0 + col;
          float s[32], g[32];
          uint32_t pp[16], pd[16];
          tc::tmem_ld32(trow + T_S + col, s);
          tc::tmem_ld32(trow + T_DP + col, g);
          if (q0c > qhi || q0c + 31 < qlo) {
#pragma unroll
            for (int i = 0; i < 16; ++i) pp[i] = pd[i] = 0u;
          } else {
            // the 32 columns' LSE / D come from smem as float4 broadcasts
            float lv[32], dv[32];
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              *reinterpret_cast<float4*>(&lv[i]) = *reinterpret_cast<const float4*>(&ls[col + i]);
              *reinterpret_cast<float4*>(&dv[i]) = *reinterpret_cast<const float4*>(&dd[col + i]);
            }
            if (q0c >= qlo && q0c + 31 <= qhi) {
#pragma unroll
              for (int i = 0; i < 32; i += 2) {
                const float p0 = ex2(fmaf(s[i], c2, -lv[i])), p1 = ex2(fmaf(s[i + 1], c2, -lv[i + 1]));
                pp[i >> 1] = tc::pack_bf16(p0, p1);
                pd[i >> 1] = tc::pack_bf16(p0 * (g[i] - dv[i]), p1 * (g[i + 1] - dv[i + 1]));
              }
            } else {
#pragma unroll
              for (int i = 0; i < 32; i += 2) {
                float pr[2], dsv[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                  const int qi = q0c + i + u;
                  pr[u] = (qi >= qlo && qi <= qhi) ? ex2(fmaf(s[i + u], c2, -lv[i + u])) : 0.f;
                  dsv[u] = pr[u] * (g[i + u] - dv[i + u]);
                }
                pp[i >> 1] = tc::pack_bf16(pr[0], pr[1]);
                pd[i >> 1] = tc::pack_bf16(dsv[0], dsv[1]);
              }
            }
          }
          store_sw(sPT, r, col, pp);
          store_sw(sDT, r, col, pd);
        }
        tc::fence_before();
        tc::fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          tc::mbar_arrive(sdp_empty);
          tc::mbar_arrive(pd_full);
        }
        ++sdp;
        ++pdc;
      }
      tc::mbar_wait(acc_full, t & 1);
      tc::fence_after();
      {
        float v[32];
        const bool ok = key < p.T;
#pragma unroll
        for (int which = 0; which < 2; ++which) {  // 0: dK (scaled), 1: dV
          tc::tmem_ld32(trow + (which ? T_DV : T_DK) + hf * 32, v);
          const float sc = which ? 1.f : p.scale;
          if (ok) {
            uint4* o = reinterpret_cast<uint4*>(out + (long long)key * p.ld_qkv + (which ? 2 : 1) * HD + hf * 32);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              uint4 u;
              u.x = tc::pack_bf16(v[8 * c + 0] * sc, v[8 * c + 1] * sc);
              u.y = tc::pack_bf16(v[8 * c + 2] * sc, v[8 * c + 3] * sc);
              u.z = tc::pack_bf16(v[8 * c + 4] * sc, v[8 * c + 5] * sc);
              u.w = tc::pack_bf16(v[8 * c + 6] * sc, v[8 * c + 7] * sc);
              o[c] = u;
            }
          }
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(acc_empty);
      ++t;
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

size_t dkv_smem_bytes() { return 1024 + 2 * TILE + KVS * 2 * TILE + 2 * PBLK + 14 * 8 + 16; }

}  // namespace v2

// ---------------------------------------------------------------------------
// dK / dV v3: key-block-major like v2, but over 64-query half-blocks so the
// score pair (S^T, dP^T: 2 x 64 TMEM columns) is triple-buffered next to the
// dK / dV accumulators (3 x 128 + 128 = 512 columns).  Two issue warps: one
// runs the S^T / dP^T products up to three half-blocks ahead, the other the
// dV += P^T dO, dK += dS^T Q products of each block as soon as its P^T / dS^T
// land in smem.  Two gradient warpgroups take alternate half-blocks
// (ping-pong; one P^T / dS^T smem slot each).  K / V are double-buffered so
// the next key block's scores start before the current block's products
// finish; Q / dO arrive as 64-row boxes in a 4-slot ring, kept across
// consecutive key blocks of a sequence (slots the next key block does not
// see are released as soon as their products complete).  LSE / D of a tile's
// query band are staged once per tile, the next tile's prefetched into
// registers.  The issue warps walk their tiles with incremental coordinates:
// a single thread's integer bookkeeping is on the critical path.
namespace v3 {

using v2::ex2;
using v2::named_bar;
constexpr int HB = 64;                  // query half-block
constexpr int QR = 4;                   // Q | dO half-block ring slots
constexpr int HTILE = HB * DH * 2;      // 8 KB: 64 x 64 bf16
constexpr int PH = TB * HB * 2;         // 16 KB: 128 x 64 bf16 (P^T or dS^T)
constexpr int MAXQ = 6 * HB;            // queries of a tile's band
constexpr uint32_t IDESC_S64 = tc::idesc_bf16(128, 64, 0, 0);

constexpr int NT3 = 352;  // warp 0 TMA, warp 1 S^T/dP^T MMAs, warps 2..9 gradients, warp 10 dV/dK MMAs
constexpr int SDR = 2;
// pipeline clock stamps of CTA 0 (scripts/r2/swa_trace.py); compiled in only with -DKL_SWA_TRACE_BUILD
#ifdef KL_SWA_TRACE_BUILD
#define SWT(ev, idx)                                                                          \
  do {                                                                                        \
    if (p.trace && blockIdx.x == 0 && (idx) < 1024) p.trace[(ev) * 1024 + (idx)] = clock64(); \
  } while (0)
#else
#define SWT(ev, idx) \
  do {               \
  } while (0)
#endif    // dK / dV kernel: S^T | dP^T TMEM slots (the other 256 columns: two dV | dK accumulators)

struct Tile {
  int b, h, k0, len, lo, n;  // lo, n: 64-query half-blocks that see keys [k0, k0 + 128)
  bool real;
};

// Half-blocks of the band of 128-block k0: queries that see keys [k0, k0+128)
// (dK / dV, QM = false) or keys seen by queries [k0, k0+128) (dQ, QM = true).
template <bool QM = false>
__device__ __forceinline__ void band_of(const SwaP& p, Tile& t) {
  t.real = t.k0 < t.len;
  t.lo = t.n = 0;
  if (t.real) {
    int lo = max(0, t.k0 - p.w);
    int hi = min(t.len - 1, t.k0 + TB - 1 + p.w);
    if (p.causal) {
      if (QM)
        hi = min(hi, t.k0 + TB - 1);
      else
        lo = max(lo, t.k0);
    }
    t.lo = lo / HB;
    t.n = hi / HB - lo / HB + 1;
  }
}

// Walks a CTA's contiguous tile range [i0, i1) with incremental coordinates
// (no divisions on the issue threads' critical path).  Sequence order is
// head-major: with contiguous per-CTA ranges, CTAs c, c + 148/H, ... work on
// the same (sample, key block) of different heads at the same time, so the
// heads' 128-byte row pieces of Q / K / V / dO are read from DRAM together.
// Also keeps the ring position of each half-block's Q | dO load (loads are
// issued once per block of a sequence, in increasing block order).
struct Walk {
  int idx, i1, nT, kt, bh, j, t;  // t: real-tile ordinal
  int seg_bh, seg_base, seg_first, ld_end;
  Tile tl;
  bool done;
  // the length of sample lb: a sequence's tiles are consecutive, so the
  // walkers read lengths[] once per sequence instead of a dependent global
  // load on every tile
  int lb = -1, lv = 0;
};

template <bool QM = false>
__device__ __forceinline__ void walk_fill(const SwaP& p, Walk& w) {
  w.tl.k0 = w.kt * TB;
  if (w.tl.b != w.lb) {
    w.lb = w.tl.b;
    w.lv = p.lengths[w.tl.b];
  }
  w.tl.len = w.lv;
  band_of<QM>(p, w.tl);
}
__device__ __forceinline__ void walk_adv(const SwaP& p, Walk& w) {
  ++w.idx;
  if (++w.kt == w.nT) {
    w.kt = 0;
    ++w.bh;
    if (++w.tl.b == p.B) {
      w.tl.b = 0;
      ++w.tl.h;
    }
  }
}
// Move to the next real tile at or after the current position.
template <bool QM = false>
__device__ __forceinline__ void walk_settle(const SwaP& p, Walk& w) {
  for (; w.idx < w.i1; walk_adv(p, w)) {
    walk_fill<QM>(p, w);
    if (!w.tl.real) continue;
    if (w.bh != w.seg_bh) {
      w.seg_bh = w.bh;
      w.seg_base = w.ld_end;
      w.seg_first = w.tl.lo;
    }
    w.ld_end = max(w.ld_end, w.seg_base + (w.tl.lo + w.tl.n - w.seg_first));
    w.j = w.tl.lo;
    ++w.t;
    return;
  }
  w.done = true;
}
template <bool QM = false>
__device__ __forceinline__ void walk_init(const SwaP& p, Walk& w, int i0, int i1, int nT) {
  w.idx = i0;
  w.i1 = i1;
  w.nT = nT;
  w.kt = i0 % nT;
  w.bh = i0 / nT;
  w.tl.b = w.bh % p.B;
  w.tl.h = w.bh / p.B;
  w.t = -1;
  w.seg_bh = -1;
  w.seg_base = w.seg_first = w.ld_end = 0;
  w.done = false;
  walk_settle<QM>(p, w);
}
template <bool QM = false>
__device__ __forceinline__ void walk_next_tile(const SwaP& p, Walk& w) {
  walk_adv(p, w);
  walk_settle<QM>(p, w);
}
template <bool QM = false>
__device__ __forceinline__ void walk_step(const SwaP& p, Walk& w) {
  if (w.j + 1 < w.tl.lo + w.tl.n)
    ++w.j;
  else
    walk_next_tile<QM>(p, w);
}
__device__ __forceinline__ int load_index(const Walk& w, int j) { return w.seg_base + j - w.seg_first; }

__global__ void __launch_bounds__(NT3, 1)
    swa_bwd_dkv_tc3_kernel(const __grid_constant__ CUtensorMap tkv, const __grid_constant__ CUtensorMap tq64,
                           const __grid_constant__ CUtensorMap tdo64, SwaP p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sKV = sm;                    // 2 x (K 16 KB | V 16 KB)
  uint8_t* sQG = sKV + 2 * 2 * TILE;    // QR x (Q 8 KB | dO 8 KB)
  uint8_t* sPD = sQG + QR * 2 * HTILE;  // 2 x (P^T 16 KB | dS^T 16 KB)
  __shared__ __align__(16) float sLD[2][2][2][MAXQ];  // [warpgroup][tile parity][LSE (log2) | D][band query]
  uint64_t* bar = (uint64_t*)(sPD + 2 * 2 * PH);
  uint64_t* kv_full = bar;                 // [2]
  uint64_t* kv_empty = bar + 2;            // [2]
  uint64_t* qg_full = bar + 4;             // [QR]
  uint64_t* qg_empty = qg_full + QR;       // [QR]
  uint64_t* sd_full = qg_empty + QR;       // [SDR]
  uint64_t* sd_empty = sd_full + SDR;      // [SDR]
  uint64_t* pd_full = sd_empty + SDR;      // [2]
  uint64_t* pd_empty = pd_full + 2;        // [2]
  uint64_t* acc_full = pd_empty + 2;      // [2]: dV / dK accumulators double-buffered by tile parity
  uint64_t* acc_empty = acc_full + 2;     // [2]
  uint32_t* tslot = (uint32_t*)(acc_empty + 2);

  const int nT = (p.T + TB - 1) / TB;
  const int W = p.B * p.H * nT;
  const int i0 = (int)((long long)W * blockIdx.x / gridDim.x);
  const int i1 = (int)((long long)W * (blockIdx.x + 1) / gridDim.x);
  const int HD = p.H * DH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tkv);
    tc::prefetch_tmap(&tq64);
    tc::prefetch_tmap(&tdo64);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&kv_full[i], 1);
      tc::mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < QR; ++i) {
      tc::mbar_init(&qg_full[i], 1);
      tc::mbar_init(&qg_empty[i], 1);
    }
    for (int i = 0; i < SDR; ++i) {
      tc::mbar_init(&sd_full[i], 1);
      tc::mbar_init(&sd_empty[i], 4);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&pd_full[i], 4);
      tc::mbar_init(&pd_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&acc_full[i], 1);
      tc::mbar_init(&acc_empty[i], 4);
    }
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tslot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  KL_PDL_ENTRY();
  // TMEM: SDR x (S^T | dP^T) 128-column slots, then two (dV | dK) 128-column accumulators
  const uint32_t T_ACC = SDR * 128;

  if (warp == 0) {
    if (lane == 0) {
      Walk w;
      walk_init(p, w, i0, i1, nT);
      int loaded = 0;  // Q | dO loads issued (ring position)
      while (!w.done) {
        const Tile& tl = w.tl;
        const int kb = w.t & 1;
        SWT(10, w.t);
        tc::mbar_wait(&kv_empty[kb], ((w.t >> 1) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&kv_full[kb], 2 * TILE);
        tc::tma_load_3d(sKV + kb * 2 * TILE, &tkv, &kv_full[kb], HD + tl.h * DH, tl.k0, tl.b);
        tc::tma_load_3d(sKV + kb * 2 * TILE + TILE, &tkv, &kv_full[kb], 2 * HD + tl.h * DH, tl.k0, tl.b);
        for (int j = tl.lo; j < tl.lo + tl.n; ++j) {
          const int li = load_index(w, j);
          if (li < loaded) continue;  // kept from the previous key block
          const int s = li % QR;
          tc::mbar_wait(&qg_empty[s], ((li / QR) & 1) ^ 1);
          tc::mbar_arrive_expect_tx(&qg_full[s], 2 * HTILE);
          tc::tma_load_3d(sQG + s * 2 * HTILE, &tq64, &qg_full[s], tl.h * DH, j * HB, tl.b);
          tc::tma_load_3d(sQG + s * 2 * HTILE + HTILE, &tdo64, &qg_full[s], tl.h * DH, j * HB, tl.b);
          loaded = li + 1;
        }
        walk_next_tile(p, w);
      }
    }
  } else if (warp == 1) {
    // S^T = K Q_j^T and dP^T = V dO_j^T into the 3-slot TMEM ring
    if (lane == 0) {
      Walk a;
      walk_init(p, a, i0, i1, nT);
      int n = 0, waited = 0;
      const uint32_t kv0 = tc::smem_u32(sKV), qg0 = tc::smem_u32(sQG);
      while (!a.done) {
        const int kb = a.t & 1;
        SWT(0, n);
        if (a.j == a.tl.lo) tc::mbar_wait(&kv_full[kb], (a.t >> 1) & 1);
        const int li = load_index(a, a.j);
        if (li >= waited) {
          tc::mbar_wait(&qg_full[li % QR], (li / QR) & 1);
          waited = li + 1;
        }
        const int ss = n % SDR;
        SWT(1, n);
        tc::mbar_wait(&sd_empty[ss], ((n / SDR) & 1) ^ 1);
        SWT(2, n);
        tc::fence_after();
        const uint32_t ka = kv0 + kb * 2 * TILE, va = ka + TILE;
        const uint32_t qa = qg0 + (li % QR) * 2 * HTILE, ga = qa + HTILE;
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk)
          tc::mma_bf16(tmem + ss * 128, d_kmaj64(ka, kk), d_kmaj64(qa, kk), IDESC_S64, kk > 0);
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk)
          tc::mma_bf16(tmem + ss * 128 + 64, d_kmaj64(va, kk), d_kmaj64(ga, kk), IDESC_S64, kk > 0);
        tc::mma_commit(&sd_full[ss]);
        if (a.j == a.tl.lo + a.tl.n - 1) tc::mma_commit(&kv_empty[kb]);  // K / V of this tile no longer read
        ++n;
        walk_step(p, a);
      }
    }
  } else if (warp == 10) {
    // dV += P^T dO_j, dK += dS^T Q_j into the TMEM accumulators
    if (lane == 0) {
      Walk b;
      walk_init(p, b, i0, i1, nT);
      int n = 0, keep = 0;
      const uint32_t qg0 = tc::smem_u32(sQG), pd0 = tc::smem_u32(sPD);
      while (!b.done) {
        const bool first = b.j == b.tl.lo, last = b.j == b.tl.lo + b.tl.n - 1;
        if (first) {
          tc::mbar_wait(&acc_empty[b.t & 1], ((b.t >> 1) & 1) ^ 1);
          // half-blocks below `keep` are not seen by the next key block of
          // this sequence: their ring slots are released after their products
          keep = b.tl.lo + b.tl.n;
          if (b.idx + 1 < b.i1 && b.kt + 1 < nT) {
            Tile nx;
            nx.k0 = (b.kt + 1) * TB;
            nx.len = b.tl.len;
            band_of(p, nx);
            if (nx.real) keep = nx.lo;
          }
        }
        const int ps = n & 1;
        SWT(3, n);
        tc::mbar_wait(&pd_full[ps], (n >> 1) & 1);
        SWT(4, n);
        tc::fence_after();
        const int li = load_index(b, b.j);
        const uint32_t qa = qg0 + (li % QR) * 2 * HTILE, ga = qa + HTILE;
        const uint32_t pt = pd0 + ps * 2 * PH, dt = pt + PH;
#pragma unroll
        for (int kk = 0; kk < HB / 16; ++kk)
          tc::mma_bf16(tmem + T_ACC + (b.t & 1) * 128, d_kmaj64(pt, kk), d_mn(ga, kk), IDESC_PV,
                       (!first || kk > 0) ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < HB / 16; ++kk)
          tc::mma_bf16(tmem + T_ACC + (b.t & 1) * 128 + 64, d_kmaj64(dt, kk), d_mn(qa, kk), IDESC_PV,
                       (!first || kk > 0) ? 1u : 0u);
        tc::mma_commit(&pd_empty[ps]);
        if (b.j < keep) tc::mma_commit(&qg_empty[li % QR]);
        if (last) tc::mma_commit(&acc_full[b.t & 1]);
        ++n;
        walk_step(p, b);
      }
    }
  } else {
    // Two warpgroups take alternate half-blocks (ping-pong): one turns its
    // S^T / dP^T into P^T / dS^T while the other loads its scores, so TMEM
    // reads, the exp / FMA math and the smem stores of the two overlap.  A
    // thread owns one key row and the 64 query columns of its items.
    const int wg = (warp - 2) >> 2, qtr = warp & 3;
    const int r = qtr * 32 + lane;
    const int wtid = (warp - 2 - 4 * wg) * 32 + lane;  // 0..127 within the warpgroup
    const uint32_t trow = tmem + ((uint32_t)(qtr * 32) << 16);
    const float c2 = p.scale * 1.4426950408889634f;
    bf16* dqkv = (bf16*)p.dQKV;
    int n_item = 0, t = 0;
    // the next real tile's LSE (log2 units) / D, 3 band entries per thread,
    // prefetched into registers while the current tile runs
    struct LD3 {
      float l[3], d[3];
    };
    // raw loads only (in-range addresses; masked and scaled when staged): an
    // instruction that consumed the loaded values here would stall the warp
    // for the full DRAM latency at every tile
    auto fetch = [](const SwaP& pp, const Tile& tl, int tid) {
      LD3 v;
      const float* LSE = pp.LSE + ((long long)tl.b * pp.H + tl.h) * pp.T;
      const float* D = pp.Dbuf + ((long long)tl.b * pp.H + tl.h) * pp.T;
#pragma unroll
      for (int u = 0; u < 3; ++u) {
        const int q = min(tl.lo * HB + tid + u * 128, pp.T - 1);
        v.l[u] = LSE[q];
        v.d[u] = D[q];
      }
      return v;
    };
    Walk w;  // all tiles, real or not (padding key blocks get zero rows)
    w.idx = i0;
    w.i1 = i1;
    w.nT = nT;
    w.kt = i0 % nT;
    w.bh = i0 / nT;
    w.tl.b = w.bh % p.B;
    w.tl.h = w.bh / p.B;
    Walk pw = w;  // prefetch cursor: the next real tile after w
    walk_fill(p, pw);
    while (pw.idx < i1 && !pw.tl.real) {
      walk_adv(p, pw);
      if (pw.idx < i1) walk_fill(p, pw);
    }
    LD3 nx = fetch(p, pw.idx < i1 ? pw.tl : w.tl, wtid);
    for (; w.idx < i1; walk_adv(p, w)) {
      walk_fill(p, w);
      const Tile tl = w.tl;
      bf16* out = dqkv + (long long)tl.b * p.bs_qkv + tl.h * DH;
      if (!tl.real) {  // keys past the length: zero dK (warpgroup 0) / dV (1)
        zero_rows(out + (1 + wg) * HD, p.ld_qkv, tl.k0, TB, p.T, wtid, 128);
        continue;
      }
      float* ls = sLD[wg][t & 1][0];
      float* dd = sLD[wg][t & 1][1];
      if (wtid == 0) SWT(11 + wg, t);
#pragma unroll
      for (int u = 0; u < 3; ++u) {
        const int i = wtid + u * 128, q = tl.lo * HB + i;
        const bool in = i < tl.n * HB && q < tl.len;
        ls[i] = in ? nx.l[u] * 1.4426950408889634f : INFINITY;
        dd[i] = in ? nx.d[u] : 0.f;
      }
      if (wtid == 0) SWT(13 + wg, t);
      named_bar(1 + wg, 128);
      if (wtid == 0) SWT(15 + wg, t);
      pw = w;
      do {
        walk_adv(p, pw);
        if (pw.idx < i1) walk_fill(p, pw);
      } while (pw.idx < i1 && !pw.tl.real);
      nx = fetch(p, pw.idx < i1 ? pw.tl : tl, wtid);
      const int key = tl.k0 + r;
      int qlo = max(0, key - p.w), qhi = min(tl.len - 1, key + p.w);
      if (p.causal) qlo = max(qlo, key);
      if (key >= tl.len) qhi = -1;
      const int last_item = n_item + tl.n - 1;
      if (wtid == 0) SWT(17 + wg, t);
      for (int jj = 0; jj < tl.n; ++jj, ++n_item) {
        if ((n_item & 1) != wg) continue;
        const int ss = n_item % SDR;
        uint8_t* blk = sPD + wg * 2 * PH;
        if (wtid == 0) SWT(5, n_item);
        tc::mbar_wait(&sd_full[ss], (n_item / SDR) & 1);
        if (wtid == 0) SWT(6, n_item);
        tc::fence_after();
#pragma unroll 1
        for (int ch = 0; ch < 2; ++ch) {
          const int q0c = (tl.lo + jj) * HB + ch * 32;
          const int lb = jj * HB + ch * 32;  // staged band index of column 0
          float s[32], g[32];
          tc::tmem_ld32x2(trow + ss * 128 + ch * 32, s, trow + ss * 128 + 64 + ch * 32, g);
          if (ch == 1) {
            tc::fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&sd_empty[ss]);
          }
          uint32_t pp[16], pd[16];
          // warp-uniform paths (a row-dependent band edge would otherwise split
          // the warp between the full and the per-element path): all rows
          // outside the band -> zeros; all rows fully inside -> no masking;
          // else every lane runs the full math with a per-element select
          const bool none = q0c > qhi || q0c + 31 < qlo, full = q0c >= qlo && q0c + 31 <= qhi;
          if (__all_sync(0xffffffffu, none)) {
#pragma unroll
            for (int i = 0; i < 16; ++i) pp[i] = pd[i] = 0u;
          } else {
            const bool all_full = __all_sync(0xffffffffu, full);
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              const float4 l4 = *reinterpret_cast<const float4*>(&ls[lb + i]);
              const float4 d4 = *reinterpret_cast<const float4*>(&dd[lb + i]);
              float p0 = ex2(fmaf(s[i], c2, -l4.x)), p1 = ex2(fmaf(s[i + 1], c2, -l4.y));
              float p2 = ex2(fmaf(s[i + 2], c2, -l4.z)), p3 = ex2(fmaf(s[i + 3], c2, -l4.w));
              if (!all_full) {
                const int qi = q0c + i;
                p0 = (qi >= qlo && qi <= qhi) ? p0 : 0.f;
                p1 = (qi + 1 >= qlo && qi + 1 <= qhi) ? p1 : 0.f;
                p2 = (qi + 2 >= qlo && qi + 2 <= qhi) ? p2 : 0.f;
                p3 = (qi + 3 >= qlo && qi + 3 <= qhi) ? p3 : 0.f;
              }
              pp[i >> 1] = tc::pack_bf16(p0, p1);
              pp[(i >> 1) + 1] = tc::pack_bf16(p2, p3);
              pd[i >> 1] = tc::pack_bf16(p0 * (g[i] - d4.x), p1 * (g[i + 1] - d4.y));
              pd[(i >> 1) + 1] = tc::pack_bf16(p2 * (g[i + 2] - d4.z), p3 * (g[i + 3] - d4.w));
            }
          }
          // this warpgroup's P^T / dS^T slot is free once the products of
          // its previous item (two items back) have completed
          if (ch == 0) tc::mbar_wait(&pd_empty[wg], ((n_item >> 1) & 1) ^ 1);
          store_sw(blk, r, ch * 32, pp);
          store_sw(blk + PH, r, ch * 32, pd);
        }
        tc::fence_async_smem();
        __syncwarp();
        if (wtid == 0) SWT(7, n_item);
        if (lane == 0) tc::mbar_arrive(&pd_full[wg]);
      }
      // the warpgroup that took the tile's last half-block writes dK / dV
      if ((last_item & 1) == wg) {
        if (wtid == 0) SWT(8, t);
        tc::mbar_wait(&acc_full[t & 1], (t >> 1) & 1);
        if (wtid == 0) SWT(9, t);
        tc::fence_after();
        // staged in this warpgroup's P^T | dS^T slot: acc_full says every
        // product of the tile (those reading the slot included) has completed
        uint8_t* stg = sPD + wg * 2 * PH + qtr * 4096;
        const int row0 = tl.k0 + qtr * 32, nvalid = max(0, min(32, p.T - row0));
#pragma unroll 1
        for (int which = 0; which < 2; ++which) {  // 0: dK (scaled), 1: dV
          const float sc = which ? 1.f : p.scale;
          float v[64];
          const uint32_t ta = trow + T_ACC + (t & 1) * 128 + (which ? 0 : 64);
          tc::tmem_ld32x2(ta, v, ta + 32, v + 32);
          if (which == 1) {
            tc::fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&acc_empty[t & 1]);
          }
          uint32_t pk[32];
#pragma unroll
          for (int c = 0; c < 32; ++c) pk[c] = tc::pack_bf16(v[2 * c] * sc, v[2 * c + 1] * sc);
          store_rows64_co(stg, pk, out + (1 + which) * HD, p.ld_qkv, row0, nvalid);
        }
        (void)key;
        if (wtid == 0) SWT(19, t);
      }
      ++t;
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

size_t dkv_smem_bytes() { return 1024 + 2 * 2 * TILE + QR * 2 * HTILE + 2 * 2 * PH + (4 + 2 * QR + 2 * SDR + 4 + 4) * 8 + 16; }

// ---------------------------------------------------------------------------
// dQ v3: the query-block-major mirror of dK / dV v3.  A tile is a 128-query
// block, its items the 64-key half-blocks of its key band: S = Q K_j^T and
// dP = dO V_j^T (2 x 64 TMEM columns, triple-buffered) by one issue warp,
// dQ += dS_j K_j by another, two gradient warpgroups ping-ponging on
// alternate half-blocks (thread = query row: its LSE / D are two registers,
// the next tile's prefetched).  Q / dO are double-buffered per tile; K / V
// arrive as 64-row boxes in a 6-slot ring kept across consecutive query
// blocks of a sequence.
constexpr int KR = 6;  // K | V half-block ring slots
constexpr float RESCALE2 = 8.f;  // lazy-rescale threshold (log2 units)

__global__ void __launch_bounds__(NT3, 1)
    swa_bwd_dq_tc3_kernel(const __grid_constant__ CUtensorMap tqg, const __grid_constant__ CUtensorMap tdo,
                          const __grid_constant__ CUtensorMap tkv64, const __grid_constant__ CUtensorMap to, SwaP p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sQG = sm;                    // 2 x (Q 16 KB | dO 16 KB)
  uint8_t* sKV = sQG + 2 * 2 * TILE;    // KR x (K 8 KB | V 8 KB)
  uint8_t* sDS = sKV + KR * 2 * HTILE;  // 2 x dS 16 KB (one per warpgroup)
  // p.dq_rowdot: 2 x O 16 KB (the tile's O rows: D = rowsum(dO * O) is formed
  // here, replacing the separate row-dot pass over O and dO)
  uint8_t* sO = sDS + 2 * PH;
  uint64_t* bar = (uint64_t*)(sO + (p.dq_rowdot ? 2 * TILE : 0));
  uint64_t* qg_full = bar;                 // [2]
  uint64_t* qg_empty = bar + 2;            // [2]
  uint64_t* kv_full = bar + 4;             // [KR]
  uint64_t* kv_empty = kv_full + KR;       // [KR]
  uint64_t* sd_full = kv_empty + KR;       // [3]
  uint64_t* sd_empty = sd_full + 3;        // [3]
  uint64_t* ds_full = sd_empty + 3;        // [2]
  uint64_t* ds_empty = ds_full + 2;        // [2]
  uint64_t* acc_full = ds_empty + 2;
  uint64_t* acc_empty = acc_full + 1;
  uint64_t* o_empty = acc_empty + 1;       // [2] (p.dq_rowdot)
  uint32_t* tslot = (uint32_t*)(o_empty + 2);

  const int nT = (p.T + TB - 1) / TB;
  const int W = p.B * p.H * nT;
  const int i0 = (int)((long long)W * blockIdx.x / gridDim.x);
  const int i1 = (int)((long long)W * (blockIdx.x + 1) / gridDim.x);
  const int HD = p.H * DH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tqg);
    tc::prefetch_tmap(&tdo);
    tc::prefetch_tmap(&tkv64);
    if (p.dq_rowdot) tc::prefetch_tmap(&to);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&qg_full[i], 1);
      tc::mbar_init(&qg_empty[i], 1);
      tc::mbar_init(&ds_full[i], 4);
      tc::mbar_init(&ds_empty[i], 1);
      tc::mbar_init(&o_empty[i], 8);
    }
    for (int i = 0; i < KR; ++i) {
      tc::mbar_init(&kv_full[i], 1);
      tc::mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 3; ++i) {
      tc::mbar_init(&sd_full[i], 1);
      tc::mbar_init(&sd_empty[i], 4);
    }
    tc::mbar_init(acc_full, 1);
    tc::mbar_init(acc_empty, 4);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tslot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  KL_PDL_ENTRY();
  const uint32_t T_DQ = 384;

  if (warp == 0) {
    if (lane == 0) {
      Walk w;
      walk_init<true>(p, w, i0, i1, nT);
      int loaded = 0;  // K | V loads issued (ring position)
      while (!w.done) {
        const Tile& tl = w.tl;
        const int qb = w.t & 1;
        tc::mbar_wait(&qg_empty[qb], ((w.t >> 1) & 1) ^ 1);
        if (p.dq_rowdot) tc::mbar_wait(&o_empty[qb], ((w.t >> 1) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&qg_full[qb], (p.dq_rowdot ? 3 : 2) * TILE);
        tc::tma_load_3d(sQG + qb * 2 * TILE, &tqg, &qg_full[qb], tl.h * DH, tl.k0, tl.b);
        tc::tma_load_3d(sQG + qb * 2 * TILE + TILE, &tdo, &qg_full[qb], tl.h * DH, tl.k0, tl.b);
        if (p.dq_rowdot) tc::tma_load_3d(sO + qb * TILE, &to, &qg_full[qb], tl.h * DH, tl.k0, tl.b);
        for (int j = tl.lo; j < tl.lo + tl.n; ++j) {
          const int li = load_index(w, j);
          if (li < loaded) continue;  // kept from the previous query block
          const int s = li % KR;
          tc::mbar_wait(&kv_empty[s], ((li / KR) & 1) ^ 1);
          tc::mbar_arrive_expect_tx(&kv_full[s], 2 * HTILE);
          tc::tma_load_3d(sKV + s * 2 * HTILE, &tkv64, &kv_full[s], HD + tl.h * DH, j * HB, tl.b);
          tc::tma_load_3d(sKV + s * 2 * HTILE + HTILE, &tkv64, &kv_full[s], 2 * HD + tl.h * DH, j * HB, tl.b);
          loaded = li + 1;
        }
        walk_next_tile<true>(p, w);
      }
    }
  } else if (warp == 1) {
    // S = Q K_j^T and dP = dO V_j^T into the 3-slot TMEM ring
    if (lane == 0) {
      Walk a;
      walk_init<true>(p, a, i0, i1, nT);
      int n = 0, waited = 0;
      const uint32_t qg0 = tc::smem_u32(sQG), kv0 = tc::smem_u32(sKV);
      while (!a.done) {
        const int qb = a.t & 1;
        if (a.j == a.tl.lo) tc::mbar_wait(&qg_full[qb], (a.t >> 1) & 1);
        const int li = load_index(a, a.j);
        if (li >= waited) {
          tc::mbar_wait(&kv_full[li % KR], (li / KR) & 1);
          waited = li + 1;
        }
        const int ss = n % 3;
        tc::mbar_wait(&sd_empty[ss], ((n / 3) & 1) ^ 1);
        tc::fence_after();
        const uint32_t qa = qg0 + qb * 2 * TILE, ga = qa + TILE;
        const uint32_t ka = kv0 + (li % KR) * 2 * HTILE, va = ka + HTILE;
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk)
          tc::mma_bf16(tmem + ss * 128, d_kmaj64(qa, kk), d_kmaj64(ka, kk), IDESC_S64, kk > 0);
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk)
          tc::mma_bf16(tmem + ss * 128 + 64, d_kmaj64(ga, kk), d_kmaj64(va, kk), IDESC_S64, kk > 0);
        tc::mma_commit(&sd_full[ss]);
        if (a.j == a.tl.lo + a.tl.n - 1) tc::mma_commit(&qg_empty[qb]);  // Q / dO of this tile no longer read
        ++n;
        walk_step<true>(p, a);
      }
    }
  } else if (warp == 10) {
    // dQ += dS_j K_j into the TMEM accumulator
    if (lane == 0) {
      Walk b;
      walk_init<true>(p, b, i0, i1, nT);
      int n = 0, keep = 0;
      const uint32_t kv0 = tc::smem_u32(sKV), ds0 = tc::smem_u32(sDS);
      while (!b.done) {
        const bool first = b.j == b.tl.lo, last = b.j == b.tl.lo + b.tl.n - 1;
        if (first) {
          tc::mbar_wait(acc_empty, (b.t & 1) ^ 1);
          // key half-blocks below `keep` are not seen by the next query block
          // of this sequence: their ring slots are released after the product
          keep = b.tl.lo + b.tl.n;
          if (b.idx + 1 < b.i1 && b.kt + 1 < nT) {
            Tile nx;
            nx.k0 = (b.kt + 1) * TB;
            nx.len = b.tl.len;
            band_of<true>(p, nx);
            if (nx.real) keep = nx.lo;
          }
        }
        const int ps = n & 1;
        tc::mbar_wait(&ds_full[ps], (n >> 1) & 1);
        tc::fence_after();
        const int li = load_index(b, b.j);
        const uint32_t ka = kv0 + (li % KR) * 2 * HTILE;
        const uint32_t da = ds0 + ps * PH;
#pragma unroll
        for (int kk = 0; kk < HB / 16; ++kk)
          tc::mma_bf16(tmem + T_DQ, d_kmaj64(da, kk), d_mn(ka, kk), IDESC_PV, (!first || kk > 0) ? 1u : 0u);
        tc::mma_commit(&ds_empty[ps]);
        if (b.j < keep) tc::mma_commit(&kv_empty[li % KR]);
        if (last) tc::mma_commit(acc_full);
        ++n;
        walk_step<true>(p, b);
      }
    }
  } else {
    const int wg = (warp - 2) >> 2, qtr = warp & 3;
    const int r = qtr * 32 + lane;
    const int wtid = (warp - 2 - 4 * wg) * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(qtr * 32) << 16);
    const float c2 = p.scale * 1.4426950408889634f;
    bf16* dq = (bf16*)p.dQKV;
    int n_item = 0, t = 0;
    Walk w;  // all tiles, real or not (padding query blocks get zero rows)
    w.idx = i0;
    w.i1 = i1;
    w.nT = nT;
    w.kt = i0 % nT;
    w.bh = i0 / nT;
    w.tl.b = w.bh % p.B;
    w.tl.h = w.bh / p.B;
    // this row's LSE (log2 units) / D of the next real tile, prefetched
    // raw loads (masked / scaled at the tile that uses them, see dK / dV)
    auto fetch = [&](const Tile& tl, float& l2, float& dr) {
      const int q = min(tl.k0 + r, p.T - 1);
      const long long off = ((long long)tl.b * p.H + tl.h) * p.T + q;
      l2 = p.LSE[off];
      dr = p.dq_rowdot ? 0.f : p.Dbuf[off];
    };
    Walk pw = w;
    walk_fill<true>(p, pw);
    while (pw.idx < i1 && !pw.tl.real) {
      walk_adv(p, pw);
      if (pw.idx < i1) walk_fill<true>(p, pw);
    }
    float nl = 0.f, nd = 0.f;
    fetch(pw.idx < i1 ? pw.tl : w.tl, nl, nd);
    for (; w.idx < i1; walk_adv(p, w)) {
      walk_fill<true>(p, w);
      const Tile tl = w.tl;
      bf16* out = dq + (long long)tl.b * p.bs_qkv + tl.h * DH;
      if (!tl.real) {
        zero_rows(out, p.ld_qkv, tl.k0, TB, p.T, wg * 128 + wtid, 256);
        continue;
      }
      const bool qin = tl.k0 + r < tl.len;
      float drow = nd;
      if (p.dq_rowdot) {
        // D = rowsum(dO * O) of this row from the tile's smem copies (SW128
        // K-major rows of 128 B); both warpgroups form it, warpgroup 0 stores it
        // for the dK / dV kernel, which runs after this one
        const int qb = t & 1;
        tc::mbar_wait(&qg_full[qb], (t >> 1) & 1);
        const uint8_t* go = sQG + qb * 2 * TILE + TILE + r * 128;
        const uint8_t* oo = sO + qb * TILE + r * 128;
        float acc = 0.f;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int off = (c ^ (r & 7)) << 4;
          const uint4 gu = *reinterpret_cast<const uint4*>(go + off);
          const uint4 ou = *reinterpret_cast<const uint4*>(oo + off);
          const uint32_t gw[4] = {gu.x, gu.y, gu.z, gu.w}, ow[4] = {ou.x, ou.y, ou.z, ou.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&gw[i]));
            const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ow[i]));
            acc = fmaf(a.x, b.x, fmaf(a.y, b.y, acc));
          }
        }
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&o_empty[qb]);
        drow = acc;
        if (wg == 0 && tl.k0 + r < p.T) p.Dbuf[((long long)tl.b * p.H + tl.h) * p.T + tl.k0 + r] = acc;
      }
      const float lse2 = qin ? nl * 1.4426950408889634f : 0.f, dr = qin ? drow : 0.f;
      pw = w;
      do {
        walk_adv(p, pw);
        if (pw.idx < i1) walk_fill<true>(p, pw);
      } while (pw.idx < i1 && !pw.tl.real);
      fetch(pw.idx < i1 ? pw.tl : tl, nl, nd);
      const int q = tl.k0 + r;
      int klo = max(0, q - p.w), khi = min(tl.len - 1, q + p.w);
      if (p.causal) khi = min(khi, q);
      if (q >= tl.len) khi = -1;
      const int last_item = n_item + tl.n - 1;
      for (int jj = 0; jj < tl.n; ++jj, ++n_item) {
        if ((n_item & 1) != wg) continue;
        const int ss = n_item % 3;
        uint8_t* blk = sDS + wg * PH;
        tc::mbar_wait(&sd_full[ss], (n_item / 3) & 1);
        tc::fence_after();
#pragma unroll 1
        for (int ch = 0; ch < 2; ++ch) {
          const int k0c = (tl.lo + jj) * HB + ch * 32;
          float sv[32], g[32];
          tc::tmem_ld32x2(trow + ss * 128 + ch * 32, sv, trow + ss * 128 + 64 + ch * 32, g);
          if (ch == 1) {
            tc::fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&sd_empty[ss]);
          }
          uint32_t pk[16];
          // warp-uniform paths (see the dK / dV kernel)
          const bool none = k0c > khi || k0c + 31 < klo, full = k0c >= klo && k0c + 31 <= khi;
          if (__all_sync(0xffffffffu, none)) {
#pragma unroll
            for (int i = 0; i < 16; ++i) pk[i] = 0u;
          } else if (__all_sync(0xffffffffu, full)) {
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              const float a0 = ex2(fmaf(sv[i], c2, -lse2)) * (g[i] - dr);
              const float a1 = ex2(fmaf(sv[i + 1], c2, -lse2)) * (g[i + 1] - dr);
              pk[i >> 1] = tc::pack_bf16(a0, a1);
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              const bool ok0 = k0c + i >= klo && k0c + i <= khi, ok1 = k0c + i + 1 >= klo && k0c + i + 1 <= khi;
              const float e0 = ex2(fmaf(sv[i], c2, -lse2)) * (g[i] - dr);
              const float e1 = ex2(fmaf(sv[i + 1], c2, -lse2)) * (g[i + 1] - dr);
              pk[i >> 1] = tc::pack_bf16(ok0 ? e0 : 0.f, ok1 ? e1 : 0.f);
            }
          }
          if (ch == 0) tc::mbar_wait(&ds_empty[wg], ((n_item >> 1) & 1) ^ 1);
          store_sw(blk, r, ch * 32, pk);
        }
        tc::fence_async_smem();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&ds_full[wg]);
      }
      if ((last_item & 1) == wg) {
        tc::mbar_wait(acc_full, t & 1);
        tc::fence_after();
        {
          // staged in this warpgroup's dS slot (every dQ product has completed)
          float v[64];
          tc::tmem_ld32x2(trow + T_DQ, v, trow + T_DQ + 32, v + 32);
          tc::fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(acc_empty);
          uint32_t pk[32];
#pragma unroll
          for (int c = 0; c < 32; ++c) pk[c] = tc::pack_bf16(v[2 * c] * p.scale, v[2 * c + 1] * p.scale);
          const int row0 = tl.k0 + qtr * 32;
          store_rows64_co(sDS + wg * PH + qtr * 4096, pk, out, p.ld_qkv, row0, max(0, min(32, p.T - row0)));
        }
      }
      ++t;
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

size_t dq_smem_bytes() { return 1024 + 2 * 2 * TILE + KR * 2 * HTILE + 2 * PH + 2 * TILE + (4 + 2 * KR + 6 + 4 + 2 + 2) * 8 + 16; }

// ---------------------------------------------------------------------------
// Forward v3: 128-query tiles, 64-key half-block items, online softmax with
// lazy rescaling (the reference max moves only when a block max exceeds it
// by > 8 in log2 units; O is rescaled in TMEM then), two CTAs per SM.
//   warp 0     TMA: the tile's Q (128 x 64), K / V half-blocks (64 x 64) in a
//              3-slot ring
//   warp 1     S_j = Q K_j^T (N = 64) into a 3-slot TMEM ring
//   warp 2     O += P_j V_j (K = 64) into the TMEM accumulator
//   warps 3-6  softmax, thread = query row: block max, rescale, P_j = exp2
//              -> smem (2 slots), epilogue O / l -> bf16, LSE
// TMEM 256 columns (3 x 64 S + 64 O) and ~97 KB smem per CTA: two CTAs share
// an SM, so one CTA's softmax overlaps the other's MMAs and loads.
constexpr int NTF = 224;
constexpr int FNS = 3;  // S ring slots
constexpr int FKR = 3;  // K | V ring slots

__global__ void __launch_bounds__(NTF, 2)
    swa_fwd_tc3_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tkv64, SwaP p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sQ = sm;                      // 16 KB
  uint8_t* sKV = sQ + TILE;              // FKR x (K 8 KB | V 8 KB)
  uint8_t* sP = sKV + FKR * 2 * HTILE;   // 2 x P 16 KB
  uint64_t* bar = (uint64_t*)(sP + 2 * PH);
  uint64_t* q_full = bar;
  uint64_t* q_empty = bar + 1;
  uint64_t* kv_full = bar + 2;            // [FKR]
  uint64_t* kv_empty = kv_full + FKR;     // [FKR]
  uint64_t* s_full = kv_empty + FKR;      // [FNS]
  uint64_t* s_empty = s_full + FNS;       // [FNS]
  uint64_t* p_full = s_empty + FNS;       // [2]
  uint64_t* p_empty = p_full + 2;         // [2]
  uint64_t* o_full = p_empty + 2;
  uint64_t* o_empty = o_full + 1;
  uint32_t* tslot = (uint32_t*)(o_empty + 1);

  const int nT = (p.T + TB - 1) / TB;
  const int W = p.B * p.H * nT;
  const int i0 = (int)((long long)W * blockIdx.x / gridDim.x);
  const int i1 = (int)((long long)W * (blockIdx.x + 1) / gridDim.x);
  const int HD = p.H * DH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tq);
    tc::prefetch_tmap(&tkv64);
    tc::mbar_init(q_full, 1);
    tc::mbar_init(q_empty, 1);
    for (int i = 0; i < FKR; ++i) {
      tc::mbar_init(&kv_full[i], 1);
      tc::mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < FNS; ++i) {
      tc::mbar_init(&s_full[i], 1);
      tc::mbar_init(&s_empty[i], 4);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&p_full[i], 4);
      tc::mbar_init(&p_empty[i], 1);
    }
    tc::mbar_init(o_full, 1);
    tc::mbar_init(o_empty, 4);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tslot, 256);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  KL_PDL_ENTRY();
  const uint32_t T_O = FNS * 64;

  if (warp == 0) {
    if (lane == 0) {
      Walk w;
      walk_init<true>(p, w, i0, i1, nT);
      int n = 0;
      while (!w.done) {
        const Tile& tl = w.tl;
        SWT(10, w.t);
        tc::mbar_wait(q_empty, (w.t & 1) ^ 1);
        tc::mbar_arrive_expect_tx(q_full, TILE);
        tc::tma_load_3d(sQ, &tq, q_full, tl.h * DH, tl.k0, tl.b);
        for (int j = tl.lo; j < tl.lo + tl.n; ++j, ++n) {
          const int s = n % FKR;
          tc::mbar_wait(&kv_empty[s], ((n / FKR) & 1) ^ 1);
          tc::mbar_arrive_expect_tx(&kv_full[s], 2 * HTILE);
          tc::tma_load_3d(sKV + s * 2 * HTILE, &tkv64, &kv_full[s], HD + tl.h * DH, j * HB, tl.b);
          tc::tma_load_3d(sKV + s * 2 * HTILE + HTILE, &tkv64, &kv_full[s], 2 * HD + tl.h * DH, j * HB, tl.b);
        }
        walk_next_tile<true>(p, w);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      Walk a;
      walk_init<true>(p, a, i0, i1, nT);
      int n = 0;
      const uint32_t qa = tc::smem_u32(sQ), kv0 = tc::smem_u32(sKV);
      while (!a.done) {
        SWT(0, n);
        if (a.j == a.tl.lo) tc::mbar_wait(q_full, a.t & 1);
        const int s = n % FKR, ss = n % FNS;
        tc::mbar_wait(&kv_full[s], (n / FKR) & 1);
        SWT(1, n);
        tc::mbar_wait(&s_empty[ss], ((n / FNS) & 1) ^ 1);
        SWT(2, n);
        tc::fence_after();
        const uint32_t ka = kv0 + s * 2 * HTILE;
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk)
          tc::mma_bf16(tmem + ss * 64, d_kmaj64(qa, kk), d_kmaj64(ka, kk), IDESC_S64, kk > 0);
        tc::mma_commit(&s_full[ss]);
        if (a.j == a.tl.lo + a.tl.n - 1) tc::mma_commit(q_empty);
        ++n;
        walk_step<true>(p, a);
      }
    }
  } else if (warp == 2) {
    if (lane == 0) {
      Walk b;
      walk_init<true>(p, b, i0, i1, nT);
      int n = 0;
      const uint32_t kv0 = tc::smem_u32(sKV), p0 = tc::smem_u32(sP);
      while (!b.done) {
        const bool first = b.j == b.tl.lo, last = b.j == b.tl.lo + b.tl.n - 1;
        if (first) tc::mbar_wait(o_empty, (b.t & 1) ^ 1);
        const int ps = n & 1, s = n % FKR;
        SWT(3, n);
        tc::mbar_wait(&p_full[ps], (n >> 1) & 1);
        SWT(4, n);
        tc::fence_after();
        const uint32_t va = kv0 + s * 2 * HTILE + HTILE, pa = p0 + ps * PH;
#pragma unroll
        for (int kk = 0; kk < HB / 16; ++kk)
          tc::mma_bf16(tmem + T_O, d_kmaj64(pa, kk), d_mn(va, kk), IDESC_PV, (!first || kk > 0) ? 1u : 0u);
        tc::mma_commit(&p_empty[ps]);
        tc::mma_commit(&kv_empty[s]);  // S_j was read before P_j existed: K_j and V_j are done
        if (last) tc::mma_commit(o_full);
        ++n;
        walk_step<true>(p, b);
      }
    }
  } else {
    const int qtr = warp & 3;
    const int r = qtr * 32 + lane;
    const int ctid = threadIdx.x - 96;
    const uint32_t trow = tmem + ((uint32_t)(qtr * 32) << 16);
    const float c2 = p.scale * 1.4426950408889634f;
    bf16* Obase = (bf16*)p.O;
    int n = 0, t = 0;
    Walk w;
    w.idx = i0;
    w.i1 = i1;
    w.nT = nT;
    w.kt = i0 % nT;
    w.bh = i0 / nT;
    w.tl.b = w.bh % p.B;
    w.tl.h = w.bh / p.B;
    for (; w.idx < i1; walk_adv(p, w)) {
      walk_fill<true>(p, w);
      const Tile tl = w.tl;
      bf16* O = Obase + (long long)tl.b * p.bs_o + tl.h * DH;
      float* LSE = p.LSE + ((long long)tl.b * p.H + tl.h) * p.T;
      if (!tl.real) {  // padding-only query block
        zero_rows(O, p.ld_o, tl.k0, TB, p.T, ctid, 128);
        if (tl.k0 + ctid < p.T) LSE[tl.k0 + ctid] = INFINITY;
        continue;
      }
      const int q = tl.k0 + r;
      int klo = max(0, q - p.w), khi = min(tl.len - 1, q + p.w);
      if (p.causal) khi = min(khi, q);
      if (q >= tl.len) khi = -1;
      float mref = -INFINITY, l = 0.f;
      for (int jj = 0; jj < tl.n; ++jj, ++n) {
        const int ss = n % FNS, ps = n & 1;
        const int k0 = (tl.lo + jj) * HB;
        float v[64];
        if (ctid == 0) SWT(5, n);
        tc::mbar_wait(&s_full[ss], (n / FNS) & 1);
        if (ctid == 0) SWT(6, n);
        tc::fence_after();
        tc::tmem_ld32x2(trow + ss * 64, v, trow + ss * 64 + 32, v + 32);
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&s_empty[ss]);
        // mask to -inf outside [klo, khi]; block max in log2 units
        float mb = -INFINITY;
        if (__all_sync(0xffffffffu, k0 >= klo && k0 + 63 <= khi)) {  // warp-uniform (band edges cross warps)
#pragma unroll
          for (int i = 0; i < 64; ++i) mb = fmaxf(mb, v[i]);
        } else {
#pragma unroll
          for (int i = 0; i < 64; ++i) {
            const bool ok = k0 + i >= klo && k0 + i <= khi;
            v[i] = ok ? v[i] : -INFINITY;
            mb = fmaxf(mb, v[i]);
          }
        }
        mb = mb == -INFINITY ? -INFINITY : mb * c2;
        const bool up = mb > mref + RESCALE2;
        // the P slot is free once the product of the item two back completed
        if (ctid == 0) SWT(7, n);
        tc::mbar_wait(&p_empty[ps], ((n >> 1) & 1) ^ 1);
        if (ctid == 0) SWT(8, n);
        if (jj > 0 && __any_sync(0xffffffffu, up)) {
          // O must be stable: the previous item's product has completed too
          tc::mbar_wait(&p_empty[ps ^ 1], (((n - 1) >> 1) & 1));
          tc::fence_after();
          const float al = up ? ex2(mref - mb) : 1.f;
          l *= al;
#pragma unroll 1
          for (int c0 = 0; c0 < DH; c0 += 16) {
            float o[16];
            uint32_t u[16];
            tc::tmem_ld16(trow + T_O + c0, o);
#pragma unroll
            for (int i = 0; i < 16; ++i) u[i] = __float_as_uint(o[i] * al);
            tc::tmem_st16(trow + T_O + c0, u);
          }
          tc::fence_before();
        }
        if (up) mref = mb;
        const float mr = mref == -INFINITY ? 0.f : mref;  // nothing visible yet: every P is exp2(-inf) = 0
        uint32_t pk[32];
#pragma unroll
        for (int i = 0; i < 64; i += 2) {
          const float a0 = ex2(fmaf(v[i], c2, -mr)), a1 = ex2(fmaf(v[i + 1], c2, -mr));
          l += a0 + a1;
          pk[i >> 1] = tc::pack_bf16(a0, a1);
        }
        uint8_t* blk = sP + ps * PH;
        store_sw(blk, r, 0, pk);
        store_sw(blk, r, 32, pk + 16);
        tc::fence_async_smem();
        __syncwarp();
        if (ctid == 0) SWT(9, n);
        if (lane == 0) tc::mbar_arrive(&p_full[ps]);
      }
      if (ctid == 0) SWT(11, t);
      tc::mbar_wait(o_full, t & 1);
      if (ctid == 0) SWT(12, t);
      tc::fence_after();
      float o[64];
      tc::tmem_ld32(trow + T_O, o);
      tc::tmem_ld32(trow + T_O + 32, o + 32);
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(o_empty);
      {
        // staged in P slot 0 (this warp's 32 rows of it): o_full says the
        // tile's P V products, the last readers of P, have completed
        const float inv = l > 0.f ? 1.f / l : 0.f;
        uint32_t pk[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) pk[c] = tc::pack_bf16(o[2 * c] * inv, o[2 * c + 1] * inv);
        const int row0 = q - lane;
        store_rows64_co(sP + qtr * 4096, pk, O, p.ld_o, row0, max(0, min(32, p.T - row0)));
        if (q < p.T) LSE[q] = l > 0.f ? (mref + __log2f(l)) * 0.6931471805599453f : INFINITY;
      }
      if (ctid == 0) SWT(13, t);
      ++t;
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 256);
}

size_t fwd_smem_bytes() { return 1024 + TILE + FKR * 2 * HTILE + 2 * PH + (2 + 2 * FKR + 2 * FNS + 4 + 2) * 8 + 16; }

}  // namespace v3

bool map3(CUtensorMap* m, const void* ptr, long long inner, int T, int B, long long ld, long long bs,
          unsigned rows = 128) {
  auto fn = tc_encode_fn();
  if (!fn) return false;
  if (((uintptr_t)ptr & 15) || (ld * 2) % 16 || (bs * 2) % 16) return false;
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)T, (cuuint64_t)B};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * 2), (cuuint64_t)(bs * 2)};
  cuuint32_t box[3] = {64, rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// The tile walks hold a band of at most three 128-blocks (the dK / dV kernel
// stages the LSE / D of <= 6 64-query half-blocks per tile): w <= 128.  Wider
// windows (mha_full) run the SIMT kernels.
bool supported(const SwaP& p) {
  return p.dtype == KL_BF16 && p.d_h == DH && p.w <= TB && kl_tcgen05_available();
}

}  // namespace

int swa_rowdot(const SwaP& p, cudaStream_t s);

int swa_fwd_tc(const SwaP& p0, cudaStream_t s) {
  if (!supported(p0)) return KL_EUNSUPPORTED;
  SwaP p = p0;
  if (const char* tv = getenv("KL_SWA_TRACE_FWD")) p.trace = (unsigned long long*)strtoull(tv, nullptr, 0);  // testing
  CUtensorMap tq;
  if (!map3(&tq, p.QKV, 3LL * p.H * DH, p.T, p.B, p.ld_qkv, p.bs_qkv)) return KL_EUNSUPPORTED;
  if (getenv("KL_SWA_FWD_V1")) {
    const size_t smem = 1024 + 7 * TILE + 3 * PBLK + 64 + 16;
    cudaFuncSetAttribute(swa_fwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 grid((p.T + TB - 1) / TB, p.H, p.B);
    launch_k(swa_fwd_tc_kernel, grid, NT, smem, s, tq, p);
  } else {
    const int W = p.B * p.H * ((p.T + TB - 1) / TB);
    CUtensorMap tkv64;
    if (!getenv("KL_SWA_FWD_V2") && map3(&tkv64, p.QKV, 3LL * p.H * DH, p.T, p.B, p.ld_qkv, p.bs_qkv, 64)) {
      const size_t smem = v3::fwd_smem_bytes();
      cudaFuncSetAttribute(v3::swa_fwd_tc3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      const int grid = std::min(W, 2 * tc_num_sms());
      launch_k(v3::swa_fwd_tc3_kernel, grid, v3::NTF, smem, s, tq, tkv64, p);
    } else {
      const size_t smem = v2::smem_bytes();
      cudaFuncSetAttribute(v2::swa_fwd_tc2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      const int grid = std::min(W, tc_num_sms());
      launch_k(v2::swa_fwd_tc2_kernel, grid, v2::NT2, smem, s, tq, p);
    }
  }
  count_launch();
  count_path(KL_PATH_SWA_FWD_TC);
  return launch_check("swa_fwd_tc");
}

int swa_bwd_tc(const SwaP& p, cudaStream_t s) {
  if (!supported(p)) return KL_EUNSUPPORTED;
  CUtensorMap tq, tdo;
  if (!map3(&tq, p.QKV, 3LL * p.H * DH, p.T, p.B, p.ld_qkv, p.bs_qkv)) return KL_EUNSUPPORTED;
  if (!map3(&tdo, p.dO, (long long)p.H * DH, p.T, p.B, p.ld_o, p.bs_o)) return KL_EUNSUPPORTED;
  // default v3 path: the dQ kernel forms D = rowsum(dO * O) itself and runs
  // first (the dK / dV kernel reads D); other paths keep the row-dot pass
  const bool fuse_d = !getenv("KL_SWA_BWD_V1") && !getenv("KL_SWA_DKV_V2") && !getenv("KL_SWA_DQ_V2") &&
                      !getenv("KL_SWA_ROWDOT");
  CUtensorMap to;
  const bool to_ok = fuse_d && map3(&to, p.O, (long long)p.H * DH, p.T, p.B, p.ld_o, p.bs_o);
  if (!to_ok) {
    int rc = swa_rowdot(p, s);
    if (rc) return rc;
  }
  SwaP pt = p;
  if (const char* tv = getenv("KL_SWA_TRACE")) pt.trace = (unsigned long long*)strtoull(tv, nullptr, 0);  // testing
  if (!getenv("KL_SWA_BWD_V1")) {
    const int W = p.B * p.H * ((p.T + TB - 1) / TB);
    const int grid = std::min(W, tc_num_sms());
    const size_t s2 = v2::dq_smem_bytes();
    static int dkv_v = -1;
    if (dkv_v < 0) dkv_v = getenv("KL_SWA_DKV_V2") ? 2 : 3;
    CUtensorMap tq64, tdo64, tkv64;
    if (to_ok && map3(&tkv64, p.QKV, 3LL * p.H * DH, p.T, p.B, p.ld_qkv, p.bs_qkv, 64)) {
      SwaP pq = p;
      pq.dq_rowdot = 1;
      const size_t s3 = v3::dq_smem_bytes();
      cudaFuncSetAttribute(v3::swa_bwd_dq_tc3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s3);
      launch_k(v3::swa_bwd_dq_tc3_kernel, grid, v3::NT3, s3, s, tq, tdo, tkv64, to, pq);
    }
    if (dkv_v == 3 && map3(&tq64, p.QKV, 3LL * p.H * DH, p.T, p.B, p.ld_qkv, p.bs_qkv, 64) &&
        map3(&tdo64, p.dO, (long long)p.H * DH, p.T, p.B, p.ld_o, p.bs_o, 64)) {
      const size_t s1 = v3::dkv_smem_bytes();
      cudaFuncSetAttribute(v3::swa_bwd_dkv_tc3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1);
      launch_k(v3::swa_bwd_dkv_tc3_kernel, grid, v3::NT3, s1, s, tq, tq64, tdo64, pt);
    } else {
      const size_t s1 = v2::dkv_smem_bytes();
      cudaFuncSetAttribute(v2::swa_bwd_dkv_tc2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1);
      launch_k(v2::swa_bwd_dkv_tc2_kernel, grid, v2::NT2, s1, s, tq, tdo, p);
    }
    if (to_ok) {
      // dQ already ran (it formed D)
    } else if (!getenv("KL_SWA_DQ_V2") && map3(&tkv64, p.QKV, 3LL * p.H * DH, p.T, p.B, p.ld_qkv, p.bs_qkv, 64)) {
      const size_t s3 = v3::dq_smem_bytes();
      cudaFuncSetAttribute(v3::swa_bwd_dq_tc3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s3);
      launch_k(v3::swa_bwd_dq_tc3_kernel, grid, v3::NT3, s3, s, tq, tdo, tkv64, tkv64, p);
    } else {
      cudaFuncSetAttribute(v2::swa_bwd_dq_tc2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s2);
      launch_k(v2::swa_bwd_dq_tc2_kernel, grid, v2::NT2, s2, s, tq, tdo, p);
    }
    count_launch(2);
    count_path(KL_PATH_SWA_BWD_TC);
    return launch_check("swa_bwd_tc2");
  }
  dim3 grid((p.T + TB - 1) / TB, p.H, p.B);
  const size_t smem1 = 1024 + 8 * TILE + 2 * PBLK + 6 * TB * 4 + 64 + 16;
  cudaFuncSetAttribute(swa_bwd_dkv_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1);
  launch_k(swa_bwd_dkv_tc_kernel, grid, NT, smem1, s, tq, tdo, p);
  const size_t smem2 = 1024 + 8 * TILE + PBLK + 64 + 16;
  cudaFuncSetAttribute(swa_bwd_dq_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
  launch_k(swa_bwd_dq_tc_kernel, grid, NT, smem2, s, tq, tdo, p);
  count_launch(2);
  count_path(KL_PATH_SWA_BWD_TC);
  return launch_check("swa_bwd_tc");
}

}  // namespace kl
