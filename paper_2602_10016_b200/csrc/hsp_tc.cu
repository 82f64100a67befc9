// Fused Hierarchical Seed Pooling / PMA cross-attention on tcgen05 (sm_100a).
//
// Reference: hsp_seed_attend / pma (seqsum.py:26-34, 96-102) =
// multi_head_attention(queries, S, S) (attention.py:69-93) with batch-shared
// queries and keys = values = the event sequence S.  The B200 path folds the
// key projection into the queries once per step (Qt = q W_q^T W_k / sqrt(d_h),
// SURVEY.md §7.3 item 7), so per sample the pooling is
//     Z = Qt S^T  (HQ x T),   P = softmax over t < len  (row-wise in Z),
//     pooled = P S            (HQ x d)
// i.e. flash attention with HQ query rows, T key rows, head dim d, and the
// value matrix equal to the key matrix.  Empty sequences pool to zeros.
//
// Forward, persistent CTAs over (query tile, sample) items (query tile-major,
// so consecutive items of a CTA reuse the query tile in smem):
//   warp 0     TMA: Qt tile (128 x d, once per query tile), 2-slot ring of
//              S blocks (128 rows x d, SWIZZLE_128B atoms of 64 columns)
//   warp 1     MMA: Z_j = Qt S_j^T into a double-buffered TMEM accumulator
//              (2 x 128 columns); O += P_j S_j (S_j read as the MN-major B
//              operand, N = d <= 256 columns of TMEM)
//   warps 2-5  softmax: thread = query row.  Online softmax in log2 units with
//              lazy rescaling (the reference max moves only when a block max
//              exceeds it by > 8, i.e. P <= 256 in bf16), P_j -> smem (bf16,
//              the K-major A operand of the second MMA); epilogue O / l ->
//              bf16 rows of the seed / CLS outputs, LSE (natural log) saved
//              for the backward.
// Traffic per sample: S read once (T*d*2 bytes) + the tiny pooled rows.
#include <cudaTypedefs.h>

#include <stdlib.h>

#include <algorithm>

#include "common.cuh"
#include "tc_common.cuh"

namespace kl {

PFN_cuTensorMapEncodeTiled_v12000 tc_encode_fn();
int tc_num_sms();

namespace hsp {

constexpr int TB = 128;                // rows of a query tile / an S block
constexpr int NT = 192;                // warp 0 TMA, warp 1 MMA, warps 2-5 softmax
constexpr uint32_t ATOM = TB * 128;    // 128 rows x 64 bf16 (16 KB)
constexpr float LOG2E = 1.4426950408889634f;
constexpr float RESCALE = 8.f;         // lazy-rescale threshold (log2 units)

struct FwdP {
  int B, T, HQ, n1, qtiles;
  int qg;  // samples per query set: sample b pools with query set b / qg (grouped event types)
  const int* lengths;
  bf16* O1;  // query rows [0, n1): (B, n1, D), batch stride o1_bs
  long long o1_bs;
  bf16* O2;  // query rows [n1, HQ): (B, HQ - n1, D)
  long long o2_bs;
  float* LSE;  // (B, HQ), natural log; +inf for empty samples
  unsigned* trace;  // debug: host-mapped [cta][role][4] progress words, or NULL
};

#define HSP_TRACE(role, a, b, c)                                                        \
  do {                                                                                  \
    if (p.trace) {                                                                      \
      volatile unsigned* tr_ = p.trace + (blockIdx.x * 8 + (role)) * 4;                 \
      tr_[0] = (unsigned)(a);                                                           \
      tr_[1] = (unsigned)(b);                                                           \
      tr_[2] = (unsigned)(c);                                                           \
      tr_[3] += 1u;                                                                     \
      __threadfence_system();                                                           \
    }                                                                                   \
  } while (0)

__device__ __forceinline__ uint64_t dk(uint32_t base, int kk) {
  return tc::sdesc(base + (kk >> 2) * ATOM + (kk & 3) * 32, 16, 1024);
}
__device__ __forceinline__ uint64_t dmn(uint32_t base, int kk) { return tc::sdesc(base + kk * 2048, ATOM, 1024); }

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 32 x 32 bf16 staging tile: row R, 16-byte chunk c at R*64 + (c ^ (R>>1 & 3))*16 (conflict-free
// for row-per-thread writes and 8-rows-per-instruction reads)
__device__ __forceinline__ uint32_t stg_off(int R, int c) { return R * 64 + ((c ^ ((R >> 1) & 3)) << 4); }

__device__ __forceinline__ int nblocks(const int* lengths, int b) {
  const int len = lengths[b];
  return len > 0 ? (len + TB - 1) / TB : 0;
}

// 32 bf16 of row r, columns [c0, c0 + 32), into a K-major SWIZZLE_128B 128-row tile.
__device__ __forceinline__ void store_sw(uint8_t* blk, int r, int c0, const uint32_t* pk) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint4 u = make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
    *reinterpret_cast<uint4*>(blk + tc::sw128_off(r, c0 + 8 * c, TB)) = u;
  }
}

template <int D>
__global__ void __launch_bounds__(NT, 1)
    hsp_fwd_kernel(const __grid_constant__ CUtensorMap tmS, const __grid_constant__ CUtensorMap tmQ, FwdP p) {
  constexpr int NA = D / 64;
  constexpr uint32_t BLK = NA * ATOM;  // one 128-row x D tile
  constexpr uint32_t IDESC_Z = tc::idesc_bf16(TB, TB, 0, 0);
  constexpr uint32_t IDESC_O = tc::idesc_bf16(TB, D, 0, 1);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sQ = sm;
  uint8_t* sS = sQ + BLK;        // 2 slots
  uint8_t* sP = sS + 2 * BLK;    // 128 x 128 bf16
  uint64_t* bar = (uint64_t*)(sP + 2 * ATOM);
  uint64_t* q_full = bar + 0;
  uint64_t* q_empty = bar + 1;
  uint64_t* s_full = bar + 2;   // [2]
  uint64_t* s_empty = bar + 4;  // [2]
  uint64_t* z_full = bar + 6;   // [2]
  uint64_t* z_empty = bar + 8;  // [2]
  uint64_t* p_full = bar + 10;
  uint64_t* p_empty = bar + 11;
  uint64_t* o_full = bar + 12;
  uint64_t* o_empty = bar + 13;
  uint32_t* tslot = (uint32_t*)(bar + 14);

  const int W = p.B * p.qtiles;
  const int i0 = (int)((long long)W * blockIdx.x / gridDim.x);
  const int i1 = (int)((long long)W * (blockIdx.x + 1) / gridDim.x);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tmS);
    tc::prefetch_tmap(&tmQ);
    tc::mbar_init(q_full, 1);
    tc::mbar_init(q_empty, 1);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&s_full[i], 1);
      tc::mbar_init(&s_empty[i], 1);
      tc::mbar_init(&z_full[i], 1);
      tc::mbar_init(&z_empty[i], 4);
    }
    tc::mbar_init(p_full, 4);
    tc::mbar_init(p_empty, 1);
    tc::mbar_init(o_full, 1);
    tc::mbar_init(o_empty, 4);
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
  const uint32_t T_O = 256;

  // the (query tile, query set) of the next item with work (-1: none) -> release Q after this item?
  auto next_qt = [&](int idx) {
    for (int k = idx + 1; k < i1; ++k)
      if (nblocks(p.lengths, k % p.B) > 0) return (k / p.B) * p.B + (k % p.B) / p.qg;
    return -1;
  };

  if (warp == 0) {
    if (lane == 0) {
      int cur_q = -1, nq = 0, sc = 0;
      for (int idx = i0; idx < i1; ++idx) {
        const int qt = idx / p.B, b = idx % p.B;
        const int nb = nblocks(p.lengths, b);
        if (nb == 0) continue;
        const int qkey = qt * p.B + b / p.qg;  // (query tile, query set)
        if (qkey != cur_q) {
          if (nq > 0) tc::mbar_wait(q_empty, (nq - 1) & 1);
          tc::mbar_arrive_expect_tx(q_full, BLK);
#pragma unroll
          for (int a = 0; a < NA; ++a) tc::tma_load_3d(sQ + a * ATOM, &tmQ, q_full, a * 64, qt * TB, b / p.qg);
          cur_q = qkey;
          ++nq;
        }
        for (int j = 0; j < nb; ++j, ++sc) {
          const int s = sc & 1;
          HSP_TRACE(0, idx, j, 1);
          tc::mbar_wait(&s_empty[s], ((sc >> 1) & 1) ^ 1);
          HSP_TRACE(0, idx, j, 2);
          tc::mbar_arrive_expect_tx(&s_full[s], BLK);
#pragma unroll
          for (int a = 0; a < NA; ++a) tc::tma_load_3d(sS + s * BLK + a * ATOM, &tmS, &s_full[s], a * 64, j * TB, b);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int cur_q = -1, nq = 0, sc = 0, zc = 0, pc = 0, t = 0;
      const uint32_t qa = tc::smem_u32(sQ), pa = tc::smem_u32(sP);
      for (int idx = i0; idx < i1; ++idx) {
        const int qt = idx / p.B, b = idx % p.B;
        const int nb = nblocks(p.lengths, b);
        if (nb == 0) continue;
        const int qkey = qt * p.B + b / p.qg;
        if (qkey != cur_q) {
          tc::mbar_wait(q_full, nq & 1);
          ++nq;
          cur_q = qkey;
        }
        auto mma_z = [&](int j) {  // S block sc0 + j, Z buffer zc0 + j
          const int s = (sc + j) & 1, z = (zc + j) & 1;
          HSP_TRACE(1, idx, j, 10);
          tc::mbar_wait(&s_full[s], ((sc + j) >> 1) & 1);
          HSP_TRACE(1, idx, j, 11);
          tc::mbar_wait(&z_empty[z], (((zc + j) >> 1) & 1) ^ 1);
          HSP_TRACE(1, idx, j, 12);
          tc::fence_after();
          const uint32_t sa = tc::smem_u32(sS + s * BLK);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) tc::mma_bf16(tmem + z * TB, dk(qa, kk), dk(sa, kk), IDESC_Z, kk > 0);
          tc::mma_commit(&z_full[z]);
        };
        mma_z(0);
        for (int j = 0; j < nb; ++j) {
          if (j + 1 < nb) mma_z(j + 1);
          HSP_TRACE(1, idx, j, 13);
          tc::mbar_wait(p_full, pc & 1);
          HSP_TRACE(1, idx, j, 14);
          if (j == 0) tc::mbar_wait(o_empty, (t & 1) ^ 1);  // the epilogue has read the previous O
          HSP_TRACE(1, idx, j, 15);
          tc::fence_after();
          const uint32_t sa = tc::smem_u32(sS + ((sc + j) & 1) * BLK);
#pragma unroll
          for (int kk = 0; kk < TB / 16; ++kk) tc::mma_bf16(tmem + T_O, dk(pa, kk), dmn(sa, kk), IDESC_O, (j | kk) > 0);
          tc::mma_commit(p_empty);
          tc::mma_commit(&s_empty[(sc + j) & 1]);
          ++pc;
        }
        tc::mma_commit(o_full);
        if (next_qt(idx) != qkey) tc::mma_commit(q_empty);
        sc += nb;
        zc += nb;
        ++t;
      }
    }
  } else {
    const int qtr = warp & 3;  // TMEM lane quarter of this warp
    const int r = qtr * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(qtr * 32) << 16);
    int zc = 0, pc = 0, t = 0;
    for (int idx = i0; idx < i1; ++idx) {
      const int qt = idx / p.B, b = idx % p.B;
      const int len = p.lengths[b];
      const int nb = nblocks(p.lengths, b);
      const int q = qt * TB + r;
      bf16* orow = nullptr;
      if (q < p.HQ)
        orow = q < p.n1 ? p.O1 + (long long)b * p.o1_bs + (long long)q * D
                        : p.O2 + (long long)b * p.o2_bs + (long long)(q - p.n1) * D;
      if (nb == 0) {  // empty sequence: pooled rows are zeros (seqsum.py:32-33, 99-100)
        if (orow) {
          const uint4 z4 = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll 4
          for (int c = 0; c < D; c += 8) *reinterpret_cast<uint4*>(orow + c) = z4;
          p.LSE[(long long)b * p.HQ + q] = INFINITY;
        }
        continue;
      }
      float mref = -INFINITY, l = 0.f;
      for (int j = 0; j < nb; ++j, ++zc, ++pc) {
        const int z = zc & 1;
        const uint32_t tz = trow + z * TB;
        const int tv = len - j * TB;  // valid columns of this block
        if (lane == 0) HSP_TRACE(2 + qtr, idx, j, 20);
        tc::mbar_wait(&z_full[z], (zc >> 1) & 1);
        if (lane == 0) HSP_TRACE(2 + qtr, idx, j, 21);
        tc::fence_after();
        // pass 1: block max (log2 units)
        float mb = -INFINITY;
#pragma unroll
        for (int c0 = 0; c0 < TB; c0 += 32) {
          float v[32];
          tc::tmem_ld32(tz + c0, v);
          if (c0 + 32 <= tv) {
#pragma unroll
            for (int i = 0; i < 32; ++i) mb = fmaxf(mb, v[i]);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (c0 + i < tv) mb = fmaxf(mb, v[i]);
          }
        }
        mb *= LOG2E;
        // P_{j-1} consumed by its MMA (O is stable) before P_j is written
        if (lane == 0) HSP_TRACE(2 + qtr, idx, j, 22);
        tc::mbar_wait(p_empty, (pc & 1) ^ 1);
        if (lane == 0) HSP_TRACE(2 + qtr, idx, j, 23);
        tc::fence_after();
        // lazy rescale of O and l to a new reference max; the TMEM accesses
        // are warp-collective, so the warp rescales if any of its rows must
        // (rows that need not use factor 1)
        const bool up = mb > mref + RESCALE;
        if (j > 0 && __any_sync(0xffffffffu, up)) {
          const float al = up ? ex2(mref - mb) : 1.f;
          l *= al;
#pragma unroll 1
          for (int c0 = 0; c0 < D; c0 += 16) {
            float v[16];
            uint32_t u[16];
            tc::tmem_ld16(trow + T_O + c0, v);
#pragma unroll
            for (int i = 0; i < 16; ++i) u[i] = __float_as_uint(v[i] * al);
            tc::tmem_st16(trow + T_O + c0, u);
          }
        }
        if (up) mref = mb;
        // pass 2: P = exp2(z log2e - mref) -> bf16 A tile
#pragma unroll
        for (int c0 = 0; c0 < TB; c0 += 32) {
          float v[32];
          uint32_t pk[16];
          tc::tmem_ld32(tz + c0, v);
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const float a = c0 + i < tv ? ex2(fmaf(v[i], LOG2E, -mref)) : 0.f;
            const float bq = c0 + i + 1 < tv ? ex2(fmaf(v[i + 1], LOG2E, -mref)) : 0.f;
            l += a + bq;
            pk[i >> 1] = tc::pack_bf16(a, bq);
          }
          store_sw(sP, r, c0, pk);
        }
        tc::fence_async_smem();
        tc::fence_before();
        __syncwarp();
        if (lane == 0) {
          tc::mbar_arrive(&z_empty[z]);
          tc::mbar_arrive(p_full);
        }
      }
      // epilogue: O / l -> bf16 pooled rows
      if (lane == 0) HSP_TRACE(2 + qtr, idx, 99, 24);
      tc::mbar_wait(o_full, t & 1);
      if (lane == 0) HSP_TRACE(2 + qtr, idx, 99, 25);
      tc::fence_after();
      const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll 1
      for (int c0 = 0; c0 < D; c0 += 32) {
        float v[32];
        tc::tmem_ld32(trow + T_O + c0, v);
        if (orow) {
          uint4* o = reinterpret_cast<uint4*>(orow + c0);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint4 u;
            u.x = tc::pack_bf16(v[8 * c + 0] * inv, v[8 * c + 1] * inv);
            u.y = tc::pack_bf16(v[8 * c + 2] * inv, v[8 * c + 3] * inv);
            u.z = tc::pack_bf16(v[8 * c + 4] * inv, v[8 * c + 5] * inv);
            u.w = tc::pack_bf16(v[8 * c + 6] * inv, v[8 * c + 7] * inv);
            o[c] = u;
          }
        }
      }
      if (orow) p.LSE[(long long)b * p.HQ + q] = (mref + __log2f(l)) * 0.6931471805599453f;
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

// ---------------------------------------------------------------------------
// Backward, persistent CTAs over (sample, 128-row block of S) items, each
// looping over the query tiles (the dS block accumulates over them in TMEM):
//   MMA   Z = Qt S_j^T, dP = dO S_j^T                 (TMEM [0,128), [128,256))
//   warps P = exp(Z - LSE) (t < len) -> smem (bf16, [q][t])
//   MMA   dS_j += P^T dO                              (TMEM [256, 256 + d))
//   warps dZ = P (dP - Dq) -> smem (same buffer) and to HBM (hi + lo split,
//         (B, HQ, T) rows: the input of the batch-reduced dQ GEMM)
//   MMA   dS_j += dZ^T Qt
//   warps (after the last query tile) dS_j -> bf16 rows of dS.
// Dq = rowsum(dO * O) comes precomputed (B, HQ).  Blocks past the sequence
// length only zero their dZ / dS rows.
struct BwdP {
  int B, T, HQ, qtiles, tblocks;
  int qg;  // samples per query set (see FwdP)
  const int* lengths;
  const float* LSE;  // (B, HQ)
  const float* Dq;   // (B, HQ)
  bf16* dS;
  long long ds_rs, ds_bs;
  int acc_ds;
  bf16* dZ;  // (B, HQ, T)
  bf16* dZlo;
  int z_tma;   // dZ (hi) rows TMA-stored from the swizzled P/dZ tile (tmZ; T % 8 == 0)
  int ds_tma;  // dS rows staged through that tile and TMA-stored (tmD; not when accumulating)
};

template <int D>
__global__ void __launch_bounds__(NT, 1)
    hsp_bwd_kernel(const __grid_constant__ CUtensorMap tmS, const __grid_constant__ CUtensorMap tmQ,
                   const __grid_constant__ CUtensorMap tmG, const __grid_constant__ CUtensorMap tmZ,
                   const __grid_constant__ CUtensorMap tmD, BwdP p) {
  constexpr int NA = D / 64;
  constexpr uint32_t BLK = NA * ATOM;
  constexpr uint32_t IDESC_Z = tc::idesc_bf16(TB, TB, 0, 0);
  constexpr uint32_t IDESC_DS = tc::idesc_bf16(TB, D, 1, 1);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sS = sm;
  uint8_t* sQ = sS + BLK;
  uint8_t* sG = sQ + BLK;   // dO tile
  uint8_t* sPZ = sG + BLK;  // 128 x 128 bf16, P then dZ
  uint64_t* bar = (uint64_t*)(sPZ + 2 * ATOM);
  uint64_t* s_full = bar + 0;
  uint64_t* s_empty = bar + 1;
  uint64_t* qg_full = bar + 2;
  uint64_t* qg_empty = bar + 3;
  uint64_t* zdp_full = bar + 4;
  uint64_t* zdp_empty = bar + 5;
  uint64_t* pz_full = bar + 6;
  uint64_t* pz_empty = bar + 7;
  uint64_t* ds_full = bar + 8;
  uint64_t* ds_empty = bar + 9;
  uint32_t* tslot = (uint32_t*)(bar + 10);

  const int W = p.B * p.tblocks;
  const int i0 = (int)((long long)W * blockIdx.x / gridDim.x);
  const int i1 = (int)((long long)W * (blockIdx.x + 1) / gridDim.x);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tmS);
    tc::prefetch_tmap(&tmQ);
    tc::prefetch_tmap(&tmG);
    tc::mbar_init(s_full, 1);
    tc::mbar_init(s_empty, 1);
    tc::mbar_init(qg_full, 1);
    tc::mbar_init(qg_empty, 1);
    tc::mbar_init(zdp_full, 1);
    tc::mbar_init(zdp_empty, 4);
    tc::mbar_init(pz_full, 4);
    tc::mbar_init(pz_empty, 1);
    tc::mbar_init(ds_full, 1);
    tc::mbar_init(ds_empty, 4);
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
  const uint32_t T_Z = 0, T_DP = 128, T_DS = 256;

  if (warp == 0) {
    if (lane == 0) {
      int n = 0, nq = 0;
      for (int idx = i0; idx < i1; ++idx) {
        const int b = idx / p.tblocks, j = idx % p.tblocks;
        if (j >= nblocks(p.lengths, b)) continue;
        tc::mbar_wait(s_empty, (n & 1) ^ 1);
        tc::mbar_arrive_expect_tx(s_full, BLK);
#pragma unroll
        for (int a = 0; a < NA; ++a) tc::tma_load_3d(sS + a * ATOM, &tmS, s_full, a * 64, j * TB, b);
        ++n;
        for (int qt = 0; qt < p.qtiles; ++qt, ++nq) {
          tc::mbar_wait(qg_empty, (nq & 1) ^ 1);
          tc::mbar_arrive_expect_tx(qg_full, 2 * BLK);
#pragma unroll
          for (int a = 0; a < NA; ++a) {
            tc::tma_load_3d(sQ + a * ATOM, &tmQ, qg_full, a * 64, qt * TB, b / p.qg);
            tc::tma_load_3d(sG + a * ATOM, &tmG, qg_full, a * 64, qt * TB, b);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int n = 0, nq = 0, pzc = 0;
      const uint32_t sa = tc::smem_u32(sS), qa = tc::smem_u32(sQ), ga = tc::smem_u32(sG), pa = tc::smem_u32(sPZ);
      for (int idx = i0; idx < i1; ++idx) {
        const int b = idx / p.tblocks, j = idx % p.tblocks;
        if (j >= nblocks(p.lengths, b)) continue;
        tc::mbar_wait(s_full, n & 1);
        for (int qt = 0; qt < p.qtiles; ++qt, ++nq) {
          tc::mbar_wait(qg_full, nq & 1);
          tc::mbar_wait(zdp_empty, (nq & 1) ^ 1);
          tc::fence_after();
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            tc::mma_bf16(tmem + T_Z, dk(qa, kk), dk(sa, kk), IDESC_Z, kk > 0);
            tc::mma_bf16(tmem + T_DP, dk(ga, kk), dk(sa, kk), IDESC_Z, kk > 0);
          }
          tc::mma_commit(zdp_full);
          // dS += P^T dO
          tc::mbar_wait(pz_full, pzc & 1);
          if (qt == 0) tc::mbar_wait(ds_empty, (n & 1) ^ 1);
          tc::fence_after();
#pragma unroll
          for (int kk = 0; kk < TB / 16; ++kk)
            tc::mma_bf16(tmem + T_DS, dmn(pa, kk), dmn(ga, kk), IDESC_DS, (qt | kk) > 0);
          tc::mma_commit(pz_empty);
          ++pzc;
          // dS += dZ^T Qt
          tc::mbar_wait(pz_full, pzc & 1);
          tc::fence_after();
#pragma unroll
          for (int kk = 0; kk < TB / 16; ++kk) tc::mma_bf16(tmem + T_DS, dmn(pa, kk), dmn(qa, kk), IDESC_DS, 1u);
          tc::mma_commit(pz_empty);
          ++pzc;
          tc::mma_commit(qg_empty);
        }
        tc::mma_commit(ds_full);
        tc::mma_commit(s_empty);
        ++n;
      }
    }
  } else {
    const int qtr = warp & 3;
    const int r = qtr * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(qtr * 32) << 16);
    int n = 0, nq = 0, pzc = 0;
    for (int idx = i0; idx < i1; ++idx) {
      const int b = idx / p.tblocks, j = idx % p.tblocks;
      const int len = p.lengths[b];
      const int tv = len - j * TB;  // valid t columns of this block
      const int t0 = j * TB;
      if (j >= nblocks(p.lengths, b)) {  // past the sequence: zero dZ rows and (unless accumulating) dS rows
        const uint4 z4 = make_uint4(0u, 0u, 0u, 0u);
        for (int qt = 0; qt < p.qtiles; ++qt) {
          const int q = qt * TB + r;
          if (q >= p.HQ) continue;
          bf16* zr = p.dZ + ((long long)b * p.HQ + q) * p.T + t0;
          bf16* lr = p.dZlo + ((long long)b * p.HQ + q) * p.T + t0;
          const int cols = min(TB, p.T - t0);
          if ((p.T & 7) == 0) {
            for (int c = 0; c < cols; c += 8) {
              *reinterpret_cast<uint4*>(zr + c) = z4;
              *reinterpret_cast<uint4*>(lr + c) = z4;
            }
          } else {
            for (int c = 0; c < cols; ++c) zr[c] = lr[c] = __float2bfloat16(0.f);
          }
        }
        if (!p.acc_ds && t0 + r < p.T) {
          bf16* dr = p.dS + (long long)b * p.ds_bs + (long long)(t0 + r) * p.ds_rs;
          for (int c = 0; c < D; c += 8) *reinterpret_cast<uint4*>(dr + c) = z4;
        }
        continue;
      }
      for (int qt = 0; qt < p.qtiles; ++qt, ++nq) {
        const int q = qt * TB + r;
        const bool qv = q < p.HQ;
        const float lse2 = qv ? p.LSE[(long long)b * p.HQ + q] * LOG2E : INFINITY;
        const float dq = qv ? p.Dq[(long long)b * p.HQ + q] : 0.f;
        tc::mbar_wait(zdp_full, nq & 1);
        tc::fence_after();
        // phase P: P = exp2(Z log2e - lse2) -> smem
        tc::mbar_wait(pz_empty, (pzc & 1) ^ 1);
        if (p.z_tma | p.ds_tma) {  // this warp's TMA stores out of the tile have read it
          if (lane == 0) tc::bulk_wait_read0();
          __syncwarp();
        }
#pragma unroll
        for (int c0 = 0; c0 < TB; c0 += 32) {
          float v[32];
          uint32_t pk[16];
          tc::tmem_ld32(trow + T_Z + c0, v);
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const float a = c0 + i < tv ? ex2(fmaf(v[i], LOG2E, -lse2)) : 0.f;
            const float bq = c0 + i + 1 < tv ? ex2(fmaf(v[i + 1], LOG2E, -lse2)) : 0.f;
            pk[i >> 1] = tc::pack_bf16(a, bq);
          }
          store_sw(sPZ, r, c0, pk);
        }
        tc::fence_async_smem();
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(pz_full);
        ++pzc;
        // phase dZ: dZ = P (dP - Dq) -> smem (after P^T dO consumed P) and HBM
        tc::mbar_wait(pz_empty, (pzc & 1) ^ 1);
        bf16* zr = qv ? p.dZ + ((long long)b * p.HQ + q) * p.T + t0 : nullptr;
        bf16* lr = qv ? p.dZlo + ((long long)b * p.HQ + q) * p.T + t0 : nullptr;
        const bool vec = (p.T & 7) == 0;
#pragma unroll 1
        for (int c0 = 0; c0 < TB; c0 += 32) {
          float v[32], g[32];
          uint32_t pk[16], lo[16];
          tc::tmem_ld32(trow + T_Z + c0, v);
          tc::tmem_ld32(trow + T_DP + c0, g);
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            float z2[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const float pr = c0 + i + u < tv ? ex2(fmaf(v[i + u], LOG2E, -lse2)) : 0.f;
              z2[u] = pr * (g[i + u] - dq);
            }
            pk[i >> 1] = tc::pack_bf16(z2[0], z2[1]);
            const __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(&pk[i >> 1]);
            const float2 hf = __bfloat1622float2(h);
            lo[i >> 1] = tc::pack_bf16(z2[0] - hf.x, z2[1] - hf.y);
          }
          store_sw(sPZ, r, c0, pk);
          if (zr && t0 + c0 < p.T) {
            if (vec && t0 + c0 + 32 <= p.T) {
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                if (!p.z_tma)
                  *reinterpret_cast<uint4*>(zr + c0 + 8 * c) = make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
                *reinterpret_cast<uint4*>(lr + c0 + 8 * c) = make_uint4(lo[4 * c], lo[4 * c + 1], lo[4 * c + 2], lo[4 * c + 3]);
              }
            } else {
              for (int i = 0; i < 32 && t0 + c0 + i < p.T; ++i) {
                const uint32_t w = pk[i >> 1], wl = lo[i >> 1];
                const unsigned short hs = (i & 1) ? (unsigned short)(w >> 16) : (unsigned short)(w & 0xffffu);
                const unsigned short ls = (i & 1) ? (unsigned short)(wl >> 16) : (unsigned short)(wl & 0xffffu);
                if (!p.z_tma) reinterpret_cast<unsigned short*>(zr)[c0 + i] = hs;
                reinterpret_cast<unsigned short*>(lr)[c0 + i] = ls;
              }
            }
          }
        }
        tc::fence_async_smem();
        tc::fence_before();
        __syncwarp();
        if (lane == 0) {
          tc::mbar_arrive(pz_full);
          tc::mbar_arrive(zdp_empty);
          // the warp's 32 dZ rows x 128 columns straight out of the swizzled
          // tile (two 64-column boxes; rows past HQ / columns past T clipped)
          if (p.z_tma && qt * TB + qtr * 32 < p.HQ) {
            tc::tma_store_3d(&tmZ, sPZ + qtr * 4096, t0, qt * TB + qtr * 32, b);
            tc::tma_store_3d(&tmZ, sPZ + ATOM + qtr * 4096, t0 + 64, qt * TB + qtr * 32, b);
            tc::bulk_commit();
          }
        }
        ++pzc;
      }
      // dS rows (thread = t row) after the last query tile
      tc::mbar_wait(ds_full, n & 1);
      tc::fence_after();
      const int t = t0 + r;
      if (p.ds_tma) {
        // dS rows through the (now free) P/dZ tile, 128 columns at a time,
        // TMA-stored as 64-column boxes of the warp's 32 rows
#pragma unroll 1
        for (int h = 0; h < D; h += TB) {
          if (lane == 0) tc::bulk_wait_read0();
          __syncwarp();
#pragma unroll 1
          for (int c0 = 0; c0 < TB; c0 += 32) {
            float v[32];
            uint32_t pk[16];
            tc::tmem_ld32(trow + T_DS + h + c0, v);
#pragma unroll
            for (int i = 0; i < 16; ++i) pk[i] = tc::pack_bf16(v[2 * i], v[2 * i + 1]);
            store_sw(sPZ, r, c0, pk);
          }
          tc::fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            tc::tma_store_3d(&tmD, sPZ + qtr * 4096, h, t0 + qtr * 32, b);
            tc::tma_store_3d(&tmD, sPZ + ATOM + qtr * 4096, h + 64, t0 + qtr * 32, b);
            tc::bulk_commit();
          }
        }
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(ds_empty);
        ++n;
        continue;
      }
      bf16* dr = t < p.T ? p.dS + (long long)b * p.ds_bs + (long long)t * p.ds_rs : nullptr;
#pragma unroll 1
      for (int c0 = 0; c0 < D; c0 += 32) {
        float v[32];
        tc::tmem_ld32(trow + T_DS + c0, v);
        if (dr) {
          uint4* o = reinterpret_cast<uint4*>(dr + c0);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            float a[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = v[8 * c + i];
            if (p.acc_ds) {
              const uint4 old = o[c];
              const uint32_t w[4] = {old.x, old.y, old.z, old.w};
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[k]));
                a[2 * k] += f.x;
                a[2 * k + 1] += f.y;
              }
            }
            o[c] = make_uint4(tc::pack_bf16(a[0], a[1]), tc::pack_bf16(a[2], a[3]), tc::pack_bf16(a[4], a[5]),
                              tc::pack_bf16(a[6], a[7]));
          }
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(ds_empty);
      ++n;
    }
    if (lane == 0) tc::bulk_wait0();
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------------------
// d = 512 (the c4 shape).  A 128 x 512 fp32 pooled accumulator alone fills
// the 512 TMEM columns and a resident 128 x 512 query tile plus one S block
// alone fill the shared memory, so the d = 512 kernels stream their operands
// in 64-column atoms:
//
// Forward, persistent CTAs over (sample, query tile, output half h) items
// (sample-major, so the query tiles and halves of one sample run on
// neighbouring CTAs and share its S blocks through L2); each item computes
// the 256-column half h of the pooled output, recomputing Z (the online
// softmax sees the same Z in both halves, so both use identical P):
//   warp 0     TMA: per S block, 8 (Qt atom, S atom) stages into a 4-slot
//              ring (Z operands), then the block's half-h S atoms (the O
//              operand) into one slot
//   warp 1     MMA: Z_j = sum_a Qt_a S_a^T into a double-buffered TMEM Z
//              (2 x 128 columns); O_h += P_j S_j[:, h] (N = 256, TMEM [256, 512))
//   warps 2-5  softmax as the d <= 256 kernel; pass epilogue O_h / l -> bf16
//              columns [256 h, 256 h + 256) of the pooled rows, LSE.
constexpr int ZST = 4;                   // Z operand ring stages
constexpr uint32_t ZSTAGE = 2 * ATOM;    // Qt atom + S atom

__global__ void __launch_bounds__(NT, 1)
    hsp_fwd512_kernel(const __grid_constant__ CUtensorMap tmS, const __grid_constant__ CUtensorMap tmQ, FwdP p) {
  constexpr int D = 512, NA = 8, DH = 256;
  constexpr uint32_t IDESC_Z = tc::idesc_bf16(TB, TB, 0, 0);
  constexpr uint32_t IDESC_O = tc::idesc_bf16(TB, DH, 0, 1);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sZ = sm;                       // ZST x (Qt atom | S atom)
  uint8_t* sO = sZ + ZST * ZSTAGE;        // 4 S atoms (half h of block j)
  uint8_t* sP = sO + 4 * ATOM;            // 128 x 128 bf16
  uint64_t* bar = (uint64_t*)(sP + 2 * ATOM);
  uint64_t* zs_full = bar;                // [ZST]
  uint64_t* zs_empty = bar + ZST;         // [ZST]
  uint64_t* os_full = bar + 2 * ZST;
  uint64_t* os_empty = os_full + 1;
  uint64_t* z_full = os_full + 2;         // [2]
  uint64_t* z_empty = os_full + 4;        // [2]
  uint64_t* p_full = os_full + 6;
  uint64_t* p_empty = os_full + 7;
  uint64_t* o_full = os_full + 8;
  uint64_t* o_empty = os_full + 9;
  uint32_t* tslot = (uint32_t*)(os_full + 10);

  const int W = p.B * p.qtiles * 2;  // (sample, query tile, output half) items
  const int i0 = (int)((long long)W * blockIdx.x / gridDim.x);
  const int i1 = (int)((long long)W * (blockIdx.x + 1) / gridDim.x);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tmS);
    tc::prefetch_tmap(&tmQ);
    for (int i = 0; i < ZST; ++i) {
      tc::mbar_init(&zs_full[i], 1);
      tc::mbar_init(&zs_empty[i], 1);
    }
    tc::mbar_init(os_full, 1);
    tc::mbar_init(os_empty, 1);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&z_full[i], 1);
      tc::mbar_init(&z_empty[i], 4);
    }
    tc::mbar_init(p_full, 4);
    tc::mbar_init(p_empty, 1);
    tc::mbar_init(o_full, 1);
    tc::mbar_init(o_empty, 4);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tslot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  KL_PDL_ENTRY();
  const uint32_t T_O = 256;

  if (warp == 0) {
    if (lane == 0) {
      int zc = 0, oc = 0;
      for (int idx = i0; idx < i1; ++idx) {
        const int b = idx / (2 * p.qtiles), qt = (idx >> 1) % p.qtiles, h = idx & 1;
        const int nb = nblocks(p.lengths, b);
        {
          for (int j = 0; j < nb; ++j) {
#pragma unroll 1
            for (int a = 0; a < NA; ++a, ++zc) {
              const int st = zc % ZST;
              tc::mbar_wait(&zs_empty[st], ((zc / ZST) & 1) ^ 1);
              tc::mbar_arrive_expect_tx(&zs_full[st], ZSTAGE);
              tc::tma_load_3d(sZ + st * ZSTAGE, &tmQ, &zs_full[st], a * 64, qt * TB, b / p.qg);
              tc::tma_load_3d(sZ + st * ZSTAGE + ATOM, &tmS, &zs_full[st], a * 64, j * TB, b);
            }
            tc::mbar_wait(os_empty, (oc & 1) ^ 1);
            tc::mbar_arrive_expect_tx(os_full, 4 * ATOM);
#pragma unroll
            for (int a = 0; a < 4; ++a) tc::tma_load_3d(sO + a * ATOM, &tmS, os_full, (4 * h + a) * 64, j * TB, b);
            ++oc;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int zc = 0, zb = 0, oc = 0, pc = 0, t = 0;
      const uint32_t z0 = tc::smem_u32(sZ), oa = tc::smem_u32(sO), pa = tc::smem_u32(sP);
      auto mma_z = [&]() {  // the next Z block into buffer zb & 1
        const int z = zb & 1;
        tc::mbar_wait(&z_empty[z], ((zb >> 1) & 1) ^ 1);
        tc::fence_after();
#pragma unroll 1
        for (int a = 0; a < NA; ++a, ++zc) {
          const int st = zc % ZST;
          tc::mbar_wait(&zs_full[st], (zc / ZST) & 1);
          tc::fence_after();
          const uint32_t qa = z0 + st * ZSTAGE, sa = qa + ATOM;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            tc::mma_bf16(tmem + z * TB, dk(qa, kk), dk(sa, kk), IDESC_Z, (a | kk) > 0 ? 1u : 0u);
          tc::mma_commit(&zs_empty[st]);
        }
        tc::mma_commit(&z_full[z]);
        ++zb;
      };
      for (int idx = i0; idx < i1; ++idx) {
        const int b = idx / (2 * p.qtiles);
        const int nb = nblocks(p.lengths, b);
        if (nb > 0) {
          mma_z();
          for (int j = 0; j < nb; ++j) {
            if (j + 1 < nb) mma_z();
            tc::mbar_wait(p_full, pc & 1);
            if (j == 0) tc::mbar_wait(o_empty, (t & 1) ^ 1);  // the epilogue has read the previous O half
            tc::mbar_wait(os_full, oc & 1);
            tc::fence_after();
#pragma unroll
            for (int kk = 0; kk < TB / 16; ++kk)
              tc::mma_bf16(tmem + T_O, dk(pa, kk), dmn(oa, kk), IDESC_O, (j | kk) > 0 ? 1u : 0u);
            tc::mma_commit(p_empty);
            tc::mma_commit(os_empty);
            ++pc;
            ++oc;
          }
          tc::mma_commit(o_full);
          ++t;
        }
      }
    }
  } else {
    const int qtr = warp & 3;
    const int r = qtr * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(qtr * 32) << 16);
    int zc = 0, pc = 0, t = 0;
    for (int idx = i0; idx < i1; ++idx) {
      const int b = idx / (2 * p.qtiles), qt = (idx >> 1) % p.qtiles, h = idx & 1;
      const int len = p.lengths[b];
      const int nb = nblocks(p.lengths, b);
      const int q = qt * TB + r;
      bf16* orow = nullptr;
      if (q < p.HQ)
        orow = q < p.n1 ? p.O1 + (long long)b * p.o1_bs + (long long)q * D
                        : p.O2 + (long long)b * p.o2_bs + (long long)(q - p.n1) * D;
      if (nb == 0) {  // empty sequence: pooled rows are zeros (seqsum.py:32-33, 99-100)
        if (orow) {
          const uint4 z4 = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll 4
          for (int c = 0; c < DH; c += 8) *reinterpret_cast<uint4*>(orow + h * DH + c) = z4;
          if (h == 1) p.LSE[(long long)b * p.HQ + q] = INFINITY;
        }
        continue;
      }
      {
        float mref = -INFINITY, l = 0.f;
        for (int j = 0; j < nb; ++j, ++zc, ++pc) {
          const int z = zc & 1;
          const uint32_t tz = trow + z * TB;
          const int tv = len - j * TB;
          tc::mbar_wait(&z_full[z], (zc >> 1) & 1);
          tc::fence_after();
          float mb = -INFINITY;
#pragma unroll
          for (int c0 = 0; c0 < TB; c0 += 32) {
            float v[32];
            tc::tmem_ld32(tz + c0, v);
            if (c0 + 32 <= tv) {
#pragma unroll
              for (int i = 0; i < 32; ++i) mb = fmaxf(mb, v[i]);
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (c0 + i < tv) mb = fmaxf(mb, v[i]);
            }
          }
          mb *= LOG2E;
          tc::mbar_wait(p_empty, (pc & 1) ^ 1);
          tc::fence_after();
          const bool up = mb > mref + RESCALE;
          if (j > 0 && __any_sync(0xffffffffu, up)) {
            const float al = up ? ex2(mref - mb) : 1.f;
            l *= al;
#pragma unroll 1
            for (int c0 = 0; c0 < DH; c0 += 16) {
              float v[16];
              uint32_t u[16];
              tc::tmem_ld16(trow + T_O + c0, v);
#pragma unroll
              for (int i = 0; i < 16; ++i) u[i] = __float_as_uint(v[i] * al);
              tc::tmem_st16(trow + T_O + c0, u);
            }
          }
          if (up) mref = mb;
#pragma unroll
          for (int c0 = 0; c0 < TB; c0 += 32) {
            float v[32];
            uint32_t pk[16];
            tc::tmem_ld32(tz + c0, v);
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              const float a = c0 + i < tv ? ex2(fmaf(v[i], LOG2E, -mref)) : 0.f;
              const float bq = c0 + i + 1 < tv ? ex2(fmaf(v[i + 1], LOG2E, -mref)) : 0.f;
              l += a + bq;
              pk[i >> 1] = tc::pack_bf16(a, bq);
            }
            store_sw(sP, r, c0, pk);
          }
          tc::fence_async_smem();
          tc::fence_before();
          __syncwarp();
          if (lane == 0) {
            tc::mbar_arrive(&z_empty[z]);
            tc::mbar_arrive(p_full);
          }
        }
        tc::mbar_wait(o_full, t & 1);
        tc::fence_after();
        const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll 1
        for (int c0 = 0; c0 < DH; c0 += 32) {
          float v[32];
          tc::tmem_ld32(trow + T_O + c0, v);
          if (orow) {
            uint4* o = reinterpret_cast<uint4*>(orow + h * DH + c0);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              uint4 u;
              u.x = tc::pack_bf16(v[8 * c + 0] * inv, v[8 * c + 1] * inv);
              u.y = tc::pack_bf16(v[8 * c + 2] * inv, v[8 * c + 3] * inv);
              u.z = tc::pack_bf16(v[8 * c + 4] * inv, v[8 * c + 5] * inv);
              u.w = tc::pack_bf16(v[8 * c + 6] * inv, v[8 * c + 7] * inv);
              o[c] = u;
            }
          }
        }
        if (orow && h == 1) p.LSE[(long long)b * p.HQ + q] = (mref + __log2f(l)) * 0.6931471805599453f;
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(o_empty);
        ++t;
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

size_t fwd512_smem() { return 1024 + ZST * ZSTAGE + 4 * ATOM + 2 * ATOM + (2 * ZST + 10) * 8 + 16; }

// ---------------------------------------------------------------------------
// d = 512 forward, balanced form.  The kernel above runs one (sample, query
// tile, half) item per CTA: 192 items on 148 SMs leave the SMs active ~60 %
// of the kernel (ncu, c4).  Here a CTA serves one lane (query set g, query
// tile qt, output half h) and an even share of that lane's 128-key blocks
// (all samples of the group, flattened), with the data path of the kernel
// above.  A sample cut by a share boundary leaves its per-part partial
// (unnormalised O half, running max, sum) in the workspace; the last part to
// arrive (per-(lane, sample) counter) merges them.  (A variant that kept the
// lane's 128 x 512 query tile resident and streamed S once in 64-key blocks
// was slower: its N = 64 score products run at 2/3 rate and the shared
// memory left for the S stream holds one block, so TMA latency paced it.)
constexpr int PARTF = 256 * 128 + 2 * 128;  // partial: O [col][row] fp32, max (log2), sum
constexpr int NTB = 224;                    // balanced kernel: + warp 6, the O operand loader

struct SplitP {
  int B, T, HQ, n1, qtiles, qg, cpl, lanes;
  const int* lengths;
  bf16* O1;
  long long o1_bs;
  bf16* O2;
  long long o2_bs;
  float* LSE;
  float* ws;       // [grid][2][PARTF]
  unsigned* cnt;   // [lanes][qg] arrival counters, zero on entry, re-zeroed by the merging CTA
};

__device__ __forceinline__ int part_start(long long NB, int p, int cpl) { return (int)(NB * p / cpl); }

// The part containing flattened block x.
__device__ __forceinline__ int part_of(long long NB, int x, int cpl) {
  int p = (int)(((long long)x * cpl) / (NB > 0 ? NB : 1));
  while (p + 1 < cpl && part_start(NB, p + 1, cpl) <= x) ++p;
  while (p > 0 && part_start(NB, p, cpl) > x) --p;
  return p;
}

// Walks the (sample, block range) segments of this CTA's part: calls
// f(b, j0, j1, whole, first, Fb) for every sample with blocks in [P0, P1)
// (first: the segment opens the part; Fb: the sample's first flattened block).
template <typename F>
__device__ __forceinline__ void walk_segments(const SplitP& p, int g, int P0, int P1, F&& f) {
  int F0 = 0;
  for (int bi = 0; bi < p.qg && F0 < P1; ++bi) {
    const int b = g * p.qg + bi;
    const int nb = nblocks(p.lengths, b);
    const int s0 = max(F0, P0), s1 = min(F0 + nb, P1);
    if (s0 < s1) f(b, s0 - F0, s1 - F0, s0 == F0 && s1 == F0 + nb, s0 == P0, F0);
    F0 += nb;
  }
}

__global__ void __launch_bounds__(NTB, 1)
    hsp_fwd512b_kernel(const __grid_constant__ CUtensorMap tmS, const __grid_constant__ CUtensorMap tmQ, SplitP p) {
  constexpr int D = 512, NA = 8, DH = 256;
  constexpr uint32_t IDESC_Z = tc::idesc_bf16(TB, TB, 0, 0);
  constexpr uint32_t IDESC_O = tc::idesc_bf16(TB, DH, 0, 1);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sZ = sm;                       // ZST x (Qt atom | S atom)
  uint8_t* sO = sZ + ZST * ZSTAGE;        // 4 S atoms (half h of block j)
  uint8_t* sP = sO + 4 * ATOM;            // 128 x 128 bf16
  uint64_t* bar = (uint64_t*)(sP + 2 * ATOM);
  uint64_t* zs_full = bar;                // [ZST]
  uint64_t* zs_empty = bar + ZST;         // [ZST]
  uint64_t* os_full = bar + 2 * ZST;
  uint64_t* os_empty = os_full + 1;
  uint64_t* z_full = os_full + 2;         // [2]
  uint64_t* z_empty = os_full + 4;        // [2]
  uint64_t* p_full = os_full + 6;
  uint64_t* p_empty = os_full + 7;
  uint64_t* o_full = os_full + 8;
  uint64_t* o_empty = os_full + 9;
  uint32_t* tslot = (uint32_t*)(os_full + 10);
  volatile int* flag = (volatile int*)(tslot + 1);

  const int lane_id = blockIdx.x / p.cpl, part = blockIdx.x % p.cpl;
  const int g = lane_id / (2 * p.qtiles), qt = (lane_id >> 1) % p.qtiles, h = lane_id & 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tmS);
    tc::prefetch_tmap(&tmQ);
    for (int i = 0; i < ZST; ++i) {
      tc::mbar_init(&zs_full[i], 1);
      tc::mbar_init(&zs_empty[i], 1);
    }
    tc::mbar_init(os_full, 1);
    tc::mbar_init(os_empty, 1);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&z_full[i], 1);
      tc::mbar_init(&z_empty[i], 4);
    }
    tc::mbar_init(p_full, 4);
    tc::mbar_init(p_empty, 1);
    tc::mbar_init(o_full, 1);
    tc::mbar_init(o_empty, 4);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tslot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tslot;
  KL_PDL_ENTRY();
  const uint32_t T_O = 256;

  long long NBl = 0;  // the lane's flattened 128-key blocks
  for (int bi = 0; bi < p.qg; ++bi) NBl += nblocks(p.lengths, g * p.qg + bi);
  const int P0 = part_start(NBl, part, p.cpl), P1 = part_start(NBl, part + 1, p.cpl);

  if (warp == 0) {
    // Z operand stages only: the O operand (half h of each S block) has its own
    // loader (warp 6), so the Z stream never waits for the single O buffer to
    // be released by the previous block's O product (264 -> 220 us at c4)
    if (lane == 0) {
      int zc = 0;
      walk_segments(p, g, P0, P1, [&](int b, int j0, int j1, bool, bool, int) {
        for (int j = j0; j < j1; ++j) {
#pragma unroll 1
          for (int a = 0; a < NA; ++a, ++zc) {
            const int st = zc % ZST;
            tc::mbar_wait(&zs_empty[st], ((zc / ZST) & 1) ^ 1);
            tc::mbar_arrive_expect_tx(&zs_full[st], ZSTAGE);
            tc::tma_load_3d(sZ + st * ZSTAGE, &tmQ, &zs_full[st], a * 64, qt * TB, g);
            tc::tma_load_3d(sZ + st * ZSTAGE + ATOM, &tmS, &zs_full[st], a * 64, j * TB, b);
          }
        }
      });
    }
  } else if (warp == 6) {
    if (lane == 0) {
      int oc = 0;
      walk_segments(p, g, P0, P1, [&](int b, int j0, int j1, bool, bool, int) {
        for (int j = j0; j < j1; ++j, ++oc) {
          tc::mbar_wait(os_empty, (oc & 1) ^ 1);
          tc::mbar_arrive_expect_tx(os_full, 4 * ATOM);
#pragma unroll
          for (int a = 0; a < 4; ++a) tc::tma_load_3d(sO + a * ATOM, &tmS, os_full, (4 * h + a) * 64, j * TB, b);
        }
      });
    }
  } else if (warp == 1) {
    if (lane == 0 && P0 < P1) {
      int zc = 0, zb = 0, oc = 0, pc = 0, t = 0;
      const uint32_t z0 = tc::smem_u32(sZ), oa = tc::smem_u32(sO), pa = tc::smem_u32(sP);
      auto mma_z = [&]() {  // the next Z block into buffer zb & 1
        const int z = zb & 1;
        tc::mbar_wait(&z_empty[z], ((zb >> 1) & 1) ^ 1);
        tc::fence_after();
#pragma unroll 1
        for (int a = 0; a < NA; ++a, ++zc) {
          const int st = zc % ZST;
          tc::mbar_wait(&zs_full[st], (zc / ZST) & 1);
          tc::fence_after();
          const uint32_t qa = z0 + st * ZSTAGE, sa = qa + ATOM;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            tc::mma_bf16(tmem + z * TB, dk(qa, kk), dk(sa, kk), IDESC_Z, (a | kk) > 0 ? 1u : 0u);
          tc::mma_commit(&zs_empty[st]);
        }
        tc::mma_commit(&z_full[z]);
        ++zb;
      };
      const int total = P1 - P0;
      mma_z();
      walk_segments(p, g, P0, P1, [&](int, int j0, int j1, bool, bool, int) {
        for (int j = j0; j < j1; ++j) {
          if (zb < total) mma_z();  // Z of the next block (possibly the next segment's) ahead of this block's O
          tc::mbar_wait(p_full, pc & 1);
          if (j == j0) tc::mbar_wait(o_empty, (t & 1) ^ 1);  // the epilogue has read the previous segment's O
          tc::mbar_wait(os_full, oc & 1);
          tc::fence_after();
#pragma unroll
          for (int kk = 0; kk < TB / 16; ++kk)
            tc::mma_bf16(tmem + T_O, dk(pa, kk), dmn(oa, kk), IDESC_O, (j > j0 || kk > 0) ? 1u : 0u);
          tc::mma_commit(p_empty);
          tc::mma_commit(os_empty);
          ++pc;
          ++oc;
        }
        tc::mma_commit(o_full);
        ++t;
      });
    }
  } else {
    const int qtr = warp & 3;
    const int r = qtr * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(qtr * 32) << 16);
    const int q = qt * TB + r;
    const bool qok = q < p.HQ;
    auto out_row = [&](int b) -> bf16* {
      return q < p.n1 ? p.O1 + (long long)b * p.o1_bs + (long long)q * D
                      : p.O2 + (long long)b * p.o2_bs + (long long)(q - p.n1) * D;
    };
    // empty samples of the group: zero rows, LSE = +inf (seqsum.py:32-33, 99-100)
    for (int bi = part; bi < p.qg; bi += p.cpl) {
      const int b = g * p.qg + bi;
      if (p.lengths[b] > 0 || !qok) continue;
      const uint4 z4 = make_uint4(0u, 0u, 0u, 0u);
      bf16* o = out_row(b) + h * DH;
#pragma unroll 4
      for (int c = 0; c < DH; c += 8) *reinterpret_cast<uint4*>(o + c) = z4;
      if (h == 1) p.LSE[(long long)b * p.HQ + q] = INFINITY;
    }
    int zc = 0, pc = 0, t = 0;
    walk_segments(p, g, P0, P1, [&](int b, int j0, int j1, bool whole, bool first_seg, int Fb) {
      const int len = p.lengths[b];
      float mref = -INFINITY, l = 0.f;
      for (int j = j0; j < j1; ++j, ++zc, ++pc) {
        const int z = zc & 1;
        const uint32_t tz = trow + z * TB;
        const int tv = len - j * TB;
        tc::mbar_wait(&z_full[z], (zc >> 1) & 1);
        tc::fence_after();
        float mb = -INFINITY;
#pragma unroll
        for (int c0 = 0; c0 < TB; c0 += 32) {
          float v[32];
          tc::tmem_ld32(tz + c0, v);
          if (c0 + 32 <= tv) {
#pragma unroll
            for (int i = 0; i < 32; ++i) mb = fmaxf(mb, v[i]);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (c0 + i < tv) mb = fmaxf(mb, v[i]);
          }
        }
        mb *= LOG2E;
        tc::mbar_wait(p_empty, (pc & 1) ^ 1);  // O of the previous block is complete (and P is free)
        tc::fence_after();
        const bool up = mb > mref + RESCALE;
        if (j > j0 && __any_sync(0xffffffffu, up)) {
          const float al = up ? ex2(mref - mb) : 1.f;
          l *= al;
#pragma unroll 1
          for (int c0 = 0; c0 < DH; c0 += 16) {
            float v[16];
            uint32_t u[16];
            tc::tmem_ld16(trow + T_O + c0, v);
#pragma unroll
            for (int i = 0; i < 16; ++i) u[i] = __float_as_uint(v[i] * al);
            tc::tmem_st16(trow + T_O + c0, u);
          }
        }
        if (up) mref = mb;
#pragma unroll
        for (int c0 = 0; c0 < TB; c0 += 32) {
          float v[32];
          uint32_t pk[16];
          tc::tmem_ld32(tz + c0, v);
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const float a = c0 + i < tv ? ex2(fmaf(v[i], LOG2E, -mref)) : 0.f;
            const float bq = c0 + i + 1 < tv ? ex2(fmaf(v[i + 1], LOG2E, -mref)) : 0.f;
            l += a + bq;
            pk[i >> 1] = tc::pack_bf16(a, bq);
          }
          store_sw(sP, r, c0, pk);
        }
        tc::fence_async_smem();
        tc::fence_before();
        __syncwarp();
        if (lane == 0) {
          tc::mbar_arrive(&z_empty[z]);
          tc::mbar_arrive(p_full);
        }
      }
      // segment epilogue
      tc::mbar_wait(o_full, t & 1);
      tc::fence_after();
      if (whole) {
        const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll 1
        for (int c0 = 0; c0 < DH; c0 += 32) {
          float v[32];
          tc::tmem_ld32(trow + T_O + c0, v);
          if (qok) {
            uint4* o = reinterpret_cast<uint4*>(out_row(b) + h * DH + c0);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              uint4 w;
              w.x = tc::pack_bf16(v[8 * c + 0] * inv, v[8 * c + 1] * inv);
              w.y = tc::pack_bf16(v[8 * c + 2] * inv, v[8 * c + 3] * inv);
              w.z = tc::pack_bf16(v[8 * c + 4] * inv, v[8 * c + 5] * inv);
              w.w = tc::pack_bf16(v[8 * c + 6] * inv, v[8 * c + 7] * inv);
              o[c] = w;
            }
          }
        }
        if (qok && h == 1) p.LSE[(long long)b * p.HQ + q] = (mref + __log2f(l)) * 0.6931471805599453f;
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(o_empty);
      } else {
        // a cut sample is its part's first segment (slot 0) or last one (slot 1):
        // unnormalised O half ([col][row]: coalesced per warp), max, sum -> workspace
        float* pw_own = p.ws + ((long long)blockIdx.x * 2 + (first_seg ? 0 : 1)) * PARTF;
#pragma unroll 1
        for (int c0 = 0; c0 < DH; c0 += 32) {
          float v[32];
          tc::tmem_ld32(trow + T_O + c0, v);
#pragma unroll
          for (int c = 0; c < 32; ++c) __stcg(pw_own + (c0 + c) * TB + r, v[c]);
        }
        __stcg(pw_own + DH * TB + r, mref);
        __stcg(pw_own + DH * TB + TB + r, l);
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(o_empty);
        __threadfence();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        // parts holding blocks of sample b (parts own no blocks when the lane has
        // fewer blocks than parts; those never arrive)
        const int plo = part_of(NBl, Fb, p.cpl), phi = part_of(NBl, Fb + nblocks(p.lengths, b) - 1, p.cpl);
        auto owns = [&](int pq) { return part_start(NBl, pq + 1, p.cpl) > part_start(NBl, pq, p.cpl); };
        int nparts = 0;
        for (int pq = plo; pq <= phi; ++pq) nparts += owns(pq);
        unsigned* cn = p.cnt + (long long)lane_id * p.qg + (b - g * p.qg);
        if (threadIdx.x == 64) *flag = (atomicAdd(cn, 1u) == (unsigned)(nparts - 1)) ? 1 : 0;
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (*flag) {  // the last part of this sample to finish merges the partials
          __threadfence();
          auto part_ws = [&](int pq) {
            const int sl = (pq == plo && part_start(NBl, plo, p.cpl) < Fb) ? 1 : 0;
            return p.ws + ((long long)(lane_id * p.cpl + pq) * 2 + sl) * PARTF;
          };
          float M = -INFINITY;
          for (int pq = plo; pq <= phi; ++pq)
            if (owns(pq)) M = fmaxf(M, __ldcg(part_ws(pq) + DH * TB + r));
          float L = 0.f;
          for (int pq = plo; pq <= phi; ++pq) {
            if (!owns(pq)) continue;
            const float* pw = part_ws(pq);
            L += __ldcg(pw + DH * TB + TB + r) * ex2(__ldcg(pw + DH * TB + r) - M);
          }
          const float inv = L > 0.f ? 1.f / L : 0.f;
#pragma unroll 1
          for (int c0 = 0; c0 < DH; c0 += 8) {
            float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            for (int pq = plo; pq <= phi; ++pq) {
              if (!owns(pq)) continue;
              const float* pw = part_ws(pq);
              const float wgt = ex2(__ldcg(pw + DH * TB + r) - M);
#pragma unroll
              for (int c = 0; c < 8; ++c) acc[c] += wgt * __ldcg(pw + (c0 + c) * TB + r);
            }
            if (qok) {
              uint4 w;
              w.x = tc::pack_bf16(acc[0] * inv, acc[1] * inv);
              w.y = tc::pack_bf16(acc[2] * inv, acc[3] * inv);
              w.z = tc::pack_bf16(acc[4] * inv, acc[5] * inv);
              w.w = tc::pack_bf16(acc[6] * inv, acc[7] * inv);
              *reinterpret_cast<uint4*>(out_row(b) + h * DH + c0) = w;
            }
          }
          if (qok && h == 1) p.LSE[(long long)b * p.HQ + q] = (M + __log2f(L)) * 0.6931471805599453f;
          if (threadIdx.x == 64) *cn = 0u;  // re-armed for the next launch
        }
      }
      ++t;
    });
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

size_t fwd512b_smem() { return fwd512_smem() + 16; }

// Backward (d = 512), persistent CTAs over (sample, 128-row S block) items,
// looping over the query tiles; the S block stays resident (8 atoms) and the
// query-tile operands stream through a 3-slot ring of (Qt atom, dO atom):
//   MMA   Z = sum_a Qt_a S_a^T, dP = sum_a dO_a S_a^T   (TMEM 2 x (128 | 128))
//   warps P = exp(Z - LSE) (t < len), dZ = P (dP - Dq): P and dZ (bf16) to the
//         rows [0, HQ) and [HQ, 2 HQ) of PZ (B, 2 HQ, T), dZ's bf16 residual
//         to dZ_lo (B, HQ, T).
// The T-length products that need the whole pooled width — dS = P^T dO +
// dZ^T Qt and dQ = sum_b dZ S — run as tcgen05 GEMMs on PZ (host).
constexpr int GST = 2;
constexpr uint32_t GSTAGE = 2 * ATOM;  // Qt atom + dO atom
constexpr uint32_t BSTG = 3 * 2048;    // per softmax warp: P | dZ | dZ_lo 32 x 32 bf16 staging tiles

__global__ void __launch_bounds__(NT, 1)
    hsp_bwd512_kernel(const __grid_constant__ CUtensorMap tmS, const __grid_constant__ CUtensorMap tmQ,
                      const __grid_constant__ CUtensorMap tmG, BwdP p) {
  constexpr int NA = 8;
  constexpr uint32_t IDESC_Z = tc::idesc_bf16(TB, TB, 0, 0);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sS = sm;                    // 8 atoms: the S block
  uint8_t* sG = sS + NA * ATOM;        // GST x (Qt atom | dO atom)
  uint8_t* sT = sG + GST * GSTAGE;     // 4 x BSTG output staging
  uint64_t* bar = (uint64_t*)(sT + 4 * BSTG);
  uint64_t* s_full = bar;
  uint64_t* s_empty = bar + 1;
  uint64_t* gs_full = bar + 2;         // [GST]
  uint64_t* gs_empty = gs_full + GST;  // [GST]
  uint64_t* zd_full = gs_empty + GST;  // [2]
  uint64_t* zd_empty = zd_full + 2;    // [2]
  uint32_t* tslot = (uint32_t*)(zd_empty + 2);

  const int W = p.B * p.tblocks;
  const int i0 = (int)((long long)W * blockIdx.x / gridDim.x);
  const int i1 = (int)((long long)W * (blockIdx.x + 1) / gridDim.x);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tmS);
    tc::prefetch_tmap(&tmQ);
    tc::prefetch_tmap(&tmG);
    tc::mbar_init(s_full, 1);
    tc::mbar_init(s_empty, 1);
    for (int i = 0; i < GST; ++i) {
      tc::mbar_init(&gs_full[i], 1);
      tc::mbar_init(&gs_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&zd_full[i], 1);
      tc::mbar_init(&zd_empty[i], 4);
    }
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
      int n = 0, gc = 0;
      for (int idx = i0; idx < i1; ++idx) {
        const int b = idx / p.tblocks, j = idx % p.tblocks;
        if (j >= nblocks(p.lengths, b)) continue;
        tc::mbar_wait(s_empty, (n & 1) ^ 1);
        tc::mbar_arrive_expect_tx(s_full, NA * ATOM);
#pragma unroll
        for (int a = 0; a < NA; ++a) tc::tma_load_3d(sS + a * ATOM, &tmS, s_full, a * 64, j * TB, b);
        ++n;
        for (int qt = 0; qt < p.qtiles; ++qt) {
#pragma unroll 1
          for (int a = 0; a < NA; ++a, ++gc) {
            const int st = gc % GST;
            tc::mbar_wait(&gs_empty[st], ((gc / GST) & 1) ^ 1);
            tc::mbar_arrive_expect_tx(&gs_full[st], GSTAGE);
            tc::tma_load_3d(sG + st * GSTAGE, &tmQ, &gs_full[st], a * 64, qt * TB, b / p.qg);
            tc::tma_load_3d(sG + st * GSTAGE + ATOM, &tmG, &gs_full[st], a * 64, qt * TB, b);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int n = 0, gc = 0, zc = 0;
      const uint32_t sa0 = tc::smem_u32(sS), g0 = tc::smem_u32(sG);
      for (int idx = i0; idx < i1; ++idx) {
        const int b = idx / p.tblocks, j = idx % p.tblocks;
        if (j >= nblocks(p.lengths, b)) continue;
        tc::mbar_wait(s_full, n & 1);
        for (int qt = 0; qt < p.qtiles; ++qt, ++zc) {
          const int z = zc & 1;
          tc::mbar_wait(&zd_empty[z], ((zc >> 1) & 1) ^ 1);
          tc::fence_after();
#pragma unroll 1
          for (int a = 0; a < NA; ++a, ++gc) {
            const int st = gc % GST;
            tc::mbar_wait(&gs_full[st], (gc / GST) & 1);
            tc::fence_after();
            const uint32_t qa = g0 + st * GSTAGE, ga = qa + ATOM, sa = sa0 + a * ATOM;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint32_t acc = (a | kk) > 0 ? 1u : 0u;
              tc::mma_bf16(tmem + z * 256, dk(qa, kk), dk(sa, kk), IDESC_Z, acc);
              tc::mma_bf16(tmem + z * 256 + TB, dk(ga, kk), dk(sa, kk), IDESC_Z, acc);
            }
            tc::mma_commit(&gs_empty[st]);
          }
          tc::mma_commit(&zd_full[z]);
        }
        tc::mma_commit(s_empty);
        ++n;
      }
    }
  } else {
    const int qtr = warp & 3;
    const int r = qtr * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(qtr * 32) << 16);
    const bool vec = (p.T & 7) == 0;
    int zc = 0;
    for (int idx = i0; idx < i1; ++idx) {
      const int b = idx / p.tblocks, j = idx % p.tblocks;
      const int len = p.lengths[b];
      const int tv = len - j * TB;
      const int t0 = j * TB;
      const bool live_blk = j < nblocks(p.lengths, b);
      for (int qt = 0; qt < p.qtiles; ++qt) {
        const int q = qt * TB + r;
        const bool qv = q < p.HQ;
        bf16* pr = qv ? p.dZ + ((long long)b * 2 * p.HQ + q) * p.T + t0 : nullptr;            // P row
        bf16* zr = qv ? p.dZ + ((long long)b * 2 * p.HQ + p.HQ + q) * p.T + t0 : nullptr;     // dZ row
        bf16* lr = qv ? p.dZlo + ((long long)b * p.HQ + q) * p.T + t0 : nullptr;
        const int cols = min(TB, p.T - t0);
        if (!live_blk) {  // past the sequence: zero rows (the GEMMs read them)
          if (qv) {
            for (int c = 0; c < cols; ++c) pr[c] = zr[c] = lr[c] = __float2bfloat16(0.f);
          }
          continue;
        }
        const int z = zc & 1;
        const float lse2 = qv ? p.LSE[(long long)b * p.HQ + q] * LOG2E : INFINITY;
        const float dq = qv ? p.Dq[(long long)b * p.HQ + q] : 0.f;
        tc::mbar_wait(&zd_full[z], (zc >> 1) & 1);
        tc::fence_after();
#pragma unroll 1
        for (int c0 = 0; c0 < TB; c0 += 32) {
          float v[32], g[32];
          uint32_t pp[16], pk[16], lo[16];
          tc::tmem_ld32(trow + z * 256 + c0, v);
          tc::tmem_ld32(trow + z * 256 + TB + c0, g);
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            float pv[2], z2[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              pv[u] = c0 + i + u < tv ? ex2(fmaf(v[i + u], LOG2E, -lse2)) : 0.f;
              z2[u] = pv[u] * (g[i + u] - dq);
            }
            pp[i >> 1] = tc::pack_bf16(pv[0], pv[1]);
            pk[i >> 1] = tc::pack_bf16(z2[0], z2[1]);
            const float2 hf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pk[i >> 1]));
            lo[i >> 1] = tc::pack_bf16(z2[0] - hf.x, z2[1] - hf.y);
          }
          if (vec && c0 + 32 <= cols) {
            // coalesced: the warp's 32 rows x 32 columns of P / dZ / dZ_lo go
            // through staging tiles so each store instruction covers 8 rows x
            // 64 B (row-per-thread 16-byte stores touch 32 lines per instruction)
            uint8_t* st0 = sT + (warp - 2) * BSTG;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const uint32_t o = stg_off(lane, c);
              *reinterpret_cast<uint4*>(st0 + o) = make_uint4(pp[4 * c], pp[4 * c + 1], pp[4 * c + 2], pp[4 * c + 3]);
              *reinterpret_cast<uint4*>(st0 + 2048 + o) = make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
              *reinterpret_cast<uint4*>(st0 + 4096 + o) = make_uint4(lo[4 * c], lo[4 * c + 1], lo[4 * c + 2], lo[4 * c + 3]);
            }
            __syncwarp();
            const int cc = lane & 3;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int R = (lane >> 2) + 8 * i, qq = qt * TB + qtr * 32 + R;
              if (qq < p.HQ) {
                const uint32_t o = stg_off(R, cc);
                const long long col = t0 + c0 + 8 * cc;
                *reinterpret_cast<uint4*>(p.dZ + ((long long)b * 2 * p.HQ + qq) * p.T + col) =
                    *reinterpret_cast<const uint4*>(st0 + o);
                *reinterpret_cast<uint4*>(p.dZ + ((long long)b * 2 * p.HQ + p.HQ + qq) * p.T + col) =
                    *reinterpret_cast<const uint4*>(st0 + 2048 + o);
                *reinterpret_cast<uint4*>(p.dZlo + ((long long)b * p.HQ + qq) * p.T + col) =
                    *reinterpret_cast<const uint4*>(st0 + 4096 + o);
              }
            }
            __syncwarp();
          } else if (qv && c0 < cols) {
            {
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                if (c0 + i >= cols) continue;
                const int sh = (i & 1) * 16;
                reinterpret_cast<unsigned short*>(pr)[c0 + i] = (unsigned short)(pp[i >> 1] >> sh);
                reinterpret_cast<unsigned short*>(zr)[c0 + i] = (unsigned short)(pk[i >> 1] >> sh);
                reinterpret_cast<unsigned short*>(lr)[c0 + i] = (unsigned short)(lo[i >> 1] >> sh);
              }
            }
          }
        }
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&zd_empty[z]);
        ++zc;
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

size_t bwd512_smem() { return 1024 + 8 * ATOM + GST * GSTAGE + 4 * BSTG + (2 + 2 * GST + 4) * 8 + 16; }

template <int D>
size_t bwd_smem() {
  return 1024 + 3 * (size_t)(D / 64) * ATOM + 2 * ATOM + 12 * 8;  // S, Qt, dO tiles, P/dZ, barriers
}

template <int D>
size_t fwd_smem() {
  return 1024 + 3 * (size_t)(D / 64) * ATOM + 2 * ATOM + 16 * 8;  // Q, 2 S slots, P, barriers
}

// 3-D bf16 tensor map (inner, rows, batch), 64 x 128 boxes, SWIZZLE_128B.
bool map3(CUtensorMap* m, const void* ptr, long long inner, long long rows, long long rs, long long nb,
          long long bs, int box_rows = TB) {
  auto fn = tc_encode_fn();
  if (!fn) return false;
  if ((rs * 2) % 16 || (bs * 2) % 16 || ((uintptr_t)ptr & 15)) return false;
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)rows, (cuuint64_t)nb};
  cuuint64_t strides[2] = {(cuuint64_t)(rs * 2), (cuuint64_t)std::max<long long>(bs * 2, rs * 2 * rows)};
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace hsp
}  // namespace kl

using namespace kl;

static long long hsp_cnt_bytes(int lanes, int qg) { return ((long long)lanes * qg * 4 + 255) / 256 * 256; }
static long long hsp_split_ws_bytes(int lanes, int cpl, int qg) {
  return hsp_cnt_bytes(lanes, qg) + (long long)lanes * cpl * 2 * hsp::PARTF * 4;
}

extern "C" long long kl_hsp_fwd_workspace_bytes(const kl_hsp_args* a) {
  if (!a || a->d != 512 || a->B < 1 || a->HQ < 1) return 0;
  const int qg = a->q_group > 0 ? a->q_group : a->B;
  if (a->B % qg) return 0;
  const int lanes = (a->B / qg) * ((a->HQ + hsp::TB - 1) / hsp::TB) * 2;
  int cpl = std::max(1, tc_num_sms() / lanes);
  if (const char* c = getenv("KL_HSP_CPL")) cpl = std::max(1, atoi(c));
  return hsp_split_ws_bytes(lanes, cpl, qg);
}

extern "C" int kl_hsp_fwd(const kl_hsp_args* a, void* stream) {
  if (!a || a->B < 0 || a->T < 0 || a->HQ < 1 || a->d < 1 || a->n1 < 0 || a->n1 > a->HQ) {
    set_error("kl_hsp_fwd: bad extents");
    return KL_EBADSHAPE;
  }
  if (a->dtype != KL_BF16 || (a->d != 128 && a->d != 256 && a->d != 512) || !kl_tcgen05_available()) {
    set_error("kl_hsp_fwd: needs bf16, d in {128, 256, 512} and an sm_100a device");
    return KL_EUNSUPPORTED;
  }
  if (a->B == 0) return KL_OK;
  bind_device((cudaStream_t)stream);
  hsp::FwdP p{};
  p.B = a->B;
  p.T = a->T;
  p.HQ = a->HQ;
  p.n1 = a->n1;
  p.qtiles = (a->HQ + hsp::TB - 1) / hsp::TB;
  const int qg = a->q_group > 0 ? a->q_group : a->B;
  if (a->B % qg) {
    set_error("kl_hsp_fwd: q_group %d does not divide B = %d", a->q_group, a->B);
    return KL_EBADSHAPE;
  }
  p.qg = qg;
  p.lengths = a->lengths;
  p.O1 = (bf16*)a->O1;
  p.o1_bs = a->o1_bs;
  p.O2 = (bf16*)a->O2;
  p.o2_bs = a->o2_bs;
  p.LSE = a->LSE;
  p.trace = nullptr;
  if (const char* tv = getenv("KL_HSP_TRACE")) p.trace = (unsigned*)strtoull(tv, nullptr, 0);  // testing
  CUtensorMap tS, tQ;
  if (!hsp::map3(&tS, a->S, a->d, a->T, a->s_rs, a->B, a->s_bs) ||
      !hsp::map3(&tQ, a->Q, a->d, a->HQ, a->d, a->B / qg, (long long)a->d * a->HQ)) {
    set_error("kl_hsp_fwd: tensor map encode failed (alignment?)");
    return KL_EUNSUPPORTED;
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (a->d == 512 && a->workspace) {  // balanced form: each lane's key blocks split evenly over the SMs
    hsp::SplitP q{};
    q.B = p.B;
    q.T = p.T;
    q.HQ = p.HQ;
    q.n1 = p.n1;
    q.qtiles = p.qtiles;
    q.qg = qg;
    q.lanes = (p.B / qg) * p.qtiles * 2;
    q.cpl = std::max(1, tc_num_sms() / q.lanes);
    if (const char* c = getenv("KL_HSP_CPL")) q.cpl = std::max(1, atoi(c));  // testing
    const long long need = hsp_split_ws_bytes(q.lanes, q.cpl, qg);
    if (a->workspace_bytes < need) {
      set_error("kl_hsp_fwd: workspace of %lld bytes, %lld needed (kl_hsp_fwd_workspace_bytes)", a->workspace_bytes,
                need);
      return KL_EBADSHAPE;
    }
    q.lengths = p.lengths;
    q.O1 = p.O1;
    q.o1_bs = p.o1_bs;
    q.O2 = p.O2;
    q.o2_bs = p.o2_bs;
    q.LSE = p.LSE;
    q.cnt = (unsigned*)a->workspace;
    q.ws = (float*)((char*)a->workspace + hsp_cnt_bytes(q.lanes, qg));
    cudaMemsetAsync(q.cnt, 0, (size_t)q.lanes * qg * sizeof(unsigned), s);
    const size_t smem = hsp::fwd512b_smem();
    cudaFuncSetAttribute(hsp::hsp_fwd512b_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_k(hsp::hsp_fwd512b_kernel, q.lanes * q.cpl, hsp::NTB, smem, s, tS, tQ, q);
    count_launch();
    count_path(KL_PATH_HSP_FWD_TC);
    count_path(KL_PATH_HSP_FWD_SPLIT);
    return launch_check("hsp_fwd");
  }
  const int items = p.B * p.qtiles * (a->d == 512 ? 2 : 1);
  int grid = std::min(items, tc_num_sms());
  if (const char* g = getenv("KL_HSP_GRID")) grid = std::max(1, std::min(grid, atoi(g)));  // testing
  if (a->d == 512) {
    const size_t smem = hsp::fwd512_smem();
    cudaFuncSetAttribute(hsp::hsp_fwd512_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_k(hsp::hsp_fwd512_kernel, grid, hsp::NT, smem, s, tS, tQ, p);
  } else if (a->d == 256) {
    const size_t smem = hsp::fwd_smem<256>();
    cudaFuncSetAttribute(hsp::hsp_fwd_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_k(hsp::hsp_fwd_kernel<256>, grid, hsp::NT, smem, s, tS, tQ, p);
  } else {
    const size_t smem = hsp::fwd_smem<128>();
    cudaFuncSetAttribute(hsp::hsp_fwd_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_k(hsp::hsp_fwd_kernel<128>, grid, hsp::NT, smem, s, tS, tQ, p);
  }
  count_launch();
  count_path(KL_PATH_HSP_FWD_TC);
  return launch_check("hsp_fwd");
}

extern "C" int kl_hsp_bwd(const kl_hsp_args* a, void* stream) {
  if (!a || a->B < 0 || a->T < 0 || a->HQ < 1 || a->d < 1) {
    set_error("kl_hsp_bwd: bad extents");
    return KL_EBADSHAPE;
  }
  if (a->dtype != KL_BF16 || (a->d != 128 && a->d != 256 && a->d != 512) || !kl_tcgen05_available()) {
    set_error("kl_hsp_bwd: needs bf16, d in {128, 256, 512} and an sm_100a device");
    return KL_EUNSUPPORTED;
  }
  if (!a->dO1 || !a->dS || !a->dZ || !a->dZ_lo || !a->LSE || !a->Dq) {
    set_error("kl_hsp_bwd: dO (all HQ rows, in dO1), Dq, LSE, dS, dZ and dZ_lo are required");
    return KL_EBADSHAPE;
  }
  if (a->B == 0 || a->T == 0) return KL_OK;
  bind_device((cudaStream_t)stream);
  hsp::BwdP p{};
  p.B = a->B;
  p.T = a->T;
  p.HQ = a->HQ;
  p.qtiles = (a->HQ + hsp::TB - 1) / hsp::TB;
  p.tblocks = (a->T + hsp::TB - 1) / hsp::TB;
  const int qg = a->q_group > 0 ? a->q_group : a->B;
  if (a->B % qg) {
    set_error("kl_hsp_bwd: q_group %d does not divide B = %d", a->q_group, a->B);
    return KL_EBADSHAPE;
  }
  p.qg = qg;
  p.lengths = a->lengths;
  p.LSE = a->LSE;
  p.Dq = a->Dq;
  p.dS = (bf16*)a->dS;
  p.ds_rs = a->ds_rs;
  p.ds_bs = a->ds_bs;
  p.acc_ds = a->accumulate_ds;
  p.dZ = (bf16*)a->dZ;
  p.dZlo = (bf16*)a->dZ_lo;
  if ((a->ds_rs % 8) || (a->ds_bs % 8) || ((uintptr_t)a->dS & 15)) {
    set_error("kl_hsp_bwd: dS rows must be 16-byte aligned");
    return KL_EUNSUPPORTED;
  }
  CUtensorMap tS, tQ, tG;
  if (!hsp::map3(&tS, a->S, a->d, a->T, a->s_rs, a->B, a->s_bs) ||
      !hsp::map3(&tQ, a->Q, a->d, a->HQ, a->d, a->B / qg, (long long)a->d * a->HQ) ||
      !hsp::map3(&tG, a->dO1, a->d, a->HQ, a->d, a->B, a->o1_bs)) {
    set_error("kl_hsp_bwd: tensor map encode failed (alignment?)");
    return KL_EUNSUPPORTED;
  }
  // d <= 256: dZ (hi) and (unless accumulating) dS leave by TMA stores
  // (KL_HSP_BWD_TMA=0 keeps the per-thread row stores: A/B testing)
  CUtensorMap tZ = tS, tD = tS;
  static int bwd_tma = -1;
  if (bwd_tma < 0) bwd_tma = (getenv("KL_HSP_BWD_TMA") && getenv("KL_HSP_BWD_TMA")[0] == '0') ? 0 : 1;
  if (a->d != 512 && bwd_tma) {
    p.z_tma = (a->T % 8) == 0 && hsp::map3(&tZ, a->dZ, a->T, a->HQ, a->T, a->B, (long long)a->HQ * a->T, 32);
    p.ds_tma = !a->accumulate_ds && (a->B == 1 || a->ds_bs >= a->ds_rs * (long long)a->T) && hsp::map3(&tD, a->dS, a->d, a->T, a->ds_rs, a->B, a->ds_bs, 32);
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int items = p.B * p.tblocks;
  int grid = std::min(items, tc_num_sms());
  if (const char* g = getenv("KL_HSP_GRID")) grid = std::max(1, std::min(grid, atoi(g)));  // testing
  if (a->d == 512) {  // P / dZ to dZ (B, 2 HQ, T), dZ's residual to dZ_lo; dS by the caller's GEMMs
    const size_t smem = hsp::bwd512_smem();
    cudaFuncSetAttribute(hsp::hsp_bwd512_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_k(hsp::hsp_bwd512_kernel, grid, hsp::NT, smem, s, tS, tQ, tG, p);
  } else if (a->d == 256) {
    const size_t smem = hsp::bwd_smem<256>();
    cudaFuncSetAttribute(hsp::hsp_bwd_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_k(hsp::hsp_bwd_kernel<256>, grid, hsp::NT, smem, s, tS, tQ, tG, tZ, tD, p);
  } else {
    const size_t smem = hsp::bwd_smem<128>();
    cudaFuncSetAttribute(hsp::hsp_bwd_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_k(hsp::hsp_bwd_kernel<128>, grid, hsp::NT, smem, s, tS, tQ, tG, tZ, tD, p);
  }
  count_launch();
  count_path(KL_PATH_HSP_BWD_TC);
  return launch_check("hsp_bwd");
}
