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

#include <algorithm>

#include "gemm.h"
#include "tc_common.cuh"

namespace kl {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int NTHREADS = 192;

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
};

template <typename TC, bool PLAIN>
__global__ void __launch_bounds__(NTHREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TcParams p,
                   Epi e) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = sA + p.stages * p.a_stage_bytes;
  float* stage_buf = (float*)(sB + p.stages * p.b_stage_bytes);  // 4 warps x 32 x 33 fp32
  uint64_t* full = (uint64_t*)(stage_buf + 4 * 32 * 33);
  uint64_t* empty = full + p.stages;
  uint64_t* tfull = empty + p.stages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tmA);
    tc::prefetch_tmap(&tmB);
    for (int s = 0; s < p.stages; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&tfull[i], 1);
      tc::mbar_init(&tempty[i], 4);
    }
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, p.tmem_cols);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

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
      for (int unit = blockIdx.x; unit < total; unit += gridDim.x) {
        const int tile = unit / p.splits, sp = unit % p.splits;
        const int it0 = (int)((long long)iters * sp / p.splits), it1 = (int)((long long)iters * (sp + 1) / p.splits);
        const int mb = tile % p.tiles_m;
        const int nb = (tile / p.tiles_m) % p.tiles_n;
        const int zo = tile / (p.tiles_m * p.tiles_n);
        const int z1o = p.red1 ? 0 : zo / nb2o, z2o = p.red2 ? 0 : zo % nb2o;
        for (int it = it0; it < it1; ++it) {
          const int r = it / p.kblocks, kb = it % p.kblocks;
          const int z1 = p.red1 ? r / r2n : z1o;
          const int z2 = p.red2 ? r % r2n : z2o;
          const int a1 = p.a_has1 ? z1 : 0, a2 = p.a_has2 ? z2 : 0;
          const int b1 = p.b_has1 ? z1 : 0, b2 = p.b_has2 ? z2 : 0;
          {
            tc::mbar_wait(&empty[stage], phase ^ 1);
            tc::mbar_arrive_expect_tx(&full[stage], tx);
            uint8_t* da = sA + stage * p.a_stage_bytes;
            uint8_t* db = sB + stage * p.b_stage_bytes;
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
            if (++stage == p.stages) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = tc::idesc_bf16(BM, p.BN, p.a_mn, p.b_mn);
      int stage = 0;
      uint32_t phase = 0;
      int t = 0;
      for (int unit = blockIdx.x; unit < total; unit += gridDim.x, ++t) {
        const int sp = unit % p.splits;
        const int it0 = (int)((long long)iters * sp / p.splits), it1 = (int)((long long)iters * (sp + 1) / p.splits);
        const int acc = t & 1;
        const uint32_t acc_phase = (t >> 1) & 1;
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
            tc::mma_bf16(d, ad, bd, idesc, (it > it0 || k > 0) ? 1u : 0u);
          }
          tc::mma_commit(&empty[stage]);
          if (++stage == p.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc::mma_commit(&tfull[acc]);
      }
    }
  } else {
    const int lane_base = (warp & 3) * 32;
    int t = 0;
    for (int unit = blockIdx.x; unit < total; unit += gridDim.x, ++t) {
      const int tile = unit / p.splits;
      const int acc = t & 1;
      const uint32_t acc_phase = (t >> 1) & 1;
      const int mb = tile % p.tiles_m;
      const int nb = (tile / p.tiles_m) % p.tiles_n;
      const int zo = tile / (p.tiles_m * p.tiles_n);
      const int z1o = p.red1 ? 0 : zo / nb2o, z2o = p.red2 ? 0 : zo % nb2o;
      TC* C = (TC*)p.C + (long long)z1o * (p.red1 ? 0 : p.c_s1) + (long long)z2o * (p.red2 ? 0 : p.c_s2);
      const TC* R = p.R ? (const TC*)p.R + (long long)z1o * (p.red1 ? 0 : p.r_s1) + (long long)z2o * (p.red2 ? 0 : p.r_s2)
                        : nullptr;
      TC* X = p.aux ? (TC*)p.aux + (long long)z1o * (p.red1 ? 0 : p.c_s1) + (long long)z2o * (p.red2 ? 0 : p.c_s2)
                    : nullptr;
      const int lim = e.row_limit ? e.row_limit[zo] : 0x7fffffff;
      const int m0 = mb * BM + lane_base;
      float* stg = stage_buf + (warp - 2) * 32 * 33;
      tc::mbar_wait(&tfull[acc], acc_phase);
      tc::fence_after();
      const uint32_t tbase = tmem + acc * p.acc_stride + ((uint32_t)lane_base << 16);
      for (int c0 = 0; c0 < p.BN; c0 += 32) {
        // TMEM row (lane) -> smem transpose -> lanes walk columns: coalesced
        // global reads (residual / C) and writes, one row per iteration.
        float v[32];
        tc::tmem_ld16(tbase + c0, v);
        if (c0 + 16 < p.BN) tc::tmem_ld16(tbase + c0 + 16, v + 16);
#pragma unroll
        for (int j = 0; j < 32; ++j) stg[lane * 33 + j] = v[j];
        __syncwarp();
        const int n = nb * p.BN + c0 + lane;
        const bool ncol = (n < p.N) && (c0 + lane < p.BN);
        const int rows = min(32, p.M - m0);
        if (p.splits > 1) {
          // split-K partial: C += alpha * partial (fp32, beta == 1 accumulate)
          float* cp = (float*)C + (long long)m0 * p.c_rs + (long long)n * p.c_cs;
          for (int r = 0; r < rows; ++r)
            if (ncol) atomicAdd(cp + (long long)r * p.c_rs, e.alpha * stg[r * 33 + lane]);
        } else if (PLAIN) {
          TC* cp = C + (long long)m0 * p.c_rs + (long long)n * p.c_cs;
          for (int r = 0; r < rows; ++r)
            if (ncol) stf(cp + (long long)r * p.c_rs, stg[r * 33 + lane]);
        } else {
          for (int r = 0; r < rows; ++r) {
            const int m = m0 + r;
            if (ncol)
              epilogue_store(e, C, R, X, (long long)m * p.c_rs + (long long)n * p.c_cs,
                             (long long)m * p.r_rs + (long long)n * p.r_cs, m, n, lim, stg[r * 33 + lane]);
          }
        }
        __syncwarp();
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, p.tmem_cols);
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
              long long s2, int nb1, long long s1, uint32_t box_inner, uint32_t box_outer, int* has2, int* has1) {
  auto fn = encode_fn();
  if (!fn) return false;
  *has2 = (s2 != 0 && nb2 > 1);
  *has1 = (s1 != 0 && nb1 > 1);
  cuuint64_t dims[4] = {(cuuint64_t)inner, (cuuint64_t)outer, (cuuint64_t)(*has2 ? nb2 : 1),
                        (cuuint64_t)(*has1 ? nb1 : 1)};
  long long so = s_outer * 2;
  long long b2 = *has2 ? s2 * 2 : std::max<long long>(so * outer, 16);
  long long b1 = *has1 ? s1 * 2 : std::max<long long>(b2 * (long long)dims[2], 16);
  auto bad = [](long long s) { return s <= 0 || (s % 16) != 0 || s >= (1ll << 40); };
  if (bad(so) || bad(b2) || bad(b1)) return false;
  b2 = (b2 + 15) / 16 * 16;
  b1 = (b1 + 15) / 16 * 16;
  cuuint64_t strides[3] = {(cuuint64_t)so, (cuuint64_t)b2, (cuuint64_t)b1};
  cuuint32_t box[4] = {box_inner, box_outer, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
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

int gemm_tc(const GemmDesc& g, const Epi& e, cudaStream_t s) {
  if (g.ab_dtype != KL_BF16) return KL_EUNSUPPORTED;
  if (!kl_tcgen05_available()) return KL_EUNSUPPORTED;
  // small problems go to the SIMT kernel unless forced
  if (gemm_path() != 2 && (long long)g.M * g.N * g.K < (1ll << 18)) return KL_EUNSUPPORTED;
  const bool a_k = (g.a_cs == 1), a_m = (g.a_rs == 1) && !a_k;
  const bool b_k = (g.b_rs == 1), b_n = (g.b_cs == 1) && !b_k;
  if (!(a_k || a_m) || !(b_k || b_n)) return KL_EUNSUPPORTED;
  if (((uintptr_t)g.A & 15) || ((uintptr_t)g.B & 15)) return KL_EUNSUPPORTED;

  TcParams p{};
  p.M = g.M;
  p.N = g.N;
  p.K = g.K;
  int tiles_n = (g.N + 255) / 256;
  int bn = (g.N + tiles_n - 1) / tiles_n;
  bn = (bn + 15) / 16 * 16;
  if (bn < 16) bn = 16;
  p.BN = bn;
  p.tiles_n = (g.N + bn - 1) / bn;
  p.tiles_m = (g.M + BM - 1) / BM;
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
  p.stages = std::min<int>(8, (190 * 1024) / stage);
  if (p.stages < 2) return KL_EUNSUPPORTED;
  p.acc_stride = bn > 128 ? 256 : (bn > 64 ? 128 : (bn > 32 ? 64 : 32));
  p.tmem_cols = 2 * p.acc_stride;
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
    if (!make_map(&tb, g.B, g.K, g.N, g.b_cs, g.nb2, g.b_s2, g.nb1, g.b_s1, BK, bn, &p.b_has2, &p.b_has1))
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

  const size_t smem = 1024 + (size_t)p.stages * stage + 4 * 32 * 33 * 4 + (2 * p.stages + 4) * 8 + 16;
  const int tiles = p.tiles_m * p.tiles_n * p.n_out;
  const int iters = ((g.red1 ? g.nb1 : 1) * (g.red2 ? g.nb2 : 1)) * p.kblocks;
  p.splits = 1;
  // Weight-gradient shape: few output tiles, a long reduction.  Spread the
  // reduction over the SMs; partial tiles accumulate with fp32 atomics, so
  // only an fp32 accumulate-into-C epilogue (beta == 1, nothing else) qualifies.
  const bool accum_only = g.c_dtype == KL_F32 && e.beta == 1.f && !e.bias && !e.row_limit && !e.aux_mode &&
                          e.n_act == 0 && !g.R;
  if (accum_only && tiles < num_sms() && iters >= 8) {
    p.splits = std::max(1, std::min(num_sms() / tiles, iters / 4));
  }
  const int total = tiles * p.splits;
  const int grid = std::min(total, num_sms());
  const bool plain = e.alpha == 1.f && e.beta == 0.f && !e.bias && !e.row_limit && !e.aux_mode && e.n_act == 0 &&
                     !g.R;
  auto launch = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, NTHREADS, smem, s>>>(ta, tb, p, e);
  };
  if (g.c_dtype == KL_BF16) {
    if (plain) launch(gemm_tc_kernel<bf16, true>);
    else launch(gemm_tc_kernel<bf16, false>);
  } else {
    if (plain) launch(gemm_tc_kernel<float, true>);
    else launch(gemm_tc_kernel<float, false>);
  }
  count_launch();
  return launch_check("gemm_tc");
}

}  // namespace kl

namespace kl {
PFN_cuTensorMapEncodeTiled_v12000 tc_encode_fn() { return encode_fn(); }
int tc_num_sms() { return num_sms(); }
}  // namespace kl
