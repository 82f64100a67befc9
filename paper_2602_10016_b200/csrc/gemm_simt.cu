// SIMT (FFMA) strided batched GEMM with fused epilogue.
//
// This is the FP32 parity path of kl_gemm (kind::tf32 is ~1e-3 accurate and
// cannot meet the 1e-5 contract) and the fallback for
// shapes the tcgen05 kernel does not take (tiny M/N, unaligned strides).
// Output tile BM x 64 (BM = 64, or 16 for the many small-M batched products of
// the summarizers / folds, 32 for the batch-shared query folds), BK = 32, 256 threads, (BM/16) x 4 register tile.
// A reduction over the batch / K space may be split across CTAs (fp32
// atomics into an accumulate-only output).
#include <algorithm>

#include "common.cuh"
#include "gemm.h"

namespace kl {

namespace {

constexpr int BN = 64, BK = 32;

template <typename TC>
__device__ __noinline__ void epilogue_store_ool(const Epi& e, TC* C, const TC* R, TC* X, long long off, long long roff,
                                                int m, int n, int lim, float acc) {
  epilogue_store(e, C, R, X, off, roff, m, n, lim, acc);
}

// Output tile BM x 64, k-tiles of 32 double-buffered in smem: the global loads
// of k-tile i+1 are in flight (registers) while k-tile i is multiplied, so a
// small-M / long-K product is not one global-latency round trip per k-step.
template <typename TA, typename TC, int BM>
__global__ void __launch_bounds__(256) gemm_simt_kernel(GemmDesc g, Epi e, int splits) {
  KL_PDL_ENTRY();
  constexpr int TM = BM / 16;        // rows per thread
  constexpr int AL = BM * BK / 256;  // A elements loaded per thread per k-tile
  constexpr int BL = BK * BN / 256;  // B elements loaded per thread per k-tile
  __shared__ float As[2][BK][BM + 4];
  __shared__ float Bs[2][BK][BN + 4];
  const TA* __restrict__ A = (const TA*)g.A;
  const TA* __restrict__ Bp = (const TA*)g.B;
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  // decompose the output batch index over the non-reduced batch dims
  const int nb2o = g.red2 ? 1 : g.nb2;
  const int zo = blockIdx.z / splits, sp = blockIdx.z % splits;
  const int z1o = g.red1 ? 0 : zo / nb2o;
  const int z2o = g.red2 ? 0 : zo % nb2o;
  const int r1n = g.red1 ? g.nb1 : 1, r2n = g.red2 ? g.nb2 : 1;

  float acc[TM][4];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  const bool a_kfast = (g.a_cs == 1);
  const bool b_nfast = (g.b_cs == 1);
  const int kbn = (g.K + BK - 1) / BK;
  const int iters = r1n * r2n * kbn;
  const int it0 = (int)((long long)iters * sp / splits), it1 = (int)((long long)iters * (sp + 1) / splits);
  float ra[AL], rb[BL];
  auto gload = [&](int it) {
    const int r = it / kbn, k0 = (it % kbn) * BK;
    const int r1 = r / r2n, r2 = r % r2n;
    const int z1 = g.red1 ? r1 : z1o;
    const int z2 = g.red2 ? r2 : z2o;
    const TA* Ab = A + (long long)z1 * g.a_s1 + (long long)z2 * g.a_s2;
    const TA* Bb = Bp + (long long)z1 * g.b_s1 + (long long)z2 * g.b_s2;
#pragma unroll
    for (int i = 0; i < AL; ++i) {
      const int e_ = tid + 256 * i;
      const int kk = a_kfast ? e_ % BK : e_ / BM;
      const int mm = a_kfast ? e_ / BK : e_ % BM;
      const int m = m0 + mm, k = k0 + kk;
      ra[i] = (m < g.M && k < g.K) ? ldf(Ab + (long long)m * g.a_rs + (long long)k * g.a_cs) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < BL; ++i) {
      const int e_ = tid + 256 * i;
      const int nn = b_nfast ? e_ % BN : e_ / BK;
      const int kk = b_nfast ? e_ / BN : e_ % BK;
      const int n = n0 + nn, k = k0 + kk;
      rb[i] = (n < g.N && k < g.K) ? ldf(Bb + (long long)k * g.b_rs + (long long)n * g.b_cs) : 0.f;
    }
  };
  auto sstore = [&](int buf) {
#pragma unroll
    for (int i = 0; i < AL; ++i) {
      const int e_ = tid + 256 * i;
      const int kk = a_kfast ? e_ % BK : e_ / BM;
      const int mm = a_kfast ? e_ / BK : e_ % BM;
      As[buf][kk][mm] = ra[i];
    }
#pragma unroll
    for (int i = 0; i < BL; ++i) {
      const int e_ = tid + 256 * i;
      const int nn = b_nfast ? e_ % BN : e_ / BK;
      const int kk = b_nfast ? e_ / BN : e_ % BK;
      Bs[buf][kk][nn] = rb[i];
    }
  };
  if (it0 < it1) {
    gload(it0);
    sstore(0);
  }
  __syncthreads();
  for (int it = it0; it < it1; ++it) {
    const int buf = (it - it0) & 1;
    const bool more = it + 1 < it1;
    if (more) gload(it + 1);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[TM], b[4];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[buf][kk][ty * TM + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[buf][kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    if (more) sstore(buf ^ 1);
    __syncthreads();
  }

  // epilogue
  TC* C = (TC*)g.C + (long long)z1o * (g.red1 ? 0 : g.c_s1) + (long long)z2o * (g.red2 ? 0 : g.c_s2);
  const TC* R = g.R ? (const TC*)g.R + (long long)z1o * (g.red1 ? 0 : g.r_s1) + (long long)z2o * (g.red2 ? 0 : g.r_s2)
                    : nullptr;
  TC* X = g.aux ? (TC*)g.aux + (long long)z1o * (g.red1 ? 0 : g.c_s1) + (long long)z2o * (g.red2 ? 0 : g.c_s2)
                : nullptr;
  const int lim = e.row_limit ? e.row_limit[zo] : 0x7fffffff;
  const int nout = gridDim.z / splits;
  // the common epilogue (alpha, bias, beta*C) inline; activations / aux /
  // residual / row limit through one out-of-line call per element (16
  // inlined copies of the generic epilogue blew the instruction cache)
  const bool simple = e.n_act == 0 && !e.aux_mode && !R && !e.row_limit;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int m = m0 + ty * TM + i;
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= g.N) continue;
      const long long off = (long long)m * g.c_rs + (long long)n * g.c_cs;
      if (splits > 1 && g.ws) {
        g.ws[((long long)sp * nout + zo) * g.M * g.N + (long long)m * g.N + n] = acc[i][j];
      } else if (splits > 1) {
        atomicAdd((float*)C + off, e.alpha * acc[i][j]);
      } else if (simple) {
        float v = e.alpha * acc[i][j];
        if (e.bias) v += e.bias[n];
        if (e.beta != 0.f) v += e.beta * ldf(C + off);
        stf(C + off, v);
      } else {
        epilogue_store_ool(e, C, R, X, off, (long long)m * g.r_rs + (long long)n * g.r_cs, m, n, lim, acc[i][j]);
      }
    }
  }
}

template <int BM>
int launch(const GemmDesc& g, const Epi& e, cudaStream_t s) {
  const int nout = (g.red1 ? 1 : g.nb1) * (g.red2 ? 1 : g.nb2);
  const long long tiles = (long long)((g.N + BN - 1) / BN) * ((g.M + BM - 1) / BM) * nout;
  const long long iters = (long long)(g.red1 ? g.nb1 : 1) * (g.red2 ? g.nb2 : 1) * ((g.K + BK - 1) / BK);
  const bool accum_only = g.c_dtype == KL_F32 && e.beta == 1.f && !e.bias && !e.row_limit && !e.aux_mode &&
                          e.n_act == 0 && !g.R;
  int splits = 1;
  GemmDesc gd = g;
  gd.ws = nullptr;
  // few output tiles: split the reduction down to 2 k-tiles per CTA so a tiny
  // product still spreads over the SMs (its latency, not its FLOPs, is the cost)
  if (accum_only && tiles < 4 * 148 && iters >= 4) {
    splits = (int)std::max<long long>(1, std::min<long long>((4 * 148) / tiles, iters / 2));
  } else if (!accum_only && g.ws && tiles < 2 * 148 && iters >= 4) {
    // any other epilogue: fp32 partials in the workspace, then one reduce +
    // epilogue pass
    int sp = (int)std::max<long long>(1, std::min<long long>((4 * 148) / tiles, iters / 2));
    const long long per = (long long)nout * g.M * g.N * 4;
    while (sp > 1 && per * sp > g.ws_bytes) --sp;
    if (sp > 1) {
      splits = sp;
      gd.ws = g.ws;
    }
  }
  dim3 grid((g.N + BN - 1) / BN, (g.M + BM - 1) / BM, nout * splits);
  if (grid.y > 65535 || grid.z > 65535) {
    set_error("kl_gemm: grid too large (M=%d, batches=%d)", g.M, nout);
    return KL_EUNSUPPORTED;
  }
  if (g.ab_dtype == KL_F32 && g.c_dtype == KL_F32)
    launch_k(gemm_simt_kernel<float, float, BM>, grid, 256, 0, s, gd, e, splits);
  else if (g.ab_dtype == KL_F32 && g.c_dtype == KL_BF16)
    launch_k(gemm_simt_kernel<float, bf16, BM>, grid, 256, 0, s, gd, e, splits);
  else if (g.ab_dtype == KL_BF16 && g.c_dtype == KL_F32)
    launch_k(gemm_simt_kernel<bf16, float, BM>, grid, 256, 0, s, gd, e, splits);
  else
    launch_k(gemm_simt_kernel<bf16, bf16, BM>, grid, 256, 0, s, gd, e, splits);
  count_launch();
  count_path(KL_PATH_GEMM_SIMT);
  int rc = launch_check("gemm_simt");
  if (rc || !gd.ws) return rc;
  return splitk_reduce(g, e, gd.ws, splits, nout, s);
}

}  // namespace

int gemm_simt(const GemmDesc& g, const Epi& e, cudaStream_t s) {
  return g.M <= 16 ? launch<16>(g, e, s) : (g.M <= 32 ? launch<32>(g, e, s) : launch<64>(g, e, s));
}

}  // namespace kl
