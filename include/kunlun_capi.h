/*
 * kunlun_capi.h — C ABI of libkunlun_sm100a.so, the B200 (sm_100a) kernels
 * behind the Kunlun layer hot path (arXiv 2602.10016).
 *
 * The reference (pkg/src/kunlun, numpy float64) has no native code; its
 * plugin point for fused kernels is `record(out, parents, vjp)`
 * (/root/reference/pkg/src/kunlun/tensor.py:185-195), with `gdpa_core`
 * (gdpa.py:141-187) as the in-tree fused-op example.  Each entry point below
 * is one device operation a `record`-style VJP (or a torch.autograd.Function
 * in paper_2602_10016_b200) binds; the comment on each names the reference
 * operation(s) it replaces.
 *
 * Conventions
 *  - Plain pointers and sizes only.  All pointers are device pointers unless
 *    stated; the caller owns every buffer (the library never allocates).
 *  - Every entry takes a cudaStream_t (as void*) and is stream-ordered and
 *    reentrant.  Return 0 on success, KL_E* on failure with a message from
 *    kl_last_error() (thread-local).
 *  - Element strides are in elements (not bytes).
 *  - dtype: KL_F32 (SIMT FFMA path, the 1e-5 parity path) or KL_BF16
 *    (tcgen05/TMEM/TMA path on sm_100a, fp32 accumulation).
 */
#ifndef KUNLUN_CAPI_H
#define KUNLUN_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KL_OK 0
#define KL_EBADSHAPE 1    /* shape / stride contract violated (ShapeError)     */
#define KL_EUNSUPPORTED 2 /* valid request the library cannot run (ValueError) */
#define KL_ELAUNCH 3      /* CUDA launch / runtime failure (RuntimeError)      */

#define KL_F32 0
#define KL_BF16 1

/* Activation tags, in the reference table order (tensor.py:431-440). */
#define KL_ACT_IDENTITY 0
#define KL_ACT_RELU 1
#define KL_ACT_SILU 2
#define KL_ACT_TANH 3
#define KL_ACT_SIGMOID 4
#define KL_ACT_EXP 5
#define KL_ACT_SQRT 6
#define KL_ACT_LOG 7

#define KL_MAX_ACT_GROUPS 32

int kl_version(void);
const char* kl_last_error(void);
/* Number of kernels this library launched since load (for bench accounting). */
unsigned long long kl_launch_count(void);
/* 1 when the device is sm_100 and the tcgen05 path is enabled. */
int kl_tcgen05_available(void);
/* Force the SIMT GEMM even for bf16 (debug / A-B testing).  0 = auto. */
void kl_set_gemm_path(int path);
/* Programmatic dependent launch of every library kernel (default on; env
 * KL_PDL=0 or kl_set_pdl(0) turns it off).  The tcgen05 kernels run their
 * prologue (barrier init, TMEM alloc, tensor-map prefetch) before waiting on
 * the previous kernel. */
void kl_set_pdl(int on);
/* Path the last kl_gemm call on this thread took: 1 tcgen05, 0 SIMT. */
int kl_last_gemm_path(void);

/* Kernel-path counters: how many launches each kernel family made since load
 * (or the last kl_reset_path_hits).  Parity tests read them to assert which
 * kernels a composed step actually ran (e.g. that the fused tcgen05 GDPA /
 * HSP / SWA kernels, not a composition or SIMT fallback, were exercised). */
#define KL_PATH_GEMM_TC 0       /* tcgen05 GEMM (kl_gemm, bf16)                */
#define KL_PATH_GEMM_SIMT 1     /* FFMA GEMM (fp32 / unsupported bf16 shapes)  */
#define KL_PATH_GDPA_FWD_TC 2   /* fused GDPA forward (kl_gdpa_fwd)            */
#define KL_PATH_GDPA_BWD_TC 3   /* fused GDPA backward (kl_gdpa_bwd)           */
#define KL_PATH_HSP_FWD_TC 4    /* fused HSP / PMA pooling forward             */
#define KL_PATH_HSP_BWD_TC 5    /* fused HSP / PMA pooling backward            */
#define KL_PATH_SWA_FWD_TC 6    /* banded flash attention forward, tcgen05     */
#define KL_PATH_SWA_BWD_TC 7    /* banded flash attention backward, tcgen05    */
#define KL_PATH_SWA_FWD_SIMT 8  /* banded attention forward, SIMT              */
#define KL_PATH_SWA_BWD_SIMT 9  /* banded attention backward, SIMT             */
#define KL_PATH_COLSOFTMAX 10   /* column softmax of the pooling composition   */
#define KL_PATH_GDPA_FWD_TC512 11 /* fused GDPA forward, d = 512 variant       */
#define KL_PATH_GDPA_BWD_TC512 12 /* fused GDPA backward, d = 512 variant      */
#define KL_PATH_HSP_FWD_SPLIT 13 /* HSP forward d = 512, balanced form       */
#define KL_PATH_GEMM_WIDE 14    /* tcgen05 GEMM, wide CTA pairs (256 x 512)  */
#define KL_PATH_COUNT 16
unsigned long long kl_path_hits(int path);
void kl_reset_path_hits(void);

/*
 * Strided, batched, optionally batch-reducing GEMM with a fused epilogue.
 * Replaces every matmul/matvec of the hot path and their VJPs
 * (tensor.py:283-297: dA = g B^T, dB = A^T g) — projections, weight
 * generation (gdpa.py:103-112), the folded GDPA contractions (gdpa.py:120-187),
 * HSP/PMA pooling (seqsum.py:26-122), Wukong/aggregate maps
 * (interaction.py:106-157) and rowwise MLPs (mlp.py:47-59).
 *
 *   for each (z1, z2):  acc = sum_k A[m,k] B[k,n]
 *   out[m,n] = act_c( alpha*acc [* act'_c(aux[m,n]) if aux_mode==2] + bias[n] )
 *              + beta*C[m,n] + R[m,n]                ([aux]=pre-act if aux_mode==1)
 *   rows m >= row_limit[z1*nb2 + z2] (if row_limit; no batch reduction) are
 *   written as 0 (pre-act 0 too).
 * A batch index with red{1,2}=1 is summed into one output (its C stride is
 * ignored).  act_c = act_codes[(n / act_group) % n_act] (n_act=0 -> identity).
 */
typedef struct kl_gemm_args {
  int M, N, K;
  int nb1, nb2;
  int red1, red2;
  int ab_dtype, c_dtype;
  const void* A;
  long long a_rs, a_cs, a_s1, a_s2;
  const void* B;
  long long b_rs, b_cs, b_s1, b_s2;
  void* C;
  long long c_rs, c_cs, c_s1, c_s2;
  const void* R; /* residual, c_dtype, or NULL */
  long long r_rs, r_cs, r_s1, r_s2;
  void* aux; /* c_dtype, C's strides */
  int aux_mode; /* 0 none, 1 write pre-activation, 2 multiply by act'(aux) */
  float alpha, beta;
  const float* bias; /* [N] fp32 or NULL */
  const int* row_limit; /* [nb1*nb2] or NULL */
  int n_act, act_group;
  int act_codes[KL_MAX_ACT_GROUPS];
  /* optional fp32 scratch for split-K of few-tile GEMMs with any epilogue
   * (partials then a reduce + epilogue pass); NULL disables it */
  void* workspace;
  long long workspace_bytes;
} kl_gemm_args;

int kl_gemm(const kl_gemm_args* args, void* stream);

/*
 * Fused GDPA core (one tcgen05/TMEM kernel per direction, TMA-fed).
 * Replaces `gdpa_core` forward and its VJP (gdpa.py:141-187) on the folded
 * per-sample weights Kt = K W_q, Vt = V W_out^T (gdpa.py:120-138):
 *   Z = S Kt^T * inv_tau, A = Act(Z) (column j uses act_codes[(j/n_kv) % n_act]),
 *   Y = S + A Vt; rows >= lengths[b] pass through (Y = S, dS = dY).
 *   bwd: dS = dY + dZ Kt, dKt = dZ^T S, dVt = A^T dY,
 *        dZ = (dY Vt^T) * Act'(Z) * inv_tau.
 * S, Y, dY, dS: (B, T, d) bf16 with row stride s_rs, batch stride s_bs.
 * Kt, Vt, dKt, dVt: (B, HK, d) bf16 contiguous.  Z and A never reach HBM.
 * Takes bf16, HK = 64, d in {128, 256}; anything else returns KL_EUNSUPPORTED
 * (the caller composes kl_gemm calls — the fp32 parity path).
 */
typedef struct kl_gdpa_args {
  int B, T, d, HK, n_kv;
  int dtype;
  float inv_tau;
  int n_act;
  int act_codes[KL_MAX_ACT_GROUPS];
  const int* lengths;
  const void* S;
  long long s_rs, s_bs;
  const void* Kt;
  const void* Vt;
  void* Y; /* forward output */
  /* backward */
  const void* dY;
  void* dS;
  void* dKt;
  void* dVt;
  /* debug: if non-NULL, 32 x 16 clock64 stamps of CTA 0's pipeline stages */
  unsigned long long* trace;
  /* d = 512 (HK = 128) backward: the kernel writes dZ and A = Act(Z) as
   * (B, T, HK) bf16 here (rows >= length zero) and the caller forms
   * dKt = dZ^T S, dVt = A^T dY with GEMMs; dKt / dVt are not written. */
  void* dZ_out;
  void* A_out;
} kl_gdpa_args;

/* bf16; (HK = 64, d in {128, 256}) or (HK = 128, d = 512); per-16-column
 * activation codes from {identity, relu, silu, tanh}. */
int kl_gdpa_fwd(const kl_gdpa_args* args, void* stream);
int kl_gdpa_bwd(const kl_gdpa_args* args, void* stream);

/*
 * Fused HSP / PMA pooling (seqsum.py:26-34, 96-102 = multi_head_attention of
 * batch-shared queries over S, attention.py:69-93), with the key projection
 * folded into the queries (Q = q W_q^T W_k / sqrt(d_h), rows ordered
 * (query, head)):  pooled[b] = softmax_t<len(Q S[b]^T) S[b].
 *   S:  (B, T, d) bf16, rows s_rs apart, samples s_bs apart.
 *   Q:  (HQ, d) bf16 contiguous (or one set per sample group, q_group).
 *   O1: query rows [0, n1) -> (B, n1, d) (batch stride o1_bs); O2: rows
 *       [n1, HQ) -> (B, HQ - n1, d).  Empty samples give zero rows.
 *   LSE: (B, HQ) fp32 natural-log normaliser (+inf for empty samples).
 * Backward: dO1 = the gradient of ALL HQ pooled rows, (B, HQ, d) with batch
 *   stride o1_bs (dO2 unused), Dq (B, HQ) fp32 = rowsum(dO * pooled), LSE ->
 *   dS (B, T, d) bf16 (rows ds_rs apart; accumulated into when accumulate_ds),
 *   dZ / dZ_lo (B, HQ, T) bf16: the score gradient split hi + lo (the input
 *   of the batch-reduced query gradient dQ = sum_b dZ S).
 * bf16, d in {128, 256}; anything else returns KL_EUNSUPPORTED.
 */
typedef struct kl_hsp_args {
  int B, T, HQ, d, n1;
  int dtype;
  const int* lengths;
  const void* S;
  long long s_rs, s_bs;
  const void* Q;
  void* O1;
  long long o1_bs;
  void* O2;
  long long o2_bs;
  float* LSE;
  /* backward */
  const void* dO1;
  const void* dO2;
  void* dS;
  long long ds_rs, ds_bs;
  int accumulate_ds;
  void* dZ;
  void* dZ_lo;
  const float* Dq;
  /* grouped event types: Q holds B / q_group query sets, (B / q_group, HQ, d)
   * contiguous, and sample b pools with set b / q_group; 0 = one set shared
   * by every sample (the reference's batch-shared queries). */
  int q_group;
  /* d = 512 forward: scratch for the split form (per-part partial pooled rows
   * + arrival counters), at least kl_hsp_fwd_workspace_bytes(args) bytes,
   * 16-byte aligned, not shared with a concurrent launch; NULL selects the
   * unsplit kernel. */
  void* workspace;
  long long workspace_bytes;
} kl_hsp_args;

int kl_hsp_fwd(const kl_hsp_args* args, void* stream);
long long kl_hsp_fwd_workspace_bytes(const kl_hsp_args* args);
int kl_hsp_bwd(const kl_hsp_args* args, void* stream);

/*
 * Sliding-window multi-head self-attention core (flash style; tiles outside
 * the band are never visited).  Replaces the score/softmax/value part of
 * `mha_window` / `mha_full` (attention.py:69-93 with band_mask & length mask,
 * attention.py:96-129; masked_softmax_lastdim tensor.py:485-505).
 *   QKV: (B, T, 3*H*d_h) packed [Q | K | V], row stride ld_qkv, batch stride bs_qkv.
 *   O:   (B, T, H*d_h), rows >= length and fully-masked rows are 0.
 *   LSE: (B, H, T) fp32 log-sum-exp of the scaled masked scores (for bwd).
 * Mask: |i-j| <= w (and j <= i when causal), i, j < lengths[b].
 */
typedef struct kl_swa_args {
  int B, T, H, d_h;
  int w, causal;
  int dtype;
  float scale; /* 1/sqrt(d_h), attention.py:83 */
  const int* lengths;
  const void* QKV;
  long long ld_qkv, bs_qkv;
  void* O;
  long long ld_o, bs_o;
  float* LSE;
  /* backward */
  const void* dO;
  void* dQKV; /* same layout as QKV; fully written */
  float* Dbuf; /* (B, H, T) fp32 scratch: rowsum(dO * O) */
} kl_swa_args;

int kl_swa_fwd(const kl_swa_args* args, void* stream);
int kl_swa_bwd(const kl_swa_args* args, void* stream);
/* Bit-exact test hook: per-query key count the SWA kernels visit, written to
 * support[b*T + i] (int32); must equal band_support_sizes (attention.py:132-139)
 * restricted to valid rows (0 for rows >= length). */
int kl_swa_debug_support(const kl_swa_args* args, int* support, void* stream);

/*
 * Column softmax over a (T x C) score block per batch, masked to rows
 * t < lengths[b]; writes P (same layout, dtype) and per-column LSE (fp32).
 * Fully-masked columns (length 0) give P = 0.  Used by HSP/PMA pooling
 * (seqsum.py:26-34, 96-102 via attention.py:69-93 with queries as columns).
 */
typedef struct kl_colsoftmax_args {
  int Bn, T, C;
  int dtype_in, dtype_out;
  const void* X;
  long long x_rs, x_bs;
  void* P;
  long long p_rs, p_bs;
  float* LSE; /* (Bn, C) or NULL */
  const int* lengths;
  /* backward: dX = P * (dP - Dcol), Dcol[c] = sum_t P[t,c] dP[t,c] */
  const void* dP;
  long long dp_rs, dp_bs;
  void* dX;
  long long dx_rs, dx_bs;
  void* dX_lo; /* optional: dX - round(dX) in dX's dtype (bf16 hi/lo split) */
  int dtype_dp; /* backward: dP's dtype (KL_F32 when zero-initialised) */
  /* backward, optional: precomputed Dcol (Bn, C) fp32 (= rowsum(dO * O) of the
   * pooled output); NULL -> reduced over t here (two passes).
   * backward, optional: X (fp32 scores, x_rs / x_bs) and LSE both set ->
   * P = exp(X - LSE) is recomputed in fp32 instead of read from P. */
  const float* Dcol;
} kl_colsoftmax_args;

int kl_colsoftmax_fwd(const kl_colsoftmax_args* args, void* stream);
int kl_colsoftmax_bwd(const kl_colsoftmax_args* args, void* stream);

/* masked_softmax_lastdim (tensor.py:485-505) over rows of n fp32 scores with a
 * boolean (uint8) mask of mask_rows x n rows, row r using mask row
 * r % mask_rows (one (n_q, n_k) mask for every batch / head); fully-masked
 * rows give 0.  Backward dx = y * (g - sum(g * y)).  The arbitrary-mask path
 * of multi_head_attention (attention.py:69-93). */
int kl_masked_softmax_fwd(long long rows, int n, const float* x, const unsigned char* mask, long long mask_rows,
                          float* y, void* stream);
int kl_masked_softmax_bwd(long long rows, int n, const float* y, const float* g, float* dx, void* stream);

/* RMSNorm over the last axis, eps inside the sqrt (tensor.py:552-556).
 * x (rows, d) fp32; y = x / sqrt(mean(x^2)+eps) * gain.  bwd writes dx and
 * dgain (fp32, dgain fully written). */
int kl_rmsnorm_fwd(int rows, int d, float eps, const float* x, const float* gain, float* y, void* stream);
int kl_rmsnorm_bwd(int rows, int d, float eps, const float* x, const float* gain, const float* dy,
                   float* dx, float* dgain, void* stream);
/* Batched forms: nb independent (rows, d) problems, element batch strides;
 * the backward writes (accumulate = 0) or adds into (accumulate = 1) dx and
 * dgain. */
int kl_rmsnorm_fwd_b(int nb, int rows, int d, float eps, const float* x, long long x_bs, const float* gain,
                     long long g_bs, float* y, long long y_bs, void* stream);
int kl_rmsnorm_bwd_b(int nb, int rows, int d, float eps, const float* x, long long x_bs, const float* gain,
                     long long g_bs, const float* dy, long long dy_bs, float* dx, long long dx_bs, float* dgain,
                     long long dg_bs, int accumulate, void* stream);

/* recent_rows (seqsum.py:186-196): out[b, r] = S[b, len-n+r] for len-n+r >= 0
 * else 0; dtype_s for S/out.  bwd accumulates into dS (dS[b, t] += dOut[b, r]). */
int kl_recent_rows_fwd(int B, int T, int d, int n_recent, int dtype, const void* S, long long s_bs,
                       const int* lengths, void* out, long long o_bs, void* stream);
int kl_recent_rows_bwd(int B, int T, int d, int n_recent, int dtype, const void* dout, long long o_bs,
                       const int* lengths, void* dS, long long s_bs, void* stream);

/* Wukong pairwise-dot block (interaction.py:63-76, 106-121):
 * tri[b, p] = x[b, r_p] . x[b, c_p] over np.triu_indices(n) order; columns
 * n(n+1)/2 .. t_bs-1 of each row (the padding of a contiguous (B, t_bs) tri)
 * are written as zeros.
 * bwd: dx[b] += (dG + dG^T) x[b] with dG scattered from dtri. */
int kl_gram_triu_fwd(int B, int n, int d, int dtype, const void* x, long long x_rs, long long x_bs,
                     void* tri, long long t_bs, void* stream);
int kl_gram_triu_bwd(int B, int n, int d, int dtype, const void* x, long long x_rs, long long x_bs,
                     const void* dtri, long long t_bs, void* dx, long long dx_rs, long long dx_bs,
                     void* stream);

/* Gated residual of a Wukong expert: out = x + gd*deep + gt*dot, gates are
 * device fp32 scalars (shape (1,), interaction.py:97-98).  bwd: ddeep = g*gd,
 * ddot = g*gt, dx += g, dgate_{deep,dot} += sum(g*deep), sum(g*dot) (fp32,
 * accumulated into the gate gradients; fp64 sums; scratch >= 2*512 doubles).  All tensors
 * (rows, d) contiguous with row strides given. */
int kl_gated_sum_fwd(int rows, int d, int dtype, const void* x, long long x_rs, const void* deep,
                     const void* dot, const float* gd, const float* gt, void* out, long long o_rs,
                     void* stream);
int kl_gated_sum_bwd(int rows, int d, int dtype, const void* g, long long g_rs, const void* deep,
                     const void* dot, const float* gd, const float* gt, void* ddeep, void* ddot,
                     float* dgd, float* dgt, float* scratch, void* stream);

/* out[r] = sum_k a[r, k] * b[r, k], fp32 accumulation (rows of length d,
 * row strides a_rs / b_rs): the softmax-VJP row term rowsum(dO * O). */
int kl_rowdot(int rows, int d, int dtype, const void* a, long long a_rs, const void* b, long long b_rs, float* out,
              void* stream);

/* out[b * out_bs + i] = sum_k a[b, i, k] * b[b, i, k], i < n: rowdot over a
 * (B, n, d) pair of strided row sets (one pooled part of the HSP backward). */
int kl_rowdot3(int B, int n, int d, int dtype, const void* a, long long a_bs, long long a_rs, const void* b,
               long long b_bs, long long b_rs, float* out, long long out_bs, void* stream);

/*
 * Row regrouping along a token axis in ONE launch: the concatenations /
 * splits of row blocks the layer composes (SummaryBundle rows [CLS | seeds |
 * recent], seqsum.py:148-162; the expert slices of [X | summaries] and their
 * re-concatenation, interaction.py:144-157).  Segment s copies `rows` rows of
 * every sample b: dst + b*dst_bs + i*dst_rs <- src + b*src_bs + i*src_rs
 * (elements; rows of d contiguous elements; src NULL writes zeros).  The
 * destination rows of the segments are enumerated in order.
 */
#define KL_MAX_SEGS 16
typedef struct kl_regroup_seg {
  const void* src;
  long long src_bs, src_rs;
  void* dst;
  long long dst_bs, dst_rs;
  int rows;
} kl_regroup_seg;
typedef struct kl_regroup_args {
  int B, d, dtype, n_seg;
  kl_regroup_seg seg[KL_MAX_SEGS];
} kl_regroup_args;
int kl_regroup(const kl_regroup_args* args, void* stream);

/* Zero `bytes` bytes of device memory (a memset node in a captured graph). */
int kl_memset(void* p, long long bytes, void* stream);

/* Mean BCE with logits (tensor.py:535-549): loss[0] = mean(...), dz = (sig(z)-y)/n.
 * z, y, dz fp32 (n,). */
int kl_bce_fwd_bwd(int n, const float* z, const float* y, float* loss, float* dz, void* stream);

/* ROTE, the rotary temporal encoding of behaviour sequences (preproc.py:155-199
 * rote_sequence / rote / gaps_from_timestamps; tensor.py:508-532 rotate_pairs).
 * Row t < lengths[b] of sample b: each (even, odd) column pair i rotates by
 *   angle = t * pos_freqs[i] + log1p(max(gap_t, 0) / tau_scale) * temp_freqs[i]
 * with gap_t = ts[t] - ts[t-1] (ts[0]: 0; gap_mode 0, "previous") or
 * ts[len-1] - ts[t] (gap_mode 1, "latest"); timestamps NULL -> tau = 0.
 * Angles in fp64, reduced to [-1/2, 1/2] turns, sin/cos in fp32 (MUFU on the
 * vector path: d % 8 == 0 with 16 B-aligned rows; |err| <= 2^-21).  inverse = 1 rotates by
 * the negative angles (the VJP).  Rows >= lengths[b] are copied unchanged.
 * x, y: (B, T, d) with row / batch strides in elements, d even; y != x. */
typedef struct kl_rote_args {
  int B, T, d, dtype;        /* dtype KL_F32 / KL_BF16 (x and y) */
  const void* x;
  long long x_rs, x_bs;
  void* y;
  long long y_rs, y_bs;
  const int* lengths;        /* (B,) or NULL (= T) */
  const double* timestamps;  /* (B, T) rows of ts_bs doubles, or NULL */
  long long ts_bs;
  const double* pos_freqs;   /* (d/2,) */
  const double* temp_freqs;  /* (d/2,) */
  double tau_scale;
  int gap_mode;              /* 0 previous, 1 latest */
  int inverse;
} kl_rote_args;
int kl_rote(const kl_rote_args* a, void* stream);

/* Non-sequence embedding, fused (preproc.py:103-136: embed_dense,
 * embed_sparse, assemble_nonseq): out (B, n_sparse + 1, d) in dtype with
 *   out[b, 0]     = proj (d, m) @ x_dense[b]          (x_dense (B, m) fp32)
 *   out[b, 1 + i] = table[offsets[i] + ids[b, i]]     (table (vocab_tot, d):
 *                   the per-feature tables stacked; ids (B, n_sparse) int64)
 * The caller validates 0 <= ids[b, i] < vocab_i (IndexError, preproc.py:121);
 * the kernel clamps to the stacked table for memory safety.
 * Backward: dtable[offsets[i] + ids[b, i]] += dout[b, 1 + i] (fp32 atomics)
 * and dproj += dout[:, 0]^T x_dense (fp32, accumulated). */
int kl_embed_nonseq_fwd(int B, int n_sparse, int d, int m, int dtype, const float* x_dense, const void* proj,
                        const void* table, const long long* offsets, const long long* ids, long long vocab_tot,
                        void* out, void* stream);
int kl_embed_nonseq_bwd(int B, int n_sparse, int d, int m, int dtype, const float* x_dense, const void* dout,
                        const long long* offsets, const long long* ids, long long vocab_tot, float* dtable,
                        float* dproj, void* stream);

/* Normalized entropy (Eq. A1-A2; SPEC.md:553-561 normalized_entropy):
 * kind 0: p holds probabilities (clipped to [1e-12, 1-1e-12]); kind 1: p holds logits.
 * y labels in {0,1}; fp64 accumulation in one block.  out (device, 4 doubles) =
 * {cross_entropy, background_entropy, ne, ctr}; ctr 0 or 1 -> ne = NaN (the
 * host wrapper raises "degenerate background entropy"). */
int kl_ne(int n, int kind, const float* p, const float* y, double* out, void* stream);

/* dtype conversion copy (fp32 <-> bf16), n elements, contiguous. */
int kl_cast(long long n, int dtype_in, const void* x, int dtype_out, void* y, void* stream);

/* Elementwise activation forward / backward with per-column-group codes
 * (same coding as kl_gemm).  (rows, cols) contiguous, row stride ld. */
int kl_act_fwd(int rows, int cols, int dtype, const void* x, long long ld, void* y, long long ld_y,
               int n_act, int act_group, const int* act_codes_host, void* stream);

/* y = g * act'(x) elementwise (the VJP of kl_act_fwd; dfn of tensor.py:431-440). */
int kl_act_bwd(int rows, int cols, int dtype, const void* g, long long ldg, const void* x, long long ldx, void* y,
               long long ld_y, int n_act, int act_group, const int* act_codes_host, void* stream);

/* Fused Adam step over a flat fp32 parameter buffer (bias-corrected; the
 * SPEC.md trainer default), optionally refreshing a bf16 mirror in place.
 * With step_dev != NULL the step count lives on the device: it is incremented
 * first and read by the kernel (CUDA-graph replayable); step == -1 with
 * step_dev reads it without incrementing (one step's Adam split over several
 * parameter ranges, kl_adam_tick issued once before them). */
int kl_adam_step(long long n, float lr, float beta1, float beta2, float eps, int step, int* step_dev, float* w,
                 const float* g, float* m, float* v, void* w_bf16, void* stream);
/* *step_dev += 1 (the device step count of a split Adam step). */
int kl_adam_tick(int* step_dev, void* stream);

/* Non-finite scan: atomically ORs 1 into *flag if any element of x is NaN/Inf
 * (NumericsError, tensor.py:21-27). */
int kl_check_finite(long long n, int dtype, const void* x, unsigned int* flag, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* KUNLUN_CAPI_H */
