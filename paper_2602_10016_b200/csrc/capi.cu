// extern "C" entry points of libkunlun_sm100a.so: argument validation,
// error reporting, and dispatch between the tcgen05 (bf16) and SIMT paths.
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>

#include <cuda.h>

#include "common.cuh"
#include "gemm.h"
#include "swa.h"

namespace kl {

static thread_local char g_err[512] = "";
static std::atomic<unsigned long long> g_launches{0};
static int g_gemm_path = 0;  // 0 auto, 1 force SIMT, 2 force tcgen05 (error if unsupported)
static int g_last_path = -1; // path the last kl_gemm took: 1 tcgen05, 0 SIMT

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int launch_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return KL_ELAUNCH;
  }
  return KL_OK;
}

void count_launch(unsigned n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

static std::atomic<unsigned long long> g_path_hits[KL_PATH_COUNT];
void count_path(int path, unsigned n) {
  if (path >= 0 && path < KL_PATH_COUNT) g_path_hits[path].fetch_add(n, std::memory_order_relaxed);
}

int gemm_path() { return g_gemm_path; }

// Tensor-map encoding is a driver-API call that needs a current context.  The
// autograd engine runs backward ops on its own worker thread, where the
// runtime may not have bound the device's primary context yet (observed:
// CUDA_ERROR_INVALID_CONTEXT from cuTensorMapEncodeTiled); bind the device of
// the launch stream first.
void bind_device(cudaStream_t s) {
  typedef CUresult (*ctx_get_fn)(CUcontext*);
  static ctx_get_fn get_ctx = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuCtxGetCurrent", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      get_ctx = (ctx_get_fn)f;
  }
  CUcontext c = nullptr;
  if (get_ctx && get_ctx(&c) == CUDA_SUCCESS && c) return;  // the common case: nothing to do (capture-safe)
  int dev = -1;
  if (!s || cudaStreamGetDevice(s, &dev) != cudaSuccess) {
    cudaGetLastError();
    cudaGetDevice(&dev);
  }
  if (dev >= 0) cudaSetDevice(dev);
}

static int g_pdl = -1;  // -1: from KL_PDL (default on)
bool pdl_enabled() {
  if (g_pdl < 0) {
    const char* v = getenv("KL_PDL");
    g_pdl = (v && v[0] == '0') ? 0 : 1;
  }
  return g_pdl == 1;
}

}  // namespace kl

using namespace kl;

extern "C" int kl_version(void) { return 1; }
extern "C" const char* kl_last_error(void) { return g_err; }
extern "C" unsigned long long kl_launch_count(void) { return g_launches.load(); }
extern "C" void kl_set_gemm_path(int path) { g_gemm_path = path; }
extern "C" void kl_set_pdl(int on) { kl::g_pdl = on ? 1 : 0; }
extern "C" int kl_last_gemm_path(void) { return kl::g_last_path; }
extern "C" unsigned long long kl_path_hits(int path) {
  return (path >= 0 && path < KL_PATH_COUNT) ? kl::g_path_hits[path].load() : 0ull;
}
extern "C" void kl_reset_path_hits(void) {
  for (auto& h : kl::g_path_hits) h.store(0);
}

extern "C" int kl_tcgen05_available(void) {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  return (major == 10 && minor == 0) ? 1 : 0;
}

// Batch folding in front of both GEMM paths.  A batch dim the B operand
// broadcasts over, with the rows of A, C (and R) continuing evenly across it,
// becomes extra M rows: one tall product instead of nb small ones (a per-sample
// M = 16 product fills 1/8 of every 128-row tile).  A reduced batch dim whose A
// columns and B rows continue across it becomes extra K: one long reduction
// instead of nb k loops each padded to whole 64-wide k blocks (K = 8 per
// sample pads 8x).  The products and sums are the same; only the fp32
// summation order of a folded reduction changes.  Only under-filled shapes
// fold (M < 128 rows, K not a multiple of 64): folding the c4 step's large
// batched GEMMs changed their tile plans and cost 0.5 ms.  Measured on the
// steps (KL_GEMM_FOLD = 0 / 1 / 2 / 3): c4 26.51, 26.54 / 26.38, 26.75 /
// 26.96, 26.68 / 26.14, 26.33 ms; c2 6.27 / 6.21 / 6.24 / 6.25 ms — the K
// folds are the default, the M folds (which cost c4 time) are opt-in.
static void fold_batches(GemmDesc& g, const Epi& e) {
  static int on = -1;
  // 1: M and K folds, 2: M folds only, 3 (default): K folds only
  if (on < 0) on = getenv("KL_GEMM_FOLD") ? atoi(getenv("KL_GEMM_FOLD")) : 3;
  if (!on) return;
  for (int pass = 0; pass < 2; ++pass) {  // batch dim 2, then 1
    int& nb = pass == 0 ? g.nb2 : g.nb1;
    int& red = pass == 0 ? g.red2 : g.red1;
    long long& as = pass == 0 ? g.a_s2 : g.a_s1;
    long long& bs = pass == 0 ? g.b_s2 : g.b_s1;
    long long& cs = pass == 0 ? g.c_s2 : g.c_s1;
    long long& rs = pass == 0 ? g.r_s2 : g.r_s1;
    if (nb <= 1) continue;
    if (!red) {
      if (on == 3) continue;
      const long long M = g.M;
      if (M >= 128 || e.row_limit || bs != 0 || g.a_rs == 0 || as != M * g.a_rs || g.c_rs == 0 || cs != M * g.c_rs ||
          (g.R && (g.r_rs == 0 || rs != M * g.r_rs)) || M * nb > (1LL << 30))
        continue;
      g.M = (int)(M * nb);
      nb = 1;
      as = bs = cs = rs = 0;
    } else {
      if (on == 2) continue;
      const long long K = g.K;
      if (K % 64 == 0 || g.a_cs == 0 || as != K * g.a_cs || g.b_rs == 0 || bs != K * g.b_rs || K * nb > (1LL << 30)) continue;
      g.K = (int)(K * nb);
      nb = 1;
      red = 0;
      as = bs = cs = rs = 0;
    }
  }
}

extern "C" int kl_gemm(const kl_gemm_args* a, void* stream) {
  if (!a) {
    set_error("kl_gemm: null args");
    return KL_EBADSHAPE;
  }
  if (a->M < 0 || a->N < 0 || a->K < 0 || a->nb1 < 1 || a->nb2 < 1) {
    set_error("kl_gemm: bad extents M=%d N=%d K=%d nb=(%d,%d)", a->M, a->N, a->K, a->nb1, a->nb2);
    return KL_EBADSHAPE;
  }
  if ((a->ab_dtype != KL_F32 && a->ab_dtype != KL_BF16) || (a->c_dtype != KL_F32 && a->c_dtype != KL_BF16)) {
    set_error("kl_gemm: bad dtype");
    return KL_EUNSUPPORTED;
  }
  if (a->n_act < 0 || a->n_act > KL_MAX_ACT_GROUPS || (a->n_act > 1 && a->act_group < 1)) {
    set_error("kl_gemm: bad activation groups (%d, %d)", a->n_act, a->act_group);
    return KL_EBADSHAPE;
  }
  if (a->aux_mode && !a->aux) {
    set_error("kl_gemm: aux_mode %d without aux buffer", a->aux_mode);
    return KL_EBADSHAPE;
  }
  if (a->row_limit && (a->red1 || a->red2)) {
    set_error("kl_gemm: row_limit cannot be combined with batch reduction");
    return KL_EBADSHAPE;
  }
  if (a->M == 0 || a->N == 0) return KL_OK;
  GemmDesc g;
  g.M = a->M; g.N = a->N; g.K = a->K;
  g.nb1 = a->nb1; g.nb2 = a->nb2; g.red1 = a->red1; g.red2 = a->red2;
  g.ab_dtype = a->ab_dtype; g.c_dtype = a->c_dtype;
  g.A = a->A; g.a_rs = a->a_rs; g.a_cs = a->a_cs; g.a_s1 = a->a_s1; g.a_s2 = a->a_s2;
  g.B = a->B; g.b_rs = a->b_rs; g.b_cs = a->b_cs; g.b_s1 = a->b_s1; g.b_s2 = a->b_s2;
  g.C = a->C; g.c_rs = a->c_rs; g.c_cs = a->c_cs; g.c_s1 = a->c_s1; g.c_s2 = a->c_s2;
  g.R = a->R; g.r_rs = a->r_rs; g.r_cs = a->r_cs; g.r_s1 = a->r_s1; g.r_s2 = a->r_s2;
  g.aux = a->aux;
  g.ws = (float*)a->workspace;
  g.ws_bytes = a->workspace ? a->workspace_bytes : 0;
  Epi e;
  e.alpha = a->alpha; e.beta = a->beta; e.bias = a->bias; e.row_limit = a->row_limit;
  e.aux_mode = a->aux_mode; e.n_act = a->n_act; e.act_group = a->act_group > 0 ? a->act_group : 1;
  for (int i = 0; i < KL_MAX_ACT_GROUPS; ++i) e.act_codes[i] = a->act_codes[i];
  fold_batches(g, e);
  cudaStream_t s = (cudaStream_t)stream;
  bind_device(s);
  if (a->ab_dtype == KL_BF16 && g_gemm_path != 1) {
    int rc = gemm_tc(g, e, s);
    g_last_path = 1;
    if (rc != KL_EUNSUPPORTED) return rc;
    if (g_gemm_path == 2) {
      set_error("kl_gemm: tcgen05 path forced but shape unsupported (M=%d N=%d K=%d)", a->M, a->N, a->K);
      return KL_EUNSUPPORTED;
    }
  }
  g_last_path = 0;
  return gemm_simt(g, e, s);
}

static int swa_validate(const kl_swa_args* a, const char* who, SwaP& p) {
  if (!a || a->B < 0 || a->T < 0 || a->H < 1 || a->d_h < 1 || a->w < 0) {
    set_error("%s: bad extents", who);
    return KL_EBADSHAPE;
  }
  if (a->dtype != KL_F32 && a->dtype != KL_BF16) {
    set_error("%s: bad dtype", who);
    return KL_EUNSUPPORTED;
  }
  p.B = a->B; p.T = a->T; p.H = a->H; p.d_h = a->d_h; p.w = a->w; p.causal = a->causal; p.dtype = a->dtype;
  p.scale = a->scale; p.lengths = a->lengths;
  p.QKV = a->QKV; p.ld_qkv = a->ld_qkv; p.bs_qkv = a->bs_qkv;
  p.O = a->O; p.ld_o = a->ld_o; p.bs_o = a->bs_o; p.LSE = a->LSE;
  p.dO = a->dO; p.dQKV = a->dQKV; p.Dbuf = a->Dbuf;
  return KL_OK;
}

extern "C" int kl_swa_fwd(const kl_swa_args* a, void* stream) {
  SwaP p;
  int rc = swa_validate(a, "kl_swa_fwd", p);
  if (rc) return rc;
  if (p.B == 0 || p.T == 0) return KL_OK;
  cudaStream_t s = (cudaStream_t)stream;
  bind_device(s);
  if (p.dtype == KL_BF16 && g_gemm_path != 1) {
    rc = swa_fwd_tc(p, s);
    if (rc != KL_EUNSUPPORTED) return rc;
  }
  return swa_fwd_simt(p, s);
}

extern "C" int kl_swa_bwd(const kl_swa_args* a, void* stream) {
  SwaP p;
  int rc = swa_validate(a, "kl_swa_bwd", p);
  if (rc) return rc;
  if (p.B == 0 || p.T == 0) return KL_OK;
  if (!p.dO || !p.dQKV || !p.Dbuf || !p.LSE) {
    set_error("kl_swa_bwd: dO, dQKV, Dbuf and LSE are required");
    return KL_EBADSHAPE;
  }
  cudaStream_t s = (cudaStream_t)stream;
  bind_device(s);
  if (p.dtype == KL_BF16 && g_gemm_path != 1) {
    rc = swa_bwd_tc(p, s);
    if (rc != KL_EUNSUPPORTED) return rc;
  }
  return swa_bwd_simt(p, s);
}

extern "C" int kl_swa_debug_support(const kl_swa_args* a, int* support, void* stream) {
  SwaP p;
  int rc = swa_validate(a, "kl_swa_debug_support", p);
  if (rc) return rc;
  if (p.B == 0 || p.T == 0) return KL_OK;
  return swa_support(p, support, (cudaStream_t)stream);
}
