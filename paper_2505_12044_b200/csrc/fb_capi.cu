// fb_capi.cu — the extern "C" boundary (include/flashbias_b200.h).
//
// Validation mirrors the reference's pre-compute checks
// (pkg/src/flashbias/attention.py:77-93 _validate_qkv/_validate_mask and
// 215-223 factor rank/row checks) and maps them onto status codes that the
// Python shim turns back into ShapeError / MaskError / ConfigError /
// ValidationError (errors.py:4-17).  No allocation, stream ordered.
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <mutex>

#include "../../include/flashbias_b200.h"
#include "fb_kernels.h"
#include "fb_sm100.cuh"

namespace fb {

static thread_local char g_err[512] = "";
// process-wide (autograd runs the backward on its own thread)
static std::atomic<int64_t> g_launches{0};

void note_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

static unsigned long long* g_trace_buf = nullptr;
static int g_trace_cta = -1;
void trace_target(unsigned long long** buf, int* cta) {
  *buf = g_trace_buf;
  *cta = g_trace_cta;
}

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

static int cuda_fail(cudaError_t e, const char* where) {
  return fail(FB_ECUDA, "%s: %s", where, cudaGetErrorString(e));
}

static size_t dtype_size(int dt) {
  switch (dt) {
    case FB_F32: return 4;
    case FB_BF16: return 2;
    case FB_F16: return 2;
    case FB_F64: return 8;
  }
  return 0;
}

static Tensor4 to_t4(const fb_tensor* t) {
  Tensor4 r;
  r.data = t->data;
  for (int i = 0; i < 4; ++i) {
    r.shape[i] = t->shape[i];
    r.stride[i] = t->shape[i] == 1 ? 0 : t->stride[i];
  }
  r.dtype = t->dtype;
  return r;
}

// ------------------------------------------------------------ tensor maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  return fn;
}

// 4-D map over a [B,H,L,C] view with box [box_cols x 128 rows].
static int make_map(CUtensorMap* map, const fb_tensor* t, int box_cols, int box_rows, int swizzle_bytes,
                    const char* name) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(FB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const size_t es = dtype_size(t->dtype);
  if (t->stride[3] != 1) return fail(FB_ESHAPE, "%s: last dim must be contiguous", name);
  if (reinterpret_cast<uintptr_t>(t->data) % 16) return fail(FB_EVALUE, "%s: data must be 16-byte aligned", name);
  cuuint64_t dims[4] = {(cuuint64_t)t->shape[3], (cuuint64_t)t->shape[2], (cuuint64_t)t->shape[1],
                        (cuuint64_t)t->shape[0]};
  cuuint64_t strides[3];
  int64_t inner = t->shape[3] * (int64_t)es;
  for (int i = 0; i < 3; ++i) {
    const int dim = 2 - i;  // L, H, B
    int64_t st = t->stride[dim] * (int64_t)es;
    if (t->shape[dim] == 1 || t->stride[dim] == 0) st = inner;  // broadcast / unit dim
    if (st % 16) return fail(FB_EVALUE, "%s: stride of dim %d (%lld bytes) not a multiple of 16", name, dim,
                             (long long)st);
    strides[i] = (cuuint64_t)st;
    inner = st * (t->shape[dim] > 0 ? t->shape[dim] : 1);
  }
  cuuint32_t box[4] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUtensorMapSwizzle sw = swizzle_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                          : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                          : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUtensorMapDataType dt = t->dtype == FB_BF16  ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                           : t->dtype == FB_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                                : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUresult r = enc(map, dt, 4, t->data, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FB_ECUDA, "%s: cuTensorMapEncodeTiled failed (%d)", name, (int)r);
  return FB_OK;
}

static inline int swz_for(int d) { return d * 2 >= 128 ? 128 : (d * 2 >= 64 ? 64 : 32); }

// ------------------------------------------------------------ validation
static int check_qkv(const fb_tensor* q, const fb_tensor* k, const fb_tensor* v) {
  if (!q || !k || !v) return fail(FB_EVALUE, "q, k, v are required");
  for (int i = 0; i < 4; ++i)
    if (q->shape[i] < 0 || k->shape[i] < 0 || v->shape[i] < 0) return fail(FB_ESHAPE, "negative extent");
  if (q->shape[3] != k->shape[3])
    return fail(FB_ESHAPE, "q and k channel counts differ: %lld vs %lld", (long long)q->shape[3],
                (long long)k->shape[3]);
  if (k->shape[2] != v->shape[2])
    return fail(FB_ESHAPE, "k and v row counts differ: %lld vs %lld", (long long)k->shape[2],
                (long long)v->shape[2]);
  if (q->shape[0] != k->shape[0] || q->shape[1] != k->shape[1] || k->shape[0] != v->shape[0] ||
      k->shape[1] != v->shape[1])
    return fail(FB_ESHAPE, "batch/head extents of q, k, v differ");
  if (q->dtype != k->dtype || k->dtype != v->dtype) return fail(FB_EVALUE, "q, k, v dtypes differ");
  if (q->shape[2] < 1 || k->shape[2] < 1) return fail(FB_ESHAPE, "empty sequence");
  return FB_OK;
}

static int check_mask(int mask, int64_t n, int64_t m) {
  if (mask != FB_MASK_NONE && mask != FB_MASK_CAUSAL) return fail(FB_EVALUE, "unknown mask %d", mask);
  if (mask == FB_MASK_CAUSAL && n != m)
    return fail(FB_EMASK, "causal mask requires N == M, got %lld x %lld", (long long)n, (long long)m);
  return FB_OK;
}

static bool bcast_ok(int64_t f, int64_t full) { return f == 1 || f == full; }

static int check_factors(const fb_tensor* q, const fb_tensor* k, const fb_tensor* uq, const fb_tensor* uk) {
  if ((uq == nullptr) != (uk == nullptr)) return fail(FB_EVALUE, "uq and uk must be given together");
  if (!uq) return FB_OK;
  if (uq->shape[3] != uk->shape[3])
    return fail(FB_ESHAPE, "factor ranks differ: %lld vs %lld", (long long)uq->shape[3], (long long)uk->shape[3]);
  if (uq->shape[2] != q->shape[2])
    return fail(FB_ESHAPE, "fq rows %lld do not match q rows %lld", (long long)uq->shape[2], (long long)q->shape[2]);
  if (uk->shape[2] != k->shape[2])
    return fail(FB_ESHAPE, "fk rows %lld do not match k rows %lld", (long long)uk->shape[2], (long long)k->shape[2]);
  if (!bcast_ok(uq->shape[0], q->shape[0]) || !bcast_ok(uq->shape[1], q->shape[1]) ||
      !bcast_ok(uk->shape[0], q->shape[0]) || !bcast_ok(uk->shape[1], q->shape[1]))
    return fail(FB_ESHAPE, "factor batch/head extents must be 1 or match q");
  return FB_OK;
}

static int check_bias(const fb_tensor* q, const fb_tensor* k, const fb_tensor* bias) {
  if (!bias) return FB_OK;
  if (bias->shape[2] != q->shape[2] || bias->shape[3] != k->shape[2])
    return fail(FB_ESHAPE, "bias shape (%lld, %lld) does not match logits (%lld, %lld)",
                (long long)bias->shape[2], (long long)bias->shape[3], (long long)q->shape[2],
                (long long)k->shape[2]);
  if (!bcast_ok(bias->shape[0], q->shape[0]) || !bcast_ok(bias->shape[1], q->shape[1]))
    return fail(FB_ESHAPE, "bias batch/head extents must be 1 or match q");
  return FB_OK;
}

}  // namespace fb

using namespace fb;

extern "C" {

const char* fb_last_error(void) { return g_err; }

/* Debug hook (not part of the public header): route kernel timeline records of
 * CTA `cta` into the device buffer `buf` (uint64, buf[0] = count).  Only the
 * FB_TRACE=1 build records anything. */
void fb_debug_set_trace(void* buf, int cta) {
  g_trace_buf = reinterpret_cast<unsigned long long*>(buf);
  g_trace_cta = cta;
}
int fb_debug_trace_enabled(void) { return FB_TRACE; }
int fb_abi_version(void) { return FB_ABI_VERSION; }
int64_t fb_launch_count(int reset) {
  return reset ? g_launches.exchange(0, std::memory_order_relaxed) : g_launches.load(std::memory_order_relaxed);
}

int64_t fb_factor_cols(int64_t rank, int split) { return rank * factor_pairs(split); }
int64_t fb_factor_rpad(int64_t rank, int split) { return (fb_factor_cols(rank, split) + 15) / 16 * 16; }

int fb_attn_fwd(const fb_tensor* q, const fb_tensor* k, const fb_tensor* v, const fb_tensor* uq,
                const fb_tensor* uk, const fb_tensor* bias, int mask, float scale, fb_tensor* o,
                fb_tensor* lse, void* stream) {
  int rc;
  if ((rc = check_qkv(q, k, v))) return rc;
  if ((rc = check_mask(mask, q->shape[2], k->shape[2]))) return rc;
  if ((rc = check_factors(q, k, uq, uk))) return rc;
  if ((rc = check_bias(q, k, bias))) return rc;
  if (!o) return fail(FB_EVALUE, "output tensor required");
  if (o->shape[0] != q->shape[0] || o->shape[1] != q->shape[1] || o->shape[2] != q->shape[2] ||
      o->shape[3] != v->shape[3])
    return fail(FB_ESHAPE, "output shape mismatch");
  if (o->dtype != q->dtype) return fail(FB_EVALUE, "output dtype must match q");
  if (!(scale > 0.f) || !isfinite(scale)) return fail(FB_EVALUE, "scale must be positive and finite");
  if (q->shape[0] * q->shape[1] == 0) return FB_OK;  // no heads: nothing to launch
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int B = (int)q->shape[0], H = (int)q->shape[1], N = (int)q->shape[2], M = (int)k->shape[2];
  const int D = (int)q->shape[3];

  if (q->dtype == FB_F32) {
    if (D > 128 || v->shape[3] != D) return fail(FB_ECONFIG, "fp32 path supports D <= 128 with dv == d");
    const int R = uq ? (int)uq->shape[3] : 0;
    if (D + R > 320) return fail(FB_ECONFIG, "fp32 path supports D + R <= 320");
    if ((uq && (uq->dtype != FB_F32 || uk->dtype != FB_F32)) || (bias && bias->dtype != FB_F32))
      return fail(FB_EVALUE, "fp32 path needs fp32 factors and bias");
    Tensor4 tq = to_t4(q), tk = to_t4(k), tv = to_t4(v), to = to_t4(o);
    if (B > 65535 || H > 65535)
      return fail(FB_ECONFIG, "fp32 path: at most 65535 batch rows and 65535 heads per call (got %lld x %lld); "
                              "pass head slices", (long long)B, (long long)H);
    SimtParams p{};
    p.B = B; p.H = H; p.N = N; p.M = M; p.D = D; p.R = R;
    p.causal = mask == FB_MASK_CAUSAL;
    p.scale = scale;
    p.q = (const float*)q->data; p.q_sb = tq.stride[0]; p.q_sh = tq.stride[1]; p.q_sn = tq.stride[2];
    p.k = (const float*)k->data; p.k_sb = tk.stride[0]; p.k_sh = tk.stride[1]; p.k_sn = tk.stride[2];
    p.v = (const float*)v->data; p.v_sb = tv.stride[0]; p.v_sh = tv.stride[1]; p.v_sn = tv.stride[2];
    if (uq) {
      Tensor4 a = to_t4(uq), c = to_t4(uk);
      p.uq = (const float*)uq->data; p.uq_sb = a.stride[0]; p.uq_sh = a.stride[1]; p.uq_sn = a.stride[2];
      p.uk = (const float*)uk->data; p.uk_sb = c.stride[0]; p.uk_sh = c.stride[1]; p.uk_sn = c.stride[2];
      if (uq->stride[3] != 1 || uk->stride[3] != 1) return fail(FB_ESHAPE, "factor last dim must be contiguous");
    }
    if (bias) {
      Tensor4 a = to_t4(bias);
      if (bias->stride[3] != 1) return fail(FB_ESHAPE, "bias last dim must be contiguous");
      p.bias = (const float*)bias->data; p.bias_sb = a.stride[0]; p.bias_sh = a.stride[1]; p.bias_sn = a.stride[2];
    }
    for (const fb_tensor* t : {q, k, v, (const fb_tensor*)o})
      if (t->stride[3] != 1) return fail(FB_ESHAPE, "last dim must be contiguous");
    p.o = (float*)o->data; p.o_sb = to.stride[0]; p.o_sh = to.stride[1]; p.o_sn = to.stride[2];
    p.lse = lse ? (float*)lse->data : nullptr;
    cudaError_t e = launch_fwd_simt_f32(p, s);
    return e == cudaSuccess ? FB_OK : cuda_fail(e, "fwd_simt_f32");
  }

  if (q->dtype != FB_BF16 && q->dtype != FB_F16) return fail(FB_EVALUE, "unsupported dtype %d", q->dtype);
  if (D != 32 && D != 64 && D != 128)
    return fail(FB_ECONFIG, "tcgen05 path supports head dim 32, 64, 128 (got %d); pad on the host", D);
  if (v->shape[3] != D) return fail(FB_ECONFIG, "tcgen05 path needs dv == d");
  int rp = 0;
  if (uq) {
    const int64_t rpad = uq->shape[3];
    const int64_t rmax = D == 128 ? 64 : 128;
    if (rpad % 16 || rpad > rmax)
      return fail(FB_ECONFIG, "factor panels must have Rpad a multiple of 16 <= %lld for head dim %d (got %lld)",
                  (long long)rmax, D, (long long)rpad);
    if (uq->dtype != q->dtype || uk->dtype != q->dtype) return fail(FB_EVALUE, "factor panels must match q dtype");
    rp = (int)(rpad / 16);
  }
  if (bias) {
    if (uq) return fail(FB_ECONFIG, "tcgen05 path takes either factors or a dense bias, not both");
    if (bias->dtype != q->dtype) return fail(FB_EVALUE, "dense bias dtype must match q");
    if ((bias->stride[2] * 2) % 16) return fail(FB_ECONFIG, "dense bias rows must be 16-byte aligned (pad the row stride)");
  }
  FwdMaps maps;
  memset(&maps, 0, sizeof(maps));
  const int sw = swz_for(D);
  if ((rc = make_map(&maps.q, q, sw / 2, 128, sw, "q"))) return rc;
  if ((rc = make_map(&maps.k, k, sw / 2, 128, sw, "k"))) return rc;
  if ((rc = make_map(&maps.v, v, sw / 2, 128, sw, "v"))) return rc;
  if (uq) {
    if ((rc = make_map(&maps.uq, uq, 16, 128, 32, "uq"))) return rc;
    if ((rc = make_map(&maps.uk, uk, 16, 128, 32, "uk"))) return rc;
  }
  if (bias && (rc = make_map(&maps.bias, bias, 64, 128, 128, "bias"))) return rc;
  if (o->stride[3] != 1 || (o->stride[2] * 2) % 16) return fail(FB_ESHAPE, "output rows must be contiguous, 16B aligned");
  FwdParams p{};
  p.B = B; p.H = H; p.N = N; p.M = M;
  p.causal = mask == FB_MASK_CAUSAL;
  p.num_pairs = (N + 255) / 256;
  p.scale_log2 = scale * 1.4426950408889634f;
  Tensor4 to = to_t4(o);
  p.o = o->data; p.o_sb = to.stride[0]; p.o_sh = to.stride[1]; p.o_sn = to.stride[2];
  p.lse = lse ? (float*)lse->data : nullptr;
  if (uq) {
    p.uq_bb = uq->shape[0] == 1; p.uq_hb = uq->shape[1] == 1;
    p.uk_bb = uk->shape[0] == 1; p.uk_hb = uk->shape[1] == 1;
  }
  if (bias) { p.bias_bb = bias->shape[0] == 1; p.bias_hb = bias->shape[1] == 1; }
  trace_target(&p.trace, &p.trace_cta);
  cudaError_t e = launch_fwd_sm100(D, rp, bias != nullptr, q->dtype == FB_BF16, maps, p, s);
  note_launch();
  return e == cudaSuccess ? FB_OK : cuda_fail(e, "fwd_sm100");
}

size_t fb_bwd_workspace_bytes(const fb_tensor* q, const fb_tensor* k) {
  (void)k;
  if (!q) return 0;
  const size_t rows = (size_t)q->shape[0] * q->shape[1] * q->shape[2];
  size_t bytes = (rows * sizeof(float) + 255) / 256 * 256 + 256;  // delta
  // fp32 dQ accumulator of the fused backwards: [B,H,N,D]
  if (q->shape[3] == 128 || q->shape[3] == 64)
    bytes += (size_t)q->shape[0] * q->shape[1] * q->shape[2] * q->shape[3] * sizeof(float);
  return bytes;
}

int fb_attn_bwd(const fb_tensor* q, const fb_tensor* k, const fb_tensor* v, const fb_tensor* uq,
                const fb_tensor* uk, const fb_tensor* bias, const fb_tensor* o, const fb_tensor* lse,
                const fb_tensor* dout, int mask, float scale, fb_tensor* dq, fb_tensor* dk,
                fb_tensor* dv, fb_tensor* duq, fb_tensor* duk, void* workspace,
                size_t workspace_bytes, void* stream) {
  return fb_attn_bwd_ex(q, k, v, uq, uk, bias, o, lse, dout, mask, scale, dq, dk, dv, duq, duk, nullptr, 0,
                        workspace, workspace_bytes, stream);
}

int fb_attn_bwd_ex(const fb_tensor* q, const fb_tensor* k, const fb_tensor* v, const fb_tensor* uq,
                   const fb_tensor* uk, const fb_tensor* bias, const fb_tensor* o, const fb_tensor* lse,
                   const fb_tensor* dout, int mask, float scale, fb_tensor* dq, fb_tensor* dk,
                   fb_tensor* dv, fb_tensor* duq, fb_tensor* duk, fb_tensor* dbias, int flags,
                   void* workspace, size_t workspace_bytes, void* stream) {
  int rc;
  if (flags & ~FB_BWD_DETERMINISTIC) return fail(FB_EVALUE, "unknown backward flags 0x%x", flags);
  if ((rc = check_qkv(q, k, v))) return rc;
  if ((rc = check_mask(mask, q->shape[2], k->shape[2]))) return rc;
  if ((rc = check_factors(q, k, uq, uk))) return rc;
  if ((rc = check_bias(q, k, bias))) return rc;
  if (!o || !lse || !dout || !dq || !dk || !dv) return fail(FB_EVALUE, "o, lse, dout, dq, dk, dv are required");
  if ((duq == nullptr) != (duk == nullptr)) return fail(FB_EVALUE, "duq and duk must be given together");
  if (duq && !uq) return fail(FB_EVALUE, "factor gradients requested without factors");
  if (q->dtype != FB_BF16 && q->dtype != FB_F16) return fail(FB_ECONFIG, "backward supports bf16/f16 only");
  const int B = (int)q->shape[0], H = (int)q->shape[1], N = (int)q->shape[2], M = (int)k->shape[2];
  const int D = (int)q->shape[3];
  if (D != 32 && D != 64 && D != 128) return fail(FB_ECONFIG, "backward supports head dim 32, 64, 128");
  if (q->shape[0] * q->shape[1] == 0) return FB_OK;  // no heads: nothing to launch
  if (workspace_bytes < fb_bwd_workspace_bytes(q, k) || !workspace) return fail(FB_ECONFIG, "workspace too small");
  int rp = 0;
  if (uq) {
    const int64_t rpad = uq->shape[3];
    if (rpad % 16 || rpad > (D == 128 ? 64 : 128))
      return fail(FB_ECONFIG, "factor panels must have Rpad a multiple of 16 <= %d", D == 128 ? 64 : 128);
    rp = (int)(rpad / 16);
  }
  if (bias && uq) return fail(FB_ECONFIG, "either factors or a dense bias, not both");
  if (dbias) {
    if (!bias) return fail(FB_EVALUE, "dbias requested without a dense bias");
    if (dbias->dtype != bias->dtype) return fail(FB_EVALUE, "dbias dtype must match the bias");
    if (dbias->shape[0] != B || dbias->shape[1] != H || dbias->shape[2] != N || dbias->shape[3] != M)
      return fail(FB_ESHAPE, "dbias must be [B,H,N,M] (reduce broadcast dims on the host)");
    if (dbias->stride[3] != 1 || dbias->stride[2] % 2 || reinterpret_cast<uintptr_t>(dbias->data) % 4)
      return fail(FB_ESHAPE, "dbias rows must be contiguous with an even, 4-byte aligned row stride");
  }
  if (bias && (bias->stride[2] * 2) % 16) return fail(FB_ECONFIG, "dense bias rows must be 16-byte aligned");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // preprocess delta = rowsum(dO * O)
  float* delta = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(workspace) + 255) & ~uintptr_t(255));
  Tensor4 tdelta{};
  tdelta.data = delta;
  tdelta.shape[0] = B; tdelta.shape[1] = H; tdelta.shape[2] = N; tdelta.shape[3] = 1;
  tdelta.stride[0] = (int64_t)H * N; tdelta.stride[1] = N; tdelta.stride[2] = 1; tdelta.stride[3] = 1;
  tdelta.dtype = FB_F32;
  cudaError_t e = launch_bwd_preprocess(to_t4(o), to_t4(dout), tdelta, s);
  if (e != cudaSuccess) return cuda_fail(e, "bwd_preprocess");

  BwdMaps maps;
  memset(&maps, 0, sizeof(maps));
  const int sw = swz_for(D);
  if ((rc = make_map(&maps.q64, q, sw / 2, 64, sw, "q"))) return rc;
  if ((rc = make_map(&maps.q128, q, sw / 2, 128, sw, "q"))) return rc;
  if ((rc = make_map(&maps.do64, dout, sw / 2, 64, sw, "dout"))) return rc;
  if ((rc = make_map(&maps.do128, dout, sw / 2, 128, sw, "dout"))) return rc;
  if ((rc = make_map(&maps.k128, k, sw / 2, 128, sw, "k"))) return rc;
  if ((rc = make_map(&maps.k64, k, sw / 2, 64, sw, "k"))) return rc;
  if ((rc = make_map(&maps.v128, v, sw / 2, 128, sw, "v"))) return rc;
  if ((rc = make_map(&maps.v64, v, sw / 2, 64, sw, "v"))) return rc;
  if (uq) {
    if ((rc = make_map(&maps.uq64, uq, 16, 64, 32, "uq"))) return rc;
    if ((rc = make_map(&maps.uq128, uq, 16, 128, 32, "uq"))) return rc;
    if ((rc = make_map(&maps.uk64, uk, 16, 64, 32, "uk"))) return rc;
    if ((rc = make_map(&maps.uk128, uk, 16, 128, 32, "uk"))) return rc;
  }
  if (bias) {
    if ((rc = make_map(&maps.biasT, bias, 64, 64, 128, "bias"))) return rc;
    if ((rc = make_map(&maps.bias, bias, 64, 128, 128, "bias"))) return rc;
  }
  for (const fb_tensor* t : {(const fb_tensor*)dq, (const fb_tensor*)dk, (const fb_tensor*)dv})
    if (t->stride[3] != 1 || (t->stride[2] * 2) % 16 || t->dtype != q->dtype || t->shape[3] != D)
      return fail(FB_ESHAPE, "gradient outputs must match q dtype/shape with contiguous rows");
  BwdParams p{};
  p.B = B; p.H = H; p.N = N; p.M = M;
  p.causal = mask == FB_MASK_CAUSAL;
  p.scale = scale;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.lse = (const float*)lse->data;
  p.delta = delta;
  Tensor4 a;
  a = to_t4(dq); p.dq = dq->data; p.dq_sb = a.stride[0]; p.dq_sh = a.stride[1]; p.dq_sn = a.stride[2];
  a = to_t4(dk); p.dk = dk->data; p.dk_sb = a.stride[0]; p.dk_sh = a.stride[1]; p.dk_sn = a.stride[2];
  a = to_t4(dv); p.dv = dv->data; p.dv_sb = a.stride[0]; p.dv_sh = a.stride[1]; p.dv_sn = a.stride[2];
  if (duq) {
    if (duq->dtype != FB_F32 || duk->dtype != FB_F32) return fail(FB_EVALUE, "factor gradients are fp32");
    a = to_t4(duq); p.duq = (float*)duq->data; p.duq_sb = a.stride[0]; p.duq_sh = a.stride[1]; p.duq_sn = a.stride[2];
    a = to_t4(duk); p.duk = (float*)duk->data; p.duk_sb = a.stride[0]; p.duk_sh = a.stride[1]; p.duk_sn = a.stride[2];
  }
  if (uq) {
    p.uq_bb = uq->shape[0] == 1; p.uq_hb = uq->shape[1] == 1;
    p.uk_bb = uk->shape[0] == 1; p.uk_hb = uk->shape[1] == 1;
  }
  if (bias) { p.bias_bb = bias->shape[0] == 1; p.bias_hb = bias->shape[1] == 1; }
  if (dbias) {
    Tensor4 td = to_t4(dbias);
    p.dbias = dbias->data; p.db_sb = td.stride[0]; p.db_sh = td.stride[1]; p.db_sn = td.stride[2];
  }
  trace_target(&p.trace, &p.trace_cta);
  static const int force_split = [] {
    const char* v = getenv("FB_FORCE_SPLIT_BWD");
    return v && v[0] == '1' ? 1 : 0;
  }();
  // FB_BWD_DETERMINISTIC (or the FB_FORCE_SPLIT_BWD=1 testing hook, read once) selects the two-kernel
  // backward: no atomics, every gradient element written once in a fixed order
  const bool deterministic = force_split || (flags & FB_BWD_DETERMINISTIC);
  static const int t128_off = [] {
    const char* v = getenv("FB_BWD_T128");
    return v && v[0] == '0' ? 1 : 0;
  }();
  // learnable factors at d = 128 ride the 128x128-tile kernel when they fit one 16-column panel
  const bool use_t128 = !t128_off && bwd_t128_supported(D, rp, bias != nullptr, duq != nullptr);
  const bool fused = !deterministic && (use_t128 || (D == 128 && duq == nullptr) || (D == 64 && rp <= 4));
  if (dbias && !fused)
    return fail(FB_ECONFIG, "the dense-bias gradient is produced by the fused backward (head dim 64/128, "
                            "not deterministic)");
  if (fused) {
    float* acc = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(delta) +
                                          ((size_t)B * H * N * sizeof(float) + 255) / 256 * 256);
    fb_tensor tacc{};
    tacc.data = acc;
    tacc.shape[0] = B; tacc.shape[1] = H; tacc.shape[2] = N; tacc.shape[3] = D;
    tacc.stride[3] = 1; tacc.stride[2] = D; tacc.stride[1] = (int64_t)N * D; tacc.stride[0] = (int64_t)H * N * D;
    tacc.dtype = FB_F32;
    CUtensorMap macc;
    if ((rc = make_map(&macc, &tacc, D, 32, 0, "dq_acc"))) return rc;
    if (use_t128) {
      // the [B,H,N,128] accumulator in 16-query x 128-dim boxes (full 512-byte rows, no swizzle)
      CUtensorMap macc16;
      if ((rc = make_map(&macc16, &tacc, D, 16, 0, "dq_acc16"))) return rc;
      e = cudaMemsetAsync(acc, 0, (size_t)B * H * N * D * sizeof(float), s);
      if (e != cudaSuccess) return cuda_fail(e, "memset dq_acc");
      CUtensorMap mduq;
      memset(&mduq, 0, sizeof(mduq));
      if (duq) {  // dUq is reduce-added in 128-query x 16-column boxes: start from zero
        if (duq->stride[3] != 1 || duq->shape[3] != 16 || duk->stride[3] != 1 || duk->shape[3] != 16 ||
            (duk->stride[2] * 4) % 16)
          return fail(FB_ESHAPE, "factor gradient outputs must be [B,H,L,16] fp32 with contiguous 16-byte rows");
        if ((rc = make_map(&mduq, duq, 16, 128, 64, "duq"))) return rc;
        for (int64_t bb = 0; bb < duq->shape[0]; ++bb)
          for (int64_t hh = 0; hh < duq->shape[1]; ++hh) {
            e = cudaMemsetAsync(static_cast<float*>(duq->data) + bb * duq->stride[0] + hh * duq->stride[1], 0,
                                (size_t)duq->shape[2] * duq->stride[2] * sizeof(float), s);
            if (e != cudaSuccess) return cuda_fail(e, "memset duq");
          }
      }
      e = launch_bwd_t128_sm100(rp, q->dtype == FB_BF16, duq != nullptr, maps, macc16, mduq, p, s);
      if (e != cudaSuccess) return cuda_fail(e, "bwd_t128_sm100");
      e = launch_dq_convert(acc, D, p, q->dtype == FB_BF16, s);
      note_launch(2);
      return e == cudaSuccess ? FB_OK : cuda_fail(e, "dq_convert");
    }
    // the 64-query kernels reduce into the untransposed [B,H,N,D] accumulator: start from zero
    e = cudaMemsetAsync(acc, 0, (size_t)B * H * N * D * sizeof(float), s);
    if (e != cudaSuccess) return cuda_fail(e, "memset dq_acc");
    if (D == 128) {
      e = launch_bwd_fused_sm100(rp, bias != nullptr, q->dtype == FB_BF16, maps, macc, p, s);
    } else {
      CUtensorMap mduq;
      memset(&mduq, 0, sizeof(mduq));
      if (uq) {
        if ((rc = make_map(&maps.uq64w, uq, 64, 64, 128, "uq"))) return rc;
        if ((rc = make_map(&maps.uk128w, uk, 64, 128, 128, "uk"))) return rc;
      }
      if (duq) {
        if (duq->stride[3] != 1 || duq->shape[3] != uq->shape[3]) return fail(FB_ESHAPE, "duq layout");
        if ((rc = make_map(&mduq, duq, (int)duq->shape[3], 32, 0, "duq"))) return rc;
        for (int64_t bb = 0; bb < duq->shape[0]; ++bb)  // TMA-reduced into: start from zero
          for (int64_t hh = 0; hh < duq->shape[1]; ++hh) {
            e = cudaMemsetAsync(static_cast<float*>(duq->data) + bb * duq->stride[0] + hh * duq->stride[1], 0,
                                (size_t)duq->shape[2] * duq->stride[2] * sizeof(float), s);
            if (e != cudaSuccess) return cuda_fail(e, "memset duq");
          }
      }
      e = launch_bwd_fused64_sm100(rp, bias != nullptr, q->dtype == FB_BF16, duq != nullptr, maps, macc, mduq, p, s);
    }
    if (e != cudaSuccess) return cuda_fail(e, "bwd_fused_sm100");
    e = launch_dq_convert(acc, D, p, q->dtype == FB_BF16, s);
    note_launch(2);
    return e == cudaSuccess ? FB_OK : cuda_fail(e, "dq_convert");
  }
  e = launch_bwd_sm100(D, rp, bias != nullptr, q->dtype == FB_BF16, duq != nullptr, maps, p, s);
  note_launch(2);
  return e == cudaSuccess ? FB_OK : cuda_fail(e, "bwd_sm100");
}

int fb_bwd_preprocess(const fb_tensor* o, const fb_tensor* dout, fb_tensor* delta, void* stream) {
  if (!o || !dout || !delta) return fail(FB_EVALUE, "null tensor");
  cudaError_t e = launch_bwd_preprocess(to_t4(o), to_t4(dout), to_t4(delta), reinterpret_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? FB_OK : cuda_fail(e, "bwd_preprocess");
}

int fb_prepare_factors(const fb_tensor* f, int side, int split, float premul, fb_tensor* out, void* stream) {
  if (!f || !out) return fail(FB_EVALUE, "null tensor");
  if (split < 1 || split > 3) return fail(FB_EVALUE, "split must be 1, 2 or 3");
  if (side != 0 && side != 1) return fail(FB_EVALUE, "side must be 0 (query) or 1 (key)");
  if (out->dtype != FB_BF16 && out->dtype != FB_F16) return fail(FB_EVALUE, "panels are bf16/f16");
  if (f->shape[3] < 1) return fail(FB_ESHAPE, "factored bias requires rank >= 1");
  if (out->shape[3] < fb_factor_cols(f->shape[3], split)) return fail(FB_ESHAPE, "panel too narrow");
  if (out->shape[2] != f->shape[2]) return fail(FB_ESHAPE, "panel rows differ from factor rows");
  cudaError_t e = launch_prepare_factors(to_t4(f), side, split, premul, to_t4(out), reinterpret_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? FB_OK : cuda_fail(e, "prepare_factors");
}

int fb_prepare_factor_pair(const fb_tensor* fq, const fb_tensor* fk, int split, float premul, fb_tensor* uq,
                           fb_tensor* uk, void* stream) {
  if (!fq || !fk || !uq || !uk) return fail(FB_EVALUE, "null tensor");
  if (split < 1 || split > 3) return fail(FB_EVALUE, "split must be 1, 2 or 3");
  if (uq->dtype != FB_BF16 && uq->dtype != FB_F16) return fail(FB_EVALUE, "panels are bf16/f16");
  if (fq->shape[3] < 1 || fq->shape[3] != fk->shape[3]) return fail(FB_ESHAPE, "factor ranks differ or are < 1");
  for (int side = 0; side < 2; ++side) {
    const fb_tensor* f = side ? fk : fq;
    const fb_tensor* o = side ? uk : uq;
    if (o->shape[3] < fb_factor_cols(f->shape[3], split)) return fail(FB_ESHAPE, "panel too narrow");
    if (o->shape[2] != f->shape[2]) return fail(FB_ESHAPE, "panel rows differ from factor rows");
    if (o->dtype != uq->dtype) return fail(FB_EVALUE, "uq and uk dtypes differ");
  }
  cudaError_t e = launch_prepare_factor_pair(to_t4(fq), to_t4(fk), split, premul, to_t4(uq), to_t4(uk),
                                             reinterpret_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? FB_OK : cuda_fail(e, "prepare_factor_pair");
}

int fb_mlp_factor_panels(const fb_tensor* x, const fb_tensor* w1, const fb_tensor* b1, const fb_tensor* w2,
                         const fb_tensor* b2, const fb_tensor* w3, const fb_tensor* b3, int side, int split,
                         float premul, fb_tensor* out, fb_tensor* factors, void* stream) {
  if (!x || !w1 || !b1 || !w2 || !b2 || !w3 || !b3 || !out) return fail(FB_EVALUE, "null tensor");
  for (const fb_tensor* t : {x, w1, b1, w2, b2, w3, b3})
    if (t->dtype != FB_F32) return fail(FB_EVALUE, "MLP inputs and weights are fp32");
  if (split < 1 || split > 3) return fail(FB_EVALUE, "split must be 1, 2 or 3");
  if (side != 0 && side != 1) return fail(FB_EVALUE, "side must be 0 (query) or 1 (key)");
  if (out->dtype != FB_BF16 && out->dtype != FB_F16) return fail(FB_EVALUE, "panels are bf16/f16");
  const int64_t L = x->shape[2], in = x->shape[3], hid = w1->shape[3], R = w3->shape[3];
  if (in < 1 || in > 8) return fail(FB_ECONFIG, "MLP input dim must be 1..8");
  if (hid < 1 || hid > 1024 || R < 1 || R > 128) return fail(FB_ECONFIG, "hidden <= 1024 and rank <= 128");
  if (w1->shape[2] != in || w2->shape[2] != hid || w2->shape[3] != hid || w3->shape[2] != hid ||
      b1->shape[3] != hid || b2->shape[3] != hid || b3->shape[3] != R)
    return fail(FB_ESHAPE, "MLP weight shapes do not chain: [in,h] [h,h] [h,R]");
  for (const fb_tensor* t : {w1, b1, w2, b2, w3, b3})
    if (t->stride[3] != 1 || (t->shape[2] > 1 && t->stride[2] != t->shape[3]))
      return fail(FB_ESHAPE, "MLP weights must be contiguous row-major");
  if (x->stride[3] != 1) return fail(FB_ESHAPE, "x rows must be contiguous");
  if (out->shape[2] != L || out->shape[3] < fb_factor_cols(R, split) || out->stride[3] != 1)
    return fail(FB_ESHAPE, "panel must be [L, >= fb_factor_cols(R, split)] with contiguous rows");
  if (factors && (factors->dtype != FB_F32 || factors->shape[2] != L || factors->shape[3] != R ||
                  factors->stride[3] != 1 || factors->stride[2] != R))
    return fail(FB_ESHAPE, "factors output must be contiguous fp32 [L, R]");
  MlpParams p{};
  p.x = static_cast<const float*>(x->data); p.x_stride = x->stride[2];
  p.L = (int)L; p.in_dim = (int)in; p.hidden = (int)hid; p.R = (int)R;
  p.w1 = static_cast<const float*>(w1->data); p.b1 = static_cast<const float*>(b1->data);
  p.w2 = static_cast<const float*>(w2->data); p.b2 = static_cast<const float*>(b2->data);
  p.w3 = static_cast<const float*>(w3->data); p.b3 = static_cast<const float*>(b3->data);
  p.side = side; p.split = split; p.rpad = (int)out->shape[3]; p.out_dtype = out->dtype;
  p.premul = side == 0 ? premul : 1.0f;
  p.out = out->data; p.out_stride = out->stride[2];
  p.factors_out = factors ? static_cast<float*>(factors->data) : nullptr;
  cudaError_t e = launch_mlp_panels(p, reinterpret_cast<cudaStream_t>(stream));
  note_launch();
  return e == cudaSuccess ? FB_OK : cuda_fail(e, "mlp_factor_panels");
}

int fb_fold_factor_grads(const fb_tensor* dpanel, int side, int split, float postmul, fb_tensor* out, void* stream) {
  if (!dpanel || !out) return fail(FB_EVALUE, "null tensor");
  if (split < 1 || split > 3) return fail(FB_EVALUE, "split must be 1, 2 or 3");
  if (dpanel->shape[3] < fb_factor_cols(out->shape[3], split)) return fail(FB_ESHAPE, "panel too narrow");
  cudaError_t e = launch_fold_factor_grads(to_t4(dpanel), side, split, postmul, to_t4(out), reinterpret_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? FB_OK : cuda_fail(e, "fold_factor_grads");
}

int fb_factor_alibi(const float* slopes, int64_t heads, int64_t n, int64_t m, fb_tensor* fq, fb_tensor* fk, void* stream) {
  if (n < 1 || m < 1) return fail(FB_EVALUE, "decompose_alibi requires n, m >= 1");
  if (!slopes || !fq || !fk) return fail(FB_EVALUE, "null argument");
  if (fq->shape[2] != n || fk->shape[2] != m || fq->shape[3] != 2 || fk->shape[3] != 2 || fq->shape[1] != heads)
    return fail(FB_ESHAPE, "alibi factor outputs must be [1,H,N,2] / [1,H,M,2]");
  cudaError_t e = launch_factor_alibi(slopes, heads, n, m, to_t4(fq), to_t4(fk), reinterpret_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? FB_OK : cuda_fail(e, "factor_alibi");
}

int fb_factor_spatial(const fb_tensor* pos_q, const fb_tensor* pos_k, const fb_tensor* w, fb_tensor* fq, fb_tensor* fk,
                      void* stream) {
  if (!pos_q || !pos_k || !fq || !fk) return fail(FB_EVALUE, "null argument");
  if (pos_q->shape[3] != 3 || pos_k->shape[3] != 3) return fail(FB_ESHAPE, "decompose_spatial requires N x 3 positions");
  if (fq->shape[3] != 9 || fk->shape[3] != 9) return fail(FB_ESHAPE, "spatial factors have rank 9");
  if (w && w->shape[3] != pos_q->shape[2]) return fail(FB_ESHAPE, "row_weights length must equal pos_q rows");
  Tensor4 tw = w ? to_t4(w) : Tensor4{};
  cudaError_t e = launch_factor_spatial(to_t4(pos_q), to_t4(pos_k), w ? &tw : nullptr, to_t4(fq), to_t4(fk),
                                        reinterpret_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? FB_OK : cuda_fail(e, "factor_spatial");
}

int fb_dense_from_factors(const fb_tensor* fq, const fb_tensor* fk, fb_tensor* out, void* stream) {
  if (!fq || !fk || !out) return fail(FB_EVALUE, "null argument");
  if (fq->shape[3] != fk->shape[3]) return fail(FB_ESHAPE, "factor ranks differ");
  if (fq->shape[3] > 64) return fail(FB_ECONFIG, "rank > 64 not supported");
  if (out->shape[2] != fq->shape[2] || out->shape[3] != fk->shape[2]) return fail(FB_ESHAPE, "output shape mismatch");
  cudaError_t e = launch_dense_from_factors(to_t4(fq), to_t4(fk), to_t4(out), reinterpret_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? FB_OK : cuda_fail(e, "dense_from_factors");
}

}  // extern "C"
