// C-ABI entry points (include/sa2pp.h): validation, buffer sizing, stream-ordered launches.
// Error behaviour mirrors the reference: shape/config problems are SA2PP_ERR_INVALID (ValueError),
// the range rule is SA2PP_ERR_RANGE (RangeConfigError, quantization.py:49-60).
#include <cuda_runtime.h>
#include <cmath>
#include <cstdio>
#include <cstdarg>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>

#include "sa2pp_internal.h"

namespace {

thread_local std::string g_last_error;
uint32_t* g_debug = nullptr;
unsigned long long* g_trace = nullptr;

int vfail(int code, const char* fmt, va_list ap) {
  char buf[512];
  vsnprintf(buf, sizeof(buf), fmt, ap);
  g_last_error = buf;
  return code;
}

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  const int rc = vfail(code, fmt, ap);
  va_end(ap);
  return rc;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(SA2PP_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

constexpr double kRangeProductLimit = 65504.0 / 32.0;  // quantization.py:26

struct Dims {
  int64_t nq_pad, np, n_qt, n_kb;
};

Dims dims_of(const sa2pp_problem& p) {
  Dims d;
  d.n_qt = (p.seq_len + 127) / 128;
  d.nq_pad = d.n_qt * 128;
  d.n_kb = (p.seq_len + 63) / 64;
  d.np = d.n_kb * 64;
  return d;
}

// NaN selects the reference default 1/sqrt(head_dim) (attention.py:87-91); any finite value,
// zero and negative included, is used as given, as AttentionConfig.softmax_scale is.
double sm_scale_of(const sa2pp_problem& p) {
  return std::isnan(p.sm_scale) ? 1.0 / std::sqrt(static_cast<double>(p.head_dim)) : p.sm_scale;
}

bool aligned16(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15u) == 0; }

}  // namespace

int sa2pp::set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  const int rc = vfail(code, fmt, ap);
  va_end(ap);
  return rc;
}

extern "C" {

int sa2pp_version(void) { return SA2PP_VERSION; }

const char* sa2pp_last_error(void) { return g_last_error.c_str(); }

int sa2pp_set_debug_buffer(void* dbg) {
  g_debug = static_cast<uint32_t*>(dbg);
  return SA2PP_OK;
}

int sa2pp_set_trace_buffer(void* buf) {
  g_trace = static_cast<unsigned long long*>(buf);
  return SA2PP_OK;
}

int sa2pp_analytic_counts(const sa2pp_problem* p, uint64_t* conversions, uint64_t* mma_invocations) {
  int rc = sa2pp_check_problem(p);
  if (rc) return rc;
  if (!conversions || !mma_invocations) return fail(SA2PP_ERR_INVALID, "output pointers must be set");
  // mma.py:67-86 as lpattn counts them per (query tile, visible key block): QK^T = rows*64 dot
  // products of ceil(D/32) k=32 MMAs, PV = rows*D of 64/32; FP16 accumulation converts each
  // output once per ceil(groups/depth) group sums (attention.py:282-303)
  const int64_t N = p->seq_len, D = p->head_dim, n_kb = (N + 63) / 64;
  uint64_t conv = 0, mma = 0;
  for (int64_t i0 = 0; i0 < N; i0 += 128) {
    const int64_t rows = std::min<int64_t>(128, N - i0);
    const int64_t stop = std::min<int64_t>(i0 + 128, N);
    const int64_t vis = p->causal ? std::min<int64_t>(n_kb, (stop + 63) / 64) : n_kb;
    mma += vis * (rows * 64 * ((D + 31) / 32) + rows * D * 2);
    if (p->pv_accum == SA2PP_ACC_F16) conv += vis * rows * D * ((2 + p->buffering_depth - 1) / p->buffering_depth);
  }
  const uint64_t heads = static_cast<uint64_t>(p->batch) * p->heads_q;
  *conversions = conv * heads;
  *mma_invocations = mma * heads;
  return SA2PP_OK;
}

int sa2pp_report_init(sa2pp_report* r, void* stream) {
  if (!r) return fail(SA2PP_ERR_INVALID, "report is NULL");
  cudaError_t e = sa2pp::launch_report_init(r, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "report init");
  return SA2PP_OK;
}

int sa2pp_check_problem(const sa2pp_problem* p) {
  if (!p) return fail(SA2PP_ERR_INVALID, "problem is NULL");
  if (p->batch < 1 || p->heads_q < 1 || p->heads_kv < 1 || p->seq_len < 1 || p->head_dim < 1)
    return fail(SA2PP_ERR_INVALID, "batch, heads, seq_len and head_dim must be positive");
  if (p->heads_q % p->heads_kv != 0)
    return fail(SA2PP_ERR_INVALID, "heads_q (%d) must be a multiple of heads_kv (%d)", p->heads_q, p->heads_kv);
  if (p->head_dim % 32 != 0)  // attention.py:242-243
    return fail(SA2PP_ERR_INVALID, "head_dim must be a multiple of 32 for the FP8 path");
  if (p->head_dim > 128)
    return fail(SA2PP_ERR_UNSUPPORTED, "head_dim %d not built (32, 64, 96, 128)", p->head_dim);
  if (p->qk_bits != 8 && p->qk_bits != 4) return fail(SA2PP_ERR_INVALID, "qk_bits must be 4 or 8");
  if (p->pv_accum != SA2PP_ACC_F16 && p->pv_accum != SA2PP_ACC_F32)
    return fail(SA2PP_ERR_INVALID, "pv_accumulator must be fp16 or fp32");
  if (p->buffering_depth != 1 && p->buffering_depth != 2)
    return fail(SA2PP_ERR_RANGE, "buffering_depth must be 1 or 2, got %d", p->buffering_depth);
  if (!(p->p_r > 0.0) || !(p->v_r > 0.0)) return fail(SA2PP_ERR_RANGE, "p_r and v_r must be positive");
  if (std::isinf(p->sm_scale)) return fail(SA2PP_ERR_INVALID, "sm_scale must be finite (NaN selects 1/sqrt(D))");
  const double bound = kRangeProductLimit / p->buffering_depth;
  if (!p->expect_overflow && p->p_r * p->v_r > bound)
    return fail(SA2PP_ERR_RANGE, "p_r*v_r = %g > %g (FP16 accumulator bound at buffering depth %d)",
                p->p_r * p->v_r, bound, p->buffering_depth);
  if (p->batch * static_cast<int64_t>(p->heads_q) > 65535)
    return fail(SA2PP_ERR_UNSUPPORTED, "batch*heads_q must be <= 65535");
  return SA2PP_OK;
}

int sa2pp_quant_sizes(const sa2pp_problem* p, sa2pp_quant_sizes_t* s) {
  int rc = sa2pp_check_problem(p);
  if (rc) return rc;
  if (!s) return fail(SA2PP_ERR_INVALID, "sizes is NULL");
  const Dims d = dims_of(*p);
  const int64_t B = p->batch, Hq = p->heads_q, Hkv = p->heads_kv, D = sa2pp::padded_dim(p->head_dim);
  s->q_codes = B * Hq * d.nq_pad * D;
  s->q_scale = B * Hq * d.n_qt * 4;
  s->q_scale64 = B * Hq * d.n_qt * 8;
  s->k_codes = B * Hkv * d.np * D;
  s->v_codes = B * Hkv * D * d.np;
  s->kv_meta = B * Hkv * d.n_kb * (4 + D) * 4;
  s->kv_scale64 = B * Hkv * d.n_kb * (1 + D) * 8;
  s->bias = B * Hq * d.np * 4;
  s->bias_l2 = B * Hq * d.np * 4;
  s->means = B * (Hq + Hkv) * D * 8;
  // the parallel exact channel means (optional: a smaller or null workspace selects the sequential kernel)
  s->workspace = sa2pp::means_ws_bytes(B, Hq + Hkv, p->seq_len, D);
  return SA2PP_OK;
}

static int check_quant(const sa2pp_quant* qt) {
  if (!qt || !qt->q_codes || !qt->q_scale || !qt->q_scale64 || !qt->k_codes || !qt->v_codes || !qt->kv_meta ||
      !qt->kv_scale64 || !qt->bias || !qt->bias_l2 || !qt->means)
    return fail(SA2PP_ERR_INVALID, "every sa2pp_quant buffer must be set");
  if (!aligned16(qt->q_codes) || !aligned16(qt->k_codes) || !aligned16(qt->v_codes) || !aligned16(qt->kv_meta) ||
      !aligned16(qt->bias_l2))
    return fail(SA2PP_ERR_INVALID, "quantized buffers must be 16-byte aligned");
  return SA2PP_OK;
}

static int check_view(const void* ptr, const int64_t st[3], int elem, const char* name) {
  if (!ptr) return fail(SA2PP_ERR_INVALID, "%s is NULL", name);
  if (!aligned16(ptr)) return fail(SA2PP_ERR_INVALID, "%s must be 16-byte aligned", name);
  for (int i = 0; i < 3; ++i)
    if (st[i] < 0 || (st[i] * elem) % 16 != 0)
      return fail(SA2PP_ERR_INVALID, "%s stride[%d]=%lld must be a non-negative multiple of 16 bytes", name, i,
                  static_cast<long long>(st[i]));
  return SA2PP_OK;
}

static int elem_size(int dt) { return dt == SA2PP_F32 ? 4 : 2; }

int sa2pp_prepass(const sa2pp_problem* p, const sa2pp_inputs* in, const sa2pp_quant* qt, void* ws, size_t ws_bytes,
                  void* stream) {
  int rc = sa2pp_check_problem(p);
  if (rc) return rc;
  if (!in) return fail(SA2PP_ERR_INVALID, "inputs is NULL");
  if (in->dtype != SA2PP_F32 && in->dtype != SA2PP_F16 && in->dtype != SA2PP_BF16)
    return fail(SA2PP_ERR_INVALID, "input dtype must be f32, f16 or bf16");
  const int es = elem_size(in->dtype);
  if ((rc = check_view(in->q, in->q_stride, es, "q")) || (rc = check_view(in->k, in->k_stride, es, "k")) ||
      (rc = check_view(in->v, in->v_stride, es, "v")) || (rc = check_quant(qt)))
    return rc;
  sa2pp_quant_sizes_t sz;
  sa2pp_quant_sizes(p, &sz);

  const Dims d = dims_of(*p);
  sa2pp::PrepassLaunch L{};
  L.dtype = in->dtype;
  L.ws_means = (ws != nullptr && ws_bytes >= sz.workspace && aligned16(ws)) ? ws : nullptr;
  L.D = sa2pp::padded_dim(p->head_dim);
  L.d_in = p->head_dim;
  L.B = p->batch;
  L.Hq = p->heads_q;
  L.Hkv = p->heads_kv;
  L.N = p->seq_len;
  L.Nq_pad = static_cast<int>(d.nq_pad);
  L.Np = static_cast<int>(d.np);
  L.n_qt = static_cast<int>(d.n_qt);
  L.n_kb = static_cast<int>(d.n_kb);
  L.qmax = (1 << (p->qk_bits - 1)) - 1;
  L.smoothing = p->smoothing ? 1 : 0;
  L.v_r = p->v_r;
  L.sm_scale_log2 = sm_scale_of(*p) * 1.4426950408889634;
  L.q = in->q;
  L.k = in->k;
  L.v = in->v;
  for (int i = 0; i < 3; ++i) {
    L.q_stride[i] = in->q_stride[i];
    L.k_stride[i] = in->k_stride[i];
    L.v_stride[i] = in->v_stride[i];
  }
  L.means = qt->means;
  L.q_codes = qt->q_codes;
  L.q_scale = qt->q_scale;
  L.q_scale64 = qt->q_scale64;
  L.k_codes = qt->k_codes;
  L.v_codes = qt->v_codes;
  L.kv_meta = qt->kv_meta;
  L.kv_scale64 = qt->kv_scale64;
  L.bias = qt->bias;
  L.bias_l2 = qt->bias_l2;
  cudaError_t e = sa2pp::launch_prepass(L, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "prepass launch");
  return SA2PP_OK;
}

int sa2pp_attn_fwd(const sa2pp_problem* p, const sa2pp_quant* qt, const sa2pp_output* out, sa2pp_report* report,
                   void* stream) {
  int rc = sa2pp_check_problem(p);
  if (rc) return rc;
  const Dims d = dims_of(*p);
  return sa2pp_attn_fwd_units(p, qt, out, report, 0, static_cast<int64_t>(p->batch) * p->heads_q * d.n_qt, stream);
}

int sa2pp_attn_fwd_units(const sa2pp_problem* p, const sa2pp_quant* qt, const sa2pp_output* out,
                         sa2pp_report* report, int64_t unit_begin, int64_t unit_count, void* stream) {
  int rc = sa2pp_check_problem(p);
  if (rc) return rc;
  if ((rc = check_quant(qt))) return rc;
  if (!out) return fail(SA2PP_ERR_INVALID, "output is NULL");
  if (out->dtype != SA2PP_F32 && out->dtype != SA2PP_F16 && out->dtype != SA2PP_BF16)
    return fail(SA2PP_ERR_INVALID, "output dtype must be f32, f16 or bf16");
  if ((rc = check_view(out->o, out->o_stride, elem_size(out->dtype), "o"))) return rc;
  const Dims d = dims_of(*p);
  sa2pp::AttnParams P{};
  P.B = p->batch;
  P.Hq = p->heads_q;
  P.Hkv = p->heads_kv;
  P.N = p->seq_len;
  P.Nq_pad = static_cast<int>(d.nq_pad);
  P.Np = static_cast<int>(d.np);
  P.n_qt = static_cast<int>(d.n_qt);
  P.n_kb = static_cast<int>(d.n_kb);
  P.group = p->heads_q / p->heads_kv;
  P.out_dtype = out->dtype;
  P.sm_scale_log2 = static_cast<float>(sm_scale_of(*p) * 1.4426950408889634);
  P.log2_pr = static_cast<float>(std::log2(p->p_r));
  P.inv_pr = static_cast<float>(1.0 / p->p_r);
  P.q_scale = qt->q_scale;
  P.kv_meta = qt->kv_meta;
  P.bias_l2 = qt->bias_l2;
  P.out = out->o;
  P.o_sb = out->o_stride[0];
  P.o_sh = out->o_stride[1];
  P.o_sn = out->o_stride[2];
  P.d_out = p->head_dim;
  P.report = report;
  P.debug = g_debug;
  P.trace = g_trace;
  const int64_t total = static_cast<int64_t>(p->batch) * p->heads_q * d.n_qt;
  if (unit_begin < 0 || unit_count < 0 || unit_begin + unit_count > total)
    return fail(SA2PP_ERR_INVALID, "query-tile units [%lld, %lld) outside [0, %lld)", static_cast<long long>(unit_begin),
                static_cast<long long>(unit_begin + unit_count), static_cast<long long>(total));
  if (total > 0x7fffffff) return fail(SA2PP_ERR_UNSUPPORTED, "more than 2^31 - 1 query tiles");
  P.unit0 = static_cast<int>(unit_begin);
  P.units = static_cast<int>(unit_count);
  P.head0 = P.unit0 / P.n_qt;
  // Causal grids in LPT (tile-major) order -- every head's heaviest query tile before any lighter one --
  // while the K/V codes stay within ~2.4x the 126 MB L2: measured +10-15 % at 1K-2K, +3-7 % at 4K-8K
  // and for Llama GQA 8K; beyond that the head-major order's K/V reuse between neighbouring CTAs wins
  // (16K D=128: 791 vs 862 TOPS tile-major vs head-major)
  const double kv_bytes = static_cast<double>(p->batch) * p->heads_kv * d.np * sa2pp::padded_dim(p->head_dim) * 2.0;
  P.tile_major = (p->causal && kv_bytes <= 300e6) ? 1 : 0;
  cudaError_t e = sa2pp::launch_attn_ws(*p, P, *qt, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "attention launch");
  if (report != nullptr) {  // v_scale min/max over every (key block, channel) (attention.py:271-275)
    e = sa2pp::launch_vscale_minmax(qt->kv_scale64, static_cast<int64_t>(p->batch) * p->heads_kv * d.n_kb,
                                    sa2pp::padded_dim(p->head_dim), p->head_dim, report, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "report launch");
  }
  return SA2PP_OK;
}

int sa2pp_sageattn(const sa2pp_problem* p, const sa2pp_inputs* in, const sa2pp_quant* qt, void* ws, size_t ws_bytes,
                   const sa2pp_output* out, sa2pp_report* report, void* stream) {
  int rc = sa2pp_prepass(p, in, qt, ws, ws_bytes, stream);
  if (rc) return rc;
  return sa2pp_attn_fwd(p, qt, out, report, stream);
}

}  // extern "C"
