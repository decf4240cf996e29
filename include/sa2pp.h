/* sa2pp.h -- C ABI of the B200 (sm_100a) SageAttention2++ quantized attention forward.
 *
 * Drop-in boundary for the reference operator
 *     lpattn.attention.attention_quantized(q, k, v, config) -> RunReport
 *     (/root/reference/pkg/src/lpattn/attention.py:232-316)
 * and for the north-star API  sageattn(q, k, v, tensor_layout, is_causal, sm_scale).
 *
 * Plain C: device pointers, sizes, element strides, a caller-owned CUDA stream.
 * No torch or C++ types cross this boundary, no exceptions, no allocation (except
 * the host-pipeline handle, which owns its buffers and streams), no host synchronisation.  Every entry point returns an sa2pp_status; the text of
 * the last failure on the calling thread is available from sa2pp_last_error().
 *
 * Mapping onto the reference (file:line of the code each entry point replaces):
 *   sa2pp_prepass   smooth_q / smooth_k / _pad_keys / quantize_int_block /
 *                   quantize_v_per_channel and the q_mean bias GEMV
 *                   (attention.py:259-281, 288-289; quantization.py:124-188)
 *   sa2pp_attn_fwd  the tile loop: INT8 QK^T, online softmax, P quantisation,
 *                   FP8 PV with FP16 (or FP32) accumulation, promotion, 1/l
 *                   (attention.py:279-305; mma.py:116-181)
 *   sa2pp_sageattn  both of the above: attention_quantized (attention.py:232)
 *   sa2pp_host_pipeline_*  the same operator on host arrays, PCIe overlapped
 *                   (attention_quantized's numpy-in / numpy-out contract)
 *   sa2pp_problem   AttentionConfig + RangeConfig (attention.py:58-95,
 *                   quantization.py:33-68)
 */
#ifndef SA2PP_H_
#define SA2PP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SA2PP_VERSION 100 /* 1.0.0 */

#if defined(__GNUC__)
#define SA2PP_API __attribute__((visibility("default")))
#else
#define SA2PP_API
#endif

typedef enum {
  SA2PP_OK = 0,
  SA2PP_ERR_INVALID = 1,     /* bad shape, stride, pointer or config (reference: ValueError) */
  SA2PP_ERR_UNSUPPORTED = 2, /* valid for the reference but not built here (head_dim > 128) */
  SA2PP_ERR_RANGE = 3,       /* p_r * v_r above 2047/depth without waiver (RangeConfigError) */
  SA2PP_ERR_CUDA = 4         /* a CUDA runtime/driver call failed */
} sa2pp_status;

typedef enum { SA2PP_F32 = 0, SA2PP_F16 = 1, SA2PP_BF16 = 2 } sa2pp_dtype;
typedef enum { SA2PP_ACC_F16 = 0, SA2PP_ACC_F32 = 1 } sa2pp_accum;

/* Problem + pipeline knobs.  Tile sizes are fixed at the reference defaults
 * block_q = 128, block_k = 64 (attention.py:62-63). */
typedef struct {
  int32_t batch;
  int32_t heads_q;
  int32_t heads_kv;       /* heads_q % heads_kv == 0 (GQA); == heads_q for MHA */
  int32_t seq_len;        /* >= 1, any value (ragged tails handled as the reference pads) */
  int32_t head_dim;       /* 32, 64, 96 or 128 (32 / 96 run the 64 / 128 kernels on zero-padded channels) */
  int32_t causal;         /* 0 / 1 */
  int32_t smoothing;      /* 0 / 1  (attention.py:66, default 1) */
  int32_t qk_bits;        /* 8 (default) or 4: INT4 codes carried in INT8 containers */
  int32_t pv_accum;       /* sa2pp_accum: FP16 (default, SageAttention2++) or FP32 */
  int32_t buffering_depth;/* 2 (default): the two k=32 group sums of a 64-key block combine in FP16 */
  int32_t expect_overflow;/* waiver for unsafe range pairs (quantization.py:47) */
  double sm_scale;        /* NaN selects 1/sqrt(head_dim) (attention.py:87-91); any finite value is used as given */
  double p_r;             /* default 224.0 */
  double v_r;             /* default 4.5   */
} sa2pp_problem;

/* Q/K/V on the device.  Element strides for (batch, head, token); the channel
 * dimension must be contiguous.  HND = [B,H,N,D], NHD = [B,N,H,D] are both just
 * strides here.  K and V have heads_kv heads. */
typedef struct {
  sa2pp_dtype dtype;
  const void* q;
  const void* k;
  const void* v;
  int64_t q_stride[3];
  int64_t k_stride[3];
  int64_t v_stride[3];
} sa2pp_inputs;

/* Quantized tensors written by sa2pp_prepass and read by sa2pp_attn_fwd.  Caller-owned
 * device buffers, sizes from sa2pp_quant_sizes().  Layouts (row-major):
 *   q_codes   int8    [B, Hq,  Nq_pad, D]      Nq_pad = ceil(N/128)*128, pad rows are 0
 *   q_scale   f32     [B, Hq,  nQT]            nQT = ceil(N/128); q_scale64 is the FP64 twin
 *   k_codes   int8    [B, Hkv, Np, D]          Np = ceil(N/64)*64
 *   v_codes   uint8   [B, Hkv, D, Np]          E4M3, transposed (channel-major)
 *   kv_meta   f32     [B, Hkv, nKB, 4 + D]     {dK, 0, 0, 0, dV[0..D)} per 64-key block
 *   kv_scale64 f64    [B, Hkv, nKB, 1 + D]     {dK, dV[0..D)} in FP64
 *   bias      f32     [B, Hq,  Np]             q_mean . Ks_j  (0 without smoothing)
 *   bias_l2   f32     [B, Hq,  Np]             bias * sm_scale * log2(e)
 *   means     f64     [B, Hq + Hkv, D]         q_mean (first Hq heads) then k_mean
 */
typedef struct {
  int8_t* q_codes;
  float* q_scale;
  double* q_scale64;
  int8_t* k_codes;
  uint8_t* v_codes;
  float* kv_meta;
  double* kv_scale64;
  float* bias;
  float* bias_l2;
  double* means;
} sa2pp_quant;

typedef struct {
  size_t q_codes, q_scale, q_scale64, k_codes, v_codes, kv_meta, kv_scale64, bias, bias_l2, means;
  size_t workspace; /* prepass scratch for the parallel exact channel means; a smaller or NULL workspace
                       selects the sequential mean kernel (same bits, slower) */
} sa2pp_quant_sizes_t;

/* Output [.., D] with element strides for (batch, head, token), same dtype choices as inputs. */
typedef struct {
  sa2pp_dtype dtype;
  void* o;
  int64_t o_stride[3];
} sa2pp_output;

/* Optional run report, device-resident (attention.py:114-125 RunReport analogue).
 * Pass NULL to skip.  Initialise it with sa2pp_report_init (or: overflow 0, p_scale_min_bits
 * 0x7f800000, p_scale_max_bits 0, v_scale_min_bits 0x7ff0000000000000, v_scale_max_bits 0) before the
 * first call; the kernels accumulate into it, so one report can span several calls. */
typedef struct {
  uint32_t overflow_events;   /* non-finite FP16 partials seen at promotion */
  uint32_t p_scale_min_bits;  /* float bits of min / max delta_P over all (query tile, key block) */
  uint32_t p_scale_max_bits;
  uint32_t reserved;
  uint64_t v_scale_min_bits;  /* double bits of min / max delta_V over all (key block, channel) */
  uint64_t v_scale_max_bits;
} sa2pp_report;

/* Host-side run report of a host-pipeline call: the reference's RunReport fields
 * (attention.py:114-125).  Conversions and MMA invocations are the reference's analytic counts
 * (mma.py:67-86); the rest are measured on the device. */
typedef struct {
  uint64_t overflow_events;
  uint64_t fp16_to_fp32_conversions;
  uint64_t mma_invocations;
  double p_scale_min, p_scale_max;
  double v_scale_min, v_scale_max;
} sa2pp_run_report;

SA2PP_API int sa2pp_version(void);
/* Reference-exact counters of one call (attention_quantized's fp16_to_fp32_conversions and
 * mma_invocations, mma.py:67-86), host-only arithmetic. */
SA2PP_API int sa2pp_analytic_counts(const sa2pp_problem* prob, uint64_t* conversions, uint64_t* mma_invocations);
/* Write the initial values of a device sa2pp_report (stream-ordered). */
SA2PP_API int sa2pp_report_init(sa2pp_report* report, void* cuda_stream);
SA2PP_API const char* sa2pp_last_error(void);

/* Validate the problem (shapes, head_dim, range rule).  No device work. */
SA2PP_API int sa2pp_check_problem(const sa2pp_problem* prob);

/* Byte sizes of every sa2pp_quant buffer and of the prepass workspace. */
SA2PP_API int sa2pp_quant_sizes(const sa2pp_problem* prob, sa2pp_quant_sizes_t* sizes);

/* Smoothing + quantization (HBM-bound kernels).  Stream-ordered. */
SA2PP_API int sa2pp_prepass(const sa2pp_problem* prob, const sa2pp_inputs* in, const sa2pp_quant* qt, void* workspace,
                  size_t workspace_bytes, void* cuda_stream);

/* The tcgen05 attention kernel over prepass outputs.  Stream-ordered. */
SA2PP_API int sa2pp_attn_fwd(const sa2pp_problem* prob, const sa2pp_quant* qt, const sa2pp_output* out,
                   sa2pp_report* report, void* cuda_stream);

/* Prepass + attention in one call: the attention_quantized / sageattn operator. */
/* sa2pp_attn_fwd over a contiguous range of query tiles only: units u in [unit_begin,
 * unit_begin + unit_count) of the flattened u = (b * heads_q + h) * ceil(N/128) + tile index; output
 * rows of other tiles are left untouched.  The quantized tensors must cover every head the range
 * touches (sa2pp_prepass of the whole problem).  This is the (b, h, q-tile) sharding unit of the
 * multi-GPU layout; sa2pp_attn_fwd is the full range. */
SA2PP_API int sa2pp_attn_fwd_units(const sa2pp_problem* prob, const sa2pp_quant* qt, const sa2pp_output* out,
                                   sa2pp_report* report, int64_t unit_begin, int64_t unit_count, void* stream);

SA2PP_API int sa2pp_sageattn(const sa2pp_problem* prob, const sa2pp_inputs* in, const sa2pp_quant* qt, void* workspace,
                   size_t workspace_bytes, const sa2pp_output* out, sa2pp_report* report, void* cuda_stream);

/* Host-memory operator (reference: attention_quantized takes and returns host arrays,
 * attention.py:232-316).  Q [B,Hq,N,D], K and V [B,Hkv,N,D], O [B,Hq,N,D], contiguous HND host
 * memory in `dtype` (pinned memory for full PCIe overlap; pageable works, serialised).
 * The (batch, kv-head) units are cut into `chunks` and pipelined through `depth` device buffer
 * sets: upload, sa2pp_sageattn and download of successive chunks overlap on three internal
 * streams, and the ring carries over between calls so back-to-back calls overlap as well.
 * This is the one entry point that owns device memory and streams (allocated at create).
 *
 * run() only enqueues.  The host inputs must be ready when it is called and stay unmodified,
 * and O is complete, once `cuda_stream` (made to wait for the last download) reaches the point
 * after the call.  The uploads do not wait for earlier work on `cuda_stream`. */
typedef struct sa2pp_host_pipeline sa2pp_host_pipeline;
SA2PP_API int sa2pp_host_pipeline_create(const sa2pp_problem* prob, int dtype, int chunks, int depth,
                                         sa2pp_host_pipeline** out);
SA2PP_API int sa2pp_host_pipeline_run(sa2pp_host_pipeline* hp, const void* q, const void* k, const void* v, void* o,
                                      void* cuda_stream);
/* The same computation with the instrumented kernels, blocking until O is in host memory, filling
 * `report` (attention_quantized's RunReport).  Slower than run(): for parity and accounting. */
SA2PP_API int sa2pp_host_pipeline_run_report(sa2pp_host_pipeline* hp, const void* q, const void* k, const void* v,
                                             void* o, sa2pp_run_report* report);
/* Block the calling host thread until every call issued on `hp` has landed in host memory
 * (for callers without a CUDA stream of their own, e.g. a numpy binding). */
SA2PP_API int sa2pp_host_pipeline_sync(sa2pp_host_pipeline* hp);
SA2PP_API int sa2pp_host_pipeline_destroy(sa2pp_host_pipeline* hp);

/* Debug/introspection: dump raw TMEM of the first block of CTA 0 (S int32 [128,64] and
 * the promoted-before-scaling PV words [128,D]) into `dbg` (device, >= 128*(64+D)*4 bytes).
 * Set to NULL to disable.  Used by the parity tests to localise failures. */
SA2PP_API int sa2pp_set_debug_buffer(void* dbg);

/* Development aid: per-phase clock64 trace of the CTAs of (batch 0, head 0) with query tile < 8,
 * written as uint64 [8][66][8] (see tools/trace_phases.py).  NULL disables. */
SA2PP_API int sa2pp_set_trace_buffer(void* buf);

#ifdef __cplusplus
}
#endif

#endif /* SA2PP_H_ */
