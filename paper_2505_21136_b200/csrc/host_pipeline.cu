// Host-memory operator (include/sa2pp.h, sa2pp_host_pipeline_*): the reference's
// attention_quantized takes host arrays and returns a host array (lpattn attention.py:232-316);
// this is the same contract on B200 with the PCIe traffic hidden behind the kernels.
//
// The (batch, kv-head) units are cut into chunks of whole GQA groups -- each chunk is an independent
// attention problem because the smoothing statistics are per head -- and chunk i's host->device
// copy, prepass + attention and device->host copy run on three streams through a ring of `depth`
// device buffer sets.  The ring position persists across calls, so consecutive calls overlap too:
// the next call's first upload only waits for its buffer set to drain, not for the previous
// call's last download.  For a bandwidth-bound step (PCIe Gen5 ~55 GB/s each way against ~7 TB/s
// of HBM) the upload stream therefore never idles.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

#include "sa2pp_internal.h"

struct sa2pp_host_pipeline {
  sa2pp_problem full{};   // the whole call's problem (for the analytic RunReport counters)
  sa2pp_problem chunk{};  // one chunk's problem: batch 1, cu*group query heads, cu kv heads
  int dtype = 0, es = 2, group = 1, units = 0, cu = 1, n_chunks = 0, depth = 1, device = 0;
  size_t q_unit = 0, kv_unit = 0;  // bytes of one unit of Q (group heads) / of K or V (one head)
  struct Set {
    char *q, *k, *v, *o;
    sa2pp_quant qt;
    void* ws;
    size_t ws_bytes;
  };
  std::vector<Set> sets;
  void* mem = nullptr;
  sa2pp_report* report = nullptr;  // device report shared by the chunks of a run_report call
  cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
  std::vector<cudaEvent_t> ev_in, ev_comp, ev_out;
  cudaEvent_t done = nullptr;
  long long ring = 0;  // chunks issued over the handle's lifetime; buffer set = ring % depth
};
// A handle is not thread-safe: one host thread issues its calls (the ring index is unsynchronised).
// Copies use cudaMemcpyDefault (UVA), so device-resident inputs/outputs also work (as D2D copies).

namespace {

size_t round_up(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

void release(sa2pp_host_pipeline* hp) {
  if (!hp) return;
  if (hp->h2d) cudaStreamSynchronize(hp->h2d);
  if (hp->comp) cudaStreamSynchronize(hp->comp);
  if (hp->d2h) cudaStreamSynchronize(hp->d2h);
  for (auto* v : {&hp->ev_in, &hp->ev_comp, &hp->ev_out})
    for (cudaEvent_t e : *v)
      if (e) cudaEventDestroy(e);
  if (hp->done) cudaEventDestroy(hp->done);
  for (cudaStream_t s : {hp->h2d, hp->comp, hp->d2h})
    if (s) cudaStreamDestroy(s);
  if (hp->mem) cudaFree(hp->mem);
  delete hp;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    int cur = 0;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != dev && cudaSetDevice(dev) == cudaSuccess) prev = cur;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace

extern "C" {

int sa2pp_host_pipeline_create(const sa2pp_problem* prob, int dtype, int chunks, int depth,
                               sa2pp_host_pipeline** out) {
  if (!out) return sa2pp::set_error(SA2PP_ERR_INVALID, "out handle is NULL");
  *out = nullptr;
  int rc = sa2pp_check_problem(prob);
  if (rc) return rc;
  if (dtype != SA2PP_F32 && dtype != SA2PP_F16 && dtype != SA2PP_BF16)
    return sa2pp::set_error(SA2PP_ERR_INVALID, "dtype must be f32, f16 or bf16");
  if (chunks < 1 || depth < 1) return sa2pp::set_error(SA2PP_ERR_INVALID, "chunks and depth must be >= 1");
  auto* hp = new sa2pp_host_pipeline();
  hp->dtype = dtype;
  hp->es = dtype == SA2PP_F32 ? 4 : 2;
  hp->group = prob->heads_q / prob->heads_kv;
  hp->units = prob->batch * prob->heads_kv;
  hp->cu = (hp->units + std::min(chunks, hp->units) - 1) / std::min(chunks, hp->units);
  hp->n_chunks = (hp->units + hp->cu - 1) / hp->cu;
  hp->depth = std::min(depth, hp->n_chunks);
  hp->kv_unit = static_cast<size_t>(prob->seq_len) * prob->head_dim * hp->es;
  hp->q_unit = hp->kv_unit * hp->group;
  hp->full = *prob;
  hp->chunk = *prob;
  hp->chunk.batch = 1;
  hp->chunk.heads_q = hp->cu * hp->group;
  hp->chunk.heads_kv = hp->cu;
  cudaGetDevice(&hp->device);

  sa2pp_quant_sizes_t qs;
  if ((rc = sa2pp_quant_sizes(&hp->chunk, &qs))) {
    release(hp);
    return rc;
  }
  const size_t qsz[] = {qs.q_codes, qs.q_scale, qs.q_scale64, qs.k_codes, qs.v_codes,
                        qs.kv_meta, qs.kv_scale64, qs.bias, qs.bias_l2, qs.means};
  size_t per_set = 2 * round_up(hp->cu * hp->q_unit) + 2 * round_up(hp->cu * hp->kv_unit) + round_up(qs.workspace);
  for (size_t b : qsz) per_set += round_up(b);
  cudaError_t e = cudaMalloc(&hp->mem, per_set * hp->depth + round_up(sizeof(sa2pp_report)));
  if (e != cudaSuccess) {
    release(hp);
    return sa2pp::set_error(SA2PP_ERR_CUDA, "host pipeline: cudaMalloc(%zu): %s", per_set * hp->depth,
                            cudaGetErrorString(e));
  }
  char* p = static_cast<char*>(hp->mem);
  auto take = [&](size_t bytes) {
    char* r = p;
    p += round_up(bytes);
    return r;
  };
  for (int s = 0; s < hp->depth; ++s) {
    sa2pp_host_pipeline::Set S{};
    S.q = take(hp->cu * hp->q_unit);
    S.o = take(hp->cu * hp->q_unit);
    S.k = take(hp->cu * hp->kv_unit);
    S.v = take(hp->cu * hp->kv_unit);
    S.qt.q_codes = reinterpret_cast<int8_t*>(take(qs.q_codes));
    S.qt.q_scale = reinterpret_cast<float*>(take(qs.q_scale));
    S.qt.q_scale64 = reinterpret_cast<double*>(take(qs.q_scale64));
    S.qt.k_codes = reinterpret_cast<int8_t*>(take(qs.k_codes));
    S.qt.v_codes = reinterpret_cast<uint8_t*>(take(qs.v_codes));
    S.qt.kv_meta = reinterpret_cast<float*>(take(qs.kv_meta));
    S.qt.kv_scale64 = reinterpret_cast<double*>(take(qs.kv_scale64));
    S.qt.bias = reinterpret_cast<float*>(take(qs.bias));
    S.qt.bias_l2 = reinterpret_cast<float*>(take(qs.bias_l2));
    S.qt.means = reinterpret_cast<double*>(take(qs.means));
    S.ws_bytes = qs.workspace;
    S.ws = take(qs.workspace);
    hp->sets.push_back(S);
  }
  hp->report = reinterpret_cast<sa2pp_report*>(take(sizeof(sa2pp_report)));
  for (cudaStream_t* s : {&hp->h2d, &hp->comp, &hp->d2h})
    if ((e = cudaStreamCreateWithFlags(s, cudaStreamNonBlocking)) != cudaSuccess) break;
  for (auto* v : {&hp->ev_in, &hp->ev_comp, &hp->ev_out}) {
    v->assign(hp->depth, nullptr);
    for (int s = 0; s < hp->depth && e == cudaSuccess; ++s) e = cudaEventCreateWithFlags(&(*v)[s], cudaEventDisableTiming);
  }
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&hp->done, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    release(hp);
    return sa2pp::set_error(SA2PP_ERR_CUDA, "host pipeline: stream/event creation: %s", cudaGetErrorString(e));
  }
  *out = hp;
  return SA2PP_OK;
}

}  // extern "C"

namespace {

int enqueue(sa2pp_host_pipeline* hp, const void* q, const void* k, const void* v, void* o, void* cuda_stream,
            sa2pp_report* report) {
  if (!hp) return sa2pp::set_error(SA2PP_ERR_INVALID, "host pipeline handle is NULL");
  if (!q || !k || !v || !o) return sa2pp::set_error(SA2PP_ERR_INVALID, "q, k, v and o must be host pointers");
  DeviceGuard guard(hp->device);
  const auto* qh = static_cast<const char*>(q);
  const auto* kh = static_cast<const char*>(k);
  const auto* vh = static_cast<const char*>(v);
  auto* oh = static_cast<char*>(o);
  const int64_t N = hp->chunk.seq_len, D = hp->chunk.head_dim;
  cudaError_t e = cudaSuccess;
  for (int i = 0; i < hp->n_chunks && e == cudaSuccess; ++i) {
    const int u0 = i * hp->cu, n = std::min(hp->units, u0 + hp->cu) - u0;
    const int s = static_cast<int>(hp->ring % hp->depth);
    const sa2pp_host_pipeline::Set& S = hp->sets[s];
    if (hp->ring >= hp->depth) e = cudaStreamWaitEvent(hp->h2d, hp->ev_out[s], 0);  // set s drained
    if (e == cudaSuccess) e = cudaMemcpyAsync(S.q, qh + u0 * hp->q_unit, n * hp->q_unit, cudaMemcpyDefault, hp->h2d);
    if (e == cudaSuccess) e = cudaMemcpyAsync(S.k, kh + u0 * hp->kv_unit, n * hp->kv_unit, cudaMemcpyDefault, hp->h2d);
    if (e == cudaSuccess) e = cudaMemcpyAsync(S.v, vh + u0 * hp->kv_unit, n * hp->kv_unit, cudaMemcpyDefault, hp->h2d);
    if (e == cudaSuccess) e = cudaEventRecord(hp->ev_in[s], hp->h2d);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(hp->comp, hp->ev_in[s], 0);
    if (e != cudaSuccess) break;
    sa2pp_problem pr = hp->chunk;
    pr.heads_q = n * hp->group;
    pr.heads_kv = n;
    sa2pp_inputs in{};
    in.dtype = static_cast<sa2pp_dtype>(hp->dtype);
    in.q = S.q;
    in.k = S.k;
    in.v = S.v;
    const int64_t qst[3] = {pr.heads_q * N * D, N * D, D}, kst[3] = {pr.heads_kv * N * D, N * D, D};
    for (int j = 0; j < 3; ++j) {
      in.q_stride[j] = qst[j];
      in.k_stride[j] = kst[j];
      in.v_stride[j] = kst[j];
    }
    sa2pp_output out{};
    out.dtype = static_cast<sa2pp_dtype>(hp->dtype);
    out.o = S.o;
    for (int j = 0; j < 3; ++j) out.o_stride[j] = qst[j];
    const int rc = sa2pp_sageattn(&pr, &in, &S.qt, S.ws, S.ws_bytes, &out, report, hp->comp);
    if (rc) return rc;
    e = cudaEventRecord(hp->ev_comp[s], hp->comp);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(hp->d2h, hp->ev_comp[s], 0);
    if (e == cudaSuccess) e = cudaMemcpyAsync(oh + u0 * hp->q_unit, S.o, n * hp->q_unit, cudaMemcpyDefault, hp->d2h);
    if (e == cudaSuccess) e = cudaEventRecord(hp->ev_out[s], hp->d2h);
    ++hp->ring;
  }
  if (e == cudaSuccess) e = cudaEventRecord(hp->done, hp->d2h);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(static_cast<cudaStream_t>(cuda_stream), hp->done, 0);
  if (e != cudaSuccess) return sa2pp::set_error(SA2PP_ERR_CUDA, "host pipeline: %s", cudaGetErrorString(e));
  return SA2PP_OK;
}

}  // namespace

extern "C" {

int sa2pp_host_pipeline_run(sa2pp_host_pipeline* hp, const void* q, const void* k, const void* v, void* o,
                            void* cuda_stream) {
  return enqueue(hp, q, k, v, o, cuda_stream, nullptr);
}

int sa2pp_host_pipeline_run_report(sa2pp_host_pipeline* hp, const void* q, const void* k, const void* v, void* o,
                                   sa2pp_run_report* report) {
  if (!hp) return sa2pp::set_error(SA2PP_ERR_INVALID, "host pipeline handle is NULL");
  if (!report) return sa2pp::set_error(SA2PP_ERR_INVALID, "report is NULL");
  DeviceGuard guard(hp->device);
  int rc = sa2pp_report_init(hp->report, hp->comp);  // ordered before every chunk's kernels
  if (rc) return rc;
  if ((rc = enqueue(hp, q, k, v, o, hp->comp, hp->report))) return rc;
  if ((rc = sa2pp_host_pipeline_sync(hp))) return rc;
  sa2pp_report r{};
  cudaError_t e = cudaMemcpy(&r, hp->report, sizeof(r), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return sa2pp::set_error(SA2PP_ERR_CUDA, "host pipeline report: %s", cudaGetErrorString(e));
  uint64_t conv = 0, mma = 0;
  if ((rc = sa2pp_analytic_counts(&hp->full, &conv, &mma))) return rc;
  float pmin, pmax;
  double vmin, vmax;
  std::memcpy(&pmin, &r.p_scale_min_bits, 4);
  std::memcpy(&pmax, &r.p_scale_max_bits, 4);
  std::memcpy(&vmin, &r.v_scale_min_bits, 8);
  std::memcpy(&vmax, &r.v_scale_max_bits, 8);
  report->overflow_events = r.overflow_events;
  report->fp16_to_fp32_conversions = conv;
  report->mma_invocations = mma;
  report->p_scale_min = pmin;
  report->p_scale_max = pmax;
  report->v_scale_min = vmin;
  report->v_scale_max = vmax;
  return SA2PP_OK;
}

int sa2pp_host_pipeline_sync(sa2pp_host_pipeline* hp) {
  if (!hp) return sa2pp::set_error(SA2PP_ERR_INVALID, "host pipeline handle is NULL");
  DeviceGuard guard(hp->device);
  cudaError_t e = cudaStreamSynchronize(hp->d2h);  // the last download of every issued chunk
  if (e == cudaSuccess) e = cudaStreamSynchronize(hp->comp);
  if (e != cudaSuccess) return sa2pp::set_error(SA2PP_ERR_CUDA, "host pipeline sync: %s", cudaGetErrorString(e));
  return SA2PP_OK;
}

int sa2pp_host_pipeline_destroy(sa2pp_host_pipeline* hp) {
  release(hp);
  return SA2PP_OK;
}

}  // extern "C"
