// Internal launch descriptors shared by the C-ABI layer and the kernels.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>

#include "../../include/sa2pp.h"

namespace sa2pp {

constexpr int kBlockQ = 128;  // attention.py:62
constexpr int kBlockK = 64;   // attention.py:63

// Record the calling thread's last error (sa2pp_last_error) and return `code`.
int set_error(int code, const char* fmt, ...);

// One-time per-device setup (cudaFuncSetAttribute and occupancy queries apply to one device's
// context): `run(f)` calls f once per device ordinal and caches success; concurrent first calls may
// both run f, which is idempotent.
struct PerDevice {
  std::atomic<uint64_t> done{0};
  std::atomic<int> value[64] = {};
  template <class F>
  cudaError_t run(F&& f) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    e = f(value[dev & 63]);
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
    return e;
  }
  int get() const {
    int dev = 0;
    cudaGetDevice(&dev);
    return value[dev & 63].load(std::memory_order_relaxed);
  }
};

// Head dims 32 and 96 run the 64 / 128 kernels on zero-padded channels: the loaders read d_in
// channels and supply zeros for the rest, which leaves every scale, code, bias and output channel
// of the real ones unchanged (per-block amax over zeros, per-channel V scales, independent PV columns).
__host__ __device__ constexpr int padded_dim(int d) { return d <= 64 ? 64 : 128; }

// workspace of the parallel exact channel means: per (b, head, 512-row chunk, channel) an FP64 sum and
// a 64-bit (max |x|, min exponent) word, plus one flag per (b, head)
constexpr int kMeansRows = 512;
inline size_t means_ws_bytes(int64_t B, int64_t Ht, int64_t N, int64_t D) {
  const int64_t n_ch = (N + kMeansRows - 1) / kMeansRows;
  return static_cast<size_t>(B * Ht * n_ch * D * 16 + B * Ht * 4);
}

struct PrepassLaunch {
  int d_in;  // channels present in the inputs (head_dim); D is the padded kernel width
  int dtype, D, B, Hq, Hkv, N, Nq_pad, Np, n_qt, n_kb, qmax, smoothing;
  double v_r, sm_scale_log2;
  const void *q, *k, *v;
  int64_t q_stride[3], k_stride[3], v_stride[3];
  double* means;
  void* ws_means;  // workspace for the parallel exact means (means_ws_bytes), or null: sequential only
  int8_t* q_codes;
  float* q_scale;
  double* q_scale64;
  int8_t* k_codes;
  uint8_t* v_codes;
  float* kv_meta;
  double* kv_scale64;
  float* bias;
  float* bias_l2;
};

struct AttnParams {
  int B, Hq, Hkv, N, Nq_pad, Np, n_qt, n_kb, group;
  int out_dtype;
  float sm_scale_log2;  // sm_scale * log2(e)
  float log2_pr;        // log2(p_r)
  float inv_pr;         // 1 / p_r
  const float* q_scale;
  const float* kv_meta;
  const float* bias_l2;
  void* out;
  int64_t o_sb, o_sh, o_sn;
  int d_out;  // channels written to out (head_dim <= the kernel's D)
  sa2pp_report* report;
  uint32_t* debug;
  unsigned long long* trace;  // optional per-phase clock trace of a few CTAs (development aid)
  // query tiles [unit0, unit0 + units) of the flattened (b * Hq + h) * n_qt + qt space (one CTA each)
  int unit0, units, head0;  // head0 = unit0 / n_qt
  int tile_major;           // causal grid order: 1 = (heads, tiles), all heads' heaviest tiles first
};

cudaError_t launch_prepass(const PrepassLaunch& L, cudaStream_t st);
cudaError_t launch_attn_ws(const sa2pp_problem& prob, const AttnParams& P, const sa2pp_quant& qt, cudaStream_t st);
cudaError_t launch_report_init(sa2pp_report* r, cudaStream_t st);
// min/max of the FP64 V scales [blocks][1 + D] (column 0 is dK) over the first d channels into
// report->v_scale_{min,max}_bits
cudaError_t launch_vscale_minmax(const double* kv_scale64, int64_t blocks, int D, int d, sa2pp_report* r,
                                 cudaStream_t st);

// 2-D uint8 TMA map (inner extent `inner` bytes, `rows` rows of `row_bytes`), box box_inner x box_rows.
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn get_encode_fn();
bool make_map_2d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t rows, uint64_t row_bytes,
                 uint32_t box_inner, uint32_t box_rows, CUtensorMapSwizzle sw);

}  // namespace sa2pp
