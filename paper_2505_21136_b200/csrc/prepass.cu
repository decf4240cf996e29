// Fused smoothing + quantization prepass (HBM-bound), sm_100a.
//
// Reproduces, bit-exactly, the quantized tensors the reference derives before
// its tile loop (lpattn attention.py:259-281):
//   * per-(b,h) FP64 channel means of Q and K            (quantization.py:124-148)
//   * Q codes: one INT8/INT4 scale per 128-token tile   (quantization.py:151-160, attention.py:279-280)
//   * K codes: one scale per 64-token block of smoothed, zero-padded K (attention.py:265-273)
//   * V codes: E4M3, one scale per (64-token block, channel), range v_r (quantization.py:178-188)
//   * per-key bias b_j = q_mean . Ks_j                   (attention.py:288-289)
// Arithmetic is FP64 with RNE division, exactly as the reference's numpy float64.
//
// Kernels:
//   channel_sums   grid (chunks, B*(Hq+Hkv))  double-double partial sums over token chunks
//   channel_means  grid (B*(Hq+Hkv))          fixed-order reduction of the partials -> FP64 mean
//   quantize_q     grid (nQT, B*Hq)           one CTA per 128-row query tile
//   quantize_kv    grid (nKB, B*Hkv)          one CTA per 64-key block (K codes, V^T codes, scales, bias)
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>

#include "sa2pp_internal.h"

namespace sa2pp {

template <typename T>
__device__ __forceinline__ double to_f64(T x);
template <>
__device__ __forceinline__ double to_f64<float>(float x) { return static_cast<double>(x); }
template <>
__device__ __forceinline__ double to_f64<__half>(__half x) { return static_cast<double>(__half2float(x)); }
template <>
__device__ __forceinline__ double to_f64<__nv_bfloat16>(__nv_bfloat16 x) {
  return static_cast<double>(__bfloat162float(x));
}

// Error-free transformation: s + e == a + b exactly.
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}
__device__ __forceinline__ void dd_add(double& hi, double& lo, double x) {
  double s, e;
  two_sum(hi, x, s, e);
  lo += e;
  hi = s;
}

template <typename T>
__device__ __forceinline__ float to_f32(T x);
template <>
__device__ __forceinline__ float to_f32<float>(float x) { return x; }
template <>
__device__ __forceinline__ float to_f32<__half>(__half x) { return __half2float(x); }
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }

// Input element (b, h, n, c) with strides in elements; channel dim contiguous.
struct InView {
  const void* base;
  int64_t sb, sh, sn;
};

template <typename T>
__device__ __forceinline__ const T* row_ptr(const InView& v, int b, int h, int n) {
  return static_cast<const T*>(v.base) + b * v.sb + h * v.sh + static_cast<int64_t>(n) * v.sn;
}

// ------------------------------------------------------------------ pass 1: channel sums
// blockDim = 256; thread t owns channels [c8*VEC, c8*VEC+VEC) of rows t/(D/VEC) + k*stride.
template <typename T, int D>
__global__ void __launch_bounds__(256) channel_sums_kernel(InView qv, InView kv, int Hq, int Hkv, int N,
                                                           int rows_per_chunk, double2* __restrict__ partial,
                                                           int n_chunks) {
  constexpr int VEC = 16 / sizeof(T);
  constexpr int LANES_PER_ROW = D / VEC;
  constexpr int ROWS_PER_PASS = 256 / LANES_PER_ROW;
  const int chunk = blockIdx.x;
  const int bh = blockIdx.y;  // in [0, B*(Hq+Hkv))
  const int Ht = Hq + Hkv;
  const int b = bh / Ht;
  const int h = bh % Ht;
  const InView& v = (h < Hq) ? qv : kv;
  const int hh = (h < Hq) ? h : h - Hq;
  const int c8 = threadIdx.x % LANES_PER_ROW;
  const int r0 = threadIdx.x / LANES_PER_ROW;
  const int n_begin = chunk * rows_per_chunk;
  const int n_end = min(N, n_begin + rows_per_chunk);
  double hi[VEC], lo[VEC];
#pragma unroll
  for (int i = 0; i < VEC; ++i) hi[i] = lo[i] = 0.0;
  for (int n = n_begin + r0; n < n_end; n += ROWS_PER_PASS) {
    const uint4 raw = *reinterpret_cast<const uint4*>(row_ptr<T>(v, b, hh, n) + c8 * VEC);
    const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
    for (int i = 0; i < VEC; ++i) dd_add(hi[i], lo[i], to_f64<T>(e[i]));
  }
  // Fixed-order combine of the ROWS_PER_PASS row-groups through shared memory.
  __shared__ double2 red[256 * VEC];
#pragma unroll
  for (int i = 0; i < VEC; ++i) red[threadIdx.x * VEC + i] = make_double2(hi[i], lo[i]);
  __syncthreads();
  if (threadIdx.x < LANES_PER_ROW) {
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      double H = 0.0, L = 0.0;
      for (int r = 0; r < ROWS_PER_PASS; ++r) {
        const double2 p = red[(r * LANES_PER_ROW + threadIdx.x) * VEC + i];
        dd_add(H, L, p.x);
        L += p.y;
      }
      partial[(static_cast<int64_t>(bh) * n_chunks + chunk) * D + threadIdx.x * VEC + i] = make_double2(H, L);
    }
  }
}

// ------------------------------------------------------------------ pass 1b: means
template <int D>
__global__ void channel_means_kernel(const double2* __restrict__ partial, int n_chunks, int N,
                                     double* __restrict__ means) {
  const int bh = blockIdx.x;
  for (int c = threadIdx.x; c < D; c += blockDim.x) {
    double H = 0.0, L = 0.0;
    for (int k = 0; k < n_chunks; ++k) {
      const double2 p = partial[(static_cast<int64_t>(bh) * n_chunks + k) * D + c];
      dd_add(H, L, p.x);
      L += p.y;
    }
    means[static_cast<int64_t>(bh) * D + c] = (H + L) / static_cast<double>(N);
  }
}

// ------------------------------------------------------------------ shared helpers
__device__ __forceinline__ double block_max_256(double x, double* scratch) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) scratch[w] = x;
  __syncthreads();
  double m = scratch[0];
#pragma unroll
  for (int i = 1; i < 8; ++i) m = fmax(m, scratch[i]);
  return m;
}

// Direct FP64 -> E4M3 ("fn") with RNE and saturation to +-448 (numerics.py:152-182).
__device__ __forceinline__ uint8_t e4m3_from_f64(double x) {
  const uint8_t sign = signbit(x) ? 0x80 : 0x00;
  const double a = fabs(x);
  if (a >= 448.0) return sign | 0x7E;
  if (a < 0.015625) {  // below the smallest normal 2^-6: fixed step 2^-9
    const double q = rint(a * 512.0);
    return sign | static_cast<uint8_t>(q);  // q == 8 is exactly the code of 2^-6
  }
  int e = ilogb(a);  // floor(log2 a), in [-6, 8]
  double q = rint(scalbn(a, 3 - e));  // significand * 8 in [8, 16]
  if (q >= 16.0) {
    q = 8.0;
    e += 1;
  }
  return sign | static_cast<uint8_t>(((e + 7) << 3) | (static_cast<int>(q) - 8));
}

// x / scale rounded to nearest-even, bit-identical to the FP64 division the reference does
// (np.round(x / scale)): multiply by the reciprocal and fall back to the correctly rounded
// division only when the product lies within 1e-9 of a rounding tie.
__device__ __forceinline__ double div_rint(double x, double scale, double inv) {
  double q = x * inv;
  const double fr = fabs(q - trunc(q));
  if (fabs(fr - 0.5) < 1e-9) q = __ddiv_rn(x, scale);
  return rint(q);
}


// E4M3 code of x / scale, bit-identical to encoding the correctly rounded FP64 quotient: the
// reciprocal product is used unless it sits within 1e-9 (relative to the grid step) of an E4M3
// rounding boundary, in which case the exact quotient is encoded.
__device__ __forceinline__ uint8_t e4m3_div(double x, double scale, double inv) {
  double q = x * inv;
  const double a = fabs(q);
  if (a < 448.0) {
    const int e = a < 0.015625 ? -6 : ilogb(a);
    const double m = scalbn(a, 3 - e);  // grid units: ties sit at k + 0.5
    const double fr = m - trunc(m);
    if (fabs(fr - 0.5) < 1e-9) q = __ddiv_rn(x, scale);
  }
  return e4m3_from_f64(q);
}



// Branch-free halves of the fast paths: the code assuming no tie, and whether the element is near
// one.  Callers OR the flags over a batch and redo the whole batch exactly in the rare case, so the
// common path carries no per-element divergence/reconvergence.
__device__ __forceinline__ int int_code_nt(float v, float mu_hi, float mu_lo, float inv32, int qmax, bool& tie) {
  const float q = ((v - mu_hi) - mu_lo) * inv32;
  const float t = q + 12582912.0f;  // 1.5 * 2^23
  tie |= fabsf(fabsf(q - (t - 12582912.0f)) - 0.5f) < 1e-4f;
  return min(max(__float_as_int(t) - 0x4B400000, -qmax), qmax);
}
__device__ __forceinline__ int int_code_exact(float v, double mu, double scale, double inv64, int qmax) {
  return min(max(static_cast<int>(div_rint(static_cast<double>(v) - mu, scale, inv64)), -qmax), qmax);
}
__device__ __forceinline__ uint32_t e4m3_nt(float v, float inv32, bool& tie) {
  const float q = v * inv32;
  const uint32_t a = __float_as_uint(q) & 0x7FFFFFFFu;
  const uint32_t d = a & 0xFFFFFu;
  const float y = __uint_as_float(a) * 512.0f;
  tie |= a >= 0x3C800000u ? (d > 0x80000u - 64u && d < 0x80000u + 64u) : (fabsf((y - truncf(y)) - 0.5f) < 1e-4f);
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(0.0f), "f"(q));
  return r & 0xFFu;
}

// ------------------------------------------------------------------ pass 2: Q tiles
// One CTA (256 threads) per 128-row tile of one (b, hq).  Rows >= N are written as zero codes.
// amax = max over channels of max(|max_c - mu_c|, |min_c - mu_c|): fl64(v - mu) is monotone in v, so
// this is the reference's max |fl64(v - mu)| over the tile with FP64 work per channel only.
template <typename T, int D>
__global__ void __launch_bounds__(256) quantize_q_kernel(InView qv, int Hq, int N, int Nq_pad, int n_qt, int qmax,
                                                         const double* __restrict__ means, int Ht,
                                                         int8_t* __restrict__ q_codes, float* __restrict__ q_scale,
                                                         double* __restrict__ q_scale64) {
  constexpr int VEC = 16 / sizeof(T);
  constexpr int LANES_PER_ROW = D / VEC;
  constexpr int ROWS_PER_PASS = 256 / LANES_PER_ROW;
  __shared__ double scratch[8];
  const int qt = blockIdx.x;
  const int bh = blockIdx.y;
  const int b = bh / Hq, h = bh % Hq;
  const int c8 = threadIdx.x % LANES_PER_ROW;
  const int r0 = threadIdx.x / LANES_PER_ROW;
  const int n0 = qt * 128;
  const int n1 = min(N, n0 + 128);
  float mn[VEC], mx[VEC];
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    mn[i] = INFINITY;
    mx[i] = -INFINITY;
  }
  for (int n = n0 + r0; n < n1; n += ROWS_PER_PASS) {
    const uint4 raw = *reinterpret_cast<const uint4*>(row_ptr<T>(qv, b, h, n) + c8 * VEC);
    const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      const float x = to_f32<T>(e[i]);
      mn[i] = fminf(mn[i], x);
      mx[i] = fmaxf(mx[i], x);
    }
  }
  const double* mup = means + (static_cast<int64_t>(b) * Ht + h) * D + c8 * VEC;
  double amax = 0.0, mumax = 0.0;
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    const double m = mup[i];
    if (mx[i] >= mn[i])
      amax = fmax(amax, fmax(fabs(static_cast<double>(mx[i]) - m), fabs(static_cast<double>(mn[i]) - m)));
    mumax = fmax(mumax, fabs(m));
  }
  amax = block_max_256(amax, scratch);
  mumax = block_max_256(mumax, scratch);
  const double scale = amax > 0.0 ? amax / static_cast<double>(qmax) : 1.0;
  if (threadIdx.x == 0) {
    q_scale[static_cast<int64_t>(bh) * n_qt + qt] = static_cast<float>(scale);
    q_scale64[static_cast<int64_t>(bh) * n_qt + qt] = scale;
  }
  const double inv = 1.0 / scale;
  const float inv32 = static_cast<float>(inv);
  const bool fast = mumax <= 65536.0 * amax;  // the error bound of int_code_nt
  float mu_hi[VEC], mu_lo[VEC];
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    mu_hi[i] = static_cast<float>(mup[i]);
    mu_lo[i] = static_cast<float>(mup[i] - static_cast<double>(mu_hi[i]));
  }
  int8_t* dst = q_codes + (static_cast<int64_t>(bh) * Nq_pad) * D;
  for (int n = n0 + r0; n < n0 + 128; n += ROWS_PER_PASS) {
    uint32_t w[VEC / 4];
#pragma unroll
    for (int i = 0; i < VEC / 4; ++i) w[i] = 0u;
    if (n < n1) {
      const uint4 raw = *reinterpret_cast<const uint4*>(row_ptr<T>(qv, b, h, n) + c8 * VEC);
      const T* e = reinterpret_cast<const T*>(&raw);
      bool tie = !fast;
#pragma unroll
      for (int i = 0; i < VEC; ++i)
        w[i >> 2] |= (static_cast<uint32_t>(int_code_nt(to_f32<T>(e[i]), mu_hi[i], mu_lo[i], inv32, qmax, tie)) & 0xFFu)
                     << (8 * (i & 3));
      if (tie) {  // rare: near a rounding tie or |mu| >> amax -> the FP64 quotient for the batch
#pragma unroll
        for (int i = 0; i < VEC / 4; ++i) w[i] = 0u;
#pragma unroll
        for (int i = 0; i < VEC; ++i)
          w[i >> 2] |= (static_cast<uint32_t>(int_code_exact(to_f32<T>(e[i]), mup[i], scale, inv, qmax)) & 0xFFu)
                       << (8 * (i & 3));
      }
    }
    int8_t* o = dst + static_cast<int64_t>(n) * D + c8 * VEC;
    if constexpr (VEC == 8) {
      *reinterpret_cast<uint2*>(o) = make_uint2(w[0], w[1]);
    } else {
      *reinterpret_cast<uint32_t*>(o) = w[0];
    }
  }
}

// ------------------------------------------------------------------ pass 3: K/V blocks
// One CTA (256 threads) per 64-key block of one (b, hkv).  The raw K and V tiles are staged in
// shared memory once; everything else works from there.
//   k_codes  [B, Hkv, Np, D]          int8
//   v_codes  [B, Hkv, D, Np]          E4M3, transposed so the PV operand is K-major
//   kv_meta  [B, Hkv, nKB, 4 + D]     f32 {dK, 0, 0, 0, dV[0..D)}
//   bias     [B, Hq, Np]              f32 q_mean . Ks_j ; bias_l2 = bias * sm_scale * log2(e)
template <typename T, int D>
__host__ __device__ constexpr int kv_smem_bytes() {
  return 2 * 64 * D * static_cast<int>(sizeof(T)) + 3 * D * 8 + 2 * D * 4 + 64;
}

template <typename T, int D>
__global__ void __launch_bounds__(256) quantize_kv_kernel(InView kv_in, InView v_in, int Hq, int Hkv, int N, int Np,
                                                          int n_kb, int qmax, double v_r, int smoothing,
                                                          double sm_scale_log2, const double* __restrict__ means,
                                                          int Ht, int8_t* __restrict__ k_codes,
                                                          uint8_t* __restrict__ v_codes, float* __restrict__ kv_meta,
                                                          double* __restrict__ kv_scale64, float* __restrict__ bias,
                                                          float* __restrict__ bias_l2) {
  constexpr int VEC = 16 / sizeof(T);
  constexpr int NV = 64 * D / VEC;  // 16-byte vectors per tile
  extern __shared__ __align__(16) unsigned char kv_smem[];
  T* kraw = reinterpret_cast<T*>(kv_smem);
  T* vraw = kraw + 64 * D;
  double* kmu = reinterpret_cast<double*>(kv_smem + 2 * 64 * D * sizeof(T));
  double* qmu = kmu + D;
  double* vsc = qmu + D;
  float* kmu_hi = reinterpret_cast<float*>(vsc + D);
  float* kmu_lo = kmu_hi + D;
  __shared__ double scratch[8];
  const int kb = blockIdx.x;
  const int bh = blockIdx.y;
  const int b = bh / Hkv, h = bh % Hkv;
  const int n0 = kb * 64;
  const int rows = min(64, N - n0);
  const int tid = threadIdx.x;

  // ---- stage the tiles (rows past N are zero: the reference pads after smoothing)
  for (int i = tid; i < NV; i += 256) {
    const int r = i / (D / VEC), c = (i % (D / VEC)) * VEC;
    uint4 kvv = make_uint4(0, 0, 0, 0), vvv = make_uint4(0, 0, 0, 0);
    if (r < rows) {
      kvv = *reinterpret_cast<const uint4*>(row_ptr<T>(kv_in, b, h, n0 + r) + c);
      vvv = *reinterpret_cast<const uint4*>(row_ptr<T>(v_in, b, h, n0 + r) + c);
    }
    *reinterpret_cast<uint4*>(kraw + r * D + c) = kvv;
    *reinterpret_cast<uint4*>(vraw + r * D + c) = vvv;
  }
  if (tid < D) {
    const double m = means[(static_cast<int64_t>(b) * Ht + Hq + h) * D + tid];
    kmu[tid] = m;
    kmu_hi[tid] = static_cast<float>(m);
    kmu_lo[tid] = static_cast<float>(m - static_cast<double>(kmu_hi[tid]));
  }
  __syncthreads();

  // ---- K: smoothed block amax -> scale (quantization.py:151-160) from per-channel min/max
  //      (fl64(k - mu) is monotone in k: same value as the element-wise FP64 max)
  double amax = 0.0, mumax = 0.0;
  {
    constexpr int TPC = 256 / D;  // threads per channel
    const int c = tid % D;
    float mn = INFINITY, mx = -INFINITY;
    for (int r = tid / D; r < rows; r += TPC) {
      const float x = to_f32<T>(kraw[r * D + c]);
      mn = fminf(mn, x);
      mx = fmaxf(mx, x);
    }
    if (mx >= mn) amax = fmax(fabs(static_cast<double>(mx) - kmu[c]), fabs(static_cast<double>(mn) - kmu[c]));
    mumax = fabs(kmu[c]);
  }
  amax = block_max_256(amax, scratch);
  mumax = block_max_256(mumax, scratch);
  const double kscale = amax > 0.0 ? amax / static_cast<double>(qmax) : 1.0;
  const double kinv = 1.0 / kscale;
  const float kinv32 = static_cast<float>(kinv);
  const bool kfast = mumax <= 65536.0 * amax;  // the error bound of int_code_nt

  // ---- K codes: 8 consecutive channels per thread-iteration, one 8-byte store
  int8_t* kdst = k_codes + (static_cast<int64_t>(bh) * Np + n0) * D;
  for (int g = tid; g < 64 * D / 8; g += 256) {
    const int r = g / (D / 8), c = (g % (D / 8)) * 8;
    uint32_t w[2] = {0u, 0u};
    if (r < rows) {
      const uint4 raw = *reinterpret_cast<const uint4*>(kraw + r * D + c);  // 8 channels (16-bit T)
      float v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = sizeof(T) == 2 ? to_f32<T>(reinterpret_cast<const T*>(&raw)[i])
                                                         : to_f32<T>(kraw[r * D + c + i]);
      bool tie = !kfast;
#pragma unroll
      for (int i = 0; i < 8; ++i)
        w[i >> 2] |= (static_cast<uint32_t>(int_code_nt(v[i], kmu_hi[c + i], kmu_lo[c + i], kinv32, qmax, tie)) & 0xFFu)
                     << (8 * (i & 3));
      if (tie) {  // rare: near a rounding tie or |mu| >> amax -> the FP64 quotient for the batch
        w[0] = w[1] = 0u;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          w[i >> 2] |= (static_cast<uint32_t>(int_code_exact(v[i], kmu[c + i], kscale, kinv, qmax)) & 0xFFu)
                       << (8 * (i & 3));
      }
    }
    *reinterpret_cast<uint2*>(kdst + static_cast<int64_t>(r) * D + c) = make_uint2(w[0], w[1]);
  }

  // ---- V: per-channel block max -> scale (quantization.py:178-188); |x| max is exact in f32
  float* meta = kv_meta + (static_cast<int64_t>(bh) * n_kb + kb) * (4 + D);
  double* sc64 = kv_scale64 + (static_cast<int64_t>(bh) * n_kb + kb) * (1 + D);
  if (tid < D) {
    float m = 0.0f;
    for (int r = 0; r < rows; ++r) m = fmaxf(m, fabsf(to_f32<T>(vraw[r * D + tid])));
    const double sc = m > 0.0f ? static_cast<double>(m) / v_r : 1.0;
    vsc[tid] = sc;
    meta[4 + tid] = static_cast<float>(sc);
    sc64[1 + tid] = sc;
  }
  if (tid < 4) meta[tid] = tid == 0 ? static_cast<float>(kscale) : 0.0f;
  if (tid == 0) sc64[0] = kscale;
  __syncthreads();

  // ---- V codes, transposed: thread -> (channel, 32-row half); 32 codes -> two 16-byte stores
  for (int t = tid; t < D * 2; t += 256) {
    const int c = t >> 1, half = t & 1;
    const double sc = vsc[c], inv = 1.0 / sc;
    const float inv32 = static_cast<float>(inv);
    uint32_t w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) w[i] = 0u;
    bool tie = false;
#pragma unroll
    for (int i = 0; i < 32; ++i)
      w[i >> 2] |= e4m3_nt(to_f32<T>(vraw[(half * 32 + i) * D + c]), inv32, tie) << (8 * (i & 3));
    if (tie) {  // rare: some element near an E4M3 rounding tie -> the exact FP64 encoder for all 32
#pragma unroll
      for (int i = 0; i < 8; ++i) w[i] = 0u;
#pragma unroll 4
      for (int i = 0; i < 32; ++i)
        w[i >> 2] |= static_cast<uint32_t>(e4m3_div(to_f64<T>(vraw[(half * 32 + i) * D + c]), sc, inv))
                     << (8 * (i & 3));
    }
    uint8_t* vdst = v_codes + (static_cast<int64_t>(bh) * D + c) * Np + n0 + half * 32;
    *reinterpret_cast<uint4*>(vdst) = make_uint4(w[0], w[1], w[2], w[3]);
    *reinterpret_cast<uint4*>(vdst + 16) = make_uint4(w[4], w[5], w[6], w[7]);
  }

  // ---- bias for every query head sharing this KV head: b_j = q_mean . Ks_j (attention.py:288-289)
  const int group = Hq / Hkv;
  const int r = tid >> 2, qq = tid & 3;  // row, quarter of the channels
  for (int g = 0; g < group; ++g) {
    const int hq = h * group + g;
    __syncthreads();
    if (tid < D) qmu[tid] = smoothing ? means[(static_cast<int64_t>(b) * Ht + hq) * D + tid] : 0.0;
    __syncthreads();
    double acc = 0.0;
    if (r < rows) {
      double a4[4] = {0.0, 0.0, 0.0, 0.0};  // four independent FMA chains (latency)
#pragma unroll
      for (int c = 0; c < D / 4; ++c) {
        const int cc = qq * (D / 4) + c;
        a4[c & 3] = fma(qmu[cc], static_cast<double>(to_f32<T>(kraw[r * D + cc])) - kmu[cc], a4[c & 3]);
      }
      acc = (a4[0] + a4[1]) + (a4[2] + a4[3]);
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    if (qq == 0) {
      const int64_t o = (static_cast<int64_t>(b) * Hq + hq) * Np + n0 + r;
      bias[o] = static_cast<float>(acc);
      bias_l2[o] = static_cast<float>(acc * sm_scale_log2);
    }
  }
}

// ------------------------------------------------------------------ host launcher
template <typename T, int D>
static cudaError_t launch_prepass_t(const PrepassLaunch& L, cudaStream_t st) {
  InView qv{L.q, L.q_stride[0], L.q_stride[1], L.q_stride[2]};
  InView kv{L.k, L.k_stride[0], L.k_stride[1], L.k_stride[2]};
  InView vv{L.v, L.v_stride[0], L.v_stride[1], L.v_stride[2]};
  const int Ht = L.Hq + L.Hkv;
  if (L.smoothing) {
    dim3 g1(L.n_chunks, L.B * Ht);
    channel_sums_kernel<T, D><<<g1, 256, 0, st>>>(qv, kv, L.Hq, L.Hkv, L.N, L.rows_per_chunk, L.partial,
                                                  L.n_chunks);
    channel_means_kernel<D><<<L.B * Ht, 128, 0, st>>>(L.partial, L.n_chunks, L.N, L.means);
  } else {
    cudaMemsetAsync(L.means, 0, sizeof(double) * L.B * Ht * D, st);
  }
  dim3 gq(L.n_qt, L.B * L.Hq);
  quantize_q_kernel<T, D><<<gq, 256, 0, st>>>(qv, L.Hq, L.N, L.Nq_pad, L.n_qt, L.qmax, L.means, Ht, L.q_codes,
                                              L.q_scale, L.q_scale64);
  dim3 gk(L.n_kb, L.B * L.Hkv);
  constexpr int kv_smem = kv_smem_bytes<T, D>();
  static bool attr_set = false;  // per template instance; benign race (idempotent)
  if (!attr_set && kv_smem > 48 * 1024) {
    cudaFuncSetAttribute(quantize_kv_kernel<T, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, kv_smem);
  }
  attr_set = true;
  quantize_kv_kernel<T, D><<<gk, 256, kv_smem, st>>>(kv, vv, L.Hq, L.Hkv, L.N, L.Np, L.n_kb, L.qmax, L.v_r, L.smoothing,
                                               L.sm_scale_log2, L.means, Ht, L.k_codes, L.v_codes, L.kv_meta,
                                               L.kv_scale64, L.bias, L.bias_l2);
  return cudaGetLastError();
}

cudaError_t launch_prepass(const PrepassLaunch& L, cudaStream_t st) {
  switch (L.dtype * 1000 + L.D) {
    case SA2PP_F32 * 1000 + 64: return launch_prepass_t<float, 64>(L, st);
    case SA2PP_F32 * 1000 + 128: return launch_prepass_t<float, 128>(L, st);
    case SA2PP_F16 * 1000 + 64: return launch_prepass_t<__half, 64>(L, st);
    case SA2PP_F16 * 1000 + 128: return launch_prepass_t<__half, 128>(L, st);
    case SA2PP_BF16 * 1000 + 64: return launch_prepass_t<__nv_bfloat16, 64>(L, st);
    case SA2PP_BF16 * 1000 + 128: return launch_prepass_t<__nv_bfloat16, 128>(L, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace sa2pp
