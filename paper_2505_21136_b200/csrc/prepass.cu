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
//   channel_means  grid (B*(Hq+Hkv))          sequential FP64 channel sums in token order -> mean
//   quantize_q     grid (nQT, B*Hq)           one CTA per 128-row query tile
//   quantize_k     grid (nKB, B*Hkv)          one CTA per 64-key block (K codes, dK, bias)
//   quantize_v     grid (nKB, B*Hkv)          one CTA per 64-key block (V^T codes, dV)
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <algorithm>
#include <cstdint>
#include <type_traits>

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

// ------------------------------------------------------------------ pass 1: channel means
// numpy's x.mean(axis=0) over a C-ordered (N, D) float64 array is a SEQUENTIAL float64 sum per
// channel in token order followed by one division by N (quantization.py:133,147; checked against
// numpy in tests/test_gpu_parity.py), so each channel is one FP64 add chain here too: one CTA per
// (b, head) of Q and K, thread t owns channel t (SA2PP_MEANS_CPT = 1; 2 was 5 % slower); the head's rows
// stream through a 4-stage cp.async ring in shared memory (16 KB per stage) and every thread adds its
// channel row by row.  The FP64 add chain (one dependent add per token) sets the kernel's time.
#ifndef SA2PP_MEANS_CPT
#define SA2PP_MEANS_CPT 1  // channels (independent FP64 add chains) per thread
#endif
template <typename T, int D>
struct MeansCfg {
  static constexpr int kCpt = SA2PP_MEANS_CPT;
  static constexpr int kThreads = D / kCpt;
  static constexpr int kRowBytes = D * static_cast<int>(sizeof(T));
  static constexpr int kStageBytes = 16384;
  static constexpr int kRows = kStageBytes / kRowBytes;  // rows per stage
  static constexpr int kStages = 4;
  static constexpr int kPieces = kStageBytes / 16 / kThreads;  // 16-byte cp.async per thread per stage
};

template <typename T>
__device__ __forceinline__ void two_f64(const void* p, double& a, double& b) {
  if constexpr (sizeof(T) == 4) {
    const float2 f = *reinterpret_cast<const float2*>(p);
    a = static_cast<double>(f.x);
    b = static_cast<double>(f.y);
  } else if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    const uint32_t w = *reinterpret_cast<const uint32_t*>(p);
    a = static_cast<double>(__uint_as_float(w << 16));
    b = static_cast<double>(__uint_as_float(w & 0xFFFF0000u));
  } else {
    const __half2 h = *reinterpret_cast<const __half2*>(p);
    a = static_cast<double>(__low2float(h));
    b = static_cast<double>(__high2float(h));
  }
}

template <typename T, int D>
__global__ void __launch_bounds__(D / SA2PP_MEANS_CPT) channel_means_kernel(InView qv, InView kv, int Hq, int Hkv, int N,
                                                              double* __restrict__ means, int dc,
                                                              const int* __restrict__ need) {
  using M = MeansCfg<T, D>;
  extern __shared__ __align__(16) unsigned char ms_smem[];
  const int bh = blockIdx.x;  // in [0, B*(Hq+Hkv))
  if (need != nullptr && need[bh] == 0) return;  // the parallel path's certificate held for this head
  const int Ht = Hq + Hkv;
  const int b = bh / Ht, h = bh % Ht;
  const InView& v = (h < Hq) ? qv : kv;
  const int hh = (h < Hq) ? h : h - Hq;
  const int t = threadIdx.x;
  const int n_st = (N + M::kRows - 1) / M::kRows;
  // a thread's 16-byte pieces all sit at the same column of their rows, so the padded-channel
  // test (head_dim 32 / 96) is one per thread
  static_assert(M::kThreads % (M::kRowBytes / 16) == 0, "piece column must not depend on the piece");
  const int c16 = t % (M::kRowBytes / 16);
  const int col = c16 * (16 / static_cast<int>(sizeof(T))) < dc ? 16 * c16 : -1;
  auto issue = [&](int s) {
    if (s < n_st) {
      unsigned char* dst = ms_smem + (s % M::kStages) * M::kStageBytes;
#pragma unroll
      for (int i = 0; i < M::kPieces; ++i) {
        const int piece = i * M::kThreads + t;  // 16-byte piece of the stage
        const int r = piece / (M::kRowBytes / 16);
        const int n = s * M::kRows + r;
        const bool ok = n < N && col >= 0;
        const unsigned char* src =
            reinterpret_cast<const unsigned char*>(row_ptr<T>(v, b, hh, n < N ? n : 0)) + (col >= 0 ? col : 0);
        const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst + 16 * piece));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(ok ? 16 : 0) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");  // empty groups keep the wait count uniform
  };
#pragma unroll
  for (int s = 0; s < M::kStages - 1; ++s) issue(s);
  double s0 = 0.0, s1 = 0.0;
  for (int s = 0; s < n_st; ++s) {
    asm volatile("cp.async.wait_group %0;" ::"n"(M::kStages - 2) : "memory");
    __syncthreads();  // stage s landed for every thread; stage s-1 is no longer read
    issue(s + M::kStages - 1);
    const unsigned char* src = ms_smem + (s % M::kStages) * M::kStageBytes + t * M::kCpt * sizeof(T);
    const int rows = min(M::kRows, N - s * M::kRows);
    if constexpr (M::kCpt == 1) {
#pragma unroll 16
      for (int r = 0; r < rows; ++r) s0 += static_cast<double>(to_f32<T>(*reinterpret_cast<const T*>(src + r * M::kRowBytes)));
    } else if (rows == M::kRows) {
#pragma unroll 16
      for (int r = 0; r < M::kRows; ++r) {
        double a, c;
        two_f64<T>(src + r * M::kRowBytes, a, c);
        s0 += a;
        s1 += c;
      }
    } else {
      for (int r = 0; r < rows; ++r) {
        double a, c;
        two_f64<T>(src + r * M::kRowBytes, a, c);
        s0 += a;
        s1 += c;
      }
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  const double n = static_cast<double>(N);
  if constexpr (M::kCpt == 1) {
    means[static_cast<int64_t>(bh) * D + t] = s0 / n;
    return;
  }
  *reinterpret_cast<double2*>(means + static_cast<int64_t>(bh) * D + 2 * t) = make_double2(s0 / n, s1 / n);
}

// Parallel exact means for 16-bit inputs.  numpy's sequential FP64 sum rounds nothing when every
// partial sum is representable: all elements are multiples of u = 2^(E_min - (p - 1)) (E_min the
// smallest exponent among the channel's nonzero elements, p the input precision) and every partial
// sum is at most N * max|x|, so N * max|x| < 2^53 * u makes the sequential sum exact and therefore
// equal to a sum in any order.  means_partial sums kMeansRows-row chunks per channel in FP64
// and records max|x| and E_min; means_finalize adds the chunks, checks the certificate per channel
// and writes the mean, or flags the head for the sequential kernel (channel_means_kernel), which
// then runs only for flagged heads.
#ifndef SA2PP_MEANS_PAR
#define SA2PP_MEANS_PAR 1
#endif

template <typename T>
__device__ __forceinline__ T __ushort_as_bf16_or_half(unsigned short u);
template <>
__device__ __forceinline__ __nv_bfloat16 __ushort_as_bf16_or_half<__nv_bfloat16>(unsigned short u) {
  return __ushort_as_bfloat16(u);
}
template <>
__device__ __forceinline__ __half __ushort_as_bf16_or_half<__half>(unsigned short u) {
  return __ushort_as_half(u);
}

template <typename T>
struct Bits16;  // exponent/precision of the 16-bit input formats
template <>
struct Bits16<__nv_bfloat16> {
  static constexpr int kMantBits = 7, kBias = 127;
};
template <>
struct Bits16<__half> {
  static constexpr int kMantBits = 10, kBias = 15;
};

// 256 threads: lane group of D/8 threads covers a row with 16-byte loads (8 channels each), 256/(D/8)
// row groups stride the chunk; per-channel FP64 sums and (max |x|, min nonzero |x|) as packed 16-bit
// SIMD, reduced across row groups in shared memory (exact under the certificate, so order-free)
template <typename T, int D>
__global__ void __launch_bounds__(256) means_partial_kernel(InView qv, InView kv, int Hq, int Hkv, int N, int dc,
                                                            double* __restrict__ part,
                                                            unsigned long long* __restrict__ stat) {
  constexpr int LPR = D / 8, RG = 256 / LPR;
  __shared__ double s_acc[RG][D];
  __shared__ uint32_t s_mx[RG][D / 2], s_mn[RG][D / 2];
  const int ch = blockIdx.x, bh = blockIdx.y, n_ch = gridDim.x;
  const int Ht = Hq + Hkv;
  const int b = bh / Ht, h = bh % Ht;
  const InView& v = (h < Hq) ? qv : kv;
  const int hh = (h < Hq) ? h : h - Hq;
  const int tid = threadIdx.x, c8 = tid % LPR, rg = tid / LPR, c0 = c8 * 8;
  const int r0 = ch * kMeansRows, r1 = min(N, r0 + kMeansRows);
  double acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.0;
  uint32_t mx[4] = {0u, 0u, 0u, 0u}, mn[4] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu};
  if (c0 < dc) {
#pragma unroll 4
    for (int r = r0 + rg; r < r1; r += RG) {
      const uint4 w4 = __ldcs(reinterpret_cast<const uint4*>(row_ptr<T>(v, b, hh, r) + c0));
      const uint32_t w[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t mag = w[i] & 0x7FFF7FFFu;
        mx[i] = __vmaxu2(mx[i], mag);
        mn[i] = __vminu2(mn[i], mag | __vcmpeq2(mag, 0u));  // zeros do not count toward the min
        const float lo = to_f32<T>(__ushort_as_bf16_or_half<T>(static_cast<unsigned short>(w[i] & 0xFFFFu)));
        const float hi = to_f32<T>(__ushort_as_bf16_or_half<T>(static_cast<unsigned short>(w[i] >> 16)));
        acc[2 * i] += static_cast<double>(lo);
        acc[2 * i + 1] += static_cast<double>(hi);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) s_acc[rg][c0 + i] = acc[i];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    s_mx[rg][c0 / 2 + i] = mx[i];
    s_mn[rg][c0 / 2 + i] = mn[i];
  }
  __syncthreads();
  if (tid < D) {
    const int c = tid, sh = (c & 1) * 16;
    double a = 0.0;
    uint32_t m = 0u, n = 0xFFFFu;
    for (int g = 0; g < RG; ++g) {
      a += s_acc[g][c];
      m = max(m, (s_mx[g][c / 2] >> sh) & 0xFFFFu);
      n = min(n, (s_mn[g][c / 2] >> sh) & 0xFFFFu);
    }
    const uint32_t emin = n == 0xFFFFu ? 0xFFFFu : max(n >> Bits16<T>::kMantBits, 1u);
    const int64_t o = (static_cast<int64_t>(bh) * n_ch + ch) * D + c;
    part[o] = a;
    stat[o] = (static_cast<unsigned long long>(m) << 32) | emin;
  }
}

template <typename T, int D>
__global__ void __launch_bounds__(D) means_finalize_kernel(const double* __restrict__ part,
                                                           const unsigned long long* __restrict__ stat, int n_ch,
                                                           int N, double* __restrict__ means, int* __restrict__ need) {
  constexpr int MB = Bits16<T>::kMantBits, BIAS = Bits16<T>::kBias;
  const int bh = blockIdx.x, c = threadIdx.x;
  double acc = 0.0;
  uint32_t mx = 0u, emin = 0xFFFFu;
  for (int k = 0; k < n_ch; ++k) {
    const int64_t o = (static_cast<int64_t>(bh) * n_ch + k) * D + c;
    acc += part[o];  // exact when certified, so the order is free
    const unsigned long long s = stat[o];
    mx = max(mx, static_cast<uint32_t>(s >> 32));
    emin = min(emin, static_cast<uint32_t>(s & 0xFFFFu));
  }
  bool ok = true;
  if (mx != 0u) {
    const float xmax = to_f32<T>(__ushort_as_bf16_or_half<T>(static_cast<unsigned short>(mx)));
    const int ulp_exp = static_cast<int>(emin) - BIAS - MB;  // u = 2^ulp_exp
    ok = static_cast<double>(N) * static_cast<double>(xmax) < ldexp(1.0, 53 + ulp_exp);
  }
  if (ok) means[static_cast<int64_t>(bh) * D + c] = acc / static_cast<double>(N);
  const int any_fail = __syncthreads_or(!ok);
  if (c == 0) need[bh] = any_fail;
}

// ------------------------------------------------------------------ shared helpers

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

// The exact integer code: the FP64 quotient of the smoothed value (quantization.py:151-160).
__device__ __forceinline__ int int_code_exact(float v, double mu, double scale, double inv64, int qmax) {
  return min(max(static_cast<int>(div_rint(static_cast<double>(v) - mu, scale, inv64)), -qmax), qmax);
}

// Integer-code tie window of the FP32 fast path.  Under the fast-path condition |mu| <= 65536*amax,
// |q_fp32 - q_fp64| <= 2^-22 * qmax (two f32 roundings of d = (v - mu_hi) - mu_lo relative to amax, the
// f32 reciprocal and the product), i.e. 3.03e-5 at qmax = 127; codes whose fractional part lies within
// 4e-5 of .5 are recomputed from the FP64 quotient.
constexpr float kTieEdge = 0.5f - 4e-5f;

// Rare-path encoders kept out of line so the unrolled fast paths stay small in the i-cache.
__device__ __noinline__ uint32_t k_codes_exact8(const float* x, const double* mu, double scale, double inv, int qmax,
                                                 uint32_t* w1) {
  uint32_t w0 = 0u, hi = 0u;
  for (int i = 0; i < 8; ++i) {
    const uint32_t code = static_cast<uint32_t>(int_code_exact(x[i], mu[i], scale, inv, qmax)) & 0xFFu;
    if (i < 4) {
      w0 |= code << (8 * i);
    } else {
      hi |= code << (8 * (i - 4));
    }
  }
  *w1 = hi;
  return w0;
}
__device__ __noinline__ uint8_t v_code_exact(float x, double sc) {
  return e4m3_div(static_cast<double>(x), sc, 1.0 / sc);
}

template <typename T>
struct KvTile {
  static constexpr int kWords = 8 * static_cast<int>(sizeof(T)) / 4;  // 32-bit words per 8 channels
  uint32_t w[kWords];
  // 16-bit -> f32 on the FMA pipe: the sm_100 mixed-precision add of -0.0 (FHADD / FHADD.BF16), exact
  // for every input; shifts/masks or HADD2.F32 would load the half-rate ALU pipe these kernels lean on.
  __device__ __forceinline__ float get(int i) const {
    if constexpr (sizeof(T) == 4) {
      return __uint_as_float(w[i]);
    } else {
      float r;
      if constexpr (std::is_same<T, __nv_bfloat16>::value) {
        if (i & 1) {
          asm("{.reg .b16 l, h;\n\tmov.b32 {l, h}, %1;\n\tadd.rn.f32.bf16 %0, h, %2;}" : "=f"(r) : "r"(w[i >> 1]), "f"(-0.0f));
        } else {
          asm("{.reg .b16 l, h;\n\tmov.b32 {l, h}, %1;\n\tadd.rn.f32.bf16 %0, l, %2;}" : "=f"(r) : "r"(w[i >> 1]), "f"(-0.0f));
        }
      } else {
        if (i & 1) {
          asm("{.reg .f16 l, h;\n\tmov.b32 {l, h}, %1;\n\tadd.rn.f32.f16 %0, h, %2;}" : "=f"(r) : "r"(w[i >> 1]), "f"(-0.0f));
        } else {
          asm("{.reg .f16 l, h;\n\tmov.b32 {l, h}, %1;\n\tadd.rn.f32.f16 %0, l, %2;}" : "=f"(r) : "r"(w[i >> 1]), "f"(-0.0f));
        }
      }
      return r;
    }
  }
  __device__ __forceinline__ float2 get2(int i) const { return make_float2(get(i), get(i + 1)); }
};

// ------------------------------------------------------------------ pass 2: Q tiles
// Persistent CTAs (256 threads) walk the 128-row tiles of all (b, hq).  Thread (rg, c8) owns channels
// [8*c8, 8*c8+8) of the RT consecutive rows [rg*RT, rg*RT+RT): it cp.asyncs exactly those bytes of
// the NEXT tile into its own shared-memory slots while it quantizes the current one from registers,
// so every CTA keeps a tile in flight (the kernel is HBM-latency-bound otherwise) and no barrier is
// needed for the staging.  Rows >= N are written as zero codes.  amax = max over channels of
// max(|max_c - mu_c|, |min_c - mu_c|): fl64(v - mu) is monotone in v, so this is the reference's
// max |fl64(v - mu)| over the tile (quantization.py:151-160) with FP64 work per channel only.
template <typename T, int D>
__host__ __device__ constexpr int q_smem_bytes() {
  return 2 * 128 * D * static_cast<int>(sizeof(T));
}

template <typename T>
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc, bool valid) {
  const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(gsrc), "r"(valid ? 16 : 0) : "memory");
}

template <typename T, int D>
__global__ void __launch_bounds__(256, 2) quantize_q_kernel(InView qv, int Hq, int N, int Nq_pad, int n_qt, int n_tiles, int qmax,
                                                            const double* __restrict__ means, int Ht,
                                                            int8_t* __restrict__ q_codes, float* __restrict__ q_scale,
                                                            double* __restrict__ q_scale64, int dc) {
  constexpr int LPR = D / 8;      // lanes per row
  constexpr int RPP = 256 / LPR;  // row groups per CTA
  constexpr int RT = 128 / RPP;   // consecutive rows per thread (8 for D=128, 4 for D=64)
  constexpr int NW = sizeof(T) == 4 ? 2 : 1;  // 16-byte pieces per 8 channels
  constexpr int SLOT = RT * NW;               // 16-byte pieces per thread per tile
  extern __shared__ __align__(16) unsigned char q_smem[];
  uint4* stage = reinterpret_cast<uint4*>(q_smem);  // [2][SLOT][256]
  __shared__ float s_mn[8 * D], s_mx[8 * D];
  __shared__ double s_red[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c8 = tid % LPR, rg = tid / LPR;
  const int c0 = c8 * 8;
  const int qcol = c0 < dc ? c0 : -1;  // padded channels (head_dim 32 / 96) load as zeros
  auto prefetch = [&](int tile, int slot) {
    const int qt = tile % n_qt, bh = tile / n_qt;
    const int b = bh / Hq, h = bh % Hq;
    const int n0 = qt * 128;
#pragma unroll
    for (int rr = 0; rr < RT; ++rr) {
      const int r = n0 + rg * RT + rr;
      const bool ok = r < N && qcol >= 0;
      const T* src = row_ptr<T>(qv, b, h, r < N ? r : 0) + (qcol >= 0 ? qcol : 0);
#pragma unroll
      for (int u = 0; u < NW; ++u)
        cp_async16<T>(&stage[(slot * SLOT + rr * NW + u) * 256 + tid], reinterpret_cast<const uint4*>(src) + u, ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int slot = 0;
  if (static_cast<int>(blockIdx.x) < n_tiles) prefetch(blockIdx.x, 0);
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, slot ^= 1) {
    const int qt = tile % n_qt, bh = tile / n_qt;
    const int b = bh / Hq, h = bh % Hq;
    const int n0 = qt * 128;
    const int rows = min(128, N - n0);
    const double* mu_g = means + (static_cast<int64_t>(b) * Ht + h) * D;
    const int next = tile + gridDim.x;
    if (next < n_tiles) {
      prefetch(next, slot ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    KvTile<T> x[RT];
#pragma unroll
    for (int rr = 0; rr < RT; ++rr)
#pragma unroll
      for (int u = 0; u < NW; ++u) {
        const uint4 v4 = stage[(slot * SLOT + rr * NW + u) * 256 + tid];
        x[rr].w[4 * u] = v4.x; x[rr].w[4 * u + 1] = v4.y; x[rr].w[4 * u + 2] = v4.z; x[rr].w[4 * u + 3] = v4.w;
      }
    const double mu_c = tid < D ? mu_g[tid] : 0.0;
    float2 mh[4], ml[4];
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      const double2 m2 = *reinterpret_cast<const double2*>(mu_g + c0 + i);
      mh[i / 2] = make_float2(static_cast<float>(m2.x), static_cast<float>(m2.y));
      ml[i / 2] = make_float2(static_cast<float>(m2.x - static_cast<double>(mh[i / 2].x)),
                              static_cast<float>(m2.y - static_cast<double>(mh[i / 2].y)));
    }

    {  // per-channel min/max over the tile's valid rows
      float mn[8], mx[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        mn[i] = INFINITY;
        mx[i] = -INFINITY;
      }
      if (rows == 128) {
#pragma unroll
        for (int rr = 0; rr < RT; ++rr)
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            mn[i] = fminf(mn[i], x[rr].get(i));
            mx[i] = fmaxf(mx[i], x[rr].get(i));
          }
      } else {
#pragma unroll
        for (int rr = 0; rr < RT; ++rr) {
          const bool ok = rg * RT + rr < rows;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            mn[i] = fminf(mn[i], ok ? x[rr].get(i) : INFINITY);
            mx[i] = fmaxf(mx[i], ok ? x[rr].get(i) : -INFINITY);
          }
        }
      }
#pragma unroll
      for (int o = LPR; o < 32; o <<= 1)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          mn[i] = fminf(mn[i], __shfl_xor_sync(0xffffffffu, mn[i], o));
          mx[i] = fmaxf(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], o));
        }
      if (lane < LPR) {
        float* d0 = s_mn + warp * D + c0;
        float* d1 = s_mx + warp * D + c0;
        *reinterpret_cast<float4*>(d0) = make_float4(mn[0], mn[1], mn[2], mn[3]);
        *reinterpret_cast<float4*>(d0 + 4) = make_float4(mn[4], mn[5], mn[6], mn[7]);
        *reinterpret_cast<float4*>(d1) = make_float4(mx[0], mx[1], mx[2], mx[3]);
        *reinterpret_cast<float4*>(d1 + 4) = make_float4(mx[4], mx[5], mx[6], mx[7]);
      }
    }
    __syncthreads();
    if (tid < D) {
      float mn = INFINITY, mx = -INFINITY;
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        mn = fminf(mn, s_mn[w * D + tid]);
        mx = fmaxf(mx, s_mx[w * D + tid]);
      }
      double amax = 0.0;
      if (mx >= mn) amax = fmax(fabs(static_cast<double>(mx) - mu_c), fabs(static_cast<double>(mn) - mu_c));
      double mumax = fabs(mu_c);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
        mumax = fmax(mumax, __shfl_xor_sync(0xffffffffu, mumax, o));
      }
      if (lane == 0) {
        s_red[warp] = amax;
        s_red[4 + warp] = mumax;
      }
    }
    __syncthreads();
    double amax = s_red[0], mumax = s_red[4];
#pragma unroll
    for (int w = 1; w < D / 32; ++w) {
      amax = fmax(amax, s_red[w]);
      mumax = fmax(mumax, s_red[4 + w]);
    }
    const double scale = amax > 0.0 ? amax / static_cast<double>(qmax) : 1.0;
    if (tid == 0) {
      q_scale[static_cast<int64_t>(bh) * n_qt + qt] = static_cast<float>(scale);
      q_scale64[static_cast<int64_t>(bh) * n_qt + qt] = scale;
    }
    const double inv = 1.0 / scale;
    const float inv32 = static_cast<float>(inv);
    const bool fast = mumax <= 65536.0 * amax && amax >= 0x1p-100;  // see quantize_k

    // codes: ((q - mu_hi) - mu_lo) * inv rounded with the 1.5*2^23 trick; the code is the low byte
    // of the rounded float's bits (|q| <= qmax + 3e-5 under `fast`, so no clamp is needed)
    const float2 inv2 = make_float2(inv32, inv32);
    const float2 magic2 = make_float2(12582912.0f, 12582912.0f);
    int8_t* dst = q_codes + (static_cast<int64_t>(bh) * Nq_pad + n0 + rg * RT) * D + c0;
#pragma unroll
    for (int rr = 0; rr < RT; ++rr) {
      uint32_t tb[8];
      bool tie = !fast;
#pragma unroll
      for (int i = 0; i < 8; i += 2) {
        const float2 d = __fadd2_rn(__fadd2_rn(x[rr].get2(i), make_float2(-mh[i / 2].x, -mh[i / 2].y)),
                                    make_float2(-ml[i / 2].x, -ml[i / 2].y));
        const float2 t = __ffma2_rn(d, inv2, magic2);
        const float2 q = __fmul2_rn(d, inv2);
        const float2 f = __fadd2_rn(q, __fadd2_rn(make_float2(-t.x, -t.y), magic2));  // q - round(q)
        tie |= (fabsf(f.x) > kTieEdge) | (fabsf(f.y) > kTieEdge);
        tb[i] = __float_as_uint(t.x);
        tb[i + 1] = __float_as_uint(t.y);
      }
      uint32_t w0 = __byte_perm(__byte_perm(tb[0], tb[1], 0x0040), __byte_perm(tb[2], tb[3], 0x0040), 0x5410);
      uint32_t w1 = __byte_perm(__byte_perm(tb[4], tb[5], 0x0040), __byte_perm(tb[6], tb[7], 0x0040), 0x5410);
      const bool valid = rg * RT + rr < rows;
      if (tie && valid) {  // rare: near a rounding tie or |mu| >> amax -> FP64 quotients for these 8
        float xs[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) xs[i] = x[rr].get(i);
        w0 = k_codes_exact8(xs, mu_g + c0, scale, inv, qmax, &w1);
      }
      if (!valid) w0 = w1 = 0u;
      *reinterpret_cast<uint2*>(dst + rr * D) = make_uint2(w0, w1);
    }
  }
}

// ------------------------------------------------------------------ pass 3: K blocks and V blocks
// Two kernels, one CTA (256 threads) per 64-key block of one (b, hkv) each.  Thread (rg, c8) holds
// channels [8*c8, 8*c8+8) of the RT consecutive keys [rg*RT, rg*RT+RT) in registers, so every block
// is read from HBM exactly once and every output is produced from registers:
//   quantize_k:  k_codes [B, Hkv, Np, D] int8 (8-byte stores), kv_meta dK, bias / bias_l2 [B, Hq, Np]
//                (b_j = q_mean . Ks_j for every query head of the GQA group)
//   quantize_v:  v_codes [B, Hkv, D, Np] E4M3 (transposed through a swizzled 64-byte-per-channel smem
//                tile), kv_meta dV[0..D)
// Per-channel statistics (K min/max, V |max|) are reduced across the row groups with shuffles and
// across warps through shared memory.  Splitting K from V halves the live registers, so three CTAs
// share an SM instead of two (the single K+V kernel stalled on its three CTA barriers at two CTAs/SM).
// three-input FMNMX3 (sm_100)
__device__ __forceinline__ float max3f(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ float min3f(float a, float b, float c) {
  float d;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

template <typename T, int D>
struct KvGeom {
  static constexpr int LPR = D / 8;                     // lanes per key row
  static constexpr int RPP = 256 / LPR;                 // row groups per CTA
  static constexpr int RT = 64 / RPP;                   // consecutive keys per thread (4 at D=128, 2 at D=64)
  static constexpr int UPR = 64 / RT;                   // RT-byte units per 64-key V^T row
  static constexpr int NW = sizeof(T) == 4 ? 2 : 1;     // 16-byte loads per 8 channels
};

template <typename T, int D>
__device__ __forceinline__ void load_rows(const InView& in, int b, int h, int n0, int rg, int c0, int rows,
                                          KvTile<T> (&x)[KvGeom<T, D>::RT]) {
  using G = KvGeom<T, D>;
#pragma unroll
  for (int rr = 0; rr < G::RT; ++rr) {
    const int r = rg * G::RT + rr;
#pragma unroll
    for (int u = 0; u < G::NW; ++u) {
      uint4 v4 = make_uint4(0, 0, 0, 0);
      if (r < rows) v4 = __ldcs(reinterpret_cast<const uint4*>(row_ptr<T>(in, b, h, n0 + r) + c0) + u);
      x[rr].w[4 * u] = v4.x; x[rr].w[4 * u + 1] = v4.y; x[rr].w[4 * u + 2] = v4.z; x[rr].w[4 * u + 3] = v4.w;
    }
  }
}

#ifndef SA2PP_K_MINB
#define SA2PP_K_MINB 3
#endif
#ifndef SA2PP_K_SMEM_SPLIT
#define SA2PP_K_SMEM_SPLIT 0  // 1: the (hi, lo) split of the K means made once per channel in smem (A/B: profiles/r02/kernel_experiments.md)
#endif
#ifndef SA2PP_K_RSCATTER
#define SA2PP_K_RSCATTER 1  // bias: reduce-scatter butterfly instead of a full butterfly per row
#endif
// PAD: head_dim < D (32 / 96), threads of the padded channels load nothing (zeros); a separate
// instantiation so the unpadded kernel keeps its register allocation
template <typename T, int D, bool PAD>
__global__ void __launch_bounds__(256, SA2PP_K_MINB) quantize_k_kernel(InView kv_in, int Hq, int Hkv, int N, int Np, int n_kb,
                                                            int qmax, int smoothing, double sm_scale_log2,
                                                            const double* __restrict__ means, int Ht,
                                                            int8_t* __restrict__ k_codes, float* __restrict__ kv_meta,
                                                            double* __restrict__ kv_scale64, float* __restrict__ bias,
                                                            float* __restrict__ bias_l2, int dc) {
  using G = KvGeom<T, D>;
  constexpr int LPR = G::LPR, RT = G::RT;
  __shared__ float s_kmn[8 * D], s_kmx[8 * D];
  __shared__ double s_red[8];
#if SA2PP_K_SMEM_SPLIT
  __shared__ __align__(16) float2 s_mhl[D];  // (hi, lo) float split of the channel means, made once per channel
#endif
  const int kb = blockIdx.x;
  const int bh = blockIdx.y;
  const int b = bh / Hkv, h = bh % Hkv;
  const int n0 = kb * 64;
  const int rows = min(64, N - n0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c8 = tid % LPR, rg = tid / LPR;
  const int c0 = c8 * 8;

  KvTile<T> kt[RT];  // rows past N are zero (padding after smoothing)
  load_rows<T, D>(kv_in, b, h, n0, rg, c0, PAD && c0 >= dc ? 0 : rows, kt);
  const double* kmu_g = means + (static_cast<int64_t>(b) * Ht + Hq + h) * D;

  // ---- per-channel min/max over the block's valid rows
  {
    float mn[8], mx[8];
    if (rows == 64) {  // every block but a ragged last one: no validity selects
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        mn[i] = kt[0].get(i);
        mx[i] = mn[i];
      }
#pragma unroll
      for (int rr = 1; rr < RT; rr += 2) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float x1 = kt[rr].get(i), x2 = rr + 1 < RT ? kt[rr + 1].get(i) : x1;
          mn[i] = min3f(mn[i], x1, x2);
          mx[i] = max3f(mx[i], x1, x2);
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        mn[i] = INFINITY;
        mx[i] = -INFINITY;
      }
#pragma unroll
      for (int rr = 0; rr < RT; ++rr) {
        const bool ok = rg * RT + rr < rows;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float x = kt[rr].get(i);
          mn[i] = fminf(mn[i], ok ? x : INFINITY);
          mx[i] = fmaxf(mx[i], ok ? x : -INFINITY);
        }
      }
    }
#pragma unroll
    for (int o = LPR; o < 32; o <<= 1) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        mn[i] = fminf(mn[i], __shfl_xor_sync(0xffffffffu, mn[i], o));
        mx[i] = fmaxf(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], o));
      }
    }
    if (lane < LPR) {
      float* d0 = s_kmn + warp * D + c0;
      float* d1 = s_kmx + warp * D + c0;
      *reinterpret_cast<float4*>(d0) = make_float4(mn[0], mn[1], mn[2], mn[3]);
      *reinterpret_cast<float4*>(d0 + 4) = make_float4(mn[4], mn[5], mn[6], mn[7]);
      *reinterpret_cast<float4*>(d1) = make_float4(mx[0], mx[1], mx[2], mx[3]);
      *reinterpret_cast<float4*>(d1 + 4) = make_float4(mx[4], mx[5], mx[6], mx[7]);
    }
  }
  __syncthreads();

  // ---- smoothed amax (quantization.py:151-160): fl64(k - mu) is monotone in k, so the channel
  //      min/max give the element-wise FP64 max
  float* meta = kv_meta + (static_cast<int64_t>(bh) * n_kb + kb) * (4 + D);
  double* sc64 = kv_scale64 + (static_cast<int64_t>(bh) * n_kb + kb) * (1 + D);
  if (tid < D) {
    float mn = INFINITY, mx = -INFINITY;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      mn = fminf(mn, s_kmn[w * D + tid]);
      mx = fmaxf(mx, s_kmx[w * D + tid]);
    }
    const double mu = kmu_g[tid];
#if SA2PP_K_SMEM_SPLIT
    {
      const float hi = static_cast<float>(mu);
      s_mhl[tid] = make_float2(hi, static_cast<float>(mu - static_cast<double>(hi)));
    }
#endif
    double amax = 0.0;
    if (mx >= mn) amax = fmax(fabs(static_cast<double>(mx) - mu), fabs(static_cast<double>(mn) - mu));
    double mumax = fabs(mu);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      mumax = fmax(mumax, __shfl_xor_sync(0xffffffffu, mumax, o));
    }
    if (lane == 0) {
      s_red[warp] = amax;
      s_red[4 + warp] = mumax;
    }
  }
  __syncthreads();
  double amax = s_red[0], mumax = s_red[4];
#pragma unroll
  for (int w = 1; w < D / 32; ++w) {
    amax = fmax(amax, s_red[w]);
    mumax = fmax(mumax, s_red[4 + w]);
  }
  const double kscale = amax > 0.0 ? amax / static_cast<double>(qmax) : 1.0;
  const double kinv = 1.0 / kscale;
  const float kinv32 = static_cast<float>(kinv);
  // the error bound of the FP32 fast path; amax >= 2^-100 keeps the f32 reciprocal finite and the
  // absolute error of subnormal intermediates (2^-150) far below a code step
  const bool kfast = mumax <= 65536.0 * amax && amax >= 0x1p-100;
  if (tid < 4) meta[tid] = tid == 0 ? static_cast<float>(kscale) : 0.0f;
  if (tid == 0) sc64[0] = kscale;

  // ---- K codes: ((k - mu_hi) - mu_lo) * inv rounded with the 1.5*2^23 trick; the code is the low
  //      byte of the rounded float's bits.  |q| <= qmax + 3e-5 under kfast, so no clamp is needed.
  {
    float2 mh[4], ml[4];
#if SA2PP_K_SMEM_SPLIT
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      const float4 a = *reinterpret_cast<const float4*>(&s_mhl[c0 + i]);  // (hi, lo) of c, c + 1
      mh[i / 2] = make_float2(a.x, a.z);
      ml[i / 2] = make_float2(a.y, a.w);
    }
#else
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      const double2 m2 = *reinterpret_cast<const double2*>(kmu_g + c0 + i);
      mh[i / 2] = make_float2(static_cast<float>(m2.x), static_cast<float>(m2.y));
      ml[i / 2] = make_float2(static_cast<float>(m2.x - static_cast<double>(mh[i / 2].x)),
                              static_cast<float>(m2.y - static_cast<double>(mh[i / 2].y)));
    }
#endif
    const float2 inv2 = make_float2(kinv32, kinv32);
    const float2 magic2 = make_float2(12582912.0f, 12582912.0f);
    int8_t* kdst = k_codes + (static_cast<int64_t>(bh) * Np + n0 + rg * RT) * D + c0;
#pragma unroll
    for (int rr = 0; rr < RT; ++rr) {
      uint32_t tb[8];
      bool tie = !kfast;
#pragma unroll
      for (int i = 0; i < 8; i += 2) {
        const float2 d = __fadd2_rn(__fadd2_rn(kt[rr].get2(i), make_float2(-mh[i / 2].x, -mh[i / 2].y)),
                                    make_float2(-ml[i / 2].x, -ml[i / 2].y));
        const float2 q = __fmul2_rn(d, inv2);
        const float2 t = __fadd2_rn(q, magic2);
        const float2 f = __fadd2_rn(q, __fadd2_rn(make_float2(-t.x, -t.y), magic2));  // q - round(q)
        tie |= (fabsf(f.x) > kTieEdge) | (fabsf(f.y) > kTieEdge);
        tb[i] = __float_as_uint(t.x);
        tb[i + 1] = __float_as_uint(t.y);
      }
      uint32_t w0 = __byte_perm(__byte_perm(tb[0], tb[1], 0x0040), __byte_perm(tb[2], tb[3], 0x0040), 0x5410);
      uint32_t w1 = __byte_perm(__byte_perm(tb[4], tb[5], 0x0040), __byte_perm(tb[6], tb[7], 0x0040), 0x5410);
      const bool valid = rg * RT + rr < rows;
      if (tie && valid) {  // rare: near a rounding tie or |mu| >> amax -> FP64 quotients for these 8
        float x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = kt[rr].get(i);
        w0 = k_codes_exact8(x, kmu_g + c0, kscale, kinv, qmax, &w1);
      }
      if (!valid) w0 = w1 = 0u;
      *reinterpret_cast<uint2*>(kdst + rr * D) = make_uint2(w0, w1);
    }
  }

  // ---- bias for every query head sharing this KV head: b_j = q_mean . Ks_j (attention.py:288-289),
  //      FP64 over this thread's 8 channels, then a butterfly over the LPR lanes of the row
  {
    const int group = Hq / Hkv;
    for (int g = 0; g < group; ++g) {
      const int hq = h * group + g;
      double acc[RT];
#pragma unroll
      for (int rr = 0; rr < RT; ++rr) acc[rr] = 0.0;
      if (smoothing) {
        const double* qm_g = means + (static_cast<int64_t>(b) * Ht + hq) * D + c0;
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
          const double2 q2 = *reinterpret_cast<const double2*>(qm_g + i);
          const double2 m2 = *reinterpret_cast<const double2*>(kmu_g + c0 + i);  // L1-resident
#pragma unroll
          for (int rr = 0; rr < RT; ++rr) {
            acc[rr] = fma(q2.x, static_cast<double>(kt[rr].get(i)) - m2.x, acc[rr]);
            acc[rr] = fma(q2.y, static_cast<double>(kt[rr].get(i + 1)) - m2.y, acc[rr]);
          }
        }
#if SA2PP_K_RSCATTER
        // reduce-scatter over the row's LPR lanes: each halving step keeps half of the live rows
        // (lanes with bit o set the upper half), so lane c8 ends with row c8 / (LPR / RT) complete
#pragma unroll
        for (int w = RT, o = LPR / 2; w > 1; w >>= 1, o >>= 1) {
          const bool up = (c8 & o) != 0;
#pragma unroll
          for (int i = 0; i < w / 2; ++i) {
            const double send = up ? acc[i] : acc[i + w / 2];
            const double keep = up ? acc[i + w / 2] : acc[i];
            acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
          }
        }
#pragma unroll
        for (int o = LPR / (2 * RT); o > 0; o >>= 1) acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], o);
#else
#pragma unroll
        for (int o = 1; o < LPR; o <<= 1) {
#pragma unroll
          for (int rr = 0; rr < RT; ++rr) acc[rr] += __shfl_xor_sync(0xffffffffu, acc[rr], o);
        }
#endif
      }
#if SA2PP_K_RSCATTER
      if (c8 % (LPR / RT) == 0) {
        const int r = rg * RT + c8 / (LPR / RT);
        double a = acc[0];
#else
      if (c8 < RT) {
        const int r = rg * RT + c8;
        double a = acc[0];
#pragma unroll
        for (int rr = 1; rr < RT; ++rr)
          if (c8 == rr) a = acc[rr];
#endif
        if (r >= rows) a = 0.0;
        const int64_t o = (static_cast<int64_t>(b) * Hq + hq) * Np + n0 + r;
        bias[o] = static_cast<float>(a);
        bias_l2[o] = static_cast<float>(a * sm_scale_log2);
      }
    }
  }
}

template <typename T, int D>
__host__ __device__ constexpr int v_smem_bytes() {
  return 8 * D * 4 + D * 64 + D * 8 + D * 4;
}

#ifndef SA2PP_V_MINB
#define SA2PP_V_MINB 4
#endif
template <typename T, int D, bool PAD>
__global__ void __launch_bounds__(256, SA2PP_V_MINB) quantize_v_kernel(InView v_in, int Hkv, int N, int Np, int n_kb, double v_r,
                                                            uint8_t* __restrict__ v_codes, float* __restrict__ kv_meta,
                                                            double* __restrict__ kv_scale64, int dc) {
  using G = KvGeom<T, D>;
  constexpr int LPR = G::LPR, RT = G::RT, UPR = G::UPR;
  extern __shared__ __align__(16) unsigned char v_smem[];
  float* s_vmx = reinterpret_cast<float*>(v_smem);              // [8 warps][D]
  uint8_t* s_vt = reinterpret_cast<uint8_t*>(s_vmx + 8 * D);    // [D][64] swizzled E4M3 codes
  double* s_vsc = reinterpret_cast<double*>(s_vt + D * 64);     // [D]
  float* s_vinv = reinterpret_cast<float*>(s_vsc + D);          // [D]
  const int kb = blockIdx.x;
  const int bh = blockIdx.y;
  const int b = bh / Hkv, h = bh % Hkv;
  const int n0 = kb * 64;
  const int rows = min(64, N - n0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c8 = tid % LPR, rg = tid / LPR;
  const int c0 = c8 * 8;

  KvTile<T> vt[RT];  // rows past N are zero (the reference pads V with zeros)
  load_rows<T, D>(v_in, b, h, n0, rg, c0, PAD && c0 >= dc ? 0 : rows, vt);

  // ---- per-channel |max| over the block (zero rows do not change it)
  {
    float va[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) va[i] = fabsf(vt[0].get(i));
#pragma unroll
    for (int rr = 1; rr < RT; rr += 2) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float x1 = fabsf(vt[rr].get(i)), x2 = rr + 1 < RT ? fabsf(vt[rr + 1].get(i)) : x1;
        va[i] = max3f(va[i], x1, x2);
      }
    }
#pragma unroll
    for (int o = LPR; o < 32; o <<= 1) {
#pragma unroll
      for (int i = 0; i < 8; ++i) va[i] = fmaxf(va[i], __shfl_xor_sync(0xffffffffu, va[i], o));
    }
    if (lane < LPR) {
      float* d2 = s_vmx + warp * D + c0;
      *reinterpret_cast<float4*>(d2) = make_float4(va[0], va[1], va[2], va[3]);
      *reinterpret_cast<float4*>(d2 + 4) = make_float4(va[4], va[5], va[6], va[7]);
    }
  }
  __syncthreads();

  // ---- V scale per (block, channel) (quantization.py:178-188)
  float* meta = kv_meta + (static_cast<int64_t>(bh) * n_kb + kb) * (4 + D);
  double* sc64 = kv_scale64 + (static_cast<int64_t>(bh) * n_kb + kb) * (1 + D);
  if (tid < D) {
    float va = 0.0f;
#pragma unroll
    for (int w = 0; w < 8; ++w) va = fmaxf(va, s_vmx[w * D + tid]);
    const double sc = va > 0.0f ? static_cast<double>(va) / v_r : 1.0;
    s_vsc[tid] = sc;
    // a channel whose block max is below 2^-100 (its f32 reciprocal may overflow, its quotients may
    // be subnormal) is encoded from the FP64 quotients; NaN marks it for the exact path below
    s_vinv[tid] = (va > 0.0f && va < 0x1p-100f) ? __int_as_float(0x7fffffff) : static_cast<float>(1.0 / sc);
    meta[4 + tid] = static_cast<float>(sc);
    sc64[1 + tid] = sc;
  }
  __syncthreads();

  // ---- V codes (E4M3, RNE, satfinite): tie test = the codes of q*(1 -+ 2^-20) differ, which brackets
  //      the exact FP64 quotient; flagged elements are re-encoded from it.  Codes go to a transposed
  //      smem tile: RT-byte unit (channel c, keys [rg*RT, +RT)) at unit index rg ^ swz(c8).
  {
    const float lo_f = 1.0f - 0x1p-20f, hi_f = 1.0f + 0x1p-20f;
    const int swz = c8 * (UPR / LPR);
    uint32_t tmask = 0u;  // bit i*RT + rr: element (channel c0+i, key rg*RT+rr) is near a tie
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int c = c0 + i;
      const float inv = s_vinv[c];
      const uint32_t all_exact = isnan(inv) ? ((1u << RT) - 1u) << (i * RT) : 0u;
      tmask |= all_exact;
      uint32_t unit = 0u;
#pragma unroll
      for (int rr = 0; rr < RT; rr += 2) {
        const float2 q = __fmul2_rn(make_float2(vt[rr].get(i), vt[rr + 1].get(i)), make_float2(inv, inv));
        const float2 ql = __fmul2_rn(q, make_float2(lo_f, lo_f));
        const float2 qh = __fmul2_rn(q, make_float2(hi_f, hi_f));
        uint16_t cq, cl, ch;
        asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(cq) : "f"(q.y), "f"(q.x));
        asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(cl) : "f"(ql.y), "f"(ql.x));
        asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(ch) : "f"(qh.y), "f"(qh.x));
        const uint32_t d = static_cast<uint32_t>(cl ^ ch);
        tmask |= (((d & 0xFFu) != 0u ? 1u : 0u) | ((d >> 8) != 0u ? 2u : 0u)) << (i * RT + rr);
        unit |= static_cast<uint32_t>(cq) << (8 * rr);
      }
      uint8_t* dst = s_vt + c * 64 + ((rg ^ swz) * RT);
      if constexpr (RT == 4) {
        *reinterpret_cast<uint32_t*>(dst) = unit;
      } else {
        *reinterpret_cast<uint16_t*>(dst) = static_cast<uint16_t>(unit);
      }
    }
    // ~0.6% of bf16 elements sit exactly on an E4M3 tie: re-encode just those from the FP64
    // quotient (a warp loops max-popcount times, ~1-2)
    while (tmask) {
      const int bit = __ffs(tmask) - 1;
      tmask &= tmask - 1u;
      const int i = bit / RT, rr = bit % RT, c = c0 + i;
      const float x = !PAD || c < dc ? to_f32<T>(row_ptr<T>(v_in, b, h, n0 + rg * RT + rr)[c]) : 0.0f;
      s_vt[c * 64 + (rg ^ swz) * RT + rr] = v_code_exact(x, s_vsc[c]);
    }
  }

  // ---- V^T codes out: lane -> (channel, 4-key word); two channels per warp instruction, 64 B each
  __syncthreads();
  constexpr int WSWZ = (UPR / LPR) * RT / 4;  // the unit swizzle in 4-byte words
#pragma unroll
  for (int it = 0; it < D / 16; ++it) {
    const int idx = it * 256 + tid;
    const int c = idx >> 4, j = idx & 15;
    const uint32_t v = *reinterpret_cast<const uint32_t*>(s_vt + c * 64 + 4 * (j ^ ((c >> 3) * WSWZ)));
    *reinterpret_cast<uint32_t*>(v_codes + (static_cast<int64_t>(bh) * D + c) * Np + n0 + 4 * j) = v;
  }
}

// ------------------------------------------------------------------ host launcher
// A non-blocking side stream and its fork/join events, per calling thread and device (created on
// first use, destroyed with the thread); nullptr stream = run everything on the caller's stream.
#ifndef SA2PP_Q_SIDE_MAXN
#define SA2PP_Q_SIDE_MAXN 2048  // quantize_q beside quantize_k up to this sequence length
#endif

struct SideStream {
  cudaStream_t stream = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr, mid = nullptr;
  int dev = -1;
  ~SideStream() {
    if (stream != nullptr) {
      int cur = 0;
      if (cudaGetDevice(&cur) == cudaSuccess && cur != dev) cudaSetDevice(dev);
      cudaEventDestroy(fork);
      cudaEventDestroy(join);
      cudaEventDestroy(mid);
      cudaStreamDestroy(stream);
      if (cur != dev) cudaSetDevice(cur);
    }
  }
};

static SideStream& side_stream() {
  static thread_local SideStream per_dev[16];
  static SideStream none;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return none;
  SideStream& s = per_dev[dev];
  if (s.stream == nullptr) {
    if (cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking) != cudaSuccess) {
      s.stream = nullptr;
      return none;
    }
    if (cudaEventCreateWithFlags(&s.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&s.join, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&s.mid, cudaEventDisableTiming) != cudaSuccess) {
      cudaStreamDestroy(s.stream);
      s.stream = nullptr;
      return none;
    }
    s.dev = dev;
  }
  return s;
}

template <typename T, int D>
static cudaError_t launch_prepass_t(const PrepassLaunch& L, cudaStream_t st) {
  InView qv{L.q, L.q_stride[0], L.q_stride[1], L.q_stride[2]};
  InView kv{L.k, L.k_stride[0], L.k_stride[1], L.k_stride[2]};
  InView vv{L.v, L.v_stride[0], L.v_stride[1], L.v_stride[2]};
  const int Ht = L.Hq + L.Hkv;
  // quantize_v needs no channel means, so it runs on a side stream beside channel_means (a long FP64
  // add chain on few CTAs) and quantize_q/k; the caller's stream joins it at the end (fork/join is
  // stream-ordered and graph-capturable).  quantize_q beside quantize_k was measured too: no gain at
  // 16K (both near their own limits)
  const dim3 gk(L.n_kb, L.B * L.Hkv);
  constexpr int v_smem = v_smem_bytes<T, D>();
  {
    static PerDevice v_once;
    cudaError_t e = v_once.run([&](std::atomic<int>&) {
      cudaError_t r = cudaFuncSetAttribute(quantize_v_kernel<T, D, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           v_smem);
      if (r == cudaSuccess)
        r = cudaFuncSetAttribute(quantize_v_kernel<T, D, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, v_smem);
      return r;
    });
    if (e != cudaSuccess) return e;
  }
  const bool pad = L.d_in < D;
  const auto vk = pad ? quantize_v_kernel<T, D, true> : quantize_v_kernel<T, D, false>;
  const auto kk = pad ? quantize_k_kernel<T, D, true> : quantize_k_kernel<T, D, false>;
  SideStream& side = side_stream();
  if (side.stream != nullptr) {
    cudaError_t e = cudaEventRecord(side.fork, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(side.stream, side.fork, 0);
    if (e != cudaSuccess) return e;
    vk<<<gk, 256, v_smem, side.stream>>>(vv, L.Hkv, L.N, L.Np, L.n_kb, L.v_r, L.v_codes,
                                                              L.kv_meta, L.kv_scale64, L.d_in);
  }
  if (L.smoothing) {
    using M = MeansCfg<T, D>;
    constexpr int smem = M::kStages * M::kStageBytes;
    static PerDevice once;
    cudaError_t e = once.run([&](std::atomic<int>&) {
      return cudaFuncSetAttribute(channel_means_kernel<T, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    });
    if (e != cudaSuccess) return e;
    const int* need = nullptr;
    if constexpr (sizeof(T) == 2) {
      // fewer (b, head) chains than SMs: the sequential kernel is pure add-chain latency (long
      // contexts, CogVideoX, the host pipeline's chunks), so the parallel certified path goes first;
      // with more chains it measured slower (it competes with quantize_v for bandwidth)
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      if (SA2PP_MEANS_PAR && L.ws_means != nullptr && L.B * Ht < sms) {
        const int n_ch = (L.N + kMeansRows - 1) / kMeansRows;
        auto* part = static_cast<double*>(L.ws_means);
        auto* stat = reinterpret_cast<unsigned long long*>(part + static_cast<int64_t>(L.B) * Ht * n_ch * D);
        int* flags = reinterpret_cast<int*>(stat + static_cast<int64_t>(L.B) * Ht * n_ch * D);
        means_partial_kernel<T, D><<<dim3(n_ch, L.B * Ht), 256, 0, st>>>(qv, kv, L.Hq, L.Hkv, L.N, L.d_in, part, stat);
        means_finalize_kernel<T, D><<<L.B * Ht, D, 0, st>>>(part, stat, n_ch, L.N, L.means, flags);
        need = flags;
      }
    }
    channel_means_kernel<T, D><<<L.B * Ht, M::kThreads, smem, st>>>(qv, kv, L.Hq, L.Hkv, L.N, L.means, L.d_in, need);
  } else {
    cudaMemsetAsync(L.means, 0, sizeof(double) * L.B * Ht * D, st);
  }
  {  // persistent: as many CTAs as fit, each walking tiles with the next one in flight
    constexpr int q_smem = q_smem_bytes<T, D>();
    static PerDevice occ;
    cudaError_t e = occ.run([&](std::atomic<int>& v) {
      cudaError_t r = cudaFuncSetAttribute(quantize_q_kernel<T, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, q_smem);
      int n = 0;
      if (r == cudaSuccess) r = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, quantize_q_kernel<T, D>, 256, q_smem);
      v.store(n < 1 ? 1 : n);
      return r;
    });
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int ctas_per_sm = occ.get();
    const int n_tiles = L.n_qt * L.B * L.Hq;
    const int grid = n_tiles < sms * ctas_per_sm ? n_tiles : sms * ctas_per_sm;
    // short sequences: quantize_q joins quantize_v on the side stream once the means are done, so
    // it runs beside quantize_k (each is a few latency-bound waves there; at 4K+ they contend)
    cudaStream_t qs = st;
    if (side.stream != nullptr && L.N <= SA2PP_Q_SIDE_MAXN) {
      e = cudaEventRecord(side.mid, st);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(side.stream, side.mid, 0);
      if (e != cudaSuccess) return e;
      qs = side.stream;
    }
    quantize_q_kernel<T, D><<<grid, 256, q_smem, qs>>>(qv, L.Hq, L.N, L.Nq_pad, L.n_qt, n_tiles, L.qmax, L.means, Ht,
                                                       L.q_codes, L.q_scale, L.q_scale64, L.d_in);
  }
  kk<<<gk, 256, 0, st>>>(kv, L.Hq, L.Hkv, L.N, L.Np, L.n_kb, L.qmax, L.smoothing, L.sm_scale_log2,
                                              L.means, Ht, L.k_codes, L.kv_meta, L.kv_scale64, L.bias, L.bias_l2, L.d_in);
  if (side.stream != nullptr) {  // join: the caller's stream waits for quantize_v
    cudaError_t e = cudaEventRecord(side.join, side.stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, side.join, 0);
    if (e != cudaSuccess) return e;
  } else {
    vk<<<gk, 256, v_smem, st>>>(vv, L.Hkv, L.N, L.Np, L.n_kb, L.v_r, L.v_codes, L.kv_meta,
                                                     L.kv_scale64, L.d_in);
  }
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

// ------------------------------------------------------------------ run-report helpers
namespace sa2pp {

__global__ void report_init_kernel(sa2pp_report* r) {
  r->overflow_events = 0u;
  r->p_scale_min_bits = 0x7f800000u;
  r->p_scale_max_bits = 0u;
  r->reserved = 0u;
  r->v_scale_min_bits = 0x7ff0000000000000ull;
  r->v_scale_max_bits = 0ull;
}

// Positive doubles order like their bit patterns, so 64-bit integer atomics give FP64 min/max.
__global__ void vscale_minmax_kernel(const double* __restrict__ s, int64_t blocks, int D, int d, sa2pp_report* r) {
  unsigned long long mn = 0x7ff0000000000000ull, mx = 0ull;
  const int64_t n = blocks * d;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const unsigned long long b = __double_as_longlong(s[(i / d) * (1 + D) + 1 + i % d]);
    mn = b < mn ? b : mn;
    mx = b > mx ? b : mx;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long a = __shfl_xor_sync(0xffffffffu, mn, o), c = __shfl_xor_sync(0xffffffffu, mx, o);
    mn = a < mn ? a : mn;
    mx = c > mx ? c : mx;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(reinterpret_cast<unsigned long long*>(&r->v_scale_min_bits), mn);
    atomicMax(reinterpret_cast<unsigned long long*>(&r->v_scale_max_bits), mx);
  }
}

cudaError_t launch_report_init(sa2pp_report* r, cudaStream_t st) {
  report_init_kernel<<<1, 1, 0, st>>>(r);
  return cudaGetLastError();
}

cudaError_t launch_vscale_minmax(const double* kv_scale64, int64_t blocks, int D, int d, sa2pp_report* r,
                                 cudaStream_t st) {
  const int64_t n = blocks * d;
  const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, 1184));
  vscale_minmax_kernel<<<grid, 256, 0, st>>>(kv_scale64, blocks, D, d, r);
  return cudaGetLastError();
}

}  // namespace sa2pp
