// SageAttention2++ forward on sm_100a: INT8 QK^T and FP8 PV on tcgen05 tensor cores.
//
// One CTA owns one query tile of 128 rows and walks the key blocks of 64 in ascending order,
// which is part of the reference's numerical contract (lpattn attention.py:6-8).  Warp roles
// (384 threads):
//   warp 0       TMA producer: the Q tile once, then a STAGES-deep ring of {K^ block, V^T block,
//                block meta (dK, dV[D]), bias row} guarded by kv_full / kv_empty mbarriers
//   warp 1       TMEM allocator + single-thread tcgen05.mma issuer
//                  S(j)  = Q^ . K^_j^T         kind::i8, M=128 N=64 K=D, S32 accumulator in TMEM
//                  PV(j) = P^(j) . V^_j         kind::f8f6f4, A (P^) from TMEM, B (V^T) from smem,
//                                              M=128 N=D K=64 (two k=32 MMAs), F16 or F32 accumulator
//   warps 4..11  softmax: two warpgroups split every query row.  Thread (h, r) owns row r, score
//                columns [32h, 32h+32) and output channels [h*D/2, (h+1)*D/2).  Per block:
//                tcgen05.ld S, dequant + bias in the log2 domain, causal/pad mask, online softmax
//                (attention.py:136-154), one E4M3 scale per 128x64 tile (quantization.py:163-175),
//                P^ -> TMEM, promotion of the previous block's PV: O = O*alpha + pv*(dP*dV[c])
//                (attention.py:303); finally O / l (attention.py:304-305).
//
// TMEM (256 columns): S[0] cols [0,64), S[1] cols [64,128), PV cols [128, 128+D).  P^ of block j
// (E4M3, 4 per column) is written over S[j&1]: keys 0-31 at cols [0,8), keys 32-63 at [32,40),
// i.e. inside the half of S that the writing warpgroup itself has already read.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda.h>
#include <cstdint>
#include <type_traits>

#include "ptx.cuh"
#include "sa2pp_internal.h"

namespace sa2pp {

template <int D>
struct AttnCfg {
  static constexpr int kStages = (D == 128) ? 4 : 6;
  static constexpr int kQBytes = 128 * D;
  static constexpr int kKBytes = 64 * D;
  static constexpr int kVBytes = D * 64;
  static constexpr int kMetaBytes = (4 + D) * 4;
  static constexpr int kBiasBytes = 64 * 4;
  static constexpr uint32_t kLayoutQK = (D == 128) ? 2u : 4u;  // SWIZZLE_128B / SWIZZLE_64B
  static constexpr uint32_t kSboQK = 8 * D;                     // bytes between 8-row core groups
  static constexpr uint32_t kLayoutV = 4u;                      // V^T rows are 64 keys = 64 B
  static constexpr uint32_t kSboV = 512;
  static constexpr int kTmemCols = 256;
  static constexpr int kHalfD = D / 2;
  // shared memory carve-up (offsets from a 1024-aligned base)
  static constexpr int kOffQ = 0;
  static constexpr int kOffK = kOffQ + kQBytes;
  static constexpr int kOffV = kOffK + kStages * kKBytes;
  static constexpr int kOffMeta = kOffV + kStages * kVBytes;
  static constexpr int kOffBias = kOffMeta + kStages * kMetaBytes;
  static constexpr int kOffF = kOffBias + kStages * kBiasBytes;     // [2][D]   dP * dV per block parity
  static constexpr int kOffHalfMax = kOffF + 2 * D * 4;             // [2][2][128] half-row maxima
  static constexpr int kOffRed = kOffHalfMax + 2 * 2 * 128 * 4;     // [2][8]   warp tile-max candidates
  static constexpr int kOffL = kOffRed + 2 * 8 * 4;                 // [2][128] final half-row sums
  static constexpr int kOffBar = kOffL + 2 * 128 * 4;
  static constexpr int kNumBars = 1 + 2 * kStages + 5;
  static constexpr int kOffTmem = kOffBar + kNumBars * 8;
  static constexpr int kSmemBytes = kOffTmem + 16 + 1024;  // + alignment slack
  static constexpr int kThreads = 384;
};

template <int N, typename OutT>
__device__ __forceinline__ void store_out(OutT* dst, const float (&O)[N], float inv_l) {
  if constexpr (sizeof(OutT) == 4) {
#pragma unroll
    for (int c = 0; c < N; c += 4) {
      float4 v = make_float4(O[c] * inv_l, O[c + 1] * inv_l, O[c + 2] * inv_l, O[c + 3] * inv_l);
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(dst) + c) = v;
    }
  } else {
#pragma unroll
    for (int c = 0; c < N; c += 8) {
      uint32_t w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float a = O[c + 2 * i] * inv_l, b = O[c + 2 * i + 1] * inv_l;
        if constexpr (std::is_same<OutT, __nv_bfloat16>::value) {
          __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
          w[i] = *reinterpret_cast<uint32_t*>(&h);
        } else {
          __half2 h = __floats2half2_rn(a, b);
          w[i] = *reinterpret_cast<uint32_t*>(&h);
        }
      }
      *reinterpret_cast<uint4*>(dst + c) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

template <int D, bool CAUSAL, bool ACC16, typename OutT>
__global__ void __launch_bounds__(384, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const AttnParams p) {
  using C = AttnCfg<D>;
  constexpr int S = C::kStages;
  constexpr int HD = C::kHalfD;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // ---- work decode: grid = (B*Hq, n_qt); causal runs the heaviest query tiles first
  const int bh = blockIdx.x;
  const int b = bh / p.Hq;
  const int hq = bh % p.Hq;
  const int hkv = hq / p.group;
  const int qt = CAUSAL ? (p.n_qt - 1 - static_cast<int>(blockIdx.y)) : static_cast<int>(blockIdx.y);
  const int q0 = qt * 128;
  const int nblk = CAUSAL ? min(p.n_kb, (min(q0 + 128, p.N) + 63) / 64) : p.n_kb;

  uint64_t* bar_base = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* q_full = bar_base;
  uint64_t* kv_full = bar_base + 1;
  uint64_t* kv_empty = bar_base + 1 + S;
  uint64_t* s_full = bar_base + 1 + 2 * S;  // [2]
  uint64_t* p_full = s_full + 2;            // [2]
  uint64_t* pv_full = p_full + 2;           // [1]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + C::kOffTmem);

  if (warp == 0 && lane == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < S; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    mbar_init(&s_full[0], 1);
    mbar_init(&s_full[1], 1);
    mbar_init(&p_full[0], 256);
    mbar_init(&p_full[1], 256);
    mbar_init(pv_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_holder, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      // =========================== TMA producer ===========================
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      mbar_arrive_expect_tx(q_full, C::kQBytes);
      tma_load_2d(smem + C::kOffQ, &tm_q, q_full, 0, bh * p.Nq_pad + q0);
      const int kv_row = (b * p.Hkv + hkv) * p.Np;
      const int vt_row = (b * p.Hkv + hkv) * D;
      const float* meta_src = p.kv_meta + static_cast<int64_t>(b * p.Hkv + hkv) * p.n_kb * (4 + D);
      const float* bias_src = p.bias_l2 + static_cast<int64_t>(bh) * p.Np;
      for (int j = 0; j < nblk; ++j) {
        const int st = j % S;
        if (j >= S) mbar_wait(&kv_empty[st], ((j / S) & 1) ^ 1);
        mbar_arrive_expect_tx(&kv_full[st], C::kKBytes + C::kVBytes + C::kMetaBytes + C::kBiasBytes);
        tma_load_2d(smem + C::kOffK + st * C::kKBytes, &tm_k, &kv_full[st], 0, kv_row + j * 64);
        tma_load_2d(smem + C::kOffV + st * C::kVBytes, &tm_v, &kv_full[st], j * 64, vt_row);
        bulk_load(smem + C::kOffMeta + st * C::kMetaBytes, meta_src + static_cast<int64_t>(j) * (4 + D),
                  C::kMetaBytes, &kv_full[st]);
        bulk_load(smem + C::kOffBias + st * C::kBiasBytes, bias_src + j * 64, C::kBiasBytes, &kv_full[st]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // =========================== MMA issuer ===========================
      constexpr uint32_t idesc_qk = make_idesc(2u, 1u, 1u, 128u, 64u);             // S32 <- s8 x s8
      constexpr uint32_t idesc_pv = make_idesc(ACC16 ? 0u : 1u, 0u, 0u, 128u, D);  // F16|F32 <- e4m3 x e4m3
      const uint64_t qdesc = smem_desc(smem_u32(smem + C::kOffQ), C::kSboQK, C::kLayoutQK);
      const uint32_t pv_tm = tmem + 128;
      mbar_wait(q_full, 0);
      tc_fence_after();
      auto issue_pv = [&](int jj) {
        const int st = jj % S;
        const uint64_t vdesc = smem_desc(smem_u32(smem + C::kOffV + st * C::kVBytes), C::kSboV, C::kLayoutV);
        mbar_wait(&p_full[jj & 1], (jj >> 1) & 1);
        tc_fence_after();
        const uint32_t a_tm = tmem + (jj & 1) * 64;
        umma_f8_ts(pv_tm, a_tm, vdesc, idesc_pv, 0u);            // keys  0..31: P^ cols [0,8)
        umma_f8_ts(pv_tm, a_tm + 32, vdesc + 2, idesc_pv, 1u);   // keys 32..63: P^ cols [32,40)
        umma_commit(pv_full);
        umma_commit(&kv_empty[st]);
      };
      for (int j = 0; j < nblk; ++j) {
        const int st = j % S;
        mbar_wait(&kv_full[st], (j / S) & 1);
        tc_fence_after();
        const uint64_t kdesc = smem_desc(smem_u32(smem + C::kOffK + st * C::kKBytes), C::kSboQK, C::kLayoutQK);
        const uint32_t d_tm = tmem + (j & 1) * 64;
#pragma unroll
        for (int kk = 0; kk < D / 32; ++kk)
          umma_i8_ss(d_tm, qdesc + 2 * kk, kdesc + 2 * kk, idesc_qk, kk > 0 ? 1u : 0u);
        umma_commit(&s_full[j & 1]);
        if (j > 0) issue_pv(j - 1);
      }
      issue_pv(nblk - 1);
    }
  } else if (warp >= 4) {
    // =========================== softmax / promotion / epilogue ===========================
    const int h = (warp - 4) >> 2;   // which half of the row
    const int wq = warp & 3;         // TMEM lane quarter
    const int r = wq * 32 + lane;    // query row within the tile
    const int tid = threadIdx.x - 128;
    const int row_g = q0 + r;
    const bool row_valid = row_g < p.N;
    const float a_q = p.q_scale[static_cast<int64_t>(bh) * p.n_qt + qt] * p.sm_scale_log2;
    const uint32_t tm_row = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    float* fbuf = reinterpret_cast<float*>(smem + C::kOffF);
    float* halfmax = reinterpret_cast<float*>(smem + C::kOffHalfMax);
    float* red = reinterpret_cast<float*>(smem + C::kOffRed);
    const bool dbg = (p.debug != nullptr) && blockIdx.x == 0 && blockIdx.y == 0;

    float O[HD];
#pragma unroll
    for (int c = 0; c < HD; ++c) O[c] = 0.0f;
    float m_run = -INFINITY, l_half = 0.0f, alpha_prev = 1.0f;
    bool resc_prev = true;
    uint32_t overflow = 0;

    auto promote = [&](int jj) {
      mbar_wait(pv_full, jj & 1);
      tc_fence_after();
      const float* f = fbuf + (jj & 1) * D + h * HD;
      const bool any_resc = __any_sync(0xffffffffu, resc_prev);
#pragma unroll
      for (int c0 = 0; c0 < HD; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tm_row + 128 + h * HD + c0, v);
        tmem_wait_ld();
        if (dbg && jj == 0) {
#pragma unroll
          for (int i = 0; i < 32; ++i) p.debug[128 * 64 + r * D + h * HD + c0 + i] = v[i];
        }
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const float4 fv = *reinterpret_cast<const float4*>(f + c0 + i);
          const float fs[4] = {fv.x, fv.y, fv.z, fv.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            float pv;
            if constexpr (ACC16) {
              pv = __half2float(__ushort_as_half(static_cast<unsigned short>(v[i + u] & 0xFFFFu)));
              overflow += !isfinite(pv);
            } else {
              pv = __uint_as_float(v[i + u]);
            }
            float& o = O[c0 + i + u];
            o = any_resc ? fmaf(o, alpha_prev, pv * fs[u]) : fmaf(pv, fs[u], o);
          }
        }
        reg_fence32(&O[c0]);
      }
    };

    for (int j = 0; j < nblk; ++j) {
      const int st = j % S;
      mbar_wait(&kv_full[st], (j / S) & 1);
      mbar_wait(&s_full[j & 1], (j >> 1) & 1);
      tc_fence_after();
      uint32_t s[32];
      tmem_ld32(tm_row + (j & 1) * 64 + h * 32, s);
      tmem_wait_ld();
      if (dbg && j == 0) {
#pragma unroll
        for (int i = 0; i < 32; ++i) p.debug[r * 64 + h * 32 + i] = s[i];
      }
      const float* meta = reinterpret_cast<const float*>(smem + C::kOffMeta + st * C::kMetaBytes);
      const float* cb = reinterpret_cast<const float*>(smem + C::kOffBias + st * C::kBiasBytes) + h * 32;
      const float a = a_q * meta[0];
      float x[32];
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        const float4 c4 = *reinterpret_cast<const float4*>(cb + i);
        x[i + 0] = fmaf(static_cast<float>(static_cast<int>(s[i + 0])), a, c4.x);
        x[i + 1] = fmaf(static_cast<float>(static_cast<int>(s[i + 1])), a, c4.y);
        x[i + 2] = fmaf(static_cast<float>(static_cast<int>(s[i + 2])), a, c4.z);
        x[i + 3] = fmaf(static_cast<float>(static_cast<int>(s[i + 3])), a, c4.w);
      }
      const int key0 = j * 64 + h * 32;
      const bool need_mask = (CAUSAL && key0 + 31 > q0) || (key0 + 32 > p.N);
      if (need_mask) {
        const int lim = CAUSAL ? min(row_g + 1, p.N) : p.N;  // keys >= lim are masked
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (key0 + i >= lim) x[i] = -INFINITY;
      }
      float hmax = fmax3(x[0], x[1], x[2]);
#pragma unroll
      for (int i = 3; i < 31; i += 2) hmax = fmax3(hmax, x[i], x[i + 1]);
      hmax = fmaxf(hmax, x[31]);
      // Tile-max candidate: rowmax - m_new = min(0, rowmax - m_old) = max over halves of
      // min(0, halfmax - m_old), so each half contributes without knowing its partner.
      float d_r = row_valid ? fminf(0.0f, hmax - m_run) : -INFINITY;
      if (m_run == -INFINITY) d_r = row_valid && hmax != -INFINITY ? 0.0f : d_r;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) d_r = fmaxf(d_r, __shfl_xor_sync(0xffffffffu, d_r, o));
      float* hm_j = halfmax + (j & 1) * 256;
      float* red_j = red + (j & 1) * 8;
      hm_j[h * 128 + r] = hmax;
      if (lane == 0) red_j[warp - 4] = d_r;
      named_bar_sync(1, 256);
      const float rmax = fmaxf(hmax, hm_j[(h ^ 1) * 128 + r]);
      float Dt = red_j[0];
#pragma unroll
      for (int w = 1; w < 8; ++w) Dt = fmaxf(Dt, red_j[w]);
      const float m_new = fmaxf(m_run, rmax);
      const float dP = ex2(Dt) * p.inv_pr;  // (tile max of P~) / p_r
      const float m_eff = (m_new == -INFINITY) ? 0.0f : (m_new + Dt - p.log2_pr);
      float rowsum = 0.0f;
      uint32_t pk[8];
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        const float e0 = ex2(x[i + 0] - m_eff), e1 = ex2(x[i + 1] - m_eff);
        const float e2 = ex2(x[i + 2] - m_eff), e3 = ex2(x[i + 3] - m_eff);
        rowsum += (e0 + e1) + (e2 + e3);
        pk[i / 4] = pack_e4m3x2(e0, e1) | (pack_e4m3x2(e2, e3) << 16);
      }
      const float alpha = ex2(m_run - m_new);
      l_half = l_half * alpha + rowsum * dP;
      if (tid < D) fbuf[(j & 1) * D + tid] = dP * meta[4 + tid];
      if (p.report != nullptr && tid == 0) {
        atomicMin(&p.report->p_scale_min_bits, __float_as_uint(dP));
        atomicMax(&p.report->p_scale_max_bits, __float_as_uint(dP));
      }
      // P^(j) goes to TMEM first so its registers are free during the promotion; the MMA does
      // not read it before p_full(j), which also certifies that the PV buffer has been drained.
      tmem_st8(tm_row + (j & 1) * 64 + h * 32, pk);
      tmem_wait_st();
      if (j > 0) promote(j - 1);
      tc_fence_before();
      mbar_arrive(&p_full[j & 1]);
      resc_prev = (m_new != m_run);
      alpha_prev = alpha;
      m_run = m_new;
    }
    float* lbuf = reinterpret_cast<float*>(smem + C::kOffL);
    lbuf[h * 128 + r] = l_half;
    named_bar_sync(1, 256);  // last block's fbuf and both half-row sums visible
    promote(nblk - 1);
    if (p.report != nullptr && overflow) atomicAdd(&p.report->overflow_events, overflow);
    if (row_valid) {
      const float l = l_half + lbuf[(h ^ 1) * 128 + r];
      const float inv_l = 1.0f / (l == 0.0f ? 1.0f : l);
      OutT* dst = reinterpret_cast<OutT*>(p.out) + b * p.o_sb + hq * p.o_sh + static_cast<int64_t>(row_g) * p.o_sn +
                  h * HD;
      store_out<HD, OutT>(dst, O, inv_l);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, C::kTmemCols);
  }
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

static bool make_map_2d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t rows, uint64_t row_bytes,
                        uint32_t box_inner, uint32_t box_rows, CUtensorMapSwizzle sw) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_inner, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int D, bool CAUSAL, bool ACC16, typename OutT>
static cudaError_t launch_t(const AttnParams& P, const sa2pp_quant& qt, cudaStream_t st) {
  using C = AttnCfg<D>;
  CUtensorMap mq, mk, mv;
  const CUtensorMapSwizzle swqk = (D == 128) ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  if (!make_map_2d(&mq, qt.q_codes, D, static_cast<uint64_t>(P.B) * P.Hq * P.Nq_pad, D, D, 128, swqk) ||
      !make_map_2d(&mk, qt.k_codes, D, static_cast<uint64_t>(P.B) * P.Hkv * P.Np, D, D, 64, swqk) ||
      !make_map_2d(&mv, qt.v_codes, P.Np, static_cast<uint64_t>(P.B) * P.Hkv * D, P.Np, 64, D,
                   CU_TENSOR_MAP_SWIZZLE_64B))
    return cudaErrorInvalidValue;
  auto kern = attn_fwd_kernel<D, CAUSAL, ACC16, OutT>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid(P.B * P.Hq, P.n_qt);
  kern<<<grid, C::kThreads, C::kSmemBytes, st>>>(mq, mk, mv, P);
  return cudaGetLastError();
}

template <int D, bool CAUSAL, bool ACC16>
static cudaError_t launch_out(const AttnParams& P, const sa2pp_quant& qt, cudaStream_t st) {
  switch (P.out_dtype) {
    case SA2PP_F32: return launch_t<D, CAUSAL, ACC16, float>(P, qt, st);
    case SA2PP_F16: return launch_t<D, CAUSAL, ACC16, __half>(P, qt, st);
    case SA2PP_BF16: return launch_t<D, CAUSAL, ACC16, __nv_bfloat16>(P, qt, st);
    default: return cudaErrorInvalidValue;
  }
}

template <int D>
static cudaError_t launch_d(const sa2pp_problem& prob, const AttnParams& P, const sa2pp_quant& qt,
                            cudaStream_t st) {
  const bool acc16 = prob.pv_accum == SA2PP_ACC_F16;
  if (prob.causal) {
    return acc16 ? launch_out<D, true, true>(P, qt, st) : launch_out<D, true, false>(P, qt, st);
  }
  return acc16 ? launch_out<D, false, true>(P, qt, st) : launch_out<D, false, false>(P, qt, st);
}

cudaError_t launch_attn(const sa2pp_problem& prob, const AttnParams& P, const sa2pp_quant& qt, cudaStream_t st) {
  if (prob.head_dim == 128) return launch_d<128>(prob, P, qt, st);
  if (prob.head_dim == 64) return launch_d<64>(prob, P, qt, st);
  return cudaErrorInvalidValue;
}

}  // namespace sa2pp
