// SageAttention2++ forward on sm_100a: INT8 QK^T and FP8 PV on tcgen05 tensor cores.
//
// One CTA (256 threads = 8 warps, two CTAs resident per SM) owns one query tile of 128 rows and
// walks the key blocks of 64 in ascending order, which is part of the reference's numerical
// contract (lpattn attention.py:6-8).  All eight warps run the softmax: two warpgroups split every
// query row, thread (h, r) owning row r, score columns [32h, 32h+32) and output channels
// [h*D/2, (h+1)*D/2).  There is no producer or MMA warp: thread 0 issues the prologue (Q, the first
// STAGES K/V loads, S(0), S(1)), and afterwards lane 0 of whichever warp finishes block j last
// (a shared-memory arrival counter) issues, from a single thread:
//     PV(j)   = P^(j) . V^_j       kind::f8f6f4, A (P^) from TMEM, B (V^T) from smem, M=128 N=D
//                                  K=64 (two k=32 MMAs), F16 or F32 accumulator
//     S(j+2)  = Q^ . K^_(j+2)^T    kind::i8, M=128 N=64 K=D, S32 accumulator (double-buffered S)
//     TMA     refill of the K^/V^T/meta/bias stage freed by PV(j-1) with block j-1+STAGES.
// Keeping the issue inside the softmax warps leaves exactly 8 warps per CTA, i.e. 4 warps per SM
// sub-partition with two CTAs resident, which is what lets each thread keep 128 registers (its
// D/2 output accumulators live in registers).  The two resident CTAs run out of phase, so one
// tile's barrier/MMA waits overlap the other tile's MUFU-bound exp2 phase.
//
// Per block each softmax thread: tcgen05.ld S, dequant + bias in the log2 domain, causal/pad mask,
// half-row max, tile max through one named barrier, online softmax (attention.py:136-154), one
// E4M3 scale per 128x64 tile (quantization.py:163-175), P^ -> TMEM, promotion of the previous
// block's PV: O = O*alpha + pv*(dP*dV[c]) (attention.py:303); finally O / l (attention.py:304-305).
//
// TMEM (256 columns per CTA): S[0] cols [0,64), S[1] cols [64,128), PV cols [128, 128+D).  P^ of
// block j (E4M3, 4 per column) is written over S[j&1]: keys 0-31 at cols [0,8), keys 32-63 at
// [32,40), i.e. inside the half of S that the writing warpgroup itself has already read.
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
  static constexpr int kStages = (D == 128) ? 5 : 8;
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
  static constexpr int kOffCnt = kOffL + 2 * 128 * 4;               // [2] per-parity warp arrival counters
  static constexpr int kOffBar = kOffCnt + 16;
  static constexpr int kNumBars = 1 + 2 * kStages + 3;
  static constexpr int kOffTmem = kOffBar + kNumBars * 8;
  static constexpr int kSmemBytes = kOffTmem + 16 + 1024;  // + alignment slack
  static constexpr int kThreads = 256;
  static_assert(2 * kSmemBytes <= 227 * 1024, "two CTAs per SM must fit in shared memory");
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

template <int D, bool CAUSAL, bool ACC16, bool INSTR, typename OutT>
__global__ void __launch_bounds__(256, 2)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const AttnParams p) {
  using C = AttnCfg<D>;
  constexpr int S = C::kStages;
  constexpr int HD = C::kHalfD;
  extern __shared__ uint8_t smem_raw[];
  // pointer arithmetic on the shared array (not via integers) keeps the shared address space visible
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // ---- work decode: grid = (n_qt, B*Hq); the CTAs resident at once share one head's K/V in L2;
  //      causal runs the heaviest query tiles first
  const int bh = blockIdx.y;
  const int b = bh / p.Hq;
  const int hq = bh % p.Hq;
  const int hkv = hq / p.group;
  const int qt = CAUSAL ? (p.n_qt - 1 - static_cast<int>(blockIdx.x)) : static_cast<int>(blockIdx.x);
  const int q0 = qt * 128;
  const int nblk = CAUSAL ? min(p.n_kb, (min(q0 + 128, p.N) + 63) / 64) : p.n_kb;

  uint64_t* bar_base = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* q_full = bar_base;
  uint64_t* kv_full = bar_base + 1;
  uint64_t* kv_empty = bar_base + 1 + S;
  uint64_t* s_full = bar_base + 1 + 2 * S;  // [2]
  uint64_t* pv_full = s_full + 2;           // [1]
  int* arrive_cnt = reinterpret_cast<int*>(smem + C::kOffCnt);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + C::kOffTmem);

  if (warp == 0) {
    if (lane == 0) {
      mbar_init(q_full, 1);
      for (int s = 0; s < S; ++s) {
        mbar_init(&kv_full[s], 1);
        mbar_init(&kv_empty[s], 1);
      }
      mbar_init(&s_full[0], 1);
      mbar_init(&s_full[1], 1);
      mbar_init(pv_full, 1);
      arrive_cnt[0] = arrive_cnt[1] = 0;
      fence_barrier_init();
    }
    __syncwarp();
    tmem_alloc(tmem_holder, C::kTmemCols);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  // ---------------- MMA / TMA issue helpers (run by one thread at a time)
  const int kv_row = (b * p.Hkv + hkv) * p.Np;
  const int vt_row = (b * p.Hkv + hkv) * D;
  const float* meta_src = p.kv_meta + static_cast<int64_t>(b * p.Hkv + hkv) * p.n_kb * (4 + D);
  const float* bias_src = p.bias_l2 + static_cast<int64_t>(bh) * p.Np;
  constexpr uint32_t idesc_qk = make_idesc(2u, 1u, 1u, 128u, 64u);             // S32 <- s8 x s8
  constexpr uint32_t idesc_pv = make_idesc(ACC16 ? 0u : 1u, 0u, 0u, 128u, D);  // F16|F32 <- e4m3 x e4m3
  auto load_block = [&](int j) {
    const int st = j % S;
    mbar_arrive_expect_tx(&kv_full[st], C::kKBytes + C::kVBytes + C::kMetaBytes + C::kBiasBytes);
    tma_load_2d(smem + C::kOffK + st * C::kKBytes, &tm_k, &kv_full[st], 0, kv_row + j * 64);
    tma_load_2d(smem + C::kOffV + st * C::kVBytes, &tm_v, &kv_full[st], j * 64, vt_row);
    bulk_load(smem + C::kOffMeta + st * C::kMetaBytes, meta_src + static_cast<int64_t>(j) * (4 + D), C::kMetaBytes,
              &kv_full[st]);
    bulk_load(smem + C::kOffBias + st * C::kBiasBytes, bias_src + j * 64, C::kBiasBytes, &kv_full[st]);
  };
  auto issue_qk = [&](int j) {
    const int st = j % S;
    mbar_wait(&kv_full[st], (j / S) & 1);
    tc_fence_after();
    const uint64_t qdesc = smem_desc(smem_u32(smem + C::kOffQ), C::kSboQK, C::kLayoutQK);
    const uint64_t kdesc = smem_desc(smem_u32(smem + C::kOffK + st * C::kKBytes), C::kSboQK, C::kLayoutQK);
    const uint32_t d_tm = tmem + (j & 1) * 64;
#pragma unroll
    for (int kk = 0; kk < D / 32; ++kk) umma_i8_ss(d_tm, qdesc + 2 * kk, kdesc + 2 * kk, idesc_qk, kk > 0 ? 1u : 0u);
    umma_commit(&s_full[j & 1]);
  };
  // End of block j, run by the last warp to finish it (every thread has stored P^(j) and drained
  // PV(j-1)): PV(j), then S(j+2) into the S buffer PV(j) reads (tcgen05 MMAs from one thread
  // execute in order), then the refill of the stage freed by PV(j-1).
  auto issue_block_end = [&](int j) {
    const int st = j % S;
    const uint64_t vdesc = smem_desc(smem_u32(smem + C::kOffV + st * C::kVBytes), C::kSboV, C::kLayoutV);
    const uint32_t a_tm = tmem + (j & 1) * 64;
    umma_f8_ts(tmem + 128, a_tm, vdesc, idesc_pv, 0u);           // keys  0..31: P^ cols [0,8)
    umma_f8_ts(tmem + 128, a_tm + 32, vdesc + 2, idesc_pv, 1u);  // keys 32..63: P^ cols [32,40)
    umma_commit(pv_full);
    umma_commit(&kv_empty[st]);
    if (j + 2 < nblk) issue_qk(j + 2);  // S[j&1] is free: PV(j), issued above, read P^(j) from it
    const int jl = j - 1 + S;
    if (j >= 1 && jl < nblk) {
      mbar_wait(&kv_empty[(j - 1) % S], ((j - 1) / S) & 1);
      load_block(jl);
    }
  };
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    mbar_arrive_expect_tx(q_full, C::kQBytes);
    tma_load_2d(smem + C::kOffQ, &tm_q, q_full, 0, bh * p.Nq_pad + q0);
    for (int j = 0; j < min(S, nblk); ++j) load_block(j);
    mbar_wait(q_full, 0);
    issue_qk(0);
    if (nblk > 1) issue_qk(1);
  }
  __syncwarp();

  // =========================== softmax / promotion / epilogue ===========================
  const int h = warp >> 2;       // which half of the row
  const int wq = warp & 3;       // TMEM lane quarter accessible to this warp
  const int r = wq * 32 + lane;  // query row within the tile
  const int tid = threadIdx.x;
  const int row_g = q0 + r;
  const bool row_valid = row_g < p.N;
  const float a_q = p.q_scale[static_cast<int64_t>(bh) * p.n_qt + qt] * p.sm_scale_log2;
  const uint32_t tm_row = tmem + (static_cast<uint32_t>(wq * 32) << 16);
  float* fbuf = reinterpret_cast<float*>(smem + C::kOffF);
  float* halfmax = reinterpret_cast<float*>(smem + C::kOffHalfMax);
  float* red = reinterpret_cast<float*>(smem + C::kOffRed);
  const bool dbg = INSTR && (p.debug != nullptr) && qt == 0 && bh == 0;
  unsigned long long* trc = (INSTR && p.trace != nullptr && bh == 0 && qt < 8 && lane == 0)
                                ? p.trace + static_cast<int64_t>(qt) * 66 * 64 + warp * 8
                                : nullptr;
  auto stamp = [&](int j, int k) {
    if constexpr (INSTR) {
      if (trc != nullptr && j < 64) trc[(2 + j) * 64 + k] = clock64();
    }
  };
  if constexpr (INSTR) {
    if (trc != nullptr && tid == 0) {
      trc[0] = smid();
      trc[1] = globaltimer();
      trc[3] = nblk;
    }
  }

  float2 O[HD / 2];
#pragma unroll
  for (int c = 0; c < HD / 2; ++c) O[c] = make_float2(0.0f, 0.0f);
  float m_run = -INFINITY, l_half = 0.0f, alpha_prev = 1.0f;
  bool resc_prev = true;
  uint32_t overflow = 0;
  const bool want_overflow = ACC16 && p.report != nullptr;

  // O[c] = O[c]*alpha + pv[c]*f[c] for this thread's D/2 channels of row r (attention.py:303).
  // RESC: at least one row of the warp changed its running max, so O is rescaled by alpha.
  auto promote_impl = [&](int jj, auto resc_tag) {
    constexpr bool RESC = decltype(resc_tag)::value;
    const float* f = fbuf + (jj & 1) * D + h * HD;
    const float2 al2 = make_float2(alpha_prev, alpha_prev);
    constexpr int CH = ACC16 ? 32 : 16;  // channels per TMEM load (16 registers either way)
#pragma unroll
    for (int c0 = 0; c0 < HD; c0 += CH) {
      float2 pv[CH / 2];
      if constexpr (ACC16) {
        uint32_t v[CH / 2];
        tmem_ld16_pack16(tm_row + 128 + h * HD + c0, v);  // F16 accumulators, 2 per register
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < CH / 2; ++i) pv[i] = __half22float2(*reinterpret_cast<const __half2*>(&v[i]));
        if (want_overflow) {
#pragma unroll
          for (int i = 0; i < CH / 2; ++i)
            overflow += ((v[i] & 0x7C00u) == 0x7C00u) + ((v[i] & 0x7C000000u) == 0x7C000000u);
        }
      } else {
        uint32_t v[CH];
        tmem_ld16(tm_row + 128 + h * HD + c0, v);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < CH / 2; ++i) pv[i] = make_float2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
      }
      if constexpr (INSTR) {
        if (dbg && jj == 0) {
#pragma unroll
          for (int i = 0; i < CH / 2; ++i) {
            p.debug[128 * 64 + r * D + h * HD + c0 + 2 * i] = __float_as_uint(pv[i].x);
            p.debug[128 * 64 + r * D + h * HD + c0 + 2 * i + 1] = __float_as_uint(pv[i].y);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < CH / 2; i += 2) {
        const float4 fv = ld_shared_f4(f + c0 + 2 * i);
        if constexpr (RESC) {
          O[c0 / 2 + i] = __ffma2_rn(pv[i], make_float2(fv.x, fv.y), __fmul2_rn(O[c0 / 2 + i], al2));
          O[c0 / 2 + i + 1] = __ffma2_rn(pv[i + 1], make_float2(fv.z, fv.w), __fmul2_rn(O[c0 / 2 + i + 1], al2));
        } else {
          O[c0 / 2 + i] = __ffma2_rn(pv[i], make_float2(fv.x, fv.y), O[c0 / 2 + i]);
          O[c0 / 2 + i + 1] = __ffma2_rn(pv[i + 1], make_float2(fv.z, fv.w), O[c0 / 2 + i + 1]);
        }
      }
      if constexpr (CH == 32) {
        reg_fence32(reinterpret_cast<float*>(&O[c0 / 2]));
      } else {
        reg_fence16(reinterpret_cast<float*>(&O[c0 / 2]));
      }
    }
  };
  auto promote = [&](int jj) {
    mbar_wait(pv_full, jj & 1);
    tc_fence_after();
    stamp(jj + 1, 6);
    if (__any_sync(0xffffffffu, resc_prev)) {
      promote_impl(jj, std::true_type{});
    } else {
      promote_impl(jj, std::false_type{});
    }
  };

  // One key block.  MASK: causal diagonal / padded-tail block (attention.py:128-133, 293-294).
  auto block = [&](int j, auto mask_tag) {
    constexpr bool MASK = decltype(mask_tag)::value;
    const int st = j % S;
    mbar_wait(&kv_full[st], (j / S) & 1);
    mbar_wait(&s_full[j & 1], (j >> 1) & 1);
    tc_fence_after();
    stamp(j, 0);
    const float* meta = reinterpret_cast<const float*>(smem + C::kOffMeta + st * C::kMetaBytes);
    const float* cb = reinterpret_cast<const float*>(smem + C::kOffBias + st * C::kBiasBytes) + h * 32;
    const float a = a_q * ld_shared_f32(meta);
    const uint32_t s_addr = tm_row + (j & 1) * 64 + h * 32;
    // ---- pass 1: t = S_int * (dQ dK sm_scale log2e) + bias_j * sm_scale log2e  (attention.py:287-292)
    //      and the half-row max; t stays in registers across the tile-max barrier.
    float2 x[16];
    float hmax;
    {
      uint32_t sr[32];
      tmem_ld32(s_addr, sr);
      tmem_wait_ld();
      stamp(j, 1);
      if constexpr (INSTR) {
        if (dbg && j == 0) {
#pragma unroll
          for (int i = 0; i < 32; ++i) p.debug[r * 64 + h * 32 + i] = sr[i];
        }
      }
      const float2 a2 = make_float2(a, a);
#pragma unroll
      for (int i = 0; i < 16; i += 2) {
        const float4 c4 = ld_shared_f4(cb + 2 * i);
        x[i] = __ffma2_rn(make_float2(static_cast<float>(static_cast<int>(sr[2 * i])),
                                      static_cast<float>(static_cast<int>(sr[2 * i + 1]))),
                          a2, make_float2(c4.x, c4.y));
        x[i + 1] = __ffma2_rn(make_float2(static_cast<float>(static_cast<int>(sr[2 * i + 2])),
                                          static_cast<float>(static_cast<int>(sr[2 * i + 3]))),
                              a2, make_float2(c4.z, c4.w));
      }
      if constexpr (MASK) {
        const int key0 = j * 64 + h * 32;
        const int lim = CAUSAL ? min(row_g + 1, p.N) : p.N;  // keys >= lim are masked
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          if (key0 + 2 * i >= lim) x[i].x = -INFINITY;
          if (key0 + 2 * i + 1 >= lim) x[i].y = -INFINITY;
        }
      }
      hmax = fmax3(x[0].x, x[0].y, x[1].x);
#pragma unroll
      for (int i = 1; i < 15; ++i) hmax = fmax3(hmax, x[i].y, x[i + 1].x);
      hmax = fmaxf(hmax, x[15].y);
    }
    // Tile-max candidate: rowmax - m_new = min(0, rowmax - m_old) = max over halves of
    // min(0, halfmax - m_old), so each half contributes without knowing its partner.
    float d_r = row_valid ? fminf(0.0f, hmax - m_run) : -INFINITY;
    if (m_run == -INFINITY) d_r = row_valid && hmax != -INFINITY ? 0.0f : d_r;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d_r = fmaxf(d_r, __shfl_xor_sync(0xffffffffu, d_r, o));
    float* hm_j = halfmax + (j & 1) * 256;
    float* red_j = red + (j & 1) * 8;
    hm_j[h * 128 + r] = hmax;
    if (lane == 0) red_j[warp] = d_r;
    stamp(j, 2);
    named_bar_sync(1, 256);
    stamp(j, 3);
    const float rmax = fmaxf(hmax, hm_j[(h ^ 1) * 128 + r]);
    const float4 ra = ld_shared_f4(red_j), rb = ld_shared_f4(red_j + 4);
    const float Dt = fmaxf(fmaxf(fmaxf(ra.x, ra.y), fmaxf(ra.z, ra.w)), fmaxf(fmaxf(rb.x, rb.y), fmaxf(rb.z, rb.w)));
    const float m_new = fmaxf(m_run, rmax);
    const float m_eff = (m_new == -INFINITY) ? 0.0f : (m_new + Dt - p.log2_pr);
    const float2 nme2 = make_float2(-m_eff, -m_eff);
    // ---- pass 2: P~/dP = exp2(t - m_new) * p_r / tilemax = exp2(t - m_eff); E4M3 RNE satfinite
    float2 rs = make_float2(0.0f, 0.0f);
    uint32_t pk[8];
    {
      stamp(j, 4);
#pragma unroll
      for (int i = 0; i < 16; i += 2) {
        const float2 u0 = __fadd2_rn(x[i], nme2);
        const float2 u1 = __fadd2_rn(x[i + 1], nme2);
        const float2 e0 = make_float2(ex2(u0.x), ex2(u0.y));
        const float2 e1 = make_float2(ex2(u1.x), ex2(u1.y));
        rs = __fadd2_rn(rs, __fadd2_rn(e0, e1));
        pk[i / 2] = pack_e4m3x2(e0.x, e0.y) | (pack_e4m3x2(e1.x, e1.y) << 16);
      }
    }
    const float dP = ex2(Dt) * p.inv_pr;  // (tile max of P~) / p_r   (quantization.py:172)
    const float alpha = ex2(m_run - m_new);
    l_half = l_half * alpha + (rs.x + rs.y) * dP;
    if (tid < D) fbuf[(j & 1) * D + tid] = dP * ld_shared_f32(meta + 4 + tid);
    if (p.report != nullptr && tid == 0) {
      atomicMin(&p.report->p_scale_min_bits, __float_as_uint(dP));
      atomicMax(&p.report->p_scale_max_bits, __float_as_uint(dP));
    }
    // P^(j) goes to TMEM first so its registers are free during the promotion; PV(j) is issued
    // only once all eight warps have arrived below, which also certifies that PV(j-1) was drained.
    stamp(j, 5);
    tmem_st8(s_addr, pk);
    tmem_wait_st();
    if (j > 0) promote(j - 1);
    stamp(j, 7);
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();  // release this warp's P^ stores / PV reads to the last arriver
      if (atomicAdd(&arrive_cnt[j & 1], 1) == 7) {
        arrive_cnt[j & 1] = 0;
        __threadfence_block();
        tc_fence_after();
        issue_block_end(j);
      }
    }
    __syncwarp();
    resc_prev = (m_new != m_run);
    alpha_prev = alpha;
    m_run = m_new;
  };

  // Blocks entirely below the causal diagonal and inside the sequence need no mask.
  const int n_plain = CAUSAL ? min(nblk, q0 / 64) : ((p.N % 64 == 0) ? nblk : nblk - 1);
  int j = 0;
  for (; j < n_plain; ++j) block(j, std::false_type{});
  for (; j < nblk; ++j) block(j, std::true_type{});

  float* lbuf = reinterpret_cast<float*>(smem + C::kOffL);
  lbuf[h * 128 + r] = l_half;
  named_bar_sync(1, 256);  // last block's fbuf and both half-row sums visible
  promote(nblk - 1);
  if (want_overflow && overflow) atomicAdd(&p.report->overflow_events, overflow);
  if (row_valid) {
    const float l = l_half + lbuf[(h ^ 1) * 128 + r];
    const float inv_l = 1.0f / (l == 0.0f ? 1.0f : l);
    OutT* dst = reinterpret_cast<OutT*>(p.out) + b * p.o_sb + hq * p.o_sh + static_cast<int64_t>(row_g) * p.o_sn +
                h * HD;
    store_out<HD, OutT>(dst, reinterpret_cast<const float(&)[HD]>(O), inv_l);
  }

  if constexpr (INSTR) {
    if (trc != nullptr && tid == 0) trc[2] = globaltimer();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
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

template <int D, bool CAUSAL, bool ACC16, bool INSTR, typename OutT>
static cudaError_t launch_t(const AttnParams& P, const sa2pp_quant& qt, cudaStream_t st) {
  using C = AttnCfg<D>;
  CUtensorMap mq, mk, mv;
  const CUtensorMapSwizzle swqk = (D == 128) ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  if (!make_map_2d(&mq, qt.q_codes, D, static_cast<uint64_t>(P.B) * P.Hq * P.Nq_pad, D, D, 128, swqk) ||
      !make_map_2d(&mk, qt.k_codes, D, static_cast<uint64_t>(P.B) * P.Hkv * P.Np, D, D, 64, swqk) ||
      !make_map_2d(&mv, qt.v_codes, P.Np, static_cast<uint64_t>(P.B) * P.Hkv * D, P.Np, 64, D,
                   CU_TENSOR_MAP_SWIZZLE_64B))
    return cudaErrorInvalidValue;
  auto kern = attn_fwd_kernel<D, CAUSAL, ACC16, INSTR, OutT>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid(P.n_qt, P.B * P.Hq);
  kern<<<grid, C::kThreads, C::kSmemBytes, st>>>(mq, mk, mv, P);
  return cudaGetLastError();
}

template <int D, bool CAUSAL, bool ACC16, bool INSTR>
static cudaError_t launch_outi(const AttnParams& P, const sa2pp_quant& qt, cudaStream_t st) {
  switch (P.out_dtype) {
    case SA2PP_F32: return launch_t<D, CAUSAL, ACC16, INSTR, float>(P, qt, st);
    case SA2PP_F16: return launch_t<D, CAUSAL, ACC16, INSTR, __half>(P, qt, st);
    case SA2PP_BF16: return launch_t<D, CAUSAL, ACC16, INSTR, __nv_bfloat16>(P, qt, st);
    default: return cudaErrorInvalidValue;
  }
}

// Instrumented variants (TMEM dumps, phase traces) are separate instantiations so the production
// kernel carries no debug branches.
template <int D, bool CAUSAL, bool ACC16>
static cudaError_t launch_out(const AttnParams& P, const sa2pp_quant& qt, cudaStream_t st) {
  if (P.debug != nullptr || P.trace != nullptr) return launch_outi<D, CAUSAL, ACC16, true>(P, qt, st);
  return launch_outi<D, CAUSAL, ACC16, false>(P, qt, st);
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
