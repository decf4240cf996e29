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
// Synchronisation per block is split so that no warp waits on the whole CTA before its exp2 work:
//   * the two warps sharing a row (w, w+4) swap half-row maxima through a 64-thread named barrier;
//   * the tile-wide P scale (quantization.py:163-175: delta_P = max|P~| / p_r over all 128x64) only
//     scales P^ *after* exp2: exp2(t - m_row) is computed first, the four h=0 warps publish their
//     rows' max-shift through a split-phase mbarrier (arrive early, wait after the exponentials),
//     and P^ = P~ * p_r * 2^-Dt is formed right before the E4M3 pack.
//
// Per block each softmax thread: tcgen05.ld S, dequant + bias in the log2 domain, causal/pad mask,
// half-row max, online softmax (attention.py:136-154) with l from the unquantized P~, one E4M3 scale
// per 128x64 tile, P^ -> TMEM, promotion of the previous block's PV: O = O*alpha + pv*(dP*dV[c])
// (attention.py:303); finally O / l (attention.py:304-305).
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
  static constexpr int kStages = (D == 128) ? 4 : 8;  // powers of two: stage/parity math is masks
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
  static constexpr int kOffF = kOffBias + kStages * kBiasBytes;     // [8][D/2] per-warp dP * dV
  static constexpr int kOffHalfMax = kOffF + 8 * (D / 2) * 4;             // [2][2][128] half-row maxima
  static constexpr int kOffRed = kOffHalfMax + 2 * 2 * 128 * 4;     // [2][4]   per-warp max-shift (-Dt candidates)
  static constexpr int kOffL = kOffRed + 2 * 4 * 4;                 // [2][128] final half-row sums
  static constexpr int kOffCnt = kOffL + 2 * 128 * 4;               // [2] per-parity warp arrival counters
  static constexpr int kOffBar = kOffCnt + 16;
  static constexpr int kNumBars = 1 + kStages + 2 + 2 + 1 + 2;
  static constexpr int kOffTmem = kOffBar + kNumBars * 8;
  static constexpr int kSmemBytes = kOffTmem + 16 + 1024;  // + alignment slack
  static constexpr int kThreads = 256;
  static_assert(2 * kSmemBytes <= 227 * 1024, "two CTAs per SM must fit in shared memory");
  static_assert((kStages & (kStages - 1)) == 0, "stage count must be a power of two");
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
  uint64_t* blk_done = bar_base + 1 + S;   // [2] all eight warps finished block j (P^ stored, PV drained)
  uint64_t* s_full = blk_done + 2;          // [2]
  uint64_t* pv_full = s_full + 2;           // [1]
  uint64_t* dt_bar = pv_full + 1;           // [2] the four h=0 warps published their max-shift
  int* issue_cnt = reinterpret_cast<int*>(smem + C::kOffCnt);  // [2] per-parity election counters
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + C::kOffTmem);

  if (warp == 0) {
    if (lane == 0) {
      mbar_init(q_full, 1);
      for (int s = 0; s < S; ++s) mbar_init(&kv_full[s], 1);
      mbar_init(&blk_done[0], 8);
      mbar_init(&blk_done[1], 8);
      mbar_init(&s_full[0], 1);
      mbar_init(&s_full[1], 1);
      mbar_init(pv_full, 1);
      mbar_init(&dt_bar[0], 4);
      mbar_init(&dt_bar[1], 4);
      issue_cnt[0] = issue_cnt[1] = 0;
      fence_barrier_init();
    }
    __syncwarp();
    tmem_alloc(tmem_holder, C::kTmemCols);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  // ---------------- MMA / TMA issue.  Runs warp-uniformly in one of the h=1 warps; the single-thread
  // instructions sit under elect.sync.  Everything here derives from blockIdx and the kernel
  // parameters only, so it lives in uniform registers, not in the softmax threads' register budget.
  const int kv_row = (b * p.Hkv + hkv) * p.Np;
  const int vt_row = (b * p.Hkv + hkv) * D;
  const float* meta_src = p.kv_meta + static_cast<int64_t>(b * p.Hkv + hkv) * p.n_kb * (4 + D);
  const float* bias_src = p.bias_l2 + static_cast<int64_t>(bh) * p.Np;
  constexpr uint32_t idesc_qk = make_idesc(2u, 1u, 1u, 128u, 64u);             // S32 <- s8 x s8
  constexpr uint32_t idesc_pv = make_idesc(ACC16 ? 0u : 1u, 0u, 0u, 128u, D);  // F16|F32 <- e4m3 x e4m3
  auto load_block = [&](int j) {  // one thread
    const int st = static_cast<int>(static_cast<unsigned>(j) % S);
    mbar_arrive_expect_tx(&kv_full[st], C::kKBytes + C::kVBytes + C::kMetaBytes + C::kBiasBytes);
    tma_load_2d(smem + C::kOffK + st * C::kKBytes, &tm_k, &kv_full[st], 0, kv_row + j * 64);
    tma_load_2d(smem + C::kOffV + st * C::kVBytes, &tm_v, &kv_full[st], j * 64, vt_row);
    bulk_load(smem + C::kOffMeta + st * C::kMetaBytes, meta_src + static_cast<int64_t>(j) * (4 + D), C::kMetaBytes,
              &kv_full[st]);
    bulk_load(smem + C::kOffBias + st * C::kBiasBytes, bias_src + j * 64, C::kBiasBytes, &kv_full[st]);
  };
  auto issue_qk = [&](int j) {  // one thread; K^_j must have landed
    const int st = static_cast<int>(static_cast<unsigned>(j) % S);
    const uint64_t qdesc = smem_desc(smem_u32(smem + C::kOffQ), C::kSboQK, C::kLayoutQK);
    const uint64_t kdesc = smem_desc(smem_u32(smem + C::kOffK + st * C::kKBytes), C::kSboQK, C::kLayoutQK);
    const uint32_t d_tm = tmem + (j & 1) * 64;
#pragma unroll
    for (int kk = 0; kk < D / 32; ++kk) umma_i8_ss(d_tm, qdesc + 2 * kk, kdesc + 2 * kk, idesc_qk, kk > 0 ? 1u : 0u);
    umma_commit(&s_full[j & 1]);
  };
  auto issue_pv = [&](int jj) {  // one thread; P^(jj) stored and PV(jj-1) drained by every warp
    const int stp = static_cast<int>(static_cast<unsigned>(jj) % S);
    const uint64_t vdesc = smem_desc(smem_u32(smem + C::kOffV + stp * C::kVBytes), C::kSboV, C::kLayoutV);
    const uint32_t a_tm = tmem + (jj & 1) * 64;
    umma_f8_ts(tmem + 128, a_tm, vdesc, idesc_pv, 0u);           // keys  0..31: P^ cols [0,8)
    umma_f8_ts(tmem + 128, a_tm + 32, vdesc + 2, idesc_pv, 1u);  // keys 32..63: P^ cols [32,40)
    umma_commit(pv_full);
  };
  // During block j, once every warp has finished block j-1 (blk_done):
  //   warp 4 + (j & 3):      PV(j-1) = P^(j-1).V^_{j-1}, then S(j+1) into the S buffer PV(j-1) reads
  //                          (tcgen05 MMAs from one thread execute in order);
  //   warp 4 + ((j+2) & 3):  the refill of the stage of block j-2, whose last readers (S(j-2),
  //                          PV(j-2), the promotion of j-2) are all done.
  auto issue_mma = [&](int j, unsigned long long* tr) {
    auto istamp = [&](int k) {
      if constexpr (INSTR) {
        if (tr != nullptr && j < 64) tr[(2 + j) * 128 + 8 + k] = clock64();
      }
    };
    istamp(0);
    mbar_wait_sleep(&blk_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
    tc_fence_after();
    istamp(1);
    const bool qk = j + 1 < nblk;
    if (qk) mbar_wait(&kv_full[static_cast<unsigned>(j + 1) % S], (static_cast<unsigned>(j + 1) / S) & 1);
    if (elect_one()) {
      issue_pv(j - 1);
      istamp(2);
      if (qk) issue_qk(j + 1);
      istamp(3);
    }
    __syncwarp();
  };
  auto issue_load = [&](int j) {
    mbar_wait_sleep(&blk_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
    if (elect_one()) load_block(j - 2 + S);
    __syncwarp();
  };
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    mbar_arrive_expect_tx(q_full, C::kQBytes);
    tma_load_2d(smem + C::kOffQ, &tm_q, q_full, 0, bh * p.Nq_pad + q0);
    for (int j = 0; j < min(S, nblk); ++j) load_block(j);
    mbar_wait(q_full, 0);
    mbar_wait(&kv_full[0], 0);
    issue_qk(0);
    if (nblk > 1) {
      mbar_wait(&kv_full[1], 0);
      issue_qk(1);
    }
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
  float* halfmax = reinterpret_cast<float*>(smem + C::kOffHalfMax);
  float* red = reinterpret_cast<float*>(smem + C::kOffRed);
  const bool dbg = INSTR && (p.debug != nullptr) && qt == 0 && bh == 0;
  unsigned long long* trc = (INSTR && p.trace != nullptr && bh == 0 && qt < 8 && lane == 0)
                                ? p.trace + static_cast<int64_t>(qt) * 66 * 128 + warp * 16
                                : nullptr;
  auto stamp = [&](int j, int k) {
    if constexpr (INSTR) {
      if (trc != nullptr && j < 64) trc[(2 + j) * 128 + k] = clock64();
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
  float m_run = -INFINITY, l_half = 0.0f, alpha_prev = 1.0f, dp_prev = 1.0f;
  bool resc_prev = true;
  uint32_t overflow = 0;
  const bool want_overflow = INSTR && ACC16 && p.report != nullptr;
  // per-warp promotion factors f[c] = dP_j * dV_j[c] for this warp's D/2 channels (written and read
  // by the same warp, so only __syncwarp orders them)
  float* fw = reinterpret_cast<float*>(smem + C::kOffF) + warp * HD;

  // O[c] = O[c]*alpha + pv[c]*f[c] for this thread's D/2 channels of row r (attention.py:303).
  // RESC: at least one row of the warp changed its running max, so O is rescaled by alpha.
  auto promote_impl = [&](int jj, auto resc_tag) {
    constexpr bool RESC = decltype(resc_tag)::value;
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
        for (int i = 0; i < CH / 2; ++i) pv[i] = f16x2_to_f32x2(v[i]);
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
        const float4 fv = ld_shared_f4(fw + c0 + 2 * i);
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
  // Promotion of block jj (its stage's dV is still resident: the stage is refilled two blocks later).
  auto promote = [&](int jj) {
    {
      const float* meta = reinterpret_cast<const float*>(smem + C::kOffMeta + (static_cast<unsigned>(jj) % S) * C::kMetaBytes);
      const float2 dv = *reinterpret_cast<const float2*>(meta + 4 + h * HD + 2 * (lane % (HD / 2)));
      if (2 * lane < HD) *reinterpret_cast<float2*>(fw + 2 * lane) = make_float2(dp_prev * dv.x, dp_prev * dv.y);
    }
    mbar_wait_sleep(pv_full, static_cast<uint32_t>(jj) & 1u);
    tc_fence_after();
    __syncwarp();
    stamp(jj + 1, 6);
    if (__any_sync(0xffffffffu, resc_prev)) {
      promote_impl(jj, std::true_type{});
    } else {
      promote_impl(jj, std::false_type{});
    }
  };

  // One key block.  MASK: causal diagonal / padded-tail block (attention.py:128-133, 293-294).
  // Pass 1 turns S into t (log2-domain scores) in place in TMEM and finds the row max; while the
  // tile-wide max-shift is gathered the first warp there issues the tensor work; pass 2 reads t
  // back and forms P^ with the final shift; then the previous block's PV is promoted.
  auto block = [&](int j, auto mask_tag, auto par_tag) {
    constexpr bool MASK = decltype(mask_tag)::value;
    constexpr int P = decltype(par_tag)::value;  // j & 1, a compile-time constant per instantiation
    const int st = static_cast<int>(static_cast<unsigned>(j) % S);
    mbar_wait_sleep(&kv_full[st], (static_cast<unsigned>(j) / S) & 1);
    mbar_wait_sleep(&s_full[P], (j >> 1) & 1);
    tc_fence_after();
    stamp(j, 0);
    const float* meta = reinterpret_cast<const float*>(smem + C::kOffMeta + st * C::kMetaBytes);
    const uint32_t s_addr = tm_row + P * 64 + h * 32;
    // ---- pass 1: t = S_int * (dQ dK sm_scale log2e) + bias_j * sm_scale log2e  (attention.py:287-292)
    float hmax;
    {
      const float* cb = reinterpret_cast<const float*>(smem + C::kOffBias + st * C::kBiasBytes) + h * 32;
      const float a = a_q * ld_shared_f32(meta);
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
      float2 x[16];
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
      {  // four independent max chains (latency), then combine
        float m4[4];
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          m4[q4] = fmax3(x[4 * q4].x, x[4 * q4].y, x[4 * q4 + 1].x);
          m4[q4] = fmax3(m4[q4], x[4 * q4 + 1].y, x[4 * q4 + 2].x);
          m4[q4] = fmax3(m4[q4], x[4 * q4 + 2].y, x[4 * q4 + 3].x);
          m4[q4] = fmaxf(m4[q4], x[4 * q4 + 3].y);
        }
        hmax = fmaxf(fmax3(m4[0], m4[1], m4[2]), m4[3]);
      }
      tmem_st32(s_addr, reinterpret_cast<const uint32_t(&)[32]>(x));
    }
    // ---- row max: swap half-row maxima with the partner warp (w ^ 4) only
    float* hm_j = halfmax + P * 256;
    hm_j[h * 128 + r] = hmax;
    stamp(j, 2);
    named_bar_sync(1 + wq, 64);
    stamp(j, 3);
    const float rmax = fmaxf(hmax, hm_j[(h ^ 1) * 128 + r]);
    const float m_new = fmaxf(m_run, rmax);
    // ---- tile-max candidate: rowmax - m_new = min(0, rowmax - m_old); the warps of one half
    //      publish -that (>= 0, +inf for rows that do not count) as float bits, min-reduced.
    if (h == 0) {
      const float v = (row_valid && rmax != -INFINITY) ? fmaxf(0.0f, m_run - rmax) : INFINITY;
      const uint32_t vmin = __reduce_min_sync(0xffffffffu, __float_as_uint(v));
      if (lane == 0) {
        red[P * 4 + wq] = __uint_as_float(vmin);
        mbar_arrive(&dt_bar[P]);  // release: the store above is visible to every waiter
      }
      stamp(j, 13);
    }
    // ---- one of the h=1 warps (they publish nothing, so they reach this point first) issues
    //      PV(j-1), S(j+1) and a stage refill while the tile-max candidates are being gathered
    if (j > 0 && warp == 4 + (j & 3)) issue_mma(j, trc);
    if (j >= 2 && j - 2 + S < nblk && warp == 4 + ((j + 2) & 3)) issue_load(j);
    const float alpha = (m_new == -INFINITY) ? 1.0f : ex2(m_run - m_new);
    // ---- pass 2a (before the tile-wide shift is known): e = P~ * p_r = exp2(t - m_new + log2 p_r);
    //      l accumulates the unquantized P~ (attention.py:149-153)
    const float m_eff = (m_new == -INFINITY) ? 0.0f : (m_new - p.log2_pr);
    const float2 nme2 = make_float2(-m_eff, -m_eff);
    float2 e[16];
    {
      tmem_wait_st();  // t stored by pass 1
      uint32_t tr[32];
      tmem_ld32(s_addr, tr);
      tmem_wait_ld();
      const float2* t2 = reinterpret_cast<const float2*>(tr);
      float2 rs[4] = {make_float2(0.0f, 0.0f), make_float2(0.0f, 0.0f), make_float2(0.0f, 0.0f),
                      make_float2(0.0f, 0.0f)};
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float2 u = __fadd2_rn(t2[i], nme2);
        e[i] = make_float2(ex2(u.x), ex2(u.y));
        rs[i & 3] = __fadd2_rn(rs[i & 3], e[i]);
      }
      const float2 r2 = __fadd2_rn(__fadd2_rn(rs[0], rs[1]), __fadd2_rn(rs[2], rs[3]));
      l_half = l_half * alpha + (r2.x + r2.y) * p.inv_pr;
    }
    // ---- tile scale (quantization.py:163-175): dP = max P~ / p_r = 2^Dt / p_r,
    //      Dt = max over the tile of (rowmax - m_new) <= 0;  P^ = P~ / dP = e * 2^-Dt
    stamp(j, 14);
    mbar_wait(&dt_bar[P], (j >> 1) & 1);
    stamp(j, 4);
    const float4 rv = ld_shared_f4(red + P * 4);
    float sh = fminf(fminf(rv.x, rv.y), fminf(rv.z, rv.w));  // -Dt >= 0
    sh = (sh == INFINITY) ? 0.0f : sh;
    const float dP = ex2(-sh) * p.inv_pr;
    if (INSTR && p.report != nullptr && tid == 0) {
      atomicMin(&p.report->p_scale_min_bits, __float_as_uint(dP));
      atomicMax(&p.report->p_scale_max_bits, __float_as_uint(dP));
    }
    if (sh != 0.0f) {  // tile-uniform
      const float sc = ex2(sh);
      const float2 sc2 = make_float2(sc, sc);
#pragma unroll
      for (int i = 0; i < 16; ++i) e[i] = __fmul2_rn(e[i], sc2);
    }
    uint32_t pk[8];
#pragma unroll
    for (int i = 0; i < 16; i += 2) pk[i / 2] = pack_e4m3x2(e[i].x, e[i].y) | (pack_e4m3x2(e[i + 1].x, e[i + 1].y) << 16);
    stamp(j, 5);
    tmem_st8(s_addr, pk);
    // ---- promotion of block j-1 (PV(j-1) was issued during this block's tile-max wait)
    if (j > 0) promote(j - 1);
    tmem_wait_st();
    stamp(j, 7);
    // P^(j) is in TMEM and PV(j-1) was drained: this warp is done with block j.
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&blk_done[P]);
    resc_prev = (m_new != m_run);
    alpha_prev = alpha;
    dp_prev = dP;
    m_run = m_new;
  };

  // Blocks entirely below the causal diagonal and inside the sequence need no mask.
  const int n_plain = CAUSAL ? min(nblk, q0 / 64) : ((p.N % 64 == 0) ? nblk : nblk - 1);
  int j = 0;
  using P0 = std::integral_constant<int, 0>;
  using P1 = std::integral_constant<int, 1>;
  for (; j + 1 < n_plain; j += 2) {
    block(j, std::false_type{}, P0{});
    block(j + 1, std::false_type{}, P1{});
  }
  if (j < n_plain) {
    block(j, std::false_type{}, P0{});
    ++j;
  }
  for (; j < nblk; ++j) {
    if (j & 1) {
      block(j, std::true_type{}, P1{});
    } else {
      block(j, std::true_type{}, P0{});
    }
  }

  // ---- PV of the last block, then its promotion and the normalisation O / l
  if (warp == 0) {
    mbar_wait_sleep(&blk_done[(nblk - 1) & 1], ((nblk - 1) >> 1) & 1);
    tc_fence_after();
    if (elect_one()) issue_pv(nblk - 1);
    __syncwarp();
  }
  float* lbuf = reinterpret_cast<float*>(smem + C::kOffL);
  lbuf[h * 128 + r] = l_half;
  named_bar_sync(1 + wq, 64);  // the partner's half-row sum
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
EncodeTiledFn get_encode_fn() {
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

bool make_map_2d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t rows, uint64_t row_bytes,
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
  static PerDevice once;
  cudaError_t e = once.run([&](std::atomic<int>&) {
    cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    if (r == cudaSuccess) r = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    return r;
  });
  if (e != cudaSuccess) return e;
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

// Instrumented variants (RunReport counters, TMEM dumps, phase traces) are separate instantiations so
// the production kernel carries no debug branches.
template <int D, bool CAUSAL, bool ACC16>
static cudaError_t launch_out(const AttnParams& P, const sa2pp_quant& qt, cudaStream_t st) {
  if (P.debug != nullptr || P.trace != nullptr || P.report != nullptr)
    return launch_outi<D, CAUSAL, ACC16, true>(P, qt, st);
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
