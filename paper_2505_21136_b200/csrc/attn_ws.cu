// SageAttention2++ forward on sm_100a, warp-specialised: INT8 QK^T and FP8 PV on tcgen05 tensor cores.
//
// One CTA (256 threads, two CTAs resident per SM) owns one 128-row query tile of one (batch, head) and
// walks the 64-key blocks in ascending order, which is part of the reference's numerical contract
// (lpattn attention.py:6-8).  Two warpgroups, one query row per thread in each:
//
//   softmax warps 0-3 (thread = row r, all 64 score columns of the block)
//     tcgen05.ld S -> t = S*(dQ dK sm_scale log2e) + bias_j*sm_scale log2e, causal/pad mask
//     (attention.py:285-294); row max in-thread; online softmax with l from the unquantized P~
//     (attention.py:136-154); the tile-wide P scale (quantization.py:163-175: dP = max|P~|/p_r over
//     128x64) from the four warps' max-shifts through a split-phase mbarrier (publish after the row
//     max, wait after the exponentials); P^ = E4M3(P~/dP) into TMEM over the S columns it read;
//     alpha_j (per row) and dP_j published for the promotion.
//   promotion warps 4-7 (thread = row r, all D output channels, O in registers)
//     O = O*alpha_j + pv_j*(dP_j*dV_j[c]) with pv_j the FP16 (or FP32) PV accumulator of block j
//     (mma.py:144-166, attention.py:303); at the end O / l (attention.py:304-305).
//     Warp 4 also issues, from one elected lane, once the softmax warps finished block j and the
//     promotion warps drained PV(j-1):
//       PV(j)   = P^(j).V^_j   kind::f8f6f4, A = P^ from TMEM, B = V^T from smem, M=128 N=D, two
//                              k=32 MMAs (the reference's depth-2 grouping), F16 or F32 accumulator
//       S(j+2)  = Q^.K^_(j+2)^T kind::i8, M=128 N=64 K=D, S32 into S[j&1] (after PV(j) read P^(j):
//                              tcgen05 MMAs from one thread execute in order)
//       TMA     refill of the stage block j-1 used (its last readers were PV(j-1) and its promotion).
//
// The softmax warps never wait for the promotion and vice versa except through the single PV
// accumulator, so block j's promotion overlaps block j+1's softmax.  Registers: setmaxnreg moves
// them from the softmax warpgroup (64 score registers) to the promotion warpgroup (D accumulators).
//
// TMEM (256 columns per CTA): S[0] [0,64), S[1] [64,128), PV [128, 128+D).  P^ of block j (E4M3, four
// keys per column) is written over S[j&1] columns [0,16) of the same lane.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda.h>
#include <cstdint>
#include <type_traits>

#include "ptx.cuh"
#include "sa2pp_internal.h"

// Tuning knobs (overridable with -D for A/B builds, tools/build_variant.py)
#ifndef SA2PP_WS_REG_SOFTMAX
#define SA2PP_WS_REG_SOFTMAX 88
#endif
#ifndef SA2PP_WS_PV_CHUNK
#define SA2PP_WS_PV_CHUNK 32
#endif
#ifndef SA2PP_WS_F_PREFETCH
#define SA2PP_WS_F_PREFETCH 0
#endif
#ifndef SA2PP_WS_PIPE
#define SA2PP_WS_PIPE 1
#endif
#ifndef SA2PP_WS_STAGES128
#define SA2PP_WS_STAGES128 4
#endif
#ifndef SA2PP_WS_STAGES64
#define SA2PP_WS_STAGES64 8
#endif
// mbarrier wait policy (ptx.cuh mbar_wait_mode) of the softmax and promotion warps
// timing probes (wrong results): half of the promotion's channels / half of the exponentials
#ifndef SA2PP_WS_PROBE_HALFPROMO
#define SA2PP_WS_PROBE_HALFPROMO 0
#endif
#ifndef SA2PP_WS_PROBE_HALFEXP
#define SA2PP_WS_PROBE_HALFEXP 0
#endif
// Softmax TMEM-load pipelining: 1 = S half 1 in flight while half 0 is converted, 2 = also the t reload
// of the exponential phase in two 16-column loads.  Measured: D=64 +2.0 % with 1 (+1.1 % with 2), D=128
// -0.6 % / -2.8 %, so the default is 1 at D=64 and 0 at D=128 (-1 = that default).
#ifndef SA2PP_WS_LDPIPE
#define SA2PP_WS_LDPIPE -1
#endif
#ifndef SA2PP_WS_WAIT_SM
#define SA2PP_WS_WAIT_SM 0
#endif
#ifndef SA2PP_WS_WAIT_PR
#define SA2PP_WS_WAIT_PR 0
#endif

namespace sa2pp {

template <int D>
struct WsCfg {
  static constexpr int kStages = (D == 128) ? SA2PP_WS_STAGES128 : SA2PP_WS_STAGES64;
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
  static constexpr int kColPV = 128;
  // D=64 leaves room for two PV accumulators (128 + 2*64 = 256 columns): PV(j+1) then runs while
  // block j is promoted.  D=128 has one.
  static constexpr int kNumPV = (D == 64) ? 2 : 1;
  // shared memory carve-up (offsets from a 1024-aligned base)
  static constexpr int kOffQ = 0;
  static constexpr int kOffK = kOffQ + kQBytes;
  static constexpr int kOffV = kOffK + kStages * kKBytes;
  static constexpr int kOffMeta = kOffV + kStages * kVBytes;
  static constexpr int kOffBias = kOffMeta + kStages * kMetaBytes;
  static constexpr int kOffF = kOffBias + kStages * kBiasBytes;  // [4 promotion warps][D] dP_j*dV_j[c]
  static constexpr int kOffAlpha = kOffF + 4 * D * 4;             // [4][128] alpha_j per row (j & 3)
  static constexpr int kOffDp = kOffAlpha + 4 * 128 * 4;          // [4] dP_j (j & 3)
  static constexpr int kOffRed = kOffDp + 4 * 4;                  // [2][4] per-warp max-shift candidates
  static constexpr int kOffL = kOffRed + 2 * 4 * 4;               // [128] final row sums
  static constexpr int kOffBar = kOffL + 128 * 4;
  static constexpr int kNumBars = 1 + kStages + 2 + 2 + 2 * kNumPV + 2 + 1;
  static constexpr int kOffTmem = kOffBar + kNumBars * 8;
  static constexpr int kSmemBytes = kOffTmem + 16 + 1024;  // + alignment slack
  // No ninth (MMA-issue) warp: the register file is split per SMSP (16384 each), so with 2 x 9 warps
  // one SMSP holds 6 warps and the launch allocation drops to 96 per thread (27648 per CTA), below the
  // 128 x (88 + 168) the two warpgroups need at D=128 (a D=64 variant measured neutral).
  static constexpr int kThreads = 256;
  static constexpr uint32_t kRegLaunch = 128;  // 65536 / (2 CTAs x 256 threads)
  // register split (setmaxnreg) at D=128; D=64 keeps the launch allocation everywhere
  static constexpr uint32_t kRegSoftmax = (D == 128) ? SA2PP_WS_REG_SOFTMAX : kRegLaunch;
  static constexpr uint32_t kRegPromote = (D == 128) ? 256 - SA2PP_WS_REG_SOFTMAX : kRegLaunch;
  static constexpr int kPvChunk16 = SA2PP_WS_PV_CHUNK;  // FP16-accumulator channels per TMEM load
  static constexpr int kLdPipe = SA2PP_WS_LDPIPE >= 0 ? SA2PP_WS_LDPIPE : (D == 64 ? 1 : 0);
  static_assert(128 * (kRegSoftmax + kRegPromote) <= kThreads * kRegLaunch,
                "the warpgroups share the launch register budget");
  static_assert(2 * kSmemBytes <= 227 * 1024, "two CTAs per SM must fit in shared memory");
  // block B's stage is refilled at issue iteration B - S + kNumPV (after the promotion of block
  // B - S), and iteration j waits for block j + 2 before issuing S(j+2): B - S + kNumPV < B - 2
  static_assert(kStages >= 3 + kNumPV, "too few K/V stages: the S(j+2) issue would wait for its own refill");
};

// MASKED: channels [d_out, N) are padding (head_dim 32 / 96 on the 64 / 128 kernels) and are not
// stored.  Padded problems run the INSTR instantiation (its report/debug/trace hooks are null-guarded),
// so the production kernel keeps its unmasked epilogue.
template <int N, bool MASKED, typename OutT>
__device__ __forceinline__ void store_row(OutT* dst, const float2 (&O)[N / 2], float inv_l, int d_out) {
  if constexpr (sizeof(OutT) == 4) {
#pragma unroll
    for (int c = 0; c < N / 2; c += 2) {
      if (!MASKED || 2 * c < d_out)
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(dst) + 2 * c) =
            make_float4(O[c].x * inv_l, O[c].y * inv_l, O[c + 1].x * inv_l, O[c + 1].y * inv_l);
    }
  } else {
#pragma unroll
    for (int c = 0; c < N / 2; c += 4) {
      uint32_t w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float a = O[c + i].x * inv_l, b = O[c + i].y * inv_l;
        if constexpr (std::is_same<OutT, __nv_bfloat16>::value) {
          __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
          w[i] = *reinterpret_cast<uint32_t*>(&h);
        } else {
          __half2 h = __floats2half2_rn(a, b);
          w[i] = *reinterpret_cast<uint32_t*>(&h);
        }
      }
      if (!MASKED || 2 * c < d_out) *reinterpret_cast<uint4*>(dst + 2 * c) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

template <int D, bool CAUSAL, bool ACC16, bool INSTR, typename OutT, int G>
__global__ void __launch_bounds__(WsCfg<D>::kThreads, 2)
    attn_ws_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                   const __grid_constant__ CUtensorMap tm_v, const AttnParams p) {
  using C = WsCfg<D>;
  constexpr int S = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // ---- work decode: grid = (n_qt, heads the unit range touches); CTA (x, y) is unit
  //      u = (b*Hq + h)*n_qt + qt of head bh = head0 + y, and exits unless u lies in [unit0, unit0 + units)
  //      (only the partial first/last heads of a q-tile shard have such CTAs); causal runs each head's
  //      heaviest query tiles first -- with tile_major (small problems whose K/V fit in L2) the grid is
  //      (heads, tiles) so every head's heaviest tile starts before any lighter one (LPT order)
  const bool tm = CAUSAL && p.tile_major != 0;
  const int bh = p.head0 + static_cast<int>(tm ? blockIdx.x : blockIdx.y);
  const int qt = CAUSAL ? (p.n_qt - 1 - static_cast<int>(tm ? blockIdx.y : blockIdx.x)) : static_cast<int>(blockIdx.x);
  {
    const int u = bh * p.n_qt + qt;
    if (u < p.unit0 || u >= p.unit0 + p.units) return;
  }
  const int b = bh / p.Hq;
  const int hq = bh % p.Hq;
  const int hkv = hq / p.group;
  const int q0 = qt * 128;
  const int nblk = CAUSAL ? min(p.n_kb, (min(q0 + 128, p.N) + 63) / 64) : p.n_kb;

  uint64_t* bar_base = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* q_full = bar_base;
  uint64_t* kv_full = q_full + 1;    // [S] TMA landed
  uint64_t* s_full = kv_full + S;    // [2] S(j) in TMEM
  uint64_t* p_ready = s_full + 2;    // [2] the 4 softmax warps stored P^(j) and published alpha_j, dP_j
  uint64_t* pv_full = p_ready + 2;          // [kNumPV] PV(j) in TMEM buffer j % kNumPV
  uint64_t* pv_free = pv_full + C::kNumPV;  // [kNumPV] the 4 promotion warps drained that buffer
  uint64_t* dt_bar = pv_free + C::kNumPV;   // [2] the 4 softmax warps published their max-shift
  uint64_t* l_ready = dt_bar + 2;    // [1] final row sums written
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + C::kOffTmem);
  float* alpha_s = reinterpret_cast<float*>(smem + C::kOffAlpha);
  float* dp_s = reinterpret_cast<float*>(smem + C::kOffDp);
  float* red = reinterpret_cast<float*>(smem + C::kOffRed);
  float* lbuf = reinterpret_cast<float*>(smem + C::kOffL);

  if (warp == 0) {
    if (lane == 0) {
      mbar_init(q_full, 1);
      for (int s = 0; s < S; ++s) mbar_init(&kv_full[s], 1);
      for (int x = 0; x < 2; ++x) {
        mbar_init(&s_full[x], 1);
        mbar_init(&p_ready[x], 4);
        mbar_init(&dt_bar[x], 4);
      }
      for (int x = 0; x < C::kNumPV; ++x) {
        mbar_init(&pv_full[x], 1);
        mbar_init(&pv_free[x], 4);
      }
      mbar_init(l_ready, 4);
      fence_barrier_init();
    }
    __syncwarp();
    tmem_alloc(tmem_holder, C::kTmemCols);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  const int wq = warp & 3;       // TMEM lane quarter of this warp
  const int r = wq * 32 + lane;  // query row within the tile
  const uint32_t tm_row = tmem + (static_cast<uint32_t>(wq * 32) << 16);
  const int row_g = q0 + r;
  const bool row_valid = row_g < p.N;
  // development trace (INSTR only): clock64 per (block < 64, warp, phase) of every tile of heads 0-2
  unsigned long long* trc = (INSTR && p.trace != nullptr && bh < 3 && lane == 0)
                                ? p.trace + static_cast<int64_t>(bh * p.n_qt + qt) * 66 * 128 +
                                      warp * 16
                                : nullptr;
  auto stamp = [&](int j, int k) {
    if constexpr (INSTR) {
      if (trc != nullptr && j < 64) trc[(2 + j) * 128 + k] = clock64();
    }
  };
  if constexpr (INSTR) {
    if (trc != nullptr && threadIdx.x == 0) {
      trc[0] = smid();
      trc[1] = globaltimer();
      trc[3] = nblk;
    }
  }

  if (warp < 4) {
    // =============================== softmax warpgroup ===============================
    if constexpr (C::kRegSoftmax < C::kRegLaunch) setmaxnreg_dec<C::kRegSoftmax>();
    const float a_q = p.q_scale[static_cast<int64_t>(bh) * p.n_qt + qt] * p.sm_scale_log2;
    const bool dbg = INSTR && (p.debug != nullptr) && qt == 0 && bh == 0;
    float m_run = -INFINITY, l_run = 0.0f;

    // One key block.  MASK: causal diagonal / padded-tail block (attention.py:128-133, 293-294).
    auto block = [&](int j, auto mask_tag) {
      constexpr bool MASK = decltype(mask_tag)::value;
      const int P = j & 1;
      const int st = static_cast<int>(static_cast<unsigned>(j) % S);
      stamp(j, 0);
      mbar_wait_mode<SA2PP_WS_WAIT_SM>(&kv_full[st], (static_cast<unsigned>(j) / S) & 1);  // bias / dK
      mbar_wait_mode<SA2PP_WS_WAIT_SM>(&s_full[P], (j >> 1) & 1);
      tc_fence_after();
      stamp(j, 1);
      const float* meta = reinterpret_cast<const float*>(smem + C::kOffMeta + st * C::kMetaBytes);
      const float* cb = reinterpret_cast<const float*>(smem + C::kOffBias + st * C::kBiasBytes);
      const uint32_t s_addr = tm_row + P * 64;
      const float a = a_q * ld_shared_f32(meta);
      const float2 a2 = make_float2(a, a);
      // ---- t = S_int * (dQ dK sm_scale log2e) + bias_j * sm_scale log2e  (attention.py:287-292),
      //      causal / pad mask, row max.  Half 0 (keys 0-31) goes back into TMEM over its S columns,
      //      half 1 stays in registers.
      // SA2PP_WS_LDPIPE: the S load of half 1 is issued before half 0 is converted (latency hidden);
      // `sr` then arrives loaded (pre = true) and is converted in place
      auto scores = [&](int hlf, float2 (&x)[16], uint32_t (&sr)[32], bool pre) {
        if (!pre) {
          tmem_ld32(s_addr + hlf * 32, sr);
          tmem_wait_ld();
        }
        if constexpr (INSTR) {
          if (dbg && j == 0) {
#pragma unroll
            for (int i = 0; i < 32; ++i) p.debug[r * 64 + hlf * 32 + i] = sr[i];
          }
        }
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
          const float4 c4 = ld_shared_f4(cb + hlf * 32 + 2 * i);
          x[i] = __ffma2_rn(make_float2(static_cast<float>(static_cast<int>(sr[2 * i])),
                                        static_cast<float>(static_cast<int>(sr[2 * i + 1]))),
                            a2, make_float2(c4.x, c4.y));
          x[i + 1] = __ffma2_rn(make_float2(static_cast<float>(static_cast<int>(sr[2 * i + 2])),
                                            static_cast<float>(static_cast<int>(sr[2 * i + 3]))),
                                a2, make_float2(c4.z, c4.w));
        }
        if constexpr (MASK) {
          const int lim = CAUSAL ? min(row_g + 1, p.N) : p.N;  // keys >= lim are masked
          const int key0 = j * 64 + hlf * 32;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            if (key0 + 2 * i >= lim) x[i].x = -INFINITY;
            if (key0 + 2 * i + 1 >= lim) x[i].y = -INFINITY;
          }
        }
        float m4[4];  // four independent max chains, then combine
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          m4[q4] = fmax3(x[4 * q4].x, x[4 * q4].y, x[4 * q4 + 1].x);
          m4[q4] = fmax3(m4[q4], x[4 * q4 + 1].y, x[4 * q4 + 2].x);
          m4[q4] = fmax3(m4[q4], x[4 * q4 + 2].y, x[4 * q4 + 3].x);
          m4[q4] = fmaxf(m4[q4], x[4 * q4 + 3].y);
        }
        return fmaxf(fmax3(m4[0], m4[1], m4[2]), m4[3]);
      };
      float2 x[16];
      float rmax;
      if constexpr (C::kLdPipe != 0) {
        uint32_t s0[32], s1[32];
        tmem_ld32(s_addr, s0);
        tmem_wait_ld();
        tmem_ld32(s_addr + 32, s1);  // in flight while half 0 is converted
        rmax = scores(0, x, s0, true);
        tmem_st32(s_addr, reinterpret_cast<const uint32_t(&)[32]>(x));
        tmem_wait_ld();
        rmax = fmaxf(rmax, scores(1, x, s1, true));
      } else {
        uint32_t sr[32];
        rmax = scores(0, x, sr, false);
        tmem_st32(s_addr, reinterpret_cast<const uint32_t(&)[32]>(x));
        rmax = fmaxf(rmax, scores(1, x, sr, false));
      }
      const float m_new = fmaxf(m_run, rmax);
      // ---- tile-max candidate: rowmax - m_new = min(0, rowmax - m_old); each warp publishes the
      //      min over its rows of -that (>= 0; +inf for rows that do not count) as float bits
      {
        const float v = (row_valid && rmax != -INFINITY) ? fmaxf(0.0f, m_run - rmax) : INFINITY;
        const uint32_t vmin = __reduce_min_sync(0xffffffffu, __float_as_uint(v));
        if (lane == 0) {
          red[P * 4 + wq] = __uint_as_float(vmin);
          mbar_arrive(&dt_bar[P]);  // release: the store above is visible to every waiter
        }
      }
      const float alpha = (m_new == -INFINITY) ? 1.0f : ex2(m_run - m_new);
      // ---- tile scale (quantization.py:163-175): dP = max P~ / p_r = 2^Dt / p_r with
      //      Dt = max over the tile of (rowmax - m_new) <= 0, so P^ = P~ / dP = exp2(t - m_new + log2 p_r - Dt)
      //      in one exponential; l accumulates the unquantized P~ = P^ * dP (attention.py:149-153)
      stamp(j, 2);
      mbar_wait(&dt_bar[P], (j >> 1) & 1);
      stamp(j, 3);
      const float4 rv = ld_shared_f4(red + P * 4);
      float sh = fminf(fminf(rv.x, rv.y), fminf(rv.z, rv.w));  // -Dt >= 0
      sh = (sh == INFINITY) ? 0.0f : sh;
      const float dP = ex2(-sh) * p.inv_pr;
      if (INSTR && p.report != nullptr && threadIdx.x == 0) {
        atomicMin(&p.report->p_scale_min_bits, __float_as_uint(dP));
        atomicMax(&p.report->p_scale_max_bits, __float_as_uint(dP));
      }
      const float m_eff = (m_new == -INFINITY) ? 0.0f : (m_new - p.log2_pr - sh);
      const float2 nme2 = make_float2(-m_eff, -m_eff);
      uint32_t pk[16];
      float2 rs[4] = {make_float2(0.0f, 0.0f), make_float2(0.0f, 0.0f), make_float2(0.0f, 0.0f),
                      make_float2(0.0f, 0.0f)};
      auto quant = [&](const float2 (&t)[16], int w0) {  // P^ codes of 32 keys into pk[w0, w0+8)
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
          const float2 u0 = __fadd2_rn(t[i], nme2), u1 = __fadd2_rn(t[i + 1], nme2);
          const float2 e0 = make_float2(ex2(u0.x), ex2(u0.y)), e1 = make_float2(ex2(u1.x), ex2(u1.y));
          rs[(i >> 1) & 3] = __fadd2_rn(rs[(i >> 1) & 3], __fadd2_rn(e0, e1));
          pk[w0 + i / 2] = pack_e4m3x2(e0.x, e0.y) | (pack_e4m3x2(e1.x, e1.y) << 16);
        }
      };
      if constexpr (C::kLdPipe >= 2) {
        // t of keys 0-15 / 16-31 reloaded in two 16-column loads, each in flight while the previous
        // 16 or 32 keys are exponentiated
        auto quant8 = [&](const float2 (&t)[8], int w0) {  // P^ codes of 16 keys into pk[w0, w0+4)
#pragma unroll
          for (int i = 0; i < 8; i += 2) {
            const float2 u0 = __fadd2_rn(t[i], nme2), u1 = __fadd2_rn(t[i + 1], nme2);
            const float2 e0 = make_float2(ex2(u0.x), ex2(u0.y)), e1 = make_float2(ex2(u1.x), ex2(u1.y));
            rs[(i >> 1) & 3] = __fadd2_rn(rs[(i >> 1) & 3], __fadd2_rn(e0, e1));
            pk[w0 + i / 2] = pack_e4m3x2(e0.x, e0.y) | (pack_e4m3x2(e1.x, e1.y) << 16);
          }
        };
        uint32_t ta[16], tb[16];
        tmem_wait_st();
        tmem_ld16(s_addr, ta);
        quant(x, 8);  // keys 32-63 (registers)
        tmem_wait_ld();
        tmem_ld16(s_addr + 16, tb);
        quant8(reinterpret_cast<const float2(&)[8]>(ta), 0);
        tmem_wait_ld();
        quant8(reinterpret_cast<const float2(&)[8]>(tb), 4);
      } else {
      quant(x, 8);  // keys 32-63 (registers)
      {
        tmem_wait_st();
        uint32_t tr[32];
        tmem_ld32(s_addr, tr);  // keys 0-31 (t stored above)
        tmem_wait_ld();
        if constexpr (SA2PP_WS_PROBE_HALFEXP) {  // timing probe only: wrong results
#pragma unroll
          for (int i = 0; i < 8; ++i) pk[i] = tr[i];
        } else {
          quant(reinterpret_cast<const float2(&)[16]>(tr), 0);
        }
      }
      }
      const float2 r2 = __fadd2_rn(__fadd2_rn(rs[0], rs[1]), __fadd2_rn(rs[2], rs[3]));
      l_run = l_run * alpha + (r2.x + r2.y) * dP;
      tmem_st16(s_addr, pk);
      alpha_s[(j & 3) * 128 + r] = alpha;
      if (threadIdx.x == 0) dp_s[j & 3] = dP;
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_ready[P]);  // release: alpha/dP stores and P^ in TMEM
      stamp(j, 4);
      m_run = m_new;
    };

    // Blocks entirely below the causal diagonal and inside the sequence need no mask.
    const int n_plain = CAUSAL ? min(nblk, q0 / 64) : ((p.N % 64 == 0) ? nblk : nblk - 1);
    int j = 0;
    for (; j < n_plain; ++j) block(j, std::false_type{});
    for (; j < nblk; ++j) block(j, std::true_type{});
    lbuf[r] = l_run;
    __syncwarp();
    if (lane == 0) mbar_arrive(l_ready);
  } else {
    // =============================== promotion warpgroup (+ issue) ===============================
    if constexpr (C::kRegPromote > C::kRegLaunch) setmaxnreg_inc<C::kRegPromote>();
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
    auto issue_pv = [&](int u, int j, int g) {  // one thread; P^(j) stored, the PV buffer drained
      const int st = static_cast<int>(static_cast<unsigned>(j) % S);
      const uint64_t vdesc = smem_desc(smem_u32(smem + C::kOffV + st * C::kVBytes), C::kSboV, C::kLayoutV);
      const uint32_t a_tm = tmem + (j & 1) * 64;
      const int pb = u % C::kNumPV;
      const uint32_t d_tm = tmem + C::kColPV + pb * D;
      if (G == 1) {  // depth 2: the two k=32 groups chain in the FP16 (or FP32) accumulator
        umma_f8_ts(d_tm, a_tm, vdesc, idesc_pv, 0u);          // keys  0..31: P^ cols [0,8)
        umma_f8_ts(d_tm, a_tm + 8, vdesc + 2, idesc_pv, 1u);  // keys 32..63: P^ cols [8,16)
      } else {       // depth 1: group g alone
        umma_f8_ts(d_tm, a_tm + 8 * g, vdesc + 2 * g, idesc_pv, 0u);
      }
      umma_commit(&pv_full[pb]);
    };
    if (warp == 4 && elect_one()) {
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

    const int pw = warp - 4;  // promotion warp index = TMEM lane quarter
    float* fw = reinterpret_cast<float*>(smem + C::kOffF) + pw * D;
    const bool dbg = INSTR && (p.debug != nullptr) && qt == 0 && bh == 0;
    const bool want_overflow = INSTR && ACC16 && p.report != nullptr;
    uint32_t overflow = 0;
    float2 O[D / 2];
#pragma unroll
    for (int c = 0; c < D / 2; ++c) O[c] = make_float2(0.0f, 0.0f);

    // Software-pipelined promotion of the FP16 accumulator (production, INSTR off): the TMEM load of
    // chunk c+1 (16 channels, 8 registers) is in flight while chunk c is converted and accumulated.
    auto promote_pipe = [&](uint32_t pv_col, float alpha, auto resc_tag) {
      constexpr bool RESC = decltype(resc_tag)::value;
      const float2 al2 = make_float2(alpha, alpha);
      constexpr int CH = 16, NC = D / CH / (SA2PP_WS_PROBE_HALFPROMO ? 2 : 1);  // (timing probe: half)
      uint32_t va[8], vb[8];
      tmem_ld8_pack16(tm_row + pv_col, va);
      tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        uint32_t(&cur)[8] = (c & 1) ? vb : va;
        uint32_t(&nxt)[8] = (c & 1) ? va : vb;
        if (c + 1 < NC) tmem_ld8_pack16(tm_row + pv_col + (c + 1) * CH, nxt);
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
          const float4 fv = *reinterpret_cast<const float4*>(fw + c * CH + 2 * i);
          const float2 p0 = f16x2_to_f32x2(cur[i]), p1 = f16x2_to_f32x2(cur[i + 1]);
          float2& o0 = O[c * CH / 2 + i];
          float2& o1 = O[c * CH / 2 + i + 1];
          if constexpr (RESC) {
            o0 = __ffma2_rn(p0, make_float2(fv.x, fv.y), __fmul2_rn(o0, al2));
            o1 = __ffma2_rn(p1, make_float2(fv.z, fv.w), __fmul2_rn(o1, al2));
          } else {
            o0 = __ffma2_rn(p0, make_float2(fv.x, fv.y), o0);
            o1 = __ffma2_rn(p1, make_float2(fv.z, fv.w), o1);
          }
        }
        reg_fence16(reinterpret_cast<float*>(&O[c * CH / 2]));
        if (c + 1 < NC) tmem_wait_ld();
      }
    };
    // O[c] = O[c]*alpha + pv[c]*f[c] for the row's D channels (attention.py:303).
    auto promote_impl = [&](int j, uint32_t pv_col, float alpha, auto resc_tag) {
      constexpr bool RESC = decltype(resc_tag)::value;
      const float2 al2 = make_float2(alpha, alpha);
      constexpr int CH = ACC16 ? C::kPvChunk16 : 16;  // channels per TMEM load
#pragma unroll
      for (int c0 = 0; c0 < D; c0 += CH) {
        float4 fpre[SA2PP_WS_F_PREFETCH ? CH / 4 : 1];
        if constexpr (SA2PP_WS_F_PREFETCH != 0) {  // f of this chunk in flight beside the TMEM load
#pragma unroll
          for (int i = 0; i < CH / 4; ++i) fpre[i] = *reinterpret_cast<const float4*>(fw + c0 + 4 * i);
        }
        float2 pv[CH / 2];
        if constexpr (ACC16) {
          uint32_t v[CH / 2];
          if constexpr (CH == 32) {
            tmem_ld16_pack16(tm_row + pv_col + c0, v);  // F16 accumulators, 2 per register
          } else {
            tmem_ld8_pack16(tm_row + pv_col + c0, v);
          }
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
          tmem_ld16(tm_row + pv_col + c0, v);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < CH / 2; ++i) pv[i] = make_float2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
        }
        if constexpr (INSTR) {
          if (dbg && j == 0) {
#pragma unroll
            for (int i = 0; i < CH / 2; ++i) {
              p.debug[128 * 64 + r * D + c0 + 2 * i] = __float_as_uint(pv[i].x);
              p.debug[128 * 64 + r * D + c0 + 2 * i + 1] = __float_as_uint(pv[i].y);
            }
          }
        }
#pragma unroll
        for (int i = 0; i < CH / 2; i += 2) {
          const float4 fv = SA2PP_WS_F_PREFETCH ? fpre[SA2PP_WS_F_PREFETCH ? i / 2 : 0] : ld_shared_f4(fw + c0 + 2 * i);
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

    // Sub-blocks: G = 1 normally; G = 2 for buffering depth 1 with the FP16 accumulator
    // (mma.py:144-152): each k=32 group of a block is its own FP16 accumulation, converted to FP32
    // and promoted on its own (the FP32 sum of the two groups is formed in O instead of in a
    // temporary, which differs only by FP32 rounding).
    for (int u = 0; u < nblk * G; ++u) {
      const int j = (G == 1) ? u : (u >> 1);
      const int g = (G == 1) ? 0 : (u & 1);
      const int st = static_cast<int>(static_cast<unsigned>(j) % S);
      const int pb = u % C::kNumPV;
      stamp(j, 0);
      if (warp == 4) {  // ---- issue PV(j) [group g], S(j+2), refill of block j-1's stage
        if (g == 0) mbar_wait_mode<SA2PP_WS_WAIT_PR>(&p_ready[j & 1], (j >> 1) & 1);
        stamp(j, 8);
        if (u >= C::kNumPV) mbar_wait(&pv_free[pb], (u / C::kNumPV - 1) & 1);
        stamp(j, 9);
        tc_fence_after();
        if (elect_one()) {  // one elected region: every UTC* op in a divergent region pays an ELECT loop
          issue_pv(u, j, g);
          if (g == G - 1) {  // P^(j) fully consumed once the last group's MMA is issued (in order)
            if (j + 2 < nblk) {
              mbar_wait(&kv_full[static_cast<unsigned>(j + 2) % S], (static_cast<unsigned>(j + 2) / S) & 1);
              issue_qk(j + 2);
            }
          }
          // the stage of block j-1: the promotion that last read it was waited for just above
          const int jr = (u - C::kNumPV) / G;  // block whose promotion is complete
          if (u >= C::kNumPV && (u - C::kNumPV) % G == G - 1 && jr + S < nblk) load_block(jr + S);
        }
        __syncwarp();
        stamp(j, 12);
      }
      // ---- promotion of block j (group g): f[c] = dP_j * dV_j[c] for this warp's copy
      mbar_wait_mode<SA2PP_WS_WAIT_PR>(&kv_full[st], (static_cast<unsigned>(j) / S) & 1);  // dV visible
      stamp(j, 1);
      mbar_wait_mode<SA2PP_WS_WAIT_PR>(&pv_full[pb], static_cast<uint32_t>(u / C::kNumPV) & 1u);
      tc_fence_after();
      stamp(j, 2);
      const float dP = dp_s[j & 3];
      const float alpha = g == 0 ? alpha_s[(j & 3) * 128 + r] : 1.0f;
      if (g == 0) {
        const float* meta = reinterpret_cast<const float*>(smem + C::kOffMeta + st * C::kMetaBytes);
#pragma unroll
        for (int c = 4 * lane; c < D; c += 128) {
          const float4 dv = ld_shared_f4(meta + 4 + c);
          *reinterpret_cast<float4*>(fw + c) = make_float4(dP * dv.x, dP * dv.y, dP * dv.z, dP * dv.w);
        }
      }
      __syncwarp();
      // the pipelined promotion is the production path; the instrumented build keeps it too unless a
      // debug dump or the overflow count needs the chunked variant (so traces time the real code)
      constexpr bool kPipeOk = SA2PP_WS_PIPE != 0 && ACC16;
      const bool pipe = kPipeOk && (!INSTR || (!dbg && !want_overflow));
      const uint32_t pv_col = C::kColPV + pb * D;
      if (__any_sync(0xffffffffu, alpha != 1.0f)) {
        if (pipe) {
          if constexpr (kPipeOk) promote_pipe(pv_col, alpha, std::true_type{});
        } else {
          promote_impl(j, pv_col, alpha, std::true_type{});
        }
      } else {
        if (pipe) {
          if constexpr (kPipeOk) promote_pipe(pv_col, alpha, std::false_type{});
        } else {
          promote_impl(j, pv_col, alpha, std::false_type{});
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&pv_free[pb]);
      stamp(j, 3);
    }
    if (want_overflow && overflow) atomicAdd(&p.report->overflow_events, overflow);
    // ---- O / l (attention.py:304-305)
    mbar_wait_sleep(l_ready, 0);
    if (row_valid) {
      const float l = lbuf[r];
      const float inv_l = 1.0f / (l == 0.0f ? 1.0f : l);
      OutT* dst = reinterpret_cast<OutT*>(p.out) + b * p.o_sb + hq * p.o_sh + static_cast<int64_t>(row_g) * p.o_sn;
      store_row<D, INSTR, OutT>(dst, O, inv_l, p.d_out);
    }
  }

  tc_fence_before();
  __syncthreads();
  if constexpr (INSTR) {
    if (trc != nullptr && threadIdx.x == 0) trc[2] = globaltimer();
  }
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, C::kTmemCols);
  }
}

// ------------------------------------------------------------------ host side
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda at link time); the
// static is written with the same value by any racing first callers.
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

template <int D, bool CAUSAL, bool ACC16, bool INSTR, typename OutT, int G>
static cudaError_t launch_ws_t(const AttnParams& P, const sa2pp_quant& qt, cudaStream_t st) {
  using C = WsCfg<D>;
  CUtensorMap mq, mk, mv;
  const CUtensorMapSwizzle swqk = (D == 128) ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  if (!make_map_2d(&mq, qt.q_codes, D, static_cast<uint64_t>(P.B) * P.Hq * P.Nq_pad, D, D, 128, swqk) ||
      !make_map_2d(&mk, qt.k_codes, D, static_cast<uint64_t>(P.B) * P.Hkv * P.Np, D, D, 64, swqk) ||
      !make_map_2d(&mv, qt.v_codes, P.Np, static_cast<uint64_t>(P.B) * P.Hkv * D, P.Np, 64, D,
                   CU_TENSOR_MAP_SWIZZLE_64B))
    return cudaErrorInvalidValue;
  auto kern = attn_ws_kernel<D, CAUSAL, ACC16, INSTR, OutT, G>;
  static PerDevice once;
  cudaError_t e = once.run([&](std::atomic<int>&) {
    cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    if (r == cudaSuccess) r = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    return r;
  });
  if (e != cudaSuccess) return e;
  if (P.units <= 0) return cudaSuccess;
  const int h1 = (P.unit0 + P.units - 1) / P.n_qt;
  const dim3 grid = (CAUSAL && P.tile_major) ? dim3(h1 - P.head0 + 1, P.n_qt) : dim3(P.n_qt, h1 - P.head0 + 1);
  kern<<<grid, C::kThreads, C::kSmemBytes, st>>>(mq, mk, mv, P);
  return cudaGetLastError();
}

template <int D, bool CAUSAL, bool ACC16, bool INSTR, int G>
static cudaError_t launch_ws_outi(const AttnParams& P, const sa2pp_quant& qt, cudaStream_t st) {
  switch (P.out_dtype) {
    case SA2PP_F32: return launch_ws_t<D, CAUSAL, ACC16, INSTR, float, G>(P, qt, st);
    case SA2PP_F16: return launch_ws_t<D, CAUSAL, ACC16, INSTR, __half, G>(P, qt, st);
    case SA2PP_BF16: return launch_ws_t<D, CAUSAL, ACC16, INSTR, __nv_bfloat16, G>(P, qt, st);
    default: return cudaErrorInvalidValue;
  }
}

template <int D, bool CAUSAL, bool ACC16, int G>
static cudaError_t launch_ws_out(const AttnParams& P, const sa2pp_quant& qt, cudaStream_t st) {
  if (P.debug != nullptr || P.report != nullptr || P.trace != nullptr || P.d_out < D)
    return launch_ws_outi<D, CAUSAL, ACC16, true, G>(P, qt, st);
  return launch_ws_outi<D, CAUSAL, ACC16, false, G>(P, qt, st);
}

template <int D>
static cudaError_t launch_ws_d(const sa2pp_problem& prob, const AttnParams& P, const sa2pp_quant& qt,
                               cudaStream_t st) {
  const bool acc16 = prob.pv_accum == SA2PP_ACC_F16;
  if (acc16 && prob.buffering_depth == 1) {  // FP16 accumulation per k=32 group (mma.py:144-152)
    return prob.causal ? launch_ws_out<D, true, true, 2>(P, qt, st) : launch_ws_out<D, false, true, 2>(P, qt, st);
  }
  if (prob.causal) {
    return acc16 ? launch_ws_out<D, true, true, 1>(P, qt, st) : launch_ws_out<D, true, false, 1>(P, qt, st);
  }
  return acc16 ? launch_ws_out<D, false, true, 1>(P, qt, st) : launch_ws_out<D, false, false, 1>(P, qt, st);
}

cudaError_t launch_attn_ws(const sa2pp_problem& prob, const AttnParams& P, const sa2pp_quant& qt, cudaStream_t st) {
  if (padded_dim(prob.head_dim) == 128) return launch_ws_d<128>(prob, P, qt, st);
  if (padded_dim(prob.head_dim) == 64) return launch_ws_d<64>(prob, P, qt, st);
  return cudaErrorInvalidValue;
}

}  // namespace sa2pp
