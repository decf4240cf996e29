// Microbenchmarks of the sm_100a resources the attention kernel is bound by (B200, one SM).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2505_21136_b200/csrc \
//        tools/microbench.cu -o build/microbench
// Each test runs one CTA per SM on all SMs and reports per-SM throughput per clock.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#include "ptx.cuh"

using namespace sa2pp;

__device__ __forceinline__ uint64_t clk() {
  uint64_t c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}

// ---------------------------------------------------------------- TMEM load throughput
template <int MODE>  // 0: 32x32b.x32 b32, 1: 32x32b.x16.pack::16b
__global__ void tmem_ld_bench(int iters, uint32_t* sink, unsigned long long* cycles) {
  __shared__ uint32_t holder;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc(&holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = holder + ((static_cast<uint32_t>(warp & 3) * 32) << 16) + (warp / 4) * 32;
  uint32_t acc = 0;
  __syncthreads();
  const uint64_t t0 = clk();
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0) {
      uint32_t r[32];
      tmem_ld32(tm + (i & 3) * 64, r);
      tmem_wait_ld();
#pragma unroll
      for (int k = 0; k < 32; ++k) acc ^= r[k];
    } else {
      uint32_t r[16];
      tmem_ld16_pack16(tm + (i & 3) * 64, r);
      tmem_wait_ld();
#pragma unroll
      for (int k = 0; k < 16; ++k) acc ^= r[k];
    }
  }
  __syncthreads();
  const uint64_t t1 = clk();
  if (threadIdx.x == 0) atomicMax(cycles, t1 - t0);
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(holder, 512);
}

// ---------------------------------------------------------------- ALU/XU throughputs
template <int OP>
__global__ void alu_bench(int iters, float* sink, unsigned long long* cycles) {
  float a[8], b2 = 1.0001f;
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3f + k;
  uint32_t u[8];
  for (int k = 0; k < 8; ++k) u[k] = threadIdx.x + k;
  float2 f2[8];
  for (int k = 0; k < 8; ++k) f2[k] = make_float2(a[k], a[k] + 1);
  __syncthreads();
  const uint64_t t0 = clk();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (OP == 0) a[k] = ex2(a[k] * -0.001f);                 // MUFU.EX2 (+FMUL)
      if (OP == 1) f2[k] = __ffma2_rn(f2[k], make_float2(b2, b2), make_float2(1e-7f, 1e-7f));  // FFMA2
      if (OP == 2) a[k] = __int_as_float(static_cast<int>(u[k] += 3)) + static_cast<float>(static_cast<int>(u[k]));  // I2FP
      if (OP == 3) u[k] = pack_e4m3x2(a[k], a[k] + 1.f) ^ u[k];  // F2FP e4m3
      if (OP == 4) a[k] = fmax3(a[k], a[(k + 1) & 7] * 0.5f, a[(k + 2) & 7]);  // FMNMX3 (+FMUL)
      if (OP == 5) a[k] = fmaf(a[k], b2, 1e-7f);               // FFMA
      if (OP == 6) {                                           // HADD2.F32 (f16 -> f32), 2 per reg
        const __half2 h = *reinterpret_cast<const __half2*>(&u[k]);
        const float2 g = __half22float2(h);
        a[k] += g.x * g.y;
        u[k] += 0x00010001u;
      }
      if (OP == 7) a[k] = __int_as_float(static_cast<int>(u[k] += 0x4B400000u)) * b2;  // VIADD magic (+FMUL)
      if (OP == 8) u[k] = __float_as_uint(__int2float_rn(static_cast<int>(u[k]) >> 3));  // I2F
    }
  }
  const uint64_t t1 = clk();
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(cycles, t1 - t0);
  float s = 0;
  for (int k = 0; k < 8; ++k) s += a[k] + f2[k].x + f2[k].y + u[k];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// ---------------------------------------------------------------- UMMA throughput
// kind: 0 = i8 SS  M128 N64 K32 (x4 per "tile": K=128), S32
//       1 = f8f6f4 TS M128 N128 K32 (x2: K=64), F16 acc
//       2 = f8f6f4 TS M128 N128 K32 (x2), F32 acc
template <int KIND>
__global__ void umma_bench(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t holder;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x / 32;
  uint8_t* base = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  for (int i = threadIdx.x; i < 32768; i += blockDim.x) base[i] = static_cast<uint8_t>(i * 7 + 1) & 0x3F;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  fence_proxy_async();
  if (warp == 0) tmem_alloc(&holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = holder;
  if (warp == 0 && threadIdx.x == 0) {
    const uint64_t t0 = clk();
    const uint64_t a = smem_desc(smem_u32(base), 1024, 2);
    const uint64_t b = smem_desc(smem_u32(base + 16384), 1024, 2);
    const uint64_t v = smem_desc(smem_u32(base + 16384), 512, 4);
    for (int i = 0; i < iters; ++i) {
      if (KIND == 0) {
        const uint32_t idesc = make_idesc(2, 1, 1, 128, 64);
#pragma unroll
        for (int k = 0; k < 4; ++k) umma_i8_ss(tm + (i & 1) * 64, a + 2 * k, b + 2 * k, idesc, k > 0);
      } else {
        const uint32_t idesc = make_idesc(KIND == 1 ? 0 : 1, 0, 0, 128, 128);
        umma_f8_ts(tm + 256, tm + (i & 1) * 64, v, idesc, 0);
        umma_f8_ts(tm + 256, tm + (i & 1) * 64 + 32, v + 2, idesc, 1);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    const uint64_t t1 = clk();
    atomicMax(cycles, t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(holder, 512);
}

template <typename K, typename... Args>
static double run(K kern, int grid, int block, int smem, Args... args) {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  cudaMemset(d, 0, 8);
  if (smem) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  kern<<<grid, block, smem>>>(args..., d);
  cudaMemset(d, 0, 8);
  kern<<<grid, block, smem>>>(args..., d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error: %s\n", cudaGetErrorString(e));
    return -1;
  }
  unsigned long long c;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return static_cast<double>(c);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* sinku;
  float* sinkf;
  cudaMalloc(&sinku, 4 * 1024 * 1024);
  cudaMalloc(&sinkf, 4 * 1024 * 1024);
  const int it = 4096;
  for (int warps : {4, 8, 16}) {
    double c = run(tmem_ld_bench<0>, sms, warps * 32, 0, it, sinku);
    printf("tmem ld 32x32b.x32 (f32) warps=%2d: %.1f B/clk/SM\n", warps, warps * 32.0 * 32 * 4 * it / c);
    c = run(tmem_ld_bench<1>, sms, warps * 32, 0, it, sinku);
    printf("tmem ld 32x32b.x16.pack16 (16b cols) warps=%2d: %.1f B/clk/SM (register bytes), %.1f cols*lanes/clk\n",
           warps, warps * 32.0 * 16 * 4 * it / c, warps * 32.0 * 32 * it / c);
  }
  const char* names[] = {"MUFU.EX2(+FMUL)", "FFMA2 (2 flops lanes)", "I2FP(+IADD,FADD)", "F2FP e4m3x2(+LOP)",
                         "FMNMX3(+FMUL)", "FFMA", "HADD2.F32 x2 (+FFMA)", "VIADD magic(+FMUL)", "I2F(+SHF)"};
  for (int warps : {8, 16}) {
    double c;
    c = run(alu_bench<0>, sms, warps * 32, 0, it, sinkf);
    printf("%-24s warps=%2d: %.1f ops/clk/SM\n", names[0], warps, warps * 32.0 * 8 * it / c);
    c = run(alu_bench<1>, sms, warps * 32, 0, it, sinkf);
    printf("%-24s warps=%2d: %.1f instr-lanes/clk/SM\n", names[1], warps, warps * 32.0 * 8 * it / c);
    c = run(alu_bench<2>, sms, warps * 32, 0, it, sinkf);
    printf("%-24s warps=%2d: %.1f ops/clk/SM\n", names[2], warps, warps * 32.0 * 8 * it / c);
    c = run(alu_bench<3>, sms, warps * 32, 0, it, sinkf);
    printf("%-24s warps=%2d: %.1f ops/clk/SM\n", names[3], warps, warps * 32.0 * 8 * it / c);
    c = run(alu_bench<4>, sms, warps * 32, 0, it, sinkf);
    printf("%-24s warps=%2d: %.1f ops/clk/SM\n", names[4], warps, warps * 32.0 * 8 * it / c);
    c = run(alu_bench<5>, sms, warps * 32, 0, it, sinkf);
    printf("%-24s warps=%2d: %.1f ops/clk/SM\n", names[5], warps, warps * 32.0 * 8 * it / c);
    for (int op = 6; op <= 8; ++op) {
      c = op == 6 ? run(alu_bench<6>, sms, warps * 32, 0, it, sinkf)
                  : op == 7 ? run(alu_bench<7>, sms, warps * 32, 0, it, sinkf) : run(alu_bench<8>, sms, warps * 32, 0, it, sinkf);
      printf("%-24s warps=%2d: %.1f ops/clk/SM\n", names[op], warps, warps * 32.0 * 8 * it / c);
    }
  }
  const int mit = 20000;
  double c0 = run(umma_bench<0>, sms, 128, 34 * 1024, mit);
  printf("UMMA i8 SS M128 N64 K128 (4 instr): %.0f MAC/clk/SM (%.1f clk per K128 tile)\n",
         128.0 * 64 * 128 * mit / c0, c0 / mit);
  double c1 = run(umma_bench<1>, sms, 128, 34 * 1024, mit);
  printf("UMMA f8f6f4 TS M128 N128 K64 F16 acc: %.0f MAC/clk/SM (%.1f clk per block)\n",
         128.0 * 128 * 64 * mit / c1, c1 / mit);
  double c2 = run(umma_bench<2>, sms, 128, 34 * 1024, mit);
  printf("UMMA f8f6f4 TS M128 N128 K64 F32 acc: %.0f MAC/clk/SM (%.1f clk per block)\n",
         128.0 * 128 * 64 * mit / c2, c2 / mit);
  return 0;
}
