// Issue and completion latency of tcgen05.mma from one thread (B200, one CTA per SM), idle and with
// other warps streaming tcgen05.ld (the promotion's TMEM traffic) and FFMA work at the same time.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_2505_21136_b200/csrc \
//        tools/umma_latency.cu -o build/umma_latency
#include <cuda.h>
#include <cstdio>
#include <cstdint>

#include "ptx.cuh"

using namespace sa2pp;

__device__ __forceinline__ uint64_t clk() {
  uint64_t c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}

// LOAD: 0 idle, 1 = warps 4..7 stream tcgen05.ld over PV-like columns, 2 = they run FFMA chains
template <int KIND, int LOAD>
__global__ void lat_bench(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t holder;
  __shared__ uint64_t bar;
  __shared__ volatile int stop;
  const int warp = threadIdx.x / 32;
  uint8_t* base = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  for (int i = threadIdx.x; i < 32768; i += blockDim.x) base[i] = static_cast<uint8_t>(i * 7 + 1) & 0x3F;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
    stop = 0;
  }
  fence_proxy_async();
  if (warp == 0) tmem_alloc(&holder, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = holder;
  if (warp == 0) {
    if (threadIdx.x == 0) {
      uint64_t issue = 0, total = 0;
      const uint64_t a = smem_desc(smem_u32(base), 1024, 2);
      const uint64_t b = smem_desc(smem_u32(base + 16384), 1024, 2);
      const uint64_t v = smem_desc(smem_u32(base + 16384), 512, 4);
      for (int i = 0; i < iters; ++i) {
        const uint64_t t0 = clk();
        if (KIND == 2) {  // one PV MMA
          const uint32_t idesc = make_idesc(0, 0, 0, 128, 128);
          umma_f8_ts(tm + 128, tm + (i & 1) * 64, v, idesc, 0);
        } else if (KIND == 3) {  // eight QK MMAs (two tiles)
          const uint32_t idesc = make_idesc(2, 1, 1, 128, 64);
#pragma unroll
          for (int k = 0; k < 8; ++k) umma_i8_ss(tm + (k >> 2) * 64, a + 2 * (k & 3), b + 2 * (k & 3), idesc, (k & 3) > 0);
        } else if (KIND == 4) {  // commit only
        } else if (KIND == 0) {  // QK: i8 SS M128 N64 K128 (4 instr)
          const uint32_t idesc = make_idesc(2, 1, 1, 128, 64);
#pragma unroll
          for (int k = 0; k < 4; ++k) umma_i8_ss(tm + (i & 1) * 64, a + 2 * k, b + 2 * k, idesc, k > 0);
        } else {  // PV: f8f6f4 TS M128 N128 K64 F16 (2 instr)
          const uint32_t idesc = make_idesc(0, 0, 0, 128, 128);
          umma_f8_ts(tm + 128, tm + (i & 1) * 64, v, idesc, 0);
          umma_f8_ts(tm + 128, tm + (i & 1) * 64 + 8, v + 2, idesc, 1);
        }
        umma_commit(&bar);
        const uint64_t t1 = clk();
        mbar_wait(&bar, i & 1);
        const uint64_t t2 = clk();
        issue += t1 - t0;
        total += t2 - t0;
      }
      atomicMax(&out[0], issue / iters);
      atomicMax(&out[1], total / iters);
      stop = 1;
    }
  } else if (warp >= 4 && LOAD != 0) {
    const uint32_t row = tm + ((static_cast<uint32_t>(warp & 3) * 32) << 16);
    uint32_t acc = 0;
    float f = threadIdx.x;
    while (!stop) {
      if (LOAD == 1) {
        uint32_t r[16];
        tmem_ld16_pack16(row + 128, r);
        tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < 16; ++k) acc += r[k];
      } else {
#pragma unroll
        for (int k = 0; k < 64; ++k) f = fmaf(f, 1.0001f, 0.5f);
      }
    }
    if (acc == 12345 || f == 1.0f) out[2] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(holder, 256);
}

template <int KIND, int LOAD>
static void run(const char* name, int sms) {
  unsigned long long* d;
  cudaMalloc(&d, 24);
  auto k = lat_bench<KIND, LOAD>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 34 * 1024);
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(d, 0, 24);
    k<<<sms, 256, 34 * 1024>>>(2000, d);
  }
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[3];
  cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
  printf("%-40s issue %5llu clk  issue->complete %5llu clk  (%s)\n", name, h[0], h[1], cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0, 0>("QK i8 SS 128x64x128, idle", sms);
  run<1, 0>("PV f8 TS 128x128x64 F16, idle", sms);
  run<2, 0>("1 PV MMA, idle", sms);
  run<3, 0>("8 QK MMAs, idle", sms);
  run<4, 0>("commit only, idle", sms);
  run<0, 1>("QK, 4 warps streaming tcgen05.ld", sms);
  run<1, 1>("PV, 4 warps streaming tcgen05.ld", sms);
  run<0, 2>("QK, 4 warps FFMA chains", sms);
  run<1, 2>("PV, 4 warps FFMA chains", sms);
  return 0;
}
