// Issue throughput of the softmax/promotion instruction mix on sm_100a: 8 independent chains per
// thread, 16 warps per SM on every SM; reports warp-instructions per clock per SM (4.0 = one per
// scheduler per clock).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/pipe_bench.cu
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint64_t clk() {
  uint64_t c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}

template <int OP>
__global__ void bench(int iters, uint32_t* sink, unsigned long long* cyc) {
  uint32_t r[8];
  float f[8];
  for (int i = 0; i < 8; ++i) {
    r[i] = threadIdx.x * 2654435761u + i * 40503u;
    f[i] = 1.0f + 1e-3f * (threadIdx.x + i);
  }
  __syncthreads();
  const uint64_t t0 = clk();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if constexpr (OP == 0) {  // cvt.f32.f16 (HADD2.F32), both halves
        float a, b;
        asm volatile("{.reg .f16 l, h;\n mov.b32 {l, h}, %2;\n cvt.f32.f16 %0, l;\n cvt.f32.f16 %1, h;}"
                     : "=f"(a), "=f"(b) : "r"(r[i]));
        r[i] = __float_as_uint(a) ^ __float_as_uint(b);
      } else if constexpr (OP == 1) {  // FFMA2
        float2 x = make_float2(f[i], __uint_as_float(r[i] | 0x3f800000u));
        float2 y;
        asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(*reinterpret_cast<unsigned long long*>(&y))
                     : "l"(*reinterpret_cast<unsigned long long*>(&x)), "l"(*reinterpret_cast<unsigned long long*>(&x)),
                       "l"(*reinterpret_cast<unsigned long long*>(&x)));
        f[i] = y.x;
        r[i] = __float_as_uint(y.y);
      } else if constexpr (OP == 2) {  // FFMA
        asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(f[i]));
      } else if constexpr (OP == 3) {  // I2F (cvt.rn.f32.s32)
        float a;
        asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(a) : "r"(r[i]));
        r[i] = __float_as_uint(a);
      } else if constexpr (OP == 4) {  // MUFU.EX2
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[i]));
      } else if constexpr (OP == 5) {  // F2FP e4m3x2
        uint16_t h;
        asm volatile("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(h) : "f"(f[i]), "f"(__uint_as_float(r[i])));
        r[i] += h;
      } else if constexpr (OP == 6) {  // integer f16->f32 bits: ((h & 0x7fff) << 13) | sign, 2 ALU ops per value
        uint32_t lo;
        asm volatile("{.reg .b32 t;\n lop3.b32 t, %1, 0x7fff, 0, 0xc0;\n shf.l.wrap.b32 %0, t, t, 13;}"
                     : "=r"(lo) : "r"(r[i]));
        r[i] = lo;
      } else if constexpr (OP == 7) {  // FMNMX3 via max of 3
        float a;
        asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(a) : "f"(f[i]), "f"(__uint_as_float(r[i])), "f"(f[(i + 1) & 7]));
        f[i] = a;
      } else if constexpr (OP == 8) {  // LOP3
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[i]) : "r"(r[(i + 1) & 7]), "r"(r[(i + 2) & 7]));
      } else if constexpr (OP == 9) {  // FADD2
        float2 x = make_float2(f[i], __uint_as_float(r[i] | 0x3f800000u));
        float2 y;
        asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(*reinterpret_cast<unsigned long long*>(&y))
                     : "l"(*reinterpret_cast<unsigned long long*>(&x)), "l"(*reinterpret_cast<unsigned long long*>(&x)));
        f[i] = y.x;
        r[i] = __float_as_uint(y.y);
      } else if constexpr (OP == 11) {  // FHADD: f32 = f16 + f32 (add.rn.f32.f16), both halves
        float a, b;
        asm volatile("{.reg .f16 l, h;\n mov.b32 {l, h}, %2;\n add.rn.f32.f16 %0, l, %3;\n add.rn.f32.f16 %1, h, %3;}"
                     : "=f"(a), "=f"(b) : "r"(r[i]), "f"(-0.0f));
        r[i] = __float_as_uint(a) ^ __float_as_uint(b);
      } else if constexpr (OP == 12) {  // MUFU.EX2 on f16x2: two exponentials per lane
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(r[i]));
      } else if constexpr (OP == 13) {  // MUFU.EX2 on bf16x2
        asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(r[i]));
      } else if constexpr (OP == 10) {  // PRMT
        asm volatile("prmt.b32 %0, %0, %1, 0x5410;" : "+r"(r[i]) : "r"(r[(i + 3) & 7]));
      }
    }
  }
  const uint64_t t1 = clk();
  uint32_t acc = 0;
  for (int i = 0; i < 8; ++i) acc ^= r[i] ^ __float_as_uint(f[i]);
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int per_op, int sms, uint32_t* sink, unsigned long long* cyc) {
  const int iters = 4096, threads = 512;
  bench<OP><<<sms, threads>>>(iters, sink, cyc);
  cudaDeviceSynchronize();
  bench<OP><<<sms, threads>>>(iters, sink, cyc);
  unsigned long long c[1024];
  cudaMemcpy(c, cyc, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < sms; ++i) mean += c[i];
  mean /= sms;
  const double warp_instr = double(iters) * 8 * per_op * (threads / 32);
  printf("%-44s %6.2f warp-instr/clk/SM  (%.1f lanes/clk/SM)\n", name, warp_instr / mean, 32 * warp_instr / mean);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* sink;
  unsigned long long* cyc;
  cudaMalloc(&sink, sms * 512 * 4);
  cudaMalloc(&cyc, sms * 8);
  run<0>("HADD2.F32 (cvt.f32.f16), per conversion", 2, sms, sink, cyc);
  run<1>("FFMA2 (fma.rn.f32x2)", 1, sms, sink, cyc);
  run<2>("FFMA", 1, sms, sink, cyc);
  run<3>("I2F (cvt.rn.f32.s32)", 1, sms, sink, cyc);
  run<4>("MUFU.EX2", 1, sms, sink, cyc);
  run<5>("F2FP e4m3x2 (+IADD)", 2, sms, sink, cyc);
  run<6>("LOP3+SHF (int f16->f32 bits)", 2, sms, sink, cyc);
  run<7>("FMNMX3 (max.f32 a,b,c)", 1, sms, sink, cyc);
  run<8>("LOP3", 1, sms, sink, cyc);
  run<9>("FADD2 (add.rn.f32x2)", 1, sms, sink, cyc);
  run<10>("PRMT", 1, sms, sink, cyc);
  run<11>("FHADD (add.rn.f32.f16), per conversion", 2, sms, sink, cyc);
  run<12>("MUFU.EX2 f16x2 (2 exps per lane)", 1, sms, sink, cyc);
  run<13>("MUFU.EX2 bf16x2 (2 exps per lane)", 1, sms, sink, cyc);
  return 0;
}
