// Microbenchmark: sustained warp-instruction throughput per SM for the
// instruction classes the glint draw loop uses (B200, sm_100a).
// Each thread runs 8 independent dependency chains of one op type.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

#define CH 8
#define ITERS 4096

template <int OP>
__global__ void k(uint32_t* out, uint32_t seed) {
  uint32_t v[CH];
  float f[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) { v[c] = seed * (threadIdx.x + 1) + c * 7919; f[c] = (float)v[c] * 1e-9f; }
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (OP == 0) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v[c]) : "r"(v[(c + 1) % CH]), "r"(seed));
      if (OP == 1) { uint32_t t; asm volatile("shr.b32 %0, %1, 15;" : "=r"(t) : "r"(v[c])); v[c] ^= t + seed; }
      if (OP == 2) asm volatile("mad.lo.u32 %0, %0, 0x7feb352d, %1;" : "+r"(v[c]) : "r"(seed));
      if (OP == 3) asm volatile("mad.hi.u32 %0, %0, 0x7feb352d, %0;" : "+r"(v[c]));
      if (OP == 4) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[c]) : "f"(f[(c + 1) % CH]), "f"(0.5f));
      if (OP == 5) asm volatile("max.f32 %0, %0, %1;" : "+f"(f[c]) : "f"(f[(c + 3) % CH]));
      if (OP == 6) asm volatile("cvt.rmi.f32.f32 %0, %0;" : "+f"(f[c]));
      if (OP == 7) asm volatile("add.u32 %0, %0, %1;" : "+r"(v[c]) : "r"(v[(c + 1) % CH]));
      if (OP == 8) asm volatile("{.reg .pred p; setp.gt.u32 p, %0, %1; selp.u32 %0, %0, %1, p;}" : "+r"(v[c]) : "r"(seed));
      if (OP == 9) asm volatile("fma.rn.f32 %0, %0, 0f3F000000, 0f3F800000;" : "+f"(f[c]));
      if (OP == 10) { v[c] = v[c] + (v[c] >> 15); v[c] = v[c] * 0x846ca68bU + seed; }
      if (OP == 11) { v[c] = v[c] ^ (v[c] >> 15); v[c] = v[c] * 0x846ca68bU + seed; }
      if (OP == 12) { v[c] = v[c] * 0x846ca68bU + seed; }
      if (OP == 13) asm volatile("rsqrt.approx.f32 %0, %0;" : "+f"(f[c]));
      if (OP == 14) asm volatile("{.reg .f32 t; rcp.approx.f32 t, %0; add.f32 %0, t, %1;}" : "+f"(f[c]) : "f"(f[(c + 1) % CH]));
      if (OP == 15) asm volatile("ex2.approx.f32 %0, %0;" : "+f"(f[c]));
      if (OP == 16) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(f[c]) : "f"(f[(c + 3) % CH]), "f"(f[(c + 5) % CH]));
      if (OP == 18) asm volatile("{.reg .pred p; add.u32 %1, %1, %2; setp.le.u32 p, %1, %2; @p fma.rn.f32 %0, %0, %3, %3;}" : "+f"(f[c]), "+r"(v[c]) : "r"(seed), "f"(0.5f));
      if (OP == 19) asm volatile("{add.u32 %1, %1, %2; fma.rn.f32 %0, %0, %3, %3;}" : "+f"(f[c]), "+r"(v[c]) : "r"(seed), "f"(0.5f));
      if (OP == 17) { extern __shared__ float sm[]; f[c] += sm[(v[c] + c * 33) & 4095]; v[c] += 0x9e3779b9u; }
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) acc ^= v[c] ^ __float_as_uint(f[c]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int OP>
float run(const char* name, int sms, uint32_t* d) {
  dim3 grid(sms * 4), block(512);
  const size_t smem = OP == 17 ? 16384 : 0;
  k<OP><<<grid, block, smem>>>(d, 3);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<OP><<<grid, block, smem>>>(d, 3);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double warp_inst = (double)grid.x * block.x / 32 * ITERS * CH;
  double cyc = ms * 1e-3 * clk * 1e3;
  printf("%-28s %7.3f warp-inst/clk/SM (%.3f ms)\n", name, warp_inst / cyc / sms, ms);
  return ms;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* d; cudaMalloc(&d, sizeof(uint32_t) * sms * 4 * 512);
  run<0>("LOP3", sms, d);
  run<1>("shr+xor+add step (3 inst)", sms, d);
  run<2>("IMAD (mad.lo imm)", sms, d);
  run<3>("IMAD.HI (mad.hi)", sms, d);
  run<4>("FFMA (reg)", sms, d);
  run<5>("FMNMX", sms, d);
  run<6>("FRND.FLOOR", sms, d);
  run<7>("IADD", sms, d);
  run<8>("ISETP+SEL", sms, d);
  run<9>("FFMA (imm)", sms, d);
  run<10>("add-shift + IMAD (2 ops?)", sms, d);
  run<11>("xor-shift + IMAD (3 ops)", sms, d);
  run<12>("IMAD only", sms, d);
  run<13>("MUFU.RSQ", sms, d);
  run<14>("MUFU.RCP (+FADD)", sms, d);
  run<15>("MUFU.EX2", sms, d);
  run<16>("FMNMX3 (3-input max)", sms, d);
  run<17>("LDS (+FADD, IADD)", sms, d);
  run<18>("IADD + ISETP + @p FFMA (3 inst)", sms, d);
  run<19>("IADD + FFMA (2 inst, control)", sms, d);
  return 0;
}
