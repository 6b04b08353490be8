// Microbenchmark: which instruction classes share an issue pipe on B200, and
// what one gated draw (S4b + S7) costs in isolation, per variant.
//
// Part 1 (pairs): each step issues one op of class A and one of class B on
// independent chains; if A and B sit on different half-rate pipes the pair
// runs at the issue peak (4 warp-inst/clk/SM), if they share one at 2.
// Part 2 (draw loop): 12 draws x 4 grids per iteration with the kernel's
// instruction sequence (quantile table in shared memory); variants change
// only the count clamp. Reports SM cycles per warp-draw.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

#define CH 8
#define ITERS 4096

template <int A, int B>
__global__ void pair_k(uint32_t* out, uint32_t seed) {
  uint32_t v[CH], w[CH];
  float f[CH], g[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    v[c] = seed * (threadIdx.x + 1) + c * 7919; w[c] = v[c] * 3u + 1u;
    f[c] = (float)v[c] * 1e-9f; g[c] = (float)w[c] * 1e-9f;
  }
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
#define OPX(OP, V, F)                                                                                     \
  if (OP == 0) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(V[c]) : "r"(V[(c + 1) % CH]), "r"(seed)); \
  if (OP == 1) asm volatile("max.f32 %0, %0, %1;" : "+f"(F[c]) : "f"(F[(c + 3) % CH]));                   \
  if (OP == 2) asm volatile("mad.lo.u32 %0, %0, 0x7feb352d, %1;" : "+r"(V[c]) : "r"(seed));               \
  if (OP == 3) asm volatile("shf.r.wrap.b32 %0, %0, %0, 11;" : "+r"(V[c]));                                \
  if (OP == 4) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(F[c]) : "f"(F[(c + 1) % CH]), "f"(0.5f));  \
  if (OP == 5) asm volatile("{.reg .pred p; setp.le.u32 p, %0, %1; selp.u32 %0, 1, 2, p;}" : "+r"(V[c]) : "r"(seed)); \
  if (OP == 6) asm volatile("cvt.rmi.f32.f32 %0, %0;" : "+f"(F[c]));                                       \
  if (OP == 7) asm volatile("add.u32 %0, %0, %1;" : "+r"(V[c]) : "r"(V[(c + 1) % CH]));                    \
  if (OP == 8) asm volatile("shr.u32 %0, %0, 7;" : "+r"(V[c]));                                            \
  if (OP == 9) asm volatile("fma.rn.sat.f32 %0, %0, %1, %2;" : "+f"(F[c]) : "f"(F[(c + 1) % CH]), "f"(0.5f)); \
  if (OP == 10) asm volatile("prmt.b32 %0, %0, %1, 0x3210;" : "+r"(V[c]) : "r"(seed));                     \
  if (OP == 11) asm volatile("min.u32 %0, %0, %1;" : "+r"(V[c]) : "r"(V[(c + 1) % CH]));
      OPX(A, v, f)
      OPX(B, w, g)
#undef OPX
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) acc ^= v[c] ^ w[c] ^ __float_as_uint(f[c]) ^ __float_as_uint(g[c]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

static const char* kName[] = {"LOP3", "FMNMX", "IMAD", "SHF.W", "FFMA", "ISETP+SEL", "FRND", "IADD",
                              "SHF.R", "FFMA.SAT", "PRMT", "IMNMX"};

template <int A, int B>
void run_pair(int sms, uint32_t* d, int clk) {
  dim3 grid(sms * 4), block(512);
  pair_k<A, B><<<grid, block>>>(d, 3);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  pair_k<A, B><<<grid, block>>>(d, 3);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const int per = (A == 5 ? 2 : 1) + (B == 5 ? 2 : 1);
  double warp_inst = (double)grid.x * block.x / 32 * ITERS * CH * per;
  double cyc = ms * 1e-3 * clk * 1e3;
  printf("pair %-10s + %-10s %6.3f warp-inst/clk/SM\n", kName[A], kName[B], warp_inst / cyc / sms);
}

// ---------------------------------------------------------------- draw loop
template <int V>
__global__ void __launch_bounds__(512, 1) draw_k(uint32_t* out, const float* Z, uint32_t seed, int iters) {
  __shared__ float sZ[4096 + 32];
  for (int i = threadIdx.x; i < 4096 + 32; i += blockDim.x) sZ[i] = Z[i & 4095];
  __syncthreads();
  uint32_t hsC[12], kaC[4];
  float bw[12];
  uint32_t x = seed * 0x9e3779b9u + (blockIdx.x * blockDim.x + threadIdx.x) * 0x85ebca6bu;
#pragma unroll
  for (int t = 0; t < 12; ++t) { x = x * 0x7feb352du + 0x1234567u; hsC[t] = x; bw[t] = (float)(x >> 9) * 0x1p-23f; }
#pragma unroll
  for (int t = 0; t < 4; ++t) { x = x * 0x846ca68bu + 0x7654321u; kaC[t] = x; }
  float A[4] = {0.f, 0.f, 0.f, 0.f};
  const uint32_t lane4 = (threadIdx.x & 31u) << 2;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      // per-grid parameters vary with the iteration so nothing is hoisted
      const float sigma = 3.0f + (float)((it + i) & 7), m1 = 40.0f + (float)(it & 15), capk = 64.0f;
      const uint32_t G = 0x00100000u * (uint32_t)(1 + ((it + i) & 3));
      const float s2 = sigma * (1.0f / 63.0f), m2 = m1 * (1.0f / 63.0f) - (1.0f / 63.0f);   // V1 (sat)
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const float bk = bw[i * 3 + k];
#pragma unroll
        for (int jn = 0; jn < 4; ++jn) {
          uint32_t y = hsC[i * 3 + k] + kaC[jn];
          y ^= __funnelshift_r(y, y, 11) ^ __funnelshift_r(y, y, 19);
          y *= 0x846ca68bU;
          const uint32_t s16 = y >> 16;
          float z;
          if (V <= 4) z = *reinterpret_cast<const float*>(reinterpret_cast<const char*>(sZ) + ((y ^ s16) & 0x3FFCu));
          if (V == 5) z = *reinterpret_cast<const float*>(reinterpret_cast<const char*>(sZ) + (((y ^ s16) & 0x3F80u) | lane4));
          if (V == 6) z = __uint_as_float(((y ^ s16) & 0x3FFCu) | 0x40000000u) - 3.0f;
          if (V == 7) z = *reinterpret_cast<const float*>(reinterpret_cast<const char*>(sZ) + ((y ^ s16) & 0x3FFCu) + lane4);
          float c;
          if (V == 0 || V >= 5) c = floorf(fminf(fmaxf(__fmaf_rn(sigma, z, m1), 1.0f), capk));
          if (V == 1) c = floorf(__fmaf_rn(__saturatef(__fmaf_rn(s2, z, m2)), capk - 1.0f, 1.0f));
          if (V == 2) c = floorf(fminf(__fmaf_rn(sigma, z, m1), capk));
          if (V == 3) c = floorf(__fmaf_rn(sigma, z, m1));
          if (V == 4) c = __fmaf_rn(sigma, z, m1);
          if (y <= G) A[jn] = __fmaf_rn(bk, c, A[jn]);
        }
        hsC[i * 3 + k] += 0x9e3779b9u;   // next iteration: new texel words
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = __float_as_uint(A[0] + A[1] + A[2] + A[3]);
}

template <int V>
void run_draw(const char* name, int sms, uint32_t* d, const float* Z, int clk) {
  const int iters = 256;
  dim3 grid(sms), block(512);
  draw_k<V><<<grid, block>>>(d, Z, 3, iters);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  draw_k<V><<<grid, block>>>(d, Z, 3, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double warp_draws_per_smsp = (double)block.x / 32 / 4 * iters * 48;
  const double cyc = ms * 1e-3 * clk * 1e3;
  printf("draw %-34s %6.2f SMSP cycles per warp-draw (%.3f ms)\n", name, cyc / warp_draws_per_smsp, ms);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  uint32_t* d; cudaMalloc(&d, sizeof(uint32_t) * sms * 4 * 512);
  run_pair<0, 0>(sms, d, clk);
  run_pair<0, 1>(sms, d, clk);
  run_pair<0, 2>(sms, d, clk);
  run_pair<1, 2>(sms, d, clk);
  run_pair<3, 2>(sms, d, clk);
  run_pair<3, 0>(sms, d, clk);
  run_pair<3, 1>(sms, d, clk);
  run_pair<8, 2>(sms, d, clk);
  run_pair<8, 0>(sms, d, clk);
  run_pair<0, 4>(sms, d, clk);
  run_pair<1, 4>(sms, d, clk);
  run_pair<5, 0>(sms, d, clk);
  run_pair<5, 2>(sms, d, clk);
  run_pair<6, 0>(sms, d, clk);
  run_pair<6, 4>(sms, d, clk);
  run_pair<7, 0>(sms, d, clk);
  run_pair<7, 2>(sms, d, clk);
  run_pair<9, 0>(sms, d, clk);
  run_pair<10, 0>(sms, d, clk);
  run_pair<10, 2>(sms, d, clk);
  run_pair<11, 0>(sms, d, clk);
  run_pair<11, 2>(sms, d, clk);
  float hz[4096];
  for (int i = 0; i < 4096; ++i) hz[i] = -3.5f + 7.0f * (i + 0.5f) / 4096.0f;
  float* Z; cudaMalloc(&Z, sizeof(hz));
  cudaMemcpy(Z, hz, sizeof(hz), cudaMemcpyHostToDevice);
  run_draw<0>("V0 kernel: clamp [1, cap] (2 FMNMX)", sms, d, Z, clk);
  run_draw<1>("V1 FFMA.SAT clamp", sms, d, Z, clk);
  run_draw<2>("V2 upper clamp only", sms, d, Z, clk);
  run_draw<3>("V3 no clamp", sms, d, Z, clk);
  run_draw<4>("V4 no clamp, no floor", sms, d, Z, clk);
  run_draw<5>("V5 V0 + conflict-free LDS (lane bank)", sms, d, Z, clk);
  run_draw<6>("V6 V0 without LDS (z from bits)", sms, d, Z, clk);
  run_draw<7>("V7 V0 + lane offset (still random)", sms, d, Z, clk);
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
