// glint_device.cuh -- device-side arithmetic of the glint path (sm_100a).
//
// Every function here implements one step of the fp32 arithmetic contract of
// DESIGN.md §4 (bit-exact with the CPU oracle on every value that decides an
// integer). The translation unit is compiled with -fmad=false so that a*b+c
// stays two roundings; FMAs appear only as explicit __fmaf_rn where the
// contract writes fma. No fast-math, no FTZ; division and square root on the
// decision path only through the contract's rcp_c / rsqrt_c (Newton steps from a
// magic-constant seed, no MUFU), plus one IEEE division per scene (1 / beta).
//
// P:Lnnn = line of the paper's text (arXiv 2306.05051).
#pragma once
#include <stdint.h>

namespace glint {

__device__ __forceinline__ float pow2i(int k) { return __uint_as_float((uint32_t)(k + 127) << 23); }

// 2^(e/2) = 2^floor(e/2) * (e odd ? fp32(sqrt 2) : 1)   (grid stretch, Eq. 12 / R-14)
__device__ __forceinline__ float pow2half(int e) {
  float s = pow2i(e >> 1);
  return (e & 1) ? s * 0x1.6a09e6p+0f : s;
}

// exp2c(y), y <= 0 (Eq. 16 (1-p)^n and the Beckmann exponential). DESIGN §4.2.
__device__ __forceinline__ float exp2c(float y) {
  const bool under = !(y >= -125.0f);   // -> 0 (branch-free: the polynomial always runs)
  y = under ? 0.0f : y;
  // k = rint(y) by the 1.5 2^23 magic number; 2^k from K's bits
  const float K = y + 12582912.0f;
  const float k = K - 12582912.0f;
  const float f = y - k;
  float q = 0x1.ffcbfcp-17f;
  q = __fmaf_rn(q, f, 0x1.430912p-13f);
  q = __fmaf_rn(q, f, 0x1.5d87fep-10f);
  q = __fmaf_rn(q, f, 0x1.3b2ab6p-7f);
  q = __fmaf_rn(q, f, 0x1.c6b08ep-5f);
  q = __fmaf_rn(q, f, 0x1.ebfbe0p-3f);
  q = __fmaf_rn(q, f, 0x1.62e430p-1f);
  q = __fmaf_rn(q, f, 1.0f);
  const float p2 = __uint_as_float((__float_as_uint(K) - 0x4B3FFF81u) << 23);   // 2^k
  return (q * p2) * (under ? 0.0f : 1.0f);   // a select as a multiply keeps ptxas from branching
}

// 1/x for normal x > 0: magic start + 3 Newton steps, branch-free;
// replaces IEEE division on the decision path
__device__ __forceinline__ float rcp_c(float x) {
  float y = __uint_as_float(0x7ef311c7U - __float_as_uint(x));
  float e;
  e = __fmaf_rn(-x, y, 1.0f); y = __fmaf_rn(y, e, y);
  e = __fmaf_rn(-x, y, 1.0f); y = __fmaf_rn(y, e, y);
  e = __fmaf_rn(-x, y, 1.0f); y = __fmaf_rn(y, e, y);
  return y;
}

// s * atanh(s)/s series to s^15 (Horner in s^2)
__device__ __forceinline__ float atanh_s(float s) {
  float z = s * s;
  float q = 0x1.111112p-4f;
  q = __fmaf_rn(q, z, 0x1.3b13b2p-4f);
  q = __fmaf_rn(q, z, 0x1.745d18p-4f);
  q = __fmaf_rn(q, z, 0x1.c71c72p-4f);
  q = __fmaf_rn(q, z, 0x1.24924ap-3f);
  q = __fmaf_rn(q, z, 0x1.99999ap-3f);
  q = __fmaf_rn(q, z, 0x1.555556p-2f);
  q = __fmaf_rn(q, z, 1.0f);
  return s * q;
}

// log2(1 - p), p in (0, 1). DESIGN §4.2.
__device__ __forceinline__ float log2_1mp(float p) {
  if (p < 0.5f) {
    float s = p * rcp_c(2.0f - p);
    return -(atanh_s(s) * 0x1.715476p+1f);
  }
  float q = 1.0f - p;
  uint32_t b = __float_as_uint(q);
  int e = (int)((b >> 23) & 255u) - 127;
  float m = __uint_as_float((b & 0x7FFFFFu) | 0x3F800000u);
  if (m > 0x1.555556p+0f) { m = m * 0.5f; e = e + 1; }
  float s = (m - 1.0f) * rcp_c(m + 1.0f);
  return __fmaf_rn(atanh_s(s), 0x1.715476p+1f, (float)e);
}

// atan2(y, x) in turns, (-1/2, 1/2]. DESIGN §4.2.
__device__ __forceinline__ float atan2_turns(float y, float x) {
  float ax = fabsf(x), ay = fabsf(y);
  float mx = ax > ay ? ax : ay;
  float mn = ax > ay ? ay : ax;
  if (!(mx >= 0x1p-126f)) return 0.0f;   // zero or subnormal: no direction
  float t = mn * rcp_c(mx);
  const bool red = t > 0x1.a8279ap-2f;   // reduce by 1/8 turn (select, branch-free)
  const float tr = (t - 1.0f) * rcp_c(t + 1.0f);
  t = red ? tr : t;
  const float base = red ? 0.125f : 0.0f;
  float z = t * t;
  float q = 0x1.32c69ep-7f;
  q = __fmaf_rn(q, z, -0x1.5bade6p-7f);
  q = __fmaf_rn(q, z, 0x1.912b1cp-7f);
  q = __fmaf_rn(q, z, -0x1.da1bacp-7f);
  q = __fmaf_rn(q, z, 0x1.21bb94p-6f);
  q = __fmaf_rn(q, z, -0x1.748376p-6f);
  q = __fmaf_rn(q, z, 0x1.04c26cp-5f);
  q = __fmaf_rn(q, z, -0x1.b2995ep-5f);
  q = __fmaf_rn(q, z, 0x1.45f306p-3f);
  float a = __fmaf_rn(t, q, base);
  if (ay > ax) a = 0.25f - a;
  if (x < 0.0f) a = 0.5f - a;
  if (y < 0.0f) a = -a;
  return a;
}

// published "lowbias32" mixer (R-23)
__device__ __forceinline__ uint32_t lowbias32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}
__device__ __forceinline__ float dot3(float ax, float ay, float az, float bx, float by, float bz) {
  return __fmaf_rn(az, bz, __fmaf_rn(ay, by, ax * bx));
}
// 1/sqrt(x), normal x > 0: magic start + 3 Newton steps, branch-free
__device__ __forceinline__ float rsqrt_c(float x) {
  float y = __uint_as_float(0x5f3759dfU - (__float_as_uint(x) >> 1));
  const float hx = 0.5f * x;
  y = y * __fmaf_rn(-hx, y * y, 1.5f);
  y = y * __fmaf_rn(-hx, y * y, 1.5f);
  y = y * __fmaf_rn(-hx, y * y, 1.5f);
  return y;
}
__device__ __forceinline__ void normalize3(float& x, float& y, float& z) {
  const float inv = rsqrt_c(dot3(x, y, z, x, y, z));
  x = x * inv; y = y * inv; z = z * inv;
}

// Gate parameters of one grid (Eq. 16-17, readings R-1..R-4). DESIGN §4.3 S6.
struct Gate {
  uint32_t T;
  float sigma, m1, cap;
};
// the gate threshold T alone (what the gate phase of the draws needs)
__device__ __forceinline__ uint32_t gate_T(float n, float p, float L2) {
  // L2 = log2(1 - p) for p in (0,1) and -inf for p = 1 (then exp2c(n L2) = 0
  // and P>=1 = 1 with no select), precomputed once per (pixel, light);
  // branch-free. For n <= 0 or p <= 0 only T needs forcing (to 0): the
  // sigma / m1 / cap of such a grid are never used (its count is 0), and
  // the DEBUG record reports the contract's values (0, 1, 1) explicitly.
  const bool none = !(n > 0.0f) || !(p > 0.0f);
  const float pge1 = 1.0f - exp2c(n * L2);
  const uint32_t T = __float2uint_ru(pge1 * 0x1p23f);   // = (uint32_t)ceil(P>=1 2^23), exact
  return none ? 0u : T;
}
// the count parameters sigma, m1, cap (needed only when some draw passes)
__device__ __forceinline__ void gate_counts(float n, float p, Gate& g) {
  const float nm1 = n - 1.0f;
  const float mu = nm1 > 0.0f ? nm1 * p : 0.0f;
  const float var = mu * (1.0f - p);
  const float rv = rsqrt_c(fmaxf(var, 0x1p-126f));          // always computed: no branch
  g.sigma = var >= 0x1p-126f ? var * rv : 0.0f;              // contract sqrt (subnormal -> 0)
  g.m1 = 1.0f + mu;
  g.cap = ceilf(n);
}
__device__ __forceinline__ Gate gate_params(float n, float p, float L2) {
  Gate g;
  g.T = gate_T(n, p, L2);
  gate_counts(n, p, g);
  return g;
}

}  // namespace glint
