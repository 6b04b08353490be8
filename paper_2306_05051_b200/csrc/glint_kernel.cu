// glint_kernel.cu -- the fused sm_100a glint evaluation kernel (S0..S9).
//
// One thread shades one pixel for all lights. Per pixel (shared by every
// light): S0 coalesced float4 loads, S1 footprint, S2 lattice
// (4 grids), S3 grid transform + simplex (12 texels), S4a spatial seeds.
// Per light: S5 half-vector / p / angular nodes, S6 gate parameters of the 4
// grids, S7 the 48 gated draws (fully unrolled, hashes finished in
// registers, quantiles from a shared-memory table), S8 blend, S9 radiance.
//
// Persistent grid: one 512-thread block per SM (128 registers) claims
// 1024-pixel tiles dynamically from a per-launch counter, so the 18 KB of
// tables are staged into shared memory once per block. For contiguous
// G-buffers each tile's 5 planes (80 KB) stream HBM -> shared memory by the
// TMA bulk-copy engine (cp.async.bulk + mbarrier) into a 2-stage ring, issued
// two tiles ahead by the last warp to finish a stage, so the DRAM latency is
// off the critical path. Every grid triggers its programmatic dependents at
// entry and waits for its predecessor before exiting (glint_eval_batch chains
// a step's frames).
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "../../include/glint.h"
#include "glint_device.cuh"
#include "glint_kernel.h"
#include "glint_tma.cuh"

// -DGLINT_CHECKED: device asserts on every computed index (compute-sanitizer
// is not available on this pool); tests/test_gpu_checked.py runs the parity
// suite's inputs against a checked build
#ifdef GLINT_CHECKED
#include <cassert>
#define GL_ASSERT(c) assert(c)
#else
#define GL_ASSERT(c) ((void)0)
#endif

// production MODE 0: evaluate a grid's 12 gates before its counts and skip
// the counts when no lane of the warp passes (0 = the dense loop, for A/B)
#ifndef GLINT_GATE_FIRST
#define GLINT_GATE_FIRST 1
#endif
// production MODE 0-2 with several lights: angular node seeds from a
// per-launch shared-memory table (0 = computed per pixel-light, for A/B)
#ifndef GLINT_KA_TABLE
#define GLINT_KA_TABLE 1
#endif

namespace glint {

// ---------------------------------------------------------------------------
// S2: lattice location (Eq. 10/13, Fig. 6-7, P:L628-635, L752-758;
// readings R-5, R-9..R-13). Output: 4 slots (ls, lr, jo, w).
// ---------------------------------------------------------------------------
struct Slot {
  int ls, lr, jo;
  float w;
};

__device__ __forceinline__ void lattice(float P, float r, float psi, int K, Slot s[4], uint32_t& flags) {
  uint32_t pb = __float_as_uint(P);
  int es = (int)((pb >> 23) & 255u) - 127;
  float ts = __uint_as_float((pb & 0x7FFFFFu) | 0x3F800000u) - 1.0f;

  int er;
  float tr;
  if (!(r >= 1.0f)) r = 1.0f;
  float rmax = pow2i(K);
  if (r >= rmax) {
    if (r > rmax) flags |= GLINT_FLAG_RATIO_CLAMPED;
    er = K - 1;
    tr = 1.0f;
  } else {
    uint32_t rb = __float_as_uint(r);
    er = (int)((rb >> 23) & 255u) - 127;
    tr = __uint_as_float((rb & 0x7FFFFFu) | 0x3F800000u) - 1.0f;
  }

  float A = psi * pow2i(er);
  float jf = floorf(A);
  float a = A - jf;
  int j = (int)jf;
  int nI = 1 << er, nO = 2 << er;
  // pentagon vertices as packed keys (lr << 9 | jo)
  int kA00 = (er << 9) | j;
  int kA01 = (er << 9) | ((j + 1) & (nI - 1));
  int kA10 = ((er + 1) << 9) | (2 * j);
  int kA11 = ((er + 1) << 9) | (2 * j + 1);
  int kA12 = ((er + 1) << 9) | ((2 * j + 2) & (nO - 1));

  // triangle of the pentagon (tr, a) (R-11), branch-free: every candidate
  // weight is computed with the contract's ops and selected (same bits)
  const float ht = 0.5f * tr;
  const bool c0 = a <= ht;                    // T0 = {A00, A10, A11}
  const bool c2 = !c0 && (a >= 1.0f - ht);    // T2 = {A01, A11, A12}; else T1 = {A00, A11, A01}
  const float om = 1.0f - a;
  const float two_a = a + a, two_om = om + om;
  const float omt = 1.0f - tr;
  int k0 = c2 ? kA01 : kA00;
  int k1 = c0 ? kA10 : kA11;
  int k2 = c0 ? kA11 : (c2 ? kA12 : kA01);
  float w0 = (c0 || c2) ? omt : (om - ht);
  float w1 = c0 ? (tr - two_a) : (c2 ? two_om : tr);
  float w2 = c0 ? two_a : (c2 ? (tr - two_om) : (a - ht));
  // merge coincident vertices (ring 0), in (0,1), (0,2), (1,2) order (R-13)
  { const bool m = k1 == k0; w0 = m ? w0 + w1 : w0; w1 = m ? 0.0f : w1; }
  { const bool m = k2 == k0; w0 = m ? w0 + w2 : w0; w2 = m ? 0.0f : w2; }
  { const bool m = k2 == k1; w1 = m ? w1 + w2 : w1; w2 = m ? 0.0f : w2; }
  // stable sort by key: compare-swaps (0,1), (1,2), (0,1)  (R-12 global order)
#define GL_CSWAP(ka, wa, kb, wb)                                 \
  {                                                              \
    const bool sw = ka > kb;                                     \
    const int tk = sw ? kb : ka; kb = sw ? ka : kb; ka = tk;      \
    const float tw = sw ? wb : wa; wb = sw ? wa : wb; wa = tw;    \
  }
  GL_CSWAP(k0, w0, k1, w1);
  GL_CSWAP(k1, w1, k2, w2);
  GL_CSWAP(k0, w0, k1, w1);
#undef GL_CSWAP
  // prism -> 3 tetrahedra, staircase fill of the top level (R-12)
  const float al = w0, be = w1, ga = w2;
  const float t = ts;
  const float ab = al + be;
  const bool s0 = t <= al, s1 = !s0 && (t <= ab);   // else s2
  int kk[4], ll[4];
  float ww[4];
  kk[0] = s0 ? k0 : (s1 ? k1 : k2); ll[0] = es;
  ww[0] = s0 ? al - t : (s1 ? ab - t : 1.0f - t);
  kk[1] = s0 ? k1 : (s1 ? k2 : k0); ll[1] = (s0 || s1) ? es : es + 1;
  ww[1] = s0 ? be : (s1 ? ga : al);
  kk[2] = s0 ? k2 : (s1 ? k0 : k1); ll[2] = s0 ? es : es + 1;
  ww[2] = s0 ? ga : (s1 ? al : be);
  kk[3] = s0 ? k0 : (s1 ? k1 : k2); ll[3] = es + 1;
  ww[3] = s0 ? t : (s1 ? t - al : (t - al) - be);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    s[i].ls = ll[i];
    s[i].lr = kk[i] >> 9;
    s[i].jo = kk[i] & 511;
    s[i].w = ww[i];
  }
}

// S2 for the 160-draw ablation: all 10 prism vertices (2 LODs x pentagon),
// linear in ts / tr, linear in a on the inner ring, hats at a = 0, 1/2, 1 on
// the outer ring; coincident ring-0 vertices merged (reading R-29).
__device__ __forceinline__ void lattice10(float P, float r, float psi, int K, int ls[10], int lr[10], int jo[10],
                                          float w[10], uint32_t& flags) {
  const uint32_t pb = __float_as_uint(P);
  const int es = (int)((pb >> 23) & 255u) - 127;
  const float ts = __uint_as_float((pb & 0x7FFFFFu) | 0x3F800000u) - 1.0f;
  int er;
  float tr;
  if (!(r >= 1.0f)) r = 1.0f;
  const float rmax = pow2i(K);
  if (r >= rmax) {
    if (r > rmax) flags |= GLINT_FLAG_RATIO_CLAMPED;
    er = K - 1;
    tr = 1.0f;
  } else {
    const uint32_t rb = __float_as_uint(r);
    er = (int)((rb >> 23) & 255u) - 127;
    tr = __uint_as_float((rb & 0x7FFFFFu) | 0x3F800000u) - 1.0f;
  }
  const float A = psi * pow2i(er);
  const float jf = floorf(A);
  const float a = A - jf;
  const int j = (int)jf;
  const int nI = 1 << er, nO = 2 << er;
  int vk[5] = {(er << 9) | j, (er << 9) | ((j + 1) & (nI - 1)), ((er + 1) << 9) | (2 * j),
               ((er + 1) << 9) | (2 * j + 1), ((er + 1) << 9) | ((2 * j + 2) & (nO - 1))};
  const float a2 = a + a, omt = 1.0f - tr;
  const bool lo = a2 <= 1.0f;
  float pw[5] = {omt * (1.0f - a), omt * a, tr * (lo ? 1.0f - a2 : 0.0f), tr * (lo ? a2 : 2.0f - a2),
                 tr * (lo ? 0.0f : a2 - 1.0f)};
#pragma unroll
  for (int p = 0; p < 5; ++p)
#pragma unroll
    for (int q = p + 1; q < 5; ++q) {
      const bool m = vk[p] == vk[q];
      pw[p] = m ? pw[p] + pw[q] : pw[p];
      pw[q] = m ? 0.0f : pw[q];
    }
#pragma unroll
  for (int lv = 0; lv < 2; ++lv) {
    const float sw = lv ? ts : 1.0f - ts;
#pragma unroll
    for (int p = 0; p < 5; ++p) {
      ls[lv * 5 + p] = es + lv;
      lr[lv * 5 + p] = vk[p] >> 9;
      jo[lv * 5 + p] = vk[p] & 511;
      w[lv * 5 + p] = sw * pw[p];
    }
  }
}

// ---------------------------------------------------------------------------
// Decisions shared by the shading kernel and the evaluation counter (so both
// take them with the same operations): S1 footprint moments and validity
// (R-7, R-25, R-30b), the S5 viewer and the per-light activity test
// (R-27, R-27b).
// ---------------------------------------------------------------------------
struct Foot {
  float P, lam, a, b, c;
};
__device__ __forceinline__ Foot s1_moments(float4 duv) {
  const float dudx = duv.x, dvdx = duv.y, dudy = duv.z, dvdy = duv.w;
  const float det = dudx * dvdy - dvdx * dudy;
  Foot f;
  f.a = dudx * dudx + dudy * dudy;
  f.b = dudx * dvdx + dudy * dvdy;
  f.c = dvdx * dvdx + dvdy * dvdy;
  const float hm = 0.5f * (f.a - f.c);
  const float dv = hm * hm + f.b * f.b;
  const float disc = dv >= 0x1p-126f ? dv * rsqrt_c(dv) : 0.0f;   // contract sqrt (subnormal -> 0)
  f.lam = 0.5f * (f.a + f.c) + disc;
  f.P = fabsf(det);
  return f;
}
__device__ __forceinline__ bool s1_valid(const Foot& f) { return f.P >= 0x1p-64f && f.P < 0x1p64f && f.lam < 0x1p126f; }
__device__ __forceinline__ bool uv_ok(float4 uvm) {
  return (__float_as_uint(uvm.w) & 1u) != 0 && fabsf(uvm.x) <= 0x1p24f && fabsf(uvm.y) <= 0x1p24f;
}
// unnormalised direction d towards the light, |d|^2 and n.d
__device__ __forceinline__ void light_dir(const glint_light& lt, float4 pos, float nx, float ny, float nz, float& dx,
                                          float& dy, float& dz, float& d2, float& nd) {
  if (lt.kind == 0) { dx = lt.pos_or_dir[0] - pos.x; dy = lt.pos_or_dir[1] - pos.y; dz = lt.pos_or_dir[2] - pos.z; }
  else { dx = lt.pos_or_dir[0]; dy = lt.pos_or_dir[1]; dz = lt.pos_or_dir[2]; }
  d2 = dot3(dx, dy, dz, dx, dy, dz);
  nd = dot3(nx, ny, nz, dx, dy, dz);
}
__device__ __forceinline__ bool light_active(float ni, float nd, float d2) {
  return ni > 0.0f && nd > 0.0f && d2 >= 0x1p-126f && d2 <= 0x1p120f;
}
__device__ __forceinline__ void view_dir(const glint_scene& sc, float4 pos, float& wix, float& wiy, float& wiz) {
  if (sc.view_kind == 0) { wix = sc.view[0] - pos.x; wiy = sc.view[1] - pos.y; wiz = sc.view[2] - pos.z; }
  else { wix = sc.view[0]; wiy = sc.view[1]; wiz = sc.view[2]; }
  normalize3(wix, wiy, wiz);
}

// ---------------------------------------------------------------------------
// S9 radiance shell (Eq. 1-2; readings R-21, R-27), tolerance
// path (1e-4 relative against the oracle's fp64). Two tiers, chosen per
// lane by the same rule in the production and DEBUG kernels (so both give the
// same bits):
//  * radiance_shell32, fp32 with MUFU rsqrt / reciprocals, for the
//    well-conditioned lanes: both shading cosines >= 2^-6 and every f0 >=
//    2^-10 (DESIGN.md §4.1 error budget: <= ~4e-5 worst case, 2e-6 measured);
//  * radiance_shell64 for the rest (grazing view or light, tiny f0, factors
//    out of fp32's comfortable range): the cosines, the irradiance and
//    Schlick's 1 - w_i.h in fp64 from the raw fp32 inputs.
// Both run only in the warp-uniform "some lane has C > 0" block.
// ---------------------------------------------------------------------------
// rcp / rsqrt from the MUFU double-precision seeds (rcp.approx / rsqrt.approx
// .f64) plus one Newton step: relative error far below the tolerance
__device__ __forceinline__ double rcp_d(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return fma(r, fma(-x, r, 1.0), r);     // one Newton step
}
__device__ __forceinline__ double rsqrt_d(double x) {
  double y;
  asm("rsqrt.approx.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y * fma(-0.5 * x, y * y, 1.5);  // one Newton step
}
__device__ __forceinline__ double dot3d(double ax, double ay, double az, double bx, double by, double bz) {
  return fma(az, bz, fma(ay, by, ax * bx));
}
// Smith G2 = 1 / (1 + Lambda(w_i) + Lambda(w_o)) (R-21) as one fraction,
// Lambda = num / den per direction (num = 0, den = 1 for Lambda = 0): GGX
// exact Lambda = s / (2 c (c + sqrt(c^2 + s))), Beckmann Walter 2007
// rational in a = c / sqrt(s) (0 from a >= 1.6). s = ax^2 wx^2 + ay^2 wy^2
// (tangential part), c = n.w (fp64, relative accuracy at grazing).
__device__ __forceinline__ void lambda_frac(int kind, double s, double c, double& num, double& den) {
  num = 0.0;
  den = 1.0;
  if (!(s > 0.0)) return;
  if (kind == 0) {
    const double t = fma(c, c, s);
    num = s;
    den = 2.0 * c * (c + t * rsqrt_d(t));
    return;
  }
  const double a = c * rsqrt_d(s);
  if (a >= 1.6) return;
  num = fma(a, fma(0.396, a, -1.259), 1.0);
  den = a * fma(2.181, a, 3.535);
}
// F G2 D_P E / (4 n.wi) of one light for the pixel (Eq. 1-4, R-20, R-21):
// the cosines n.wi, n.wo, the irradiance E and Schlick's 1 - w_i.h in fp64
// from the raw fp32 inputs (exact differences view - pos, light - pos and
// exact products: relative accuracy at grazing and near retro-reflection);
// the tangential parts of w_i, w_o in the fp32 frame of the decision path
// (they enter only Lambda's s, which needs absolute accuracy ~1e-7: DESIGN.md
// §4.1); D_P = C / (pi ax ay R N P) from the fp32 denominator (relative 3e-7).
// Nothing when C = 0 or an fp64 cosine is not > 0 (DESIGN.md §4.3 S9).
// Out of line: inlined, its code and registers cost the draw loop ~10 % even
// though few lanes take it. Every scene value arrives as a scalar argument (a
// pointer into the kernel's parameter space would force a local copy of the
// whole scene per thread).
__device__ __noinline__ float3 radiance_shell64(int ndf_kind, int view_kind, int light_kind, float vx, float vy, float vz,
                                                float lx, float ly, float lz, float ir, float ig, float ib, float f0r,
                                                float f0g, float f0b, float4 nrm, float4 pos, float ti, float bi,
                                                float to, float bo, float ax2, float ay2, float den_f, float C) {
  const float3 zero = make_float3(0.0f, 0.0f, 0.0f);
  if (!(C > 0.0f)) return zero;
  const double px = pos.x, py = pos.y, pz = pos.z;
  const double nx = nrm.x, ny = nrm.y, nz = nrm.z;
  double wx = vx, wy = vy, wz = vz;   // towards the viewer (pinhole camera or direction)
  if (view_kind == 0) { wx -= px; wy -= py; wz -= pz; }
  double ox = lx, oy = ly, oz = lz;   // towards the light
  if (light_kind == 0) { ox -= px; oy -= py; oz -= pz; }
  const double rn = rsqrt_d(dot3d(nx, ny, nz, nx, ny, nz));
  const double ri = rsqrt_d(dot3d(wx, wy, wz, wx, wy, wz));
  const double ro = rsqrt_d(dot3d(ox, oy, oz, ox, oy, oz));
  const double ci = dot3d(nx, ny, nz, wx, wy, wz) * rn * ri;
  const double co = dot3d(nx, ny, nz, ox, oy, oz) * rn * ro;
  if (!(ci > 0.0) || !(co > 0.0)) return zero;
  // Schlick F = f0 + (1 - f0)(1 - w_i.h)^5, h = normalize(w_i + w_o)
  wx *= ri; wy *= ri; wz *= ri;
  ox *= ro; oy *= ro; oz *= ro;
  const double hx = wx + ox, hy = wy + oy, hz = wz + oz;
  const double cih = dot3d(wx, wy, wz, hx, hy, hz) * rsqrt_d(dot3d(hx, hy, hz, hx, hy, hz));
  const double om = 1.0 - cih;
  const double om2 = om * om;
  const double om5 = om2 * om2 * om;
  // G2 D_P E / (4 n.wi) = C E G2 / (4 n.wi pi ax ay R N P), one reciprocal
  double ni_, di_, no_, do_;
  lambda_frac(ndf_kind, (double)__fmaf_rn(ax2, ti * ti, ay2 * (bi * bi)), ci, ni_, di_);
  lambda_frac(ndf_kind, (double)__fmaf_rn(ax2, to * to, ay2 * (bo * bo)), co, no_, do_);
  const double dd = di_ * do_;
  const double E = light_kind == 0 ? ro * ro : 1.0;
  const double k = ((double)C * E) * dd * rcp_d((fma(ni_, do_, dd) + no_ * di_) * (4.0 * ci) * (double)den_f);
  const double f0d[3] = {f0r, f0g, f0b};
  return make_float3((float)(fma(1.0 - f0d[0], om5, f0d[0]) * k * (double)ir),
                     (float)(fma(1.0 - f0d[1], om5, f0d[1]) * k * (double)ig),
                     (float)(fma(1.0 - f0d[2], om5, f0d[2]) * k * (double)ib));
}

// The fp32 tier. Its cosines come from the decision path (fp32-normalised
// vectors, fp32 differences: absolute error <= ~5e-7, so relative <= 3.2e-5
// at 2^-6); Lambda's tangential parts need only absolute accuracy (~2e-7,
// the fp32 frame); Schlick's (1 - w_i.h)^5 with absolute error ~3e-7 adds
// <= 5e-6 relative when f0 >= 2^-10.
// MUFU reciprocal / rsqrt with flush-to-zero (one instruction each; without
// .ftz the compiler wraps every MUFU op in ~4 instructions of subnormal
// scaling). Every value the fp32 tier accepts is a normal float: its
// cosines are >= 2^-6 and k is range-checked; a flushed operand can only
// yield 0 / inf / NaN in k (rejected: the lane takes the fp64 tier) or a
// Beckmann a = inf (Lambda = 0, the s -> 0 limit).
__device__ __forceinline__ float rcp_ftz(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rsqrt_ftz(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float lambda32(int kind, float s, float c) {
  if (!(s > 0.0f)) return 0.0f;
  if (kind == 0) {
    const float t = __fmaf_rn(c, c, s);
    return s * rcp_ftz(2.0f * c * (c + t * rsqrt_ftz(t)));
  }
  const float a = c * rsqrt_ftz(s);
  if (a >= 1.6f) return 0.0f;
  return __fmaf_rn(a, __fmaf_rn(0.396f, a, -1.259f), 1.0f) * rcp_ftz(a * __fmaf_rn(2.181f, a, 3.535f));
}
// one light's contribution; ci, lam_i, dq: the pixel's cosine, Lambda(w_i)
// and 4 n.wi pi ax ay R N P; rs = rsqrt_c(|d|^2). Only k = C G2 E / dq needs
// a range check: F in [2^-10, 1], so F k stays normal, and the final product
// with the intensity is one correctly rounded multiplication (an fp32 result
// beyond fp32's range is that value's rounding)
__device__ __forceinline__ bool radiance_shell32(const glint_scene& sc, int ndf, const glint_light& lt, float ci, float lam_i,
                                                 float co, float cih, float to, float bo, float ax2, float ay2,
                                                 float dq, float rs, float C, float3& rgb) {
  const float om = 1.0f - cih;
  const float om2 = om * om;
  const float om5 = om2 * om2 * om;
  const float g2 = rcp_ftz(1.0f + lam_i + lambda32(ndf, __fmaf_rn(ax2, to * to, ay2 * (bo * bo)), co));
  const float E = lt.kind == 0 ? rs * rs : 1.0f;
  const float k = (C * g2) * rcp_ftz(dq) * E;
  // one exit (no branches): a lane outside the tier adds an exact +0 and
  // returns false, so the caller's fp64 tier adds its contribution instead
  const bool ok = ci >= 0x1p-6f && co >= 0x1p-6f && k >= 0x1p-100f && k <= 0x1p100f;
  const float kk = ok ? k : 0.0f;
  rgb.x += ((sc.f0[0] + (1.0f - sc.f0[0]) * om5) * kk) * lt.intensity[0];
  rgb.y += ((sc.f0[1] + (1.0f - sc.f0[1]) * om5) * kk) * lt.intensity[1];
  rgb.z += ((sc.f0[2] + (1.0f - sc.f0[2]) * om5) * kk) * lt.intensity[2];
  return ok;
}

// shared tables at namespace scope: fixed shared-window offsets, so the
// quantile lookup in the draw loop is a single LDS with an immediate base
__shared__ __align__(128) float g_sZ[GLINT_ZQ];
__shared__ __align__(16) float2 g_sCS[GLINT_NANG];
// angular node seeds ka(cx, cy) * C1 of every node a pixel-light can reach
// (|h_x|, |h_y| <= 1: cx in [-ceil(1/beta) - 2, ceil(1/beta) + 2]), built per
// launch by each block: four LDS per pixel-light instead of four lowbias32.
// Same values as the direct computation (production == DEBUG tests).
__shared__ __align__(16) uint32_t g_sKA[kKaMax];

// ---------------------------------------------------------------------------
// Shading of one pixel (S1..S9). Inputs already in registers; `outp` is the
// pixel's output float4, `rec` its first debug record (DEBUG only).
// ---------------------------------------------------------------------------
// NDF: the scene's ndf_kind fixed at compile time (0 GGX, 1 Beckmann) for the
// production kernel of the method, -1 = read from the scene (DEBUG, ablations,
// baseline): the GGX / Beckmann branches of S5 and of the shell disappear
template <bool DEBUG, int MODE, int NDF, bool KAT>
__device__ __forceinline__ void shade_pixel(const glint_scene& sc, const float* __restrict__ sZ,
                                            const float2* __restrict__ sCS, float4* outp, glint_debug_rec* rec,
                                            float4 duv, float4 uvm, float4 nrm, float4 pos, float4 mat,
                                            uint32_t seed_h, float inv_beta, uint32_t c1s, uint32_t c1n,
                                            bool f0_fast, int ka_lo, int ka_n) {
  const int ndf = NDF >= 0 ? NDF : sc.ndf_kind;
  const int L = sc.n_lights;
  uint32_t flags = 0;
  const uint32_t meta = __float_as_uint(uvm.w);
  const float u = uvm.x, v = uvm.y;
  bool ok = uv_ok(uvm);
  if (!ok) flags = (meta & 1u) ? (GLINT_FLAG_INVALID | GLINT_FLAG_UV_RANGE) : GLINT_FLAG_INVALID;
  // ---------------- S1: footprint (R-7, R-8)
  float P = 0.0f, r = 0.0f, psi = 0.0f;
  float zex = 1.0f, zey = 0.0f, zsmax = 0.0f;   // MODE 3: major axis, sigma_max (R-32)
  if (ok) {
    const Foot f = s1_moments(duv);
    const float a = f.a, b = f.b, c = f.c, lam = f.lam;
    P = f.P;
    r = lam * rcp_c(P);
    const float at = atan2_turns(2.0f * b, a - c);
    psi = at < 0.0f ? at + 1.0f : at;
    if (psi >= 1.0f) psi = 0.0f;
    if (!s1_valid(f)) {   // R-25, R-30b
      flags = GLINT_FLAG_DEGENERATE;
      ok = false;
    }
    if (MODE == 3) {
      float ex = a >= c ? lam - c : b;
      float ey = a >= c ? b : lam - a;
      const float l2 = ex * ex + ey * ey;
      if (l2 >= 0x1p-126f) {
        const float il = rsqrt_c(l2);
        ex = ex * il;
        ey = ey * il;
      } else {
        ex = 1.0f;
        ey = 0.0f;
      }
      zex = ex;
      zey = ey;
      zsmax = lam >= 0x1p-126f ? lam * rsqrt_c(lam) : 0.0f;
    }
  }
  if (!ok) {
    __stcs(outp, make_float4(0.0f, 0.0f, 0.0f, __uint_as_float(flags)));
    if (DEBUG) {
      for (int l = 0; l < L; ++l) {
        uint32_t* w = reinterpret_cast<uint32_t*>(rec + l);
        for (int q = 0; q < (int)(sizeof(glint_debug_rec) / 4); ++q) w[q] = 0u;
        rec[l].flags = flags;
      }
    }
    return;
  }

  // ---------------- S2: 4 grids + distribution weights, n_i = w_i N 2^ls
  Slot sl[4];
  constexpr int NGA = MODE == 2 ? 10 : 4;   // ablation grid list (MODE 1: the same 4 grids)
  int als[NGA], alr[NGA], ajo[NGA];
  float aw[NGA];
  int znp = 1;            // MODE 3: probes, their area and half-step (R-31, R-32)
  float zA = 0.0f, zq = 0.0f;
  if (MODE == 3) {
    for (int i = 0; i < 4; ++i) { sl[i].ls = 0; sl[i].lr = 0; sl[i].jo = 0; sl[i].w = 0.0f; }
    const float cr = ceilf(r);
    if (cr > 16.0f) flags |= GLINT_FLAG_RATIO_CLAMPED;
    znp = cr >= 16.0f ? 16 : (cr >= 1.0f ? (int)cr : 1);
    const float rn = rcp_c((float)znp);
    zA = P * rn;
    zq = 0.5f * rn;
  } else if (MODE == 2) {
    lattice10(P, r, psi, sc.max_ratio_level, als, alr, ajo, aw, flags);
    for (int i = 0; i < 4; ++i) { sl[i].ls = 0; sl[i].lr = 0; sl[i].jo = 0; sl[i].w = 0.0f; }
  } else {
    lattice(P, r, psi, sc.max_ratio_level, sl, flags);
    if (MODE == 1)
      for (int i = 0; i < 4; ++i) { als[i] = sl[i].ls; alr[i] = sl[i].lr; ajo[i] = sl[i].jo; aw[i] = sl[i].w; }
  }
  // material domain (R-37): roughness in [2^-16, 16], flake density in
  // [0, 2^40], ratio R in [0, 16]; NaN goes to the lower bound (max.f32 also
  // maps -0 to +0). Trial counts N 2^ls then stay below 2^104 and the radiance
  // denominator pi ax ay R N P below 2^116: no fp32 overflow anywhere
  const float ax = fminf(fmaxf(mat.x, 0x1p-16f), 16.0f), ay = fminf(fmaxf(mat.y, 0x1p-16f), 16.0f);
  const float N = fminf(fmaxf(mat.z, 0.0f), 0x1p40f);
  const float R = fminf(fmaxf(mat.w, 0.0f), 16.0f);
  float n[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) n[i] = sl[i].w * (N * pow2i(sl[i].ls));

  // ---------------- S3 + S4a: grid transform, simplex, spatial seeds (12)
  // hsC = hs * C1: the draw hash draw_hash(hs + ka) starts with (hs + ka) * C1 =
  // hsC + kaC, one add per draw.
  const uint32_t so = lowbias32(__float_as_uint(uvm.z) ^ seed_h);
  uint32_t hsC[12];
  float beta[12];
  uint32_t dlx[DEBUG ? 12 : 1], dly[DEBUG ? 12 : 1], dhs[DEBUG ? 12 : 1];
  float dfx[DEBUG ? 4 : 1] = {}, dfy[DEBUG ? 4 : 1] = {};
#pragma unroll
  for (int i = 0; i < (MODE == 0 ? 4 : 0); ++i) {
    GL_ASSERT(sl[i].lr >= 0 && sl[i].lr <= 8 && sl[i].jo >= 0 && (sl[i].jo >> sl[i].lr) == 0);
    const float2 cs = sCS[sl[i].jo << (8 - sl[i].lr)];
    const float xr = __fmaf_rn(cs.x, u, cs.y * v);
    const float yr = __fmaf_rn(cs.x, v, -(cs.y * u));
    // 2^((lr-ls)/2) = 2^(-(ls+lr)/2) * 2^lr exactly (power-of-two scaling)
    const float sxs = pow2half(-(sl[i].ls + sl[i].lr));
    const float gx = xr * sxs;
    const float gy = yr * (sxs * pow2i(sl[i].lr));
    const float xs = gx + 0.5f * gy;
    const float fxs = floorf(xs), fys = floorf(gy);
    const float fx = xs - fxs, fy = gy - fys;
    const uint32_t ix = (uint32_t)(long long)fxs, iy = (uint32_t)(long long)fys;
    const bool lower = fx >= fy;
    beta[i * 3 + 0] = 1.0f - (lower ? fx : fy);
    beta[i * 3 + 1] = lower ? fx - fy : fy - fx;
    beta[i * 3 + 2] = lower ? fy : fx;
    const uint32_t key = ((uint32_t)sl[i].ls & 511u) | ((uint32_t)sl[i].lr << 9) | ((uint32_t)sl[i].jo << 13);
    // seed of texel (key; lattice vertex): lowbias32(so + key K + lx A + ly B);
    // vertices (ix,iy), lower ? (ix+1,iy) : (ix,iy+1), (ix+1,iy+1)
    const uint32_t base = so + key * 0x9e3779b1U + ix * 0x8da6b343U + iy * 0xd8163841U;
    const uint32_t lin1 = base + (lower ? 0x8da6b343U : 0xd8163841U);
    const uint32_t lin2 = base + (0x8da6b343U + 0xd8163841U);
    const uint32_t h0 = lowbias32(base), h1 = lowbias32(lin1), h2 = lowbias32(lin2);
    hsC[i * 3 + 0] = h0 * c1s;
    hsC[i * 3 + 1] = h1 * c1s;
    hsC[i * 3 + 2] = h2 * c1s;
    if (DEBUG) {
      dfx[i] = fx; dfy[i] = fy;
      dlx[i * 3 + 0] = ix; dly[i * 3 + 0] = iy;
      dlx[i * 3 + 1] = lower ? ix + 1u : ix; dly[i * 3 + 1] = lower ? iy : iy + 1u;
      dlx[i * 3 + 2] = ix + 1u; dly[i * 3 + 2] = iy + 1u;
      dhs[i * 3 + 0] = h0; dhs[i * 3 + 1] = h1; dhs[i * 3 + 2] = h2;
    }
  }

  // ---------------- per-pixel shading frame (fp32 contract; R-17)
  float nx = nrm.x, ny = nrm.y, nz = nrm.z;
  normalize3(nx, ny, nz);
  const float sgn = copysignf(1.0f, nz);
  const float oa = -(sgn * rcp_c(1.0f + fabsf(nz)));   // = -1/(sgn + nz)
  const float ob = (nx * ny) * oa;
  const float tx = 1.0f + sgn * ((nx * nx) * oa), ty = sgn * ob, tz = -(sgn * nx);
  const float bx = ob, by = sgn + (ny * ny) * oa, bz = -ny;
  float wix, wiy, wiz;
  view_dir(sc, pos, wix, wiy, wiz);
  const float ni = dot3(nx, ny, nz, wix, wiy, wiz);
  const float iax = rcp_c(ax), iay = rcp_c(ay);
  // radiance accumulator, the fp32 tangential parts of w_i in the frame, and
  // the pixel's shell constants (computed at its first glint, S9)
  float3 rgb = make_float3(0.0f, 0.0f, 0.0f);
  bool have_px = false;
  float ci_c = 0.0f, lam_i = 0.0f, dq = 0.0f;
  const float ti = dot3(wix, wiy, wiz, tx, ty, tz), bi = dot3(wix, wiy, wiz, bx, by, bz);

  for (int l = 0; l < L; ++l) {
    const glint_light& lt = sc.lights[l];
    // ---------------- S5: light direction d (unnormalised), activity, h, p
    float dx, dy, dz, d2, nd;   // nd: sign of n.wo
    light_dir(lt, pos, nx, ny, nz, dx, dy, dz, d2, nd);
    glint_debug_rec* rc = DEBUG ? rec + l : nullptr;
    if (DEBUG) {
      uint32_t* w = reinterpret_cast<uint32_t*>(rc);
      for (int q = 0; q < (int)(sizeof(glint_debug_rec) / 4); ++q) w[q] = 0u;
      rc->P = P; rc->r = r; rc->psi = psi;
      for (int i = 0; i < 4; ++i) { rc->ls[i] = sl[i].ls; rc->lr[i] = sl[i].lr; rc->jo[i] = sl[i].jo; rc->w[i] = sl[i].w; rc->n[i] = n[i]; }
      for (int q = 0; q < 12; ++q) { rc->lx[q] = (int32_t)dlx[q]; rc->ly[q] = (int32_t)dly[q]; }
      for (int i = 0; i < 4; ++i) { rc->sfx[i] = dfx[i]; rc->sfy[i] = dfy[i]; }
    }
    // light below the horizon (R-27); |d|^2 a normal float (R-27b)
    if (!light_active(ni, nd, d2)) continue;
    if (DEBUG) rc->light_active = 1u;
    // h = normalize(|d| wi + d)  (proportional to wi + wo, one division less)
    const float dl = d2 * rsqrt_c(d2);
    float hx_ = __fmaf_rn(dl, wix, dx), hy_ = __fmaf_rn(dl, wiy, dy), hz_ = __fmaf_rn(dl, wiz, dz);
    normalize3(hx_, hy_, hz_);
    const float hx = dot3(hx_, hy_, hz_, tx, ty, tz);
    const float hy = dot3(hx_, hy_, hz_, bx, by, bz);
    const float hz = dot3(hx_, hy_, hz_, nx, ny, nz);
    // Eq. 4: p = R D(h)/D(n), GGX / Beckmann (R-19, R-22)
    float ratio = 0.0f;
    if (hz > 0.0f) {
      const float X = hx * iax, Y = hy * iay;
      const float s2 = X * X + Y * Y;
      const float hz2 = hz * hz;
      if (ndf == 0) {
        const float q = s2 + hz2;
        ratio = rcp_c(q * q);
      } else {
        const float e2 = s2 * rcp_c(hz2);
        ratio = exp2c(-(e2 * 0x1.715476p+0f)) * rcp_c(hz2 * hz2);
      }
    }
    float p = R * ratio;
    if (p > 1.0f) { p = 1.0f; flags |= GLINT_FLAG_P_CLAMPED; }
    if (!(p > 0.0f)) p = 0.0f;
    // Eq. 14 angular grid (R-17); angular seeds pre-multiplied by C1
    const float gxa = __fmaf_rn(hx, inv_beta, -0.5f), gya = __fmaf_rn(hy, inv_beta, -0.5f);
    const float cxf = floorf(gxa), cyf = floorf(gya);
    const float fxa = gxa - cxf, fya = gya - cyf;
    const int cx0 = (int)cxf, cy0 = (int)cyf;
    const float vj[4] = {(1.0f - fxa) * (1.0f - fya), fxa * (1.0f - fya), (1.0f - fxa) * fya, fxa * fya};
    uint32_t kaC[4];
    const uint32_t kix = (uint32_t)(cx0 - ka_lo), kiy = (uint32_t)(cy0 - ka_lo);
    if (KAT && ka_n > 0 && kix < (uint32_t)(ka_n - 1) && kiy < (uint32_t)(ka_n - 1)) {
      const int e = (int)kiy * ka_n + (int)kix;
      GL_ASSERT(e >= 0 && e + ka_n + 1 < kKaMax);
      kaC[0] = g_sKA[e]; kaC[1] = g_sKA[e + 1]; kaC[2] = g_sKA[e + ka_n]; kaC[3] = g_sKA[e + ka_n + 1];
    } else {
#pragma unroll
      for (int jn = 0; jn < 4; ++jn) {
        const uint32_t cx = (uint32_t)(cx0 + (jn & 1)), cy = (uint32_t)(cy0 + (jn >> 1));
        const uint32_t ka0 = lowbias32(cx * 0xcb1ab31fU + cy * 0x165667b1U + 0x27d4eb2fU);
        kaC[jn] = MODE == 3 ? ka0 : ka0 * c1n;
      }
    }
    if (DEBUG) { rc->p = p; rc->cx0 = cx0; rc->cy0 = cy0; rc->afx = fxa; rc->afy = fya; }

    // ---------------- S6 + S7 + S8: 48 gated draws, blended
    const float L2 = p >= 1.0f ? -__int_as_float(0x7f800000) : (p > 0.0f ? log2_1mp(p) : 0.0f);   // see gate_params
    float A[4] = {0.0f, 0.0f, 0.0f, 0.0f};   // A_j = sum_ik beta_ik c_ikj
    if (MODE == 3) {
      // ---- Zirr & Kaplanyan-style baseline: per LOD of
      // the pair around the probe area (Eq. 7 output mix, R-33), per probe
      // along the major axis (R-31/32), 4 bilinear texels x 4 angular nodes,
      // each an Eq. 15 classical binomial (R-34/35). Variable cost by design.
      const int32_t ez = (int32_t)((__float_as_uint(zA) >> 23) & 255u) - 127;
      const int32_t kz = ez >> 1;
      const float wt = (zA * pow2i(-2 * kz) - 1.0f) * (1.0f / 3.0f);
      const uint32_t Tp = (uint32_t)ceilf(p * 0x1p24f);
#pragma unroll 1
      for (int lev = 0; lev < 2; ++lev) {
        const int32_t lv = kz + lev;
        const float wl = lev ? wt : 1.0f - wt;
        float nt = N * pow2i(2 * lv);
        if (!(nt <= 0x1p64f)) nt = 0x1p64f;
        const float np_ = nt * p;
        const bool gauss = np_ > 5.0f || nt > 16.0f;
        const float sv = np_ * (1.0f - p);
        const float sg = sv >= 0x1p-126f ? sv * rsqrt_c(sv) : 0.0f;
        const float capz = ceilf(nt);
        const float nf = floorf(nt);
        const int nfi = gauss ? 0 : (int)nf;
        const uint32_t Tf = (uint32_t)ceilf(((nt - nf) * p) * 0x1p24f);
        const float s = pow2i(-lv);
        const uint32_t lkey = so + (uint32_t)lv * 0x5bd1e995U + 0x68e31da4U;
#pragma unroll 1
        for (int k = 0; k < znp; ++k) {
          const float off = ((float)(2 * k + 1 - znp) * zq) * zsmax;
          const float uk = __fmaf_rn(off, zex, u), vk = __fmaf_rn(off, zey, v);
          const float gx = __fmaf_rn(uk, s, -0.5f), gy = __fmaf_rn(vk, s, -0.5f);
          const float fxs = floorf(gx), fys = floorf(gy);
          const float fx = gx - fxs, fy = gy - fys;
          const uint32_t ix = (uint32_t)(long long)fxs, iy = (uint32_t)(long long)fys;
          const float bq[4] = {(1.0f - fx) * (1.0f - fy), fx * (1.0f - fy), (1.0f - fx) * fy, fx * fy};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t hz = lowbias32(lkey + (ix + (uint32_t)(q & 1)) * 0x8da6b343U +
                                          (iy + (uint32_t)(q >> 1)) * 0xd8163841U);
            const float wq = wl * bq[q];
#pragma unroll
            for (int jn = 0; jn < 4; ++jn) {
              const uint32_t w = lowbias32(hz + kaC[jn]);
              float c;
              if (gauss) {
                const float z = sZ[(w >> 2) & (GLINT_ZQ - 1)];
                float x = __fmaf_rn(sg, z, np_);
                x = x < 0.0f ? 0.0f : x;
                x = x > capz ? capz : x;
                c = floorf(x);
              } else {
                int cnt = (lowbias32(w + 16u * 0x9e3779b9U) >> 8) < Tf ? 1 : 0;
#pragma unroll 1
                for (int t = 0; t < nfi; ++t) cnt += (lowbias32(w + (uint32_t)t * 0x9e3779b9U) >> 8) < Tp ? 1 : 0;
                c = (float)cnt;
              }
              A[jn] = __fmaf_rn(wq, c, A[jn]);
            }
          }
        }
      }
    }
    if (MODE == 1 || MODE == 2) {
      // ---- ablations: NGA grids x 4 bilinear texels x 4 nodes,
      // everything per light (one grid at a time, rolled: small code)
#pragma unroll 1
      for (int g = 0; g < NGA; ++g) {
        const float ng = aw[g] * (N * pow2i(als[g]));
        const Gate gt = gate_params(ng, p, L2);
        const uint32_t G = (gt.T << 9) - 1u;
        const float capk = gt.T ? gt.cap : 0.0f;
        GL_ASSERT(alr[g] >= 0 && alr[g] <= 8 && ajo[g] >= 0 && (ajo[g] >> alr[g]) == 0);
        const float2 cs = sCS[ajo[g] << (8 - alr[g])];
        const float xr = __fmaf_rn(cs.x, u, cs.y * v);
        const float yr = __fmaf_rn(cs.x, v, -(cs.y * u));
        const float sxs = pow2half(-(als[g] + alr[g]));
        const float gx = xr * sxs;
        const float gy = yr * (sxs * pow2i(alr[g]));
        const float fxs = floorf(gx), fys = floorf(gy);
        const float fx = gx - fxs, fy = gy - fys;
        const uint32_t ix = (uint32_t)(long long)fxs, iy = (uint32_t)(long long)fys;
        const float bw[4] = {(1.0f - fx) * (1.0f - fy), fx * (1.0f - fy), (1.0f - fx) * fy, fx * fy};
        const uint32_t key = ((uint32_t)als[g] & 511u) | ((uint32_t)alr[g] << 9) | ((uint32_t)ajo[g] << 13);
        const uint32_t base = so + key * 0x9e3779b1U + ix * 0x8da6b343U + iy * 0xd8163841U;
        const uint32_t lin[4] = {base, base + 0x8da6b343U, base + 0xd8163841U, base + (0x8da6b343U + 0xd8163841U)};
        uint32_t hC[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) hC[k] = lowbias32(lin[k]) * c1s;
        if (!DEBUG && GLINT_GATE_FIRST) {
          // gates before counts, as for the method's 48 draws (a fair ablation)
          bool pass = false;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
#pragma unroll
            for (int jn = 0; jn < 4; ++jn) {
              uint32_t y = hC[k] + kaC[jn];
              y ^= __funnelshift_r(y, y, 11) ^ __funnelshift_r(y, y, 19);
              y *= 0x846ca68bU;
              pass = pass || (y <= G);
            }
          }
          if (!__any_sync(__activemask(), pass && gt.T != 0u)) continue;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
#pragma unroll
          for (int jn = 0; jn < 4; ++jn) {
            uint32_t y = hC[k] + kaC[jn];
            y ^= __funnelshift_r(y, y, 11) ^ __funnelshift_r(y, y, 19);
            y *= 0x846ca68bU;
            const uint32_t s16 = y >> 16;
            const float z = *reinterpret_cast<const float*>(reinterpret_cast<const char*>(sZ) + ((y ^ s16) & 0x3FFCu));
            const float c = floorf(fminf(fmaxf(__fmaf_rn(gt.sigma, z, gt.m1), 1.0f), capk));
            if (y <= G) A[jn] = __fmaf_rn(bw[k], c, A[jn]);
          }
        }
      }
    }
    // lanes shading this light (invalid pixels and lights below the horizon
    // left earlier); warp votes below use this mask
    const uint32_t am = __activemask();
#pragma unroll
    for (int i = 0; i < (MODE == 0 ? 4 : 0); ++i) {
      // a grid with no trials (zero distribution weight: ring-0 merges,
      // isotropic footprints) or p = 0 draws only zeros; neighbouring pixels
      // share their grid structure, so skip it when the whole warp agrees
      // (results unchanged)
      if (!DEBUG && !__any_sync(am, n[i] > 0.0f && p > 0.0f)) continue;
      // gate (y >> 9) < T  <=>  y <= T*512 - 1; T = 0 wraps to "always" but its
      // cap is forced to 0 so the count is 0 (same result, one compare)
      Gate gt;
      if (DEBUG || !GLINT_GATE_FIRST) {
        gt = gate_params(n[i], p, L2);
      } else {
        // gates first (production): a grid none of whose 12 x 32 lane-draws
        // passes its gate adds nothing, so its count work (sigma / m1 / cap,
        // quantile load, clamp, floor, accumulate) is skipped by a warp vote.
        // Glints are sparse: on C2 / C4 only 20-50 % of the warp-grids have
        // a passing draw. Results unchanged (production == DEBUG tests).
        gt.T = gate_T(n[i], p, L2);
        const uint32_t Gg = (gt.T << 9) - 1u;
        bool pass = false;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
#pragma unroll
          for (int jn = 0; jn < 4; ++jn) {
            uint32_t y = hsC[i * 3 + k] + kaC[jn];
            y ^= __funnelshift_r(y, y, 11) ^ __funnelshift_r(y, y, 19);
            y *= 0x846ca68bU;
            pass = pass || (y <= Gg);
          }
        }
        if (!__any_sync(am, pass && gt.T != 0u)) continue;
        gate_counts(n[i], p, gt);
      }
      const uint32_t G = (gt.T << 9) - 1u;
      const float capk = gt.T ? gt.cap : 0.0f;
      if (DEBUG) {
        const bool none = !(n[i] > 0.0f) || !(p > 0.0f);
        rc->T[i] = gt.T;
        rc->sigma[i] = none ? 0.0f : gt.sigma;
        rc->m1[i] = none ? 1.0f : gt.m1;
        rc->cap[i] = none ? 1.0f : gt.cap;
        rc->pge1[i] = none ? 0.0f : 1.0f - exp2c(n[i] * L2);   // gate_T's P>=1
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const float bk = beta[i * 3 + k];
#pragma unroll
        for (int jn = 0; jn < 4; ++jn) {
          uint32_t y = hsC[i * 3 + k] + kaC[jn];        // (hs + ka) * C1
          y ^= __funnelshift_r(y, y, 11) ^ __funnelshift_r(y, y, 19);   // bijective xor-rotate (R-23b)
          y *= 0x846ca68bU;                              // y: gate bits 9..31
          const uint32_t s16 = y >> 16;                  // h = y ^ (y >> 16): quantile bits 2..13
          const float z = *reinterpret_cast<const float*>(reinterpret_cast<const char*>(sZ) + ((y ^ s16) & 0x3FFCu));
          const float c = floorf(fminf(fmaxf(__fmaf_rn(gt.sigma, z, gt.m1), 1.0f), capk));
          if (y <= G) A[jn] = __fmaf_rn(bk, c, A[jn]);
          if (DEBUG) { rc->hash[i * 12 + k * 4 + jn] = y ^ s16; rc->count[i * 12 + k * 4 + jn] = (y <= G) ? c : 0.0f; }
        }
      }
    }
    const float C = __fmaf_rn(vj[3], A[3], __fmaf_rn(vj[2], A[2], __fmaf_rn(vj[1], A[1], vj[0] * A[0])));
    if (DEBUG) {
      rc->C = C;
      rc->Dp = C > 0.0f ? (float)((double)C * rcp_d(3.141592653589793 * (double)ax * (double)ay * (double)R * (double)N *
                                                    (double)P))
                        : 0.0f;
    }
    // ---------------- S8/S9: D_P and radiance (Eq. 1-3), fp64 shell.
    // Warp-uniform: lanes with C = 0 add exactly nothing (the shell returns
    // at once), so the block runs without per-lane divergence
    if (DEBUG ? (C > 0.0f) : __any_sync(am, C > 0.0f)) {
      if (C > 0.0f) {
        if (!have_px) {   // the pixel's shell constants, once (per-pixel work shared by the lights)
          have_px = true;
          ci_c = ni;
          lam_i = lambda32(ndf, __fmaf_rn(ax * ax, ti * ti, ay * ay * (bi * bi)), ci_c);
          dq = 3.14159265358979f * ax * ay * R * N * P * (4.0f * ci_c);
        }
        // w_o's tangential parts by reflecting w_i about h (fp32 frame): w_o = 2 (w_i.h) h - w_i
        const float cih = dot3(wix, wiy, wiz, hx_, hy_, hz_);
        const float to = __fmaf_rn(2.0f * cih, hx, -ti), bo = __fmaf_rn(2.0f * cih, hy, -bi);
        const float rs = rsqrt_c(d2);   // the decision path's (dl = d2 rs)
        if (!(f0_fast && radiance_shell32(sc, ndf, lt, ci_c, lam_i, nd * rs, cih, to, bo, ax * ax, ay * ay, dq, rs, C, rgb))) {
          const float3 c = radiance_shell64(ndf, sc.view_kind, lt.kind, sc.view[0], sc.view[1], sc.view[2],
                                            lt.pos_or_dir[0], lt.pos_or_dir[1], lt.pos_or_dir[2], lt.intensity[0],
                                            lt.intensity[1], lt.intensity[2], sc.f0[0], sc.f0[1], sc.f0[2], nrm, pos,
                                            ti, bi, to, bo, ax * ax, ay * ay, 3.14159265358979f * ax * ay * R * N * P,
                                            C);
          rgb.x += c.x;
          rgb.y += c.y;
          rgb.z += c.z;
        }
      }
    }
  }
  if (DEBUG) for (int l = 0; l < L; ++l) rec[l].flags = flags;
  __stcs(outp, make_float4(rgb.x, rgb.y, rgb.z, __uint_as_float(flags)));
}

// ---------------------------------------------------------------------------
// The kernel: persistent blocks over kTile-pixel tiles, claimed dynamically
// (the first two are blockIdx.x and one claim, later ones come from this
// launch's counter: balances per-tile cost variance and the tail). Tiles
// stream through a ring of kStages shared-memory stages; each stage has a
// full mbarrier (tile id + bytes landed) and a counter of warps done with it.
// The LAST warp to finish a stage knows it is free: it claims the tile
// kStages iterations ahead and (TMA: contiguous G-buffer, pitch == width)
// issues its 5 bulk copies into that stage. No producer warp, no block-wide
// barrier inside the loop; a warp can run up to kStages - 1 tiles ahead of
// the slowest one. Without TMA the ring carries only tile ids.
// ---------------------------------------------------------------------------
template <bool DEBUG, bool TMA, int MODE, int NDF, bool KAT>
__global__ void __launch_bounds__(kBlock, kMinBlocks) glint_eval_kernel(const KParams prm) {
  float* sZ = g_sZ;
  float2* sCS = g_sCS;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* tbar = reinterpret_cast<uint64_t*>(smem);   // tables loaded
  uint64_t* full = tbar + 1;                             // [kStages] tile (and its bytes) ready
  long long* s_tile = reinterpret_cast<long long*>(full + kStages);   // [kStages] tile ids
  uint32_t* s_done = reinterpret_cast<uint32_t*>(s_tile + kStages);   // [kStages] warps done
  float4* tiles = reinterpret_cast<float4*>(smem + kSmemTables);
  const int tid = threadIdx.x, lane = tid & 31;

  const glint_scene& sc = prm.sc;
  const int64_t n_pix = (int64_t)prm.width * prm.height;
  const int64_t n_tiles = (n_pix + kTile - 1) / kTile;
  const float inv_beta = 1.0f / sc.beta;
  const uint32_t seed_h = lowbias32(sc.seed);
  const bool flat_out = prm.out_pitch == prm.width;
  // node-seed table extent: cx, cy in [ka_lo, ka_lo + ka_n) (ka_n = 0: none)
  int ka_lo = 0, ka_n = 0;
  if (KAT && inv_beta <= 29.0f) {
    const int cb = (int)ceilf(inv_beta);
    ka_lo = -cb - 2;
    ka_n = 2 * cb + 5;
  }

  auto issue = [&](int64_t t, int b) {   // one thread: tile t into stage b (or just its id)
    s_tile[b] = t;
    if (TMA && t < n_tiles) {
      const int64_t base = t * kTile;
      const int64_t cnt = (n_pix - base) < kTile ? (n_pix - base) : kTile;
      GL_ASSERT(t >= 0 && base < n_pix && cnt > 0 && b >= 0 && b < kStages);
      const uint32_t bytes = (uint32_t)cnt * 16u;
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&full[b], 5u * bytes);
      bulk_g2s(tiles + (b * 5 + 0) * kTile, prm.duv + base, bytes, &full[b]);
      bulk_g2s(tiles + (b * 5 + 1) * kTile, prm.uvm + base, bytes, &full[b]);
      bulk_g2s(tiles + (b * 5 + 2) * kTile, prm.nrm + base, bytes, &full[b]);
      bulk_g2s(tiles + (b * 5 + 3) * kTile, prm.pos + base, bytes, &full[b]);
      bulk_g2s(tiles + (b * 5 + 4) * kTile, prm.mat + base, bytes, &full[b]);
    } else {
      mbar_arrive(&full[b]);
    }
  };
  auto claim = [&]() -> int64_t { return (int64_t)gridDim.x + (int64_t)atomicAdd(&prm.sched[0], 1ull); };

  // the next frame of a glint_eval_batch may launch now: its blocks fill the
  // SMs this grid's blocks free at its tail (frames of a batch are independent)
  pdl_launch_dependents();
  if (tid == 0) {
    mbar_init(tbar, 1);
    for (int s = 0; s < kStages; ++s) { mbar_init(&full[s], 1); s_done[s] = 0u; }
    fence_mbar_init();
    // tables: one bulk copy each (16 KB quantiles, 2 KB orientations)
    mbar_arrive_expect_tx(tbar, (uint32_t)(kSmemZ + kSmemCS));
    bulk_g2s(sZ, prm.ztab, (uint32_t)kSmemZ, tbar);
    bulk_g2s(sCS, prm.cstab, (uint32_t)kSmemCS, tbar);
    const bool any = (int64_t)blockIdx.x < n_tiles;
    issue(blockIdx.x, 0);
    for (int s = 1; s < kStages; ++s) issue(any ? claim() : n_tiles, s);
  }
  for (int e = tid; e < ka_n * ka_n; e += kBlock) {   // node-seed table (same arithmetic as S5's)
    const int iy = e / ka_n, ix = e - iy * ka_n;
    const uint32_t cx = (uint32_t)(ka_lo + ix), cy = (uint32_t)(ka_lo + iy);
    g_sKA[e] = lowbias32(cx * 0xcb1ab31fU + cy * 0x165667b1U + 0x27d4eb2fU) * prm.c1n;
  }
  __syncthreads();   // barriers initialised, node-seed table built
  mbar_wait(tbar, 0u);

  for (int it = 0;; ++it) {
    const int s = it % kStages;
    mbar_wait(&full[s], (uint32_t)(it / kStages) & 1u);
    const int64_t t = s_tile[s];
    if (t >= n_tiles) break;
#pragma unroll 1
    for (int q = 0; q < kPPT; ++q) {
      const int slot = q * kBlock + tid;
      const int64_t idx = t * kTile + slot;
      if (idx >= n_pix) break;
      float4 duv, uvm, nrm, pos, mat;
      int64_t oi = idx;
      if (TMA) {
        const float4* tb = tiles + s * 5 * kTile + slot;
        duv = tb[0]; uvm = tb[kTile]; nrm = tb[2 * kTile]; pos = tb[3 * kTile]; mat = tb[4 * kTile];
        if (!flat_out) {
          const uint32_t y = (uint32_t)idx / (uint32_t)prm.width;
          oi = (int64_t)y * prm.out_pitch + ((uint32_t)idx - y * (uint32_t)prm.width);
        }
      } else {
        const uint32_t y = (uint32_t)idx / (uint32_t)prm.width;
        const uint32_t x = (uint32_t)idx - y * (uint32_t)prm.width;
        const int64_t gi = (int64_t)y * prm.pitch + x;
        duv = __ldcs(prm.duv + gi); uvm = __ldcs(prm.uvm + gi); nrm = __ldcs(prm.nrm + gi);
        pos = __ldcs(prm.pos + gi); mat = __ldcs(prm.mat + gi);
        oi = (int64_t)y * prm.out_pitch + x;
      }
      GL_ASSERT(idx >= 0 && idx < n_pix && oi >= 0 &&
                oi < (int64_t)(prm.height - 1) * prm.out_pitch + prm.width && slot < kTile);
      shade_pixel<DEBUG, MODE, NDF, KAT>(sc, sZ, sCS, prm.out + oi, DEBUG ? prm.dbg + idx * sc.n_lights : nullptr, duv, uvm,
                               nrm, pos, mat, seed_h, inv_beta, prm.c1s, prm.c1n, prm.f0_fast != 0, ka_lo, ka_n);
    }
    __syncwarp();
    if (lane == 0) {
      // this warp is done with stage s (its reads ordered before the count)
      __threadfence_block();
      if (atomicAdd(&s_done[s], 1u) == (uint32_t)(kWarps - 1)) {
        __threadfence_block();
        s_done[s] = 0u;
        issue(claim(), s);   // the tile kStages iterations ahead
      }
    }
  }
  // all claims of this block precede its finish; the last block to finish
  // resets this launch's counters for the next use of the slot
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(&prm.sched[1], 1ull) == (unsigned long long)(gridDim.x - 1)) {
      prm.sched[0] = 0ull;
      prm.sched[1] = 0ull;
      __threadfence();
    }
    // a batch frame completes only after the frame before it: work that
    // follows the batch in the stream then sees every frame complete
    pdl_wait_prerequisites();
  }
}

template <bool DEBUG, bool TMA, int MODE, int NDF = -1, bool KAT = false>
static cudaError_t launch_t(const KParams& prm, int grid, cudaStream_t stream, bool pdl) {
  const size_t smem = TMA ? kSmemTma : kSmemTables;
  // the dynamic shared-memory opt-in, once per (instantiation, device);
  // concurrent first launches from several host threads may both set it
  // (idempotent), the flag itself is atomic
  static std::atomic<uint64_t> configured{0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (!(configured.load(std::memory_order_acquire) & bit)) {
    e = cudaFuncSetAttribute(glint_eval_kernel<DEBUG, TMA, MODE, NDF, KAT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    if (e != cudaSuccess) return e;
    configured.fetch_or(bit, std::memory_order_release);
  }
  if (!pdl) {
    glint_eval_kernel<DEBUG, TMA, MODE, NDF, KAT><<<grid, kBlock, smem, stream>>>(prm);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kBlock);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, glint_eval_kernel<DEBUG, TMA, MODE, NDF, KAT>, prm);
}

cudaError_t launch_eval(const KParams& prm, int grid, bool debug, cudaStream_t stream, bool pdl) {
  const bool tma = (prm.pitch == prm.width) && (((uintptr_t)prm.duv | (uintptr_t)prm.uvm | (uintptr_t)prm.nrm |
                                                  (uintptr_t)prm.pos | (uintptr_t)prm.mat) % 16 == 0);
  if (debug)
    return tma ? launch_t<true, true, 0>(prm, grid, stream, pdl) : launch_t<true, false, 0>(prm, grid, stream, pdl);
  // the angular node-seed table (see g_sKA) pays with several lights; with one
  // light the four independent hash chains hide better than its LDS latency
  // (C2 -0.4 % with the table), and small beta would overflow it
  const bool kat = GLINT_KA_TABLE && prm.sc.n_lights >= 2 && 1.0f / prm.sc.beta <= 29.0f;
  switch (prm.sc.eval_mode) {
    case 1:
      if (kat) return tma ? launch_t<false, true, 1, -1, true>(prm, grid, stream, pdl) : launch_t<false, false, 1, -1, true>(prm, grid, stream, pdl);
      return tma ? launch_t<false, true, 1>(prm, grid, stream, pdl) : launch_t<false, false, 1>(prm, grid, stream, pdl);
    case 2:
      if (kat) return tma ? launch_t<false, true, 2, -1, true>(prm, grid, stream, pdl) : launch_t<false, false, 2, -1, true>(prm, grid, stream, pdl);
      return tma ? launch_t<false, true, 2>(prm, grid, stream, pdl) : launch_t<false, false, 2>(prm, grid, stream, pdl);
    case 3:
      return tma ? launch_t<false, true, 3>(prm, grid, stream, pdl) : launch_t<false, false, 3>(prm, grid, stream, pdl);
    default:
      if (kat) {
        if (prm.sc.ndf_kind == 0)
          return tma ? launch_t<false, true, 0, 0, true>(prm, grid, stream, pdl) : launch_t<false, false, 0, 0, true>(prm, grid, stream, pdl);
        return tma ? launch_t<false, true, 0, 1, true>(prm, grid, stream, pdl) : launch_t<false, false, 0, 1, true>(prm, grid, stream, pdl);
      }
      if (prm.sc.ndf_kind == 0)
        return tma ? launch_t<false, true, 0, 0>(prm, grid, stream, pdl) : launch_t<false, false, 0, 0>(prm, grid, stream, pdl);
      return tma ? launch_t<false, true, 0, 1>(prm, grid, stream, pdl) : launch_t<false, false, 0, 1>(prm, grid, stream, pdl);
  }
}

// ---------------------------------------------------------------------------
// glint_count_active: the (pixel, light) pairs whose S5-S9 work glint_eval
// does, with the kernel's own decision functions (uv_ok, s1_moments/s1_valid,
// view_dir, light_dir/light_active). Grid-stride, one warp-reduced atomic per
// warp into the caller's counter.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) count_active_kernel(const float4* __restrict__ duv, const float4* __restrict__ uvm,
                                                           const float4* __restrict__ nrm, const float4* __restrict__ pos,
                                                           int32_t width, int64_t n_pix, int64_t pitch,
                                                           const glint_scene sc, unsigned long long* count) {
  unsigned long long c = 0;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n_pix; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t y = idx / width, x = idx - y * width;
    const int64_t gi = y * pitch + x;
    const float4 u = uvm[gi];
    if (!uv_ok(u)) continue;
    if (!s1_valid(s1_moments(duv[gi]))) continue;
    const float4 nr = nrm[gi], ps = pos[gi];
    float nx = nr.x, ny = nr.y, nz = nr.z;
    normalize3(nx, ny, nz);
    float wix, wiy, wiz;
    view_dir(sc, ps, wix, wiy, wiz);
    const float ni = dot3(nx, ny, nz, wix, wiy, wiz);
    for (int l = 0; l < sc.n_lights; ++l) {
      float dx, dy, dz, d2, nd;
      light_dir(sc.lights[l], ps, nx, ny, nz, dx, dy, dz, d2, nd);
      c += light_active(ni, nd, d2) ? 1ull : 0ull;
    }
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

cudaError_t launch_count_active(const float4* duv, const float4* uvm, const float4* nrm, const float4* pos, int32_t width,
                                int32_t height, int64_t pitch, const glint_scene& sc, unsigned long long* count,
                                int grid, cudaStream_t stream) {
  count_active_kernel<<<grid, 256, 0, stream>>>(duv, uvm, nrm, pos, width, (int64_t)width * height, pitch, sc, count);
  return cudaGetLastError();
}

cudaError_t occupancy_blocks_per_sm(int* out) {
  cudaError_t e = cudaFuncSetAttribute(glint_eval_kernel<false, true, 0, 0, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)kSmemTma);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, glint_eval_kernel<false, true, 0, 0, false>, kBlock, kSmemTma);
}

}  // namespace glint
