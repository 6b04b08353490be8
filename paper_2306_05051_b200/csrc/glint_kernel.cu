// glint_kernel.cu -- the fused sm_100a glint evaluation kernel (S0..S9).
//
// One thread shades one pixel for all lights. Per pixel (shared by every
// light): S0 coalesced float4 loads, S1 footprint, S2 lattice
// (4 grids), S3 grid transform + simplex (12 texels), S4a spatial seeds.
// Per light: S5 half-vector / p / angular nodes, S6 gate parameters of the 4
// grids, S7 the 48 gated draws (fully unrolled, hashes finished in
// registers, quantiles from a shared-memory table), S8 blend, S9 radiance.
//
// The block count is capped at (#SMs x resident blocks per SM) and blocks
// stride over the image, so the 18 KB of tables are staged into shared memory
// once per resident block, not once per 256 pixels.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/glint.h"
#include "glint_device.cuh"
#include "glint_kernel.h"

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

  int k0, k1, k2;
  float w0, w1, w2;
  float ht = 0.5f * tr;
  if (a <= ht) {                       // T0 = {A00, A10, A11}
    k0 = kA00; k1 = kA10; k2 = kA11;
    w0 = 1.0f - tr;
    w2 = a + a;
    w1 = tr - w2;
  } else if (a >= 1.0f - ht) {         // T2 = {A01, A11, A12}
    float om = 1.0f - a;
    k0 = kA01; k1 = kA11; k2 = kA12;
    w0 = 1.0f - tr;
    w1 = om + om;
    w2 = tr - w1;
  } else {                             // T1 = {A00, A11, A01}
    k0 = kA00; k1 = kA11; k2 = kA01;
    w0 = (1.0f - a) - ht;
    w1 = tr;
    w2 = a - ht;
  }
  // merge coincident vertices (ring 0), in (0,1), (0,2), (1,2) order (R-13)
  if (k1 == k0) { w0 = w0 + w1; w1 = 0.0f; }
  if (k2 == k0) { w0 = w0 + w2; w2 = 0.0f; }
  if (k2 == k1) { w1 = w1 + w2; w2 = 0.0f; }
  // stable sort by key: compare-swaps (0,1), (1,2), (0,1)  (R-12 global order)
#define GL_CSWAP(ka, wa, kb, wb) \
  if (ka > kb) { int tk = ka; ka = kb; kb = tk; float tw = wa; wa = wb; wb = tw; }
  GL_CSWAP(k0, w0, k1, w1);
  GL_CSWAP(k1, w1, k2, w2);
  GL_CSWAP(k0, w0, k1, w1);
#undef GL_CSWAP
  // prism -> 3 tetrahedra, staircase fill of the top level (R-12)
  float al = w0, be = w1, ga = w2;
  float t = ts;
  float ab = al + be;
  int kk[4], ll[4];
  float ww[4];
  if (t <= al) {
    kk[0] = k0; ll[0] = es;     ww[0] = al - t;
    kk[1] = k1; ll[1] = es;     ww[1] = be;
    kk[2] = k2; ll[2] = es;     ww[2] = ga;
    kk[3] = k0; ll[3] = es + 1; ww[3] = t;
  } else if (t <= ab) {
    kk[0] = k1; ll[0] = es;     ww[0] = ab - t;
    kk[1] = k2; ll[1] = es;     ww[1] = ga;
    kk[2] = k0; ll[2] = es + 1; ww[2] = al;
    kk[3] = k1; ll[3] = es + 1; ww[3] = t - al;
  } else {
    kk[0] = k2; ll[0] = es;     ww[0] = 1.0f - t;
    kk[1] = k0; ll[1] = es + 1; ww[1] = al;
    kk[2] = k1; ll[2] = es + 1; ww[2] = be;
    kk[3] = k2; ll[3] = es + 1; ww[3] = (t - al) - be;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    s[i].ls = ll[i];
    s[i].lr = kk[i] >> 9;
    s[i].jo = kk[i] & 511;
    s[i].w = ww[i];
  }
}

// fp32 Smith Lambda for the radiance path (R-21)
__device__ __forceinline__ float smith_lambda(int kind, float ax2, float ay2, float wx, float wy, float wz) {
  float s = ax2 * (wx * wx) + ay2 * (wy * wy);
  if (!(s > 0.0f)) return 0.0f;
  if (kind == 0) {
    float q = s / (wz * wz);
    return q / (2.0f * (1.0f + sqrtf(1.0f + q)));
  }
  float a = wz * rsqrtf(s);
  if (a >= 1.6f) return 0.0f;
  return __fdividef(1.0f - 1.259f * a + 0.396f * a * a, 3.535f * a + 2.181f * a * a);
}

// ---------------------------------------------------------------------------
// The kernel
// ---------------------------------------------------------------------------
template <bool DEBUG>
__global__ void __launch_bounds__(kBlock) glint_eval_kernel(const KParams prm) {
  __shared__ float sZ[GLINT_ZQ];
  __shared__ float2 sCS[GLINT_NANG];
  for (int i = threadIdx.x; i < GLINT_ZQ; i += kBlock) sZ[i] = prm.ztab[i];
  for (int i = threadIdx.x; i < GLINT_NANG; i += kBlock) sCS[i] = prm.cstab[i];
  __syncthreads();

  const glint_scene& sc = prm.sc;
  const int L = sc.n_lights;
  const int64_t n_pix = (int64_t)prm.width * prm.height;
  const float inv_beta = 1.0f / sc.beta;
  const uint32_t seed_h = lowbias32(sc.seed);

  for (int64_t idx = (int64_t)blockIdx.x * kBlock + threadIdx.x; idx < n_pix;
       idx += (int64_t)gridDim.x * kBlock) {
    const int y = (int)(idx / prm.width);
    const int x = (int)(idx - (int64_t)y * prm.width);
    const int64_t gi = (int64_t)y * prm.pitch + x;
    // ---------------- S0: coalesced float4 loads (read-once, streaming)
    const float4 duv = __ldcs(prm.duv + gi);
    const float4 uvm = __ldcs(prm.uvm + gi);
    const float4 nrm = __ldcs(prm.nrm + gi);
    const float4 pos = __ldcs(prm.pos + gi);
    const float4 mat = __ldcs(prm.mat + gi);
    glint_debug_rec* rec = DEBUG ? prm.dbg + idx * L : nullptr;

    uint32_t flags = 0;
    float3 rgb = make_float3(0.0f, 0.0f, 0.0f);
    const uint32_t meta = __float_as_uint(uvm.w);
    const float u = uvm.x, v = uvm.y;
    bool ok = (meta & 1u) != 0;
    if (!ok) flags = GLINT_FLAG_INVALID;
    if (ok && !(fabsf(u) <= 0x1p24f && fabsf(v) <= 0x1p24f)) {
      flags = GLINT_FLAG_INVALID | GLINT_FLAG_UV_RANGE;
      ok = false;
    }
    // ---------------- S1: footprint (R-7, R-8)
    float P = 0.0f, r = 0.0f, psi = 0.0f;
    if (ok) {
      const float dudx = duv.x, dvdx = duv.y, dudy = duv.z, dvdy = duv.w;
      const float det = dudx * dvdy - dvdx * dudy;
      const float a = dudx * dudx + dudy * dudy;
      const float b = dudx * dvdx + dudy * dvdy;
      const float c = dvdx * dvdx + dvdy * dvdy;
      const float hm = 0.5f * (a - c);
      const float disc = sqrtf(hm * hm + b * b);
      const float lam = 0.5f * (a + c) + disc;
      P = fabsf(det);
      r = lam / P;
      const float at = atan2_turns(2.0f * b, a - c);
      psi = at < 0.0f ? at + 1.0f : at;
      if (psi >= 1.0f) psi = 0.0f;
      if (!(P >= 0x1p-64f && P < 0x1p64f)) {
        flags = GLINT_FLAG_DEGENERATE;
        ok = false;
      }
    }
    if (!ok) {
      prm.out[(int64_t)y * prm.out_pitch + x] = make_float4(0.0f, 0.0f, 0.0f, __uint_as_float(flags));
      if (DEBUG) {
        for (int l = 0; l < L; ++l) {
          uint32_t* w = reinterpret_cast<uint32_t*>(rec + l);
          for (int q = 0; q < (int)(sizeof(glint_debug_rec) / 4); ++q) w[q] = 0u;
          rec[l].flags = flags;
        }
      }
      continue;
    }

    // ---------------- S2: 4 grids + distribution weights, n_i = w_i N 2^ls
    Slot sl[4];
    lattice(P, r, psi, sc.max_ratio_level, sl, flags);
    const float ax = mat.x, ay = mat.y, N = mat.z, R = mat.w;
    float n[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) n[i] = sl[i].w * (N * pow2i(sl[i].ls));

    // ---------------- S3 + S4a: grid transform, simplex, spatial seeds
    const uint32_t so = lowbias32(__float_as_uint(uvm.z) ^ seed_h);
    uint32_t hsx[12];   // lowbias32 spatial hash, pre-xorshifted by 16 for the draw hash
    float beta[12];
    uint32_t dlx[DEBUG ? 12 : 1], dly[DEBUG ? 12 : 1];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 cs = sCS[sl[i].jo << (8 - sl[i].lr)];
      const float xr = __fmaf_rn(cs.x, u, cs.y * v);
      const float yr = __fmaf_rn(cs.x, v, -(cs.y * u));
      const float gx = xr * pow2half(-(sl[i].ls + sl[i].lr));
      const float gy = yr * pow2half(sl[i].lr - sl[i].ls);
      const float xs = gx + 0.5f * gy;
      const float fxs = floorf(xs), fys = floorf(gy);
      const float fx = xs - fxs, fy = gy - fys;
      const uint32_t ix = (uint32_t)(long long)fxs, iy = (uint32_t)(long long)fys;
      const bool lower = fx >= fy;
      // vertices: (ix,iy), lower ? (ix+1,iy) : (ix,iy+1), (ix+1,iy+1)
      const uint32_t lx1 = lower ? ix + 1u : ix, ly1 = lower ? iy : iy + 1u;
      beta[i * 3 + 0] = 1.0f - (lower ? fx : fy);
      beta[i * 3 + 1] = lower ? fx - fy : fy - fx;
      beta[i * 3 + 2] = lower ? fy : fx;
      const uint32_t key = ((uint32_t)sl[i].ls & 511u) | ((uint32_t)sl[i].lr << 9) | ((uint32_t)sl[i].jo << 13);
      const uint32_t g = lowbias32(so ^ key);
      const uint32_t lxs[3] = {ix, lx1, ix + 1u}, lys[3] = {iy, ly1, iy + 1u};
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const uint32_t hs = lowbias32(g ^ (lxs[k] * 0x8da6b343U + lys[k] * 0xd8163841U));
        hsx[i * 3 + k] = hs ^ (hs >> 16);
        if (DEBUG) { dlx[i * 3 + k] = lxs[k]; dly[i * 3 + k] = lys[k]; }
      }
    }

    // ---------------- per-pixel shading frame (fp32 contract; R-17)
    float nx = nrm.x, ny = nrm.y, nz = nrm.z;
    normalize3(nx, ny, nz);
    const float sgn = copysignf(1.0f, nz);
    const float oa = -1.0f / (sgn + nz);
    const float ob = (nx * ny) * oa;
    const float tx = 1.0f + sgn * ((nx * nx) * oa), ty = sgn * ob, tz = -(sgn * nx);
    const float bx = ob, by = sgn + (ny * ny) * oa, bz = -ny;
    float wix, wiy, wiz;
    if (sc.view_kind == 0) { wix = sc.view[0] - pos.x; wiy = sc.view[1] - pos.y; wiz = sc.view[2] - pos.z; }
    else { wix = sc.view[0]; wiy = sc.view[1]; wiz = sc.view[2]; }
    normalize3(wix, wiy, wiz);
    const float ni = dot3(nx, ny, nz, wix, wiy, wiz);
    const float wilx = dot3(wix, wiy, wiz, tx, ty, tz), wily = dot3(wix, wiy, wiz, bx, by, bz);
    const float ax2 = ax * ax, ay2 = ay * ay;
    const float lam_i = smith_lambda(sc.ndf_kind, ax2, ay2, wilx, wily, ni);
    // D_P = C * Dn / (R N P) with D(n) = 1 / (pi ax ay)  (Eq. 3-4, R-20)
    const float dp_scale = 1.0f / (3.14159265358979f * ax * ay * R * N * P);

    for (int l = 0; l < L; ++l) {
      const glint_light& lt = sc.lights[l];
      // ---------------- S5: light direction, activity, h, p, angular nodes
      float wox, woy, woz;
      if (lt.kind == 0) { wox = lt.pos_or_dir[0] - pos.x; woy = lt.pos_or_dir[1] - pos.y; woz = lt.pos_or_dir[2] - pos.z; }
      else { wox = lt.pos_or_dir[0]; woy = lt.pos_or_dir[1]; woz = lt.pos_or_dir[2]; }
      const float d2 = dot3(wox, woy, woz, wox, woy, woz);
      normalize3(wox, woy, woz);
      const float no = dot3(nx, ny, nz, wox, woy, woz);
      glint_debug_rec* rc = DEBUG ? rec + l : nullptr;
      if (DEBUG) {
        uint32_t* w = reinterpret_cast<uint32_t*>(rc);
        for (int q = 0; q < (int)(sizeof(glint_debug_rec) / 4); ++q) w[q] = 0u;
        rc->P = P; rc->r = r; rc->psi = psi;
        for (int i = 0; i < 4; ++i) { rc->ls[i] = sl[i].ls; rc->lr[i] = sl[i].lr; rc->jo[i] = sl[i].jo; rc->w[i] = sl[i].w; rc->n[i] = n[i]; }
        for (int q = 0; q < 12; ++q) { rc->lx[q] = (int32_t)dlx[q]; rc->ly[q] = (int32_t)dly[q]; }
      }
      if (!(ni > 0.0f && no > 0.0f)) continue;   // light below the horizon (R-27)
      if (DEBUG) rc->light_active = 1u;
      float hx_ = wix + wox, hy_ = wiy + woy, hz_ = wiz + woz;
      normalize3(hx_, hy_, hz_);
      const float hx = dot3(hx_, hy_, hz_, tx, ty, tz);
      const float hy = dot3(hx_, hy_, hz_, bx, by, bz);
      const float hz = dot3(hx_, hy_, hz_, nx, ny, nz);
      // Eq. 4: p = R D(h)/D(n), GGX / Beckmann (R-19, R-22)
      float ratio = 0.0f;
      if (hz > 0.0f) {
        const float X = hx / ax, Y = hy / ay;
        const float s2 = X * X + Y * Y;
        const float hz2 = hz * hz;
        if (sc.ndf_kind == 0) {
          const float q = s2 + hz2;
          ratio = 1.0f / (q * q);
        } else {
          const float e2 = s2 / hz2;
          ratio = exp2c(-(e2 * 0x1.715476p+0f)) / (hz2 * hz2);
        }
      }
      float p = R * ratio;
      if (p > 1.0f) { p = 1.0f; flags |= GLINT_FLAG_P_CLAMPED; }
      if (!(p > 0.0f)) p = 0.0f;
      // Eq. 14 angular grid (R-17)
      const float gxa = __fmaf_rn(hx, inv_beta, -0.5f), gya = __fmaf_rn(hy, inv_beta, -0.5f);
      const float cxf = floorf(gxa), cyf = floorf(gya);
      const float fxa = gxa - cxf, fya = gya - cyf;
      const int cx0 = (int)cxf, cy0 = (int)cyf;
      const float vj[4] = {(1.0f - fxa) * (1.0f - fya), fxa * (1.0f - fya), (1.0f - fxa) * fya, fxa * fya};
      uint32_t kax[4];
#pragma unroll
      for (int jn = 0; jn < 4; ++jn) {
        const uint32_t cx = (uint32_t)(cx0 + (jn & 1)), cy = (uint32_t)(cy0 + (jn >> 1));
        const uint32_t ka = lowbias32(cx * 0xcb1ab31fU + cy * 0x165667b1U + 0x27d4eb2fU);
        kax[jn] = ka ^ (ka >> 16);
      }
      if (DEBUG) { rc->p = p; rc->cx0 = cx0; rc->cy0 = cy0; }

      // ---------------- S6 + S7 + S8: 48 gated draws, blended
      const float L2 = (p > 0.0f && p < 1.0f) ? log2_1mp(p) : 0.0f;
      float C = 0.0f;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const Gate gt = gate_params(n[i], p, L2);
        if (DEBUG) { rc->T[i] = gt.T; rc->sigma[i] = gt.sigma; rc->m1[i] = gt.m1; rc->cap[i] = gt.cap; }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          float cik = 0.0f;
#pragma unroll
          for (int jn = 0; jn < 4; ++jn) {
            const uint32_t h = lowbias32_tail(hsx[i * 3 + k] ^ kax[jn]);
            const float c = gated_count(h, gt, sZ);
            cik = __fmaf_rn(vj[jn], c, cik);
            if (DEBUG) { rc->hash[i * 12 + k * 4 + jn] = h; rc->count[i * 12 + k * 4 + jn] = c; }
          }
          C = __fmaf_rn(beta[i * 3 + k], cik, C);
        }
      }
      // ---------------- S8/S9: D_P and radiance (Eq. 1-3)
      const float Dp = C * dp_scale;
      if (DEBUG) { rc->C = C; rc->Dp = Dp; }
      if (C > 0.0f) {
        const float E = (lt.kind == 0) ? 1.0f / d2 : 1.0f;
        const float wolx = dot3(wox, woy, woz, tx, ty, tz), woly = dot3(wox, woy, woz, bx, by, bz);
        const float G2 = 1.0f / (1.0f + lam_i + smith_lambda(sc.ndf_kind, ax2, ay2, wolx, woly, no));
        const float cih = dot3(wix, wiy, wiz, hx_, hy_, hz_);
        const float om = 1.0f - cih;
        const float om2 = om * om;
        const float om5 = om2 * om2 * om;
        const float k = G2 * Dp * E / (4.0f * ni);
        rgb.x += (sc.f0[0] + (1.0f - sc.f0[0]) * om5) * k * lt.intensity[0];
        rgb.y += (sc.f0[1] + (1.0f - sc.f0[1]) * om5) * k * lt.intensity[1];
        rgb.z += (sc.f0[2] + (1.0f - sc.f0[2]) * om5) * k * lt.intensity[2];
      }
    }
    if (DEBUG) for (int l = 0; l < L; ++l) rec[l].flags = flags;
    __stcs(prm.out + (int64_t)y * prm.out_pitch + x, make_float4(rgb.x, rgb.y, rgb.z, __uint_as_float(flags)));
  }
}

template __global__ void glint_eval_kernel<false>(const KParams);
template __global__ void glint_eval_kernel<true>(const KParams);

cudaError_t launch_eval(const KParams& prm, int grid, bool debug, cudaStream_t stream) {
  if (debug)
    glint_eval_kernel<true><<<grid, kBlock, 0, stream>>>(prm);
  else
    glint_eval_kernel<false><<<grid, kBlock, 0, stream>>>(prm);
  return cudaGetLastError();
}

cudaError_t occupancy_blocks_per_sm(int* out) {
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, glint_eval_kernel<false>, kBlock, 0);
}

}  // namespace glint
