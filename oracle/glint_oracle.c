/*
 * glint_oracle.c -- CPU ORACLE for the per-pixel glint BRDF (arXiv 2306.05051).
 *
 * TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs; never by the product path.
 * It shares no code, header, table or constant generator with the CUDA path.
 *
 * The method is a stochastic approximation with discrete choices, so there is
 * no closed-form "answer" to compare with: this file follows the paper's
 * algorithm step by step, in the paper's order and notation (S1..S9 of
 * DESIGN.md §2), taking DESIGN.md §5's reading wherever the paper is silent.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fno-tree-vectorize
 * (no contraction: every fp32 op rounds exactly as DESIGN.md §4 writes it; fmaf
 * appears only where the contract says fma).
 *
 * Citations: P:Lnnn = line of /root/reference/PAPER.md.
 */
#include "glint_oracle.h"

#include <math.h>
#include <string.h>

/* ---------------------------------------------------------------------- */
/* fp32 bit helpers                                                         */
/* ---------------------------------------------------------------------- */
static uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
/* 2^k as an fp32, k in [-126, 127] (exact) */
static float pow2i(int32_t k) { return u2f((uint32_t)(k + 127) << 23); }

/* ---------------------------------------------------------------------- */
/* Tables ("a small texture of random numbers that we precompute")  */
/* ---------------------------------------------------------------------- */
static float g_z[ORC_ZQ];      /* Z[k] = fp32(Phi^-1((k + 1/2) / Q))   (reading R-2) */
static float g_cos[ORC_NANG];  /* fp32(cos(m pi / 256))  (orientation phi_j, Fig. 6) */
static float g_sin[ORC_NANG];
static int g_init = 0;

/* standard normal CDF, fp64: Phi(x) = erfc(-x / sqrt 2) / 2 */
static double phi_cdf(double x) { return 0.5 * erfc(-x / sqrt(2.0)); }

/* Phi^-1 by plain bisection to full double resolution (slow, obviously correct). */
static double phi_inv_bisect(double q) {
  double lo = -40.0, hi = 40.0;
  for (int it = 0; it < 400; ++it) {
    double mid = 0.5 * (lo + hi);
    if (mid == lo || mid == hi) break;
    if (phi_cdf(mid) < q) lo = mid; else hi = mid;
  }
  return 0.5 * (lo + hi);
}

int orc_init(void) {
  if (g_init) return 0;
  for (int k = 0; k < ORC_ZQ; ++k)
    g_z[k] = (float)phi_inv_bisect(((double)k + 0.5) / (double)ORC_ZQ);
  for (int m = 0; m < ORC_NANG; ++m) {
    g_cos[m] = (float)cos((double)m * M_PI / 256.0);
    g_sin[m] = (float)sin((double)m * M_PI / 256.0);
  }
  g_init = 1;
  return 0;
}
const float* orc_ztable(void) { orc_init(); return g_z; }
const float* orc_costable(void) { orc_init(); return g_cos; }
const float* orc_sintable(void) { orc_init(); return g_sin; }

/* ---------------------------------------------------------------------- */
/* Contract transcendentals. IEEE + - * / sqrt, fmaf only.  */
/* ---------------------------------------------------------------------- */

/* 2^y for y <= 0 (used for (1-p)^N = 2^(N log2(1-p)), Eq. 16, and Beckmann
 * exp). k = floor(y + 1/2), f = y - k in [-1/2, 1/2], degree-7 Taylor
 * of e^(f ln2) in Horner form, times 2^k. y < -125 -> 0. */
float orc_exp2(float y) {
  if (!(y >= -125.0f)) return 0.0f;
  /* k = rint(y) by the 1.5 2^23 magic number; 2^k from K's bits */
  float K = y + 12582912.0f;
  float k = K - 12582912.0f;
  float f = y - k;
  float q = 0x1.ffcbfcp-17f;           /* ln2^7/7! */
  q = fmaf(q, f, 0x1.430912p-13f);     /* ln2^6/6! */
  q = fmaf(q, f, 0x1.5d87fep-10f);     /* ln2^5/5! */
  q = fmaf(q, f, 0x1.3b2ab6p-7f);      /* ln2^4/4! */
  q = fmaf(q, f, 0x1.c6b08ep-5f);      /* ln2^3/3! */
  q = fmaf(q, f, 0x1.ebfbe0p-3f);      /* ln2^2/2! */
  q = fmaf(q, f, 0x1.62e430p-1f);      /* ln2 */
  q = fmaf(q, f, 1.0f);
  return q * u2f((f2u(K) - 0x4B3FFF81u) << 23);   /* 2^k: (K bits - 0x4B400000 + 127) << 23 */
}

/* atanh(s)/s = 1 + s^2/3 + s^4/5 + ... + s^14/15 (Horner in z = s^2) */
static float atanh_series(float s) {
  float z = s * s;
  float q = 0x1.111112p-4f;            /* 1/15 */
  q = fmaf(q, z, 0x1.3b13b2p-4f);      /* 1/13 */
  q = fmaf(q, z, 0x1.745d18p-4f);      /* 1/11 */
  q = fmaf(q, z, 0x1.c71c72p-4f);      /* 1/9 */
  q = fmaf(q, z, 0x1.24924ap-3f);      /* 1/7 */
  q = fmaf(q, z, 0x1.99999ap-3f);      /* 1/5 */
  q = fmaf(q, z, 0x1.555556p-2f);      /* 1/3 */
  q = fmaf(q, z, 1.0f);
  return s * q;
}

/* log2(1 - p) for p in (0, 1): log(1-p) = -2 atanh(p / (2 - p)) for p < 1/2;
 * otherwise 1 - p (exact) = 2^e m, m in [2/3, 4/3], log2 = e + 2 atanh((m-1)/(m+1))/ln2. */
float orc_log2_1mp(float p) {
  if (p < 0.5f) {
    float s = p * orc_rcp(2.0f - p);
    return -(atanh_series(s) * 0x1.715476p+1f); /* 2/ln2 */
  }
  float q = 1.0f - p;
  uint32_t b = f2u(q);
  int32_t e = (int32_t)((b >> 23) & 255u) - 127;
  float m = u2f((b & 0x7FFFFFu) | 0x3F800000u); /* [1, 2) */
  if (m > 0x1.555556p+0f) { m = m * 0.5f; e = e + 1; }
  float s = (m - 1.0f) * orc_rcp(m + 1.0f);
  return fmaf(atanh_series(s), 0x1.715476p+1f, (float)e);
}

/* atan2(y, x) in turns, in (-1/2, 1/2]. t = min/max in [0,1]; if t > tan(pi/8)
 * reduce t' = (t-1)/(t+1) (+1/8 turn); odd Taylor series to t^17, coefficients
 * fp32((-1)^k / ((2k+1) 2pi)); octant/quadrant fix-ups are exact in turns. */
float orc_atan2_turns(float y, float x) {
  float ax = fabsf(x), ay = fabsf(y);
  float mx = ax > ay ? ax : ay;
  float mn = ax > ay ? ay : ax;
  if (!(mx >= 0x1p-126f)) return 0.0f;   /* zero or subnormal: no direction */
  float t = mn * orc_rcp(mx);
  float base = 0.0f;
  if (t > 0x1.a8279ap-2f) { t = (t - 1.0f) * orc_rcp(t + 1.0f); base = 0.125f; }
  float z = t * t;
  float q = 0x1.32c69ep-7f;
  q = fmaf(q, z, -0x1.5bade6p-7f);
  q = fmaf(q, z, 0x1.912b1cp-7f);
  q = fmaf(q, z, -0x1.da1bacp-7f);
  q = fmaf(q, z, 0x1.21bb94p-6f);
  q = fmaf(q, z, -0x1.748376p-6f);
  q = fmaf(q, z, 0x1.04c26cp-5f);
  q = fmaf(q, z, -0x1.b2995ep-5f);
  q = fmaf(q, z, 0x1.45f306p-3f);
  float a = fmaf(t, q, base);
  if (ay > ax) a = 0.25f - a;
  if (x < 0.0f) a = 0.5f - a;
  if (y < 0.0f) a = -a;
  return a;
}

/* 1/x for normal x > 0: magic start 0x7ef311c7 - bits, three Newton steps
 * e = 1 - x y, y <- y + y e (fma). Replaces IEEE division. */
float orc_rcp(float x) {
  float y = u2f(0x7ef311c7U - f2u(x));
  float e;
  e = fmaf(-x, y, 1.0f); y = fmaf(y, e, y);
  e = fmaf(-x, y, 1.0f); y = fmaf(y, e, y);
  e = fmaf(-x, y, 1.0f); y = fmaf(y, e, y);
  return y;
}

/* 1/sqrt(x) for normal x > 0: magic-constant start 0x5f3759df - (bits >> 1),
 * then three Newton steps y <- y (3/2 - (x/2) y^2) with the fma written out
 * (DESIGN.md §4.2). Used to normalise directions. */
float orc_rsqrt(float x) {
  float y = u2f(0x5f3759dfU - (f2u(x) >> 1));
  float hx = 0.5f * x;
  y = y * fmaf(-hx, y * y, 1.5f);
  y = y * fmaf(-hx, y * y, 1.5f);
  y = y * fmaf(-hx, y * y, 1.5f);
  return y;
}

/* sqrt(v) = v rsqrt(v) for normal v > 0, 0 otherwise (subnormals included:
 * the Newton steps would overflow to inf * 0) (contract sqrt) */
static float sqrt_c(float v) { return v >= 0x1p-126f ? v * orc_rsqrt(v) : 0.0f; }


/* ---------------------------------------------------------------------- */
/* Hash ("random seeds theta are distributed in a spatial and angular
 * grid"; reading R-23). Published "lowbias32" integer mixer.                */
/* ---------------------------------------------------------------------- */
uint32_t orc_lowbias32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

/* the per-draw hash h = draw_hash(hs + ka) of the spatial seed hs and the
 * angular seed ka (both full lowbias32 outputs): the last four steps of
 * lowbias32 with the middle xor-shift replaced by a three-term xor-rotate
 * x ^ rotr(x, 11) ^ rotr(x, 19) (reading R-23b). The shift leaves chi-square-
 * detectable dependence between the 4 node draws of a texel, whose sums
 * differ by fixed offsets; the rotations feed the top bits of x*C1 back into
 * the low bits. An odd number of rotation terms makes the step invertible
 * (1 + t^11 + t^19 is a unit modulo t^32 - 1 over GF(2)), so draw_hash is a
 * bijection of 32-bit words and theta0 stays exactly uniform. */
uint32_t orc_draw_hash(uint32_t x) {
  x *= 0x7feb352dU;
  x ^= ((x >> 11) | (x << 21)) ^ ((x >> 19) | (x << 13));
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

/* ---------------------------------------------------------------------- */
/* S1  Footprint: "we use screen-space derivatives to obtain the
 * minor/major axis"; phi = orientation of the major axis v0, r = |v0|/|v1|.
 * Reading R-7/R-8: P = |det J|, M = J J^T, lambda+ = major eigenvalue,
 * r = lambda+ / P = sigma_max/sigma_min, psi = phi/pi = atan2(2b, a-c)/(2pi) mod 1.
 * duv = (du/dx, dv/dx, du/dy, dv/dy). Returns 0 if degenerate.              */
/* ---------------------------------------------------------------------- */
int orc_footprint(const float duv[4], float* P, float* r, float* psi) {
  float dudx = duv[0], dvdx = duv[1], dudy = duv[2], dvdy = duv[3];
  float det = dudx * dvdy - dvdx * dudy;
  float a = dudx * dudx + dudy * dudy;
  float b = dudx * dvdx + dudy * dvdy;
  float c = dvdx * dvdx + dvdy * dvdy;
  float hm = 0.5f * (a - c);
  float disc = sqrt_c(hm * hm + b * b);
  float lam = 0.5f * (a + c) + disc;
  *P = fabsf(det);
  *r = lam * orc_rcp(*P);
  float at = orc_atan2_turns(2.0f * b, a - c);
  float ps = at < 0.0f ? at + 1.0f : at;
  if (ps >= 1.0f) ps = 0.0f;
  *psi = ps;
  /* reading R-25: valid footprint area is [2^-64, 2^64); R-30b: and the
   * major eigenvalue below 2^126 (so a, c, 2b, a - c are finite) */
  return (*P >= 0x1p-64f && *P < 0x1p64f && lam < 0x1p126f) ? 1 : 0;
}

/* ---------------------------------------------------------------------- */
/* S2  Lattice location: scale enclosure (Eq. 13, reading R-5),
 * ratio levels and orientation bins that refine per ratio level (P:L635,
 * Fig. 6, readings R-9/R-10), pentagon -> 3 triangles and prism ->
 * 3 tetrahedra (Fig. 7 edges P:L804-807, readings R-11..R-13).
 * Output: 4 grid vertices (ls = log2 texel area, lr = ratio level, jo =
 * orientation index) with distribution weights w (Eq. 10 generalised to 4
 * areas, "distributing over more than 2 areas").                     */
/* ---------------------------------------------------------------------- */
typedef struct { int32_t lr, jo; float w; } tri_vtx;

int orc_lattice(float P, float r, float psi, int32_t K, int32_t ls[4], int32_t lr[4],
                int32_t jo[4], float w[4], uint32_t* flags) {
  /* scale: P = 2^es (1 + ts); bottom level es, top level es + 1 (Eq. 13 with
   * the power-of-two tie resolved as reading R-5): w_top = ts (Eq. 10). */
  uint32_t pb = f2u(P);
  int32_t es = (int32_t)((pb >> 23) & 255u) - 127;
  float ts = u2f((pb & 0x7FFFFFu) | 0x3F800000u) - 1.0f;

  /* ratio: r = 2^er (1 + tr), er in [0, K-1]; r >= 2^K -> (K-1, 1) (R-25) */
  int32_t er;
  float tr;
  if (!(r >= 1.0f)) r = 1.0f;
  if (r >= pow2i(K)) {
    if (r > pow2i(K)) *flags |= ORC_FLAG_RATIO_CLAMPED;
    er = K - 1;
    tr = 1.0f;
  } else {
    uint32_t rb = f2u(r);
    er = (int32_t)((rb >> 23) & 255u) - 127;
    tr = u2f((rb & 0x7FFFFFu) | 0x3F800000u) - 1.0f;
  }

  /* orientation: ring er has 2^er vertices at psi = j / 2^er (R-9) */
  float A = psi * pow2i(er);
  float jf = floorf(A);
  float a = A - jf;
  int32_t j = (int32_t)jf;
  int32_t nI = 1 << er, nO = 2 << er;
  tri_vtx A00 = {er, j, 0.0f}, A01 = {er, (j + 1) & (nI - 1), 0.0f};
  tri_vtx A10 = {er + 1, 2 * j, 0.0f}, A11 = {er + 1, 2 * j + 1, 0.0f};
  tri_vtx A12 = {er + 1, (2 * j + 2) & (nO - 1), 0.0f};

  /* pentagon (tr, a) with A00=(0,0) A01=(0,1) A10=(1,0) A11=(1,1/2) A12=(1,1):
   * T0 = {A00,A10,A11}, T1 = {A00,A11,A01}, T2 = {A01,A11,A12} (reading R-11) */
  tri_vtx v[3];
  float ht = 0.5f * tr;
  if (a <= ht) {
    v[0] = A00; v[1] = A10; v[2] = A11;
    v[0].w = 1.0f - tr;
    v[2].w = a + a;
    v[1].w = tr - v[2].w;
  } else if (a >= 1.0f - ht) {
    float om = 1.0f - a;
    v[0] = A01; v[1] = A11; v[2] = A12;
    v[0].w = 1.0f - tr;
    v[1].w = om + om;
    v[2].w = tr - v[1].w;
  } else {
    v[0] = A00; v[1] = A11; v[2] = A01;
    v[0].w = (1.0f - a) - ht;
    v[1].w = tr;
    v[2].w = a - ht;
  }

  /* merge coincident grid vertices (ring 0: A00 == A01, A10 == A12; R-13) */
  for (int p = 0; p < 3; ++p)
    for (int q = p + 1; q < 3; ++q)
      if (v[p].lr == v[q].lr && v[p].jo == v[q].jo) { v[p].w = v[p].w + v[q].w; v[q].w = 0.0f; }

  /* global vertex order by key (lr, jo), stable (R-12) */
#define KEY(t) (((t).lr << 9) | (t).jo)
#define CSWAP(p, q) if (KEY(v[p]) > KEY(v[q])) { tri_vtx tmp_ = v[p]; v[p] = v[q]; v[q] = tmp_; }
  CSWAP(0, 1);
  CSWAP(1, 2);
  CSWAP(0, 1);
#undef CSWAP
#undef KEY

  /* prism (triangle x [es, es+1]) -> 3 tetrahedra, staircase fill of the top
   * level in global order (R-12); t = ts */
  float al = v[0].w, be = v[1].w, ga = v[2].w;
  float t = ts;
  float ab = al + be;
  if (t <= al) {
    ls[0] = es;     lr[0] = v[0].lr; jo[0] = v[0].jo; w[0] = al - t;
    ls[1] = es;     lr[1] = v[1].lr; jo[1] = v[1].jo; w[1] = be;
    ls[2] = es;     lr[2] = v[2].lr; jo[2] = v[2].jo; w[2] = ga;
    ls[3] = es + 1; lr[3] = v[0].lr; jo[3] = v[0].jo; w[3] = t;
  } else if (t <= ab) {
    ls[0] = es;     lr[0] = v[1].lr; jo[0] = v[1].jo; w[0] = ab - t;
    ls[1] = es;     lr[1] = v[2].lr; jo[1] = v[2].jo; w[1] = ga;
    ls[2] = es + 1; lr[2] = v[0].lr; jo[2] = v[0].jo; w[2] = al;
    ls[3] = es + 1; lr[3] = v[1].lr; jo[3] = v[1].jo; w[3] = t - al;
  } else {
    ls[0] = es;     lr[0] = v[2].lr; jo[0] = v[2].jo; w[0] = 1.0f - t;
    ls[1] = es + 1; lr[1] = v[0].lr; jo[1] = v[0].jo; w[1] = al;
    ls[2] = es + 1; lr[2] = v[1].lr; jo[2] = v[1].jo; w[2] = be;
    ls[3] = es + 1; lr[3] = v[2].lr; jo[3] = v[2].jo; w[3] = (t - al) - be;
  }
  (void)ga;
  return 0;
}

/* The naive 10-grid distribution the paper starts from before its tetrahedral
 * split ("2 x 5 anisotropic grids with linear blending"; "trilinear
 * weights"), reading R-29: linear in ts between the two LODs, linear
 * in tr between the two ratio rings, linear in a between the inner ring's two
 * orientations and piecewise linear (hats at a = 0, 1/2, 1) over the outer
 * ring's three. Slots: LOD es then es+1, each A00 A01 A10 A11 A12; coincident
 * ring-0 vertices merged as in R-13. Used only by the 160-draw ablation. */
int orc_lattice10(float P, float r, float psi, int32_t K, int32_t ls[10], int32_t lr[10],
                  int32_t jo[10], float w[10], uint32_t* flags) {
  uint32_t pb = f2u(P);
  int32_t es = (int32_t)((pb >> 23) & 255u) - 127;
  float ts = u2f((pb & 0x7FFFFFu) | 0x3F800000u) - 1.0f;
  int32_t er;
  float tr;
  if (!(r >= 1.0f)) r = 1.0f;
  if (r >= pow2i(K)) {
    if (r > pow2i(K)) *flags |= ORC_FLAG_RATIO_CLAMPED;
    er = K - 1;
    tr = 1.0f;
  } else {
    uint32_t rb = f2u(r);
    er = (int32_t)((rb >> 23) & 255u) - 127;
    tr = u2f((rb & 0x7FFFFFu) | 0x3F800000u) - 1.0f;
  }
  float A = psi * pow2i(er);
  float jf = floorf(A);
  float a = A - jf;
  int32_t j = (int32_t)jf;
  int32_t nI = 1 << er, nO = 2 << er;
  int32_t vlr[5] = {er, er, er + 1, er + 1, er + 1};
  int32_t vjo[5] = {j, (j + 1) & (nI - 1), 2 * j, 2 * j + 1, (2 * j + 2) & (nO - 1)};
  float a2 = a + a;
  float omt = 1.0f - tr;
  float pw[5];
  pw[0] = omt * (1.0f - a);
  pw[1] = omt * a;
  pw[2] = tr * (a2 <= 1.0f ? 1.0f - a2 : 0.0f);
  pw[3] = tr * (a2 <= 1.0f ? a2 : 2.0f - a2);
  pw[4] = tr * (a2 <= 1.0f ? 0.0f : a2 - 1.0f);
  for (int p = 0; p < 5; ++p)
    for (int q = p + 1; q < 5; ++q)
      if (vlr[p] == vlr[q] && vjo[p] == vjo[q]) { pw[p] = pw[p] + pw[q]; pw[q] = 0.0f; }
  for (int lv = 0; lv < 2; ++lv) {
    float sw = lv ? ts : 1.0f - ts;
    for (int p = 0; p < 5; ++p) {
      ls[lv * 5 + p] = es + lv;
      lr[lv * 5 + p] = vlr[p];
      jo[lv * 5 + p] = vjo[p];
      w[lv * 5 + p] = sw * pw[p];
    }
  }
  return 0;
}

/* ---------------------------------------------------------------------- */
/* S3  Anisotropic grid transform (Eq. 12, reading R-14):
 * rotate by phi_j = m pi / 256 (m = jo 2^(8-lr)), then area-preserving stretch:
 * x = (c u + s v) 2^(-(ls+lr)/2), y = (c v - s u) 2^((lr-ls)/2).             */
/* ---------------------------------------------------------------------- */
static float pow2half(int32_t e) { /* 2^(e/2): odd e -> fp32(sqrt 2) * 2^floor(e/2) */
  int32_t h = e >> 1;  /* arithmetic shift = floor */
  float s = pow2i(h);
  return (e & 1) ? s * 0x1.6a09e6p+0f : s;
}

void orc_grid_uv(float u, float v, int32_t ls, int32_t lr, int32_t jo, float* x, float* y) {
  orc_init();
  int32_t m = jo << (8 - lr);
  float c = g_cos[m], s = g_sin[m];
  float xr = fmaf(c, u, s * v);
  float yr = fmaf(c, v, -(s * u));
  *x = xr * pow2half(-(ls + lr));
  *y = yr * pow2half(lr - ls);
}

/* S3  Simplex surface grid (Fig. 8 shear P:L882, reading R-15):
 * lattice coordinates (x + y/2, y); triangle {(0,0),(1,0),(1,1)} if fx >= fy
 * else {(0,0),(0,1),(1,1)}; barycentric weights. */
void orc_simplex(float x, float y, int64_t lx[3], int64_t ly[3], float beta[3]) {
  float xs = x + 0.5f * y;
  float fxs = floorf(xs), fys = floorf(y);
  float fx = xs - fxs, fy = y - fys;
  int64_t ix = (int64_t)fxs, iy = (int64_t)fys;
  if (fx >= fy) {
    lx[0] = ix;     ly[0] = iy;     beta[0] = 1.0f - fx;
    lx[1] = ix + 1; ly[1] = iy;     beta[1] = fx - fy;
    lx[2] = ix + 1; ly[2] = iy + 1; beta[2] = fy;
  } else {
    lx[0] = ix;     ly[0] = iy;     beta[0] = 1.0f - fy;
    lx[1] = ix;     ly[1] = iy + 1; beta[1] = fy - fx;
    lx[2] = ix + 1; ly[2] = iy + 1; beta[2] = fx;
  }
}

/* Square spatial grid with bilinear weights (the 4-texel spatial blending the
 * simplex grid replaces); used by the 64- and 160-draw ablations. */
void orc_bilinear(float x, float y, int64_t lx[4], int64_t ly[4], float beta[4]) {
  float fxs = floorf(x), fys = floorf(y);
  float fx = x - fxs, fy = y - fys;
  int64_t ix = (int64_t)fxs, iy = (int64_t)fys;
  lx[0] = ix;     ly[0] = iy;     beta[0] = (1.0f - fx) * (1.0f - fy);
  lx[1] = ix + 1; ly[1] = iy;     beta[1] = fx * (1.0f - fy);
  lx[2] = ix;     ly[2] = iy + 1; beta[2] = (1.0f - fx) * fy;
  lx[3] = ix + 1; ly[3] = iy + 1; beta[3] = fx * fy;
}

/* ---------------------------------------------------------------------- */
/* S6  Gated Gaussian binomial (Eq. 16-18, readings R-1..R-4):
 * P>=1 = 1 - (1-p)^n; mu = (n-1)p, sigma = sqrt((n-1)p(1-p)); gate succeeds
 * iff theta0 < P>=1 with theta0 = (y >> 9) 2^-23, i.e. (y >> 9) < T, where
 * y = h ^ (h >> 16) is the hash before its final xor-shift (the same top 16
 * bits as h) and T = ceil(P>=1 2^23); z = Z[(h >> 2) & 4095] (bits 2..13);
 * count = floor(clamp(1 + mu + sigma z, 1, ceil(n))) (reading R-3).         */
/* ---------------------------------------------------------------------- */
/* P>=1 = 1 - (1-p)^n (Eq. 16) for n > 0, p > 0; 0 otherwise (no trials) */
static float pge1_of(float n, float p) {
  if (!(n > 0.0f) || !(p > 0.0f)) return 0.0f;
  if (p >= 1.0f) return 1.0f;
  float y = n * orc_log2_1mp(p);        /* log2((1-p)^n) */
  return 1.0f - orc_exp2(y);            /* Eq. 16 */
}

void orc_gate_params(float n, float p, uint32_t* T, float* sigma, float* m1, float* cap) {
  if (!(n > 0.0f) || !(p > 0.0f)) { *T = 0; *sigma = 0.0f; *m1 = 1.0f; *cap = 1.0f; return; }
  float Pge1 = pge1_of(n, p);
  *T = (uint32_t)ceilf(Pge1 * 0x1p23f);
  float nm1 = n - 1.0f;
  float mu = nm1 > 0.0f ? nm1 * p : 0.0f; /* Eq. 17 (R-4: n < 1 -> mu = 0) */
  float var = mu * (1.0f - p);
  *sigma = sqrt_c(var); /* contract sqrt */
  *m1 = 1.0f + mu;
  *cap = ceilf(n);
}

float orc_gated_count(uint32_t h, uint32_t T, float sigma, float m1, float cap) {
  orc_init();
  uint32_t y = h ^ (h >> 16);                     /* undo the final xor-shift */
  if (!((y >> 9) < T)) return 0.0f;               /* H(P>=1 - theta0) gate, R-1 */
  float z = g_z[(h >> 2) & (ORC_ZQ - 1)];         /* N(theta1) via quantile table, R-2 */
  float x = fmaf(sigma, z, m1);                   /* 1 + N(theta1; mu, sigma) */
  x = x < 1.0f ? 1.0f : x;                        /* R-3 clamp */
  x = x > cap ? cap : x;
  return floorf(x);                               /* Eq. 18 floor, R-26 */
}

/* exact test sampler (sampler = 1): Bin(floor n, p) + Bernoulli(frac(n) p),
 * trials driven by the same per-draw hash; mean is exactly n p. fp64. */
static float exact_count(uint32_t h, float n, float p) {
  if (!(n > 0.0f) || !(p > 0.0f)) return 0.0f;
  double dn = (double)n, dp = (double)p;
  int64_t nf = (int64_t)floor(dn);
  int32_t c = 0;
  for (int64_t t = 0; t < nf; ++t) {
    uint32_t u = orc_lowbias32(h ^ orc_lowbias32((uint32_t)t * 0x9e3779b9U + 0x632be5abU));
    if ((double)u * 0x1p-32 < dp) ++c;
  }
  uint32_t u = orc_lowbias32(h ^ 0xa5a5a5a5U);
  if ((double)u * 0x1p-32 < (dn - (double)nf) * dp) ++c;
  return (float)c;
}

/* ---------------------------------------------------------------------- */
/* S5  NDF ratio D(h)/D(n) (Eq. 4; targets P:L148, L1211; anisotropic
 * alpha reading R-22). GGX: 1/q^2, q = X^2+Y^2+hz^2; Beckmann:
 * exp(-(X^2+Y^2)/hz^2)/hz^4; X = hx/ax, Y = hy/ay.                           */
/* ---------------------------------------------------------------------- */
float orc_ratio(int32_t ndf_kind, float ax, float ay, float hx, float hy, float hz) {
  if (!(hz > 0.0f)) return 0.0f;
  float X = hx * orc_rcp(ax), Y = hy * orc_rcp(ay);
  float s2 = X * X + Y * Y;
  float hz2 = hz * hz;
  if (ndf_kind == 0) {
    float q = s2 + hz2;
    return orc_rcp(q * q);
  }
  float e2 = s2 * orc_rcp(hz2);
  return orc_exp2(-(e2 * 0x1.715476p+0f)) * orc_rcp(hz2 * hz2);
}

/* fp32 contract vector helpers */
float orc_rcp(float x);
static float dot3f(const float a[3], const float b[3]) {
  return fmaf(a[2], b[2], fmaf(a[1], b[1], a[0] * b[0]));
}
static void normalize3f(float v[3]) {
  float inv = orc_rsqrt(dot3f(v, v));
  v[0] = v[0] * inv; v[1] = v[1] * inv; v[2] = v[2] * inv;
}
/* Duff et al. 2017 branchless ONB from n (reading R-17) */
static void onb_f(const float n[3], float t[3], float bt[3]) {
  float sgn = copysignf(1.0f, n[2]);
  float a = -(sgn * orc_rcp(1.0f + fabsf(n[2])));   /* = -1/(sgn + nz) */
  float b = (n[0] * n[1]) * a;
  float nxxa = (n[0] * n[0]) * a;
  float nyya = (n[1] * n[1]) * a;
  t[0] = 1.0f + sgn * nxxa; t[1] = sgn * b; t[2] = -(sgn * n[0]);
  bt[0] = b; bt[1] = sgn + nyya; bt[2] = -n[1];
}

/* fp64 radiance helpers (tolerance path; Eq. 1-2, reading R-21) */
static double dot3d(const double a[3], const double b[3]) { return a[0]*b[0] + a[1]*b[1] + a[2]*b[2]; }
static void normalize3d(double v[3]) { double l = sqrt(dot3d(v, v)); v[0] /= l; v[1] /= l; v[2] /= l; }
static void onb_d(const double n[3], double t[3], double bt[3]) {
  double sgn = copysign(1.0, n[2]);   /* as onb_f (DESIGN §4.3 S5): -0 gives -1 */
  double a = -1.0 / (sgn + n[2]);
  double b = n[0] * n[1] * a;
  t[0] = 1.0 + sgn * n[0] * n[0] * a; t[1] = sgn * b; t[2] = -sgn * n[0];
  bt[0] = b; bt[1] = sgn + n[1] * n[1] * a; bt[2] = -n[1];
}
/* Smith Lambda (height-correlated G2 = 1/(1 + L(wi) + L(wo))) */
static double smith_lambda(int kind, double ax, double ay, const double wl[3]) {
  double s = ax * ax * wl[0] * wl[0] + ay * ay * wl[1] * wl[1];
  if (s <= 0.0) return 0.0;
  if (kind == 0) { /* GGX, exact: (-1 + sqrt(1 + s/wz^2))/2, stable form */
    double q = s / (wl[2] * wl[2]);
    return q / (2.0 * (1.0 + sqrt(1.0 + q)));
  }
  double a = wl[2] / sqrt(s); /* Beckmann, Walter et al. 2007 rational fit */
  if (a >= 1.6) return 0.0;
  return (1.0 - 1.259 * a + 0.396 * a * a) / (3.535 * a + 2.181 * a * a);
}

/* radiance-path terms exported for pin tests (fp64; reading R-21):
 * G2 = 1/(1 + Lambda(wi) + Lambda(wo)) in the local (t, b, n) frame, and
 * Schlick F = f0 + (1 - f0)(1 - cos)^5. */
double orc_smith_g2(int32_t kind, double ax, double ay, const double wi_l[3], const double wo_l[3]) {
  return 1.0 / (1.0 + smith_lambda(kind, ax, ay, wi_l) + smith_lambda(kind, ax, ay, wo_l));
}
double orc_schlick(double f0, double cos_t) {
  double om = 1.0 - cos_t;
  return f0 + (1.0 - f0) * om * om * om * om * om;
}

/* ---------------------------------------------------------------------- */
/* Zirr & Kaplanyan-style baseline (eval_mode 3), from the
 * paper's description of that method only (their code is not available):
 *  - anisotropic footprints are filtered by probing: "the counting law needs
 *    to be manually evaluated for each texel under the pixel footprint"
 *    (P:L188), with the anisotropy capped at x16 beyond which the footprint
 *    grows isotropically;
 *  - LOD levels whose cells quadruple in area, two at a time, blended
 *    by OUTPUT: b = mix(b(N P_top, p), b(N P_bottom, p), w) (Eq. 7);
 *  - random seeds on a spatial and an angular grid, evaluations bilinearly
 *    interpolated;
 *  - the classical binomial: floor(N(theta0; mu, sigma^2)) if N p > 5, else the
 *    sum of N Bernoulli trials H(theta_k - p), looped up to N = 16 (Eq. 15,
 *    P:L975-983).
 * The readings that make this concrete are DESIGN.md R-31..R-36. */
/* ---------------------------------------------------------------------- */

/* R-31/R-32: probes along the footprint's major axis. From M = J J^T (S1's
 * a, b, c, lambda): n = min(ceil(r), 16) probes, each of area P / n, centred
 * at uv + ((2k + 1 - n) (1/2) / n) sigma_max e, e = unit major-axis direction
 * (the eigenvector of M for lambda, from its better-conditioned row), and
 * sigma_max = sqrt(lambda). Returns n; flags RATIO_CLAMPED if ceil(r) > 16. */
int orc_zk_probes(const float duv[4], float u, float v, float uk[16], float vk[16], float* area,
                  uint32_t* flags) {
  float dudx = duv[0], dvdx = duv[1], dudy = duv[2], dvdy = duv[3];
  float det = dudx * dvdy - dvdx * dudy;
  float a = dudx * dudx + dudy * dudy;
  float b = dudx * dvdx + dudy * dvdy;
  float c = dvdx * dvdx + dvdy * dvdy;
  float hm = 0.5f * (a - c);
  float disc = sqrt_c(hm * hm + b * b);
  float lam = 0.5f * (a + c) + disc;
  float P = fabsf(det);
  float r = lam * orc_rcp(P);
  float ex = a >= c ? lam - c : b;
  float ey = a >= c ? b : lam - a;
  float l2 = ex * ex + ey * ey;
  if (l2 >= 0x1p-126f) { float il = orc_rsqrt(l2); ex = ex * il; ey = ey * il; }
  else { ex = 1.0f; ey = 0.0f; }
  float cr = ceilf(r);
  if (cr > 16.0f) *flags |= ORC_FLAG_RATIO_CLAMPED;
  int n = cr >= 16.0f ? 16 : (cr >= 1.0f ? (int)cr : 1);
  float rn = orc_rcp((float)n);
  *area = P * rn;
  float smax = sqrt_c(lam);
  float q = 0.5f * rn;
  for (int k = 0; k < n; ++k) {
    float off = ((float)(2 * k + 1 - n) * q) * smax;
    uk[k] = fmaf(off, ex, u);
    vk[k] = fmaf(off, ey, v);
  }
  return n;
}

/* R-33: LOD pair of a probe of area A. Level l has cells of side 2^l (area
 * 4^l); A = 4^kz (1 + t), t in [0, 3) from A's exponent bits (kz = floor(e/2));
 * the output mix puts weight wt = t/3 on level kz + 1 and 1 - wt on kz, so
 * that (1 - wt) 4^kz + wt 4^(kz+1) = A (Eq. 7 with E[b] = N A p). */
void orc_zk_lod(float A, int32_t* kz, float* t) {
  int32_t e = (int32_t)((f2u(A) >> 23) & 255u) - 127;
  int32_t k = e >> 1;                   /* floor(e / 2) */
  *kz = k;
  *t = A * pow2i(-2 * k) - 1.0f;       /* exact: power-of-2 scaling, result in [0, 3) */
}

/* R-34: the classical binomial of Eq. 15 for one (texel, angular node) with
 * nt = N 4^l trials and draw word w: Gaussian floor(mu + sigma z) clamped to
 * [0, ceil(nt)] (z = Z[(w >> 2) & 4095], mu = nt p, sigma = sqrt(nt p (1-p)))
 * when nt p > 5 or nt > 16; otherwise floor(nt) Bernoulli trials
 * theta_k = lowbias32(w + k 0x9e3779b9) >> 8 < ceil(p 2^24) plus one
 * fractional trial (k = 16) with probability frac(nt) p (R-35), so that
 * E = nt p exactly in the looped regime. */
float orc_zk_count(uint32_t w, float nt, float p) {
  orc_init();
  float np = nt * p;
  if (np > 5.0f || nt > 16.0f) {
    float sg = sqrt_c(np * (1.0f - p));
    float z = g_z[(w >> 2) & (ORC_ZQ - 1)];
    float x = fmaf(sg, z, np);
    float cap = ceilf(nt);
    x = x < 0.0f ? 0.0f : x;
    x = x > cap ? cap : x;
    return floorf(x);
  }
  float nf = floorf(nt);
  uint32_t Tp = (uint32_t)ceilf(p * 0x1p24f);
  uint32_t Tf = (uint32_t)ceilf(((nt - nf) * p) * 0x1p24f);
  int c = 0;
  for (int k = 0; k < (int)nf; ++k)
    if ((orc_lowbias32(w + (uint32_t)k * 0x9e3779b9U) >> 8) < Tp) ++c;
  if ((orc_lowbias32(w + 16u * 0x9e3779b9U) >> 8) < Tf) ++c;
  return (float)c;
}

/* R-36: texel seed of the ZK random texture (its own key domain): level l,
 * texel (lx, ly) of the side-2^l grid, object/seed word so. */
static uint32_t zk_texel_seed(uint32_t so, int32_t l, int64_t lx, int64_t ly) {
  return orc_lowbias32(so + (uint32_t)l * 0x5bd1e995U + (uint32_t)lx * 0x8da6b343U +
                       (uint32_t)ly * 0xd8163841U + 0x68e31da4U);
}

/* blended count C of one pixel-light (fp64 weights, exact integer counts) */
static double zk_blend(int npr, const float uk[16], const float vk[16], float A, uint32_t so,
                       float N, float p, const uint32_t ka[4], const double vj[4]) {
  int32_t kz; float t;
  orc_zk_lod(A, &kz, &t);
  double wt = (double)t / 3.0;
  double C = 0.0;
  for (int k = 0; k < npr; ++k) {
    for (int lev = 0; lev < 2; ++lev) {
      int32_t l = kz + lev;
      double wl = lev ? wt : 1.0 - wt;
      float nt = N * pow2i(2 * l);
      if (!(nt <= 0x1p64f)) nt = 0x1p64f;
      float s = pow2i(-l);
      float gx = fmaf(uk[k], s, -0.5f), gy = fmaf(vk[k], s, -0.5f);
      float fxs = floorf(gx), fys = floorf(gy);
      double fx = (double)(gx - fxs), fy = (double)(gy - fys);
      int64_t ix = (int64_t)fxs, iy = (int64_t)fys;
      double bq[4] = {(1.0 - fx) * (1.0 - fy), fx * (1.0 - fy), (1.0 - fx) * fy, fx * fy};
      for (int q = 0; q < 4; ++q) {
        uint32_t hz = zk_texel_seed(so, l, ix + (q & 1), iy + (q >> 1));
        double Cq = 0.0;
        for (int jn = 0; jn < 4; ++jn)
          Cq += vj[jn] * (double)orc_zk_count(orc_lowbias32(hz + ka[jn]), nt, p);
        C += wl * bq[q] * Cq;
      }
    }
  }
  return C;
}

/* ---------------------------------------------------------------------- */
/* S9  Radiance shell of one light (Eq. 1-2: L = F G D_P E / (4
 * n.wi) for a punctual light; readings R-21, R-27). Everything in
 * fp64 from the raw fp32 inputs (normal, position, view, light): no fp32
 * rounding of a cosine reaches the radiance. Called for a light the fp32
 * decision path found active; adds nothing when D_P = 0 (no flake reflects)
 * or when an fp64 cosine n.wi, n.wo is not > 0 (the exact geometry is at or
 * below the horizon although the fp32 decision said otherwise). Adds the
 * light's RGB contribution to rgb; returns 1 if it added anything.         */
/* ---------------------------------------------------------------------- */
int orc_shell(const orc_scene* sc, int32_t l, const float nrm[3], const float pos[3], float ax, float ay,
              double Dp, double rgb[3]) {
  if (!(Dp > 0.0)) return 0;
  const orc_light* lt = &sc->lights[l];
  double nd[3] = {nrm[0], nrm[1], nrm[2]};
  normalize3d(nd);
  double td[3], bd[3];
  onb_d(nd, td, bd);
  double wid[3];  /* towards the viewer: pinhole camera (R-27) or direction */
  if (sc->view_kind == 0) { wid[0] = (double)sc->view[0] - pos[0]; wid[1] = (double)sc->view[1] - pos[1]; wid[2] = (double)sc->view[2] - pos[2]; }
  else { wid[0] = sc->view[0]; wid[1] = sc->view[1]; wid[2] = sc->view[2]; }
  normalize3d(wid);
  double wod[3], E[3];  /* towards the light; irradiance E = I / d^2 (point) or I */
  if (lt->kind == 0) {
    wod[0] = (double)lt->pos_or_dir[0] - pos[0]; wod[1] = (double)lt->pos_or_dir[1] - pos[1]; wod[2] = (double)lt->pos_or_dir[2] - pos[2];
    double d2 = dot3d(wod, wod);
    for (int ch = 0; ch < 3; ++ch) E[ch] = (double)lt->intensity[ch] / d2;
  } else {
    wod[0] = lt->pos_or_dir[0]; wod[1] = lt->pos_or_dir[1]; wod[2] = lt->pos_or_dir[2];
    for (int ch = 0; ch < 3; ++ch) E[ch] = (double)lt->intensity[ch];
  }
  normalize3d(wod);
  double nid = dot3d(nd, wid), nod = dot3d(nd, wod);
  if (!(nid > 0.0) || !(nod > 0.0)) return 0;
  double hd[3] = {wid[0] + wod[0], wid[1] + wod[1], wid[2] + wod[2]};
  normalize3d(hd);
  double cih = dot3d(wid, hd);
  double wil[3] = {dot3d(wid, td), dot3d(wid, bd), nid};
  double wol[3] = {dot3d(wod, td), dot3d(wod, bd), nod};
  double G2 = orc_smith_g2(sc->ndf_kind, ax, ay, wil, wol);
  for (int ch = 0; ch < 3; ++ch) {
    double F = orc_schlick((double)sc->f0[ch], cih);
    rgb[ch] += F * G2 * Dp * E[ch] / (4.0 * nid);
  }
  return 1;
}

/* ---------------------------------------------------------------------- */
/* S0..S9 for one pixel                                                     */
/* ---------------------------------------------------------------------- */
static void eval_pixel(const float duv[4], const float uvm[4], const float nrm[4],
                       const float pos[4], const float mat[4], const orc_scene* sc,
                       double rgb[3], uint32_t* flags_out, orc_rec* rec) {
  int L = sc->n_lights;
  uint32_t flags = 0;
  rgb[0] = rgb[1] = rgb[2] = 0.0;
  if (rec) memset(rec, 0, sizeof(orc_rec) * (size_t)L);

  uint32_t meta = f2u(uvm[3]);
  float u = uvm[0], v = uvm[1];
  if (!(meta & 1u)) { *flags_out = ORC_FLAG_INVALID; goto fill_flags; }
  if (!(fabsf(u) <= 0x1p24f && fabsf(v) <= 0x1p24f)) {
    *flags_out = ORC_FLAG_INVALID | ORC_FLAG_UV_RANGE; goto fill_flags;
  }

  /* S1 footprint */
  float P, r, psi;
  if (!orc_footprint(duv, &P, &r, &psi)) { *flags_out = ORC_FLAG_DEGENERATE; goto fill_flags; }

  /* S2 lattice: 4 grids (tetrahedron of the prism) + distribution
   * weights; n_i = w_i N 2^ls_i (R-14: "N_i proportional to its area",
   * P:L633). Ablation mode 2 (160 draws) uses all 10 prism vertices (R-29). */
  const int mode = sc->eval_mode;
  const int NG = mode == 3 ? 0 : (mode == 2 ? 10 : 4);   /* grids (mode 3: ZK probes instead) */
  const int NS = mode == 0 ? 3 : 4;           /* spatial texels per grid */
  int32_t ls[10], lr[10], jo[10];
  float w[10], n[10];
  float zuk[16], zvk[16], zA = 0.0f;
  int znp = 0;
  if (mode == 3) {
    znp = orc_zk_probes(duv, u, v, zuk, zvk, &zA, &flags);
    for (int i = 0; i < 4; ++i) { ls[i] = lr[i] = jo[i] = 0; w[i] = 0.0f; }
  } else if (mode == 2) orc_lattice10(P, r, psi, sc->max_ratio_level, ls, lr, jo, w, &flags);
  else orc_lattice(P, r, psi, sc->max_ratio_level, ls, lr, jo, w, &flags);
  /* reading R-37: the material domain -- roughness in [2^-16, 16], flake
   * density in [0, 2^40], ratio R in [0, 16]; NaN (and -0) go to the lower
   * bound -- so N 2^ls < 2^104 and pi ax ay R N P < 2^116: no fp32 overflow */
  float ax = mat[0] >= 0x1p-16f ? mat[0] : 0x1p-16f;
  ax = ax <= 16.0f ? ax : 16.0f;
  float ay = mat[1] >= 0x1p-16f ? mat[1] : 0x1p-16f;
  ay = ay <= 16.0f ? ay : 16.0f;
  float N = mat[2] > 0.0f ? mat[2] : 0.0f;
  N = N > 0x1p40f ? 0x1p40f : N;
  float R = mat[3] > 0.0f ? mat[3] : 0.0f;
  R = R <= 16.0f ? R : 16.0f;
  for (int i = 0; i < NG; ++i) n[i] = w[i] * (N * pow2i(ls[i]));

  /* S3 + S4a: per grid, 3 simplex lattice vertices -- or, in the
   * 64/160 ablations, 4 square-lattice texels with bilinear weights -- and
   * their spatial seeds */
  uint32_t obj = f2u(uvm[2]);
  uint32_t so = orc_lowbias32(obj ^ orc_lowbias32(sc->seed));
  uint32_t hs[10][4];
  int64_t lxs[10][4], lys[10][4];
  double betad[10][4];
  float sfx[4] = {0, 0, 0, 0}, sfy[4] = {0, 0, 0, 0};   /* simplex fractions (records) */
  for (int i = 0; i < NG; ++i) {
    float x, y, be[4];
    orc_grid_uv(u, v, ls[i], lr[i], jo[i], &x, &y);
    if (mode == 0) {
      orc_simplex(x, y, lxs[i], lys[i], be);
      /* barycentrics recomputed in fp64 from the exact fp32 fractions */
      float xs = x + 0.5f * y;
      double fx = (double)(xs - floorf(xs)), fy = (double)(y - floorf(y));
      sfx[i] = (float)fx; sfy[i] = (float)fy;
      if (fx >= fy) { betad[i][0] = 1.0 - fx; betad[i][1] = fx - fy; betad[i][2] = fy; }
      else          { betad[i][0] = 1.0 - fy; betad[i][1] = fy - fx; betad[i][2] = fx; }
    } else {
      orc_bilinear(x, y, lxs[i], lys[i], be);
      double fx = (double)(x - floorf(x)), fy = (double)(y - floorf(y));
      betad[i][0] = (1.0 - fx) * (1.0 - fy); betad[i][1] = fx * (1.0 - fy);
      betad[i][2] = (1.0 - fx) * fy;         betad[i][3] = fx * fy;
    }
    /* spatial seed of texel (grid key, lattice vertex): one hash of the
     * object/seed word plus a linear code of (key, lx, ly) (reading R-23) */
    uint32_t gk = ((uint32_t)ls[i] & 511u) | ((uint32_t)lr[i] << 9) | ((uint32_t)jo[i] << 13);
    for (int k = 0; k < NS; ++k) {
      uint32_t lin = gk * 0x9e3779b1U + (uint32_t)lxs[i][k] * 0x8da6b343U + (uint32_t)lys[i][k] * 0xd8163841U;
      hs[i][k] = orc_lowbias32(so + lin);
    }
  }

  /* shading frame (fp32 contract; decides light activity, p, angular nodes) */
  float nf[3] = {nrm[0], nrm[1], nrm[2]};
  normalize3f(nf);
  float tf[3], bf[3];
  onb_f(nf, tf, bf);
  float wi[3];
  if (sc->view_kind == 0) { wi[0] = sc->view[0] - pos[0]; wi[1] = sc->view[1] - pos[1]; wi[2] = sc->view[2] - pos[2]; }
  else { wi[0] = sc->view[0]; wi[1] = sc->view[1]; wi[2] = sc->view[2]; }
  normalize3f(wi);
  float ni = dot3f(nf, wi);
  float inv_beta = 1.0f / sc->beta;

  for (int l = 0; l < L; ++l) {
    const orc_light* lt = &sc->lights[l];
    orc_rec* rc = rec ? &rec[l] : 0;
    if (rc) {
      rc->P = P; rc->r = r; rc->psi = psi;
      for (int i = 0; i < 4; ++i) { rc->ls[i] = ls[i]; rc->lr[i] = lr[i]; rc->jo[i] = jo[i]; rc->w[i] = w[i]; rc->n[i] = n[i]; }
      for (int i = 0; i < 4; ++i) for (int k = 0; k < 3; ++k) { rc->lx[i*3+k] = (int32_t)(uint32_t)lxs[i][k]; rc->ly[i*3+k] = (int32_t)(uint32_t)lys[i][k]; }
      for (int i = 0; i < 4; ++i) { rc->sfx[i] = sfx[i]; rc->sfy[i] = sfy[i]; }
    }
    /* S5: light direction d toward the light (P:L1228 punctual lights only,
     * reading R-27); w_o = d/|d|. The light is active iff n.w_i > 0 and
     * n.d > 0; h = normalize(|d| w_i + d), proportional to w_i + w_o. */
    float d[3];
    if (lt->kind == 0) { d[0] = lt->pos_or_dir[0] - pos[0]; d[1] = lt->pos_or_dir[1] - pos[1]; d[2] = lt->pos_or_dir[2] - pos[2]; }
    else { d[0] = lt->pos_or_dir[0]; d[1] = lt->pos_or_dir[1]; d[2] = lt->pos_or_dir[2]; }
    float d2 = dot3f(d, d);
    float n_d = dot3f(nf, d);
    /* light below the horizon: 0; R-27b: |d|^2 must be a normal float (else
     * the contract sqrt cannot form |d| and h) */
    if (!(ni > 0.0f && n_d > 0.0f && d2 >= 0x1p-126f && d2 <= 0x1p120f)) continue;
    if (rc) rc->light_active = 1;
    float dl = d2 * orc_rsqrt(d2);
    float hv[3] = {fmaf(dl, wi[0], d[0]), fmaf(dl, wi[1], d[1]), fmaf(dl, wi[2], d[2])};
    normalize3f(hv);
    float hx = dot3f(hv, tf), hy = dot3f(hv, bf), hz = dot3f(hv, nf);
    /* Eq. 4: p = R D(h)/D(n), clamped to 1 (reading R-19) */
    float p = R * orc_ratio(sc->ndf_kind, ax, ay, hx, hy, hz);
    if (p > 1.0f) { p = 1.0f; flags |= ORC_FLAG_P_CLAMPED; }
    if (!(p > 0.0f)) p = 0.0f;
    /* Eq. 14 angular grid: orthographic projection of h, cell size beta (R-17) */
    float gx = fmaf(hx, inv_beta, -0.5f), gy = fmaf(hy, inv_beta, -0.5f);
    float cxf = floorf(gx), cyf = floorf(gy);
    double fxa = (double)(gx - cxf), fya = (double)(gy - cyf);
    int32_t cx0 = (int32_t)cxf, cy0 = (int32_t)cyf;
    double vj[4] = {(1.0 - fxa) * (1.0 - fya), fxa * (1.0 - fya), (1.0 - fxa) * fya, fxa * fya};
    uint32_t ka[4];
    for (int jn = 0; jn < 4; ++jn) {
      uint32_t cx = (uint32_t)(cx0 + (jn & 1)), cy = (uint32_t)(cy0 + (jn >> 1));
      ka[jn] = orc_lowbias32(cx * 0xcb1ab31fU + cy * 0x165667b1U + 0x27d4eb2fU);
    }
    if (rc) { rc->p = p; rc->cx0 = cx0; rc->cy0 = cy0; rc->afx = (float)fxa; rc->afy = (float)fya; }

    /* S6 + S7 + S8: 4 grids x 3 spatial x 4 angular = 48 draws
     * (ablations: 4 x 4 x 4 = 64; 10 x 4 x 4 = 160) */
    double C = mode == 3 ? zk_blend(znp, zuk, zvk, zA, so, N, p, ka, vj) : 0.0;
    for (int i = 0; i < NG; ++i) {
      uint32_t T; float sig, m1, cap;
      orc_gate_params(n[i], p, &T, &sig, &m1, &cap);
      if (rc) { rc->T[i] = T; rc->sigma[i] = sig; rc->m1[i] = m1; rc->cap[i] = cap; rc->pge1[i] = pge1_of(n[i], p); }
      double Ci = 0.0; /* b_theta_i(w_i N_i, p), interpolated (Eq. 14, R-16) */
      for (int k = 0; k < NS; ++k) {
        double Cik = 0.0;
        for (int jn = 0; jn < 4; ++jn) {
          uint32_t h = orc_draw_hash(hs[i][k] + ka[jn]);
          float c = sc->sampler == 1 ? exact_count(h, n[i], p) : orc_gated_count(h, T, sig, m1, cap);
          if (rc) { rc->hash[i*12 + k*4 + jn] = h; rc->count[i*12 + k*4 + jn] = c; }
          Cik += vj[jn] * (double)c;
        }
        Ci += betad[i][k] * Cik;
      }
      C += Ci; /* distributed law: sum over the grids (Eq. 10/13) */
    }

    /* S8: Eq. 3-4, D_P = D(n)/R * b / N(P), N(P) = N P (reading R-20); no
     * flake reflects (C = 0, e.g. N = 0 or p = 0): D_P = 0, not 0/0 */
    double Dp = C > 0.0 ? C / (M_PI * (double)ax * (double)ay * (double)R * (double)N * (double)P) : 0.0;
    /* S9: Eq. 1-2, fp64 shell from the raw fp32 inputs */
    orc_shell(sc, l, nrm, pos, ax, ay, Dp, rgb);
    if (rc) { rc->C = (float)C; rc->Dp = (float)Dp; }
  }
  *flags_out = flags;
fill_flags:
  if (rec) for (int l = 0; l < L; ++l) rec[l].flags = *flags_out;
}

int orc_eval(const float* duv, const float* uvm, const float* nrm, const float* pos,
             const float* mat, int64_t n, const orc_scene* sc, double* rgb,
             uint32_t* flags, orc_rec* rec) {
  orc_init();
  if (sc->n_lights < 0 || sc->n_lights > ORC_MAX_LIGHTS) return -1;
  if (sc->eval_mode < 0 || sc->eval_mode > 3) return -1;
  if (rec && sc->eval_mode != 0) return -1;   /* debug records describe the 48-draw path */
  for (int64_t i = 0; i < n; ++i)
    eval_pixel(duv + 4 * i, uvm + 4 * i, nrm + 4 * i, pos + 4 * i, mat + 4 * i, sc,
               rgb + 3 * i, flags + i, rec ? rec + i * sc->n_lights : 0);
  return 0;
}


/* ---------------------------------------------------------------------- */
/* Exhaustive contract-math checksums (SURVEY 8c-2 "Contract math itself"):
 * an order-independent 64-bit sum over an input range of
 * bits(f(x)) * (index * golden | 1), NaN results canonicalised (payload bits
 * differ between CPU and GPU). The GPU test library computes the same sum
 * with the product's device functions; equal sums over all 2^32 inputs mean
 * bit-equal functions. fn: 0 exp2 (y <= 0 or NaN), 1 log2(1-p) (0 < p < 1),
 * 2 rcp (normal x > 0), 3 rsqrt (normal x > 0), 4 atan2 in turns on hashed
 * finite pairs, 5 lowbias32 (all inputs). Test infrastructure.            */
/* ---------------------------------------------------------------------- */
static uint64_t cs_term(uint64_t idx, uint32_t bits) {
  return (uint64_t)bits * ((idx * 0x9E3779B97F4A7C15ull) | 1ull);
}
static uint32_t cs_bits(float r) { return r != r ? 0x7FC00000u : f2u(r); }

uint64_t orc_contract_checksum(int32_t fn, uint64_t lo, uint64_t hi) {
  orc_init();
  uint64_t acc = 0;
  for (uint64_t i = lo; i < hi; ++i) {
    uint32_t b = (uint32_t)i;
    float x = u2f(b);
    switch (fn) {
      case 0: if (!(x > 0.0f)) acc += cs_term(i, cs_bits(orc_exp2(x))); break;
      case 1: if (x > 0.0f && x < 1.0f) acc += cs_term(i, cs_bits(orc_log2_1mp(x))); break;
      case 2: if (x >= 0x1p-126f && x <= 0x1.fffffep127f) acc += cs_term(i, cs_bits(orc_rcp(x))); break;
      case 3: if (x >= 0x1p-126f && x <= 0x1.fffffep127f) acc += cs_term(i, cs_bits(orc_rsqrt(x))); break;
      case 4: {
        float yy = u2f(orc_lowbias32(b)), xx = u2f(orc_lowbias32(b ^ 0x9e3779b9u));
        if (fabsf(yy) <= 0x1.fffffep127f && fabsf(xx) <= 0x1.fffffep127f)
          acc += cs_term(i, cs_bits(orc_atan2_turns(yy, xx)));
        break;
      }
      case 5: acc += cs_term(i, orc_lowbias32(b)); break;
      default: break;
    }
  }
  return acc;
}
