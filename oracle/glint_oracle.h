/*
 * glint_oracle.h -- CPU ORACLE for the glint hot path (TEST INFRASTRUCTURE ONLY).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library. The product path (the CUDA library
 * under paper_2306_05051_b200/csrc) never includes, links or calls it, and
 * this file shares no code with it.
 *
 * Plain, slow, scalar C. Decision-path values (everything that feeds an
 * integer: lattice keys, simplex vertices, angular nodes, hashes, gates,
 * counts) follow the fp32 arithmetic contract of DESIGN.md §4 op by op;
 * the radiance path (Eq. 1-4 factors) is computed in fp64.
 *
 * Paper = /root/reference/PAPER.md (arXiv 2306.05051), cited as P:Lnnn.
 */
#ifndef GLINT_ORACLE_H
#define GLINT_ORACLE_H
#include <stdint.h>

#define ORC_MAX_LIGHTS 16
#define ORC_ZQ 4096 /* quantile-table size (reading R-2) */
#define ORC_NANG 256 /* orientation table: m*pi/256, m < 256 */

/* output flag bits (same meaning as the product's GLINT_FLAG_*) */
#define ORC_FLAG_INVALID 1u
#define ORC_FLAG_DEGENERATE 2u
#define ORC_FLAG_RATIO_CLAMPED 4u
#define ORC_FLAG_P_CLAMPED 8u
#define ORC_FLAG_UV_RANGE 16u

typedef struct {
  int32_t kind;          /* 0 = point (pos), 1 = directional (dir toward light) */
  float pos_or_dir[3];
  float intensity[3];
  int32_t pad_;
} orc_light;

typedef struct {
  uint32_t seed;
  int32_t ndf_kind;        /* 0 = GGX, 1 = Beckmann */
  int32_t max_ratio_level; /* K in [1, 8] */
  float beta;              /* angular cell size (micro-roughness), > 0 */
  float f0[3];
  int32_t view_kind;       /* 0 = point camera at view[], 1 = directional view[] */
  float view[3];
  int32_t n_lights;
  int32_t sampler;         /* 0 = gated Gaussian (Eq. 18), 1 = exact Bernoulli sum (tests) */
  int32_t eval_mode;       /* draws per pixel-light: 0 = 48 (tetrahedra x simplex x angular),
                              1 = 64 (tetrahedra x bilinear x angular), 2 = 160 (10 prism
                              vertices x bilinear x angular) -- P:L749, L758, L928;
                              3 = Zirr & Kaplanyan-style baseline */
  int32_t pad_[2];
  orc_light lights[ORC_MAX_LIGHTS];
} orc_scene;

/* per (pixel, light) debug record -- 184 x 4-byte words */
typedef struct {
  float P, r, psi;                 /* footprint (S1) */
  int32_t ls[4], lr[4], jo[4];     /* 4 lattice slots (S2) */
  float w[4], n[4];                /* distributed weights, trial counts */
  int32_t lx[12], ly[12];          /* simplex lattice vertices (S3) */
  float p;                         /* success probability (Eq. 4) */
  int32_t cx0, cy0;                /* angular base node (Eq. 14) */
  uint32_t T[4];                   /* gate thresholds, ceil(P>=1 * 2^23) */
  float sigma[4], m1[4], cap[4];   /* Eq. 17 parameters */
  uint32_t hash[48];               /* per-draw 32-bit hash */
  float count[48];                 /* per-draw flake count (integer-valued fp32) */
  float C;                         /* blended count (fp32 view of the fp64 value) */
  float Dp;                        /* D_P(h) (Eq. 3), fp32 view */
  uint32_t flags;
  uint32_t light_active;           /* 1 if n.wi > 0 and n.wo > 0 */
  float sfx[4], sfy[4];            /* simplex cell fractions per grid (S3) */
  float afx, afy;                  /* angular cell fractions (Eq. 14) */
  float pge1[4];                   /* P>=1 per grid (Eq. 16; 0 if n <= 0 or p <= 0) */
  uint32_t pad_[4];
} orc_rec;

int orc_init(void);
const float* orc_ztable(void);
const float* orc_costable(void);
const float* orc_sintable(void);

/* Evaluate n pixels (SoA float4 planes, row-major, contiguous). rgb: n*3
 * doubles; flags: n words; rec: n*n_lights records or NULL. */
int orc_eval(const float* duv, const float* uvm, const float* nrm, const float* pos,
             const float* mat, int64_t n, const orc_scene* sc, double* rgb,
             uint32_t* flags, orc_rec* rec);

/* contract primitives, exported for pin tests */
float orc_exp2(float y);
float orc_rsqrt(float x);
float orc_rcp(float x);
float orc_log2_1mp(float p);
float orc_atan2_turns(float y, float x);
uint32_t orc_lowbias32(uint32_t x);
uint32_t orc_draw_hash(uint32_t x);
int orc_footprint(const float duv[4], float* P, float* r, float* psi);
int orc_lattice(float P, float r, float psi, int32_t K, int32_t ls[4], int32_t lr[4],
                int32_t jo[4], float w[4], uint32_t* flags);
int orc_lattice10(float P, float r, float psi, int32_t K, int32_t ls[10], int32_t lr[10],
                  int32_t jo[10], float w[10], uint32_t* flags);
void orc_bilinear(float x, float y, int64_t lx[4], int64_t ly[4], float beta[4]);
void orc_grid_uv(float u, float v, int32_t ls, int32_t lr, int32_t jo, float* x, float* y);
void orc_simplex(float x, float y, int64_t lx[3], int64_t ly[3], float beta[3]);
void orc_gate_params(float n, float p, uint32_t* T, float* sigma, float* m1, float* cap);
float orc_gated_count(uint32_t h, uint32_t T, float sigma, float m1, float cap);
float orc_ratio(int32_t ndf_kind, float ax, float ay, float hx, float hy, float hz);
double orc_smith_g2(int32_t kind, double ax, double ay, const double wi_l[3], const double wo_l[3]);
double orc_schlick(double f0, double cos_t);
/* S9 shell of light l (fp64 from the raw fp32 inputs): adds F G2 Dp E / (4 n.wi)
 * to rgb when Dp > 0 and both fp64 cosines are > 0; returns 1 if it added. */
int orc_shell(const orc_scene* sc, int32_t l, const float nrm[3], const float pos[3], float ax, float ay,
              double Dp, double rgb[3]);
int orc_zk_probes(const float duv[4], float u, float v, float uk[16], float vk[16], float* area,
                  uint32_t* flags);
void orc_zk_lod(float A, int32_t* kz, float* t);
float orc_zk_count(uint32_t w, float nt, float p);
uint64_t orc_contract_checksum(int32_t fn, uint64_t lo, uint64_t hi);
#endif
