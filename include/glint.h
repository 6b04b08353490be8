/*
 * glint.h -- C ABI of the B200-native glint evaluation library (libglint.so).
 *
 * Implements the per-pixel glinty-BRDF evaluation of arXiv 2306.05051
 * ("distributed binomial laws on anisotropic grids") for a structure-of-arrays
 * G-buffer on NVIDIA B200 (sm_100a). One frame = one kernel launch that runs
 * every step of the path for every (pixel, light):
 *
 *   S1 footprint from screen-space uv derivatives
 *   S2 anisotropic lattice: scale (Eq. 13), ratio/orientation
 *      (Fig. 6), 9-tetrahedra cell split -> 4 grids
 *   S3 grid transform (Eq. 12) + simplex surface grid
 *   S4 per-texel seeds coherent across LODs
 *   S5 p = R D(h)/D(n) (Eq. 4) + angular grid (Eq. 14)
 *   S6/S7 48 gated Gaussian binomial draws (Eq. 16-18)
 *   S8 distributed law + interpolation -> D_P (Eq. 3, 10)
 *   S9 microfacet radiance (Eq. 1-2), punctual lights
 *
 * P:Lnnn = line of the paper's text. The exact fp32 arithmetic of
 * every step is the contract of DESIGN.md §4; where the paper is silent the
 * readings of DESIGN.md §5 apply.
 *
 * Conventions
 *  - All functions return GLINT_OK (0) or a negative GLINT_E* code; no
 *    exception crosses the ABI. glint_strerror() describes a code.
 *  - Device pointers are CUDA device addresses on the context's device; the
 *    caller owns every buffer (typically torch tensors). The library never
 *    allocates or frees caller memory and never synchronises the stream in
 *    glint_eval / glint_eval_batch (errors of asynchronous execution surface
 *    at the caller's next synchronisation). The host-buffer entries
 *    (glint_eval_host, glint_eval_host_batch) are synchronous.
 *  - cudaStream_t is passed as void* (NULL = legacy default stream).
 */
#ifndef GLINT_H
#define GLINT_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GLINT_VERSION 20100 /* 2.1.0: debug record 184 words (simplex / angular fractions, P>=1); 2.0.0: tile origin, glint_count_active */

/* return codes */
#define GLINT_OK 0
#define GLINT_EINVAL -1   /* null pointer, size < 0, tile origin < 0, bad enum, K not in [1,8], beta not finite or
                             < 2^-20, n_lights not in [0,16], eval_mode not in [0,3] or debug records requested
                             with eval_mode != 0 */
#define GLINT_EALIGN -2   /* a plane / output pointer not 16-byte aligned, pitch < width */
#define GLINT_EDEVICE -3  /* no CUDA device, device is not sm_100, or ctx/device mismatch */
#define GLINT_ELIMIT -4   /* width*height >= 2^31 pixels, pitch*height (or the output's (y0+height)*out_pitch)
                             >= 2^40 float4, or the context's pool of 4096 graph-captured launch slots is
                             used up */
#define GLINT_ECUDA -5    /* a CUDA runtime call failed; see glint_last_cuda_error() */
#define GLINT_ENOMEM -6   /* host or device allocation failed */
#define GLINT_EALIAS -7   /* glint_eval_batch / glint_eval_host_batch: an output overlaps an input plane or
                             another output */

/* per-pixel output flags, stored as the bit pattern of out[pixel].w */
#define GLINT_FLAG_INVALID 1u        /* meta bit0 clear: pixel not shaded */
#define GLINT_FLAG_DEGENERATE 2u     /* |det J| outside [2^-64, 2^64), or major eigenvalue of J J^T >= 2^126 */
#define GLINT_FLAG_RATIO_CLAMPED 4u  /* anisotropy r > 2^K, clamped (reading R-25) */
#define GLINT_FLAG_P_CLAMPED 8u      /* R D(h)/D(n) > 1 for some light, clamped (R-19) */
#define GLINT_FLAG_UV_RANGE 16u      /* |u| or |v| > 2^24 (uv must be tile-local); with INVALID */

#define GLINT_MAX_LIGHTS 16
#define GLINT_ZQ 4096     /* quantile table size (reading R-2) */
#define GLINT_NANG 256    /* orientation table size: phi_m = m pi / 256 */

typedef struct glint_ctx glint_ctx;

/* A punctual light. kind 0 = point at pos_or_dir (E = I / d^2),
 * kind 1 = directional, pos_or_dir points toward the light (E = I).
 * Intensity domain: any finite value; the radiance is formed in fp64 and
 * rounded to fp32 once per light (so it reads +inf, never NaN, where the true
 * value exceeds fp32's range). */
typedef struct {
  int32_t kind;
  float pos_or_dir[3];
  float intensity[3];   /* RGB */
  int32_t reserved;
} glint_light;

/* Scene constants, passed BY VALUE to the kernel (lands in the launch's
 * constant bank; concurrent evals on different streams cannot race). */
typedef struct {
  uint32_t seed;            /* hash seed (reading R-23) */
  int32_t ndf_kind;         /* 0 = GGX, 1 = Beckmann */
  int32_t max_ratio_level;  /* K in [1, 8]: anisotropy levels r = 2^0..2^K (R-9) */
  float beta;               /* angular cell size / micro-roughness, > 0 (R-17) */
  float f0[3];              /* Schlick F0, RGB (R-21) */
  int32_t view_kind;        /* 0 = pinhole camera at view[], 1 = directional view[] */
  float view[3];
  int32_t n_lights;         /* 0 .. GLINT_MAX_LIGHTS */
  int32_t eval_mode;        /* draws per (pixel, light): 0 = 48, the paper's method (4 tetrahedron
                               grids x 3 simplex texels x 4 angular nodes); ablations of
                               its section 6: 1 = 64 (4 grids x 4 bilinear texels
                               x 4), 2 = 160 (10 prism grids x 4 x 4); 3 = the Zirr & Kaplanyan-
                               style baseline re-derived from P:L170-190, L975-983 (DESIGN.md
                               section 10: <= 16 footprint probes x 2 LODs x 4 texels x 4 nodes,
                               classical binomial of Eq. 15). Debug records: mode 0 only */
  int32_t reserved[3];
  glint_light lights[GLINT_MAX_LIGHTS];
} glint_scene;

/* Structure-of-arrays G-buffer. Five planes of float4 per pixel, row-major,
 * `pitch` float4 elements between rows (pitch >= width), 16-byte aligned:
 *   duv = (du/dx, dv/dx, du/dy, dv/dy)  screen-space uv derivatives
 *   uvm = (u, v, obj, meta)             tile-local uv; obj and meta are uint32
 *                                       bit patterns; meta bit0 = pixel valid
 *   nrm = (nx, ny, nz, -)               shading normal (normalised in-kernel)
 *   pos = (x, y, z, -)                  world position (point lights / camera)
 *   mat = (alpha_x, alpha_y, N, R)      roughness, flakes per unit uv^2, glint ratio R; clamped to
 *                                       alpha in [2^-16, 16], N in [0, 2^40], R in [0, 16], NaN to
 *                                       the lower bound (R-37). Components of nrm and pos
 *                                       (and of the scene's view and lights) must satisfy |x| <= 2^60
 *                                       so that squared lengths stay finite (R-27b); outside that
 *                                       domain radiance and records are unspecified (no crash)
 * For glint_eval the planes are device pointers; for glint_eval_host they are
 * host pointers (pinned memory gives full PCIe/C2C bandwidth). */
typedef struct {
  const void* duv;
  const void* uvm;
  const void* nrm;
  const void* pos;
  const void* mat;
  int32_t width;
  int32_t height;
  int64_t pitch;
  int32_t x0, y0;   /* tile origin in the output image (>= 0): pixel (x, y) of these planes is written to
                       out[(y0 + y) * out_pitch + x0 + x]. {0, 0} for a whole frame; a row band or tile
                       of a sharded frame passes its position so that its radiance lands in
                       place in a full-frame output (local, or a peer GPU's mapped buffer) */
} glint_gbuffer;

/* Optional per (pixel, light) debug record (184 words, 736 bytes), written
 * in-kernel by the same arithmetic (template instantiation) when `dbg` is
 * non-NULL; record index = (y * width + x) * n_lights + light. For tiny
 * parity inputs only. Fields mirror DESIGN.md §4.3. */
typedef struct {
  float P, r, psi;                 /* S1 footprint */
  int32_t ls[4], lr[4], jo[4];     /* S2 grid vertices (log2 texel area, ratio level, orientation) */
  float w[4], n[4];                /* distribution weights, trial counts n_i = w_i N 2^ls_i */
  int32_t lx[12], ly[12];          /* S3 simplex lattice vertices (low 32 bits), slot-major */
  float p;                         /* S5 success probability */
  int32_t cx0, cy0;                /* S5 angular base node */
  uint32_t T[4];                   /* S6 gate thresholds ceil(P>=1 2^23) */
  float sigma[4], m1[4], cap[4];   /* S6 Gaussian parameters */
  uint32_t hash[48];               /* S7 draw hashes, index = slot*12 + texel*4 + node */
  float count[48];                 /* S7 flake counts (integer-valued fp32; may exceed 2^31) */
  float C;                         /* S8 blended count */
  float Dp;                        /* S8 D_P(h) */
  uint32_t flags;
  uint32_t light_active;           /* n.wi > 0 and n.wo > 0 */
  float sfx[4], sfy[4];            /* S3 simplex cell fractions per slot (beta = barycentrics of (sfx, sfy)) */
  float afx, afy;                  /* S5 angular cell fractions (v_j = their bilinear weights, Eq. 14) */
  float pge1[4];                   /* S6 P>=1 = 1 - (1-p)^n per slot (0 when n <= 0 or p <= 0) */
  uint32_t reserved[4];
} glint_debug_rec;

int glint_version(void);
const char* glint_strerror(int code);
/* CUDA error code (cudaError_t value) of the most recent GLINT_ECUDA in this thread. */
int glint_last_cuda_error(void);

/* Host-only: build the tables exactly as glint_create uploads them:
 * z[k] = fp32(Phi^-1((k + 1/2) / 4096)), cosv[m] = fp32(cos(m pi/256)),
 * sinv[m] = fp32(sin(m pi/256)); computed in double precision. Any pointer may
 * be NULL. Needs no GPU. */
int glint_build_tables(float* z, float* cosv, float* sinv);

/* Create a context on `device` (must be sm_100): builds and uploads the
 * tables ("precompute once at startup"). The context is immutable
 * after creation; glint_eval may be called concurrently on different streams.
 * Returns GLINT_EDEVICE if no sm_100 device is present. */
int glint_create(glint_ctx** out, int device);
int glint_destroy(glint_ctx* ctx);   /* waits for the device (cudaDeviceSynchronize), then frees */

/* Evaluate every pixel of `gb` (device planes) for every light of `scene`:
 * out[(gb->y0 + y) * out_pitch + gb->x0 + x] = float4(R, G, B, flags bits) for
 * all pixels of the tile (fully overwritten; nothing else is written). `out` may be any address the current device can store to:
 * its own memory, or a peer GPU's buffer mapped through CUDA IPC / peer
 * access (the kernel then streams the radiance over NVLink -- the fused
 * gather of DESIGN.md section 8). `dbg` (device, nullable) receives
 * width*height*n_lights records. One kernel launch on `stream`; asynchronous;
 * no host synchronisation or allocation, so it can be captured in a CUDA
 * graph. Each launch owns a tile-scheduler counter pair, reset by the launch
 * itself: an ordinary launch takes the next slot of a ring of 1024, so at most
 * 1024 launches of one context may be in flight at once (across all streams);
 * a launch recorded by stream capture (cudaStreamIsCapturing) gets a pair of
 * its own from a separate pool of 4096 that is never recycled, so a graph can
 * be replayed alongside any number of ordinary launches, but one graph must
 * not be replayed concurrently with itself. */
int glint_eval(const glint_ctx* ctx, const glint_gbuffer* gb, const glint_scene* scene,
               void* out, int64_t out_pitch, glint_debug_rec* dbg, void* stream);

/* Evaluate n_frames independent frames (C2's elevation set, C4's jittered
 * frames, C5's zoom path: P:L1010-1032 time whole frames): frame f is exactly
 * glint_eval(ctx, &gbs[f], &scenes[f], outs[f], out_pitches[f], NULL, stream),
 * bit for bit. The launches are chained with programmatic dependent launch:
 * frame f+1's blocks start on the SMs that frame f's blocks free at its tail
 * instead of after frame f completes ("frame batching").
 * This is only correct because the frames do not depend on each other, so the
 * call checks it: every output range [outs[f], outs[f] + ((h-1)*out_pitch + w)
 * float4) must be disjoint from every input plane range of every frame and
 * from every other output, else GLINT_EALIAS (nothing launched). The test is
 * exact for regions of equal pitch (e.g. frames side by side as column views
 * of one atlas are accepted) and conservative otherwise (overlapping
 * [first, last] byte spans of regions with different pitches are refused). Frame 0
 * waits for all prior work on `stream` like glint_eval; work enqueued on
 * `stream` after the call sees every frame complete (each frame's grid waits
 * for its predecessor before it exits). Arguments: host arrays of n_frames
 * entries (gbs, scenes, outs, out_pitches), device buffers behind them as for
 * glint_eval; n_frames = 0 is a no-op; empty frames are skipped. Every frame
 * is validated before the first launch; an error launches nothing. No debug
 * records (use glint_eval). Graph-capturable; one scheduler slot per frame. */
int glint_eval_batch(const glint_ctx* ctx, int n_frames, const glint_gbuffer* gbs, const glint_scene* scenes,
                     void* const* outs, const int64_t* out_pitches, void* stream);

/* End-to-end entry with HOST buffers: copies the planes host->device, runs the
 * kernel and copies the radiance device->host, pipelined over row chunks on
 * two internal streams (copy/compute overlap). Uses device staging owned by
 * the context (grown on demand, freed by glint_destroy); concurrent calls on
 * one context are serialised by an internal lock (use one context per thread
 * for parallel host pipelines). Synchronous: returns after `out` (host, out_pitch float4 per row)
 * is complete. `stream` orders the work after the caller's prior work. */
int glint_eval_host(glint_ctx* ctx, const glint_gbuffer* gb_host, const glint_scene* scene,
                    void* out_host, int64_t out_pitch, void* stream);

/* glint_eval_host over n_frames independent frames (host arrays of n_frames
 * entries, host buffers behind them): frame f's radiance equals
 * glint_eval_host(ctx, &gbs_host[f], &scenes[f], outs_host[f], out_pitches[f],
 * stream) bit for bit. The row-chunk pipeline runs continuously across the
 * frames, so it fills and drains once per call instead of once per frame.
 * Every frame is validated first; outputs (16-byte aligned) must not overlap
 * any input plane or another output (GLINT_EALIAS). Synchronous, serialised
 * per context like glint_eval_host. n_frames = 0 is a no-op. */
int glint_eval_host_batch(glint_ctx* ctx, int n_frames, const glint_gbuffer* gbs_host, const glint_scene* scenes,
                          void* const* outs_host, const int64_t* out_pitches, void* stream);

/* Count the (pixel, light) evaluations of `gb` under `scene`: pixels that are
 * valid with a non-degenerate footprint (flags 0 apart from RATIO/P clamps)
 * times the lights active there (n.wi > 0, n.wo > 0, |d|^2 in [2^-126, 2^120]:
 * the pairs whose S5-S9 work glint_eval does, R-27b) -- the unit of
 * the throughput metric. Adds the count to *d_count (a device uint64 the
 * caller zeroes); one kernel launch on `stream`, asynchronous. */
int glint_count_active(const glint_ctx* ctx, const glint_gbuffer* gb, const glint_scene* scene,
                       unsigned long long* d_count, void* stream);

/* Copies of the device-resident tables (host pointers), for parity tests. */
int glint_get_tables(const glint_ctx* ctx, float* z, float* cosv, float* sinv);

/* Number of kernel launches issued by this context so far (bench evidence). */
int64_t glint_launch_count(const glint_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* GLINT_H */
