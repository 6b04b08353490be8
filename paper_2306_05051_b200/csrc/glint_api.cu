// glint_api.cu -- host side of the C ABI declared in include/glint.h.
//
// Validation, table construction (double precision on the host, rounded to
// fp32: "a small texture of random numbers that we precompute once at
// startup"), launch-shape selection and the end-to-end host-buffer pipeline.
// No arithmetic of the glint path runs here.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <mutex>
#include <vector>

#include "../../include/glint.h"
#include "glint_kernel.h"

static thread_local int g_last_cuda = 0;

#define GL_CUDA(call)                                \
  do {                                               \
    cudaError_t e_ = (call);                         \
    if (e_ != cudaSuccess) {                         \
      g_last_cuda = (int)e_;                         \
      return GLINT_ECUDA;                            \
    }                                                \
  } while (0)

struct glint_ctx {
  int device;
  int sm_count;
  int blocks_per_sm;
  float* d_z;
  float2* d_cs;
  float h_z[GLINT_ZQ];
  float h_cos[GLINT_NANG], h_sin[GLINT_NANG];
  std::atomic<int64_t> launches;
  unsigned long long* d_sched;   // (kSchedSlots + kCaptureSlots) x [tile counter, finished blocks], zeroed
  std::atomic<int64_t> sched_next;     // ring of kSchedSlots for ordinary launches
  std::atomic<int64_t> capture_next;   // pool of kCaptureSlots for graph-captured launches (never recycled)
  // glint_eval_host staging (2 buffers x (5 planes + out)), grown on demand
  size_t stage_px;
  float4* d_stage[2][6];
  cudaStream_t st[2];
  cudaEvent_t ev_in, ev_done[2];
  std::mutex host_mu;   // serialises glint_eval_host (staging and streams are per context)
};

static_assert(sizeof(glint_debug_rec) == 184 * 4, "glint.h 2.1: the debug record is 184 words");
extern "C" int glint_version(void) { return GLINT_VERSION; }

extern "C" const char* glint_strerror(int code) {
  switch (code) {
    case GLINT_OK: return "ok";
    case GLINT_EALIAS: return "an output overlaps an input plane or another output of the batch";
    case GLINT_EINVAL: return "invalid argument";
    case GLINT_EALIGN: return "pointer not 16-byte aligned or pitch < width";
    case GLINT_EDEVICE: return "no suitable sm_100 device / context-device mismatch";
    case GLINT_ELIMIT: return "image too large (>= 2^31 pixels or >= 2^40 float4 spans), or graph-capture slots exhausted";
    case GLINT_ECUDA: return "CUDA runtime error (see glint_last_cuda_error)";
    case GLINT_ENOMEM: return "allocation failed";
    default: return "unknown error";
  }
}

extern "C" int glint_last_cuda_error(void) { return g_last_cuda; }

// ---------------------------------------------------------------------------
// Tables. Z[k] = fp32(Phi^-1((k + 1/2)/4096)): Abramowitz & Stegun 26.2.23
// rational start, then Halley iterations on Phi(x) - q with Phi from erfc,
// to double precision (the oracle uses a different method: bisection).
// ---------------------------------------------------------------------------
static double norm_quantile(double q) {
  double pp = q < 0.5 ? q : 1.0 - q;
  double t = sqrt(-2.0 * log(pp));
  double x = t - (2.515517 + 0.802853 * t + 0.010328 * t * t) /
                     (1.0 + 1.432788 * t + 0.189269 * t * t + 0.001308 * t * t * t);
  if (q < 0.5) x = -x;
  for (int it = 0; it < 6; ++it) {
    double e = 0.5 * erfc(-x / sqrt(2.0)) - q;
    double u = e * sqrt(2.0 * M_PI) * exp(0.5 * x * x);
    double dx = u / (1.0 + 0.5 * x * u);
    x -= dx;
    if (fabs(dx) <= 1e-17 * (1.0 + fabs(x))) break;
  }
  return x;
}

extern "C" int glint_build_tables(float* z, float* cosv, float* sinv) {
  if (z)
    for (int k = 0; k < GLINT_ZQ; ++k) z[k] = (float)norm_quantile(((double)k + 0.5) / (double)GLINT_ZQ);
  for (int m = 0; m < GLINT_NANG; ++m) {
    double ang = (double)m * M_PI / 256.0;
    if (cosv) cosv[m] = (float)cos(ang);
    if (sinv) sinv[m] = (float)sin(ang);
  }
  return GLINT_OK;
}

// ---------------------------------------------------------------------------
// Context
// ---------------------------------------------------------------------------
extern "C" int glint_create(glint_ctx** out, int device) {
  if (!out) return GLINT_EINVAL;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0) {
    cudaGetLastError();
    return GLINT_EDEVICE;
  }
  if (device < 0 || device >= ndev) return GLINT_EDEVICE;
  cudaDeviceProp prop;
  GL_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10 || prop.minor != 0) return GLINT_EDEVICE;   // built for sm_100a only
  int prev = 0;
  GL_CUDA(cudaGetDevice(&prev));
  GL_CUDA(cudaSetDevice(device));
  glint_ctx* c = new (std::nothrow) glint_ctx();
  if (!c) return GLINT_ENOMEM;
  c->device = device;
  c->sm_count = prop.multiProcessorCount;
  c->launches = 0;
  c->sched_next = 0;
  c->capture_next = 0;
  int rc = GLINT_OK;
  float2 cs[GLINT_NANG];
  glint_build_tables(c->h_z, c->h_cos, c->h_sin);
  for (int m = 0; m < GLINT_NANG; ++m) cs[m] = make_float2(c->h_cos[m], c->h_sin[m]);
  cudaError_t e = glint::occupancy_blocks_per_sm(&c->blocks_per_sm);
  if (e == cudaSuccess) e = cudaMalloc(&c->d_z, sizeof(float) * GLINT_ZQ);
  if (e == cudaSuccess) e = cudaMalloc(&c->d_cs, sizeof(float2) * GLINT_NANG);
  const size_t sched_bytes = sizeof(unsigned long long) * 2 * (glint::kSchedSlots + glint::kCaptureSlots);
  if (e == cudaSuccess) e = cudaMalloc(&c->d_sched, sched_bytes);
  if (e == cudaSuccess) e = cudaMemset(c->d_sched, 0, sched_bytes);
  if (e == cudaSuccess) e = cudaMemcpy(c->d_z, c->h_z, sizeof(float) * GLINT_ZQ, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(c->d_cs, cs, sizeof(float2) * GLINT_NANG, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    g_last_cuda = (int)e;
    rc = GLINT_ECUDA;
    if (c->d_z) cudaFree(c->d_z);
    if (c->d_cs) cudaFree(c->d_cs);
    if (c->d_sched) cudaFree(c->d_sched);
    delete c;
    c = nullptr;
  } else if (c->blocks_per_sm < 1) {
    c->blocks_per_sm = 1;
  }
  cudaSetDevice(prev);
  *out = c;
  return rc;
}

static void free_stage(glint_ctx* c) {
  for (int b = 0; b < 2; ++b)
    for (int p = 0; p < 6; ++p)
      if (c->d_stage[b][p]) { cudaFree(c->d_stage[b][p]); c->d_stage[b][p] = nullptr; }
  c->stage_px = 0;
}

extern "C" int glint_destroy(glint_ctx* c) {
  if (!c) return GLINT_EINVAL;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(c->device);
  // launches still in flight on callers' streams read the tables and the
  // scheduler counters freed below: wait for the device first
  cudaDeviceSynchronize();
  free_stage(c);
  for (int b = 0; b < 2; ++b) {
    if (c->st[b]) cudaStreamDestroy(c->st[b]);
    if (c->ev_done[b]) cudaEventDestroy(c->ev_done[b]);
  }
  if (c->ev_in) cudaEventDestroy(c->ev_in);
  cudaFree(c->d_z);
  cudaFree(c->d_cs);
  cudaFree(c->d_sched);
  cudaSetDevice(prev);
  delete c;
  return GLINT_OK;
}

extern "C" int glint_get_tables(const glint_ctx* c, float* z, float* cosv, float* sinv) {
  if (!c) return GLINT_EINVAL;
  int prev = 0;
  GL_CUDA(cudaGetDevice(&prev));
  GL_CUDA(cudaSetDevice(c->device));
  float2 cs[GLINT_NANG];
  cudaError_t e = cudaSuccess;
  if (z) e = cudaMemcpy(z, c->d_z, sizeof(float) * GLINT_ZQ, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(cs, c->d_cs, sizeof(cs), cudaMemcpyDeviceToHost);
  cudaSetDevice(prev);
  if (e != cudaSuccess) { g_last_cuda = (int)e; return GLINT_ECUDA; }
  for (int m = 0; m < GLINT_NANG; ++m) {
    if (cosv) cosv[m] = cs[m].x;
    if (sinv) sinv[m] = cs[m].y;
  }
  return GLINT_OK;
}

extern "C" int64_t glint_launch_count(const glint_ctx* c) { return c ? c->launches.load() : -1; }

// ---------------------------------------------------------------------------
// Validation
// ---------------------------------------------------------------------------
static bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

static int validate_scene(const glint_scene* s) {
  if (!s) return GLINT_EINVAL;
  if (s->ndf_kind != 0 && s->ndf_kind != 1) return GLINT_EINVAL;
  if (s->view_kind != 0 && s->view_kind != 1) return GLINT_EINVAL;
  if (s->max_ratio_level < 1 || s->max_ratio_level > 8) return GLINT_EINVAL;
  if (!(s->beta > 0.0f) || !isfinite(s->beta) || s->beta < 0x1p-20f) return GLINT_EINVAL;
  if (s->n_lights < 0 || s->n_lights > GLINT_MAX_LIGHTS) return GLINT_EINVAL;
  if (s->eval_mode < 0 || s->eval_mode > 3) return GLINT_EINVAL;
  for (int l = 0; l < s->n_lights; ++l)
    if (s->lights[l].kind != 0 && s->lights[l].kind != 1) return GLINT_EINVAL;
  return GLINT_OK;
}

static int validate_gbuffer(const glint_gbuffer* g, int64_t out_pitch) {
  if (!g) return GLINT_EINVAL;
  if (g->width < 0 || g->height < 0 || g->x0 < 0 || g->y0 < 0) return GLINT_EINVAL;
  if (g->width == 0 || g->height == 0) return GLINT_OK;
  if (!g->duv || !g->uvm || !g->nrm || !g->pos || !g->mat) return GLINT_EINVAL;
  if (g->pitch < g->width || out_pitch < g->width) return GLINT_EALIGN;
  if (!aligned16(g->duv) || !aligned16(g->uvm) || !aligned16(g->nrm) || !aligned16(g->pos) || !aligned16(g->mat))
    return GLINT_EALIGN;
  if ((int64_t)g->width * g->height >= (int64_t)1 << 31) return GLINT_ELIMIT;
  if (g->pitch * (int64_t)g->height >= (int64_t)1 << 40) return GLINT_ELIMIT;
  if (out_pitch >= (int64_t)1 << 40 || ((int64_t)g->y0 + g->height) * out_pitch + g->x0 >= (int64_t)1 << 40)
    return GLINT_ELIMIT;
  return GLINT_OK;
}

// the tile's first output element: out + y0 * out_pitch + x0 (float4)
static void* tile_out(void* out, const glint_gbuffer* g, int64_t out_pitch) {
  return (void*)((float4*)out + (int64_t)g->y0 * out_pitch + g->x0);
}

// A scheduler counter pair for this launch: ordinary launches take the next
// slot of a ring (reused kSchedSlots launches later); a launch recorded by
// stream capture owns a slot of a separate pool for good (its graph may be
// replayed at any time alongside ordinary launches).
struct Slots {
  int64_t first;   // first slot index of this call's run
  bool ring;       // ordinary launches (ring) or graph-captured ones (pool)
};
static int sched_slots(const glint_ctx* c, cudaStream_t stream, int n, Slots* out) {
  glint_ctx* cm = const_cast<glint_ctx*>(c);
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  GL_CUDA(cudaStreamIsCapturing(stream, &st));
  out->ring = st != cudaStreamCaptureStatusActive;
  if (out->ring) {
    out->first = cm->sched_next.fetch_add(n);
  } else {
    out->first = cm->capture_next.fetch_add(n);
    if (out->first + n > glint::kCaptureSlots) return GLINT_ELIMIT;
  }
  return GLINT_OK;
}
// the counter pair of the i-th launch of a run
static unsigned long long* slot_at(const glint_ctx* c, const Slots& s, int i) {
  return s.ring ? c->d_sched + 2 * ((s.first + i) % glint::kSchedSlots)
                : c->d_sched + 2 * (glint::kSchedSlots + s.first + i);
}

static void make_params(const glint_ctx* c, const glint_gbuffer* gb, const glint_scene* sc, void* out,
                        int64_t out_pitch, glint_debug_rec* dbg, unsigned long long* slot, glint::KParams* kp) {
  glint::KParams& k = *kp;
  k.sched = slot;
  k.duv = (const float4*)gb->duv;
  k.uvm = (const float4*)gb->uvm;
  k.nrm = (const float4*)gb->nrm;
  k.pos = (const float4*)gb->pos;
  k.mat = (const float4*)gb->mat;
  k.out = (float4*)tile_out(out, gb, out_pitch);
  k.dbg = dbg;
  k.ztab = c->d_z;
  k.cstab = c->d_cs;
  k.width = gb->width;
  k.height = gb->height;
  k.pitch = gb->pitch;
  k.out_pitch = out_pitch;
  k.c1s = 0x7feb352du;   // the draw hash's first multiplier, twice (see KParams)
  k.c1n = 0x7feb352du;
  k.sc = *sc;
  k.f0_fast = sc->f0[0] >= 0x1p-10f && sc->f0[1] >= 0x1p-10f && sc->f0[2] >= 0x1p-10f;
}

static int grid_for(const glint_ctx* c, int64_t n_pix) {
  int64_t need = (n_pix + glint::kTile - 1) / glint::kTile;
  int64_t cap = (int64_t)c->sm_count * c->blocks_per_sm;
  return (int)(need < cap ? need : cap);
}

// ---------------------------------------------------------------------------
// glint_eval: device buffers, one launch, asynchronous
// ---------------------------------------------------------------------------
extern "C" int glint_eval(const glint_ctx* c, const glint_gbuffer* gb, const glint_scene* sc, void* out,
                          int64_t out_pitch, glint_debug_rec* dbg, void* stream) {
  if (!c) return GLINT_EINVAL;
  int rc = validate_scene(sc);
  if (rc) return rc;
  rc = validate_gbuffer(gb, out_pitch);
  if (rc) return rc;
  if (gb->width == 0 || gb->height == 0) return GLINT_OK;
  if (!out) return GLINT_EINVAL;
  if (dbg && sc->eval_mode != 0) return GLINT_EINVAL;
  if (!aligned16(out)) return GLINT_EALIGN;
  int cur = -1;
  GL_CUDA(cudaGetDevice(&cur));
  if (cur != c->device) return GLINT_EDEVICE;
  Slots slot;
  rc = sched_slots(c, (cudaStream_t)stream, 1, &slot);
  if (rc) return rc;
  glint::KParams k;
  make_params(c, gb, sc, out, out_pitch, dbg, slot_at(c, slot, 0), &k);
  int64_t n_pix = (int64_t)gb->width * gb->height;
  GL_CUDA(glint::launch_eval(k, grid_for(c, n_pix), dbg != nullptr, (cudaStream_t)stream));
  const_cast<glint_ctx*>(c)->launches++;
  return GLINT_OK;
}

// ---------------------------------------------------------------------------
// glint_eval_batch: independent frames, launches chained with programmatic
// dependent launch (frame f+1 fills the SMs frame f frees at its tail)
// ---------------------------------------------------------------------------
namespace {
// a pitched region: h rows of w float4 at lo + r * pitch float4 (bytes below)
struct Range { uintptr_t lo, hi; int64_t pitch, w, h; };   // [lo, hi): its whole span
Range plane_range(const void* p, int64_t pitch, int w, int h) {
  const uintptr_t lo = (uintptr_t)p;
  return {lo, lo + (uintptr_t)(((int64_t)(h - 1) * pitch + w) * 16), pitch * 16, (int64_t)w * 16, h};
}
// do two regions share a byte? Disjoint spans: no. Equal pitches P: with
// b.lo - a.lo = q P + rem (0 <= rem < P), b's row s starts at column rem of
// a's row q + s and, if rem + b.w > P, runs on into a's row q + s + 1: exact
// in O(1). Unequal pitches: the spans' overlap (conservative).
bool overlap_one_way(const Range& a, const Range& b) {   // b.lo >= a.lo, same pitch (width <= pitch)
  const int64_t P = a.pitch, d = (int64_t)(b.lo - a.lo);
  const int64_t q = d / P, rem = d % P;
  // rows of a that b's rows land on: q .. q + b.h - 1 (same column rem)
  const bool same_row = rem < a.w && q < a.h;                 // b row 0 meets a row q (q >= 0)
  const bool next_row = rem + b.w > P && q + 1 < a.h;          // b row 0 wraps into a row q + 1
  return same_row || next_row;
}
bool overlap(Range a, Range b) {
  if (!(a.lo < b.hi && b.lo < a.hi)) return false;
  // a single row has no pitch of its own: it can take the other's if it fits
  if (a.h == 1 && a.w <= b.pitch) a.pitch = b.pitch;
  if (b.h == 1 && b.w <= a.pitch) b.pitch = a.pitch;
  if (a.pitch != b.pitch) return true;
  return a.lo <= b.lo ? overlap_one_way(a, b) : overlap_one_way(b, a);
}
}  // namespace

// every frame valid; no output overlaps any input plane or another output
// (frames of a batch run concurrently); the outputs non-null and aligned
static int validate_batch_impl(int n_frames, const glint_gbuffer* gbs, const glint_scene* scenes,
                               void* const* outs, const int64_t* out_pitches) {
  std::vector<Range> outr, inr;
  for (int f = 0; f < n_frames; ++f) {
    int rc = validate_scene(&scenes[f]);
    if (rc) return rc;
    rc = validate_gbuffer(&gbs[f], out_pitches[f]);
    if (rc) return rc;
    const glint_gbuffer& g = gbs[f];
    if (g.width == 0 || g.height == 0) continue;
    if (!outs[f]) return GLINT_EINVAL;
    if (!aligned16(outs[f])) return GLINT_EALIGN;
    outr.push_back(plane_range(tile_out(outs[f], &g, out_pitches[f]), out_pitches[f], g.width, g.height));
    for (const void* p : {g.duv, g.uvm, g.nrm, g.pos, g.mat}) inr.push_back(plane_range(p, g.pitch, g.width, g.height));
  }
  for (size_t a = 0; a < outr.size(); ++a) {
    for (const Range& r : inr)
      if (overlap(outr[a], r)) return GLINT_EALIAS;
    for (size_t b = a + 1; b < outr.size(); ++b)
      if (overlap(outr[a], outr[b])) return GLINT_EALIAS;
  }
  return GLINT_OK;
}

// no exception crosses the ABI: an allocation failure of the range lists is
// GLINT_ENOMEM
static int validate_batch(int n_frames, const glint_gbuffer* gbs, const glint_scene* scenes, void* const* outs,
                          const int64_t* out_pitches) {
  try {
    return validate_batch_impl(n_frames, gbs, scenes, outs, out_pitches);
  } catch (...) {
    return GLINT_ENOMEM;
  }
}

extern "C" int glint_eval_batch(const glint_ctx* c, int n_frames, const glint_gbuffer* gbs, const glint_scene* scenes,
                                void* const* outs, const int64_t* out_pitches, void* stream) {
  if (!c || n_frames < 0) return GLINT_EINVAL;
  if (n_frames == 0) return GLINT_OK;
  if (!gbs || !scenes || !outs || !out_pitches) return GLINT_EINVAL;
  int rc = validate_batch(n_frames, gbs, scenes, outs, out_pitches);
  if (rc) return rc;
  int cur = -1;
  GL_CUDA(cudaGetDevice(&cur));
  if (cur != c->device) return GLINT_EDEVICE;
  int n_launch = 0;
  for (int f = 0; f < n_frames; ++f) n_launch += (gbs[f].width > 0 && gbs[f].height > 0) ? 1 : 0;
  Slots slots;
  rc = sched_slots(c, (cudaStream_t)stream, n_launch, &slots);
  if (rc) return rc;
  int i = 0;
  for (int f = 0; f < n_frames; ++f) {
    const glint_gbuffer& g = gbs[f];
    if (g.width == 0 || g.height == 0) continue;
    glint::KParams k;
    make_params(c, &g, &scenes[f], outs[f], out_pitches[f], nullptr, slot_at(c, slots, i), &k);
    GL_CUDA(glint::launch_eval(k, grid_for(c, (int64_t)g.width * g.height), false, (cudaStream_t)stream, i > 0));
    const_cast<glint_ctx*>(c)->launches++;
    ++i;
  }
  return GLINT_OK;
}

// ---------------------------------------------------------------------------
// glint_eval_host: host planes in, host radiance out; row chunks pipelined
// over two streams so H2D(chunk c+1) and D2H(chunk c-1) overlap kernel(c).
// ---------------------------------------------------------------------------
static int ensure_stage(glint_ctx* c, size_t px) {
  if (!c->st[0]) {
    for (int b = 0; b < 2; ++b) {
      GL_CUDA(cudaStreamCreateWithFlags(&c->st[b], cudaStreamNonBlocking));
      GL_CUDA(cudaEventCreateWithFlags(&c->ev_done[b], cudaEventDisableTiming));
    }
    GL_CUDA(cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming));
  }
  if (c->stage_px >= px) return GLINT_OK;
  free_stage(c);
  for (int b = 0; b < 2; ++b)
    for (int p = 0; p < 6; ++p) {
      cudaError_t e = cudaMalloc(&c->d_stage[b][p], px * sizeof(float4));
      if (e != cudaSuccess) { g_last_cuda = (int)e; free_stage(c); return GLINT_ENOMEM; }
    }
  c->stage_px = px;
  return GLINT_OK;
}

// The enqueue part of host_pipeline: H2D of each row chunk into staging
// buffer b = chunk & 1, the kernel, D2H into the caller's output (at the
// frame's tile origin) -- all on internal stream b. Returns at the first error.
static int host_pipeline_enqueue(glint_ctx* c, int n, const glint_gbuffer* gbs, const glint_scene* scs,
                                 void* const* outs, const int64_t* out_pitches, void* stream, int64_t chunk_px) {
  GL_CUDA(cudaEventRecord(c->ev_in, (cudaStream_t)stream));
  for (int b = 0; b < 2; ++b) GL_CUDA(cudaStreamWaitEvent(c->st[b], c->ev_in, 0));
  int chunk = 0;
  for (int f = 0; f < n; ++f) {
    const glint_gbuffer* gb = &gbs[f];
    const int W = gb->width, H = gb->height;
    if (W == 0 || H == 0) continue;
    int rows = (int)(chunk_px / W);
    rows = rows < 1 ? 1 : (rows > H ? H : rows);
    const void* planes[5] = {gb->duv, gb->uvm, gb->nrm, gb->pos, gb->mat};
    const size_t rowb = (size_t)W * sizeof(float4);
    float4* out_tile = (float4*)tile_out(outs[f], gb, out_pitches[f]);
    for (int y0 = 0; y0 < H; y0 += rows, ++chunk) {
      const int b = chunk & 1;
      const int nr = (y0 + rows <= H) ? rows : H - y0;
      cudaStream_t s = c->st[b];
      for (int p = 0; p < 5; ++p)
        GL_CUDA(cudaMemcpy2DAsync(c->d_stage[b][p], rowb, (const float4*)planes[p] + (int64_t)y0 * gb->pitch,
                                  (size_t)gb->pitch * sizeof(float4), rowb, nr, cudaMemcpyHostToDevice, s));
      glint_gbuffer sub;
      sub.duv = c->d_stage[b][0];
      sub.uvm = c->d_stage[b][1];
      sub.nrm = c->d_stage[b][2];
      sub.pos = c->d_stage[b][3];
      sub.mat = c->d_stage[b][4];
      sub.width = W;
      sub.height = nr;
      sub.pitch = W;
      sub.x0 = 0;
      sub.y0 = 0;
      Slots slot;
      const int rc = sched_slots(c, s, 1, &slot);
      if (rc) return rc;
      glint::KParams k;
      make_params(c, &sub, &scs[f], c->d_stage[b][5], W, nullptr, slot_at(c, slot, 0), &k);
      GL_CUDA(glint::launch_eval(k, grid_for(c, (int64_t)W * nr), false, s));
      c->launches++;
      GL_CUDA(cudaMemcpy2DAsync(out_tile + (int64_t)y0 * out_pitches[f], (size_t)out_pitches[f] * sizeof(float4),
                                c->d_stage[b][5], rowb, rowb, nr, cudaMemcpyDeviceToHost, s));
    }
  }
  return GLINT_OK;
}

// One continuous chunk stream over n frames: H2D of the next chunk (of this
// or the next frame) overlaps the kernel and D2H of the previous one, so the
// pipeline fills and drains once per call, not once per frame.
static int host_pipeline(glint_ctx* c, int n, const glint_gbuffer* gbs, const glint_scene* scs, void* const* outs,
                         const int64_t* out_pitches, void* stream) {
  // chunk size (pixels, at least 1 row): GLINT_HOST_CHUNK_PX if set at build
  // time, else 1M (80 MB in, 16 MB out) for calls under 8M pixels and 2M for
  // larger ones. Measured on C2: one 1080p frame per call reaches 96.5 % of the
  // pinned H2D bandwidth at 1M, and 256K / 128K chunks lose more to per-chunk
  // copies and launches (91 / 89 %) than they gain from a shorter fill and
  // drain; a 10-frame batch moves 50.1 GB/s at 1M, 50.7 at 2M and 4M, 48.5 at
  // 512K (the fill and drain are paid once per call)
  int64_t total_px = 0;
  for (int f = 0; f < n; ++f) total_px += (int64_t)gbs[f].width * gbs[f].height;
#ifdef GLINT_HOST_CHUNK_PX
  const int64_t chunk_px = GLINT_HOST_CHUNK_PX;
#else
  const int64_t chunk_px = total_px >= ((int64_t)8 << 20) ? ((int64_t)2 << 20) : ((int64_t)1 << 20);
#endif
  size_t stage_px = 0;
  for (int f = 0; f < n; ++f) {
    const glint_gbuffer& g = gbs[f];
    if (g.width == 0 || g.height == 0) continue;
    int rows = (int)(chunk_px / g.width);
    rows = rows < 1 ? 1 : (rows > g.height ? g.height : rows);
    const size_t px = (size_t)rows * g.width;
    stage_px = px > stage_px ? px : stage_px;
  }
  if (stage_px == 0) return GLINT_OK;
  int rc = ensure_stage(c, stage_px);
  if (rc) return rc;
  // from the first enqueue on, an error must not return while earlier chunks'
  // copies into the caller's host buffers are still in flight (the call is
  // synchronous): drain both internal streams, keep the first error
  try {
    rc = host_pipeline_enqueue(c, n, gbs, scs, outs, out_pitches, stream, chunk_px);
  } catch (...) {
    rc = GLINT_ENOMEM;
  }
  for (int b = 0; b < 2; ++b) {
    const cudaError_t e = cudaStreamSynchronize(c->st[b]);
    if (e != cudaSuccess && rc == GLINT_OK) {
      g_last_cuda = (int)e;
      rc = GLINT_ECUDA;
    }
  }
  return rc;
}

extern "C" int glint_eval_host(glint_ctx* c, const glint_gbuffer* gb, const glint_scene* sc, void* out_host,
                               int64_t out_pitch, void* stream) {
  if (!c) return GLINT_EINVAL;
  int rc = validate_scene(sc);
  if (rc) return rc;
  rc = validate_gbuffer(gb, out_pitch);
  if (rc) return rc;
  if (gb->width == 0 || gb->height == 0) return GLINT_OK;
  if (!out_host) return GLINT_EINVAL;
  int cur = -1;
  GL_CUDA(cudaGetDevice(&cur));
  if (cur != c->device) return GLINT_EDEVICE;
  std::lock_guard<std::mutex> lock(c->host_mu);
  void* outs[1] = {out_host};
  return host_pipeline(c, 1, gb, sc, outs, &out_pitch, stream);
}

extern "C" int glint_eval_host_batch(glint_ctx* c, int n_frames, const glint_gbuffer* gbs, const glint_scene* scenes,
                                     void* const* outs, const int64_t* out_pitches, void* stream) {
  if (!c || n_frames < 0) return GLINT_EINVAL;
  if (n_frames == 0) return GLINT_OK;
  if (!gbs || !scenes || !outs || !out_pitches) return GLINT_EINVAL;
  int rc = validate_batch(n_frames, gbs, scenes, outs, out_pitches);
  if (rc) return rc;
  int cur = -1;
  GL_CUDA(cudaGetDevice(&cur));
  if (cur != c->device) return GLINT_EDEVICE;
  std::lock_guard<std::mutex> lock(c->host_mu);
  return host_pipeline(c, n_frames, gbs, scenes, outs, out_pitches, stream);
}

// ---------------------------------------------------------------------------
// glint_count_active: the throughput metric's unit, counted on the device
// with the kernel's own decision functions
// ---------------------------------------------------------------------------
extern "C" int glint_count_active(const glint_ctx* c, const glint_gbuffer* gb, const glint_scene* sc,
                                  unsigned long long* d_count, void* stream) {
  if (!c || !d_count) return GLINT_EINVAL;
  int rc = validate_scene(sc);
  if (rc) return rc;
  rc = validate_gbuffer(gb, gb ? gb->width : 0);
  if (rc) return rc;
  if (gb->width == 0 || gb->height == 0) return GLINT_OK;
  int cur = -1;
  GL_CUDA(cudaGetDevice(&cur));
  if (cur != c->device) return GLINT_EDEVICE;
  const int64_t n_pix = (int64_t)gb->width * gb->height;
  int64_t grid = (n_pix + 255) / 256;
  const int64_t cap = (int64_t)c->sm_count * 8;
  grid = grid < cap ? grid : cap;
  GL_CUDA(glint::launch_count_active((const float4*)gb->duv, (const float4*)gb->uvm, (const float4*)gb->nrm,
                                     (const float4*)gb->pos, gb->width, gb->height, gb->pitch, *sc, d_count,
                                     (int)grid, (cudaStream_t)stream));
  return GLINT_OK;
}
