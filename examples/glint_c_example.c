/*
 * glint_c_example.c -- the C ABI used from plain C (no Python, no torch).
 *
 * Builds a 64x64 G-buffer of a flat quad (the C1 layout of BASELINE.json:
 * uv = pixel/64, duv/dx = (1/64, 0), duv/dy = (0, 1/64), normal +z, isotropic
 * GGX roughness 0.3, 1e5 flakes per unit uv^2, R = 0.034), one directional
 * light in the mirror configuration, uploads it with the CUDA runtime, calls
 * glint_eval, and prints the number of glinting pixels and a checksum of the
 * radiance. Also runs the host-buffer entry glint_eval_host and checks that
 * both entries return the same bits, and shades two frames (the same quad
 * under two seeds) with one glint_eval_batch call: frame 0 must equal the
 * single glint_eval bit for bit, and an output aliasing an input is refused.
 *
 * Build: gcc -O2 -I include examples/glint_c_example.c \
 *          -L paper_2306_05051_b200 -lglint -L /usr/local/cuda/lib64 -lcudart \
 *          -Wl,-rpath,$PWD/paper_2306_05051_b200 -o glint_c_example
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "glint.h"

#define W 64
#define H 64

static float bits_f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

#define CHECK(call)                                                                  \
  do {                                                                               \
    int rc_ = (call);                                                                \
    if (rc_) { fprintf(stderr, "%s failed: %s\n", #call, glint_strerror(rc_)); return 1; } \
  } while (0)

int main(void) {
  const size_t n = (size_t)W * H;
  float* host[5];
  for (int p = 0; p < 5; ++p) host[p] = (float*)calloc(4 * n, sizeof(float));
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      size_t i = 4 * ((size_t)y * W + x);
      host[0][i + 0] = 1.0f / 64; host[0][i + 3] = 1.0f / 64;             /* duv */
      host[1][i + 0] = x / 64.0f; host[1][i + 1] = y / 64.0f;             /* uvm */
      host[1][i + 2] = bits_f(0u); host[1][i + 3] = bits_f(1u);            /* obj 0, valid */
      host[2][i + 2] = 1.0f;                                               /* nrm */
      host[4][i + 0] = 0.3f; host[4][i + 1] = 0.3f;                        /* mat */
      host[4][i + 2] = 1e5f; host[4][i + 3] = 0.034f;
    }

  glint_ctx* ctx = NULL;
  CHECK(glint_create(&ctx, 0));
  void* dev[5];
  for (int p = 0; p < 5; ++p) {
    if (cudaMalloc(&dev[p], 16 * n) != cudaSuccess) return 1;
    cudaMemcpy(dev[p], host[p], 16 * n, cudaMemcpyHostToDevice);
  }
  void* dout;
  if (cudaMalloc(&dout, 16 * n) != cudaSuccess) return 1;

  glint_gbuffer gb;
  memset(&gb, 0, sizeof gb);
  gb.duv = dev[0]; gb.uvm = dev[1]; gb.nrm = dev[2]; gb.pos = dev[3]; gb.mat = dev[4];
  gb.width = W; gb.height = H; gb.pitch = W;

  glint_scene sc;
  memset(&sc, 0, sizeof sc);
  const float s30 = 0.5f, c30 = 0.8660254f;
  sc.seed = 1; sc.ndf_kind = 0; sc.max_ratio_level = 8; sc.beta = 0.05f;
  sc.f0[0] = sc.f0[1] = sc.f0[2] = 0.9f;
  sc.view_kind = 1; sc.view[0] = s30; sc.view[2] = c30;
  sc.n_lights = 1; sc.eval_mode = 0;
  sc.lights[0].kind = 1;
  sc.lights[0].pos_or_dir[0] = -s30; sc.lights[0].pos_or_dir[2] = c30;
  sc.lights[0].intensity[0] = sc.lights[0].intensity[1] = sc.lights[0].intensity[2] = 1.0f;

  CHECK(glint_eval(ctx, &gb, &sc, dout, W, NULL, NULL));
  float* out = (float*)malloc(16 * n);
  if (cudaMemcpy(out, dout, 16 * n, cudaMemcpyDeviceToHost) != cudaSuccess) return 1;

  /* the host-buffer entry on the same inputs */
  glint_gbuffer gh = gb;
  gh.duv = host[0]; gh.uvm = host[1]; gh.nrm = host[2]; gh.pos = host[3]; gh.mat = host[4];
  float* out_h = (float*)malloc(16 * n);
  CHECK(glint_eval_host(ctx, &gh, &sc, out_h, W, NULL));

  /* two independent frames in one call (launches chained on the GPU) */
  void* dout2;
  if (cudaMalloc(&dout2, 16 * n) != cudaSuccess) return 1;
  glint_gbuffer gbs[2] = {gb, gb};
  glint_scene scs[2] = {sc, sc};
  scs[1].seed = 2;
  void* outs[2] = {dout, dout2};
  int64_t pitches[2] = {W, W};
  CHECK(glint_eval_batch(ctx, 2, gbs, scs, outs, pitches, NULL));
  float* out_b = (float*)malloc(16 * n);
  if (cudaMemcpy(out_b, dout, 16 * n, cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
  int batch_same = memcmp(out, out_b, 16 * n) == 0;
  void* bad_outs[2] = {dout, dev[4]};   /* frame 1 would overwrite the material plane */
  int alias_rc = glint_eval_batch(ctx, 2, gbs, scs, bad_outs, pitches, NULL);
  cudaFree(dout2);
  free(out_b);

  /* the same frame as two row bands (a sharded frame): each band's
     planes start at its first row, its tile origin (x0, y0) places it in one
     full-frame output; the assembled frame equals the whole-frame launch */
  void* dband;
  if (cudaMalloc(&dband, 16 * n) != cudaSuccess) return 1;
  const int H0 = 24;
  glint_gbuffer bands[2] = {gb, gb};
  bands[0].height = H0;
  bands[1].height = H - H0;
  bands[1].y0 = H0;
  bands[1].duv = (const char*)gb.duv + 16 * (size_t)H0 * W;
  bands[1].uvm = (const char*)gb.uvm + 16 * (size_t)H0 * W;
  bands[1].nrm = (const char*)gb.nrm + 16 * (size_t)H0 * W;
  bands[1].pos = (const char*)gb.pos + 16 * (size_t)H0 * W;
  bands[1].mat = (const char*)gb.mat + 16 * (size_t)H0 * W;
  glint_scene bsc[2] = {sc, sc};
  void* bouts[2] = {dband, dband};
  CHECK(glint_eval_batch(ctx, 2, bands, bsc, bouts, pitches, NULL));
  float* out_bands = (float*)malloc(16 * n);
  if (cudaMemcpy(out_bands, dband, 16 * n, cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
  int bands_same = memcmp(out, out_bands, 16 * n) == 0;
  cudaFree(dband);
  free(out_bands);

  /* the metric's unit: active (pixel, light) pairs */
  unsigned long long* dcount;
  unsigned long long active = 0;
  if (cudaMalloc((void**)&dcount, sizeof *dcount) != cudaSuccess) return 1;
  cudaMemset(dcount, 0, sizeof *dcount);
  CHECK(glint_count_active(ctx, &gb, &sc, dcount, NULL));
  if (cudaMemcpy(&active, dcount, sizeof active, cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
  cudaFree(dcount);

  int glints = 0;
  double sum = 0.0;
  for (size_t i = 0; i < n; ++i) {
    if (out[4 * i] > 0.0f) ++glints;
    sum += out[4 * i] + out[4 * i + 1] + out[4 * i + 2];
  }
  int same = memcmp(out, out_h, 16 * n) == 0;
  printf("glinting pixels %d of %zu, radiance sum %.9g, host entry identical %d, batch identical %d, "
         "aliased batch refused %d, bands identical %d, active pairs %llu, launches %lld\n", glints, n, sum, same,
         batch_same, alias_rc == GLINT_EALIAS, bands_same, active, (long long)glint_launch_count(ctx));
  CHECK(glint_destroy(ctx));
  for (int p = 0; p < 5; ++p) { cudaFree(dev[p]); free(host[p]); }
  cudaFree(dout);
  free(out);
  free(out_h);
  return (glints > 0 && same && batch_same && alias_rc == GLINT_EALIAS && bands_same && active == n) ? 0 : 2;
}
