/* oracle_asan_main.c -- test driver (tests/test_oracle_sanitizers.py): runs
 * the CPU oracle under AddressSanitizer + UndefinedBehaviorSanitizer on input
 * planes read from a file, writes rgb / flags / records back, so the test can
 * compare them with the uninstrumented build bit for bit.
 * file in : int64 n, orc_scene, 5 x n x 4 floats (duv, uvm, nrm, pos, mat)
 * file out: n x 3 doubles, n uint32 flags, n x n_lights orc_rec */
#include <stdio.h>
#include <stdlib.h>

#include "../oracle/glint_oracle.h"

int main(int argc, char** argv) {
  if (argc != 3) return 2;
  FILE* f = fopen(argv[1], "rb");
  if (!f) return 3;
  int64_t n = 0;
  orc_scene sc;
  if (fread(&n, sizeof n, 1, f) != 1 || fread(&sc, sizeof sc, 1, f) != 1) return 4;
  float* planes[5];
  for (int p = 0; p < 5; ++p) {
    planes[p] = (float*)malloc(sizeof(float) * 4 * (size_t)(n ? n : 1));
    if (fread(planes[p], sizeof(float) * 4, (size_t)n, f) != (size_t)n) return 5;
  }
  fclose(f);
  double* rgb = (double*)malloc(sizeof(double) * 3 * (size_t)(n ? n : 1));
  uint32_t* flags = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(n ? n : 1));
  size_t nrec = (size_t)n * (size_t)(sc.n_lights > 0 ? sc.n_lights : 0);
  orc_rec* rec = sc.eval_mode == 0 ? (orc_rec*)malloc(sizeof(orc_rec) * (nrec ? nrec : 1)) : NULL;
  int rc = orc_eval(planes[0], planes[1], planes[2], planes[3], planes[4], n, &sc, rgb, flags, rec);
  if (rc) return 6;
  FILE* o = fopen(argv[2], "wb");
  fwrite(rgb, sizeof(double) * 3, (size_t)n, o);
  fwrite(flags, sizeof(uint32_t), (size_t)n, o);
  if (rec) fwrite(rec, sizeof(orc_rec), nrec, o);
  fclose(o);
  for (int p = 0; p < 5; ++p) free(planes[p]);
  free(rgb);
  free(flags);
  free(rec);
  return 0;
}
