/* A C caller of the drop-in boundary: the whole unwrap through pu_unwrap
 * (include/pu_unwrap.h), no Python involved.
 *
 *   gcc -O2 -I include examples/unwrap_demo.c -L paper_2401_09961_b200/_lib \
 *       -Wl,-rpath,$PWD/paper_2401_09961_b200/_lib -lpu_unwrap -lm -o unwrap_demo
 *   ./unwrap_demo in.f64 n m out.f64 [fp32]
 *
 * in.f64: n*m raw little-endian doubles (wrapped phase in [0, 2pi));
 * out.f64: the unwrapped u (n*m doubles).  Prints one line per IRLS
 * iteration (the reference's trace fields, cli.py:158-173) and exits with the
 * reference CLI's codes: 0 ok, 2 bad input, 4 numerical breakdown. */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "pu_unwrap.h"

int main(int argc, char** argv) {
  if (argc < 5) {
    fprintf(stderr, "usage: %s in.f64 n m out.f64 [fp32]\n", argv[0]);
    return 2;
  }
  const int n = atoi(argv[2]), m = atoi(argv[3]);
  const int dtype = (argc > 5 && strcmp(argv[5], "fp32") == 0) ? PU_F32 : PU_F64;
  if (n < 1 || m < 1) return 2;
  double* x = malloc(sizeof(double) * (size_t)n * m);
  double* u = malloc(sizeof(double) * (size_t)n * m);
  double* vv = malloc(sizeof(double) * (size_t)(n > 1 ? n - 1 : 1) * m);
  double* vh = malloc(sizeof(double) * (size_t)n * (m > 1 ? m - 1 : 1));
  FILE* f = fopen(argv[1], "rb");
  if (!f || fread(x, sizeof(double), (size_t)n * m, f) != (size_t)n * m) {
    fprintf(stderr, "error: cannot read %s\n", argv[1]);
    return 2;
  }
  fclose(f);
  pu_irls_params p;
  pu_irls_params_default(&p);
  pu_iteration_record trace[128];
  int len = 0, brk = -1;
  const int rc = pu_unwrap(x, n, m, NULL, NULL, 1e-2, 1e-6, &p, -3.141592653589793, dtype, 0, u, vv, vh, trace, 128,
                           &len, &brk);
  if (rc != PU_OK) {
    fprintf(stderr, "error: %s\n", pu_last_error());
    return rc == PU_ERR_BREAKDOWN ? 4 : (rc == PU_ERR_ARG ? 2 : 1);
  }
  for (int i = 0; i < len && i < 128; ++i)
    printf("{\"k\": %d, \"m_cg\": %d, \"h_delta\": %.17g, \"cg_iters\": %d, \"fallback\": %s}\n", trace[i].k,
           trace[i].m_cg, trace[i].h_delta, trace[i].cg_iters, trace[i].fallback_used ? "true" : "false");
  f = fopen(argv[4], "wb");
  if (!f || fwrite(u, sizeof(double), (size_t)n * m, f) != (size_t)n * m) return 1;
  fclose(f);
  free(x); free(u); free(vv); free(vh);
  return 0;
}
