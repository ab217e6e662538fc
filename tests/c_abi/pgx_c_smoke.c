/* pgx_c_smoke.c -- the C ABI used from plain C (no Python, no torch).
 *
 *   host : ABI version, workspace size queries, error codes and messages
 *   gpu  : a complete connected_components run (algorithms.py:87-113) on
 *          a 6-vertex graph through pgx_offsets_to_i32 / pgx_graph_prepare /
 *          pgx_cc_run with cudaMalloc'd buffers; prints the labels and the
 *          superstep statistics for the test to compare with the oracle.
 *
 * Built by tests/test_c_abi.py with gcc against include/pgx.h and libpgx.so.
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "pgx.h"

#ifdef PGX_SMOKE_GPU
#include <cuda_runtime_api.h>
#define CK(x)                                                          \
  do {                                                                 \
    int rc_ = (int)(x);                                                \
    if (rc_ != 0) {                                                    \
      fprintf(stderr, "%s failed: %d (%s)\n", #x, rc_, pgx_last_error()); \
      return 1;                                                        \
    }                                                                  \
  } while (0)
#endif

static int host_checks(void) {
  size_t b = 0;
  if (pgx_abi_version() != PGX_ABI_VERSION) return 10;
  if (pgx_graph_workspace_bytes(1000, 5000, &b) != PGX_OK || b < 1000 * 4) return 11;
  if (pgx_run_workspace_bytes(PGX_APP_CC, 1000, 5000, 16, &b) != PGX_OK || b < 1000 * 4)
    return 12;
  if (pgx_run_workspace_bytes(7, 10, 10, 1, &b) != PGX_EINVAL) return 13;
  if (strstr(pgx_last_error(), "bad run workspace") == NULL) return 14;
  if (pgx_set_option(99, 1) != PGX_EINVAL) return 15;
  printf("host ok abi=%d\n", pgx_abi_version());
  return 0;
}

#ifdef PGX_SMOKE_GPU
static int gpu_run(void) {
  /* two triangles 0-1-2 and 3-4-5, stored in both directions, rows sorted */
  const int32_t n = 6;
  const int64_t m = 12;
  const int64_t off[7] = {0, 2, 4, 6, 8, 10, 12};
  const int32_t tgt[12] = {1, 2, 0, 2, 0, 1, 4, 5, 3, 5, 3, 4};
  const int32_t max_steps = 64;
  int64_t *d_off;
  int32_t *d_row, *d_col;
  uint32_t *d_lab;
  int64_t *d_stats;
  void *gws, *rws;
  size_t gb = 0, rb = 0;
  CK(cudaMalloc((void **)&d_off, sizeof off));
  CK(cudaMalloc((void **)&d_row, sizeof(int32_t) * (n + 1)));
  CK(cudaMalloc((void **)&d_col, sizeof tgt));
  CK(cudaMalloc((void **)&d_lab, sizeof(uint32_t) * n));
  CK(cudaMalloc((void **)&d_stats, sizeof(int64_t) * (PGX_STAT_HDR + PGX_STAT_FIELDS * max_steps)));
  CK(cudaMemcpy(d_off, off, sizeof off, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_col, tgt, sizeof tgt, cudaMemcpyHostToDevice));
  CK(pgx_offsets_to_i32(d_off, d_row, n + 1, 0));
  CK(pgx_graph_workspace_bytes(n, m, &gb));
  CK(cudaMalloc(&gws, gb));
  CK(pgx_graph_prepare(n, m, d_row, gws, gb, 0));
  CK(pgx_run_workspace_bytes(PGX_APP_CC, n, m, max_steps, &rb));
  CK(cudaMalloc(&rws, rb));
  CK(pgx_cc_run(n, m, d_row, d_col, gws, NULL, 0, max_steps, d_lab, rws, rb, d_stats, 0));
  CK(cudaDeviceSynchronize());
  uint32_t lab[6];
  int64_t st[PGX_STAT_HDR + PGX_STAT_FIELDS * 64];
  CK(cudaMemcpy(lab, d_lab, sizeof lab, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(st, d_stats, sizeof st, cudaMemcpyDeviceToHost));
  printf("labels");
  for (int v = 0; v < n; v++) printf(" %u", lab[v]);
  printf("\nsteps %lld cap %lld\nactive", (long long)st[0], (long long)st[1]);
  for (int s = 0; s < st[0]; s++) printf(" %lld", (long long)st[PGX_STAT_HDR + s * PGX_STAT_FIELDS]);
  printf("\nsent");
  for (int s = 0; s < st[0]; s++)
    printf(" %lld", (long long)st[PGX_STAT_HDR + s * PGX_STAT_FIELDS + 1]);
  printf("\n");
  /* a bad source is an EINVAL with a message, not a crash */
  if (pgx_sssp_run(n, m, d_row, d_col, gws, NULL, 0, 99, max_steps, d_lab, rws, rb, d_stats, 0) !=
      PGX_EINVAL)
    return 20;
  cudaFree(d_off); cudaFree(d_row); cudaFree(d_col); cudaFree(d_lab); cudaFree(d_stats);
  cudaFree(gws); cudaFree(rws);
  return 0;
}
#endif

int main(int argc, char **argv) {
  int rc = host_checks();
  if (rc) {
    fprintf(stderr, "host check %d failed: %s\n", rc, pgx_last_error());
    return rc;
  }
#ifdef PGX_SMOKE_GPU
  if (argc > 1 && strcmp(argv[1], "gpu") == 0) return gpu_run();
#endif
  (void)argc;
  (void)argv;
  return 0;
}
