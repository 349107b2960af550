/* A plain C consumer of the C ABI (include/wmd.h): no Python, no torch.
 *
 *   abi_consumer          host-only entry points (any machine)
 *   abi_consumer gpu      plus one query on device 0, checked against a closed form
 *
 * The closed form (tests/test_oracle_pins.py P4): with a single query word the transport plan
 * is forced (all of each target word's mass goes to it), so for any lambda and any iteration
 * count WMD_j = sum_e c_ej * ||E[q] - E[k_e]||_2 (PAPER.md:66 with u, v at their fixed point).
 * Exit status 0 on success. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "wmd.h"

#define CHECK(cond, ...)                       \
  do {                                         \
    if (!(cond)) {                             \
      fprintf(stderr, "FAIL: " __VA_ARGS__);   \
      fprintf(stderr, "\n");                   \
      return 1;                                \
    }                                          \
  } while (0)

static int host_checks(void) {
  CHECK(wmd_version() && strlen(wmd_version()) > 0, "wmd_version");
  CHECK(strlen(wmd_status_string(WMD_ERR_EMPTY_DOCUMENT)) > 0, "wmd_status_string");
  /* nnz split of 4 documents with 1, 3, 2, 2 nonzeros over 2 parts: the boundary snaps to the
   * document holding nonzero ceil(8/2) = 4 -> bounds {0, 2, 4} */
  const int64_t col_ptr[5] = {0, 1, 4, 6, 8};
  int64_t bounds[3] = {-1, -1, -1};
  CHECK(wmd_partition(col_ptr, 4, 2, bounds) == WMD_OK, "wmd_partition status");
  CHECK(bounds[0] == 0 && bounds[1] == 2 && bounds[2] == 4, "wmd_partition bounds %lld %lld %lld",
        (long long)bounds[0], (long long)bounds[1], (long long)bounds[2]);
  const int32_t ids[2] = {3, 3};
  const float w[2] = {0.5f, 0.5f};
  int64_t bad = -1;
  CHECK(wmd_validate_query(ids, w, 2, 10, &bad) == WMD_ERR_BAD_WEIGHTS, "duplicate id not rejected");
  const int32_t ids2[1] = {11};
  const float w2[1] = {1.f};
  CHECK(wmd_validate_query(ids2, w2, 1, 10, &bad) == WMD_ERR_INDEX_OUT_OF_RANGE && bad == 0,
        "id >= V not rejected");
  return 0;
}

static int gpu_checks(void) {
  enum { V = 64, D = 8, N = 3 };
  float E[V * D];
  unsigned s = 12345u;
  for (int i = 0; i < V * D; ++i) {  /* deterministic values in [-1, 1) */
    s = s * 1664525u + 1013904223u;
    E[i] = (float)((s >> 8) & 0xFFFF) / 32768.f - 1.f;
  }
  /* three target documents (CSC over the vocabulary, rows ascending), weights summing to 1 */
  const int64_t col_ptr[N + 1] = {0, 2, 5, 6};
  const int32_t row_idx[6] = {1, 7, 3, 10, 42, 5};
  const float val[6] = {0.25f, 0.75f, 0.5f, 0.25f, 0.25f, 1.f};
  wmd_handle* h = NULL;
  wmd_status st = wmd_create(E, V, D, 0, &h);
  CHECK(st == WMD_OK, "wmd_create: %s", wmd_status_string(st));
  st = wmd_set_targets(h, col_ptr, row_idx, val, N, 6);
  CHECK(st == WMD_OK, "wmd_set_targets: %s (%s)", wmd_status_string(st), wmd_last_error(h));
  const int32_t q[1] = {20};
  const float qw[1] = {1.f};
  float dist[N];
  st = wmd_query(h, q, qw, 1, 10.f, 7, dist);
  CHECK(st == WMD_OK, "wmd_query: %s (%s)", wmd_status_string(st), wmd_last_error(h));
  st = wmd_sync(h);
  CHECK(st == WMD_OK, "wmd_sync: %s", wmd_status_string(st));
  for (int j = 0; j < N; ++j) {
    double ref = 0.0;
    for (int64_t e = col_ptr[j]; e < col_ptr[j + 1]; ++e) {
      double m2 = 0.0;
      for (int t = 0; t < D; ++t) {
        const double x = (double)E[q[0] * D + t] - (double)E[row_idx[e] * D + t];
        m2 += x * x;
      }
      ref += (double)val[e] * sqrt(m2);
    }
    CHECK(fabs(dist[j] - ref) <= 1e-4 * fabs(ref) + 1e-5, "doc %d: gpu %.7g vs closed form %.7g", j,
          (double)dist[j], ref);
  }
  wmd_destroy(h);
  printf("abi_consumer gpu ok: %g %g %g\n", (double)dist[0], (double)dist[1], (double)dist[2]);
  return 0;
}

int main(int argc, char** argv) {
  if (host_checks()) return 1;
  printf("abi_consumer host ok (%s)\n", wmd_version());
  if (argc > 1 && strcmp(argv[1], "gpu") == 0) return gpu_checks();
  return 0;
}
