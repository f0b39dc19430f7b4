/* c_api_demo.c — the GRASS hot path driven from plain C99 through
 * include/grass.h (no C++, no Python, no torch).  Checks closed forms:
 *   - Eq. 2 on g = [3, 4]: r = sqrt(25 / 2);
 *   - one AdamW step with g = 1, lr = 0.1, theta = 0: theta' = -0.1 / (1 + 1e-8)
 *     (bias correction cancels at t = 1);
 *   - gamma = N_L sampling returns every layer once;
 *   - the P2P data-parallel path (world 1) gives the same AdamW step, and the
 *     P2P barrier self-test reports no mismatch.
 * Exit code 0 on success.  Build: see tests/test_c_api.py. */
#include <cuda_runtime_api.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "grass.h"

#define CHECK(x)                                                                    \
  do {                                                                              \
    grass_status s_ = (x);                                                          \
    if (s_ != GRASS_OK) {                                                           \
      fprintf(stderr, "%s failed: %d %s\n", #x, (int)s_, grass_last_error(ctx));     \
      return 1;                                                                     \
    }                                                                               \
  } while (0)

int main(void) {
  grass_ctx* ctx = NULL;
  const int64_t numel[2] = {2, 4096};
  grass_config cfg;
  if (grass_config_init(&cfg) != GRASS_OK) return 1;
  cfg.n_layers = 2;
  cfg.layer_numel = numel;
  cfg.gamma = 2;
  CHECK(grass_create(&cfg, &ctx));

  float *g0, *g1, *p1;
  if (cudaMalloc((void**)&g0, 2 * sizeof(float)) || cudaMalloc((void**)&g1, 4096 * sizeof(float)) ||
      cudaMalloc((void**)&p1, 4096 * sizeof(float)))
    return 1;
  const float h0[2] = {3.0f, 4.0f};
  float* h1 = (float*)malloc(4096 * sizeof(float));
  for (int i = 0; i < 4096; ++i) h1[i] = 1.0f;
  cudaMemcpy(g0, h0, sizeof(h0), cudaMemcpyHostToDevice);
  cudaMemcpy(g1, h1, 4096 * sizeof(float), cudaMemcpyHostToDevice);
  cudaMemset(p1, 0, 4096 * sizeof(float));

  /* probing: Eq. 2 norms of both layers */
  const int32_t all[2] = {0, 1};
  const float* grads[2] = {g0, g1};
  CHECK(grass_mgn_accumulate(ctx, all, 2, grads, NULL));
  double S[2], probs[2];
  int64_t c[2];
  CHECK(grass_get_mgn(ctx, NULL, S, c, NULL, NULL));
  if (c[0] != 1 || fabs(S[0] - sqrt(12.5)) > 0.0 || S[1] != 1.0) {
    fprintf(stderr, "norms: %.17g %.17g\n", S[0], S[1]);
    return 2;
  }
  CHECK(grass_update_probs(ctx, probs));
  if (fabs(probs[0] + probs[1] - 1.0) > 1e-12) return 3;

  int32_t ids[2];
  CHECK(grass_sample_layers(ctx, NULL, 0, ids));
  if (!((ids[0] == 0 && ids[1] == 1) || (ids[0] == 1 && ids[1] == 0))) return 4;

  /* one AdamW step of layer 1 */
  const int32_t one[1] = {1};
  float* params[1] = {p1};
  const float* g[1] = {g1};
  CHECK(grass_step_layers(ctx, one, 1, params, g, 0.1f, NULL));
  CHECK(grass_sync(ctx));
  cudaMemcpy(h1, p1, 4096 * sizeof(float), cudaMemcpyDeviceToHost);
  const double want = -0.1 / (1.0 + 1e-8);
  for (int i = 0; i < 4096; ++i)
    if (fabs(h1[i] - want) > 1e-5 * fabs(want)) {
      fprintf(stderr, "theta[%d] = %.9g want %.9g\n", i, h1[i], want);
      return 5;
    }
  int64_t t = 0;
  CHECK(grass_read_state(ctx, 1, NULL, NULL, &t));
  if (t != 1) return 6;

  grass_destroy(ctx);

  /* P2P data parallelism at world 1: register the buffers, one step */
  grass_config pc;
  if (grass_config_init(&pc) != GRASS_OK) return 7;
  pc.n_layers = 2;
  pc.layer_numel = numel;
  pc.gamma = 2;
  pc.dp_mode = GRASS_DP_P2P;
  CHECK(grass_create(&pc, &ctx));
  void* blk = NULL;
  int64_t blk_bytes = 0;
  CHECK(grass_p2p_exchange_block(ctx, &blk, &blk_bytes));
  CHECK(grass_p2p_attach(ctx, &blk));
  cudaMemset(p1, 0, 4096 * sizeof(float));
  void* pp[1] = {p1};
  const void* gg[1] = {g1};
  CHECK(grass_p2p_register_layer(ctx, 1, pp, gg));
  CHECK(grass_step_layers(ctx, one, 1, params, g, 0.1f, NULL));
  CHECK(grass_sync(ctx));
  cudaMemcpy(h1, p1, 4096 * sizeof(float), cudaMemcpyDeviceToHost);
  for (int i = 0; i < 4096; ++i)
    if (fabs(h1[i] - want) > 1e-5 * fabs(want)) return 8;
  grass_destroy(ctx);
  ctx = NULL;
  int64_t mismatches = -1;
  int32_t timed_out = -1;
  CHECK(grass_selftest_p2p(0, 4, 200, &mismatches, &timed_out));
  if (mismatches != 0 || timed_out != 0) return 9;

  cudaFree(g0);
  cudaFree(g1);
  cudaFree(p1);
  free(h1);
  printf("c api demo ok\n");
  return 0;
}
