/* A plain-C host of the C ABI (include/mgwfbp.h) — what a non-Python
 * framework binds: plan a 3-layer model with the
 * reference solver, run one fused all-reduce + SGD per group on one GPU
 * (P = 1: the update is w -= lr * g), and check the result on the host.
 *
 *   build: see tests/test_c_example.py (gcc -Iinclude ... -lmgwfbp -lcudart)
 *   run:   ./mgw_c_host   (needs a GPU; exit 0 = bit-exact)
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "mgwfbp.h"

#define CHECK(x)                                                                 \
  do {                                                                           \
    int rc_ = (x);                                                               \
    if (rc_ != 0) {                                                              \
      fprintf(stderr, "%s failed (%d): %s\n", #x, rc_, mgw_last_error());        \
      return 1;                                                                  \
    }                                                                            \
  } while (0)

int main(void) {
  enum { L = 3 };
  const uint64_t counts[L] = {1000, 4096, 77};
  const double t_b[L] = {2e-4, 1e-4, 5e-5};
  uint8_t tags[L];
  /* the reference's optimal_plan (planner.hpp:63-98) with a + b*M */
  CHECK(mgw_plan_optimal(counts, t_b, L, 1e-3, 4, 2e-5, 1e-9, tags));

  float* h_g[L];
  float* h_w[L];
  float* d_g[L];
  float* d_w[L];
  for (int l = 0; l < L; ++l) {
    h_g[l] = (float*)malloc(counts[l] * sizeof(float));
    h_w[l] = (float*)malloc(counts[l] * sizeof(float));
    for (uint64_t i = 0; i < counts[l]; ++i) {
      h_g[l][i] = (float)((i * 37 + l) % 101) / 50.0f - 1.0f;
      h_w[l][i] = (float)((i * 11 + 3 * l) % 97) / 97.0f;
    }
    if (cudaMalloc((void**)&d_g[l], counts[l] * sizeof(float)) != cudaSuccess ||
        cudaMalloc((void**)&d_w[l], counts[l] * sizeof(float)) != cudaSuccess) {
      fprintf(stderr, "cudaMalloc failed\n");
      return 1;
    }
    cudaMemcpy(d_g[l], h_g[l], counts[l] * sizeof(float), cudaMemcpyHostToDevice);
    cudaMemcpy(d_w[l], h_w[l], counts[l] * sizeof(float), cudaMemcpyHostToDevice);
  }
  mgw_comm* comm = NULL;
  mgw_plan* plan = NULL;
  CHECK(mgw_comm_create(0, 1, 0, 1 << 20, &comm));
  CHECK(mgw_plan_create(comm, L, d_g, d_w, counts, tags, &plan));
  int G = 0;
  CHECK(mgw_plan_num_groups(plan, &G));
  const float lr = 0.125f;
  for (int g = G - 1; g >= 0; --g) {  /* backward order */
    CHECK(mgw_group_allreduce(plan, g, lr, MGW_SGD, MGW_ALGO_AUTO, NULL));
  }
  if (cudaDeviceSynchronize() != cudaSuccess) return 1;
  int bad = 0;
  for (int l = 0; l < L; ++l) {
    float* w = (float*)malloc(counts[l] * sizeof(float));
    cudaMemcpy(w, d_w[l], counts[l] * sizeof(float), cudaMemcpyDeviceToHost);
    for (uint64_t i = 0; i < counts[l]; ++i) {
      const volatile float step = lr * h_g[l][i]; /* two roundings, like the kernel */
      const float want = h_w[l][i] - step;
      if (w[i] != want) ++bad;
    }
    free(w);
  }
  CHECK(mgw_plan_destroy(plan));
  CHECK(mgw_comm_destroy(comm));
  printf("groups=%d mismatches=%d (%s)\n", G, bad, mgw_version());
  return bad == 0 ? 0 : 2;
}
