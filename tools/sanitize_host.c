/* Plain-C driver for compute-sanitizer (memcheck / racecheck / synccheck /
 * initcheck): the fused kernels on a loopback communicator of P emulated
 * ranks — standalone group launches (one-shot, two-shot, LL) and the
 * persistent engine in standalone drain mode (every group ready, so no
 * concurrent replay kernel is needed under the sanitizer's serialisation) —
 * with a bit-exact host check of the rank-order result. No Python / torch
 * under the sanitizer.
 *
 *   build: tools/sanitize.sh (gcc -Iinclude ... -lmgwfbp -lcudart)
 *   run:   compute-sanitizer --tool T --error-exitcode 9 ./sanitize_host P
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "mgwfbp.h"

#define CHECK(x)                                                          \
  do {                                                                    \
    int rc_ = (x);                                                        \
    if (rc_ != 0) {                                                       \
      fprintf(stderr, "%s failed (%d): %s\n", #x, rc_, mgw_last_error()); \
      exit(1);                                                            \
    }                                                                     \
  } while (0)

enum { L = 9, MAXP = 8 };
static const uint64_t kCounts[L] = {1000, 0, 7, 9000, 4096, 13, 70000, 3, 20000};

static float lcg(uint32_t* s) {
  *s = *s * 1664525u + 1013904223u;
  return (float)(*s >> 8) / 8388608.0f - 1.0f;
}

/* one SGD step of the rank-order mean (x 1/P per source, two roundings) */
static void host_step(int P, float* g[MAXP][L], float* w[MAXP][L], float lr) {
  const float s = 1.0f / (float)P;
  for (int l = 0; l < L; ++l) {
    for (uint64_t i = 0; i < kCounts[l]; ++i) {
      volatile float acc = g[0][l][i] * s;
      for (int r = 1; r < P; ++r) {
        volatile float t = g[r][l][i] * s;
        acc = acc + t;
      }
      for (int r = 0; r < P; ++r) {
        volatile float step = lr * acc;
        w[r][l][i] = w[r][l][i] - step;
      }
    }
  }
}

int main(int argc, char** argv) {
  const int P = argc > 1 ? atoi(argv[1]) : 2;
  const float lr = 0.01f;
  float* hg[MAXP][L];
  float* hw[MAXP][L];
  void* dg[MAXP * L];
  float* dw[MAXP * L];
  uint32_t seed = 12345u;
  for (int r = 0; r < P; ++r) {
    for (int l = 0; l < L; ++l) {
      const size_t n = kCounts[l] ? kCounts[l] : 1;
      hg[r][l] = (float*)malloc(n * sizeof(float));
      hw[r][l] = (float*)malloc(n * sizeof(float));
      for (uint64_t i = 0; i < kCounts[l]; ++i) {
        hg[r][l][i] = lcg(&seed);
        hw[r][l][i] = lcg(&seed);
      }
      if (cudaMalloc(&dg[r * L + l], n * sizeof(float)) != cudaSuccess ||
          cudaMalloc((void**)&dw[r * L + l], n * sizeof(float)) != cudaSuccess) {
        fprintf(stderr, "cudaMalloc failed\n");
        return 1;
      }
      cudaMemcpy(dg[r * L + l], hg[r][l], n * sizeof(float), cudaMemcpyHostToDevice);
      cudaMemcpy(dw[r * L + l], hw[r][l], n * sizeof(float), cudaMemcpyHostToDevice);
    }
  }
  const double t_b[L] = {1e-5, 1e-5, 1e-5, 1e-5, 1e-5, 1e-5, 1e-5, 1e-5, 1e-5};
  const uint8_t tags[L] = {0, 1, 0, 1, 0, 0, 1, 0, 0};
  mgw_comm* comm = NULL;
  mgw_plan* plan = NULL;
  if (P == 1) {
    CHECK(mgw_comm_create(0, 1, 0, 1 << 20, &comm));
  } else {
    CHECK(mgw_comm_create_loopback(P, 0, 1 << 20, &comm));
    CHECK(mgw_comm_set_oneshot_max(comm, 32 << 10)); /* groups of 1..5 tiles: LL, one-shot, two-shot */
    CHECK(mgw_comm_set_ll_max(comm, 8 << 10));
  }
  CHECK(mgw_plan_create_ex(comm, L, dg, dw, kCounts, tags, MGW_DTYPE_F32, &plan));
  int G = 0;
  CHECK(mgw_plan_num_groups(plan, &G));
  int steps = 0;
  const int algos[3] = {MGW_ALGO_ONESHOT, MGW_ALGO_TWOSHOT, MGW_ALGO_AUTO};
  for (int a = 0; a < (P > 1 ? 3 : 1); ++a) {
    for (int g = G - 1; g >= 0; --g) CHECK(mgw_group_allreduce(plan, g, lr, MGW_SGD, algos[a], NULL));
    ++steps;
  }
  mgw_pipeline* pipe = NULL;
  CHECK(mgw_pipeline_create(plan, t_b, 1e-5, lr, MGW_ALGO_AUTO, 1, 0, -1, &pipe));
  float ms[2];
  CHECK(mgw_pipeline_drain(pipe, 2, ms));
  steps += 2;
  if (cudaDeviceSynchronize() != cudaSuccess) {
    fprintf(stderr, "sync failed\n");
    return 1;
  }
  int failed = 0;
  CHECK(mgw_comm_error(comm, &failed));
  for (int k = 0; k < steps; ++k) host_step(P, hg, hw, lr);
  long bad = 0;
  for (int r = 0; r < P; ++r) {
    for (int l = 0; l < L; ++l) {
      const size_t n = kCounts[l] ? kCounts[l] : 1;
      float* w = (float*)malloc(n * sizeof(float));
      cudaMemcpy(w, dw[r * L + l], n * sizeof(float), cudaMemcpyDeviceToHost);
      for (uint64_t i = 0; i < kCounts[l]; ++i) bad += w[i] != hw[r][l][i];
      free(w);
    }
  }
  CHECK(mgw_pipeline_destroy(pipe));
  CHECK(mgw_plan_destroy(plan));
  CHECK(mgw_comm_destroy(comm));
  printf("P=%d groups=%d steps=%d mismatches=%ld comm_failed=%d\n", P, G, steps, bad, failed);
  return (bad == 0 && failed == 0) ? 0 : 2;
}
