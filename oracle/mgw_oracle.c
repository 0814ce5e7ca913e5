/*
 * mgw_oracle.c — CPU restatement of the MG-WFBP path. TEST INFRASTRUCTURE
 * ONLY (see mgw_oracle.h for who may load it). Compiled with -O2
 * -ffp-contract=off (no FMA), matching the reference's x86-64 Release build
 * (proj/CMakeLists.txt:6-8, no -march) so double arithmetic rounds the same.
 *
 * Each function is a deliberately literal restatement of the reference
 * (O(L^2) DP with no pruning, greedy with full tau_c recomputation) so it
 * checks the optimised product code through a different path.
 *
 * Pinning: the solver / predictor / fit restatements are pinned to the
 * reference itself (oracle/_ref, built from the unmodified headers, and the
 * golden vectors in tests/golden). The reduction part (pack, rank-order
 * all-reduce + SGD, the CPU Algorithm-2 pipeline) has NO reference code —
 * the reference only models it — so its parity is UNPINNED by the
 * reference: it restates PAPER.md:117-120 (Eq. 2) and PAPER.md:562-563,
 * and only its bf16 rounding is pinned (to torch's conversion).
 */
#define _GNU_SOURCE
#include "mgw_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ---------------------------------------------------------------- solver */

/* timeline.hpp:99-108 — tau_b[L-1] = t_f; tau_b[i] = tau_b[i+1] + t_b[i+1]. */
static void backward_starts(const double* t_b, size_t L, double t_f, double* tau_b) {
  tau_b[L - 1] = t_f;
  for (size_t i = L - 1; i-- > 0;) tau_b[i] = tau_b[i + 1] + t_b[i + 1];
}

/* trace.hpp:108-116 — bytes = (double)params * (double)bpe. */
static double bytes_of(const uint64_t* params, int bpe, size_t i) {
  return (double)params[i] * (double)bpe;
}

/* comm_model.hpp:194-199 */
static double cost(double a, double b, double m) { return a + b * m; }

int orc_optimal_plan(const uint64_t* params, const double* t_b, size_t L, double t_f, int bpe,
                     double a, double b, uint8_t* tags) {
  /* planner.hpp:36-45 */
  if (!(a > 0.0) || !(b >= 0.0)) return 3;
  if (L == 0) return 2;
  double* tau_b = malloc(L * sizeof(double));
  double* ready = malloc(L * sizeof(double));
  double* best_finish = malloc((L + 1) * sizeof(double));
  size_t* next_head = malloc((L + 1) * sizeof(size_t));
  backward_starts(t_b, L, t_f, tau_b);
  /* planner.hpp:66-70 */
  for (size_t i = 0; i < L; ++i) ready[i] = tau_b[i] + t_b[i];
  /* planner.hpp:72-92, literal O(L^2) form */
  best_finish[L] = -INFINITY;
  next_head[L] = L;
  for (size_t g = L; g-- > 0;) {
    double best = 0.0, group_bytes = 0.0;
    size_t choice = L;
    for (size_t u = g + 1; u <= L; ++u) {
      group_bytes += bytes_of(params, bpe, u - 1);
      const double hi = best_finish[u] > ready[g] ? best_finish[u] : ready[g];
      const double finish = hi + cost(a, b, group_bytes);
      if (u == g + 1 || finish < best) {
        best = finish;
        choice = u;
      }
    }
    best_finish[g] = best;
    next_head[g] = choice;
  }
  /* planner.hpp:93-97 */
  for (size_t i = 0; i < L; ++i) tags[i] = 1;
  for (size_t g = 0; g < L; g = next_head[g]) tags[g] = 0;
  free(tau_b);
  free(ready);
  free(best_finish);
  free(next_head);
  return 0;
}

/* planner.hpp:120-129 */
static void comm_start_times(const double* tau_b, const double* t_b, const double* t_c, size_t L,
                             double* tau_c) {
  tau_c[L - 1] = tau_b[L - 1] + t_b[L - 1];
  for (size_t i = L - 1; i-- > 0;) {
    const double x = tau_c[i + 1] + t_c[i + 1];
    const double y = tau_b[i] + t_b[i];
    tau_c[i] = x < y ? y : x; /* std::max(x, y) returns x unless x < y */
  }
}

int orc_greedy_plan(const uint64_t* params, const double* t_b, size_t L, double t_f, int bpe,
                    double a, double b, uint8_t* tags) {
  if (!(a > 0.0) || !(b >= 0.0)) return 3;
  if (L == 0) return 2;
  double* tau_b = malloc(L * sizeof(double));
  double* bytes = malloc(L * sizeof(double));
  double* t_c = malloc(L * sizeof(double));
  double* tau_c = malloc(L * sizeof(double));
  backward_starts(t_b, L, t_f, tau_b);
  for (size_t i = 0; i < L; ++i) {
    bytes[i] = bytes_of(params, bpe, i);
    t_c[i] = cost(a, b, bytes[i]);
    tags[i] = 0;
  }
  comm_start_times(tau_b, t_b, t_c, L, tau_c);
  /* planner.hpp:138-146 (paper Algorithm 1 lines 9-19) */
  for (size_t i = L - 1; i >= 1; --i) {
    if (tau_b[i - 1] + t_b[i - 1] - tau_c[i] < a) {
      t_c[i] = 0.0;
      bytes[i - 1] += bytes[i];
      t_c[i - 1] = cost(a, b, bytes[i - 1]);
      comm_start_times(tau_b, t_b, t_c, L, tau_c);
      tags[i] = 1;
    }
  }
  free(tau_b);
  free(bytes);
  free(t_c);
  free(tau_c);
  return 0;
}

double orc_iteration_time(const uint64_t* params, const double* t_b, size_t L, double t_f,
                          int bpe, double a, double b, const uint8_t* tags) {
  double* tau_b = malloc(L * sizeof(double));
  double* gbytes = calloc(L, sizeof(double));
  size_t* head = malloc(L * sizeof(size_t));
  double* t_c = malloc(L * sizeof(double));
  double* tau_c = malloc(L * sizeof(double));
  backward_starts(t_b, L, t_f, tau_b);
  /* timeline.hpp:113-126: fold ascending into the nearest lower normal */
  size_t h = 0;
  for (size_t i = 0; i < L; ++i) {
    if (tags[i] == 0) h = i;
    head[i] = h;
    gbytes[h] += bytes_of(params, bpe, i);
  }
  /* timeline.hpp:140-153 */
  for (size_t i = 0; i < L; ++i) t_c[i] = head[i] == i ? cost(a, b, gbytes[i]) : 0.0;
  comm_start_times(tau_b, t_b, t_c, L, tau_c);
  const double it = tau_c[0] + t_c[0]; /* timeline.hpp:172 */
  free(tau_b);
  free(gbytes);
  free(head);
  free(t_c);
  free(tau_c);
  return it;
}

int orc_fit(const uint64_t* sizes, const double* times, size_t n, double* a, double* b) {
  /* comm_model.hpp:209-251 */
  if (n < 2) return 2;
  int distinct = 0;
  for (size_t i = 0; i < n; ++i) {
    if (!(times[i] > 0.0)) return 2;
    if (sizes[i] != sizes[0]) distinct = 1;
  }
  if (!distinct) return 2;
  double sw = 0.0, sx = 0.0, sy = 0.0;
  for (size_t i = 0; i < n; ++i) {
    const double w = 1.0 / (times[i] * times[i]);
    sw += w;
    sx += w * (double)sizes[i];
    sy += w * times[i];
  }
  const double xbar = sx / sw, ybar = sy / sw;
  double sxx = 0.0, sxy = 0.0;
  for (size_t i = 0; i < n; ++i) {
    const double w = 1.0 / (times[i] * times[i]);
    const double dx = (double)sizes[i] - xbar;
    sxx += w * dx * dx;
    sxy += w * dx * (times[i] - ybar);
  }
  *b = sxy / sxx;
  *a = ybar - *b * xbar;
  if (!(*a > 0.0) || !(*b >= 0.0)) return 2;
  return 0;
}

/* ------------------------------------------------------------- reduction */

void orc_merge_offsets(const uint64_t* counts, size_t L, uint64_t* offs) {
  offs[0] = 0;
  for (size_t l = 0; l < L; ++l) offs[l + 1] = offs[l] + ((counts[l] + 3u) & ~(uint64_t)3u);
}

void orc_pack(const float* const* grads, const uint64_t* counts, const uint64_t* offs,
              size_t first, size_t last, float scale, float* merge) {
  for (size_t l = first; l < last; ++l) {
    float* dst = merge + (offs[l] - offs[first]);
    const uint64_t padded = offs[l + 1] - offs[l];
    for (uint64_t j = 0; j < padded; ++j) dst[j] = j < counts[l] ? grads[l][j] * scale : 0.0f;
  }
}

/* Reduce one contiguous layer range for P ranks: rank-order sum of the
 * scaled gradients, then SGD. Split by element chunks for OpenMP. */
static void reduce_layer(int P, float* const* grads, float* const* weights, size_t L, size_t l,
                         uint64_t begin, uint64_t end, float scale, float lr, int write_grad) {
  for (uint64_t j = begin; j < end; ++j) {
    float acc = grads[l][j] * scale;
    for (int r = 1; r < P; ++r) acc = acc + grads[(size_t)r * L + l][j] * scale;
    for (int r = 0; r < P; ++r) {
      float* w = weights[(size_t)r * L + l];
      if (w) {
        w[j] = w[j] - lr * acc; /* two roundings: -ffp-contract=off, no FMA */
      }
    }
    if (write_grad) {
      for (int r = 0; r < P; ++r) grads[(size_t)r * L + l][j] = acc;
    }
  }
}

void orc_allreduce_sgd(int P, float* const* grads, float* const* weights, const uint64_t* counts,
                       size_t L, const uint8_t* tags, float lr, int write_grad) {
  const float scale = 1.0f / (float)P;
  (void)tags; /* grouping does not change per-element values */
  for (size_t l = 0; l < L; ++l) {
    reduce_layer(P, grads, weights, L, l, 0, counts[l], scale, lr, write_grad);
  }
}

/* NVLS variant (the switch-reduced all-reduce, SURVEY §5 "optional, flagged"):
 * the NVSwitch's multimem.ld_reduce returns the EXACT sum of the P scaled
 * fp32 values rounded once to fp32 (nearest even) — measured on B200,
 * tools/nvls_probe.cu; at P = 2 that equals the rank-order sum. Restated
 * with an x87 80-bit accumulator: exact whenever the P addends' exponents
 * span <= 37 bits (64-bit significand), which holds for every test input
 * here (uniform gradients); then one rounding to fp32. Not pinned to the
 * reference: the reference models no runtime. */
void orc_allreduce_sgd_nvls(int P, float* const* grads, float* const* weights, const uint64_t* counts,
                            size_t L, const uint8_t* tags, float lr, int write_grad) {
  const float scale = 1.0f / (float)P;
  (void)tags;
  for (size_t l = 0; l < L; ++l) {
    for (uint64_t j = 0; j < counts[l]; ++j) {
      long double exact = 0.0L;
      for (int r = 0; r < P; ++r) exact += (long double)(grads[(size_t)r * L + l][j] * scale);
      const float acc = (float)exact;
      for (int r = 0; r < P; ++r) {
        float* w = weights[(size_t)r * L + l];
        if (w) w[j] = w[j] - lr * acc;
      }
      if (write_grad) {
        for (int r = 0; r < P; ++r) grads[(size_t)r * L + l][j] = acc;
      }
    }
  }
}

/* ------------------------------------------------------- bf16 gradients */

uint16_t orc_f32_to_bf16(float x) {
  uint32_t u;
  memcpy(&u, &x, sizeof u);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40u); /* quiet NaN */
  u += 0x7fffu + ((u >> 16) & 1u); /* round to nearest, ties to even */
  return (uint16_t)(u >> 16);
}

float orc_bf16_to_f32(uint16_t h) {
  const uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, sizeof f);
  return f;
}

void orc_merge_offsets_granule(const uint64_t* counts, size_t L, uint64_t granule, uint64_t* offs) {
  offs[0] = 0;
  for (size_t l = 0; l < L; ++l) offs[l + 1] = offs[l] + ((counts[l] + granule - 1) / granule) * granule;
}

void orc_pack_bf16(const uint16_t* const* grads, const uint64_t* counts, const uint64_t* offs,
                   size_t first, size_t last, float scale, uint16_t* merge) {
  for (size_t l = first; l < last; ++l) {
    uint16_t* dst = merge + (offs[l] - offs[first]);
    const uint64_t padded = offs[l + 1] - offs[l];
    for (uint64_t j = 0; j < padded; ++j) {
      dst[j] = j < counts[l] ? orc_f32_to_bf16(orc_bf16_to_f32(grads[l][j]) * scale) : 0;
    }
  }
}

void orc_allreduce_sgd_bf16(int P, uint16_t* const* grads, float* const* weights, const uint64_t* counts,
                            size_t L, const uint8_t* tags, float lr, int write_grad) {
  const float scale = 1.0f / (float)P;
  (void)tags; /* grouping does not change per-element values */
  for (size_t l = 0; l < L; ++l) {
    for (uint64_t j = 0; j < counts[l]; ++j) {
      float acc = orc_bf16_to_f32(grads[l][j]) * scale;
      for (int r = 1; r < P; ++r) acc = acc + orc_bf16_to_f32(grads[(size_t)r * L + l][j]) * scale;
      const uint16_t red_bits = orc_f32_to_bf16(acc);
      const float red = orc_bf16_to_f32(red_bits);
      for (int r = 0; r < P; ++r) {
        float* w = weights[(size_t)r * L + l];
        if (w) {
          w[j] = w[j] - lr * red; /* two roundings: -ffp-contract=off, no FMA */
        }
      }
      if (write_grad) {
        for (int r = 0; r < P; ++r) grads[(size_t)r * L + l][j] = red_bits;
      }
    }
  }
}

/* --------------------------------------------------- CPU Algorithm 2 run */

static double now_sec(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

typedef struct {
  int P, threads, write_grad;
  float lr;
  float* const* grads;
  float* const* weights;
  const uint64_t* counts;
  size_t L, G;
  const size_t* heads; /* ascending, G+1 entries (heads[G] = L) */
  float** merge;       /* per-rank merge buffers (padded layout) */
  const uint64_t* offs;
  _Atomic long ready_groups; /* groups made ready by the compute thread this iter */
  _Atomic long done_groups;
  _Atomic int iter_go;       /* iteration index the comm thread may start */
  _Atomic int quit;
} pipe_ctx;

/* Group g (ascending index): pack every rank x 1/P into its merge buffer,
 * rank-order sum, SGD on every rank — paper SynchonizedAllReduce(lb). */
static void cpu_group(pipe_ctx* c, size_t g) {
  const size_t first = c->heads[g], last = c->heads[g + 1];
  const uint64_t base = c->offs[first], span = c->offs[last] - base;
  const float scale = 1.0f / (float)c->P;
  for (int r = 0; r < c->P; ++r) {
    float* const* gr = c->grads + (size_t)r * c->L;
    float* m = c->merge[r] + base;
    for (size_t l = first; l < last; ++l) {
      float* dst = m + (c->offs[l] - base);
      const uint64_t padded = c->offs[l + 1] - c->offs[l];
      const long long cnt = (long long)c->counts[l];
      const float* src = gr[l];
#pragma omp parallel for num_threads(c->threads) schedule(static) if (cnt > 65536)
      for (long long j = 0; j < cnt; ++j) dst[j] = src[j] * scale;
      for (uint64_t j = (uint64_t)cnt; j < padded; ++j) dst[j] = 0.0f;
    }
  }
  const long long n = (long long)span;
#pragma omp parallel for num_threads(c->threads) schedule(static) if (n > 65536)
  for (long long j = 0; j < n; ++j) {
    float acc = c->merge[0][base + (uint64_t)j];
    for (int r = 1; r < c->P; ++r) acc = acc + c->merge[r][base + (uint64_t)j];
    c->merge[0][base + (uint64_t)j] = acc;
  }
  for (size_t l = first; l < last; ++l) {
    const float* red = c->merge[0] + c->offs[l];
    const long long cnt = (long long)c->counts[l];
    for (int r = 0; r < c->P; ++r) {
      float* w = c->weights[(size_t)r * c->L + l];
#pragma omp parallel for num_threads(c->threads) schedule(static) if (cnt > 65536)
      for (long long j = 0; j < cnt; ++j) w[j] = w[j] - c->lr * red[j]; /* -ffp-contract=off */
    }
  }
}

static void* comm_thread(void* arg) {
  pipe_ctx* c = arg;
  int iter = 0;
  for (;;) {
    while (atomic_load(&c->iter_go) <= iter) {
      if (atomic_load(&c->quit)) return NULL;
    }
    /* FIFO in backward order: groups G-1 .. 0 */
    for (long k = 0; k < (long)c->G; ++k) {
      while (atomic_load(&c->ready_groups) <= k) {
      }
      cpu_group(c, c->G - 1 - (size_t)k);
      atomic_store(&c->done_groups, k + 1);
    }
    ++iter;
  }
}

int orc_pipeline_run(int P, float* const* grads, float* const* weights, const uint64_t* counts,
                     const double* t_b, size_t L, double t_f, const uint8_t* tags, float lr,
                     int threads, int iters, double* iter_sec_out) {
  if (P < 1 || L == 0 || iters < 0) return 2;
  pipe_ctx c;
  memset(&c, 0, sizeof c);
  c.P = P;
  /* the calling thread spins on the replay clock: leave it a core */
  c.threads = threads > 1 ? threads - 1 : 1;
  c.lr = lr;
  c.grads = grads;
  c.weights = weights;
  c.counts = counts;
  c.L = L;
  size_t* heads = malloc((L + 1) * sizeof(size_t));
  size_t G = 0;
  for (size_t i = 0; i < L; ++i) {
    if (i == 0 || tags[i] == 0) heads[G++] = i;
  }
  heads[G] = L;
  c.G = G;
  c.heads = heads;
  uint64_t* offs = malloc((L + 1) * sizeof(uint64_t));
  orc_merge_offsets(counts, L, offs);
  c.offs = offs;
  c.merge = malloc((size_t)P * sizeof(float*));
  for (int r = 0; r < P; ++r) c.merge[r] = calloc(offs[L] ? offs[L] : 1, sizeof(float));
  double* tau_b = malloc(L * sizeof(double));
  backward_starts(t_b, L, t_f, tau_b);

  pthread_t th;
  pthread_create(&th, NULL, comm_thread, &c);
  for (int it = 0; it < iters; ++it) {
    atomic_store(&c.ready_groups, 0);
    atomic_store(&c.done_groups, 0);
    const double t0 = now_sec();
    atomic_store(&c.iter_go, it + 1);
    /* compute thread: layers L-1..0 finish at tau_b[l] + t_b[l]; a group is
     * pushed when its head (lowest layer) finishes (Algorithm 2 lines 20-23). */
    for (long k = 0; k < (long)G; ++k) {
      const size_t head = heads[G - 1 - (size_t)k];
      const double due = t0 + tau_b[head] + t_b[head];
      while (now_sec() < due) {
      }
      atomic_store(&c.ready_groups, k + 1);
    }
    while (atomic_load(&c.done_groups) < (long)G) {
    }
    iter_sec_out[it] = now_sec() - t0;
  }
  atomic_store(&c.quit, 1);
  pthread_join(th, NULL);
  for (int r = 0; r < P; ++r) free(c.merge[r]);
  free(c.merge);
  free(heads);
  free(offs);
  free(tau_b);
  return 0;
}
