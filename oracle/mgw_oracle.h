/*
 * mgw_oracle.h — CPU restatement of the MG-WFBP path. TEST INFRASTRUCTURE.
 *
 * This is the parity checker, not the product. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load liboracle (oracle/_build/libmgw_oracle.so). The product
 * (libmgwfbp.so) never links or calls it and fails loudly without its CUDA
 * kernels.
 *
 * Pinning: the solver/predictor/fit restatements are checked bit-for-bit
 * against the reference itself compiled from /root/reference
 * (oracle/_ref/libgradsched_ref.so, see oracle/ref_shim.cpp) and against the
 * golden vectors in tests/golden/. The reduction restatement (pack x 1/P,
 * rank-order fp32 sum, SGD) has no reference code to pin against — the
 * reference only charges a + b*M for it — so its "parity" is our own
 * restatement of PAPER.md:117-120 (Eq. 2) and PAPER.md:562-563 (merge
 * buffers): PARITY UNPINNED for reduced values, by construction.
 */
#ifndef MGW_ORACLE_H_
#define MGW_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* --- solver / predictor (reference planner.hpp, timeline.hpp) --- */

/* Returns 0, or 3 if a <= 0 or b < 0 (PlannerError). */
int orc_optimal_plan(const uint64_t* params, const double* t_b, size_t L, double t_f, int bpe,
                     double a, double b, uint8_t* tags);
int orc_greedy_plan(const uint64_t* params, const double* t_b, size_t L, double t_f, int bpe,
                    double a, double b, uint8_t* tags);
double orc_iteration_time(const uint64_t* params, const double* t_b, size_t L, double t_f,
                          int bpe, double a, double b, const uint8_t* tags);
/* Returns 0, or 2 on an unusable fit. */
int orc_fit(const uint64_t* sizes, const double* times_sec, size_t n, double* a, double* b);

/* --- merge layout and reduction (the build's semantics) --- */

/* Element offset of every layer in the padded merge layout: each layer starts
 * on a 4-element (16-byte) boundary. offs has L+1 entries. */
void orc_merge_offsets(const uint64_t* counts, size_t L, uint64_t* offs);

/* Gather layers [first, last) times `scale` into merge (padded, zero pad),
 * merge[0] being the element at offs[first]. */
void orc_pack(const float* const* grads, const uint64_t* counts, const uint64_t* offs,
              size_t first, size_t last, float scale, float* merge);

/* One synchronous DP iteration for P ranks held as host arrays:
 * grads[r*L + l], weights[r*L + l]. For every group of `tags`: pack with
 * scale 1/P per rank, sum ranks 0..P-1 in order (fl(fl(x0)+x1)+...),
 * w = fl(w - fl(lr * g)) on every rank, grads overwritten with the reduced
 * value when write_grad. */
void orc_allreduce_sgd(int P, float* const* grads, float* const* weights, const uint64_t* counts,
                       size_t L, const uint8_t* tags, float lr, int write_grad);

/* NVLS variant: the per-element sum is the exact sum of the P scaled values
 * rounded once to fp32 (what the NVSwitch's multimem.ld_reduce returns). */
void orc_allreduce_sgd_nvls(int P, float* const* grads, float* const* weights, const uint64_t* counts,
                            size_t L, const uint8_t* tags, float lr, int write_grad);

/* --- bf16 gradients (reference trace.hpp:50
 * bytes_per_element = 2). The build's semantics, restated: every source is
 * widened to fp32 (exact), times 1/P, summed in rank order in fp32; the sum
 * is rounded ONCE to bf16 (round to nearest even) and that value is the
 * reduced gradient of every rank: w = fl(w - fl(lr * red)) on fp32 weights,
 * grads overwritten with it when write_grad. --- */

/* fp32 -> bf16 bits, round to nearest even (NaN -> quiet NaN). */
uint16_t orc_f32_to_bf16(float x);
float orc_bf16_to_f32(uint16_t h);

/* Merge layout with layers starting on a `granule`-element boundary (16
 * bytes: 4 for fp32, 8 for bf16). */
void orc_merge_offsets_granule(const uint64_t* counts, size_t L, uint64_t granule, uint64_t* offs);

/* bf16 pack: merge[j] = bf16(f32(g[j]) * scale), zero padding. */
void orc_pack_bf16(const uint16_t* const* grads, const uint64_t* counts, const uint64_t* offs,
                   size_t first, size_t last, float scale, uint16_t* merge);

void orc_allreduce_sgd_bf16(int P, uint16_t* const* grads, float* const* weights, const uint64_t* counts,
                            size_t L, const uint8_t* tags, float lr, int write_grad);

/* --- CPU runtime of paper Algorithm 2 (bench reference arm) --- */

/* Runs `iters` iterations: the calling thread replays the backward schedule
 * (busy-wait to each layer's ready time, t_f + backward of the layers above)
 * and a communication thread performs each group's CPU all-reduce + SGD
 * (OpenMP over `threads` cores) as soon as its head layer is ready, FIFO in
 * backward order. Writes per-iteration wall seconds. */
int orc_pipeline_run(int P, float* const* grads, float* const* weights, const uint64_t* counts,
                     const double* t_b, size_t L, double t_f, const uint8_t* tags, float lr,
                     int threads, int iters, double* iter_sec_out);

#ifdef __cplusplus
}
#endif

#endif /* MGW_ORACLE_H_ */
