/*
 * mgwfbp.h — C ABI of the B200-native MG-WFBP runtime (libmgwfbp.so).
 *
 * The reference (arxiv 1912.09268, `gradsched`) exposes a header-only C++
 * API and no FFI. This header is the thin, plain-pointer boundary that a
 * binding (ctypes, cgo, JNI, ...) or a C++ host calls. It has two halves:
 *
 *  HOST (pure, thread-safe, no CUDA): the solver, predictor and calibration
 *  fit, bit-exact with the reference C++ functions they replace.
 *
 *  DEVICE (sm_100a, one process per GPU): symmetric merge arenas mapped over
 *  NVLink with CUDA IPC, the pack kernel, the fused pack -> one-shot/two-shot
 *  all-reduce -> unpack+SGD kernel, the backward-replay pipeline and the
 *  on-box calibration sweep. The reference only *models* these (paper
 *  Algorithm 2; cost model comm_model.hpp:194-199).
 *
 * Conventions
 *  - Every function returns an mgw_status. On failure mgw_last_error()
 *    returns a thread-local message. No C++ exception crosses this ABI.
 *  - Status codes mirror the reference CLI exit codes (tools/main.cpp:31-35):
 *    2 = bad input (ValidationError / ParseError / FitError),
 *    3 = planner rejection (PlannerError), 4 = guard refusal (GuardError).
 *  - Tags: 0 = normal (group head), 1 = merged (folds into the next lower
 *    layer), indexed in forward order like ModelTrace::layers.
 *  - Times in seconds (double) unless a name says otherwise.
 *  - Streams are cudaStream_t passed as void*. Device pointers are
 *    caller-owned fp32 buffers; nothing on the hot path allocates.
 *  - Device functions of one communicator are collective: every rank calls
 *    them in the same order with the same arguments (sizes, plans, groups).
 */
#ifndef MGWFBP_H_
#define MGWFBP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MGW_OK = 0,
  MGW_ERR_INPUT = 2,
  MGW_ERR_PLANNER = 3,
  MGW_ERR_GUARD = 4,
  MGW_ERR_CUDA = 6,
  MGW_ERR_INTERNAL = 7,
} mgw_status;

/* One calibration sample. Same fields as gradsched::CommMeasurement
 * (reference comm_model.hpp:121-130). */
typedef struct {
  uint64_t size_bytes;
  double time_sec;
} mgw_meas;

const char* mgw_last_error(void);
/* Class of the last error: "ValidationError", "ParseError", "FitError",
 * "PlannerError", "GuardError", "CudaError" or "Error". */
const char* mgw_last_error_kind(void);
const char* mgw_version(void);

/* ------------------------------------------------------------------ HOST */

/* gradsched::fit_model (comm_model.hpp:209-251): 1/t^2-weighted least
 * squares -> T(M) = a + b*M. */
int mgw_fit(const mgw_meas* samples, size_t n, double* a_out, double* b_out);

/* gradsched::load_measurements_csv (comm_model.hpp:255-308). Two-call
 * pattern: pass out=NULL to get the count, then a buffer of that size. */
int mgw_load_measurements_csv(const char* path, mgw_meas* out, size_t cap, size_t* n_out);

/* gradsched::coefficients_for (comm_model.hpp:140-191). algo: 0 binary
 * tree, 1 recursive doubling, 2 recursive halving/doubling, 3 double binary
 * trees, 4 ring. */
int mgw_coefficients(int algo, double alpha, double beta, double gamma, int n_workers,
                     int dbt_literal, double* a_out, double* b_out);

/* A trace in the reference schema (trace.hpp:38-94): L layers in forward
 * order, params[i] gradient elements, t_b[i] backward seconds. */

/* gradsched::load_trace (trace.hpp:148-219). Two-call pattern on params /
 * t_b (pass NULL to query L). */
int mgw_load_trace(const char* path, size_t* L_out, double* t_f_out, int* bpe_out,
                   uint64_t* params_out, double* t_b_out, size_t cap);

/* gradsched::optimal_plan (planner.hpp:63-98), bit-exact tags. */
int mgw_plan_optimal(const uint64_t* params, const double* t_b, size_t L, double t_f,
                     int bpe, double a, double b, uint8_t* tags_out);

/* gradsched::greedy_plan (planner.hpp:112-148; paper Algorithm 1). */
int mgw_plan_greedy(const uint64_t* params, const double* t_b, size_t L, double t_f,
                    int bpe, double a, double b, uint8_t* tags_out);

/* gradsched::brute_force_plan (planner.hpp:159-200); L <= max_layers. */
int mgw_plan_brute_force(const uint64_t* params, const double* t_b, size_t L, double t_f,
                         int bpe, double a, double b, size_t max_layers, uint8_t* tags_out,
                         double* iter_time_out);

/* gradsched::iteration_time (timeline.hpp:158-177). Any of the per-layer
 * outputs may be NULL. */
int mgw_predict(const uint64_t* params, const double* t_b, size_t L, double t_f, int bpe,
                double a, double b, const uint8_t* tags, double* iter_time_out,
                double* comm_nonoverlap_out, double* tau_b_out, double* tau_c_out,
                double* t_c_out);

/* B200 extension (no reference counterpart): optimal_plan's exact DP and
 * iteration_time's FIFO timeline with T(M) interpolated from measured
 * (size, time) pairs — piecewise linear, non-decreasing, flat below the
 * smallest size, last slope above the largest — instead of a + b*M. The
 * fused kernel's cost is piecewise (LL / one-shot / two-shot). */
int mgw_plan_optimal_table(const uint64_t* params, const double* t_b, size_t L, double t_f, int bpe,
                           const mgw_meas* meas, size_t n_meas, uint8_t* tags_out);
int mgw_predict_table(const uint64_t* params, const double* t_b, size_t L, double t_f, int bpe,
                      const mgw_meas* meas, size_t n_meas, const uint8_t* tags, double* iter_time_out);

/* gradsched::synceasgd_time / naive_time (timeline.hpp:196-221). */
int mgw_baseline_times(const uint64_t* params, const double* t_b, size_t L, double t_f,
                       int bpe, double a, double b, double* synceasgd_out, double* naive_out);

/* gradsched::synth_trace + save_trace (trace.hpp:257-346, :221-248): the
 * canonical JSON text of a deterministic synthetic trace, NUL-terminated in
 * buf when cap > length. Returns the length, or -status on error. */
long mgw_synth_trace_json(size_t n_layers, uint64_t total_params, double total_backward_time,
                          double forward_time, double size_skew, int bpe, uint64_t seed, char* buf,
                          size_t cap);

/* ---------------------------------------------------------------- DEVICE */

typedef struct mgw_comm mgw_comm;
typedef struct mgw_plan mgw_plan;
typedef struct mgw_pipeline mgw_pipeline;

/* Per-rank communicator on `device`: allocates the symmetric merge arena
 * (nranks slots of arena_bytes: slot r receives rank r's scaled gradients
 * as posted NVLink stores) and the signal area. arena_bytes must hold the
 * padded merge layout of every plan used with it. nranks in {1, 2, 4, 8}. */
int mgw_comm_create(int rank, int nranks, int device, size_t arena_bytes, mgw_comm** out);

/* CUDA IPC handles of this rank's arena + signal area (opaque bytes). */
size_t mgw_comm_handle_size(void);
int mgw_comm_export_handle(mgw_comm* comm, void* handle_out);
/* all_handles: nranks * mgw_comm_handle_size() bytes in rank order. Maps
 * every peer's arena and signals into this process (NVLink P2P). */
int mgw_comm_open_peers(mgw_comm* comm, const void* all_handles);
int mgw_comm_destroy(mgw_comm* comm);
/* Ranks whose arena + signal area this communicator can address (itself
 * included): nranks once mgw_comm_open_peers mapped every peer. */
int mgw_comm_num_peers(const mgw_comm* comm, int* mapped);

/* Single-GPU emulation of `nranks` ranks (all arenas on one device, every
 * collective launched as ONE kernel over all emulated ranks: a cooperative
 * group launch, or one persistent-engine grid (ctas, nranks) for pipelines).
 * Used by the parity tests on one B200; never by the multi-GPU path. */
int mgw_comm_create_loopback(int nranks, int device, size_t arena_bytes, mgw_comm** out);

/* Device-side plan: the layer table of this rank (grads[i], weights[i]
 * are device fp32 pointers with counts[i] elements; weights may be NULL
 * when lr is never used) and the merge tags. For a loopback comm the
 * arrays hold nranks*L pointers, emulated rank r at [r*L, (r+1)*L).
 * Group g (0-based, ascending head index) is [head_g, head_{g+1}). */
int mgw_plan_create(mgw_comm* comm, size_t L, float* const* grads, float* const* weights,
                    const uint64_t* counts, const uint8_t* tags, mgw_plan** out);

/* Gradient element type (reference trace.hpp:50
 * bytes_per_element). Weights are always fp32 (master weights). */
typedef enum { MGW_DTYPE_F32 = 0, MGW_DTYPE_BF16 = 1 } mgw_dtype;

/* mgw_plan_create with the gradient element type. bf16: gradients and the
 * merge arena are bf16 (half the NVLink and HBM bytes); every source is
 * widened to fp32, scaled by 1/P and summed in rank order in fp32; the sum
 * is rounded once to bf16 (nearest even) and THAT value is the reduced
 * gradient on every rank (SGD on the fp32 weights, grad write-back). The
 * merge layout pads every layer to 16 bytes (8 bf16 elements). */
int mgw_plan_create_ex(mgw_comm* comm, size_t L, void* const* grads, float* const* weights,
                       const uint64_t* counts, const uint8_t* tags, int dtype, mgw_plan** out);
int mgw_plan_destroy(mgw_plan* plan);
int mgw_plan_num_groups(const mgw_plan* plan, int* n_groups_out);
/* Padded element span of group g inside the merge layout (layers start
 * 16-byte aligned). */
int mgw_plan_group_span(const mgw_plan* plan, int group, uint64_t* elem_begin,
                        uint64_t* elem_count, uint64_t* bytes_unpadded);

/* Pack kernel: gather group g's layer gradients, times `scale`, into the
 * contiguous merge buffer `merge_buf` (>= elem_count elements of the plan's
 * gradient type, padded layout). Rank-local. */
int mgw_pack(mgw_plan* plan, int group, float scale, void* merge_buf, void* stream);

/* Unpack + SGD: for every layer of group g, w -= lr * red (non-contracted
 * fp32) and, if write_grad, grad = red. Rank-local. */
int mgw_unpack_sgd(mgw_plan* plan, int group, const void* merge_buf, float lr, int write_grad,
                   void* stream);

/* Algorithm selection for the merged all-reduce. */
typedef enum { MGW_ALGO_AUTO = 0, MGW_ALGO_ONESHOT = 1, MGW_ALGO_TWOSHOT = 2, MGW_ALGO_NVLS = 3 } mgw_algo;
/* Epilogue flags. */
enum { MGW_SGD = 1, MGW_WRITE_GRAD = 2 };

/* The fused hot op, collective: pack (x 1/P) -> all-reduce over NVLink in
 * rank order -> unpack + SGD, one kernel per group. */
int mgw_group_allreduce(mgw_plan* plan, int group, float lr, int epilogue, int algo,
                        void* stream);

/* One-shot/two-shot crossover (bytes) used by MGW_ALGO_AUTO (default: the
 * B200-measured crossover for the communicator's rank count). */
int mgw_comm_set_oneshot_max(mgw_comm* comm, uint64_t bytes);
int mgw_comm_get_oneshot_max(const mgw_comm* comm, uint64_t* bytes);
/* Tuning knobs (defaults: the B200 measurements in DESIGN.md §4.1). Every
 * rank must set the same values before creating plans / pipelines.
 *  ll_max: one-shot groups up to this many bytes travel as LL (flag-in-data)
 *    packets; 0 disables LL.
 *  small_tile_max: groups below this many bytes are cut into 8 KiB tiles
 *    (more CTAs) instead of 32 KiB tiles.
 *  protocol: MGW_PROTO_AUTO (default) — chunked at P > 1 (the shorter
 *    iteration for every measured MG-WFBP plan), the TMA-fed engine at
 *    P = 1; MGW_PROTO_STREAM — the persistent engine streams: the producer
 *    warp streams tiles and publishes per-tile delivery counts, the data
 *    warps consume them as they arrive (no barrier after the launch's entry
 *    barrier), and a replay pipeline launches its last-ready group as a
 *    chunked standalone launch after the engine (an isolated large group is
 *    the streamed protocol's weak case); standalone launches stay chunked
 *    unless STREAM is set; MGW_PROTO_CHUNKED — everything chunked: a CTA's
 *    tiles run in
 *    pipelined chunks with one cross-rank barrier per chunk (chunk_tiles /
 *    min_chunks: at most chunk_tiles tiles per chunk, two-shot chunk_tiles /
 *    P super-tiles, and at least min_chunks chunks when the CTA owns enough
 *    tiles). At P = 1, CHUNKED selects the register engine instead of the
 *    TMA-fed one. */
#define MGW_PROTO_STREAM 0
#define MGW_PROTO_CHUNKED 1
#define MGW_PROTO_AUTO 2
int mgw_comm_set_ll_max(mgw_comm* comm, uint64_t bytes);
int mgw_comm_set_small_tile_max(mgw_comm* comm, uint64_t bytes);
int mgw_comm_set_chunk_tiles(mgw_comm* comm, uint32_t max_tiles, uint32_t min_chunks);
int mgw_comm_set_protocol(mgw_comm* comm, int protocol);
/* Streamed protocol: a producer publishes its delivery count every
 * credit_batch (1, 2, 4 or 8) bulk items; a two-shot owner publishes its
 * reduced tiles every ag_batch owned super-tiles. */
int mgw_comm_set_stream_batches(mgw_comm* comm, uint32_t credit_batch, uint32_t ag_batch);
int mgw_comm_get_protocol(const mgw_comm* comm, int* protocol);
/* Current knob values (any output may be NULL). */
int mgw_comm_get_tuning(const mgw_comm* comm, uint64_t* oneshot_max, uint64_t* ll_max,
                        uint64_t* small_tile_max, uint32_t* chunk_tiles, uint32_t* min_chunks);
/* 1 in *failed once any kernel of this communicator gave up a bounded wait
 * (a peer or the compute side never arrived; the kernels then skip their
 * SGD epilogues). Reads host-mapped memory: no CUDA call, no sync — cheap
 * enough to poll every iteration. A failed communicator stays failed. */
int mgw_comm_error(const mgw_comm* comm, int* failed);
/* NVLS (NVLink SHARP, the optional switch-reduced variant of SURVEY §5):
 * every rank's copy of one arena slot is bound to a multicast object; the
 * owner of each vector reads the P copies' SUM through the multicast
 * address (multimem.ld_reduce: the NVSwitch reduces) and stores it to all P
 * copies (multimem.st), then every rank unpacks + applies SGD locally. NVLink
 * bytes per rank: S each way instead of 2(P-1)/P*S. Numerics: the switch
 * returns the exact sum of the P scaled fp32 values rounded once (nearest
 * even) — the rank-order sum at P = 2, the oracle's exact-sum variant at
 * P >= 4 (deterministic, identical on every rank). fp32 only; standalone
 * group launches only (mgw_group_allreduce, mgw_allreduce, calibration, the
 * pipelines' launch mode and tail launches), never the persistent engine.
 * Setup is collective, three phases (the caller moves rank 0's handle to
 * every rank and puts a barrier between join and bind):
 *   mgw_comm_nvls_create  rank 0 creates + exports the multicast object into
 *                         handle_out (mgw_nvls_handle_size() bytes; other ranks
 *                         get zeros);
 *   mgw_comm_nvls_join    every rank: import rank 0's handle, add its GPU;
 *   mgw_comm_nvls_bind    every rank, after all joined: bind + map.
 * mgw_comm_set_nvls: MGW_ALGO_AUTO sends fp32 groups of at least min_bytes
 * through NVLS (0: never, the default); chunk_tiles (1..16, default 4): tiles
 * per pipelined chunk of a CTA. MGW_ALGO_NVLS forces it for any size. */
size_t mgw_nvls_handle_size(void);
int mgw_comm_nvls_supported(const mgw_comm* comm, int* supported);
int mgw_comm_nvls_create(mgw_comm* comm, void* handle_out);
int mgw_comm_nvls_join(mgw_comm* comm, const void* handle0);
int mgw_comm_nvls_bind(mgw_comm* comm);
int mgw_comm_nvls_ready(const mgw_comm* comm, int* ready);
int mgw_comm_set_nvls(mgw_comm* comm, uint64_t min_bytes, uint32_t chunk_tiles);
/* Profiling aid (results are WRONG while set): 1 skips the NVLS kernel's
 * pack / unpack (HBM) phases, 2 skips its switch reduce; 0 restores. */
int mgw_comm_set_nvls_skip(mgw_comm* comm, uint32_t mask);
/* Cap on the CTAs per rank of a standalone fused launch (mgw_group_allreduce,
 * mgw_allreduce); 0 = one per SM (default). A real backward that launches
 * groups while it runs leaves the other SMs to the compute kernels. */
int mgw_comm_set_max_ctas(mgw_comm* comm, int max_ctas);

/* Backward-replay pipeline (paper Algorithm 2): a compute stream spins
 * until each group head's ready time (t_f + backward of the layers above,
 * trace order), a comm stream launches each group the moment its head is
 * ready, FIFO in backward order; the whole iteration is one CUDA graph.
 * t_b: L backward seconds, t_f: forward seconds. l2_flush_bytes > 0 adds
 * a memset of that many bytes on a side branch at iteration start (it
 * overlaps the forward replay, as a real forward evicts L2), which the first
 * group waits for, so no iteration reads gradients/weights hot from L2.
 * engine_ctas selects the comm side: 0 = one fused kernel launch per group,
 * each gated by its head's ready event; != 0 = the persistent comm engine,
 * ONE kernel per iteration with engine_ctas CTAs (< 0: one per SM) that
 * runs the groups in backward order as the replay marks them ready (no
 * per-group launch cost; the paper's comm daemon thread, on the GPU). */
int mgw_pipeline_create(mgw_plan* plan, const double* t_b, double t_f, float lr, int algo,
                        int record_group_times, size_t l2_flush_bytes, int engine_ctas,
                        mgw_pipeline** out);
/* Same, with the step's host I/O captured into the graph: h2d_bytes from
 * pinned h2d_src to device h2d_dst on the comm branch at iteration start
 * (every group waits for it; it overlaps the forward replay), and d2h_bytes
 * from device d2h_src to pinned d2h_dst after the last group. One launch =
 * one end-to-end step. */
int mgw_pipeline_create_io(mgw_plan* plan, const double* t_b, double t_f, float lr, int algo,
                           int record_group_times, size_t l2_flush_bytes, int engine_ctas,
                           const void* h2d_src, void* h2d_dst, size_t h2d_bytes, void* d2h_dst,
                           const void* d2h_src, size_t d2h_bytes, mgw_pipeline** out);
int mgw_pipeline_destroy(mgw_pipeline* pipe);
/* Launch `iters` iterations back to back on the pipeline's compute stream
 * (asynchronous). */
int mgw_pipeline_launch(mgw_pipeline* pipe, int iters);
/* Synchronous: run iters iterations, write per-iteration device times (ms,
 * CUDA events on the compute stream). */
int mgw_pipeline_run(mgw_pipeline* pipe, int iters, float* iter_ms_out);
/* Per-group kernel durations (ms) of the last launched iteration, in group
 * order; requires record_group_times. */
int mgw_pipeline_group_times(mgw_pipeline* pipe, float* group_ms_out);
/* The compute stream (cudaStream_t) the pipeline runs on. */
int mgw_pipeline_stream(mgw_pipeline* pipe, void** stream_out);
/* Diagnostics, readable while the pipeline runs: engine state {groups made
 * ready, iteration, CTA exit count, ready-timeout flag} and the replay clock
 * {iteration start, last replay completion} (%globaltimer ns). */
int mgw_pipeline_debug(mgw_pipeline* pipe, uint32_t* engine_state4, uint64_t* clock2);
/* Standalone drain of an engine pipeline (roofline and ncu runs): launch the
 * persistent engine `iters` times with EVERY group ready at launch (no
 * replay, no ready flags), each launch preceded by the pipeline's L2 flush;
 * writes each engine launch's device time (ms, CUDA events on the engine's
 * stream). The plan's whole merged all-reduce + SGD streams through the
 * engine back to back. Collective. */
int mgw_pipeline_drain(mgw_pipeline* pipe, int iters, float* ms_out);
/* Engine pipelines with record_group_times: the last iteration's raw
 * (start, end) %globaltimer stamps of every group, 2*G values in group
 * order (zero for groups without tiles). */
int mgw_pipeline_stamps(mgw_pipeline* pipe, uint64_t* stamps_2g);
/* 1 in *streamed when the pipeline's persistent engine runs the streamed
 * protocol (0: chunked, or no engine). */
int mgw_pipeline_streamed(const mgw_pipeline* pipe, int* streamed);
/* Debug: the raw per-(group, CTA) (start, end) %globaltimer stamps of the
 * last engine launch, [G][cols][2] (cols = CTAs of all emulated ranks). */
int mgw_pipeline_stamps_raw(mgw_pipeline* pipe, uint64_t* out, size_t cap, size_t* cols_out);

/* Host-driven persistent comm engine for a REAL backward (SURVEY §8f row
 * 2; paper Algorithm 2 with the daemon thread on the GPU): instead of the
 * replay, the framework marks each group ready on its compute stream after
 * the backward of the group's layers (e.g. from autograd post-accumulate
 * hooks). Per iteration: mgw_engine_begin (launch the engine after the work
 * queued on after_stream; NULL = the legacy default stream), mgw_engine_mark_ready per group (1-thread kernel
 * on the compute stream; groups may complete in any order, they are reduced
 * FIFO in backward order), mgw_engine_join (stream waits until every group's
 * SGD is done). engine_ctas > 0 should be small so the backward keeps SMs.
 * Timing / destroy through mgw_pipeline_group_times / mgw_pipeline_stamps /
 * mgw_pipeline_destroy. */
int mgw_engine_create(mgw_plan* plan, float lr, int algo, int engine_ctas, int record_group_times,
                      mgw_pipeline** out);
int mgw_engine_begin(mgw_pipeline* engine, void* after_stream);
int mgw_engine_mark_ready(mgw_pipeline* engine, int group, void* stream);
int mgw_engine_join(mgw_pipeline* engine, void* stream);
/* Leave groups [0, n_tail) — the last ones the backward makes ready — to
 * the caller: the engine reduces groups [n_tail, G) only, and after
 * mgw_engine_join the caller runs mgw_group_allreduce for the tail groups at
 * full width (the backward no longer needs the SMs then). */
int mgw_engine_set_tail(mgw_pipeline* engine, int n_tail);
/* Synchronise the engine and report a barrier / ready timeout as an error. */
int mgw_engine_check(mgw_pipeline* engine);

/* Copy-engine mode for a real backward (P > 1): no SM is taken from the
 * backward. Each finished group's gradients travel to every peer's merge
 * arena as copy-engine (DMA) writes over NVLink the moment the group is
 * marked ready; after the backward ONE full-width kernel reduces every tile
 * in rank order from the local arena (own contribution in place), fused
 * with SGD. The merge plan sets the number of copies (the a of the
 * copy-engine cost model, mgw_calibrate_ce). Needs the gradients in one flat
 * buffer laid out like the merge layout (layer l at element offs[l], see
 * mgw_plan_group_span) and weights for every layer. Reduced values are
 * bit-identical to mgw_group_allreduce's (same rank-order arithmetic).
 *   begin(after_stream)   at the start of an iteration (the peers finished
 *                         reducing the previous one before any copy lands)
 *   mark_ready(g, stream) after group g's gradients were produced on stream
 *   join(stream)          after the backward: the reduce + SGD, `stream`
 *                         waits for it. */
typedef struct mgw_ce mgw_ce;
int mgw_ce_create(mgw_plan* plan, float lr, mgw_ce** out);
int mgw_ce_begin(mgw_ce* ce, void* after_stream);
int mgw_ce_mark_ready(mgw_ce* ce, int group, void* stream);
int mgw_ce_join(mgw_ce* ce, void* stream);
/* Groups [0, n_tail) (the last the backward makes ready) are left to the
 * caller (e.g. mgw_group_allreduce after the backward): no copy, no reduce.
 * Launch those fused kernels after mgw_ce_join on the same stream unless
 * mgw_ce_signals_without_sm: a fused launch pairs its CTAs with the peers'
 * and may hold every SM while waiting, which must not starve a peer's
 * signal kernel. */
int mgw_ce_set_tail(mgw_ce* ce, int n_tail);
/* 1 in *out when "iteration delivered" is signalled with stream memory
 * operations (cuStreamWriteValue64: no SM needed). Then the tail groups'
 * fused launches may go BEFORE mgw_ce_join and overlap the reduce; with 0
 * (a 1-thread signal kernel) they must follow it. */
int mgw_ce_signals_without_sm(const mgw_ce* ce, int* out);
/* Synchronise and report a timed-out wait as an error. */
int mgw_ce_check(mgw_ce* ce);
int mgw_ce_destroy(mgw_ce* ce);
/* Copy-engine calibration: per size, the median of `reps` timed device-to-
 * peer copies (rank -> rank+1; P = 1: local). */
int mgw_calibrate_ce(mgw_comm* comm, const uint64_t* sizes_bytes, size_t n, int warmup, int reps,
                     mgw_meas* out);

/* On-box calibration sweep (N1): for each size, warmup + reps timed runs
 * of the fused group kernel on a single-layer group of size/4 elements;
 * writes the median per size. Collective. */
int mgw_calibrate(mgw_comm* comm, const uint64_t* sizes_bytes, size_t n, int warmup, int reps,
                  int algo, mgw_meas* out);

/* Calibration of the persistent comm engine: per size, `reps` iterations of
 * an engine running ONE group of that size, made ready 100 us into the
 * iteration (the engine is already waiting, as in a pipeline); the median group
 * device duration (%globaltimer, first CTA start -> last CTA end) is the
 * sample (L2 evicted before every rep). This is the T(M) the planner sees in
 * engine pipelines. */
int mgw_calibrate_engine(mgw_comm* comm, const uint64_t* sizes_bytes, size_t n, int warmup,
                         int reps, int algo, int engine_ctas, mgw_meas* out);
/* The same with the gradient type of the groups (sizes stay in bytes). */
int mgw_calibrate_engine_ex(mgw_comm* comm, const uint64_t* sizes_bytes, size_t n, int warmup,
                            int reps, int algo, int engine_ctas, int dtype, mgw_meas* out);

/* Plain in-place sum all-reduce of a contiguous fp32 device buffer in rank
 * order (no scale, no SGD), through the same kernel. Collective. */
int mgw_allreduce(mgw_comm* comm, float* buf, size_t n_elems, int algo, void* stream);

/* Device counts / kernels launched by this library since load (evidence
 * for the bench's gpu_launches). */
uint64_t mgw_kernel_launches(void);

#ifdef __cplusplus
}
#endif

#endif /* MGWFBP_H_ */
