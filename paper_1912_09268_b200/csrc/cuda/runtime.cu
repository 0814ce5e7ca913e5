// mgwfbp-b200: device half of the C ABI (include/mgwfbp.h) — communicator
// (symmetric merge arenas mapped over NVLink with CUDA IPC), device plans
// (tile tables for every merge group), the standalone pack / unpack+SGD ops,
// the fused per-group all-reduce, the backward-replay pipeline captured as
// one CUDA graph per plan, and the on-box calibration sweep.
//
// Paper mapping: Algorithm 2 runs a comm daemon thread
// that pops layers and calls SynchonizedAllReduce(lb) on each normal layer;
// here the comm "thread" is a CUDA stream whose kernels wait on per-group
// events of the compute stream, FIFO in backward order — exactly the
// serialised schedule of reference timeline.hpp:128-154.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <string>
#include <cstdlib>
#include <condition_variable>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include <cuda.h>  // driver types only (cuStreamWriteValue64 is fetched with cudaGetDriverEntryPoint)
#include <cuda_runtime.h>

#include "capi_common.hpp"
#include "gradsched/errors.hpp"
#include "mgw_device.cuh"
#include "mgwfbp.h"
#include "nvls.hpp"

namespace mgw {

cudaError_t launch_nvls_group(const GroupLaunch& L, int ctas, cudaStream_t stream);
cudaError_t nvls_ctas_per_sm(int nranks, int* out);
cudaError_t launch_group_allreduce(const GroupLaunch& L, int ctas_per_rank, bool two_shot,
                                   bool loopback, cudaStream_t stream);
cudaError_t max_ctas_per_sm(int nranks, bool two_shot, bool loopback, int dtype, int* out);
cudaError_t launch_pack(const Tile* tiles, uint32_t n_tiles, float* const* grads, void* merge,
                        uint64_t begin, float scale, int dtype, int ctas, cudaStream_t stream);
cudaError_t launch_unpack_sgd(const Tile* tiles, uint32_t n_tiles, float* const* grads,
                              float* const* weights, const void* merge, uint64_t begin, float lr,
                              int epi, int dtype, int ctas, cudaStream_t stream);
cudaError_t launch_replay(unsigned long long* clock, unsigned long long deadline_ns, int first,
                          uint32_t* ready, cudaStream_t stream);
cudaError_t launch_engine(const EngineLaunch& E, int ctas, int ranks, cudaStream_t stream);
cudaError_t launch_replay_all(unsigned long long* clock, const unsigned long long* deadlines_ns,
                              uint32_t n, const uint32_t* pipe, uint32_t* flags,
                              cudaStream_t stream, int gate);
cudaError_t launch_mark_ready(const uint32_t* pipe, uint32_t* flags, uint32_t g,
                              cudaStream_t stream);
cudaError_t preload_kernels();
cudaError_t launch_ce(int what, const CeLaunch& C, int n_views, int ctas, cudaStream_t stream);
cudaError_t engine_ctas_per_sm(int nranks, int dtype, int* out);
cudaError_t launch_l2_flush(void* buf, size_t bytes, int ctas, cudaStream_t stream);

std::atomic<uint64_t> g_kernel_launches{0};

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw CudaFailure(std::string(what) + ": " + cudaGetErrorString(e));
  }
}

// Bad arguments are input errors (MGW_ERR_INPUT), like the reference's
// ValidationError.
void require(bool ok, const std::string& msg) {
  if (!ok) throw gradsched::ValidationError(msg);
}

struct IpcBlob {
  cudaIpcMemHandle_t arena;
  cudaIpcMemHandle_t signal;
};

}  // namespace
}  // namespace mgw

using mgw::ck;
using mgw::require;

struct mgw_comm {
  int rank = 0;
  int nranks = 1;
  int device = 0;
  bool loopback = false;
  size_t arena_elems = 0;  // per copy
  uint64_t oneshot_max = 512 * 1024;
  int num_sms = 148;
  uint32_t chunk_tiles = 16;  // max tiles of a CTA's pipelined chunk (mgw_comm_set_chunk_tiles)
  uint32_t min_chunks = 1;    // a CTA splits its tiles into at least this many chunks (mgw_comm_set_chunk_tiles)
  uint32_t credit_batch = 8;  // streamed: bulk items per published delivery count (mgw_comm_set_stream_batches)
  uint32_t ag_batch = 4;      // streamed two-shot: owned super-tiles per all-gather publication
  int protocol = MGW_PROTO_AUTO;  // mgw_comm_set_protocol: STREAM, CHUNKED or AUTO (P > 1 chunked,
                                 // P = 1 the TMA-fed engine)
  uint64_t ll_max = 64 << 10; // one-shot groups up to this many bytes use LL packets (mgw_comm_set_ll_max)
  int max_ctas = 0;           // cap on the CTAs of a standalone group launch (0: one per SM)
  uint64_t small_tile_max = 0; // groups below this many bytes use kTileElems / 4 tiles (mgw_comm_set_small_tile_max)
  uint32_t* host_err = nullptr;   // host-mapped error word (kernels raise it on a timeout)
  uint32_t* host_err_d = nullptr; // its device alias
  // own allocations (loopback: one per emulated rank)
  std::vector<float*> arenas;
  std::vector<uint32_t*> signals;
  std::vector<uint32_t*> states;
  // peer mappings opened through IPC (real mode)
  std::vector<void*> opened;
  float* peer_arena[mgw::kMaxRanks] = {};
  uint32_t* peer_signal[mgw::kMaxRanks] = {};
  bool peers_ready = false;
  cudaStream_t stream = nullptr;  // calibrate / plain all-reduce
  unsigned long long* d_clock = nullptr;  // calibration spin clock
  uint64_t ce_seq = 0;  // copy-engine mode iterations run on this communicator (identical on every rank)
  int occ_cache[2][2] = {{0, 0}, {0, 0}};  // [dtype][two_shot]           // CTAs/SM of the one-shot / two-shot kernel
  // NVLS (mgw_comm_nvls_*): multicast-bound buffer of one arena slot
  mgw::NvlsArena* nvls = nullptr;
  bool nvls_bound = false;
  uint64_t nvls_min = 0;       // AUTO: fp32 groups of at least this many bytes use NVLS (0: never)
  uint32_t nvls_chunk = 4;     // tiles per pipelined chunk of a CTA
  int nvls_occ = 0;            // resident NVLS CTAs per SM (occupancy query, cached)
  uint32_t nvls_skip = 0;      // profiling only (mgw_comm_set_nvls_skip): 1 skip pack/unpack, 2 skip the reduce
  // cached single-buffer plan for mgw_allreduce
  mgw_plan* ar_plan = nullptr;
  float* ar_buf = nullptr;
  size_t ar_n = 0;
};

struct mgw_plan {
  mgw_comm* comm = nullptr;
  size_t L = 0;
  int dtype = MGW_DTYPE_F32;        // gradient / arena element type
  size_t esize = 4;                 // bytes per gradient element
  uint64_t slot_stride = 0;         // arena slot stride in gradient elements
  int n_views = 1;
  std::vector<uint64_t> counts;
  std::vector<uint64_t> offs;       // L+1 padded element offsets
  std::vector<size_t> heads;        // G+1, ascending, heads[G] = L
  std::vector<uint32_t> tile_first; // G+1 tile ranges per group
  std::vector<uint32_t> ll_pkt;     // G: first LL packet of a small group (kNoLL: too large / no room)
  mgw::Tile* d_tiles = nullptr;
  float** d_grads = nullptr;        // n_views * L
  float** d_weights = nullptr;      // n_views * L
  std::vector<float*> h_grads;
  std::vector<float*> h_weights;
  int G() const { return static_cast<int>(heads.size()) - 1; }
};

struct mgw_pipeline {
  mgw_plan* plan = nullptr;
  cudaStream_t compute = nullptr;
  cudaStream_t comm = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  std::vector<cudaEvent_t> ready;
  std::vector<cudaEvent_t> g_start, g_end;
  unsigned long long* d_clock = nullptr;
  void* flush_buf = nullptr;
  size_t flush_bytes = 0;
  int iter_flush_value = 0x5a;
  bool timed_groups = false;
  int kernels_per_iter = 0;
  // persistent comm engine mode
  bool engine = false;
  int engine_ctas = 0;
  uint32_t* d_pipe = nullptr;             // ready count, iteration, exit count
  unsigned long long* d_stamps = nullptr; // [G][stamp_cols][2] per-CTA (start, end)
  size_t stamp_cols = 0;                  // CTAs (all emulated ranks) per stamp row
  int grid_y = 1;                         // emulated ranks of the engine grid (loopback)
  mgw::EngineGroup* d_groups = nullptr;   // G
  uint32_t* d_sched = nullptr;            // per-CTA participating groups, FIFO order (CSR)
  uint32_t* d_sched_off = nullptr;        // engine_ctas + 1 offsets into d_sched
  unsigned long long* d_deadlines = nullptr;  // G group-head ready times (ns), backward order
  uint32_t* d_ready = nullptr;            // G ready flags (iteration stamps)
  mgw::EngineLaunch args{};               // engine kernel arguments
  bool manual = false;                    // host-driven engine (real backward), no graph
  int tail_launch = 0;                    // replay pipelines, streamed protocol: groups [0, tail_launch)
                                          // run as chunked standalone launches after the engine
  cudaEvent_t replay_done = nullptr;
};

namespace mgw {
namespace {

void set_device(const mgw_comm* c) { ck(cudaSetDevice(c->device), "cudaSetDevice"); }

uint32_t* alloc_zero_u32(size_t words) {
  uint32_t* p = nullptr;
  ck(cudaMalloc(&p, words * sizeof(uint32_t)), "cudaMalloc(signal)");
  ck(cudaMemset(p, 0, words * sizeof(uint32_t)), "cudaMemset(signal)");
  return p;
}

// One slot of `elems` floats per source rank (push data path).
float* alloc_arena(size_t elems, int nranks) {
  float* p = nullptr;
  const size_t n = std::max<size_t>(static_cast<size_t>(nranks) * elems, 4);
  ck(cudaMalloc(&p, n * sizeof(float)), "cudaMalloc(arena)");
  ck(cudaMemset(p, 0, n * sizeof(float)), "cudaMemset(arena)");
  return p;
}

void init_common(mgw_comm* c, int device, size_t arena_bytes) {
  c->device = device;
  c->arena_elems = (arena_bytes / sizeof(float) + 3) & ~size_t{3};
  ck(cudaSetDevice(device), "cudaSetDevice");
  ck(cudaHostAlloc(&c->host_err, sizeof(uint32_t), cudaHostAllocMapped), "cudaHostAlloc(error word)");
  *c->host_err = 0;
  ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->host_err_d), c->host_err, 0), "error word alias");
  ck(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device), "sm count");
  ck(preload_kernels(), "preload kernels (lazy module loading would deadlock the engine)");
  ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream");
  ck(cudaMalloc(&c->d_clock, 2 * sizeof(unsigned long long)), "cudaMalloc(clock)");
  ck(cudaMemset(c->d_clock, 0, 2 * sizeof(unsigned long long)), "memset(clock)");
}

RankView make_view(const mgw_comm* c, int r, float* const* grads, float* const* weights) {
  RankView v{};
  for (int q = 0; q < c->nranks; ++q) {
    if (c->loopback) {
      v.arena[q] = c->arenas[q];
      v.signal[q] = c->signals[q];
    } else {
      v.arena[q] = c->peer_arena[q];
      v.signal[q] = c->peer_signal[q];
    }
  }
  v.state = c->states[c->loopback ? r : 0];
  v.host_err = c->host_err_d;
  v.grads = grads;
  v.weights = weights;
  v.arena_bytes = std::max<uint64_t>(static_cast<uint64_t>(c->nranks) * c->arena_elems, 4) * sizeof(float);
  v.rank = c->loopback ? r : c->rank;
  return v;
}

// Default one-shot/two-shot crossover, measured on B200 NVLink with the
// persistent engine (tools/probe_bw.py): one-shot pushes (P-1)*S bytes per
// rank behind one barrier, two-shot 2(P-1)/P*S behind two.
uint64_t default_oneshot_max(int nranks) {
  if (nranks <= 2) return 8ull << 20;
  if (nranks <= 4) return 3ull << 20;
  return 1ull << 20;
}

// Signal allocation: the flags, then one LL slot per source rank.
size_t signal_words(int nranks) {
  return kLLWord + static_cast<size_t>(nranks) * kLLSlotPackets * 2;
}

// Largest one-shot group that travels as LL packets (0 disables LL).
// Measured on B200 (tools/probe_bw.py, engine, LL vs barrier one-shot): LL
// wins up to 512 KiB at P = 2 (8.0 vs 10.7 us) and 128 KiB at P = 4 (8.5
// vs 12.4 us); LL sends 2(P-1) x the bytes, so P = 8 gets 32 KiB.
// Tuning knobs are C-ABI setters (mgw_comm_set_*), never environment
// variables: every rank must hold the same values.
uint64_t default_ll_max(int nranks) {
  if (nranks <= 2) return 512ull << 10;
  if (nranks <= 4) return 128ull << 10;
  return 32ull << 10;
}

// Groups below this many bytes are cut into kTileElems / 4 tiles so they
// spread over more CTAs. Measured on B200 (tools/probe_bw.py, engine): 1 MiB
// P = 2 one-shot 11.0 -> 9.9 us, 2 MiB P = 4 two-shot 23.4 -> 21.2 us; from
// 4 MiB on the 32 KiB tiles are as fast or faster (P = 2 8 MiB 24.2 vs 28.1).
constexpr uint64_t kDefaultSmallTileMax = 3ull << 20;

// NVLS: opt-in (mgw_comm_set_nvls) or forced (MGW_ALGO_NVLS); fp32 only,
// real ranks only (a multicast object spans distinct GPUs).
bool use_nvls(const mgw_comm* c, uint64_t bytes, int algo, int dtype) {
  if (algo == MGW_ALGO_NVLS) {
    require(c->nvls_bound, "MGW_ALGO_NVLS needs mgw_comm_nvls_create / _join / _bind first");
    require(dtype == MGW_DTYPE_F32, "MGW_ALGO_NVLS reduces fp32 gradients only");
    return true;
  }
  return algo == MGW_ALGO_AUTO && c->nvls_bound && c->nvls_min > 0 && bytes >= c->nvls_min &&
         dtype == MGW_DTYPE_F32 && c->nranks > 1;
}

// NVLS grid: one CTA per tile up to (resident CTAs per SM) x SMs, capped by
// mgw_comm_set_max_ctas.
int nvls_grid(mgw_comm* c, uint32_t n_tiles) {
  if (c->nvls_occ == 0) ck(nvls_ctas_per_sm(c->nranks, &c->nvls_occ), "nvls occupancy");
  int cap = std::min(std::max(1, c->nvls_occ) * c->num_sms, kMaxCtas);
  if (c->max_ctas > 0) cap = std::min(cap, c->max_ctas);
  return static_cast<int>(std::max<uint32_t>(1, std::min<uint32_t>(n_tiles, static_cast<uint32_t>(cap))));
}

bool use_two_shot(const mgw_comm* c, uint64_t bytes, int algo) {
  if (c->nranks == 1) return false;
  if (algo == MGW_ALGO_ONESHOT) return false;
  if (algo == MGW_ALGO_TWOSHOT) return true;
  return bytes > c->oneshot_max;
}

int grid_for(mgw_comm* c, uint32_t n_tiles, bool two_shot, int dtype = MGW_DTYPE_F32, bool ll = false) {
  int& occ = c->occ_cache[dtype == MGW_DTYPE_BF16 ? 1 : 0][two_shot ? 1 : 0];
  if (occ == 0) ck(max_ctas_per_sm(c->nranks, two_shot, c->loopback, dtype, &occ), "occupancy");
  int cap = std::max(1, occ) * c->num_sms;
  if (c->loopback) cap = std::max(1, cap / c->nranks);
  cap = std::min(cap, kMaxCtas);
  if (c->max_ctas > 0) cap = std::min(cap, c->max_ctas);
  const uint32_t units = two_shot ? (n_tiles + c->nranks - 1) / c->nranks
                                  : (ll ? n_tiles * kLLParts : n_tiles);
  return static_cast<int>(std::max<uint32_t>(1, std::min<uint32_t>(units, cap)));
}

uint64_t group_bytes(const mgw_plan* p, int g) {
  uint64_t s = 0;
  for (size_t l = p->heads[g]; l < p->heads[g + 1]; ++l) s += p->counts[l] * p->esize;
  return s;
}

// Fused pack -> all-reduce -> unpack+SGD for group g.
void launch_group(mgw_plan* p, int g, float lr, int epilogue, int algo, cudaStream_t stream,
                  bool force_chunked = false, unsigned long long* stamps = nullptr, uint32_t stamp_row = 0) {
  mgw_comm* c = p->comm;
  require(c->loopback || c->nranks == 1 || c->peers_ready,
          "communicator peers not opened (call mgw_comm_open_peers)");
  require(g >= 0 && g < p->G(), "group index out of range");
  GroupLaunch L{};
  L.tiles = p->d_tiles + p->tile_first[g];
  L.n_tiles = p->tile_first[g + 1] - p->tile_first[g];
  L.nranks = c->nranks;
  L.scale = 1.0f / static_cast<float>(c->nranks);
  L.lr = lr;
  L.epilogue = epilogue;
  L.slot_stride = p->slot_stride;
  L.chunk = c->chunk_tiles;
  L.min_chunks = c->min_chunks;
  L.stream = (!force_chunked && c->protocol == MGW_PROTO_STREAM) ? 1u : 0u;  // AUTO: chunked when standalone
  L.credit_batch = c->credit_batch;
  L.ag_batch = c->ag_batch;
  L.dtype = p->dtype;
  L.stamps = stamps;
  L.stamp_group = static_cast<uint32_t>(g);
  L.stamp_row = stamp_row;
  for (int r = 0; r < p->n_views; ++r) {
    L.views[r] = make_view(c, r, p->d_grads + static_cast<size_t>(r) * p->L,
                           p->d_weights + static_cast<size_t>(r) * p->L);
  }
  if (use_nvls(c, group_bytes(p, g), algo, p->dtype)) {
    L.nvls_uc = nvls_uc(c->nvls);
    L.nvls_mc = nvls_mc(c->nvls);
    L.chunk = c->nvls_chunk;
    L.nvls_skip = c->nvls_skip;
    L.nvls_elems = nvls_bytes(c->nvls) / sizeof(float);
    L.ll_pkt = kNoLL;
    ck(launch_nvls_group(L, nvls_grid(c, L.n_tiles), stream), "nvls group launch");
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
    return;
  }
  const bool two = use_two_shot(c, group_bytes(p, g), algo);
  L.ll_pkt = two ? kNoLL : p->ll_pkt[g];
  L.mbase = static_cast<uint32_t>(p->offs[p->heads[g]]);
  ck(launch_group_allreduce(L, grid_for(c, L.n_tiles, two, p->dtype, L.ll_pkt != kNoLL), two, c->loopback,
                            stream),
     "group_allreduce launch");
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

void check_barrier_flags(const mgw_comm* c) {
  for (uint32_t* st : c->states) {
    uint32_t flag = 0;
    ck(cudaMemcpy(&flag, st + kStateError, sizeof flag, cudaMemcpyDeviceToHost), "read barrier flag");
    if (flag != 0) throw CudaFailure("cross-rank wait timed out (a peer never arrived); the communicator is failed");
  }
}

void destroy_plan(mgw_plan* p) {
  if (p == nullptr) return;
  cudaFree(p->d_tiles);
  cudaFree(p->d_grads);
  cudaFree(p->d_weights);
  delete p;
}

mgw_plan* build_plan(mgw_comm* c, size_t L, float* const* grads, float* const* weights,
                     const uint64_t* counts, const uint8_t* tags, int dtype = MGW_DTYPE_F32) {
  require(c != nullptr, "comm is NULL");
  require(L >= 1, "plan needs at least one layer");
  require(grads != nullptr && counts != nullptr && tags != nullptr, "NULL plan arrays");
  require(tags[0] == 0, "the first layer cannot be merged (tags[0] must be 0)");
  set_device(c);
  // held by a unique_ptr until every check and allocation succeeded: any
  // throw below frees the plan and its device tables
  std::unique_ptr<mgw_plan, void (*)(mgw_plan*)> owner(new mgw_plan(), destroy_plan);
  mgw_plan* p = owner.get();
  p->comm = c;
  p->L = L;
  require(dtype == MGW_DTYPE_F32 || dtype == MGW_DTYPE_BF16, "dtype must be MGW_DTYPE_F32 or MGW_DTYPE_BF16");
  p->dtype = dtype;
  p->esize = dtype == MGW_DTYPE_BF16 ? 2 : 4;
  p->slot_stride = c->arena_elems * (sizeof(float) / p->esize);  // the arena is reinterpreted
  const uint64_t granule = 16 / p->esize;                         // layers start 16-byte aligned
  p->n_views = c->loopback ? c->nranks : 1;
  p->counts.assign(counts, counts + L);
  p->offs.resize(L + 1, 0);
  for (size_t l = 0; l < L; ++l) {
    require(tags[l] <= 1, "tags must be 0 or 1");
    require(counts[l] < (uint64_t{1} << 32), "layer too large (>= 2^32 elements)");
    p->offs[l + 1] = p->offs[l] + ((counts[l] + granule - 1) & ~(granule - 1));
    if (l == 0 || tags[l] == 0) p->heads.push_back(l);
  }
  p->heads.push_back(L);
  if (p->offs[L] > p->slot_stride) {
    throw gradsched::ValidationError("plan needs " + std::to_string(p->offs[L] * p->esize) +
                                     " arena bytes; communicator has " + std::to_string(c->arena_elems * 4));
  }
  require(p->offs[L] < (uint64_t{1} << 32), "model too large for 32-bit tile offsets");
  const size_t nv = static_cast<size_t>(p->n_views);
  p->h_grads.assign(grads, grads + nv * L);
  p->h_weights.assign(nv * L, nullptr);
  if (weights != nullptr) p->h_weights.assign(weights, weights + nv * L);

  std::vector<Tile> tiles;
  for (int g = 0; g + 1 < static_cast<int>(p->heads.size()); ++g) {
    p->tile_first.push_back(static_cast<uint32_t>(tiles.size()));
    // medium groups: smaller tiles spread the group over more CTAs
    uint64_t gbytes = 0;
    for (size_t l = p->heads[g]; l < p->heads[g + 1]; ++l) gbytes += counts[l] * p->esize;
    const uint64_t tile_elems = (c->nranks > 1 && gbytes < c->small_tile_max) ? kTileElems / 4 : kTileElems;
    for (size_t l = p->heads[g]; l < p->heads[g + 1]; ++l) {
      uint32_t flags = 0;
      for (size_t r = 0; r < nv; ++r) {
        if (reinterpret_cast<uintptr_t>(p->h_grads[r * L + l]) % 16) flags |= kGradUnaligned;
        if (reinterpret_cast<uintptr_t>(p->h_weights[r * L + l]) % 16) flags |= kWeightUnaligned;
        require(counts[l] == 0 || p->h_grads[r * L + l] != nullptr, "NULL gradient pointer");
      }
      for (uint64_t s = 0; s < counts[l]; s += tile_elems) {
        Tile t;
        t.layer = static_cast<uint32_t>(l) | flags;
        t.len = static_cast<uint32_t>(std::min<uint64_t>(tile_elems, counts[l] - s));
        t.src = static_cast<uint32_t>(s);
        t.moff = static_cast<uint32_t>(p->offs[l] + s);
        tiles.push_back(t);
      }
    }
  }
  p->tile_first.push_back(static_cast<uint32_t>(tiles.size()));
  require(L <= kLayerMask, "too many layers");
  // LL packets for the small groups, in backward (engine FIFO) order, while
  // the LL slot has room; 4 data bytes per packet, padded layout
  p->ll_pkt.assign(p->G(), kNoLL);
  if (c->nranks > 1) {
    uint64_t next = 0;
    for (int g = p->G() - 1; g >= 0; --g) {
      if (group_bytes(p, g) > c->ll_max) continue;
      const uint64_t pk = (p->offs[p->heads[g + 1]] - p->offs[p->heads[g]]) * p->esize / 4;
      if (next + pk > kLLSlotPackets) break;
      p->ll_pkt[g] = static_cast<uint32_t>(next);
      next += pk;
    }
  }
  ck(cudaMalloc(&p->d_tiles, std::max<size_t>(tiles.size(), 1) * sizeof(Tile)), "cudaMalloc(tiles)");
  if (!tiles.empty()) {
    ck(cudaMemcpy(p->d_tiles, tiles.data(), tiles.size() * sizeof(Tile), cudaMemcpyHostToDevice),
       "upload tiles");
  }
  ck(cudaMalloc(&p->d_grads, nv * L * sizeof(float*)), "cudaMalloc(grads table)");
  ck(cudaMalloc(&p->d_weights, nv * L * sizeof(float*)), "cudaMalloc(weights table)");
  ck(cudaMemcpy(p->d_grads, p->h_grads.data(), nv * L * sizeof(float*), cudaMemcpyHostToDevice),
     "upload grads table");
  ck(cudaMemcpy(p->d_weights, p->h_weights.data(), nv * L * sizeof(float*),
                cudaMemcpyHostToDevice),
     "upload weights table");
  return owner.release();
}

// Optional per-step host I/O captured into the pipeline graph (e2e runs).
struct StepIo {
  const void* h2d_src = nullptr;  // pinned host input (e.g. the step's gradients)
  void* h2d_dst = nullptr;
  size_t h2d_bytes = 0;
  void* d2h_dst = nullptr;        // pinned host result (e.g. a weight checksum)
  const void* d2h_src = nullptr;
  size_t d2h_bytes = 0;
};

mgw_pipeline* build_pipeline(mgw_plan* p, const double* t_b, double t_f, float lr, int algo,
                             bool timed, size_t l2_flush_bytes, int engine_ctas,
                             const StepIo& io = StepIo{}, bool gate_replay = false);

}  // namespace
}  // namespace mgw

extern "C" {

uint64_t mgw_kernel_launches(void) { return mgw::g_kernel_launches.load(); }

size_t mgw_comm_handle_size(void) { return sizeof(mgw::IpcBlob); }

int mgw_comm_create(int rank, int nranks, int device, size_t arena_bytes, mgw_comm** out) {
  MGW_TRY {
    require(out != nullptr, "out is NULL");
    require(nranks == 1 || nranks == 2 || nranks == 4 || nranks == 8, "nranks must be 1, 2, 4 or 8");
    require(rank >= 0 && rank < nranks, "rank out of range");
    auto* c = new mgw_comm();
    c->rank = rank;
    c->nranks = nranks;
    c->oneshot_max = mgw::default_oneshot_max(nranks);
    c->ll_max = mgw::default_ll_max(nranks);
    c->small_tile_max = mgw::kDefaultSmallTileMax;
    mgw::init_common(c, device, arena_bytes);
    c->arenas.push_back(mgw::alloc_arena(c->arena_elems, nranks));
    c->signals.push_back(mgw::alloc_zero_u32(mgw::signal_words(nranks)));
    c->states.push_back(mgw::alloc_zero_u32(mgw::kStateWords));
    ck(cudaDeviceSynchronize(), "init sync");
    c->peer_arena[rank] = c->arenas[0];
    c->peer_signal[rank] = c->signals[0];
    c->peers_ready = nranks == 1;
    *out = c;
  }
  MGW_CATCH
}

int mgw_comm_create_loopback(int nranks, int device, size_t arena_bytes, mgw_comm** out) {
  MGW_TRY {
    require(out != nullptr, "out is NULL");
    require(nranks == 1 || nranks == 2 || nranks == 4 || nranks == 8, "nranks must be 1, 2, 4 or 8");
    auto* c = new mgw_comm();
    c->nranks = nranks;
    c->oneshot_max = mgw::default_oneshot_max(nranks);
    c->ll_max = mgw::default_ll_max(nranks);
    c->small_tile_max = mgw::kDefaultSmallTileMax;
    c->loopback = true;
    mgw::init_common(c, device, arena_bytes);
    for (int r = 0; r < nranks; ++r) {
      c->arenas.push_back(mgw::alloc_arena(c->arena_elems, nranks));
      c->signals.push_back(mgw::alloc_zero_u32(mgw::signal_words(nranks)));
      c->states.push_back(mgw::alloc_zero_u32(mgw::kStateWords));
    }
    ck(cudaDeviceSynchronize(), "init sync");
    c->peers_ready = true;
    *out = c;
  }
  MGW_CATCH
}

int mgw_comm_export_handle(mgw_comm* c, void* handle_out) {
  MGW_TRY {
    require(c != nullptr && handle_out != nullptr && !c->loopback, "bad communicator/handle");
    mgw::set_device(c);
    mgw::IpcBlob blob;
    ck(cudaIpcGetMemHandle(&blob.arena, c->arenas[0]), "cudaIpcGetMemHandle(arena)");
    ck(cudaIpcGetMemHandle(&blob.signal, c->signals[0]), "cudaIpcGetMemHandle(signal)");
    std::memcpy(handle_out, &blob, sizeof blob);
  }
  MGW_CATCH
}

int mgw_comm_open_peers(mgw_comm* c, const void* all_handles) {
  MGW_TRY {
    require(c != nullptr && all_handles != nullptr && !c->loopback, "bad communicator/handles");
    mgw::set_device(c);
    const auto* blobs = static_cast<const mgw::IpcBlob*>(all_handles);
    for (int q = 0; q < c->nranks; ++q) {
      if (q == c->rank) continue;
      void* a = nullptr;
      void* s = nullptr;
      ck(cudaIpcOpenMemHandle(&a, blobs[q].arena, cudaIpcMemLazyEnablePeerAccess),
         "cudaIpcOpenMemHandle(arena)");
      ck(cudaIpcOpenMemHandle(&s, blobs[q].signal, cudaIpcMemLazyEnablePeerAccess),
         "cudaIpcOpenMemHandle(signal)");
      c->opened.push_back(a);
      c->opened.push_back(s);
      c->peer_arena[q] = static_cast<float*>(a);
      c->peer_signal[q] = static_cast<uint32_t*>(s);
    }
    c->peers_ready = true;
  }
  MGW_CATCH
}

int mgw_comm_num_peers(const mgw_comm* c, int* mapped) {
  MGW_TRY {
    require(c != nullptr && mapped != nullptr, "NULL argument");
    int n = 0;
    for (int q = 0; q < c->nranks; ++q) {
      if (c->loopback) {
        n += c->arenas.size() > static_cast<size_t>(q) ? 1 : 0;
      } else {
        n += (c->peer_arena[q] != nullptr && c->peer_signal[q] != nullptr) ? 1 : 0;
      }
    }
    *mapped = n;
  }
  MGW_CATCH
}

int mgw_comm_set_oneshot_max(mgw_comm* c, uint64_t bytes) {
  MGW_TRY {
    require(c != nullptr, "comm is NULL");
    c->oneshot_max = bytes;
  }
  MGW_CATCH
}

int mgw_comm_set_max_ctas(mgw_comm* c, int max_ctas) {
  MGW_TRY {
    require(c != nullptr && max_ctas >= 0, "bad communicator / CTA cap");
    c->max_ctas = max_ctas;
  }
  MGW_CATCH
}

int mgw_comm_set_ll_max(mgw_comm* c, uint64_t bytes) {
  MGW_TRY {
    require(c != nullptr, "comm is NULL");
    c->ll_max = bytes;
  }
  MGW_CATCH
}

int mgw_comm_set_small_tile_max(mgw_comm* c, uint64_t bytes) {
  MGW_TRY {
    require(c != nullptr, "comm is NULL");
    c->small_tile_max = bytes;
  }
  MGW_CATCH
}

int mgw_comm_set_chunk_tiles(mgw_comm* c, uint32_t max_tiles, uint32_t min_chunks) {
  MGW_TRY {
    require(c != nullptr && max_tiles >= 1 && min_chunks >= 1, "chunk tiles and min chunks must be >= 1");
    c->chunk_tiles = max_tiles;
    c->min_chunks = min_chunks;
  }
  MGW_CATCH
}

int mgw_comm_set_protocol(mgw_comm* c, int protocol) {
  MGW_TRY {
    require(c != nullptr, "comm is NULL");
    require(protocol == MGW_PROTO_STREAM || protocol == MGW_PROTO_CHUNKED || protocol == MGW_PROTO_AUTO,
            "protocol must be MGW_PROTO_STREAM, MGW_PROTO_CHUNKED or MGW_PROTO_AUTO");
    c->protocol = protocol;
  }
  MGW_CATCH
}

int mgw_comm_set_stream_batches(mgw_comm* c, uint32_t credit_batch, uint32_t ag_batch) {
  MGW_TRY {
    require(c != nullptr, "comm is NULL");
    require(credit_batch == 1 || credit_batch == 2 || credit_batch == 4 || credit_batch == 8,
            "credit_batch must be 1, 2, 4 or 8");
    require(ag_batch >= 1, "ag_batch must be >= 1");
    c->credit_batch = credit_batch;
    c->ag_batch = ag_batch;
  }
  MGW_CATCH
}

int mgw_comm_get_protocol(const mgw_comm* c, int* protocol) {
  MGW_TRY {
    require(c != nullptr && protocol != nullptr, "NULL argument");
    *protocol = c->protocol;
  }
  MGW_CATCH
}

int mgw_comm_get_tuning(const mgw_comm* c, uint64_t* oneshot_max, uint64_t* ll_max, uint64_t* small_tile_max,
                        uint32_t* chunk_tiles, uint32_t* min_chunks) {
  MGW_TRY {
    require(c != nullptr, "comm is NULL");
    if (oneshot_max) *oneshot_max = c->oneshot_max;
    if (ll_max) *ll_max = c->ll_max;
    if (small_tile_max) *small_tile_max = c->small_tile_max;
    if (chunk_tiles) *chunk_tiles = c->chunk_tiles;
    if (min_chunks) *min_chunks = c->min_chunks;
  }
  MGW_CATCH
}

int mgw_comm_error(const mgw_comm* c, int* failed) {
  MGW_TRY {
    require(c != nullptr && failed != nullptr, "NULL argument");
    *failed = *reinterpret_cast<volatile const uint32_t*>(c->host_err) != 0 ? 1 : 0;
  }
  MGW_CATCH
}

int mgw_comm_get_oneshot_max(const mgw_comm* c, uint64_t* bytes) {
  MGW_TRY {
    require(c != nullptr && bytes != nullptr, "comm / out is NULL");
    *bytes = c->oneshot_max;
  }
  MGW_CATCH
}

size_t mgw_nvls_handle_size(void) { return mgw::kNvlsBlobBytes; }

int mgw_comm_nvls_supported(const mgw_comm* c, int* supported) {
  MGW_TRY {
    require(c != nullptr && supported != nullptr, "NULL argument");
    *supported = (!c->loopback && c->nranks > 1 && mgw::nvls_supported(c->device)) ? 1 : 0;
  }
  MGW_CATCH
}

int mgw_comm_nvls_create(mgw_comm* c, void* handle_out) {
  MGW_TRY {
    require(c != nullptr && handle_out != nullptr, "NULL argument");
    require(!c->loopback && c->nranks > 1, "NVLS needs a real communicator of P > 1 ranks");
    require(c->nvls == nullptr, "NVLS already set up on this communicator");
    require(c->peers_ready, "open the peers (mgw_comm_open_peers) before NVLS");
    mgw::set_device(c);
    c->nvls = mgw::nvls_create(c->device, c->rank, c->nranks, c->arena_elems * sizeof(float), handle_out);
  }
  MGW_CATCH
}

int mgw_comm_nvls_join(mgw_comm* c, const void* handle0) {
  MGW_TRY {
    require(c != nullptr && handle0 != nullptr && c->nvls != nullptr, "call mgw_comm_nvls_create first");
    mgw::set_device(c);
    try {
      mgw::nvls_join(c->nvls, handle0);
    } catch (...) {  // leave the communicator without NVLS (a later create may retry)
      mgw::nvls_destroy(c->nvls);
      c->nvls = nullptr;
      throw;
    }
  }
  MGW_CATCH
}

int mgw_comm_nvls_bind(mgw_comm* c) {
  MGW_TRY {
    require(c != nullptr && c->nvls != nullptr, "call mgw_comm_nvls_create / _join first");
    mgw::set_device(c);
    try {
      mgw::nvls_bind(c->nvls);
    } catch (...) {
      mgw::nvls_destroy(c->nvls);
      c->nvls = nullptr;
      throw;
    }
    c->nvls_bound = true;
  }
  MGW_CATCH
}

int mgw_comm_nvls_ready(const mgw_comm* c, int* ready) {
  MGW_TRY {
    require(c != nullptr && ready != nullptr, "NULL argument");
    *ready = c->nvls_bound ? 1 : 0;
  }
  MGW_CATCH
}

int mgw_comm_set_nvls(mgw_comm* c, uint64_t min_bytes, uint32_t chunk_tiles) {
  MGW_TRY {
    require(c != nullptr, "comm is NULL");
    require(min_bytes == 0 || c->nvls_bound, "NVLS is not set up on this communicator");
    require(chunk_tiles >= 1 && chunk_tiles <= 16, "chunk_tiles must be in [1, 16]");
    c->nvls_min = min_bytes;
    c->nvls_chunk = chunk_tiles;
  }
  MGW_CATCH
}

int mgw_pipeline_streamed(const mgw_pipeline* pipe, int* streamed) {
  MGW_TRY {
    require(pipe != nullptr && streamed != nullptr, "NULL argument");
    *streamed = pipe->engine && pipe->args.stream ? 1 : 0;
  }
  MGW_CATCH
}

int mgw_comm_set_nvls_skip(mgw_comm* c, uint32_t mask) {
  MGW_TRY {
    require(c != nullptr && mask <= 3, "mask must be 0..3");
    c->nvls_skip = mask;
  }
  MGW_CATCH
}

int mgw_comm_destroy(mgw_comm* c) {
  MGW_TRY {
    if (c == nullptr) return 0;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    mgw::destroy_plan(c->ar_plan);
    mgw::nvls_destroy(c->nvls);
    for (void* p : c->opened) cudaIpcCloseMemHandle(p);
    for (float* a : c->arenas) cudaFree(a);
    for (uint32_t* s : c->signals) cudaFree(s);
    for (uint32_t* s : c->states) cudaFree(s);
    if (c->stream) cudaStreamDestroy(c->stream);
    if (c->d_clock) cudaFree(c->d_clock);
    if (c->host_err) cudaFreeHost(c->host_err);
    delete c;
  }
  MGW_CATCH
}

int mgw_plan_create(mgw_comm* comm, size_t L, float* const* grads, float* const* weights,
                    const uint64_t* counts, const uint8_t* tags, mgw_plan** out) {
  MGW_TRY {
    require(out != nullptr, "out is NULL");
    *out = mgw::build_plan(comm, L, grads, weights, counts, tags);
  }
  MGW_CATCH
}

int mgw_plan_create_ex(mgw_comm* comm, size_t L, void* const* grads, float* const* weights,
                       const uint64_t* counts, const uint8_t* tags, int dtype, mgw_plan** out) {
  MGW_TRY {
    require(out != nullptr, "out is NULL");
    // the layer tables hold untyped device pointers; kernels reinterpret
    // them as the plan's element type
    *out = mgw::build_plan(comm, L, reinterpret_cast<float* const*>(grads), weights, counts, tags, dtype);
  }
  MGW_CATCH
}

int mgw_plan_destroy(mgw_plan* plan) {
  MGW_TRY {
    if (plan) cudaSetDevice(plan->comm->device);
    mgw::destroy_plan(plan);
  }
  MGW_CATCH
}

int mgw_plan_num_groups(const mgw_plan* plan, int* n) {
  MGW_TRY {
    require(plan != nullptr && n != nullptr, "NULL argument");
    *n = plan->G();
  }
  MGW_CATCH
}

int mgw_plan_group_span(const mgw_plan* p, int g, uint64_t* begin, uint64_t* count,
                        uint64_t* bytes) {
  MGW_TRY {
    require(p != nullptr && g >= 0 && g < p->G(), "bad plan/group");
    if (begin) *begin = p->offs[p->heads[g]];
    if (count) *count = p->offs[p->heads[g + 1]] - p->offs[p->heads[g]];
    if (bytes) *bytes = mgw::group_bytes(p, g);
  }
  MGW_CATCH
}

int mgw_pack(mgw_plan* p, int g, float scale, void* merge_buf, void* stream) {
  MGW_TRY {
    require(p != nullptr && merge_buf != nullptr && g >= 0 && g < p->G(), "bad pack arguments");
    mgw::set_device(p->comm);
    const uint32_t n = p->tile_first[g + 1] - p->tile_first[g];
    const int ctas = static_cast<int>(std::max<uint32_t>(1, std::min<uint32_t>(n, 4 * p->comm->num_sms)));
    ck(mgw::launch_pack(p->d_tiles + p->tile_first[g], n, p->d_grads, merge_buf,
                        p->offs[p->heads[g]], scale, p->dtype, ctas, static_cast<cudaStream_t>(stream)),
       "pack launch");
    mgw::g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  }
  MGW_CATCH
}

int mgw_unpack_sgd(mgw_plan* p, int g, const void* merge_buf, float lr, int write_grad,
                   void* stream) {
  MGW_TRY {
    require(p != nullptr && merge_buf != nullptr && g >= 0 && g < p->G(), "bad unpack arguments");
    mgw::set_device(p->comm);
    const uint32_t n = p->tile_first[g + 1] - p->tile_first[g];
    const int ctas = static_cast<int>(std::max<uint32_t>(1, std::min<uint32_t>(n, 4 * p->comm->num_sms)));
    const int epi = MGW_SGD | (write_grad ? MGW_WRITE_GRAD : 0);
    ck(mgw::launch_unpack_sgd(p->d_tiles + p->tile_first[g], n, p->d_grads, p->d_weights,
                              merge_buf, p->offs[p->heads[g]], lr, epi, p->dtype, ctas,
                              static_cast<cudaStream_t>(stream)),
       "unpack launch");
    mgw::g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  }
  MGW_CATCH
}

int mgw_group_allreduce(mgw_plan* p, int g, float lr, int epilogue, int algo, void* stream) {
  MGW_TRY {
    require(p != nullptr, "plan is NULL");
    mgw::set_device(p->comm);
    mgw::launch_group(p, g, lr, epilogue, algo, static_cast<cudaStream_t>(stream));
  }
  MGW_CATCH
}

int mgw_allreduce(mgw_comm* c, float* buf, size_t n, int algo, void* stream) {
  MGW_TRY {
    require(c != nullptr && buf != nullptr && n > 0 && !c->loopback, "bad all-reduce arguments");
    mgw::set_device(c);
    if (c->ar_plan == nullptr || c->ar_buf != buf || c->ar_n != n) {
      mgw::destroy_plan(c->ar_plan);
      c->ar_plan = nullptr;
      const uint64_t cnt = n;
      const uint8_t tag = 0;
      float* g[1] = {buf};
      c->ar_plan = mgw::build_plan(c, 1, g, nullptr, &cnt, &tag);
      c->ar_buf = buf;
      c->ar_n = n;
    }
    // A plain SUM all-reduce: same kernel, pack scale 1, result written
    // back into buf, no SGD.
    mgw_plan* p = c->ar_plan;
    mgw::GroupLaunch L{};
    L.tiles = p->d_tiles;
    L.n_tiles = p->tile_first[1];
    L.nranks = c->nranks;
    L.scale = 1.0f;
    L.lr = 0.0f;
    L.epilogue = MGW_WRITE_GRAD;
    L.slot_stride = p->slot_stride;
    L.chunk = c->chunk_tiles;
    L.min_chunks = c->min_chunks;
    L.stream = c->protocol == MGW_PROTO_STREAM ? 1u : 0u;
    L.credit_batch = c->credit_batch;
    L.ag_batch = c->ag_batch;
    L.dtype = MGW_DTYPE_F32;
    L.ll_pkt = mgw::kNoLL;
    L.mbase = 0;
    L.views[0] = mgw::make_view(c, 0, p->d_grads, p->d_weights);
    if (mgw::use_nvls(c, static_cast<uint64_t>(n) * 4, algo, MGW_DTYPE_F32)) {
      L.nvls_uc = mgw::nvls_uc(c->nvls);
      L.nvls_mc = mgw::nvls_mc(c->nvls);
      L.chunk = c->nvls_chunk;
      L.nvls_skip = c->nvls_skip;
      L.nvls_elems = mgw::nvls_bytes(c->nvls) / sizeof(float);
      ck(mgw::launch_nvls_group(L, mgw::nvls_grid(c, L.n_tiles), static_cast<cudaStream_t>(stream)),
         "nvls all-reduce launch");
      mgw::g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
      return 0;
    }
    const bool two = mgw::use_two_shot(c, static_cast<uint64_t>(n) * 4, algo);
    ck(mgw::launch_group_allreduce(L, mgw::grid_for(c, L.n_tiles, two), two, false,
                                   static_cast<cudaStream_t>(stream)),
       "allreduce launch");
    mgw::g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  }
  MGW_CATCH
}

int mgw_calibrate(mgw_comm* c, const uint64_t* sizes, size_t n, int warmup, int reps, int algo,
                  mgw_meas* out) {
  MGW_TRY {
    require(c != nullptr && sizes != nullptr && out != nullptr && reps >= 1, "bad calibrate args");
    require(!c->loopback, "calibration runs on a real communicator");
    mgw::set_device(c);
    uint64_t max_bytes = 16;
    for (size_t i = 0; i < n; ++i) max_bytes = std::max(max_bytes, sizes[i]);
    const size_t max_elems = (max_bytes + 3) / 4;
    float* grad = nullptr;
    float* w = nullptr;
    ck(cudaMalloc(&grad, max_elems * sizeof(float)), "cudaMalloc(calib grad)");
    ck(cudaMalloc(&w, max_elems * sizeof(float)), "cudaMalloc(calib w)");
    ck(cudaMemset(grad, 0, max_elems * sizeof(float)), "memset");
    ck(cudaMemset(w, 0, max_elems * sizeof(float)), "memset");
    std::vector<cudaEvent_t> ev(2 * static_cast<size_t>(reps));
    for (auto& e : ev) ck(cudaEventCreate(&e), "event");
    std::vector<float> ms(reps);
    try {
      for (size_t i = 0; i < n; ++i) {
        const uint64_t cnt = (sizes[i] + 3) / 4;
        const uint8_t tag = 0;
        float* gp[1] = {grad};
        float* wp[1] = {w};
        mgw_plan* p = mgw::build_plan(c, 1, gp, wp, &cnt, &tag);
        // Hold the stream with a spin so every rep below is already queued
        // when the GPU reaches it: the event-to-event times then measure
        // the device-side cost (kernel + stream gap), not host launch latency.
        const unsigned long long spin_ns = 100000ull + 30000ull * (warmup + reps);
        ck(mgw::launch_replay(c->d_clock, spin_ns, 1, nullptr, c->stream), "calibration spin");
        for (int k = 0; k < warmup; ++k) mgw::launch_group(p, 0, 0.0f, MGW_SGD, algo, c->stream);
        for (int k = 0; k < reps; ++k) {
          ck(cudaEventRecord(ev[2 * k], c->stream), "record");
          mgw::launch_group(p, 0, 0.0f, MGW_SGD, algo, c->stream);
          ck(cudaEventRecord(ev[2 * k + 1], c->stream), "record");
        }
        ck(cudaStreamSynchronize(c->stream), "calibrate sync");
        for (int k = 0; k < reps; ++k) {
          ck(cudaEventElapsedTime(&ms[k], ev[2 * k], ev[2 * k + 1]), "elapsed");
        }
        std::sort(ms.begin(), ms.end());
        const double med = reps % 2 ? ms[reps / 2] : 0.5 * (ms[reps / 2 - 1] + ms[reps / 2]);
        out[i].size_bytes = sizes[i];
        out[i].time_sec = med * 1e-3;
        mgw::destroy_plan(p);
      }
      mgw::check_barrier_flags(c);
    } catch (...) {
      for (auto& e : ev) cudaEventDestroy(e);
      cudaFree(grad);
      cudaFree(w);
      throw;
    }
    for (auto& e : ev) cudaEventDestroy(e);
    cudaFree(grad);
    cudaFree(w);
  }
  MGW_CATCH
}

int mgw_pipeline_create(mgw_plan* p, const double* t_b, double t_f, float lr, int algo,
                        int record_group_times, size_t l2_flush_bytes, int engine_ctas,
                        mgw_pipeline** out) {
  MGW_TRY {
    require(p != nullptr && t_b != nullptr && out != nullptr, "bad pipeline arguments");
    *out = mgw::build_pipeline(p, t_b, t_f, lr, algo, record_group_times != 0, l2_flush_bytes,
                               engine_ctas);
  }
  MGW_CATCH
}

int mgw_pipeline_create_io(mgw_plan* p, const double* t_b, double t_f, float lr, int algo,
                           int record_group_times, size_t l2_flush_bytes, int engine_ctas,
                           const void* h2d_src, void* h2d_dst, size_t h2d_bytes, void* d2h_dst,
                           const void* d2h_src, size_t d2h_bytes, mgw_pipeline** out) {
  MGW_TRY {
    require(p != nullptr && t_b != nullptr && out != nullptr, "bad pipeline arguments");
    require(h2d_bytes == 0 || (h2d_src != nullptr && h2d_dst != nullptr), "bad h2d buffers");
    require(d2h_bytes == 0 || (d2h_src != nullptr && d2h_dst != nullptr), "bad d2h buffers");
    mgw::StepIo io;
    io.h2d_src = h2d_src;
    io.h2d_dst = h2d_dst;
    io.h2d_bytes = h2d_bytes;
    io.d2h_dst = d2h_dst;
    io.d2h_src = d2h_src;
    io.d2h_bytes = d2h_bytes;
    *out = mgw::build_pipeline(p, t_b, t_f, lr, algo, record_group_times != 0, l2_flush_bytes,
                               engine_ctas, io);
  }
  MGW_CATCH
}

}  // extern "C"

namespace mgw {
namespace {

// Persistent-engine resources of a pipeline: group table, ready flags,
// counters, stamps, and the kernel arguments (fixed for the pipeline's life).
// Loopback communicators run ONE engine grid (ctas, P) for all emulated
// ranks; the replay's ready flags are shared by them.
// The engine's protocol. AUTO: chunked at P > 1 — measured, it gives the
// shorter iteration for every MG-WFBP plan (replayed BERT-large N = 2 / 4
// 33.826 / 33.949 ms against 33.832 / 33.964 streamed; comm-bound regime
// 1-4 % faster); the streamed protocol only wins drains of
// many small groups that are all ready at once (WFBP plans in the
// comm-bound regime, the standalone drain). P = 1: the TMA-fed engine.
bool engine_streamed(const mgw_comm* c) {
  if (c->protocol == MGW_PROTO_STREAM) return true;
  if (c->protocol == MGW_PROTO_CHUNKED) return false;
  return c->nranks == 1;
}

void setup_engine(mgw_pipeline* pipe, mgw_plan* p, int algo, int engine_ctas, float lr, bool timed) {
  mgw_comm* c = p->comm;
  const int G = p->G();
  int occ = 1;
  ck(engine_ctas_per_sm(c->nranks, p->dtype, &occ), "engine occupancy");
  // The engine runs concurrently with the compute stream, whose kernels must
  // still find SMs: measured on B200, a 1-thread replay kernel is NOT
  // scheduled next to engine CTAs when every SM holds one (the engine then
  // waits forever for a ready signal), so kFreeSms SMs are always left
  // without an engine CTA. A real backward needs SMs too (use few CTAs).
  // Every CTA of the grid must be resident at once (cross-rank barriers pair
  // CTA b with CTA b of every peer): at most one CTA per SM, fewer CTAs than
  // SMs.
  constexpr int kFreeSms = 8;
  pipe->grid_y = c->loopback ? c->nranks : 1;
  const int cap = std::max(1, std::min({kMaxCtas, (std::max(1, occ) * c->num_sms - 1) / pipe->grid_y,
                                        (c->num_sms - kFreeSms) / pipe->grid_y}));
  pipe->engine_ctas = std::min(cap, engine_ctas < 0 ? cap : engine_ctas);
  const size_t g1 = static_cast<size_t>(std::max(G, 1));
  pipe->stamp_cols = static_cast<size_t>(pipe->engine_ctas) * pipe->grid_y;
  ck(cudaMalloc(&pipe->d_pipe, 4 * sizeof(uint32_t)), "cudaMalloc(pipe)");
  ck(cudaMemset(pipe->d_pipe, 0, 4 * sizeof(uint32_t)), "memset(pipe)");
  ck(cudaMalloc(&pipe->d_ready, g1 * sizeof(uint32_t)), "cudaMalloc(ready)");
  ck(cudaMemset(pipe->d_ready, 0, g1 * sizeof(uint32_t)), "memset(ready)");
  if (timed) {
    const size_t n = 2 * g1 * pipe->stamp_cols;
    ck(cudaMalloc(&pipe->d_stamps, n * sizeof(unsigned long long)), "cudaMalloc(stamps)");
    ck(cudaMemset(pipe->d_stamps, 0, n * sizeof(unsigned long long)), "memset(stamps)");
  }
  // Groups in FIFO (backward) order rotate over the CTAs: group k starts at
  // the CTA after the last one group k-1 used (a pure function of the plan
  // and the CTA count, so identical on every rank).
  const uint32_t ncta = static_cast<uint32_t>(pipe->engine_ctas);
  std::vector<EngineGroup> groups(G);
  uint64_t next = 0;
  for (int g = G - 1; g >= 0; --g) {
    EngineGroup& e = groups[g];
    e.tile_first = p->tile_first[g];
    e.n_tiles = p->tile_first[g + 1] - p->tile_first[g];
    e.two_shot = use_two_shot(c, group_bytes(p, g), algo) ? 1u : 0u;
    e.ll_pkt = e.two_shot ? kNoLL : p->ll_pkt[g];
    e.mbase = static_cast<uint32_t>(p->offs[p->heads[g]]);
    const uint32_t P = static_cast<uint32_t>(c->nranks);
    e.units = (P > 1 && e.two_shot) ? (e.n_tiles + P - 1) / P
                                    : (P > 1 && e.ll_pkt != kNoLL ? e.n_tiles * kLLParts : e.n_tiles);
    e.cta0 = static_cast<uint32_t>(next % ncta);
    next += std::min<uint32_t>(e.units, ncta);
  }
  ck(cudaMalloc(&pipe->d_groups, g1 * sizeof(EngineGroup)), "cudaMalloc(groups)");
  if (G > 0) {
    ck(cudaMemcpy(pipe->d_groups, groups.data(), G * sizeof(EngineGroup), cudaMemcpyHostToDevice),
       "upload groups");
  }
  // Per-CTA schedules: CTA b's participating groups in FIFO order (CSR), so
  // a CTA never walks the groups it has no unit in (measured: ~0.15 us per
  // skipped group even from shared memory; GoogLeNet's CTAs take part in 7
  // of 173 groups). Identical on every rank (a function of plan and grid).
  std::vector<uint32_t> off(ncta + 1, 0), sched;
  {
    std::vector<std::vector<uint32_t>> per(ncta);
    for (int g = G - 1; g >= 0; --g) {
      const uint32_t u = std::min<uint32_t>(groups[g].units, ncta);
      for (uint32_t k = 0; k < u; ++k) per[(groups[g].cta0 + k) % ncta].push_back(static_cast<uint32_t>(g));
    }
    for (uint32_t b = 0; b < ncta; ++b) {
      off[b + 1] = off[b] + static_cast<uint32_t>(per[b].size());
      sched.insert(sched.end(), per[b].begin(), per[b].end());
    }
  }
  ck(cudaMalloc(&pipe->d_sched_off, off.size() * sizeof(uint32_t)), "cudaMalloc(schedule offsets)");
  ck(cudaMemcpy(pipe->d_sched_off, off.data(), off.size() * sizeof(uint32_t), cudaMemcpyHostToDevice),
     "upload schedule offsets");
  ck(cudaMalloc(&pipe->d_sched, std::max<size_t>(sched.size(), 1) * sizeof(uint32_t)), "cudaMalloc(schedule)");
  if (!sched.empty()) {
    ck(cudaMemcpy(pipe->d_sched, sched.data(), sched.size() * sizeof(uint32_t), cudaMemcpyHostToDevice),
       "upload schedule");
  }
  EngineLaunch& E = pipe->args;
  E = EngineLaunch{};
  for (int r = 0; r < p->n_views; ++r) {
    E.views[r] = make_view(c, r, p->d_grads + static_cast<size_t>(r) * p->L,
                           p->d_weights + static_cast<size_t>(r) * p->L);
  }
  E.tiles = p->d_tiles;
  E.groups = pipe->d_groups;
  E.sched = pipe->d_sched;
  E.sched_off = pipe->d_sched_off;
  E.G = static_cast<uint32_t>(G);
  E.nranks = c->nranks;
  E.scale = 1.0f / static_cast<float>(c->nranks);
  E.lr = lr;
  E.epilogue = MGW_SGD;
  E.slot_stride = p->slot_stride;
  E.chunk = c->chunk_tiles;
  E.min_chunks = c->min_chunks;
  E.stream = engine_streamed(c) ? 1u : 0u;
  E.credit_batch = c->credit_batch;
  E.ag_batch = c->ag_batch;
  E.dtype = p->dtype;
  E.pipe = pipe->d_pipe;
  E.ready = pipe->d_ready;
  E.no_wait = 0;
  E.stamps = timed ? pipe->d_stamps : nullptr;
}

// Reduce the per-CTA stamps of the last engine launch to (start, end) per
// group: the earliest CTA start and the latest CTA end (0, 0 for groups no
// CTA takes part in).
void read_group_stamps(mgw_pipeline* pipe, std::vector<unsigned long long>& out) {
  const int G = pipe->plan->G();
  std::vector<unsigned long long> raw(2 * static_cast<size_t>(G) * pipe->stamp_cols);
  if (!raw.empty()) {
    ck(cudaMemcpy(raw.data(), pipe->d_stamps, raw.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost),
       "read stamps");
  }
  out.assign(2 * static_cast<size_t>(G), 0ull);
  for (int g = 0; g < G; ++g) {
    unsigned long long lo = ~0ull, hi = 0;
    for (size_t k = 0; k < pipe->stamp_cols; ++k) {
      const unsigned long long a = raw[(g * pipe->stamp_cols + k) * 2];
      const unsigned long long b = raw[(g * pipe->stamp_cols + k) * 2 + 1];
      if (a == 0 || b == 0) continue;
      lo = std::min(lo, a);
      hi = std::max(hi, b);
    }
    if (hi > 0) {
      out[2 * g] = lo;
      out[2 * g + 1] = hi;
    }
  }
}

// Backward-replay pipeline as one CUDA graph per iteration. engine_ctas == 0:
// one fused kernel launch per group, each waiting on its head's ready event;
// engine_ctas != 0: ONE persistent engine kernel (engine_ctas CTAs, < 0 =
// one per SM) that the replay kernels feed through a device ready counter.
mgw_pipeline* build_pipeline(mgw_plan* p, const double* t_b, double t_f, float lr, int algo,
                             bool timed, size_t l2_flush_bytes, int engine_ctas, const StepIo& io,
                             bool gate_replay) {
  {
    require(t_f >= 0.0, "t_f must be >= 0");
    require(!p->comm->loopback || engine_ctas != 0,
            "loopback pipelines run the persistent engine (engine_ctas != 0)");
    set_device(p->comm);
    const size_t L = p->L;
    // Ready time of every layer, reference timeline.hpp:99-108 / planner.hpp:67-70.
    std::vector<double> tau_b(L);
    tau_b[L - 1] = t_f;
    for (size_t i = L - 1; i-- > 0;) tau_b[i] = tau_b[i + 1] + t_b[i + 1];

    auto* pipe = new mgw_pipeline();
    pipe->plan = p;
    pipe->timed_groups = timed;
    pipe->engine = engine_ctas != 0;
    const int G = p->G();
    mgw_comm* c = p->comm;
    if (pipe->engine) {
      setup_engine(pipe, p, algo, engine_ctas, lr, timed);
      // Streamed protocol: it wins where groups follow each other and loses
      // on an isolated large group — the last group the
      // backward makes ready is exactly that, and the only one exposed. It
      // runs as a chunked standalone launch (full grid) after the engine and
      // the replay; the engine takes groups [1, G).
      if (c->nranks > 1 && pipe->args.stream && G > 1) {
        pipe->tail_launch = 1;
        pipe->args.g_lo = 1;
      }
      // ready time of every group head, in backward (comm) order
      std::vector<unsigned long long> dl;
      for (int g = G - 1; g >= 0; --g) {
        const size_t head = p->heads[g];
        dl.push_back(static_cast<unsigned long long>(std::llround((tau_b[head] + t_b[head]) * 1e9)));
      }
      ck(cudaMalloc(&pipe->d_deadlines, std::max<size_t>(dl.size(), 1) * sizeof(unsigned long long)),
         "cudaMalloc(deadlines)");
      ck(cudaMemcpy(pipe->d_deadlines, dl.data(), dl.size() * sizeof(unsigned long long),
                    cudaMemcpyHostToDevice),
         "upload deadlines");
    }
    ck(cudaStreamCreateWithFlags(&pipe->compute, cudaStreamNonBlocking), "stream");
    ck(cudaStreamCreateWithFlags(&pipe->comm, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreateWithFlags(&pipe->fork, cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&pipe->join, cudaEventDisableTiming), "event");
    pipe->ready.resize(pipe->engine ? 0 : G);
    for (auto& e : pipe->ready) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    if (pipe->timed_groups && !pipe->engine) {
      pipe->g_start.resize(G);
      pipe->g_end.resize(G);
      for (auto& e : pipe->g_start) ck(cudaEventCreate(&e), "event");
      for (auto& e : pipe->g_end) ck(cudaEventCreate(&e), "event");
    }
    ck(cudaMalloc(&pipe->d_clock, 2 * sizeof(unsigned long long)), "cudaMalloc(clock)");
    ck(cudaMemset(pipe->d_clock, 0, 2 * sizeof(unsigned long long)), "memset(clock)");
    if (l2_flush_bytes > 0) {
      ck(cudaMalloc(&pipe->flush_buf, l2_flush_bytes), "cudaMalloc(l2 flush)");
      ck(cudaMemset(pipe->flush_buf, 0, l2_flush_bytes), "memset(l2 flush)");  // the flush reads it
      pipe->flush_bytes = l2_flush_bytes;
    }

    ck(cudaStreamBeginCapture(pipe->compute, cudaStreamCaptureModeThreadLocal), "begin capture");
    try {
      ck(cudaEventRecord(pipe->fork, pipe->compute), "fork");
      ck(cudaStreamWaitEvent(pipe->comm, pipe->fork, 0), "fork wait");
      if (io.h2d_bytes > 0) {
        // the step's input arrives on the comm branch while the compute
        // stream replays the forward pass; every group kernel follows it
        ck(cudaMemcpyAsync(io.h2d_dst, io.h2d_src, io.h2d_bytes, cudaMemcpyHostToDevice, pipe->comm),
           "h2d input");
      }
      if (pipe->flush_bytes > 0) {
        // The comm stream is idle until the first group is ready: evict L2
        // there while the compute stream replays the forward pass — on all
        // but 8 SMs (a full-grid flush kept the 1-thread replay kernel from
        // being scheduled; 16 CTAs took ~170 us, longer than a short
        // forward, and delayed the engine).
        const int flush_ctas = std::max(16, p->comm->num_sms - 8);
        ck(launch_l2_flush(pipe->flush_buf, pipe->flush_bytes, flush_ctas, pipe->comm), "l2 flush");
      }
      if (pipe->engine) {
        ck(launch_engine(pipe->args, pipe->engine_ctas, pipe->grid_y, pipe->comm), "engine launch");
        // one replay kernel walks every group head's ready time
        ck(launch_replay_all(pipe->d_clock, pipe->d_deadlines, static_cast<uint32_t>(G), pipe->d_pipe,
                             pipe->d_ready, pipe->compute, gate_replay ? 1 : 0),
           "replay");
        if (pipe->tail_launch > 0) {
          // the replay kernel ends right after marking group 0 (last in backward order) ready
          ck(cudaEventCreateWithFlags(&pipe->replay_done, cudaEventDisableTiming), "event");
          ck(cudaEventRecord(pipe->replay_done, pipe->compute), "replay done");
          ck(cudaStreamWaitEvent(pipe->comm, pipe->replay_done, 0), "replay done wait");
          for (int g = pipe->tail_launch - 1; g >= 0; --g) {
            launch_group(p, g, lr, MGW_SGD, algo, pipe->comm, /*force_chunked=*/true,
                         pipe->timed_groups ? pipe->d_stamps : nullptr, static_cast<uint32_t>(pipe->stamp_cols));
          }
        }
      }
      bool first = true;
      for (int g = G - 1; g >= 0 && !pipe->engine; --g) {
        const size_t head = p->heads[g];
        const double ready_s = tau_b[head] + t_b[head];
        const auto deadline = static_cast<unsigned long long>(std::llround(ready_s * 1e9));
        ck(launch_replay(pipe->d_clock, deadline, first ? 1 : 0, nullptr, pipe->compute), "replay");
        first = false;
        ck(cudaEventRecord(pipe->ready[g], pipe->compute), "ready");
        ck(cudaStreamWaitEvent(pipe->comm, pipe->ready[g], 0), "ready wait");
        if (pipe->timed_groups) {
          ck(cudaEventRecordWithFlags(pipe->g_start[g], pipe->comm, cudaEventRecordExternal),
             "group start");
        }
        launch_group(p, g, lr, MGW_SGD, algo, pipe->comm);
        if (pipe->timed_groups) {
          ck(cudaEventRecordWithFlags(pipe->g_end[g], pipe->comm, cudaEventRecordExternal),
             "group end");
        }
      }
      ck(cudaEventRecord(pipe->join, pipe->comm), "join");
      ck(cudaStreamWaitEvent(pipe->compute, pipe->join, 0), "join wait");
      if (io.d2h_bytes > 0) {
        ck(cudaMemcpyAsync(io.d2h_dst, io.d2h_src, io.d2h_bytes, cudaMemcpyDeviceToHost, pipe->compute),
           "d2h result");
      }
    } catch (...) {
      cudaGraph_t g = nullptr;
      cudaStreamEndCapture(pipe->compute, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    ck(cudaStreamEndCapture(pipe->compute, &pipe->graph), "end capture");
    ck(cudaGraphInstantiate(&pipe->exec, pipe->graph, 0), "graph instantiate");
    if (!pipe->engine) {
      // the capture counted kernels once; graph replays add per launch
      g_kernel_launches.fetch_sub(static_cast<uint64_t>(G), std::memory_order_relaxed);
    }
    if (pipe->engine && pipe->tail_launch > 0) {
      g_kernel_launches.fetch_sub(static_cast<uint64_t>(pipe->tail_launch), std::memory_order_relaxed);
    }
    // engine + replay (+ tail launches), or replay + group kernel per group; plus the L2 flush
    pipe->kernels_per_iter = (pipe->engine ? 2 + pipe->tail_launch : 2 * G) + (pipe->flush_bytes > 0 ? 1 : 0);
    return pipe;
  }
}

}  // namespace
}  // namespace mgw

extern "C" {

int mgw_pipeline_destroy(mgw_pipeline* pipe) {
  MGW_TRY {
    if (pipe == nullptr) return 0;
    cudaSetDevice(pipe->plan->comm->device);
    cudaStreamSynchronize(pipe->compute);
    cudaStreamSynchronize(pipe->comm);
    if (pipe->exec) cudaGraphExecDestroy(pipe->exec);
    if (pipe->graph) cudaGraphDestroy(pipe->graph);
    for (auto e : pipe->ready) cudaEventDestroy(e);
    for (auto e : pipe->g_start) cudaEventDestroy(e);
    for (auto e : pipe->g_end) cudaEventDestroy(e);
    cudaEventDestroy(pipe->fork);
    cudaEventDestroy(pipe->join);
    if (pipe->replay_done) cudaEventDestroy(pipe->replay_done);
    cudaFree(pipe->d_clock);
    if (pipe->flush_buf) cudaFree(pipe->flush_buf);
    if (pipe->d_pipe) cudaFree(pipe->d_pipe);
    if (pipe->d_stamps) cudaFree(pipe->d_stamps);
    if (pipe->d_groups) cudaFree(pipe->d_groups);
    if (pipe->d_sched) cudaFree(pipe->d_sched);
    if (pipe->d_sched_off) cudaFree(pipe->d_sched_off);
    if (pipe->d_deadlines) cudaFree(pipe->d_deadlines);
    if (pipe->d_ready) cudaFree(pipe->d_ready);
    cudaStreamDestroy(pipe->compute);
    cudaStreamDestroy(pipe->comm);
    delete pipe;
  }
  MGW_CATCH
}

int mgw_pipeline_launch(mgw_pipeline* pipe, int iters) {
  MGW_TRY {
    require(pipe != nullptr && iters >= 0 && !pipe->manual, "bad pipeline launch");
    mgw::set_device(pipe->plan->comm);
    for (int i = 0; i < iters; ++i) {
      ck(cudaGraphLaunch(pipe->exec, pipe->compute), "graph launch");
      mgw::g_kernel_launches.fetch_add(pipe->kernels_per_iter, std::memory_order_relaxed);
    }
  }
  MGW_CATCH
}

int mgw_pipeline_run(mgw_pipeline* pipe, int iters, float* iter_ms) {
  MGW_TRY {
    require(pipe != nullptr && iters >= 1 && iter_ms != nullptr && !pipe->manual,
            "bad pipeline run");
    mgw::set_device(pipe->plan->comm);
    std::vector<cudaEvent_t> ev(static_cast<size_t>(iters) + 1);
    for (auto& e : ev) ck(cudaEventCreate(&e), "event");
    try {
      ck(cudaEventRecord(ev[0], pipe->compute), "record");
      for (int i = 0; i < iters; ++i) {
        ck(cudaGraphLaunch(pipe->exec, pipe->compute), "graph launch");
        mgw::g_kernel_launches.fetch_add(pipe->kernels_per_iter, std::memory_order_relaxed);
        ck(cudaEventRecord(ev[i + 1], pipe->compute), "record");
      }
      ck(cudaEventSynchronize(ev[iters]), "pipeline sync");
      for (int i = 0; i < iters; ++i) ck(cudaEventElapsedTime(&iter_ms[i], ev[i], ev[i + 1]), "elapsed");
      mgw::check_barrier_flags(pipe->plan->comm);
      if (pipe->d_pipe != nullptr) {
        uint32_t st[4];
        ck(cudaMemcpy(st, pipe->d_pipe, sizeof st, cudaMemcpyDeviceToHost), "read pipe state");
        if (st[3] != 0) {
          throw mgw::CudaFailure("comm engine timed out waiting for a ready group "
                                 "(compute stream did not run concurrently?)");
        }
      }
    } catch (...) {
      for (auto e : ev) cudaEventDestroy(e);
      throw;
    }
    for (auto e : ev) cudaEventDestroy(e);
  }
  MGW_CATCH
}

int mgw_pipeline_group_times(mgw_pipeline* pipe, float* group_ms) {
  MGW_TRY {
    require(pipe != nullptr && group_ms != nullptr && pipe->timed_groups,
            "pipeline was created without record_group_times");
    mgw::set_device(pipe->plan->comm);
    ck(cudaStreamSynchronize(pipe->compute), "sync");
    ck(cudaStreamSynchronize(pipe->comm), "sync");
    if (pipe->engine) {
      const int G = pipe->plan->G();
      std::vector<unsigned long long> st;
      mgw::read_group_stamps(pipe, st);
      for (int g = 0; g < G; ++g) {
        // zero-tile groups are no-ops in the engine (no CTA active)
        group_ms[g] = st[2 * g + 1] > st[2 * g] ? static_cast<float>(st[2 * g + 1] - st[2 * g]) * 1e-6f
                                                : 0.0f;
      }
      return 0;
    }
    for (size_t g = 0; g < pipe->g_start.size(); ++g) {
      ck(cudaEventElapsedTime(&group_ms[g], pipe->g_start[g], pipe->g_end[g]), "elapsed");
    }
  }
  MGW_CATCH
}

int mgw_calibrate_engine(mgw_comm* c, const uint64_t* sizes, size_t n, int warmup, int reps,
                         int algo, int engine_ctas, mgw_meas* out) {
  return mgw_calibrate_engine_ex(c, sizes, n, warmup, reps, algo, engine_ctas, MGW_DTYPE_F32, out);
}

int mgw_calibrate_engine_ex(mgw_comm* c, const uint64_t* sizes, size_t n, int warmup, int reps,
                            int algo, int engine_ctas, int dtype, mgw_meas* out) {
  MGW_TRY {
    require(dtype == MGW_DTYPE_F32 || dtype == MGW_DTYPE_BF16, "bad dtype");
    const uint64_t esize = dtype == MGW_DTYPE_BF16 ? 2 : 4;
    require(c != nullptr && sizes != nullptr && out != nullptr && reps >= 1, "bad calibrate args");
    require(!c->loopback, "calibration runs on a real communicator");
    mgw::set_device(c);
    uint64_t max_bytes = 16;
    for (size_t i = 0; i < n; ++i) max_bytes = std::max(max_bytes, sizes[i]);
    const size_t max_elems = (max_bytes + esize - 1) / esize;  // gradient elements
    // ONE group per iteration: the planner's cost T(M) is a group's time on
    // an idle engine (back-to-back groups overlap at CTA
    // granularity, which made per-group stamps of a multi-group iteration
    // unreliable at large sizes).
    constexpr int kGroups = 1;
    float* grad = nullptr;
    float* w = nullptr;
    ck(cudaMalloc(&grad, max_elems * esize + 16), "cudaMalloc(calib grad)");
    ck(cudaMalloc(&w, max_elems * sizeof(float)), "cudaMalloc(calib w)");
    ck(cudaMemset(grad, 0, max_elems * esize + 16), "memset");
    ck(cudaMemset(w, 0, max_elems * sizeof(float)), "memset");
    try {
      for (size_t i = 0; i < n; ++i) {
        // R layers of `cnt` elements that all alias the same buffers (the
        // kernel reads grads / updates weights; aliasing is harmless for
        // timing), one group each, every group ready at iteration start.
        const uint64_t cnt = std::max<uint64_t>(1, (sizes[i] + esize - 1) / esize);
        const int R = kGroups;
        std::vector<float*> gp(R, grad), wp(R, w);
        std::vector<uint64_t> counts(R, cnt);
        std::vector<uint8_t> tags(R, 0);
        std::vector<double> tb(R, 0.0);
        mgw_plan* p = mgw::build_plan(c, R, gp.data(), wp.data(), counts.data(), tags.data(), dtype);
        mgw_pipeline* pipe = nullptr;
        try {
          // L2 evicted before every rep (256 MiB > the 126 MB L2, on the comm
          // branch before the engine; the group's stamps start after it):
          // cold-HBM group times, as in a pipeline iteration — a warm L2 made
          // the P = 1 slope look faster than HBM
          // the group becomes ready 100 us into the iteration, after the L2
          // flush: the engine is already waiting for it, as in a pipeline,
          // so T(M) is the ready -> reduced latency the planner trades
          pipe = mgw::build_pipeline(p, tb.data(), 100e-6, 0.0f, algo, true, size_t{256} << 20, engine_ctas,
                                     mgw::StepIo{}, /*gate_replay=*/true);
          std::vector<float> ms;
          std::vector<float> gm(R);
          for (int k = 0; k < warmup + reps; ++k) {
            ck(cudaGraphLaunch(pipe->exec, pipe->compute), "graph launch");
            if (mgw_pipeline_group_times(pipe, gm.data()) != 0) throw mgw::CudaFailure("stamps");
            if (k >= warmup) ms.insert(ms.end(), gm.begin(), gm.end());
          }
          std::sort(ms.begin(), ms.end());
          out[i].size_bytes = sizes[i];
          out[i].time_sec = 1e-3 * ms[ms.size() / 2];
        } catch (...) {
          mgw_pipeline_destroy(pipe);
          mgw::destroy_plan(p);
          throw;
        }
        mgw_pipeline_destroy(pipe);
        mgw::destroy_plan(p);
      }
      mgw::check_barrier_flags(c);
    } catch (...) {
      cudaFree(grad);
      cudaFree(w);
      throw;
    }
    cudaFree(grad);
    cudaFree(w);
  }
  MGW_CATCH
}

int mgw_pipeline_stream(mgw_pipeline* pipe, void** stream_out) {
  MGW_TRY {
    require(pipe != nullptr && stream_out != nullptr, "NULL argument");
    *stream_out = pipe->compute;
  }
  MGW_CATCH
}

int mgw_engine_create(mgw_plan* p, float lr, int algo, int engine_ctas, int record_group_times,
                      mgw_pipeline** out) {
  MGW_TRY {
    require(p != nullptr && out != nullptr, "bad engine arguments");
    require(engine_ctas != 0, "engine_ctas must be non-zero (< 0: default)");
    mgw::set_device(p->comm);
    auto* pipe = new mgw_pipeline();
    pipe->plan = p;
    pipe->timed_groups = record_group_times != 0;
    pipe->engine = true;
    pipe->manual = true;
    mgw::setup_engine(pipe, p, algo, engine_ctas, lr, pipe->timed_groups);
    ck(cudaStreamCreateWithFlags(&pipe->compute, cudaStreamNonBlocking), "stream");
    ck(cudaStreamCreateWithFlags(&pipe->comm, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreateWithFlags(&pipe->fork, cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&pipe->join, cudaEventDisableTiming), "event");
    ck(cudaMalloc(&pipe->d_clock, 2 * sizeof(unsigned long long)), "cudaMalloc(clock)");
    ck(cudaMemset(pipe->d_clock, 0, 2 * sizeof(unsigned long long)), "memset(clock)");
    pipe->kernels_per_iter = 1 + p->G();  // engine + one mark kernel per group
    *out = pipe;
  }
  MGW_CATCH
}

int mgw_engine_begin(mgw_pipeline* pipe, void* after_stream) {
  MGW_TRY {
    require(pipe != nullptr && pipe->manual, "not a host-driven engine");
    mgw::set_device(pipe->plan->comm);
    // NULL is the legacy default stream (torch's default), not "no stream"
    ck(cudaEventRecord(pipe->fork, static_cast<cudaStream_t>(after_stream)), "fork");
    ck(cudaStreamWaitEvent(pipe->comm, pipe->fork, 0), "fork wait");
    ck(mgw::launch_engine(pipe->args, pipe->engine_ctas, pipe->grid_y, pipe->comm), "engine launch");
    mgw::g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  }
  MGW_CATCH
}

int mgw_engine_mark_ready(mgw_pipeline* pipe, int group, void* stream) {
  MGW_TRY {
    require(pipe != nullptr && pipe->manual, "not a host-driven engine");
    require(group >= 0 && group < pipe->plan->G(), "group index out of range");
    mgw::set_device(pipe->plan->comm);
    ck(mgw::launch_mark_ready(pipe->d_pipe, pipe->d_ready, static_cast<uint32_t>(group),
                              static_cast<cudaStream_t>(stream)),
       "mark ready");
    mgw::g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  }
  MGW_CATCH
}

int mgw_engine_join(mgw_pipeline* pipe, void* stream) {
  MGW_TRY {
    require(pipe != nullptr && pipe->manual, "not a host-driven engine");
    mgw::set_device(pipe->plan->comm);
    ck(cudaEventRecord(pipe->join, pipe->comm), "join");
    ck(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), pipe->join, 0), "join wait");
  }
  MGW_CATCH
}

int mgw_engine_set_tail(mgw_pipeline* pipe, int n_tail) {
  MGW_TRY {
    require(pipe != nullptr && pipe->manual, "not a host-driven engine");
    require(n_tail >= 0 && n_tail <= pipe->plan->G(), "tail group count out of range");
    pipe->args.g_lo = static_cast<uint32_t>(n_tail);
  }
  MGW_CATCH
}

int mgw_engine_check(mgw_pipeline* pipe) {
  MGW_TRY {
    require(pipe != nullptr && pipe->engine, "not an engine");
    mgw::set_device(pipe->plan->comm);
    ck(cudaStreamSynchronize(pipe->comm), "engine sync");
    mgw::check_barrier_flags(pipe->plan->comm);
    uint32_t st[4];
    ck(cudaMemcpy(st, pipe->d_pipe, sizeof st, cudaMemcpyDeviceToHost), "read pipe state");
    if (st[3] != 0) {
      throw mgw::CudaFailure("comm engine timed out waiting for a ready group (a group was never "
                             "marked ready, or the compute stream could not run)");
    }
  }
  MGW_CATCH
}

int mgw_pipeline_drain(mgw_pipeline* pipe, int iters, float* ms_out) {
  MGW_TRY {
    require(pipe != nullptr && pipe->engine && iters >= 1 && ms_out != nullptr, "bad drain arguments");
    mgw::set_device(pipe->plan->comm);
    mgw_comm* c = pipe->plan->comm;
    mgw::EngineLaunch E = pipe->args;
    E.no_wait = 1;  // every group ready at launch: the engine streams the whole plan
    if (pipe->tail_launch > 0) E.g_lo = 0;  // (including the pipeline's tail group)
    std::vector<cudaEvent_t> ev(2 * static_cast<size_t>(iters));
    for (auto& e : ev) ck(cudaEventCreate(&e), "event");
    try {
      for (int i = 0; i < iters; ++i) {
        if (pipe->flush_buf != nullptr) {
          ck(mgw::launch_l2_flush(pipe->flush_buf, pipe->flush_bytes, c->num_sms, pipe->comm), "l2 flush");
          mgw::g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
        }
        ck(cudaEventRecord(ev[2 * i], pipe->comm), "record");
        ck(mgw::launch_engine(E, pipe->engine_ctas, pipe->grid_y, pipe->comm), "engine launch");
        mgw::g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
        ck(cudaEventRecord(ev[2 * i + 1], pipe->comm), "record");
      }
      ck(cudaEventSynchronize(ev.back()), "drain sync");
      for (int i = 0; i < iters; ++i) ck(cudaEventElapsedTime(&ms_out[i], ev[2 * i], ev[2 * i + 1]), "elapsed");
      mgw::check_barrier_flags(c);
    } catch (...) {
      for (auto e : ev) cudaEventDestroy(e);
      throw;
    }
    for (auto e : ev) cudaEventDestroy(e);
  }
  MGW_CATCH
}

int mgw_pipeline_stamps(mgw_pipeline* pipe, uint64_t* stamps_2g) {
  MGW_TRY {
    require(pipe != nullptr && stamps_2g != nullptr && pipe->engine && pipe->timed_groups,
            "stamps need an engine pipeline created with record_group_times");
    mgw::set_device(pipe->plan->comm);
    ck(cudaStreamSynchronize(pipe->compute), "sync");
    ck(cudaStreamSynchronize(pipe->comm), "sync");
    std::vector<unsigned long long> st;
    mgw::read_group_stamps(pipe, st);
    std::copy(st.begin(), st.end(), stamps_2g);
  }
  MGW_CATCH
}

int mgw_pipeline_stamps_raw(mgw_pipeline* pipe, uint64_t* out, size_t cap, size_t* cols_out) {
  MGW_TRY {
    require(pipe != nullptr && out != nullptr && cols_out != nullptr && pipe->engine && pipe->timed_groups &&
                pipe->d_stamps != nullptr,
            "raw stamps need an engine pipeline created with record_group_times");
    mgw::set_device(pipe->plan->comm);
    ck(cudaStreamSynchronize(pipe->comm), "sync");
    const size_t n = static_cast<size_t>(pipe->plan->G()) * pipe->stamp_cols * 2;
    require(cap >= n, "raw stamps buffer too small (G x CTAs x 2)");
    ck(cudaMemcpy(out, pipe->d_stamps, n * sizeof(uint64_t), cudaMemcpyDeviceToHost), "read stamps");
    *cols_out = pipe->stamp_cols;
  }
  MGW_CATCH
}

int mgw_pipeline_debug(mgw_pipeline* pipe, uint32_t* engine_state4, uint64_t* clock2) {
  MGW_TRY {
    require(pipe != nullptr, "NULL pipeline");
    mgw::set_device(pipe->plan->comm);
    // Read on a private stream: must not wait behind a stuck pipeline.
    cudaStream_t s = nullptr;
    ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
    if (engine_state4 != nullptr) {
      if (pipe->d_pipe) {
        ck(cudaMemcpyAsync(engine_state4, pipe->d_pipe, 4 * sizeof(uint32_t), cudaMemcpyDeviceToHost, s),
           "read pipe");
      } else {
        std::memset(engine_state4, 0, 4 * sizeof(uint32_t));
      }
    }
    if (clock2 != nullptr) {
      ck(cudaMemcpyAsync(clock2, pipe->d_clock, 2 * sizeof(uint64_t), cudaMemcpyDeviceToHost, s),
         "read clock");
    }
    ck(cudaStreamSynchronize(s), "debug sync");
    cudaStreamDestroy(s);
  }
  MGW_CATCH
}

}  // extern "C"

// ---- copy-engine mode (real backward, no SMs during the backward) ----------
// The paper's communication daemon thread, on the host:
// the backward's hook only appends (group, compute stream) to a single-
// producer / single-consumer ring — no CUDA call on the main thread; a C++
// worker thread (spinning between begin and join, asleep otherwise) records
// the group's ready event on the compute stream (the hook ran right after
// autograd enqueued the group's last gradient kernel, so the event covers it;
// recording a little later only adds work before it, never less), makes the
// comm stream wait for it and queues the group's copy-engine pushes.
struct mgw_ce {
  mgw_plan* plan = nullptr;
  cudaStream_t comm = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  std::vector<cudaEvent_t> ready;  // G
  struct Copy {
    void* dst;
    const void* src;
    size_t bytes;
  };
  std::vector<std::vector<Copy>> copies;  // [G]: every view's copies to every peer
  mgw::CeLaunch args{};
  uint32_t* d_done = nullptr;  // per view: reduce-kernel CTA counter
  int n_views = 1;
  int reduce_ctas = 0;
  int n_tail = 0;  // groups [0, n_tail) are not copied nor reduced here (the caller's full-width launches)
  // "iteration delivered" signals as stream memory operations (no SM):
  // per (view, peer) the peer's ce_pushed word; nullptr fn: signal kernel
  using WriteValue64 = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
  WriteValue64 write_value = nullptr;
  std::vector<CUdeviceptr> signal_words;
  bool begun = false;
  // daemon
  std::vector<int> ring;              // G + 1 slots (each group at most once per iteration)
  std::vector<cudaStream_t> ring_stream;  // the compute stream of each appended group
  std::atomic<uint64_t> head{0};      // groups appended by the main thread (this iteration and before)
  std::atomic<uint64_t> tail{0};      // groups whose copies the worker queued
  std::atomic<bool> active{false};    // between begin and join: the worker spins
  std::atomic<bool> stop{false};
  std::mutex mu;
  std::condition_variable cv;
  std::thread worker;
  std::string error;                  // first CUDA error of the worker (guarded by mu)
};

namespace mgw {
namespace {

void ce_worker(mgw_ce* e) {
  if (cudaSetDevice(e->plan->comm->device) != cudaSuccess) return;
  const size_t n = e->ring.size();
  for (;;) {
    {
      std::unique_lock<std::mutex> lk(e->mu);
      e->cv.wait(lk, [&] { return e->stop.load() || e->active.load() ||
                                  e->tail.load() != e->head.load(std::memory_order_acquire); });
      if (e->stop.load()) return;  // destroy: copies still queued are moot
    }
    // spin while the iteration is open: a hook's append is picked up at once
    while (!e->stop.load(std::memory_order_relaxed)) {
      const uint64_t t = e->tail.load(std::memory_order_relaxed);
      if (t == e->head.load(std::memory_order_acquire)) {
        if (!e->active.load(std::memory_order_acquire)) break;
        continue;
      }
      const int g = e->ring[t % n];
      cudaError_t err = cudaEventRecord(e->ready[g], e->ring_stream[t % n]);
      if (err == cudaSuccess) err = cudaStreamWaitEvent(e->comm, e->ready[g], 0);
      for (const auto& cp : e->copies[g]) {
        if (err != cudaSuccess) break;
        err = cudaMemcpyAsync(cp.dst, cp.src, cp.bytes, cudaMemcpyDeviceToDevice, e->comm);
      }
      if (err != cudaSuccess) {
        std::lock_guard<std::mutex> lk(e->mu);
        if (e->error.empty()) e->error = std::string("copy-engine push: ") + cudaGetErrorString(err);
      }
      e->tail.store(t + 1, std::memory_order_release);
    }
  }
}

}  // namespace
}  // namespace mgw

int mgw_ce_create(mgw_plan* p, float lr, mgw_ce** out) {
  MGW_TRY {
    require(p != nullptr && out != nullptr, "NULL argument");
    mgw_comm* c = p->comm;
    require(c->nranks > 1, "copy-engine mode needs P > 1 (P = 1 has no exchange)");
    require(c->loopback || c->peers_ready, "communicator peers not opened (call mgw_comm_open_peers)");
    mgw::set_device(c);
    const size_t L = p->L;
    // gradients must be laid out like the merge layout (one flat buffer,
    // layer l at element offs[l]): a group is then ONE contiguous copy
    std::vector<const char*> base(static_cast<size_t>(p->n_views), nullptr);
    for (int r = 0; r < p->n_views; ++r) {
      for (size_t l = 0; l < L; ++l) {
        if (p->counts[l] == 0) continue;
        const char* g = reinterpret_cast<const char*>(p->h_grads[static_cast<size_t>(r) * L + l]);
        if (base[r] == nullptr) base[r] = g - p->offs[l] * p->esize;
        require(g == base[r] + p->offs[l] * p->esize,
                "copy-engine mode needs the gradients in one flat buffer laid out like the merge layout "
                "(layer l at element offs[l], 16-byte aligned layers)");
      }
      require(base[r] != nullptr, "plan has no gradient elements");
      for (size_t l = 0; l < L; ++l) {
        require(p->counts[l] == 0 || p->h_weights[static_cast<size_t>(r) * L + l] != nullptr,
                "copy-engine mode applies SGD: every layer needs its weights");
      }
    }
    std::unique_ptr<mgw_ce> e(new mgw_ce());
    e->plan = p;
    e->n_views = p->n_views;
    const int G = p->G();
    e->copies.resize(G);
    for (int g = 0; g < G; ++g) {
      // the group's data span: its first layer's start to the end of its last
      // non-empty layer (not the padded end: the caller's buffer may stop
      // at the last element)
      const uint64_t lo = p->offs[p->heads[g]];
      uint64_t hi = lo;
      for (size_t l = p->heads[g]; l < p->heads[g + 1]; ++l) {
        if (p->counts[l] > 0) hi = p->offs[l] + p->counts[l];
      }
      const size_t bytes = (hi - lo) * p->esize;
      if (bytes == 0) continue;
      for (int r = 0; r < p->n_views; ++r) {
        const int me = c->loopback ? r : c->rank;
        for (int q = 0; q < c->nranks; ++q) {
          if (q == me) continue;
          char* arena = reinterpret_cast<char*>(c->loopback ? c->arenas[q] : c->peer_arena[q]);
          e->copies[g].push_back(
              {arena + (static_cast<uint64_t>(me) * p->slot_stride + lo) * p->esize, base[r] + lo * p->esize, bytes});
        }
      }
    }
    mgw::CeLaunch& C = e->args;
    for (int r = 0; r < p->n_views; ++r) {
      C.views[r] = mgw::make_view(c, r, p->d_grads + static_cast<size_t>(r) * L, p->d_weights + static_cast<size_t>(r) * L);
    }
    C.tiles = p->d_tiles;
    C.n_tiles = p->tile_first.back();
    C.nranks = c->nranks;
    C.scale = 1.0f / static_cast<float>(c->nranks);
    C.lr = lr;
    C.epilogue = MGW_SGD;
    C.slot_stride = p->slot_stride;
    C.dtype = p->dtype;
    ck(cudaMalloc(&e->d_done, sizeof(uint32_t) * mgw::kMaxRanks), "cudaMalloc(ce done)");
    ck(cudaMemset(e->d_done, 0, sizeof(uint32_t) * mgw::kMaxRanks), "memset(ce done)");
    C.done = e->d_done;
    e->reduce_ctas = c->num_sms;
    // SM-free signalling: cuStreamWriteValue64 (a system-scope memory fence
    // before the write, scoped to the stream — the copies ahead of it on the
    // comm stream are visible before the flag). Without it, a 1-thread
    // signal kernel (then a fused tail launch must follow mgw_ce_join).
    {
      int ok = 0;
      cudaDeviceGetAttribute(&ok, static_cast<cudaDeviceAttr>(CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS),
                             c->device);
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
      if (ok && cudaGetDriverEntryPoint("cuStreamWriteValue64", &fn, cudaEnableDefault, &q) == cudaSuccess &&
          q == cudaDriverEntryPointSuccess && fn != nullptr) {
        e->write_value = reinterpret_cast<mgw_ce::WriteValue64>(fn);
      }
      cudaGetLastError();
      for (int r = 0; r < p->n_views; ++r) {
        const int me = c->loopback ? r : c->rank;
        for (int q2 = 0; q2 < c->nranks; ++q2) {
          if (q2 == me) continue;
          uint32_t* sig = c->loopback ? c->signals[q2] : c->peer_signal[q2];
          e->signal_words.push_back(reinterpret_cast<CUdeviceptr>(sig + mgw::kCeWord) +
                                    static_cast<CUdeviceptr>(me) * sizeof(uint64_t));
        }
      }
    }
    ck(cudaStreamCreateWithFlags(&e->comm, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreateWithFlags(&e->fork, cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&e->join, cudaEventDisableTiming), "event");
    e->ready.resize(G);
    for (auto& ev : e->ready) ck(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
    e->ring.assign(static_cast<size_t>(G) + 1, 0);
    e->ring_stream.assign(static_cast<size_t>(G) + 1, nullptr);
    e->worker = std::thread(mgw::ce_worker, e.get());
    *out = e.release();
  }
  MGW_CATCH
}

int mgw_ce_begin(mgw_ce* e, void* after_stream) {
  MGW_TRY {
    require(e != nullptr, "NULL engine");
    require(!e->begun, "mgw_ce_begin twice without mgw_ce_join");
    mgw_comm* c = e->plan->comm;
    mgw::set_device(c);
    ck(cudaEventRecord(e->fork, static_cast<cudaStream_t>(after_stream)), "fork");
    ck(cudaStreamWaitEvent(e->comm, e->fork, 0), "fork wait");
    e->args.iter = ++c->ce_seq;
    // the peers finished reducing the previous iteration out of their arenas
    ck(mgw::launch_ce(0, e->args, e->n_views, 1, e->comm), "ce wait");
    mgw::g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
    e->begun = true;
    {
      std::lock_guard<std::mutex> lk(e->mu);
      e->active.store(true, std::memory_order_release);
    }
    e->cv.notify_one();
  }
  MGW_CATCH
}

int mgw_ce_set_tail(mgw_ce* e, int n_tail) {
  MGW_TRY {
    require(e != nullptr && !e->begun, "mgw_ce_set_tail inside an iteration");
    const mgw_plan* p = e->plan;
    require(n_tail >= 0 && n_tail < p->G(), "tail group count out of range (the engine needs >= 1 group)");
    e->n_tail = n_tail;
    e->args.tiles = p->d_tiles + p->tile_first[n_tail];
    e->args.n_tiles = p->tile_first.back() - p->tile_first[n_tail];
  }
  MGW_CATCH
}

int mgw_ce_mark_ready(mgw_ce* e, int g, void* stream) {
  MGW_TRY {
    require(e != nullptr && e->begun, "mgw_ce_mark_ready outside mgw_ce_begin / mgw_ce_join");
    require(g >= 0 && g < e->plan->G(), "group index out of range");
    if (g < e->n_tail) return 0;  // a tail group: the caller reduces it after the backward
    const uint64_t h = e->head.load(std::memory_order_relaxed);
    require(h - e->tail.load(std::memory_order_acquire) < e->ring.size(), "group marked ready twice");
    e->ring[h % e->ring.size()] = g;
    e->ring_stream[h % e->ring.size()] = static_cast<cudaStream_t>(stream);
    e->head.store(h + 1, std::memory_order_release);  // the spinning worker picks it up
  }
  MGW_CATCH
}

int mgw_ce_join(mgw_ce* e, void* stream) {
  MGW_TRY {
    require(e != nullptr && e->begun, "mgw_ce_join without mgw_ce_begin");
    mgw::set_device(e->plan->comm);
    // every appended group's copies are queued on the comm stream
    while (e->tail.load(std::memory_order_acquire) != e->head.load(std::memory_order_relaxed)) {
    }
    e->active.store(false, std::memory_order_release);
    {
      std::lock_guard<std::mutex> lk(e->mu);
      if (!e->error.empty()) throw mgw::CudaFailure(e->error);
    }
    bool signalled = false;
    if (e->write_value != nullptr) {
      signalled = true;
      for (CUdeviceptr w : e->signal_words) {
        if (e->write_value(reinterpret_cast<CUstream>(e->comm), w, e->args.iter, CU_STREAM_WRITE_VALUE_DEFAULT) !=
            CUDA_SUCCESS) {
          signalled = false;  // the kernel below re-signals every peer (same value: idempotent)
          e->write_value = nullptr;
          break;
        }
      }
    }
    if (!signalled) {
      ck(mgw::launch_ce(1, e->args, e->n_views, 1, e->comm), "ce signal");
      mgw::g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
    }
    ck(mgw::launch_ce(2, e->args, e->n_views, e->reduce_ctas, e->comm), "ce reduce");
    mgw::g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
    ck(cudaEventRecord(e->join, e->comm), "join");
    ck(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), e->join, 0), "join wait");
    e->begun = false;
  }
  MGW_CATCH
}

int mgw_ce_signals_without_sm(const mgw_ce* e, int* out) {
  MGW_TRY {
    require(e != nullptr && out != nullptr, "NULL argument");
    *out = e->write_value != nullptr ? 1 : 0;
  }
  MGW_CATCH
}

int mgw_ce_check(mgw_ce* e) {
  MGW_TRY {
    require(e != nullptr, "NULL engine");
    mgw::set_device(e->plan->comm);
    ck(cudaStreamSynchronize(e->comm), "ce sync");
    mgw::check_barrier_flags(e->plan->comm);
  }
  MGW_CATCH
}

int mgw_ce_destroy(mgw_ce* e) {
  MGW_TRY {
    if (e == nullptr) return 0;
    {
      std::lock_guard<std::mutex> lk(e->mu);
      e->stop.store(true);
      e->active.store(false);
    }
    e->cv.notify_one();
    if (e->worker.joinable()) e->worker.join();
    mgw::set_device(e->plan->comm);
    cudaStreamSynchronize(e->comm);
    for (auto ev : e->ready) cudaEventDestroy(ev);
    cudaEventDestroy(e->fork);
    cudaEventDestroy(e->join);
    cudaStreamDestroy(e->comm);
    cudaFree(e->d_done);
    delete e;
  }
  MGW_CATCH
}

int mgw_calibrate_ce(mgw_comm* c, const uint64_t* sizes_bytes, size_t n, int warmup, int reps, mgw_meas* out) {
  MGW_TRY {
    require(c != nullptr && sizes_bytes != nullptr && out != nullptr && n >= 1 && reps >= 1, "bad arguments");
    require(c->loopback || c->nranks == 1 || c->peers_ready, "communicator peers not opened");
    mgw::set_device(c);
    const int me = c->loopback ? 0 : c->rank;
    const int q = (me + 1) % c->nranks;
    char* dst = reinterpret_cast<char*>(c->nranks == 1 ? c->arenas[0]
                                                       : (c->loopback ? c->arenas[q] : c->peer_arena[q]));
    uint64_t top = 0;
    for (size_t i = 0; i < n; ++i) top = std::max(top, sizes_bytes[i]);
    require(top <= c->arena_elems * sizeof(float), "calibration size exceeds the arena");
    void* src = nullptr;
    ck(cudaMalloc(&src, std::max<uint64_t>(top, 16)), "cudaMalloc(calibration source)");
    cudaEvent_t e0, e1;
    ck(cudaEventCreate(&e0), "event");
    ck(cudaEventCreate(&e1), "event");
    try {
      for (size_t i = 0; i < n; ++i) {
        std::vector<float> ts;
        for (int k = 0; k < warmup + reps; ++k) {
          ck(cudaEventRecord(e0, c->stream), "record");
          ck(cudaMemcpyAsync(dst, src, sizes_bytes[i], cudaMemcpyDeviceToDevice, c->stream), "copy");
          ck(cudaEventRecord(e1, c->stream), "record");
          ck(cudaEventSynchronize(e1), "sync");
          float ms = 0;
          ck(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
          if (k >= warmup) ts.push_back(ms);
        }
        std::sort(ts.begin(), ts.end());
        out[i].size_bytes = sizes_bytes[i];
        out[i].time_sec = ts[ts.size() / 2] * 1e-3;
      }
    } catch (...) {
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      cudaFree(src);
      throw;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(src);
  }
  MGW_CATCH
}
