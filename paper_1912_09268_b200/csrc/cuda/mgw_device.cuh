// mgwfbp-b200: device-side data layout and PTX helpers shared by the
// kernels (kernels.cu) and the host runtime (runtime.cu).
//
// Data layout in HBM (per rank):
//   merge arena   P slots x (padded model elements) fp32; slot r receives
//                 rank r's scaled gradients (posted NVLink stores — the push
//                 data path). Layer l of the plan lives at element offs[l]
//                 of a slot (16-byte aligned), so every merge group
//                 [head_g, head_{g+1}) is one contiguous span — the paper's
//                 pre-allocated merge buffers laid out
//                 once for all groups. Reuse across launches is made safe by
//                 an entry barrier, not by double buffering.
//   signal area   kMaxCtas x kMaxRanks uint32 flags: flag [b][q] holds the
//                 barrier count CTA b of rank q last published (written by
//                 q over NVLink with st.release.sys, spun on locally with
//                 ld.acquire.sys).
//   state         [2] timeout error flag, [3] launch sequence number (the
//                 LL epoch source: identical on every rank, +1 per collective
//                 launch), [4] exit count of the running launch, [64 + b]
//                 barrier count of CTA index b (identical on every rank).
// Work unit: a Tile = up to kTileElems consecutive elements of ONE layer,
// so pack/unpack read and write contiguous 16-byte vectors.
#ifndef MGWFBP_DEVICE_CUH_
#define MGWFBP_DEVICE_CUH_

#include <cstdint>

namespace mgw {

constexpr int kMaxRanks = 8;
constexpr int kMaxCtas = 1024;           // per-rank CTAs of one collective launch
constexpr int kBlock = 512;              // threads per CTA of the fused kernel (16 warps, 128 regs)
constexpr int kThreads = kBlock - 32;    // data threads; the last warp is the TMA producer
constexpr uint32_t kTileElems = 8192;    // 32 KiB of fp32 (one TMA stage); <= 5 float4 per data thread
constexpr uint32_t kVecPerThread = (kTileElems / 4 + kThreads - 1) / kThreads;
constexpr uint32_t kLayerMask = 0x3fffffffu;
constexpr uint32_t kGradUnaligned = 0x80000000u;
constexpr uint32_t kWeightUnaligned = 0x40000000u;
constexpr int kSignalWords = kMaxCtas * kMaxRanks;  // flag [cta][src rank]
// state words: [kStateError] barrier-timeout flag, [kStateCtaBase + b] the
// barrier count of CTA index b (persists across launches)
constexpr int kStateError = 2;
constexpr int kStateSeq = 3;
constexpr int kStateExit = 4;
constexpr int kStateCtaBase = 64;
constexpr int kStateWords = kStateCtaBase + kMaxCtas;
// LL (flag-in-data) area, right after the signal flags of every rank's
// signal allocation: one slot per source rank of kLLSlotPackets 8-byte
// packets {32-bit data word, 32-bit epoch}. Small one-shot groups travel as
// packets (no barrier, no release/acquire round trip); LL doubles the bytes,
// so a slot holds kLLSlotPackets * 4 bytes of gradient data per plan.
constexpr uint64_t kLLSlotPackets = 1ull << 21;  // 16 MiB per source rank
constexpr uint32_t kNoLL = 0xffffffffu;
// LL work unit: a PART of a tile, one vector per data thread.
constexpr uint32_t kLLParts = (kTileElems / 4 + kThreads - 1) / kThreads;  // parts per tile
// Stream flags (the streamed protocol, no per-chunk barrier): two arrays of
// 64-bit words [cta][src rank] after the barrier flags of every rank's signal
// allocation. rs[b][q] = (launch epoch << 32) | tiles CTA b of rank q has
// delivered into this rank's arena in the current launch (its producer's
// gradient pushes); ag[b][q] = the same for owner q's reduced (all-gather)
// tiles. Written by the source over NVLink with st.release.sys.u64, polled
// locally with ld.acquire.sys.u64; the epoch makes every older launch's
// value compare lower.
constexpr int kStreamFlagWords = 2 * kMaxCtas * kMaxRanks * 2;  // in uint32 words
constexpr int kStreamRsWord = kSignalWords;                     // first rs flag (uint32 index)
constexpr int kStreamAgWord = kSignalWords + kMaxCtas * kMaxRanks * 2;
// Copy-engine mode (real backward without SMs): per source rank, the
// iteration whose gradients that rank's copy engine has delivered into this
// rank's arena (ce_pushed), and the iteration this rank's peers have finished
// reducing from their arenas (ce_reduced, guards the next pushes). 64-bit.
constexpr int kCeWord = kSignalWords + kStreamFlagWords;         // [2][kMaxRanks] uint64
constexpr int kCeWords = 2 * kMaxRanks * 2;
constexpr int kLLWord = kCeWord + kCeWords;                      // first LL packet (uint32 index)

struct Tile {
  uint32_t layer;  // layer index | alignment flags
  uint32_t len;    // valid elements in this tile
  uint32_t src;    // first element inside the layer
  uint32_t moff;   // first element in the merge layout (multiple of 4)
};
static_assert(sizeof(Tile) == 16, "tile descriptor is one 16-byte load");

// Everything one (possibly emulated) rank needs inside a collective launch.
struct RankView {
  float* arena[kMaxRanks];       // every rank's merge arena (peer-mapped)
  uint32_t* signal[kMaxRanks];   // every rank's signal area (peer-mapped)
  uint32_t* state;               // this rank's counters
  uint32_t* host_err;            // host-mapped error word of the communicator (may be NULL)
  float* const* grads;           // this rank's layer gradient pointers
  float* const* weights;         // this rank's layer weight pointers (may hold NULLs)
  uint64_t arena_bytes;          // size of every rank's merge arena (bounds checks)
  int rank;
};

struct GroupLaunch {
  const Tile* tiles;     // this group's tiles
  uint32_t n_tiles;
  uint32_t ll_pkt;       // first LL packet of the group (kNoLL: not an LL group)
  uint32_t mbase;        // merge-layout element offset of the group's first element
  int nranks;
  float scale;           // 1/P, applied in the pack phase
  float lr;
  int epilogue;          // MGW_SGD | MGW_WRITE_GRAD
  uint64_t slot_stride;  // elements between the per-source-rank slots of an arena
  uint32_t chunk;        // max tiles per pipelined chunk of one CTA (two-shot: max(1, chunk/P) super-tiles)
  uint32_t min_chunks;   // a CTA with enough tiles splits them into at least this many chunks
  uint32_t stream;       // 1: streamed protocol (per-tile flags), 0: chunked (per-chunk barriers)
  uint32_t credit_batch; // streamed: bulk items per published delivery count (1, 2, 4, 8)
  uint32_t ag_batch;     // streamed two-shot: owned super-tiles per all-gather publication
  int dtype;             // MGW_DTYPE_* of the gradients / arena
  unsigned long long* stamps;  // optional: engine-layout stamps [G][row][2] of group stamp_group
  uint32_t stamp_group;        //   (a pipeline's tail group launched standalone after the engine)
  uint32_t stamp_row;          //   row width (engine CTAs x emulated ranks)
  float* nvls_uc;              // NVLS groups: this rank's copy of the multicast-bound buffer
  float* nvls_mc;              //   and the multicast address of the same bytes (all P copies)
  uint32_t nvls_skip;          //   profiling mask (mgw_comm_set_nvls_skip; 0 in production)
  uint64_t nvls_elems;         //   fp32 elements of the buffer (bounds checks)
  RankView views[kMaxRanks];  // [0] for a real rank; [r] per emulated rank in loopback
};

// One merge group as the persistent comm engine sees it.
struct EngineGroup {
  uint32_t tile_first;
  uint32_t n_tiles;
  uint32_t two_shot;
  uint32_t ll_pkt;       // kNoLL unless the group travels as LL packets (one-shot only)
  uint32_t mbase;        // merge-layout element offset of the group's first element
  uint32_t cta0;         // first CTA of the group: groups rotate over the CTAs in FIFO order,
                         // so consecutive small groups run on different SMs concurrently
  uint32_t units;        // work units (tiles / super-tiles / LL parts); min(units, ncta) CTAs take part
  uint32_t pad;
};

// The persistent comm engine (paper Algorithm 2's communication daemon, on
// the GPU): ONE kernel per iteration walks the groups in backward order,
// each one the moment the compute side marks its head layer ready.
struct EngineLaunch {
  RankView views[kMaxRanks];     // [0] for a real rank; [r] per emulated rank (loopback, blockIdx.y)
  const Tile* tiles;
  const EngineGroup* groups;     // ascending group index
  const uint32_t* sched;         // CTA b's participating groups in FIFO order: sched[sched_off[b] ..
  const uint32_t* sched_off;     //   sched_off[b+1]) (host-built; identical on every rank)
  uint32_t G;
  uint32_t g_lo;                 // the engine runs groups [g_lo, G) (the rest: caller's tail launches)
  int nranks;
  float scale;
  float lr;
  int epilogue;
  uint64_t slot_stride;
  uint32_t chunk;                // as GroupLaunch::chunk
  uint32_t min_chunks;           // as GroupLaunch::min_chunks
  uint32_t stream;               // as GroupLaunch::stream
  uint32_t credit_batch;         // as GroupLaunch::credit_batch
  uint32_t ag_batch;             // as GroupLaunch::ag_batch
  int dtype;                     // MGW_DTYPE_* of the gradients / arena
  uint32_t* pipe;                // [1] iteration, [2] CTA exit count, [3] ready-timeout flag
  const uint32_t* ready;         // G flags: group g ready for iteration i when >= i + 1
  uint32_t no_wait;              // 1: every group is ready (standalone drain: roofline / ncu runs)
  unsigned long long* stamps;    // [G][ranks*ncta][2]: (start, end) %globaltimer of each group on each
                                 // CTA (NULL: no timing); the group's span is min start .. max end
};

// Copy-engine mode: the after-backward reduce of every group (the data
// arrived during the backward as copy-engine writes into the arenas).
struct CeLaunch {
  RankView views[kMaxRanks];  // [0] for a real rank; [r] per emulated rank (loopback, blockIdx.y)
  const Tile* tiles;          // the whole plan's tiles
  uint32_t n_tiles;
  int nranks;
  float scale;
  float lr;
  int epilogue;
  uint64_t slot_stride;
  uint64_t iter;              // this iteration's sequence number (>= 1, identical on every rank)
  uint32_t* done;             // per view: CTA completion counter
  int dtype;
};

#ifdef __CUDACC__

// Device bounds checks of the remote-write sites (arena stores, LL packets,
// barrier flags), compiled in with -DMGW_BOUNDS_CHECK (make
// EXTRA_NVCC=-DMGW_BOUNDS_CHECK): the pool has no compute-sanitizer, so a
// checked build runs the parity suites instead (tools/bounds_check.sh). A
// violation prints the site and traps (the test fails loudly).
#ifdef MGW_BOUNDS_CHECK
#define MGW_DCHECK(cond, what)                                                                       \
  do {                                                                                              \
    if (!(cond)) {                                                                                  \
      printf("MGW_BOUNDS_CHECK failed: %s (block %d,%d thread %d)\n", what, blockIdx.x, blockIdx.y, \
             threadIdx.x);                                                                          \
      __trap();                                                                                     \
    }                                                                                               \
  } while (0)
#else
#define MGW_DCHECK(cond, what) \
  do {                         \
  } while (0)
#endif

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t ld_acquire_sys_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Peer / merge-arena loads: L1-bypassing (.cg), so data written by another
// GPU after this SM last cached the line is never read stale.
__device__ __forceinline__ float4 ld_cg_v4(const float* p) {
  float4 v;
  asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

// Streaming gradient reads: read once per iteration, L2 only. Not .nc: in
// a real backward the gradients are written by other kernels while the
// persistent engine runs, so they are not read-only for the kernel's life.
__device__ __forceinline__ float4 ld_stream_v4(const float* p) {
  float4 v;
  asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ float4 ld_v4(const float* p) {
  return *reinterpret_cast<const float4*>(p);
}

__device__ __forceinline__ void st_v4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }

__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z),
                     __fadd_rn(a.w, b.w));
}

__device__ __forceinline__ float4 mul4(float4 a, float s) {
  return make_float4(__fmul_rn(a.x, s), __fmul_rn(a.y, s), __fmul_rn(a.z, s), __fmul_rn(a.w, s));
}

// w - lr*g with two roundings (never an FMA): the oracle's semantics.
__device__ __forceinline__ float sgd1(float w, float g, float lr) {
  return __fsub_rn(w, __fmul_rn(lr, g));
}

#endif  // __CUDACC__

}  // namespace mgw

#endif  // MGWFBP_DEVICE_CUH_
