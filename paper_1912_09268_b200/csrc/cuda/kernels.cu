// mgwfbp-b200 sm_100a kernels.
//
//  run_group<P, T>  — THE hot op, shared by both launch styles: for one
//      merge group, the gradient push over NVLink into the peers' merge
//      arenas -> rank-order reduction (x 1/P per source, fp32) from local HBM
//      -> unpack + SGD into the fp32 layer weights. T = float or bf16
//      gradients. Warp roles: a producer warp pushes gradients with TMA bulk
//      copies (global -> smem -> peer), 15 data warps reduce / apply / push
//      all-gather results.
//        one-shot: every rank pushes its tiles to every rank; 1 barrier per
//          chunk of 16 tiles per CTA.
//        two-shot: tile s*P+q is owned by rank q; ranks push each tile to its
//          owner (reduce-scatter), owners reduce + push the result to every
//          peer (all-gather) fused with SGD; pipelined RS(c) | RA(c-1) |
//          AP(c-2), one barrier per chunk.
//        LL: small one-shot groups as flag-in-data packets, no barrier.
//  engine_kernel<P, T> — the persistent comm engine: one launch per
//      iteration runs every group in backward order as soon as the compute
//      side marks it ready (paper Algorithm 2's daemon thread, on the GPU;
//      no per-group launch latency).
//  group_allreduce_kernel<P, TWO_SHOT, LOOPBACK, T> — one launch per group
//      (standalone C-ABI op, calibration of that op, the full-width tail of
//      a real backward, and the single-GPU loopback emulation of P ranks in
//      one cooperative launch).
//  pack_kernel / unpack_sgd_kernel — the standalone pack and unpack+SGD
//      ops of the C ABI (rank-local, HBM-bound).
//  replay_all_kernel / replay_kernel / mark_ready_kernel — backward replay
//      on %globaltimer and ready marks for the engine.
//
// Cross-rank synchronisation is per CTA index: CTA b of every rank handles
// the same tiles, so CTA b only waits for CTA b of the peers. Each CTA index
// counts its barriers (state counters, persisted across launches; identical
// on every rank because every rank runs the same launches); a barrier
// publishes the count to the peers' flag [b][me] (st.release.sys over
// NVLink) and waits until every peer's flag [b][q] reached it. Every
// collective launch starts with an entry barrier, so no rank overwrites a
// peer's merge arena while that peer may still read it from an earlier
// launch. Reductions use __fadd_rn / __fmul_rn / __fsub_rn only: no FMA
// contraction, bit-exact with the CPU oracle's fl(fl(x0*s) + x1*s)... in
// rank order.
#include <cstdint>
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "mgw_device.cuh"
#include "mgwfbp.h"

namespace mgw {

namespace {

constexpr uint64_t kTimeoutNs = 10ull * 1000 * 1000 * 1000;  // 10 s: error, never a hang
constexpr int kStages = 3;                           // TMA ring depth (32 KiB stages)
// Per-data-thread staging slots (16 B each) for the reduction's inputs,
// filled with cp.async so a whole batch (P sources + weights of up to 5
// vectors) is in flight without holding registers: 480 x 15 x 16 B.
constexpr uint32_t kStageSlots = 15;
constexpr uint32_t kStageBytes = kTileElems * 4;
// Software pipelining: a CTA walks its tiles in CHUNKS; while the producer
// warp pushes chunk c over NVLink the data warps reduce / apply chunk c-1
// (c-2); one barrier per chunk.

__device__ __forceinline__ float4 load_tail(const float* p, uint32_t n) {
  float4 v;
  v.x = n > 0 ? p[0] : 0.0f;
  v.y = n > 1 ? p[1] : 0.0f;
  v.z = n > 2 ? p[2] : 0.0f;
  v.w = n > 3 ? p[3] : 0.0f;
  return v;
}

// ---- gradient element types ------------------------------------------------
// Gradients and merge arenas are fp32 or bf16; weights
// and every sum are fp32. A "vector" is 4 consecutive elements (16 bytes of
// fp32, 8 of bf16) carried as a float4; bf16 -> fp32 is exact, fp32 -> bf16
// rounds to nearest even (__float2bfloat16_rn).
using bf16 = __nv_bfloat16;

template <typename T>
struct Elem;
template <>
struct Elem<float> {
  static constexpr uint32_t kVec = 4;  // elements per 16 bytes (TMA / layout granule)
};
template <>
struct Elem<bf16> {
  static constexpr uint32_t kVec = 8;
};

template <typename T>
__device__ __forceinline__ T* as(float* p) {
  return reinterpret_cast<T*>(p);
}

__device__ __forceinline__ float4 unpack_bf16x4(uint32_t a, uint32_t b) {
  return make_float4(__uint_as_float(a << 16), __uint_as_float(a & 0xffff0000u), __uint_as_float(b << 16),
                     __uint_as_float(b & 0xffff0000u));
}

__device__ __forceinline__ uint32_t bf16_bits(float x) {
  return static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(x)));
}

// 4 elements -> float4: L1-bypassing (peer-written arena data)
template <typename T>
__device__ __forceinline__ float4 ld4_cg(const T* p);
template <>
__device__ __forceinline__ float4 ld4_cg<float>(const float* p) {
  return ld_cg_v4(p);
}
template <>
__device__ __forceinline__ float4 ld4_cg<bf16>(const bf16* p) {
  uint32_t a, b;
  asm volatile("ld.global.cg.v2.u32 {%0,%1}, [%2];" : "=r"(a), "=r"(b) : "l"(p));
  return unpack_bf16x4(a, b);
}

// 4 elements -> float4: streaming read-once gradients
template <typename T>
__device__ __forceinline__ float4 ld4_stream(const T* p);
template <>
__device__ __forceinline__ float4 ld4_stream<float>(const float* p) {
  return ld_stream_v4(p);
}
template <>
__device__ __forceinline__ float4 ld4_stream<bf16>(const bf16* p) {
  uint32_t a, b;
  asm volatile("ld.global.cg.v2.u32 {%0,%1}, [%2];" : "=r"(a), "=r"(b) : "l"(p));
  return unpack_bf16x4(a, b);
}

template <typename T>
__device__ __forceinline__ float4 ld4(const T* p) {
  if constexpr (sizeof(T) == 4) {
    return ld_v4(reinterpret_cast<const float*>(p));
  } else {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    return unpack_bf16x4(u.x, u.y);
  }
}

// First n (< 4 allowed) elements, zero-filled, any alignment.
template <typename T>
__device__ __forceinline__ float4 ld4_tail(const T* p, uint32_t n) {
  if constexpr (sizeof(T) == 4) {
    return load_tail(reinterpret_cast<const float*>(p), n);
  } else {
    float4 v;
    v.x = n > 0 ? __bfloat162float(p[0]) : 0.0f;
    v.y = n > 1 ? __bfloat162float(p[1]) : 0.0f;
    v.z = n > 2 ? __bfloat162float(p[2]) : 0.0f;
    v.w = n > 3 ? __bfloat162float(p[3]) : 0.0f;
    return v;
  }
}

// float4 -> 4 elements (bf16: round to nearest even)
template <typename T>
__device__ __forceinline__ void st4(T* p, float4 v) {
  if constexpr (sizeof(T) == 4) {
    st_v4(reinterpret_cast<float*>(p), v);
  } else {
    *reinterpret_cast<uint2*>(p) =
        make_uint2(bf16_bits(v.x) | (bf16_bits(v.y) << 16), bf16_bits(v.z) | (bf16_bits(v.w) << 16));
  }
}

template <typename T>
__device__ __forceinline__ void st_tail(T* p, float4 v, uint32_t n) {
  if constexpr (sizeof(T) == 4) {
    if (n > 0) p[0] = v.x;
    if (n > 1) p[1] = v.y;
    if (n > 2) p[2] = v.z;
    if (n > 3) p[3] = v.w;
  } else {
    if (n > 0) p[0] = __float2bfloat16_rn(v.x);
    if (n > 1) p[1] = __float2bfloat16_rn(v.y);
    if (n > 2) p[2] = __float2bfloat16_rn(v.z);
    if (n > 3) p[3] = __float2bfloat16_rn(v.w);
  }
}

// The reduced gradient in the gradient type: identity for fp32; bf16 rounds
// the fp32 rank-order sum once, and every rank applies that same value.
template <typename T>
__device__ __forceinline__ float4 round4(float4 v) {
  if constexpr (sizeof(T) == 4) {
    return v;
  } else {
    return unpack_bf16x4(bf16_bits(v.x) | (bf16_bits(v.y) << 16), bf16_bits(v.z) | (bf16_bits(v.w) << 16));
  }
}

// Standalone pack of tile t: gather + x scale into the merge buffer; each
// thread has all its kPackVec loads in flight before any store.
constexpr uint32_t kPackVec = kTileElems / 4 / kBlock;
template <typename T>
__device__ __forceinline__ void pack_tile(const Tile& t, float* const* grads, T* dst_base, float scale) {
  const T* src = as<T>(grads[t.layer & kLayerMask]) + t.src;
  T* dst = dst_base + t.moff;
  const bool aligned = !(t.layer & kGradUnaligned);
  const uint32_t nvec = (t.len + 3) >> 2;
  float4 x[kPackVec];
#pragma unroll
  for (uint32_t k = 0; k < kPackVec; ++k) {
    const uint32_t i = threadIdx.x + k * kBlock;
    const uint32_t e = i * 4;
    if (i < nvec) x[k] = (aligned && e + 4 <= t.len) ? ld4_stream<T>(src + e) : ld4_tail<T>(src + e, t.len - e);
  }
#pragma unroll
  for (uint32_t k = 0; k < kPackVec; ++k) {
    const uint32_t i = threadIdx.x + k * kBlock;
    if (i < nvec) st4<T>(dst + i * 4, mul4(x[k], scale));
  }
}

// Element group e..e+3 of tile t receives the reduced gradient `g`.
template <typename T>
__device__ __forceinline__ void epilogue(const Tile& t, uint32_t e, float4 g, float* w_layer, T* g_layer,
                                         float lr, int epi) {
  const uint32_t n = t.len - e < 4 ? t.len - e : 4;
  if ((epi & MGW_SGD) && w_layer != nullptr) {
    float* w = w_layer + t.src + e;
    if (n == 4 && !(t.layer & kWeightUnaligned)) {
      float4 wv = ld_v4(w);
      wv.x = sgd1(wv.x, g.x, lr);
      wv.y = sgd1(wv.y, g.y, lr);
      wv.z = sgd1(wv.z, g.z, lr);
      wv.w = sgd1(wv.w, g.w, lr);
      st_v4(w, wv);
    } else {  // ragged tail or unaligned layer: scalar, no local-memory array
      if (n > 0) w[0] = sgd1(w[0], g.x, lr);
      if (n > 1) w[1] = sgd1(w[1], g.y, lr);
      if (n > 2) w[2] = sgd1(w[2], g.z, lr);
      if (n > 3) w[3] = sgd1(w[3], g.w, lr);
    }
  }
  if (epi & MGW_WRITE_GRAD) {
    T* d = g_layer + t.src + e;
    if (n == 4 && !(t.layer & kGradUnaligned)) {
      st4<T>(d, g);
    } else {
      st_tail<T>(d, g, n);
    }
  }
}

// Errors: a bounded wait (10 s of %globaltimer) expired — a peer or the
// compute side never arrived. The error is recorded in the rank's state word
// and in the communicator's host-mapped word (the host reads it without a
// CUDA call); every later wait gives up at once, a CTA that gave up stops
// publishing its barrier flags (so its peers time out too instead of
// reducing partial data), and no SGD / write-back epilogue runs on data that
// was never synchronised. A communicator that raised an error stays failed.
__device__ __forceinline__ void raise_error(const RankView& v) {
  atomicExch(v.state + kStateError, 1u);
  if (v.host_err != nullptr) *reinterpret_cast<volatile uint32_t*>(v.host_err) = 1u;
}

__device__ __forceinline__ bool error_raised(const RankView& v) {
  return ld_volatile_u32(v.state + kStateError) != 0;
}

// Spin until done() holds; false on timeout or when an error was raised
// elsewhere (checked every 64 polls, off the fast path).
template <typename Done>
__device__ __forceinline__ bool spin_until(const RankView& v, Done done) {
  if (done()) return true;
  const uint64_t t0 = globaltimer_ns();
  for (uint32_t n = 1;; ++n) {
    if (done()) return true;
    if ((n & 63) == 0) {
      if (error_raised(v)) return false;
      if (globaltimer_ns() - t0 > kTimeoutNs) {
        raise_error(v);
        return false;
      }
    }
  }
}

// Everything a CTA needs to run groups: its barrier counter, the launch's LL
// epoch, the abort state and, for the producer warp, the TMA ring.
struct PushRing {
  uint32_t head;
  uint32_t phase;  // bit k: parity to wait for on stage k
};

struct CtaCtx {
  uint32_t count;     // barrier count of this CTA index (identical on every rank)
  uint32_t epoch;     // LL epoch of this launch: the rank's launch sequence + 1
  bool abort;         // a wait of this CTA gave up: no more epilogues, no more flags
  uint32_t* s_abort;  // CTA-shared abort word
  PushRing ring;
  uint8_t* stages;
  float4* staging;  // data warps' cp.async slots (after the TMA ring)
  uint64_t* bars;
  bool producer;
};

// Barrier of CTA index `cta` with the same CTA index of every rank.
// bar.sync orders every warp's posted NVLink stores (and the producer warp's
// completed, proxy-fenced bulk copies) before the flag writers'
// st.release.sys; release is cumulative at system scope, so a peer that
// acquires the flag sees the data (no per-thread fence.sys).
//
// The flag slot is the PHYSICAL CTA index (blockIdx.x), whose counter cx.count
// is: inside the engine a CTA runs groups under a rotated, group-local index,
// and two CTAs with different counters must never share a slot.
__device__ __forceinline__ void cta_barrier(const RankView& v, int P, CtaCtx& cx) {
  const uint32_t cta = blockIdx.x;
  ++cx.count;
  __syncthreads();
  if (threadIdx.x < P && !cx.abort) {
    const int q = threadIdx.x;
    const uint32_t want = cx.count;
    MGW_DCHECK(cta < static_cast<uint32_t>(kMaxCtas), "barrier flag CTA index");
    st_release_sys(v.signal[q] + cta * kMaxRanks + v.rank, want);
    const uint32_t* mine = v.signal[v.rank] + cta * kMaxRanks + q;
    if (!spin_until(v, [&] { return static_cast<int32_t>(ld_acquire_sys(mine) - want) >= 0; })) {
      *cx.s_abort = 1u;
    }
  }
  __syncthreads();
  cx.abort = *reinterpret_cast<volatile uint32_t*>(cx.s_abort) != 0;
}

// ---- push data path -------------------------------------------------------
// Every rank's merge arena holds one SLOT per source rank (slot r at element
// r * slot_stride, laid out like the merge buffer). Transfers are posted
// NVLink writes into the peers' slots (no remote-load latency on the
// critical path); every reduction reads local HBM only.
//
// Warp roles inside a CTA (kBlock = 16 warps):
//   data warps (threads [0, kThreads))  reduce / SGD / all-gather pushes
//   producer warp (the last warp)       the gradient pushes, as TMA bulk
//       copies: lane 0 streams tiles global -> shared (cp.async.bulk +
//       mbarrier complete_tx) -> the peers' arenas (cp.async.bulk
//       shared -> global over NVLink), kStages x 32 KiB in flight, no
//       register traffic. The whole warp handles the rare tiles TMA cannot
//       (16-byte-unaligned layer views) and the < 4-element layer tails.
// The gradients are pushed UNSCALED; the receiver multiplies every source
// by 1/P before the rank-order sum — fl(x * 1/P) is the same value wherever
// it is computed, so the result is unchanged bit for bit. A rank's own
// contribution is read straight from its gradients (no self-slot copy).

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void ring_init(uint64_t* bars) {
#pragma unroll
  for (int k = 0; k < kStages; ++k) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bars + k)) : "memory");
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void tma_load(uint32_t stage_addr, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(stage_addr),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void tma_store(void* dst, uint32_t stage_addr, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(stage_addr), "r"(bytes)
               : "memory");
}

// Wait for stage `bar` to reach `parity` (bounded like every wait).
__device__ __forceinline__ bool mbar_wait(const RankView& v, uint32_t bar, uint32_t parity) {
  return spin_until(v, [&] {
    uint32_t done = 0;
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    return done != 0;
  });
}

// Bulk copies of the tile's 16-byte body (a multiple of Elem<T>::kVec
// elements) are the TMA's; the rest (unaligned layer view: the whole tile;
// else the < 16-byte tail) goes through registers.
template <typename T>
__device__ __forceinline__ bool tma_able(const Tile& t) {
  return !(t.layer & kGradUnaligned) && t.len >= Elem<T>::kVec;
}

template <typename T>
__device__ __forceinline__ uint32_t tma_body(const Tile& t) {
  return t.len & ~(Elem<T>::kVec - 1);
}

// One push item: a tile and the ranks it goes to.
struct PushItem {
  Tile t;
  uint32_t mask;  // bit q: push into rank q's arena (0: no tile)
};

// Push the items of one chunk, enumerated by `item(i)`. Producer warp only.
template <int P, typename T, typename Item>
__device__ __forceinline__ void push_items(const RankView& v, uint32_t n_items, uint64_t my_slot,
                                           PushRing& ring, uint8_t* stages, uint64_t* bars,
                                           uint32_t* s_abort, Item item) {
  const uint32_t lane = threadIdx.x & 31;
  if (lane == 0) {
    // gradients were written by generic-proxy stores (backward / earlier
    // kernels, ordered by the ready flag): make them visible to the TMA
    asm volatile("fence.proxy.async.global;" ::: "memory");
    const uint32_t s0 = smem_u32(stages);
    uint32_t iL = 0, iS = 0, nl = 0, ns = 0;
    for (;;) {
      // prefill kStages loads; then refill the stage of item nl - kStages
      // once its store group has read it: wait_group.read 1 leaves only the
      // latest group (item ns - 1) pending, so that needs nl <= ns + kStages - 2
      while (iL < n_items && (nl < kStages || nl + 2 <= ns + kStages)) {
        const PushItem it = item(iL++);
        if (it.mask == 0 || !tma_able<T>(it.t)) continue;
        if (nl >= kStages) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        const uint32_t k = (ring.head + nl) % kStages;
        tma_load(s0 + k * kStageBytes, as<T>(v.grads[it.t.layer & kLayerMask]) + it.t.src,
                 tma_body<T>(it.t) * static_cast<uint32_t>(sizeof(T)), smem_u32(bars + k));
        ++nl;
      }
      if (ns == nl) break;
      PushItem it;
      do {
        it = item(iS++);
      } while (it.mask == 0 || !tma_able<T>(it.t));
      const uint32_t k = (ring.head + ns) % kStages;
      if (!mbar_wait(v, smem_u32(bars + k), (ring.phase >> k) & 1u)) *s_abort = 1u;
      ring.phase ^= 1u << k;
      const uint32_t bytes = tma_body<T>(it.t) * static_cast<uint32_t>(sizeof(T));
#pragma unroll
      for (int q = 0; q < P; ++q) {
        MGW_DCHECK((my_slot + it.t.moff) * sizeof(T) + bytes <= v.arena_bytes, "TMA push into a peer arena");
        if (it.mask & (1u << q)) tma_store(as<T>(v.arena[q]) + my_slot + it.t.moff, s0 + k * kStageBytes, bytes);
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      ++ns;
    }
    ring.head = (ring.head + nl) % kStages;
  }
  __syncwarp();
  // register path: unaligned tiles (whole warp) and tails (lane 0)
  for (uint32_t i = 0; i < n_items; ++i) {
    const PushItem it = item(i);
    if (it.mask == 0 || (tma_able<T>(it.t) && tma_body<T>(it.t) == it.t.len)) continue;
    const T* src = as<T>(v.grads[it.t.layer & kLayerMask]) + it.t.src;
    const uint32_t first = tma_able<T>(it.t) ? tma_body<T>(it.t) : 0;  // elements the TMA did
    const uint32_t nvec = (it.t.len - first + 3) >> 2;
    for (uint32_t j = lane; j < nvec; j += 32) {
      const uint32_t e = first + j * 4;
      const float4 x = ld4_tail<T>(src + e, it.t.len - e);  // (bf16 -> fp32 -> bf16 is exact)
#pragma unroll
      for (int q = 0; q < P; ++q) {
        MGW_DCHECK((my_slot + it.t.moff + e + 4) * sizeof(T) <= v.arena_bytes, "register push into a peer arena");
        if (it.mask & (1u << q)) st4<T>(as<T>(v.arena[q]) + my_slot + it.t.moff + e, x);
      }
    }
  }
}

// End of a step for the producer: its bulk copies are complete (written to
// the peers) and ordered before the generic-proxy flag release.
__device__ __forceinline__ void push_drain() {
  if ((threadIdx.x & 31) == 0) {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    asm volatile("fence.proxy.async.global;" ::: "memory");
  }
  __syncwarp();
}

// Weight vectors of B vectors of tile t (thread vector indices i0, i0 +
// stride, ...), loaded up front so their latency overlaps the gradient loads.
template <uint32_t B>
__device__ __forceinline__ void load_w_batch(const Tile& t, uint32_t i0, uint32_t stride, const float* w_layer,
                                             int epi, float4 (&wv)[B]) {
  const uint32_t nvec = (t.len + 3) >> 2;
  const bool vec_w = (epi & MGW_SGD) && w_layer != nullptr && !(t.layer & kWeightUnaligned);
#pragma unroll
  for (uint32_t j = 0; j < B; ++j) {
    const uint32_t i = i0 + j * stride;
    if (vec_w && i < nvec && i * 4 + 4 <= t.len) wv[j] = ld_v4(w_layer + t.src + i * 4);
  }
}

// SGD (+ optional grad write-back) for the B vectors, with their weights wv
// from load_w_batch.
template <uint32_t B, typename T>
__device__ __forceinline__ void apply_batch(const Tile& t, uint32_t i0, uint32_t stride,
                                            const float4 (&g)[B], const float4 (&wv)[B], float* w_layer,
                                            T* g_layer, float lr, int epi) {
  const uint32_t nvec = (t.len + 3) >> 2;
  const bool vec_w = (epi & MGW_SGD) && w_layer != nullptr && !(t.layer & kWeightUnaligned);
#pragma unroll
  for (uint32_t j = 0; j < B; ++j) {
    const uint32_t i = i0 + j * stride;
    if (i >= nvec) continue;
    const uint32_t e = i * 4;
    if (vec_w && e + 4 <= t.len) {
      float4 w = wv[j];
      w.x = sgd1(w.x, g[j].x, lr);
      w.y = sgd1(w.y, g[j].y, lr);
      w.z = sgd1(w.z, g[j].z, lr);
      w.w = sgd1(w.w, g[j].w, lr);
      st_v4(w_layer + t.src + e, w);
      if (epi & MGW_WRITE_GRAD) epilogue<T>(t, e, g[j], nullptr, g_layer, lr, MGW_WRITE_GRAD);
    } else {
      epilogue<T>(t, e, g[j], w_layer, g_layer, lr, epi);  // tail / unaligned / no-SGD
    }
  }
}

// cp.async (LDGSTS, L2-only .cg) of 16 bytes into this thread's staging slot.
__device__ __forceinline__ void cp_async16(float4* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}

// 8-byte cp.async (a bf16 vector). .ca (the only 8-byte form) may allocate
// in L1; safe here: within a launch every arena address is read at most once
// per CTA (groups and phases use disjoint bytes), and kernel boundaries
// invalidate L1.
__device__ __forceinline__ void cp_async8(float4* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}

template <typename T>
__device__ __forceinline__ void cp_async_vec(float4* smem, const T* gmem) {
  if constexpr (sizeof(T) == 4) {
    cp_async16(smem, gmem);
  } else {
    cp_async8(smem, gmem);
  }
}

// A staged vector: fp32 as is; bf16 as its raw 8 bytes in the slot's first half.
template <typename T>
__device__ __forceinline__ float4 slot_load(const float4* slot) {
  if constexpr (sizeof(T) == 4) {
    return *slot;
  } else {
    const uint2 u = *reinterpret_cast<const uint2*>(slot);
    return unpack_bf16x4(u.x, u.y);
  }
}

template <typename T>
__device__ __forceinline__ void slot_store(float4* slot, float4 v) {  // v exact in T
  if constexpr (sizeof(T) == 4) {
    *slot = v;
  } else {
    *reinterpret_cast<uint2*>(slot) = make_uint2((__float_as_uint(v.x) >> 16) | (__float_as_uint(v.y) & 0xffff0000u),
                                                 (__float_as_uint(v.z) >> 16) | (__float_as_uint(v.w) & 0xffff0000u));
  }
}

// Reduction with staged inputs: for a batch of B vectors per thread,
// every source slot, the own gradient and the weight vector are copied
// global -> shared with cp.async (one memory latency per batch, B * (P + 1)
// <= kStageSlots 16-byte slots per thread, conflict-free: slot k of thread t
// at stage[k * kThreads + t]); then each vector is summed in rank order from
// shared memory, pushed to the peers (all-gather) and applied. Bit-identical
// to reduce_tile: the same operands, the same operation order.
template <int P>
struct StagedBatch {
  static constexpr uint32_t raw = kStageSlots / (P + 1);
  static constexpr uint32_t value = raw < kVecPerThread ? raw : kVecPerThread;
};

template <int P, typename T>
__device__ __forceinline__ void reduce_tile_staged(const RankView& v, const Tile& t, uint64_t slot_stride,
                                                   bool push_to_peers, uint64_t my_slot, float scale, float lr,
                                                   int epi, float4* stage) {
  constexpr uint32_t B = StagedBatch<P>::value;
  static_assert(B >= 1, "staging slots too few for P");
  const T* base = as<T>(v.arena[v.rank]) + t.moff;
  const uint32_t nvec = (t.len + 3) >> 2;
  const uint32_t layer = t.layer & kLayerMask;
  float* w = v.weights[layer];
  T* g = as<T>(v.grads[layer]);
  const T* own = g + t.src;
  const bool own_aligned = !(t.layer & kGradUnaligned);
  const bool vec_w = (epi & MGW_SGD) && w != nullptr && !(t.layer & kWeightUnaligned);
  float4* my = stage + threadIdx.x;
  auto slot = [&](uint32_t k) { return my + k * kThreads; };
#pragma unroll 1
  for (uint32_t k0 = 0; k0 < kVecPerThread; k0 += B) {
    const uint32_t i0 = threadIdx.x + k0 * kThreads;
    if (i0 >= nvec) break;
#pragma unroll
    for (uint32_t j = 0; j < B; ++j) {
      const uint32_t i = i0 + j * kThreads;
      if (i >= nvec) continue;
      const uint32_t e = i * 4;
      const bool full = e + 4 <= t.len;
#pragma unroll
      for (int r = 0; r < P; ++r) {
        if (r != v.rank) cp_async_vec<T>(slot(j * (P + 1) + r), base + r * slot_stride + e);
      }
      if (own_aligned && full) cp_async_vec<T>(slot(j * (P + 1) + v.rank), own + e);
      else slot_store<T>(slot(j * (P + 1) + v.rank), ld4_tail<T>(own + e, t.len - e));
      if (vec_w && full) cp_async16(slot(j * (P + 1) + P), w + t.src + e);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll 1
    for (uint32_t j = 0; j < B; ++j) {
      const uint32_t i = i0 + j * kThreads;
      if (i >= nvec) break;
      float4 s[1], wv[1];
      s[0] = mul4(slot_load<T>(slot(j * (P + 1))), scale);
#pragma unroll
      for (int r = 1; r < P; ++r) s[0] = add4(s[0], mul4(slot_load<T>(slot(j * (P + 1) + r)), scale));
      s[0] = round4<T>(s[0]);
      wv[0] = *slot(j * (P + 1) + P);  // (unused by the scalar epilogue paths)
      if (push_to_peers) {
#pragma unroll
        for (int q = 0; q < P; ++q) {
          MGW_DCHECK((my_slot + t.moff + i * 4 + 4) * sizeof(T) <= v.arena_bytes, "all-gather push into a peer arena");
          if (q != v.rank) st4<T>(as<T>(v.arena[q]) + my_slot + t.moff + i * 4, s[0]);
        }
      }
      apply_batch<1, T>(t, i, kThreads, s, wv, w, g, lr, epi);
    }
  }
}

// ---- LL (flag-in-data) one-shot for small groups ----------------------------
// Every 32-bit word of gradient data travels with a 32-bit epoch in ONE
// naturally aligned 8-byte store (single-copy atomic), so a receiver that
// sees the epoch sees the data: no barrier, no release/acquire round trip —
// one NVLink trip per group. The epoch is the CTA's barrier count after the
// launch's entry barrier (identical on every rank for CTA index b, strictly
// increasing across launches; LL groups of one launch use disjoint packets).

__device__ __forceinline__ uint64_t* ll_slot(const RankView& v, int q, int src) {
  return reinterpret_cast<uint64_t*>(v.signal[q] + kLLWord) + static_cast<uint64_t>(src) * kLLSlotPackets;
}

// The 4-element vector's raw gradient words: fp32 4 words, bf16 2.
template <typename T>
__device__ __forceinline__ void ll_send(uint64_t* dst, float4 x, uint32_t epoch) {
  const uint64_t e = static_cast<uint64_t>(epoch) << 32;
  if constexpr (sizeof(T) == 4) {
    asm volatile("st.volatile.global.v2.b64 [%0], {%1, %2};" ::"l"(dst), "l"(e | __float_as_uint(x.x)),
                 "l"(e | __float_as_uint(x.y))
                 : "memory");
    asm volatile("st.volatile.global.v2.b64 [%0], {%1, %2};" ::"l"(dst + 2), "l"(e | __float_as_uint(x.z)),
                 "l"(e | __float_as_uint(x.w))
                 : "memory");
  } else {  // bf16 values are exact in fp32: repack the raw bits
    const uint32_t w0 = (__float_as_uint(x.x) >> 16) | (__float_as_uint(x.y) & 0xffff0000u);
    const uint32_t w1 = (__float_as_uint(x.z) >> 16) | (__float_as_uint(x.w) & 0xffff0000u);
    asm volatile("st.volatile.global.v2.b64 [%0], {%1, %2};" ::"l"(dst), "l"(e | w0), "l"(e | w1) : "memory");
  }
}

__device__ __forceinline__ bool ll_pair(const uint64_t* p, uint32_t epoch, uint32_t& w0, uint32_t& w1) {
  uint64_t a, b;
  asm volatile("ld.volatile.global.v2.b64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
  w0 = static_cast<uint32_t>(a);
  w1 = static_cast<uint32_t>(b);
  return static_cast<uint32_t>(a >> 32) == epoch && static_cast<uint32_t>(b >> 32) == epoch;
}

// Spin until the vector's packets carry `epoch` (bounded); false if the
// wait gave up (the caller then skips this vector's epilogue).
template <typename T>
__device__ __forceinline__ bool ll_recv(const RankView& v, const uint64_t* src, uint32_t epoch, float4& out) {
  uint32_t w[4] = {0, 0, 0, 0};
  constexpr int kPairs = sizeof(T) == 4 ? 2 : 1;
  bool ok = true;
#pragma unroll
  for (int k = 0; k < kPairs; ++k) {
    ok = ok && spin_until(v, [&] { return ll_pair(src + 2 * k, epoch, w[2 * k], w[2 * k + 1]); });
  }
  if constexpr (sizeof(T) == 4) {
    out = make_float4(__uint_as_float(w[0]), __uint_as_float(w[1]), __uint_as_float(w[2]), __uint_as_float(w[3]));
  } else {
    out = unpack_bf16x4(w[0], w[1]);
  }
  return ok;
}

// A small one-shot group over LL packets, all 16 warps. Work unit: one
// kBlock-vector PART of a tile (one vector per thread), so even a 2-tile
// group spreads over 8 CTAs — the group is latency-bound, not per-CTA
// bandwidth-bound. Send the vector to every peer, then receive, rank-order
// sum (own contribution in place), SGD. Tile t's packets start at
// ll_pkt + (t.moff - mbase) * sizeof(T) / 4. The epoch is the launch's
// (unique per launch of the communicator, identical on every rank), so a
// packet left in a slot by an earlier launch — any plan, any CTA mapping —
// never matches.
// (kLLParts: mgw_device.cuh; the data threads [0, kThreads) take part.)
template <int P, typename T>
__device__ __noinline__ void ll_group(const RankView& v, const Tile* tiles, uint32_t n_tiles, uint32_t ll_pkt,
                                      uint32_t mbase, float scale, float lr, int epi, uint32_t cta,
                                      uint32_t ncta, uint32_t epoch) {
  constexpr uint32_t kW = sizeof(T);  // packets per 4-element vector
  const int me = v.rank;
  if (threadIdx.x >= kThreads) return;
  for (uint32_t u = cta; u < n_tiles * kLLParts; u += ncta) {
    const Tile t = tiles[u / kLLParts];
    const uint32_t i = (u % kLLParts) * kThreads + threadIdx.x;  // this thread's vector
    const uint32_t nvec = (t.len + 3) >> 2;
    if (i >= nvec) continue;
    const uint32_t layer = t.layer & kLayerMask;
    T* g = as<T>(v.grads[layer]);
    const T* own = g + t.src;
    float* w = v.weights[layer];
    const uint32_t e = i * 4;
    const uint64_t pkt = ll_pkt + static_cast<uint64_t>(t.moff - mbase) * sizeof(T) / 4 + static_cast<uint64_t>(i) * kW;
    float4 x[1], wv[1];
    x[0] = (!(t.layer & kGradUnaligned) && e + 4 <= t.len) ? ld4_stream<T>(own + e) : ld4_tail<T>(own + e, t.len - e);
#pragma unroll
    for (int q = 0; q < P; ++q) {
      MGW_DCHECK(pkt + kW <= kLLSlotPackets, "LL packet slot");
      if (q != me) ll_send<T>(ll_slot(v, q, me) + pkt, x[0], epoch);
    }
    load_w_batch<1>(t, i, kThreads, w, epi, wv);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    bool ok = true;
#pragma unroll
    for (int r = 0; r < P; ++r) {
      float4 xr = x[0];
      if (r != me) ok = ll_recv<T>(v, ll_slot(v, me, r) + pkt, epoch, xr) && ok;
      acc = r == 0 ? mul4(xr, scale) : add4(acc, mul4(xr, scale));
    }
    x[0] = round4<T>(acc);
    if (ok) apply_batch<1, T>(t, i, kThreads, x, wv, w, g, lr, epi);
  }
}

// Chunk of a CTA's pipelined loop: at most `cap` units, and small enough
// that a CTA with `mine` units runs at least `min_chunks` chunks (so the
// push of chunk c overlaps the reduction of chunk c-1 even for mid-size
// groups where every CTA owns only a few units).
__device__ __forceinline__ uint32_t chunk_units(uint32_t mine, uint32_t cap, uint32_t min_chunks) {
  const uint32_t m = min_chunks > 0 ? min_chunks : 1;
  const uint32_t c = (mine + m - 1) / m;
  return c < 1 ? 1 : (c > cap ? cap : c);
}

// One-shot, pipelined over chunks of this CTA's tiles (cta + j*ncta):
//   step t: producer pushes chunk t to every peer (TMA) | data warps reduce
//   + SGD chunk t-1 from the local slots; barrier (if t < n).
// NVLink: (P-1) * S posted writes per rank.
template <int P, typename T>
__device__ __forceinline__ void one_shot_group(const RankView& v, const Tile* tiles,
                                               uint32_t n_tiles, uint64_t slot_stride, float scale,
                                               float lr, int epi, uint32_t cta, uint32_t ncta,
                                               uint32_t chunk, uint32_t min_chunks, CtaCtx& cx) {
  const uint64_t my_slot = static_cast<uint64_t>(v.rank) * slot_stride;
  const uint32_t mine = cta < n_tiles ? (n_tiles - cta + ncta - 1) / ncta : 0;  // my tiles
  const uint32_t C = chunk_units(mine, chunk, min_chunks);
  const uint32_t n_chunks = (mine + C - 1) / C;
  const uint32_t peers = ((1u << P) - 1u) & ~(1u << v.rank);
#pragma unroll 1
  for (uint32_t t = 0; t <= n_chunks && n_chunks > 0; ++t) {
    if (cx.producer) {
      if (t < n_chunks && !cx.abort) {
        const uint32_t j0 = t * C;
        const uint32_t n = mine - j0 < C ? mine - j0 : C;
        push_items<P, T>(v, n, my_slot, cx.ring, cx.stages, cx.bars, cx.s_abort, [&](uint32_t i) {
          return PushItem{tiles[cta + (j0 + i) * ncta], peers};
        });
        push_drain();
      }
    } else if (t >= 1 && !cx.abort) {
#pragma unroll 1
      for (uint32_t j = (t - 1) * C; j < mine && j < t * C; ++j) {
        reduce_tile_staged<P, T>(v, tiles[cta + j * ncta], slot_stride, false, my_slot, scale, lr, epi, cx.staging);
      }
    }
    if (t < n_chunks) cta_barrier(v, P, cx);
  }
}

// Two-shot: super-tile s = tiles [s*P, s*P+P), tile s*P+q owned by rank q.
//   RS(c):  push each tile of chunk c to its owner's slot `me` (producer, TMA)
//   RA(c):  owner: rank-order sum of its tile, SGD, push the result into
//           slot `owner` of every peer (all-gather)
//   AP(c):  apply the other owners' results from the local slots (SGD)
// step t: RS(t) [producer] | RA(t-1), AP(t-2) [data warps]; barrier (t <= n).
// NVLink: 2 (P-1)/P * S posted writes per rank.
template <int P, typename T>
__device__ __forceinline__ void two_shot_group(const RankView& v, const Tile* tiles,
                                               uint32_t n_tiles, uint64_t slot_stride, float scale,
                                               float lr, int epi, uint32_t cta, uint32_t ncta,
                                               uint32_t chunk, uint32_t min_chunks, CtaCtx& cx) {
  const uint64_t my_slot = static_cast<uint64_t>(v.rank) * slot_stride;
  const uint32_t n_super = (n_tiles + P - 1) / P;
  const uint32_t mine = cta < n_super ? (n_super - cta + ncta - 1) / ncta : 0;  // my super-tiles
  const uint32_t C = chunk_units(mine, chunk > P ? chunk / P : 1, min_chunks);
  const uint32_t n_chunks = (mine + C - 1) / C;
  const int me = v.rank;
#pragma unroll 1
  for (uint32_t t = 0; t <= n_chunks + 1 && n_chunks > 0; ++t) {
    if (cx.producer) {
      if (t < n_chunks && !cx.abort) {
        const uint32_t j0 = t * C;
        const uint32_t ns = mine - j0 < C ? mine - j0 : C;
        push_items<P, T>(v, ns * (P - 1), my_slot, cx.ring, cx.stages, cx.bars, cx.s_abort,
                         [&](uint32_t i) {
                           const uint32_t s = cta + (j0 + i / (P - 1)) * ncta;
                           const int qi = static_cast<int>(i % (P - 1));
                           const int q = qi < me ? qi : qi + 1;
                           const uint32_t ti = s * P + q;
                           return ti < n_tiles ? PushItem{tiles[ti], 1u << q} : PushItem{Tile{}, 0u};
                         });
        push_drain();
      }
    } else if (!cx.abort) {
      if (t >= 1 && t <= n_chunks) {  // RA(t-1)
#pragma unroll 1
        for (uint32_t j = (t - 1) * C; j < mine && j < t * C; ++j) {
          const uint32_t ti = (cta + j * ncta) * P + me;
          if (ti < n_tiles) reduce_tile_staged<P, T>(v, tiles[ti], slot_stride, true, my_slot, scale, lr, epi, cx.staging);
        }
      }
      if (t >= 2) {  // AP(t-2)
#pragma unroll 1
        for (uint32_t j = (t - 2) * C; j < mine && j < (t - 1) * C; ++j) {
          const uint32_t s = cta + j * ncta;
#pragma unroll 1
          for (int q = 0; q < P; ++q) {
            const uint32_t ti = s * P + q;
            if (q == me || ti >= n_tiles) continue;
            const Tile tl = tiles[ti];
            const T* red = as<T>(v.arena[me]) + static_cast<uint64_t>(q) * slot_stride + tl.moff;
            const uint32_t layer = tl.layer & kLayerMask;
            const uint32_t nvec = (tl.len + 3) >> 2;
            float4 x[kVecPerThread], wv[kVecPerThread];
#pragma unroll
            for (uint32_t k = 0; k < kVecPerThread; ++k) {
              const uint32_t i = threadIdx.x + k * kThreads;
              if (i < nvec) x[k] = ld4_cg<T>(red + i * 4);
            }
            load_w_batch<kVecPerThread>(tl, threadIdx.x, kThreads, v.weights[layer], epi, wv);
            apply_batch<kVecPerThread, T>(tl, threadIdx.x, kThreads, x, wv, v.weights[layer],
                                          as<T>(v.grads[layer]), lr, epi);
          }
        }
      }
    }
    if (t <= n_chunks) cta_barrier(v, P, cx);
  }
}

// ---- streamed protocol: no per-chunk barrier --------------------------------
// The producer warp and the data warps of a CTA run DECOUPLED over the CTA's
// whole work list (every group of the launch in FIFO order). The producer
// streams gradient tiles to their destinations with TMA bulk copies and, once
// a tile's copies have completed (cp.async.bulk.wait_group, two tiles of
// lag), raises the destination's rs[b][me] delivery count; the data warps
// consume tiles in the same order as their counts arrive (two-shot owners
// push the reduced tile to every peer with register stores and raise
// ag[b][me]). Every tile of a launch lands in its own arena bytes, so no
// one ever waits for a consumer: the only cross-rank waits are data
// arrivals, the NVLink pipe never drains between chunks, and the producer
// runs ahead into the next group while the data warps still reduce the
// previous one. The launch's entry barrier (cta_ctx_init) keeps arena reuse
// across launches safe.

__device__ __forceinline__ uint64_t* rs_flag(const RankView& v, int at, uint32_t cta, int src) {
  return reinterpret_cast<uint64_t*>(v.signal[at] + kStreamRsWord) + cta * kMaxRanks + src;
}

__device__ __forceinline__ uint64_t* ag_flag(const RankView& v, int at, uint32_t cta, int src) {
  return reinterpret_cast<uint64_t*>(v.signal[at] + kStreamAgWord) + cta * kMaxRanks + src;
}

// Named barrier of the data warps only (the producer never joins it).
__device__ __forceinline__ void data_bar() { asm volatile("bar.sync 1, %0;" ::"n"(kThreads) : "memory"); }

// Producer bookkeeping (lane 0 of the producer warp). Delivery counts are
// published per BATCH of kCreditBatch bulk items, one batch behind: when a
// batch closes, cp.async.bulk.wait_group kCreditBatch completes the batch
// before it (the newest batch stays in flight), so a publication never
// drains this CTA's NVLink pipe, and the system-scope release it needs is
// paid once per batch.
constexpr uint32_t kCreditBatch = 8;

template <int P>
struct Producer {
  uint64_t cur;       // items per destination (byte q) of the open batch
  uint64_t prev;      // items per destination of the closed batch still in flight
  uint32_t n_cur;     // items in the open batch
  uint32_t batch;     // items per batch at full speed (kCreditBatch unless tuned: 1, 2, 4, 8)
  uint32_t cur_batch; // size of the open batch: ramps 1, 2, 4, ... up to `batch` from each group's
                      // first item, so a group's first tiles are published after ~3 items, not 2 batches
  uint64_t epoch_hi;  // launch epoch << 32
  uint32_t* done;     // shared [kMaxRanks]: counts published so far (this launch)
};

// Publish `counts` (byte q: newly completed items into rank q's arena):
// async-proxy fence (the completed bulk copies before the generic release),
// then a system-scope release of the new total per destination.
template <int P>
__device__ __forceinline__ void publish(const RankView& v, Producer<P>& pr, uint64_t counts) {
  if (counts == 0) return;
  asm volatile("fence.proxy.async.global;" ::: "memory");
#pragma unroll
  for (int q = 0; q < P; ++q) {
    const uint32_t c = static_cast<uint32_t>(counts >> (8 * q)) & 0xffu;
    if (c != 0) {
      pr.done[q] += c;
      st_release_sys_u64(rs_flag(v, q, blockIdx.x, v.rank), pr.epoch_hi | pr.done[q]);
    }
  }
}

__device__ __forceinline__ uint64_t mask_counts(uint32_t mask) {
  uint64_t c = 0;
#pragma unroll
  for (int q = 0; q < kMaxRanks; ++q) c |= static_cast<uint64_t>((mask >> q) & 1u) << (8 * q);
  return c;
}

// One bulk item (destinations `mask`) was committed; a batch closes every
// pr.batch items (1, 2, 4 or 8: the wait_group operand is an immediate).
template <int P>
__device__ __forceinline__ void committed(const RankView& v, Producer<P>& pr, uint32_t mask) {
  pr.cur += mask_counts(mask);
  if (++pr.n_cur == pr.cur_batch) {
    switch (pr.cur_batch) {
      case 1: asm volatile("cp.async.bulk.wait_group 1;" ::: "memory"); break;
      case 2: asm volatile("cp.async.bulk.wait_group 2;" ::: "memory"); break;
      case 4: asm volatile("cp.async.bulk.wait_group 4;" ::: "memory"); break;
      default: asm volatile("cp.async.bulk.wait_group 8;" ::: "memory"); break;
    }
    publish<P>(v, pr, pr.prev);
    pr.prev = pr.cur;
    pr.cur = 0;
    pr.n_cur = 0;
    if (pr.cur_batch < pr.batch) pr.cur_batch *= 2;
  }
}

// Complete and publish everything committed (before the producer blocks on
// a group that is not ready yet, before a register-path item, at the end).
template <int P>
__device__ __forceinline__ void flush(const RankView& v, Producer<P>& pr) {
  if (pr.prev == 0 && pr.cur == 0) return;
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  publish<P>(v, pr, pr.prev + pr.cur);  // bytes <= 2 * kCreditBatch: no carries
  pr.prev = 0;
  pr.cur = 0;
  pr.n_cur = 0;
}

// This CTA's push items of one group (unit j of ncta): one-shot, every tile
// to every peer; two-shot, tile s*P+q of each super-tile s to its owner q.
template <int P>
__device__ __forceinline__ uint32_t stream_items(const Tile* tiles, uint32_t n_tiles, bool two_shot, uint32_t j,
                                                 uint32_t ncta) {
  if (!two_shot) return j < n_tiles ? (n_tiles - j + ncta - 1) / ncta : 0;
  const uint32_t n_super = (n_tiles + P - 1) / P;
  return (j < n_super ? (n_super - j + ncta - 1) / ncta : 0) * (P - 1);
}

template <int P>
__device__ __forceinline__ PushItem stream_item(const Tile* tiles, uint32_t n_tiles, bool two_shot, uint32_t j,
                                                uint32_t ncta, int me, uint32_t i) {
  if (!two_shot) return PushItem{tiles[j + i * ncta], ((1u << P) - 1u) & ~(1u << me)};
  const uint32_t s = j + (i / (P - 1)) * ncta;
  const int qi = static_cast<int>(i % (P - 1));
  const int q = qi < me ? qi : qi + 1;
  const uint32_t ti = s * P + q;
  return ti < n_tiles ? PushItem{tiles[ti], 1u << q} : PushItem{Tile{}, 0u};
}

// Producer warp: push one group's items in order. The whole warp runs the
// loop (uniform control flow); lane 0 drives the TMA: loads run up to two
// items ahead in the kStages ring (a stage is reused once the store that
// read it has finished reading: wait_group.read 1), each item is stored to
// every destination from its stage and committed as one bulk group; the
// < 16-byte tail goes through lane 0's registers. Tiles TMA cannot take
// (16-byte-unaligned layer views) go through the whole warp's registers,
// after a flush so the published counts stay in item order.
template <int P, typename T>
__device__ __forceinline__ void produce_group(const RankView& v, const Tile* tiles, uint32_t n_tiles,
                                              bool two_shot, uint32_t j, uint32_t ncta, uint64_t my_slot,
                                              Producer<P>& pr, CtaCtx& cx) {
  const uint32_t lane = threadIdx.x & 31;
  const int me = v.rank;
  const uint32_t n = stream_items<P>(tiles, n_tiles, two_shot, j, ncta);
  const uint32_t s0 = smem_u32(cx.stages);
  auto item = [&](uint32_t i) { return stream_item<P>(tiles, n_tiles, two_shot, j, ncta, me, i); };
  uint32_t iL = 0, iS = 0, nl = 0, ns = 0;  // next item to load / store; TMA loads / stores issued
  if (lane == 0 && pr.n_cur == 0) pr.cur_batch = 1;  // ramp the publication batch for this group
  for (;;) {
    // loads ahead, up to the first register-path item
    while (iL < n && (nl < kStages || nl + 2 <= ns + kStages)) {
      const PushItem it = item(iL);
      if (it.mask == 0) {
        ++iL;
        continue;
      }
      if (!tma_able<T>(it.t)) break;
      if (lane == 0) {
        if (nl >= kStages) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        const uint32_t k = (cx.ring.head + nl) % kStages;
        tma_load(s0 + k * kStageBytes, as<T>(v.grads[it.t.layer & kLayerMask]) + it.t.src,
                 tma_body<T>(it.t) * static_cast<uint32_t>(sizeof(T)), smem_u32(cx.bars + k));
      }
      ++nl;
      ++iL;
    }
    while (iS < n && item(iS).mask == 0) ++iS;
    if (iS >= n) break;
    const PushItem it = item(iS);
    const T* src = as<T>(v.grads[it.t.layer & kLayerMask]) + it.t.src;
    if (tma_able<T>(it.t)) {
      if (lane == 0) {
        const uint32_t k = (cx.ring.head + ns) % kStages;
        if (!mbar_wait(v, smem_u32(cx.bars + k), (cx.ring.phase >> k) & 1u)) *cx.s_abort = 1u;
        cx.ring.phase ^= 1u << k;
        const uint32_t bytes = tma_body<T>(it.t) * static_cast<uint32_t>(sizeof(T));
#pragma unroll
        for (int q = 0; q < P; ++q) {
          MGW_DCHECK((my_slot + it.t.moff) * sizeof(T) + bytes <= v.arena_bytes, "TMA push into a peer arena");
        if (it.mask & (1u << q)) tma_store(as<T>(v.arena[q]) + my_slot + it.t.moff, s0 + k * kStageBytes, bytes);
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        for (uint32_t e = tma_body<T>(it.t); e < it.t.len; e += 4) {  // tail (< one 16-byte vector)
          const float4 x = ld4_tail<T>(src + e, it.t.len - e);
#pragma unroll
          for (int q = 0; q < P; ++q) {
            MGW_DCHECK((my_slot + it.t.moff + e + 4) * sizeof(T) <= v.arena_bytes, "register push into a peer arena");
        if (it.mask & (1u << q)) st4<T>(as<T>(v.arena[q]) + my_slot + it.t.moff + e, x);
          }
        }
        committed<P>(v, pr, it.mask);
      }
      ++ns;
    } else {  // register path; every earlier item is stored (loads stop here)
      if (lane == 0) flush<P>(v, pr);
      __syncwarp();
      const uint32_t nvec = (it.t.len + 3) >> 2;
      for (uint32_t jv = lane; jv < nvec; jv += 32) {
        const uint32_t e = jv * 4;
        const float4 x = ld4_tail<T>(src + e, it.t.len - e);
#pragma unroll
        for (int q = 0; q < P; ++q) {
          MGW_DCHECK((my_slot + it.t.moff + e + 4) * sizeof(T) <= v.arena_bytes, "register push into a peer arena");
        if (it.mask & (1u << q)) st4<T>(as<T>(v.arena[q]) + my_slot + it.t.moff + e, x);
        }
      }
      __syncwarp();
      if (lane == 0) publish<P>(v, pr, mask_counts(it.mask));
      if (iL == iS) ++iL;
    }
    ++iS;
    __syncwarp();
    // a wait of this CTA gave up: stop pushing and publishing
    if (__shfl_sync(0xffffffffu, lane == 0 ? *reinterpret_cast<volatile uint32_t*>(cx.s_abort) : 0u, 0)) {
      if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      return;
    }
  }
  cx.ring.head = (cx.ring.head + nl) % kStages;
}

// Consumer bookkeeping (data threads). Delivery counts observed by the
// pollers (thread t < P watches peer t) are cached: a later tile whose count
// was already seen needs no poll and no barrier (the acquire that saw it and
// the data barrier after it already ordered the reads).

struct Consumer {
  uint32_t rs;        // tiles expected from every peer's producer so far (this launch)
  uint32_t rs_avail;  // min over the peers of the counts observed (identical in every data thread)
  uint32_t ag;        // thread t < P: reduced tiles expected from owner t so far
  uint32_t ag_out;    // reduced tiles published as an owner
  uint32_t round;     // poll rounds (parity selects the exchange buffer)
  uint32_t ag_batch;  // two-shot: owned super-tiles per all-gather publication
  uint64_t epoch_hi;
  uint32_t* s_cnt;    // shared [2][kMaxRanks]: counts seen by the pollers, per round parity
};

template <int P>
__device__ __forceinline__ void wait_flag(const RankView& v, const uint64_t* flag, uint64_t want, uint32_t* seen,
                                          CtaCtx& cx) {
  uint64_t val = 0;
  if (!spin_until(v, [&] {
        val = ld_acquire_sys_u64(flag);
        return val >= want;
      })) {
    *cx.s_abort = 1u;
  }
  *seen = static_cast<uint32_t>(val);
}

// All data threads: the first `cs.rs` tiles of every peer's producer have
// arrived (false: a wait gave up).
template <int P>
__device__ __forceinline__ bool arrived_rs(const RankView& v, Consumer& cs, CtaCtx& cx) {
  if (cs.rs_avail >= cs.rs) return true;
  const int t = static_cast<int>(threadIdx.x);
  const int me = v.rank;
  uint32_t* cnt = cs.s_cnt + (cs.round & 1u) * kMaxRanks;
  if (t < P && t != me && !cx.abort) wait_flag<P>(v, rs_flag(v, me, blockIdx.x, t), cs.epoch_hi | cs.rs, cnt + t, cx);
  data_bar();
  cx.abort = *reinterpret_cast<volatile uint32_t*>(cx.s_abort) != 0;
  uint32_t m = 0xffffffffu;
#pragma unroll
  for (int q = 0; q < P; ++q) {
    if (q != me) m = min(m, cnt[q]);
  }
  cs.rs_avail = m;
  ++cs.round;
  return !cx.abort;
}

// AP of owned super-tiles [s_lo, s_hi) (stride ncta): wait for the other
// owners' reduced tiles, then SGD from the local slots.
template <int P, typename T>
__device__ __forceinline__ bool apply_batch_supers(const RankView& v, const Tile* tiles, uint32_t n_tiles,
                                                   uint32_t s_lo, uint32_t n_s, uint32_t ncta, uint64_t slot_stride,
                                                   float lr, int epi, Consumer& cs, CtaCtx& cx) {
  const int me = v.rank;
  const int t = static_cast<int>(threadIdx.x);
  if (t < P && t != me) {
    uint32_t add = 0;  // owner t's tiles in this batch (none: t publishes nothing for it)
    for (uint32_t m = 0; m < n_s; ++m) add += (s_lo + m * ncta) * P + t < n_tiles ? 1u : 0u;
    cs.ag += add;
    uint32_t seen;
    if (add != 0 && !cx.abort) wait_flag<P>(v, ag_flag(v, me, blockIdx.x, t), cs.epoch_hi | cs.ag, &seen, cx);
  }
  data_bar();
  cx.abort = *reinterpret_cast<volatile uint32_t*>(cx.s_abort) != 0;
  if (cx.abort) return false;
#pragma unroll 1
  for (uint32_t m = 0; m < n_s; ++m) {
    const uint32_t s = s_lo + m * ncta;
#pragma unroll 1
    for (int q = 0; q < P; ++q) {
      const uint32_t ti = s * P + q;
      if (q == me || ti >= n_tiles) continue;
      const Tile tl = tiles[ti];
      const T* red = as<T>(v.arena[me]) + static_cast<uint64_t>(q) * slot_stride + tl.moff;
      const uint32_t layer = tl.layer & kLayerMask;
      const uint32_t nvec = (tl.len + 3) >> 2;
      float4 x[kVecPerThread], wv[kVecPerThread];
#pragma unroll
      for (uint32_t k = 0; k < kVecPerThread; ++k) {
        const uint32_t i = threadIdx.x + k * kThreads;
        if (i < nvec) x[k] = ld4_cg<T>(red + i * 4);
      }
      load_w_batch<kVecPerThread>(tl, threadIdx.x, kThreads, v.weights[layer], epi, wv);
      apply_batch<kVecPerThread, T>(tl, threadIdx.x, kThreads, x, wv, v.weights[layer], as<T>(v.grads[layer]),
                                    lr, epi);
    }
  }
  return true;
}

// Data warps: consume one group (unit j of ncta) as its tiles arrive.
//   one-shot: per tile, every peer's delivery, then the rank-order reduce + SGD.
//   two-shot: per batch of kAgBatch owned super-tiles, RA (reduce + SGD of
//   the owned tile, result pushed to every peer), one ag publication, then
//   AP of the previous batch (the other owners' results, SGD).
template <int P, typename T>
__device__ __forceinline__ void consume_group(const RankView& v, const Tile* tiles, uint32_t n_tiles,
                                              bool two_shot, uint32_t ll_pkt, uint32_t mbase, uint64_t slot_stride,
                                              float scale, float lr, int epi, uint32_t j, uint32_t ncta,
                                              Consumer& cs, CtaCtx& cx) {
  const int me = v.rank;
  const int t = static_cast<int>(threadIdx.x);
  const uint64_t my_slot = static_cast<uint64_t>(me) * slot_stride;
  if (ll_pkt != kNoLL) {
    ll_group<P, T>(v, tiles, n_tiles, ll_pkt, mbase, scale, lr, epi, j, ncta, cx.epoch);
    return;
  }
  if (!two_shot) {
#pragma unroll 1
    for (uint32_t ti = j; ti < n_tiles; ti += ncta) {
      ++cs.rs;
      if (!arrived_rs<P>(v, cs, cx)) return;
      reduce_tile_staged<P, T>(v, tiles[ti], slot_stride, false, my_slot, scale, lr, epi, cx.staging);
    }
    return;
  }
  const uint32_t n_super = (n_tiles + P - 1) / P;
  const uint32_t mine = j < n_super ? (n_super - j + ncta - 1) / ncta : 0;
  uint32_t prev_lo = 0, prev_n = 0;
  // all-gather publication batches ramp 1, 2, 4, ... up to ag_batch from the
  // group's first owned super-tile (the peers' first AP is not held back)
  uint32_t agb = 1;
#pragma unroll 1
  for (uint32_t b0 = 0; b0 < mine; b0 += agb, agb = agb * 2 < cs.ag_batch ? agb * 2 : cs.ag_batch) {
    const uint32_t nb = mine - b0 < agb ? mine - b0 : agb;
    uint32_t owned = 0;
#pragma unroll 1
    for (uint32_t m = b0; m < b0 + nb; ++m) {
      const uint32_t ti = (j + m * ncta) * P + me;
      if (ti >= n_tiles) continue;
      ++cs.rs;
      if (!arrived_rs<P>(v, cs, cx)) return;
      reduce_tile_staged<P, T>(v, tiles[ti], slot_stride, true, my_slot, scale, lr, epi, cx.staging);
      ++owned;
    }
    // AP of the previous batch BEFORE publishing this one: its local HBM
    // work overlaps the NVLink drain of this batch's result stores, which
    // the release below has to wait for
    if (prev_n != 0 && !apply_batch_supers<P, T>(v, tiles, n_tiles, j + prev_lo * ncta, prev_n, ncta, slot_stride,
                                                 lr, epi, cs, cx)) {
      return;
    }
    if (owned != 0) {
      data_bar();  // every data warp's result stores precede the release
      cs.ag_out += owned;
      if (t < P && t != me) st_release_sys_u64(ag_flag(v, t, blockIdx.x, me), cs.epoch_hi | cs.ag_out);
    }
    prev_lo = b0;
    prev_n = nb;
  }
  if (prev_n != 0) {
    apply_batch_supers<P, T>(v, tiles, n_tiles, j + prev_lo * ncta, prev_n, ncta, slot_stride, lr, epi, cs, cx);
  }
}

// Group-level parameters shared by both launch styles.
struct GroupArgs {
  const Tile* tiles;
  uint32_t n_tiles;
  uint64_t slot_stride;
  float scale;
  float lr;
  int epi;
  uint32_t chunk;
  uint32_t min_chunks;
  uint32_t ll_pkt;
  uint32_t mbase;
};

// One merge group, executed by CTA `cta` of `ncta`.
template <int P, typename T>
__device__ __forceinline__ void run_group(bool two_shot, const RankView& v, const GroupArgs& a, uint32_t cta,
                                          uint32_t ncta, CtaCtx& cx) {
  if constexpr (P > 1) {
    if (a.ll_pkt != kNoLL) {
      ll_group<P, T>(v, a.tiles, a.n_tiles, a.ll_pkt, a.mbase, a.scale, a.lr, a.epi, cta, ncta, cx.epoch);
      return;
    }
  }
  if constexpr (P == 1) {
    // Single rank: no exchange. grad x 1/P (= 1) straight into the epilogue;
    // all kB gradient and weight loads of a thread are in flight together.
    constexpr uint32_t kB = kTileElems / 4 / kBlock;
    for (uint32_t ti = cta; ti < a.n_tiles; ti += ncta) {
      const Tile t = a.tiles[ti];
      const uint32_t layer = t.layer & kLayerMask;
      T* g = as<T>(v.grads[layer]);
      const T* src = g + t.src;
      float* w = v.weights[layer];
      const bool aligned = !(t.layer & kGradUnaligned);
      const uint32_t nvec = (t.len + 3) >> 2;
      float4 x[kB], wv[kB];
#pragma unroll
      for (uint32_t k = 0; k < kB; ++k) {
        const uint32_t i = threadIdx.x + k * kBlock;
        const uint32_t e = i * 4;
        if (i < nvec) x[k] = (aligned && e + 4 <= t.len) ? ld4_stream<T>(src + e) : ld4_tail<T>(src + e, t.len - e);
      }
      load_w_batch<kB>(t, threadIdx.x, kBlock, w, a.epi, wv);
#pragma unroll
      for (uint32_t k = 0; k < kB; ++k) x[k] = round4<T>(mul4(x[k], a.scale));
      apply_batch<kB, T>(t, threadIdx.x, kBlock, x, wv, w, g, a.lr, a.epi);
    }
  } else if (two_shot) {
    two_shot_group<P, T>(v, a.tiles, a.n_tiles, a.slot_stride, a.scale, a.lr, a.epi, cta, ncta, a.chunk,
                         a.min_chunks, cx);
  } else {
    one_shot_group<P, T>(v, a.tiles, a.n_tiles, a.slot_stride, a.scale, a.lr, a.epi, cta, ncta, a.chunk,
                         a.min_chunks, cx);
  }
}

// Per-CTA set-up: barrier counter, launch epoch, TMA ring (P > 1), then the
// entry barrier: every peer has left every older launch of the communicator
// before this CTA index pushes into their arenas or LL slots.
template <int P>
__device__ __forceinline__ void cta_ctx_init(CtaCtx& cx, const RankView& v, uint8_t* dsmem, uint64_t* bars,
                                             uint32_t* s_abort) {
  __shared__ uint32_t s_init[2];
  cx.producer = threadIdx.x >= kThreads;
  cx.stages = dsmem;
  cx.staging = reinterpret_cast<float4*>(dsmem + static_cast<size_t>(kStages) * kStageBytes);
  cx.bars = bars;
  cx.ring.head = 0;
  cx.ring.phase = 0;
  cx.count = 0;
  cx.epoch = 0;
  cx.abort = false;
  cx.s_abort = s_abort;
  if (threadIdx.x == 0) *s_abort = 0u;
  if constexpr (P > 1) {
    if (threadIdx.x == kThreads) ring_init(bars);
    if (threadIdx.x == 0) {
      s_init[0] = ld_volatile_u32(v.state + kStateCtaBase + blockIdx.x);
      s_init[1] = ld_volatile_u32(v.state + kStateSeq);
    }
    __syncthreads();  // (also publishes the ring init)
    cx.count = s_init[0];
    cx.epoch = s_init[1] + 1u;
    cta_barrier(v, P, cx);
  } else {
    __syncthreads();
  }
}

// Per-CTA exit: persist the barrier counter; the last CTA of this rank's
// launch advances the launch sequence (the next launch's LL epoch). Every CTA
// read the sequence at entry, before any CTA can get here.
template <int P>
__device__ __forceinline__ void cta_exit(const RankView& v, const CtaCtx& cx) {
  if constexpr (P > 1) {
    if (threadIdx.x == 0) {
      v.state[kStateCtaBase + blockIdx.x] = cx.count;
      __threadfence();
      if (atomicAdd(v.state + kStateExit, 1u) == gridDim.x - 1) {
        v.state[kStateExit] = 0u;
        v.state[kStateSeq] = cx.epoch;
      }
    }
  }
}

template <int P, bool TWO_SHOT, bool LOOPBACK, typename T>
__global__ void __launch_bounds__(kBlock, 1) group_allreduce_kernel(const __grid_constant__ GroupLaunch L) {
  extern __shared__ __align__(1024) uint8_t dsmem[];
  __shared__ __align__(8) uint64_t bars[kStages];
  __shared__ uint32_t s_abort;
  __shared__ uint32_t s_stream[3 * kMaxRanks];  // producer counts, consumer poll exchange [2][ranks]
  const RankView& v = L.views[LOOPBACK ? blockIdx.y : 0];
  if (threadIdx.x < 3 * kMaxRanks) s_stream[threadIdx.x] = 0u;
  CtaCtx cx;
  cta_ctx_init<P>(cx, v, dsmem, bars, &s_abort);
  // a pipeline's tail group: stamps in the engine's layout (only CTAs that
  // fit the engine's row are stamped; min start / max end is the group span)
  const uint32_t stamp_col = (LOOPBACK ? blockIdx.y : 0u) * (L.stamp_row / (LOOPBACK ? gridDim.y : 1u)) + blockIdx.x;
  const bool stamped = L.stamps != nullptr && threadIdx.x == 0 && blockIdx.x < L.stamp_row / (LOOPBACK ? gridDim.y : 1u);
  if (stamped) L.stamps[(static_cast<size_t>(L.stamp_group) * L.stamp_row + stamp_col) * 2] = globaltimer_ns();
  if constexpr (P > 1) {
    if (L.stream) {
      const uint64_t epoch_hi = static_cast<uint64_t>(cx.epoch) << 32;
      if (cx.producer) {
        if (L.ll_pkt == kNoLL && !cx.abort) {
          Producer<P> pr{};
          pr.epoch_hi = epoch_hi;
          pr.done = s_stream;
          pr.batch = L.credit_batch;
          pr.cur_batch = 1;
          if ((threadIdx.x & 31) == 0) asm volatile("fence.proxy.async.global;" ::: "memory");
          produce_group<P, T>(v, L.tiles, L.n_tiles, TWO_SHOT, blockIdx.x, gridDim.x,
                              static_cast<uint64_t>(v.rank) * L.slot_stride, pr, cx);
          if ((threadIdx.x & 31) == 0 && *reinterpret_cast<volatile uint32_t*>(cx.s_abort) == 0) flush<P>(v, pr);
        }
      } else if (!cx.abort) {
        Consumer cs{0, 0, 0, 0, 0, L.ag_batch, epoch_hi, s_stream + kMaxRanks};
        consume_group<P, T>(v, L.tiles, L.n_tiles, TWO_SHOT, L.ll_pkt, L.mbase, L.slot_stride, L.scale, L.lr,
                            L.epilogue, blockIdx.x, gridDim.x, cs, cx);
      }
      __syncthreads();
      if (stamped) L.stamps[(static_cast<size_t>(L.stamp_group) * L.stamp_row + stamp_col) * 2 + 1] = globaltimer_ns();
      cta_exit<P>(v, cx);
      return;
    }
  }
  const GroupArgs a{L.tiles, L.n_tiles, L.slot_stride, L.scale, L.lr, L.epilogue,
                    L.chunk, L.min_chunks, L.ll_pkt, L.mbase};
  run_group<P, T>(TWO_SHOT, v, a, blockIdx.x, gridDim.x, cx);
  if (L.stamps != nullptr) {
    __syncthreads();
    if (stamped) L.stamps[(static_cast<size_t>(L.stamp_group) * L.stamp_row + stamp_col) * 2 + 1] = globaltimer_ns();
  }
  cta_exit<P>(v, cx);
}

// Group descriptors are read-only for the engine's lifetime: every CTA walks
// the whole table (skipping the groups it has no unit in), so the loads go
// through the non-coherent L1 path and the table is prefetched into L1 at
// launch — a skipped group costs an L1 hit, not an L2 round trip (many-group
// plans: DenseNet-201 has 604 groups).
__device__ __forceinline__ EngineGroup ld_group(const EngineGroup* g) {
  static_assert(sizeof(EngineGroup) == 32, "two 16-byte loads");
  const uint4 a = __ldg(reinterpret_cast<const uint4*>(g));
  const uint4 b = __ldg(reinterpret_cast<const uint4*>(g) + 1);
  EngineGroup r;
  r.tile_first = a.x;
  r.n_tiles = a.y;
  r.two_shot = a.z;
  r.ll_pkt = a.w;
  r.mbase = b.x;
  r.cta0 = b.y;
  r.units = b.z;
  r.pad = b.w;
  return r;
}

// CTA b walks only its own schedule (host-built: the groups it has a unit
// in, FIFO order); j = its unit index inside the group (groups rotate over
// the CTAs from cta0).
__device__ __forceinline__ uint32_t unit_of(const EngineGroup& g) {
  const uint32_t b = blockIdx.x;
  return b >= g.cta0 ? b - g.cta0 : b + gridDim.x - g.cta0;
}

__device__ __forceinline__ bool is_ll_oneshot(const EngineGroup& g) { return !g.two_shot && g.ll_pkt != kNoLL; }

// Off the critical path of a group: while thread 0 waits for the group's
// ready flag, warp 1 warms what the first tile of this CTA needs — its
// descriptor and the layer's pointer-table entries into L1 (read-only for
// the kernel's life), the weight lines into L2 — so once the flag flips only
// the gradient load (written by the backward, so read after the flag) is a
// memory round trip.
template <int P>
__device__ __forceinline__ void warm_group(const RankView& v, const Tile* tiles, const EngineGroup& grp, uint32_t j,
                                           float lr_nonzero) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t ti;
  if (P > 1 && grp.two_shot) {
    ti = j * P + static_cast<uint32_t>(v.rank);
  } else if (P > 1 && grp.ll_pkt != kNoLL) {
    ti = j / kLLParts;
  } else {
    ti = j;
  }
  if (ti >= grp.n_tiles) return;
  const Tile t = tiles[grp.tile_first + ti];
  const uint32_t layer = t.layer & kLayerMask;
  asm volatile("prefetch.global.L1 [%0];" ::"l"(v.grads + layer));
  const float* w = v.weights[layer];
  if (w == nullptr || lr_nonzero == 0.0f) return;
  const char* wb = reinterpret_cast<const char*>(w + t.src);
  const uint32_t bytes = t.len * 4u;
  for (uint32_t off = lane * 128u; off < bytes; off += 32u * 128u) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(wb + off));
  }
}

// ---- P = 1: TMA-fed gradient -> SGD pipeline ---------------------------------
// The single-rank engine (no exchange: W -= lr * round(g * 1/P)) is HBM-bound;
// its loads are decoupled from the math: the producer warp streams each
// tile's gradient and weight bodies into a kP1Stages ring of shared-memory
// stages with TMA bulk copies (one mbarrier complete_tx per stage) while the
// data warps apply SGD from shared memory and store the weights — the
// tile-descriptor -> pointer -> data dependency chain and the HBM latency
// leave the critical path. Tiles TMA cannot take (unaligned views, no
// weights) go through the data warps' registers.
constexpr uint32_t kP1Stages = 3;
constexpr uint32_t kP1StageBytes = 2 * kStageBytes;  // gradient body (<= 32 KiB) + weight body (32 KiB)
constexpr size_t kSmemP1 = static_cast<size_t>(kP1Stages) * kP1StageBytes;

template <typename T>
__device__ __forceinline__ bool p1_tma_able(const Tile& t, const float* w, int epi) {
  return !(t.layer & (kGradUnaligned | kWeightUnaligned)) && w != nullptr && (epi & MGW_SGD) &&
         t.len >= Elem<T>::kVec;
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  asm volatile(
      "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
      : "=r"(done)
      : "r"(bar), "r"(parity)
      : "memory");
  return done != 0;
}

template <typename T>
__device__ __noinline__ void engine_p1(const EngineLaunch& E, const RankView& v, uint8_t* dsmem, uint64_t* full,
                                       uint64_t* empty, uint32_t* s_abort, uint32_t iter, uint32_t slot, size_t row) {
  const uint32_t ncta = gridDim.x;
  const uint32_t target = iter + 1;
  const bool producer = threadIdx.x >= kThreads;
  const uint32_t s0 = smem_u32(dsmem);
  if (producer) {
    if ((threadIdx.x & 31) != 0) return;
    uint32_t n = 0, pe = 0;
    const uint32_t e_end = E.sched_off[blockIdx.x + 1];
    for (uint32_t e = E.sched_off[blockIdx.x]; e < e_end; ++e) {
      const uint32_t gi = E.sched[e];
      if (gi < E.g_lo) break;  // FIFO order: the caller's tail groups come last
      const EngineGroup grp = ld_group(E.groups + gi);
      const uint32_t j = unit_of(grp);
      if (!E.no_wait) {
        const uint32_t* flag = E.ready + gi;
        if (!spin_until(v, [&] { return static_cast<int32_t>(ld_acquire_gpu(flag) - target) >= 0; })) {
          atomicExch(E.pipe + 3, 1u);
          *s_abort = 1u;
        }
      }
      if (*reinterpret_cast<volatile uint32_t*>(s_abort)) return;
      // gradients written by generic-proxy stores and published by the ready
      // flag just acquired: visible to the TMA (a drain — every group ready at
      // launch — has them ordered by the kernel boundary)
      if (!E.no_wait) asm volatile("fence.proxy.async.global;" ::: "memory");
      const Tile* tiles = E.tiles + grp.tile_first;
      for (uint32_t ti = j; ti < grp.n_tiles; ti += ncta) {
        const Tile t = tiles[ti];
        const uint32_t layer = t.layer & kLayerMask;
        const float* w = v.weights[layer];
        if (!p1_tma_able<T>(t, w, E.epilogue)) continue;
        const uint32_t st = n % kP1Stages;
        if (n >= kP1Stages) {
          if (!spin_until(v, [&] { return mbar_try(smem_u32(empty + st), (pe >> st) & 1u); })) {
            *s_abort = 1u;
            return;
          }
          pe ^= 1u << st;
        }
        const uint32_t body = tma_body<T>(t);
        const uint32_t gb = body * static_cast<uint32_t>(sizeof(T)), wb = body * 4u;
        const uint32_t bar = smem_u32(full + st);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(gb + wb) : "memory");
        const uint32_t dst = s0 + st * kP1StageBytes;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
            "l"(as<T>(v.grads[layer]) + t.src), "r"(gb), "r"(bar)
            : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                dst + kStageBytes),
            "l"(w + t.src), "r"(wb), "r"(bar)
            : "memory");
        ++n;
      }
    }
    return;
  }
  uint32_t m = 0, pf = 0;
  const int tid = static_cast<int>(threadIdx.x);
  const uint32_t e_end = E.sched_off[blockIdx.x + 1];
  for (uint32_t e = E.sched_off[blockIdx.x]; e < e_end; ++e) {
    const uint32_t gi = E.sched[e];
    if (gi < E.g_lo) break;  // FIFO order: the caller's tail groups come last
    const EngineGroup grp = ld_group(E.groups + gi);
    const uint32_t j = unit_of(grp);
    if (tid == 0) {
      if (!E.no_wait && !*reinterpret_cast<volatile uint32_t*>(s_abort)) {
        const uint32_t* flag = E.ready + gi;
        if (!spin_until(v, [&] { return static_cast<int32_t>(ld_acquire_gpu(flag) - target) >= 0; })) {
          atomicExch(E.pipe + 3, 1u);
          *s_abort = 1u;
        }
      }
      if (E.stamps != nullptr) E.stamps[(gi * row + slot) * 2] = globaltimer_ns();
    }
    data_bar();
    if (*reinterpret_cast<volatile uint32_t*>(s_abort)) return;
    const Tile* tiles = E.tiles + grp.tile_first;
    for (uint32_t ti = j; ti < grp.n_tiles; ti += ncta) {
      const Tile t = tiles[ti];
      const uint32_t layer = t.layer & kLayerMask;
      float* w = v.weights[layer];
      T* g = as<T>(v.grads[layer]);
      if (p1_tma_able<T>(t, w, E.epilogue)) {
        const uint32_t st = m % kP1Stages;
        const uint32_t bar = smem_u32(full + st);
        if (!spin_until(v, [&] { return mbar_try(bar, (pf >> st) & 1u); })) *s_abort = 1u;
        pf ^= 1u << st;
        const uint8_t* sg = dsmem + st * kP1StageBytes;
        const float4* sw = reinterpret_cast<const float4*>(sg + kStageBytes);
        const uint32_t body = tma_body<T>(t);
        for (uint32_t i = tid; i < body / 4; i += kThreads) {
          float4 x;
          if constexpr (sizeof(T) == 4) {
            x = reinterpret_cast<const float4*>(sg)[i];
          } else {
            const uint2 u = reinterpret_cast<const uint2*>(sg)[i];
            x = unpack_bf16x4(u.x, u.y);
          }
          x = round4<T>(mul4(x, E.scale));
          float4 wv = sw[i];
          wv.x = sgd1(wv.x, x.x, E.lr);
          wv.y = sgd1(wv.y, x.y, E.lr);
          wv.z = sgd1(wv.z, x.z, E.lr);
          wv.w = sgd1(wv.w, x.w, E.lr);
          st_v4(w + t.src + i * 4, wv);
          if (E.epilogue & MGW_WRITE_GRAD) st4<T>(g + t.src + i * 4, x);
        }
        if (tid == 0) {  // the < one-vector tail from global memory
          for (uint32_t e = body; e < t.len; e += 4) {
            const float4 x = round4<T>(mul4(ld4_tail<T>(g + t.src + e, t.len - e), E.scale));
            epilogue<T>(t, e, x, w, g, E.lr, E.epilogue);
          }
        }
        data_bar();  // every data thread has read the stage
        if (tid == 0) mbar_arrive(smem_u32(empty + st));
        ++m;
      } else {
        const bool aligned = !(t.layer & kGradUnaligned);
        const uint32_t nvec = (t.len + 3) >> 2;
        for (uint32_t i = tid; i < nvec; i += kThreads) {
          const uint32_t e = i * 4;
          float4 x[1], wv[1];
          x[0] = (aligned && e + 4 <= t.len) ? ld4_stream<T>(g + t.src + e) : ld4_tail<T>(g + t.src + e, t.len - e);
          load_w_batch<1>(t, i, kThreads, w, E.epilogue, wv);
          x[0] = round4<T>(mul4(x[0], E.scale));
          apply_batch<1, T>(t, i, kThreads, x, wv, w, g, E.lr, E.epilogue);
        }
      }
    }
    if (E.stamps != nullptr) {
      data_bar();
      if (tid == 0) E.stamps[(gi * row + slot) * 2 + 1] = globaltimer_ns();
    }
  }
}

// The engine's streamed body (P > 1): the producer warp walks the groups
// pushing tiles (waiting for each group's ready flag, after publishing what
// it has in flight), the data warps walk the same groups consuming them.
template <int P, typename T>
__device__ __forceinline__ void engine_stream(const EngineLaunch& E, const RankView& v, CtaCtx& cx, uint32_t iter,
                                              uint32_t slot, size_t row, uint32_t* s_stream) {
  const uint32_t ncta = gridDim.x;
  const uint64_t epoch_hi = static_cast<uint64_t>(cx.epoch) << 32;
  const uint32_t target = iter + 1;
  if (cx.producer) {
    const uint32_t lane = threadIdx.x & 31;
    Producer<P> pr{};
    pr.epoch_hi = epoch_hi;
    pr.done = s_stream;
    pr.batch = E.credit_batch;
    pr.cur_batch = 1;
    const uint64_t my_slot = static_cast<uint64_t>(v.rank) * E.slot_stride;
    const uint32_t e_end = E.sched_off[blockIdx.x + 1];
    for (uint32_t e = E.sched_off[blockIdx.x]; e < e_end; ++e) {
      const uint32_t gi = E.sched[e];
      if (gi < E.g_lo) break;  // FIFO order: the caller's tail groups come last
      const EngineGroup grp = ld_group(E.groups + gi);
      if (is_ll_oneshot(grp)) continue;  // LL groups: the data warps alone
      const uint32_t j = unit_of(grp);
      uint32_t abort = 0;
      if (lane == 0) {
        abort = *reinterpret_cast<volatile uint32_t*>(cx.s_abort);
        const uint32_t* flag = E.ready + gi;
        if (!abort && !E.no_wait && static_cast<int32_t>(ld_acquire_gpu(flag) - target) < 0) {
          flush<P>(v, pr);  // publish what is in flight before blocking
          if (!spin_until(v, [&] { return static_cast<int32_t>(ld_acquire_gpu(flag) - target) >= 0; })) {
            atomicExch(E.pipe + 3, 1u);
            *cx.s_abort = 1u;
            abort = 1;
          }
        }
        // gradients written by generic-proxy stores: visible to the TMA
        // (drain: ordered by the kernel boundary)
        if (!E.no_wait) asm volatile("fence.proxy.async.global;" ::: "memory");
      }
      if (__shfl_sync(0xffffffffu, abort, 0)) break;
      produce_group<P, T>(v, E.tiles + grp.tile_first, grp.n_tiles, grp.two_shot != 0, j, ncta, my_slot, pr, cx);
    }
    if (lane == 0 && *reinterpret_cast<volatile uint32_t*>(cx.s_abort) == 0) flush<P>(v, pr);
    __syncwarp();
    return;
  }
  Consumer cs{0, 0, 0, 0, 0, E.ag_batch, epoch_hi, s_stream + kMaxRanks};
  const uint32_t e_end = E.sched_off[blockIdx.x + 1];
  for (uint32_t e = E.sched_off[blockIdx.x]; e < e_end; ++e) {
    const uint32_t gi = E.sched[e];
    if (gi < E.g_lo) break;  // FIFO order: the caller's tail groups come last
    const EngineGroup grp = ld_group(E.groups + gi);
    const uint32_t j = unit_of(grp);
    if (threadIdx.x >= 32 && threadIdx.x < 64) warm_group<P>(v, E.tiles, grp, j, E.lr);
    if (threadIdx.x == 0) {
      if (!E.no_wait && !cx.abort) {
        const uint32_t* flag = E.ready + gi;
        if (!spin_until(v, [&] { return static_cast<int32_t>(ld_acquire_gpu(flag) - target) >= 0; })) {
          atomicExch(E.pipe + 3, 1u);
          *cx.s_abort = 1u;
        }
      }
      if (E.stamps != nullptr) E.stamps[(gi * row + slot) * 2] = globaltimer_ns();
    }
    data_bar();
    cx.abort = *reinterpret_cast<volatile uint32_t*>(cx.s_abort) != 0;
    if (cx.abort) break;
    consume_group<P, T>(v, E.tiles + grp.tile_first, grp.n_tiles, grp.two_shot != 0,
                        grp.two_shot ? kNoLL : grp.ll_pkt, grp.mbase, E.slot_stride, E.scale, E.lr, E.epilogue, j,
                        ncta, cs, cx);
    if (E.stamps != nullptr) {
      data_bar();
      if (threadIdx.x == 0) E.stamps[(gi * row + slot) * 2 + 1] = globaltimer_ns();
    }
  }
}

// The persistent comm engine. Grid (ncta, 1) for a real rank, (ncta, P) in
// loopback (blockIdx.y = emulated rank). Groups run FIFO in backward order;
// group k's units go to CTAs cta0_k, cta0_k + 1, ... (mod ncta), where cta0
// rotates by the CTAs the previous groups used — so a run of small groups
// spreads over the SMs and their latencies overlap instead of queueing on
// CTA 0. The mapping is a pure function of the plan: CTA index b does the
// same groups, tiles and barriers on every rank.
// STREAM: the streamed protocol (a separate kernel, so each protocol gets
// the whole register budget).
template <int P, typename T, bool STREAM>
__global__ void __launch_bounds__(kBlock, 1) engine_kernel(const __grid_constant__ EngineLaunch E) {
  extern __shared__ __align__(1024) uint8_t dsmem[];
  __shared__ __align__(8) uint64_t bars[kStages];
  __shared__ uint32_t s_iter;
  __shared__ uint32_t s_abort;
  __shared__ uint32_t s_stream[3 * kMaxRanks];  // producer counts, consumer poll exchange [2][ranks]
  if (threadIdx.x < 3 * kMaxRanks) s_stream[threadIdx.x] = 0u;
  const RankView& v = E.views[blockIdx.y];
  if (threadIdx.x == 0) s_iter = ld_volatile_u32(E.pipe + 1);
  // Entry barrier inside (runs while the compute stream replays the forward
  // pass): every peer has finished every older launch before any push.
  CtaCtx cx;
  cta_ctx_init<P>(cx, v, dsmem, bars, &s_abort);
  const uint32_t iter = s_iter;
  // past the entry barrier: a gated replay (calibration) may start its clock
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) st_release_gpu(E.pipe, iter + 1);
  const uint32_t ncta = gridDim.x;
  const uint32_t slot = blockIdx.y * gridDim.x + blockIdx.x;      // stamp column
  const size_t row = static_cast<size_t>(gridDim.x) * gridDim.y;  // stamp row width
  if constexpr (P > 1 && STREAM) {
    engine_stream<P, T>(E, v, cx, iter, slot, row, s_stream);
    __syncthreads();
  }
  if constexpr (P == 1 && STREAM) {
    __shared__ __align__(8) uint64_t p1_empty[kP1Stages];
    if (threadIdx.x == kThreads) {
      for (uint32_t k = 0; k < kP1Stages; ++k) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bars + k)) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(p1_empty + k)) : "memory");
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    engine_p1<T>(E, v, dsmem, bars, p1_empty, &s_abort, iter, slot, row);
    __syncthreads();
  }
  // this CTA's groups in backward order: FIFO like timeline.hpp:133-154
  // (the schedule is identical on every rank: no barrier to skip)
  const uint32_t e_end = STREAM ? 0u : E.sched_off[blockIdx.x + 1];
  for (uint32_t e = STREAM ? 0u : E.sched_off[blockIdx.x]; e < e_end; ++e) {
    const uint32_t gi = E.sched[e];
    if (gi < E.g_lo) break;
    const EngineGroup grp = ld_group(E.groups + gi);
    const uint32_t j = unit_of(grp);  // this CTA's index inside the group
    if (threadIdx.x >= 32 && threadIdx.x < 64) warm_group<P>(v, E.tiles, grp, j, E.lr);
    if (threadIdx.x == 0) {
      // group gi is ready for iteration `iter` once its flag reached iter+1
      // (set by the replay, or by a mark kernel after the real backward of
      // the group's layers — groups may complete out of FIFO order)
      if (!E.no_wait && !cx.abort) {
        const uint32_t target = iter + 1;
        const uint32_t* flag = E.ready + gi;
        if (!spin_until(v, [&] { return static_cast<int32_t>(ld_acquire_gpu(flag) - target) >= 0; })) {
          atomicExch(E.pipe + 3, 1u);  // compute side never signalled
          s_abort = 1u;
        }
      }
      if (E.stamps != nullptr) E.stamps[(gi * row + slot) * 2] = globaltimer_ns();
    }
    __syncthreads();
    cx.abort = *reinterpret_cast<volatile uint32_t*>(&s_abort) != 0;
    if (!cx.abort) {
      const GroupArgs a{E.tiles + grp.tile_first, grp.n_tiles, E.slot_stride, E.scale, E.lr, E.epilogue,
                        E.chunk, E.min_chunks, grp.two_shot ? kNoLL : grp.ll_pkt, grp.mbase};
      run_group<P, T>(P > 1 && grp.two_shot != 0, v, a, j, ncta, cx);
    }
    if (E.stamps != nullptr) {
      __syncthreads();
      if (threadIdx.x == 0) E.stamps[(gi * row + slot) * 2 + 1] = globaltimer_ns();
    }
  }
  cta_exit<P>(v, cx);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(E.pipe + 2, 1u) == gridDim.x * gridDim.y - 1) {
      atomicExch(E.pipe + 2, 0u);
      __threadfence();
      atomicExch(E.pipe + 1, iter + 1);
    }
  }
}

// ---- NVLS (NVLink SHARP) two-shot ---------------------------------------------
// The NVSwitch does the reduction: each rank packs its scaled gradients into
// its own NVLS buffer (local HBM; the buffers of all ranks are bound to one
// multicast object), then the owner of each vector loads it through the
// multicast address with multimem.ld_reduce (the switch returns the sum of
// the P copies) and stores the sum back with multimem.st (the switch writes
// it into all P copies); every rank then unpacks + applies SGD from its local
// copy. NVLink bytes per rank: S in and S out, against 2(P-1)/P*S each way
// for the push two-shot — the win grows with P.
// Numerics (measured on B200, tools/nvls_probe.cu): the switch returns the
// EXACT sum of the P fp32 inputs rounded once to fp32 (round to nearest
// even) — at P = 2 that is the rank-order sum bit for bit; at P >= 4 it is
// deterministic, identical on every rank and pinned by the oracle's
// exact-sum variant (mgw_oracle_nvls), but not the rank-order fold.
//
// Pipeline per CTA (its tiles j = b, b + ncta, ..., in chunks of `chunk`
// tiles), step s: the HBM warps pack chunk s and unpack + SGD chunk s - 2,
// the switch warps reduce chunk s - 1; ONE cross-rank barrier per step
// certifies both "chunk s packed everywhere" and "chunk s - 1's sums landed
// everywhere". No entry barrier: every byte a launch reads remotely was
// certified by a barrier of the launch that wrote it, and the previous
// launch's last remote access precedes its last barrier.
// 256-thread CTAs, several per SM: a CTA waiting on its step barrier leaves
// the SM to the others (the per-step latency chain — ld_reduce round trip,
// the multicast stores' fence, the barrier round trip — is ~3 NVLink round
// trips, and one CTA per SM would serialise them).
constexpr uint32_t kNvlsBlock = 256;
constexpr uint32_t kNvlsWarps = 4;                    // switch warps (the other 4: HBM warps)
constexpr uint32_t kNvlsThreads = kNvlsWarps * 32;    // per role
constexpr uint32_t kNvlsMaxChunk = 16;                // tiles per chunk (<= 32: one lane per tile)
constexpr uint32_t kNvlsU = 4;                        // vectors in flight per thread and batch

__device__ __forceinline__ float4 mc_ld_reduce(const float* mc) {
  float4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(mc)
               : "memory");
  return v;
}

__device__ __forceinline__ void mc_st(float* mc, float4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}

// One chunk's tiles as a flat vector index space: entry k covers vectors
// [pre[k], pre[k+1]) (pre[0] = 0); built by one warp, lane k = tile k.
struct NvlsChunk {
  uint32_t pre[kNvlsMaxChunk + 1];
  uint32_t base[kNvlsMaxChunk];   // first vector: merge-layout vector index (reduce) / 0 (pack, unpack)
  Tile t[kNvlsMaxChunk];
  float* w[kNvlsMaxChunk];        // layer weights (unpack)
  float* g[kNvlsMaxChunk];        // layer gradients
};

__device__ __forceinline__ uint32_t nvls_find(const NvlsChunk& c, uint32_t nt, uint32_t idx) {
  uint32_t k = 0;
  while (k + 1 < nt && idx >= c.pre[k + 1]) ++k;
  return k;
}

// Lane k < nt of the calling warp describes tile k of chunk `m0` (CTA b's
// tiles m0 .. m0+nt-1, stride ncta); part = true: only this rank's 1/P of
// every tile's vectors (the switch reduce).
template <int P>
__device__ __forceinline__ void nvls_describe(NvlsChunk& c, const GroupLaunch& L, const RankView& v, uint32_t m0,
                                              uint32_t nt, bool part) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t n = 0;
  if (lane < nt) {
    const Tile t = L.tiles[blockIdx.x + (m0 + lane) * gridDim.x];
    const uint32_t nv = (t.len + 3) >> 2;
    const uint32_t l = t.layer & kLayerMask;
    c.t[lane] = t;
    if (part) {
      const uint32_t lo = nv * static_cast<uint32_t>(v.rank) / P;
      const uint32_t hi = nv * static_cast<uint32_t>(v.rank + 1) / P;
      c.base[lane] = t.moff / 4 + lo;
      n = hi - lo;
    } else {
      c.base[lane] = 0;
      c.w[lane] = v.weights[l];
      c.g[lane] = v.grads[l];
      n = nv;
    }
  }
  // inclusive scan of n over the warp
  uint32_t x = n;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (static_cast<int>(lane) >= d) x += y;
  }
  if (lane < nt) c.pre[lane + 1] = x;
  if (lane == 0) c.pre[0] = 0;
}

// Switch warps: this rank's part of every tile of the chunk through the
// multicast address (ld_reduce -> st), kNvlsU vectors in flight per thread.
__device__ __forceinline__ void nvls_reduce(float* mc, const NvlsChunk& c, uint32_t nt, uint32_t tid,
                                            uint64_t cap) {
  const uint32_t total = c.pre[nt];
  for (uint32_t i0 = tid; i0 < total; i0 += kNvlsU * kNvlsThreads) {
    float4 x[kNvlsU];
    size_t at[kNvlsU];
#pragma unroll
    for (uint32_t u = 0; u < kNvlsU; ++u) {
      const uint32_t i = i0 + u * kNvlsThreads;
      if (i < total) {
        const uint32_t k = nvls_find(c, nt, i);
        at[u] = static_cast<size_t>(c.base[k] + (i - c.pre[k])) * 4;
        MGW_DCHECK(at[u] + 4 <= cap, "NVLS multicast reduce / store");
        x[u] = mc_ld_reduce(mc + at[u]);
      }
    }
#pragma unroll
    for (uint32_t u = 0; u < kNvlsU; ++u) {
      if (i0 + u * kNvlsThreads < total) mc_st(mc + at[u], x[u]);
    }
  }
}

// HBM warps: pack (x 1/P into this rank's copy), 2 kNvlsU vectors in flight.
__device__ __forceinline__ void nvls_pack(float* uc, const NvlsChunk& c, uint32_t nt, float scale, uint32_t tid,
                                          uint64_t cap) {
  constexpr uint32_t U = 2 * kNvlsU;
  const uint32_t total = c.pre[nt];
  for (uint32_t i0 = tid; i0 < total; i0 += U * kNvlsThreads) {
    float4 x[U];
    float* dst[U];
#pragma unroll
    for (uint32_t u = 0; u < U; ++u) {
      const uint32_t i = i0 + u * kNvlsThreads;
      if (i < total) {
        const uint32_t k = nvls_find(c, nt, i);
        const Tile& t = c.t[k];
        const uint32_t e = (i - c.pre[k]) * 4;
        const float* src = c.g[k] + t.src + e;
        x[u] = (!(t.layer & kGradUnaligned) && e + 4 <= t.len) ? ld_stream_v4(src) : load_tail(src, t.len - e);
        dst[u] = uc + t.moff + e;
        MGW_DCHECK(static_cast<uint64_t>(t.moff) + e + 4 <= cap, "NVLS pack into the local copy");
      }
    }
#pragma unroll
    for (uint32_t u = 0; u < U; ++u) {
      if (i0 + u * kNvlsThreads < total) st_v4(dst[u], mul4(x[u], scale));
    }
  }
}

// HBM warps: unpack + SGD from this rank's copy of the sums.
__device__ __forceinline__ void nvls_unpack(const float* uc, const NvlsChunk& c, uint32_t nt, float lr, int epi,
                                            uint32_t tid) {
  const uint32_t total = c.pre[nt];
  for (uint32_t i0 = tid; i0 < total; i0 += kNvlsU * kNvlsThreads) {
    float4 sv[kNvlsU], wv[kNvlsU];
    uint32_t kk[kNvlsU], ee[kNvlsU];
    bool fast[kNvlsU];
#pragma unroll
    for (uint32_t u = 0; u < kNvlsU; ++u) {
      const uint32_t i = i0 + u * kNvlsThreads;
      fast[u] = false;
      if (i < total) {
        const uint32_t k = nvls_find(c, nt, i);
        const Tile& t = c.t[k];
        const uint32_t e = (i - c.pre[k]) * 4;
        kk[u] = k;
        ee[u] = e;
        sv[u] = ld_cg_v4(uc + t.moff + e);
        fast[u] = (epi & MGW_SGD) && c.w[k] != nullptr && e + 4 <= t.len && !(t.layer & kWeightUnaligned);
        if (fast[u]) wv[u] = ld_v4(c.w[k] + t.src + e);
      }
    }
#pragma unroll
    for (uint32_t u = 0; u < kNvlsU; ++u) {
      if (i0 + u * kNvlsThreads >= total) continue;
      const Tile& t = c.t[kk[u]];
      if (fast[u]) {
        float4 w = wv[u];
        w.x = sgd1(w.x, sv[u].x, lr);
        w.y = sgd1(w.y, sv[u].y, lr);
        w.z = sgd1(w.z, sv[u].z, lr);
        w.w = sgd1(w.w, sv[u].w, lr);
        st_v4(c.w[kk[u]] + t.src + ee[u], w);
        if (epi & MGW_WRITE_GRAD) epilogue<float>(t, ee[u], sv[u], nullptr, c.g[kk[u]], lr, MGW_WRITE_GRAD);
      } else {
        epilogue<float>(t, ee[u], sv[u], c.w[kk[u]], c.g[kk[u]], lr, epi);
      }
    }
  }
}

template <int P>
__global__ void __launch_bounds__(kNvlsBlock, 2) nvls_group_kernel(const __grid_constant__ GroupLaunch L) {
  __shared__ uint32_t s_abort;
  __shared__ uint32_t s_init[2];
  __shared__ NvlsChunk s_red, s_pack, s_unpack;
  const RankView& v = L.views[0];
  CtaCtx cx{};
  cx.s_abort = &s_abort;
  cx.producer = false;
  if (threadIdx.x == 0) {
    s_abort = 0u;
    s_init[0] = ld_volatile_u32(v.state + kStateCtaBase + blockIdx.x);
    s_init[1] = ld_volatile_u32(v.state + kStateSeq);
  }
  __syncthreads();
  cx.count = s_init[0];
  cx.epoch = s_init[1] + 1u;
  // a pipeline's tail group: stamps in the engine's layout (as group_allreduce_kernel)
  const bool stamped = L.stamps != nullptr && threadIdx.x == 0 && blockIdx.x < L.stamp_row;
  const size_t stamp_at = (static_cast<size_t>(L.stamp_group) * L.stamp_row + blockIdx.x) * 2;
  if (stamped) L.stamps[stamp_at] = globaltimer_ns();
  const uint32_t ncta = gridDim.x;
  const uint32_t b = blockIdx.x;
  const uint32_t mine = L.n_tiles > b ? (L.n_tiles - b + ncta - 1) / ncta : 0u;  // tiles j = b + m * ncta
  const uint32_t chunk = L.chunk < 1 ? 1u : (L.chunk > kNvlsMaxChunk ? kNvlsMaxChunk : L.chunk);
  const uint32_t nchunks = (mine + chunk - 1) / chunk;
  const uint32_t warp = threadIdx.x >> 5;
  const bool hbm = threadIdx.x >= kNvlsThreads;
  const uint32_t tid = hbm ? threadIdx.x - kNvlsThreads : threadIdx.x;
  auto nt_of = [&](uint32_t c) { return min(chunk, mine - c * chunk); };
  // step s: pack chunk s | reduce chunk s - 1 | unpack chunk s - 2; one barrier
  for (uint32_t s = 0; s < nchunks + 2; ++s) {
    const bool do_pack = s < nchunks, do_red = s >= 1 && s - 1 < nchunks, do_unpack = s >= 2;
    if (warp == 0 && do_red) nvls_describe<P>(s_red, L, v, (s - 1) * chunk, nt_of(s - 1), true);
    if (warp == kNvlsWarps && do_pack) nvls_describe<P>(s_pack, L, v, s * chunk, nt_of(s), false);
    if (warp == kNvlsWarps + 1 && do_unpack) nvls_describe<P>(s_unpack, L, v, (s - 2) * chunk, nt_of(s - 2), false);
    __syncthreads();
    if (!cx.abort) {
      if (!hbm) {
        if (do_red && !(L.nvls_skip & 2u)) {
          nvls_reduce(L.nvls_mc, s_red, nt_of(s - 1), tid, L.nvls_elems);
          asm volatile("fence.acq_rel.sys;" ::: "memory");  // the multicast stores before the barrier's release
        }
      } else {
        if (do_pack && !(L.nvls_skip & 1u)) nvls_pack(L.nvls_uc, s_pack, nt_of(s), L.scale, tid, L.nvls_elems);
        if (do_unpack && !(L.nvls_skip & 1u)) nvls_unpack(L.nvls_uc, s_unpack, nt_of(s - 2), L.lr, L.epilogue, tid);
      }
    }
    if (s < nchunks + 1) cta_barrier(v, P, cx);  // the last step (unpack only) needs none
    else __syncthreads();
  }
  if (stamped) L.stamps[stamp_at + 1] = globaltimer_ns();
  cta_exit<P>(v, cx);
}

// ---- copy-engine mode ---------------------------------------------------------
// During a real backward the gradients of each finished group travel to the
// peers' arenas as copy-engine (DMA) writes over NVLink — no SM is taken
// from the backward. After it: ce_signal_kernel publishes "iteration delivered"
// to every peer, ce_reduce_kernel (full width) waits for every peer's
// delivery, reduces every tile in rank order from the local arena (own
// contribution in place) fused with SGD, and, when its last CTA is done,
// publishes "iteration reduced" so the peers may overwrite the arena with the
// next iteration's copies (ce_wait_kernel, before the first copy).

__device__ __forceinline__ uint64_t* ce_pushed(const RankView& v, int at, int src) {
  return reinterpret_cast<uint64_t*>(v.signal[at] + kCeWord) + src;
}

__device__ __forceinline__ uint64_t* ce_reduced(const RankView& v, int at, int src) {
  return reinterpret_cast<uint64_t*>(v.signal[at] + kCeWord) + kMaxRanks + src;
}

// One thread per (emulated) rank: every peer has reduced iteration iter-1.
template <int P>
__global__ void ce_wait_kernel_t(const __grid_constant__ CeLaunch C, int n_views) {
  if (static_cast<int>(threadIdx.x) >= n_views) return;
  const RankView& v = C.views[threadIdx.x];
  const uint64_t want = C.iter - 1;
#pragma unroll 1
  for (int q = 0; q < P; ++q) {
    if (q == v.rank) continue;
    const uint64_t* f = ce_reduced(v, v.rank, q);
    if (!spin_until(v, [&] { return ld_acquire_sys_u64(f) >= want; })) return;
  }
}

// One thread per (emulated) rank: this rank's copies of iteration `iter`
// (queued before this kernel on its stream) are complete; tell every peer.
template <int P>
__global__ void ce_signal_kernel(const __grid_constant__ CeLaunch C, int n_views) {
  if (static_cast<int>(threadIdx.x) >= n_views) return;
  const RankView& v = C.views[threadIdx.x];
  __threadfence_system();
#pragma unroll 1
  for (int q = 0; q < P; ++q) {
    if (q != v.rank) st_release_sys_u64(ce_pushed(v, q, v.rank), C.iter);
  }
}

// Full-width reduce + SGD of every tile of the plan from the local arena.
// kThreads threads (the data-thread layout of reduce_tile_staged).
template <int P, typename T>
__global__ void __launch_bounds__(kThreads, 1) ce_reduce_kernel(const __grid_constant__ CeLaunch C) {
  extern __shared__ __align__(1024) uint8_t dsmem[];
  __shared__ uint32_t s_ok;
  const RankView& v = C.views[blockIdx.y];
  const int t = static_cast<int>(threadIdx.x);
  if (t == 0) s_ok = 1u;
  __syncthreads();
  if (t < P && t != v.rank) {
    const uint64_t* f = ce_pushed(v, v.rank, t);
    if (!spin_until(v, [&] { return ld_acquire_sys_u64(f) >= C.iter; })) s_ok = 0u;
  }
  __syncthreads();
  if (s_ok) {
    float4* staging = reinterpret_cast<float4*>(dsmem);
    const uint64_t my_slot = static_cast<uint64_t>(v.rank) * C.slot_stride;
    for (uint32_t ti = blockIdx.x; ti < C.n_tiles; ti += gridDim.x) {
      reduce_tile_staged<P, T>(v, C.tiles[ti], C.slot_stride, false, my_slot, C.scale, C.lr, C.epilogue, staging);
    }
  }
  __syncthreads();
  if (t == 0 && s_ok) {
    // every CTA of this rank has read its arena tiles: the last one lets the
    // peers push the next iteration
    __threadfence();
    uint32_t* done = C.done + blockIdx.y;
    if (atomicAdd(done, 1u) == gridDim.x - 1) {
      *done = 0u;
      __threadfence_system();
#pragma unroll 1
      for (int q = 0; q < P; ++q) {
        if (q != v.rank) st_release_sys_u64(ce_reduced(v, q, v.rank), C.iter);
      }
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(kBlock) pack_kernel(const Tile* tiles, uint32_t n_tiles, float* const* grads,
                                                       T* merge, uint64_t begin, float scale) {
  for (uint32_t ti = blockIdx.x; ti < n_tiles; ti += gridDim.x) {
    Tile t = tiles[ti];
    t.moff = static_cast<uint32_t>(t.moff - begin);
    pack_tile<T>(t, grads, merge, scale);
  }
}

template <typename T>
__global__ void __launch_bounds__(kBlock) unpack_sgd_kernel(const Tile* tiles, uint32_t n_tiles,
                                                             float* const* grads, float* const* weights,
                                                             const T* merge, uint64_t begin, float lr,
                                                             int epi) {
  for (uint32_t ti = blockIdx.x; ti < n_tiles; ti += gridDim.x) {
    const Tile t = tiles[ti];
    const uint32_t layer = t.layer & kLayerMask;
    const T* red = merge + (t.moff - begin);
    float* w = weights[layer];
    T* g = as<T>(grads[layer]);
    const uint32_t nvec = (t.len + 3) >> 2;
    float4 x[kPackVec], wv[kPackVec];
#pragma unroll
    for (uint32_t k = 0; k < kPackVec; ++k) {
      const uint32_t i = threadIdx.x + k * kBlock;
      if (i < nvec) x[k] = ld4<T>(red + i * 4);
    }
    load_w_batch<kPackVec>(t, threadIdx.x, kBlock, w, epi, wv);
    apply_batch<kPackVec, T>(t, threadIdx.x, kBlock, x, wv, w, g, lr, epi);
  }
}

// The whole backward replay of one iteration in ONE thread (engine
// pipelines): spin to each group head's ready time in backward order and
// mark the group ready for the comm engine. No per-group kernel launches, so
// the emulated compute stream is continuously busy and its timing exact.
__global__ void replay_all_kernel(unsigned long long* clock, const unsigned long long* deadlines,
                                  uint32_t n, const uint32_t* pipe, uint32_t* flags, int gate) {
  if (threadIdx.x != 0) return;
  // the engine of the previous iteration has finished (graph join), so the
  // iteration counter is this iteration's
  const uint32_t stamp = ld_volatile_u32(pipe + 1) + 1;
  // gate (calibration): the replay clock starts when this rank's engine has
  // passed its entry barrier (pipe[0]), so every rank's group becomes ready
  // at the same time and T(M) excludes the ranks' launch skew
  if (gate) {
    const uint64_t w0 = globaltimer_ns();
    while (static_cast<int32_t>(ld_acquire_gpu(pipe) - stamp) < 0 && globaltimer_ns() - w0 < kTimeoutNs) {
    }
  }
  const unsigned long long t0 = globaltimer_ns();
  clock[0] = t0;
  unsigned long long now = t0;
  for (uint32_t k = 0; k < n; ++k) {
    const unsigned long long due = t0 + deadlines[k];
    while (now < due) now = globaltimer_ns();
    st_release_gpu(flags + (n - 1 - k), stamp);  // groups in backward order
  }
  clock[1] = now;
}

// Real-backward integration: after the backward of every layer of group g
// has been enqueued on the compute stream, this 1-thread kernel marks g
// ready for the comm engine of the running iteration (stream order makes
// the group's gradients complete before it runs).
__global__ void mark_ready_kernel(const uint32_t* pipe, uint32_t* flags, uint32_t g) {
  if (threadIdx.x == 0) st_release_gpu(flags + g, ld_volatile_u32(pipe + 1) + 1);
}

// One group head of the replay (per-group-launch pipelines). clock[0]:
// iteration start (written by the first replay kernel of an iteration),
// clock[1]: completion time of the latest replay kernel. When `ready` is
// given, the group is marked ready for the comm engine.
__global__ void replay_kernel(unsigned long long* clock, unsigned long long deadline_ns, int first,
                              uint32_t* ready) {
  if (threadIdx.x != 0) return;
  unsigned long long t0;
  if (first) {
    t0 = globaltimer_ns();
    clock[0] = t0;
  } else {
    t0 = *reinterpret_cast<volatile unsigned long long*>(clock);
  }
  const unsigned long long due = t0 + deadline_ns;
  unsigned long long now = globaltimer_ns();
  while (now < due) now = globaltimer_ns();
  clock[1] = now;
  if (ready != nullptr) {
    __threadfence();
    atomicAdd(ready, 1u);
  }
}

// L2 eviction between iterations: READS of a buffer larger than L2 from a
// FEW CTAs, so the flush never occupies every SM (a full-grid memset delayed
// the concurrently launched one-thread replay kernel by the whole flush,
// measured ~40 us per iteration). Reads, not stores: a store flush leaves up
// to the whole L2 DIRTY, and the next kernel would pay its write-back (~126
// MB at HBM speed, ~20 us: a third of a small plan's drain); a read flush
// writes back the previous kernel's dirty lines itself and leaves clean ones.
__global__ void __launch_bounds__(512) l2_flush_kernel(float4* buf, size_t n_vec, uint32_t salt) {
  float acc = 0.0f;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n_vec;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const float4 x = __ldcg(buf + i);
    acc += x.x + x.y + x.z + x.w;
  }
  if (__float_as_uint(acc) == salt) buf[0].y = acc;  // (keeps the loads; practically never taken)
}

constexpr size_t kSmemBytes =
    static_cast<size_t>(kStages) * kStageBytes + static_cast<size_t>(kThreads) * kStageSlots * 16;

constexpr size_t smem_for(int P) { return P > 1 ? kSmemBytes : 0; }
// The engine: P > 1 the push ring + staging; P = 1 with STREAM the TMA SGD ring.
constexpr size_t smem_for_engine(int P, bool stream) { return P > 1 ? kSmemBytes : (stream ? kSmemP1 : 0); }

template <int P, bool TWO, bool LB, typename T>
cudaError_t launch_t(const GroupLaunch& L, dim3 grid, cudaStream_t stream) {
  auto* fn = group_allreduce_kernel<P, TWO, LB, T>;
  if constexpr (LB) {
    void* args[] = {const_cast<GroupLaunch*>(&L)};
    return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(fn), grid, dim3(kBlock), args, smem_for(P),
                                       stream);
  } else {
    fn<<<grid, kBlock, smem_for(P), stream>>>(L);
    return cudaGetLastError();
  }
}

template <bool LB, typename T>
cudaError_t launch_lb(const GroupLaunch& L, dim3 grid, bool two, cudaStream_t s) {
  switch (L.nranks) {
    case 1: return launch_t<1, false, LB, T>(L, grid, s);
    case 2: return two ? launch_t<2, true, LB, T>(L, grid, s) : launch_t<2, false, LB, T>(L, grid, s);
    case 4: return two ? launch_t<4, true, LB, T>(L, grid, s) : launch_t<4, false, LB, T>(L, grid, s);
    case 8: return two ? launch_t<8, true, LB, T>(L, grid, s) : launch_t<8, false, LB, T>(L, grid, s);
    default: return cudaErrorInvalidValue;
  }
}

template <typename T, bool S>
const void* engine_fn_t(int nranks) {
  switch (nranks) {
    case 1: return reinterpret_cast<const void*>(engine_kernel<1, T, S>);
    case 2: return reinterpret_cast<const void*>(engine_kernel<2, T, S>);
    case 4: return reinterpret_cast<const void*>(engine_kernel<4, T, S>);
    case 8: return reinterpret_cast<const void*>(engine_kernel<8, T, S>);
    default: return nullptr;
  }
}

const void* engine_fn(int nranks, int dtype, bool stream) {
  if (stream) return dtype == MGW_DTYPE_BF16 ? engine_fn_t<bf16, true>(nranks) : engine_fn_t<float, true>(nranks);
  return dtype == MGW_DTYPE_BF16 ? engine_fn_t<bf16, false>(nranks) : engine_fn_t<float, false>(nranks);
}

template <typename T>
const void* group_fn_t(int nranks, bool two_shot, bool loopback) {
#define MGW_PICK(P, TWO, LB) return reinterpret_cast<const void*>(group_allreduce_kernel<P, TWO, LB, T>)
  if (loopback) {
    if (nranks == 1) MGW_PICK(1, false, true);
    if (nranks == 2) { if (two_shot) MGW_PICK(2, true, true); MGW_PICK(2, false, true); }
    if (nranks == 4) { if (two_shot) MGW_PICK(4, true, true); MGW_PICK(4, false, true); }
    if (nranks == 8) { if (two_shot) MGW_PICK(8, true, true); MGW_PICK(8, false, true); }
  } else {
    if (nranks == 1) MGW_PICK(1, false, false);
    if (nranks == 2) { if (two_shot) MGW_PICK(2, true, false); MGW_PICK(2, false, false); }
    if (nranks == 4) { if (two_shot) MGW_PICK(4, true, false); MGW_PICK(4, false, false); }
    if (nranks == 8) { if (two_shot) MGW_PICK(8, true, false); MGW_PICK(8, false, false); }
  }
#undef MGW_PICK
  return nullptr;
}

const void* group_fn(int nranks, bool two_shot, bool loopback, int dtype) {
  return dtype == MGW_DTYPE_BF16 ? group_fn_t<bf16>(nranks, two_shot, loopback)
                                 : group_fn_t<float>(nranks, two_shot, loopback);
}

}  // namespace

cudaError_t launch_group_allreduce(const GroupLaunch& L, int ctas_per_rank, bool two_shot,
                                   bool loopback, cudaStream_t stream) {
  const dim3 grid(ctas_per_rank, loopback ? L.nranks : 1);
  if (L.dtype == MGW_DTYPE_BF16) {
    return loopback ? launch_lb<true, bf16>(L, grid, two_shot, stream)
                    : launch_lb<false, bf16>(L, grid, two_shot, stream);
  }
  return loopback ? launch_lb<true, float>(L, grid, two_shot, stream)
                  : launch_lb<false, float>(L, grid, two_shot, stream);
}

cudaError_t launch_nvls_group(const GroupLaunch& L, int ctas, cudaStream_t stream) {
  switch (L.nranks) {
    case 2: nvls_group_kernel<2><<<ctas, kNvlsBlock, 0, stream>>>(L); break;
    case 4: nvls_group_kernel<4><<<ctas, kNvlsBlock, 0, stream>>>(L); break;
    case 8: nvls_group_kernel<8><<<ctas, kNvlsBlock, 0, stream>>>(L); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t nvls_ctas_per_sm(int nranks, int* out) {
  const void* fn = nranks == 2 ? reinterpret_cast<const void*>(nvls_group_kernel<2>)
                   : nranks == 4 ? reinterpret_cast<const void*>(nvls_group_kernel<4>)
                                 : reinterpret_cast<const void*>(nvls_group_kernel<8>);
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, fn, kNvlsBlock, 0);
}

cudaError_t launch_engine(const EngineLaunch& E, int ctas, int ranks, cudaStream_t stream) {
  const void* fn = engine_fn(E.nranks, E.dtype, E.stream != 0);
  if (fn == nullptr) return cudaErrorInvalidValue;
  void* args[] = {const_cast<EngineLaunch*>(&E)};
  return cudaLaunchKernel(fn, dim3(ctas, ranks), dim3(kBlock), args, smem_for_engine(E.nranks, E.stream != 0),
                          stream);
}

cudaError_t engine_ctas_per_sm(int nranks, int dtype, int* out) {
  const void* fn = engine_fn(nranks, dtype, true);
  if (fn == nullptr) return cudaErrorInvalidValue;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, fn, kBlock, smem_for_engine(nranks, true));
}

cudaError_t max_ctas_per_sm(int nranks, bool two_shot, bool loopback, int dtype, int* out) {
  const void* fn = group_fn(nranks, two_shot, loopback, dtype);
  if (fn == nullptr) return cudaErrorInvalidValue;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, fn, kBlock, smem_for(nranks));
}

cudaError_t launch_pack(const Tile* tiles, uint32_t n_tiles, float* const* grads, void* merge,
                        uint64_t begin, float scale, int dtype, int ctas, cudaStream_t stream) {
  if (dtype == MGW_DTYPE_BF16) {
    pack_kernel<bf16><<<ctas, kBlock, 0, stream>>>(tiles, n_tiles, grads, static_cast<bf16*>(merge), begin, scale);
  } else {
    pack_kernel<float><<<ctas, kBlock, 0, stream>>>(tiles, n_tiles, grads, static_cast<float*>(merge), begin,
                                                     scale);
  }
  return cudaGetLastError();
}

cudaError_t launch_unpack_sgd(const Tile* tiles, uint32_t n_tiles, float* const* grads,
                              float* const* weights, const void* merge, uint64_t begin, float lr,
                              int epi, int dtype, int ctas, cudaStream_t stream) {
  if (dtype == MGW_DTYPE_BF16) {
    unpack_sgd_kernel<bf16><<<ctas, kBlock, 0, stream>>>(tiles, n_tiles, grads, weights,
                                                          static_cast<const bf16*>(merge), begin, lr, epi);
  } else {
    unpack_sgd_kernel<float><<<ctas, kBlock, 0, stream>>>(tiles, n_tiles, grads, weights,
                                                           static_cast<const float*>(merge), begin, lr, epi);
  }
  return cudaGetLastError();
}

cudaError_t launch_replay(unsigned long long* clock, unsigned long long deadline_ns, int first,
                          uint32_t* ready, cudaStream_t stream) {
  replay_kernel<<<1, 32, 0, stream>>>(clock, deadline_ns, first, ready);
  return cudaGetLastError();
}

cudaError_t launch_l2_flush(void* buf, size_t bytes, int ctas, cudaStream_t stream) {
  l2_flush_kernel<<<ctas, 512, 0, stream>>>(static_cast<float4*>(buf), bytes / sizeof(float4), 0x5a5a);
  return cudaGetLastError();
}

cudaError_t launch_replay_all(unsigned long long* clock, const unsigned long long* deadlines_ns,
                              uint32_t n, const uint32_t* pipe, uint32_t* flags,
                              cudaStream_t stream, int gate) {
  replay_all_kernel<<<1, 32, 0, stream>>>(clock, deadlines_ns, n, pipe, flags, gate);
  return cudaGetLastError();
}

// CUDA 12 loads modules lazily, at a kernel's first launch, and that load
// waits for the context to go idle. A 1-thread mark / replay kernel launched
// for the first time while the persistent engine spins waiting for it would
// therefore deadlock (measured: the engine hit its 10 s ready timeout, then
// the mark kernel ran). Every kernel is loaded up front instead.
cudaError_t preload_ce_kernels();

cudaError_t preload_kernels() {
  const void* fns[] = {
      reinterpret_cast<const void*>(mark_ready_kernel),
      reinterpret_cast<const void*>(replay_all_kernel),
      reinterpret_cast<const void*>(replay_kernel),
      reinterpret_cast<const void*>(l2_flush_kernel),
      reinterpret_cast<const void*>(pack_kernel<float>),
      reinterpret_cast<const void*>(pack_kernel<bf16>),
      reinterpret_cast<const void*>(unpack_sgd_kernel<float>),
      reinterpret_cast<const void*>(unpack_sgd_kernel<bf16>),
      reinterpret_cast<const void*>(nvls_group_kernel<2>),
      reinterpret_cast<const void*>(nvls_group_kernel<4>),
      reinterpret_cast<const void*>(nvls_group_kernel<8>),
  };
  for (const void* f : fns) {
    cudaFuncAttributes attr;
    const cudaError_t e = cudaFuncGetAttributes(&attr, f);
    if (e != cudaSuccess) return e;
  }
  {
    const cudaError_t e = preload_ce_kernels();
    if (e != cudaSuccess) return e;
  }
  for (int dt : {MGW_DTYPE_F32, MGW_DTYPE_BF16}) {
    for (int p : {1, 2, 4, 8}) {
      const void* ks[] = {engine_fn(p, dt, true), engine_fn(p, dt, false), group_fn(p, false, false, dt), group_fn(p, true, false, dt),
                          group_fn(p, false, true, dt), group_fn(p, true, true, dt)};
      for (const void* f : ks) {
        cudaFuncAttributes attr;
        cudaError_t e = cudaFuncGetAttributes(&attr, f);
        // the TMA ring lives in dynamic shared memory (> the 48 KiB default)
        if (e == cudaSuccess && p > 1) {
          e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemBytes));
        }
        if (e == cudaSuccess && p == 1 && f == engine_fn(1, dt, true)) {
          e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemP1));
        }
        if (e != cudaSuccess) return e;
      }
    }
  }
  return cudaSuccess;
}

cudaError_t launch_mark_ready(const uint32_t* pipe, uint32_t* flags, uint32_t g,
                              cudaStream_t stream) {
  mark_ready_kernel<<<1, 32, 0, stream>>>(pipe, flags, g);
  return cudaGetLastError();
}


namespace {
template <int P>
cudaError_t ce_launch_p(int what, const CeLaunch& C, int n_views, int ctas, cudaStream_t s) {
  if (what == 0) {
    ce_wait_kernel_t<P><<<1, 32, 0, s>>>(C, n_views);
  } else if (what == 1) {
    ce_signal_kernel<P><<<1, 32, 0, s>>>(C, n_views);
  } else {
    const size_t smem = static_cast<size_t>(kThreads) * kStageSlots * 16;
    const dim3 grid(ctas, n_views);
    if (C.dtype == MGW_DTYPE_BF16) {
      ce_reduce_kernel<P, bf16><<<grid, kThreads, smem, s>>>(C);
    } else {
      ce_reduce_kernel<P, float><<<grid, kThreads, smem, s>>>(C);
    }
  }
  return cudaGetLastError();
}
}  // namespace

// what: 0 wait (peers reduced iter-1), 1 signal (iter delivered), 2 reduce.
cudaError_t launch_ce(int what, const CeLaunch& C, int n_views, int ctas, cudaStream_t stream) {
  switch (C.nranks) {
    case 2: return ce_launch_p<2>(what, C, n_views, ctas, stream);
    case 4: return ce_launch_p<4>(what, C, n_views, ctas, stream);
    case 8: return ce_launch_p<8>(what, C, n_views, ctas, stream);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t preload_ce_kernels() {
  const size_t smem = static_cast<size_t>(kThreads) * kStageSlots * 16;
  const void* fns[] = {
      reinterpret_cast<const void*>(ce_reduce_kernel<2, float>), reinterpret_cast<const void*>(ce_reduce_kernel<4, float>),
      reinterpret_cast<const void*>(ce_reduce_kernel<8, float>), reinterpret_cast<const void*>(ce_reduce_kernel<2, bf16>),
      reinterpret_cast<const void*>(ce_reduce_kernel<4, bf16>), reinterpret_cast<const void*>(ce_reduce_kernel<8, bf16>)};
  for (const void* f : fns) {
    const cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  const void* small[] = {reinterpret_cast<const void*>(ce_wait_kernel_t<2>), reinterpret_cast<const void*>(ce_wait_kernel_t<4>),
                         reinterpret_cast<const void*>(ce_wait_kernel_t<8>), reinterpret_cast<const void*>(ce_signal_kernel<2>),
                         reinterpret_cast<const void*>(ce_signal_kernel<4>), reinterpret_cast<const void*>(ce_signal_kernel<8>)};
  for (const void* f : small) {
    cudaFuncAttributes attr;
    const cudaError_t e = cudaFuncGetAttributes(&attr, f);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace mgw
