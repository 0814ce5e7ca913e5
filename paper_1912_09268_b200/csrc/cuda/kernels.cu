// mgwfbp-b200 sm_100a kernels.
//
//  run_group<P>  — THE hot op, shared by both launch styles: for one merge
//      group, pack (gather layer grads x 1/P) fused with a push over NVLink
//      into the peers' merge arenas -> rank-order reduction from local HBM ->
//      unpack + SGD into the layer weights.
//        one-shot: every rank pushes its tiles to every rank; 1 barrier per
//          chunk.
//        two-shot: tile t is owned by rank t % P; ranks push each tile to its
//          owner (reduce-scatter), owners reduce + push the result to every
//          peer (all-gather) fused with SGD; 2 barriers per chunk.
//      A CTA walks its tiles in 256 KiB CHUNKS, software-pipelined: chunk
//      c+1's posted NVLink stores are issued before chunk c's local work.
//  engine_kernel<P> — the persistent comm engine: one launch per iteration
//      runs every group in backward order as soon as the compute side marks
//      its head ready (paper Algorithm 2's daemon thread, on the GPU; no
//      per-group launch latency).
//  group_allreduce_kernel<P, TWO_SHOT, LOOPBACK> — one launch per group
//      (standalone C-ABI op, calibration of that op, and the single-GPU
//      loopback emulation of P ranks in one cooperative launch).
//  pack_kernel / unpack_sgd_kernel — the standalone pack and unpack+SGD
//      ops of the C ABI (rank-local, HBM-bound).
//  replay_all_kernel / replay_kernel — backward-pass replay on %globaltimer.
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
#include <cuda_runtime.h>

#include "mgw_device.cuh"
#include "mgwfbp.h"

namespace mgw {

namespace {

constexpr uint64_t kTimeoutNs = 10ull * 1000 * 1000 * 1000;  // 10 s: error, never a hang
// Software pipelining of the push data path. A CTA walks its tiles in
// CHUNKS and issues chunk c+1's posted NVLink stores BEFORE chunk c's local
// HBM work, so the stores drain while the CTA reduces / applies SGD; one
// barrier per chunk. (Measured on 2x B200, 256 MiB: a non-overlapped
// barrier per 4-tile chunk cost more than it bought — 296 / 221 GB/s vs
// 400 / 478 unchunked; the overlap below is what chunks are for, and a
// chunk is 256 KiB per CTA so barriers stay rare.)
constexpr uint32_t kOneShotChunk = 16;  // tiles of this CTA per chunk (256 KiB)

template <int P>
struct TwoShotChunk {  // super-tiles (P tiles each) of this CTA per chunk: 256 KiB
  static constexpr uint32_t value = 16 / P;
};

__device__ __forceinline__ float4 load_tail(const float* p, uint32_t n) {
  float4 v;
  v.x = n > 0 ? p[0] : 0.0f;
  v.y = n > 1 ? p[1] : 0.0f;
  v.z = n > 2 ? p[2] : 0.0f;
  v.w = n > 3 ? p[3] : 0.0f;
  return v;
}

__device__ __forceinline__ void pack_tile(const Tile& t, float* const* grads, float* dst_base,
                                          float scale) {
  const float* src = grads[t.layer & kLayerMask] + t.src;
  float* dst = dst_base + t.moff;
  const bool aligned = !(t.layer & kGradUnaligned);
  const uint32_t nvec = (t.len + 3) >> 2;
  for (uint32_t i = threadIdx.x; i < nvec; i += blockDim.x) {
    const uint32_t e = i * 4;
    const float4 x = (aligned && e + 4 <= t.len) ? ld_stream_v4(src + e) : load_tail(src + e, t.len - e);
    st_v4(dst + e, mul4(x, scale));
  }
}

// Element group e..e+3 of tile t receives the reduced gradient `g`.
__device__ __forceinline__ void epilogue(const Tile& t, uint32_t e, float4 g, float* w_layer,
                                         float* g_layer, float lr, int epi) {
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
    float* d = g_layer + t.src + e;
    if (n == 4 && !(t.layer & kGradUnaligned)) {
      st_v4(d, g);
    } else {
      if (n > 0) d[0] = g.x;
      if (n > 1) d[1] = g.y;
      if (n > 2) d[2] = g.z;
      if (n > 3) d[3] = g.w;
    }
  }
}

// Barrier of CTA index `cta` with the same CTA index of every rank.
// `count` is this CTA's barrier counter (same value in every thread).
__device__ __forceinline__ void cta_barrier(const RankView& v, int P, uint32_t cta, uint32_t& count,
                                            bool after_remote_stores) {
  ++count;
  // bar.sync orders every warp's posted NVLink stores before the flag
  // writers' st.release.sys, and release is cumulative at system scope, so
  // a peer that acquires the flag sees the data (no per-thread fence.sys).
  (void)after_remote_stores;
  __syncthreads();
  if (threadIdx.x < P) {
    const int q = threadIdx.x;
    st_release_sys(v.signal[q] + cta * kMaxRanks + v.rank, count);
    const uint32_t* mine = v.signal[v.rank] + cta * kMaxRanks + q;
    if (static_cast<int32_t>(ld_acquire_sys(mine) - count) < 0) {
      const uint64_t t0 = globaltimer_ns();
      while (static_cast<int32_t>(ld_acquire_sys(mine) - count) < 0) {
        if (globaltimer_ns() - t0 > kTimeoutNs) {
          atomicExch(v.state + kStateError, 1u);
          break;
        }
      }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ uint32_t load_cta_count(const RankView& v, uint32_t cta) {
  __shared__ uint32_t s_count;
  if (threadIdx.x == 0) s_count = ld_volatile_u32(v.state + kStateCtaBase + cta);
  __syncthreads();
  return s_count;
}

__device__ __forceinline__ void store_cta_count(const RankView& v, uint32_t cta, uint32_t count) {
  if (threadIdx.x == 0) v.state[kStateCtaBase + cta] = count;
}

// ---- push data path -------------------------------------------------------
// Every rank's merge arena holds one SLOT per source rank (slot r at element
// r * slot_stride, laid out like the merge buffer). Transfers are posted
// NVLink stores into the peers' slots (no remote-load latency on the
// critical path); every reduction reads local HBM only.

// Gather + scale tile t of this rank's gradients and store it into slot
// `me` of the arenas of ranks [q_begin, q_end) — the pack kernel fused with
// the scatter. kVecPerThread loads are issued before any store.
template <int P>
__device__ __forceinline__ void scatter_tile(const RankView& v, const Tile& t, int q_begin, int q_end,
                                             uint64_t my_slot, float scale) {
  const float* src = v.grads[t.layer & kLayerMask] + t.src;
  const bool aligned = !(t.layer & kGradUnaligned);
  const uint32_t nvec = (t.len + 3) >> 2;
  float4 x[kVecPerThread];
#pragma unroll
  for (uint32_t k = 0; k < kVecPerThread; ++k) {
    const uint32_t i = threadIdx.x + k * kThreads;
    if (i < nvec) {
      const uint32_t e = i * 4;
      x[k] = (aligned && e + 4 <= t.len) ? ld_stream_v4(src + e) : load_tail(src + e, t.len - e);
      x[k] = mul4(x[k], scale);
    }
  }
#pragma unroll
  for (uint32_t k = 0; k < kVecPerThread; ++k) {
    const uint32_t i = threadIdx.x + k * kThreads;
    if (i < nvec) {
#pragma unroll
      for (int q = 0; q < P; ++q) {
        if (q >= q_begin && q < q_end) st_v4(v.arena[q] + my_slot + t.moff + i * 4, x[k]);
      }
    }
  }
}

// Vectors of a thread reduced per batch: all slot loads of a batch are in
// flight together (B * P <= 8 float4 per thread keeps the engine at <= 128
// registers without spills).
template <int P>
struct RedBatch {
  static constexpr uint32_t raw = P >= 4 ? 1 : 4 / P;
  static constexpr uint32_t value = raw < kVecPerThread ? raw : kVecPerThread;
};

// SGD (+ optional grad write-back) for B vectors of tile t (thread vector
// indices i0, i0 + stride, ...): the W loads of the whole batch are issued
// before any store, so their latency overlaps.
template <uint32_t B>
__device__ __forceinline__ void apply_batch(const Tile& t, uint32_t i0, uint32_t stride,
                                            const float4 (&g)[B], float* w_layer, float* g_layer,
                                            float lr, int epi) {
  const uint32_t nvec = (t.len + 3) >> 2;
  const bool vec_w = (epi & MGW_SGD) && w_layer != nullptr && !(t.layer & kWeightUnaligned);
  float4 wv[B];
#pragma unroll
  for (uint32_t j = 0; j < B; ++j) {
    const uint32_t i = i0 + j * stride;
    if (vec_w && i < nvec && i * 4 + 4 <= t.len) wv[j] = ld_v4(w_layer + t.src + i * 4);
  }
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
      if (epi & MGW_WRITE_GRAD) epilogue(t, e, g[j], nullptr, g_layer, lr, MGW_WRITE_GRAD);
    } else {
      epilogue(t, e, g[j], w_layer, g_layer, lr, epi);  // tail / unaligned / no-SGD
    }
  }
}

// Rank-order sum of tile t over the P local slots (x0 + x1 + ... + x_{P-1},
// each already scaled by 1/P; .cg loads: peers wrote them), B vectors per
// batch; optionally push each sum into slot `my_slot` of every peer (the
// two-shot owner's all-gather), then SGD.
template <int P>
__device__ __forceinline__ void reduce_tile(const RankView& v, const Tile& t, uint64_t slot_stride,
                                            bool push_to_peers, uint64_t my_slot, float lr, int epi) {
  constexpr uint32_t B = RedBatch<P>::value;
  const float* base = v.arena[v.rank] + t.moff;
  const uint32_t nvec = (t.len + 3) >> 2;
  const uint32_t layer = t.layer & kLayerMask;
  float* w = v.weights[layer];
  float* g = v.grads[layer];
#pragma unroll 1
  for (uint32_t k0 = 0; k0 < kVecPerThread; k0 += B) {
    const uint32_t i0 = threadIdx.x + k0 * kThreads;
    if (i0 >= nvec) break;
    float4 x[B][P];
#pragma unroll
    for (uint32_t j = 0; j < B; ++j) {
      const uint32_t i = i0 + j * kThreads;
      if (i < nvec) {
#pragma unroll
        for (int r = 0; r < P; ++r) x[j][r] = ld_cg_v4(base + r * slot_stride + i * 4);
      }
    }
    float4 s[B];
#pragma unroll
    for (uint32_t j = 0; j < B; ++j) {
      s[j] = x[j][0];
#pragma unroll
      for (int r = 1; r < P; ++r) s[j] = add4(s[j], x[j][r]);
    }
    if (push_to_peers) {
#pragma unroll
      for (uint32_t j = 0; j < B; ++j) {
        const uint32_t i = i0 + j * kThreads;
        if (i >= nvec) continue;
#pragma unroll
        for (int q = 0; q < P; ++q) {
          if (q != v.rank) st_v4(v.arena[q] + my_slot + t.moff + i * 4, s[j]);
        }
      }
    }
    apply_batch<B>(t, i0, kThreads, s, w, g, lr, epi);
  }
}

// One-shot, pipelined over chunks of this CTA's tiles (cta + j*ncta):
//   push(0); barrier; for c: push(c+1); reduce+SGD(c); barrier (if c+1<n)
// push = gather x 1/P into slot `me` of every rank; reduce = rank-order sum
// of the P local slots. NVLink: (P-1) * S posted writes per rank.
template <int P>
__device__ __forceinline__ void one_shot_group(const RankView& v, const Tile* tiles,
                                               uint32_t n_tiles, uint64_t slot_stride, float scale,
                                               float lr, int epi, uint32_t cta, uint32_t ncta,
                                               uint32_t& count) {
  const uint64_t my_slot = static_cast<uint64_t>(v.rank) * slot_stride;
  const uint32_t mine = cta < n_tiles ? (n_tiles - cta + ncta - 1) / ncta : 0;  // my tiles
  const uint32_t n_chunks = (mine + kOneShotChunk - 1) / kOneShotChunk;
  auto push = [&](uint32_t c) {
#pragma unroll 1
    for (uint32_t j = c * kOneShotChunk; j < mine && j < (c + 1) * kOneShotChunk; ++j) {
      scatter_tile<P>(v, tiles[cta + j * ncta], 0, P, my_slot, scale);
    }
  };
  // step t: push(t) [t < n], reduce+SGD(t-1) [t >= 1], barrier [t < n]
#pragma unroll 1
  for (uint32_t t = 0; t <= n_chunks && n_chunks > 0; ++t) {
    if (t < n_chunks) push(t);
    if (t >= 1) {
#pragma unroll 1
      for (uint32_t j = (t - 1) * kOneShotChunk; j < mine && j < t * kOneShotChunk; ++j) {
        reduce_tile<P>(v, tiles[cta + j * ncta], slot_stride, false, my_slot, lr, epi);
      }
    }
    if (t < n_chunks) cta_barrier(v, P, cta, count, true);
  }
}

// Two-shot: super-tile s = tiles [s*P, s*P+P), tile s*P+q owned by rank q.
//   RS(c):  push each tile of chunk c to its owner's slot `me`
//   RA(c):  owner: rank-order sum of its tile's P local slots, SGD, push the
//           result into slot `owner` of every peer (all-gather)
//   AP(c):  apply the other owners' results from the local slots (SGD)
// Pipelined: RS(0); bar; RA(0); RS(1); bar; for c: RA(c+1); RS(c+2); AP(c);
// bar (if c+1<n). NVLink: 2 (P-1)/P * S posted writes per rank.
template <int P>
__device__ __forceinline__ void two_shot_group(const RankView& v, const Tile* tiles,
                                               uint32_t n_tiles, uint64_t slot_stride, float scale,
                                               float lr, int epi, uint32_t cta, uint32_t ncta,
                                               uint32_t& count) {
  constexpr uint32_t C = TwoShotChunk<P>::value;
  const uint64_t my_slot = static_cast<uint64_t>(v.rank) * slot_stride;
  const uint32_t n_super = (n_tiles + P - 1) / P;
  const uint32_t mine = cta < n_super ? (n_super - cta + ncta - 1) / ncta : 0;  // my super-tiles
  const uint32_t n_chunks = (mine + C - 1) / C;
  auto rs = [&](uint32_t c) {
#pragma unroll 1
    for (uint32_t j = c * C; j < mine && j < (c + 1) * C; ++j) {
      const uint32_t s = cta + j * ncta;
#pragma unroll 1
      for (int q = 0; q < P; ++q) {
        const uint32_t ti = s * P + q;
        if (ti < n_tiles) scatter_tile<P>(v, tiles[ti], q, q + 1, my_slot, scale);
      }
    }
  };
  auto ra = [&](uint32_t c) {
#pragma unroll 1
    for (uint32_t j = c * C; j < mine && j < (c + 1) * C; ++j) {
      const uint32_t ti = (cta + j * ncta) * P + v.rank;
      if (ti < n_tiles) reduce_tile<P>(v, tiles[ti], slot_stride, true, my_slot, lr, epi);
    }
  };
  auto ap = [&](uint32_t c) {
#pragma unroll 1
    for (uint32_t j = c * C; j < mine && j < (c + 1) * C; ++j) {
      const uint32_t s = cta + j * ncta;
#pragma unroll 1
      for (int q = 0; q < P; ++q) {
        const uint32_t ti = s * P + q;
        if (q == v.rank || ti >= n_tiles) continue;
        const Tile t = tiles[ti];
        const float* red = v.arena[v.rank] + static_cast<uint64_t>(q) * slot_stride + t.moff;
        const uint32_t layer = t.layer & kLayerMask;
        const uint32_t nvec = (t.len + 3) >> 2;
        float4 x[kVecPerThread];
#pragma unroll
        for (uint32_t k = 0; k < kVecPerThread; ++k) {
          const uint32_t i = threadIdx.x + k * kThreads;
          if (i < nvec) x[k] = ld_cg_v4(red + i * 4);
        }
        apply_batch<kVecPerThread>(t, threadIdx.x, kThreads, x, v.weights[layer], v.grads[layer], lr, epi);
      }
    }
  };
  // step t: RA(t-1) [1 <= t <= n], RS(t) [t < n], AP(t-2) [t >= 2],
  // barrier [t <= n] (covers the posted stores of RS(t) and RA(t-1))
#pragma unroll 1
  for (uint32_t t = 0; t <= n_chunks + 1 && n_chunks > 0; ++t) {
    if (t >= 1 && t <= n_chunks) ra(t - 1);
    if (t < n_chunks) rs(t);
    if (t >= 2) ap(t - 2);
    if (t <= n_chunks) cta_barrier(v, P, cta, count, true);
  }
}

// One merge group, executed by CTA `cta` of `ncta`.
template <int P>
__device__ __forceinline__ void run_group(bool two_shot, const RankView& v, const Tile* tiles,
                                          uint32_t n_tiles, uint64_t slot_stride, float scale,
                                          float lr, int epi, uint32_t cta, uint32_t ncta,
                                          uint32_t& count) {
  if constexpr (P == 1) {
    // Single rank: no exchange. grad x 1/P (= 1) straight into the epilogue.
    for (uint32_t ti = cta; ti < n_tiles; ti += ncta) {
      const Tile t = tiles[ti];
      const uint32_t layer = t.layer & kLayerMask;
      const float* src = v.grads[layer] + t.src;
      float* w = v.weights[layer];
      float* g = v.grads[layer];
      const bool aligned = !(t.layer & kGradUnaligned);
      const uint32_t nvec = (t.len + 3) >> 2;
      for (uint32_t i = threadIdx.x; i < nvec; i += blockDim.x) {
        const uint32_t e = i * 4;
        const float4 x = (aligned && e + 4 <= t.len) ? ld_stream_v4(src + e) : load_tail(src + e, t.len - e);
        epilogue(t, e, mul4(x, scale), w, g, lr, epi);
      }
    }
  } else if (two_shot) {
    two_shot_group<P>(v, tiles, n_tiles, slot_stride, scale, lr, epi, cta, ncta, count);
  } else {
    one_shot_group<P>(v, tiles, n_tiles, slot_stride, scale, lr, epi, cta, ncta, count);
  }
}

template <int P, bool TWO_SHOT, bool LOOPBACK>
__global__ void __launch_bounds__(kThreads, 1)
    group_allreduce_kernel(const __grid_constant__ GroupLaunch L) {
  const RankView& v = L.views[LOOPBACK ? blockIdx.y : 0];
  uint32_t count = 0;
  if constexpr (P > 1) {
    count = load_cta_count(v, blockIdx.x);
    cta_barrier(v, P, blockIdx.x, count, false);  // entry: peers have left every older launch
  }
  run_group<P>(TWO_SHOT, v, L.tiles, L.n_tiles, L.slot_stride, L.scale, L.lr, L.epilogue,
               blockIdx.x, gridDim.x, count);
  if constexpr (P > 1) store_cta_count(v, blockIdx.x, count);
}

template <int P>
__global__ void __launch_bounds__(kThreads, 1) engine_kernel(const __grid_constant__ EngineLaunch E) {
  const RankView& v = E.v;
  __shared__ uint32_t s_iter;
  if (threadIdx.x == 0) s_iter = ld_volatile_u32(E.pipe + 1);
  uint32_t count = 0;
  if constexpr (P > 1) {
    count = load_cta_count(v, blockIdx.x);
    // Entry barrier (runs while the compute stream replays the forward
    // pass): every peer has finished every older launch before any push.
    cta_barrier(v, P, blockIdx.x, count, false);
  } else {
    __syncthreads();
  }
  const uint32_t iter = s_iter;
  for (uint32_t k = 0; k < E.G; ++k) {
    const uint32_t gi = E.G - 1 - k;  // backward order: FIFO like timeline.hpp:133-154
    const EngineGroup grp = E.groups[gi];
    const bool two = P > 1 && grp.two_shot != 0;
    const uint32_t units = two ? (grp.n_tiles + P - 1) / P : grp.n_tiles;
    if (blockIdx.x >= units) continue;  // same on every rank: no barrier to skip
    if (threadIdx.x == 0) {
      // group gi is ready for iteration `iter` once its flag reached iter+1
      // (set by the replay, or by a mark kernel after the real backward of
      // the group's layers — groups may complete out of FIFO order)
      const uint32_t target = iter + 1;
      const uint32_t* flag = E.ready + gi;
      if (static_cast<int32_t>(ld_acquire_gpu(flag) - target) < 0) {
        const uint64_t t0 = globaltimer_ns();
        while (static_cast<int32_t>(ld_acquire_gpu(flag) - target) < 0) {
          if (globaltimer_ns() - t0 > kTimeoutNs) {  // compute side never signalled
            atomicExch(E.pipe + 3, 1u);
            break;
          }
        }
      }
      if (E.stamps != nullptr && blockIdx.x == 0) E.stamps[2 * gi] = globaltimer_ns();
    }
    __syncthreads();
    run_group<P>(two, v, E.tiles + grp.tile_first, grp.n_tiles, E.slot_stride, E.scale, E.lr,
                 E.epilogue, blockIdx.x, gridDim.x, count);
    if (E.stamps != nullptr) {
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        const uint32_t active = units < gridDim.x ? units : gridDim.x;
        if (atomicAdd(E.group_done + gi, 1u) == active - 1) {
          E.group_done[gi] = 0;
          E.stamps[2 * gi + 1] = globaltimer_ns();
        }
      }
    }
  }
  if constexpr (P > 1) store_cta_count(v, blockIdx.x, count);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(E.pipe + 2, 1u) == gridDim.x - 1) {
      atomicExch(E.pipe + 2, 0u);
      __threadfence();
      atomicExch(E.pipe + 1, iter + 1);
    }
  }
}

__global__ void __launch_bounds__(kThreads) pack_kernel(const Tile* tiles, uint32_t n_tiles,
                                                         float* const* grads, float* merge,
                                                         uint64_t begin, float scale) {
  for (uint32_t ti = blockIdx.x; ti < n_tiles; ti += gridDim.x) {
    Tile t = tiles[ti];
    t.moff = static_cast<uint32_t>(t.moff - begin);
    pack_tile(t, grads, merge, scale);
  }
}

__global__ void __launch_bounds__(kThreads) unpack_sgd_kernel(const Tile* tiles, uint32_t n_tiles,
                                                               float* const* grads,
                                                               float* const* weights,
                                                               const float* merge, uint64_t begin,
                                                               float lr, int epi) {
  for (uint32_t ti = blockIdx.x; ti < n_tiles; ti += gridDim.x) {
    const Tile t = tiles[ti];
    const uint32_t layer = t.layer & kLayerMask;
    const float* red = merge + (t.moff - begin);
    float* w = weights[layer];
    float* g = grads[layer];
    const uint32_t nvec = (t.len + 3) >> 2;
    for (uint32_t i = threadIdx.x; i < nvec; i += blockDim.x) {
      epilogue(t, i * 4, ld_v4(red + i * 4), w, g, lr, epi);
    }
  }
}

// The whole backward replay of one iteration in ONE thread (engine
// pipelines): spin to each group head's ready time in backward order and
// mark the group ready for the comm engine. No per-group kernel launches, so
// the emulated compute stream is continuously busy and its timing exact.
__global__ void replay_all_kernel(unsigned long long* clock, const unsigned long long* deadlines,
                                  uint32_t n, const uint32_t* pipe, uint32_t* flags) {
  if (threadIdx.x != 0) return;
  // the engine of the previous iteration has finished (graph join), so the
  // iteration counter is this iteration's
  const uint32_t stamp = ld_volatile_u32(pipe + 1) + 1;
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

// L2 eviction between iterations: streaming stores over a buffer larger
// than L2 from a FEW CTAs, so the flush never occupies every SM (a full-grid
// memset delayed the concurrently launched one-thread replay kernel by the
// whole flush, measured ~40 us per iteration).
__global__ void __launch_bounds__(512) l2_flush_kernel(float4* buf, size_t n_vec, uint32_t salt) {
  const float4 v = make_float4(__uint_as_float(salt), 0.0f, 0.0f, 0.0f);
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n_vec;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    __stcs(buf + i, v);
  }
}

template <int P, bool TWO, bool LB>
cudaError_t launch_t(const GroupLaunch& L, dim3 grid, cudaStream_t stream) {
  auto* fn = group_allreduce_kernel<P, TWO, LB>;
  if constexpr (LB) {
    void* args[] = {const_cast<GroupLaunch*>(&L)};
    return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(fn), grid, dim3(kThreads), args, 0,
                                       stream);
  } else {
    fn<<<grid, kThreads, 0, stream>>>(L);
    return cudaGetLastError();
  }
}

template <bool LB>
cudaError_t launch_lb(const GroupLaunch& L, dim3 grid, bool two, cudaStream_t s) {
  switch (L.nranks) {
    case 1: return launch_t<1, false, LB>(L, grid, s);
    case 2: return two ? launch_t<2, true, LB>(L, grid, s) : launch_t<2, false, LB>(L, grid, s);
    case 4: return two ? launch_t<4, true, LB>(L, grid, s) : launch_t<4, false, LB>(L, grid, s);
    case 8: return two ? launch_t<8, true, LB>(L, grid, s) : launch_t<8, false, LB>(L, grid, s);
    default: return cudaErrorInvalidValue;
  }
}

const void* engine_fn(int nranks) {
  switch (nranks) {
    case 1: return reinterpret_cast<const void*>(engine_kernel<1>);
    case 2: return reinterpret_cast<const void*>(engine_kernel<2>);
    case 4: return reinterpret_cast<const void*>(engine_kernel<4>);
    case 8: return reinterpret_cast<const void*>(engine_kernel<8>);
    default: return nullptr;
  }
}

}  // namespace

cudaError_t launch_group_allreduce(const GroupLaunch& L, int ctas_per_rank, bool two_shot,
                                   bool loopback, cudaStream_t stream) {
  const dim3 grid(ctas_per_rank, loopback ? L.nranks : 1);
  return loopback ? launch_lb<true>(L, grid, two_shot, stream)
                  : launch_lb<false>(L, grid, two_shot, stream);
}

cudaError_t launch_engine(const EngineLaunch& E, int ctas, cudaStream_t stream) {
  const void* fn = engine_fn(E.nranks);
  if (fn == nullptr) return cudaErrorInvalidValue;
  void* args[] = {const_cast<EngineLaunch*>(&E)};
  return cudaLaunchKernel(fn, dim3(ctas), dim3(kThreads), args, 0, stream);
}

cudaError_t engine_ctas_per_sm(int nranks, int* out) {
  const void* fn = engine_fn(nranks);
  if (fn == nullptr) return cudaErrorInvalidValue;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, fn, kThreads, 0);
}

cudaError_t max_ctas_per_sm(int nranks, bool two_shot, bool loopback, int* out) {
  const void* fn = nullptr;
#define MGW_PICK(P, TWO, LB) fn = reinterpret_cast<const void*>(group_allreduce_kernel<P, TWO, LB>)
  if (loopback) {
    if (nranks == 1) MGW_PICK(1, false, true);
    else if (nranks == 2) { if (two_shot) MGW_PICK(2, true, true); else MGW_PICK(2, false, true); }
    else if (nranks == 4) { if (two_shot) MGW_PICK(4, true, true); else MGW_PICK(4, false, true); }
    else { if (two_shot) MGW_PICK(8, true, true); else MGW_PICK(8, false, true); }
  } else {
    if (nranks == 1) MGW_PICK(1, false, false);
    else if (nranks == 2) { if (two_shot) MGW_PICK(2, true, false); else MGW_PICK(2, false, false); }
    else if (nranks == 4) { if (two_shot) MGW_PICK(4, true, false); else MGW_PICK(4, false, false); }
    else { if (two_shot) MGW_PICK(8, true, false); else MGW_PICK(8, false, false); }
  }
#undef MGW_PICK
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, fn, kThreads, 0);
}

cudaError_t launch_pack(const Tile* tiles, uint32_t n_tiles, float* const* grads, float* merge,
                        uint64_t begin, float scale, int ctas, cudaStream_t stream) {
  pack_kernel<<<ctas, kThreads, 0, stream>>>(tiles, n_tiles, grads, merge, begin, scale);
  return cudaGetLastError();
}

cudaError_t launch_unpack_sgd(const Tile* tiles, uint32_t n_tiles, float* const* grads,
                              float* const* weights, const float* merge, uint64_t begin, float lr,
                              int epi, int ctas, cudaStream_t stream) {
  unpack_sgd_kernel<<<ctas, kThreads, 0, stream>>>(tiles, n_tiles, grads, weights, merge, begin,
                                                   lr, epi);
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
                              cudaStream_t stream) {
  replay_all_kernel<<<1, 32, 0, stream>>>(clock, deadlines_ns, n, pipe, flags);
  return cudaGetLastError();
}

// CUDA 12 loads modules lazily, at a kernel's first launch, and that load
// waits for the context to go idle. A 1-thread mark / replay kernel launched
// for the first time while the persistent engine spins waiting for it would
// therefore deadlock (measured: the engine hit its 10 s ready timeout, then
// the mark kernel ran). Every kernel is loaded up front instead.
cudaError_t preload_kernels() {
  const void* fns[] = {
      reinterpret_cast<const void*>(mark_ready_kernel),
      reinterpret_cast<const void*>(replay_all_kernel),
      reinterpret_cast<const void*>(replay_kernel),
      reinterpret_cast<const void*>(l2_flush_kernel),
      reinterpret_cast<const void*>(pack_kernel),
      reinterpret_cast<const void*>(unpack_sgd_kernel),
      engine_fn(1), engine_fn(2), engine_fn(4), engine_fn(8),
  };
  for (const void* f : fns) {
    cudaFuncAttributes attr;
    const cudaError_t e = cudaFuncGetAttributes(&attr, f);
    if (e != cudaSuccess) return e;
  }
  for (bool lb : {false, true}) {
    for (int p : {1, 2, 4, 8}) {
      for (bool two : {false, true}) {
        int occ = 0;
        const cudaError_t e = max_ctas_per_sm(p, two, lb, &occ);
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

}  // namespace mgw
