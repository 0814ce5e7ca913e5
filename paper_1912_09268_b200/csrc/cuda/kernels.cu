// mgwfbp-b200 sm_100a kernels.
//
//  group_allreduce_kernel<P, TWO_SHOT, LOOPBACK>  — THE hot op: for one merge
//      group, pack (gather layer grads x 1/P into the merge arena) ->
//      all-reduce over NVLink peer memory, summed in rank order ->
//      unpack + SGD into the layer weights. One launch per group.
//        one-shot: every rank reads every peer's packed tiles; 1 barrier.
//        two-shot: tile t is owned by rank t % P; owners reduce their tiles
//          in place (reduce-scatter), then every rank pulls the other
//          owners' reduced tiles (all-gather) fused with SGD; 2 barriers.
//  pack_kernel / unpack_sgd_kernel — the standalone pack and unpack+SGD
//      ops of the C ABI (rank-local, HBM-bound).
//  replay_kernel — backward-pass replay: one thread spins on %globaltimer
//      until a group head's ready time (pipeline.cu).
//
// Cross-rank synchronisation is per CTA index: CTA b of every rank handles
// the same tiles, so CTA b only waits for CTA b of the peers (flag plane
// [b][src_rank], epoch = launch counter + 1, monotone, never reset).
// Reductions use __fadd_rn / __fmul_rn / __fsub_rn only: no FMA contraction,
// bit-exact with the CPU oracle's fl(fl(x0*s) + x1*s)... rank order.
#include <cstdint>
#include <cuda_runtime.h>

#include "mgw_device.cuh"
#include "mgwfbp.h"

namespace mgw {

namespace {

constexpr uint64_t kBarrierTimeoutNs = 10ull * 1000 * 1000 * 1000;  // 10 s

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
    } else {
      const float gs[4] = {g.x, g.y, g.z, g.w};
      for (uint32_t j = 0; j < n; ++j) w[j] = sgd1(w[j], gs[j], lr);
    }
  }
  if (epi & MGW_WRITE_GRAD) {
    float* d = g_layer + t.src + e;
    if (n == 4 && !(t.layer & kGradUnaligned)) {
      st_v4(d, g);
    } else {
      const float gs[4] = {g.x, g.y, g.z, g.w};
      for (uint32_t j = 0; j < n; ++j) d[j] = gs[j];
    }
  }
}

// CTA-index barrier across ranks on barrier plane `plane`.
__device__ __forceinline__ void rank_barrier(const RankView& v, int P, int plane, uint32_t epoch) {
  __syncthreads();
  if (threadIdx.x < P) {
    const int q = threadIdx.x;
    const uint32_t slot = plane * kSignalPlane + blockIdx.x * kMaxRanks;
    st_release_sys(v.signal[q] + slot + v.rank, epoch);
    const uint32_t* mine = v.signal[v.rank] + slot + q;
    if (static_cast<int32_t>(ld_acquire_sys(mine) - epoch) < 0) {
      const uint64_t t0 = globaltimer_ns();
      while (static_cast<int32_t>(ld_acquire_sys(mine) - epoch) < 0) {
        if (globaltimer_ns() - t0 > kBarrierTimeoutNs) {
          atomicExch(v.state + 2, 1u);
          break;
        }
      }
    }
  }
  __syncthreads();
}

// Last CTA of this rank bumps the launch counter (epoch + parity source).
__device__ __forceinline__ void finish_launch(const RankView& v, uint32_t seq) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const uint32_t prev = atomicAdd(v.state + 1, 1u);
    if (prev == gridDim.x - 1) {
      atomicExch(v.state + 1, 0u);
      __threadfence();
      atomicExch(v.state, seq + 1);
    }
  }
}

template <int P>
__device__ __forceinline__ void reduce_tile_rank_order(const RankView& v, const Tile& t,
                                                       uint64_t copy_off, float4 (&acc)[kVecPerThread],
                                                       bool (&live)[kVecPerThread]) {
  float4 x[kVecPerThread][P];
  const uint32_t nvec = (t.len + 3) >> 2;
#pragma unroll
  for (uint32_t k = 0; k < kVecPerThread; ++k) {
    const uint32_t i = threadIdx.x + k * kThreads;
    live[k] = i < nvec;
    if (live[k]) {
#pragma unroll
      for (int q = 0; q < P; ++q) x[k][q] = ld_cg_v4(v.arena[q] + copy_off + t.moff + i * 4);
    }
  }
#pragma unroll
  for (uint32_t k = 0; k < kVecPerThread; ++k) {
    if (live[k]) {
      float4 s = x[k][0];
#pragma unroll
      for (int q = 1; q < P; ++q) s = add4(s, x[k][q]);
      acc[k] = s;
    }
  }
}

template <int P, bool TWO_SHOT, bool LOOPBACK>
__global__ void __launch_bounds__(kThreads) group_allreduce_kernel(const GroupLaunch L) {
  const RankView& v = L.views[LOOPBACK ? blockIdx.y : 0];
  __shared__ uint32_t s_seq;
  if (threadIdx.x == 0) s_seq = ld_volatile_u32(v.state);
  __syncthreads();
  const uint32_t seq = s_seq;
  const uint32_t epoch = seq + 1;
  const uint64_t copy_off = static_cast<uint64_t>(seq & 1u) * L.copy_stride;
  const Tile* tiles = L.tiles;
  const uint32_t n_tiles = L.n_tiles;

  if constexpr (P == 1) {
    // Single rank: no exchange. grad x 1/P (= 1) straight into the epilogue.
    for (uint32_t ti = blockIdx.x; ti < n_tiles; ti += gridDim.x) {
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
        epilogue(t, e, mul4(x, L.scale), w, g, L.lr, L.epilogue);
      }
    }
  } else if constexpr (!TWO_SHOT) {
    float* mine = v.arena[v.rank] + copy_off;
    for (uint32_t ti = blockIdx.x; ti < n_tiles; ti += gridDim.x) {
      pack_tile(tiles[ti], v.grads, mine, L.scale);
    }
    rank_barrier(v, P, 0, epoch);
    for (uint32_t ti = blockIdx.x; ti < n_tiles; ti += gridDim.x) {
      const Tile t = tiles[ti];
      float4 acc[kVecPerThread];
      bool live[kVecPerThread];
      reduce_tile_rank_order<P>(v, t, copy_off, acc, live);
      const uint32_t layer = t.layer & kLayerMask;
      float* w = v.weights[layer];
      float* g = v.grads[layer];
#pragma unroll
      for (uint32_t k = 0; k < kVecPerThread; ++k) {
        if (live[k]) epilogue(t, (threadIdx.x + k * kThreads) * 4, acc[k], w, g, L.lr, L.epilogue);
      }
    }
  } else {
    // Tiles are dealt to owners round-robin: super-tile s = tiles [s*P, s*P+P).
    const uint32_t n_super = (n_tiles + P - 1) / P;
    float* mine = v.arena[v.rank] + copy_off;
    for (uint32_t s = blockIdx.x; s < n_super; s += gridDim.x) {
#pragma unroll
      for (int q = 0; q < P; ++q) {
        const uint32_t ti = s * P + q;
        if (ti < n_tiles) pack_tile(tiles[ti], v.grads, mine, L.scale);
      }
    }
    rank_barrier(v, P, 0, epoch);
    // Reduce-scatter: this rank's tile of every super-tile, reduced in place.
    for (uint32_t s = blockIdx.x; s < n_super; s += gridDim.x) {
      const uint32_t ti = s * P + v.rank;
      if (ti >= n_tiles) continue;
      const Tile t = tiles[ti];
      float4 acc[kVecPerThread];
      bool live[kVecPerThread];
      reduce_tile_rank_order<P>(v, t, copy_off, acc, live);
      const uint32_t layer = t.layer & kLayerMask;
      float* w = v.weights[layer];
      float* g = v.grads[layer];
#pragma unroll
      for (uint32_t k = 0; k < kVecPerThread; ++k) {
        if (live[k]) {
          const uint32_t e = (threadIdx.x + k * kThreads) * 4;
          st_v4(mine + t.moff + e, acc[k]);
          epilogue(t, e, acc[k], w, g, L.lr, L.epilogue);
        }
      }
    }
    rank_barrier(v, P, 1, epoch);
    // All-gather fused with unpack + SGD: pull every other owner's tile.
    for (uint32_t s = blockIdx.x; s < n_super; s += gridDim.x) {
      float4 x[P][kVecPerThread];
#pragma unroll
      for (int q = 0; q < P; ++q) {
        const uint32_t ti = s * P + q;
        if (q == v.rank || ti >= n_tiles) continue;
        const Tile t = tiles[ti];
        const uint32_t nvec = (t.len + 3) >> 2;
#pragma unroll
        for (uint32_t k = 0; k < kVecPerThread; ++k) {
          const uint32_t i = threadIdx.x + k * kThreads;
          if (i < nvec) x[q][k] = ld_cg_v4(v.arena[q] + copy_off + t.moff + i * 4);
        }
      }
#pragma unroll
      for (int q = 0; q < P; ++q) {
        const uint32_t ti = s * P + q;
        if (q == v.rank || ti >= n_tiles) continue;
        const Tile t = tiles[ti];
        const uint32_t layer = t.layer & kLayerMask;
        const uint32_t nvec = (t.len + 3) >> 2;
        float* w = v.weights[layer];
        float* g = v.grads[layer];
#pragma unroll
        for (uint32_t k = 0; k < kVecPerThread; ++k) {
          const uint32_t i = threadIdx.x + k * kThreads;
          if (i < nvec) epilogue(t, i * 4, x[q][k], w, g, L.lr, L.epilogue);
        }
      }
    }
  }
  finish_launch(v, seq);
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

// clock[0]: iteration start (written by the first replay kernel of an
// iteration), clock[1]: completion time of the latest replay kernel.
__global__ void replay_kernel(unsigned long long* clock, unsigned long long deadline_ns,
                              int first) {
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

}  // namespace

cudaError_t launch_group_allreduce(const GroupLaunch& L, int ctas_per_rank, bool two_shot,
                                   bool loopback, cudaStream_t stream) {
  const dim3 grid(ctas_per_rank, loopback ? L.nranks : 1);
  return loopback ? launch_lb<true>(L, grid, two_shot, stream)
                  : launch_lb<false>(L, grid, two_shot, stream);
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
                          cudaStream_t stream) {
  replay_kernel<<<1, 32, 0, stream>>>(clock, deadline_ns, first);
  return cudaGetLastError();
}

}  // namespace mgw
