// NVLink egress micro-probe (tools only): GPU 0 writes a 256 MiB buffer into
// GPU 1 (peer access, one process) with
//   (a) SM stores, 16-byte per thread (st.global.v4),
//   (b) SM stores, 32-byte per thread (two v4 to adjacent addresses),
//   (c) TMA bulk copies smem -> peer global (cp.async.bulk), 16 KiB chunks,
// for several CTA counts, and cudaMemcpyPeerAsync as the copy-engine
// reference. Prints GB/s.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvlink_probe tools/nvlink_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

__global__ void st16(float4* dst, size_t n_vec, float v) {
  const float4 x = make_float4(v, v, v, v);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n_vec; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = x;
}

__global__ void st32(float4* dst, size_t n_vec, float v) {
  const float4 x = make_float4(v, v, v, v);
  for (size_t i = 2 * (blockIdx.x * (size_t)blockDim.x + threadIdx.x); i + 1 < n_vec;
       i += 2 * (size_t)gridDim.x * blockDim.x) {
    dst[i] = x;
    dst[i + 1] = x;
  }
}

// Each CTA: fill a 16 KiB smem chunk once, then bulk-copy it to successive
// destination chunks, keeping up to 8 bulk groups in flight.
__global__ void tma_bulk(char* dst, size_t bytes, float v) {
  constexpr int kChunk = 16384;
  __shared__ __align__(128) float buf[kChunk / 4];
  for (int i = threadIdx.x; i < kChunk / 4; i += blockDim.x) buf[i] = v;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(buf);
    int inflight = 0;
    for (size_t off = (size_t)blockIdx.x * kChunk; off + kChunk <= bytes; off += (size_t)gridDim.x * kChunk) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + off), "r"(s),
                   "n"(kChunk) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      if (++inflight >= 8) {
        asm volatile("cp.async.bulk.wait_group.read 7;" ::: "memory");
      }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

// local -> remote copy, 4 float4 per thread per step (loads batched before
// stores); optionally a system fence + __syncthreads every `fence_every`
// steps (what a barrier per chunk costs).
__global__ void copy_batched(const float4* __restrict__ src, float4* dst, size_t n_vec, int fence_every) {
  const size_t stride = (size_t)gridDim.x * blockDim.x * 4;
  int step = 0;
  for (size_t base = (size_t)blockIdx.x * blockDim.x * 4 + threadIdx.x; base < n_vec; base += stride) {
    float4 x[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const size_t i = base + (size_t)k * blockDim.x;
      if (i < n_vec) x[k] = __ldg(src + i);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const size_t i = base + (size_t)k * blockDim.x;
      if (i < n_vec) dst[i] = x[k];
    }
    if (fence_every > 0 && ++step % fence_every == 0) {
      __threadfence_system();
      __syncthreads();
    }
  }
}

// TMA copy: global -> smem (cp.async.bulk + mbarrier) -> peer global
// (cp.async.bulk bulk_group). One elected thread per CTA drives kStages
// 16 KiB stages; no register traffic at all.
__global__ void tma_copy(const char* src, char* dst, size_t bytes) {
  constexpr int kChunk = 16384, kStages = 8;
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) unsigned long long bar[kStages];
  if (threadIdx.x != 0) return;
  const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(sm);
  for (int i = 0; i < kStages; ++i) {
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[i]);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint32_t phase[kStages] = {};
  const size_t step = (size_t)gridDim.x * kChunk;
  size_t off0 = (size_t)blockIdx.x * kChunk;
  int k = 0;
  // prologue: fill stages
  size_t next_load = off0;
  for (int i = 0; i < kStages && next_load + kChunk <= bytes; ++i, next_load += step) {
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[i]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "n"(kChunk) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s0 + i * kChunk),
                 "l"(src + next_load), "n"(kChunk), "r"(b) : "memory");
  }
  for (size_t off = off0; off + kChunk <= bytes; off += step, k = (k + 1) % kStages) {
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[k]);
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(b), "r"(phase[k]) : "memory");
    phase[k] ^= 1;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + off), "r"(s0 + k * kChunk), "n"(kChunk) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (next_load + kChunk <= bytes) {
      // reuse stage k once its store has read smem
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "n"(kChunk) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s0 + k * kChunk),
                   "l"(src + next_load), "n"(kChunk), "r"(b) : "memory");
      next_load += step;
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) { std::printf("need 2 GPUs\n"); return 0; }
  const size_t bytes = 256ull << 20;
  float *src = nullptr, *dst = nullptr;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&dst, bytes));
  CK(cudaSetDevice(0));
  CK(cudaMalloc(&src, bytes));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto timeit = [&](auto launch) -> double {
    for (int w = 0; w < 2; ++w) launch();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    return bytes * 5 / (ms * 1e-3) / 1e9;
  };
  std::printf("copy engine cudaMemcpyPeerAsync: %.1f GB/s\n",
              timeit([&] { cudaMemcpyPeerAsync(dst, 1, src, 0, bytes); }));
  for (int ctas : {16, 32, 64, 140, 296}) {
    const double a = timeit([&] { st16<<<ctas, 512>>>((float4*)dst, bytes / 16, 1.0f); });
    const double b = timeit([&] { st32<<<ctas, 512>>>((float4*)dst, bytes / 16, 1.0f); });
    const double c = timeit([&] { tma_bulk<<<ctas, 128>>>((char*)dst, bytes, 1.0f); });
    std::printf("ctas=%3d  st16 %.1f  st32 %.1f  tma_bulk %.1f GB/s\n", ctas, a, b, c);
  }
  for (int ctas : {8, 16, 32, 140}) {
    const double d = timeit([&] { copy_batched<<<ctas, 512>>>((const float4*)src, (float4*)dst, bytes / 16, 0); });
    const double e = timeit([&] { copy_batched<<<ctas, 512>>>((const float4*)src, (float4*)dst, bytes / 16, 16); });
    const double f = timeit([&] { copy_batched<<<ctas, 512>>>((const float4*)src, (float4*)dst, bytes / 16, 2); });
    std::printf("ctas=%3d  copy(ld local, st peer) %.1f  +fence/256KiB %.1f  +fence/32KiB %.1f GB/s\n", ctas, d,
                e, f);
  }
  CK(cudaFuncSetAttribute(tma_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384));
  for (int ctas : {8, 16, 32, 64, 140}) {
    const double g = timeit([&] { tma_copy<<<ctas, 32, 8 * 16384>>>((const char*)src, (char*)dst, bytes); });
    std::printf("ctas=%3d  tma_copy(bulk ld local -> smem -> bulk st peer) %.1f GB/s\n", ctas, g);
  }
  // bidirectional: GPU0 -> GPU1 and GPU1 -> GPU0 at the same time
  float *src1 = nullptr, *dst0 = nullptr;
  CK(cudaMalloc(&dst0, bytes));
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&src1, bytes));
  CK(cudaDeviceEnablePeerAccess(0, 0));
  CK(cudaFuncSetAttribute(tma_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384));
  cudaStream_t s1;
  cudaEvent_t f0, f1;
  CK(cudaStreamCreate(&s1));
  CK(cudaEventCreate(&f0));
  CK(cudaEventCreate(&f1));
  CK(cudaSetDevice(0));
  for (int mode = 0; mode < 2; ++mode) {
    for (int ctas : {32, 64, 140}) {
      auto go = [&] {
        CK(cudaSetDevice(0));
        if (mode == 0) copy_batched<<<ctas, 512>>>((const float4*)src, (float4*)dst, bytes / 16, 0);
        else tma_copy<<<ctas, 32, 8 * 16384>>>((const char*)src, (char*)dst, bytes);
        CK(cudaSetDevice(1));
        if (mode == 0) copy_batched<<<ctas, 512, 0, s1>>>((const float4*)src1, (float4*)dst0, bytes / 16, 0);
        else tma_copy<<<ctas, 32, 8 * 16384, s1>>>((const char*)src1, (char*)dst0, bytes);
        CK(cudaSetDevice(0));
        return 0;
      };
      for (int w = 0; w < 2; ++w) go();
      CK(cudaDeviceSynchronize());
      CK(cudaSetDevice(1));
      CK(cudaDeviceSynchronize());
      CK(cudaSetDevice(0));
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) go();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      CK(cudaSetDevice(1));
      CK(cudaDeviceSynchronize());
      CK(cudaSetDevice(0));
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      std::printf("bidirectional %s ctas=%3d: GPU0->1 %.1f GB/s per direction (GPU0 clock)\n",
                  mode == 0 ? "copy_batched" : "tma_copy", ctas, bytes * 5 / (ms * 1e-3) / 1e9);
    }
  }
  CK(cudaGetLastError());
  return 0;
}
