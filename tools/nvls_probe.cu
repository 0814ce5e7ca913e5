// NVLS (NVLink SHARP / multicast) micro-probe (tools only, one process, every
// visible GPU): does this pool support multicast objects, and what does a
// switch-reduced all-reduce reach?
//
//   buffer: cuMemCreate on every GPU, bound to one multicast object
//   kernel: per CTA an entry barrier (multimem.red on a flag word, local
//           acquire poll), then for the rank's shard
//           multimem.ld_reduce.add.v4.f32 (the switch sums the P copies) ->
//           multimem.st.v4.f32 (the switch writes the sum to all P copies),
//           then an exit barrier.
//   bus GB/s = 2(P-1)/P * S / t (the NCCL busbw convention).
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvls_probe tools/nvls_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

#define CU(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s_ = nullptr; cuGetErrorString(r_, &s_); \
  std::printf("CU error %d (%s) at %s:%d: %s\n", (int)r_, s_ ? s_ : "?", __FILE__, __LINE__, #x); return 1; } } while (0)
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

__device__ __forceinline__ void mc_red_add(uint32_t* mc, uint32_t v) {
  asm volatile("multimem.red.release.sys.global.add.u32 [%0], %1;" ::"l"(mc), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void cta_barrier(uint32_t* flag_mc, uint32_t* flag_uc, uint32_t target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    mc_red_add(flag_mc, 1u);
    for (uint64_t spin = 0; ld_acquire(flag_uc) < target; ++spin) {
      if (spin > (1ull << 24)) { printf("barrier timeout cta %d\n", blockIdx.x); asm volatile("trap;"); }
    }
  }
  __syncthreads();
}

// data_mc: multicast view of the buffer; flags: [2 * gridDim.x] words
__global__ void __launch_bounds__(512) nvls_allreduce(float* data_mc, size_t n_vec, int rank, int nranks,
                                                      uint32_t* flags_mc, uint32_t* flags_uc, uint32_t epoch,
                                                      int unroll, int iters, size_t out_off_vec) {
 for (int it = 0; it < iters; ++it) {
  const uint32_t target = (epoch + it) * static_cast<uint32_t>(nranks);
  cta_barrier(flags_mc + 2 * blockIdx.x, flags_uc + 2 * blockIdx.x, target);
  const size_t shard = n_vec / nranks;
  const size_t lo = shard * rank;
  const size_t hi = rank == nranks - 1 ? n_vec : lo + shard;
  float4* base = reinterpret_cast<float4*>(data_mc);
  float4* out = base + (out_off_vec ? out_off_vec : 0);  // out-of-place when timing (values do not grow)
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  size_t i = lo + static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (unroll == 4) {
    for (; i + 3 * stride < hi; i += 4 * stride) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(v[u].x), "=f"(v[u].y), "=f"(v[u].z), "=f"(v[u].w)
                     : "l"(base + i + u * stride) : "memory");
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(out + i + u * stride),
                     "f"(v[u].x), "f"(v[u].y), "f"(v[u].z), "f"(v[u].w) : "memory");
      }
    }
  }
  for (; i < hi; i += stride) {
    float4 v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(base + i) : "memory");
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(out + i), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w) : "memory");
  }
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  cta_barrier(flags_mc + 2 * blockIdx.x + 1, flags_uc + 2 * blockIdx.x + 1, target);
 }
}

__global__ void fill(float* p, size_t n, float base) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = __fadd_rn(base, __fmul_rn(static_cast<float>((i * 7919u) % 977u), 0.00123f));
}

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  CU(cuInit(0));
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  const int P = argc > 1 ? std::atoi(argv[1]) : ndev;
  if (P < 2 || P > ndev) { std::printf("need 2..%d GPUs\n", ndev); return 1; }
  for (int d = 0; d < P; ++d) {
    CUdevice dev; CU(cuDeviceGet(&dev, d));
    int mc = 0, fab = 0;
    CU(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
    cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
    std::printf("dev %d: MULTICAST_SUPPORTED=%d FABRIC_HANDLE=%d\n", d, mc, fab);
    if (!mc) { std::printf("NVLS: multicast unsupported on this pool\n"); return 0; }
  }
  const size_t max_bytes = static_cast<size_t>(1) << 30;
  const int nblk_max = 1024;
  CUmulticastObjectProp mp{};
  mp.numDevices = static_cast<unsigned>(P);
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  mp.size = max_bytes;
  CU(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  const size_t flag_bytes = ((2 * nblk_max * 4 + gran - 1) / gran) * gran;
  const size_t total = ((max_bytes + gran - 1) / gran) * gran + flag_bytes;
  mp.size = total;
  std::printf("multicast granularity %zu, object %zu bytes\n", gran, total);
  CUmemGenericAllocationHandle mch;
  CU(cuMulticastCreate(&mch, &mp));
  for (int d = 0; d < P; ++d) {
    CUdevice dev; CU(cuDeviceGet(&dev, d));
    CU(cuMulticastAddDevice(mch, dev));
  }
  std::vector<CUdeviceptr> uc(P), mcp(P);
  std::vector<CUcontext> ctx(P);
  for (int d = 0; d < P; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaFree(nullptr));
    CU(cuCtxGetCurrent(&ctx[d]));
    CUmemAllocationProp ap{};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = d;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    CUmemGenericAllocationHandle ph;
    CU(cuMemCreate(&ph, total, &ap, 0));
    CU(cuMulticastBindMem(mch, 0, ph, 0, total, 0));
    CUmemAccessDesc acc{};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = d;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CU(cuMemAddressReserve(&uc[d], total, gran, 0, 0));
    CU(cuMemMap(uc[d], total, 0, ph, 0));
    CU(cuMemSetAccess(uc[d], total, &acc, 1));
    CU(cuMemAddressReserve(&mcp[d], total, gran, 0, 0));
    CU(cuMemMap(mcp[d], total, 0, mch, 0));
    CU(cuMemSetAccess(mcp[d], total, &acc, 1));
    CK(cudaMemset(reinterpret_cast<void*>(uc[d] + total - flag_bytes), 0, flag_bytes));
  }
  for (int d = 0; d < P; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
  uint32_t epoch = 0;
  // correctness at 4 MiB: rank r holds base r+1
  {
    const size_t n = (4u << 20) / 4;
    for (int d = 0; d < P; ++d) {
      CK(cudaSetDevice(d));
      fill<<<148, 512>>>(reinterpret_cast<float*>(uc[d]), n, static_cast<float>(d + 1));
    }
    for (int d = 0; d < P; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
    std::vector<std::vector<float>> in(P, std::vector<float>(n));
    for (int d = 0; d < P; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaMemcpy(in[d].data(), reinterpret_cast<void*>(uc[d]), n * 4, cudaMemcpyDeviceToHost));
    }
    ++epoch;
    for (int d = 0; d < P; ++d) {
      CK(cudaSetDevice(d));
      nvls_allreduce<<<148, 512>>>(reinterpret_cast<float*>(mcp[d]), n / 4, d, P,
                                   reinterpret_cast<uint32_t*>(mcp[d] + total - flag_bytes),
                                   reinterpret_cast<uint32_t*>(uc[d] + total - flag_bytes), epoch, 4, 1, 0);
      CK(cudaGetLastError());
    }
    for (int d = 0; d < P; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
    std::vector<float> h(n);
    size_t bad = 0, bad_exact = 0, bad_once = 0;
    for (int d = 0; d < P; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaMemcpy(h.data(), reinterpret_cast<void*>(uc[d]), n * 4, cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < n; ++i) {
        float ref = in[0][i];  // rank order
        for (int r = 1; r < P; ++r) ref += in[r][i];
        double exact = 0.0;  // the exact sum (rounded once)
        for (int r = 0; r < P; ++r) exact += in[r][i];
        if (std::abs(h[i] - ref) > 1e-5f * std::abs(ref)) ++bad;
        if (h[i] != ref) ++bad_exact;
        if (h[i] != static_cast<float>(exact)) ++bad_once;
      }
    }
    std::printf("correctness P=%d (%zu elements x %d GPUs): %zu off 1e-5 rel, %zu != rank-order fp32 sum, "
                "%zu != correctly rounded exact sum\n", P, n, P, bad, bad_exact, bad_once);
  }
  const size_t sizes[] = {4u << 10, 16u << 10, 64u << 10, 256u << 10, 1u << 20, 4u << 20, 16u << 20, 64u << 20, 128u << 20, 256u << 20, 512u << 20};
  const int blocks_list[] = {16, 32, 64, 148};
  std::vector<cudaEvent_t> e0(P), e1(P);
  for (int d = 0; d < P; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
  }
  for (int nb : blocks_list) {
    // every CTA index restarts at epoch 0 (a CTA count change would leave flags behind)
    for (int d = 0; d < P; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaMemset(reinterpret_cast<void*>(uc[d] + total - flag_bytes), 0, flag_bytes));
    }
    for (int d = 0; d < P; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
    epoch = 0;
    for (size_t bytes : sizes) {
      const size_t nvec = bytes / 16;
      const int reps = bytes >= (256u << 20) ? 10 : 50;
      float best = 1e30f;
      for (int trial = 0; trial < 3; ++trial) {
        for (int d = 0; d < P; ++d) {
          CK(cudaSetDevice(d));
          CK(cudaEventRecord(e0[d]));
        }
        // one launch of `reps` back-to-back all-reduces (host launch cost excluded)
        for (int d = 0; d < P; ++d) {
          CK(cudaSetDevice(d));
          nvls_allreduce<<<nb, 512>>>(reinterpret_cast<float*>(mcp[d]), nvec, d, P,
                                      reinterpret_cast<uint32_t*>(mcp[d] + total - flag_bytes),
                                      reinterpret_cast<uint32_t*>(uc[d] + total - flag_bytes), epoch + 1, 4, reps, (max_bytes / 2) / 16);
        }
        epoch += reps;
        float worst = 0.f;
        for (int d = 0; d < P; ++d) {
          CK(cudaSetDevice(d));
          CK(cudaEventRecord(e1[d]));
        }
        for (int d = 0; d < P; ++d) {
          CK(cudaSetDevice(d));
          CK(cudaEventSynchronize(e1[d]));
          float ms = 0.f;
          CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
          worst = std::max(worst, ms);
        }
        best = std::min(best, worst / reps);
      }
      const double bus = 2.0 * (P - 1) / P * static_cast<double>(bytes) / (best * 1e-3) / 1e9;
      std::printf("P=%d ctas=%d size=%zu KiB: %.2f us  bus %.1f GB/s (%.3f of 900)\n", P, nb, bytes >> 10,
                  best * 1e3, bus, bus / 900.0);
    }
  }
  return 0;
}
