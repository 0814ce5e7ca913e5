// mgwfbp-b200: NVLS multicast buffer management (see nvls.hpp).
//
// Driver entry points are fetched with cudaGetDriverEntryPoint (the library
// does not link libcuda directly). The multicast object is shared as a POSIX
// file descriptor: rank 0 exports it, the peers duplicate it out of rank 0's
// process with pidfd_open + pidfd_getfd (same host, same user) and import it.
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cstring>
#include <string>

#include <cuda.h>
#include <cuda_runtime.h>

#include "capi_common.hpp"
#include "nvls.hpp"

namespace mgw {

namespace {

struct Driver {
  decltype(&cuDeviceGet) dev_get = nullptr;
  decltype(&cuDeviceGetAttribute) dev_attr = nullptr;
  decltype(&cuMulticastGetGranularity) mc_gran = nullptr;
  decltype(&cuMulticastCreate) mc_create = nullptr;
  decltype(&cuMulticastAddDevice) mc_add = nullptr;
  decltype(&cuMulticastBindMem) mc_bind = nullptr;
  decltype(&cuMulticastUnbind) mc_unbind = nullptr;
  decltype(&cuMemCreate) mem_create = nullptr;
  decltype(&cuMemRelease) mem_release = nullptr;
  decltype(&cuMemAddressReserve) va_reserve = nullptr;
  decltype(&cuMemAddressFree) va_free = nullptr;
  decltype(&cuMemMap) map = nullptr;
  decltype(&cuMemUnmap) unmap = nullptr;
  decltype(&cuMemSetAccess) set_access = nullptr;
  decltype(&cuMemGetAllocationGranularity) alloc_gran = nullptr;
  decltype(&cuMemExportToShareableHandle) export_handle = nullptr;
  decltype(&cuMemImportFromShareableHandle) import_handle = nullptr;
  bool ok = false;
};

template <typename F>
bool entry(const char* name, F& fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess ||
      p == nullptr) {
    cudaGetLastError();
    return false;
  }
  fn = reinterpret_cast<F>(p);
  return true;
}

const Driver& drv() {
  static const Driver d = [] {
    Driver x;
    x.ok = entry("cuDeviceGet", x.dev_get) && entry("cuDeviceGetAttribute", x.dev_attr) && entry("cuMulticastGetGranularity", x.mc_gran) &&
           entry("cuMulticastCreate", x.mc_create) && entry("cuMulticastAddDevice", x.mc_add) &&
           entry("cuMulticastBindMem", x.mc_bind) && entry("cuMulticastUnbind", x.mc_unbind) &&
           entry("cuMemCreate", x.mem_create) && entry("cuMemRelease", x.mem_release) &&
           entry("cuMemAddressReserve", x.va_reserve) && entry("cuMemAddressFree", x.va_free) &&
           entry("cuMemMap", x.map) && entry("cuMemUnmap", x.unmap) && entry("cuMemSetAccess", x.set_access) &&
           entry("cuMemGetAllocationGranularity", x.alloc_gran) &&
           entry("cuMemExportToShareableHandle", x.export_handle) &&
           entry("cuMemImportFromShareableHandle", x.import_handle);
    return x;
  }();
  return d;
}

void cu(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) throw CudaFailure(std::string("NVLS ") + what + ": CUresult " + std::to_string(r));
}

// What rank 0 exports (kNvlsBlobBytes, plain data).
struct Blob {
  uint32_t magic;
  int32_t pid;
  int32_t fd;
  int32_t nranks;
  uint64_t bytes;  // multicast object size
  uint8_t pad[kNvlsBlobBytes - 24];
};
static_assert(sizeof(Blob) == kNvlsBlobBytes, "blob size");
constexpr uint32_t kMagic = 0x534c564eu;  // "NVLS"

}  // namespace

struct NvlsArena {
  int device = 0;
  int rank = 0;
  int nranks = 1;
  size_t bytes = 0;       // multicast object / each local buffer
  size_t gran = 0;
  CUmemGenericAllocationHandle mc = 0;
  bool have_mc = false;
  bool added = false;
  int export_fd = -1;     // rank 0: kept open until destroy (the peers duplicate it)
  CUmemGenericAllocationHandle phys = 0;
  bool have_phys = false;
  bool bound = false;
  CUdeviceptr uc = 0, mcp = 0;
  bool uc_mapped = false, mc_mapped = false;
};

bool nvls_supported(int device) {
  const Driver& d = drv();
  if (!d.ok) return false;
  int v = 0;
  CUdevice dev = 0;
  if (d.dev_get(&dev, device) != CUDA_SUCCESS) return false;
  if (d.dev_attr(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev) != CUDA_SUCCESS) return false;
  return v != 0;
}

NvlsArena* nvls_create(int device, int rank, int nranks, size_t bytes, void* blob_out) {
  const Driver& d = drv();
  if (!d.ok) throw CudaFailure("NVLS: driver entry points unavailable");
  if (!nvls_supported(device)) throw CudaFailure("NVLS: multicast objects are not supported on this device");
  auto* a = new NvlsArena();
  try {
    a->device = device;
    a->rank = rank;
    a->nranks = nranks;
    CUmulticastObjectProp mp{};
    mp.numDevices = static_cast<unsigned>(nranks);
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    mp.size = bytes;
    // sizes and offsets at the RECOMMENDED multicast granularity (512 MiB on
    // B200) — what tools/nvls_probe.cu binds successfully
    cu(d.mc_gran(&a->gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED), "multicast granularity");
    size_t ag = 0;
    CUmemAllocationProp ap{};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = device;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    cu(d.alloc_gran(&ag, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "allocation granularity");
    a->gran = std::max(a->gran, ag);
    a->bytes = (std::max<size_t>(bytes, 1) + a->gran - 1) / a->gran * a->gran;
    Blob b{};
    if (rank == 0) {
      mp.size = a->bytes;
      cu(d.mc_create(&a->mc, &mp), "cuMulticastCreate");
      a->have_mc = true;
      int fd = -1;
      cu(d.export_handle(&fd, a->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0), "export");
      a->export_fd = fd;
      b.magic = kMagic;
      b.pid = static_cast<int32_t>(getpid());
      b.fd = fd;
      b.nranks = nranks;
      b.bytes = a->bytes;
    }
    std::memcpy(blob_out, &b, sizeof b);
    return a;
  } catch (...) {
    nvls_destroy(a);
    throw;
  }
}

void nvls_join(NvlsArena* a, const void* blob0) {
  const Driver& d = drv();
  Blob b;
  std::memcpy(&b, blob0, sizeof b);
  if (b.magic != kMagic || b.nranks != a->nranks) throw CudaFailure("NVLS: bad handle from rank 0");
  if (a->rank != 0) {
    a->bytes = b.bytes;
    const int pidfd = static_cast<int>(syscall(SYS_pidfd_open, b.pid, 0));
    if (pidfd < 0) throw CudaFailure("NVLS: pidfd_open(rank 0) failed: errno " + std::to_string(errno));
    const int fd = static_cast<int>(syscall(SYS_pidfd_getfd, pidfd, b.fd, 0));
    close(pidfd);
    if (fd < 0) throw CudaFailure("NVLS: pidfd_getfd failed: errno " + std::to_string(errno));
    const CUresult r = d.import_handle(&a->mc, reinterpret_cast<void*>(static_cast<uintptr_t>(fd)),
                                       CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
    close(fd);
    cu(r, "import");
    a->have_mc = true;
  }
  CUdevice dev = 0;
  cu(d.dev_get(&dev, a->device), "cuDeviceGet");
  cu(d.mc_add(a->mc, dev), "cuMulticastAddDevice");
  a->added = true;
}

void nvls_bind(NvlsArena* a) {
  const Driver& d = drv();
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = a->device;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;  // as the multicast object's
  cu(d.mem_create(&a->phys, a->bytes, &ap, 0), "cuMemCreate");
  a->have_phys = true;
  cu(d.mc_bind(a->mc, 0, a->phys, 0, a->bytes, 0), "cuMulticastBindMem");
  a->bound = true;
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = a->device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  cu(d.va_reserve(&a->uc, a->bytes, a->gran, 0, 0), "reserve");
  cu(d.map(a->uc, a->bytes, 0, a->phys, 0), "map");
  a->uc_mapped = true;
  cu(d.set_access(a->uc, a->bytes, &acc, 1), "access");
  cu(d.va_reserve(&a->mcp, a->bytes, a->gran, 0, 0), "reserve (multicast)");
  cu(d.map(a->mcp, a->bytes, 0, a->mc, 0), "map (multicast)");
  a->mc_mapped = true;
  cu(d.set_access(a->mcp, a->bytes, &acc, 1), "access (multicast)");
  if (cudaMemset(reinterpret_cast<void*>(a->uc), 0, a->bytes) != cudaSuccess ||
      cudaDeviceSynchronize() != cudaSuccess) {
    throw CudaFailure("NVLS: clearing the buffer failed");
  }
}

float* nvls_uc(const NvlsArena* a) { return reinterpret_cast<float*>(a->uc); }
float* nvls_mc(const NvlsArena* a) { return reinterpret_cast<float*>(a->mcp); }
size_t nvls_bytes(const NvlsArena* a) { return a->bytes; }

void nvls_destroy(NvlsArena* a) {
  if (a == nullptr) return;
  const Driver& d = drv();
  if (d.ok) {
    if (a->mc_mapped) d.unmap(a->mcp, a->bytes);
    if (a->mcp) d.va_free(a->mcp, a->bytes);
    if (a->uc_mapped) d.unmap(a->uc, a->bytes);
    if (a->uc) d.va_free(a->uc, a->bytes);
    CUdevice dev = 0;
    if (a->bound && d.dev_get(&dev, a->device) == CUDA_SUCCESS) d.mc_unbind(a->mc, dev, 0, a->bytes);
    if (a->have_phys) d.mem_release(a->phys);
    if (a->have_mc) d.mem_release(a->mc);
  }
  if (a->export_fd >= 0) close(a->export_fd);
  delete a;
}

}  // namespace mgw
