// mgwfbp-b200: NVLS (NVLink SHARP) buffer — one multicast object over the P
// ranks' GPUs with every rank's local buffer bound to it (nvls.cu). Host-only
// driver-API plumbing; the kernels that use it are in kernels.cu.
//
// Setup is three collective phases (the caller exchanges the blob and puts
// a barrier between join and bind — every device must be added to the
// multicast object before any rank binds memory to it):
//   nvls_create  rank 0 creates the multicast object and exports it (a POSIX
//                file descriptor, fetched by the peers with pidfd_getfd);
//   nvls_join    every other rank imports it; every rank adds its device;
//   nvls_bind    every rank allocates + binds its local buffer and maps the
//                unicast and multicast views.
#ifndef MGWFBP_NVLS_HPP_
#define MGWFBP_NVLS_HPP_

#include <cstddef>
#include <cstdint>

namespace mgw {

struct NvlsArena;

constexpr size_t kNvlsBlobBytes = 64;  // what nvls_create exports (rank 0's object)

bool nvls_supported(int device);
// bytes: usable buffer size (rounded up to the multicast granularity)
NvlsArena* nvls_create(int device, int rank, int nranks, size_t bytes, void* blob_out);
void nvls_join(NvlsArena* a, const void* blob0);
void nvls_bind(NvlsArena* a);
float* nvls_uc(const NvlsArena* a);   // this rank's copy (local HBM)
float* nvls_mc(const NvlsArena* a);   // the multicast address of the same bytes
size_t nvls_bytes(const NvlsArena* a);
void nvls_destroy(NvlsArena* a);

}  // namespace mgw

#endif  // MGWFBP_NVLS_HPP_
