// mgwfbp-b200: shared C-ABI plumbing (status mapping, CUDA error type).
#ifndef MGWFBP_CAPI_COMMON_HPP_
#define MGWFBP_CAPI_COMMON_HPP_

#include <stdexcept>
#include <string>

namespace mgw {

// A failed CUDA runtime call; mapped to MGW_ERR_CUDA at the ABI.
class CudaFailure : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

void set_error(const std::string& msg);
// Call from inside a catch block: records the message, returns the status.
int status_from_current_exception();

}  // namespace mgw

#define MGW_TRY try
#define MGW_CATCH                                \
  catch (...) {                                  \
    return mgw::status_from_current_exception(); \
  }                                              \
  return 0;

#endif  // MGWFBP_CAPI_COMMON_HPP_
