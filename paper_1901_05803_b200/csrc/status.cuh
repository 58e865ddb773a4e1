// Thread-local error reporting for the C ABI (ralpb_last_error()).
#pragma once
#include <cuda_runtime.h>
#include <string>

namespace ralpb {

std::string& last_error_slot();

inline int set_status(cudaError_t e, const std::string& why) {
  if (e == cudaSuccess) return 0;
  std::string msg = why.empty() ? std::string(cudaGetErrorString(e))
                                : why + " (" + cudaGetErrorString(e) + ")";
  last_error_slot() = msg;
  return static_cast<int>(e) == 0 ? 1 : static_cast<int>(e);
}

inline int set_error(const std::string& why, int code = 1) {
  last_error_slot() = why;
  return code;
}

}  // namespace ralpb
