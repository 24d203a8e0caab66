// internal.hpp — shared host-side definitions of libgh (not part of the ABI).
#pragma once
#include <string>

#include "gh/gh.h"

namespace gh {

// thread-local last-error message (gh_last_error)
void set_error(const std::string& msg);
inline gh_status fail(gh_status s, const std::string& msg) {
  set_error(msg);
  return s;
}

}  // namespace gh

#define GH_CUDA(call)                                                                      \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return ::gh::fail(GH_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));     \
  } while (0)

#define GH_TRY(call)                       \
  do {                                     \
    gh_status s_ = (call);                 \
    if (s_ != GH_OK) return s_;            \
  } while (0)
