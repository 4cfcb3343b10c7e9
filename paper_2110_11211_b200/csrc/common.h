// Shared helpers: status/error plumbing and CUDA checks.
#pragma once
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "../../include/sfcdd_b200.h"

namespace sfcdd {

// Exceptions carry the C-ABI status they map to.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);

#define SFCDD_REQUIRE(cond, code, msg)                                    \
  do {                                                                    \
    if (!(cond)) throw ::sfcdd::Error((code), (msg));                     \
  } while (0)

}  // namespace sfcdd

#ifdef __CUDACC__
#include <cuda_runtime.h>
#define CUDA_CHECK(expr)                                                          \
  do {                                                                            \
    cudaError_t _e = (expr);                                                      \
    if (_e != cudaSuccess)                                                        \
      throw ::sfcdd::Error(SFCDD_ECUDA, std::string(#expr) + ": " +               \
                                            cudaGetErrorString(_e) + " at " +     \
                                            __FILE__ + ":" + std::to_string(__LINE__)); \
  } while (0)
#endif

// Wrap a C-ABI body: translate exceptions into status codes.
#define SFCDD_API_BEGIN try {
#define SFCDD_API_END                                                     \
  return SFCDD_OK;                                                        \
  }                                                                       \
  catch (const ::sfcdd::Error& e) {                                       \
    ::sfcdd::set_last_error(e.what());                                    \
    return e.code;                                                        \
  }                                                                       \
  catch (const std::bad_alloc&) {                                         \
    ::sfcdd::set_last_error("host out of memory");                        \
    return SFCDD_EINTERNAL;                                               \
  }                                                                       \
  catch (const std::exception& e) {                                       \
    ::sfcdd::set_last_error(e.what());                                    \
    return SFCDD_EINTERNAL;                                               \
  }
