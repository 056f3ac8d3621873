// Error plumbing shared by the extern "C" entry points.
#pragma once
#include <cstdarg>
#include <cstdio>
#include <string>

#include <cuda_runtime.h>

#include "singa_b200.h"

namespace sg {

void set_error(const char* fmt, ...);
const char* get_error();

#define SG_FAIL(code, ...)       \
  do {                           \
    ::sg::set_error(__VA_ARGS__); \
    return (code);               \
  } while (0)

#define SG_CUDA(expr)                                                                                  \
  do {                                                                                                 \
    cudaError_t _e = (expr);                                                                           \
    if (_e != cudaSuccess) SG_FAIL(SG_ERR_CUDA, "CUDA error %s at %s:%d (%s)", cudaGetErrorString(_e), \
                                   __FILE__, __LINE__, #expr);                                         \
  } while (0)

#define SG_CHECK(cond, code, ...) \
  do {                            \
    if (!(cond)) SG_FAIL(code, __VA_ARGS__); \
  } while (0)

#define SG_TRY(expr)             \
  do {                           \
    sg_status _s = (expr);       \
    if (_s != SG_OK) return _s;  \
  } while (0)

}  // namespace sg
