// Library-level C ABI: error reporting and launch accounting.
#include <cstdarg>

#include "common.cuh"

namespace accel {

static thread_local std::string t_last_error;
std::atomic<unsigned long long> g_launches{0};

void set_error(const std::string& msg) { t_last_error = msg; }

int fail(int status, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  t_last_error = buf;
  return status;
}

}  // namespace accel

extern "C" const char* accel_last_error(void) { return accel::t_last_error.c_str(); }

extern "C" unsigned long long accel_launch_count(void) {
  return accel::g_launches.load(std::memory_order_relaxed);
}

extern "C" int accel_version(void) { return 4; }

#ifndef ACCEL_BUILD_ID
#define ACCEL_BUILD_ID "unknown"
#endif
// Hash of the sources and flags this library was built from (build.py):
// the Python loader refuses a library whose id does not match its sources.
extern "C" const char* accel_build_id(void) { return ACCEL_BUILD_ID; }

// One strided DMA (host <-> device or device <-> device): uploads row-major
// host arrays into pitched device storage (16-byte aligned rows for TMA).
extern "C" int accel_copy_2d(void* dst, size_t dpitch, const void* src, size_t spitch,
                             size_t width, size_t height, void* stream) {
  if (height == 0 || width == 0) return accel::kOk;
  if (!dst || !src || dpitch < width || spitch < width)
    return accel::fail(accel::kDimension, "copy_2d: bad arguments");
  return accel::check_cuda(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height,
                                             cudaMemcpyDefault, accel::as_stream(stream)),
                           "copy_2d");
}
