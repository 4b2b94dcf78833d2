// Error plumbing and device queries of the C-ABI (include/mpm.h).
#include <stdarg.h>
#include "common.cuh"

namespace mpm {
static thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}
}  // namespace mpm

extern "C" int mpm_abi_version(void) { return MPM_ABI_VERSION; }

extern "C" const char* mpm_last_error(void) { return mpm::g_last_error.c_str(); }

extern "C" int mpm_sm_count(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  return n;
}

extern "C" int mpm_copy_async(void* dst, const void* src, size_t bytes, int direction, void* stream) {
  cudaMemcpyKind kind;
  switch (direction) {
    case MPM_COPY_D2H: kind = cudaMemcpyDeviceToHost; break;
    case MPM_COPY_H2D: kind = cudaMemcpyHostToDevice; break;
    case MPM_COPY_D2D: kind = cudaMemcpyDeviceToDevice; break;
    default: mpm::set_error("mpm_copy_async: bad direction %d", direction); return MPM_ERR_INVALID;
  }
  if (bytes == 0) return 0;
  MPM_CUDA_RET(cudaMemcpyAsync(dst, src, bytes, kind, (cudaStream_t)stream));
  return 0;
}
