// Error plumbing and device queries of the C-ABI (include/mpm.h).
#include <stdarg.h>
#include <atomic>
#include <stdlib.h>
#include "common.cuh"

namespace mpm {
static thread_local std::string g_last_error;

static std::atomic<unsigned long long> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("MPM_PDL");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

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

extern "C" unsigned long long mpm_launch_count(void) { return mpm::g_launches.load(); }

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

// ---------------------------------------------------------------- events
// Thin wrappers so the host executor (runtime.py) issues its cross-stream
// waits with one C call each.
extern "C" int mpm_event_create(int timing, void** ev_out) {
  MPM_CHECK_ARG(ev_out != nullptr, "null event out");
  cudaEvent_t ev;
  MPM_CUDA_RET(cudaEventCreateWithFlags(&ev, timing ? cudaEventDefault : cudaEventDisableTiming));
  *ev_out = ev;
  return 0;
}

extern "C" int mpm_event_destroy(void* ev) {
  if (ev) MPM_CUDA_RET(cudaEventDestroy((cudaEvent_t)ev));
  return 0;
}

extern "C" int mpm_event_record(void* ev, void* stream) {
  MPM_CUDA_RET(cudaEventRecord((cudaEvent_t)ev, (cudaStream_t)stream));
  return 0;
}

extern "C" int mpm_stream_wait(void* stream, void* ev) {
  MPM_CUDA_RET(cudaStreamWaitEvent((cudaStream_t)stream, (cudaEvent_t)ev, 0));
  return 0;
}

extern "C" int mpm_event_elapsed_ms(void* start, void* end, float* ms) {
  MPM_CUDA_RET(cudaEventSynchronize((cudaEvent_t)end));
  MPM_CUDA_RET(cudaEventElapsedTime(ms, (cudaEvent_t)start, (cudaEvent_t)end));
  return 0;
}
