// Exchange watchdog: turns a stalled peer exchange into a loud process abort.
//
// A chunk exchange waits on flags that peers raise (stream memory-op waits,
// csrc/p2p.cu).  If a peer process dies or hangs, those waits never complete
// and the survivor's streams block forever — the failure mode the reference's
// SPEC does not cover and NCCL's own watchdog exists for.  mpm_watchdog_watch
// records an event behind the work issued so far on a stream; one host thread
// polls every watched event and, when one has not completed within its
// timeout, prints the tag and aborts the process (torchrun then tears the job
// down), instead of leaving every rank hanging.  Events are owned here, so the
// caller's buffers and streams may go away while a watch is pending.
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <mutex>
#include <string>
#include <thread>

#include "common.cuh"

namespace mpm {
namespace {

struct Watch {
  cudaEvent_t ev;
  int device;
  std::chrono::steady_clock::time_point deadline;
  std::string tag;
};

struct Watchdog {
  std::mutex mu;
  std::condition_variable cv;
  std::deque<Watch> pending;
  std::thread thread;
  bool running = false;
  std::atomic<unsigned long long> fired{0};

  void loop() {
    // relaxed capture mode for this thread: its event queries must neither fail nor invalidate a
    // CUDA-graph capture another thread runs in global mode (MoELayer.step_graph)
    cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
    cudaThreadExchangeStreamCaptureMode(&mode);
    std::unique_lock<std::mutex> lock(mu);
    while (running) {
      cv.wait_for(lock, std::chrono::milliseconds(50));
      const auto now = std::chrono::steady_clock::now();
      for (auto it = pending.begin(); it != pending.end();) {
        cudaSetDevice(it->device);
        const cudaError_t q = cudaEventQuery(it->ev);
        if (q == cudaSuccess) {
          cudaEventDestroy(it->ev);
          it = pending.erase(it);
          continue;
        }
        if (q != cudaErrorNotReady) cudaGetLastError();  // transient (e.g. capture in progress): retry
        if (now > it->deadline) {
          fired++;
          fprintf(stderr,
                  "[mpm watchdog] %s: device work did not complete within its timeout (%s); a peer of the "
                  "expert-parallel group is likely dead or stalled. Aborting this rank.\n",
                  it->tag.c_str(), q == cudaErrorNotReady ? "still pending" : cudaGetErrorString(q));
          fflush(stderr);
          if (!getenv("MPM_WATCHDOG_NO_ABORT")) std::abort();
          cudaEventDestroy(it->ev);
          it = pending.erase(it);
          continue;
        }
        ++it;
      }
    }
  }
};

Watchdog& dog() {
  static Watchdog* d = new Watchdog();  // never destroyed: the thread may outlive static teardown
  return *d;
}

}  // namespace
}  // namespace mpm

extern "C" int mpm_watchdog_watch(void* stream, double timeout_s, const char* tag) {
  MPM_CHECK_ARG(timeout_s > 0, "watchdog timeout must be > 0");
  cudaStream_t s = (cudaStream_t)stream;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  MPM_CUDA_RET(cudaStreamIsCapturing(s, &cap));
  if (cap != cudaStreamCaptureStatusNone) return 0;  // a graph is watched at replay, not at capture
  int device = 0;
  MPM_CUDA_RET(cudaGetDevice(&device));
  cudaEvent_t ev;
  MPM_CUDA_RET(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  MPM_CUDA_RET(cudaEventRecord(ev, s));
  auto& d = mpm::dog();
  std::lock_guard<std::mutex> lock(d.mu);
  if (!d.running) {
    d.running = true;
    d.thread = std::thread([&d] { d.loop(); });
    d.thread.detach();
  }
  d.pending.push_back({ev, device,
                       std::chrono::steady_clock::now() + std::chrono::microseconds((int64_t)(timeout_s * 1e6)),
                       tag ? std::string(tag) : std::string("mpm exchange")});
  return 0;
}

extern "C" int mpm_watchdog_pending(void) {
  auto& d = mpm::dog();
  std::lock_guard<std::mutex> lock(d.mu);
  return (int)d.pending.size();
}

extern "C" unsigned long long mpm_watchdog_fired(void) { return mpm::dog().fired.load(); }
