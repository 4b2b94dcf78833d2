// Measurement helper for bench.py: SM clock + clock-event (throttle) reasons
// sampled from NVML by a native thread every `period_us`, stamped with
// CLOCK_MONOTONIC.  A native thread, because a Python sampler starves on the
// GIL while the step is being issued and a sampler process sees NVML calls
// slow down ~10x under another process's GPU load.  NVML is dlopen'ed, so the
// library has no link-time dependency on it; no NVML -> start returns an error
// and the caller falls back.
#include <dlfcn.h>
#include <cstdlib>
#include <time.h>
#include <atomic>
#include <mutex>
#include <thread>
#include <vector>
#include "common.cuh"

namespace {
typedef int (*nvml_init_t)(void);
typedef int (*nvml_handle_by_pci_t)(const char*, void**);
typedef int (*nvml_clock_t)(void*, int, unsigned int*);
typedef int (*nvml_reasons_t)(void*, unsigned long long*);
constexpr int NVML_CLOCK_SM = 1;

struct Sampler {
  std::thread th;
  std::atomic<bool> run{false};
  std::mutex mu;
  std::vector<double> rows;  // [sm_mhz, max_mhz, reasons, t]
  ~Sampler() {  // a sampler left running at exit: stop it instead of std::terminate
    run = false;
    if (th.joinable()) th.join();
  }
};
Sampler g_s;

double mono() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + ts.tv_nsec * 1e-9;
}
}  // namespace

extern "C" int mpm_clock_sampler_start(const char* pci_bus_id, int period_us) {
  if (g_s.run.load()) { mpm::set_error("clock sampler already running"); return MPM_ERR_INVALID; }
  void* lib = dlopen("libnvidia-ml.so.1", RTLD_NOW | RTLD_LOCAL);
  if (!lib) { mpm::set_error("libnvidia-ml.so.1 not found"); return MPM_ERR_INVALID; }
  auto init = (nvml_init_t)dlsym(lib, "nvmlInit_v2");
  auto by_pci = (nvml_handle_by_pci_t)dlsym(lib, "nvmlDeviceGetHandleByPciBusId_v2");
  auto clock = (nvml_clock_t)dlsym(lib, "nvmlDeviceGetClockInfo");
  auto maxclock = (nvml_clock_t)dlsym(lib, "nvmlDeviceGetMaxClockInfo");
  auto reasons = (nvml_reasons_t)dlsym(lib, "nvmlDeviceGetCurrentClocksEventReasons");
  if (!reasons) reasons = (nvml_reasons_t)dlsym(lib, "nvmlDeviceGetCurrentClocksThrottleReasons");
  if (!init || !by_pci || !clock || !maxclock || !reasons) { mpm::set_error("NVML symbols missing"); return MPM_ERR_INVALID; }
  void* dev = nullptr;
  if (init() != 0 || by_pci(pci_bus_id, &dev) != 0) { mpm::set_error("NVML init / device %s failed", pci_bus_id); return MPM_ERR_INVALID; }
  unsigned int mx = 0;
  maxclock(dev, NVML_CLOCK_SM, &mx);
  {
    std::lock_guard<std::mutex> lk(g_s.mu);
    g_s.rows.clear();
  }
  g_s.run = true;
  const int period = period_us > 0 ? period_us : 1000;
  g_s.th = std::thread([=] {
    while (g_s.run.load()) {
      unsigned int sm = 0;
      unsigned long long why = 0;
      clock(dev, NVML_CLOCK_SM, &sm);
      reasons(dev, &why);
      const double t = mono();
      {
        std::lock_guard<std::mutex> lk(g_s.mu);
        g_s.rows.insert(g_s.rows.end(), {(double)sm, (double)mx, (double)why, t});
      }
      timespec ts{0, (long)period * 1000};
      nanosleep(&ts, nullptr);
    }
  });
  return 0;
}

// Stops the thread; copies up to max_rows samples (4 doubles each) into out.
extern "C" int mpm_clock_sampler_stop(double* out, int max_rows, int* n_rows) {
  if (g_s.run.exchange(false) && g_s.th.joinable()) g_s.th.join();
  std::lock_guard<std::mutex> lk(g_s.mu);
  const int n = (int)(g_s.rows.size() / 4);
  const int m = n < max_rows ? n : max_rows;
  if (out && m > 0) std::copy(g_s.rows.begin(), g_s.rows.begin() + 4 * m, out);
  if (n_rows) *n_rows = m;
  return 0;
}

// CLOCK_MONOTONIC seconds (the samplers' time base; Python's time.monotonic is the same clock).
extern "C" double mpm_monotonic(void) { return mono(); }

// In-kernel SM clock trace: one thread (a 1-warp CTA, co-resident with any kernel) records
// (globaltimer ns, clock64) every `interval_ns` for `samples` samples, so the effective SM clock
// of the SM it lands on can be read at microsecond scale while a step runs (the NVML clock is a
// ~1 ms average and misses fast power-limit clock drops).
__global__ void clock_trace_kernel(unsigned long long* out, int samples, unsigned long long interval_ns,
                                   unsigned sleep_ns) {
  if (threadIdx.x != 0) return;
  unsigned long long next = 0;
  for (int i = 0; i < samples;) {
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    if (gt >= next) {
      out[2 * i] = gt;
      out[2 * i + 1] = clock64();
      next = gt + interval_ns;
      ++i;
    } else if (sleep_ns) {
      __nanosleep(sleep_ns);  // stay off the SM's issue slots between samples
    }
  }
}

extern "C" int mpm_clock_trace(unsigned long long* out, int samples, long long interval_ns, void* stream) {
  MPM_CHECK_ARG(out != nullptr && samples > 0 && interval_ns > 0, "clock_trace: bad arguments");
  // the warp sleeps between samples: a spinning warp takes issue slots from the GEMM CTA on its
  // SM, and the static tile order makes the whole GEMM wait for that SM (measured: 1.42 -> 2.10 ms
  // per cfg2 step with a spinning tracer, unchanged with the sleeping one)
  clock_trace_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(out, samples, (unsigned long long)interval_ns, 500u);
  MPM_LAUNCH_CHECK("clock_trace_kernel");
  return 0;
}
