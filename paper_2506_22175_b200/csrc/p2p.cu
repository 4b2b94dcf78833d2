// Chunk exchanges over NVLink peer memory.
//
// The pipelined layer moves one chunk per all-to-all (
// reference ops S_i / R_i / BS_i / RC_i / BR_i, pipesim/schedule.py:252-340)
// while the persistent tcgen05 GEMMs hold every SM.  A collective that needs
// shared memory would wait for the GEMM to drain (the paper's interference
// factors mu / sigma); here each exchange is one light copy
// kernel (no shared memory: it fits beside a GEMM CTA) or, selectably, copy
// engine transfers:
//
//   * every rank exports one device window per step arena through CUDA IPC
//     (the dispatch-side buffers T_I / T_O / g_o / g_i, the gate-gradient
//     staging and a flag array, at identical offsets on every rank);
//   * a pull (dispatch, re-dispatch, grad dispatch) waits for the source
//     rank's "ready" flag, then copies the E_loc blocks of the chunk straight
//     out of the peer's window into the local expert rows;
//   * a push (combine, grad combine) copies local expert rows into each
//     owner's window, bumps a flag there, and waits for the peers' flags in
//     the local window (the data of the chunk has arrived).
//
// Waits are stream memory operations (cuStreamWaitValue32 on local memory:
// no SM, no host); a one-thread release store per peer raises a flag.  Flag
// values are the arena's step epoch, identical on every rank.  Host cost per
// exchange is a handful of driver calls: one batched wait (cuStreamBatchMemOp),
// one batched copy of every row of every peer block (cudaMemcpyBatchAsync),
// one signal launch, one batched arrival wait.
#include <cuda.h>
#include <string.h>
#include <mutex>
#include <unordered_map>
#include <vector>
#include "common.cuh"

namespace mpm {
namespace {

typedef CUresult (*PFN_waitValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_batchMemOp)(CUstream, unsigned int, CUstreamBatchMemOpParams*, unsigned int);

PFN_batchMemOp batch_fn() {
  static PFN_batchMemOp fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamBatchMemOp", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_batchMemOp>(ptr);
  });
  return fn;
}

PFN_waitValue32 wait_fn() {
  static PFN_waitValue32 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_waitValue32>(ptr);
  });
  return fn;
}

// 1 = stream memory-op waits, 0 = spin kernel (MPM_P2P_WAIT=kernel forces it)
int wait_mode() {
  static int mode = -1;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* e = getenv("MPM_P2P_WAIT");
    if (e && strcmp(e, "kernel") == 0) { mode = 0; return; }
    // stream memory operations are on by default since CUDA 12; a failing
    // wait reports itself per call (MPM_P2P_WAIT=kernel then selects the spin kernel)
    mode = wait_fn() ? 1 : 0;
  });
  return mode;
}

struct FlagPtrs {
  uint32_t* p[MPM_MAX_PEERS];
};

__global__ void signal_kernel(FlagPtrs f, int n, uint32_t epoch) {
  const int i = threadIdx.x;
  if (i < n) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f.p[i]), "r"(epoch) : "memory");
}

struct ConstFlagPtrs {
  const uint32_t* p[MPM_MAX_PEERS];
};

// fallback wait: one thread per flag polls with acquire loads (wrap-safe compare)
__global__ void spin_wait_kernel(ConstFlagPtrs f, int n, uint32_t epoch) {
  const int i = threadIdx.x;
  if (i >= n) return;
  for (;;) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f.p[i]) : "memory");
    if ((int32_t)(v - epoch) >= 0) break;
    __nanosleep(256);
  }
}

__global__ void sum_slices_kernel(const float* __restrict__ s, int n, int64_t stride, int64_t count,
                                  float* __restrict__ out) {
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i >= count) return;
  float4 acc = __ldg(reinterpret_cast<const float4*>(s + i));
  for (int r = 1; r < n; ++r) {  // rank order: every rank computes the same bits
    const float4 v = __ldg(reinterpret_cast<const float4*>(s + r * stride + i));
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  *reinterpret_cast<float4*>(out + i) = acc;
}

// All copies of one exchange in one light grid: blockIdx.y = copy (peer block),
// blockIdx.x strides its rows x 16-byte vectors with 4 vectors per thread in
// flight.  No shared memory, 256 threads: a CTA fits beside a persistent GEMM
// CTA on the same SM, so the exchange overlaps the expert GEMMs instead of
// waiting for SMs.  The last CTA to finish (device counter) fences
// system-wide and raises the peer flags, so every row is visible to the
// peers before any flag is.
struct CopyList {
  int n_copy;
  int n_signal;
  mpm_p2p_copy c[MPM_MAX_PEERS];
  uint32_t* sig[MPM_MAX_PEERS];
};
constexpr int SM_COPY_THREADS = 256, SM_COPY_UNROLL = 4;

__global__ void __launch_bounds__(SM_COPY_THREADS)
p2p_copy_kernel(const __grid_constant__ CopyList L, uint32_t epoch, uint32_t* counter) {
  const mpm_p2p_copy& c = L.c[blockIdx.y];
  // 32-bit index math (a block is far below 2^32 vectors; the host checks): the row split
  // of every vector index is one 32-bit division instead of an emulated 64-bit one
  const uint32_t vpr = (uint32_t)(c.width >> 4);  // 16-byte vectors per row
  const uint32_t total = vpr * (uint32_t)c.height;
  const uint32_t stride = gridDim.x * SM_COPY_THREADS;
  const char* src = static_cast<const char*>(c.src);
  char* dst = static_cast<char*>(c.dst);
  for (uint32_t v0 = blockIdx.x * SM_COPY_THREADS + threadIdx.x; v0 < total; v0 += stride * SM_COPY_UNROLL) {
    uint4 u[SM_COPY_UNROLL];
    int64_t so[SM_COPY_UNROLL], dso[SM_COPY_UNROLL];
#pragma unroll
    for (int q = 0; q < SM_COPY_UNROLL; ++q) {
      const uint32_t v = v0 + q * stride;
      if (v < total) {
        const uint32_t h = v / vpr, x = v - h * vpr;
        so[q] = (int64_t)h * c.spitch + ((int64_t)x << 4);
        dso[q] = (int64_t)h * c.dpitch + ((int64_t)x << 4);
        u[q] = __ldcg(reinterpret_cast<const uint4*>(src + so[q]));
      }
    }
#pragma unroll
    for (int q = 0; q < SM_COPY_UNROLL; ++q)
      if (v0 + q * stride < total) *reinterpret_cast<uint4*>(dst + dso[q]) = u[q];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();  // this CTA's rows are visible system-wide
    const unsigned blocks = gridDim.x * gridDim.y;
    if (atomicAdd(counter, 1u) == blocks - 1) {
      __threadfence_system();
      for (int i = 0; i < L.n_signal; ++i)
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(L.sig[i]), "r"(epoch) : "memory");
      *counter = 0u;  // ready for the next launch (stream-ordered)
    }
  }
}

int wait_flags(const uint32_t* const* flags, int n, uint32_t epoch, cudaStream_t s) {
  if (n <= 0) return 0;
  if (wait_mode() == 1) {
    if (batch_fn()) {  // all waits of the exchange in one driver call
      CUstreamBatchMemOpParams ops[MPM_MAX_PEERS];
      memset(ops, 0, sizeof(CUstreamBatchMemOpParams) * n);
      for (int j = 0; j < n; ++j) {
        ops[j].waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_32;
        ops[j].waitValue.address = (CUdeviceptr)flags[j];
        ops[j].waitValue.value = epoch;
        ops[j].waitValue.flags = CU_STREAM_WAIT_VALUE_GEQ;
      }
      CUresult r = batch_fn()((CUstream)s, (unsigned)n, ops, 0);
      if (r != CUDA_SUCCESS) {
        set_error("cuStreamBatchMemOp(wait) failed (%d); set MPM_P2P_WAIT=kernel", (int)r);
        return 3000 + (int)r;
      }
      return 0;
    }
    for (int j = 0; j < n; ++j) {
      CUresult r = wait_fn()((CUstream)s, (CUdeviceptr)flags[j], epoch, CU_STREAM_WAIT_VALUE_GEQ);
      if (r != CUDA_SUCCESS) {
        set_error("cuStreamWaitValue32 failed (%d); set MPM_P2P_WAIT=kernel", (int)r);
        return 3000 + (int)r;
      }
    }
    return 0;
  }
  ConstFlagPtrs f{};
  for (int j = 0; j < n; ++j) f.p[j] = flags[j];
  spin_wait_kernel<<<1, 64, 0, s>>>(f, n, epoch);
  MPM_LAUNCH_CHECK("spin_wait_kernel");
  return 0;
}

// Copy fan-out: the copies of one exchange go to different peers, and each
// copy engine drives one transfer at a time, so one stream would serialise
// them.  Every issuing stream gets its own small set of helper streams (a
// fork event, one join event per helper; events are re-recorded per call,
// which is safe because each wait captures the record it follows).  Sets are
// per issuing stream so exchanges issued on different streams never queue
// behind each other's flag waits.
constexpr int MAX_FANOUT = 8;
struct FanOut {
  cudaStream_t aux[MAX_FANOUT];
  cudaEvent_t fork;
  cudaEvent_t join[MAX_FANOUT];
};

int fanout_for(cudaStream_t s, FanOut** out) {
  static std::mutex mu;
  static std::unordered_map<cudaStream_t, FanOut*> sets;
  std::lock_guard<std::mutex> lock(mu);
  auto it = sets.find(s);
  if (it != sets.end()) { *out = it->second; return 0; }
  FanOut* f = new FanOut();
  MPM_CUDA_RET(cudaEventCreateWithFlags(&f->fork, cudaEventDisableTiming));
  for (int j = 0; j < MAX_FANOUT; ++j) {
    MPM_CUDA_RET(cudaStreamCreateWithFlags(&f->aux[j], cudaStreamNonBlocking));
    MPM_CUDA_RET(cudaEventCreateWithFlags(&f->join[j], cudaEventDisableTiming));
  }
  sets[s] = f;
  *out = f;
  return 0;
}

// How the copies of one exchange are issued (MPM_P2P_COPY):
//   batch  one cudaMemcpyBatchAsync of every row of every peer block
//          (the driver schedules them over the copy engines; prefer-overlap hint)
//   fanout one cudaMemcpy2DAsync per peer block, spread over helper streams
//   serial one cudaMemcpy2DAsync per peer block on the issuing stream
//   sm     (default) one light SM kernel for every block + the fenced signal
enum { COPY_BATCH = 0, COPY_FANOUT = 1, COPY_SERIAL = 2, COPY_SM = 3 };
int copy_mode() {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("MPM_P2P_COPY");
    mode = !e ? COPY_SM
              : strcmp(e, "fanout") == 0 ? COPY_FANOUT
              : strcmp(e, "serial") == 0 ? COPY_SERIAL
              : strcmp(e, "batch") == 0 ? COPY_BATCH : COPY_SM;
  }
  return mode;
}

}  // namespace
}  // namespace mpm

extern "C" int mpm_ipc_alloc(size_t bytes, void** ptr_out, void* host_handle_out) {
  MPM_CHECK_ARG(ptr_out && host_handle_out && bytes > 0, "bad ipc alloc arguments");
  static_assert(sizeof(cudaIpcMemHandle_t) == MPM_IPC_HANDLE_BYTES, "IPC handle size");
  void* p = nullptr;
  MPM_CUDA_RET(cudaMalloc(&p, bytes));
  MPM_CUDA_RET(cudaMemset(p, 0, bytes));  // flags start below every epoch; padding reads as zeros
  MPM_CUDA_RET(cudaDeviceSynchronize());
  cudaIpcMemHandle_t h;
  MPM_CUDA_RET(cudaIpcGetMemHandle(&h, p));
  memcpy(host_handle_out, &h, sizeof(h));
  *ptr_out = p;
  return 0;
}

extern "C" int mpm_ipc_open(const void* host_handle, void** ptr_out) {
  MPM_CHECK_ARG(host_handle && ptr_out, "bad ipc open arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, host_handle, sizeof(h));
  MPM_CUDA_RET(cudaIpcOpenMemHandle(ptr_out, h, cudaIpcMemLazyEnablePeerAccess));
  return 0;
}

extern "C" int mpm_ipc_close(void* ptr) {
  if (ptr) MPM_CUDA_RET(cudaIpcCloseMemHandle(ptr));
  return 0;
}

extern "C" int mpm_ipc_free(void* ptr) {
  if (ptr) MPM_CUDA_RET(cudaFree(ptr));
  return 0;
}

extern "C" int mpm_p2p_wait_mode(void) { return mpm::wait_mode(); }

extern "C" int mpm_p2p_run(const mpm_p2p_plan* plan, uint32_t epoch, void* stream) {
  MPM_CHECK_ARG(plan != nullptr, "null plan");
  MPM_CHECK_ARG(plan->n_wait >= 0 && plan->n_wait <= MPM_MAX_PEERS && plan->n_copy >= 0 &&
                    plan->n_copy <= MPM_MAX_PEERS && plan->n_signal >= 0 && plan->n_signal <= MPM_MAX_PEERS &&
                    plan->n_arrive >= 0 && plan->n_arrive <= MPM_MAX_PEERS,
                "plan counts out of range");
  cudaStream_t s = (cudaStream_t)stream;
  if (int rc = mpm::wait_flags(plan->wait, plan->n_wait, epoch, s)) return rc;
  std::vector<int> live;
  for (int j = 0; j < plan->n_copy; ++j) {
    const mpm_p2p_copy& c = plan->copy[j];
    if (c.width > 0 && c.height > 0 && c.dst != c.src) live.push_back(j);
  }
  auto copy = [&](int j, cudaStream_t on) -> int {
    const mpm_p2p_copy& c = plan->copy[j];
    MPM_CUDA_RET(cudaMemcpy2DAsync(c.dst, (size_t)c.dpitch, c.src, (size_t)c.spitch, (size_t)c.width,
                                   (size_t)c.height, cudaMemcpyDeviceToDevice, on));
    return 0;
  };
  int mode = mpm::copy_mode();
  if (mode == mpm::COPY_SM) {
    bool ok = plan->counter != nullptr && !live.empty();
    for (int j : live) {
      const mpm_p2p_copy& c = plan->copy[j];
      ok = ok && ((c.width | c.dpitch | c.spitch) & 15) == 0 && ((uintptr_t)c.dst & 15) == 0 &&
           ((uintptr_t)c.src & 15) == 0;
    }
    if (ok) {
      mpm::CopyList L{};
      L.n_copy = (int)live.size();
      int64_t biggest = 0;
      for (size_t q = 0; q < live.size(); ++q) {
        L.c[q] = plan->copy[live[q]];
        const int64_t v = (L.c[q].width >> 4) * L.c[q].height;
        biggest = v > biggest ? v : biggest;
      }
      MPM_CHECK_ARG(biggest < (int64_t(1) << 31), "p2p copy block too large (%lld vectors)", (long long)biggest);
      L.n_signal = plan->n_signal;
      for (int j = 0; j < plan->n_signal; ++j) L.sig[j] = plan->signal[j];
      // ~128 CTAs in total: enough 16-byte loads in flight for NVLink, light enough to co-reside
      int64_t bx = mpm::ceil_div(128, (int64_t)live.size());
      const int64_t need = mpm::ceil_div(biggest, (int64_t)mpm::SM_COPY_THREADS * mpm::SM_COPY_UNROLL);
      bx = bx < need ? bx : need;
      mpm::p2p_copy_kernel<<<dim3((unsigned)(bx < 1 ? 1 : bx), (unsigned)live.size()), mpm::SM_COPY_THREADS, 0,
                             s>>>(L, epoch, plan->counter);
      MPM_LAUNCH_CHECK("p2p_copy_kernel");
      return mpm::wait_flags(plan->arrive, plan->n_arrive, epoch, s);
    }
    mode = mpm::COPY_SERIAL;  // nothing to copy, no counter, or unaligned: copy engines
  }
  const bool legacy = s == nullptr || s == cudaStreamLegacy;  // the batch API refuses the legacy stream
  if (live.size() > 0 && mode == mpm::COPY_BATCH && !legacy) {
    std::vector<void*> dsts, srcs;
    std::vector<size_t> sizes;
    for (int j : live) {
      const mpm_p2p_copy& c = plan->copy[j];
      for (int64_t h = 0; h < c.height; ++h) {  // one entry per row of the 2-D block
        dsts.push_back(static_cast<char*>(c.dst) + h * c.dpitch);
        srcs.push_back(const_cast<char*>(static_cast<const char*>(c.src)) + h * c.spitch);
        sizes.push_back((size_t)c.width);
      }
    }
    cudaMemcpyAttributes attr{};
    attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
    attr.flags = cudaMemcpyFlagPreferOverlapWithCompute;
    size_t idx0 = 0, fail = 0;
    cudaError_t e = cudaMemcpyBatchAsync(dsts.data(), srcs.data(), sizes.data(), dsts.size(), &attr, &idx0, 1,
                                         &fail, s);
    if (e != cudaSuccess) {
      mpm::set_error("cudaMemcpyBatchAsync failed: %s (copy %zu of %zu); MPM_P2P_COPY=serial avoids it",
                     cudaGetErrorString(e), fail, dsts.size());
      return (int)e;
    }
  } else if (live.size() <= 1 || mode == mpm::COPY_SERIAL || legacy) {
    for (int j : live)
      if (int rc = copy(j, s)) return rc;
  } else {
    // one helper stream per copy (round robin beyond MAX_FANOUT), joined before the signal
    mpm::FanOut* f = nullptr;
    if (int rc = mpm::fanout_for(s, &f)) return rc;
    const int lanes = (int)live.size() < mpm::MAX_FANOUT ? (int)live.size() : mpm::MAX_FANOUT;
    MPM_CUDA_RET(cudaEventRecord(f->fork, s));
    for (int l = 0; l < lanes; ++l) MPM_CUDA_RET(cudaStreamWaitEvent(f->aux[l], f->fork, 0));
    for (size_t q = 0; q < live.size(); ++q)
      if (int rc = copy(live[q], f->aux[q % lanes])) return rc;
    for (int l = 0; l < lanes; ++l) {
      MPM_CUDA_RET(cudaEventRecord(f->join[l], f->aux[l]));
      MPM_CUDA_RET(cudaStreamWaitEvent(s, f->join[l], 0));
    }
  }
  if (plan->n_signal > 0) {
    mpm::FlagPtrs f{};
    for (int j = 0; j < plan->n_signal; ++j) f.p[j] = plan->signal[j];
    mpm::signal_kernel<<<1, 64, 0, s>>>(f, plan->n_signal, epoch);
    MPM_LAUNCH_CHECK("signal_kernel");
  }
  return mpm::wait_flags(plan->arrive, plan->n_arrive, epoch, s);
}

extern "C" int mpm_sum_slices(const float* slices, int n, int64_t stride, int64_t count, float* out,
                              void* stream) {
  MPM_CHECK_ARG(n >= 1 && count % 4 == 0 && stride % 4 == 0, "sum_slices: n >= 1, count/stride multiples of 4");
  if (count == 0) return 0;
  const int64_t threads = count / 4;
  mpm::sum_slices_kernel<<<(unsigned)mpm::ceil_div(threads, 256), 256, 0, (cudaStream_t)stream>>>(
      slices, n, stride, count, out);
  MPM_LAUNCH_CHECK("sum_slices_kernel");
  return 0;
}
