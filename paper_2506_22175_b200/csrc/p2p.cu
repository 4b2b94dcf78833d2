// Chunk exchanges over NVLink peer memory.
//
// The pipelined layer moves one chunk per all-to-all (
// reference ops S_i / R_i / BS_i / RC_i / BR_i, pipesim/schedule.py:252-340)
// while the persistent tcgen05 GEMMs hold every SM.  A collective that needs
// shared memory would wait for the GEMM to drain (the paper's interference
// factors mu / sigma); here each exchange is one light copy
// kernel (no shared memory: it fits beside a GEMM CTA):
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
// Waits are stream memory operations (cuStreamBatchMemOp wait-value on local
// memory: no SM, no host); the copy kernel's last CTA raises the peer flags
// with release stores after a system fence.  A flag is raised once per step
// (value 1) and reset to 0 by its last waiter of the step, so no per-step
// value enters an exchange and a CUDA graph of the whole step replays as
// captured.  Host cost per exchange: one batched wait, one copy-kernel
// launch, one batched arrival wait (+ one batched reset).
#include <cuda.h>
#include <string.h>
#include <mutex>
#include "common.cuh"

namespace mpm {
namespace {

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

struct FlagPtrs {
  uint32_t* p[MPM_MAX_PEERS];
};

__global__ void signal_kernel(FlagPtrs f, int n, uint32_t value) {
  const int i = threadIdx.x;
  if (i < n) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f.p[i]), "r"(value) : "memory");
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

// Waits on local flags (>= value) as stream memory operations: no SM, no host thread; all
// waits of one exchange in one driver call.
int wait_flags(const uint32_t* const* flags, int n, uint32_t value, cudaStream_t s) {
  if (n <= 0) return 0;
  MPM_CHECK_ARG(batch_fn() != nullptr, "cuStreamBatchMemOp unavailable from the driver");
  CUstreamBatchMemOpParams ops[MPM_MAX_PEERS];
  memset(ops, 0, sizeof(CUstreamBatchMemOpParams) * n);
  for (int j = 0; j < n; ++j) {
    ops[j].waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_32;
    ops[j].waitValue.address = (CUdeviceptr)flags[j];
    ops[j].waitValue.value = value;
    ops[j].waitValue.flags = CU_STREAM_WAIT_VALUE_GEQ;
  }
  CUresult r = batch_fn()((CUstream)s, (unsigned)n, ops, 0);
  if (r != CUDA_SUCCESS) {
    set_error("cuStreamBatchMemOp(wait) failed (%d)", (int)r);
    return 3000 + (int)r;
  }
  return 0;
}

// Local flags back to 0 once their last waiter of the step has passed them (stream-ordered
// writes after the waits): every flag is raised once per step and consumed once, so the
// exchanges carry no per-step value and a captured CUDA graph replays them unchanged.
int reset_flags(uint32_t* const* flags, int n, cudaStream_t s) {
  if (n <= 0) return 0;
  MPM_CHECK_ARG(batch_fn() != nullptr, "cuStreamBatchMemOp unavailable from the driver");
  CUstreamBatchMemOpParams ops[MPM_MAX_PEERS];
  memset(ops, 0, sizeof(CUstreamBatchMemOpParams) * n);
  for (int j = 0; j < n; ++j) {
    ops[j].writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_32;
    ops[j].writeValue.address = (CUdeviceptr)flags[j];
    ops[j].writeValue.value = 0;
    ops[j].writeValue.flags = CU_STREAM_WRITE_VALUE_DEFAULT;
  }
  CUresult r = batch_fn()((CUstream)s, (unsigned)n, ops, 0);
  if (r != CUDA_SUCCESS) {
    set_error("cuStreamBatchMemOp(reset) failed (%d)", (int)r);
    return 3000 + (int)r;
  }
  return 0;
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

extern "C" int mpm_p2p_run(const mpm_p2p_plan* plan, uint32_t value, void* stream) {
  MPM_CHECK_ARG(plan != nullptr, "null plan");
  MPM_CHECK_ARG(plan->n_wait >= 0 && plan->n_wait <= MPM_MAX_PEERS && plan->n_copy >= 0 &&
                    plan->n_copy <= MPM_MAX_PEERS && plan->n_signal >= 0 && plan->n_signal <= MPM_MAX_PEERS &&
                    plan->n_arrive >= 0 && plan->n_arrive <= MPM_MAX_PEERS && plan->n_reset >= 0 &&
                    plan->n_reset <= MPM_MAX_PEERS,
                "plan counts out of range");
  cudaStream_t s = (cudaStream_t)stream;
  if (int rc = mpm::wait_flags(plan->wait, plan->n_wait, value, s)) return rc;
  mpm::CopyList L{};
  int64_t biggest = 0;
  for (int j = 0; j < plan->n_copy; ++j) {
    const mpm_p2p_copy& c = plan->copy[j];
    if (c.width <= 0 || c.height <= 0 || c.dst == c.src) continue;
    MPM_CHECK_ARG(((c.width | c.dpitch | c.spitch) & 15) == 0 && ((uintptr_t)c.dst & 15) == 0 &&
                      ((uintptr_t)c.src & 15) == 0,
                  "peer copies move 16-byte vectors: rows, pitches and addresses must be 16-byte aligned "
                  "(width %lld, pitches %lld/%lld)", (long long)c.width, (long long)c.dpitch, (long long)c.spitch);
    L.c[L.n_copy++] = c;
    const int64_t v = (c.width >> 4) * c.height;
    biggest = v > biggest ? v : biggest;
  }
  L.n_signal = plan->n_signal;
  for (int j = 0; j < plan->n_signal; ++j) L.sig[j] = plan->signal[j];
  if (L.n_copy > 0) {
    MPM_CHECK_ARG(plan->counter != nullptr, "a plan with copies needs its completion counter");
    MPM_CHECK_ARG(biggest < (int64_t(1) << 31), "p2p copy block too large (%lld vectors)", (long long)biggest);
    // ~128 CTAs in total: enough 16-byte loads in flight for NVLink, light enough to co-reside
    int64_t bx = mpm::ceil_div(128, (int64_t)L.n_copy);
    const int64_t need = mpm::ceil_div(biggest, (int64_t)mpm::SM_COPY_THREADS * mpm::SM_COPY_UNROLL);
    bx = bx < need ? bx : need;
    mpm::p2p_copy_kernel<<<dim3((unsigned)(bx < 1 ? 1 : bx), (unsigned)L.n_copy), mpm::SM_COPY_THREADS, 0, s>>>(
        L, value, plan->counter);
    MPM_LAUNCH_CHECK("p2p_copy_kernel");
  } else if (plan->n_signal > 0) {
    mpm::FlagPtrs f{};
    for (int j = 0; j < plan->n_signal; ++j) f.p[j] = plan->signal[j];
    mpm::signal_kernel<<<1, 64, 0, s>>>(f, plan->n_signal, value);
    MPM_LAUNCH_CHECK("signal_kernel");
  }
  if (int rc = mpm::wait_flags(plan->arrive, plan->n_arrive, value, s)) return rc;
  return mpm::reset_flags(plan->reset, plan->n_reset, s);
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
