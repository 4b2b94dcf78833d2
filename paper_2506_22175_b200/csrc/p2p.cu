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

// Fused dispatch: one warp per destination row (destination d, local expert el, slot s) of this
// rank's part of a chunk; the row is gathered from the token rows through the slot-owner map
// (assignment a = t*k + j -> token row t, scaled by scale[a] for the routed gradient w * dy) and
// stored straight into destination d's expert-side buffer over NVLink (no local T_I staging).
// Unused slots get zero rows.  Light grid, no shared memory: co-resident with the GEMM CTAs.
struct PushArgs {
  int nranks, rank;
  char* dst[MPM_MAX_PEERS];
  uint32_t* flag[MPM_MAX_PEERS];
  int64_t e_loc, capacity, e0, ne, s0, cs, x_stride, x_row0;
  const int32_t* kept_all;  // [nranks][E] every source's kept counts: compacted expert-side rows (or null)
};

// Compacted expert-side layout (kept_all given; one slot part per expert group, so a chunk holds
// every slot of its experts): source s's valid rows of expert e start at the sum of the lower
// sources' kept counts, so every expert's routed rows are one contiguous prefix and its capacity
// padding is a single tail that the GEMMs skip (valid rows / valid K).
// Routed rows of (source s, expert e) inside the chunk's slot range [s0, s0 + cs): slots fill in order,
// so they are a prefix of the range.
__device__ __forceinline__ int64_t chunk_rows(const int32_t* __restrict__ kept_all, int64_t E, int64_t e, int s,
                                              int64_t s0, int64_t cs) {
  const int64_t v = (int64_t)kept_all[(int64_t)s * E + e] - s0;
  return v < 0 ? 0 : (v > cs ? cs : v);
}
__device__ __forceinline__ int64_t compact_offset(const int32_t* __restrict__ kept_all, int64_t E, int64_t e,
                                                  int src, int64_t s0 = 0, int64_t cs = INT64_MAX) {
  int64_t o = 0;
  for (int s = 0; s < src; ++s) o += chunk_rows(kept_all, E, e, s, s0, cs);
  return o;
}

template <typename T>
__global__ void __launch_bounds__(256)
dispatch_push_kernel(const __grid_constant__ PushArgs P, const uint4* __restrict__ src, int64_t vec_per_row, int k,
                     const int32_t* __restrict__ inv, const float* __restrict__ scale, uint32_t value,
                     uint32_t* counter) {
  const int lane = threadIdx.x & 31;
  const int64_t rows = (int64_t)P.nranks * P.ne * P.cs;
  const int64_t E = (int64_t)P.nranks * P.e_loc;
  // compacted: the last source also zeroes each expert's rows from its routed total up to the next
  // 64-row boundary (the weight-gradient K blocks read them); NT such rows per (destination, expert)
  constexpr int64_t NT = 64;
  const bool compact = P.kept_all != nullptr;
  const int64_t tail = compact && P.rank == P.nranks - 1 ? (int64_t)P.nranks * P.ne * NT : 0;
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows + tail;
       r += (int64_t)gridDim.x * (blockDim.x >> 5)) {
    if (r >= rows) {  // zero tail (compacted layout, last source)
      const int64_t q = r - rows;
      const int64_t d = q / (P.ne * NT);
      const int64_t el = P.e0 + (q - d * P.ne * NT) / NT;
      const int64_t z = q % NT;
      const int64_t e = d * P.e_loc + el;
      const int64_t tot = compact_offset(P.kept_all, E, e, P.nranks, P.s0, P.cs);
      const int64_t row = tot + z;
      if (row >= ((tot + NT - 1) / NT) * NT || row >= (int64_t)P.nranks * P.cs) continue;
      uint4* out = reinterpret_cast<uint4*>(P.dst[d]) + ((el - P.e0) * P.x_stride + P.x_row0 + row) * vec_per_row;
      for (int64_t v = lane; v < vec_per_row; v += 32) out[v] = make_uint4(0, 0, 0, 0);
      continue;
    }
    const int64_t d = r / (P.ne * P.cs);
    const int64_t rem = r - d * P.ne * P.cs;
    const int64_t el = P.e0 + rem / P.cs;
    const int64_t s = P.s0 + rem % P.cs;
    const int32_t a = inv[(d * P.e_loc + el) * P.capacity + s];
    if (compact && a < 0) continue;  // padding: not sent (the receiver's GEMMs stop at the routed rows)
    const int64_t xrow = compact ? compact_offset(P.kept_all, E, d * P.e_loc + el, P.rank, P.s0, P.cs) + (s - P.s0)
                                 : (int64_t)P.rank * P.cs + (s - P.s0);
    uint4* out = reinterpret_cast<uint4*>(P.dst[d]) + ((el - P.e0) * P.x_stride + P.x_row0 + xrow) * vec_per_row;
    if (a < 0) {
      for (int64_t v = lane; v < vec_per_row; v += 32) out[v] = make_uint4(0, 0, 0, 0);
      continue;
    }
    const uint4* in = src + (int64_t)(a / k) * vec_per_row;
    const float w = scale ? scale[a] : 1.f;
    for (int64_t v0 = 0; v0 < vec_per_row; v0 += 32 * 4) {  // 4 vectors per lane in flight
      uint4 u[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t v = v0 + lane + 32 * q;
        if (v < vec_per_row) u[q] = __ldg(in + v);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t v = v0 + lane + 32 * q;
        if (v >= vec_per_row) continue;
        if (scale) {  // the routed gradient: w * dy, rounded like combine_bwd's g_o rows
          uint4 o = u[q];
          if constexpr (sizeof(T) == 2) {
            __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float2 f = __bfloat1622float2(h[i]);
              h[i] = __floats2bfloat162_rn(f.x * w, f.y * w);
            }
          } else {
            o.x = __float_as_uint(__uint_as_float(o.x) * w); o.y = __float_as_uint(__uint_as_float(o.y) * w);
            o.z = __float_as_uint(__uint_as_float(o.z) * w); o.w = __float_as_uint(__uint_as_float(o.w) * w);
          }
          u[q] = o;
        }
        out[v] = u[q];
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();  // this CTA's rows are visible system-wide
    if (atomicAdd(counter, 1u) == gridDim.x - 1) {
      __threadfence_system();
      for (int d = 0; d < P.nranks; ++d)
        if (d != P.rank) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(P.flag[d]), "r"(value) : "memory");
      *counter = 0u;
    }
  }
}

// Combine-type push of one chunk in the compacted layout (R_i: T_DO -> owners' T_O; BR_i: g_di ->
// g_i): one warp per row; owner d's rows of local expert el are the kept_all[d][e] rows at d's
// compact offset, copied to d's dispatch-side rows (expert e, slots s0 ...).  The last CTA fences
// system-wide and raises flag (slot, rank) in every peer.
__global__ void __launch_bounds__(256)
combine_push_kernel(const __grid_constant__ PushArgs P, const uint4* __restrict__ src, int64_t vec_per_row,
                    uint32_t value, uint32_t* counter) {
  const int lane = threadIdx.x & 31;
  const int64_t E = (int64_t)P.nranks * P.e_loc;
  const int64_t rows = (int64_t)P.nranks * P.ne * P.cs;  // capacity-sized enumeration, unused rows skipped
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows;
       r += (int64_t)gridDim.x * (blockDim.x >> 5)) {
    const int64_t d = r / (P.ne * P.cs);
    const int64_t rem = r - d * P.ne * P.cs;
    const int64_t el = P.e0 + rem / P.cs;
    const int64_t j = rem % P.cs;
    const int64_t e = (int64_t)P.rank * P.e_loc + el;  // this rank's expert
    if (j >= chunk_rows(P.kept_all, E, e, (int)d, P.s0, P.cs)) continue;
    const uint4* in = src + ((el - P.e0) * P.x_stride + P.x_row0 +
                             compact_offset(P.kept_all, E, e, (int)d, P.s0, P.cs) + j) * vec_per_row;
    uint4* out = reinterpret_cast<uint4*>(P.dst[d]) + (e * P.capacity + P.s0 + j) * vec_per_row;
    for (int64_t v0 = 0; v0 < vec_per_row; v0 += 32 * 4) {
      uint4 u[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t v = v0 + lane + 32 * q;
        if (v < vec_per_row) u[q] = __ldcg(in + v);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t v = v0 + lane + 32 * q;
        if (v < vec_per_row) out[v] = u[q];
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    if (atomicAdd(counter, 1u) == gridDim.x - 1) {
      __threadfence_system();
      for (int d = 0; d < P.nranks; ++d)
        if (d != P.rank) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(P.flag[d]), "r"(value) : "memory");
      *counter = 0u;
    }
  }
}

// Routed rows per local expert in the compacted layout of a chunk's slot range:
// rows[el] = sum over sources of their routed rows of expert (rank, el) in [s0, s0 + cs).
__global__ void compact_rows_kernel(const int32_t* __restrict__ kept_all, int nranks, int64_t E, int64_t e_loc,
                                    int rank, int64_t s0, int64_t cs, int32_t* __restrict__ rows) {
  const int64_t el = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (el >= e_loc) return;
  rows[el] = (int32_t)compact_offset(kept_all, E, (int64_t)rank * e_loc + el, nranks, s0, cs);
}

// Dispatch-type pull of one chunk into the compacted layout (memory reuse: the expert side is a ring
// slot that peers cannot address, so the receiver pulls): source s's routed rows of local expert el in
// the chunk's slot range are read from s's dispatch-side buffer (P.dst[s] = T_I or g_o) and land at the
// lower sources' prefix; the rows from the routed total up to the next 64-row boundary are zeroed.
__global__ void __launch_bounds__(256)
compact_pull_kernel(const __grid_constant__ PushArgs P, uint4* __restrict__ dst, int64_t vec_per_row) {
  const int lane = threadIdx.x & 31;
  const int64_t E = (int64_t)P.nranks * P.e_loc;
  constexpr int64_t NT = 64;
  const int64_t rows = (int64_t)P.nranks * P.ne * P.cs;
  const int64_t tail = (int64_t)P.ne * NT;
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows + tail;
       r += (int64_t)gridDim.x * (blockDim.x >> 5)) {
    if (r >= rows) {  // zero tail of expert el
      const int64_t el = P.e0 + (r - rows) / NT, z = (r - rows) % NT;
      const int64_t tot = compact_offset(P.kept_all, E, (int64_t)P.rank * P.e_loc + el, P.nranks, P.s0, P.cs);
      const int64_t row = tot + z;
      if (row >= ((tot + NT - 1) / NT) * NT || row >= (int64_t)P.nranks * P.cs) continue;
      uint4* out = dst + ((el - P.e0) * P.x_stride + P.x_row0 + row) * vec_per_row;
      for (int64_t v = lane; v < vec_per_row; v += 32) out[v] = make_uint4(0, 0, 0, 0);
      continue;
    }
    const int64_t s = r / (P.ne * P.cs);
    const int64_t rem = r - s * P.ne * P.cs;
    const int64_t el = P.e0 + rem / P.cs;
    const int64_t j = rem % P.cs;
    const int64_t e = (int64_t)P.rank * P.e_loc + el;
    if (j >= chunk_rows(P.kept_all, E, e, (int)s, P.s0, P.cs)) continue;
    const uint4* in = reinterpret_cast<const uint4*>(P.dst[s]) + (e * P.capacity + P.s0 + j) * vec_per_row;
    uint4* out = dst + ((el - P.e0) * P.x_stride + P.x_row0 + compact_offset(P.kept_all, E, e, (int)s, P.s0, P.cs) + j) *
                           vec_per_row;
    for (int64_t v0 = 0; v0 < vec_per_row; v0 += 32 * 4) {
      uint4 u[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t v = v0 + lane + 32 * q;
        if (v < vec_per_row) u[q] = __ldcg(in + v);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t v = v0 + lane + 32 * q;
        if (v < vec_per_row) out[v] = u[q];
      }
    }
  }
}

// Slot owners: inv[e*C + s] = the assignment (t*k + j) holding slot s of expert e, -1 if unused.
__global__ void slot_owner_kernel(const int32_t* __restrict__ idx, const int32_t* __restrict__ slot,
                                  const int32_t* __restrict__ kept, int64_t Tk, int64_t E, int64_t C,
                                  int32_t* __restrict__ inv) {
  pdl_begin();
  const int64_t EC = E * C;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < EC + Tk; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < EC) {
      if (i % C >= kept[i / C]) inv[i] = -1;
    } else {
      const int64_t a = i - EC;
      const int32_t sl = slot[a];
      if (sl >= 0) inv[(int64_t)idx[a] * C + sl] = (int32_t)a;
    }
  }
}

}  // namespace
}  // namespace mpm

extern "C" int mpm_slot_owners(const int32_t* idx, const int32_t* slot, const int32_t* kept, int64_t T, int64_t E,
                               int k, int64_t capacity, int32_t* inv, void* stream) {
  MPM_CHECK_ARG(T >= 0 && E > 0 && k >= 1 && capacity >= 1 && E * capacity + T * k < (int64_t(1) << 31),
                "slot_owners: bad sizes");
  const int64_t items = E * capacity + T * k;
  const int64_t blocks = mpm::ceil_div(items, 256);
  MPM_PDL_LAUNCH(mpm::slot_owner_kernel, dim3((unsigned)(blocks < 4 * 148 ? blocks : 4 * 148)), dim3(256), 0,
                 (cudaStream_t)stream, idx, slot, kept, T * k, E, capacity, inv);
  return 0;
}

extern "C" int mpm_dispatch_push(const mpm_push_plan* plan, const void* src, int dtype, int64_t M, int k,
                                 const int32_t* inv, const float* scale, uint32_t value, void* stream) {
  MPM_CHECK_ARG(plan && src && inv && plan->counter, "dispatch_push: null argument");
  MPM_CHECK_ARG(plan->nranks >= 1 && plan->nranks <= MPM_MAX_PEERS && plan->rank >= 0 && plan->rank < plan->nranks,
                "dispatch_push: bad ranks");
  MPM_CHECK_ARG(dtype == MPM_BF16 || dtype == MPM_F32, "dispatch_push: dtype");
  const int64_t row_bytes = M * (int64_t)mpm::dtype_size(dtype);
  MPM_CHECK_ARG(row_bytes % 16 == 0 && ((uintptr_t)src & 15) == 0, "dispatch_push: rows must be 16-byte vectors");
  mpm::PushArgs P{};
  P.nranks = plan->nranks;
  P.rank = plan->rank;
  for (int d = 0; d < plan->nranks; ++d) {
    P.dst[d] = static_cast<char*>(plan->dst[d]);
    P.flag[d] = plan->flag[d];
    MPM_CHECK_ARG(((uintptr_t)plan->dst[d] & 15) == 0, "dispatch_push: unaligned destination");
  }
  P.e_loc = plan->e_loc; P.capacity = plan->capacity; P.e0 = plan->e0; P.ne = plan->ne; P.s0 = plan->s0;
  P.cs = plan->cs; P.x_stride = plan->x_stride; P.x_row0 = plan->x_row0;
  P.kept_all = plan->kept_all;
  MPM_CHECK_ARG(!P.kept_all || (P.s0 == 0 && P.cs == P.capacity),
                "dispatch_push: the compacted layout needs whole-capacity chunks (one slot part per expert group)");
  const int64_t rows = (int64_t)plan->nranks * plan->ne * plan->cs;
  if (rows == 0) return 0;
  // ~128 CTAs of 8 warps: NVLink stores in flight from every SM pair, light enough to co-reside
  const int64_t blocks = mpm::ceil_div(rows, 8);
  const unsigned grid = (unsigned)(blocks < 128 ? blocks : 128);
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t vpr = row_bytes / 16;
  if (dtype == MPM_BF16)
    mpm::dispatch_push_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(P, (const uint4*)src, vpr, k, inv, scale, value,
                                                                  plan->counter);
  else
    mpm::dispatch_push_kernel<float><<<grid, 256, 0, s>>>(P, (const uint4*)src, vpr, k, inv, scale, value,
                                                          plan->counter);
  MPM_LAUNCH_CHECK("dispatch_push_kernel");
  return 0;
}

extern "C" int mpm_combine_push(const mpm_push_plan* plan, const void* src, int dtype, int64_t M, uint32_t value,
                                void* stream) {
  MPM_CHECK_ARG(plan && src && plan->counter && plan->kept_all, "combine_push: null argument");
  MPM_CHECK_ARG(plan->nranks >= 1 && plan->nranks <= MPM_MAX_PEERS && plan->rank >= 0 && plan->rank < plan->nranks,
                "combine_push: bad ranks");
  MPM_CHECK_ARG(dtype == MPM_BF16 || dtype == MPM_F32, "combine_push: dtype");
  MPM_CHECK_ARG(plan->s0 >= 0 && plan->cs >= 0 && plan->s0 + plan->cs <= plan->capacity, "combine_push: slot range");
  const int64_t row_bytes = M * (int64_t)mpm::dtype_size(dtype);
  MPM_CHECK_ARG(row_bytes % 16 == 0 && ((uintptr_t)src & 15) == 0, "combine_push: rows must be 16-byte vectors");
  mpm::PushArgs P{};
  P.nranks = plan->nranks;
  P.rank = plan->rank;
  for (int d = 0; d < plan->nranks; ++d) {
    P.dst[d] = static_cast<char*>(plan->dst[d]);
    P.flag[d] = plan->flag[d];
    MPM_CHECK_ARG(((uintptr_t)plan->dst[d] & 15) == 0, "combine_push: unaligned destination");
  }
  P.e_loc = plan->e_loc; P.capacity = plan->capacity; P.e0 = plan->e0; P.ne = plan->ne; P.s0 = plan->s0;
  P.cs = plan->cs; P.x_stride = plan->x_stride; P.x_row0 = plan->x_row0;
  P.kept_all = plan->kept_all;
  const int64_t rows = (int64_t)plan->nranks * plan->ne * plan->cs;
  if (rows == 0) return 0;
  const int64_t blocks = mpm::ceil_div(rows, 8);
  const unsigned grid = (unsigned)(blocks < 128 ? blocks : 128);
  mpm::combine_push_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(P, (const uint4*)src, row_bytes / 16, value,
                                                                   plan->counter);
  MPM_LAUNCH_CHECK("combine_push_kernel");
  return 0;
}

extern "C" int mpm_compact_rows(const int32_t* kept_all, int nranks, int64_t E, int64_t e_loc, int rank,
                                int64_t s0, int64_t cs, int32_t* rows, void* stream) {
  MPM_CHECK_ARG(kept_all && rows && nranks >= 1 && E == (int64_t)nranks * e_loc && rank >= 0 && rank < nranks &&
                    s0 >= 0 && cs >= 0,
                "compact_rows: bad arguments");
  if (e_loc == 0) return 0;
  mpm::compact_rows_kernel<<<(unsigned)mpm::ceil_div(e_loc, 128), 128, 0, (cudaStream_t)stream>>>(
      kept_all, nranks, E, e_loc, rank, s0, cs, rows);
  MPM_LAUNCH_CHECK("compact_rows_kernel");
  return 0;
}

extern "C" int mpm_compact_pull(const mpm_push_plan* plan, void* dst, int dtype, int64_t M, void* stream) {
  MPM_CHECK_ARG(plan && dst && plan->kept_all, "compact_pull: null argument");
  MPM_CHECK_ARG(plan->nranks >= 1 && plan->nranks <= MPM_MAX_PEERS && plan->rank >= 0 && plan->rank < plan->nranks,
                "compact_pull: bad ranks");
  MPM_CHECK_ARG(dtype == MPM_BF16 || dtype == MPM_F32, "compact_pull: dtype");
  MPM_CHECK_ARG(plan->s0 >= 0 && plan->cs >= 0 && plan->s0 + plan->cs <= plan->capacity, "compact_pull: slot range");
  const int64_t row_bytes = M * (int64_t)mpm::dtype_size(dtype);
  MPM_CHECK_ARG(row_bytes % 16 == 0 && ((uintptr_t)dst & 15) == 0, "compact_pull: rows must be 16-byte vectors");
  mpm::PushArgs P{};
  P.nranks = plan->nranks;
  P.rank = plan->rank;
  for (int d = 0; d < plan->nranks; ++d) {
    P.dst[d] = static_cast<char*>(plan->dst[d]);
    MPM_CHECK_ARG(((uintptr_t)plan->dst[d] & 15) == 0, "compact_pull: unaligned source");
  }
  P.e_loc = plan->e_loc; P.capacity = plan->capacity; P.e0 = plan->e0; P.ne = plan->ne; P.s0 = plan->s0;
  P.cs = plan->cs; P.x_stride = plan->x_stride; P.x_row0 = plan->x_row0;
  P.kept_all = plan->kept_all;
  const int64_t rows = (int64_t)plan->nranks * plan->ne * plan->cs + plan->ne * 64;
  if (plan->ne == 0) return 0;
  const int64_t blocks = mpm::ceil_div(rows, 8);
  const unsigned grid = (unsigned)(blocks < 128 ? blocks : 128);
  mpm::compact_pull_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(P, (uint4*)dst, row_bytes / 16);
  MPM_LAUNCH_CHECK("compact_pull_kernel");
  return 0;
}

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
