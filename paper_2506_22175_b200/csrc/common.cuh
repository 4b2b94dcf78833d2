// Shared helpers for the libmpm kernels (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>
#include <string>

#include "../../include/mpm.h"

namespace mpm {

void set_error(const char* fmt, ...);
void note_launch();  // counts every libmpm kernel launch (mpm_launch_count)

#define MPM_CHECK_ARG(cond, ...)            \
  do {                                      \
    if (!(cond)) {                          \
      ::mpm::set_error(__VA_ARGS__);        \
      return MPM_ERR_INVALID;               \
    }                                       \
  } while (0)

#define MPM_CUDA_RET(expr)                                                   \
  do {                                                                       \
    cudaError_t e_ = (expr);                                                 \
    if (e_ != cudaSuccess) {                                                 \
      ::mpm::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                       __FILE__, __LINE__);                                  \
      return (int)e_;                                                        \
    }                                                                        \
  } while (0)

// Launch-error check after a <<<>>> launch; counts the launch.
#define MPM_LAUNCH_CHECK(name)          \
  do {                                  \
    MPM_CUDA_RET(cudaGetLastError());   \
    ::mpm::note_launch();               \
  } while (0)

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Top-k on fp32 logits, lowest expert index wins exact ties (oracle/moe_oracle.py route):
// a sorted insertion list of k <= KM entries.
__device__ __forceinline__ bool better(float v, int i, float bv, int bi) {
  return v > bv || (v == bv && i < bi);
}
template <int KM>
__device__ __forceinline__ void topk_insert(float (&tv)[KM], int (&ti)[KM], int k, float v, int e) {
  constexpr int NONE = 0x7fffffff;
  float cv = v;
  int ci = e;
#pragma unroll
  for (int j = 0; j < KM; ++j) {
    if (j < k && ci != NONE && (ti[j] == NONE || better(cv, ci, tv[j], ti[j]))) {
      const float fv = tv[j];
      const int fi = ti[j];
      tv[j] = cv; ti[j] = ci;
      cv = fv; ci = fi;
    }
  }
}



// Routing fused into the gate GEMM's epilogue (sm100::run with `route`): the epilogue thread that
// owns token row t in TMEM sums the three partial logits of its experts in the routing kernel's
// fixed order, writes the logits row, keeps a top-k, writes idx / weights, and each epilogue warp
// (32 rows = one routing block) writes the block's per-(k-rank, expert) counts.
struct RouteEpi {
  int64_t T;
  int E, Ec, k, renorm, nblk;
  float* logits;      // [T][E]
  int32_t* idx;       // [T][k]
  float* weights;     // [T][k]
  int32_t* counts;    // [k][nblk][E]
};

// Slot geometry of the dispatch buffers (expert-major [E][C][row]).  The
// capacity C is split into n chunks with the reference's balanced rule
// (core.py:102-105: the first C mod n parts get one extra slot); chunk i is
// slot range [s_i, s_i + c_i) of every expert, so within an expert all
// chunks are contiguous (one weight-gradient GEMM covers every chunk).
struct ChunkGeom {
  int64_t C;
  int n;
  int64_t q, r;  // C = q*n + r
  __host__ __device__ ChunkGeom(int64_t C_, int n_) : C(C_), n(n_), q(C_ / n_), r(C_ % n_) {}
  // chunk index and its first slot / size for a slot s in [0, C)
  __host__ __device__ inline void locate(int64_t s, int* chunk, int64_t* start, int64_t* size) const {
    int64_t big = r * (q + 1);
    if (s < big) {
      int64_t i = s / (q + 1);
      *chunk = (int)i; *start = i * (q + 1); *size = q + 1;
    } else {
      int64_t i = r + (s - big) / q;
      *chunk = (int)i; *start = big + (i - r) * q; *size = q;
    }
  }
  // row of (expert e, slot s) in a dispatch buffer of E experts
  __host__ __device__ inline int64_t row(int64_t /*E*/, int64_t e, int64_t s) const { return e * C + s; }
};

// bf16x3 split of an fp32 value: h = bf16(v), l = bf16(v - h), l2 = bf16(v - h - l) (24 mantissa
// bits in total; bf16 x bf16 products are exact in an fp32 tensor-core accumulator).
__device__ __forceinline__ void split3(float v, __nv_bfloat16 (&t)[3]) {
  t[0] = __float2bfloat16_rn(v);
  const float r1 = v - __bfloat162float(t[0]);
  t[1] = __float2bfloat16_rn(r1);
  t[2] = __float2bfloat16_rn(r1 - __bfloat162float(t[1]));
}

// Gate backward operands in the gate workspace (csrc/gate.cu): for T tokens, M, E experts
// (Ec = E rounded up to 32) the bf16x3 split of dlogits as
//   dla [T][3Ec]  h | l | l2   A (MN-major, rows = 3Ec) of dWg = dl^T x, one pass over x
//   dlc [T][3Ec]  h | l | h    A of the dense gate term dx_g = dl . Wg (three cross terms)
// written by the fused combine-backward / gate kernel (csrc/routing.cu) or gate_bwd_split_kernel.
struct GateBwdOperands {
  __nv_bfloat16* dla;
  __nv_bfloat16* dlc;
  int64_t Ec;
};
GateBwdOperands gate_bwd_operands(int64_t T, int64_t M, int64_t E, void* workspace);

// dlogits of one token (one warp; lane-strided over the padded expert axis) through the routing
// weights: softmax Jacobian, or the top-k renormalisation when k > 1 and renorm (then only the k
// chosen experts are nonzero); written as fp32 and as the split operands above (null: skipped).
template <int KM>
__device__ __forceinline__ void gate_token_dlogits(const float* __restrict__ logits_row, const int (&ex)[KM],
                                                   const float (&wv)[KM], const float (&dp)[KM], int k, int E,
                                                   int Ec, bool rn, int lane, float* __restrict__ dl_row,
                                                   __nv_bfloat16* __restrict__ dla_row,
                                                   __nv_bfloat16* __restrict__ dlc_row) {
  float s = 0.f;  // sum_j w_j dP_j
#pragma unroll
  for (int j = 0; j < KM; ++j)
    if (j < k) s = fmaf(wv[j], dp[j], s);
  float mx = -INFINITY, part = 0.f;
  if (!rn) {  // p = softmax(logits row), recomputed exactly as in route_kernel
    for (int e = lane; e < E; e += 32) mx = fmaxf(mx, logits_row[e]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    for (int e = lane; e < E; e += 32) part += expf(logits_row[e] - mx);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
  }
  for (int e = lane; e < Ec; e += 32) {
    float d = 0.f;
    if (e < E) {
      d = rn ? 0.f : -(expf(logits_row[e] - mx) / part) * s;
#pragma unroll
      for (int j = 0; j < KM; ++j)
        if (j < k && ex[j] == e) d += rn ? wv[j] * (dp[j] - s) : dp[j] * wv[j];
      dl_row[e] = d;
    }
    __nv_bfloat16 h[3];
    split3(d, h);
    if (dla_row) { dla_row[e] = h[0]; dla_row[Ec + e] = h[1]; dla_row[2 * Ec + e] = h[2]; }
    if (dlc_row) { dlc_row[e] = h[0]; dlc_row[Ec + e] = h[1]; dlc_row[2 * Ec + e] = h[0]; }
  }
}

__device__ __forceinline__ float to_f32(float v) { return v; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T> __device__ __forceinline__ T from_f32(float v);
template <> __device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

inline size_t dtype_size(int dt) { return dt == MPM_BF16 ? 2 : 4; }

// Programmatic dependent launch: kernels on a stream are launched with the
// programmatic-serialization attribute; the short HBM kernels start with
// pdl_begin() (let the next kernel be scheduled, then wait for the previous
// grid to complete and its memory to be visible), the persistent GEMM only
// waits (after its prologue) and lets dependents launch as its CTAs exit, so
// launch latency and prologues overlap the previous kernel's tail without
// parking waiting CTAs beside a running GEMM.  MPM_PDL=0 disables the
// attribute (the instructions are then no-ops).
bool pdl_enabled();

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_begin() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  pdl_wait();
}

template <typename... KArgs, typename... Args>
inline cudaError_t pdl_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<Args&&>(args)...);
}

#define MPM_PDL_LAUNCH(...)                          \
  do {                                               \
    MPM_CUDA_RET(::mpm::pdl_launch(__VA_ARGS__));    \
    ::mpm::note_launch();                            \
  } while (0)

// Warp-per-item grid-stride loop (the HBM-bound kernels run persistent grids).
#define MPM_WARP_LOOP(var, total)                                                            \
  for (int64_t var = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); var < (total); \
       var += (int64_t)gridDim.x * (blockDim.x >> 5))

// Per-device caches (a process may drive several GPUs): index of the current device.
constexpr int MAX_DEVICES = 64;
inline int device_index() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= MAX_DEVICES) d = 0;
  return d;
}
// SM count of the current device, cached per device.
inline int device_sms() {
  static int sms[MAX_DEVICES] = {0};
  const int d = device_index();
  if (sms[d] <= 0) {
    const int n = mpm_sm_count();
    sms[d] = n > 0 ? n : 148;
  }
  return sms[d];
}

// Persistent grid for a warp-per-item kernel: enough blocks for `warps` items,
// capped at the number of blocks that are resident at once (no partial last wave).
template <auto Kern>
unsigned persistent_grid(int threads, int64_t warps) {
  static int per_sm[MAX_DEVICES] = {0};
  const int d = device_index();
  if (per_sm[d] <= 0) {
    int v = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, Kern, threads, 0) != cudaSuccess || v < 1) v = 1;
    per_sm[d] = v;
  }
  const int64_t need = ceil_div(warps, threads / 32);
  const int64_t cap = (int64_t)per_sm[d] * device_sms();
  return (unsigned)(need < 1 ? 1 : (need < cap ? need : cap));
}

}  // namespace mpm
