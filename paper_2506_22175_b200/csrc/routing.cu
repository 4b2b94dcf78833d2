// Routing, permute and combine kernels (K1/K2/K7/K8/K13 of SURVEY.md §2.2).
//
// The reference excludes routing from its model (memmodel.py:7-8,
// README.md:153-154); the semantics here are the ones pinned in
// oracle/moe_oracle.py (top-k on fp32 logits with lowest-index tie-break,
// capacity C per (source rank, expert), slot priority (k-rank, token)),
// following PAPER.md:124 (gate -> dispatch -> expert -> combine) and
// PAPER.md:517-518 (top-k gate).
//
// All of these are HBM-bound: rows move as 16-byte vectors, one warp per
// token, and every reduction runs in a fixed order so results are
// bit-reproducible run to run.
#include "common.cuh"

namespace mpm {

constexpr int ROUTE_TB = 256;      // tokens per routing block
constexpr int ROUTE_THREADS = 256; // 8 warps
constexpr int MAX_E_PER_LANE = 8;  // E <= 256
constexpr int MAX_K = 8;

int simt_gemm_launch(const mpm_gemm_args* a, int a_dtype, int b_dtype, cudaStream_t s);

__device__ __forceinline__ bool better(float v, int i, float bv, int bi) {
  return v > bv || (v == bv && i < bi);
}

// One warp per token: top-k over logits, softmax weights, per-block counts.
__global__ void __launch_bounds__(ROUTE_THREADS)
route_kernel(const float* __restrict__ logits, int64_t T, int E, int k, int renorm,
             int32_t* __restrict__ idx_out, float* __restrict__ w_out,
             int32_t* __restrict__ counts /* [k][nblk][E] */, int nblk) {
  extern __shared__ int s_cnt[];  // [k][E]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < k * E; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  const int64_t t0 = (int64_t)blockIdx.x * ROUTE_TB;
  for (int tt = warp; tt < ROUTE_TB; tt += ROUTE_THREADS / 32) {
    const int64_t t = t0 + tt;
    if (t >= T) break;
    const float* row = logits + t * E;
    float v[MAX_E_PER_LANE];
    bool taken[MAX_E_PER_LANE];
#pragma unroll
    for (int q = 0; q < MAX_E_PER_LANE; ++q) {
      int e = lane + 32 * q;
      v[q] = (e < E) ? row[e] : -INFINITY;
      taken[q] = (e >= E);
    }
    int sel[MAX_K];
    float selv[MAX_K];
    for (int j = 0; j < k; ++j) {
      float bv = -INFINITY; int bi = 0x7fffffff;
#pragma unroll
      for (int q = 0; q < MAX_E_PER_LANE; ++q) {
        int e = lane + 32 * q;
        if (!taken[q] && (bi == 0x7fffffff || better(v[q], e, bv, bi))) { bv = v[q]; bi = e; }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        float ov = __shfl_xor_sync(0xffffffffu, bv, off);
        int oi = __shfl_xor_sync(0xffffffffu, bi, off);
        if (oi != 0x7fffffff && (bi == 0x7fffffff || better(ov, oi, bv, bi))) { bv = ov; bi = oi; }
      }
      sel[j] = bi; selv[j] = bv;
#pragma unroll
      for (int q = 0; q < MAX_E_PER_LANE; ++q)
        if (lane + 32 * q == bi) taken[q] = true;
    }
    const float mx = selv[0];
    if (k > 1 && renorm) {
      // softmax restricted to the chosen logits (== renormalised top-k probs)
      float den = 0.f;
      for (int j = 0; j < k; ++j) den += expf(selv[j] - mx);
      if (lane == 0)
        for (int j = 0; j < k; ++j) {
          idx_out[t * k + j] = sel[j];
          w_out[t * k + j] = expf(selv[j] - mx) / den;
        }
    } else {
      float part = 0.f;
#pragma unroll
      for (int q = 0; q < MAX_E_PER_LANE; ++q)
        if (lane + 32 * q < E) part += expf(v[q] - mx);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
      if (lane == 0)
        for (int j = 0; j < k; ++j) {
          idx_out[t * k + j] = sel[j];
          w_out[t * k + j] = expf(selv[j] - mx) / part;
        }
    }
    if (lane == 0)
      for (int j = 0; j < k; ++j) atomicAdd(&s_cnt[j * E + sel[j]], 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < k * E; i += blockDim.x) {
    int j = i / E, e = i % E;
    counts[((int64_t)j * nblk + blockIdx.x) * E + e] = s_cnt[i];
  }
}

// Exclusive prefix over (k-rank, block) per expert: the slot priority order.
__global__ void scan_kernel(const int32_t* __restrict__ counts, int32_t* __restrict__ offs,
                            int nblk, int E, int k, int64_t C, int32_t* __restrict__ kept) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  int64_t run = 0;
  for (int j = 0; j < k; ++j)
    for (int b = 0; b < nblk; ++b) {
      int64_t o = ((int64_t)j * nblk + b) * E + e;
      offs[o] = (int32_t)run;
      run += counts[o];
    }
  kept[e] = (int32_t)(run < C ? run : C);
}

// Slot of every (token, k-rank): block prefix + warp prefix + rank in warp.
__global__ void __launch_bounds__(ROUTE_THREADS)
slot_kernel(const int32_t* __restrict__ idx, int64_t T, int E, int k, int64_t C,
            const int32_t* __restrict__ offs, int nblk, int32_t* __restrict__ slot) {
  extern __shared__ int s_w[];  // [8][E]
  const int j = blockIdx.y, blk = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 8 * E; i += blockDim.x) s_w[i] = 0;
  __syncthreads();
  const int64_t t = (int64_t)blk * ROUTE_TB + threadIdx.x;
  const bool valid = t < T;
  const int e = valid ? idx[t * k + j] : -1;
  const unsigned peers = __match_any_sync(0xffffffffu, e);
  const unsigned lt = (1u << lane) - 1u;
  const int rank = __popc(peers & lt);
  if (valid && rank == 0) s_w[warp * E + e] = __popc(peers);
  __syncthreads();
  if (!valid) return;
  int pre = 0;
  for (int w = 0; w < warp; ++w) pre += s_w[w * E + e];
  int64_t s = (int64_t)offs[((int64_t)j * nblk + blk) * E + e] + pre + rank;
  slot[t * k + j] = s < C ? (int32_t)s : -1;
}

// Row scatter: one warp per (token, k-rank) assignment, 16-byte vectors.
__global__ void permute_kernel(const uint4* __restrict__ x, const int32_t* __restrict__ idx,
                               const int32_t* __restrict__ slot, int64_t T, int E, int k,
                               ChunkGeom g, int64_t vec_per_row, uint4* __restrict__ send) {
  const int64_t a = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (a >= T * k) return;
  const int32_t s = slot[a];
  if (s < 0) return;
  const int64_t t = a / k;
  const int64_t r = g.row(E, idx[a], s);
  const uint4* src = x + t * vec_per_row;
  uint4* dst = send + r * vec_per_row;
  for (int64_t v = lane; v < vec_per_row; v += 32) dst[v] = src[v];
}

// Zero the unused slots [kept[e], C) of every expert (one block per expert).
__global__ void zero_tail_kernel(const int32_t* __restrict__ kept, int E, ChunkGeom g,
                                 int64_t vec_per_row, uint4* __restrict__ buf) {
  const int e = blockIdx.x;
  const int64_t first = kept[e];
  const uint4 z = make_uint4(0, 0, 0, 0);
  const int64_t total = (g.C - first) * vec_per_row;
  for (int64_t i = threadIdx.x; i < total; i += blockDim.x) {
    int64_t s = first + i / vec_per_row, v = i % vec_per_row;
    buf[g.row(E, e, s) * vec_per_row + v] = z;
  }
}

template <typename T>
struct Vec8 {  // 16 bytes of T
  static constexpr int N = 16 / sizeof(T);
};

template <typename T>
__device__ __forceinline__ void load_vec(const uint4& u, float* f) {
  if constexpr (sizeof(T) == 2) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) { float2 p = __bfloat1622float2(h[i]); f[2 * i] = p.x; f[2 * i + 1] = p.y; }
  } else {
    f[0] = __uint_as_float(u.x); f[1] = __uint_as_float(u.y);
    f[2] = __uint_as_float(u.z); f[3] = __uint_as_float(u.w);
  }
}
template <typename T>
__device__ __forceinline__ uint4 store_vec(const float* f) {
  uint4 u;
  if constexpr (sizeof(T) == 2) {
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  } else {
    u.x = __float_as_uint(f[0]); u.y = __float_as_uint(f[1]);
    u.z = __float_as_uint(f[2]); u.w = __float_as_uint(f[3]);
  }
  return u;
}

// y[t] = sum_j w[t,j] * t_o[row_j]; one warp per token.
template <typename T>
__global__ void combine_kernel(const uint4* __restrict__ t_o, const int32_t* __restrict__ idx,
                               const int32_t* __restrict__ slot, const float* __restrict__ w,
                               int64_t Tn, int E, int k, ChunkGeom g, int64_t vec_per_row,
                               uint4* __restrict__ y) {
  constexpr int NV = Vec8<T>::N;
  const int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= Tn) return;
  int64_t rows[MAX_K];
  float ws[MAX_K];
  for (int j = 0; j < k; ++j) {
    int32_t s = slot[t * k + j];
    rows[j] = s < 0 ? -1 : g.row(E, idx[t * k + j], s);
    ws[j] = w[t * k + j];
  }
  for (int64_t v = lane; v < vec_per_row; v += 32) {
    float acc[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) acc[i] = 0.f;
    for (int j = 0; j < k; ++j) {
      if (rows[j] < 0) continue;
      float f[NV];
      load_vec<T>(t_o[rows[j] * vec_per_row + v], f);
#pragma unroll
      for (int i = 0; i < NV; ++i) acc[i] = fmaf(ws[j], f[i], acc[i]);
    }
    y[t * vec_per_row + v] = store_vec<T>(acc);
  }
}

// dprob[t,j] = <dy[t], t_o[row_j]>;  g_o[row_j] = w[t,j] * dy[t].
template <typename T>
__global__ void combine_bwd_kernel(const uint4* __restrict__ dy, const uint4* __restrict__ t_o,
                                   const int32_t* __restrict__ idx, const int32_t* __restrict__ slot,
                                   const float* __restrict__ w, int64_t Tn, int E, int k, ChunkGeom g,
                                   int64_t vec_per_row, float* __restrict__ dprob,
                                   uint4* __restrict__ g_o) {
  constexpr int NV = Vec8<T>::N;
  const int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= Tn) return;
  for (int j = 0; j < k; ++j) {
    const int32_t s = slot[t * k + j];
    if (s < 0) {
      if (lane == 0) dprob[t * k + j] = 0.f;
      continue;
    }
    const int64_t r = g.row(E, idx[t * k + j], s);
    const float wj = w[t * k + j];
    float part = 0.f;
    for (int64_t v = lane; v < vec_per_row; v += 32) {
      float a[NV], b[NV];
      load_vec<T>(dy[t * vec_per_row + v], a);
      load_vec<T>(t_o[r * vec_per_row + v], b);
#pragma unroll
      for (int i = 0; i < NV; ++i) { part = fmaf(a[i], b[i], part); a[i] *= wj; }
      g_o[r * vec_per_row + v] = store_vec<T>(a);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
    if (lane == 0) dprob[t * k + j] = part;
  }
}

// dlogits through the routing weights; one warp per token.
__global__ void gate_bwd_logits_kernel(const float* __restrict__ logits, const int32_t* __restrict__ idx,
                                       const float* __restrict__ w, const float* __restrict__ dprob,
                                       int64_t Tn, int E, int k, int renorm,
                                       float* __restrict__ dlogits) {
  const int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= Tn) return;
  float s = 0.f;  // sum_j w_j dP_j
  for (int j = 0; j < k; ++j) s = fmaf(w[t * k + j], dprob[t * k + j], s);
  float* out = dlogits + t * E;
  if (k > 1 && renorm) {
    for (int e = lane; e < E; e += 32) out[e] = 0.f;
    __syncwarp();
    if (lane == 0)
      for (int j = 0; j < k; ++j) out[idx[t * k + j]] = w[t * k + j] * (dprob[t * k + j] - s);
    return;
  }
  // p = softmax(logits row), recomputed exactly as in route_kernel
  const float* row = logits + t * E;
  float mx = -INFINITY;
  for (int e = lane; e < E; e += 32) mx = fmaxf(mx, row[e]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  float part = 0.f;
  for (int q = 0; q < MAX_E_PER_LANE; ++q) {
    int e = lane + 32 * q;
    if (e < E) part += expf(row[e] - mx);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
  for (int e = lane; e < E; e += 32) {
    float p = expf(row[e] - mx) / part;
    float d = -p * s;
    for (int j = 0; j < k; ++j)
      if (idx[t * k + j] == e) d += dprob[t * k + j] * w[t * k + j];
    out[e] = d;
  }
}

// dx[t] = sum_j g_i[row_j] + dlogits[t] . wg.  A block owns GB_TOK tokens
// and 1024 columns (256 threads x float4); wg rows stream from L2 and each
// float4 feeds GB_TOK*4 FMAs.
constexpr int GB_TOK = 16;
template <typename T>
__global__ void __launch_bounds__(256)
gather_bwd_kernel(const T* __restrict__ g_i, const int32_t* __restrict__ idx,
                  const int32_t* __restrict__ slot, const float* __restrict__ dlogits,
                  const float* __restrict__ wg, int64_t Tn, int64_t M, int E, int k,
                  ChunkGeom g, T* __restrict__ dx) {
  extern __shared__ float s_dl[];  // [GB_TOK][E]
  __shared__ int64_t s_rows[GB_TOK][MAX_K];
  const int64_t t0 = (int64_t)blockIdx.x * GB_TOK;
  const int64_t c = ((int64_t)blockIdx.y * 256 + threadIdx.x) * 4;
  for (int i = threadIdx.x; i < GB_TOK * E; i += blockDim.x) {
    int tt = i / E, e = i % E;
    s_dl[i] = (t0 + tt < Tn) ? dlogits[(t0 + tt) * E + e] : 0.f;
  }
  for (int i = threadIdx.x; i < GB_TOK * k; i += blockDim.x) {
    int tt = i / k, j = i % k;
    int64_t r = -1;
    if (t0 + tt < Tn) {
      int32_t s = slot[(t0 + tt) * k + j];
      if (s >= 0) r = g.row(E, idx[(t0 + tt) * k + j], s);
    }
    s_rows[tt][j] = r;
  }
  __syncthreads();
  if (c >= M) return;
  float acc[GB_TOK][4];
#pragma unroll
  for (int tt = 0; tt < GB_TOK; ++tt)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[tt][i] = 0.f;
  for (int e = 0; e < E; ++e) {
    const float4 wv = *reinterpret_cast<const float4*>(wg + (int64_t)e * M + c);
#pragma unroll
    for (int tt = 0; tt < GB_TOK; ++tt) {
      const float d = s_dl[tt * E + e];
      acc[tt][0] = fmaf(d, wv.x, acc[tt][0]);
      acc[tt][1] = fmaf(d, wv.y, acc[tt][1]);
      acc[tt][2] = fmaf(d, wv.z, acc[tt][2]);
      acc[tt][3] = fmaf(d, wv.w, acc[tt][3]);
    }
  }
#pragma unroll
  for (int tt = 0; tt < GB_TOK; ++tt) {
    if (t0 + tt >= Tn) break;
    float gsum[4] = {0.f, 0.f, 0.f, 0.f};
    for (int j = 0; j < k; ++j) {
      int64_t r = s_rows[tt][j];
      if (r < 0) continue;
      const T* src = g_i + r * M + c;
#pragma unroll
      for (int i = 0; i < 4; ++i) gsum[i] += to_f32(src[i]);
    }
    T* dst = dx + (t0 + tt) * M + c;
#pragma unroll
    for (int i = 0; i < 4; ++i) dst[i] = from_f32<T>(gsum[i] + acc[tt][i]);
  }
}

static int check_common(int dtype, int64_t M, int E, int k) {
  MPM_CHECK_ARG(dtype == MPM_F32 || dtype == MPM_BF16, "unsupported dtype %d", dtype);
  MPM_CHECK_ARG(E >= 1 && E <= 32 * MAX_E_PER_LANE, "num_experts %d outside [1, %d]", E, 32 * MAX_E_PER_LANE);
  MPM_CHECK_ARG(k >= 1 && k <= MAX_K && k <= E, "top_k %d outside [1, min(%d, E)]", k, MAX_K);
  MPM_CHECK_ARG((M * (int64_t)dtype_size(dtype)) % 16 == 0, "row bytes (M=%lld) must be a multiple of 16",
                (long long)M);
  return 0;
}

}  // namespace mpm

using namespace mpm;

static inline int nblk_of(int64_t T) { return (int)ceil_div(T, ROUTE_TB); }

extern "C" size_t mpm_route_workspace_bytes(int64_t T, int64_t E, int k) {
  return (size_t)2 * k * nblk_of(T) * E * sizeof(int32_t);
}

extern "C" int mpm_gate_fwd(const void* x, int x_dtype, const float* wg, float* logits, int64_t T,
                            int64_t M, int64_t E, void* stream) {
  MPM_CHECK_ARG(x_dtype == MPM_F32 || x_dtype == MPM_BF16, "unsupported dtype %d", x_dtype);
  if (T == 0) return 0;
  mpm_gemm_args a{};
  a.dtype = x_dtype; a.epilogue = MPM_EPI_NONE;
  a.batches = 1; a.rows = T; a.n = E; a.k = M;
  a.a = x; a.a_ld = M; a.a_mn_major = 0;
  a.b = wg; a.b_ld = M; a.b_mn_major = 0;
  a.c = logits; a.c_ld = E; a.c_dtype = MPM_F32;
  return simt_gemm_launch(&a, x_dtype, MPM_F32, (cudaStream_t)stream);
}

extern "C" int mpm_gate_wgrad(const float* dlogits, const void* x, int x_dtype, int64_t T, int64_t M,
                              int64_t E, float* dwg, void* stream) {
  MPM_CHECK_ARG(x_dtype == MPM_F32 || x_dtype == MPM_BF16, "unsupported dtype %d", x_dtype);
  mpm_gemm_args a{};
  a.dtype = x_dtype; a.epilogue = MPM_EPI_STORE_F32;
  a.batches = 1; a.rows = E; a.n = M; a.k = T;
  a.a = dlogits; a.a_ld = E; a.a_mn_major = 1;   // A(e, t) = dlogits[t][e]
  a.b = x; a.b_ld = M; a.b_mn_major = 1;         // B(m, t) = x[t][m]
  a.c = dwg; a.c_ld = M; a.c_dtype = MPM_F32;
  if (T == 0) { MPM_CUDA_RET(cudaMemsetAsync(dwg, 0, E * M * sizeof(float), (cudaStream_t)stream)); return 0; }
  return simt_gemm_launch(&a, MPM_F32, x_dtype, (cudaStream_t)stream);
}

extern "C" int mpm_route(const float* logits, int64_t T, int64_t E, int k, int renorm, int32_t* idx,
                         float* weights, void* workspace, void* stream) {
  if (int rc = check_common(MPM_F32, 4, (int)E, k)) return rc;
  if (T == 0) return 0;
  int nblk = nblk_of(T);
  route_kernel<<<nblk, ROUTE_THREADS, k * E * sizeof(int), (cudaStream_t)stream>>>(
      logits, T, (int)E, k, renorm, idx, weights, (int32_t*)workspace, nblk);
  MPM_LAUNCH_CHECK("route_kernel");
  return 0;
}

extern "C" int mpm_assign_slots(const int32_t* idx, int64_t T, int64_t E, int k, int64_t capacity,
                                void* workspace, int32_t* slot, int32_t* kept, void* stream) {
  if (int rc = check_common(MPM_F32, 4, (int)E, k)) return rc;
  MPM_CHECK_ARG(capacity >= 0 && capacity < (1ll << 31), "capacity %lld out of range", (long long)capacity);
  cudaStream_t s = (cudaStream_t)stream;
  if (T == 0) { MPM_CUDA_RET(cudaMemsetAsync(kept, 0, E * sizeof(int32_t), s)); return 0; }
  int nblk = nblk_of(T);
  int32_t* counts = (int32_t*)workspace;
  int32_t* offs = counts + (size_t)k * nblk * E;
  scan_kernel<<<(int)ceil_div(E, 128), 128, 0, s>>>(counts, offs, nblk, (int)E, k, capacity, kept);
  MPM_LAUNCH_CHECK("scan_kernel");
  slot_kernel<<<dim3(nblk, k), ROUTE_THREADS, 8 * E * sizeof(int), s>>>(idx, T, (int)E, k, capacity, offs,
                                                                         nblk, slot);
  MPM_LAUNCH_CHECK("slot_kernel");
  return 0;
}

extern "C" int mpm_permute(const void* x, int dtype, const int32_t* idx, const int32_t* slot,
                           const int32_t* kept, int64_t T, int64_t M, int64_t E, int k, int64_t capacity,
                           int n_chunks, void* send, void* stream) {
  if (int rc = check_common(dtype, M, (int)E, k)) return rc;
  MPM_CHECK_ARG(n_chunks >= 1 && n_chunks <= (capacity > 0 ? capacity : 1), "n_chunks %d invalid for C=%lld",
                n_chunks, (long long)capacity);
  cudaStream_t s = (cudaStream_t)stream;
  if (capacity == 0) return 0;
  ChunkGeom g(capacity, n_chunks);
  int64_t vpr = M * dtype_size(dtype) / 16;
  if (T > 0) {
    int64_t nasg = T * k;
    permute_kernel<<<(int)ceil_div(nasg, 8), 256, 0, s>>>((const uint4*)x, idx, slot, T, (int)E, k, g, vpr,
                                                            (uint4*)send);
    MPM_LAUNCH_CHECK("permute_kernel");
  }
  zero_tail_kernel<<<(int)E, 256, 0, s>>>(kept, (int)E, g, vpr, (uint4*)send);
  MPM_LAUNCH_CHECK("zero_tail_kernel");
  return 0;
}

extern "C" int mpm_combine(const void* t_o, int dtype, const int32_t* idx, const int32_t* slot,
                           const float* weights, int64_t T, int64_t M, int64_t E, int k, int64_t capacity,
                           int n_chunks, void* y, void* stream) {
  if (int rc = check_common(dtype, M, (int)E, k)) return rc;
  if (T == 0) return 0;
  ChunkGeom g(capacity > 0 ? capacity : 1, n_chunks);
  int64_t vpr = M * dtype_size(dtype) / 16;
  dim3 grid((unsigned)ceil_div(T, 8));
  if (dtype == MPM_BF16)
    combine_kernel<__nv_bfloat16><<<grid, 256, 0, (cudaStream_t)stream>>>(
        (const uint4*)t_o, idx, slot, weights, T, (int)E, k, g, vpr, (uint4*)y);
  else
    combine_kernel<float><<<grid, 256, 0, (cudaStream_t)stream>>>((const uint4*)t_o, idx, slot, weights, T,
                                                                   (int)E, k, g, vpr, (uint4*)y);
  MPM_LAUNCH_CHECK("combine_kernel");
  return 0;
}

extern "C" int mpm_combine_bwd(const void* dy, const void* t_o, int dtype, const int32_t* idx,
                               const int32_t* slot, const int32_t* kept, const float* weights, int64_t T,
                               int64_t M, int64_t E, int k, int64_t capacity, int n_chunks, float* dprob,
                               void* g_o, void* stream) {
  if (int rc = check_common(dtype, M, (int)E, k)) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  if (capacity == 0) {
    if (T > 0) MPM_CUDA_RET(cudaMemsetAsync(dprob, 0, T * k * sizeof(float), s));
    return 0;
  }
  ChunkGeom g(capacity, n_chunks);
  int64_t vpr = M * dtype_size(dtype) / 16;
  if (T > 0) {
    dim3 grid((unsigned)ceil_div(T, 8));
    if (dtype == MPM_BF16)
      combine_bwd_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>((const uint4*)dy, (const uint4*)t_o, idx, slot,
                                                              weights, T, (int)E, k, g, vpr, dprob, (uint4*)g_o);
    else
      combine_bwd_kernel<float><<<grid, 256, 0, s>>>((const uint4*)dy, (const uint4*)t_o, idx, slot, weights,
                                                      T, (int)E, k, g, vpr, dprob, (uint4*)g_o);
    MPM_LAUNCH_CHECK("combine_bwd_kernel");
  }
  zero_tail_kernel<<<(int)E, 256, 0, s>>>(kept, (int)E, g, vpr, (uint4*)g_o);
  MPM_LAUNCH_CHECK("zero_tail_kernel");
  return 0;
}

extern "C" int mpm_gate_bwd_logits(const float* logits, const int32_t* idx, const float* weights,
                                   const float* dprob, int64_t T, int64_t E, int k, int renorm, float* dlogits,
                                   void* stream) {
  if (int rc = check_common(MPM_F32, 4, (int)E, k)) return rc;
  if (T == 0) return 0;
  gate_bwd_logits_kernel<<<(unsigned)ceil_div(T, 8), 256, 0, (cudaStream_t)stream>>>(
      logits, idx, weights, dprob, T, (int)E, k, renorm, dlogits);
  MPM_LAUNCH_CHECK("gate_bwd_logits_kernel");
  return 0;
}

extern "C" int mpm_gather_bwd(const void* g_i, int dtype, const int32_t* idx, const int32_t* slot,
                              const float* dlogits, const float* wg, int64_t T, int64_t M, int64_t E, int k,
                              int64_t capacity, int n_chunks, void* dx, void* stream) {
  if (int rc = check_common(dtype, M, (int)E, k)) return rc;
  MPM_CHECK_ARG(M % 4 == 0, "M must be a multiple of 4");
  if (T == 0) return 0;
  ChunkGeom g(capacity > 0 ? capacity : 1, n_chunks);
  dim3 grid((unsigned)ceil_div(T, GB_TOK), (unsigned)ceil_div(M, 1024));
  size_t smem = GB_TOK * E * sizeof(float);
  if (dtype == MPM_BF16)
    gather_bwd_kernel<__nv_bfloat16><<<grid, 256, smem, (cudaStream_t)stream>>>(
        (const __nv_bfloat16*)g_i, idx, slot, dlogits, wg, T, M, (int)E, k, g, (__nv_bfloat16*)dx);
  else
    gather_bwd_kernel<float><<<grid, 256, smem, (cudaStream_t)stream>>>((const float*)g_i, idx, slot, dlogits,
                                                                         wg, T, M, (int)E, k, g, (float*)dx);
  MPM_LAUNCH_CHECK("gather_bwd_kernel");
  return 0;
}
