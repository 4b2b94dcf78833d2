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
#include <type_traits>
#include "common.cuh"

namespace mpm {

constexpr int ROUTE_TB = 32;       // tokens per routing block (= one warp's worth for slot ranks)
constexpr int MAX_E_PER_LANE = 8;  // E <= 256
constexpr int MAX_K = 8;

int simt_gemm_launch(const mpm_gemm_args* a, int a_dtype, int b_dtype, cudaStream_t s);

// Routing: 8 lanes per token (4 tokens per warp, a 256-thread block = one
// ROUTE_TB = 32-token routing block).  Each lane keeps a streaming top-k of
// the logits e = lane8 + 8q (lowest expert index wins exact ties), the 8
// lanes merge their lists in three xor rounds, then softmax weights and the
// block's per-(k-rank, expert) counts (shared-memory atomics).
constexpr int ROUTE_G = 8;

template <int KM>
__global__ void __launch_bounds__(256)
route_kernel(const float* __restrict__ logits, int64_t T, int E, int k, int renorm,
             int32_t* __restrict__ idx_out, float* __restrict__ w_out,
             int32_t* __restrict__ counts /* [k][nblk][E] */, int nblk,
             const float* __restrict__ parts = nullptr, int pitch = 0, float* __restrict__ logits_out = nullptr) {
  pdl_begin();
  static_assert(256 / ROUTE_G == ROUTE_TB, "one block = one routing block");
  constexpr int NONE = 0x7fffffff;
  extern __shared__ int s_cnt[];  // [k][E]
  for (int i = threadIdx.x; i < k * E; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  const int g8 = threadIdx.x & (ROUTE_G - 1);
  const int64_t t = (int64_t)blockIdx.x * ROUTE_TB + (threadIdx.x >> 3);
  const bool valid = t < T;
  float tv[KM];
  int ti[KM];
#pragma unroll
  for (int j = 0; j < KM; ++j) { tv[j] = -INFINITY; ti[j] = NONE; }
  // logits row: given, or (fused gate) the fixed-order sum of the stacked-term gate GEMM's
  // three partial logits [t][h | l | l2], written out for the backward on the way
  const float* row = logits + t * E;
  const float* prow = parts + t * 3 * pitch;
  auto logit = [&](int e) -> float {
    return parts ? (__ldg(prow + e) + __ldg(prow + pitch + e)) + __ldg(prow + 2 * pitch + e) : __ldg(row + e);
  };
  if (valid)
    for (int e = g8; e < E; e += ROUTE_G) {
      const float v = logit(e);
      if (parts) logits_out[t * E + e] = v;
      topk_insert<KM>(tv, ti, k, v, e);
    }
  // merge the 8 lanes' lists (xor partners stay inside the token's lane group)
#pragma unroll
  for (int off = 1; off < ROUTE_G; off <<= 1) {
    float pv[KM];
    int pi[KM];
#pragma unroll
    for (int j = 0; j < KM; ++j) {
      pv[j] = __shfl_xor_sync(0xffffffffu, tv[j], off);
      pi[j] = __shfl_xor_sync(0xffffffffu, ti[j], off);
    }
#pragma unroll
    for (int j = 0; j < KM; ++j)
      if (j < k) topk_insert<KM>(tv, ti, k, pv[j], pi[j]);
  }
  const float mx = tv[0];
  float den = 0.f;
  if (k > 1 && renorm) {
#pragma unroll
    for (int j = 0; j < KM; ++j)
      if (j < k) den += expf(tv[j] - mx);
  } else {
    if (valid)
      for (int e = g8; e < E; e += ROUTE_G) den += expf(logit(e) - mx);
#pragma unroll
    for (int off = 1; off < ROUTE_G; off <<= 1) den += __shfl_xor_sync(0xffffffffu, den, off);
  }
  if (valid && g8 == 0) {
#pragma unroll
    for (int j = 0; j < KM; ++j) {
      if (j >= k) break;
      idx_out[t * k + j] = ti[j];
      w_out[t * k + j] = expf(tv[j] - mx) / den;
      atomicAdd(&s_cnt[j * E + ti[j]], 1);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < k * E; i += blockDim.x) {
    const int j = i / E, e = i % E;
    counts[((int64_t)j * nblk + blockIdx.x) * E + e] = s_cnt[i];
  }
}

// Exclusive prefix over (k-rank, block) per expert: the slot priority order.
// One CTA per expert; each thread scans a contiguous run, then a CTA scan.
constexpr int SCAN_THREADS = 256;
__global__ void __launch_bounds__(SCAN_THREADS)
scan_kernel(const int32_t* __restrict__ counts, int32_t* __restrict__ offs, int nblk, int E, int k, int64_t C,
            int32_t* __restrict__ kept) {
  pdl_begin();
  __shared__ int s_warp[SCAN_THREADS / 32];
  const int e = blockIdx.x;
  const int L = k * nblk;
  const int per = (L + SCAN_THREADS - 1) / SCAN_THREADS;
  const int lo = threadIdx.x * per, hi = min(lo + per, L);
  int local = 0;
  for (int i = lo; i < hi; ++i) local += counts[(int64_t)i * E + e];
  // inclusive warp scan then CTA scan of warp totals
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = local;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    int o = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += o;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  int wbase = 0;
  for (int w = 0; w < warp; ++w) wbase += s_warp[w];
  int run = wbase + incl - local;  // exclusive prefix of this thread's run
  for (int i = lo; i < hi; ++i) {
    const int64_t o = (int64_t)i * E + e;
    offs[o] = run;
    run += counts[o];
  }
  if (threadIdx.x == SCAN_THREADS - 1) kept[e] = (int32_t)(run < C ? run : C);
}

// Slot of every (token, k-rank): one warp per (block, k-rank); the block's 32
// tokens are the warp's lanes, so the in-block rank is a match_any prefix.
__global__ void __launch_bounds__(256)
slot_kernel(const int32_t* __restrict__ idx, int64_t T, int E, int k, int64_t C,
            const int32_t* __restrict__ offs, int nblk, int32_t* __restrict__ slot) {
  pdl_begin();
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= nblk * k) return;
  const int j = w / nblk, blk = w % nblk;
  const int64_t t = (int64_t)blk * ROUTE_TB + lane;
  const bool valid = t < T;
  const int e = valid ? idx[t * k + j] : -1;
  const unsigned peers = __match_any_sync(0xffffffffu, e);
  const int rank = __popc(peers & ((1u << lane) - 1u));
  if (!valid) return;
  const int64_t s = (int64_t)offs[((int64_t)j * nblk + blk) * E + e] + rank;
  slot[t * k + j] = s < C ? (int32_t)s : -1;
}

// Unused slots (beyond the expert's kept count) get zero rows.  One warp item covers G consecutive
// slots of one expert: it reads kept[e] once and zeroes only the unused rows.  The combine
// backward kernels use G = 32 (E*C/32 dependent kept[] loads instead of E*C: 45 -> 43 us at
// configs[1], where ~2 % of the slots are unused); the permute keeps G = 1, whose zero items end
// its grid (a 32-slot item there leaves one warp zeroing a run of rows as the grid's tail).
template <int G>
__host__ __device__ inline int64_t zero_items(int64_t E, int64_t C) { return E * ((C + G - 1) / G); }
template <int G>
__device__ __forceinline__ void zero_unused_rows(int64_t w, const int32_t* __restrict__ kept, int E, const ChunkGeom& g,
                                                 int64_t vec_per_row, uint4* __restrict__ buf, int lane) {
  const int64_t groups = (g.C + G - 1) / G;
  if (w >= (int64_t)E * groups) return;
  // 32-bit index math (E*C < 2^31, checked on the host): a 64-bit division is an emulated sequence
  const uint32_t gr = (uint32_t)groups;
  const int e = (int)((uint32_t)w / gr);
  const int64_t s0 = (int64_t)((uint32_t)w - (uint32_t)e * gr) * G;
  const int64_t s1 = s0 + G < g.C ? s0 + G : g.C;
  const int64_t ks = kept[e];
  const uint4 z = make_uint4(0, 0, 0, 0);
  for (int64_t s = s0 > ks ? s0 : ks; s < s1; ++s) {
    uint4* dst = buf + g.row(E, e, s) * vec_per_row;
    for (int64_t v = lane; v < vec_per_row; v += 32) dst[v] = z;
  }
}

// Row scatter: one warp per (token, k-rank) assignment, 16-byte vectors;
// warps past the T*k assignments zero the unused slots of every expert.
__global__ void permute_kernel(const uint4* __restrict__ x, const int32_t* __restrict__ idx,
                               const int32_t* __restrict__ slot, const int32_t* __restrict__ kept, int64_t T, int E,
                               int k, ChunkGeom g, int64_t vec_per_row, uint4* __restrict__ send) {
  pdl_begin();
  const int lane = threadIdx.x & 31;
  MPM_WARP_LOOP(a, T * k + zero_items<1>(E, g.C)) {
    if (a >= T * k) {
      zero_unused_rows<1>(a - T * k, kept, E, g, vec_per_row, send, lane);
      continue;
    }
    const int32_t s = slot[a];
    if (s < 0) continue;
    const int64_t t = (uint32_t)a / (uint32_t)k;
    const int64_t r = g.row(E, idx[a], s);
    const uint4* src = x + t * vec_per_row;
    uint4* dst = send + r * vec_per_row;
    for (int64_t v0 = 0; v0 < vec_per_row; v0 += 32 * 4) {  // 4 vectors per lane in flight
      uint4 u[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t v = v0 + lane + 32 * q;
        if (v < vec_per_row) u[q] = __ldg(src + v);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t v = v0 + lane + 32 * q;
        if (v < vec_per_row) dst[v] = u[q];
      }
    }
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

// y[t] = sum_j w[t,j] * t_o[row_j]; one warp per token (persistent grid-stride).
// KM = compile-time bound on k (1/2/4/8): the loads of all k rows are issued
// before any FMA and routing state stays in registers.  CU vectors per lane
// per row are in flight (KM*CU <= 8).
template <int KM> struct CombineCfg { static constexpr int CU = KM <= 2 ? 4 : (KM == 4 ? 2 : 1); };

template <typename T, int KM>
__global__ void __launch_bounds__(256)
combine_kernel(const uint4* __restrict__ t_o, const int32_t* __restrict__ idx,
               const int32_t* __restrict__ slot, const float* __restrict__ w,
               int64_t Tn, int E, int k, ChunkGeom g, int64_t vec_per_row,
               uint4* __restrict__ y) {
  pdl_begin();
  constexpr int NV = Vec8<T>::N;
  constexpr int CU = CombineCfg<KM>::CU;
  const int lane = threadIdx.x & 31;
  MPM_WARP_LOOP(t, Tn) {
    int64_t rows[KM];
    float ws[KM];
#pragma unroll
    for (int j = 0; j < KM; ++j) {
      const int32_t s = j < k ? slot[t * k + j] : -1;
      rows[j] = s < 0 ? -1 : g.row(E, idx[t * k + j], s);
      ws[j] = j < k ? w[t * k + j] : 0.f;
    }
    for (int64_t v0 = 0; v0 < vec_per_row; v0 += 32 * CU) {
      uint4 raw[KM][CU];
#pragma unroll
      for (int j = 0; j < KM; ++j)
#pragma unroll
        for (int u = 0; u < CU; ++u) {
          const int64_t v = v0 + lane + 32 * u;
          raw[j][u] = (rows[j] >= 0 && v < vec_per_row) ? __ldg(t_o + rows[j] * vec_per_row + v)
                                                         : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
      for (int u = 0; u < CU; ++u) {
        float acc[NV];
#pragma unroll
        for (int i = 0; i < NV; ++i) acc[i] = 0.f;
#pragma unroll
        for (int j = 0; j < KM; ++j) {  // fixed order j = 0..k-1 (dropped rows add 0 * 0)
          float f[NV];
          load_vec<T>(raw[j][u], f);
#pragma unroll
          for (int i = 0; i < NV; ++i) acc[i] = fmaf(ws[j], f[i], acc[i]);
        }
        const int64_t v = v0 + lane + 32 * u;
        if (v < vec_per_row) y[t * vec_per_row + v] = store_vec<T>(acc);
      }
    }
  }
}

// dprob[t,j] = <dy[t], t_o[row_j]>;  g_o[row_j] = w[t,j] * dy[t].  dy is read once;
// warps past the tokens zero the unused slots of g_o.  DP / GO select the halves
// (the g_o half gates the expert backward; the dprob half only the gate's).
template <typename T, int KM, bool DP, bool GO>
__global__ void __launch_bounds__(256)
combine_bwd_kernel(const uint4* __restrict__ dy, const uint4* __restrict__ t_o,
                   const int32_t* __restrict__ idx, const int32_t* __restrict__ slot,
                   const float* __restrict__ w, int64_t Tn, int E, int k, ChunkGeom g,
                   int64_t vec_per_row, float* __restrict__ dprob, uint4* __restrict__ g_o,
                   const int32_t* __restrict__ kept) {
  pdl_begin();
  constexpr int NV = Vec8<T>::N;
  constexpr int CU = CombineCfg<KM>::CU;
  const int lane = threadIdx.x & 31;
  MPM_WARP_LOOP(t, Tn + (GO ? zero_items<32>(E, g.C) : 0)) {
    if (t >= Tn) {
      zero_unused_rows<32>(t - Tn, kept, E, g, vec_per_row, g_o, lane);
      continue;
    }
    int64_t rows[KM];
    float ws[KM], part[KM];
#pragma unroll
    for (int j = 0; j < KM; ++j) {
      const int32_t s = j < k ? slot[t * k + j] : -1;
      rows[j] = s < 0 ? -1 : g.row(E, idx[t * k + j], s);
      ws[j] = j < k ? w[t * k + j] : 0.f;
      part[j] = 0.f;
    }
    for (int64_t v0 = 0; v0 < vec_per_row; v0 += 32 * CU) {
      uint4 da[CU], raw[KM][CU];
#pragma unroll
      for (int u = 0; u < CU; ++u) {
        const int64_t v = v0 + lane + 32 * u;
        da[u] = v < vec_per_row ? __ldg(dy + t * vec_per_row + v) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int j = 0; j < KM; ++j)
#pragma unroll
        for (int u = 0; u < CU; ++u) {
          const int64_t v = v0 + lane + 32 * u;
          raw[j][u] = (DP && rows[j] >= 0 && v < vec_per_row) ? __ldg(t_o + rows[j] * vec_per_row + v)
                                                               : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
      for (int u = 0; u < CU; ++u) {
        const int64_t v = v0 + lane + 32 * u;
        float a[NV];
        load_vec<T>(da[u], a);
#pragma unroll
        for (int j = 0; j < KM; ++j) {
          if (rows[j] < 0) continue;
          if (DP) {
            float b[NV];
            load_vec<T>(raw[j][u], b);
#pragma unroll
            for (int i = 0; i < NV; ++i) part[j] = fmaf(a[i], b[i], part[j]);
          }
          if (GO) {
            float o[NV];
#pragma unroll
            for (int i = 0; i < NV; ++i) o[i] = a[i] * ws[j];
            if (v < vec_per_row) g_o[rows[j] * vec_per_row + v] = store_vec<T>(o);
          }
        }
      }
    }
    if (DP) {
#pragma unroll
      for (int j = 0; j < KM; ++j) {
        float p = part[j];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) p += __shfl_xor_sync(0xffffffffu, p, off);
        if (lane == 0 && j < k) dprob[t * k + j] = rows[j] < 0 ? 0.f : p;
      }
    }
  }
}

// Fused combine backward + gate softmax backward, one warp per token: dy is read once and the k
// routed rows of t_o once; the g_o rows (GO; warps past the tokens zero the unused slots),
// dprob (optional), dlogits and the bf16x3 split operands of the gate GEMMs (dla / dlc of
// GateBwdOperands; null on the exact-fp32 path) in one pass.  The separate route was combine_bwd
// (dy and t_o) + gate_bwd_split_kernel (dprob and logits again): one more pass over dy, two more
// launches.
template <typename T, int KM, bool GO>
__global__ void __launch_bounds__(256, 3)  // 3 CTAs (24 warps) per SM: the row loads need the warps
combine_bwd_gate_kernel(const uint4* __restrict__ dy, const uint4* __restrict__ t_o,
                        const int32_t* __restrict__ idx, const int32_t* __restrict__ slot,
                        const float* __restrict__ w, const float* __restrict__ logits, int64_t Tn, int E, int Ec,
                        int k, int renorm, ChunkGeom g, int64_t vec_per_row, float* __restrict__ dprob,
                        uint4* __restrict__ g_o, const int32_t* __restrict__ kept, float* __restrict__ dlogits,
                        __nv_bfloat16* __restrict__ dla, __nv_bfloat16* __restrict__ dlc) {
  pdl_begin();
  constexpr int NV = Vec8<T>::N;
  constexpr int CU = CombineCfg<KM>::CU;
  const int lane = threadIdx.x & 31;
  MPM_WARP_LOOP(t, Tn + (GO ? zero_items<32>(E, g.C) : 0)) {
    if (t >= Tn) {
      zero_unused_rows<32>(t - Tn, kept, E, g, vec_per_row, g_o, lane);
      continue;
    }
    int64_t rows[KM];
    int ex[KM];
    float ws[KM], part[KM];
#pragma unroll
    for (int j = 0; j < KM; ++j) {
      const int32_t s = j < k ? slot[t * k + j] : -1;
      ex[j] = j < k ? idx[t * k + j] : -1;
      rows[j] = s < 0 ? -1 : g.row(E, ex[j], s);
      ws[j] = j < k ? w[t * k + j] : 0.f;
      part[j] = 0.f;
    }
    for (int64_t v0 = 0; v0 < vec_per_row; v0 += 32 * CU) {
      uint4 da[CU], raw[KM][CU];
#pragma unroll
      for (int u = 0; u < CU; ++u) {
        const int64_t v = v0 + lane + 32 * u;
        da[u] = v < vec_per_row ? __ldg(dy + t * vec_per_row + v) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int j = 0; j < KM; ++j)
#pragma unroll
        for (int u = 0; u < CU; ++u) {
          const int64_t v = v0 + lane + 32 * u;
          raw[j][u] = (rows[j] >= 0 && v < vec_per_row) ? __ldg(t_o + rows[j] * vec_per_row + v)
                                                         : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
      for (int u = 0; u < CU; ++u) {
        const int64_t v = v0 + lane + 32 * u;
        float a[NV];
        load_vec<T>(da[u], a);
#pragma unroll
        for (int j = 0; j < KM; ++j) {
          if (rows[j] < 0) continue;
          float b[NV];
          load_vec<T>(raw[j][u], b);
#pragma unroll
          for (int i = 0; i < NV; ++i) part[j] = fmaf(a[i], b[i], part[j]);
          if (GO) {
            float o[NV];
#pragma unroll
            for (int i = 0; i < NV; ++i) o[i] = a[i] * ws[j];
            if (v < vec_per_row) g_o[rows[j] * vec_per_row + v] = store_vec<T>(o);
          }
        }
      }
    }
    float dp[KM];
#pragma unroll
    for (int j = 0; j < KM; ++j) {  // butterfly: every lane holds the dot products
      float p = part[j];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) p += __shfl_xor_sync(0xffffffffu, p, off);
      dp[j] = (j < k && rows[j] >= 0) ? p : 0.f;
      if (dprob && lane == 0 && j < k) dprob[t * k + j] = dp[j];
    }
    gate_token_dlogits<KM>(logits + t * E, ex, ws, dp, k, E, Ec, k > 1 && renorm, lane, dlogits + t * E,
                           dla ? dla + t * 3 * Ec : nullptr, dlc ? dlc + t * 3 * Ec : nullptr);
  }
}

// dlogits through the routing weights; one warp per token.
__global__ void gate_bwd_logits_kernel(const float* __restrict__ logits, const int32_t* __restrict__ idx,
                                       const float* __restrict__ w, const float* __restrict__ dprob,
                                       int64_t Tn, int E, int k, int renorm,
                                       float* __restrict__ dlogits) {
  pdl_begin();
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

// Calls f(element tag, integral_constant<KM>) with the smallest KM in {1, 2, 4, 8} >= k.
template <typename F>
static cudaError_t dispatch_k(int dtype, int k, F&& f) {
  auto by_k = [&](auto tag) -> cudaError_t {
    if (k <= 1) return f(tag, std::integral_constant<int, 1>{});
    if (k <= 2) return f(tag, std::integral_constant<int, 2>{});
    if (k <= 4) return f(tag, std::integral_constant<int, 4>{});
    return f(tag, std::integral_constant<int, 8>{});
  };
  if (dtype == MPM_BF16) return by_k(__nv_bfloat16{});
  return by_k(float{});
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

extern "C" int mpm_route(const float* logits, int64_t T, int64_t E, int k, int renorm, int32_t* idx,
                         float* weights, void* workspace, void* stream) {
  if (int rc = check_common(MPM_F32, 4, (int)E, k)) return rc;
  if (T == 0) return 0;
  const int nblk = nblk_of(T);
  cudaStream_t s = (cudaStream_t)stream;
  int32_t* counts = (int32_t*)workspace;
  const size_t sm = (size_t)k * E * sizeof(int);
  auto kern = k <= 1 ? route_kernel<1> : k <= 2 ? route_kernel<2> : k <= 4 ? route_kernel<4> : route_kernel<8>;
  MPM_PDL_LAUNCH(kern, dim3(nblk), dim3(256), sm, s, logits, T, (int)E, k, renorm, idx, weights, counts, nblk,
                 (const float*)nullptr, 0, (float*)nullptr);
  return 0;
}

namespace mpm {
int gate_partials(const void* x, int x_dtype, const float* wg, int64_t T, int64_t M, int64_t E, float* logits,
                  void* workspace, cudaStream_t s, const float** parts, int64_t* pitch);
int gate_route_fused(const void* x, int x_dtype, const float* wg, int64_t T, int64_t M, int64_t E, int k, int renorm,
                     float* logits, int32_t* idx, float* weights, int32_t* counts, void* workspace, cudaStream_t s);
}

extern "C" int mpm_gate_route(const void* x, int x_dtype, const float* wg, int64_t T, int64_t M, int64_t E, int k,
                              int renorm, float* logits, int32_t* idx, float* weights, void* gate_ws,
                              void* route_ws, void* stream) {
  if (int rc = check_common(MPM_F32, 4, (int)E, k)) return rc;
  if (T == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  // E <= 64 on the tensor-core path: the routing runs in the gate GEMM's epilogue (no partial logits,
  // no routing kernel); otherwise the GEMM stores the partials and route_kernel sums them
  const int fused = gate_route_fused(x, x_dtype, wg, T, M, E, k, renorm, logits, idx, weights,
                                     (int32_t*)route_ws, gate_ws, s);
  if (fused >= 0) return fused;
  const float* parts = nullptr;  // non-null: the routing kernel sums the partial logits
  int64_t pitch = 0;
  if (int rc = gate_partials(x, x_dtype, wg, T, M, E, logits, gate_ws, s, &parts, &pitch)) return rc;
  const int nblk = nblk_of(T);
  int32_t* counts = (int32_t*)route_ws;
  const size_t sm = (size_t)k * E * sizeof(int);
  auto kern = k <= 1 ? route_kernel<1> : k <= 2 ? route_kernel<2> : k <= 4 ? route_kernel<4> : route_kernel<8>;
  MPM_PDL_LAUNCH(kern, dim3(nblk), dim3(256), sm, s, (const float*)logits, T, (int)E, k, renorm, idx, weights, counts,
                 nblk, parts, (int)pitch, logits);
  return 0;
}

__global__ void chunk_rows_kernel(const int32_t* __restrict__ kept, int E, ChunkGeom g, int32_t* __restrict__ out) {
  pdl_begin();
  const int i = blockIdx.y;
  const int64_t big = g.r;  // the first C mod n chunks hold q + 1 slots (core.py:102-105)
  const int64_t start = i < big ? i * (g.q + 1) : big * (g.q + 1) + (i - big) * g.q;
  const int64_t size = i < big ? g.q + 1 : g.q;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    const int64_t v = (int64_t)kept[e] - start;
    out[(int64_t)i * E + e] = (int32_t)(v < 0 ? 0 : (v > size ? size : v));
  }
}

extern "C" int mpm_chunk_rows(const int32_t* kept, int64_t E, int64_t capacity, int n_chunks, int32_t* rows_out,
                              void* stream) {
  MPM_CHECK_ARG(E > 0 && E < (1 << 30) && n_chunks >= 1 && capacity >= n_chunks && capacity < (1ll << 31),
                "chunk_rows: bad sizes (E=%lld, C=%lld, n=%d)", (long long)E, (long long)capacity, n_chunks);
  MPM_PDL_LAUNCH(chunk_rows_kernel, dim3((unsigned)ceil_div(E, 256), (unsigned)n_chunks), dim3(256), 0,
                 (cudaStream_t)stream, kept, (int)E, ChunkGeom(capacity, n_chunks), rows_out);
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
  MPM_PDL_LAUNCH(scan_kernel, dim3((unsigned)E), dim3(SCAN_THREADS), 0, s, (const int32_t*)counts, offs, nblk,
                 (int)E, k, capacity, kept);
  MPM_PDL_LAUNCH(slot_kernel, dim3((unsigned)ceil_div((int64_t)nblk * k, 8)), dim3(256), 0, s, idx, T, (int)E, k,
                 capacity, (const int32_t*)offs, nblk, slot);
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
  const int64_t warps = T * k + zero_items<1>(E, capacity);
  MPM_CHECK_ARG(warps < (int64_t(1) << 31), "T*k + E*C too large (%lld)", (long long)warps);
  MPM_PDL_LAUNCH(permute_kernel, dim3(persistent_grid<permute_kernel>(256, warps)), dim3(256), 0, s,
                 (const uint4*)x, idx, slot, kept, T, (int)E, k, g, vpr, (uint4*)send);
  return 0;
}

extern "C" int mpm_combine(const void* t_o, int dtype, const int32_t* idx, const int32_t* slot,
                           const float* weights, int64_t T, int64_t M, int64_t E, int k, int64_t capacity,
                           int n_chunks, void* y, void* stream) {
  if (int rc = check_common(dtype, M, (int)E, k)) return rc;
  if (T == 0) return 0;
  ChunkGeom g(capacity > 0 ? capacity : 1, n_chunks);
  int64_t vpr = M * dtype_size(dtype) / 16;
  cudaStream_t s = (cudaStream_t)stream;
  auto launch = [&](auto tag, auto km) -> cudaError_t {
    using TT = decltype(tag);
    constexpr int KM = decltype(km)::value;
    return ::mpm::pdl_launch(combine_kernel<TT, KM>, dim3(persistent_grid<combine_kernel<TT, KM>>(256, T)), dim3(256),
                             0, s, (const uint4*)t_o, idx, slot, weights, T, (int)E, k, g, vpr, (uint4*)y);
  };
  MPM_CUDA_RET(dispatch_k(dtype, k, launch));
  note_launch();
  return 0;
}

extern "C" int mpm_combine_bwd(const void* dy, const void* t_o, int dtype, const int32_t* idx,
                               const int32_t* slot, const int32_t* kept, const float* weights, int64_t T,
                               int64_t M, int64_t E, int k, int64_t capacity, int n_chunks, float* dprob,
                               void* g_o, void* stream) {
  if (int rc = check_common(dtype, M, (int)E, k)) return rc;
  MPM_CHECK_ARG(dprob != nullptr || g_o != nullptr, "combine_bwd: nothing to compute (dprob and g_o NULL)");
  cudaStream_t s = (cudaStream_t)stream;
  if (capacity == 0) {
    if (T > 0 && dprob) MPM_CUDA_RET(cudaMemsetAsync(dprob, 0, T * k * sizeof(float), s));
    return 0;
  }
  ChunkGeom g(capacity, n_chunks);
  int64_t vpr = M * dtype_size(dtype) / 16;
  const int64_t items = T + (g_o ? zero_items<32>(E, capacity) : 0);
  MPM_CHECK_ARG(E * capacity < (int64_t(1) << 31), "E*C too large (%lld)", (long long)(E * capacity));
  auto launch = [&](auto tag, auto km) -> cudaError_t {
    using TT = decltype(tag);
    constexpr int KM = decltype(km)::value;
#define MPM_CB(DP, GO)                                                                                       \
  ::mpm::pdl_launch(combine_bwd_kernel<TT, KM, DP, GO>,                                                      \
                    dim3(persistent_grid<combine_bwd_kernel<TT, KM, DP, GO>>(256, items)), dim3(256), 0, s, \
                    (const uint4*)dy, (const uint4*)t_o, idx, slot, weights, T, (int)E, k, g, vpr, dprob,   \
                    (uint4*)g_o, kept)
    if (dprob && g_o) return MPM_CB(true, true);
    if (dprob) return MPM_CB(true, false);
    return MPM_CB(false, true);
#undef MPM_CB
  };
  MPM_CUDA_RET(dispatch_k(dtype, k, launch));
  note_launch();
  return 0;
}

namespace mpm { bool gate_bwd_tensor_path(int dtype, int64_t T, int64_t M, int64_t E); }

extern "C" int mpm_combine_bwd_gate(const void* dy, const void* t_o, int dtype, const int32_t* idx,
                                    const int32_t* slot, const int32_t* kept, const float* weights,
                                    const float* logits, int64_t T, int64_t M, int64_t E, int k, int renorm,
                                    int64_t capacity, int n_chunks, void* g_o, float* dprob, float* dlogits,
                                    void* gate_ws, void* stream) {
  if (int rc = check_common(dtype, M, (int)E, k)) return rc;
  MPM_CHECK_ARG(dlogits != nullptr && gate_ws != nullptr, "combine_bwd_gate: dlogits and the gate workspace are required");
  MPM_CHECK_ARG(capacity >= 0 && E * capacity < (int64_t(1) << 31), "E*C too large (%lld)", (long long)(E * capacity));
  if (T == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  const bool cap0 = capacity == 0;
  ChunkGeom g(cap0 ? 1 : capacity, cap0 ? 1 : n_chunks);
  void* go = cap0 ? nullptr : g_o;  // C = 0: every assignment dropped, no rows to write
  int64_t vpr = M * dtype_size(dtype) / 16;
  // split operands for the tcgen05 gate GEMMs (dlc only for the dense gate term: the top-k
  // renormalised gradient is sparse and enters dx in the gather)
  __nv_bfloat16 *dla = nullptr, *dlc = nullptr;
  int64_t Ec = ceil_div(E, 32) * 32;
  if (gate_bwd_tensor_path(dtype, T, M, E)) {
    const GateBwdOperands op = gate_bwd_operands(T, M, E, gate_ws);
    dla = op.dla;
    dlc = (k > 1 && renorm) ? nullptr : op.dlc;
    Ec = op.Ec;
  }
  const int64_t items = T + (go ? zero_items<32>(E, g.C) : 0);
  auto launch = [&](auto tag, auto km) -> cudaError_t {
    using TT = decltype(tag);
    constexpr int KM = decltype(km)::value;
#define MPM_CBG(GO)                                                                                            \
  ::mpm::pdl_launch(combine_bwd_gate_kernel<TT, KM, GO>,                                                        \
                    dim3(persistent_grid<combine_bwd_gate_kernel<TT, KM, GO>>(256, items)), dim3(256), 0, s,   \
                    (const uint4*)dy, (const uint4*)t_o, idx, slot, weights, logits, T, (int)E, (int)Ec, k,    \
                    renorm, g, vpr, dprob, (uint4*)go, kept, dlogits, dla, dlc)
    if (go) return MPM_CBG(true);
    return MPM_CBG(false);
#undef MPM_CBG
  };
  MPM_CUDA_RET(dispatch_k(dtype, k, launch));
  note_launch();
  return 0;
}

extern "C" int mpm_gate_bwd_logits(const float* logits, const int32_t* idx, const float* weights,
                                   const float* dprob, int64_t T, int64_t E, int k, int renorm, float* dlogits,
                                   void* stream) {
  if (int rc = check_common(MPM_F32, 4, (int)E, k)) return rc;
  if (T == 0) return 0;
  MPM_PDL_LAUNCH(gate_bwd_logits_kernel, dim3((unsigned)ceil_div(T, 8)), dim3(256), 0, (cudaStream_t)stream, logits,
                 idx, weights, dprob, T, (int)E, k, renorm, dlogits);
  return 0;
}

