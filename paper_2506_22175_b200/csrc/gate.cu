// Gate (router) GEMMs on tensor cores with fp32-accurate split precision.
//
// The gate is replicated / data parallel with E*M fp32
// parameters (Eq. 1).  Its three GEMMs are tiny next to the
// expert FFN (6*M*E vs 12*k*M*H flops per token) but GEMM-shaped, so they
// run on tcgen05 like the experts, in "bf16x3" split precision:
//
//   an fp32 value v is carried as three bf16 terms h = bf16(v),
//   l = bf16(v - h), l2 = bf16(v - h - l) (24 mantissa bits in total);
//   bf16 x bf16 products are exact in the fp32 TMEM accumulator.
//
//   logits = x . Wg^T     x (bf16, exact) against [Wg_h; Wg_l; Wg_l2] stacked
//                         along N (3E columns, one pass over x), then a
//                         fixed-order sum of the three partial logits
//   dWg    = dl^T . x     [dl_h; dl_l; dl_l2] against x (b_k_period = T),
//                         split-K over the token dimension + fixed-order reduce
//   dx_g   = dl . Wg      [dl_h | dl_l | dl_h] . [Wg_h; Wg_h; Wg_l] (the
//                         three leading cross terms, ~2^-16 relative)
//
// so logits and dWg carry fp32-level accuracy and every result is a fixed
// order sum (deterministic).  Any expert count runs here: the expert axis of
// every split operand is padded with zeros to Ec = E rounded up to 32 (the
// epilogue's column slice), so E = 4 / 8 / 48 take the same kernels as
// E = 64.  fp32 activations (the parity configuration) take the exact-fp32
// FMA kernels instead.
#include <type_traits>
#include "common.cuh"

namespace mpm {
int simt_gemm_launch(const mpm_gemm_args* a, int a_dtype, int b_dtype, cudaStream_t s);
namespace sm100 { int run(const mpm_gemm_args* a, cudaStream_t s, const RouteEpi* route = nullptr); }

constexpr int MAX_K_GATE = 8;

// src [rows][cols] f32 -> n_slots bf16 copies of the terms named by
// `pattern` (2 bits per slot).  stack == 0: dst[r][s*cols_pad + c]
// (concatenated along columns); stack == 1: dst[s*rows_pad + r][c].
// Padding (c >= cols or r >= rows) is written as zero.
__global__ void split_kernel(const float* __restrict__ src, int64_t rows, int64_t cols, int n_slots,
                             uint32_t pattern, int stack, int64_t rows_pad, int64_t cols_pad,
                             __nv_bfloat16* __restrict__ dst) {
  pdl_begin();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t r = (uint32_t)i / (uint32_t)cols_pad, c = (uint32_t)i - (uint32_t)r * (uint32_t)cols_pad;
  if (r >= rows_pad) return;
  __nv_bfloat16 t[3];
  const float v = (r < rows && c < cols) ? src[r * cols + c] : 0.f;
  split3(v, t);
  for (int sl = 0; sl < n_slots; ++sl) {
    const int term = (pattern >> (2 * sl)) & 3;
    if (stack) dst[((int64_t)sl * rows_pad + r) * cols_pad + c] = t[term];
    else dst[r * (n_slots * cols_pad) + (int64_t)sl * cols_pad + c] = t[term];
  }
}

// logits[t][e] = (p[t][e] + p[t][P+e]) + p[t][2P+e]: the h / l / l2 partial logits
// of the stacked-term gate GEMM (pitch P = Ec per term), summed in a fixed order;
// four experts per thread (E % 4 == 0, P % 4 == 0 on this path).
__global__ void __launch_bounds__(256)
sum3_kernel(const float* __restrict__ part, int64_t T, int64_t E, int64_t P, float* __restrict__ logits) {
  pdl_begin();
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= T * E / 4) return;
  const uint32_t qe = (uint32_t)(E / 4);
  const int64_t t = (uint32_t)q / qe, e = ((uint32_t)q - (uint32_t)t * qe) * 4;
  const float* r = part + t * 3 * P + e;
  const float4 a = __ldg(reinterpret_cast<const float4*>(r));
  const float4 b = __ldg(reinterpret_cast<const float4*>(r + P));
  const float4 c = __ldg(reinterpret_cast<const float4*>(r + 2 * P));
  *reinterpret_cast<float4*>(logits + t * E + e) =
      make_float4((a.x + b.x) + c.x, (a.y + b.y) + c.y, (a.z + b.z) + c.z, (a.w + b.w) + c.w);
}
// same, one expert per thread (E % 4 != 0)
__global__ void __launch_bounds__(256)
sum3_scalar_kernel(const float* __restrict__ part, int64_t T, int64_t E, int64_t P, float* __restrict__ logits) {
  pdl_begin();
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= T * E) return;
  const int64_t t = (uint32_t)q / (uint32_t)E, e = (uint32_t)q - (uint32_t)t * (uint32_t)E;
  const float* r = part + t * 3 * P + e;
  logits[t * E + e] = (__ldg(r) + __ldg(r + P)) + __ldg(r + 2 * P);
}

// dx[t] = base + sum_j g_i[row_j].  Dense gate gradient (SPARSE = false): in place, dx already
// holds the gate term dlogits[t] . Wg (written there by the gate GEMM), so no [T][M] scratch
// exists.  Sparse gate gradient (SPARSE: top-k renormalisation, k > 1, where dlogits has only
// the k chosen experts nonzero): base = sum_j dlogits[t][idx_j] * Wg[idx_j] in exact fp32 from
// the k Wg rows (E x M fp32, L2-resident), so the gate term costs no GEMM and no dx round trip.
// One warp per token (persistent grid-stride), 16-byte vectors, all KM rows' loads in flight
// before the adds, fixed summation order.
template <typename T, int KM, bool SPARSE>
__global__ void __launch_bounds__(256, 3)
gather_kernel(const uint4* __restrict__ g_i, const int32_t* __restrict__ idx, const int32_t* __restrict__ slot,
              int64_t Tn, int64_t M, int E, int k, ChunkGeom g, T* dx, const float* __restrict__ dlogits,
              const float* __restrict__ wg) {
  pdl_begin();
  constexpr int NV = 16 / sizeof(T);
  constexpr int CU = KM <= 2 ? 4 : (KM == 4 ? 2 : 1);
  const int lane = threadIdx.x & 31;
  const int64_t vpr = M / NV;
  MPM_WARP_LOOP(t, Tn) {
    int64_t rows[KM];
    int ex[KM];
    float dl[KM];
#pragma unroll
    for (int j = 0; j < KM; ++j) {
      const int32_t s = j < k ? slot[t * k + j] : -1;
      ex[j] = j < k ? idx[t * k + j] : 0;
      rows[j] = s < 0 ? -1 : g.row(E, ex[j], s);
      dl[j] = (SPARSE && j < k) ? __ldg(dlogits + t * E + ex[j]) : 0.f;
    }
    uint4* drow = reinterpret_cast<uint4*>(dx + t * M);
    for (int64_t v0 = 0; v0 < vpr; v0 += 32 * CU) {
      uint4 base[CU], add[KM][CU];
      if (!SPARSE) {
#pragma unroll
        for (int u = 0; u < CU; ++u) {
          const int64_t v = v0 + lane + 32 * u;
          base[u] = v < vpr ? drow[v] : make_uint4(0, 0, 0, 0);
        }
      }
#pragma unroll
      for (int j = 0; j < KM; ++j)
#pragma unroll
        for (int u = 0; u < CU; ++u) {
          const int64_t v = v0 + lane + 32 * u;
          add[j][u] = (rows[j] >= 0 && v < vpr) ? __ldg(g_i + rows[j] * vpr + v) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
      for (int u = 0; u < CU; ++u) {
        const int64_t v = v0 + lane + 32 * u;
        float acc[NV];
        if (SPARSE) {
#pragma unroll
          for (int i = 0; i < NV; ++i) acc[i] = 0.f;
          if (v < vpr) {
#pragma unroll
            for (int j = 0; j < KM; ++j) {  // gate term, fixed order j = 0..k-1
              if (j >= k) break;
              const float4* wr = reinterpret_cast<const float4*>(wg + (int64_t)ex[j] * M + v * NV);
#pragma unroll
              for (int q = 0; q < NV / 4; ++q) {
                const float4 wv = __ldg(wr + q);
                acc[4 * q] = fmaf(dl[j], wv.x, acc[4 * q]);
                acc[4 * q + 1] = fmaf(dl[j], wv.y, acc[4 * q + 1]);
                acc[4 * q + 2] = fmaf(dl[j], wv.z, acc[4 * q + 2]);
                acc[4 * q + 3] = fmaf(dl[j], wv.w, acc[4 * q + 3]);
              }
            }
          }
        } else {
          const T* h0 = reinterpret_cast<const T*>(&base[u]);
#pragma unroll
          for (int i = 0; i < NV; ++i) acc[i] = to_f32(h0[i]);
        }
#pragma unroll
        for (int j = 0; j < KM; ++j) {
          if (rows[j] < 0) continue;
          const T* h = reinterpret_cast<const T*>(&add[j][u]);
#pragma unroll
          for (int i = 0; i < NV; ++i) acc[i] += to_f32(h[i]);
        }
        if (v >= vpr) continue;
        uint4 out;
        T* o = reinterpret_cast<T*>(&out);
#pragma unroll
        for (int i = 0; i < NV; ++i) o[i] = from_f32<T>(acc[i]);
        drow[v] = out;
      }
    }
  }
}

template <typename T, bool SPARSE = false>
static cudaError_t launch_gather(const void* g_i, const int32_t* idx, const int32_t* slot, int64_t T_, int64_t M,
                                 int E, int k, ChunkGeom g, void* dx, cudaStream_t s,
                                 const float* dlogits = nullptr, const float* wg = nullptr) {
  auto go = [&](auto km) -> cudaError_t {
    constexpr int KM = decltype(km)::value;
    auto kern = gather_kernel<T, KM, SPARSE>;
    return pdl_launch(kern, dim3(persistent_grid<gather_kernel<T, KM, SPARSE>>(256, T_)), dim3(256), 0, s,
                      (const uint4*)g_i, idx, slot, T_, M, E, k, g, (T*)dx, dlogits, wg);
  };
  if (k <= 1) return go(std::integral_constant<int, 1>{});
  if (k <= 2) return go(std::integral_constant<int, 2>{});
  if (k <= 4) return go(std::integral_constant<int, 4>{});
  return go(std::integral_constant<int, 8>{});
}

// dlogits through the routing weights (softmax Jacobian; top-k renormalisation when k > 1 and
// renorm) from a given dprob, one token per warp, emitted as fp32 dlogits and the split operands
// dla / dlc (GateBwdOperands, common.cuh).  The layer's backward computes dprob and this in one
// pass instead (combine_bwd_gate_kernel, csrc/routing.cu).
template <int KM>
__global__ void __launch_bounds__(256)
gate_bwd_split_kernel(const float* __restrict__ logits, const int32_t* __restrict__ idx,
                      const float* __restrict__ w, const float* __restrict__ dprob, int64_t Tn, int E, int Ec,
                      int k, int renorm, float* __restrict__ dlogits, __nv_bfloat16* __restrict__ dla,
                      __nv_bfloat16* __restrict__ dlc) {
  pdl_begin();
  const int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= Tn) return;
  int ex[KM];
  float wv[KM], dp[KM];
#pragma unroll
  for (int j = 0; j < KM; ++j) {
    ex[j] = j < k ? idx[t * k + j] : -1;
    wv[j] = j < k ? w[t * k + j] : 0.f;
    dp[j] = j < k ? dprob[t * k + j] : 0.f;
  }
  gate_token_dlogits<KM>(logits + t * E, ex, wv, dp, k, E, Ec, k > 1 && renorm, lane, dlogits + t * E,
                         dla ? dla + t * 3 * Ec : nullptr, dlc ? dlc + t * 3 * Ec : nullptr);
}

// dWg[e][m] = sum over the split-K partials part[s][3Ec][M] of dla^T x of the three term rows
// ((h + l) + l2).  One block per 128 columns of one expert row: warp w sums splits w, w + 8, ... in
// order (coalesced 512 B loads, a warp's splits all in flight), then warp 0 adds the eight warp
// sums in order — a fixed summation order (bitwise reproducible, identical on every rank).  (The
// previous warp-per-four-columns form read 16 B per split row per lane, half of every sector.)
__global__ void __launch_bounds__(256)
dwg_reduce_kernel(const float* __restrict__ part, int64_t splits, int64_t Ec, int64_t E, int64_t M,
                  float* __restrict__ dwg) {
  pdl_begin();
  __shared__ float4 red[8][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t mb = ceil_div(M, 128);
  const int64_t e = blockIdx.x / mb, m = (blockIdx.x % mb) * 128 + lane * 4;
  const bool ok = e < E && m < M;
  const int64_t term = Ec * M, stride = 3 * Ec * M;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (ok) {
#pragma unroll 4
    for (int64_t sp = warp; sp < splits; sp += 8) {
      const float* p = part + sp * stride + e * M + m;
      const float4 h = __ldg(reinterpret_cast<const float4*>(p));
      const float4 l = __ldg(reinterpret_cast<const float4*>(p + term));
      const float4 l2 = __ldg(reinterpret_cast<const float4*>(p + 2 * term));
      acc.x += (h.x + l.x) + l2.x; acc.y += (h.y + l.y) + l2.y;
      acc.z += (h.z + l.z) + l2.z; acc.w += (h.w + l.w) + l2.w;
    }
  }
  red[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && ok) {
    float4 t = red[0][lane];
#pragma unroll
    for (int w = 1; w < 8; ++w) {
      const float4 v = red[w][lane];
      t.x += v.x; t.y += v.y; t.z += v.z; t.w += v.w;
    }
    *reinterpret_cast<float4*>(dwg + e * M + m) = t;
  }
}

struct GateGeom {
  int64_t T, M, E;
  int64_t Tp, Mp, Ep, Ec;  // padded to 64 / 64 / 8 / 32
  GateGeom(int64_t T_, int64_t M_, int64_t E_)
      : T(T_), M(M_), E(E_), Tp(ceil_div(T_, 64) * 64), Mp(ceil_div(M_, 64) * 64), Ep(ceil_div(E_, 8) * 8),
        Ec(ceil_div(E_, 32) * 32) {}
  int64_t splits() const {  // split-K count for dWg (dlogits given): ~one wave of 148 SMs
    const int64_t tiles = ceil_div(E, 128) * ceil_div(M, 256);
    int64_t s = 148 / (tiles > 0 ? tiles : 1);
    return s < 1 ? 1 : (s > 64 ? 64 : s);
  }
  // split-K count of the fused backward's dWg (rows = the 3Ec term rows; 2-CTA 256-row tiles when
  // 3Ec > 128): ~one wave of tiles, at least 4 k-blocks of tokens per split
  int64_t bwd_splits() const {
    const bool pair = 3 * Ec > 128 && M > 128;
    const int64_t tiles = ceil_div(3 * Ec, pair ? 256 : 128) * ceil_div(M, 256);
    const int64_t units = pair ? 74 : 148;
    int64_t s = units / (tiles > 0 ? tiles : 1);
    const int64_t cap = ceil_div(T, 256);
    s = s > cap ? cap : s;
    return s < 1 ? 1 : (s > 64 ? 64 : s);
  }
  // bf16 workspace needs (bytes), each segment 256-aligned
  static size_t al(size_t b) { return (b + 255) & ~size_t(255); }
  // forward: stacked terms [3Ec][Mp] bf16 | partial logits [T][3Ec] f32
  size_t fwd_bytes() const { return al(Ec * 3 * Mp * 2) + al(T * 3 * Ec * 4); }
  size_t wgrad_bytes() const { return al(3 * Tp * Ec * 2) + al(splits() * E * M * 4); }
  size_t gather_bytes() const { return al(T * 3 * Ep * 2) + al(3 * Ep * M * 2); }
  // fused backward: dla | dlc | wst | partials  (the gate term of dx goes straight into dx)
  size_t off_dlc() const { return al(T * 3 * Ec * 2); }
  size_t off_wst() const { return off_dlc() + al(T * 3 * Ec * 2); }
  size_t off_part() const { return off_wst() + al(3 * Ec * M * 2); }
  size_t bwd_bytes() const {
    const int64_t sp = bwd_splits() > splits() ? bwd_splits() : splits();
    return off_part() + al(sp * 3 * Ec * M * 4);
  }
};

GateBwdOperands gate_bwd_operands(int64_t T, int64_t M, int64_t E, void* workspace) {
  GateGeom g(T, M, E);
  char* ws = static_cast<char*>(workspace);
  return {reinterpret_cast<__nv_bfloat16*>(ws), reinterpret_cast<__nv_bfloat16*>(ws + g.off_dlc()), g.Ec};
}

// tcgen05 path: bf16 activations, M a multiple of 64 (the K period of the
// split-precision operand equals the operand's true K extent, so a 64-wide K
// block never straddles terms); any E (padded to Ec in the split operands).
static bool tc_ok(int x_dtype, int64_t M, int64_t E) {
  return x_dtype == MPM_BF16 && M % 64 == 0 && E > 0;
}

static int split(const float* src, int64_t rows, int64_t cols, int n_slots, uint32_t pattern, int stack,
                 int64_t rows_pad, int64_t cols_pad, void* dst, cudaStream_t s) {
  const int64_t n = rows_pad * cols_pad;
  if (n == 0) return 0;
  MPM_CHECK_ARG(n < (int64_t(1) << 31), "split: %lld elements", (long long)n);
  MPM_PDL_LAUNCH(split_kernel, dim3((unsigned)ceil_div(n, 256)), dim3(256), 0, s, src, rows, cols, n_slots, pattern,
                 stack, rows_pad, cols_pad, static_cast<__nv_bfloat16*>(dst));
  return 0;
}

}  // namespace mpm

using namespace mpm;

extern "C" size_t mpm_gate_workspace_bytes(int64_t T, int64_t M, int64_t E) {
  GateGeom g(T, M, E);
  size_t b = g.fwd_bytes();
  if (g.wgrad_bytes() > b) b = g.wgrad_bytes();
  if (g.gather_bytes() > b) b = g.gather_bytes();
  if (g.bwd_bytes() > b) b = g.bwd_bytes();
  return b;
}

namespace mpm {
// The gate GEMM.  tcgen05 path: the three bf16 terms of Wg stacked along N ([Wg_h; Wg_l; Wg_l2],
// each term Ec = E rounded up to 32 rows, zero-padded) give the three partial logits side by side in
// one pass over x; *parts points at them ([T][3Ec] f32 in the workspace, term pitch *pitch = Ec) and
// the caller sums them in a fixed order (sum3_kernel, or the routing kernel when fused).
// Exact-fp32 path: logits written directly, *parts = nullptr.
int gate_partials(const void* x, int x_dtype, const float* wg, int64_t T, int64_t M, int64_t E, float* logits,
                  void* workspace, cudaStream_t s, const float** parts, int64_t* pitch) {
  MPM_CHECK_ARG(x_dtype == MPM_F32 || x_dtype == MPM_BF16, "unsupported dtype %d", x_dtype);
  *parts = nullptr;
  mpm_gemm_args a{};
  a.epilogue = MPM_EPI_NONE;
  a.batches = 1; a.rows = T; a.n = E;
  a.a = x; a.a_ld = M; a.a_mn_major = 0;
  a.c = logits; a.c_ld = E; a.c_dtype = MPM_F32;
  if (!tc_ok(x_dtype, M, E)) {
    a.dtype = x_dtype; a.k = M;
    a.b = wg; a.b_ld = M; a.b_mn_major = 0;
    return simt_gemm_launch(&a, x_dtype, MPM_F32, s);
  }
  MPM_CHECK_ARG(workspace != nullptr, "gate workspace required");
  GateGeom g(T, M, E);
  void* wst = workspace;
  float* part = reinterpret_cast<float*>(static_cast<char*>(workspace) + GateGeom::al(g.Ec * 3 * g.Mp * 2));
  if (int rc = split(wg, E, M, 3, 0b100100u, 1, g.Ec, g.Mp, wst, s)) return rc;  // zero rows E..Ec-1
  a.dtype = MPM_BF16; a.epilogue = MPM_EPI_STORE_F32;
  a.n = 3 * g.Ec; a.k = M;
  a.b = wst; a.b_ld = g.Mp; a.b_mn_major = 0;
  a.c = part; a.c_ld = 3 * g.Ec;
  if (int rc = sm100::run(&a, s)) return rc;
  *parts = part;
  *pitch = g.Ec;
  return 0;
}

// Gate GEMM with the routing in its epilogue (E <= 64: one N tile holds the three stacked terms):
// logits, idx, weights and the per-block counts come straight out of TMEM, so the [T][3Ec] partial
// logits never reach memory and no routing kernel runs.  Returns -1 (nothing launched) when the
// shape needs the two-kernel route, else a status code.
int gate_route_fused(const void* x, int x_dtype, const float* wg, int64_t T, int64_t M, int64_t E, int k, int renorm,
                     float* logits, int32_t* idx, float* weights, int32_t* counts, void* workspace, cudaStream_t s) {
  GateGeom g(T, M, E);
  if (!tc_ok(x_dtype, M, E) || g.Ec > 64 || workspace == nullptr) return -1;
  void* wst = workspace;
  if (int rc = split(wg, E, M, 3, 0b100100u, 1, g.Ec, g.Mp, wst, s)) return rc;  // zero rows E..Ec-1
  mpm_gemm_args a{};
  a.dtype = MPM_BF16; a.epilogue = MPM_EPI_STORE_F32;
  a.batches = 1; a.rows = T; a.n = 3 * g.Ec; a.k = M;
  a.a = x; a.a_ld = M; a.a_mn_major = 0;
  a.b = wst; a.b_ld = g.Mp; a.b_mn_major = 0;
  a.c = logits; a.c_ld = 3 * g.Ec; a.c_dtype = MPM_F32;  // never stored: the epilogue writes the routing outputs
  RouteEpi r{};
  r.T = T; r.E = (int)E; r.Ec = (int)g.Ec; r.k = k; r.renorm = renorm; r.nblk = (int)ceil_div(T, 32);
  r.logits = logits; r.idx = idx; r.weights = weights; r.counts = counts;
  return sm100::run(&a, s, &r);
}
}  // namespace mpm

extern "C" int mpm_gate_fwd(const void* x, int x_dtype, const float* wg, float* logits, int64_t T, int64_t M,
                            int64_t E, void* workspace, void* stream) {
  if (T == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  const float* part = nullptr;
  int64_t pitch = 0;
  if (int rc = gate_partials(x, x_dtype, wg, T, M, E, logits, workspace, s, &part, &pitch)) return rc;
  if (!part) return 0;
  MPM_CHECK_ARG(T * E < (int64_t(1) << 31), "gate: T*E too large");
  if (E % 4 == 0)
    MPM_PDL_LAUNCH(sum3_kernel, dim3((unsigned)ceil_div(T * E / 4, 256)), dim3(256), 0, s, part, T, E, pitch, logits);
  else
    MPM_PDL_LAUNCH(sum3_scalar_kernel, dim3((unsigned)ceil_div(T * E, 256)), dim3(256), 0, s, part, T, E, pitch,
                   logits);
  return 0;
}

extern "C" int mpm_gate_wgrad(const float* dlogits, const void* x, int x_dtype, int64_t T, int64_t M, int64_t E,
                              float* dwg, void* workspace, void* stream) {
  MPM_CHECK_ARG(x_dtype == MPM_F32 || x_dtype == MPM_BF16, "unsupported dtype %d", x_dtype);
  cudaStream_t s = (cudaStream_t)stream;
  if (T == 0) { MPM_CUDA_RET(cudaMemsetAsync(dwg, 0, E * M * sizeof(float), s)); return 0; }
  mpm_gemm_args a{};
  a.epilogue = MPM_EPI_STORE_F32;
  a.batches = 1; a.rows = E; a.n = M;
  a.b = x; a.b_ld = M; a.b_mn_major = 1;          // B(m, t) = x[t][m]
  a.c = dwg; a.c_ld = M; a.c_dtype = MPM_F32;
  if (!tc_ok(x_dtype, M, E) || T % 64 != 0) {
    a.dtype = x_dtype; a.k = T;
    a.a = dlogits; a.a_ld = E; a.a_mn_major = 1;  // A(e, t) = dlogits[t][e]
    // the output is tiny (E x M) and K = T long: split K over ~2 waves of blocks
    const int64_t tiles = ceil_div(E, 64) * ceil_div(M, 64);
    int64_t splits = ceil_div(296, tiles);
    const int64_t max_splits = ceil_div(T, 256);  // >= 256 tokens per split
    if (splits > max_splits) splits = max_splits;
    if (splits > GateGeom(T, M, E).splits()) splits = GateGeom(T, M, E).splits();  // workspace bound
    if (splits <= 1 || workspace == nullptr) return simt_gemm_launch(&a, MPM_F32, x_dtype, s);
    float* part = static_cast<float*>(workspace);
    a.c = part; a.k_splits = splits; a.split_stride = E * M;
    if (int rc = simt_gemm_launch(&a, MPM_F32, x_dtype, s)) return rc;
    return mpm_splitk_reduce(part, splits, E * M, E * M, dwg, MPM_F32, 0, stream);
  }
  MPM_CHECK_ARG(workspace != nullptr, "gate workspace required");
  GateGeom g(T, M, E);
  char* ws = static_cast<char*>(workspace);
  void* dl3 = ws;                                   // [3][Tp][Ec] bf16: dl_h; dl_l; dl_l2
  float* part = reinterpret_cast<float*>(ws + GateGeom::al(3 * g.Tp * g.Ec * 2));
  if (int rc = split(dlogits, T, E, 3, 0b100100u, 1, g.Tp, g.Ec, dl3, s)) return rc;
  a.dtype = MPM_BF16;
  a.k = 3 * g.Tp; a.b_k_period = g.Tp;
  a.a = dl3; a.a_ld = g.Ec; a.a_mn_major = 1;
  a.c = part; a.k_splits = g.splits(); a.split_stride = E * M;
  if (int rc = sm100::run(&a, s)) return rc;
  // the kernel may merge splits so that none is empty: recompute the count it used
  const int64_t kblocks = ceil_div(a.k, 64);
  const int64_t per = ceil_div(kblocks, g.splits() < kblocks ? g.splits() : kblocks);
  return mpm_splitk_reduce(part, ceil_div(kblocks, per), E * M, E * M, dwg, MPM_F32, 0, stream);
}

extern "C" int mpm_gather_bwd(const void* g_i, int dtype, const int32_t* idx, const int32_t* slot,
                              const float* dlogits, const float* wg, int64_t T, int64_t M, int64_t E, int k,
                              int64_t capacity, int n_chunks, void* dx, void* workspace, void* stream) {
  MPM_CHECK_ARG(dtype == MPM_F32 || dtype == MPM_BF16, "unsupported dtype %d", dtype);
  MPM_CHECK_ARG(k >= 1 && k <= MAX_K_GATE, "top_k %d unsupported", k);
  MPM_CHECK_ARG((M * (int64_t)dtype_size(dtype)) % 16 == 0, "row bytes must be a multiple of 16");
  MPM_CHECK_ARG(workspace != nullptr, "gate workspace required");
  if (T == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  GateGeom gg(T, M, E);
  char* ws = static_cast<char*>(workspace);
  mpm_gemm_args a{};
  a.epilogue = MPM_EPI_NONE;
  a.batches = 1; a.rows = T; a.n = M;
  const bool tc = tc_ok(dtype, M, E);
  // the gate term dl . Wg is written into dx itself; the gather then adds the rows in place
  a.c = dx; a.c_ld = M; a.c_dtype = dtype;
  if (!tc) {
    a.dtype = MPM_F32; a.k = E;
    a.a = dlogits; a.a_ld = E; a.a_mn_major = 0;
    a.b = wg; a.b_ld = M; a.b_mn_major = 1;        // B(m, e) = wg[e][m]
    if (int rc = simt_gemm_launch(&a, MPM_F32, MPM_F32, s)) return rc;
  } else {
    void* dlc = ws;                                                   // [T][3*Ep]: dl_h | dl_l | dl_h
    void* wst = ws + GateGeom::al(T * 3 * gg.Ep * 2);                 // [3*Ep][M]: Wg_h; Wg_h; Wg_l
    if (int rc = split(dlogits, T, E, 3, 0b000100u, 0, T, gg.Ep, dlc, s)) return rc;
    if (int rc = split(wg, E, M, 3, 0b010000u, 1, gg.Ep, M, wst, s)) return rc;
    a.dtype = MPM_BF16; a.k = 3 * gg.Ep;
    a.a = dlc; a.a_ld = 3 * gg.Ep; a.a_mn_major = 0;
    a.b = wst; a.b_ld = M; a.b_mn_major = 1;
    if (int rc = sm100::run(&a, s)) return rc;
  }
  ChunkGeom g(capacity > 0 ? capacity : 1, n_chunks);
  MPM_CUDA_RET(dtype == MPM_BF16 ? launch_gather<__nv_bfloat16>(g_i, idx, slot, T, M, (int)E, k, g, dx, s)
                                  : launch_gather<float>(g_i, idx, slot, T, M, (int)E, k, g, dx, s));
  note_launch();
  return 0;
}

static bool gate_bwd_tc(int dtype, int64_t T, int64_t M, int64_t E) { return tc_ok(dtype, M, E) && T % 64 == 0 && T > 0; }

namespace mpm {
bool gate_bwd_tensor_path(int dtype, int64_t T, int64_t M, int64_t E) { return gate_bwd_tc(dtype, T, M, E); }

// dWg = dl^T x from the split operand dla [T][3Ec] in the workspace: the three term rows stacked
// along M (3Ec rows; 2-CTA 256-row tiles when 3Ec > 128), so each N tile streams its x columns
// once; split-K over tokens into [splits][3Ec][M] fp32 partials, then the fixed-order term and
// split reduce (dwg_reduce_kernel).
static int gate_dwg_from_operands(const void* x, int64_t T, int64_t M, int64_t E, float* dwg, void* workspace,
                                  cudaStream_t s) {
  GateGeom gg(T, M, E);
  char* ws = static_cast<char*>(workspace);
  float* part = reinterpret_cast<float*>(ws + gg.off_part());
  mpm_gemm_args a{};
  a.dtype = MPM_BF16; a.epilogue = MPM_EPI_STORE_F32;
  a.batches = 1; a.rows = 3 * gg.Ec; a.n = M; a.k = T;
  a.a = ws; a.a_ld = 3 * gg.Ec; a.a_mn_major = 1;   // A(r, t) = dla[t][r]
  a.b = x; a.b_ld = M; a.b_mn_major = 1;            // B(m, t) = x[t][m]
  a.c = part; a.c_ld = M; a.c_dtype = MPM_F32;
  a.k_splits = gg.bwd_splits(); a.split_stride = 3 * gg.Ec * M;
  if (int rc = sm100::run(&a, s)) return rc;
  const int64_t kblocks = ceil_div(T, 64);  // the kernel merges splits so that none is empty
  const int64_t per = ceil_div(kblocks, a.k_splits < kblocks ? a.k_splits : kblocks);
  MPM_CHECK_ARG(M % 4 == 0, "dWg reduce: M %% 4 != 0 (M=%lld)", (long long)M);
  MPM_PDL_LAUNCH(dwg_reduce_kernel, dim3((unsigned)(E * ceil_div(M, 128))), dim3(256), 0, s, (const float*)part,
                 ceil_div(kblocks, per), gg.Ec, E, M, dwg);
  return 0;
}

// Dense gate term dx = dl . Wg (three leading cross terms: dlc [T][3Ec] h|l|h against
// [Wg_h; Wg_h; Wg_l]), written into dx; the gather then adds the expert rows in place.
static int gate_dx_dense(const float* wg, int64_t T, int64_t M, int64_t E, void* dx, void* workspace,
                         cudaStream_t s) {
  GateGeom gg(T, M, E);
  char* ws = static_cast<char*>(workspace);
  void* wst = ws + gg.off_wst();
  if (int rc = split(wg, E, M, 3, 0b010000u, 1, gg.Ec, M, wst, s)) return rc;  // Wg_h; Wg_h; Wg_l (zero rows >= E)
  mpm_gemm_args d{};
  d.dtype = MPM_BF16; d.epilogue = MPM_EPI_NONE;
  d.batches = 1; d.rows = T; d.n = M; d.k = 3 * gg.Ec;
  d.a = ws + gg.off_dlc(); d.a_ld = 3 * gg.Ec; d.a_mn_major = 0;
  d.b = wst; d.b_ld = M; d.b_mn_major = 1;
  d.c = dx; d.c_ld = M; d.c_dtype = MPM_BF16;
  return sm100::run(&d, s);
}
}  // namespace mpm

extern "C" int mpm_gate_backward_gate(const float* logits, const int32_t* idx, const float* weights,
                                      const float* dprob, const void* x, int dtype, const float* wg, int64_t T,
                                      int64_t M, int64_t E, int k, int renorm, float* dlogits, float* dwg,
                                      void* dx, void* workspace, void* stream) {
  MPM_CHECK_ARG(dtype == MPM_F32 || dtype == MPM_BF16, "unsupported dtype %d", dtype);
  MPM_CHECK_ARG(k >= 1 && k <= MAX_K_GATE && E <= 256, "top_k %d / E %lld unsupported", k, (long long)E);
  MPM_CHECK_ARG(workspace != nullptr, "gate workspace required");
  cudaStream_t s = (cudaStream_t)stream;
  if (!gate_bwd_tc(dtype, T, M, E)) {
    // exact-fp32 route: dlogits kernel, then the FMA gate GEMM (dl . wg is fused into the gather)
    if (int rc = mpm_gate_bwd_logits(logits, idx, weights, dprob, T, E, k, renorm, dlogits, stream)) return rc;
    return mpm_gate_wgrad(dlogits, x, dtype, T, M, E, dwg, workspace, stream);
  }
  const GateBwdOperands op = gate_bwd_operands(T, M, E, workspace);
  auto go = [&](auto km) -> cudaError_t {
    constexpr int KM = decltype(km)::value;
    return pdl_launch(gate_bwd_split_kernel<KM>, dim3((unsigned)ceil_div(T, 8)), dim3(256), 0, s, logits, idx,
                      weights, dprob, T, (int)E, (int)op.Ec, k, renorm, dlogits, op.dla, op.dlc);
  };
  MPM_CUDA_RET(k <= 1 ? go(std::integral_constant<int, 1>{}) : k <= 2 ? go(std::integral_constant<int, 2>{})
               : k <= 4 ? go(std::integral_constant<int, 4>{}) : go(std::integral_constant<int, 8>{}));
  note_launch();
  if (int rc = gate_dwg_from_operands(x, T, M, E, dwg, workspace, s)) return rc;
  return gate_dx_dense(wg, T, M, E, dx, workspace, s);  // dx = dl Wg; the gather adds the expert rows
}

extern "C" int mpm_gate_backward_gemms(const void* x, int dtype, const float* wg, const float* dlogits, int64_t T,
                                       int64_t M, int64_t E, int k, int renorm, float* dwg, void* dx,
                                       void* workspace, void* stream) {
  MPM_CHECK_ARG(dtype == MPM_F32 || dtype == MPM_BF16, "unsupported dtype %d", dtype);
  MPM_CHECK_ARG(k >= 1 && k <= MAX_K_GATE && E <= 256, "top_k %d / E %lld unsupported", k, (long long)E);
  MPM_CHECK_ARG(workspace != nullptr, "gate workspace required");
  cudaStream_t s = (cudaStream_t)stream;
  if (!gate_bwd_tc(dtype, T, M, E))  // exact fp32: FMA dWg; the dense dx term is computed by mpm_gate_gather
    return mpm_gate_wgrad(dlogits, x, dtype, T, M, E, dwg, workspace, stream);
  if (int rc = gate_dwg_from_operands(x, T, M, E, dwg, workspace, s)) return rc;
  if (k > 1 && renorm) return 0;  // sparse gate gradient: the gather adds the term from the Wg rows
  return gate_dx_dense(wg, T, M, E, dx, workspace, s);
}

extern "C" int mpm_gate_gather(const void* g_i, int dtype, const int32_t* idx, const int32_t* slot,
                               const float* dlogits, const float* wg, int64_t T, int64_t M, int64_t E, int k,
                               int renorm, int64_t capacity, int n_chunks, void* dx, void* workspace, void* stream) {
  MPM_CHECK_ARG(dtype == MPM_F32 || dtype == MPM_BF16, "unsupported dtype %d", dtype);
  MPM_CHECK_ARG(k >= 1 && k <= MAX_K_GATE, "top_k %d unsupported", k);
  MPM_CHECK_ARG((M * (int64_t)dtype_size(dtype)) % 16 == 0, "row bytes must be a multiple of 16");
  MPM_CHECK_ARG(workspace != nullptr, "gate workspace required");
  if (T == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  ChunkGeom g(capacity > 0 ? capacity : 1, n_chunks);
  if (k > 1 && renorm) {
    MPM_CHECK_ARG((reinterpret_cast<uintptr_t>(wg) & 15) == 0, "wg must be 16-byte aligned");
    const cudaError_t e = dtype == MPM_BF16
                              ? launch_gather<__nv_bfloat16, true>(g_i, idx, slot, T, M, (int)E, k, g, dx, st, dlogits, wg)
                              : launch_gather<float, true>(g_i, idx, slot, T, M, (int)E, k, g, dx, st, dlogits, wg);
    MPM_CUDA_RET(e);
    note_launch();
    return 0;
  }
  if (!gate_bwd_tc(dtype, T, M, E))
    return mpm_gather_bwd(g_i, dtype, idx, slot, dlogits, wg, T, M, E, k, capacity, n_chunks, dx, workspace, stream);
  MPM_CUDA_RET(launch_gather<__nv_bfloat16>(g_i, idx, slot, T, M, (int)E, k, g, dx, st));
  note_launch();
  return 0;
}

extern "C" int mpm_gate_backward_gather(const void* g_i, int dtype, const int32_t* idx, const int32_t* slot,
                                        const float* dlogits, const float* wg, int64_t T, int64_t M, int64_t E,
                                        int k, int64_t capacity, int n_chunks, void* dx, void* workspace,
                                        void* stream) {
  MPM_CHECK_ARG(dtype == MPM_F32 || dtype == MPM_BF16, "unsupported dtype %d", dtype);
  MPM_CHECK_ARG(workspace != nullptr, "gate workspace required");
  if (!gate_bwd_tc(dtype, T, M, E))
    return mpm_gather_bwd(g_i, dtype, idx, slot, dlogits, wg, T, M, E, k, capacity, n_chunks, dx, workspace, stream);
  ChunkGeom g(capacity > 0 ? capacity : 1, n_chunks);
  MPM_CUDA_RET(launch_gather<__nv_bfloat16>(g_i, idx, slot, T, M, (int)E, k, g, dx, (cudaStream_t)stream));
  note_launch();
  return 0;
}

extern "C" int mpm_gate_backward(const float* logits, const int32_t* idx, const float* weights, const float* dprob,
                                 const void* x, const void* g_i, const int32_t* slot, int dtype, const float* wg,
                                 int64_t T, int64_t M, int64_t E, int k, int renorm, int64_t capacity, int n_chunks,
                                 float* dlogits, void* dx, float* dwg, void* workspace, void* stream) {
  if (int rc = mpm_gate_backward_gate(logits, idx, weights, dprob, x, dtype, wg, T, M, E, k, renorm, dlogits, dwg,
                                      dx, workspace, stream))
    return rc;
  return mpm_gate_backward_gather(g_i, dtype, idx, slot, dlogits, wg, T, M, E, k, capacity, n_chunks, dx, workspace,
                                  stream);
}
