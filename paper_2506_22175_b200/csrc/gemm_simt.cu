// Exact-fp32 batched GEMM on the FMA pipe.
//
// Used for (a) the fp32 parity configuration (BASELINE.json configs[0]:
// "fp32 (CPU reference oracle)"), where tcgen05 kind::tf32 would miss the
// north-star fp32 tolerance (rtol 1e-5), and (b) the small fp32 gate GEMMs
// (E x M weights).  The K loop runs in index order, so every
// output is a fixed-order fp32 sum (bit-reproducible).  Split-K (k_splits > 1,
// one batch): split s sums its contiguous K range into the f32 partial at
// c + s*split_stride; mpm_splitk_reduce adds the partials in split order.
#include "common.cuh"

namespace mpm {

constexpr int SB_M = 64, SB_N = 64, SB_K = 16;

template <typename TA, typename TB>
__global__ void __launch_bounds__(256)
simt_gemm_kernel(mpm_gemm_args p) {
  __shared__ float As[SB_K][SB_M + 4];
  __shared__ float Bs[SB_K][SB_N + 4];
  const bool split = p.k_splits > 1;
  const int64_t b = split ? 0 : blockIdx.z;
  const int64_t m0 = (int64_t)blockIdx.y * SB_M, n0 = (int64_t)blockIdx.x * SB_N;
  if (p.valid_rows && m0 >= p.valid_rows[b]) return;
  const TA* A = reinterpret_cast<const TA*>(p.a) + b * p.a_batch_stride;
  const TB* B = reinterpret_cast<const TB*>(p.b) + b * p.b_batch_stride;
  // this block's K range (the whole K unless split)
  const int64_t k_per = split ? (p.k + p.k_splits - 1) / p.k_splits : p.k;
  const int64_t k_lo = split ? (int64_t)blockIdx.z * k_per : 0;
  int64_t k_hi = split ? (k_lo + k_per < p.k ? k_lo + k_per : p.k) : p.k;
  if (p.valid_k && p.valid_k[b] < k_hi) k_hi = p.valid_k[b] < k_lo ? k_lo : p.valid_k[b];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  for (int64_t k0 = k_lo; k0 < k_hi; k0 += SB_K) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int i = tid + 256 * q;
      int kk, mm;
      if (p.a_mn_major) { mm = i & 63; kk = i >> 6; } else { kk = i & 15; mm = i >> 4; }
      int64_t m = m0 + mm, k = k0 + kk;
      float v = 0.f;
      if (m < p.rows && k < k_hi) v = to_f32(p.a_mn_major ? A[k * p.a_ld + m] : A[m * p.a_ld + k]);
      As[kk][mm] = v;
      int nn;
      if (p.b_mn_major) { nn = i & 63; kk = i >> 6; } else { kk = i & 15; nn = i >> 4; }
      int64_t n = n0 + nn;
      k = k0 + kk;
      float u = 0.f;
      if (n < p.n && k < k_hi) u = to_f32(p.b_mn_major ? B[k * p.b_ld + n] : B[n * p.b_ld + k]);
      Bs[kk][nn] = u;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SB_K; ++kk) {
      float a[4], bb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bb[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], bb[j], acc[i][j]);
    }
    __syncthreads();
  }

#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t m = m0 + ty * 4 + i;
    if (m >= p.rows) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int64_t n = n0 + tx * 4 + j;
      if (n >= p.n) continue;
      float v = acc[i][j];
      int64_t co = (split ? (int64_t)blockIdx.z * p.split_stride : b * p.c_batch_stride) + m * p.c_ld + n;
      int64_t ao = b * p.aux_batch_stride + m * p.aux_ld + n;
      switch (p.epilogue) {
        case MPM_EPI_RELU: v = fmaxf(v, 0.f); break;
        case MPM_EPI_DRELU: {
          float g = p.dtype == MPM_BF16 ? to_f32(reinterpret_cast<const __nv_bfloat16*>(p.aux)[ao])
                                        : reinterpret_cast<const float*>(p.aux)[ao];
          v = g > 0.f ? v : 0.f;
          break;
        }
        case MPM_EPI_ACCUM_F32: v += reinterpret_cast<float*>(p.c)[co]; break;
        case MPM_EPI_ACCUM:
          v += p.c_dtype == MPM_BF16 ? __bfloat162float(reinterpret_cast<__nv_bfloat16*>(p.c)[co])
                                     : reinterpret_cast<float*>(p.c)[co];
          break;
        case MPM_EPI_ADD_AUX_F32: v += reinterpret_cast<const float*>(p.aux)[ao]; break;
        default: break;
      }
      if (p.c_dtype == MPM_BF16) reinterpret_cast<__nv_bfloat16*>(p.c)[co] = __float2bfloat16_rn(v);
      else reinterpret_cast<float*>(p.c)[co] = v;
    }
  }
}

int simt_gemm_launch(const mpm_gemm_args* a, int a_dtype, int b_dtype, cudaStream_t s) {
  MPM_CHECK_ARG(a->epilogue != MPM_EPI_RELU_MASK && a->epilogue != MPM_EPI_DMASK,
                "ReLU-mask epilogues are tcgen05-path features (bf16 operands)");
  MPM_CHECK_ARG(a->rows >= 0 && a->n >= 0 && a->k >= 0 && a->batches >= 0, "negative GEMM extent");
  MPM_CHECK_ARG(a->batches < 65536, "too many batches");
  if (a->rows == 0 || a->n == 0 || a->batches == 0) return 0;
  const bool split = a->k_splits > 1;
  if (split)
    MPM_CHECK_ARG(a->batches == 1 && a->c_dtype == MPM_F32 &&
                      (a->epilogue == MPM_EPI_STORE_F32 || a->epilogue == MPM_EPI_NONE) && a->split_stride > 0,
                  "simt split-K: one batch, f32 partials (EPI_STORE_F32) with a split stride");
  dim3 grid((unsigned)ceil_div(a->n, SB_N), (unsigned)ceil_div(a->rows, SB_M),
            (unsigned)(split ? a->k_splits : a->batches));
  MPM_CHECK_ARG(grid.y < 65536, "too many row tiles");
  if (a_dtype == MPM_F32 && b_dtype == MPM_F32) simt_gemm_kernel<float, float><<<grid, 256, 0, s>>>(*a);
  else if (a_dtype == MPM_BF16 && b_dtype == MPM_BF16)
    simt_gemm_kernel<__nv_bfloat16, __nv_bfloat16><<<grid, 256, 0, s>>>(*a);
  else if (a_dtype == MPM_BF16 && b_dtype == MPM_F32)
    simt_gemm_kernel<__nv_bfloat16, float><<<grid, 256, 0, s>>>(*a);
  else if (a_dtype == MPM_F32 && b_dtype == MPM_BF16)
    simt_gemm_kernel<float, __nv_bfloat16><<<grid, 256, 0, s>>>(*a);
  else { set_error("simt gemm: bad dtypes %d/%d", a_dtype, b_dtype); return MPM_ERR_INVALID; }
  MPM_LAUNCH_CHECK("simt_gemm_kernel");
  return 0;
}

int validate_gemm(const mpm_gemm_args* a) {
  MPM_CHECK_ARG(a != nullptr, "null gemm args");
  MPM_CHECK_ARG(a->dtype == MPM_F32 || a->dtype == MPM_BF16, "bad operand dtype %d", a->dtype);
  MPM_CHECK_ARG(a->c_dtype == MPM_F32 || a->c_dtype == MPM_BF16, "bad output dtype %d", a->c_dtype);
  MPM_CHECK_ARG(a->epilogue >= MPM_EPI_NONE && a->epilogue <= MPM_EPI_ACCUM, "bad epilogue %d", a->epilogue);
  if (a->epilogue == MPM_EPI_RELU_MASK || a->epilogue == MPM_EPI_DMASK)
    MPM_CHECK_ARG(a->aux != nullptr, "ReLU-mask epilogues need the mask buffer (aux)");
  if (a->epilogue == MPM_EPI_STORE_F32 || a->epilogue == MPM_EPI_ACCUM_F32)
    MPM_CHECK_ARG(a->c_dtype == MPM_F32, "epilogue %d needs an f32 output", a->epilogue);
  if (a->epilogue == MPM_EPI_DRELU || a->epilogue == MPM_EPI_ADD_AUX_F32)
    MPM_CHECK_ARG(a->aux != nullptr, "epilogue %d needs aux", a->epilogue);
  return 0;
}

}  // namespace mpm

extern "C" int mpm_grouped_gemm_simt(const mpm_gemm_args* args, void* stream) {
  if (int rc = mpm::validate_gemm(args)) return rc;
  return mpm::simt_gemm_launch(args, args->dtype, args->dtype, (cudaStream_t)stream);
}
