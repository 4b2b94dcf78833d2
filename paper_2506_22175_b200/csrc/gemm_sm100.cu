// Batched expert GEMM on 5th-gen tensor cores (tcgen05 + TMEM + TMA), sm_100a.
//
// Realises the GeMM units of the reference schedule: C_i (fc1 + fc2,
// pipesim/schedule.py:253), RE_i (recompute, :327-332), G2_i / G1_i
// (dgrad + wgrad, :335-339).  One batch per local expert; every batch has
// the same (capacity-padded) row count, so a single persistent launch covers
// all experts of a chunk.
//
// Structure (one CTA per SM, persistent over (expert, n-tile, m-tile) with
// m fastest so consecutive CTAs share the weight tile through L2; the wide
// expert GEMMs run as 2-CTA clusters, cta_group::2, 256 x 256 pair tiles):
//   warp 0      TMA producer: ring of {A 128x64, B (BN or BN/2)x64} bf16
//               stages (6 for pairs, 4 single-CTA; ~192 KiB), 128B-swizzled,
//               K-major boxes or, for MN-major operands, one 4-D box per k-slab
//   warp 1      MMA issuer (the pair leader): one thread issues tcgen05.mma
//               (M 256 x N 256 x K 16 per pair, 128 x BN single-CTA) into a
//               double-buffered TMEM accumulator (2 x BN fp32 columns)
//   warp 2      TMEM allocator
//   warps 4-7   epilogue: tcgen05.ld 32x32b -> registers -> fused ReLU (+1-bit
//               mask) / mask' / fp32 or bf16 accumulate -> swizzled smem ->
//               TMA store or TMA reduce-add (64-column boxes for bf16)
// Launched with programmatic dependent launch: the prologue (barriers, TMEM,
// tensor-map prefetch) overlaps the previous kernel's tail.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include "common.cuh"

namespace mpm {
int simt_gemm_launch(const mpm_gemm_args* a, int a_dtype, int b_dtype, cudaStream_t s);
int validate_gemm(const mpm_gemm_args* a);

namespace sm100 {

int run(const mpm_gemm_args* a, cudaStream_t s, const RouteEpi* route = nullptr);

constexpr int BM = 128, BK = 64;
constexpr int A_STAGE = BM * BK * 2;       // 16 KiB
constexpr int MN_BLOCK_BYTES = BK * 128;   // one 64-wide MN block of a 64-deep K slab
// Epilogue staging for TMA stores: per epilogue warp two 4 KiB buffers, each
// one 32-row slice of 128 B rows (fp32: 32 columns; bf16: 64 columns, or 32
// columns in 64 B rows when N < 64), swizzled like the tensor map so the
// row-per-thread writes are bank-conflict free.
constexpr int EPI_BUF = 4096;

// Per-(BN, PAIR) configuration: N tile, pipeline depth (~192 KiB of stages),
// TMEM columns.  PAIR = 2-CTA cluster issuing cta_group::2 MMAs of M = 256:
// each CTA stages its own 128 A rows and half of the BN B rows.
// EW = epilogue warps: 4 (one per TMEM lane quarter) or 8 (two per quarter, each taking half of
// the tile's columns) for store-bound GEMMs with few k-blocks per tile; 8 warps' staging costs a
// ring stage.
// staging buffers per warp of the 8-warp epilogue (1 keeps six ring stages but serialises each
// warp's stores: measured slower both at K=80 (1.293 vs 1.280 ms layer step) and K=512)
#ifndef EPI_NB8
#define EPI_NB8 2
#endif
template <int BN, bool PAIR = false, int EW = 4>
struct Cfg {
  static constexpr int B_STAGE = (PAIR ? BN / 2 : BN) * BK * 2;
  static constexpr int STAGE_BYTES = A_STAGE + B_STAGE;
  static constexpr int EPI_NB = EW == 4 ? 2 : EPI_NB8;  // staging buffers per epilogue warp
  static constexpr int EPI_BYTES = EW * EPI_NB * EPI_BUF;
  static constexpr int BUDGET = (EPI_BYTES <= 32 * 1024 ? 192 : 160) * 1024;
  static constexpr int STAGES = BUDGET / STAGE_BYTES > 8 ? 8 : BUDGET / STAGE_BYTES;
  static constexpr int TMEM_COLS = 2 * BN;  // double-buffered accumulator
  static constexpr int THREADS_ = 128 + 32 * EW;
  static constexpr size_t SMEM_BYTES = (size_t)STAGES * STAGE_BYTES + 1024 + 256 + EPI_BYTES;
};

struct Params {
  int64_t rows, n, k;
  int64_t m_tiles, n_tiles, k_blocks, total_tiles, tiles_per_split;
  int64_t k_splits, kb_per_split, split_stride;  // split-K: partial outputs at c + s*split_stride
  int64_t a_k_period, b_k_period;                // K-periodic operands (0 = off)
  void* c; int64_t c_ld, c_bs; int c_dtype;
  const void* aux; int64_t aux_ld, aux_bs;
  const int32_t* valid_rows;
  const int32_t* valid_k;  // per-batch K limit (weight gradients of under-filled experts)
  int epilogue;
  int op_dtype;
  int use_tma;     // TMA store / reduce-add of the output tile
  int wide_store;  // bf16 output staged 64 columns per TMA store (128B swizzle) instead of 32
  int a_mn4, b_mn4;  // MN-major operand loaded as one 4-D box per k-slab (MN extent % 64 == 0)
  RouteEpi route;    // the gate GEMM's routing epilogue (ROUTE instantiations only)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// 4-D load: an MN-major operand viewed as {64 MN, K, MN/64 blocks, batch} so one
// TMA op brings every 64-wide MN block of a k-slab ([blocks][K][64] in smem).
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d_pair(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                                 int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, "
      "%6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on the barrier at the same smem offset in CTA `rank` of the cluster
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
// 2-SM TMA load: data lands in this CTA's smem, bytes are counted on the
// leader CTA's barrier (peer bit cleared, as CUTLASS SM100_TMA_2SM_LOAD does)
__device__ __forceinline__ void tma_load_3d_pair(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                                 int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void umma_pair(uint32_t d_tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
// commit of the pair's MMAs, arriving on the barrier at this offset in both CTAs
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// Shared-memory matrix descriptor, SWIZZLE_128B, sm100 version bit.
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// Instruction descriptor: D f32, A/B bf16, M=128, N=bn.
__host__ __device__ constexpr uint32_t make_idesc(bool a_mn, bool b_mn, int bn, int bm = BM) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(bn >> 3) << 17) | ((uint32_t)(bm >> 4) << 24);
}

__device__ __forceinline__ void umma(uint32_t d_tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// 64 consecutive accumulator columns of this thread's TMEM lane in one load and one wait (the wide bf16
// epilogue's two 32-column slices): half the load-to-use round trips of two tmem_ld32 calls.
__device__ __forceinline__ void tmem_ld64(uint32_t taddr, uint32_t (&r)[64]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];\n"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(taddr)
      : "memory");
}

// Tile t -> (split, batch, n-tile, m-tile), m fastest; k-block range of the split.
// 32-bit index math (the host checks total_tiles < 2^31): the MMA issuer decodes
// the next tile between two tiles' MMAs, and 64-bit division is a long
// emulated sequence on that single thread.
template <int BN, int TILE_M = BM>
__device__ __forceinline__ bool decode_tile(const Params& p, int64_t t64, int64_t& b, int64_t& m0, int64_t& n0,
                                            int64_t& kb0, int64_t& kb1, int64_t& split) {
  const uint32_t t = (uint32_t)t64;
  const uint32_t mt_n = (uint32_t)p.m_tiles;
  const uint32_t per_b = mt_n * (uint32_t)p.n_tiles;
  const uint32_t per_s = (uint32_t)p.tiles_per_split;
  const uint32_t sp = per_s ? t / per_s : 0u;
  const uint32_t r0 = t - sp * per_s;
  const uint32_t bb = r0 / per_b;
  const uint32_t r = r0 - bb * per_b;
  const uint32_t nt = r / mt_n, mt = r - nt * mt_n;
  split = sp;
  b = bb;
  m0 = (int64_t)mt * TILE_M;
  n0 = (int64_t)nt * BN;
  kb0 = split * p.kb_per_split;
  kb1 = kb0 + p.kb_per_split < p.k_blocks ? kb0 + p.kb_per_split : p.k_blocks;
  if (p.valid_k) {  // K rows past the expert's routed tokens are padding: stop at the covering block
    const int64_t kv = ((int64_t)p.valid_k[b] + BK - 1) / BK;
    kb1 = kb1 < kv ? kb1 : kv;
    kb1 = kb1 > kb0 ? kb1 : kb0;  // kb1 == kb0: a zero tile (no MMA; the epilogue writes zeros)
  }
  return !(p.valid_rows && m0 >= p.valid_rows[b]);
}

// Direct epilogue (row per thread) for the epilogues that read a dense aux
// tensor (ADD_AUX_F32, DRELU with a bf16 aux): 32 consecutive columns.
__device__ __forceinline__ void epilogue_store(const Params& p, int64_t b, int64_t m, int64_t n, int64_t split,
                                               const uint32_t (&r)[32]) {
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
  const int64_t co = split * p.split_stride + b * p.c_bs + m * p.c_ld + n;
  switch (p.epilogue) {
    case MPM_EPI_RELU:
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
      break;
    case MPM_EPI_DRELU: {
      const uint4* ap = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(p.aux) +
                                                       b * p.aux_bs + m * p.aux_ld + n);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 u = ap[q];
        const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[q * 8 + i] = __bfloat162float(h[i]) > 0.f ? v[q * 8 + i] : 0.f;
      }
      break;
    }
    case MPM_EPI_ACCUM_F32: {
      const float4* cp = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(p.c) + co);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float4 u = cp[q];
        v[4 * q] += u.x; v[4 * q + 1] += u.y; v[4 * q + 2] += u.z; v[4 * q + 3] += u.w;
      }
      break;
    }
    case MPM_EPI_ACCUM:
      if (p.c_dtype == MPM_BF16) {
        const uint4* cp = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(p.c) + co);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 u = cp[q];
          const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
          for (int i = 0; i < 8; ++i) v[q * 8 + i] += __bfloat162float(h[i]);
        }
      } else {
        const float4* cp = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(p.c) + co);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          float4 u = cp[q];
          v[4 * q] += u.x; v[4 * q + 1] += u.y; v[4 * q + 2] += u.z; v[4 * q + 3] += u.w;
        }
      }
      break;
    case MPM_EPI_ADD_AUX_F32: {
      const float4* ap = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(p.aux) + b * p.aux_bs +
                                                         m * p.aux_ld + n);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float4 u = ap[q];
        v[4 * q] += u.x; v[4 * q + 1] += u.y; v[4 * q + 2] += u.z; v[4 * q + 3] += u.w;
      }
      break;
    }
    default: break;
  }
  if (p.c_dtype == MPM_BF16) {
    uint32_t w[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      __nv_bfloat162 h2 = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
      w[i] = *reinterpret_cast<uint32_t*>(&h2);
    }
    __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.c) + co;
    if ((reinterpret_cast<uintptr_t>(dst) & 31) == 0) {  // two 256-bit stores: one full 32-byte sector each
#pragma unroll
      for (int q = 0; q < 2; ++q)
        asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst + 16 * q),
                     "r"(w[8 * q]), "r"(w[8 * q + 1]), "r"(w[8 * q + 2]), "r"(w[8 * q + 3]), "r"(w[8 * q + 4]),
                     "r"(w[8 * q + 5]), "r"(w[8 * q + 6]), "r"(w[8 * q + 7])
                     : "memory");
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        reinterpret_cast<uint4*>(dst)[q] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
    }
  } else {
    float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(p.c) + co);
#pragma unroll
    for (int q = 0; q < 8; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  }
}


// Routing epilogue of the gate GEMM (one thread = one token row of the accumulator; the three bf16x3
// partial logits of expert e sit in columns e, Ec + e, 2Ec + e; Ec <= 64).  Bit-identical to
// route_kernel over the stored partials: the same fixed-order partial sum, the same top-k (value,
// then lowest index: a strict total order, so any reduction tree selects the same experts), the same
// softmax denominator order (8 interleaved partial sums e = g (mod 8), combined as route_kernel's
// three xor rounds combine its 8 lanes).  The top-k is k selection passes, each a depth-6 max tree
// over the 64 logits held in registers (an insertion list over 64 experts is a ~4K-instruction
// dependent chain per thread: 35 us for the 128-row tiles at configs[1]).
// MPM_EPI_PROBE builds only (tools/epi_probe.py): SM-clock cycles spent in each wait of the
// warp roles, summed over CTAs (slot meanings in tools/epi_probe.py).
#ifdef MPM_EPI_PROBE
__device__ unsigned long long g_epi_probe[16];
#define PROBE_T(v) const long long v = clock64()
#define PROBE_ADD(slot, t0) (probe_acc[slot] += (unsigned long long)(clock64() - (t0)))
#else
#define PROBE_T(v)
#define PROBE_ADD(slot, t0)
#endif

__device__ __forceinline__ void route_epilogue(const RouteEpi& R, uint32_t tbase, int64_t row0, int lane) {
  constexpr int KX = 8;
  constexpr int NONE = 0x7fffffff;
  const int64_t t = row0 + lane;
  const bool valid = t < R.T;
#ifdef MPM_EPI_PROBE
  const long long rq0 = clock64();
  long long rq1 = 0, rq2 = 0, rq3 = 0;
#endif
  float lg[64];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (h * 32 >= R.Ec) {
#pragma unroll
      for (int i = 0; i < 32; ++i) lg[h * 32 + i] = -INFINITY;
      continue;
    }
    uint32_t a[32], b[32];
    tmem_ld32(tbase + h * 32, a);
    tmem_ld32(tbase + R.Ec + h * 32, b);
#pragma unroll
    for (int i = 0; i < 32; ++i) lg[h * 32 + i] = __uint_as_float(a[i]) + __uint_as_float(b[i]);
    tmem_ld32(tbase + 2 * R.Ec + h * 32, a);
#pragma unroll
    for (int i = 0; i < 32; ++i) lg[h * 32 + i] += __uint_as_float(a[i]);
  }
#ifdef MPM_EPI_PROBE
  rq1 = clock64();
#endif
  if (valid) {
    float* out = R.logits + t * R.E;
    if ((R.E & 3) == 0) {
#pragma unroll
      for (int q = 0; q < 16; ++q)
        if (4 * q < R.E)
          reinterpret_cast<float4*>(out)[q] = make_float4(lg[4 * q], lg[4 * q + 1], lg[4 * q + 2], lg[4 * q + 3]);
    } else {
#pragma unroll
      for (int i = 0; i < 64; ++i)
        if (i < R.E) out[i] = lg[i];
    }
  }
#ifdef MPM_EPI_PROBE
  rq2 = clock64();
#endif
  // k selection passes; `sel` marks the experts already chosen (and the padded ones, never chosen)
  uint64_t sel = R.E >= 64 ? 0ull : ~((1ull << R.E) - 1ull);
  float tv[KX];
  int ti[KX];
  auto pick = [](float& bv, int& bi, float v, int i) {
    if (v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
  };
#pragma unroll
  for (int j = 0; j < KX; ++j) {
    tv[j] = -INFINITY;
    ti[j] = NONE;
    if (j >= R.k) continue;
    float gv[8];
    int gi[8];
#pragma unroll
    for (int g = 0; g < 8; ++g) {  // groups of 8 leaves, then the 8 group winners
      gv[g] = -INFINITY;
      gi[g] = NONE;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = 8 * g + u;
        if (!((sel >> e) & 1ull)) pick(gv[g], gi[g], lg[e], e);
      }
    }
#pragma unroll
    for (int g = 0; g < 8; ++g) pick(tv[j], ti[j], gv[g], gi[g]);
    sel |= 1ull << (ti[j] & 63);
  }
  const float mx = tv[0];
  float den = 0.f;
  if (R.k > 1 && R.renorm) {
#pragma unroll
    for (int j = 0; j < KX; ++j)
      if (j < R.k) den += expf(tv[j] - mx);
  } else {
    float pp[8];
#pragma unroll
    for (int g = 0; g < 8; ++g) pp[g] = 0.f;
#pragma unroll
    for (int i = 0; i < 64; ++i)
      if (i < R.E) pp[i & 7] += expf(lg[i] - mx);
    den = ((pp[0] + pp[1]) + (pp[2] + pp[3])) + ((pp[4] + pp[5]) + (pp[6] + pp[7]));
  }
  if (valid) {
#pragma unroll
    for (int j = 0; j < KX; ++j) {
      if (j >= R.k) break;
      R.idx[t * R.k + j] = ti[j];
      R.weights[t * R.k + j] = expf(tv[j] - mx) / den;
    }
  }
#ifdef MPM_EPI_PROBE
  rq3 = clock64();
#endif
  // this warp's 32 rows are one routing block: its per-(k-rank, expert) counts (zeros, then the
  // count of every chosen expert written by the first lane that chose it)
  const int64_t blk = row0 / 32;
  if (blk < R.nblk) {
#pragma unroll
    for (int j = 0; j < KX; ++j) {
      if (j >= R.k) break;
      int32_t* cnt = R.counts + ((int64_t)j * R.nblk + blk) * R.E;
      for (int e = lane; e < R.E; e += 32) cnt[e] = 0;
      __syncwarp();
      const unsigned peers = __match_any_sync(0xffffffffu, valid ? ti[j] : -1 - lane);
      if (valid && (peers & ((1u << lane) - 1u)) == 0u) cnt[ti[j]] = __popc(peers);
      __syncwarp();
    }
  }
#ifdef MPM_EPI_PROBE
  if (lane == 0) {
    const long long rq4 = clock64();
    atomicAdd(&g_epi_probe[12], (unsigned long long)(rq1 - rq0));  // TMEM loads + partial sums
    atomicAdd(&g_epi_probe[13], (unsigned long long)(rq2 - rq1));  // logits row stores
    atomicAdd(&g_epi_probe[14], (unsigned long long)(rq3 - rq2));  // top-k, softmax, idx / weights
    atomicAdd(&g_epi_probe[15], (unsigned long long)(rq4 - rq3));  // block counts
  }
#endif
}


template <bool A_MN, bool B_MN, int BN, bool PAIR, int EW = 4, bool ROUTE = false>
// 8-warp epilogue: registers capped so ~16K of the SM's 64K stay free for the co-resident exchange copy
// kernel and the gather (256 x 40 and 256 x ~100 registers) beside the persistent CTA
__global__ void __launch_bounds__(128 + 32 * EW) __maxnreg__(EW == 8 ? 128 : 168)
umma_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const __grid_constant__ CUtensorMap tmC, const Params p) {
  using K = Cfg<BN, PAIR, EW>;
  constexpr int TILE_M = PAIR ? 2 * BM : BM;  // rows per (cluster) tile
  constexpr int B_ROWS = PAIR ? BN / 2 : BN;  // B rows staged by this CTA
  constexpr int STAGES = K::STAGES;
  constexpr int STAGE_BYTES = K::STAGE_BYTES;
  PROBE_T(k_entry);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* epi_smem = smem + STAGES * STAGE_BYTES;  // 1 KiB aligned
  uint64_t* full = reinterpret_cast<uint64_t*>(epi_smem + K::EPI_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = PAIR ? cluster_rank() : 0;
  const bool leader = rank == 0;
  // cluster tiles: both CTAs of a pair walk the same tile sequence
  const int64_t first_tile = PAIR ? (blockIdx.x >> 1) : blockIdx.x;
  const int64_t tile_step = PAIR ? (gridDim.x >> 1) : gridDim.x;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], PAIR ? 2 : 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], PAIR ? 2 * EW : EW); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    if (p.use_tma) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmC)) : "memory");
  }
  if (warp == 2) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(K::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(K::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  if (PAIR) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
#ifdef MPM_EPI_PROBE
  unsigned long long probe_acc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#endif
  pdl_wait();  // prologue done; from here on global memory of the previous kernel is read/written
#ifdef MPM_EPI_PROBE
  if (threadIdx.x == 32) PROBE_ADD(9, k_entry);  // entry -> after the dependency wait
#endif

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t t = first_tile; t < p.total_tiles; t += tile_step) {
      int64_t b, m0, n0, kb0, kb1, split;
      if (!decode_tile<BN, TILE_M>(p, t, b, m0, n0, kb0, kb1, split)) continue;
      const int am0 = (int)(m0 + rank * BM);      // this CTA's A rows
      const int bn0 = (int)(n0 + rank * B_ROWS);  // this CTA's B rows
      for (int64_t kb = kb0; kb < kb1; ++kb) {
        PROBE_T(pe0);
        mbar_wait(&empty[stage], phase ^ 1);
        PROBE_ADD(0, pe0);
        if (!PAIR) mbar_expect_tx(&full[stage], STAGE_BYTES);
        else if (leader) mbar_expect_tx(&full[stage], 2 * STAGE_BYTES);
        else mbar_arrive_cluster(&full[stage], 0);
        uint8_t* sa = smem + stage * STAGE_BYTES;
        uint8_t* sb = sa + A_STAGE;
        const int64_t kk = kb * BK;
        const int ka = (int)(p.a_k_period ? kk % p.a_k_period : kk);
        const int kbb = (int)(p.b_k_period ? kk % p.b_k_period : kk);
        auto load = [&](void* dst, const CUtensorMap* map, int c0, int c1) {
          if (PAIR) tma_load_3d_pair(dst, map, &full[stage], c0, c1, (int)b);
          else tma_load_3d(dst, map, &full[stage], c0, c1, (int)b);
        };
        auto load4 = [&](void* dst, const CUtensorMap* map, int c1, int c2) {
          if (PAIR) tma_load_4d_pair(dst, map, &full[stage], 0, c1, c2, (int)b);
          else tma_load_4d(dst, map, &full[stage], 0, c1, c2, (int)b);
        };
        if (!A_MN) {
          load(sa, &tmA, ka, am0);
        } else if (p.a_mn4) {
          load4(sa, &tmA, ka, am0 / 64);
        } else {
#pragma unroll
          for (int j = 0; j < BM / 64; ++j) load(sa + j * MN_BLOCK_BYTES, &tmA, am0 + 64 * j, ka);
        }
        if (!B_MN) {
          load(sb, &tmB, kbb, bn0);
        } else if (p.b_mn4) {
          load4(sb, &tmB, kbb, bn0 / 64);
        } else {
#pragma unroll
          for (int j = 0; j < B_ROWS / 64; ++j) load(sb + j * MN_BLOCK_BYTES, &tmB, bn0 + 64 * j, kbb);
        }
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1 && lane == 0 && leader) {
    // ---------------- MMA issuer (the leader CTA issues for the pair)
    constexpr uint32_t idesc = make_idesc(A_MN, B_MN, BN, TILE_M);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    PROBE_T(mt0);
    for (int64_t t = first_tile; t < p.total_tiles; t += tile_step) {
      int64_t b, m0, n0, kb0, kb1, split;
      if (!decode_tile<BN, TILE_M>(p, t, b, m0, n0, kb0, kb1, split)) continue;
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      PROBE_T(me0);
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      PROBE_ADD(1, me0);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int64_t kb = kb0; kb < kb1; ++kb) {
        PROBE_T(mf0);
        mbar_wait(&full[stage], phase);
        PROBE_ADD(2, mf0);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
        const uint32_t sb = sa + A_STAGE;
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk) {
          const uint64_t da = A_MN ? make_desc(sa + kk * 2048, MN_BLOCK_BYTES, 1024) : make_desc(sa + kk * 32, 16, 1024);
          const uint64_t db = B_MN ? make_desc(sb + kk * 2048, MN_BLOCK_BYTES, 1024) : make_desc(sb + kk * 32, 16, 1024);
          if (PAIR) umma_pair(d_tmem, da, db, idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
          else umma(d_tmem, da, db, idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
        }
        if (PAIR) umma_commit_pair(&empty[stage]); else umma_commit(&empty[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (PAIR) umma_commit_pair(&tfull[acc]); else umma_commit(&tfull[acc]);
      ++it;
    }
    PROBE_ADD(8, mt0);
  } else if (warp >= 4) {
    // ---------------- epilogue
    const int ew = warp - 4;
    const int qw = ew & 3;  // TMEM lane quarter this warp may access (warp id % 4)
    constexpr int CC_PER = (BN / 32) / (EW / 4);  // 32-column slices per warp
    const int cc_lo = EW == 4 ? 0 : (ew >> 2) * CC_PER, cc_hi = cc_lo + CC_PER;
    uint8_t* stg = epi_smem + ew * K::EPI_NB * EPI_BUF;
    const bool f32_out = p.c_dtype == MPM_F32;
    int buf = 0;
    int it = 0;
    for (int64_t t = first_tile; t < p.total_tiles; t += tile_step) {
      int64_t b, m0, n0, kb0, kb1, split;
      if (!decode_tile<BN, TILE_M>(p, t, b, m0, n0, kb0, kb1, split)) continue;
      m0 += rank * BM;  // this CTA's rows of the (pair) tile
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int64_t m = m0 + qw * 32 + lane;
      const bool row_ok = m < p.rows;
      // ReLU-mask words of this row for the whole tile, issued before the accumulator wait
      uint32_t mw[BN / 32];
      if (p.epilogue == MPM_EPI_DMASK) {
        const uint32_t* mp = reinterpret_cast<const uint32_t*>(p.aux) + b * p.aux_bs + m * p.aux_ld + n0 / 32;
#pragma unroll
        for (int cc = 0; cc < BN / 32; ++cc) mw[cc] = (row_ok && n0 + cc * 32 < p.n) ? __ldg(mp + cc) : 0u;
      }
      PROBE_T(ef0);
      mbar_wait(&tfull[acc], acc_phase);
      if (lane == 0) PROBE_ADD(3, ef0);
      PROBE_T(et0);
      tc_fence_after();
      const bool zero_tile = kb1 <= kb0;  // no k-block (valid_k == 0): the tile is all zeros
#if defined(MPM_EPI_SKIP) && MPM_EPI_SKIP >= 3  // probe builds: release the accumulator untouched
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR) mbar_arrive_cluster(&tempty[acc], 0);
        else mbar_arrive(&tempty[acc]);
      }
      ++it;
      continue;
#endif
      const uint32_t tbase = tmem_base + ((uint32_t)(qw * 32) << 16) + acc * BN;
      if constexpr (ROUTE) {  // the gate GEMM: routing in the epilogue, no C stores
        PROBE_T(rt0);
        route_epilogue(p.route, tbase, m0 + qw * 32, lane);
        if (lane == 0) PROBE_ADD(10, rt0);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (PAIR) mbar_arrive_cluster(&tempty[acc], 0);
          else mbar_arrive(&tempty[acc]);
        }
        ++it;
        continue;
      }
      // epilogue math of one 32-column slice (in place on v)
      auto apply = [&](int cc, int64_t n, float (&v)[32]) {
        if (p.epilogue == MPM_EPI_RELU || p.epilogue == MPM_EPI_RELU_MASK) {
          // mask bit by a predicated OR (compare + one LOP3 per element; the C++ form compiled to
          // compare + select + multiply-add): these epilogues pace the K = 1024 tiles
          uint32_t word = 0;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            asm("{\n.reg .pred p;\nsetp.gt.f32 p, %1, 0f00000000;\n@p or.b32 %0, %0, %2;\n}"
                : "+r"(word) : "f"(v[i]), "r"(1u << i));
            v[i] = fmaxf(v[i], 0.f);
          }
          if (p.epilogue == MPM_EPI_RELU_MASK) {  // kept in registers, stored once per tile row
#pragma unroll
            for (int q = 0; q < BN / 32; ++q)
              if (q == cc) mw[q] = word;
          }
        } else if (p.epilogue == MPM_EPI_DMASK) {
          uint32_t word = 0;
#pragma unroll
          for (int q = 0; q < BN / 32; ++q)
            if (q == cc) word = mw[q];
#pragma unroll
          for (int i = 0; i < 32; ++i)  // bit test straight into a predicate, then a select
            asm("{\n.reg .pred p;\n.reg .b32 t;\nand.b32 t, %1, %2;\nsetp.eq.u32 p, t, 0;\n@p mov.f32 %0, 0f00000000;\n}"
                : "+f"(v[i]) : "r"(word), "r"(1u << i));
        }
      };
      // bf16 outputs go out 64 columns (128 B rows) per TMA store: half the stores of 32-column slices
      const bool wide = p.wide_store && !f32_out && p.use_tma;
      const int step = wide ? 2 : 1;
#pragma unroll 1
      for (int cc = cc_lo; cc < cc_hi; cc += step) {
        const int64_t n = n0 + cc * 32;
        if (n >= p.n) break;  // warp-uniform
        float v[32], v2[32];
        if (wide) {  // both 32-column slices of the 64-column store in one TMEM load
          uint32_t r2[64];
          if (zero_tile) {
#pragma unroll
            for (int i = 0; i < 64; ++i) r2[i] = 0u;
          } else {
            PROBE_T(el0);
            tmem_ld64(tbase + cc * 32, r2);
            if (lane == 0) PROBE_ADD(4, el0);
          }
#pragma unroll
          for (int i = 0; i < 32; ++i) { v[i] = __uint_as_float(r2[i]); v2[i] = __uint_as_float(r2[32 + i]); }
#if !(defined(MPM_EPI_SKIP) && MPM_EPI_SKIP == 4)
          apply(cc, n, v);
          apply(cc + 1, n + 32, v2);
#endif
        } else {
          uint32_t r[32];
          if (zero_tile) {
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = 0u;
          } else {
            tmem_ld32(tbase + cc * 32, r);
          }
          if (!p.use_tma) {
            if (row_ok) epilogue_store(p, b, m, n, split, r);
            continue;
          }
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
          apply(cc, n, v);
        }
#if defined(MPM_EPI_SKIP) && MPM_EPI_SKIP == 4  // probe builds: TMEM loads only
        {
          if (__float_as_uint(v[0]) == 0x7f800001u && __float_as_uint(v2[31]) == 0x7f800001u)
            *reinterpret_cast<float*>(p.c) = v[1];
          continue;
        }
#endif
#if defined(MPM_EPI_SKIP) && MPM_EPI_SKIP == 2  // probe builds: TMEM loads and math only
        {
          float z = 0.f;
#pragma unroll
          for (int i = 0; i < 32; ++i) z += v[i] + v2[i];
          if (z == 12345.678f) *reinterpret_cast<float*>(p.c) = z;
          continue;
        }
#endif
        // staging buffer `buf` is free once the TMA store issued two stores ago has read it
        if (lane == 0) {
          PROBE_T(ew0);
          if (K::EPI_NB == 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          PROBE_ADD(5, ew0);
        }
        __syncwarp();
        uint8_t* sb = stg + buf * EPI_BUF;
        if (f32_out) {
          uint8_t* row = sb + lane * 128;
#pragma unroll
          for (int q = 0; q < 8; ++q)
            *reinterpret_cast<float4*>(row + ((q ^ (lane & 7)) << 4)) =
                make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        } else if (wide) {
          uint8_t* row = sb + lane * 128;  // 64 bf16 = 8 chunks of 16 B, 128B swizzle
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float* src = q < 4 ? v + 8 * q : v2 + 8 * (q - 4);
            uint4 u;
            __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
            for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(src[2 * i], src[2 * i + 1]);
            *reinterpret_cast<uint4*>(row + ((q ^ (lane & 7)) << 4)) = u;
          }
        } else {
          uint8_t* row = sb + lane * 64;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 u;
            __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
            for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[8 * q + 2 * i], v[8 * q + 2 * i + 1]);
            *reinterpret_cast<uint4*>(row + ((q ^ ((lane >> 1) & 3)) << 4)) = u;
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
#if defined(MPM_EPI_SKIP) && MPM_EPI_SKIP == 1  // probe builds: staging writes but no TMA store
        if (false) {
#else
        if (lane == 0) {
#endif
          const int c0 = (int)n, c1 = (int)(m0 + qw * 32), c2 = (int)(p.k_splits > 1 ? split : b);
          if (p.epilogue == MPM_EPI_ACCUM_F32 || p.epilogue == MPM_EPI_ACCUM)
            asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.bulk_group [%0, {%2, %3, %4}], [%1];"
                         ::"l"(reinterpret_cast<uint64_t>(&tmC)), "r"(smem_u32(sb)), "r"(c0), "r"(c1), "r"(c2)
                         : "memory");
          else
            asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];"
                         ::"l"(reinterpret_cast<uint64_t>(&tmC)), "r"(smem_u32(sb)), "r"(c0), "r"(c1), "r"(c2)
                         : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        if (K::EPI_NB == 2) buf ^= 1;
      }
      if (p.epilogue == MPM_EPI_RELU_MASK && row_ok) {
        // this row's BN/32 mask words: whole 32-byte sectors when the tile is full and aligned
        uint32_t* mp = reinterpret_cast<uint32_t*>(const_cast<void*>(p.aux)) + b * p.aux_bs + m * p.aux_ld + n0 / 32;
        if (CC_PER % 4 == 0 && n0 + BN <= p.n && (reinterpret_cast<uintptr_t>(mp + cc_lo) & 15) == 0) {
#pragma unroll
          for (int g4 = 0; g4 < BN / 128; ++g4)  // groups of 4 words; compile-time register indices
            if (4 * g4 >= cc_lo && 4 * g4 < cc_hi)
              *reinterpret_cast<uint4*>(mp + 4 * g4) =
                  make_uint4(mw[4 * g4], mw[4 * g4 + 1], mw[4 * g4 + 2], mw[4 * g4 + 3]);
        } else {
#pragma unroll
          for (int q = 0; q < BN / 32; ++q)
            if (q >= cc_lo && q < cc_hi && n0 + q * 32 < p.n) mp[q] = mw[q];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        PROBE_ADD(6, et0);
#ifdef MPM_EPI_PROBE
        probe_acc[7] += 1;
#endif
        if (PAIR) mbar_arrive_cluster(&tempty[acc], 0);  // the leader's MMA waits for both CTAs
        else mbar_arrive(&tempty[acc]);
      }
      ++it;
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }

#ifdef MPM_EPI_PROBE
  if (threadIdx.x == 128) PROBE_ADD(11, k_entry);  // first epilogue warp: entry -> done
#pragma unroll
  for (int i = 0; i < 12; ++i)
    if (probe_acc[i]) atomicAdd(&g_epi_probe[i], probe_acc[i]);
#endif
  tc_fence_before();
  if (PAIR) cluster_sync(); else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(K::TMEM_COLS));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(K::TMEM_COLS));
  }
}

// ---------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

// 3D bf16 tensor map: inner dim d0 (contiguous), d1 rows (pitch s1 elems),
// d2 batches (pitch s2 elems), box {64, box1, 1}, 128B swizzle, zero OOB.
static int make_map(CUtensorMap* map, const void* base, int64_t d0, int64_t d1, int64_t d2, int64_t s1, int64_t s2,
                    int box1) {
  auto fn = encode_fn();
  MPM_CHECK_ARG(fn != nullptr, "cuTensorMapEncodeTiled unavailable from the driver");
  if (d2 <= 1) s2 = s1 * d1;
  cuuint64_t dims[3] = {(cuuint64_t)d0, (cuuint64_t)d1, (cuuint64_t)(d2 < 1 ? 1 : d2)};
  cuuint64_t strides[2] = {(cuuint64_t)(s1 * 2), (cuuint64_t)(s2 * 2)};
  cuuint32_t box[3] = {64, (cuuint32_t)box1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  MPM_CHECK_ARG(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed (%d): dims %lld x %lld x %lld pitch %lld/%lld",
                (int)r, (long long)d0, (long long)d1, (long long)d2, (long long)s1, (long long)s2);
  return 0;
}

// MN-major operand as a 4-D map {64 MN, K, MN/64 blocks, batches}: one box {64, BK,
// blocks, 1} per k-slab lands as [blocks][BK][64] — the layout of `blocks` 3-D
// loads (MN_BLOCK_BYTES apart).  Needs MN % 64 == 0 (every block in bounds).
static int make_map_mn4(CUtensorMap* map, const void* base, int64_t mn, int64_t kext, int64_t batches, int64_t s1,
                        int64_t s2, int blocks) {
  auto fn = encode_fn();
  MPM_CHECK_ARG(fn != nullptr, "cuTensorMapEncodeTiled unavailable from the driver");
  if (batches <= 1) s2 = s1 * kext;
  cuuint64_t dims[4] = {64, (cuuint64_t)kext, (cuuint64_t)(mn / 64), (cuuint64_t)(batches < 1 ? 1 : batches)};
  cuuint64_t strides[3] = {(cuuint64_t)(s1 * 2), 128, (cuuint64_t)(s2 * 2)};
  cuuint32_t box[4] = {64, (cuuint32_t)BK, (cuuint32_t)blocks, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -1;  // caller falls back to 3-D loads
}

// Output map for TMA stores: {N, rows, batches|splits}; box 32 x 32 fp32 (128B
// swizzle), 64 x 32 bf16 when N >= 64 (`wide`, 128B swizzle) else 32 x 32 bf16
// (64B swizzle) — matching the epilogue's staging layouts.
static int make_out_map(CUtensorMap* map, const mpm_gemm_args* a, bool wide) {
  auto fn = encode_fn();
  MPM_CHECK_ARG(fn != nullptr, "cuTensorMapEncodeTiled unavailable from the driver");
  const bool f32 = a->c_dtype == MPM_F32;
  const int64_t esz = f32 ? 4 : 2;
  const int64_t z = a->k_splits > 1 ? a->k_splits : a->batches;
  int64_t zs = a->k_splits > 1 ? a->split_stride : a->c_batch_stride;
  if (z <= 1) zs = a->c_ld * a->rows;
  cuuint64_t dims[3] = {(cuuint64_t)a->n, (cuuint64_t)a->rows, (cuuint64_t)(z < 1 ? 1 : z)};
  cuuint64_t strides[2] = {(cuuint64_t)(a->c_ld * esz), (cuuint64_t)(zs * esz)};
  cuuint32_t box[3] = {(cuuint32_t)(wide ? 64 : 32), 32, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, a->c, dims,
                  strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  (f32 || wide) ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  MPM_CHECK_ARG(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled(out) failed (%d)", (int)r);
  return 0;
}

template <bool A_MN, bool B_MN, int BN, bool PAIR, int EW = 4, bool ROUTE = false>
static int launch(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc, const Params& p,
                  cudaStream_t s) {
  using K = Cfg<BN, PAIR, EW>;
  static bool attr_set[MAX_DEVICES] = {false};  // the smem opt-in is per device
  auto kern = umma_gemm_kernel<A_MN, B_MN, BN, PAIR, EW, ROUTE>;
  const int dev = device_index();
  if (!attr_set[dev]) {
    MPM_CUDA_RET(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K::SMEM_BYTES));
    attr_set[dev] = true;
  }
  const int sms = device_sms();
  const int64_t units = PAIR ? sms / 2 : sms;  // CTAs, or CTA pairs
  const int64_t grid = (p.total_tiles < units ? p.total_tiles : units) * (PAIR ? 2 : 1);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(K::THREADS_);
  cfg.dynamicSmemBytes = K::SMEM_BYTES;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = PAIR ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  MPM_CUDA_RET(cudaLaunchKernelEx(&cfg, kern, ta, tb, tc, p));
  MPM_LAUNCH_CHECK("umma_gemm_kernel");
  return 0;
}

template <int BN, bool PAIR, int EW = 4>
static int launch_bn(const mpm_gemm_args* a, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc,
                     const Params& p, cudaStream_t s) {
  if (!a->a_mn_major && !a->b_mn_major) return launch<false, false, BN, PAIR, EW>(ta, tb, tc, p, s);
  if (!a->a_mn_major && a->b_mn_major) return launch<false, true, BN, PAIR, EW>(ta, tb, tc, p, s);
  if (a->a_mn_major && !a->b_mn_major) return launch<true, false, BN, PAIR, EW>(ta, tb, tc, p, s);
  return launch<true, true, BN, PAIR, EW>(ta, tb, tc, p, s);
}

// 8 epilogue warps for store-bound tiles: few k-blocks per tile (the epilogue, not the MMA,
// paces the tile loop).  MPM_GEMM_EW=4|8 forces either (A/B testing).
static bool use_ew8(const Params& p) {
  static int env = -1;
  if (env < 0) { const char* e = getenv("MPM_GEMM_EW"); env = e ? atoi(e) : 0; }
  if (env == 4) return false;
  if (env == 8) return true;
  return p.kb_per_split <= 2;
}

// 2-CTA pairs (cta_group::2, 256 x 256 cluster tiles: each SM stages its
// 128 A rows and half of B, halving B's L2->SMEM traffic) for the wide
// expert GEMMs; MPM_GEMM_PAIR=0 forces single-CTA tiles (A/B testing).
// Pairs only when there are enough pair tiles for every CTA pair to get about two: a small GEMM
// (the gate GEMMs: 64 pair tiles of 16 k-blocks at T = 16K) is one latency-bound wave, and
// single-CTA 128-row tiles give twice the tiles with half the MMA work per k-block each.
static bool use_pair(const mpm_gemm_args* a, int bn) {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("MPM_GEMM_PAIR");
    env = (e && e[0] == '0') ? 0 : 1;
  }
  if (!(env == 1 && bn == 256 && a->rows > BM)) return false;
  const int64_t splits = a->k_splits > 1 ? a->k_splits : 1;
  const int64_t pair_tiles = a->batches * ceil_div(a->rows, 2 * BM) * ceil_div(a->n, bn) * splits;
  if (pair_tiles >= device_sms()) return true;
  // split-K GEMMs size their split count to one wave of pairs (the dWg GEMM: 4 N tiles x 18 splits of
  // the 192 stacked term rows): there a pair stages half of B per CTA and computes the 192 rows as one
  // 256-row tile, where single CTAs stage all of B for two 128-row tiles (the second half empty)
  return splits > 1 && 10 * pair_tiles >= 9 * (device_sms() / 2);
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int run(const mpm_gemm_args* a, cudaStream_t s, const RouteEpi* route) {
  MPM_CHECK_ARG(a->n % 32 == 0, "tcgen05 path needs N %% 32 == 0 (N=%lld)", (long long)a->n);
  MPM_CHECK_ARG(a->a_ld % 8 == 0 && a->b_ld % 8 == 0 && a->a_batch_stride % 8 == 0 && a->b_batch_stride % 8 == 0,
                "operand pitches must be multiples of 8 elements");
  MPM_CHECK_ARG(aligned16(a->a) && aligned16(a->b) && aligned16(a->c), "operands must be 16-byte aligned");
  MPM_CHECK_ARG(a->a_k_period % BK == 0 && a->b_k_period % BK == 0 && a->a_k_period >= 0 && a->b_k_period >= 0,
                "K periods must be multiples of %d", BK);
  const int csz = (int)dtype_size(a->c_dtype);
  MPM_CHECK_ARG((a->c_ld * csz) % 16 == 0 && (a->c_batch_stride * csz) % 16 == 0, "output pitch alignment");
  if (a->aux && (a->epilogue == MPM_EPI_DRELU || a->epilogue == MPM_EPI_ADD_AUX_F32))
    MPM_CHECK_ARG(aligned16(a->aux) && a->aux_ld % 4 == 0 && a->aux_batch_stride % 4 == 0, "aux alignment");
  if (a->epilogue == MPM_EPI_RELU_MASK || a->epilogue == MPM_EPI_DMASK)
    MPM_CHECK_ARG(a->n % 32 == 0 && aligned16(a->aux), "ReLU-mask epilogues need N %% 32 == 0 and an aligned mask");
  const int64_t splits_req = a->k_splits > 1 ? a->k_splits : 1;
  if (splits_req > 1)
    MPM_CHECK_ARG(a->epilogue == MPM_EPI_STORE_F32 && a->c_dtype == MPM_F32 && a->split_stride > 0,
                  "split-K writes f32 partials (EPI_STORE_F32) with a split stride");
  MPM_CHECK_ARG(!(a->valid_k && (splits_req > 1 || a->a_k_period || a->b_k_period)),
                "valid_k does not combine with split-K or K-periodic operands");

  // bn: widest N tile that does not exceed N (skinny gate GEMMs use 64/128)
  const int bn = a->n <= 64 ? 64 : a->n <= 128 ? 128 : 256;
  const bool pair = use_pair(a, bn);
  const int b_box = pair ? bn / 2 : bn;  // B rows per CTA (K-major B box)
  const int64_t ka = a->a_k_period ? a->a_k_period : a->k;
  const int64_t kb = a->b_k_period ? a->b_k_period : a->k;
  CUtensorMap ta, tb;
  static int mn4_env = -1;
  if (mn4_env < 0) { const char* e = getenv("MPM_GEMM_MN4"); mn4_env = (e && e[0] == '0') ? 0 : 1; }
  bool a_mn4 = false, b_mn4 = false;
  if (!a->a_mn_major) { if (int rc = make_map(&ta, a->a, ka, a->rows, a->batches, a->a_ld, a->a_batch_stride, BM)) return rc; }
  else {
    a_mn4 = mn4_env && a->rows % 64 == 0 &&
            make_map_mn4(&ta, a->a, a->rows, ka, a->batches, a->a_ld, a->a_batch_stride, BM / 64) == 0;
    if (!a_mn4) { if (int rc = make_map(&ta, a->a, a->rows, ka, a->batches, a->a_ld, a->a_batch_stride, BK)) return rc; }
  }
  if (!a->b_mn_major) { if (int rc = make_map(&tb, a->b, kb, a->n, a->batches, a->b_ld, a->b_batch_stride, b_box)) return rc; }
  else {
    b_mn4 = mn4_env && a->n % 64 == 0 &&
            make_map_mn4(&tb, a->b, a->n, kb, a->batches, a->b_ld, a->b_batch_stride, b_box / 64) == 0;
    if (!b_mn4) { if (int rc = make_map(&tb, a->b, a->n, kb, a->batches, a->b_ld, a->b_batch_stride, BK)) return rc; }
  }

  Params p{};
  p.rows = a->rows; p.n = a->n; p.k = a->k;
  p.a_mn4 = a_mn4; p.b_mn4 = b_mn4;
  p.m_tiles = ceil_div(a->rows, pair ? 2 * BM : BM);
  p.n_tiles = ceil_div(a->n, bn);
  p.k_blocks = ceil_div(a->k, BK);
  // every split gets >= 1 k-block (an empty split would leave its TMEM accumulator unwritten)
  p.kb_per_split = ceil_div(p.k_blocks, splits_req < p.k_blocks ? splits_req : p.k_blocks);
  p.k_splits = ceil_div(p.k_blocks, p.kb_per_split);
  p.split_stride = a->split_stride;
  p.a_k_period = a->a_k_period; p.b_k_period = a->b_k_period;
  p.tiles_per_split = a->batches * p.m_tiles * p.n_tiles;
  p.total_tiles = p.k_splits * p.tiles_per_split;
  MPM_CHECK_ARG(p.total_tiles < (int64_t(1) << 31), "too many tiles (%lld)", (long long)p.total_tiles);
  p.c = a->c; p.c_ld = a->c_ld; p.c_bs = a->c_batch_stride; p.c_dtype = a->c_dtype;
  p.aux = a->aux; p.aux_ld = a->aux_ld; p.aux_bs = a->aux_batch_stride;
  p.valid_rows = a->valid_rows;
  p.valid_k = a->valid_k;
  p.epilogue = a->epilogue;
  p.op_dtype = a->dtype;
  // TMA store epilogue unless the epilogue reads a dense aux tensor per element
  p.use_tma = !(a->epilogue == MPM_EPI_ADD_AUX_F32 || a->epilogue == MPM_EPI_DRELU) &&
              (a->k_splits <= 1 || a->batches == 1);
  if (route) {  // routing epilogue: one N tile holds every expert's three partial logits
    MPM_CHECK_ARG(a->n <= 256 && a->batches == 1 && a->k_splits <= 1 && route->k >= 1 && route->k <= 8 &&
                      3 * route->Ec <= a->n && route->Ec % 32 == 0 && route->E <= route->Ec,
                  "routing epilogue: unsupported gate GEMM shape");
    p.use_tma = 0;
    p.route = *route;
  }
  CUtensorMap tc;
  memset(&tc, 0, sizeof(tc));
  p.wide_store = p.use_tma && a->c_dtype == MPM_BF16 && a->n >= 64 && bn >= 64;
  if (p.use_tma) {
    if (int rc = make_out_map(&tc, a, p.wide_store != 0)) return rc;
  }
  if (p.total_tiles == 0) return 0;
  if (route) {  // the gate GEMM (K-major x and stacked Wg terms)
    MPM_CHECK_ARG(!a->a_mn_major && !a->b_mn_major && (bn == 128 || bn == 256), "routing epilogue: layout");
    if (bn == 128) return launch<false, false, 128, false, 4, true>(ta, tb, tc, p, s);
    if (pair) return launch<false, false, 256, true, 4, true>(ta, tb, tc, p, s);
    return launch<false, false, 256, false, 4, true>(ta, tb, tc, p, s);
  }
  if (bn == 64) return launch_bn<64, false>(a, ta, tb, tc, p, s);
  if (bn == 128) return launch_bn<128, false>(a, ta, tb, tc, p, s);
  if (pair) return use_ew8(p) ? launch_bn<256, true, 8>(a, ta, tb, tc, p, s) : launch_bn<256, true>(a, ta, tb, tc, p, s);
  return use_ew8(p) ? launch_bn<256, false, 8>(a, ta, tb, tc, p, s) : launch_bn<256, false>(a, ta, tb, tc, p, s);
}

// Fixed-order sum of split-K partials: out[i] = sum_s part[s*stride + i] (+ out[i] if accumulate).
__global__ void splitk_reduce_kernel(const float* __restrict__ part, int64_t splits, int64_t stride, int64_t count,
                                     void* __restrict__ out, int out_dtype, int accumulate) {
  pdl_begin();
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i >= count) return;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  int64_t sp = 0;
  for (; sp + 8 <= splits; sp += 8) {  // 8 loads in flight, summed in split order
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldg(reinterpret_cast<const float4*>(part + (sp + u) * stride + i));
#pragma unroll
    for (int u = 0; u < 8; ++u) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
  }
  for (; sp < splits; ++sp) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(part + sp * stride + i));
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  if (out_dtype == MPM_F32) {
    float4* o = reinterpret_cast<float4*>(static_cast<float*>(out) + i);
    if (accumulate) { float4 b = *o; acc.x += b.x; acc.y += b.y; acc.z += b.z; acc.w += b.w; }
    *o = acc;
  } else {
    __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>(static_cast<__nv_bfloat16*>(out) + i);
    o[0] = __floats2bfloat162_rn(acc.x, acc.y);
    o[1] = __floats2bfloat162_rn(acc.z, acc.w);
  }
}

}  // namespace sm100
}  // namespace mpm

extern "C" int mpm_grouped_gemm(const mpm_gemm_args* args, void* stream) {
  if (int rc = mpm::validate_gemm(args)) return rc;
  if (args->rows == 0 || args->n == 0 || args->batches == 0) return 0;
  if (args->dtype == MPM_F32 || args->k == 0) {
    MPM_CHECK_ARG(args->k_splits <= 1 && args->a_k_period == 0 && args->b_k_period == 0,
                  "split-K / K periods are tcgen05-path features (bf16 operands)");
    return mpm::simt_gemm_launch(args, args->dtype, args->dtype, (cudaStream_t)stream);
  }
  return mpm::sm100::run(args, (cudaStream_t)stream);
}

extern "C" int mpm_splitk_reduce(const float* partials, int64_t splits, int64_t split_stride, int64_t count,
                                 void* out, int out_dtype, int accumulate, void* stream) {
  MPM_CHECK_ARG(count % 4 == 0 && split_stride % 4 == 0, "count and stride must be multiples of 4");
  MPM_CHECK_ARG(out_dtype == MPM_F32 || out_dtype == MPM_BF16, "bad dtype");
  MPM_CHECK_ARG(!(accumulate && out_dtype != MPM_F32), "accumulate needs an f32 output");
  if (count == 0) return 0;
  const int64_t threads = count / 4;
  MPM_PDL_LAUNCH(mpm::sm100::splitk_reduce_kernel, dim3((unsigned)mpm::ceil_div(threads, 128)), dim3(128), 0,
                 (cudaStream_t)stream, partials, splits, split_stride, count, out, out_dtype, accumulate);
  return 0;
}

#ifdef MPM_EPI_PROBE
// probe builds only: copy out (and optionally clear) the wait-cycle sums
extern "C" int mpm_debug_epi_probe(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, mpm::sm100::g_epi_probe, sizeof(unsigned long long) * 16) != cudaSuccess) return 1;
  if (reset) {
    unsigned long long z[16] = {0};
    if (cudaMemcpyToSymbol(mpm::sm100::g_epi_probe, z, sizeof(z)) != cudaSuccess) return 1;
  }
  return 0;
}
#endif
