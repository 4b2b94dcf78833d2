/*
 * mpm.h — C-ABI of the B200-native pipelined expert-parallel MoE layer
 * (MPipeMoE, arxiv 2506.22175).  Built from paper_2506_22175_b200/csrc/*.cu
 * into paper_2506_22175_b200/libmpm.so for sm_100a.
 *
 * The reference (`/root/reference`, package `moepipesim`) has no FFI and no
 * numerics: it *models* each operation below as an op node of its schedule
 * DAG.  Each entry point cites the modelled op it realises:
 *
 *   S_i  dispatch all-to-all       pipesim/schedule.py:252   -> mpm_a2a_chunk(dir=DISPATCH)
 *   C_i  expert compute (2 GeMMs)  pipesim/schedule.py:253   -> mpm_grouped_gemm (FC1 relu, FC2)
 *   R_i  combine all-to-all        pipesim/schedule.py:254   -> mpm_a2a_chunk(dir=COMBINE)
 *   Ddi_i/Dm_i offload copies      pipesim/schedule.py:261-270 -> mpm_copy_async(D2H)
 *   BS_i grad dispatch             pipesim/schedule.py:300   -> mpm_a2a_chunk(dir=DISPATCH)
 *   RC_i re-dispatch (S2/S4)       pipesim/schedule.py:306-310 -> mpm_a2a_chunk(dir=DISPATCH)
 *   Hdi_i/Hm_i prefetch copies     pipesim/schedule.py:311-326 -> mpm_copy_async(H2D)
 *   RE_i recompute (S3/S4)         pipesim/schedule.py:327-332 -> mpm_grouped_gemm (FC1 relu)
 *   G2_i fc2 dgrad+wgrad           pipesim/schedule.py:335   -> mpm_grouped_gemm (DRELU, WGRAD)
 *   G1_i fc1 dgrad+wgrad           pipesim/schedule.py:338   -> mpm_grouped_gemm (NONE, WGRAD)
 *   BR_i grad combine              pipesim/schedule.py:340   -> mpm_a2a_chunk(dir=COMBINE)
 * and the routing / combine kernels the reference excludes from its model
 * (memmodel.py:7-8): mpm_gate_fwd, mpm_route,
 * mpm_gate_route (the two fused),
 * mpm_assign_slots, mpm_permute, mpm_combine, mpm_combine_bwd,
 * mpm_gate_bwd_logits, mpm_gather_bwd.
 *
 * Conventions
 *  - Every function returns 0 on success, else a nonzero status (a
 *    cudaError_t / ncclResult_t code, or MPM_ERR_INVALID for bad
 *    arguments); mpm_last_error() returns the message of the last failure
 *    on the calling thread.
 *  - Pointers are device pointers unless named host_*.  The caller owns
 *    every buffer; nothing here allocates device memory or synchronises
 *    with the host (the comm init is the only blocking call).
 *  - `stream` is a cudaStream_t passed as void*.
 *  - Slot layout (expert-major): a dispatch buffer holds E*C rows of M,
 *    row e*C + s for slot s of expert e (e = dest*E_loc + e_loc).  The
 *    capacity C is split into n chunks with the reference's balanced rule
 *    (core.py:102-105): the first C mod n chunks hold C/n+1 slots, the rest
 *    C/n; chunk i is slot range [s_i, s_i+c_i) of every expert.  Per
 *    destination and chunk a rank sends E_loc blocks of c_i contiguous rows.
 */
#ifndef MPM_H_
#define MPM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPM_ABI_VERSION 1

enum { MPM_OK = 0, MPM_ERR_INVALID = 1000, MPM_ERR_UNSUPPORTED = 1001 };

/* element types */
enum { MPM_F32 = 0, MPM_BF16 = 1 };

/* GEMM epilogues (applied to the fp32 accumulator `acc`) */
enum {
  MPM_EPI_NONE = 0,       /* c = cast(acc)                                 */
  MPM_EPI_RELU = 1,       /* c = cast(max(acc, 0))          (fc1 forward)  */
  MPM_EPI_DRELU = 2,      /* c = cast(acc * (aux > 0))      (fc2 dgrad: aux = relu output T_M) */
  MPM_EPI_STORE_F32 = 3,  /* c(f32) = acc                   (first wgrad chunk) */
  MPM_EPI_ACCUM_F32 = 4,  /* c(f32) += acc                  (middle wgrad chunks) */
  MPM_EPI_ADD_AUX_F32 = 5, /* c = cast(acc + aux(f32))      (last wgrad chunk) */
  MPM_EPI_RELU_MASK = 6,   /* c = cast(max(acc, 0)); aux (uint32 [b][rows][N/32]) = bit (acc > 0) */
  MPM_EPI_DMASK = 7,       /* c = cast(acc * bit(aux mask)) (fc2 dgrad against the fc1 mask) */
  MPM_EPI_ACCUM = 8        /* c += acc in c's dtype (f32, or bf16 rounded once per call):
                              wgrad accumulation across chunks without fp32 scratch */
};

/* all-to-all directions */
enum { MPM_A2A_DISPATCH = 0, MPM_A2A_COMBINE = 1 };

/* copy directions */
enum { MPM_COPY_D2H = 0, MPM_COPY_H2D = 1, MPM_COPY_D2D = 2 };

int mpm_abi_version(void);
const char* mpm_last_error(void);
/* Number of SMs of the current device (grid sizing); -1 on error. */
int mpm_sm_count(void);
/* Kernels libmpm has launched in this process (all threads). */
unsigned long long mpm_launch_count(void);

/* ---------------------------------------------------------------- routing */

/* Bytes of the workspace mpm_gate_fwd / mpm_gate_wgrad / mpm_gather_bwd need. */
size_t mpm_gate_workspace_bytes(int64_t T, int64_t M, int64_t E);

/* logits[T][E] (f32) = x[T][M] (x_dtype) . wg[E][M]^T (f32).  bf16 x with
 * M % 64 == 0: tcgen05 in bf16x3 split precision (fp32 accurate, any E: the
 * expert axis is zero-padded to a multiple of 32 in the workspace, see
 * csrc/gate.cu); otherwise exact-fp32 FMA.  Deterministic.
 * Gate of PAPER.md:124,517. */
int mpm_gate_fwd(const void* x, int x_dtype, const float* wg, float* logits,
                 int64_t T, int64_t M, int64_t E, void* workspace, void* stream);

/* Bytes of the routing workspace shared by mpm_route/mpm_assign_slots. */
size_t mpm_route_workspace_bytes(int64_t T, int64_t E, int k);

/* Top-k of each logits row (lowest expert index wins exact ties), routing
 * weights (k == 1: softmax probability of the chosen expert; k > 1 and
 * renorm: softmax over the k chosen logits), and per-block expert counts in
 * `workspace`.  idx[T][k] int32, weights[T][k] f32. */
int mpm_route(const float* logits, int64_t T, int64_t E, int k, int renorm,
              int32_t* idx, float* weights, void* workspace, void* stream);

/* Gate + top-k routing in one call (the layer's forward front end): logits
 * (f32, written for the backward), idx, weights and the per-block expert
 * counts for mpm_assign_slots, bit-identical to mpm_gate_fwd followed by
 * mpm_route.  On the tcgen05 path with E <= 64 the routing runs in the gate
 * GEMM's epilogue (the partial logits never leave TMEM, no routing kernel);
 * for larger E the three partial logits of the stacked-term gate GEMM are
 * summed inside the routing kernel instead of in a separate pass. */
int mpm_gate_route(const void* x, int x_dtype, const float* wg, int64_t T,
                   int64_t M, int64_t E, int k, int renorm, float* logits,
                   int32_t* idx, float* weights, void* gate_workspace,
                   void* route_workspace, void* stream);

/* Capacity-bounded slot assignment, priority (k-rank, token index): slot[T][k]
 * int32 (-1 = dropped), kept[E] int32 = min(arrivals, C).  Bit-exact with
 * oracle/moe_oracle.py:assign_slots. */
int mpm_assign_slots(const int32_t* idx, int64_t T, int64_t E, int k,
                     int64_t capacity, void* workspace, int32_t* slot,
                     int32_t* kept, void* stream);

/* Valid (routed) rows of every expert in every chunk: rows[i][e] =
 * clamp(kept[e] - s_i, 0, c_i) for the balanced split of `capacity` into
 * n_chunks (core.py:102-105).  Slots fill in order, so chunk i's rows of
 * expert e are a valid prefix followed by zero padding: the expert GEMMs skip
 * the padded row tiles (valid_rows) and the weight gradients the padded K
 * blocks (valid_k).  rows_out holds n_chunks * E int32. */
int mpm_chunk_rows(const int32_t* kept, int64_t E, int64_t capacity, int n_chunks,
                   int32_t* rows_out, void* stream);

/* Scatter rows of x into the expert-major dispatch buffer (dtype), zero the
 * unused slots of every expert.  send holds E*C rows of M. */
int mpm_permute(const void* x, int dtype, const int32_t* idx,
                const int32_t* slot, const int32_t* kept, int64_t T,
                int64_t M, int64_t E, int k, int64_t capacity, int n_chunks,
                void* send, void* stream);

/* y[t] = sum_j weights[t][j] * t_o[row(idx[t][j], slot[t][j])], dropped
 * assignments contribute 0 (fp32 accumulation). */
int mpm_combine(const void* t_o, int dtype, const int32_t* idx,
                const int32_t* slot, const float* weights, int64_t T,
                int64_t M, int64_t E, int k, int64_t capacity, int n_chunks,
                void* y, void* stream);

/* Backward of mpm_combine: dprob[t][j] = <dy[t], t_o[row]> (f32, 0 when
 * dropped); g_o[row] = weights[t][j] * dy[t]; unused slots of g_o zeroed.
 * Either output may be NULL to compute only the other half (dprob == NULL:
 * no t_o reads; g_o == NULL: no scatter), e.g. the g_o half on the compute
 * stream (it gates the expert backward) and the dprob half on a side stream. */
int mpm_combine_bwd(const void* dy, const void* t_o, int dtype,
                    const int32_t* idx, const int32_t* slot,
                    const int32_t* kept, const float* weights, int64_t T,
                    int64_t M, int64_t E, int k, int64_t capacity,
                    int n_chunks, float* dprob, void* g_o, void* stream);

/* dlogits[T][E] (f32) from dprob through the routing weights (softmax
 * Jacobian; top-k renormalisation when k > 1 and renorm). */
int mpm_gate_bwd_logits(const float* logits, const int32_t* idx,
                        const float* weights, const float* dprob, int64_t T,
                        int64_t E, int k, int renorm, float* dlogits,
                        void* stream);

/* dx[t] = sum_j g_i[row(idx[t][j], slot[t][j])] + dlogits[t] . wg   (dtype) */
int mpm_gather_bwd(const void* g_i, int dtype, const int32_t* idx,
                   const int32_t* slot, const float* dlogits, const float* wg,
                   int64_t T, int64_t M, int64_t E, int k, int64_t capacity,
                   int n_chunks, void* dx, void* workspace, void* stream);

/* Fused gate backward: dlogits (as mpm_gate_bwd_logits), dwg = dlogits^T x,
 * dx = gathered g_i rows + dlogits . wg.  bf16 with M % 64 == 0 and
 * T % 64 == 0 (any E): one kernel emits dlogits and both bf16x3 operands,
 * then two tcgen05 GEMMs (split-K for dwg) and the gather; otherwise the
 * exact-fp32 kernels (split-K over tokens for dwg). */
int mpm_gate_backward(const float* logits, const int32_t* idx,
                      const float* weights, const float* dprob, const void* x,
                      const void* g_i, const int32_t* slot, int dtype,
                      const float* wg, int64_t T, int64_t M, int64_t E, int k,
                      int renorm, int64_t capacity, int n_chunks,
                      float* dlogits, void* dx, float* dwg, void* workspace,
                      void* stream);

/* The two halves of mpm_gate_backward, for overlapping the gate part with
 * the expert backward (it needs only dprob, x and wg; the expert-side g_i
 * enters in the gather).  _gate: dlogits, dwg and (tcgen05 path) the gate
 * term dlogits.wg written into dx; _gather: dx += the gathered g_i rows (in
 * place; on the exact-fp32 path it computes the gate term into dx first).
 * Issue _gather after _gate with the same dx and workspace (stream-ordered
 * by the caller).  No [T][M] scratch exists on either path. */
int mpm_gate_backward_gate(const float* logits, const int32_t* idx,
                           const float* weights, const float* dprob,
                           const void* x, int dtype, const float* wg,
                           int64_t T, int64_t M, int64_t E, int k, int renorm,
                           float* dlogits, float* dwg, void* dx,
                           void* workspace, void* stream);
int mpm_gate_backward_gather(const void* g_i, int dtype, const int32_t* idx,
                             const int32_t* slot, const float* dlogits,
                             const float* wg, int64_t T, int64_t M, int64_t E,
                             int k, int64_t capacity, int n_chunks, void* dx,
                             void* workspace, void* stream);

/* The layer's backward of combine + gate in three stream-ordered calls
 * (PAPER.md:124,174 combine / gate backward; the schedule's backward starts
 * after them, pipesim/schedule.py:300-340):
 *   mpm_combine_bwd_gate   one pass per token: g_o rows (g_o may be NULL, e.g.
 *                          when the grad-dispatch gathers w*dy itself), dprob
 *                          (may be NULL), dlogits, and the bf16x3 split
 *                          operands of the gate GEMMs in the gate workspace
 *                          (tcgen05 path: bf16, M % 64 == 0, T % 64 == 0);
 *   mpm_gate_backward_gemms  dwg = dlogits^T x (term rows stacked along M,
 *                          split-K, fixed-order reduce) and, for the dense
 *                          gate gradient (k == 1 or no renorm), the gate term
 *                          dlogits . wg written into dx;
 *   mpm_gate_gather        dx = gathered g_i rows + the gate term: in place on
 *                          the dense term, or (k > 1 with renorm, where
 *                          dlogits has only the k chosen experts nonzero)
 *                          from the k rows of wg in exact fp32.
 * Same workspace and dlogits across the three; results are deterministic. */
int mpm_combine_bwd_gate(const void* dy, const void* t_o, int dtype,
                         const int32_t* idx, const int32_t* slot,
                         const int32_t* kept, const float* weights,
                         const float* logits, int64_t T, int64_t M, int64_t E,
                         int k, int renorm, int64_t capacity, int n_chunks,
                         void* g_o, float* dprob, float* dlogits,
                         void* gate_workspace, void* stream);
int mpm_gate_backward_gemms(const void* x, int dtype, const float* wg,
                            const float* dlogits, int64_t T, int64_t M,
                            int64_t E, int k, int renorm, float* dwg, void* dx,
                            void* gate_workspace, void* stream);
int mpm_gate_gather(const void* g_i, int dtype, const int32_t* idx,
                    const int32_t* slot, const float* dlogits, const float* wg,
                    int64_t T, int64_t M, int64_t E, int k, int renorm,
                    int64_t capacity, int n_chunks, void* dx,
                    void* gate_workspace, void* stream);

/* dwg[E][M] (f32) = dlogits^T . x  (tcgen05 split-K when x is bf16) */
int mpm_gate_wgrad(const float* dlogits, const void* x, int x_dtype,
                   int64_t T, int64_t M, int64_t E, float* dwg,
                   void* workspace, void* stream);

/* ------------------------------------------------------------ expert GEMM */

/* Batched (one batch per local expert) GEMM  C[b] = A[b] . B[b]^T  with
 * A logically rows x K and B logically N x K.
 *   a_mn_major = 0: A stored [b][rows][K] (row pitch a_ld elements)
 *   a_mn_major = 1: A stored [b][K][rows] (pitch a_ld)          (wgrad)
 *   b_mn_major = 0: B stored [b][N][K]                            (fwd)
 *   b_mn_major = 1: B stored [b][K][N]                            (dgrad/wgrad)
 * C stored [b][rows][N] with pitch c_ld, dtype c_dtype.  aux has C's
 * geometry (operand dtype for DRELU, f32 for ADD_AUX_F32).  bf16 operands
 * run on tcgen05 (TMEM accumulators, TMA-fed, 128x256x64 tiles, persistent);
 * f32 operands run an exact-fp32 FMA kernel (parity path). */
typedef struct mpm_gemm_args {
  int dtype;        /* operand dtype: MPM_BF16 or MPM_F32 */
  int epilogue;     /* MPM_EPI_* */
  int64_t batches, rows, n, k;
  const void* a; int64_t a_ld, a_batch_stride; int a_mn_major;
  const void* b; int64_t b_ld, b_batch_stride; int b_mn_major;
  void* c; int64_t c_ld, c_batch_stride; int c_dtype;
  const void* aux; int64_t aux_ld, aux_batch_stride;
  /* optional: valid rows per batch (int32[batches]); tiles whose rows are
   * all >= valid are skipped and their outputs left untouched. NULL = all */
  const int32_t* valid_rows;
  /* tcgen05 path only.  K-periodic operands: the operand holds only
   * `*_k_period` columns of K and logical column k reads column k mod
   * period (multiples of 64; 0 = off) — how split-precision "bf16x3" GEMMs
   * reuse one bf16 operand against three bf16 terms of an fp32 one.
   * Split-K: k_splits > 1 writes f32 partial sums of split s at
   * c + s*split_stride (EPI_STORE_F32); sum them with mpm_splitk_reduce. */
  int64_t a_k_period, b_k_period;
  int64_t k_splits, split_stride;
  /* optional: valid K per batch (int32[batches]); batch b's K loop stops at
   * the 64-aligned block covering valid_k[b] (the operands' K rows beyond it
   * are capacity padding and are not read; rows up to the 64 boundary must be
   * zero).  valid_k[b] == 0 writes zeros.  NULL = all K.  Weight gradients of
   * experts with fewer routed tokens than their capacity. */
  const int32_t* valid_k;
} mpm_gemm_args;

int mpm_grouped_gemm(const mpm_gemm_args* args, void* stream);

/* out[i] (+)= sum over s in [0, splits) of partials[s*split_stride + i] in
 * split order (deterministic); out f32 (accumulate allowed) or bf16. */
int mpm_splitk_reduce(const float* partials, int64_t splits, int64_t split_stride,
                      int64_t count, void* out, int out_dtype, int accumulate,
                      void* stream);

/* Force the exact-fp32/SIMT kernel for bf16 operands too (test hook). */
int mpm_grouped_gemm_simt(const mpm_gemm_args* args, void* stream);

/* ------------------------------------------------------ communication */

/* NCCL communicator for the expert-parallel group (pip NCCL 2.28). */
int mpm_comm_unique_id(void* host_id_out /* 128 bytes */);
int mpm_comm_init(const void* host_id, int nranks, int rank, int device,
                  void** comm_out);
int mpm_comm_destroy(void* comm);

/* One chunk's all-to-all (S_i/R_i/BS_i/RC_i/BR_i) as an explicit block plan:
 * for b in [0, n_blocks): send src[host_send_off[b] ...+block_elems) to
 * host_peer[b] and receive from host_peer[b] into dst[host_recv_off[b] ...]
 * (offsets in elements; grouped ncclSend/ncclRecv, pairs matched in plan
 * order per peer).  The plan for the layer's layouts
 *   DISPATCH: rows [e*C + s_i, +c_i) of the source's [E][C][M] buffer ->
 *             rows [row0 + src*c_i, +c_i) of local expert e_loc's region
 *             (expert stride X) of the destination's expert-side buffer
 *   COMBINE : the reverse
 * comes from comm.py:block_plan.  nranks == 1 with comm == NULL: device
 * copies; with a (single-rank) communicator the NCCL path runs (tests). */
int mpm_a2a_chunk(void* comm, int nranks, int n_blocks, const int32_t* host_peer,
                  const int64_t* host_send_off, const int64_t* host_recv_off,
                  int64_t block_elems, int dtype, const void* src, void* dst,
                  void* stream);

/* ------------------------------------------------ peer-memory exchange */

/* The production N > 1 data path (csrc/p2p.cu): every rank exports one
 * device *window* per step arena through CUDA IPC (dispatch-side buffers,
 * gate-gradient staging, a uint32 flag array; identical offsets on every
 * rank).  A chunk exchange is one mpm_p2p_run: wait until flags in the local
 * window reach `value` (stream memory ops: no SM), one light SM kernel that
 * moves every 2-D block between local rows and peer windows over NVLink
 * (no shared memory, so it runs beside the persistent GEMM CTAs; its last
 * CTA fences system-wide and raises `value` in the peers' flags), a wait
 * for the peers' flags (their pushes have landed), and finally a reset of
 * the listed local flags to 0 (each flag is raised once per step and reset
 * by its last waiter, so the layer passes value 1 every step and a captured
 * CUDA graph replays the exchanges unchanged).  Rows, pitches and addresses
 * must be 16-byte aligned.  Same modelled ops as mpm_a2a_chunk
 * (schedule.py:252-340). */
#define MPM_MAX_PEERS 64
#define MPM_IPC_HANDLE_BYTES 64

/* cudaMalloc'd, zero-filled window and its IPC handle (host, 64 bytes). */
int mpm_ipc_alloc(size_t bytes, void** ptr_out, void* host_handle_out);
/* Map a peer process's window (lazy peer access). */
int mpm_ipc_open(const void* host_handle, void** ptr_out);
int mpm_ipc_close(void* ptr);
int mpm_ipc_free(void* ptr);

typedef struct mpm_p2p_copy {
  void* dst; const void* src;               /* device (local or peer-window) */
  int64_t dpitch, spitch, width, height;     /* bytes, rows (cudaMemcpy2D) */
} mpm_p2p_copy;

typedef struct mpm_p2p_plan {
  int n_wait;   const uint32_t* wait[MPM_MAX_PEERS];    /* local flags >= value before the copies */
  int n_copy;   mpm_p2p_copy copy[MPM_MAX_PEERS];
  int n_signal; uint32_t* signal[MPM_MAX_PEERS];        /* peer flags := value after the copies */
  int n_arrive; const uint32_t* arrive[MPM_MAX_PEERS];  /* local flags >= value at the end */
  int n_reset;  uint32_t* reset[MPM_MAX_PEERS];         /* local flags := 0 last (their final wait passed) */
  /* zero-initialised device uint32 owned by this plan: completion count of
   * the SM copy kernel (the last CTA fences and raises the peer flags). */
  uint32_t* counter;
} mpm_p2p_plan;

int mpm_p2p_run(const mpm_p2p_plan* plan, uint32_t value, void* stream);

/* Fused dispatch (no memory reuse): the dispatch-type exchanges S_i / BS_i
 * (schedule.py:252,300) without the local T_I / g_o staging.  The sender
 * gathers its rows of a chunk (local experts [e0, e0+ne) of every
 * destination, slots [s0, s0+cs)) from the token rows through the
 * slot-owner map and stores them straight into every destination's
 * expert-side buffer (its window) at row
 *   (el - e0)*x_stride + x_row0 + rank*cs + (s - s0)
 * (x when scale == NULL, else scale[a] * dy[t] for assignment a = t*k + j,
 * rounded like mpm_combine_bwd's g_o rows; zero rows for unused slots), then
 * its last CTA fences system-wide and raises `value` in flag[d] of every
 * destination d != rank.  The receiver waits for those flags (mpm_p2p_run
 * with only arrivals).  counter: a zeroed device uint32 owned by the plan. */
typedef struct mpm_push_plan {
  int nranks, rank;
  void* dst[MPM_MAX_PEERS];       /* destination d's expert-side buffer (window address) */
  uint32_t* flag[MPM_MAX_PEERS];  /* destination d's arrival flag for (this chunk, this rank) */
  int64_t e_loc, capacity, e0, ne, s0, cs, x_stride, x_row0;
  uint32_t* counter;
  /* Compacted expert-side layout (null: capacity layout): [nranks][E] kept
   * counts of every source (this rank's window copy).  Source s's routed
   * rows of expert e land at the sum of the lower sources' counts; padding
   * slots are not sent and the last source zeroes the rows up to the next
   * 64-row boundary.  Needs whole-capacity chunks (s0 = 0, cs = capacity). */
  const int32_t* kept_all;
} mpm_push_plan;

int mpm_dispatch_push(const mpm_push_plan* plan, const void* src, int dtype, int64_t M, int k,
                      const int32_t* inv, const float* scale, uint32_t value, void* stream);

/* Combine-type exchange of one chunk in the compacted layout (R_i: T_DO ->
 * the owners' T_O; BR_i: g_di -> g_i; pipesim/schedule.py:252-340): dst[d] =
 * owner d's dispatch-side buffer (window), src = this rank's expert-side
 * rows; owner d's routed rows of each local expert e in the slot range
 * [s0, s0 + cs) are copied to those slots and flag[d] is raised in every peer
 * after a system fence.
 * The caller then waits for its own arrival flags (mpm_p2p_run). */
int mpm_combine_push(const mpm_push_plan* plan, const void* src, int dtype, int64_t M, uint32_t value,
                     void* stream);

/* rows[el] = routed rows of local expert el in the compacted layout of the
 * chunk slot range [s0, s0 + cs) (the sum over sources of their routed rows
 * of expert rank * e_loc + el there): the GEMMs' valid rows / the weight
 * gradients' valid K. */
int mpm_compact_rows(const int32_t* kept_all, int nranks, int64_t E, int64_t e_loc, int rank, int64_t s0,
                     int64_t cs, int32_t* rows, void* stream);

/* Dispatch-type pull of one chunk into the compacted layout (memory reuse:
 * S_i / BS_i / RC_i into a ring slot): dst[s] = source s's dispatch-side
 * buffer (T_I or g_o, window), `dst` argument = this rank's expert-side
 * rows; source s's routed rows of each local expert land at the lower
 * sources' prefix, and the rows up to the next 64-row boundary are zeroed.
 * The caller waits for the sources' ready flags first (mpm_p2p_run). */
int mpm_compact_pull(const mpm_push_plan* plan, void* dst, int dtype, int64_t M, void* stream);

/* Slot owners: inv[e*C + s] = t*k + j for the assignment holding slot s of
 * expert e, -1 for unused slots (slot >= kept[e]). */
int mpm_slot_owners(const int32_t* idx, const int32_t* slot, const int32_t* kept, int64_t T, int64_t E,
                    int k, int64_t capacity, int32_t* inv, void* stream);

/* Exchange watchdog (csrc/watchdog.cu): record an event behind the work
 * issued so far on `stream`; a host thread aborts the process with `tag` if
 * it has not completed within timeout_s (a dead or stalled peer would
 * otherwise leave the flag waits blocked forever).  No-op while the stream
 * is being captured into a graph.  _pending: watches not yet completed;
 * _fired: timeouts seen (MPM_WATCHDOG_NO_ABORT=1 reports instead of abort). */
int mpm_watchdog_watch(void* stream, double timeout_s, const char* tag);
int mpm_watchdog_pending(void);
unsigned long long mpm_watchdog_fired(void);

/* out[i] = sum over r in [0, n) of slices[r*stride + i], in rank order
 * (fp32; every rank computes identical bits) — the gate-gradient
 * all-reduce over pushed slices (data parallel gate). */
int mpm_sum_slices(const float* slices, int n, int64_t stride, int64_t count,
                   float* out, void* stream);

/* cudaMemcpyAsync wrapper for offload (D2H) / prefetch (H2D) on the copy
 * stream (S1-S3).  Host pointers must be pinned for the copy to overlap. */
int mpm_copy_async(void* dst, const void* src, size_t bytes, int direction,
                   void* stream);

/* ----------------------------------------------------------- events */

/* CUDA events for the host executor's cross-stream dependencies (the
 * schedule DAG edges of pipesim/schedule.py become event waits). */
int mpm_event_create(int timing, void** ev_out);
int mpm_event_destroy(void* ev);
int mpm_event_record(void* ev, void* stream);
int mpm_stream_wait(void* stream, void* ev);
int mpm_event_elapsed_ms(void* start, void* end, float* ms); /* syncs on end */

/* ---- measurement helper (bench.py), not part of the layer path ----------
 * Native NVML sampler: SM clock, max SM clock and clock-event reasons every
 * period_us from its own thread, stamped with CLOCK_MONOTONIC (rows of 4
 * doubles: sm_mhz, max_mhz, reasons bitmask, t).  NVML is dlopen'ed; start
 * fails (nonzero) when it is unavailable. */
int mpm_clock_sampler_start(const char* pci_bus_id, int period_us);
int mpm_clock_sampler_stop(double* out, int max_rows, int* n_rows);
/* In-kernel SM clock trace (measurement): one warp records (globaltimer ns,
 * clock64) pairs every interval_ns into out[2*samples], co-resident with
 * whatever runs; the effective SM clock at microsecond scale. */
int mpm_clock_trace(unsigned long long* out, int samples, long long interval_ns,
                    void* stream);
double mpm_monotonic(void);

#ifdef __cplusplus
}
#endif

#endif /* MPM_H_ */
