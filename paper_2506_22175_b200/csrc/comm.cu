// Chunked all-to-all over NCCL (pip NCCL 2.28, the copy torch loads).
//
// One call moves one pipeline chunk (the token batch is
// split along the batch dimension and every chunk is a full N-way
// all-to-all; reference ops S_i / R_i / BS_i / RC_i / BR_i,
// pipesim/schedule.py:252-340).  The receive side lands expert-major so the
// grouped GEMM reads one contiguous [N*c_i][M] block per local expert:
//
//   dispatch: src[d][el][c][M] on rank s  ->  dst[el][s][c][M] on rank d
//   combine : src[el][d][c][M] on rank s  ->  dst[s][el][c][M] on rank d
//
// Every (peer, local expert) block is c_i*M contiguous elements, so the
// exchange is E_loc grouped ncclSend/ncclRecv pairs per peer.  The block
// plan (peer, send offset, recv offset per block) is computed on the host by
// paper_2506_22175_b200/comm.py:block_plan — one definition of the layout,
// exercised by the world-size-2 gloo tests — and executed here.
#include <nccl.h>
#include "common.cuh"

#define MPM_NCCL_RET(expr)                                                              \
  do {                                                                                  \
    ncclResult_t r_ = (expr);                                                           \
    if (r_ != ncclSuccess) {                                                            \
      ::mpm::set_error("%s failed: %s (%s:%d)", #expr, ncclGetErrorString(r_), __FILE__, \
                       __LINE__);                                                       \
      return 2000 + (int)r_;                                                            \
    }                                                                                   \
  } while (0)

extern "C" int mpm_comm_unique_id(void* host_id_out) {
  MPM_CHECK_ARG(host_id_out != nullptr, "null id buffer");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  MPM_NCCL_RET(ncclGetUniqueId(&id));
  memcpy(host_id_out, &id, sizeof(id));
  return 0;
}

extern "C" int mpm_comm_init(const void* host_id, int nranks, int rank, int device, void** comm_out) {
  MPM_CHECK_ARG(host_id && comm_out, "null argument");
  MPM_CHECK_ARG(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank %d of %d", rank, nranks);
  MPM_CUDA_RET(cudaSetDevice(device));
  ncclUniqueId id;
  memcpy(&id, host_id, sizeof(id));
  ncclComm_t comm;
  MPM_NCCL_RET(ncclCommInitRank(&comm, nranks, id, rank));
  *comm_out = comm;
  return 0;
}

extern "C" int mpm_comm_destroy(void* comm) {
  if (!comm) return 0;
  MPM_NCCL_RET(ncclCommDestroy((ncclComm_t)comm));
  return 0;
}

extern "C" int mpm_a2a_chunk(void* comm, int nranks, int n_blocks, const int32_t* host_peer,
                             const int64_t* host_send_off, const int64_t* host_recv_off, int64_t block_elems,
                             int dtype, const void* src, void* dst, void* stream) {
  MPM_CHECK_ARG(dtype == MPM_F32 || dtype == MPM_BF16, "bad dtype %d", dtype);
  MPM_CHECK_ARG(nranks >= 1, "bad nranks %d", nranks);
  MPM_CHECK_ARG(n_blocks >= 0 && (n_blocks == 0 || (host_peer && host_send_off && host_recv_off)),
                "bad block plan");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t esz = mpm::dtype_size(dtype);
  if (block_elems <= 0 || n_blocks == 0) return 0;
  const char* sp = static_cast<const char*>(src);
  char* dp = static_cast<char*>(dst);
  if (nranks == 1 && comm == nullptr) {
    // every block stays on this rank: plain device copies (none when aliased)
    for (int b = 0; b < n_blocks; ++b) {
      MPM_CHECK_ARG(host_peer[b] == 0, "peer %d with nranks=1", host_peer[b]);
      const char* from = sp + host_send_off[b] * esz;
      char* to = dp + host_recv_off[b] * esz;
      if (from != to) MPM_CUDA_RET(cudaMemcpyAsync(to, from, block_elems * esz, cudaMemcpyDeviceToDevice, s));
    }
    return 0;
  }
  MPM_CHECK_ARG(comm != nullptr, "null communicator for nranks=%d", nranks);
  const ncclDataType_t nt = dtype == MPM_BF16 ? ncclBfloat16 : ncclFloat32;
  // every peer is validated before the group opens: an early return must never leave an
  // NCCL group open on this thread
  for (int b = 0; b < n_blocks; ++b)
    MPM_CHECK_ARG(host_peer[b] >= 0 && host_peer[b] < nranks, "peer %d out of range", host_peer[b]);
  MPM_NCCL_RET(ncclGroupStart());
  ncclResult_t r = ncclSuccess;
  for (int b = 0; b < n_blocks && r == ncclSuccess; ++b) {
    const int peer = host_peer[b];
    r = ncclSend(sp + host_send_off[b] * esz, (size_t)block_elems, nt, peer, (ncclComm_t)comm, s);
    if (r == ncclSuccess)
      r = ncclRecv(dp + host_recv_off[b] * esz, (size_t)block_elems, nt, peer, (ncclComm_t)comm, s);
  }
  const ncclResult_t end = ncclGroupEnd();  // closed on the error path too
  MPM_NCCL_RET(r);
  MPM_NCCL_RET(end);
  return 0;
}
