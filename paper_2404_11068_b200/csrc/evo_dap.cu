// evo_dap.cu — Dynamic Axial Parallelism exchange steps (include/evo_dap.h): the all-to-all
// transpose between the two sharded axes of an Evoformer activation, the pair-bias all-gather
// and the dbias reduce-scatter, on one NCCL communicator per DAP group (NVLink 5 / NVSwitch).
//
// PAPER.md L207 (DAP splits activations along a non-reductive axis), L243 (DAP's all-gather and
// all-to-all communications), L233 (a global synchronisation before the NCCL kernels);
// SURVEY.md §8(e) for the per-module shard axes.
//
// The only device code here is the pack/unpack of the transpose: a 16-byte-vector swap of the
// two leading axes of [X][Y][W bytes] (HBM-bound copy, grid sized to the SM count).  The receive
// side of the forward transpose and the send side of the reverse one are contiguous already, so
// each direction costs one pack OR one unpack plus one ncclAlltoAll.
#include <cuda_runtime.h>
#include <nccl.h>

#include <chrono>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>

#include "evo_dap.h"

struct evo_dap {
  ncclComm_t comm;
  int nranks, rank, device;
};

namespace {

thread_local std::string g_detail;

evo_status_t fail(evo_status_t s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_detail = buf;
  return s;
}

evo_status_t nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return EVO_OK;
  return fail(EVO_E_CUDA, "%s: %s", what, ncclGetErrorString(r));
}

evo_status_t cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return EVO_OK;
  return fail(EVO_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// dst[y][x][:] = src[x][y][:] over rows of W16 16-byte vectors.  `tpr` threads (a power of two
// dividing the block) share one output row, so the row's (x, y) decomposition is one integer
// division per thread per row — amortised over W16 / tpr vectors — instead of a 64-bit
// division/modulo per 16-byte element.
__global__ void __launch_bounds__(256) swap01_kernel(const uint4* __restrict__ src,
                                                     uint4* __restrict__ dst, int64_t X,
                                                     int64_t Y, int64_t W16, int tpr) {
  const int64_t rows = X * Y;
  const int rpb = blockDim.x / tpr;  // rows per block per iteration
  const int sub = threadIdx.x % tpr;
  for (int64_t r = (int64_t)blockIdx.x * rpb + threadIdx.x / tpr; r < rows;
       r += (int64_t)gridDim.x * rpb) {
    const int64_t y = r / X, x = r - y * X;  // output row r = y * X + x
    const uint4* s = src + (x * Y + y) * W16;
    uint4* d = dst + r * W16;
    for (int64_t w = sub; w < W16; w += tpr) d[w] = __ldg(&s[w]);
  }
}

evo_status_t launch_swap01(const void* src, void* dst, int64_t X, int64_t Y, int64_t W_bytes,
                           cudaStream_t st) {
  const int64_t W16 = W_bytes / 16;
  const int64_t rows = X * Y;
  if (rows * W16 == 0) return EVO_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int tpr = 1;
  while (tpr < 256 && tpr < W16) tpr <<= 1;
  const int64_t rpb = 256 / tpr;
  int64_t blocks = (rows + rpb - 1) / rpb;
  const int64_t cap = (int64_t)sms * 8;  // 8 resident 256-thread CTAs per SM
  if (blocks > cap) blocks = cap;
  swap01_kernel<<<(unsigned)blocks, 256, 0, st>>>(static_cast<const uint4*>(src),
                                                   static_cast<uint4*>(dst), X, Y, W16, tpr);
  return cuda_check(cudaGetLastError(), "swap01 launch");
}

}  // namespace

extern "C" {

const char* evo_dap_last_error_detail(void) { return g_detail.c_str(); }

evo_status_t evo_dap_unique_id(void* uid) {
  if (!uid) return fail(EVO_E_INVALID, "uid is NULL");
  ncclUniqueId id;
  evo_status_t s = nccl_check(ncclGetUniqueId(&id), "ncclGetUniqueId");
  if (s != EVO_OK) return s;
  static_assert(sizeof(ncclUniqueId) == EVO_DAP_UID_BYTES, "NCCL unique id size");
  memcpy(uid, &id, sizeof id);
  return EVO_OK;
}

evo_status_t evo_dap_init(int32_t nranks, int32_t rank, const void* uid, int32_t device,
                          evo_dap_t** out) {
  if (!out) return fail(EVO_E_INVALID, "out is NULL");
  *out = nullptr;
  if (!uid) return fail(EVO_E_INVALID, "uid is NULL");
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return fail(EVO_E_INVALID, "rank %d of %d", rank, nranks);
  evo_status_t s = cuda_check(cudaSetDevice(device), "cudaSetDevice");
  if (s != EVO_OK) return s;
  ncclUniqueId id;
  memcpy(&id, uid, sizeof id);
  ncclComm_t comm;
  s = nccl_check(ncclCommInitRank(&comm, nranks, id, rank), "ncclCommInitRank");
  if (s != EVO_OK) return s;
  *out = new evo_dap{comm, nranks, rank, device};
  return EVO_OK;
}

evo_status_t evo_dap_destroy(evo_dap_t* dap) {
  if (!dap) return EVO_OK;
  evo_status_t s = dap->comm ? nccl_check(ncclCommDestroy(dap->comm), "ncclCommDestroy") : EVO_OK;
  delete dap;
  return s;
}

int32_t evo_dap_nranks(const evo_dap_t* dap) { return dap ? dap->nranks : 0; }
int32_t evo_dap_rank(const evo_dap_t* dap) { return dap ? dap->rank : -1; }

size_t evo_dap_a2a_staging_bytes(const evo_dap_t* dap, int64_t A, int64_t Bd, int64_t C_bytes) {
  if (!dap || dap->nranks == 1 || A <= 0 || Bd <= 0 || C_bytes <= 0) return 0;
  return (size_t)(A / dap->nranks) * (size_t)Bd * (size_t)C_bytes;
}

evo_status_t evo_dap_pack(const void* src, void* dst, int32_t n, int64_t A_loc, int64_t Bd,
                          int64_t C_bytes, int32_t dir, void* stream) {
  if (n < 1) return fail(EVO_E_INVALID, "n = %d", n);
  if (A_loc < 0 || Bd < 0 || C_bytes < 0) return fail(EVO_E_SHAPE, "negative extent");
  if (Bd % n) return fail(EVO_E_SHAPE, "Bd = %lld is not a multiple of n = %d", (long long)Bd, n);
  if (C_bytes % 16) return fail(EVO_E_ALIGN, "C_bytes = %lld is not a multiple of 16",
                                (long long)C_bytes);
  if (dir != 0 && dir != 1) return fail(EVO_E_INVALID, "dir = %d", dir);
  if ((long long)A_loc * Bd * C_bytes == 0) return EVO_OK;
  if (!src || !dst) return fail(EVO_E_INVALID, "NULL buffer");
  if (!aligned16(src) || !aligned16(dst)) return fail(EVO_E_ALIGN, "buffer not 16-byte aligned");
  const int64_t W = (Bd / n) * C_bytes;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // dir 0: src [A_loc][n][W] -> dst [n][A_loc][W];  dir 1: src [n][A_loc][W] -> dst [A_loc][n][W]
  return dir == 0 ? launch_swap01(src, dst, A_loc, n, W, st) : launch_swap01(src, dst, n, A_loc, W, st);
}

evo_status_t evo_dap_alltoall_transpose(evo_dap_t* dap, const void* src, void* dst, void* staging,
                                        size_t staging_bytes, int64_t A, int64_t Bd,
                                        int64_t C_bytes, int32_t dir, void* stream) {
  if (!dap || !dap->comm) return fail(EVO_E_INVALID, "dap is NULL or its communicator was aborted");
  const int n = dap->nranks;
  if (A < 0 || Bd < 0 || C_bytes < 0) return fail(EVO_E_SHAPE, "negative extent");
  if (A % n || Bd % n)
    return fail(EVO_E_SHAPE, "A = %lld and Bd = %lld must be multiples of nranks = %d",
                (long long)A, (long long)Bd, n);
  if (C_bytes % 16) return fail(EVO_E_ALIGN, "C_bytes = %lld is not a multiple of 16",
                                (long long)C_bytes);
  if (dir != 0 && dir != 1) return fail(EVO_E_INVALID, "dir = %d", dir);
  const size_t shard = (size_t)(A / n) * (size_t)Bd * (size_t)C_bytes;
  if (shard == 0) return EVO_OK;
  if (!src || !dst) return fail(EVO_E_INVALID, "NULL buffer");
  if (!aligned16(src) || !aligned16(dst)) return fail(EVO_E_ALIGN, "buffer not 16-byte aligned");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n == 1)  // the row shard and the column shard are the same tensor
    return cuda_check(cudaMemcpyAsync(dst, src, shard, cudaMemcpyDeviceToDevice, st), "copy");
  if (!staging || staging_bytes < shard)
    return fail(EVO_E_WORKSPACE, "staging %zu bytes < %zu", staging_bytes, shard);
  if (!aligned16(staging)) return fail(EVO_E_ALIGN, "staging not 16-byte aligned");
  const size_t per_peer = shard / n;
  evo_status_t s;
  if (dir == 0) {
    // pack [A/n][n][Bd/n·C] -> [n][A/n][Bd/n·C]; peer j receives block j; what arrives from rank i
    // is rows i·A/n.. of this rank's column block: dst = [A][Bd/n][C] contiguous, no unpack
    s = evo_dap_pack(src, staging, n, A / n, Bd, C_bytes, 0, stream);
    if (s != EVO_OK) return s;
    return nccl_check(ncclAlltoAll(staging, dst, per_peer, ncclUint8, dap->comm, st), "ncclAlltoAll");
  }
  // reverse: rows j·A/n.. of the column shard go to rank j (contiguous), blocks arrive as
  // [n][A/n][Bd/n·C] and are unpacked into the row shard [A/n][Bd][C]
  s = nccl_check(ncclAlltoAll(src, staging, per_peer, ncclUint8, dap->comm, st), "ncclAlltoAll");
  if (s != EVO_OK) return s;
  return evo_dap_pack(staging, dst, n, A / n, Bd, C_bytes, 1, stream);
}

evo_status_t evo_dap_allgather(evo_dap_t* dap, const void* src, void* dst, size_t bytes_per_rank,
                               void* stream) {
  if (!dap || !dap->comm) return fail(EVO_E_INVALID, "dap is NULL or its communicator was aborted");
  if (bytes_per_rank == 0) return EVO_OK;
  if (!src || !dst) return fail(EVO_E_INVALID, "NULL buffer");
  if (bytes_per_rank % 16 || !aligned16(src) || !aligned16(dst))
    return fail(EVO_E_ALIGN, "allgather buffers/size must be 16-byte multiples");
  return nccl_check(ncclAllGather(src, dst, bytes_per_rank, ncclUint8, dap->comm,
                                  static_cast<cudaStream_t>(stream)),
                    "ncclAllGather");
}

evo_status_t evo_dap_reduce_scatter_f32(evo_dap_t* dap, const float* src, float* dst,
                                        size_t count_per_rank, void* stream) {
  if (!dap || !dap->comm) return fail(EVO_E_INVALID, "dap is NULL or its communicator was aborted");
  if (count_per_rank == 0) return EVO_OK;
  if (!src || !dst) return fail(EVO_E_INVALID, "NULL buffer");
  if (!aligned16(src) || !aligned16(dst)) return fail(EVO_E_ALIGN, "buffer not 16-byte aligned");
  return nccl_check(ncclReduceScatter(src, dst, count_per_rank, ncclFloat32, ncclSum, dap->comm,
                                      static_cast<cudaStream_t>(stream)),
                    "ncclReduceScatter");
}

evo_status_t evo_dap_wait(evo_dap_t* dap, void* stream, double timeout_s) {
  if (!dap || !dap->comm) return fail(EVO_E_INVALID, "dap is NULL or its communicator was aborted");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    ncclResult_t ar = ncclSuccess;
    ncclResult_t r = ncclCommGetAsyncError(dap->comm, &ar);
    if (r != ncclSuccess || (ar != ncclSuccess && ar != ncclInProgress)) {
      ncclCommAbort(dap->comm);
      dap->comm = nullptr;
      return fail(EVO_E_CUDA, "NCCL asynchronous error on rank %d: %s (communicator aborted)",
                  dap->rank, ncclGetErrorString(r != ncclSuccess ? r : ar));
    }
    const cudaError_t q = cudaStreamQuery(st);
    if (q == cudaSuccess) return EVO_OK;
    if (q != cudaErrorNotReady) return cuda_check(q, "cudaStreamQuery");
    const double el =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (timeout_s > 0 && el > timeout_s) {
      ncclCommAbort(dap->comm);
      dap->comm = nullptr;
      return fail(EVO_E_CUDA, "rank %d: stream not done after %.1f s (a peer is missing or "
                  "hung; communicator aborted)", dap->rank, el);
    }
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

evo_status_t evo_dap_barrier(evo_dap_t* dap, float* scratch, void* stream) {
  if (!dap || !dap->comm) return fail(EVO_E_INVALID, "dap is NULL or its communicator was aborted");
  if (!scratch) return fail(EVO_E_INVALID, "scratch is NULL");
  return nccl_check(ncclAllReduce(scratch, scratch, 1, ncclFloat32, ncclSum, dap->comm,
                                  static_cast<cudaStream_t>(stream)),
                    "ncclAllReduce(barrier)");
}

}  // extern "C"
