/*
 * evo_dap.h — C ABI of the Dynamic Axial Parallelism (DAP) exchange steps around the Evoformer
 * attention core (libevodap.so; NCCL 2.28 over NVLink 5 / NVSwitch).
 *
 * What it implements (§2 "Dynamic Axial Parallelism": DAP "splits intermediate
 * activations and associated computations of a single training sample along a non-reductive
 * axis"; L243: DAP's "all-gather and all-to-all communications"):
 *
 *   - the all-to-all TRANSPOSE that moves a 3-axis activation between the two sharded axes
 *     (MSA m: S-sharded for row attention <-> R-sharded for column attention; pair z:
 *     I-sharded for triangle-start <-> J-sharded for triangle-end), forward and reverse;
 *   - the ALL-GATHER of the pair-bias shards (each rank computes the bias rows of its own z
 *     shard; every rank's attention needs the whole [Lq, H, Lk] bias);
 *   - the REDUCE-SCATTER of the fp32 bias-gradient partials (each rank's evo_attn_bwd sums dbias
 *     over its local batch rows; the sum over ranks is scattered back to the owner of each
 *     bias row).
 *
 * Layout convention.  A "row-sharded" tensor on rank r is X[r*A/n : (r+1)*A/n,
 * :, :] of a logical [A][Bd][C] tensor, stored contiguously as [A/n][Bd][C]; a "column-sharded"
 * tensor is X[:, r*Bd/n : (r+1)*Bd/n, :], stored contiguously as [A][Bd/n][C].  C is given in
 * BYTES (the transpose never looks inside an element).  Bias shards are row-sharded along the
 * query axis of the head-major-inner storage [Lq][H][Lk] (so the gathered bias is one
 * contiguous [Lq][H][Lk] tensor that evo_attn consumes through its bias strides), and dbias is
 * produced in the same storage and reduce-scattered along Lq.
 *
 * Ownership and calling convention (as evo_attn.h):
 *   - every data pointer is caller-owned DEVICE memory, 16-byte aligned; the library allocates
 *     nothing on the hot path (staging buffers come from the caller);
 *   - calls are asynchronous and stream-ordered on `stream`; inputs are never written; dst must
 *     not alias src;
 *   - all ranks must call the collectives in the same order with the same sizes (NCCL rule);
 *   - errors are returned as evo_status_t (values of evo_attn.h) and detailed by
 *     evo_dap_last_error_detail() (thread-local); NCCL failures map to EVO_E_CUDA.
 */
#ifndef EVO_DAP_H
#define EVO_DAP_H

#include <stddef.h>
#include <stdint.h>

#include "evo_attn.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct evo_dap evo_dap_t; /* one NCCL communicator over the DAP group + its device */

#define EVO_DAP_UID_BYTES 128

/* Rank 0 creates the 128-byte NCCL unique id; the caller ships it to the other ranks out of
 * band (the Python layer uses the torch.distributed store). */
evo_status_t evo_dap_unique_id(void* uid /* out, EVO_DAP_UID_BYTES */);

/* Collective over the group: every rank calls it with the same uid and nranks, its own rank, and
 * the CUDA device it drives.  *out receives the handle (NULL on failure). */
evo_status_t evo_dap_init(int32_t nranks, int32_t rank, const void* uid, int32_t device,
                          evo_dap_t** out);
evo_status_t evo_dap_destroy(evo_dap_t* dap); /* NULL is a no-op */
int32_t evo_dap_nranks(const evo_dap_t* dap);
int32_t evo_dap_rank(const evo_dap_t* dap);

/* Bytes of the staging buffer evo_dap_alltoall_transpose needs: the local shard size
 * (A/n)·Bd·C_bytes.  0 when nranks == 1. */
size_t evo_dap_a2a_staging_bytes(const evo_dap_t* dap, int64_t A, int64_t Bd, int64_t C_bytes);

/* All-to-all transpose of a logical [A][Bd][C] tensor between the two sharded axes.
 *   dir = 0 (row -> column): src = this rank's row shard [A/n][Bd][C],
 *                            dst = this rank's column shard [A][Bd/n][C].
 *   dir = 1 (column -> row): src = column shard [A][Bd/n][C], dst = row shard [A/n][Bd][C].
 * A and Bd must be multiples of nranks (EVO_E_SHAPE); C_bytes a multiple of 16 (EVO_E_ALIGN).
 * One pack (dir 0) or unpack (dir 1) kernel through `staging` plus one ncclAlltoAll. */
evo_status_t evo_dap_alltoall_transpose(evo_dap_t* dap, const void* src, void* dst, void* staging,
                                        size_t staging_bytes, int64_t A, int64_t Bd,
                                        int64_t C_bytes, int32_t dir, void* stream /* cudaStream_t */);

/* All-gather: dst[r*bytes_per_rank : (r+1)*bytes_per_rank] = src of rank r (bytes_per_rank a
 * multiple of 16).  Used for the pair-bias rows. */
evo_status_t evo_dap_allgather(evo_dap_t* dap, const void* src, void* dst, size_t bytes_per_rank,
                               void* stream);

/* fp32 sum-reduce-scatter: dst (count_per_rank floats) = Σ_ranks src[rank*count_per_rank ...].
 * Used for the dbias partials. */
evo_status_t evo_dap_reduce_scatter_f32(evo_dap_t* dap, const float* src, float* dst,
                                        size_t count_per_rank, void* stream /* cudaStream_t */);

/* The layout step of the transpose on its own (no communication; tests and fused callers):
 *   dir = 0: dst[j][a][c'] = src[a][j][c']   for src viewed [A_loc][n][W], dst [n][A_loc][W]
 *   dir = 1: dst[a][j][c'] = src[j][a][c']   (the inverse)
 * with W = (Bd/n)·C_bytes bytes.  Bd a multiple of n, C_bytes a multiple of 16. */
evo_status_t evo_dap_pack(const void* src, void* dst, int32_t n, int64_t A_loc, int64_t Bd,
                          int64_t C_bytes, int32_t dir, void* stream /* cudaStream_t */);

/* Global barrier on `stream` over the group (a one-element all-reduce): PAPER.md L233 inserts a
 * synchronisation before the DAP collectives so that stragglers show up as their own time
 * instead of inflating the NCCL kernels of the fast ranks. */
evo_status_t evo_dap_barrier(evo_dap_t* dap, float* scratch /* 1 float, device */,
                             void* stream);

/* Wait for the work enqueued on `stream` (a cudaStream_t) while polling the communicator for an
 * asynchronous NCCL error (ncclCommGetAsyncError): returns EVO_OK once the stream is idle;
 * on an asynchronous error, or when `timeout_s` > 0 seconds pass first (a peer rank died or
 * hangs), aborts the communicator (ncclCommAbort; every later collective call on `dap` fails
 * with EVO_E_INVALID) and returns EVO_E_CUDA with the rank and reason in
 * evo_dap_last_error_detail().  Host-blocking; use it instead of a bare stream synchronise
 * around DAP steps (SURVEY.md §5 failure detection). */
evo_status_t evo_dap_wait(evo_dap_t* dap, void* stream, double timeout_s);

const char* evo_dap_last_error_detail(void);

#ifdef __cplusplus
}
#endif
#endif /* EVO_DAP_H */
