// comm.h -- NCCL plumbing of libattnsm.so (internal).
//
// The gradient exchange of the data-parallel stage ("GPU 0 as
// the root for accumulating and synchronizing") is a rootless NCCL sum
// allreduce over NVLink / NVSwitch.  NCCL is resolved at run time with
// dlopen("libnccl.so.2") (the copy torch already loaded), so the library has
// no link-time NCCL dependency and single-GPU use never touches it.
#pragma once
#include <cuda_runtime.h>

#include "../../include/attn_softmax.h"

// One in-flight fwd_bwd call's use of the communicator: the compute stream
// forks to the comm stream after each finished gradient block and joins back
// at the end.
struct CommRun {
  int n_enqueued = 0;
};

attn_status_t comm_begin(attn_comm_t* c, cudaStream_t compute, CommRun* run);
// Enqueue an in-place fp32 sum allreduce of buf[0..count) that starts once
// `compute` reaches this point, on the communicator's own stream.
attn_status_t comm_enqueue_allreduce(attn_comm_t* c, CommRun* run, cudaStream_t compute,
                                     float* buf, size_t count);
// Fork the comm stream off `compute` at this point (for work enqueued with
// comm_stream() / comm_allreduce_forked: it starts after everything `compute`
// has enqueued so far, without waiting for what `compute` enqueues later).
attn_status_t comm_fork(attn_comm_t* c, CommRun* run, cudaStream_t compute);
cudaStream_t comm_stream(attn_comm_t* c);
// In-place fp32 sum allreduce enqueued on the comm stream as it stands.
attn_status_t comm_allreduce_forked(attn_comm_t* c, CommRun* run, float* buf, size_t count);
// Make `compute` wait for every allreduce enqueued in this run.
attn_status_t comm_end(attn_comm_t* c, CommRun* run, cudaStream_t compute);

// NEXT-2 (sharded optimizer step): communicator size / rank, in-place fp32 sum
// reduce-scatter (rank r's shard at buf + r * shard) and in-place bf16
// all-gather, both enqueued on stream s.
int comm_nranks(const attn_comm_t* c);
int comm_rank(const attn_comm_t* c);
attn_status_t comm_reduce_scatter_f32(attn_comm_t* c, float* buf, size_t shard, cudaStream_t s);
attn_status_t comm_all_gather_bf16(attn_comm_t* c, void* buf, size_t shard, cudaStream_t s);
// CTA cap the communicator gave NCCL (0 = NCCL's default); the stage's
// persistent GEMMs leave that many SMs free while gradients are in flight.
int comm_max_ctas(const attn_comm_t* c);
extern int g_comm_max_ctas;
extern int g_comm_reserve_1rank;
