// comm.cu -- NCCL communicator of libattnsm.so (see comm.h).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <chrono>
#include <cstdarg>
#include <thread>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "comm.h"
#include "nvtx.cuh"

// Minimal NCCL ABI (nccl.h 2.x): opaque comm, 128-byte unique id, enums.
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef int ncclResult_t;
enum { ncclSuccess_ = 0, ncclInProgress_ = 7 };
enum { ncclFloat32_ = 7, ncclBfloat16_ = 9 };
enum { ncclSum_ = 0 };

// ncclConfig_t of NCCL 2.28 (nccl.h ncclConfig_v22800), so the communicator can
// cap the CTAs NCCL's kernels use (the stage's persistent GEMMs leave that
// many SMs free while a gradient allreduce is in flight).
struct NcclConfigV22800 {
  size_t size;
  unsigned int magic;
  unsigned int version;
  int blocking, cgaClusterSize, minCTAs, maxCTAs;
  const char* netName;
  int splitShare, trafficClass;
  const char* commName;
  int collnetEnable, CTAPolicy, shrinkShare, nvlsCTAs, nChannelsPerNetPeer, nvlinkCentricSched;
};
static NcclConfigV22800 nccl_config(int max_ctas) {
  const int U = (int)0x80000000;   // NCCL_CONFIG_UNDEF_INT
  NcclConfigV22800 c;
  c.size = sizeof(NcclConfigV22800);
  c.magic = 0xcafebeef;
  c.version = 22809;
  c.blocking = U; c.cgaClusterSize = U; c.minCTAs = U; c.maxCTAs = max_ctas > 0 ? max_ctas : U;
  c.netName = nullptr; c.splitShare = U; c.trafficClass = U; c.commName = nullptr;
  c.collnetEnable = U; c.CTAPolicy = U; c.shrinkShare = U; c.nvlsCTAs = U;
  c.nChannelsPerNetPeer = U; c.nvlinkCentricSched = U;
  return c;
}

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommInitRankConfig)(ncclComm_t*, int, ncclUniqueId, int, void*) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  bool ok = false;
  std::string why;
};

static NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    void* h = nullptr;
    for (const char* n : names) {
      h = dlopen(n, RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
      if (!h) h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) {
      api.why = std::string("dlopen(libnccl.so.2) failed: ") + (dlerror() ? dlerror() : "?");
      return;
    }
    api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
    api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
    api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
    api.ReduceScatter = (decltype(api.ReduceScatter))dlsym(h, "ncclReduceScatter");
    api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
    api.CommInitRankConfig = (decltype(api.CommInitRankConfig))dlsym(h, "ncclCommInitRankConfig");
    api.GetVersion = (decltype(api.GetVersion))dlsym(h, "ncclGetVersion");
    api.CommGetAsyncError = (decltype(api.CommGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
    api.CommAbort = (decltype(api.CommAbort))dlsym(h, "ncclCommAbort");
    api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
    api.Send = (decltype(api.Send))dlsym(h, "ncclSend");
    api.Recv = (decltype(api.Recv))dlsym(h, "ncclRecv");
    api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
    api.ok = api.GetUniqueId && api.CommInitRank && api.AllReduce && api.CommDestroy &&
             api.ReduceScatter && api.AllGather;
    if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
  });
  return api;
}

struct attn_comm {
  ncclComm_t comm = nullptr;
  cudaStream_t stream = nullptr;
  std::vector<cudaEvent_t> events;  // fork events, reused round-robin
  cudaEvent_t join = nullptr;
  int device = 0;
  int nranks = 1, rank = 0;
  int max_ctas = 0;   // the CTA cap given to NCCL (0 = NCCL's default)
  cudaEvent_t done = nullptr;   // attn_comm_poll: marks the end of the enqueued comm work
  bool aborted = false;
};

// "comm_max_ctas" option (attn_softmax.cu): CTA cap for communicators created
// afterwards (0 = NCCL default); the stage reserves that many SMs.
int g_comm_max_ctas = 8;

// errors are reported through attn_last_error(); defined in attn_softmax.cu
attn_status_t attn_set_error(attn_status_t code, const char* msg);

static attn_status_t err(attn_status_t code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  return attn_set_error(code, buf);
}

#define CUDA_OK(expr)                                                                            \
  do {                                                                                           \
    cudaError_t e_ = (expr);                                                                     \
    if (e_ != cudaSuccess) return err(ATTN_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)
#define NCCL_OK(expr)                                                                        \
  do {                                                                                       \
    ncclResult_t r_ = (expr);                                                                \
    if (r_ != ncclSuccess_)                                                                  \
      return err(ATTN_ERR_NCCL, "%s: %s", #expr,                                             \
                 nccl().GetErrorString ? nccl().GetErrorString(r_) : "nccl error");          \
  } while (0)

extern "C" attn_status_t attn_comm_get_unique_id(uint8_t id[128]) {
  if (!id) return err(ATTN_ERR_INVALID_ARG, "id is NULL");
  NcclApi& api = nccl();
  if (!api.ok) return err(ATTN_ERR_NCCL, "%s", api.why.c_str());
  ncclUniqueId u;
  NCCL_OK(api.GetUniqueId(&u));
  memcpy(id, u.internal, 128);
  return ATTN_OK;
}

extern "C" attn_status_t attn_comm_init(const uint8_t id[128], int nranks, int rank, int device,
                                        attn_comm_t** out) {
  if (!id || !out) return err(ATTN_ERR_INVALID_ARG, "id / out is NULL");
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return err(ATTN_ERR_INVALID_ARG, "rank %d of %d is invalid", rank, nranks);
  NcclApi& api = nccl();
  if (!api.ok) return err(ATTN_ERR_NCCL, "%s", api.why.c_str());
  CUDA_OK(cudaSetDevice(device));
  attn_comm* c = new attn_comm();
  c->device = device;
  c->nranks = nranks;
  c->rank = rank;
  ncclUniqueId u;
  memcpy(u.internal, id, 128);
  ncclResult_t r;
  int ver = 0;
  if (api.GetVersion) api.GetVersion(&ver);
  if (g_comm_max_ctas > 0 && api.CommInitRankConfig && ver >= 22800) {
    NcclConfigV22800 cfg = nccl_config(g_comm_max_ctas);
    r = api.CommInitRankConfig(&c->comm, nranks, u, rank, &cfg);
    if (r == ncclSuccess_) {
      c->max_ctas = g_comm_max_ctas;
    } else {
      // every rank sees the same library and config, so all fall back together
      c->comm = nullptr;
      r = api.CommInitRank(&c->comm, nranks, u, rank);
    }
  } else {
    r = api.CommInitRank(&c->comm, nranks, u, rank);
  }
  if (r != ncclSuccess_) {
    delete c;
    return err(ATTN_ERR_NCCL, "ncclCommInitRank: %s", api.GetErrorString ? api.GetErrorString(r) : "?");
  }
  // high-priority comm stream so the allreduce kernels get SMs as GEMM CTAs retire
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  CUDA_OK(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, hi));
  c->events.resize(64);
  for (auto& e : c->events) CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CUDA_OK(cudaEventCreateWithFlags(&c->join, cudaEventDisableTiming));
  CUDA_OK(cudaEventCreateWithFlags(&c->done, cudaEventDisableTiming));
  *out = c;
  return ATTN_OK;
}

extern "C" attn_status_t attn_comm_destroy(attn_comm_t* c) {
  if (!c) return ATTN_OK;
  if (!c->aborted) cudaStreamSynchronize(c->stream);
  if (c->comm && nccl().ok) {
    if (c->aborted) { /* ncclCommAbort already freed the communicator */ }
    else nccl().CommDestroy(c->comm);
  }
  if (c->done) cudaEventDestroy(c->done);
  for (auto& e : c->events) cudaEventDestroy(e);
  cudaEventDestroy(c->join);
  cudaStreamDestroy(c->stream);
  delete c;
  return ATTN_OK;
}

extern "C" int attn_comm_nranks(const attn_comm_t* c) { return c ? c->nranks : 1; }

extern "C" attn_status_t attn_comm_poll(attn_comm_t* c, int64_t timeout_ms) {
  if (!c) return err(ATTN_ERR_INVALID_ARG, "comm is NULL");
  if (c->aborted) return err(ATTN_ERR_NCCL, "communicator was aborted by an earlier attn_comm_poll");
  CUDA_OK(cudaSetDevice(c->device));
  CUDA_OK(cudaEventRecord(c->done, c->stream));
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t q = cudaEventQuery(c->done);
    if (q == cudaSuccess) return ATTN_OK;
    if (q != cudaErrorNotReady) return err(ATTN_ERR_CUDA, "comm stream: %s", cudaGetErrorString(q));
    ncclResult_t ae = ncclSuccess_;
    if (nccl().CommGetAsyncError && nccl().CommGetAsyncError(c->comm, &ae) == ncclSuccess_ &&
        ae != ncclSuccess_ && ae != ncclInProgress_) {
      if (nccl().CommAbort) nccl().CommAbort(c->comm);
      c->aborted = true;
      return err(ATTN_ERR_NCCL, "rank %d of %d: NCCL asynchronous error %d (%s); communicator aborted",
                 c->rank, c->nranks, (int)ae,
                 nccl().GetErrorString ? nccl().GetErrorString(ae) : "?");
    }
    const long long ms = std::chrono::duration_cast<std::chrono::milliseconds>(
                             std::chrono::steady_clock::now() - t0).count();
    if (timeout_ms > 0 && ms >= timeout_ms) {
      if (nccl().CommAbort) nccl().CommAbort(c->comm);
      c->aborted = true;
      return err(ATTN_ERR_NCCL, "rank %d of %d: collectives not complete after %lld ms (a rank hung "
                 "or left); communicator aborted", c->rank, c->nranks, (long long)timeout_ms);
    }
    std::this_thread::sleep_for(std::chrono::milliseconds(1));
  }
}

extern "C" attn_status_t attn_grad_allreduce(attn_comm_t* c, float* buf, size_t count, void* stream) {
  attnsm::NvtxRange nvtx_range_("attn_grad_allreduce");
  if (!c || (!buf && count)) return err(ATTN_ERR_INVALID_ARG, "comm / buf is NULL");
  if (count == 0) return ATTN_OK;
  NCCL_OK(nccl().AllReduce(buf, buf, count, ncclFloat32_, ncclSum_, c->comm, (cudaStream_t)stream));
  return ATTN_OK;
}

attn_status_t comm_begin(attn_comm_t* c, cudaStream_t compute, CommRun* run) {
  (void)compute;
  run->n_enqueued = 0;
  return c ? ATTN_OK : err(ATTN_ERR_INVALID_ARG, "comm is NULL");
}

attn_status_t comm_enqueue_allreduce(attn_comm_t* c, CommRun* run, cudaStream_t compute, float* buf,
                                     size_t count) {
  cudaEvent_t e = c->events[run->n_enqueued % c->events.size()];
  CUDA_OK(cudaEventRecord(e, compute));
  CUDA_OK(cudaStreamWaitEvent(c->stream, e, 0));
  NCCL_OK(nccl().AllReduce(buf, buf, count, ncclFloat32_, ncclSum_, c->comm, c->stream));
  run->n_enqueued++;
  return ATTN_OK;
}

attn_status_t comm_fork(attn_comm_t* c, CommRun* run, cudaStream_t compute) {
  cudaEvent_t e = c->events[run->n_enqueued % c->events.size()];
  CUDA_OK(cudaEventRecord(e, compute));
  CUDA_OK(cudaStreamWaitEvent(c->stream, e, 0));
  run->n_enqueued++;
  return ATTN_OK;
}

cudaStream_t comm_stream(attn_comm_t* c) { return c->stream; }

attn_status_t comm_allreduce_forked(attn_comm_t* c, CommRun* run, float* buf, size_t count) {
  (void)run;
  NCCL_OK(nccl().AllReduce(buf, buf, count, ncclFloat32_, ncclSum_, c->comm, c->stream));
  return ATTN_OK;
}

attn_status_t comm_end(attn_comm_t* c, CommRun* run, cudaStream_t compute) {
  (void)run;
  CUDA_OK(cudaEventRecord(c->join, c->stream));
  CUDA_OK(cudaStreamWaitEvent(compute, c->join, 0));
  return ATTN_OK;
}

int comm_nranks(const attn_comm_t* c) { return c ? c->nranks : 1; }
int comm_rank(const attn_comm_t* c) { return c ? c->rank : 0; }

attn_status_t comm_reduce_scatter_f32(attn_comm_t* c, float* buf, size_t shard, cudaStream_t s) {
  // in place: rank r's summed shard lands at buf + r * shard
  NCCL_OK(nccl().ReduceScatter(buf, buf + (size_t)c->rank * shard, shard, ncclFloat32_, ncclSum_,
                               c->comm, s));
  return ATTN_OK;
}

attn_status_t comm_all_gather_bf16(attn_comm_t* c, void* buf, size_t shard, cudaStream_t s) {
  // in place: rank r contributes buf + r * shard
  char* b = static_cast<char*>(buf);
  NCCL_OK(nccl().AllGather(b + (size_t)c->rank * shard * 2, b, shard, ncclBfloat16_, c->comm, s));
  return ATTN_OK;
}

// one rank: the "allreduce" moves nothing, so no SMs are set aside
// "comm_reserve_1rank" option (tests): reserve the communicator's SMs on a
// 1-rank communicator too, so one GPU exercises the reduced-grid launches
int g_comm_reserve_1rank = 0;
int comm_max_ctas(const attn_comm_t* c) {
  return c && (c->nranks > 1 || g_comm_reserve_1rank) ? c->max_ctas : 0;
}

// NEXT-3: MP -> DP scatter of the hidden states (attn_softmax.h).  Shards are
// contiguous sentence ranges, sizes differing by at most one, lower ranks
// first (the same rule as synthetic.shard_range and the stage's partitioning).
static void shard_of(int B, int R, int r, int* lo, int* n) {
  const int base = B / R, extra = B % R;
  *lo = r * base + (r < extra ? r : extra);
  *n = base + (r < extra ? 1 : 0);
}

extern "C" attn_status_t attn_hidden_scatter(attn_comm_t* c, int root, int B_global, int rows,
                                             int hidden, const void* full, void* shard, void* stream) {
  attnsm::NvtxRange nvtx_range_("attn_hidden_scatter");
  if (!c) return err(ATTN_ERR_INVALID_ARG, "hidden_scatter: comm is NULL");
  if (B_global < 0 || rows < 1 || hidden < 1 || root < 0 || root >= c->nranks)
    return err(ATTN_ERR_SHAPE, "hidden_scatter: B_global %d, rows %d, hidden %d, root %d of %d ranks",
               B_global, rows, hidden, root, c->nranks);
  if (!shard || (c->rank == root && !full)) return err(ATTN_ERR_INVALID_ARG, "hidden_scatter: NULL buffer");
  if (!nccl().Send || !nccl().Recv || !nccl().GroupStart || !nccl().GroupEnd)
    return err(ATTN_ERR_NCCL, "hidden_scatter: libnccl lacks ncclSend / ncclRecv / ncclGroup*");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t row_bytes = (size_t)rows * hidden * 2;   // one sentence, bf16
  int lo = 0, n = 0;
  if (c->rank == root) {
    NCCL_OK(nccl().GroupStart());
    for (int r = 0; r < c->nranks; ++r) {
      shard_of(B_global, c->nranks, r, &lo, &n);
      if (r == root || n == 0) continue;
      NCCL_OK(nccl().Send(static_cast<const char*>(full) + (size_t)lo * row_bytes, (size_t)n * row_bytes,
                          0 /* ncclInt8: raw bytes */, r, c->comm, s));
    }
    NCCL_OK(nccl().GroupEnd());
    shard_of(B_global, c->nranks, root, &lo, &n);
    if (n > 0) {
      cudaError_t e = cudaMemcpyAsync(shard, static_cast<const char*>(full) + (size_t)lo * row_bytes,
                                      (size_t)n * row_bytes, cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) return err(ATTN_ERR_CUDA, "hidden_scatter: %s", cudaGetErrorString(e));
    }
  } else {
    shard_of(B_global, c->nranks, c->rank, &lo, &n);
    if (n > 0) NCCL_OK(nccl().Recv(shard, (size_t)n * row_bytes, 0, root, c->comm, s));
  }
  return ATTN_OK;
}
