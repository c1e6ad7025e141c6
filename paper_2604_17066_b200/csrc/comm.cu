// Multi-GPU exchange entry points of the C ABI: the per-iteration
// collectives of the sample-sharded path for a caller that is not Python --
// all-reduce of class counts, all-gather of new reference rows, and the OR-reduce of
// classifier hit flags across reference shards.  The reference has no communication
// (its only parallel seam is the thread pool of classify.py:140-142); the Python
// package does the same exchanges through torch.distributed (dist.py).
//
// NCCL is bound at run time (dlopen of libnccl.so.2: in a PyTorch process this finds
// the already-loaded torch copy by soname, so one NCCL serves both), with the types
// and enum values of nccl.h.  Every call is stream-ordered on the caller's stream.
#include <dlfcn.h>
#include <nccl.h>

#include "common.cuh"

namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*);
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*comm_destroy)(ncclComm_t);
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t);
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                             cudaStream_t);
  const char* (*get_error_string)(ncclResult_t);
  bool ok;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a{};
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
    a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(h, "ncclAllGather"));
    a.get_error_string =
        reinterpret_cast<decltype(a.get_error_string)>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.get_unique_id && a.comm_init_rank && a.comm_destroy && a.all_reduce &&
           a.all_gather && a.get_error_string;
    return a;
  }();
  return api;
}

#define RSR_NCCL(expr)                                                                   \
  do {                                                                                   \
    const ncclResult_t r_ = (expr);                                                      \
    if (r_ != ncclSuccess) {                                                             \
      rsr::set_error("%s: %s", #expr, nccl().get_error_string(r_));                      \
      return RSR_ENCCL;                                                                  \
    }                                                                                    \
  } while (0)

#define RSR_NEED_NCCL()                                                                  \
  do {                                                                                   \
    if (!nccl().ok) {                                                                    \
      rsr::set_error("libnccl.so.2 not found or incomplete");                            \
      return RSR_EUNSUPPORTED;                                                           \
    }                                                                                    \
  } while (0)

// flags (bit0 lower hit, bit1 upper hit) -> two 0/1 planes; NCCL has no bitwise OR,
// but MAX over 0/1 planes is OR (MAX over the raw bytes would turn 1 | 2 into 2)
__global__ void split_planes_kernel(const uint8_t* __restrict__ flags, int64_t S,
                                    uint8_t* __restrict__ planes) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < S;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint8_t f = flags[i];
    planes[i] = f & 1u;
    planes[S + i] = (f >> 1) & 1u;
  }
}

__global__ void merge_planes_kernel(const uint8_t* __restrict__ planes, int64_t S,
                                    uint8_t* __restrict__ flags) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < S;
       i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = (uint8_t)(planes[i] | (planes[S + i] << 1));
}

unsigned grid_for(int64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = rsr::ceil_div(n, 256);
  return (unsigned)(want < 8 * sms ? (want > 0 ? want : 1) : 8 * sms);
}

}  // namespace

extern "C" int rsr_comm_unique_id(uint8_t* out_id) {
  RSR_NEED_NCCL();
  RSR_REQUIRE(out_id != nullptr, "rsr_comm_unique_id: null output");
  ncclUniqueId id;
  RSR_NCCL(nccl().get_unique_id(&id));
  memcpy(out_id, id.internal, RSR_COMM_ID_BYTES);
  return RSR_OK;
}

extern "C" int rsr_comm_init(const uint8_t* unique_id, int world, int rank, void** out_comm) {
  RSR_NEED_NCCL();
  RSR_REQUIRE(unique_id && out_comm, "rsr_comm_init: null pointer");
  RSR_REQUIRE(world >= 1 && rank >= 0 && rank < world, "rsr_comm_init: bad rank %d of %d", rank,
              world);
  ncclUniqueId id;
  memcpy(id.internal, unique_id, RSR_COMM_ID_BYTES);
  ncclComm_t c = nullptr;
  RSR_NCCL(nccl().comm_init_rank(&c, world, id, rank));
  *out_comm = c;
  return RSR_OK;
}

extern "C" int rsr_comm_destroy(void* comm) {
  RSR_NEED_NCCL();
  if (comm) RSR_NCCL(nccl().comm_destroy(static_cast<ncclComm_t>(comm)));
  return RSR_OK;
}

extern "C" int rsr_allreduce_counts(void* comm, int64_t* counts, int n, void* stream) {
  RSR_NEED_NCCL();
  RSR_REQUIRE(comm && counts && n >= 0, "rsr_allreduce_counts: bad arguments");
  if (n == 0) return RSR_OK;
  RSR_NCCL(nccl().all_reduce(counts, counts, (size_t)n, ncclInt64, ncclSum,
                             static_cast<ncclComm_t>(comm), rsr::as_stream(stream)));
  return RSR_OK;
}

extern "C" int rsr_allgather_refs(void* comm, const uint8_t* send, int64_t bytes_per_rank,
                                  uint8_t* recv, void* stream) {
  RSR_NEED_NCCL();
  RSR_REQUIRE(comm && bytes_per_rank >= 0, "rsr_allgather_refs: bad arguments");
  if (bytes_per_rank == 0) return RSR_OK;
  RSR_REQUIRE(send && recv, "rsr_allgather_refs: null buffer");
  RSR_NCCL(nccl().all_gather(send, recv, (size_t)bytes_per_rank, ncclUint8,
                             static_cast<ncclComm_t>(comm), rsr::as_stream(stream)));
  return RSR_OK;
}

extern "C" int rsr_or_reduce_flags(void* comm, uint8_t* flags, int64_t S, uint8_t* scratch,
                                   void* stream) {
  RSR_NEED_NCCL();
  RSR_REQUIRE(comm && S >= 0, "rsr_or_reduce_flags: bad arguments");
  if (S == 0) return RSR_OK;
  RSR_REQUIRE(flags && scratch, "rsr_or_reduce_flags: null buffer");
  cudaStream_t st = rsr::as_stream(stream);
  const unsigned g = grid_for(S);
  split_planes_kernel<<<g, 256, 0, st>>>(flags, S, scratch);
  int rc = rsr::check_launch("split_planes_kernel");
  if (rc) return rc;
  RSR_NCCL(nccl().all_reduce(scratch, scratch, (size_t)(2 * S), ncclUint8, ncclMax,
                             static_cast<ncclComm_t>(comm), st));
  merge_planes_kernel<<<g, 256, 0, st>>>(scratch, S, flags);
  return rsr::check_launch("merge_planes_kernel");
}
