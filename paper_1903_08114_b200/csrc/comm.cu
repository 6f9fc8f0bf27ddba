// Single-process multi-GPU collectives over NCCL (one host thread drives
// every device with group calls; NVLink / NVSwitch underneath).
//
// Reference seam: the reference spreads the row blocks of every MVM over the
// threads of a WorkerPool (partition.py:46-57, :155-183) inside one process;
// the device equivalent splits the symmetric kernel's work items over the
// GPUs of one process and combines the 64-bit fixed-point partial sums with a
// reduce-scatter (SURVEY §8(b) "Collectives": gp_comm_init ->
// ncclCommInitAll, group calls). The torchrun path (one process per GPU,
// torch.distributed) uses the same partial/finalize entry points.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2, the copy the process
// already has loaded when torch is imported), so the library has no
// link-time NCCL dependency and loads on hosts without it.
#include "gp_common.cuh"

#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <vector>

namespace gp {
namespace {

struct NcclApi {
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
#define GP_NCCL_SYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name))
    GP_NCCL_SYM(CommInitAll, "ncclCommInitAll");
    GP_NCCL_SYM(CommDestroy, "ncclCommDestroy");
    GP_NCCL_SYM(GroupStart, "ncclGroupStart");
    GP_NCCL_SYM(GroupEnd, "ncclGroupEnd");
    GP_NCCL_SYM(Broadcast, "ncclBroadcast");
    GP_NCCL_SYM(AllGather, "ncclAllGather");
    GP_NCCL_SYM(ReduceScatter, "ncclReduceScatter");
    GP_NCCL_SYM(AllReduce, "ncclAllReduce");
    GP_NCCL_SYM(GetErrorString, "ncclGetErrorString");
#undef GP_NCCL_SYM
    api.ok = api.CommInitAll && api.CommDestroy && api.GroupStart && api.GroupEnd && api.Broadcast &&
             api.AllGather && api.ReduceScatter && api.AllReduce && api.GetErrorString;
  });
  return api;
}

}  // namespace
}  // namespace gp

struct gp_comm {
  std::vector<ncclComm_t> comms;
  std::vector<int> devices;
};

using namespace gp;

#define GP_NCCL_TRY(expr)                                                                       \
  do {                                                                                          \
    ncclResult_t _r = (expr);                                                                   \
    if (_r != ncclSuccess)                                                                      \
      return set_error(GP_ENCCL, "%s failed: %s", #expr, nccl().GetErrorString(_r));            \
  } while (0)

namespace {

int check_comm(const gp_comm* c) {
  GP_REQUIRE(c != nullptr && !c->comms.empty(), "gp_comm: null or empty communicator");
  return GP_OK;
}

// one group call over every device of the communicator: f(rank) issues the
// collective of that rank on its stream (the current device set to it)
template <class F>
int group_call(gp_comm* c, F f) {
  if (int rc = check_comm(c)) return rc;
  int prev = 0;
  GP_CUDA_TRY(cudaGetDevice(&prev));
  GP_NCCL_TRY(nccl().GroupStart());
  int rc = GP_OK;
  for (size_t r = 0; r < c->comms.size() && rc == GP_OK; ++r) {
    cudaError_t e = cudaSetDevice(c->devices[r]);
    if (e != cudaSuccess) {
      rc = set_error(GP_ECUDA, "cudaSetDevice(%d): %s", c->devices[r], cudaGetErrorString(e));
      break;
    }
    ncclResult_t nr = f((int)r);
    if (nr != ncclSuccess) rc = set_error(GP_ENCCL, "NCCL collective failed: %s", nccl().GetErrorString(nr));
  }
  ncclResult_t end = nccl().GroupEnd();
  cudaSetDevice(prev);
  if (rc != GP_OK) return rc;
  GP_NCCL_TRY(end);
  return GP_OK;
}

}  // namespace

extern "C" {

int gp_comm_available(void) { return nccl().ok ? 1 : 0; }

int gp_comm_init(int ndev, const int* devices_host, gp_comm** out) {
  GP_REQUIRE(out != nullptr && ndev >= 1 && devices_host != nullptr, "gp_comm_init: ndev=%d", ndev);
  if (!nccl().ok) return set_error(GP_ENCCL, "gp_comm_init: libnccl.so.2 not found or incomplete");
  int count = 0;
  GP_CUDA_TRY(cudaGetDeviceCount(&count));
  for (int r = 0; r < ndev; ++r) {
    GP_REQUIRE(devices_host[r] >= 0 && devices_host[r] < count, "gp_comm_init: device %d of %d",
               devices_host[r], count);
    for (int q = 0; q < r; ++q)
      GP_REQUIRE(devices_host[q] != devices_host[r], "gp_comm_init: device %d listed twice", devices_host[r]);
  }
  gp_comm* c = new gp_comm;
  c->devices.assign(devices_host, devices_host + ndev);
  c->comms.resize(ndev);
  ncclResult_t r = nccl().CommInitAll(c->comms.data(), ndev, devices_host);
  if (r != ncclSuccess) {
    delete c;
    return set_error(GP_ENCCL, "ncclCommInitAll(%d devices): %s", ndev, nccl().GetErrorString(r));
  }
  *out = c;
  return GP_OK;
}

int gp_comm_destroy(gp_comm* comm) {
  if (!comm) return GP_OK;
  int rc = GP_OK;
  for (ncclComm_t h : comm->comms) {
    ncclResult_t r = nccl().CommDestroy(h);
    if (r != ncclSuccess && rc == GP_OK) rc = set_error(GP_ENCCL, "ncclCommDestroy: %s", nccl().GetErrorString(r));
  }
  delete comm;
  return rc;
}

int gp_comm_size(const gp_comm* comm) { return comm ? (int)comm->comms.size() : 0; }

int gp_comm_broadcast(gp_comm* comm, void* const* bufs, int64_t bytes, int root, void* const* streams) {
  GP_REQUIRE(bufs && streams && bytes >= 0, "gp_comm_broadcast: null argument");
  GP_REQUIRE(comm && root >= 0 && root < (int)comm->comms.size(), "gp_comm_broadcast: root %d", root);
  return group_call(comm, [&](int r) {
    return nccl().Broadcast(bufs[r], bufs[r], (size_t)bytes, ncclUint8, root, comm->comms[r],
                            (cudaStream_t)streams[r]);
  });
}

int gp_comm_allgather(gp_comm* comm, const void* const* send, void* const* recv, int64_t bytes_per_rank,
                      void* const* streams) {
  GP_REQUIRE(send && recv && streams && bytes_per_rank >= 0, "gp_comm_allgather: null argument");
  return group_call(comm, [&](int r) {
    return nccl().AllGather(send[r], recv[r], (size_t)bytes_per_rank, ncclUint8, comm->comms[r],
                            (cudaStream_t)streams[r]);
  });
}

int gp_comm_reduce_scatter_i64(gp_comm* comm, const int64_t* const* send, int64_t* const* recv,
                               int64_t count_per_rank, void* const* streams) {
  GP_REQUIRE(send && recv && streams && count_per_rank >= 0, "gp_comm_reduce_scatter_i64: null argument");
  return group_call(comm, [&](int r) {
    return nccl().ReduceScatter(send[r], recv[r], (size_t)count_per_rank, ncclInt64, ncclSum, comm->comms[r],
                                (cudaStream_t)streams[r]);
  });
}

int gp_comm_reduce_scatter_i32(gp_comm* comm, const int32_t* const* send, int32_t* const* recv,
                               int64_t count_per_rank, void* const* streams) {
  GP_REQUIRE(send && recv && streams && count_per_rank >= 0, "gp_comm_reduce_scatter_i32: null argument");
  return group_call(comm, [&](int r) {
    return nccl().ReduceScatter(send[r], recv[r], (size_t)count_per_rank, ncclInt32, ncclSum, comm->comms[r],
                                (cudaStream_t)streams[r]);
  });
}

int gp_comm_allreduce_f64(gp_comm* comm, double* const* bufs, int64_t count, void* const* streams) {
  GP_REQUIRE(bufs && streams && count >= 0, "gp_comm_allreduce_f64: null argument");
  return group_call(comm, [&](int r) {
    return nccl().AllReduce(bufs[r], bufs[r], (size_t)count, ncclFloat64, ncclSum, comm->comms[r],
                            (cudaStream_t)streams[r]);
  });
}

}  // extern "C"
