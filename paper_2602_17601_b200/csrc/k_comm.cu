// Native data plane of the node-partitioned step (SURVEY 8b gm_init_comm,
// 8e): an NCCL communicator owned by a context, grouped point-to-point
// send/recv of the halo buffers and the all-reduce of [H | g | C | d], all
// stream-ordered with no host synchronisation, so a rank's whole RTI step
// (kernels + exchanges) can be captured in one CUDA graph.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2): inside a PyTorch
// process that is the library torch already loaded, so both share one NCCL;
// the reference has no counterpart (its only parallelism is the node-chunk
// thread pool of condensing.py:208-227, which the partition generalises).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <type_traits>

#include "common.cuh"

namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      return fn != nullptr;
    };
    api.ok = sym(api.GetUniqueId, "ncclGetUniqueId") && sym(api.CommInitRank, "ncclCommInitRank") &&
             sym(api.CommDestroy, "ncclCommDestroy") && sym(api.AllReduce, "ncclAllReduce") &&
             sym(api.Send, "ncclSend") && sym(api.Recv, "ncclRecv") && sym(api.GroupStart, "ncclGroupStart") &&
             sym(api.GroupEnd, "ncclGroupEnd") && sym(api.GetErrorString, "ncclGetErrorString");
  });
  return api;
}

int nccl_fail(gm_ctx* ctx, ncclResult_t r, const char* what) {
  const NcclApi& a = nccl();
  return gm_fail(ctx, GM_ERR_CUDA,
                 std::string(what) + ": " + (a.GetErrorString ? a.GetErrorString(r) : "NCCL error"));
}

#define GM_NCCL(ctx, expr)                                   \
  do {                                                       \
    ncclResult_t _r = (expr);                                \
    if (_r != ncclSuccess) return nccl_fail((ctx), _r, #expr); \
  } while (0)

int need_comm(gm_ctx* ctx) {
  int rc = gm_need_device(ctx);
  if (rc) return rc;
  if (!ctx->nccl_comm) return gm_fail(ctx, GM_ERR_CONFIG, "no communicator (gm_init_comm)");
  return GM_OK;
}

}  // namespace

void gm_comm_release(gm_ctx* ctx) {
  if (ctx && ctx->nccl_comm && nccl().ok) nccl().CommDestroy((ncclComm_t)ctx->nccl_comm);
  if (ctx) ctx->nccl_comm = nullptr;
}

extern "C" {

int gm_comm_available(void) { return nccl().ok ? 1 : 0; }

int gm_comm_unique_id(void* out) {
  if (!out) return GM_ERR_CONFIG;
  const NcclApi& a = nccl();
  if (!a.ok) return GM_ERR_CUDA;
  ncclUniqueId id;
  if (a.GetUniqueId(&id) != ncclSuccess) return GM_ERR_CUDA;
  std::memcpy(out, &id, sizeof(id));
  return GM_OK;
}

int gm_init_comm(gm_ctx* ctx, const void* unique_id, int rank, int world) {
  int rc = gm_need_device(ctx);
  if (rc) return rc;
  if (!unique_id || world < 1 || rank < 0 || rank >= world)
    return gm_fail(ctx, GM_ERR_CONFIG, "gm_init_comm: need a unique id and 0 <= rank < world");
  const NcclApi& a = nccl();
  if (!a.ok) return gm_fail(ctx, GM_ERR_CUDA, "libnccl.so.2 not found");
  gm_comm_release(ctx);
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  ncclComm_t comm = nullptr;
  GM_NCCL(ctx, a.CommInitRank(&comm, world, id, rank));
  ctx->nccl_comm = comm;
  ctx->comm_rank = rank;
  ctx->comm_world = world;
  return GM_OK;
}

int gm_comm_destroy(gm_ctx* ctx) {
  if (!ctx) return GM_ERR_CONFIG;
  gm_comm_release(ctx);
  return GM_OK;
}

// in-place sum over the ranks (fp64: [H | g | C | d] of the partitioned step)
int gm_allreduce_sum(gm_ctx* ctx, double* buf, int64_t count, void* stream) {
  int rc = need_comm(ctx);
  if (rc) return rc;
  if (count < 0 || (count > 0 && !buf)) return gm_fail(ctx, GM_ERR_CONFIG, "gm_allreduce_sum: bad buffer");
  if (count == 0) return GM_OK;
  GM_NCCL(ctx, nccl().AllReduce(buf, buf, (size_t)count, ncclFloat64, ncclSum, (ncclComm_t)ctx->nccl_comm,
                                (cudaStream_t)stream));
  return GM_OK;
}

// one grouped batch of byte transfers: send_bufs[i] (send_bytes[i]) to rank
// send_peers[i], recv_bufs[j] (recv_bytes[j]) from rank recv_peers[j]; the
// host arrays are read during the call only
int gm_sendrecv(gm_ctx* ctx, int nsend, const int* send_peers, void* const* send_bufs, const int64_t* send_bytes,
                int nrecv, const int* recv_peers, void* const* recv_bufs, const int64_t* recv_bytes,
                void* stream) {
  int rc = need_comm(ctx);
  if (rc) return rc;
  if (nsend < 0 || nrecv < 0 || (nsend && (!send_peers || !send_bufs || !send_bytes)) ||
      (nrecv && (!recv_peers || !recv_bufs || !recv_bytes)))
    return gm_fail(ctx, GM_ERR_CONFIG, "gm_sendrecv: bad peer lists");
  for (int i = 0; i < nsend; ++i)
    if (send_peers[i] < 0 || send_peers[i] >= ctx->comm_world || send_bytes[i] < 0)
      return gm_fail(ctx, GM_ERR_CONFIG, "gm_sendrecv: bad send peer / size");
  for (int j = 0; j < nrecv; ++j)
    if (recv_peers[j] < 0 || recv_peers[j] >= ctx->comm_world || recv_bytes[j] < 0)
      return gm_fail(ctx, GM_ERR_CONFIG, "gm_sendrecv: bad recv peer / size");
  if (nsend + nrecv == 0) return GM_OK;
  const NcclApi& a = nccl();
  ncclComm_t comm = (ncclComm_t)ctx->nccl_comm;
  cudaStream_t st = (cudaStream_t)stream;
  GM_NCCL(ctx, a.GroupStart());
  for (int i = 0; i < nsend; ++i) {
    const ncclResult_t r = a.Send(send_bufs[i], (size_t)send_bytes[i], ncclInt8, send_peers[i], comm, st);
    if (r != ncclSuccess) {
      a.GroupEnd();
      return nccl_fail(ctx, r, "ncclSend");
    }
  }
  for (int j = 0; j < nrecv; ++j) {
    const ncclResult_t r = a.Recv(recv_bufs[j], (size_t)recv_bytes[j], ncclInt8, recv_peers[j], comm, st);
    if (r != ncclSuccess) {
      a.GroupEnd();
      return nccl_fail(ctx, r, "ncclRecv");
    }
  }
  GM_NCCL(ctx, a.GroupEnd());
  return GM_OK;
}

}  // extern "C"
