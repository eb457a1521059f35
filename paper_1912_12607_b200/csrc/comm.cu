// comm.cu -- the data-parallel collectives of the gradient quantiser inside the
// library: an NCCL communicator owned by the i8t_ctx, so the per-layer DSGC
// statistics (max|g|, the d_c / eps / g_hat sums, the search candidates' sums;
// SURVEY.md 8e) are combined by NCCL on the context's stream -- no host
// callback, no host sync, capturable in a CUDA graph.  NCCL is resolved at run
// time (dlopen of libnccl.so.2; the copy PyTorch already loaded is reused), so
// the library keeps no link-time NCCL dependency.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <string>

#include "internal.cuh"

namespace i8t_dev {

namespace {
struct NcclApi {
  bool ok = false;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's NCCL (PyTorch's), if loaded
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return api;
  api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
  api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
  api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
  api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
  api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
  api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_gather && api.error_string;
  return api;
}

int nccl_error(const char* what, ncclResult_t r) {
  return set_error(I8T_ECUDA, std::string(what) + ": " + (nccl().error_string ? nccl().error_string(r) : "?"));
}

// totals[j] = fold over the ranks' rows in rank order: [0] MAX (when op == 2,
// or every j when op == 1), SUM otherwise -- identical on every rank.
__global__ void k_fold_gathered(const double* __restrict__ rows, int64_t count, int world, int op, double* out) {
  pdl_entry();
  for (int64_t j = threadIdx.x; j < count; j += blockDim.x) {
    const bool mx = op == 1 || (op == 2 && j == 0);
    double v = rows[j];
    for (int r = 1; r < world; ++r) {
      const double x = rows[static_cast<int64_t>(r) * count + j];
      v = mx ? fmax(v, x) : v + x;
    }
    out[j] = v;
  }
}
}  // namespace

// The collective behind ctx_allreduce when the context owns a communicator:
// one all-gather of every rank's buffer and a fixed-order fold (a single
// latency-bound collective for the mixed MAX / SUM buffers of op 2).
int ctx_allreduce_nccl(Ctx* c, double* buf, int64_t count, int op) {
  if (count > c->gather_cap) return set_error(I8T_EUNSUPPORTED, "allreduce: buffer larger than the gather scratch");
  const ncclResult_t r = nccl().all_gather(buf, c->d_gather, static_cast<size_t>(count), ncclFloat64,
                                           reinterpret_cast<ncclComm_t>(c->nccl_comm), c->stream);
  if (r != ncclSuccess) return nccl_error("ncclAllGather", r);
  launch_k(k_fold_gathered, 1, 256, 0, c->stream, c->d_gather, count, c->world, op, buf);
  count_launch(1);
  return cuda_check("k_fold_gathered");
}

int ctx_comm_destroy(Ctx* c) {
  if (c->nccl_comm) nccl().comm_destroy(reinterpret_cast<ncclComm_t>(c->nccl_comm));
  c->nccl_comm = nullptr;
  if (c->d_gather) cudaFree(c->d_gather);
  c->d_gather = nullptr;
  c->gather_cap = 0;
  return I8T_OK;
}

}  // namespace i8t_dev

using namespace i8t_dev;

extern "C" {

int i8t_nccl_unique_id(uint8_t* out, int64_t bytes) {
  if (!out || bytes < static_cast<int64_t>(sizeof(ncclUniqueId))) return set_error(I8T_EINVAL, "nccl_unique_id: buffer");
  if (!nccl().ok) return set_error(I8T_EUNSUPPORTED, "nccl_unique_id: libnccl.so.2 not available");
  ncclUniqueId id;
  const ncclResult_t r = nccl().get_unique_id(&id);
  if (r != ncclSuccess) return nccl_error("ncclGetUniqueId", r);
  std::memcpy(out, &id, sizeof(id));
  return I8T_OK;
}

int i8t_ctx_set_nccl(i8t_ctx* ctx, const uint8_t* id, int64_t bytes, int rank, int world) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return set_error(I8T_EINVAL, "ctx_set_nccl: null ctx");
  ctx_comm_destroy(c);
  if (!id) {  // detach
    c->rank = 0;
    c->world = 1;
    return I8T_OK;
  }
  if (bytes < static_cast<int64_t>(sizeof(ncclUniqueId)) || world < 1 || rank < 0 || rank >= world)
    return set_error(I8T_EINVAL, "ctx_set_nccl: bad id / rank / world");
  if (!nccl().ok) return set_error(I8T_EUNSUPPORTED, "ctx_set_nccl: libnccl.so.2 not available");
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t comm = nullptr;
  const ncclResult_t r = nccl().comm_init_rank(&comm, world, uid, rank);
  if (r != ncclSuccess) return nccl_error("ncclCommInitRank", r);
  c->gather_cap = 128;
  if (cudaMalloc(&c->d_gather, sizeof(double) * c->gather_cap * world) != cudaSuccess) {
    nccl().comm_destroy(comm);
    return set_error(I8T_ECUDA, "ctx_set_nccl: gather scratch");
  }
  c->nccl_comm = comm;
  c->rank = rank;
  c->world = world;
  return I8T_OK;
}

}  // extern "C"
