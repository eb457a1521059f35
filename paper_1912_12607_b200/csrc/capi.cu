// capi.cu -- context, error reporting and scratch management behind i8t_cuda.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstdio>
#include <string>

#include "internal.cuh"

namespace i8t_dev {

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

void count_launch(int n) { g_launches.fetch_add(static_cast<uint64_t>(n), std::memory_order_relaxed); }

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("I8T_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

int set_error(int status, const std::string& msg) {
  g_last_error = msg;
  return status;
}

int cuda_check(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(I8T_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return I8T_OK;
}

double* ensure_partials(Ctx* c, size_t doubles) {
  if (doubles <= c->partials_cap) return c->d_partials;
  // growth is rare (first use of a larger reduction); keep ordering on the stream
  cudaStreamSynchronize(c->stream);
  if (c->d_partials) cudaFree(c->d_partials);
  c->d_partials = nullptr;
  size_t cap = doubles < 4096 ? 4096 : doubles * 2;
  if (cudaMalloc(&c->d_partials, cap * sizeof(double)) != cudaSuccess) {
    c->partials_cap = 0;
    return nullptr;
  }
  c->partials_cap = cap;
  return c->d_partials;
}

void* ensure_scratch(Ctx* c, size_t bytes) {
  if (bytes <= c->scratch_cap) return c->d_scratch;
  cudaStreamSynchronize(c->stream);
  if (c->d_scratch) cudaFree(c->d_scratch);
  c->d_scratch = nullptr;
  size_t cap = bytes < 65536 ? 65536 : bytes * 2;
  if (cudaMalloc(&c->d_scratch, cap) != cudaSuccess) {
    c->scratch_cap = 0;
    return nullptr;
  }
  cudaMemset(c->d_scratch, 0, cap);
  c->scratch_cap = cap;
  return c->d_scratch;
}

void* ensure_wgrad(Ctx* c, size_t bytes) {
  if (bytes <= c->wgrad_cap) return c->d_wgrad;
  cudaStreamSynchronize(c->stream);
  if (c->d_wgrad) cudaFree(c->d_wgrad);
  c->d_wgrad = nullptr;
  size_t cap = bytes + bytes / 4;
  if (cudaMalloc(&c->d_wgrad, cap) != cudaSuccess) {
    c->wgrad_cap = 0;
    return nullptr;
  }
  c->wgrad_cap = cap;
  return c->d_wgrad;
}

void* ensure_fold(Ctx* c, size_t bytes) {
  if (bytes <= c->fold_cap) return c->d_fold;
  cudaStreamSynchronize(c->stream);
  if (c->d_fold) cudaFree(c->d_fold);
  c->d_fold = nullptr;
  if (cudaMalloc(&c->d_fold, bytes) != cudaSuccess) {
    c->fold_cap = 0;
    return nullptr;
  }
  c->fold_cap = bytes;
  return c->d_fold;
}

int ctx_allreduce(Ctx* c, double* buf, int64_t count, int op) {
  if (count <= 0) return I8T_OK;
  if (c->nccl_comm) return ctx_allreduce_nccl(c, buf, count, op);
  if (!c->allreduce) return I8T_OK;
  const int rc = c->allreduce(c->allreduce_user, buf, count, 0, op, c->stream);
  return rc ? set_error(I8T_ECUDA, "allreduce hook failed") : I8T_OK;
}

}  // namespace i8t_dev

using namespace i8t_dev;

extern "C" {

int i8t_abi_version(void) { return I8T_ABI_VERSION; }

const char* i8t_last_error(void) { return g_last_error.c_str(); }

uint64_t i8t_launch_count(void) { return g_launches.load(); }

int i8t_ctx_create(void* stream, i8t_ctx** out) {
  if (!out) return set_error(I8T_EINVAL, "ctx_create: null output");
  int dev_count = 0;
  if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0)
    return set_error(I8T_ECUDA, "ctx_create: no CUDA device (this library has no CPU fallback)");
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, dev);
  if (prop.major != 10) return set_error(I8T_EUNSUPPORTED, "ctx_create: requires an sm_100 (B200) device");
  Ctx* c = new Ctx();
  c->stream = reinterpret_cast<cudaStream_t>(stream);
  if (cudaMalloc(&c->d_err, sizeof(int)) != cudaSuccess || cudaMalloc(&c->d_totals, 128 * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&c->d_ticket, sizeof(unsigned)) != cudaSuccess) {
    delete c;
    return set_error(I8T_ECUDA, "ctx_create: cudaMalloc failed");
  }
  cudaMemset(c->d_err, 0, sizeof(int));
  cudaMemset(c->d_totals, 0, 128 * sizeof(double));
  cudaMemset(c->d_ticket, 0, sizeof(unsigned));
  cudaDeviceSynchronize();
  *out = reinterpret_cast<i8t_ctx*>(c);
  return cuda_check("ctx_create");
}

int i8t_device_alloc(i8t_ctx* ctx, uint64_t bytes, void** out) {
  if (!ctx || !out) return set_error(I8T_EINVAL, "device_alloc: bad arguments");
  *out = nullptr;
  if (bytes == 0) return I8T_OK;
  if (cudaMalloc(out, bytes) != cudaSuccess) return set_error(I8T_ECUDA, "device_alloc: cudaMalloc failed");
  return I8T_OK;
}

int i8t_device_free(i8t_ctx* ctx, void* ptr) {
  if (!ctx) return set_error(I8T_EINVAL, "device_free: null ctx");
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (ptr) {
    cudaStreamSynchronize(c->stream);
    cudaFree(ptr);
  }
  return cuda_check("device_free");
}

int i8t_memcpy(i8t_ctx* ctx, void* dst, const void* src, uint64_t bytes, int kind) {
  if (!ctx || (bytes && (!dst || !src)) || kind < 0 || kind > 2) return set_error(I8T_EINVAL, "memcpy: bad arguments");
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!bytes) return I8T_OK;
  const cudaMemcpyKind k = kind == 0 ? cudaMemcpyHostToDevice : (kind == 1 ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice);
  cudaMemcpyAsync(dst, src, bytes, k, c->stream);
  cudaStreamSynchronize(c->stream);
  return cuda_check("memcpy");
}

int i8t_ctx_set_stream(i8t_ctx* ctx, void* stream) {
  if (!ctx) return set_error(I8T_EINVAL, "ctx_set_stream: null ctx");
  reinterpret_cast<Ctx*>(ctx)->stream = reinterpret_cast<cudaStream_t>(stream);
  return I8T_OK;
}

int i8t_ctx_set_allreduce(i8t_ctx* ctx, i8t_allreduce_fn fn, void* user) {
  if (!ctx) return set_error(I8T_EINVAL, "ctx_set_allreduce: null ctx");
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  c->allreduce = fn;
  c->allreduce_user = user;
  return I8T_OK;
}

int i8t_ctx_set_shard(i8t_ctx* ctx, int rank, int world) {
  if (!ctx || world < 1 || rank < 0 || rank >= world) return set_error(I8T_EINVAL, "ctx_set_shard: bad rank/world");
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  c->rank = rank;
  c->world = world;
  return I8T_OK;
}

int i8t_ctx_destroy(i8t_ctx* ctx) {
  if (!ctx) return I8T_OK;
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  cudaStreamSynchronize(c->stream);
  ctx_comm_destroy(c);
  if (c->d_err) cudaFree(c->d_err);
  if (c->d_partials) cudaFree(c->d_partials);
  if (c->d_scratch) cudaFree(c->d_scratch);
  if (c->d_totals) cudaFree(c->d_totals);
  if (c->d_wgrad) cudaFree(c->d_wgrad);
  if (c->d_fold) cudaFree(c->d_fold);
  if (c->d_hist) cudaFree(c->d_hist);
  if (c->d_ticket) cudaFree(c->d_ticket);
  if (c->d_tickets) cudaFree(c->d_tickets);
  if (c->d_set_tickets) cudaFree(c->d_set_tickets);
  delete c;
  return I8T_OK;
}

// dst <- src (bytes) iff *flag != 0, on the stream (no host round trip): the
// trainer's restore of the pre-backward device state on a diverged step.
static __global__ void k_copy_if(const int32_t* flag, uint4* dst, const uint4* src, int64_t n16, uint8_t* dtail,
                                 const uint8_t* stail, int tail) {
  pdl_entry();
  if (!*flag) return;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n16; i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = src[i];
  if (blockIdx.x == 0 && static_cast<int>(threadIdx.x) < tail) dtail[threadIdx.x] = stail[threadIdx.x];
}

int i8t_copy_if(i8t_ctx* ctx, const int32_t* flag, void* dst, const void* src, int64_t bytes) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !flag || !dst || !src || bytes < 0) return set_error(I8T_EINVAL, "copy_if: bad arguments");
  if ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15u)
    return set_error(I8T_EUNSUPPORTED, "copy_if: 16-byte alignment");
  const int64_t n16 = bytes / 16;
  const int tail = static_cast<int>(bytes - n16 * 16);
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>(std::max<int64_t>((n16 + 255) / 256, 1), 148 * 4));
  launch_k(k_copy_if, blocks, 256, 0, c->stream, flag, static_cast<uint4*>(dst), static_cast<const uint4*>(src), n16,
           static_cast<uint8_t*>(dst) + n16 * 16, static_cast<const uint8_t*>(src) + n16 * 16, tail);
  count_launch(1);
  return cuda_check("k_copy_if");
}

int i8t_ctx_error_word(i8t_ctx* ctx, int32_t** out) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !out) return set_error(I8T_EINVAL, "ctx_error_word: bad arguments");
  *out = reinterpret_cast<int32_t*>(c->d_err);
  return I8T_OK;
}

int i8t_ctx_check(i8t_ctx* ctx) {
  if (!ctx) return set_error(I8T_EINVAL, "ctx_check: null ctx");
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return set_error(I8T_ECUDA, std::string("stream: ") + cudaGetErrorString(e));
  int h = 0;
  cudaMemcpy(&h, c->d_err, sizeof(int), cudaMemcpyDeviceToHost);
  cudaMemset(c->d_err, 0, sizeof(int));
  if (h & ERR_NONFINITE) return set_error(I8T_EDOMAIN, "quantize: non-finite input element");
  if (h) return set_error(I8T_ECUDA, "device error word set");
  return cuda_check("ctx_check");
}

}  // extern "C"
