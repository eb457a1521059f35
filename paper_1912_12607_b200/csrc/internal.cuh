// internal.cuh -- shared declarations of the sm_100a kernels behind i8t_cuda.h.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <utility>

#include "../../include/i8t_cuda.h"

namespace i8t_dev {

constexpr uint32_t LCG_A = 1664525u;
constexpr uint32_t LCG_C = 1013904223u;

// affine map x -> a*x + c (mod 2^32); composition of LCG steps.
struct Affine {
  uint32_t a, c;
};

__host__ __device__ inline Affine lcg_jump_map(uint64_t k) {
  uint32_t mul = 1u, add = 0u, am = LCG_A, cm = LCG_C;
  while (k) {
    if (k & 1u) {
      mul = am * mul;
      add = am * add + cm;
    }
    cm = am * cm + cm;
    am = am * am;
    k >>= 1u;
  }
  return {mul, add};
}

// error bits latched in the context's device error word
enum : int { ERR_NONFINITE = 1, ERR_INTERNAL = 2 };

// Device-side DSGC state (public view first, search scratch after).
struct DsgcState {
  i8t_dsgc_view v;
  // --- search scratch (clip.cpp:30-78)
  float m;            // max_abs(g) of the search
  float best_clip;
  double best_dc;
  double sq_g;        // sum g^2
  double lo, hi, x1, x2, f1, f2;
  int32_t active;     // search in progress and not short-circuited
  int32_t ncand;      // candidates in cand[]
  int32_t phase;      // 0 grid, 1 golden-init, 2.. rounds
  int32_t grid_done;  // grid candidates consumed so far
  float cand[32];
  float prev_clip;
  int32_t pad_;
  int32_t hist;         // the grid pass runs on the boundary histogram (dsgc.cu)
  int32_t grid_active;  // active && !hist: the per-candidate grid pass runs instead
};

// Context: stream, error word, scratch, data-parallel hooks.
struct Ctx {
  cudaStream_t stream = nullptr;
  int* d_err = nullptr;                // latched error bits
  double* d_partials = nullptr;        // per-block reduction partials
  size_t partials_cap = 0;             // in doubles
  double* d_totals = nullptr;          // grid-reduced totals (128 doubles)
  unsigned* d_ticket = nullptr;        // last-block ticket (self-resetting)
  unsigned* d_tickets = nullptr;       // per-group tickets of the BN column reductions
  unsigned* d_set_tickets = nullptr;   // per-(group, set) tickets of their two-level reduction
  void* d_scratch = nullptr;           // misc scratch (temp states, small buffers)
  size_t scratch_cap = 0;
  void* d_wgrad = nullptr;             // per-split int32 wgrad partial tiles
  size_t wgrad_cap = 0;
  void* d_fold = nullptr;              // tap-folded activations / weights (narrow-channel convs)
  size_t fold_cap = 0;
  void* d_hist = nullptr;              // DSGC grid-search boundary histogram (dsgc.cu)
  // data parallel: the gradient of this rank is shard `rank` of `world` equal
  // shards of the global batch; statistics are combined through `allreduce`.
  i8t_allreduce_fn allreduce = nullptr;
  void* allreduce_user = nullptr;
  int rank = 0, world = 1;
  // or an NCCL communicator owned by the context (comm.cu): the statistics are
  // all-gathered on `stream` and folded in rank order
  void* nccl_comm = nullptr;
  double* d_gather = nullptr;  // [world][gather_cap]
  int64_t gather_cap = 0;
};

int ctx_allreduce_nccl(Ctx* c, double* buf, int64_t count, int op);
// data parallelism active: statistics must be combined across ranks
inline bool ctx_dp(const Ctx* c) { return c->allreduce != nullptr || c->nccl_comm != nullptr; }
int ctx_comm_destroy(Ctx* c);

// Runs the allreduce hook (if any) on `count` device doubles: op 0 = SUM, 1 = MAX.
int ctx_allreduce(Ctx* c, double* buf, int64_t count, int op);

// partial buffer layout helpers
constexpr int RED_THREADS = 256;

double* ensure_partials(Ctx* c, size_t doubles);
void* ensure_scratch(Ctx* c, size_t bytes);
void* ensure_wgrad(Ctx* c, size_t bytes);
void* ensure_fold(Ctx* c, size_t bytes);

void count_launch(int n = 1);
// 64 self-resetting tickets: [0, 32) BN column-sum groups, [32, 64) K4 candidate groups
unsigned* group_tickets(Ctx* c);

// Programmatic dependent launch: every kernel of this library starts with
// pdl_entry() (wait until the preceding grid of the stream has completed and
// its writes are visible), and launch_k() sets the programmatic-serialization
// attribute, so a grid is launched and its blocks scheduled while its
// predecessor drains instead of after it.  Most kernels do not trigger early
// (griddepcontrol.launch_dependents): the dependents of a persistent
// multi-block-per-SM grid would land on the SMs that free up first and lose
// their one-wave balance (measured slower).  I8T_PDL=0 turns the attribute off.
bool pdl_enabled();

__device__ __forceinline__ void pdl_entry() {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 900)
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
// Early trigger, only in kernels whose successor is a conv grid (one CTA per
// SM by its shared memory, so it cannot pile onto the SMs that free up first):
// the gradient quantiser before its grid reduction, the BN-apply passes after
// their main loops.  The conv kernels wait after their prologue.
__device__ __forceinline__ void pdl_trigger() {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 900)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

// launch_k with a thread-block cluster of `cluster_x` CTAs along x.
template <typename... KArgs, typename... Args>
inline void launch_k_cluster(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                             unsigned cluster_x, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster_x;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

template <typename... KArgs, typename... Args>
inline void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                     Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// shifted-window stride-1 convolution (conv_sw.cu)
bool conv_sw_eligible(const i8t_conv_geom* g, int64_t Cred, int Ng, int OH, int OW, const void* in, const void* out,
                      int64_t ldw);
int conv_sw_run(Ctx* c, bool dgrad, const i8t_conv_geom* g, const int8_t* in, int64_t Cred, int IH, int IW,
                const int8_t* wts, int64_t ldw, int Ng, int OH, int OW, const float* clip_x, const float* clip_y,
                float* out, int32_t* acc);
int set_error(int status, const std::string& msg);
int cuda_check(const char* what);

}  // namespace i8t_dev
