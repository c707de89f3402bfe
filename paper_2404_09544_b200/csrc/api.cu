// C-ABI glue: errors, graph load, NCCL comm, blocks handles (host code).
#include <dlfcn.h>
#include <cub/device/device_scan.cuh>
#include <limits.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <mutex>

#include "common.cuh"
#include "nccl.h"

namespace gnnv {

static thread_local std::string g_last_error;
static std::atomic<unsigned long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
static thread_local bool t_pdl_off = false;
void set_pdl(bool on) { t_pdl_off = !on; }
static std::mutex g_opt_mu;
static std::vector<std::pair<std::string, int>> g_opt_override;  // gnnv_set_option
static std::vector<std::pair<std::string, bool>> g_opt_env;      // environment, read once
bool env_on(const char* name) {
  std::lock_guard<std::mutex> lk(g_opt_mu);
  for (auto& kv : g_opt_override)
    if (kv.first == name && kv.second >= 0) return kv.second != 0;
  for (auto& kv : g_opt_env)
    if (kv.first == name) return kv.second;
  const char* e = getenv(name);
  const bool on = e && e[0] && strcmp(e, "0") != 0;
  g_opt_env.emplace_back(name, on);
  return on;
}
static std::vector<std::pair<std::string, int>> g_opt_env_int;  // integer options from the environment, read once
int env_int(const char* name, int def) {
  std::lock_guard<std::mutex> lk(g_opt_mu);
  for (auto& kv : g_opt_override)
    if (kv.first == name && kv.second >= 0) return kv.second;
  for (auto& kv : g_opt_env_int)
    if (kv.first == name) return kv.second == INT_MIN ? def : kv.second;
  const char* e = getenv(name);
  const int v = e && e[0] ? atoi(e) : INT_MIN;
  g_opt_env_int.emplace_back(name, v);
  return v == INT_MIN ? def : v;
}
static thread_local int t_grid_cap = 0;
void set_grid_cap(int cap) { t_grid_cap = cap; }
int capped_grid(int64_t grid) {
  const int64_t g = std::max<int64_t>(grid, 1);
  return (int)(t_grid_cap > 0 ? std::min<int64_t>(g, t_grid_cap) : g);
}
bool pdl_enabled() {
  static const bool on = !env_on("GNNV_NO_PDL");
  return on && !t_pdl_off;
}
void set_error(const std::string& msg) { g_last_error = msg; }
// W = 1 + 4 bias for bias in {0, 1/4, 1/2, 3/4, 1} (reading Q26), else 0
int32_t locality_weight(double bias) {
  for (int q = 0; q <= 4; ++q)
    if (bias == 0.25 * q) return 1 + q;
  return 0;
}
const char* get_error() { return g_last_error.c_str(); }

// Guarded allocations (GNNV_GUARD_ALLOC=1; the pool's compute-sanitizer is
// closed): every library allocation gets a 64 KB guard region on each side,
// filled with 0xA5; gnnv_debug_check_guards() reports any allocation whose
// guard bytes changed, i.e. an out-of-bounds write by any kernel.
constexpr size_t kGuard = 1 << 16;
struct GuardRec {
  char* base;
  size_t bytes;
  std::string what;
};
static std::mutex g_guard_mu;
static std::vector<std::pair<void*, GuardRec>> g_guard;
static bool guard_on() {
  static const bool on = env_on("GNNV_GUARD_ALLOC");
  return on;
}

void* dmalloc(size_t bytes, const char* what) {
  if (bytes == 0) bytes = 16;
  void* p = nullptr;
  const bool guard = guard_on();
  cudaError_t e = cudaMalloc(&p, guard ? bytes + 2 * kGuard : bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    char buf[256];
    snprintf(buf, sizeof(buf), "device allocation of %zu bytes for %s failed: %s", bytes, what,
             cudaGetErrorString(e));
    throw Error{e == cudaErrorMemoryAllocation ? GNNV_ERR_OOM : GNNV_ERR_CUDA, buf};
  }
  if (!guard) return p;
  char* base = static_cast<char*>(p);
  GNNV_TRY_CUDA(cudaMemset(base, 0xA5, kGuard));
  GNNV_TRY_CUDA(cudaMemset(base + kGuard + bytes, 0xA5, kGuard));
  GNNV_TRY_CUDA(cudaDeviceSynchronize());
  std::lock_guard<std::mutex> lk(g_guard_mu);
  g_guard.emplace_back(base + kGuard, GuardRec{base, bytes, what});
  return base + kGuard;
}

static int g_guard_freed_bad = 0;  // violations found when an allocation was freed
static std::string g_guard_freed_msg;

// index of the first modified guard byte of side 0 (before) / 1 (after), or kGuard
static size_t guard_first_bad(const GuardRec& r, int side) {
  std::vector<unsigned char> h(kGuard);
  const char* g = side ? r.base + kGuard + r.bytes : r.base;
  if (cudaMemcpy(h.data(), g, kGuard, cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
  for (size_t i = 0; i < kGuard; ++i)
    if (h[i] != 0xA5) return i;
  return kGuard;
}

size_t ipc_offset() { return guard_on() ? kGuard : 0; }

void dfree(void* p) {
  if (!p) return;
  if (guard_on()) {
    std::lock_guard<std::mutex> lk(g_guard_mu);
    for (size_t i = 0; i < g_guard.size(); ++i)
      if (g_guard[i].first == p) {
        const GuardRec& r = g_guard[i].second;
        cudaDeviceSynchronize();
        for (int side = 0; side < 2; ++side)
          if (guard_first_bad(r, side) < kGuard) {
            ++g_guard_freed_bad;
            g_guard_freed_msg += (g_guard_freed_msg.empty() ? "" : "; ") + r.what + " (freed): guard " +
                                 (side ? "after the end" : "before the start") + " modified";
          }
        cudaFree(r.base);
        g_guard.erase(g_guard.begin() + (long)i);
        return;
      }
  }
  cudaFree(p);
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

__global__ void k_fill_i32(int32_t* p, int64_t n, int32_t v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// ------------------------------------------------------------------ NCCL
struct NcclApi {
  void* lib = nullptr;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclAllGather) allGather = nullptr;
  decltype(&ncclGetErrorString) errStr = nullptr;
};

static NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* env = getenv("GNNV_NCCL_LIB");
    const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      if (!n) continue;
      api.lib = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (api.lib) break;
    }
    if (!api.lib) return;
    api.getUniqueId = (decltype(api.getUniqueId))dlsym(api.lib, "ncclGetUniqueId");
    api.commInitRank = (decltype(api.commInitRank))dlsym(api.lib, "ncclCommInitRank");
    api.commDestroy = (decltype(api.commDestroy))dlsym(api.lib, "ncclCommDestroy");
    api.allReduce = (decltype(api.allReduce))dlsym(api.lib, "ncclAllReduce");
    api.allGather = (decltype(api.allGather))dlsym(api.lib, "ncclAllGather");
    api.errStr = (decltype(api.errStr))dlsym(api.lib, "ncclGetErrorString");
  });
  if (!api.lib || !api.getUniqueId || !api.commInitRank || !api.allReduce || !api.allGather)
    throw Error{GNNV_ERR_COMM, "NCCL library not found (set GNNV_NCCL_LIB or preload libnccl.so.2)"};
  return api;
}

static void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    NcclApi& a = nccl();
    throw Error{GNNV_ERR_COMM, std::string(what) + ": " + (a.errStr ? a.errStr(r) : "nccl error")};
  }
}

}  // namespace gnnv

using namespace gnnv;

void* gnnv_blocks::ensure_scratch(size_t bytes, cudaStream_t s) {
  if (bytes <= scratch_bytes) return scratch;
  if (scratch) {
    GNNV_TRY_CUDA(cudaStreamSynchronize(s));
    dfree(scratch);
    scratch = nullptr;
    scratch_bytes = 0;
  }
  size_t want = std::max(bytes, (size_t)1 << 20);
  scratch = dmalloc(want, "layer scratch");
  scratch_bytes = want;
  return scratch;
}

extern "C" {

const char* gnnv_last_error(void) { return get_error(); }

gnnv_status gnnv_debug_check_guards(int32_t* n_bad) {
  return guarded([&] {
    GNNV_REQUIRE(n_bad, GNNV_ERR_PARAM, "debug_check_guards: null");
    *n_bad = 0;
    if (!guard_on()) return;
    GNNV_TRY_CUDA(cudaDeviceSynchronize());
    std::lock_guard<std::mutex> lk(g_guard_mu);
    std::string bad = g_guard_freed_msg;
    *n_bad = g_guard_freed_bad;
    g_guard_freed_bad = 0;
    g_guard_freed_msg.clear();
    for (auto& kv : g_guard) {
      const GuardRec& r = kv.second;
      for (int side = 0; side < 2; ++side) {
        const size_t first = guard_first_bad(r, side);
        if (first < kGuard) {
          ++*n_bad;
          char buf[256];
          snprintf(buf, sizeof(buf), "%s%s (%zu bytes): guard %s modified at byte %zu", bad.empty() ? "" : "; ",
                   r.what.c_str(), r.bytes, side ? "after the end" : "before the start", first);
          bad += buf;
        }
      }
    }
    if (*n_bad) set_error(bad);
  });
}

gnnv_status gnnv_set_option(const char* name, int32_t value) {
  return guarded([&] {
    static const char* known[] = {"GNNV_XROWS",      "GNNV_GEMM_PAIR",    "GNNV_BWD_PULL",   "GNNV_NO_TAIL",
                                  "GNNV_NO_PDL",     "GNNV_L2PUSH",       "GNNV_LASTUSE",    "GNNV_STATIC_TILES",
                                  "GNNV_PF_AGG",     "GNNV_NO_BF16ACT",   "GNNV_NO_BF16TABLE", "GNNV_NO_DW16",
                                  "GNNV_PF_CAP",     "GNNV_NO_FWD16",     "GNNV_NO_HID16",   "GNNV_DW16_MINKB",
                                  "GNNV_HID16_DW",   "GNNV_PF_PRIO",      "GNNV_BWD_NARROW", "GNNV_NO_TAIL16",
                                  "GNNV_NO_DA16",    "GNNV_NO_LASTROWS", "GNNV_KEEP_H1",     "GNNV_NO_BRES",   "GNNV_NO_EPPIPE"};
    GNNV_REQUIRE(name, GNNV_ERR_PARAM, "set_option: null name");
    bool ok = false;
    for (const char* k : known) ok |= strcmp(k, name) == 0;
    GNNV_REQUIRE(ok, GNNV_ERR_PARAM, std::string("set_option: unknown option ") + name);
    std::lock_guard<std::mutex> lk(g_opt_mu);
    for (auto& kv : g_opt_override)
      if (kv.first == name) {
        kv.second = value;
        return;
      }
    g_opt_override.emplace_back(name, value);
  });
}
const char* gnnv_version(void) { return GNNV_VERSION " sm_100a"; }
uint64_t gnnv_launch_count(void) { return g_launches.load(); }

}  // extern "C"
namespace gnnv {
__global__ void k_host_read(const uint4* __restrict__ h, int64_t n16, unsigned int* sink) {
  uint32_t acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 v = h[i];
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x9e3779b9u) atomicAdd(sink, 1u);  // keeps the loads
}
}  // namespace gnnv
extern "C" {

gnnv_status gnnv_host_read_probe(const void* h_buf, int64_t bytes, int32_t reps, float* ms, gnnv_stream stream) {
  return guarded([&] {
    GNNV_REQUIRE(h_buf && ms && bytes > 0 && bytes % 16 == 0 && reps >= 1, GNNV_ERR_PARAM, "host_read_probe: args");
    void* d = nullptr;
    GNNV_TRY_CUDA(cudaHostGetDevicePointer(&d, const_cast<void*>(h_buf), 0));
    unsigned int* sink = (unsigned int*)dmalloc(sizeof(unsigned int), "probe sink");
    cudaStream_t s = (cudaStream_t)stream;
    cudaEvent_t e0, e1;
    GNNV_TRY_CUDA(cudaEventCreate(&e0));
    GNNV_TRY_CUDA(cudaEventCreate(&e1));
    const int grid = num_sms() * 8;
    k_host_read<<<grid, 256, 0, s>>>(static_cast<const uint4*>(d), bytes / 16, sink);  // warm-up
    GNNV_TRY_CUDA(cudaEventRecord(e0, s));
    for (int r = 0; r < reps; ++r) k_host_read<<<grid, 256, 0, s>>>(static_cast<const uint4*>(d), bytes / 16, sink);
    GNNV_TRY_CUDA(cudaEventRecord(e1, s));
    GNNV_TRY_CUDA(cudaEventSynchronize(e1));
    GNNV_CHECK_LAUNCH();
    GNNV_TRY_CUDA(cudaEventElapsedTime(ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    dfree(sink);
  });
}
int32_t gnnv_row_stride(int32_t d) { return row_stride(d); }

// ------------------------------------------------------------------ graph
gnnv_status gnnv_graph_load(const int64_t* indptr, const int32_t* indices, int64_t n_nodes, int64_t nnz,
                            const float* host_feats, int32_t feat_dim, int32_t stride, const int32_t* labels,
                            int32_t n_classes, int32_t device, gnnv_graph** out) {
  return guarded([&] {
    GNNV_REQUIRE(out && indptr && (indices || nnz == 0) && host_feats && labels, GNNV_ERR_PARAM,
                 "graph_load: null pointer");
    GNNV_REQUIRE(n_nodes >= 1 && n_nodes < INT32_MAX && nnz >= 0, GNNV_ERR_PARAM,
                 "graph_load: n_nodes must be in [1, 2^31-1), nnz >= 0");
    GNNV_REQUIRE(feat_dim >= 1 && stride >= feat_dim && stride % 4 == 0, GNNV_ERR_PARAM,
                 "graph_load: row_stride must be >= feat_dim and a multiple of 4");
    GNNV_REQUIRE(n_classes >= 1, GNNV_ERR_PARAM, "graph_load: n_classes < 1");
    GNNV_REQUIRE(indptr[0] == 0 && indptr[n_nodes] == nnz, GNNV_ERR_PARAM,
                 "graph_load: indptr[0] must be 0 and indptr[n] == nnz");
    GNNV_REQUIRE(((uintptr_t)host_feats & 15) == 0, GNNV_ERR_PARAM, "graph_load: host_feats must be 16-byte aligned");
    GNNV_TRY_CUDA(cudaSetDevice(device));
    gnnv_graph* g = new gnnv_graph();
    g->device = device;
    g->n = n_nodes;
    g->nnz = nnz;
    g->d = feat_dim;
    g->stride = stride;
    g->n_classes = n_classes;
    try {
      g->d_indptr = (int64_t*)dmalloc((n_nodes + 1) * sizeof(int64_t), "indptr");
      g->d_indices = (int32_t*)dmalloc(std::max<int64_t>(nnz, 1) * sizeof(int32_t), "indices");
      g->d_labels = (int32_t*)dmalloc(n_nodes * sizeof(int32_t), "labels");
      GNNV_TRY_CUDA(cudaMemcpy(g->d_indptr, indptr, (n_nodes + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
      if (nnz) GNNV_TRY_CUDA(cudaMemcpy(g->d_indices, indices, nnz * sizeof(int32_t), cudaMemcpyHostToDevice));
      GNNV_TRY_CUDA(cudaMemcpy(g->d_labels, labels, n_nodes * sizeof(int32_t), cudaMemcpyHostToDevice));
      size_t fbytes = (size_t)n_nodes * stride * sizeof(float);
      cudaError_t e = cudaHostRegister((void*)host_feats, fbytes,
                                       cudaHostRegisterMapped | cudaHostRegisterPortable | cudaHostRegisterReadOnly);
      if (e == cudaErrorHostMemoryAlreadyRegistered) {
        cudaGetLastError();
      } else if (e != cudaSuccess) {
        cudaGetLastError();
        // read-only registration is not available everywhere; retry without it
        e = cudaHostRegister((void*)host_feats, fbytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
        if (e != cudaSuccess && e != cudaErrorHostMemoryAlreadyRegistered) GNNV_TRY_CUDA(e);
        cudaGetLastError();
        g->registered = (e == cudaSuccess);
      } else {
        g->registered = true;
      }
      void* dptr = nullptr;
      GNNV_TRY_CUDA(cudaHostGetDevicePointer(&dptr, (void*)host_feats, 0));
      g->h_feats = host_feats;
      g->d_feats = (const float*)dptr;
    } catch (...) {
      gnnv_graph_free(g);
      throw;
    }
    *out = g;
  });
}

gnnv_status gnnv_graph_free(gnnv_graph* g) {
  if (!g) return GNNV_OK;
  cudaSetDevice(g->device);
  dfree(g->d_indptr);
  dfree(g->d_indices);
  dfree(g->d_labels);
  if (g->registered && g->h_feats) cudaHostUnregister((void*)g->h_feats);
  delete g;
  return GNNV_OK;
}

gnnv_status gnnv_graph_info(const gnnv_graph* g, gnnv_graph_view* o) {
  return guarded([&] {
    GNNV_REQUIRE(g && o, GNNV_ERR_PARAM, "graph_info: null");
    o->n_nodes = g->n;
    o->nnz = g->nnz;
    o->feat_dim = g->d;
    o->row_stride = g->stride;
    o->n_classes = g->n_classes;
    o->device = g->device;
    o->d_indptr = g->d_indptr;
    o->d_indices = g->d_indices;
    o->d_labels = g->d_labels;
    o->d_host_feats = g->d_feats;
  });
}

// ------------------------------------------------------------------- comm
gnnv_status gnnv_comm_unique_id(void* out128) {
  return guarded([&] {
    GNNV_REQUIRE(out128, GNNV_ERR_PARAM, "comm_unique_id: null");
    ncclUniqueId id;
    nccl_check(nccl().getUniqueId(&id), "ncclGetUniqueId");
    memcpy(out128, &id, sizeof(id));
  });
}

gnnv_status gnnv_comm_init(int32_t rank, int32_t world, const void* uid, int32_t device, gnnv_comm** out) {
  return guarded([&] {
    GNNV_REQUIRE(out && world >= 1 && rank >= 0 && rank < world, GNNV_ERR_PARAM, "comm_init: bad rank/world");
    GNNV_TRY_CUDA(cudaSetDevice(device));
    ncclComm_t comm = nullptr;
    if (uid) {  // NULL: a host-only comm (rank/world; the caller exchanges data)
      ncclUniqueId id;
      memcpy(&id, uid, sizeof(id));
      nccl_check(nccl().commInitRank(&comm, world, id, rank), "ncclCommInitRank");
    }
    gnnv_comm* c = new gnnv_comm();
    c->rank = rank;
    c->world = world;
    c->device = device;
    c->nccl = comm;
    *out = c;
  });
}

gnnv_status gnnv_comm_free(gnnv_comm* c) {
  if (!c) return GNNV_OK;
  if (c->nccl) {
    try {
      nccl().commDestroy((ncclComm_t)c->nccl);
    } catch (...) {
    }
  }
  delete c;
  return GNNV_OK;
}

gnnv_status gnnv_allreduce_sum(gnnv_comm* c, float* d_buf, int64_t n, gnnv_stream s) {
  return guarded([&] {
    GNNV_REQUIRE(c && d_buf && n >= 0, GNNV_ERR_PARAM, "allreduce: bad args");
    if (c->world == 1 || n == 0) return;
    GNNV_REQUIRE(c->nccl, GNNV_ERR_STATE, "allreduce: host-only comm (created without an NCCL id)");
    nccl_check(nccl().allReduce(d_buf, d_buf, (size_t)n, ncclFloat32, ncclSum, (ncclComm_t)c->nccl,
                                (cudaStream_t)s),
               "ncclAllReduce");
  });
}

}  // extern "C"

namespace gnnv {
// all-gather `bytes` per rank through NCCL (synchronous; setup path only)
void comm_allgather_bytes(gnnv_comm* c, const void* mine, void* all, size_t bytes) {
  GNNV_REQUIRE(c && c->nccl, GNNV_ERR_STATE, "allgather: host-only comm");
  char* d = (char*)dmalloc(bytes * (c->world + 1), "allgather buffer");
  cudaStream_t s = nullptr;
  try {
    GNNV_TRY_CUDA(cudaMemcpy(d, mine, bytes, cudaMemcpyHostToDevice));
    nccl_check(nccl().allGather(d, d + bytes, bytes, ncclChar, (ncclComm_t)c->nccl, s), "ncclAllGather");
    GNNV_TRY_CUDA(cudaStreamSynchronize(s));
    GNNV_TRY_CUDA(cudaMemcpy(all, d + bytes, bytes * c->world, cudaMemcpyDeviceToHost));
  } catch (...) {
    dfree(d);
    throw;
  }
  dfree(d);
}
}  // namespace gnnv

namespace gnnv {
void blocks_enable_csc(gnnv_blocks* b, int h) {
  GNNV_REQUIRE(h >= 0 && h < b->L, GNNV_ERR_PARAM, "blocks_enable_csc: hop");
  if ((b->csc_mask >> h) & 1u) return;
  b->d_colptr[h] = (int32_t*)dmalloc((b->max_n[h + 1] + 1) * sizeof(int32_t), "block CSC colptr");
  b->d_csc[h] = (int32_t*)dmalloc(std::max<int64_t>(b->max_nnz[h], 1) * sizeof(int32_t), "block CSC rows");
  int64_t n_max = 1;
  for (int k = 0; k < b->L; ++k)
    if (((b->csc_mask >> k) & 1u) || k == h) n_max = std::max(n_max, b->max_n[k + 1] + 1);
  const size_t tmp = csc_scan_tmp_bytes(n_max);
  if (n_max > b->csc_cnt_cap) {
    GNNV_TRY_CUDA(cudaDeviceSynchronize());
    dfree(b->d_csc_cnt);
    b->d_csc_cnt = (int32_t*)dmalloc(n_max * sizeof(int32_t), "CSC counts");
    GNNV_TRY_CUDA(cudaMemset(b->d_csc_cnt, 0, n_max * sizeof(int32_t)));
    b->csc_cnt_cap = n_max;
  }
  if (tmp > b->csc_tmp_bytes) {
    dfree(b->d_csc_tmp);
    b->d_csc_tmp = dmalloc(tmp, "CSC scan temporary");
    b->csc_tmp_bytes = tmp;
  }
  b->csc_mask |= 1u << h;
  GNNV_TRY_CUDA(cudaDeviceSynchronize());
}
void blocks_enable_owner_rows(gnnv_blocks* b, int h) {
  GNNV_REQUIRE(h >= 0 && h < b->L, GNNV_ERR_PARAM, "blocks_enable_owner_rows: hop");
  GNNV_REQUIRE(!((b->csc_mask >> h) & 1u) || ((b->csc_nonowner >> h) & 1u), GNNV_ERR_STATE,
               "blocks_enable_owner_rows: hop already has a full CSC");
  if (!b->d_owner_row[h])
    b->d_owner_row[h] = (int32_t*)dmalloc(b->max_n[h + 1] * sizeof(int32_t), "owner rows");
  b->csc_nonowner |= 1u << h;
  blocks_enable_csc(b, h);
}

void blocks_set_rowidx(gnnv_blocks* b, const int32_t* d_slot, int32_t* d_rowidx, int64_t* d_stats) {
  b->rowidx_slot = d_slot;
  b->d_rowidx = d_rowidx;
  b->d_rowidx_stats = d_stats;
}
void blocks_set_last_rows(gnnv_blocks* b, const int32_t* d_slot) {
  b->last_rows = d_slot;
  // cub temporary of the last hop's offsets scan (shared with the CSC scans)
  size_t tmp = 0;
  GNNV_TRY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, b->d_cnt, b->d_indptr[b->L - 1], (int)b->max_n[b->L - 1]));
  if (tmp > b->csc_tmp_bytes) {
    dfree(b->d_csc_tmp);
    b->d_csc_tmp = dmalloc(tmp, "scan temporary");
    b->csc_tmp_bytes = tmp;
  }
}
void blocks_enable_lastuse(gnnv_blocks* b) {
  if (b->d_lastv) return;
  b->d_lastv = (uint32_t*)dmalloc(b->max_n[b->L] * sizeof(uint32_t), "last-use slots");
  GNNV_TRY_CUDA(cudaMemset(b->d_lastv, 0, b->max_n[b->L] * sizeof(uint32_t)));
}
}  // namespace gnnv

extern "C" {

// ----------------------------------------------------------------- blocks
gnnv_status gnnv_blocks_create(gnnv_graph* g, int32_t max_seeds, const int32_t* fanouts, int32_t L,
                               gnnv_blocks** out) {
  return guarded([&] {
    GNNV_REQUIRE(g && out && fanouts, GNNV_ERR_PARAM, "blocks_create: null");
    GNNV_REQUIRE(L >= 1 && L <= GNNV_MAX_LAYERS, GNNV_ERR_PARAM, "blocks_create: L must be in [1, 8]");
    GNNV_REQUIRE(max_seeds >= 1 && max_seeds <= g->n, GNNV_ERR_PARAM, "blocks_create: max_seeds must be in [1, N]");
    for (int h = 0; h < L; ++h)
      GNNV_REQUIRE(fanouts[h] >= 1 && fanouts[h] <= 32, GNNV_ERR_PARAM, "blocks_create: fanout must be in [1, 32]");
    GNNV_TRY_CUDA(cudaSetDevice(g->device));
    gnnv_blocks* b = new gnnv_blocks();
    b->g = g;
    b->L = L;
    b->max_n[0] = max_seeds;
    int64_t ell_max = 1, cnt_max = 1, tiles_max = 1;
    for (int h = 0; h < L; ++h) {
      b->fanouts[h] = fanouts[h];
      b->max_n[h + 1] = std::min<int64_t>(g->n, b->max_n[h] * (1 + (int64_t)fanouts[h]));
      b->max_nnz[h] = b->max_n[h] * fanouts[h];
      ell_max = std::max(ell_max, b->max_nnz[h]);
      cnt_max = std::max(cnt_max, b->max_n[h]);
      tiles_max = std::max(tiles_max, ceil_div(b->max_n[h], 256));
    }
    try {
      GNNV_REQUIRE(ell_max + 2 < INT32_MAX, GNNV_ERR_PARAM, "blocks_create: sampled slots exceed int32");
      b->d_tag = (int32_t*)dmalloc(g->n * sizeof(int32_t), "relabel tags");
      k_fill_i32<<<num_sms() * 4, 256>>>(b->d_tag, g->n, INT_MIN);
      GNNV_CHECK_LAUNCH();
      b->d_F = (int32_t*)dmalloc(b->max_n[L] * sizeof(int32_t), "frontiers");
      b->d_ell = (int32_t*)dmalloc(ell_max * sizeof(int32_t), "sample slots");
      b->d_cnt = (int32_t*)dmalloc(cnt_max * sizeof(int32_t), "sample counts");
      for (int h = 0; h < L; ++h) {
        b->d_indptr[h] = (int32_t*)dmalloc((b->max_n[h] + 1) * sizeof(int32_t), "block indptr");
        b->d_indices[h] = (int32_t*)dmalloc(std::max<int64_t>(b->max_nnz[h], 1) * sizeof(int32_t), "block indices");
        b->d_own[h] = (uint32_t*)dmalloc(b->max_n[h] * sizeof(uint32_t), "block owner masks");
      }
      // GNNV_BWD_PULL=1: CSC of the hops whose layer has a dX (h <= L-2),
      // for the pulled backward aggregation (measured slower than the
      // two-pass push on products; opt-in)
      b->pull_bwd = env_on("GNNV_BWD_PULL");
      if (b->pull_bwd)
        for (int h = 0; h + 1 < L; ++h) blocks_enable_csc(b, h);
      b->d_sizes = (int32_t*)dmalloc((2 * L + 2) * sizeof(int32_t), "sizes");
      GNNV_TRY_CUDA(cudaMemset(b->d_sizes, 0, (2 * L + 2) * sizeof(int32_t)));
      b->scan_words = tiles_max + 1;
      b->d_scan = (unsigned long long*)dmalloc(b->scan_words * sizeof(unsigned long long), "scan status");
      // zero once: every hop's k_map clears the words its scan used (sample.cu)
      GNNV_TRY_CUDA(cudaMemset(b->d_scan, 0, b->scan_words * sizeof(unsigned long long)));
      GNNV_TRY_CUDA(cudaDeviceSynchronize());
    } catch (...) {
      gnnv_blocks_free(b);
      throw;
    }
    *out = b;
  });
}

gnnv_status gnnv_blocks_set_locality(gnnv_blocks* b, const gnnv_cache* c, double bias) {
  return guarded([&] {
    GNNV_REQUIRE(b, GNNV_ERR_PARAM, "blocks_set_locality: null");
    const int32_t weight = locality_weight(bias);
    GNNV_REQUIRE(weight >= 1, GNNV_ERR_PARAM, "blocks_set_locality: bias must be one of 0, 0.25, 0.5, 0.75, 1");
    GNNV_REQUIRE(weight == 1 || c, GNNV_ERR_PARAM, "blocks_set_locality: a biased sampler needs the cache");
    GNNV_REQUIRE(!c || c->g == b->g, GNNV_ERR_STATE, "blocks_set_locality: cache of another graph");
    b->loc_w = weight;
    b->loc_slot = weight > 1 ? c->d_slot : nullptr;
  });
}

gnnv_status gnnv_blocks_free(gnnv_blocks* b) {
  if (!b) return GNNV_OK;
  dfree(b->d_tag);
  dfree(b->d_F);
  dfree(b->d_ell);
  dfree(b->d_cnt);
  for (int h = 0; h < GNNV_MAX_LAYERS; ++h) {
    dfree(b->d_indptr[h]);
    dfree(b->d_indices[h]);
    dfree(b->d_own[h]);
    dfree(b->d_colptr[h]);
    dfree(b->d_csc[h]);
  }
  dfree(b->d_csc_cnt);
  dfree(b->d_csc_tmp);
  dfree(b->d_lastv);
  for (int h = 0; h < GNNV_MAX_LAYERS; ++h) dfree(b->d_owner_row[h]);
  dfree(b->d_sizes);
  dfree(b->d_scan);
  dfree(b->scratch);
  delete b;
  return GNNV_OK;
}

gnnv_status gnnv_sample(gnnv_graph* g, const int32_t* d_seeds, int32_t n_seeds, const int32_t* fanouts, int32_t L,
                        uint64_t rng_seed, gnnv_blocks* b, gnnv_stream s) {
  return guarded([&] {
    GNNV_REQUIRE(g && b && d_seeds && fanouts, GNNV_ERR_PARAM, "sample: null");
    GNNV_REQUIRE(b->g == g, GNNV_ERR_STATE, "sample: blocks were created for another graph");
    GNNV_REQUIRE(L == b->L, GNNV_ERR_PARAM, "sample: L differs from blocks_create");
    for (int h = 0; h < L; ++h)
      GNNV_REQUIRE(fanouts[h] == b->fanouts[h], GNNV_ERR_PARAM, "sample: fanouts differ from blocks_create");
    GNNV_REQUIRE(n_seeds >= 1 && n_seeds <= b->max_n[0], GNNV_ERR_PARAM, "sample: n_seeds must be in [1, max_seeds]");
    launch_sample(g, b, d_seeds, n_seeds, rng_seed, (cudaStream_t)s);
    b->sampled = true;
  });
}

gnnv_status gnnv_blocks_info(gnnv_blocks* b, int32_t sync, gnnv_stream s, gnnv_block_view* v) {
  return guarded([&] {
    GNNV_REQUIRE(b && v, GNNV_ERR_PARAM, "blocks_info: null");
    std::vector<int32_t> sz(2 * b->L + 2, -1);
    if (sync) {
      GNNV_REQUIRE(b->sampled, GNNV_ERR_STATE, "blocks_info: gnnv_sample has not run on these blocks");
      GNNV_TRY_CUDA(cudaMemcpyAsync(sz.data(), b->d_sizes, sz.size() * sizeof(int32_t), cudaMemcpyDeviceToHost,
                                    (cudaStream_t)s));
      GNNV_TRY_CUDA(cudaStreamSynchronize((cudaStream_t)s));
    }
    for (int h = 0; h < b->L; ++h) {
      v[h].n_dst = sz[h];
      v[h].n_src = sz[h + 1];
      v[h].nnz = sz[b->L + 1 + h];
      v[h].max_dst = b->max_n[h];
      v[h].max_src = b->max_n[h + 1];
      v[h].max_nnz = b->max_nnz[h];
      v[h].d_indptr = b->d_indptr[h];
      v[h].d_indices = b->d_indices[h];
      v[h].d_src_global = b->d_F;
    }
    if (sync) {
      int32_t err = sz[2 * b->L + 1];
      if (err) {
        GNNV_TRY_CUDA(cudaMemsetAsync(b->d_sizes + 2 * b->L + 1, 0, sizeof(int32_t), (cudaStream_t)s));
        throw Error{GNNV_ERR_PARAM, (err & 1) ? "sample: a seed id is outside [0, N)" : "sample: repeated seed id"};
      }
    }
  });
}

const int32_t* gnnv_blocks_device_sizes(const gnnv_blocks* b) { return b ? b->d_sizes : nullptr; }
int32_t gnnv_blocks_num_layers(const gnnv_blocks* b) { return b ? b->L : 0; }

gnnv_status gnnv_sgd(float* d_params, const float* d_grads, int64_t n, float lr, gnnv_stream s) {
  return guarded([&] {
    GNNV_REQUIRE(d_params && d_grads && n >= 0, GNNV_ERR_PARAM, "sgd: bad args");
    launch_sgd(d_params, d_grads, n, lr, (cudaStream_t)s);
  });
}

}  // extern "C"
