// Internal definitions shared by the libgnnv translation units (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>
#include <utility>
#include <vector>

#include "../../include/gnnv.h"

namespace gnnv {

// ----------------------------------------------------------------- errors
void set_error(const std::string& msg);
const char* get_error();

struct Error {
  gnnv_status st;
  std::string msg;
};

#define GNNV_TRY_CUDA(expr)                                                                    \
  do {                                                                                         \
    cudaError_t _e = (expr);                                                                   \
    if (_e != cudaSuccess) {                                                                   \
      if (_e == cudaErrorMemoryAllocation) {                                                   \
        throw ::gnnv::Error{GNNV_ERR_OOM, std::string(#expr) + ": " + cudaGetErrorString(_e)}; \
      }                                                                                        \
      throw ::gnnv::Error{GNNV_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)};  \
    }                                                                                          \
  } while (0)

// Every kernel launch site ends with GNNV_CHECK_LAUNCH(), which also counts
// the launch (gnnv_launch_count(), used by bench.py's gpu_launches).
void count_launch();
#define GNNV_CHECK_LAUNCH()          \
  do {                               \
    ::gnnv::count_launch();          \
    GNNV_TRY_CUDA(cudaGetLastError()); \
  } while (0)

// Programmatic dependent launch (PDL): every kernel of the step starts with
// GNNV_PDL_ENTRY() -- it lets the next kernel in the stream be scheduled as
// soon as all of this kernel's CTAs are running, then waits for its own
// predecessor to complete (griddepcontrol.wait; a no-op without a
// programmatic dependency).  launch_k() launches with the PDL attribute, so
// launch latency and CTA rasterisation overlap the predecessor's tail.
// GNNV_NO_PDL=1 disables the attribute.
#define GNNV_PDL_ENTRY()                                          \
  do {                                                            \
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); \
    asm volatile("griddepcontrol.wait;" ::: "memory");            \
  } while (0)
bool pdl_enabled();
// off around the Eq.4 prefetch: its kernels would otherwise park waiting CTAs
// on the SMs the concurrent step needs
void set_pdl(bool on);
// integer option (gnnv_set_option override, else the environment, else def)
int env_int(const char* name, int def);
// CTA cap for the grid-stride launches of this thread (0 = none): the Eq.4
// prefetch caps its sampler / gather grids so the step's kernels keep room
// on every SM (trainer.cu)
void set_grid_cap(int cap);
int capped_grid(int64_t grid);
template <typename... KArgs, typename... Args>
inline void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  if (pdl_enabled()) {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  GNNV_TRY_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

#define GNNV_REQUIRE(cond, code, msg)                  \
  do {                                                 \
    if (!(cond)) throw ::gnnv::Error{(code), (msg)};   \
  } while (0)

// Runs `body`, converting thrown Errors to a status + thread-local message.
template <class F>
gnnv_status guarded(F&& body) {
  try {
    body();
    return GNNV_OK;
  } catch (const Error& e) {
    set_error(e.msg);
    return e.st;
  } catch (const std::exception& e) {
    set_error(e.what());
    return GNNV_ERR_CUDA;
  }
}

void* dmalloc(size_t bytes, const char* what);  // throws OOM with the byte count
// offset of a dmalloc pointer from its allocation's base (a CUDA IPC handle
// maps the base): 0, or the guard region's size with GNNV_GUARD_ALLOC
size_t ipc_offset();
void dfree(void* p);

inline int32_t row_stride(int32_t d) { return (d + 3) & ~3; }
inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

int num_sms();

// Opt-in switches, read once per process: set and not "0" = on.  Every one
// of them selects a variant measured slower than (or equal to) the default
// on the products workload and kept for A/B runs:
//   GNNV_XROWS     layer-1 GEMMs read H_dst with TMA gather4 (gemm_tma.cu)
//   GNNV_GEMM_PAIR forward GEMM on CTA pairs, cta_group::2 (gemm_tma.cu)
//   GNNV_BWD_PULL  backward aggregation pulled through a CSC (spmm.cu)
//   GNNV_NO_TAIL   per-kernel output layer instead of tail.cu
//   GNNV_NO_PDL    no programmatic dependent launch
bool env_on(const char* name);
// NEXT-2 locality weight 1 + 4 bias (1..5), 0 for an unsupported bias
int32_t locality_weight(double bias);

// ---------------------------------------------------------------- handles
}  // namespace gnnv

struct gnnv_graph {
  int device = 0;
  int64_t n = 0, nnz = 0;
  int32_t d = 0, stride = 0, n_classes = 0;
  int64_t* d_indptr = nullptr;
  int32_t* d_indices = nullptr;
  int32_t* d_labels = nullptr;
  const float* h_feats = nullptr;  // borrowed host table
  const float* d_feats = nullptr;  // device-mapped alias
  bool registered = false;         // we called cudaHostRegister
};

struct gnnv_comm {
  int rank = 0, world = 1, device = 0;
  void* nccl = nullptr;  // ncclComm_t
};

namespace gnnv {
void comm_allgather_bytes(gnnv_comm* c, const void* mine, void* all, size_t bytes);
}
struct gnnv_cache {
  gnnv_graph* g = nullptr;
  int64_t capacity = 0;
  int64_t local_rows = 0;
  int32_t world = 1, rank = 0, placement = GNNV_PLACE_REPLICA;
  int32_t* d_slot = nullptr;   // [N] degree rank if cached else -1
  int32_t* d_order = nullptr;  // [N] vertices by (deg desc, id asc)
  std::vector<float*> shards;  // per shard base pointer (local allocs or IPC-mapped peers)
  std::vector<bool> shard_owned;
  std::vector<bool> shard_ipc;
  const float** d_shard_ptrs = nullptr;  // device array [world]
  // bf16 copy of the whole local table (cache_bf16_table; the tf32 trainer's
  // layer-1 aggregation reads it -- reading Q31), row stride table16_ld
  // elements (d rounded up to 8, zero-padded); NULL until requested
  void* d_table16 = nullptr;
  int32_t table16_ld = 0;
  bool peers_ready = true;               // SHARDED: every peer's shard mapped
  // NEXT-3 dynamic cache (policy FIFO / LRU): starts empty, the misses of
  // every batch are admitted by gnnv_cache_update (cache.cu)
  int32_t policy = GNNV_POLICY_DEGREE;
  bool dynamic = false;
  int32_t step = 0;                        // batch index t (LRU stamps)
  int32_t* d_owner = nullptr;              // [C] vertex in slot, -1 free
  int32_t* d_stamp = nullptr;              // [C] last-access batch (LRU)
  int64_t* d_seq = nullptr;                // [C] admission sequence number
  unsigned long long* d_keys = nullptr;    // [2C] victim-order keys
  int32_t* d_vidx = nullptr;               // [2C] slots sorted by key
  void* d_sort_tmp = nullptr;
  size_t sort_tmp_bytes = 0;
  int32_t* d_miss = nullptr;               // [miss_cap] miss rows of the batch (ascending)
  int32_t* d_mflag = nullptr;              // [miss_cap]
  int64_t miss_cap = 0;
  void* d_sel_tmp = nullptr;
  size_t sel_tmp_bytes = 0;
  int64_t* d_ctr = nullptr;                // [6] hits, misses, replaced, admitted, seq_next, n_miss
};

struct gnnv_blocks {
  gnnv_graph* g = nullptr;
  int32_t L = 0;
  int32_t fanouts[GNNV_MAX_LAYERS] = {0};
  int64_t max_n[GNNV_MAX_LAYERS + 1] = {0};   // frontier capacities
  int64_t max_nnz[GNNV_MAX_LAYERS] = {0};
  int32_t* d_tag = nullptr;       // [N] relabel map: INT_MIN unvisited, <-1 claim, >=0 local id
  int32_t* d_F = nullptr;         // [max_n[L]] nested frontiers
  int32_t* d_ell = nullptr;       // [max over h of max_n[h]*k_h] sampled global ids
  int32_t* d_cnt = nullptr;       // [max_n[L-1]] per-row sampled count
  int32_t* d_indptr[GNNV_MAX_LAYERS] = {nullptr};
  int32_t* d_indices[GNNV_MAX_LAYERS] = {nullptr};
  int32_t* d_sizes = nullptr;     // [2L+1] + error flag
  unsigned long long* d_scan = nullptr;  // chained-scan status [1 + max tiles]
  int64_t scan_words = 0;
  uint32_t* d_own[GNNV_MAX_LAYERS] = {nullptr};  // [max_n[h]] owner-edge bit mask per dst row
  // transposed blocks (CSC) of selected hops: the in-edges of src row u of
  // hop h are d_csc[h][d_colptr[h][u] .. d_colptr[h][u+1]), their dst rows
  // (counting sort, order of arrival).  Used by the trainer's fused L2 push
  // (the layer-1 GEMM epilogue aggregates layer 2's input; hop L-2) and, with
  // GNNV_BWD_PULL, by the pulled backward aggregation (hops <= L-2).
  uint32_t csc_mask = 0;  // bit h: hop h gets a CSC (blocks_enable_csc)
  bool pull_bwd = false;   // GNNV_BWD_PULL: the CSC hops' backward aggregation pulls
  int32_t* d_colptr[GNNV_MAX_LAYERS] = {nullptr};  // [max_n[h+1] + 1]
  int32_t* d_csc[GNNV_MAX_LAYERS] = {nullptr};     // [max_nnz[h]]
  int32_t* d_csc_cnt = nullptr;    // [max n_src + 1] in-edge counts (zero between batches)
  int64_t csc_cnt_cap = 0;
  // last-use slots of hop L-1 (the layer-1 block): lastv[u] = 1 + the CSR
  // position of src id u's last edge (0: no edge); the layer-1 aggregation
  // loads a row for the last time with an L2 evict_first hint
  // (blocks_enable_lastuse; NULL: off)
  uint32_t* d_lastv = nullptr;
  // whole-table trainer (blocks_set_rowidx; NULL: off): k_reset also writes
  // rowidx[i] = slot[F[i]] for every F_L row and the all-hit gather counters
  int32_t* d_rowidx = nullptr;
  const int32_t* rowidx_slot = nullptr;
  int64_t* d_rowidx_stats = nullptr;
  // whole-table trainer (blocks_set_last_rows; NULL: off): the last hop is
  // not relabelled -- its sampled ids claim no tag, get no local id, and its
  // CSR indices are their cache-table rows last_rows[u] (F_L = F_{L-1});
  // the layer-1 aggregation reads the table rows directly
  const int32_t* last_rows = nullptr;
  // fused L2 push (blocks_enable_owner_rows): the hop's owner row of every
  // src id (the dst row whose edge discovered it; -1 for the dst prefix), and
  // its CSC holding the non-owner edges only (bit h of csc_nonowner)
  int32_t* d_owner_row[GNNV_MAX_LAYERS] = {nullptr};
  uint32_t csc_nonowner = 0;
  void* d_csc_tmp = nullptr;       // cub scan temporary storage
  size_t csc_tmp_bytes = 0;
  bool sampled = false;
  // NEXT-2 locality bias: cached neighbours (slot[u] >= 0) weigh loc_w
  // (= 1 + 4b, 1 = unbiased); see gnnv_blocks_set_locality
  const int32_t* loc_slot = nullptr;
  int32_t loc_w = 1;
  // scratch arena for the layer kernels (grows on demand)
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  void* ensure_scratch(size_t bytes, cudaStream_t s);
};

namespace gnnv {

// Named segments of a step, bracketed by CUDA events on the step's stream
// and read back after the timed region (no sync inside a step).  Segment j
// runs from mark j to mark j+1.
struct Timeline {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  std::vector<std::pair<std::string, cudaEvent_t>> marks;
  void mark(cudaStream_t s, const std::string& name) {
    if (!on) return;
    if (used == pool.size()) {
      cudaEvent_t e;
      GNNV_TRY_CUDA(cudaEventCreate(&e));
      pool.push_back(e);
    }
    cudaEvent_t e = pool[used++];
    GNNV_TRY_CUDA(cudaEventRecord(e, s));
    marks.emplace_back(name, e);
  }
  void clear() {
    used = 0;
    marks.clear();
  }
  ~Timeline() {
    for (auto e : pool) cudaEventDestroy(e);
  }
};

// kernels implemented in the .cu files -----------------------------------
// sample.cu
void launch_sample(gnnv_graph* g, gnnv_blocks* b, const int32_t* d_seeds, int32_t n_seeds, uint64_t rng_seed,
                   cudaStream_t s);
// cub scan temporary bytes for the CSC column pointers of max_items columns
size_t csc_scan_tmp_bytes(int64_t max_items);
// give hop h of b a transposed block (CSC), built by every later
// gnnv_sample on b (setup path: allocates; synchronises the device)
void blocks_enable_csc(gnnv_blocks* b, int h);
void blocks_enable_lastuse(gnnv_blocks* b);
void blocks_set_rowidx(gnnv_blocks* b, const int32_t* d_slot, int32_t* d_rowidx, int64_t* d_stats);
void blocks_set_last_rows(gnnv_blocks* b, const int32_t* d_slot);
void blocks_enable_owner_rows(gnnv_blocks* b, int h);  // + CSC of hop h's non-owner edges
// cache.cu
void launch_cache_update(gnnv_cache* c, const gnnv_blocks* b, const float* d_X, cudaStream_t s);
// builds c->d_table16 from the local table (setup path; synchronises)
void cache_bf16_table(gnnv_cache* c);
void launch_gather(const gnnv_cache* c, const gnnv_blocks* b, float* d_X, int64_t* d_stats, cudaStream_t s,
                   int32_t* d_rowidx = nullptr, bool materialize = true, void* d_X16 = nullptr, int32_t ldx16 = 0);
// spmm.cu
// rowidx != NULL: source row u is row rowidx[u] of H (the cache table)
void launch_spmm_fwd(const int32_t* d_indptr, const int32_t* d_indices, const int32_t* d_ndst, int64_t max_dst,
                     const float* H, int32_t ldh, float* A, int32_t lda, int32_t d, int32_t kind, int32_t aggr,
                     cudaStream_t s, const int32_t* rowidx = nullptr, const uint32_t* lastv = nullptr);
void launch_spmm_bwd(const int32_t* d_indptr, const int32_t* d_indices, const uint32_t* d_own, const int32_t* d_ndst,
                     int64_t max_dst, const float* dA, int32_t lda, void* dH, int32_t ldh, int32_t d, int32_t kind,
                     int32_t aggr, const uint32_t* bits, int32_t bits_ld, cudaStream_t s, bool dh_bf16 = false,
                     bool da_bf16 = false);
// the wide bf16 push (a warp per dst row, 8 columns per lane) applies
bool spmm_bwd_wide(int32_t ldh, int32_t lda, int32_t kind, bool dh_bf16);
// the forward aggregation over bf16 source rows (stride ld16 elements)
// rowidx != NULL: source row u is row rowidx[u] of H16 (the bf16 table)
void launch_spmm_fwd_h16(const int32_t* d_indptr, const int32_t* d_indices, const int32_t* d_ndst, int64_t max_dst,
                         const void* H16, int32_t ld16, float* A, int32_t lda, int32_t d, int32_t kind, int32_t aggr,
                         cudaStream_t s, const int32_t* rowidx = nullptr, void* A16 = nullptr, int32_t lda16 = 0,
                         void* X16 = nullptr, bool rows_direct = false);
// the same transposed aggregation pulled per src row (rows up to
// kPullMaxLd floats; wider ones keep the push) through the block's
// CSC (one coalesced store per dH row, no atomics; see k_spmm_bwd_pull)
constexpr int kPullMaxLd = 512;
void launch_spmm_bwd_pull(const int32_t* d_colptr, const int32_t* d_csc, const int32_t* d_indptr,
                          const int32_t* d_ndst, const int32_t* d_nsrc, int64_t max_src, const float* dA, int32_t lda,
                          float* dH, int32_t ldh, int32_t d, int32_t kind, int32_t aggr, const uint32_t* bits,
                          int32_t bits_ld, cudaStream_t s);
void launch_colsum_reduce(const float* partial, int blocks, int ld, int N, float* out, cudaStream_t s);
// gemm
struct GemmFwdArgs {
  const float* X1; int32_t ld1;  // H_dst (rows 0..M) or A' (GCN)
  const float* X2; int32_t ld2;  // A (SAGE) or nullptr
  int32_t K1;                    // width of each part (d_in)
  const float* W;                // [(X2?2:1)*K1 x N] row-major
  const float* bias;             // [N]
  float* Y; int32_t ldy;         // [M x N]
  int32_t N;
  const int32_t* d_M; int64_t max_M;
  bool relu;
  // TF32 with relu: also write the ReLU mask as bits, bits[m*mask_ld + n/32]
  // bit n%32 = (Y[m][n] > 0), for a later fused dW (NULL: none)
  uint32_t* mask_bits = nullptr;
  int32_t mask_ld = 0;
  // TF32 only: X1 row m is row x1_rows[m] of X1, a [x1_table_rows x ld1]
  // table (layer 1 reading H_dst from the whole-table cache; NULL: row m)
  const int32_t* x1_rows = nullptr;
  int64_t x1_table_rows = 0;
  // TF32 only: the next layer's aggregation fused into the epilogue (the
  // trainer's "L2 push"): for every output row u and every
  // in-edge (v, u) of the next layer's block -- push_colptr[u] ..
  // push_colptr[u+1] in push_dst -- push_out[v] += w_v * Y[u] with
  // red.global.add (w_v = 1 / (push_indptr[v+1] - push_indptr[v]) for the
  // mean, 1 for the sum); push_out must be zero.  Rows u >= *keep_rows are
  // then not stored to Y (only their ReLU bits are).  NULL: off.
  const int32_t* push_colptr = nullptr;
  const int32_t* push_dst = nullptr;
  const int32_t* push_indptr = nullptr;
  float* push_out = nullptr;
  int32_t push_ld = 0;
  bool push_mean = true;
  const int32_t* keep_rows = nullptr;
  // owner row of each output row (-1: none; NULL: the CSC holds every edge):
  // the owner edges are then reduced as runs of consecutive rows and the CSC
  // holds only the other edges
  const int32_t* push_owner = nullptr;
  // TF32: every output row also stored as bf16 (y16, row stride ld16, a
  // multiple of 32); the fp32 rows then only below *keep_rows.  NULL: off
  void* y16 = nullptr;
  int32_t ld16 = 0;
  // TF32 mode, SAGE: X1 and X2 as bf16 copies ([M x ld16in], columns past
  // K1 ignored) -- the GEMM then runs kind::f16 over bf16 operands (W
  // rounded to bf16 per call); X1/X2 unused.  NULL: off
  const void* X1_16 = nullptr;
  const void* X2_16 = nullptr;
  int32_t ld16in = 0;
};
void gemm_fwd(const GemmFwdArgs& a, int prec, cudaStream_t s);
// The trainer's fused L2 push (GemmFwdArgs::push_*): layer i's GEMM
// epilogue accumulates layer i+1's aggregate A^{i+1} over the CSC of hop
// L-i-1 into `out` (zeroed first, launch_zero_rows)
struct FwdPush {
  const int32_t *colptr, *dst, *indptr;
  float* out;
  int32_t ld;
  bool mean;
  const int32_t* keep_rows;
  const int32_t* owner;
};
void launch_zero_rows(float* p, const int32_t* d_rows, int64_t max_rows, int32_t ld, cudaStream_t s);
// The trainer's bf16 intermediates (GNNV_BF16ACT): a hidden
// layer's output H^i is also stored as bf16 for the next layer's
// aggregation (its fp32 rows only for the next layer's dst prefix), and
// dL/dH^i is produced and consumed as bf16.  Per layer call:
struct Bf16Io {
  void* y16 = nullptr;             // fwd: bf16 copy of this layer's output
  int32_t ld16 = 0;                //      its row stride (elements, % 32 == 0)
  const int32_t* keep_rows = nullptr;  // fwd: fp32 output rows kept
  const void* src16 = nullptr;     // fwd: aggregate from this bf16 copy of H_src
  int32_t src16_ld = 0;
  const int32_t* src16_rows = nullptr;  // fwd: source row u is row src16_rows[u] of src16 (the bf16 table)
  void* gsrc16 = nullptr;          // bwd: dH_src produced as bf16 (stride gsrc16_ld)
  int32_t gsrc16_ld = 0;
  const void* gdst16 = nullptr;    // bwd: this layer's G read as bf16 (stride gdst16_ld)
  int32_t gdst16_ld = 0;
  // fwd: the aggregation also writes A as bf16 (a16, stride a16_ld) and,
  // with x16 (X's dst prefix as bf16, ones column at d_in, stride a16_ld),
  // the GEMM reads [x16 | a16] (kind::f16); bwd with x16, a16 and gdst16:
  // dW and db by gemm_dw16
  void* a16 = nullptr;
  int32_t a16_ld = 0;
  const void* x16 = nullptr;
  bool keep_a32 = false;  // fwd with x16: still write the fp32 A (a TF32 dW reads it)
  void* x16_out = nullptr;  // fwd, bf16 aggregation: also copy each dst row's own bf16 row here (+ ones column)
  bool rows_direct = false;  // fwd, with src16_rows: the block's indices are already table rows (last_rows)
  // bwd with x16 and a16, G pre-masked fp32: write G's bf16 copy here (stride
  // g16_ld) and run dW over bf16 (gemm_dw16; db by the conversion pass)
  void* g16_out = nullptr;
  int32_t g16_ld = 0;
  // bwd with x16 and a16: G already as bf16 (stride g16_ld; the fused
  // output layer wrote it) with db's partial column sums dbp[ndbp][d_out]
  const void* g16_in = nullptr;
  const float* dbp = nullptr;
  int32_t ndbp = 0;
};
// Layer 1 of the trainer with the whole feature table on the device: H_dst
// (X's dst prefix) is read by the TF32 GEMMs straight from the table through
// the gather's row indices, so X is never materialised.
struct XRows {
  const float* table;
  const int32_t* rows;
  int64_t table_rows;
};
// words per row of a ReLU bit mask over N columns (16-byte rows for TMA)
inline int32_t mask_words(int32_t N) { return ((N + 31) / 32 + 3) / 4 * 4; }
void launch_relu_bits(const float* H, int32_t ldh, int32_t N, const int32_t* d_M, int64_t max_M, uint32_t* bits,
                      int32_t bits_ld, cudaStream_t s);
// dW = [X1|X2]^T G (+ bias row = colsum G): split-K over graph rows, reduced
// in a fixed order (FP32/BF16, bitwise reproducible) or added with
// red.global.add (TF32: arrival order, see gnnv_layer_bwd)
struct GemmDwArgs {
  const float* X1; int32_t ld1;
  const float* X2; int32_t ld2;
  int32_t K1;
  const float* G; int32_t ldg;
  int32_t N;
  const int32_t* d_M; int64_t max_M;
  float* dW;  // [(X2?2:1)*K1 x N]
  float* db;  // [N]
  float* partial; int32_t splits;  // workspace [splits x (rows+1) x N]
  // TF32 only: fuse G' = G * mask and db, mask = the ReLU bits of the
  // layer's output (see GemmFwdArgs::mask_bits); NULL: G is final, db elsewhere
  const uint32_t* mask_bits = nullptr;
  int32_t mask_ld = 0;
  bool db_fused = false;  // TF32 only: db = colsum(G) computed by the dW kernel (G final)
  const int32_t* x1_rows = nullptr;  // as GemmFwdArgs::x1_rows
  int64_t x1_table_rows = 0;
  bool zeroed = false;  // TF32: dW (and db) already zero (the trainer clears them in-kernel)
  const void* G16 = nullptr;  // TF32: G as bf16 (row stride ldg elements) instead of G
};
void gemm_dw(const GemmDwArgs& a, int prec, cudaStream_t s);
size_t gemm_dw_partial_floats(int32_t rows_plus_bias, int32_t N, int32_t* splits_out, int64_t max_M);
// dW = [S_0 | S_1]^T G16 over bf16 operands, MN-major on kind::f16
// (gemm_tma.cu k_tma_dw16): source s ([rows x ld] bf16, `width` features)
// fills dW rows out_row0 .. out_row0 + width; with `ones` its column
// `width` holds 1.0 and the same MMAs give db = colsum(G16).  Widths up to
// 256 (at most four 128-feature tiles), N a multiple of 64 up to 256.
struct GemmDw16Src {
  const void* p = nullptr;
  int32_t ld = 0, width = 0, out_row0 = 0;
  bool ones = false;
};
struct GemmDw16Args {
  GemmDw16Src src[2];
  const void* G16;  // [rows x ldg] bf16
  int32_t ldg, N;
  const int32_t* d_M;
  int64_t max_M;
  float* dW;  // rows: src widths summed
  float* db;  // with a ones source or G32; else untouched (may be NULL)
  bool zeroed = false;
  // G32 set: G16 is first written from this pre-masked fp32 G ([rows x
  // ldg32]) by the same call, which also sums db = colsum(G32)
  const float* G32 = nullptr;
  int32_t ldg32 = 0;
  // dbp set (no ones source, no G32): db = the sum of these partial column
  // sums [ndbp][N] in order
  const float* dbp = nullptr;
  int32_t ndbp = 0;
};
void gemm_dw16(const GemmDw16Args& a, cudaStream_t s);
struct GemmDxArgs {  // [Y1 | Y2] = G W^T  (Y1 = first K1 cols, Y2 = the rest)
  const float* G; int32_t ldg;
  int32_t N;
  const float* W;  // [(Y2?2:1)*K1 x N] row-major
  int32_t K1;
  float* Y1; int32_t ld1;
  float* Y2; int32_t ld2;
  const int32_t* d_M; int64_t max_M;
  // TF32 only: Y1 *= ReLU bits of the previous layer (NULL: none)
  const uint32_t* y1_bits = nullptr;
  int32_t y1_bits_ld = 0;
  void* Y1_16 = nullptr;  // TF32: Y1 stored as bf16 (row stride ld1, ld1 % 32 == 0) instead of Y1
  void* Y2_16 = nullptr;  // TF32 with Y1_16: Y2 stored as bf16 too (row stride ld2, ld2 % 32 == 0) instead of Y2
  // TF32 mode: G as a bf16 copy ([M x ldg16]) -- the GEMM then runs kind::f16
  // with W rounded to bf16 (reading Q34); G unused.  NULL: off
  const void* G16 = nullptr;
  int32_t ldg16 = 0;
};
void gemm_dx(const GemmDxArgs& a, int prec, cudaStream_t s);
// tail.cu: the trainer's output layer (forward, loss, backward) fused
struct TailArgs {
  const int32_t *indptr, *indices;  // hop-0 block (dst = seeds)
  const uint32_t* own;              // owner-edge masks of the hop-0 rows
  const int32_t* d_ndst;            // n_0 on the device
  int64_t max_dst;
  const float* H; int32_t ldh;      // H^{L-1} [n_1 x ldh]
  const uint32_t* hbits; int32_t hbits_ld;  // its ReLU bits
  const float *W, *bias;            // [W_s; W_n] (2d x C), b (C)
  int32_t d, C, aggr;
  float* A; int32_t lda;            // aggregates out [n_0 x lda]
  float *Z, *dZ; int32_t ldz;       // logits and dlogits [n_0 x ldz]
  const int32_t *F, *labels;
  int32_t n_global;
  float* dH; int32_t ldg;           // dL/dH^{L-1} [n_1 x ldg] (ReLU derivative applied)
  // dH16 set: dL/dH^{L-1} written as bf16 instead ([n_1 x ldg], dH unused),
  // and db_part[b][d] (b < tail_db_parts(max_dst)) gets each CTA's column
  // sums of what it wrote: db^{L-1} = their sum (the layer's bf16 dW)
  void* dH16 = nullptr;
  float* db_part = nullptr;
  float* dA;                        // scratch [n_0 x d]
  float* loss_partial;              // >= ceil(max_dst / 32) floats
  float* part;                      // tail_partial_floats(max_dst, d, C): per-CTA dW/db partials
  float *dW, *db, *d_loss;
  float* zero; int64_t zero_n;      // cleared by k_tail_a (the other layers' dW/db), may be NULL
};
bool tail_supported(int kind, int d, int C, int fanout0);
int tail_db_parts(int64_t max_dst);
size_t tail_partial_floats(int64_t max_dst, int d, int C);
void launch_tail(const TailArgs& a, cudaStream_t s, Timeline* tl, const std::string& sfx);
// layers.cu
void launch_relu_mask(const float* G, const float* H, float* Gp, int32_t ld, int32_t N, const int32_t* d_M,
                      int64_t max_M, cudaStream_t s);
void launch_ce_loss(const float* z, int32_t ldz, int32_t C, const int32_t* d_rows, const int32_t* d_F,
                    const int32_t* d_labels, int32_t n_global, float* d_loss, float* dz, float* partial,
                    unsigned int* counter, int64_t max_rows, cudaStream_t s);
void launch_sgd(float* p, const float* g, int64_t n, float lr, cudaStream_t s, float* out_loss = nullptr,
                int32_t* out_err = nullptr, const int32_t* err = nullptr);

}  // namespace gnnv
