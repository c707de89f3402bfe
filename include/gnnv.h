/*
 * gnnv.h — C-ABI of libgnnv, the B200-native hot path of one mini-batch
 * GraphSAGE/GCN training iteration as decomposed by GNNavigator
 * (arXiv 2404.09544): sample / transfer / compute.
 *
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n (the paper's
 * equations and Algorithm 1 are restated in DESIGN.md §1).
 *
 * Conventions
 *  - Every call returns gnnv_status; no exception crosses the ABI.  On error
 *    gnnv_last_error() (thread-local) holds a one-line message.
 *      GNNV_ERR_PARAM        "parameter error": ratio not in
 *                            [0,1], fanout < 1, L < 1, n_seeds < 1 or > max, a seed
 *                            id outside [0,N) or repeated, dimension mismatch.
 *      GNNV_ERR_STATE        "state error": call order violated.
 *      GNNV_ERR_OOM          device/pinned allocation failed; the message carries
 *                            the requested bytes.
 *      GNNV_ERR_CUDA         a CUDA runtime error.
 *      GNNV_ERR_COMM         an NCCL error.
 *      GNNV_ERR_UNSUPPORTED  valid but not built (FIFO/LRU policies S:183,
 *                            Bernoulli/layer-wise/subgraph-wise samplers S:96).
 *    Device-side range checks (seed ids) set a device flag that is reported
 *    as GNNV_ERR_PARAM at the next synchronising call on that handle.
 *  - Ownership.  Opaque handles are owned by the library and released with
 *    the matching *_free.  Device buffers passed as `d_*` pointers are owned
 *    by the caller; the library never frees them.  Host features are BORROWED
 *    by gnnv_graph_load (registered in place, zero-copy) and must outlive the
 *    graph.  The CSR is copied to the device.
 *  - Streams.  `gnnv_stream` is a cudaStream_t (NULL = legacy default
 *    stream).  Kernel-launching calls are stream-ordered and do NOT
 *    synchronise unless documented.  Sizes produced by sampling live on the
 *    device; every downstream kernel reads them there, so a whole iteration
 *    runs without a host round trip.
 *  - Layouts.  Row-major everywhere.  A feature/activation matrix with
 *    logical width d is stored with row stride gnnv_row_stride(d) = d rounded
 *    up to a multiple of 4 floats (16-byte rows); padding columns are written
 *    as 0 by every kernel that produces them.  The graph feature table may
 *    use any stride >= d that is a multiple of 4.
 *  - Concurrency.  The GEMM launches (gnnv_layer_*, gnnv_dense_*, gnnv_step)
 *    share per-process workspaces (weight images): on one device they must
 *    not run concurrently on different streams.  Sampling and gathering on
 *    separate blocks/buffers may (the trainer's Eq.4 prefetch does).
 *  - Determinism.  gnnv_sample output is a pure function of (graph, seeds,
 *    fanouts, rng_seed): independent of device, stream, rank and world size.
 *    gnnv_gather rows are bit-exact copies.
 */
#ifndef GNNV_H_
#define GNNV_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GNNV_MAX_LAYERS 8
#define GNNV_VERSION "0.1.0"

typedef enum gnnv_status {
  GNNV_OK = 0,
  GNNV_ERR_PARAM = 1,
  GNNV_ERR_STATE = 2,
  GNNV_ERR_OOM = 3,
  GNNV_ERR_CUDA = 4,
  GNNV_ERR_COMM = 5,
  GNNV_ERR_UNSUPPORTED = 6
} gnnv_status;

typedef struct gnnv_graph gnnv_graph;
typedef struct gnnv_cache gnnv_cache;
typedef struct gnnv_blocks gnnv_blocks;
typedef struct gnnv_trainer gnnv_trainer;
typedef struct gnnv_comm gnnv_comm;
typedef void* gnnv_stream; /* cudaStream_t */

/* Cache update policy: NONE (pyg-like, ratio treated as 0);
 * DEGREE = the static PaGraph template; FIFO / LRU = dynamic caches
 * that start empty and admit every miss (gnnv_cache_update; SURVEY §8(f)
 * NEXT-3, reading Q27). */
typedef enum { GNNV_POLICY_NONE = 0, GNNV_POLICY_DEGREE = 1, GNNV_POLICY_FIFO = 2, GNNV_POLICY_LRU = 3 } gnnv_policy;
/* Cache placement over the GPUs of one box.  REPLICA: every rank holds the
 * C = floor(ratio*N) hottest rows.  SHARDED: rank r holds the rows whose
 * degree rank i satisfies i mod G == r (at local slot i div G); peers' rows
 * are read over NVLink (CUDA IPC).  SHARDED_LOCAL: the same G-way layout with
 * all G shards resident on this device (used to test the routing on one GPU;
 * G = `virtual_shards`). */
typedef enum { GNNV_PLACE_REPLICA = 0, GNNV_PLACE_SHARDED = 1, GNNV_PLACE_SHARDED_LOCAL = 2 } gnnv_placement;
typedef enum { GNNV_KIND_SAGE = 0, GNNV_KIND_GCN = 1 } gnnv_kind;
typedef enum { GNNV_AGGR_MEAN = 0, GNNV_AGGR_SUM = 1 } gnnv_aggr;
typedef enum { GNNV_ACT_NONE = 0, GNNV_ACT_RELU = 1 } gnnv_act;
/* Precision of the dense transform (reading Q18): FP32 = SIMT FFMA (parity
 * mode); BF16 = operands rounded RNE to bf16 by the producer warps, fp32
 * accumulation on tcgen05; TF32 = fp32 operands fed by TMA straight to
 * tcgen05 kind::tf32 (10-bit mantissa, fp32 accumulation) -- the
 * throughput mode, since these GEMMs are HBM-bound on fp32 activations.
 * Aggregation (SpMM) is fp32 in every mode.  Tensor-core modes support
 * d_out <= 252 (fwd) / 256 (dW). */
typedef enum { GNNV_PREC_FP32 = 0, GNNV_PREC_BF16 = 1, GNNV_PREC_TF32 = 2 } gnnv_prec;

/* ------------------------------------------------------------------ misc */
const char* gnnv_last_error(void);
/* Named options (DESIGN.md §9 has each one's measurement on products).
 * Opt-in variants, measured slower than or equal to the default: GNNV_XROWS,
 * GNNV_GEMM_PAIR, GNNV_BWD_PULL, GNNV_L2PUSH, GNNV_LASTUSE,
 * GNNV_STATIC_TILES, GNNV_PF_AGG, GNNV_HID16_DW (a hidden layer's dW/dX over
 * a converted bf16 G), GNNV_BWD_NARROW (the 4-column bf16 push).
 * Switches back to the fp32 / TF32 form of a default path: GNNV_NO_TAIL,
 * GNNV_NO_PDL, GNNV_NO_BF16ACT (Q30), GNNV_NO_BF16TABLE (Q31), GNNV_NO_DW16
 * (Q32), GNNV_NO_FWD16 (Q33), GNNV_NO_HID16 and GNNV_NO_TAIL16 (Q34),
 * GNNV_NO_DA16 (fp32 dA in the bf16 push), GNNV_NO_BRES (the bf16 forward
 * GEMM re-reads W^T per tile instead of keeping it in shared memory),
 * GNNV_NO_EPPIPE (its epilogue loads each pass's TMEM columns at the top of
 * the pass instead of one pass ahead).
 * Integer options:
 * GNNV_PF_CAP (CTA cap of the Eq.4 prefetch's launches, 0 = none),
 * GNNV_PF_PRIO (its stream priority), GNNV_DW16_MINKB (k-blocks per CTA
 * of the bf16 dW, default 16).
 * value 1 = on, 0 = off (integers: the value, >= 0 here; a negative
 * priority only through the environment), -1 = back to the environment
 * variable of the same name (read once per process; set and not "0" = on).
 * Options that shape a trainer or blocks take effect for those created
 * afterwards, the rest for kernels launched afterwards.  PARAM on an
 * unknown name.  Process-wide; not for concurrent use with running steps. */
gnnv_status gnnv_set_option(const char* name, int32_t value);
/* Debug (GNNV_GUARD_ALLOC=1 in the environment when the first allocation is
 * made): every library allocation carries 64 KB guard regions before and
 * after it; this call synchronises the device and sets *n_bad to the number
 * of guard regions whose bytes changed (out-of-bounds writes), naming them
 * in gnnv_last_error().  0 when guards are off. */
gnnv_status gnnv_debug_check_guards(int32_t* n_bad);
const char* gnnv_version(void);
/* Number of kernels libgnnv has launched in this process (monotonic). */
uint64_t gnnv_launch_count(void);
/* Host-link probe (measurement helper, Eq.6's bound): SM zero-copy reads of
 * `bytes` of pinned host memory `h_buf` (page-locked by the caller,
 * device-mapped), 16 bytes per thread and load, the pattern of the gather's
 * cache misses at full row width; *ms = device time of `reps` passes
 * (CUDA events on `s`).  Synchronises `s`.  Errors: PARAM (null, bytes not
 * a multiple of 16), CUDA. */
gnnv_status gnnv_host_read_probe(const void* h_buf, int64_t bytes, int32_t reps, float* ms, gnnv_stream s);
/* d rounded up to a multiple of 4 (floats). */
int32_t gnnv_row_stride(int32_t d);

/* ----------------------------------------------------------------- graph */
/* G(V,E) with features h^0_v and labels (CSR invariants S:25-27).
 *  indptr   host int64[n_nodes+1], indptr[0]=0, non-decreasing, indptr[n]=nnz
 *  indices  host int32[nnz], every id in [0,n_nodes); rows need not be sorted,
 *           but sampled positions refer to the order given (reading Q5)
 *  host_feats host float32[n_nodes * row_stride], borrowed (registered
 *           mapped/read-only in place; must stay alive until gnnv_graph_free)
 *  feat_dim logical d (n_attr); row_stride >= d, multiple of 4
 *  labels   host int32[n_nodes] in [0,n_classes); copied
 *  device   CUDA ordinal the graph lives on
 * Errors: PARAM on size/stride violations; OOM; CUDA.  Synchronous. */
gnnv_status gnnv_graph_load(const int64_t* indptr, const int32_t* indices, int64_t n_nodes, int64_t nnz,
                            const float* host_feats, int32_t feat_dim, int32_t row_stride,
                            const int32_t* labels, int32_t n_classes, int32_t device, gnnv_graph** out);
gnnv_status gnnv_graph_free(gnnv_graph* g);
/* Device pointers of the graph (valid while g lives). */
typedef struct {
  int64_t n_nodes, nnz;
  int32_t feat_dim, row_stride, n_classes, device;
  const int64_t* d_indptr;
  const int32_t* d_indices;
  const int32_t* d_labels;
  const float* d_host_feats; /* device-mapped alias of the pinned host table */
} gnnv_graph_view;
gnnv_status gnnv_graph_info(const gnnv_graph* g, gnnv_graph_view* out);

/* ------------------------------------------------------------------ comm */
/* NCCL over NVLink/NVSwitch, one process per GPU.  The 128-byte unique id is
 * produced on rank 0 and exchanged by the caller (torch process group).
 * unique_id128 == NULL creates a host-only comm (rank/world only, no NCCL):
 * gnnv_allreduce_sum then fails with STATE for world > 1, and a SHARDED
 * cache needs gnnv_cache_open_peers. */
gnnv_status gnnv_comm_unique_id(void* out128);
gnnv_status gnnv_comm_init(int32_t rank, int32_t world, const void* unique_id128, int32_t device, gnnv_comm** out);
gnnv_status gnnv_comm_free(gnnv_comm* c);
/* In-place sum over ranks of d_buf[0:n) (fp32), stream-ordered. */
gnnv_status gnnv_allreduce_sum(gnnv_comm* c, float* d_buf, int64_t n, gnnv_stream s);

/* ----------------------------------------------------------------- cache */
/* Device feature cache: "initialized according to the available memory"
 * (§3.2), PaGraph static degree template.  Capacity
 * C = floor(ratio * N) in IEEE double; vertices ordered by
 * (degree desc, id asc); slot(v) = rank(v) if rank(v) < C else -1.
 *  comm            NULL => single GPU (SHARDED then has one shard)
 *  virtual_shards  G for SHARDED_LOCAL (>=1), ignored otherwise
 * Errors: PARAM (ratio not in [0,1]); UNSUPPORTED (FIFO/LRU across GPUs); OOM (message
 * carries the bytes, Γ_cache = C * row_stride * 4, Eq.10).
 * Synchronous (fills the rows from the pinned host table). */
gnnv_status gnnv_cache_build(gnnv_graph* g, double ratio, int32_t policy, int32_t placement,
                             gnnv_comm* comm, int32_t virtual_shards, gnnv_cache** out);
gnnv_status gnnv_cache_free(gnnv_cache* c);
/* SHARDED across GPUs (north_star: "the feature cache is sharded across the
 * GPUs' HBM and read peer-to-peer over NVLink"): rank r holds
 * the rows of degree rank i = j*G + r at row j, and the gather kernel reads
 * the other ranks' rows in place through CUDA IPC mappings (one-sided
 * NVLink loads, no collective on the data path).  With an NCCL comm,
 * gnnv_cache_build exchanges the IPC handles itself (all-gather, collective
 * over all ranks).  With a host-only comm the caller all-gathers the 64-byte
 * handles of gnnv_cache_ipc_handle (rank order, world * 64 bytes) and passes
 * them to gnnv_cache_open_peers; gnnv_gather / trainer creation fail with
 * STATE until then.  Both synchronous; STATE unless placement is SHARDED. */
/* Dynamic caches (policy FIFO / LRU, one device; NEXT-3): SPEC's
 * access_batch for the batch sampled in b whose rows were
 * gathered into d_X (all n_L rows, row stride = the graph's): LRU stamps the
 * hits with the batch index; the misses are admitted in ascending F_L order,
 * each into a free slot (lowest first) or evicting the resident with the
 * smallest key -- (last access, admission order) for LRU, admission order
 * for FIFO (Eq.5's "replaced stale data"); their rows are copied
 * from d_X.  Call once per gathered batch, in batch order (the trainer does,
 * after each gather, on the gather's stream).  Stream-ordered, no sync.
 * STATE for a static cache or unsampled blocks. */
gnnv_status gnnv_cache_update(gnnv_cache* c, const gnnv_blocks* b, const float* d_X, gnnv_stream s);
/* Cumulative counters of a dynamic cache: int64[4] = hits, misses, replaced
 * (evictions), admitted; zeros for a static cache.  Synchronises. */
gnnv_status gnnv_cache_counters(const gnnv_cache* c, int64_t* host4);
/* Device pointer to the slot -> vertex table (int32[capacity], -1 free) of
 * a dynamic cache (valid while c lives).  STATE for a static cache. */
gnnv_status gnnv_cache_owners(const gnnv_cache* c, const int32_t** d_owner);
gnnv_status gnnv_cache_ipc_handle(const gnnv_cache* c, void* out64);
gnnv_status gnnv_cache_open_peers(gnnv_cache* c, const void* handles);
typedef struct {
  int64_t capacity;     /* C: cached rows over all shards */
  int64_t local_rows;   /* rows resident on this device */
  int64_t bytes;        /* Γ_cache on this device */
  int32_t world, rank;  /* shard count G and this device's shard */
  int32_t placement;
  const int32_t* d_slot;   /* int32[N]: degree rank if cached else -1 */
  const int32_t* d_order;  /* int32[N]: vertices in (degree desc, id asc) order */
} gnnv_cache_view;
gnnv_status gnnv_cache_info(const gnnv_cache* c, gnnv_cache_view* out);

/* ---------------------------------------------------------------- blocks */
/* Workspace for the sampled blocks b_0..b_{L-1} of one rank, sized for the
 * upper bound n_{h+1} <= min(N, n_h (1 + k_h)) (Eq.12, tau=1). */
gnnv_status gnnv_blocks_create(gnnv_graph* g, int32_t max_seeds, const int32_t* fanouts, int32_t L,
                               gnnv_blocks** out);
gnnv_status gnnv_blocks_free(gnnv_blocks* b);
/* Locality-biased sampling (the 2PGraph template,
 * selection probability "a function of data locality"):
 * subsequent gnnv_sample calls on b draw each node's min(k, deg) neighbours
 * by successive weighted sampling without replacement, cached neighbours
 * (slot of c >= 0) weighing 1 + 4*bias and the others 1 (SPEC S:123,
 * S:159; reading Q26: bias in {0, 1/4, 1/2, 3/4, 1}, so the weight is an
 * integer 1..5 and the draws are exact integer arithmetic on the same
 * Philox words as the unbiased sampler).  bias 0 restores the unbiased
 * Floyd sampler (c may then be NULL).  c must outlive the blocks' use.
 * PARAM on any other bias or a missing cache; STATE if c belongs to
 * another graph. */
gnnv_status gnnv_blocks_set_locality(gnnv_blocks* b, const gnnv_cache* c, double bias);

/* SubgraphSampling (Algorithm 1 line 2) with the unified node-wise
 * sampler of Eq.2: for every v in F_h, min(k_h, deg v) distinct
 * neighbours uniformly without replacement (reading Q1), Philox4x32-10 draws
 * keyed by (rng_seed; hop, node, draw) fed to Floyd's algorithm (Q4),
 * ascending CSR position (Q5); F_{h+1} = F_h ++ new ids in first-appearance
 * order (Q3, Q6).  fanouts[0] applies to the seeds (Q2).
 *  d_seeds  device int32[n_seeds], unique ids in [0,N) (Q19); fanouts/L
 *           must equal the ones given to gnnv_blocks_create (fanout <= created)
 * Outputs stay in `b` until the next gnnv_sample on `b`.  Stream-ordered, no
 * host sync.  Errors: PARAM (n_seeds, fanouts; bad seed ids reported at the
 * next gnnv_blocks_info(sync=1)). */
gnnv_status gnnv_sample(gnnv_graph* g, const int32_t* d_seeds, int32_t n_seeds, const int32_t* fanouts,
                        int32_t L, uint64_t rng_seed, gnnv_blocks* b, gnnv_stream s);

/* Block b_h: dst = F_h (n_dst rows), src = F_{h+1} (n_src rows, dst prefix
 * first).  indptr int32[n_dst+1], indices int32[nnz] = local ids into
 * F_{h+1}; src_global = F_{h+1} (global ids).  max_* are the capacities. */
typedef struct {
  int64_t n_dst, n_src, nnz;
  int64_t max_dst, max_src, max_nnz;
  const int32_t* d_indptr;
  const int32_t* d_indices;
  const int32_t* d_src_global;
} gnnv_block_view;
/* Fills per_hop[0..L-1].  sync=1: synchronises `s`, copies the sizes to the
 * host and reports a pending device error; sync=0: sizes are -1 and only the
 * pointers and capacities are valid. */
gnnv_status gnnv_blocks_info(gnnv_blocks* b, int32_t sync, gnnv_stream s, gnnv_block_view* per_hop);
/* Device int32[2L+1]: n_0..n_L then nnz_0..nnz_{L-1} (written by gnnv_sample). */
const int32_t* gnnv_blocks_device_sizes(const gnnv_blocks* b);
int32_t gnnv_blocks_num_layers(const gnnv_blocks* b);

/* ---------------------------------------------------------------- gather */
/* Transfer (Algorithm 1 line 3; §3.2; Eq.6):
 * X[i,:] = feat[F_L[i], :] for i < n_L, bit-exact, full row stride of the
 * graph.  Source per row: local HBM cache slot, a peer GPU's shard over
 * NVLink, or the pinned host table (zero-copy over PCIe) on a miss.
 *  d_X      device float32[max n_L * graph row_stride] (caller-owned)
 *  d_stats  device int64[4] accumulated: rows, hits_local, hits_peer,
 *           misses_host (reading Q8: per unique row of F_L); may be NULL
 * Stream-ordered.  Errors: STATE if b was never sampled. */
gnnv_status gnnv_gather(const gnnv_cache* c, const gnnv_blocks* b, float* d_X, int64_t* d_stats, gnnv_stream s);

/* ---------------------------------------------------------------- layers */
typedef struct {
  int32_t d_in, d_out;
  int32_t in_stride;  /* row stride of H_src / dH_src (>= d_in, %4==0) */
  int32_t kind;       /* gnnv_kind */
  int32_t aggr;       /* gnnv_aggr */
  int32_t act;        /* gnnv_act */
  int32_t prec;       /* gnnv_prec */
} gnnv_layer_desc;

/* Buffer sizing for the layer calls: the row counts live on the device (the
 * step never synchronises), so every activation / gradient buffer passed
 * below must be allocated for the CAPACITY rows of its block
 * (gnnv_block_view.max_dst / max_src, available with sync=0).  Rows beyond
 * the actual counts may be read (and ignored); outputs are written for the
 * actual rows only, except dH_src rows beyond n_src which are unspecified.
 *
 * GNN layer i in 1..L on block b_{L-i} (Eq.1; Algorithm 1 lines
 * 5-6 P:110-111; reading Q11):
 *   SAGE: A = Agg(H_src), H_dst = act(H_src[0:n_dst] W_s + A W_n + b)
 *   GCN : A = (h_v + sum_u h_u)/(c_v+1) (or sum), H_dst = act(A W + b)
 *  d_Hsrc  [n_src x in_stride]; d_W [(2 or 1)*d_in x d_out] row-major
 *          ([W_s; W_n] for SAGE); d_b [d_out]
 *  d_Hdst  [n_dst x row_stride(d_out)] output; d_saveA [n_dst x
 *          row_stride(d_in)] the aggregate, kept for the backward.
 * Stream-ordered.  Errors: PARAM (layer range, dims), STATE. */
gnnv_status gnnv_layer_fwd(gnnv_blocks* b, int32_t layer, const gnnv_layer_desc* ld, const float* d_Hsrc,
                           const float* d_W, const float* d_b, float* d_Hdst, float* d_saveA, gnnv_stream s);

/* Backward of gnnv_layer_fwd (Algorithm 1 line 8):
 * G' = G * 1[H_dst > 0] (ReLU); dW = [H_dst|A]^T G' (SAGE) or A^T G' (GCN);
 * db = sum_rows G'; if d_Gsrc: dH_src = P^T (G' W_n^T) + [G' W_s^T; 0].
 *  d_Gdst  dL/dH_dst (post-activation) [n_dst x row_stride(d_out)]
 *  d_Gsrc  [n_src x in_stride] overwritten; NULL for layer 1
 *  d_dW, d_db overwritten (same layout as W, b).
 * Stream-ordered.  Summation order: FP32 and BF16 reduce dW/db split-K
 * partials in a fixed order (bitwise reproducible); TF32 adds the split-K
 * partials and db into dW/db with red.global.add.f32, so their rounding
 * depends on the order the CTAs arrive in (run-to-run differences at fp32
 * rounding level, within the tf32 tolerance); dH_src uses fp32 atomics
 * (order-dependent rounding) in every mode. */
gnnv_status gnnv_layer_bwd(gnnv_blocks* b, int32_t layer, const gnnv_layer_desc* ld, const float* d_Gdst,
                           const float* d_Hdst, const float* d_Hsrc, const float* d_saveA, const float* d_W,
                           float* d_Gsrc, float* d_dW, float* d_db, gnnv_stream s);

/* Softmax cross-entropy over the n_0 seeds (Algorithm 1 line 7 P:112):
 * loss = (1/n_global) sum_i [lse(z_i) - z_i[y_i]], dz = (softmax - onehot)/n_global.
 *  d_logits [n_0 x stride], labels from the graph indexed by F_0.
 *  d_loss   device float[1] (overwritten).  Deterministic. */
gnnv_status gnnv_ce_loss(gnnv_blocks* b, const gnnv_graph* g, const float* d_logits, int32_t n_classes,
                         int32_t stride, int32_t n_global, float* d_loss, float* d_dlogits, gnnv_stream s);

/* The layer's dense products on their own (host-side M), for kernel tests
 * and micro-benchmarks.  Layouts as in gnnv_layer_fwd/bwd:
 *  fwd: Y[M x ldy] = act([X1 | X2] W + b), X2 may be NULL (K = K1)
 *  dx : [Y1 | Y2] = G W^T, G [M x ldg] with N columns, Y2 may be NULL
 *  dw : dW = [X1 | X2]^T G (+ db = colsum(G) if d_db); fixed-order split-K
 *       in FP32/BF16, atomic (arrival-order) split-K in TF32
 * prec: gnnv_prec.  Stream-ordered. */
gnnv_status gnnv_dense_fwd(const float* d_X1, int32_t ld1, const float* d_X2, int32_t ld2, int32_t K1,
                           const float* d_W, const float* d_b, float* d_Y, int32_t ldy, int32_t N, int64_t M,
                           int32_t relu, int32_t prec, gnnv_stream s);
gnnv_status gnnv_dense_dx(const float* d_G, int32_t ldg, int32_t N, const float* d_W, int32_t K1, float* d_Y1,
                          int32_t ld1, float* d_Y2, int32_t ld2, int64_t M, int32_t prec, gnnv_stream s);
gnnv_status gnnv_dense_dw(const float* d_X1, int32_t ld1, const float* d_X2, int32_t ld2, int32_t K1,
                          const float* d_G, int32_t ldg, int32_t N, int64_t M, float* d_dW, float* d_db,
                          int32_t prec, gnnv_stream s);

/* Plain gradient descent p <- p - lr g. */
gnnv_status gnnv_sgd(float* d_params, const float* d_grads, int64_t n, float lr, gnnv_stream s);

/* --------------------------------------------------------------- trainer */
typedef struct {
  int32_t L;
  int32_t dims[GNNV_MAX_LAYERS + 1]; /* d_0 = feat_dim, ..., d_L = n_classes */
  int32_t fanouts[GNNV_MAX_LAYERS];
  int32_t max_seeds;
  int32_t kind, aggr, prec;
} gnnv_model_desc;

/* Per-phase device times in ms (Eq.4-8 decomposition). */
typedef struct {
  float sample_ms, gather_ms, fwd_ms, loss_ms, bwd_ms, allreduce_ms, update_ms, total_ms;
} gnnv_step_timing;

/* A whole iteration runner.  Parameters are a flat fp32 vector: for each
 * layer i: W_i [(2 or 1) d_{i-1} x d_i] row-major, then b_i [d_i].
 *  host_params  initial values (copied); comm NULL => single GPU. */
gnnv_status gnnv_trainer_create(gnnv_graph* g, gnnv_cache* c, const gnnv_model_desc* md,
                                const float* host_params, gnnv_comm* comm, gnnv_trainer** out);
gnnv_status gnnv_trainer_free(gnnv_trainer* t);
int64_t gnnv_trainer_num_params(const gnnv_trainer* t);
/* Copies params (and grads of the last step, if d_grads_out/host) to host; synchronises. */
gnnv_status gnnv_trainer_get(gnnv_trainer* t, float* host_params, float* host_grads);
gnnv_status gnnv_trainer_set_params(gnnv_trainer* t, const float* host_params);
/* Blocks of the last step (borrowed, do not free).  With gnnv_trainer_prefetch
 * the trainer alternates between two buffer sets, so query again after every
 * step. */
gnnv_blocks* gnnv_trainer_blocks(gnnv_trainer* t);
/* Which rows of X (activation 0) the trainer materialises: F_level, i.e.
 * L (every row of F_L), L-1 (the dst prefix F_{L-1} only) or -1 (none).
 * L-1 when the cache holds the whole table on this device (capacity N, one
 * shard): the gather then writes only the rows the layer-1 GEMMs read and
 * the layer-1 aggregation reads its source rows from the cache table
 * directly (the retrieval still goes through the cache's slot map; hit
 * counters still cover every row of F_L).  -1 when in addition the model is
 * SAGE with TF32 GEMMs and GNNV_XROWS=1 was set when the trainer was
 * created: the layer-1 GEMMs (forward and dW) then read the H_dst rows from
 * the table as well (TMA gather4 through the same row indices) and X is
 * never written (off by default: slower on products).  -1
 * also with gnnv_trainer_fwd16: layer 1 then reads only the bf16 copies
 * (gnnv_trainer_dw16_operands) and the fp32 X is never written. */
int32_t gnnv_trainer_x_level(const gnnv_trainer* t);
/* Whole-table mode (x_level < L): *d_rowidx = int32[n_L] cache-table row of
 * every F_L row of the last step (row u of layer 1's input is row
 * (*d_rowidx)[u] of *d_table, a [N x stride] fp32 table in degree-rank
 * order); both NULL otherwise.  Borrowed device pointers, valid until the
 * trainer's next step on that buffer set.  Errors: GNNV_ERR_PARAM (null). */
gnnv_status gnnv_trainer_rowidx(const gnnv_trainer* t, const int32_t** d_rowidx, const float** d_table);
/* Device pointers of the trainer's activations for layer i (0 = X) of the
 * last step (same buffer-set caveat; X holds the rows of gnnv_trainer_x_level).
 * NULL and 0 for H^1 of a 3-layer trainer whose hidden layers and output
 * layer run over bf16 (gnnv_trainer_tail16): only its bf16 copy exists
 * (gnnv_trainer_activation16) unless GNNV_KEEP_H1. */
gnnv_status gnnv_trainer_activation(gnnv_trainer* t, int32_t i, const float** d_H, int32_t* stride);
/* Layer i's aggregate A^i (1..L) of the last step: [n_dst x stride] fp32
 * (borrowed device pointer, same buffer-set caveat).  With the fused L2 push
 * (gnnv_trainer_l2push) A^{i+1} was accumulated by layer i's GEMM epilogue
 * and H^i (gnnv_trainer_activation) holds only the rows layer i+1 reads as
 * its dst prefix (the first n_dst of layer i+1); its other rows exist only
 * as their ReLU bits.  With gnnv_trainer_fwd16, A^1 exists only as its bf16
 * copy: i = 1 then gives NULL and 0.  PARAM on i outside 1..L. */
gnnv_status gnnv_trainer_aggregate(gnnv_trainer* t, int32_t i, const float** d_A, int32_t* stride);
/* TF32: layer i's ReLU bits (1..L-1) of the last step, bit n%32 of word
 * [row * words + n/32] = (H^i[row][n] > 0); NULL (and 0) otherwise. */
gnnv_status gnnv_trainer_relu_bits(gnnv_trainer* t, int32_t i, const uint32_t** d_bits, int32_t* words);
/* 1 if the trainer fuses layer i+1's aggregation into layer i's GEMM
 * epilogue (TF32 SAGE with L >= 3 and GNNV_L2PUSH), else 0. */
int32_t gnnv_trainer_l2push(const gnnv_trainer* t);
/* 1 if the trainer keeps bf16 intermediates (TF32 SAGE with L >= 3, unless
 * GNNV_NO_BF16ACT): for each hidden layer i <= L-2, H^i is also stored as bf16 (all
 * rows; the next layer aggregates this copy), its fp32 rows only for the
 * next layer's dst prefix (as with gnnv_trainer_l2push), and dL/dH^i is
 * produced and consumed as bf16. */
int32_t gnnv_trainer_bf16act(const gnnv_trainer* t);
/* 1 if layer 1 aggregates the cache's bf16 copy of the whole table (TF32
 * SAGE with the whole table on this device, unless GNNV_NO_BF16TABLE;
 * reading Q31).  The exact fp32 rows are still what gnnv_gather copies. */
int32_t gnnv_trainer_table16(const gnnv_trainer* t);
/* The bf16 copy of H^i (1..L-2) of the last step: [rows x *ld] bf16
 * (borrowed device pointer), NULL and 0 when the trainer keeps none. */
gnnv_status gnnv_trainer_activation16(gnnv_trainer* t, int32_t i, const void** d_H16, int32_t* ld);
/* The bf16 copy of dL/dH^i (after the ReLU mask) the last step's layer-i
 * dW read -- i <= L-2 with bf16 intermediates (reading Q30), hidden layers
 * 2..L-1 with their bf16 dW (reading Q34): [rows x *ld] bf16, NULL and 0
 * when the trainer keeps none. */
gnnv_status gnnv_trainer_gradient16(gnnv_trainer* t, int32_t i, const void** d_G16, int32_t* ld);
/* 1 if layer 1's dW runs over bf16 operands (gemm_dw16: bf16act and
 * table16, d_in + 1 <= 256, hidden a multiple of 64 up to 256, unless
 * GNNV_NO_DW16; reading Q32).  Its operands of the last step: the bf16
 * copy of X's dst prefix with 1.0 in column d_in (the db column) and the
 * bf16 copy of A^1, both [n_dst x *ld] (borrowed device pointers). */
int32_t gnnv_trainer_dw16(const gnnv_trainer* t);
/* 1 if layer 1's forward GEMM also reads those bf16 copies (kind::f16 over
 * [X16 | A16] and W rounded to bf16; with gnnv_trainer_dw16, unless
 * GNNV_NO_FWD16; reading Q33). */
int32_t gnnv_trainer_fwd16(const gnnv_trainer* t);
/* The bf16 copy of layer i's aggregate A^i the last step's kind::f16 GEMMs
 * read: layer 1 with gnnv_trainer_dw16 (reading Q32), hidden layers
 * 2..L-1 of a bf16-intermediate trainer unless GNNV_NO_HID16 (their forward
 * GEMM reads [bf16 H^{i-1} dst prefix | this copy], reading Q34): [n_dst x
 * *ld] bf16, NULL and 0 when there is none. */
gnnv_status gnnv_trainer_aggregate16(gnnv_trainer* t, int32_t i, const void** d_A16, int32_t* ld);
/* 1 if the fused output layer writes dL/dH^{L-1} as bf16 (with db^{L-1}'s
 * partial column sums) and layer L-1's dW / dX run over bf16 operands
 * (bf16 intermediates with the fused output layer, unless GNNV_NO_TAIL16;
 * reading Q34).  gnnv_trainer_gradient16(L-1) then returns that copy. */
int32_t gnnv_trainer_tail16(const gnnv_trainer* t);
/* 1 if the trainer's sampler leaves the last hop unrelabelled (with
 * gnnv_trainer_fwd16, unless GNNV_NO_LASTROWS or GNNV_LASTUSE): the last
 * hop's sampled ids claim no local id, so its block (gnnv_blocks_info of
 * gnnv_trainer_blocks) has n_src = n_dst and F_L = F_{L-1}, and its CSR
 * indices are the ids' cache-table rows (slot[u]; the cache's d_order maps
 * them back); gnnv_trainer_rowidx covers F_{L-1} and the gather counters
 * count F_{L-1}'s rows.  The same sampled edges as the relabelled form. */
int32_t gnnv_trainer_last_rows(const gnnv_trainer* t);
gnnv_status gnnv_trainer_dw16_operands(gnnv_trainer* t, const void** d_X16, const void** d_A16, int32_t* ld);

/* One iteration of Algorithm 1 on this rank's seed slice:
 * sample -> gather -> L x (aggregate, combine) -> loss -> L x backward ->
 * allreduce(grads, loss) over comm -> SGD.
 *  seeds        int32[n_seeds]; seeds_on_host=1: host memory (copied H2D
 *               inside the call), else device memory
 *  n_global     seeds of the iteration over all ranks (loss scale 1/n_global)
 *  loss_out     host float (loss summed over ranks) or NULL (then the call
 *               does not synchronise unless tm != NULL)
 *  tm           per-phase device times or NULL
 * Stream-ordered on `s`.  Precision (GNNV_PREC_TF32 trainer, SAGE): the
 * layer GEMMs run on tcgen05 in tf32 or, where the trainer keeps bf16
 * operand copies (readings Q30-Q34, gnnv_trainer_dw16 / fwd16 / tail16,
 * aggregate16), in bf16 (kind::f16), always with fp32 accumulation; each
 * bf16 mode has a GNNV_NO_* switch.  Summation order: the bf16 dW
 * (gemm_dw16) adds its per-CTA slices in a fixed order; the TF32 dW and the
 * backward pushes (fp32 and bf16x2 reductions) are order-dependent at their
 * rounding level, so gradients are not bitwise reproducible run to run. */
gnnv_status gnnv_step(gnnv_trainer* t, const int32_t* seeds, int32_t n_seeds, int32_t seeds_on_host,
                      int32_t n_global, uint64_t rng_seed, float lr, float* loss_out, gnnv_step_timing* tm,
                      gnnv_stream s);
/* Fine-grained timeline: with on=1 every gnnv_step records CUDA events on its
 * stream around each kernel group (sample, gather, spmm_fwd.l<i>,
 * gemm_fwd.l<i>, loss, relu_mask.l<i>, gemm_dw.l<i>, gemm_dx.l<i>,
 * spmm_bwd.l<i>, allreduce, sgd) without synchronising.  _read synchronises
 * the device and returns the per-name totals since the last read/enable. */
typedef struct {
  char name[32];
  double total_ms;
  int32_t count;
} gnnv_segment;
/* The trainer's sampler locality bias (gnnv_blocks_set_locality with the
 * trainer's cache; both buffer sets).  STATE while a prefetch is pending. */
gnnv_status gnnv_trainer_set_locality(gnnv_trainer* t, double bias);
gnnv_status gnnv_trainer_timeline(gnnv_trainer* t, int32_t on);
gnnv_status gnnv_trainer_timeline_read(gnnv_trainer* t, gnnv_segment* out, int32_t cap, int32_t* n_out);
/* Eq.4 pipelining (T = n_iter max(t_sample + t_transfer,
 * t_replace + t_compute)): enqueue the sampling and the gather of the NEXT
 * step on the trainer's side stream, into a second buffer set, so that they
 * overlap the current step's compute.  The next gnnv_step trains on this
 * batch (its seeds/n_seeds/rng_seed must match; it waits for the prefetch on
 * its stream).  At most one prefetch may be pending (else STATE).  The second
 * buffer set is allocated on the first call (synchronises once).
 * Ordering: the prefetch waits for the step that last used its buffer set
 * (two steps back) and, for DEVICE seeds, for the work already enqueued on
 * `s` -- pass the stream that produced the seeds, not the step stream, or the
 * prefetch serialises behind the step in flight.  HOST seeds are copied to a
 * pinned staging buffer (the host waits only for the previous copy out of
 * that buffer) and impose no stream dependency. */
gnnv_status gnnv_trainer_prefetch(gnnv_trainer* t, const int32_t* seeds, int32_t n_seeds, int32_t seeds_on_host,
                                  uint64_t rng_seed, gnnv_stream s);
/* Makes `s` wait for the pending prefetch (if any) to complete -- without
 * consuming it -- so that a timed region closed by an event on `s` contains
 * every batch it prefetched.  No-op without a pending prefetch. */
gnnv_status gnnv_trainer_join_prefetch(gnnv_trainer* t, gnnv_stream s);
/* Loss of the last step (summed over ranks) to the host; synchronises `s`
 * and reports a pending seed error.  Lets a pipelined loop enqueue the next
 * prefetch before blocking on the loss. */
gnnv_status gnnv_trainer_read_loss(gnnv_trainer* t, float* loss_out, gnnv_stream s);
/* Asynchronous loss read-back (the e2e loop's per-step result without a
 * per-step stream synchronisation): every step's SGD kernel writes the
 * step's all-reduced loss and seed-error flag into a mapped pinned ring
 * slot (zero-copy, no copy on the stream; a step whose batch had an
 * invalid seed writes its flag and skips its SGD update -- the flag is
 * reset by every sample, so it never outlives its batch); _loss_async records an event on
 * `s` after the last enqueued step and returns its ticket (the step index);
 * _loss_result waits for that event only and returns the loss (PARAM if the
 * step saw a bad seed).  The ring holds the last 8 steps; an older ticket
 * is STATE.  STATE before the first step. */
gnnv_status gnnv_trainer_loss_async(gnnv_trainer* t, int64_t* ticket, gnnv_stream s);
gnnv_status gnnv_trainer_loss_result(gnnv_trainer* t, int64_t ticket, float* loss_out);
/* Device counters of the last step's gather: int64[4] (see gnnv_gather). */
gnnv_status gnnv_trainer_stats(gnnv_trainer* t, int64_t* host_stats4);

#ifdef __cplusplus
}
#endif
#endif /* GNNV_H_ */
