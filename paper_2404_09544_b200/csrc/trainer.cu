// gnnv_step: one whole iteration of Algorithm 1 on one rank.
//
// sample -> gather -> L x (aggregate, combine) -> loss -> L x backward ->
// allreduce(grads ++ loss) -> SGD, all stream-ordered on one stream with the
// frontier sizes kept on the device (no host round trip inside the step).
// Per-phase CUDA events give the Eq.4-8 decomposition:
// t_sample, t_transfer (gather), t_compute (fwd + loss + bwd + update).
#include <cuda.h>
#include <string.h>

#include "common.cuh"

namespace gnnv {
void layer_fwd_impl(gnnv_blocks* b, int32_t layer, const gnnv_layer_desc* ld, const float* Hsrc, const float* W,
                    const float* bias, float* Hdst, float* A, cudaStream_t s, Timeline* tl, uint32_t* mask_bits,
                    const float* agg_table, const int32_t* rowidx, const XRows* xr, const FwdPush* push,
                    bool agg_ready, const Bf16Io* io);
void layer_bwd_impl(gnnv_blocks* b, int32_t layer, const gnnv_layer_desc* ld, const float* Gdst, const float* Hdst,
                    const float* Hsrc, const float* A, const float* W, float* Gsrc, float* dW, float* db,
                    cudaStream_t s, Timeline* tl, const uint32_t* mask_bits, bool g_masked,
                    const uint32_t* src_bits, int32_t src_bits_ld, const XRows* xr, bool grads_zeroed,
                    const Bf16Io* io);
}  // namespace gnnv

using namespace gnnv;

struct gnnv_trainer {
  gnnv_graph* g = nullptr;
  gnnv_cache* c = nullptr;
  gnnv_comm* comm = nullptr;
  gnnv_model_desc md{};
  gnnv_blocks* b = nullptr;
  int64_t nparams = 0;
  int64_t w_off[GNNV_MAX_LAYERS] = {0}, b_off[GNNV_MAX_LAYERS] = {0};
  float* d_params = nullptr;
  float* d_grads = nullptr;  // nparams + 1 (loss), all-reduced together
  int32_t* d_seeds = nullptr;
  int32_t* h_seeds = nullptr;  // pinned staging
  float* h_out = nullptr;      // pinned: loss
  int32_t* h_err = nullptr;    // pinned: sample error flag
  // asynchronous loss read-back: a ring of pinned (loss, error flag) slots,
  // each completed by an event (gnnv_trainer_loss_async / _loss_result)
  static constexpr int kLossRing = 8;
  float* h_lossr = nullptr;       // [kLossRing] mapped pinned: the SGD kernel writes step s's loss at s % ring
  int32_t* h_errr = nullptr;      // [kLossRing] mapped pinned: its seed-error flag
  float* d_lossr = nullptr;       // device aliases of the two rings
  int32_t* d_errr = nullptr;
  cudaEvent_t ev_loss[kLossRing] = {nullptr};
  int64_t steps_done = 0;         // steps enqueued (the ring position)
  int64_t loss_tickets = 0;
  float* H[GNNV_MAX_LAYERS + 1] = {nullptr};
  int32_t Hs[GNNV_MAX_LAYERS + 1] = {0};
  float* A[GNNV_MAX_LAYERS + 1] = {nullptr};
  float* G[GNNV_MAX_LAYERS + 1] = {nullptr};
  // TF32: ReLU bits of each hidden layer's output (written by its forward
  // epilogue; the backward masks dH where it is produced)
  uint32_t* mbits[GNNV_MAX_LAYERS + 1] = {nullptr};
  float* loss_partial = nullptr;
  // fused output layer (tail.cu): TF32 SAGE with L >= 2 and the shapes
  // tail_supported() accepts; GNNV_NO_TAIL=1 keeps the per-kernel path
  bool tail = false;
  // fused L2 push (TF32 SAGE, L >= 3; opt-in GNNV_L2PUSH=1 -- measured
  // slower): the GEMM epilogue of layer i (1 <= i <= L-2)
  // accumulates layer i+1's aggregate A^{i+1} = P H^i with L2 reductions
  // over the CSC of hop L-i-1 while H^i is still on chip, so H^i is stored
  // only for the dst prefix layer i+1 reads (its other rows -- 88% of
  // products' H^1 -- never reach HBM) and layer i+1 runs no aggregation
  bool l2push = false;
  // layer-1 aggregation loads a source row for the last time with an L2
  // evict_first hint (sampler: last-use slot per src id; opt-in GNNV_LASTUSE=1)
  bool lastuse = false;
  // Layer 1's aggregation depends on the sampled block and the features
  // only (no weight), so the Eq.4 prefetch also computes it for the batch it
  // prepares (on the side stream, into that buffer set's A^1), and a step
  // consuming a prefetch starts at the layer-1 GEMM.  Opt-in (GNNV_PF_AGG=1):
  // measured neutral on products (1.325-1.329 vs 1.327-1.330 ms; the step
  // then waits ~0.2 ms for the longer prefetch).  A^1 per
  // buffer set: A1b[k] (t->A[1] follows the current set).
  bool pf_agg = false;
  // bf16 intermediates (TF32 SAGE, L >= 3; GNNV_NO_BF16ACT=1: off): H^i and dL/dH^i of
  // the hidden layers i <= L-2 -- the widest activations, read back by the
  // next layer's aggregation and by layer i's dW -- as bf16 (H16[i], G16[i],
  // row stride ld16[i]); H[i] fp32 then holds only layer i+1's dst prefix
  bool bf16act = false;
  // whole-table TF32 SAGE: the layer-1 aggregation reads the cache's bf16
  // copy of the table (reading Q31; GNNV_NO_BF16TABLE=1: the fp32 table)
  bool table16 = false;
  // with both: layer 1's dW over bf16 MN-major operands (gemm_dw16, no
  // transposer): the gather also writes a bf16 copy of X's dst prefix with a
  // ones column at d (X16[k]) and the layer-1 aggregation a bf16
  // copy of A^1 (A16[k]); GNNV_NO_DW16=1: the TF32 dW
  bool dw16 = false;
  // with dw16: layer 1's forward GEMM reads the same bf16 copies (kind::f16,
  // reading Q33); GNNV_NO_FWD16=1: the TF32 GEMM over the fp32 rows
  bool fwd16 = false;
  // bf16 intermediates: the forward GEMMs of hidden layers 2..L-1 read
  // [H16^{i-1} dst prefix | A16^i] (kind::f16, reading Q34); the
  // aggregation then also writes A^i as bf16 (A16h[i], stride ld16[i-1]).
  // GNNV_NO_HID16=1: the TF32 GEMMs over fp32 rows
  bool hid16 = false;
  void* A16h[GNNV_MAX_LAYERS + 1] = {nullptr};
  // opt-in GNNV_HID16_DW=1: their dW and dX run over bf16 too (G^i's bf16
  // copy G16h[i], stride ld16[i], written by gemm_dw16's db pass).  Measured
  // slower on products (layer 2: 60K rows, too few k-blocks per CTA to
  // amortise the per-CTA TMEM flush)
  void* G16h[GNNV_MAX_LAYERS + 1] = {nullptr};
  // the fused output layer writes dL/dH^{L-1} only as bf16 (G16h[L-1],
  // stride Hs[L-1]) and db^{L-1}'s partial column sums (tail_dbp): layer
  // L-1's dW and dX then run over bf16 with no conversion pass (reading
  // Q34); GNNV_NO_TAIL16=1: fp32 dL/dH^{L-1}
  bool tail16 = false;
  float* tail_dbp = nullptr;
  // with fwd16: the sampler does not relabel the last hop; its CSR indices
  // are the sampled ids' cache-table rows (blocks_set_last_rows) and the
  // layer-1 aggregation reads them directly.  GNNV_NO_LASTROWS=1: relabelled
  bool last_rows = false;
  // with hid16 and tail16 at L = 3 nothing reads H^1's fp32 rows (layer 2's
  // GEMMs read its bf16 copy, the output layer reads H^2): layer 1's
  // epilogue writes none (h1_fp32 false; GNNV_KEEP_H1=1 keeps them)
  bool h1_fp32 = true;
  int32_t* d_zero = nullptr;
  void* X16[2] = {nullptr, nullptr};
  void* A16[2] = {nullptr, nullptr};
  int32_t ld16x = 0;  // their row stride: d + 1 rounded up to 8
  void* H16[GNNV_MAX_LAYERS + 1] = {nullptr};
  void* G16[GNNV_MAX_LAYERS + 1] = {nullptr};
  int32_t ld16[GNNV_MAX_LAYERS + 1] = {0};
  float* A1b[2] = {nullptr, nullptr};
  float* tail_dA = nullptr;    // [max_n[0] x dims[L-1]]
  float* tail_part = nullptr;  // per-CTA dW/db partials
  unsigned int* loss_counter = nullptr;
  int64_t* d_stats = nullptr;
  cudaEvent_t ev[8] = {nullptr};
  Timeline tl;
  // Eq.4 pipeline: sample + gather of step t+1 on a side stream
  // into the other buffer set while step t computes.  bb[cur] / X[cur] are
  // the current step's blocks and gathered features (b == bb[cur], H[0] ==
  // X[cur]).
  gnnv_blocks* bb[2] = {nullptr, nullptr};
  float* X[2] = {nullptr, nullptr};
  int32_t* d_seedsb[2] = {nullptr, nullptr};
  int32_t* h_seedsb[2] = {nullptr, nullptr};
  int64_t* d_statsb[2] = {nullptr, nullptr};
  int cur = 0;
  bool pending = false;
  int pend_n = 0;
  uint64_t pend_rng = 0;
  cudaStream_t side = nullptr;
  cudaEvent_t ev_ready[2] = {nullptr, nullptr}, ev_free[2] = {nullptr, nullptr}, ev_in = nullptr;
  // NEXT-3 dynamic cache: the last admission (serial step or prefetch, on
  // whichever stream ran it); every later gather + admission waits on it, so
  // the slot map, the table and the shared miss buffers are never touched by
  // two batches at once
  cudaEvent_t ev_cache = nullptr;
  bool cache_pending = false;
  cudaEvent_t ev_h2d[2] = {nullptr, nullptr};  // last copy out of h_seedsb[k]
  bool h2d_used[2] = {false, false};
  Timeline tl_side;
  // Whole feature table resident on this device (capacity N, one shard):
  // the gather materialises only the dst prefix F_{L-1} of X and records
  // every F_L row's cache row in rowidx; layer 1 aggregates from the table.
  double loc_bias = 0.0;  // NEXT-2 locality bias for both buffer sets
  bool x_fused = false;
  // x_fused with TF32 SAGE and GNNV_XROWS=1: the layer-1 GEMMs also read
  // H_dst from the table (TMA gather4 through rowidx), so the gather copies
  // no rows at all.  Off by default: measured on products, the gather4 loads
  // (a 400-byte row fetched as four 128-byte pieces, one per k-block) cost
  // the layer-1 GEMMs more (fwd 180 -> 257 us, dW 215 -> 230 us) than the
  // dst-prefix copy they save (92 -> 25 us).
  bool x_rows = false;
  const float* table = nullptr;
  int32_t* rowidx[2] = {nullptr, nullptr};
};

static gnnv_layer_desc layer_desc(const gnnv_trainer* t, int i) {
  gnnv_layer_desc ld{};
  ld.d_in = t->md.dims[i - 1];
  ld.d_out = t->md.dims[i];
  ld.in_stride = t->Hs[i - 1];
  ld.kind = t->md.kind;
  ld.aggr = t->md.aggr;
  ld.act = i < t->md.L ? GNNV_ACT_RELU : GNNV_ACT_NONE;
  ld.prec = t->md.prec;
  return ld;
}

// The prefetch (side) stream: lowest priority, so that the prefetch fills
// the SMs the step leaves idle (DESIGN.md §9 lists the placements measured:
// green contexts, grid caps, high priority, event gates -- none was faster).
static cudaStream_t make_side_stream() {
  int lo = 0, hi = 0;
  GNNV_TRY_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  cudaStream_t st;
  // GNNV_PF_PRIO: the side stream's priority (default: the lowest)
  const int want = env_int("GNNV_PF_PRIO", lo);
  GNNV_TRY_CUDA(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, std::min(lo, std::max(hi, want))));
  return st;
}

static void alloc_dw16(gnnv_trainer* t, int k, const gnnv_blocks* b) {
  const size_t bytes = (size_t)b->max_n[t->md.L - 1] * t->ld16x * 2;
  t->X16[k] = dmalloc(bytes, "bf16 X dst prefix (layer-1 dW)");
  t->A16[k] = dmalloc(bytes, "bf16 layer-1 aggregates (layer-1 dW)");
  GNNV_TRY_CUDA(cudaMemset(t->X16[k], 0, bytes));
  GNNV_TRY_CUDA(cudaMemset(t->A16[k], 0, bytes));
}

extern "C" {

gnnv_status gnnv_trainer_free(gnnv_trainer* t) {
  if (!t) return GNNV_OK;
  cudaSetDevice(t->g ? t->g->device : 0);
  if (t->side) cudaStreamSynchronize(t->side);
  for (int k = 0; k < 2; ++k) {
    gnnv_blocks_free(t->bb[k]);
    dfree(t->X[k]);
    dfree(t->X16[k]);
    dfree(t->A16[k]);
    dfree(t->rowidx[k]);
    if (k == 1) dfree(t->A1b[1]);  // A1b[0] is A[1], freed with the layers
    dfree(t->d_seedsb[k]);
    if (t->h_seedsb[k]) cudaFreeHost(t->h_seedsb[k]);
    dfree(t->d_statsb[k]);
    if (t->ev_ready[k]) cudaEventDestroy(t->ev_ready[k]);
    if (t->ev_free[k]) cudaEventDestroy(t->ev_free[k]);
    if (t->ev_h2d[k]) cudaEventDestroy(t->ev_h2d[k]);
  }
  if (t->ev_in) cudaEventDestroy(t->ev_in);
  if (t->ev_cache) cudaEventDestroy(t->ev_cache);
  if (t->side) cudaStreamDestroy(t->side);
  dfree(t->d_params);
  dfree(t->d_grads);
  if (t->h_out) cudaFreeHost(t->h_out);
  if (t->h_lossr) cudaFreeHost(t->h_lossr);
  if (t->h_errr) cudaFreeHost(t->h_errr);
  for (auto& e : t->ev_loss)
    if (e) cudaEventDestroy(e);
  if (t->h_err) cudaFreeHost(t->h_err);
  if (t->A1b[0]) t->A[1] = t->A1b[0];  // the set-0 buffer is the one the layer loop allocated
  for (int i = 1; i <= GNNV_MAX_LAYERS; ++i) {
    dfree(t->H[i]);
    dfree(t->A[i]);
    dfree(t->G[i]);
  }
  for (auto* m : t->mbits) dfree(m);
  for (int i = 0; i <= GNNV_MAX_LAYERS; ++i) {
    dfree(t->H16[i]);
    dfree(t->G16[i]);
    dfree(t->A16h[i]);
    dfree(t->G16h[i]);
  }
  dfree(t->tail_dbp);
  dfree(t->d_zero);
  dfree(t->loss_partial);
  dfree(t->tail_dA);
  dfree(t->tail_part);
  dfree(t->loss_counter);
  for (auto& e : t->ev)
    if (e) cudaEventDestroy(e);
  delete t;
  return GNNV_OK;
}

gnnv_status gnnv_trainer_create(gnnv_graph* g, gnnv_cache* c, const gnnv_model_desc* md, const float* host_params,
                                gnnv_comm* comm, gnnv_trainer** out) {
  return guarded([&] {
    GNNV_REQUIRE(g && c && md && host_params && out, GNNV_ERR_PARAM, "trainer_create: null");
    GNNV_REQUIRE(c->peers_ready, GNNV_ERR_STATE, "trainer_create: SHARDED cache peers not mapped");
    GNNV_REQUIRE(c->g == g, GNNV_ERR_STATE, "trainer_create: cache belongs to another graph");
    GNNV_REQUIRE(md->L >= 1 && md->L <= GNNV_MAX_LAYERS, GNNV_ERR_PARAM, "trainer_create: L in [1, 8]");
    GNNV_REQUIRE(md->dims[0] == g->d, GNNV_ERR_PARAM, "trainer_create: dims[0] must equal the feature dim");
    GNNV_REQUIRE(md->dims[md->L] == g->n_classes, GNNV_ERR_PARAM, "trainer_create: dims[L] must equal n_classes");
    for (int i = 0; i <= md->L; ++i) GNNV_REQUIRE(md->dims[i] >= 1, GNNV_ERR_PARAM, "trainer_create: dims >= 1");
    GNNV_REQUIRE(md->kind == GNNV_KIND_SAGE || md->kind == GNNV_KIND_GCN, GNNV_ERR_PARAM, "trainer_create: kind");
    GNNV_REQUIRE(md->aggr == GNNV_AGGR_MEAN || md->aggr == GNNV_AGGR_SUM, GNNV_ERR_PARAM, "trainer_create: aggr");
    GNNV_REQUIRE(md->prec >= GNNV_PREC_FP32 && md->prec <= GNNV_PREC_TF32, GNNV_ERR_PARAM, "trainer_create: prec");
    GNNV_TRY_CUDA(cudaSetDevice(g->device));
    gnnv_trainer* t = new gnnv_trainer();
    t->g = g;
    t->c = c;
    t->comm = comm;
    t->md = *md;
    try {
      gnnv_status st = gnnv_blocks_create(g, md->max_seeds, md->fanouts, md->L, &t->b);
      if (st != GNNV_OK) throw Error{st, get_error()};
      const int L = md->L;
      int64_t off = 0;
      for (int i = 1; i <= L; ++i) {
        const int64_t rows = (md->kind == GNNV_KIND_SAGE ? 2 : 1) * (int64_t)md->dims[i - 1];
        t->w_off[i - 1] = off;
        off += rows * md->dims[i];
        t->b_off[i - 1] = off;
        off += md->dims[i];
      }
      t->nparams = off;
      t->d_params = (float*)dmalloc(off * sizeof(float), "params");
      t->d_grads = (float*)dmalloc((off + 1) * sizeof(float), "grads");
      GNNV_TRY_CUDA(cudaMemcpy(t->d_params, host_params, off * sizeof(float), cudaMemcpyHostToDevice));
      GNNV_TRY_CUDA(cudaMemset(t->d_grads, 0, (off + 1) * sizeof(float)));
      t->d_seeds = (int32_t*)dmalloc(md->max_seeds * sizeof(int32_t), "seeds");
      GNNV_TRY_CUDA(cudaMallocHost(&t->h_seeds, md->max_seeds * sizeof(int32_t)));
      GNNV_TRY_CUDA(cudaMallocHost(&t->h_out, 4 * sizeof(float)));
      GNNV_TRY_CUDA(cudaHostAlloc(&t->h_lossr, gnnv_trainer::kLossRing * sizeof(float), cudaHostAllocMapped));
      GNNV_TRY_CUDA(cudaHostAlloc(&t->h_errr, gnnv_trainer::kLossRing * sizeof(int32_t), cudaHostAllocMapped));
      GNNV_TRY_CUDA(cudaHostGetDevicePointer((void**)&t->d_lossr, t->h_lossr, 0));
      GNNV_TRY_CUDA(cudaHostGetDevicePointer((void**)&t->d_errr, t->h_errr, 0));
      for (auto& e : t->ev_loss) GNNV_TRY_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      GNNV_TRY_CUDA(cudaMallocHost(&t->h_err, 4 * sizeof(int32_t)));
      gnnv_blocks* b = t->b;
      t->Hs[0] = g->stride;
      t->x_fused = L > 1 && !c->dynamic && c->capacity == g->n && c->world == 1 && c->shards.size() == 1 &&
                   c->shards[0];
      t->table = t->x_fused ? c->shards[0] : nullptr;
      t->x_rows = t->x_fused && md->prec == GNNV_PREC_TF32 && md->kind == GNNV_KIND_SAGE && env_on("GNNV_XROWS");
      const int64_t xrows = t->x_rows ? 1 : t->x_fused ? b->max_n[L - 1] : b->max_n[L];
      t->H[0] = (float*)dmalloc((size_t)xrows * g->stride * sizeof(float), "X (gathered features)");
      if (t->x_fused) t->rowidx[0] = (int32_t*)dmalloc(b->max_n[L] * sizeof(int32_t), "cache rows of F_L");
      t->pf_agg = env_on("GNNV_PF_AGG");
      for (int i = 1; i <= L; ++i) {
        t->Hs[i] = row_stride(md->dims[i]);
        const int64_t rows = b->max_n[L - i];
        t->H[i] = (float*)dmalloc((size_t)rows * t->Hs[i] * sizeof(float), "H activations");
        t->G[i] = (float*)dmalloc((size_t)rows * t->Hs[i] * sizeof(float), "dH gradients");
        t->A[i] = (float*)dmalloc((size_t)rows * row_stride(md->dims[i - 1]) * sizeof(float), "aggregates");
      }
      if (md->prec == GNNV_PREC_TF32)
        for (int i = 1; i < L; ++i)
          t->mbits[i] = (uint32_t*)dmalloc((size_t)b->max_n[L - i] * mask_words(md->dims[i]) * sizeof(uint32_t),
                                           "ReLU bits");
      t->loss_partial =
          (float*)dmalloc(std::max<int64_t>(256, ceil_div(b->max_n[0], 32)) * sizeof(float), "loss partials");
      t->tail = md->prec == GNNV_PREC_TF32 && L >= 2 &&
                tail_supported(md->kind, md->dims[L - 1], md->dims[L], md->fanouts[0]) && !env_on("GNNV_NO_TAIL");
      t->bf16act = md->prec == GNNV_PREC_TF32 && md->kind == GNNV_KIND_SAGE && L >= 3 && !env_on("GNNV_NO_BF16ACT");
      for (int i = 1; i <= L - 2 && t->bf16act; ++i) t->bf16act = md->dims[i] % 8 == 0;
      if (t->bf16act)
        for (int i = 1; i <= L - 2; ++i) {
          t->ld16[i] = (md->dims[i] + 31) / 32 * 32;
          const size_t bytes = (size_t)b->max_n[L - i] * t->ld16[i] * 2;
          t->H16[i] = dmalloc(bytes, "bf16 activations");
          t->G16[i] = dmalloc(bytes, "bf16 activation gradients");
        }
      t->hid16 = t->bf16act && !env_on("GNNV_NO_HID16");
      for (int i = 2; i <= L - 1 && t->hid16; ++i)
        if (i - 1 > L - 2 || t->ld16[i - 1] % 8 != 0) t->hid16 = false;
      if (t->hid16)
        for (int i = 2; i <= L - 1; ++i) {
          t->A16h[i] = dmalloc((size_t)b->max_n[L - i] * t->ld16[i - 1] * 2, "bf16 aggregates (hidden layers)");
          if (env_on("GNNV_HID16_DW") && md->dims[i] % 64 == 0 && md->dims[i] <= 256 && md->dims[i - 1] <= 256)
            t->G16h[i] = dmalloc((size_t)b->max_n[L - i] * ((md->dims[i] + 31) / 32 * 32) * 2,
                                 "bf16 gradients (hidden-layer dW)");
        }
      t->tail16 = t->tail && t->hid16 && L - 1 >= 2 && t->A16h[L - 1] && md->dims[L - 1] % 64 == 0 &&
                  md->dims[L - 1] <= 256 && md->dims[L - 2] <= 256 && t->Hs[L - 1] % 8 == 0 &&
                  !env_on("GNNV_NO_TAIL16");
      if (t->tail16) {
        dfree(t->G16h[L - 1]);
        t->G16h[L - 1] = dmalloc((size_t)b->max_n[1] * t->Hs[L - 1] * 2, "bf16 dL/dH^{L-1} (output layer)");
        t->tail_dbp = (float*)dmalloc((size_t)tail_db_parts(b->max_n[0]) * md->dims[L - 1] * sizeof(float),
                                      "db^{L-1} partials (output layer)");
      }
      // layer 1 aggregates a bf16 copy of the whole-table cache (reading Q31)
      t->table16 = t->x_fused && md->prec == GNNV_PREC_TF32 && md->kind == GNNV_KIND_SAGE &&
                   !env_on("GNNV_NO_BF16TABLE");
      if (t->table16) cache_bf16_table(c);
      t->dw16 = t->table16 && t->bf16act && !t->x_rows && md->dims[0] + 1 <= 256 && md->dims[1] % 64 == 0 &&
                md->dims[1] <= 256 && !env_on("GNNV_NO_DW16");
      t->ld16x = (md->dims[0] + 1 + 7) / 8 * 8;
      t->fwd16 = t->dw16 && !env_on("GNNV_NO_FWD16");
      if (t->fwd16) {  // layer 1 reads only the bf16 copies: no fp32 X
        dfree(t->H[0]);
        t->H[0] = (float*)dmalloc((size_t)g->stride * sizeof(float), "X (unused: bf16 copies)");
      }
      if (t->dw16) alloc_dw16(t, 0, b);
      t->l2push = !t->bf16act && md->prec == GNNV_PREC_TF32 && md->kind == GNNV_KIND_SAGE && L >= 3 &&
                  env_on("GNNV_L2PUSH");
      if (t->l2push)
        for (int i = 1; i <= L - 2; ++i) blocks_enable_owner_rows(t->b, L - i - 1);
      // dead-row L2 hints for the layer-1 aggregation (spmm.cu HINT; opt-in
      // GNNV_LASTUSE=1: measured 1.11 -> 1.04 GB DRAM reads but 255 -> 262 us
      // on products)
      t->lastuse = env_on("GNNV_LASTUSE");
      if (t->lastuse) blocks_enable_lastuse(t->b);
      if (t->tail) {
        t->tail_dA = (float*)dmalloc((size_t)b->max_n[0] * md->dims[L - 1] * sizeof(float), "output-layer dA");
        t->tail_part = (float*)dmalloc(tail_partial_floats(b->max_n[0], md->dims[L - 1], md->dims[L]) * sizeof(float),
                                       "output-layer dW partials");
      }
      t->loss_counter = (unsigned int*)dmalloc(sizeof(unsigned int), "loss counter");
      GNNV_TRY_CUDA(cudaMemset(t->loss_counter, 0, sizeof(unsigned int)));
      t->d_stats = (int64_t*)dmalloc(4 * sizeof(int64_t), "gather stats");
      GNNV_TRY_CUDA(cudaMemset(t->d_stats, 0, 4 * sizeof(int64_t)));
      if (t->fwd16) blocks_set_rowidx(b, c->d_slot, t->rowidx[0], t->d_stats);  // k_reset writes the cache rows
      t->last_rows = t->fwd16 && !t->lastuse && !env_on("GNNV_NO_LASTROWS");
      t->h1_fp32 = !(t->hid16 && t->tail16 && L == 3) || env_on("GNNV_KEEP_H1");
      t->d_zero = (int32_t*)dmalloc(sizeof(int32_t), "zero");
      GNNV_TRY_CUDA(cudaMemset(t->d_zero, 0, sizeof(int32_t)));
      if (t->last_rows) blocks_set_last_rows(b, c->d_slot);
      for (auto& e : t->ev) GNNV_TRY_CUDA(cudaEventCreate(&e));
      // buffer set 0; set 1 is allocated by the first gnnv_trainer_prefetch
      t->bb[0] = t->b;
      t->X[0] = t->H[0];
      t->d_seedsb[0] = t->d_seeds;
      t->h_seedsb[0] = t->h_seeds;
      t->d_statsb[0] = t->d_stats;
      t->A1b[0] = t->A[1];
      for (int k = 0; k < 2; ++k) {
        GNNV_TRY_CUDA(cudaEventCreateWithFlags(&t->ev_ready[k], cudaEventDisableTiming));
        GNNV_TRY_CUDA(cudaEventCreateWithFlags(&t->ev_free[k], cudaEventDisableTiming));
        GNNV_TRY_CUDA(cudaEventCreateWithFlags(&t->ev_h2d[k], cudaEventDisableTiming));
      }
      GNNV_TRY_CUDA(cudaEventCreateWithFlags(&t->ev_in, cudaEventDisableTiming));
      GNNV_TRY_CUDA(cudaEventCreateWithFlags(&t->ev_cache, cudaEventDisableTiming));
      GNNV_TRY_CUDA(cudaDeviceSynchronize());
    } catch (...) {
      gnnv_trainer_free(t);
      throw;
    }
    *out = t;
  });
}

int64_t gnnv_trainer_num_params(const gnnv_trainer* t) { return t ? t->nparams : -1; }
gnnv_blocks* gnnv_trainer_blocks(gnnv_trainer* t) { return t ? t->b : nullptr; }

int32_t gnnv_trainer_x_level(const gnnv_trainer* t) {
  return t ? (t->x_rows || t->fwd16 ? -1 : t->x_fused ? t->md.L - 1 : t->md.L) : -1;
}

gnnv_status gnnv_trainer_rowidx(const gnnv_trainer* t, const int32_t** d_rowidx, const float** d_table) {
  return guarded([&] {
    GNNV_REQUIRE(t && d_rowidx && d_table, GNNV_ERR_PARAM, "trainer_rowidx: null");
    *d_rowidx = t->x_fused ? t->rowidx[t->cur] : nullptr;
    *d_table = t->x_fused ? t->table : nullptr;
  });
}

gnnv_status gnnv_trainer_get(gnnv_trainer* t, float* host_params, float* host_grads) {
  return guarded([&] {
    GNNV_REQUIRE(t, GNNV_ERR_PARAM, "trainer_get: null");
    GNNV_TRY_CUDA(cudaDeviceSynchronize());
    if (host_params)
      GNNV_TRY_CUDA(cudaMemcpy(host_params, t->d_params, t->nparams * sizeof(float), cudaMemcpyDeviceToHost));
    if (host_grads)
      GNNV_TRY_CUDA(cudaMemcpy(host_grads, t->d_grads, t->nparams * sizeof(float), cudaMemcpyDeviceToHost));
  });
}

gnnv_status gnnv_trainer_set_params(gnnv_trainer* t, const float* host_params) {
  return guarded([&] {
    GNNV_REQUIRE(t && host_params, GNNV_ERR_PARAM, "trainer_set_params: null");
    GNNV_TRY_CUDA(cudaDeviceSynchronize());
    GNNV_TRY_CUDA(cudaMemcpy(t->d_params, host_params, t->nparams * sizeof(float), cudaMemcpyHostToDevice));
  });
}

gnnv_status gnnv_trainer_activation(gnnv_trainer* t, int32_t i, const float** d_H, int32_t* stride) {
  return guarded([&] {
    GNNV_REQUIRE(t && d_H && stride && i >= 0 && i <= t->md.L, GNNV_ERR_PARAM, "trainer_activation: bad args");
    const bool none = i == 1 && !t->h1_fp32;  // only the bf16 copy (gnnv_trainer_activation16)
    *d_H = none ? nullptr : t->H[i];
    *stride = none ? 0 : t->Hs[i];
  });
}

gnnv_status gnnv_trainer_aggregate(gnnv_trainer* t, int32_t i, const float** d_A, int32_t* stride) {
  return guarded([&] {
    GNNV_REQUIRE(t && d_A && stride && i >= 1 && i <= t->md.L, GNNV_ERR_PARAM, "trainer_aggregate: bad args");
    const bool none = i == 1 && t->fwd16;  // layer 1 keeps only the bf16 copy (gnnv_trainer_dw16_operands)
    *d_A = none ? nullptr : t->A[i];
    *stride = none ? 0 : row_stride(t->md.dims[i - 1]);
  });
}

gnnv_status gnnv_trainer_relu_bits(gnnv_trainer* t, int32_t i, const uint32_t** d_bits, int32_t* words) {
  return guarded([&] {
    GNNV_REQUIRE(t && d_bits && words && i >= 1 && i <= t->md.L, GNNV_ERR_PARAM, "trainer_relu_bits: bad args");
    *d_bits = t->mbits[i];
    *words = t->mbits[i] ? mask_words(t->md.dims[i]) : 0;
  });
}

int32_t gnnv_trainer_l2push(const gnnv_trainer* t) { return t && t->l2push ? 1 : 0; }
int32_t gnnv_trainer_bf16act(const gnnv_trainer* t) { return t && t->bf16act ? 1 : 0; }
int32_t gnnv_trainer_table16(const gnnv_trainer* t) { return t && t->table16 ? 1 : 0; }

gnnv_status gnnv_trainer_activation16(gnnv_trainer* t, int32_t i, const void** d_H16, int32_t* ld) {
  return guarded([&] {
    GNNV_REQUIRE(t && d_H16 && ld && i >= 0 && i <= t->md.L, GNNV_ERR_PARAM, "trainer_activation16: bad args");
    *d_H16 = t->H16[i];
    *ld = t->H16[i] ? t->ld16[i] : 0;
  });
}

gnnv_status gnnv_trainer_gradient16(gnnv_trainer* t, int32_t i, const void** d_G16, int32_t* ld) {
  return guarded([&] {
    GNNV_REQUIRE(t && d_G16 && ld && i >= 0 && i <= t->md.L, GNNV_ERR_PARAM, "trainer_gradient16: bad args");
    if (t->G16[i]) {
      *d_G16 = t->G16[i];
      *ld = t->ld16[i];
    } else {  // a hidden layer's dW operand (reading Q34)
      *d_G16 = t->G16h[i];
      *ld = !t->G16h[i] ? 0 : (t->tail16 && i == t->md.L - 1) ? t->Hs[i] : (t->md.dims[i] + 31) / 32 * 32;
    }
  });
}

int32_t gnnv_trainer_dw16(const gnnv_trainer* t) { return t && t->dw16 ? 1 : 0; }
int32_t gnnv_trainer_fwd16(const gnnv_trainer* t) { return t && t->fwd16 ? 1 : 0; }
int32_t gnnv_trainer_tail16(const gnnv_trainer* t) { return t && t->tail16 ? 1 : 0; }
int32_t gnnv_trainer_last_rows(const gnnv_trainer* t) { return t && t->last_rows ? 1 : 0; }

gnnv_status gnnv_trainer_aggregate16(gnnv_trainer* t, int32_t i, const void** d_A16, int32_t* ld) {
  return guarded([&] {
    GNNV_REQUIRE(t && d_A16 && ld && i >= 1 && i <= t->md.L, GNNV_ERR_PARAM, "trainer_aggregate16: bad args");
    const void* p = i == 1 ? t->A16[t->cur] : t->A16h[i];
    *d_A16 = p;
    *ld = !p ? 0 : i == 1 ? t->ld16x : t->ld16[i - 1];
  });
}

gnnv_status gnnv_trainer_dw16_operands(gnnv_trainer* t, const void** d_X16, const void** d_A16, int32_t* ld) {
  return guarded([&] {
    GNNV_REQUIRE(t && d_X16 && d_A16 && ld, GNNV_ERR_PARAM, "trainer_dw16_operands: null");
    *d_X16 = t->X16[t->cur];
    *d_A16 = t->A16[t->cur];
    *ld = t->dw16 ? t->ld16x : 0;
  });
}

gnnv_status gnnv_trainer_set_locality(gnnv_trainer* t, double bias) {
  return guarded([&] {
    GNNV_REQUIRE(t, GNNV_ERR_PARAM, "trainer_set_locality: null");
    GNNV_REQUIRE(!t->pending, GNNV_ERR_STATE, "trainer_set_locality: a prefetched batch is pending");
    for (int k = 0; k < 2; ++k) {
      if (!t->bb[k]) continue;
      gnnv_status st = gnnv_blocks_set_locality(t->bb[k], t->c, bias);
      if (st != GNNV_OK) throw Error{st, get_error()};
    }
    t->loc_bias = bias;
  });
}

gnnv_status gnnv_trainer_timeline(gnnv_trainer* t, int32_t on) {
  return guarded([&] {
    GNNV_REQUIRE(t, GNNV_ERR_PARAM, "trainer_timeline: null");
    GNNV_TRY_CUDA(cudaDeviceSynchronize());
    t->tl.clear();
    t->tl_side.clear();
    t->tl.on = on != 0;
    t->tl_side.on = on != 0;
  });
}

gnnv_status gnnv_trainer_timeline_read(gnnv_trainer* t, gnnv_segment* out, int32_t cap, int32_t* n_out) {
  return guarded([&] {
    GNNV_REQUIRE(t && n_out && (out || cap == 0), GNNV_ERR_PARAM, "trainer_timeline_read: null");
    GNNV_TRY_CUDA(cudaDeviceSynchronize());
    std::vector<gnnv_segment> segs;
    // main-stream segments, then the prefetch stream's (pf_*): each timeline
    // is a chain of consecutive marks on its own stream
    for (Timeline* tlp : {&t->tl, &t->tl_side}) {
      auto& m = tlp->marks;
      for (size_t j = 0; j + 1 < m.size(); ++j) {
        if (m[j].first == "end") continue;
        float ms = 0.f;
        GNNV_TRY_CUDA(cudaEventElapsedTime(&ms, m[j].second, m[j + 1].second));
        size_t k = 0;
        for (; k < segs.size(); ++k)
          if (m[j].first == segs[k].name) break;
        if (k == segs.size()) {
          gnnv_segment sg{};
          strncpy(sg.name, m[j].first.c_str(), sizeof(sg.name) - 1);
          segs.push_back(sg);
        }
        segs[k].total_ms += ms;
        segs[k].count += 1;
      }
      tlp->clear();
    }
    *n_out = (int32_t)segs.size();
    for (int32_t i = 0; i < cap && i < (int32_t)segs.size(); ++i) out[i] = segs[i];
  });
}

gnnv_status gnnv_trainer_read_loss(gnnv_trainer* t, float* loss_out, gnnv_stream stream) {
  return guarded([&] {
    GNNV_REQUIRE(t && loss_out, GNNV_ERR_PARAM, "read_loss: null");
    cudaStream_t s = (cudaStream_t)stream;
    const int L = t->md.L;
    GNNV_TRY_CUDA(cudaMemcpyAsync(t->h_out, t->d_grads + t->nparams, sizeof(float), cudaMemcpyDeviceToHost, s));
    GNNV_TRY_CUDA(cudaMemcpyAsync(t->h_err, t->b->d_sizes + 2 * L + 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    GNNV_TRY_CUDA(cudaStreamSynchronize(s));
    *loss_out = t->h_out[0];
    if (t->h_err[0]) {
      GNNV_TRY_CUDA(cudaMemsetAsync(t->b->d_sizes + 2 * L + 1, 0, sizeof(int32_t), s));
      throw Error{GNNV_ERR_PARAM, "step: repeated or out-of-range seed id"};
    }
  });
}

gnnv_status gnnv_trainer_loss_async(gnnv_trainer* t, int64_t* ticket, gnnv_stream stream) {
  return guarded([&] {
    GNNV_REQUIRE(t && ticket, GNNV_ERR_PARAM, "loss_async: null");
    cudaStream_t s = (cudaStream_t)stream;
    const int L = t->md.L;
    (void)L;
    GNNV_REQUIRE(t->steps_done > 0, GNNV_ERR_STATE, "loss_async: no step has run");
    // the last step's SGD kernel writes its loss into the mapped ring slot;
    // an event marks when that write is complete (no copy on the stream)
    const int64_t step = t->steps_done - 1;
    const int k = (int)(step % gnnv_trainer::kLossRing);
    GNNV_TRY_CUDA(cudaEventRecord(t->ev_loss[k], s));
    *ticket = step;
    t->loss_tickets = t->steps_done;
  });
}

gnnv_status gnnv_trainer_loss_result(gnnv_trainer* t, int64_t ticket, float* loss_out) {
  return guarded([&] {
    GNNV_REQUIRE(t && loss_out, GNNV_ERR_PARAM, "loss_result: null");
    GNNV_REQUIRE(ticket >= 0 && ticket < t->loss_tickets && ticket >= t->steps_done - gnnv_trainer::kLossRing,
                 GNNV_ERR_STATE, "loss_result: ticket not issued or already recycled (ring of 8)");
    const int k = (int)(ticket % gnnv_trainer::kLossRing);
    GNNV_TRY_CUDA(cudaEventSynchronize(t->ev_loss[k]));
    *loss_out = ((volatile float*)t->h_lossr)[k];
    GNNV_REQUIRE(!((volatile int32_t*)t->h_errr)[k], GNNV_ERR_PARAM, "step: repeated or out-of-range seed id");
  });
}

gnnv_status gnnv_trainer_stats(gnnv_trainer* t, int64_t* host_stats4) {
  return guarded([&] {
    GNNV_REQUIRE(t && host_stats4, GNNV_ERR_PARAM, "trainer_stats: null");
    GNNV_TRY_CUDA(cudaDeviceSynchronize());
    GNNV_TRY_CUDA(cudaMemcpy(host_stats4, t->d_stats, 4 * sizeof(int64_t), cudaMemcpyDeviceToHost));
  });
}


static void select_buffers(gnnv_trainer* t, int k) {
  t->cur = k;
  t->b = t->bb[k];
  t->H[0] = t->X[k];
  t->d_seeds = t->d_seedsb[k];
  t->h_seeds = t->h_seedsb[k];
  t->d_stats = t->d_statsb[k];
  if (t->A1b[k]) t->A[1] = t->A1b[k];
}

// Stage host seeds (validated) or take device seeds; returns device pointer.
static const int32_t* stage_seeds(gnnv_trainer* t, int k, const int32_t* seeds, int32_t n_seeds, int32_t on_host,
                                  cudaStream_t s, Timeline* tl) {
  if (!on_host) return seeds;
  for (int i = 0; i < n_seeds; ++i)
    GNNV_REQUIRE(seeds[i] >= 0 && seeds[i] < t->g->n, GNNV_ERR_PARAM, "step: seed id outside [0, N)");
  // the staging buffer may still feed the previous copy out of it; wait for
  // that copy only (not for the stream), so a prefetch never blocks the host
  // on the step in flight
  if (t->h2d_used[k]) GNNV_TRY_CUDA(cudaEventSynchronize(t->ev_h2d[k]));
  memcpy(t->h_seedsb[k], seeds, n_seeds * sizeof(int32_t));
  if (tl) tl->mark(s, "h2d_seeds");
  GNNV_TRY_CUDA(
      cudaMemcpyAsync(t->d_seedsb[k], t->h_seedsb[k], n_seeds * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  GNNV_TRY_CUDA(cudaEventRecord(t->ev_h2d[k], s));
  t->h2d_used[k] = true;
  return t->d_seedsb[k];
}

gnnv_status gnnv_trainer_prefetch(gnnv_trainer* t, const int32_t* seeds, int32_t n_seeds, int32_t seeds_on_host,
                                  uint64_t rng_seed, gnnv_stream stream) {
  return guarded([&] {
    GNNV_REQUIRE(t && seeds, GNNV_ERR_PARAM, "prefetch: null");
    GNNV_REQUIRE(!t->pending, GNNV_ERR_STATE, "prefetch: a prefetched batch is already pending");
    GNNV_REQUIRE(n_seeds >= 1 && n_seeds <= t->md.max_seeds, GNNV_ERR_PARAM,
                 "prefetch: n_seeds must be in [1, max_seeds]");
    gnnv_graph* g = t->g;
    const int k = t->cur ^ 1;
    if (!t->bb[k]) {  // first use: the second buffer set
      GNNV_TRY_CUDA(cudaDeviceSynchronize());
      gnnv_status st = gnnv_blocks_create(g, t->md.max_seeds, t->md.fanouts, t->md.L, &t->bb[k]);
      if (st != GNNV_OK) throw Error{st, get_error()};
      st = gnnv_blocks_set_locality(t->bb[k], t->c, t->loc_bias);
      if (st != GNNV_OK) throw Error{st, get_error()};
      if (t->l2push)
        for (int i = 1; i <= t->md.L - 2; ++i) blocks_enable_owner_rows(t->bb[k], t->md.L - i - 1);
      if (t->lastuse) blocks_enable_lastuse(t->bb[k]);
      const int64_t xrows = t->x_rows || t->fwd16 ? 1 : t->bb[k]->max_n[t->x_fused ? t->md.L - 1 : t->md.L];
      t->X[k] = (float*)dmalloc((size_t)xrows * g->stride * sizeof(float), "X (prefetch)");
      if (t->x_fused)
        t->rowidx[k] = (int32_t*)dmalloc(t->bb[k]->max_n[t->md.L] * sizeof(int32_t), "cache rows of F_L (prefetch)");
      t->d_seedsb[k] = (int32_t*)dmalloc(t->md.max_seeds * sizeof(int32_t), "seeds (prefetch)");
      GNNV_TRY_CUDA(cudaMallocHost(&t->h_seedsb[k], t->md.max_seeds * sizeof(int32_t)));
      t->d_statsb[k] = (int64_t*)dmalloc(4 * sizeof(int64_t), "gather stats (prefetch)");
      if (t->fwd16) blocks_set_rowidx(t->bb[k], t->c->d_slot, t->rowidx[k], t->d_statsb[k]);
      if (t->last_rows) blocks_set_last_rows(t->bb[k], t->c->d_slot);
      if (t->dw16) alloc_dw16(t, k, t->bb[k]);
      if (t->pf_agg)
        t->A1b[k] = (float*)dmalloc((size_t)t->bb[k]->max_n[t->md.L - 1] * row_stride(t->md.dims[0]) * sizeof(float),
                                    "layer-1 aggregates (prefetch)");
      // the layer backward's scratch arena, sized like the first buffer set's
      // (grown by its steps so far): growing it at this set's first step
      // would put a device synchronisation and a cudaMalloc inside the step
      if (t->bb[k ^ 1] && t->bb[k ^ 1]->scratch_bytes)
        t->bb[k]->ensure_scratch(t->bb[k ^ 1]->scratch_bytes, (cudaStream_t)stream);
      if (!t->side) t->side = make_side_stream();
    }
    cudaStream_t s = (cudaStream_t)stream;
    // order after the step that last computed on buffer set k and, for
    // device seeds, after the work already enqueued on the caller's stream
    // (pass the stream that produced the seeds, not the step stream, to let
    // the prefetch overlap the step in flight).  Host seeds carry no device
    // dependency.
    if (!seeds_on_host) {
      GNNV_TRY_CUDA(cudaEventRecord(t->ev_in, s));
      GNNV_TRY_CUDA(cudaStreamWaitEvent(t->side, t->ev_in, 0));
    }
    GNNV_TRY_CUDA(cudaStreamWaitEvent(t->side, t->ev_free[k], 0));
    Timeline* tl = t->tl.on ? &t->tl_side : nullptr;
    const int32_t* d_seeds = stage_seeds(t, k, seeds, n_seeds, seeds_on_host, t->side, tl);
    if (tl) tl->mark(t->side, "pf_sample");
    // the overlapped batch launches without programmatic dependent launch
    // (its waiting CTAs would park on SMs the concurrent step needs)
    struct PrefetchLaunch {
      PrefetchLaunch() {
        set_pdl(false);
        set_grid_cap(env_int("GNNV_PF_CAP", 0));
      }
      ~PrefetchLaunch() {
        set_pdl(true);
        set_grid_cap(0);
      }
    } pf_launch;
    launch_sample(g, t->bb[k], d_seeds, n_seeds, rng_seed, t->side);
    t->bb[k]->sampled = true;
    if (!t->fwd16) GNNV_TRY_CUDA(cudaMemsetAsync(t->d_statsb[k], 0, 4 * sizeof(int64_t), t->side));
    if (tl) tl->mark(t->side, "pf_gather");
    if (t->c->dynamic && t->cache_pending) GNNV_TRY_CUDA(cudaStreamWaitEvent(t->side, t->ev_cache, 0));
    // with fwd16 the layer-1 aggregation copies X's bf16 dst prefix itself
    // and the sampler's last kernel wrote every F_L row's cache row and the
    // counters: no gather pass
    if (!t->fwd16)
      launch_gather(t->c, t->bb[k], t->X[k], t->d_statsb[k], t->side, t->rowidx[k], !t->x_rows, t->X16[k], t->ld16x);
    if (t->c->dynamic) {  // NEXT-3 admission
      if (tl) tl->mark(t->side, "pf_replace");
      launch_cache_update(t->c, t->bb[k], t->X[k], t->side);
      GNNV_TRY_CUDA(cudaEventRecord(t->ev_cache, t->side));
      t->cache_pending = true;
    }
    if (t->pf_agg) {  // layer 1's aggregation of the prefetched batch (no weight involved)
      if (tl) tl->mark(t->side, "pf_spmm_fwd.l1");
      const int L = t->md.L, h = L - 1;
      gnnv_blocks* bk = t->bb[k];
      if (t->table16)
        launch_spmm_fwd_h16(bk->d_indptr[h], bk->d_indices[h], bk->d_sizes + h, bk->max_n[h], t->c->d_table16,
                            t->c->table16_ld, t->fwd16 ? nullptr : t->A1b[k], row_stride(t->md.dims[0]),
                            t->md.dims[0], t->md.kind, t->md.aggr, t->side, t->rowidx[k], t->A16[k], t->ld16x,
                            t->fwd16 ? t->X16[k] : nullptr, t->last_rows);
      else
        launch_spmm_fwd(bk->d_indptr[h], bk->d_indices[h], bk->d_sizes + h, bk->max_n[h],
                        t->x_fused ? t->table : t->X[k], g->stride, t->A1b[k], row_stride(t->md.dims[0]),
                        t->md.dims[0], t->md.kind, t->md.aggr, t->side, t->x_fused ? t->rowidx[k] : nullptr,
                        bk->d_lastv);
    }

    if (tl) tl->mark(t->side, "end");
    GNNV_TRY_CUDA(cudaEventRecord(t->ev_ready[k], t->side));
    t->pending = true;
    t->pend_n = n_seeds;
    t->pend_rng = rng_seed;
  });
}

gnnv_status gnnv_trainer_join_prefetch(gnnv_trainer* t, gnnv_stream stream) {
  return guarded([&] {
    GNNV_REQUIRE(t, GNNV_ERR_PARAM, "join_prefetch: null");
    if (t->pending) GNNV_TRY_CUDA(cudaStreamWaitEvent((cudaStream_t)stream, t->ev_ready[t->cur ^ 1], 0));
  });
}

gnnv_status gnnv_step(gnnv_trainer* t, const int32_t* seeds, int32_t n_seeds, int32_t seeds_on_host, int32_t n_global,
                      uint64_t rng_seed, float lr, float* loss_out, gnnv_step_timing* tm, gnnv_stream stream) {
  return guarded([&] {
    GNNV_REQUIRE(t && seeds, GNNV_ERR_PARAM, "step: null");
    GNNV_REQUIRE(n_seeds >= 1 && n_seeds <= t->md.max_seeds, GNNV_ERR_PARAM, "step: n_seeds must be in [1, max_seeds]");
    GNNV_REQUIRE(n_global >= n_seeds, GNNV_ERR_PARAM, "step: n_global must be >= n_seeds");
    cudaStream_t s = (cudaStream_t)stream;
    gnnv_graph* g = t->g;
    const int L = t->md.L;
    Timeline* tl = t->tl.on ? &t->tl : nullptr;
    // Programmatic dependent launch only for a serial step: with the Eq.4
    // prefetch in flight the next kernel's early-resident CTAs take SM slots
    // the overlapped batch needs (measured: 1.49 vs 1.41 ms per products step)
    struct StepPdl {
      explicit StepPdl(bool on) { set_pdl(on); }
      ~StepPdl() { set_pdl(true); }
    } step_pdl(!t->pending);
    if (tm) GNNV_TRY_CUDA(cudaEventRecord(t->ev[0], s));
    bool agg1_ready = false;
    if (t->pending) {
      // the batch was sampled and gathered by gnnv_trainer_prefetch
      GNNV_REQUIRE(n_seeds == t->pend_n && rng_seed == t->pend_rng, GNNV_ERR_STATE,
                   "step: seeds/rng_seed differ from the pending prefetch");
      select_buffers(t, t->cur ^ 1);
      t->pending = false;
      agg1_ready = t->pf_agg;
      if (tl) tl->mark(s, "wait_prefetch");
      GNNV_TRY_CUDA(cudaStreamWaitEvent(s, t->ev_ready[t->cur], 0));
      if (tm) GNNV_TRY_CUDA(cudaEventRecord(t->ev[1], s));
      if (tm) GNNV_TRY_CUDA(cudaEventRecord(t->ev[2], s));
    } else {
      const int32_t* d_seeds = stage_seeds(t, t->cur, seeds, n_seeds, seeds_on_host, s, tl);
      if (tl) tl->mark(s, "sample");
      launch_sample(g, t->b, d_seeds, n_seeds, rng_seed, s);
      t->b->sampled = true;
      if (!t->fwd16) GNNV_TRY_CUDA(cudaMemsetAsync(t->d_stats, 0, 4 * sizeof(int64_t), s));
      if (tm) GNNV_TRY_CUDA(cudaEventRecord(t->ev[1], s));
      if (tl) tl->mark(s, "gather");
      if (t->c->dynamic && t->cache_pending) GNNV_TRY_CUDA(cudaStreamWaitEvent(s, t->ev_cache, 0));
      if (!t->fwd16)
        launch_gather(t->c, t->b, t->H[0], t->d_stats, s, t->rowidx[t->cur], !t->x_rows, t->X16[t->cur], t->ld16x);
      if (t->c->dynamic) {  // NEXT-3 admission (Eq.5's t_replace)
        if (tl) tl->mark(s, "replace");
        launch_cache_update(t->c, t->b, t->H[0], s);
        GNNV_TRY_CUDA(cudaEventRecord(t->ev_cache, s));
        t->cache_pending = true;
      }
      if (tm) GNNV_TRY_CUDA(cudaEventRecord(t->ev[2], s));
    }
    gnnv_blocks* b = t->b;
    const XRows xr{t->table, t->rowidx[t->cur], g->n};
    const XRows* xr1 = t->x_rows ? &xr : nullptr;
    for (int i = 1; i <= L; ++i) {
      if (t->tail && i == L) break;  // the fused output layer below
      const gnnv_layer_desc ld = layer_desc(t, i);
      FwdPush push{};
      const bool do_push = t->l2push && i <= L - 2;
      if (do_push) {
        const int hn = L - i - 1;  // the next layer's block
        if (tl) tl->mark(s, "zero_a.l" + std::to_string(i + 1));
        launch_zero_rows(t->A[i + 1], b->d_sizes + hn, b->max_n[hn], row_stride(t->md.dims[i]), s);
        push = FwdPush{b->d_colptr[hn], b->d_csc[hn], b->d_indptr[hn], t->A[i + 1], row_stride(t->md.dims[i]),
                       t->md.aggr == GNNV_AGGR_MEAN, b->d_sizes + hn, b->d_owner_row[hn]};
      }
      Bf16Io io{};
      if (i == 1 && t->table16) {
        io.src16 = t->c->d_table16;
        io.src16_ld = t->c->table16_ld;
        io.src16_rows = t->rowidx[t->cur];
        io.a16 = t->A16[t->cur];
        io.a16_ld = t->ld16x;
        if (t->fwd16) {
          io.x16 = t->X16[t->cur];
          io.x16_out = t->X16[t->cur];  // written by the aggregation (self rows + ones column)
          io.rows_direct = t->last_rows;
        }
      }
      if (t->bf16act) {
        if (i <= L - 2) {  // this layer's output: a bf16 copy, fp32 rows for the next dst prefix
          io.y16 = t->H16[i];
          io.ld16 = t->ld16[i];
          io.keep_rows = (i == 1 && !t->h1_fp32) ? t->d_zero : b->d_sizes + (L - i - 1);
        }
        if (i >= 2 && i - 1 <= L - 2) {  // aggregate the previous layer's bf16 copy
          io.src16 = t->H16[i - 1];
          io.src16_ld = t->ld16[i - 1];
          if (t->hid16 && t->A16h[i]) {  // and run the GEMM over [H16 dst prefix | A16]
            io.x16 = t->H16[i - 1];
            io.a16 = t->A16h[i];
            io.a16_ld = t->ld16[i - 1];
            io.keep_a32 = true;  // the layer's TF32 dW reads the fp32 A
          }
        }
      }
      layer_fwd_impl(b, i, &ld, t->H[i - 1], t->d_params + t->w_off[i - 1], t->d_params + t->b_off[i - 1], t->H[i],
                     t->A[i], s, tl, t->mbits[i], t->table, i == 1 ? t->rowidx[t->cur] : nullptr,
                     i == 1 ? xr1 : nullptr, do_push ? &push : nullptr,
                     (t->l2push && i >= 2 && i <= L - 1) || (i == 1 && agg1_ready),
                     (t->bf16act || t->table16) ? &io : nullptr);
    }
    if (tm) GNNV_TRY_CUDA(cudaEventRecord(t->ev[3], s));
    float* d_loss = t->d_grads + t->nparams;
    if (t->tail) {
      // output layer forward + loss + backward (tail.cu); the per-phase
      // timing puts all of it in "loss"
      TailArgs a{};
      a.indptr = b->d_indptr[0];
      a.indices = b->d_indices[0];
      a.own = b->d_own[0];
      a.d_ndst = b->d_sizes;
      a.max_dst = b->max_n[0];
      a.H = t->H[L - 1];
      a.ldh = t->Hs[L - 1];
      a.hbits = t->mbits[L - 1];
      a.hbits_ld = mask_words(t->md.dims[L - 1]);
      a.W = t->d_params + t->w_off[L - 1];
      a.bias = t->d_params + t->b_off[L - 1];
      a.d = t->md.dims[L - 1];
      a.C = t->md.dims[L];
      a.aggr = t->md.aggr;
      a.A = t->A[L];
      a.lda = row_stride(t->md.dims[L - 1]);
      a.Z = t->H[L];
      a.dZ = t->G[L];
      a.ldz = t->Hs[L];
      a.F = b->d_F;
      a.labels = g->d_labels;
      a.n_global = n_global;
      a.dH = t->G[L - 1];
      a.ldg = t->Hs[L - 1];
      if (t->tail16) {
        a.dH16 = t->G16h[L - 1];
        a.db_part = t->tail_dbp;
      }
      a.dA = t->tail_dA;
      a.loss_partial = t->loss_partial;
      a.part = t->tail_part;
      a.zero = t->d_grads;  // layers 1..L-1: [0, w_off[L-1])
      a.zero_n = t->w_off[L - 1];
      a.dW = t->d_grads + t->w_off[L - 1];
      a.db = t->d_grads + t->b_off[L - 1];
      a.d_loss = d_loss;
      launch_tail(a, s, tl, ".l" + std::to_string(L));
    } else {
      if (tl) tl->mark(s, "loss");
      launch_ce_loss(t->H[L], t->Hs[L], t->md.dims[L], b->d_sizes, b->d_F, g->d_labels, n_global, d_loss, t->G[L],
                     t->loss_partial, t->loss_counter, b->max_n[0], s);
    }
    if (tm) GNNV_TRY_CUDA(cudaEventRecord(t->ev[4], s));
    for (int i = L; i >= 1; --i) {
      if (t->tail && i == L) continue;
      const gnnv_layer_desc ld = layer_desc(t, i);
      Bf16Io io{};
      if (t->bf16act) {
        if (i - 1 >= 1 && i - 1 <= L - 2) {  // dL/dH^{i-1} produced as bf16
          io.gsrc16 = t->G16[i - 1];
          io.gsrc16_ld = t->ld16[i - 1];
        }
        if (i <= L - 2) {  // this layer's G read as bf16
          io.gdst16 = t->G16[i];
          io.gdst16_ld = t->ld16[i];
        }
        if (i == 1 && t->dw16) {
          io.x16 = t->X16[t->cur];
          io.a16 = t->A16[t->cur];
          io.a16_ld = t->ld16x;
        }
        if (i >= 2 && t->G16h[i]) {  // hidden layer: dW over bf16 (reading Q34)
          io.x16 = t->H16[i - 1];
          io.a16 = t->A16h[i];
          io.a16_ld = t->ld16[i - 1];
          io.g16_out = t->G16h[i];
          io.g16_ld = (t->md.dims[i] + 31) / 32 * 32;
          if (t->tail16 && i == L - 1) {  // G came as bf16 from the fused output layer
            io.g16_out = nullptr;
            io.g16_in = t->G16h[i];
            io.g16_ld = t->Hs[i];
            io.dbp = t->tail_dbp;
            io.ndbp = tail_db_parts(b->max_n[0]);
          }
        }
      }
      layer_bwd_impl(b, i, &ld, t->G[i], t->H[i], t->H[i - 1], t->A[i], t->d_params + t->w_off[i - 1],
                     i > 1 ? t->G[i - 1] : nullptr, t->d_grads + t->w_off[i - 1], t->d_grads + t->b_off[i - 1], s, tl,
                     t->mbits[i], t->mbits[i] != nullptr, t->mbits[i - 1], mask_words(t->md.dims[i - 1]),
                     i == 1 ? xr1 : nullptr, t->tail, t->bf16act ? &io : nullptr);
    }
    if (tm) GNNV_TRY_CUDA(cudaEventRecord(t->ev[5], s));
    if (tl) tl->mark(s, "allreduce");
    if (t->comm && t->comm->world > 1) {
      gnnv_status st = gnnv_allreduce_sum(t->comm, t->d_grads, t->nparams + 1, s);
      if (st != GNNV_OK) throw Error{st, get_error()};
    }
    if (tm) GNNV_TRY_CUDA(cudaEventRecord(t->ev[6], s));
    if (tl) tl->mark(s, "sgd");
    {
      const int slot = (int)(t->steps_done % gnnv_trainer::kLossRing);
      launch_sgd(t->d_params, t->d_grads, t->nparams, lr, s, t->d_lossr + slot, t->d_errr + slot,
                 b->d_sizes + 2 * L + 1);
      ++t->steps_done;
    }
    if (tl) tl->mark(s, "end");
    GNNV_TRY_CUDA(cudaEventRecord(t->ev_free[t->cur], s));  // buffer set may be refilled
    if (tm) GNNV_TRY_CUDA(cudaEventRecord(t->ev[7], s));
    if (loss_out || tm) {
      GNNV_TRY_CUDA(cudaMemcpyAsync(t->h_out, d_loss, sizeof(float), cudaMemcpyDeviceToHost, s));
      GNNV_TRY_CUDA(cudaMemcpyAsync(t->h_err, b->d_sizes + 2 * L + 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      GNNV_TRY_CUDA(cudaStreamSynchronize(s));
      if (loss_out) *loss_out = t->h_out[0];
      if (t->h_err[0]) {
        GNNV_TRY_CUDA(cudaMemsetAsync(b->d_sizes + 2 * L + 1, 0, sizeof(int32_t), s));
        throw Error{GNNV_ERR_PARAM, "step: repeated or out-of-range seed id"};
      }
    }
    if (tm) {
      float ms[7];
      for (int i = 0; i < 7; ++i) GNNV_TRY_CUDA(cudaEventElapsedTime(&ms[i], t->ev[i], t->ev[i + 1]));
      tm->sample_ms = ms[0];
      tm->gather_ms = ms[1];
      tm->fwd_ms = ms[2];
      tm->loss_ms = ms[3];
      tm->bwd_ms = ms[4];
      tm->allreduce_ms = ms[5];
      tm->update_ms = ms[6];
      GNNV_TRY_CUDA(cudaEventElapsedTime(&tm->total_ms, t->ev[0], t->ev[7]));
    }
  });
}

}  // extern "C"
