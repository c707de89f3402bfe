// GNN layer forward/backward orchestration, loss, SGD (C-ABI entry points).
//
// Paper: Eq.1; Algorithm 1 lines 4-8; SPEC S:320,
// S:322 (combine = linear + ReLU except the last layer; mean/sum over
// neighbours), S:332 (softmax cross-entropy + plain gradient descent).
// Layer i in 1..L runs on block b_{L-i} (dst = F_{L-i}, src = F_{L-i+1}).
#include <cuda_bf16.h>

#include "common.cuh"

namespace gnnv {

__global__ void k_relu_mask(const float* __restrict__ G, const float* __restrict__ H, float* __restrict__ Gp, int ld,
                            const int32_t* d_M) {
  GNNV_PDL_ENTRY();
  const int64_t total = (int64_t)(*d_M) * (ld >> 2);
  const float4* G4 = reinterpret_cast<const float4*>(G);
  const float4* H4 = reinterpret_cast<const float4*>(H);
  float4* P4 = reinterpret_cast<float4*>(Gp);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const float4 g = __ldg(G4 + t), h = __ldg(H4 + t);
    P4[t] = make_float4(h.x > 0.f ? g.x : 0.f, h.y > 0.f ? g.y : 0.f, h.z > 0.f ? g.z : 0.f, h.w > 0.f ? g.w : 0.f);
  }
}

void launch_relu_mask(const float* G, const float* H, float* Gp, int32_t ld, int32_t, const int32_t* d_M,
                      int64_t max_M, cudaStream_t s) {
  const int64_t total = std::max<int64_t>(max_M, 1) * (ld / 4);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), (int64_t)num_sms() * 8));
  launch_k(k_relu_mask, grid, 256, 0, s, G, H, Gp, ld, d_M);
  GNNV_CHECK_LAUNCH();
}

// bits[m*bits_ld + n/32] bit n%32 = (H[m][n] > 0): one warp per (row, word)
__global__ void k_relu_bits(const float* __restrict__ H, int32_t ldh, int32_t N, const int32_t* d_M, uint32_t* bits,
                            int32_t bits_ld) {
  GNNV_PDL_ENTRY();
  const int64_t M = *d_M;
  const int lane = threadIdx.x & 31;
  const int64_t total = M * bits_ld;
  for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < total;
       t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t m = t / bits_ld;
    const int wd = (int)(t - m * bits_ld);
    const int n = wd * 32 + lane;
    const bool on = n < N && H[m * ldh + n] > 0.f;
    const uint32_t w = __ballot_sync(0xffffffffu, on);
    if (lane == 0) bits[t] = w;
  }
}

void launch_relu_bits(const float* H, int32_t ldh, int32_t N, const int32_t* d_M, int64_t max_M, uint32_t* bits,
                      int32_t bits_ld, cudaStream_t s) {
  const int64_t warps = std::max<int64_t>(max_M, 1) * bits_ld;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(warps, 8), (int64_t)num_sms() * 16));
  launch_k(k_relu_bits, grid, 256, 0, s, H, ldh, N, d_M, bits, bits_ld);
  GNNV_CHECK_LAUNCH();
}

// G' = G * 1[H > 0] (if H) written to Gp, plus per-block column sums of G'
// (db).  Fixed grid, contiguous row ranges, fixed in-block order: the
// bias gradient is deterministic.
constexpr int kColBlocks = 296;
__global__ void __launch_bounds__(256) k_mask_colsum(const float* __restrict__ G, const float* __restrict__ H,
                                                     float* __restrict__ Gp, int ld, const int32_t* d_M,
                                                     float* __restrict__ partial,
                                                     __nv_bfloat16* __restrict__ G16, int ld16) {
  GNNV_PDL_ENTRY();
  __shared__ float4 s_acc[256];
  const int M = *d_M;
  const int ld4 = ld >> 2;
  const int groups = max(1, (int)blockDim.x / ld4);
  const int rg = threadIdx.x / ld4, c4 = threadIdx.x - rg * ld4;
  const int per = (M + gridDim.x - 1) / gridDim.x;
  const int r0 = min(M, (int)blockIdx.x * per), r1 = min(M, r0 + per);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (rg < groups && c4 < ld4) {
    const float4* G4 = reinterpret_cast<const float4*>(G);
    const float4* H4 = reinterpret_cast<const float4*>(H);
    float4* P4 = reinterpret_cast<float4*>(Gp);
    for (int r = r0 + rg; r < r1; r += groups) {
      const int64_t i = (int64_t)r * ld4 + c4;
      float4 g = __ldg(G4 + i);
      if (H) {
        const float4 h = __ldg(H4 + i);
        g = make_float4(h.x > 0.f ? g.x : 0.f, h.y > 0.f ? g.y : 0.f, h.z > 0.f ? g.z : 0.f, h.w > 0.f ? g.w : 0.f);
        P4[i] = g;
      }
      if (G16) {  // the bf16 copy a kind::f16 dW reads
        const __nv_bfloat162 lo = __floats2bfloat162_rn(g.x, g.y), hi = __floats2bfloat162_rn(g.z, g.w);
        reinterpret_cast<uint2*>(G16)[((int64_t)r * ld16 >> 2) + c4] =
            make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
      }
      acc.x += g.x;
      acc.y += g.y;
      acc.z += g.z;
      acc.w += g.w;
    }
  }
  s_acc[threadIdx.x] = acc;
  __syncthreads();
  if (rg == 0 && c4 < ld4) {
    float4 t = s_acc[c4];
    for (int q = 1; q < groups; ++q) {
      const float4 u = s_acc[q * ld4 + c4];
      t.x += u.x;
      t.y += u.y;
      t.z += u.z;
      t.w += u.w;
    }
    reinterpret_cast<float4*>(partial)[(int64_t)blockIdx.x * ld4 + c4] = t;
  }
}

// out[n] = sum_b partial[b*ld + n], n < N: 32 columns x 8 part-groups per
// block, fixed order (deterministic); block (32, 8), grid ceil(N/32).
__global__ void __launch_bounds__(256) k_colsum_reduce(const float* __restrict__ partial, int blocks, int ld, int N,
                                                       float* db) {
  GNNV_PDL_ENTRY();
  __shared__ float s[8][33];
  const int n = blockIdx.x * 32 + threadIdx.x;
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;  // 4 loads in flight, fixed order
  if (n < N) {
    int b = threadIdx.y;
    for (; b + 24 < blocks; b += 32) {
      a0 += partial[(int64_t)b * ld + n];
      a1 += partial[(int64_t)(b + 8) * ld + n];
      a2 += partial[(int64_t)(b + 16) * ld + n];
      a3 += partial[(int64_t)(b + 24) * ld + n];
    }
    for (; b < blocks; b += 8) a0 += partial[(int64_t)b * ld + n];
  }
  s[threadIdx.y][threadIdx.x] = (a0 + a1) + (a2 + a3);
  __syncthreads();
  if (threadIdx.y == 0 && n < N) {
    float t = 0.f;
#pragma unroll
    for (int y = 0; y < 8; ++y) t += s[y][threadIdx.x];
    db[n] = t;
  }
}

void launch_colsum_reduce(const float* partial, int blocks, int ld, int N, float* out, cudaStream_t s) {
  launch_k(k_colsum_reduce, (N + 31) / 32, dim3(32, 8), 0, s, partial, blocks, ld, N, out);
  GNNV_CHECK_LAUNCH();
}

constexpr int kLossBlocks = 256;  // <= the trainer's 256 partials

// One warp per seed row; fixed grid => fixed summation order (deterministic).
__global__ void __launch_bounds__(256) k_ce_loss(const float* __restrict__ z, int ldz, int C,
                                                 const int32_t* d_rows, const int32_t* __restrict__ F,
                                                 const int32_t* __restrict__ labels, int n_global,
                                                 float* d_loss, float* __restrict__ dz, float* partial,
                                                 unsigned int* counter) {
  GNNV_PDL_ENTRY();
  __shared__ float s_w[8];
  __shared__ bool s_last;
  const int n = *d_rows;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const float inv = 1.f / (float)n_global;
  float wsum = 0.f;
  for (int row = blockIdx.x * 8 + wid; row < n; row += gridDim.x * 8) {
    const float* zr = z + (int64_t)row * ldz;
    float m = -INFINITY;
    for (int c = lane; c < C; c += 32) m = fmaxf(m, zr[c]);
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float se = 0.f;
    for (int c = lane; c < C; c += 32) se += expf(zr[c] - m);
#pragma unroll
    for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
    const int y = labels[F[row]];
    const float lse = m + logf(se);
    if (lane == 0) wsum += (lse - zr[y]);
    float* dr = dz + (int64_t)row * ldz;
    for (int c = lane; c < ldz; c += 32) {
      float g = 0.f;
      if (c < C) g = (expf(zr[c] - m) / se - (c == y ? 1.f : 0.f)) * inv;
      dr[c] = g;
    }
  }
  if (lane == 0) s_w[wid] = wsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    float b = 0.f;
    for (int w = 0; w < 8; ++w) b += s_w[w];
    partial[blockIdx.x] = b;
    __threadfence();
    s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {  // block-uniform: the last block reduces the partials (fixed tree)
    __shared__ float s_r[256];
    __threadfence();
    float t = 0.f;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) t += ((volatile float*)partial)[i];
    s_r[threadIdx.x] = t;
    __syncthreads();
    for (int o = 128; o; o >>= 1) {
      if ((int)threadIdx.x < o) s_r[threadIdx.x] += s_r[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      *d_loss = s_r[0] * inv;
      *counter = 0;
    }
  }
}

void launch_ce_loss(const float* z, int32_t ldz, int32_t C, const int32_t* d_rows, const int32_t* d_F,
                    const int32_t* d_labels, int32_t n_global, float* d_loss, float* dz, float* partial,
                    unsigned int* counter, int64_t, cudaStream_t s) {
  launch_k(k_ce_loss, kLossBlocks, 256, 0, s, z, ldz, C, d_rows, d_F, d_labels, n_global, d_loss, dz, partial, counter);
  GNNV_CHECK_LAUNCH();
}

// p -= lr g; with `out_loss` (the trainer's mapped host ring slot) thread 0
// also publishes the step's all-reduced loss g[n] and the seed-error flag,
// so the host reads the step's result without a copy on the stream.
__global__ void k_sgd(float* __restrict__ p, const float* __restrict__ g, int64_t n, float lr, float* out_loss,
                      int32_t* out_err, const int32_t* err) {
  GNNV_PDL_ENTRY();
  const int32_t bad = err ? *err : 0;
  if (out_loss && blockIdx.x == 0 && threadIdx.x == 0) {
    *out_loss = g[n];
    *out_err = bad;
    __threadfence_system();
  }
  // a batch with an invalid seed (sample.cu k_init_seeds) is not applied:
  // the step reports GNNV_ERR_PARAM and the parameters stay as they were
  if (bad) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] -= lr * g[i];
}
void launch_sgd(float* p, const float* g, int64_t n, float lr, cudaStream_t s, float* out_loss, int32_t* out_err,
                const int32_t* err) {
  if (n <= 0) return;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), (int64_t)num_sms() * 4));
  launch_k(k_sgd, grid, 256, 0, s, p, g, n, lr, out_loss, out_err, err);
  GNNV_CHECK_LAUNCH();
}

static void check_layer(const gnnv_blocks* b, int32_t layer, const gnnv_layer_desc* ld) {
  GNNV_REQUIRE(b && ld, GNNV_ERR_PARAM, "layer: null");
  GNNV_REQUIRE(b->sampled, GNNV_ERR_STATE, "layer: gnnv_sample has not run on these blocks");
  GNNV_REQUIRE(layer >= 1 && layer <= b->L, GNNV_ERR_PARAM, "layer: index must be in [1, L]");
  GNNV_REQUIRE(ld->d_in >= 1 && ld->d_out >= 1, GNNV_ERR_PARAM, "layer: dims must be >= 1");
  GNNV_REQUIRE(ld->in_stride >= ld->d_in && ld->in_stride % 4 == 0, GNNV_ERR_PARAM,
               "layer: in_stride must be >= d_in and a multiple of 4");
  GNNV_REQUIRE(ld->kind == GNNV_KIND_SAGE || ld->kind == GNNV_KIND_GCN, GNNV_ERR_PARAM, "layer: kind");
  GNNV_REQUIRE(ld->aggr == GNNV_AGGR_MEAN || ld->aggr == GNNV_AGGR_SUM, GNNV_ERR_PARAM, "layer: aggr");
  GNNV_REQUIRE(ld->act == GNNV_ACT_NONE || ld->act == GNNV_ACT_RELU, GNNV_ERR_PARAM, "layer: act");
  GNNV_REQUIRE(ld->prec == GNNV_PREC_FP32 || ld->prec == GNNV_PREC_BF16 || ld->prec == GNNV_PREC_TF32, GNNV_ERR_PARAM,
               "layer: prec");
}

__global__ void k_zero_rows(float4* __restrict__ p, const int32_t* d_rows, int32_t ld4) {
  GNNV_PDL_ENTRY();
  const int64_t n = (int64_t)*d_rows * ld4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}
void launch_zero_rows(float* p, const int32_t* d_rows, int64_t max_rows, int32_t ld, cudaStream_t s) {
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(max_rows * (ld / 4), 256), num_sms() * 8));
  launch_k(k_zero_rows, grid, 256, 0, s, reinterpret_cast<float4*>(p), d_rows, ld / 4);
  GNNV_CHECK_LAUNCH();
}

void layer_fwd_impl(gnnv_blocks* b, int32_t layer, const gnnv_layer_desc* ld, const float* Hsrc, const float* W,
                    const float* bias, float* Hdst, float* A, cudaStream_t s, Timeline* tl, uint32_t* mask_bits,
                    const float* agg_table, const int32_t* rowidx, const XRows* xr, const FwdPush* push,
                    bool agg_ready, const Bf16Io* io) {
  const std::string sfx = ".l" + std::to_string(layer);
  const int h = b->L - layer;
  const int32_t* d_ndst = b->d_sizes + h;
  const int lda = row_stride(ld->d_in), ldo = row_stride(ld->d_out);
  // rowidx: the aggregation reads its source rows from the cache table
  // (rows of Hsrc beyond the dst prefix are not materialised).  agg_ready:
  // A was already accumulated by the previous layer's GEMM epilogue (the
  // trainer's fused L2 push)
  if (!agg_ready) {
    if (tl) tl->mark(s, "spmm_fwd" + sfx);
    if (io && io->src16)
      launch_spmm_fwd_h16(b->d_indptr[h], b->d_indices[h], d_ndst, b->max_n[h], io->src16, io->src16_ld,
                          io->x16 && io->a16 && !io->keep_a32 ? nullptr : A, lda, ld->d_in, ld->kind, ld->aggr, s, io->src16_rows,
                          io->a16, io->a16_ld, io->x16_out, io->rows_direct);
    else
      launch_spmm_fwd(b->d_indptr[h], b->d_indices[h], d_ndst, b->max_n[h], rowidx ? agg_table : Hsrc,
                      ld->in_stride, A, lda, ld->d_in, ld->kind, ld->aggr, s, rowidx,
                      h == b->L - 1 ? b->d_lastv : nullptr);
  }
  GemmFwdArgs g{};
  if (ld->kind == GNNV_KIND_SAGE) {
    g.X1 = xr ? xr->table : Hsrc;
    g.ld1 = ld->in_stride;
    g.X2 = A;
    g.ld2 = lda;
    if (xr) g.x1_rows = xr->rows, g.x1_table_rows = xr->table_rows;
  } else {
    g.X1 = A;
    g.ld1 = lda;
    g.X2 = nullptr;
    g.ld2 = 0;
  }
  if (io && io->x16 && io->a16 && ld->kind == GNNV_KIND_SAGE) {  // bf16 operand copies (reading Q33)
    g.X1_16 = io->x16;
    g.X2_16 = io->a16;
    g.ld16in = io->a16_ld;
  }
  g.K1 = ld->d_in;
  g.W = W;
  g.bias = bias;
  g.Y = Hdst;
  g.ldy = ldo;
  g.N = ld->d_out;
  g.d_M = d_ndst;
  g.max_M = b->max_n[h];
  g.relu = ld->act == GNNV_ACT_RELU;
  if (mask_bits && g.relu && ld->prec == GNNV_PREC_TF32) {
    g.mask_bits = mask_bits;
    g.mask_ld = mask_words(ld->d_out);
  }
  if (push) {
    g.push_colptr = push->colptr;
    g.push_dst = push->dst;
    g.push_indptr = push->indptr;
    g.push_out = push->out;
    g.push_ld = push->ld;
    g.push_mean = push->mean;
    g.keep_rows = push->keep_rows;
    g.push_owner = push->owner;
  }
  if (io && io->y16) {
    g.y16 = io->y16;
    g.ld16 = io->ld16;
    g.keep_rows = io->keep_rows;
  }
  if (tl) tl->mark(s, "gemm_fwd" + sfx);
  gemm_fwd(g, ld->prec, s);
}

void layer_bwd_impl(gnnv_blocks* b, int32_t layer, const gnnv_layer_desc* ld, const float* Gdst, const float* Hdst,
                    const float* Hsrc, const float* A, const float* W, float* Gsrc, float* dW, float* db,
                    cudaStream_t s, Timeline* tl, const uint32_t* mask_bits, bool g_masked,
                    const uint32_t* src_bits, int32_t src_bits_ld, const XRows* xr, bool grads_zeroed,
                    const Bf16Io* io) {
  const std::string sfx = ".l" + std::to_string(layer);
  const int h = b->L - layer;
  const int32_t* d_ndst = b->d_sizes + h;
  const int64_t max_dst = b->max_n[h];
  const int lda = row_stride(ld->d_in), ldo = row_stride(ld->d_out);
  const bool sage = ld->kind == GNNV_KIND_SAGE;
  const int rows = (sage ? 2 * ld->d_in : ld->d_in) + 1;
  int32_t splits = 1;
  const size_t part_f = gemm_dw_partial_floats(rows, ld->d_out, &splits, max_dst);
  const bool relu = ld->act == GNNV_ACT_RELU;
  const bool tf32 = ld->prec == GNNV_PREC_TF32;
  const size_t gp_f = relu ? (size_t)max_dst * ldo : 0;
  const size_t da_f = Gsrc ? (size_t)max_dst * lda : 0;
  const size_t cs_f = tf32 ? (size_t)kColBlocks * ldo : 0;
  // g_masked: Gdst already carries this layer's ReLU derivative (the trainer
  // applies it where Gdst is produced: the next layer's dX epilogue and
  // backward aggregation, from the forward's bit mask), so TF32 only needs
  // db = colsum(G), fused into the dW kernel.  Otherwise the mask is applied
  // here: TF32 without dX (layer 1) fuses it into dW (bits derived from H),
  // other TF32 layers use the mask + column-sum pass.
  const bool need_mask = relu && !g_masked;
  const bool fuse_mask = tf32 && need_mask && !Gsrc;
  const int mwords = mask_words(ld->d_out);
  const size_t mb_f = (fuse_mask && !mask_bits) ? (size_t)max_dst * mwords : 0;
  auto al = [](size_t f) { return (f + 63) & ~(size_t)63; };
  float* scratch =
      (float*)b->ensure_scratch((al(part_f) + al(gp_f) + al(da_f) + al(cs_f) + al(mb_f)) * sizeof(float), s);
  float* partial = scratch;
  float* Gp = scratch + al(part_f);
  float* dA = Gp + al(gp_f);
  float* colpart = dA + al(da_f);
  const float* G = Gdst;
  if (fuse_mask && !mask_bits) {
    uint32_t* mb = reinterpret_cast<uint32_t*>(colpart + al(cs_f));
    if (tl) tl->mark(s, "relu_bits" + sfx);
    launch_relu_bits(Hdst, ldo, ld->d_out, d_ndst, max_dst, mb, mwords, s);
    mask_bits = mb;
  }
  if (tf32 && need_mask && !fuse_mask) {
    // masked gradient + deterministic column sums (db) in one pass
    if (tl) tl->mark(s, "relu_mask" + sfx);
    launch_k(k_mask_colsum, kColBlocks, 256, 0, s, Gdst, Hdst, Gp, ldo, d_ndst, colpart, (__nv_bfloat16*)nullptr, 0);
    GNNV_CHECK_LAUNCH();
    launch_colsum_reduce(colpart, kColBlocks, ldo, ld->d_out, db, s);
    G = Gp;
  } else if (need_mask && !tf32) {
    if (tl) tl->mark(s, "relu_mask" + sfx);
    launch_relu_mask(Gdst, Hdst, Gp, ldo, ld->d_out, d_ndst, max_dst, s);
    G = Gp;
  }
  GemmDwArgs w{};
  if (sage) {
    w.X1 = xr ? xr->table : Hsrc;
    w.ld1 = ld->in_stride;
    w.X2 = A;
    w.ld2 = lda;
    if (xr) w.x1_rows = xr->rows, w.x1_table_rows = xr->table_rows;
  } else {
    w.X1 = A;
    w.ld1 = lda;
  }
  w.K1 = ld->d_in;
  w.G = G;
  w.ldg = ldo;
  if (io && io->gdst16) {
    GNNV_REQUIRE(tf32 && !need_mask, GNNV_ERR_UNSUPPORTED, "layer_bwd: a bf16 G needs TF32 and a pre-masked G");
    w.G16 = io->gdst16;
    w.ldg = io->gdst16_ld;
  }
  w.N = ld->d_out;
  w.d_M = d_ndst;
  w.max_M = max_dst;
  w.dW = dW;
  w.db = db;
  w.partial = partial;
  w.splits = splits;
  if (fuse_mask) {
    w.mask_bits = mask_bits;
    w.mask_ld = mwords;
  }
  w.db_fused = tf32 && !need_mask;
  w.zeroed = tf32 && grads_zeroed;
  if (tl) tl->mark(s, "gemm_dw" + sfx);
  if (io && io->x16 && io->a16 && (io->g16_out || io->g16_in) && !need_mask && tf32 && sage) {
    // hidden layer over bf16 operands (reading Q34): G (pre-masked fp32) ->
    // its bf16 copy + db = colsum(G) in one pass, then dW = [H16_dst |
    // A16]^T G16 by the MN-major kind::f16 kernel (four feature tiles)
    GemmDw16Args w16{};
    if (io->g16_in) {  // G and db's partials from the fused output layer
      w16.dbp = io->dbp;
      w16.ndbp = io->ndbp;
    } else {
      w16.G32 = Gdst;
      w16.ldg32 = ldo;
    }
    w16.src[0] = GemmDw16Src{io->x16, io->a16_ld, ld->d_in, 0, false};
    w16.src[1] = GemmDw16Src{io->a16, io->a16_ld, ld->d_in, ld->d_in, false};
    w16.G16 = io->g16_in ? io->g16_in : io->g16_out;
    w16.ldg = io->g16_ld;
    w16.N = ld->d_out;
    w16.d_M = d_ndst;
    w16.max_M = max_dst;
    w16.dW = dW;
    w16.db = db;
    w16.zeroed = w.zeroed;
    gemm_dw16(w16, s);
  } else if (io && io->x16 && io->a16 && io->gdst16) {
    GNNV_REQUIRE(sage && !xr && w.db_fused, GNNV_ERR_UNSUPPORTED, "layer_bwd: the bf16 dW needs SAGE and a final G");
    GemmDw16Args w16{};
    w16.src[0] = GemmDw16Src{io->x16, io->a16_ld, ld->d_in, 0, true};
    w16.src[1] = GemmDw16Src{io->a16, io->a16_ld, ld->d_in, ld->d_in, false};
    w16.G16 = io->gdst16;
    w16.ldg = io->gdst16_ld;
    w16.N = ld->d_out;
    w16.d_M = d_ndst;
    w16.max_M = max_dst;
    w16.dW = dW;
    w16.db = db;
    w16.zeroed = w.zeroed;
    gemm_dw16(w16, s);
  } else {
    gemm_dw(w, ld->prec, s);
  }
  if (Gsrc) {
    GemmDxArgs x{};
    x.G = G;
    x.ldg = ldo;
    x.N = ld->d_out;
    x.W = W;
    x.K1 = ld->d_in;
    x.d_M = d_ndst;
    x.max_M = max_dst;
    if (io && (io->g16_out || io->g16_in) && io->x16 && io->a16 && !need_mask && tf32 && sage) {  // G's bf16 copy
      x.G16 = io->g16_in ? io->g16_in : io->g16_out;
      x.ldg16 = io->g16_ld;
    }
    const bool g16 = io && io->gsrc16;
    // with the wide bf16 push, dA itself goes through as bf16 (the pushed
    // rows are stored as bf16 anyway); GNNV_NO_DA16=1: fp32 dA
    const bool da16 = sage && g16 && tf32 && lda % 32 == 0 && spmm_bwd_wide(io->gsrc16_ld, lda, ld->kind, true) &&
                      !env_on("GNNV_NO_DA16");
    if (sage && g16) {  // dH_src (and its dst-prefix rows from the GEMM) as bf16
      x.Y1_16 = io->gsrc16;
      x.ld1 = io->gsrc16_ld;
      x.y1_bits = src_bits;
      x.y1_bits_ld = src_bits_ld;
      x.Y2 = dA;
      x.ld2 = lda;
      if (da16) x.Y2_16 = dA;  // the scratch holds bf16 rows then (stride lda elements)
    } else if (sage) {
      x.Y1 = Gsrc;  // dH_dst lands directly in rows [0, n_dst) of dH_src
      x.ld1 = ld->in_stride;
      if (tf32) {
        x.y1_bits = src_bits;
        x.y1_bits_ld = src_bits_ld;
      }
      x.Y2 = dA;
      x.ld2 = lda;
    } else {
      x.Y1 = dA;
      x.ld1 = lda;
      x.Y2 = nullptr;
      x.ld2 = 0;
    }
    if (tl) tl->mark(s, "gemm_dx" + sfx);
    gemm_dx(x, ld->prec, s);
    if (tl) tl->mark(s, "spmm_bwd" + sfx);
    if (!g16 && b->pull_bwd && ((b->csc_mask >> h) & 1u) && ld->in_stride <= kPullMaxLd) {
      // transposed aggregation pulled per src row through the block's CSC:
      // one coalesced store per dH_src row, no atomics
      launch_spmm_bwd_pull(b->d_colptr[h], b->d_csc[h], b->d_indptr[h], d_ndst, b->d_sizes + h + 1, b->max_n[h + 1],
                           dA, lda, Gsrc, ld->in_stride, ld->d_in, ld->kind, ld->aggr, tf32 ? src_bits : nullptr,
                           src_bits_ld, s);
    } else {
      // transposed aggregation pushed from the dst rows: owner edges store,
      // the rest add atomically -- no zeroing pass over dH_src
      if (g16)
        launch_spmm_bwd(b->d_indptr[h], b->d_indices[h], b->d_own[h], d_ndst, max_dst, dA, lda, io->gsrc16,
                        io->gsrc16_ld, ld->d_in, ld->kind, ld->aggr, src_bits, src_bits_ld, s, true, da16);
      else
        launch_spmm_bwd(b->d_indptr[h], b->d_indices[h], b->d_own[h], d_ndst, max_dst, dA, lda, Gsrc, ld->in_stride,
                        ld->d_in, ld->kind, ld->aggr, tf32 ? src_bits : nullptr, src_bits_ld, s);
    }
  }
}

}  // namespace gnnv

using namespace gnnv;

extern "C" {

gnnv_status gnnv_layer_fwd(gnnv_blocks* b, int32_t layer, const gnnv_layer_desc* ld, const float* d_Hsrc,
                           const float* d_W, const float* d_b, float* d_Hdst, float* d_saveA, gnnv_stream s) {
  return guarded([&] {
    check_layer(b, layer, ld);
    GNNV_REQUIRE(d_Hsrc && d_W && d_b && d_Hdst && d_saveA, GNNV_ERR_PARAM, "layer_fwd: null buffer");
    layer_fwd_impl(b, layer, ld, d_Hsrc, d_W, d_b, d_Hdst, d_saveA, (cudaStream_t)s, nullptr, nullptr, nullptr, nullptr,
                   nullptr, nullptr, false, nullptr);
  });
}

gnnv_status gnnv_layer_bwd(gnnv_blocks* b, int32_t layer, const gnnv_layer_desc* ld, const float* d_Gdst,
                           const float* d_Hdst, const float* d_Hsrc, const float* d_saveA, const float* d_W,
                           float* d_Gsrc, float* d_dW, float* d_db, gnnv_stream s) {
  return guarded([&] {
    check_layer(b, layer, ld);
    GNNV_REQUIRE(d_Gdst && d_Hdst && d_Hsrc && d_saveA && d_W && d_dW && d_db, GNNV_ERR_PARAM,
                 "layer_bwd: null buffer");
    layer_bwd_impl(b, layer, ld, d_Gdst, d_Hdst, d_Hsrc, d_saveA, d_W, d_Gsrc, d_dW, d_db, (cudaStream_t)s, nullptr,
                   nullptr, false, nullptr, 0, nullptr, false, nullptr);
  });
}

}  // extern "C"

namespace {
// device-side row counts for the dense entry points: a ring of slots filled
// in stream order (the kernels read M from the device, like in a step)
const int32_t* device_count(int64_t M, cudaStream_t s) {
  static int32_t* ring = nullptr;
  static int slot = 0;
  constexpr int kSlots = 1024;
  if (!ring) ring = (int32_t*)gnnv::dmalloc(kSlots * sizeof(int32_t), "dense row counts");
  int32_t* p = ring + (slot++ % kSlots);
  const int32_t v = (int32_t)M;
  GNNV_TRY_CUDA(cudaMemcpyAsync(p, &v, sizeof(v), cudaMemcpyHostToDevice, s));
  return p;
}
float* dense_scratch(size_t floats, cudaStream_t s) {
  static float* buf = nullptr;
  static size_t cap = 0;
  if (floats > cap) {
    if (buf) {
      GNNV_TRY_CUDA(cudaStreamSynchronize(s));
      gnnv::dfree(buf);
    }
    cap = std::max(floats, (size_t)1 << 20);
    buf = (float*)gnnv::dmalloc(cap * sizeof(float), "dense scratch");
  }
  return buf;
}
}  // namespace

extern "C" {

gnnv_status gnnv_dense_fwd(const float* X1, int32_t ld1, const float* X2, int32_t ld2, int32_t K1, const float* W,
                           const float* b, float* Y, int32_t ldy, int32_t N, int64_t M, int32_t relu, int32_t prec,
                           gnnv_stream st) {
  return guarded([&] {
    GNNV_REQUIRE(X1 && W && b && Y && K1 >= 1 && N >= 1 && M >= 1 && M < INT32_MAX, GNNV_ERR_PARAM, "dense_fwd: args");
    GNNV_REQUIRE(ld1 >= K1 && ld1 % 4 == 0 && (!X2 || (ld2 >= K1 && ld2 % 4 == 0)) && ldy >= N && ldy % 4 == 0,
                 GNNV_ERR_PARAM, "dense_fwd: strides");
    GNNV_REQUIRE(prec >= GNNV_PREC_FP32 && prec <= GNNV_PREC_TF32, GNNV_ERR_PARAM, "dense_fwd: prec");
    cudaStream_t s = (cudaStream_t)st;
    GemmFwdArgs g{};
    g.X1 = X1;
    g.ld1 = ld1;
    g.X2 = X2;
    g.ld2 = ld2;
    g.K1 = K1;
    g.W = W;
    g.bias = b;
    g.Y = Y;
    g.ldy = ldy;
    g.N = N;
    g.d_M = device_count(M, s);
    g.max_M = M;
    g.relu = relu != 0;
    gemm_fwd(g, prec, s);
  });
}

gnnv_status gnnv_dense_dx(const float* G, int32_t ldg, int32_t N, const float* W, int32_t K1, float* Y1, int32_t ld1,
                          float* Y2, int32_t ld2, int64_t M, int32_t prec, gnnv_stream st) {
  return guarded([&] {
    GNNV_REQUIRE(G && W && Y1 && K1 >= 1 && N >= 1 && M >= 1 && M < INT32_MAX, GNNV_ERR_PARAM, "dense_dx: args");
    GNNV_REQUIRE(ldg >= N && ldg % 4 == 0 && ld1 >= K1 && ld1 % 4 == 0 && (!Y2 || (ld2 >= K1 && ld2 % 4 == 0)),
                 GNNV_ERR_PARAM, "dense_dx: strides");
    GNNV_REQUIRE(prec >= GNNV_PREC_FP32 && prec <= GNNV_PREC_TF32, GNNV_ERR_PARAM, "dense_dx: prec");
    cudaStream_t s = (cudaStream_t)st;
    GemmDxArgs x{};
    x.G = G;
    x.ldg = ldg;
    x.N = N;
    x.W = W;
    x.K1 = K1;
    x.Y1 = Y1;
    x.ld1 = ld1;
    x.Y2 = Y2;
    x.ld2 = ld2;
    x.d_M = device_count(M, s);
    x.max_M = M;
    gemm_dx(x, prec, s);
  });
}

gnnv_status gnnv_dense_dw(const float* X1, int32_t ld1, const float* X2, int32_t ld2, int32_t K1, const float* G,
                          int32_t ldg, int32_t N, int64_t M, float* dW, float* db, int32_t prec, gnnv_stream st) {
  return guarded([&] {
    GNNV_REQUIRE(X1 && G && dW && K1 >= 1 && N >= 1 && M >= 1 && M < INT32_MAX, GNNV_ERR_PARAM, "dense_dw: args");
    GNNV_REQUIRE(ld1 >= K1 && ld1 % 4 == 0 && (!X2 || (ld2 >= K1 && ld2 % 4 == 0)) && ldg >= N && ldg % 4 == 0,
                 GNNV_ERR_PARAM, "dense_dw: strides");
    GNNV_REQUIRE(prec >= GNNV_PREC_FP32 && prec <= GNNV_PREC_TF32, GNNV_ERR_PARAM, "dense_dw: prec");
    cudaStream_t s = (cudaStream_t)st;
    const int rows = (X2 ? 2 * K1 : K1) + 1;
    int32_t splits = 1;
    const size_t part_f = gemm_dw_partial_floats(rows, N, &splits, M);
    const size_t cs_f = (size_t)kColBlocks * ldg;
    float* scratch = dense_scratch(part_f + cs_f + N, s);
    float* db_out = db ? db : scratch + part_f + cs_f;
    GemmDwArgs w{};
    w.X1 = X1;
    w.ld1 = ld1;
    w.X2 = X2;
    w.ld2 = ld2;
    w.K1 = K1;
    w.G = G;
    w.ldg = ldg;
    w.N = N;
    w.d_M = device_count(M, s);
    w.max_M = M;
    w.dW = dW;
    w.db = db_out;
    w.partial = scratch;
    w.splits = splits;
    if (prec == GNNV_PREC_TF32) {
      float* colpart = scratch + part_f;
      launch_k(k_mask_colsum, kColBlocks, 256, 0, s, G, (const float*)nullptr, (float*)nullptr, ldg, w.d_M, colpart,
               (__nv_bfloat16*)nullptr, 0);
      GNNV_CHECK_LAUNCH();
      launch_colsum_reduce(colpart, kColBlocks, ldg, N, db_out, s);
    }
    gemm_dw(w, prec, s);
  });
}

gnnv_status gnnv_ce_loss(gnnv_blocks* b, const gnnv_graph* g, const float* d_logits, int32_t n_classes, int32_t stride,
                         int32_t n_global, float* d_loss, float* d_dlogits, gnnv_stream s) {
  return guarded([&] {
    GNNV_REQUIRE(b && g && d_logits && d_loss && d_dlogits, GNNV_ERR_PARAM, "ce_loss: null");
    GNNV_REQUIRE(b->sampled, GNNV_ERR_STATE, "ce_loss: gnnv_sample has not run on these blocks");
    GNNV_REQUIRE(n_classes >= 1 && stride >= n_classes && stride % 4 == 0 && n_global >= 1, GNNV_ERR_PARAM,
                 "ce_loss: bad sizes");
    float* scratch = (float*)b->ensure_scratch(4096, (cudaStream_t)s);
    // the loss uses its own small region at the end of a fresh 4 KiB block of the arena
    unsigned int* counter = reinterpret_cast<unsigned int*>(scratch + 1000);
    static_assert(kLossBlocks <= 1000, "partials must fit");
    GNNV_TRY_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned int), (cudaStream_t)s));
    launch_ce_loss(d_logits, stride, n_classes, b->d_sizes, b->d_F, g->d_labels, n_global, d_loss, d_dlogits,
                   scratch, counter, b->max_n[0], (cudaStream_t)s);
  });
}

}  // extern "C"
