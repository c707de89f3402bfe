// Degree-ordered static feature cache and the cache-lookup + gather kernel.
//
// Paper: transmission abstraction §3.2: the device cache is
// initialised from the free device memory, looks up which part of the
// mini-batch is resident, and the rest is fetched from the host over the
// host-device link; PaGraph static template; Eq.6 t_transfer =
// f(n_attr |V_i| (1-hit)).  Readings Q7 (capacity floor(r N),
// ties by lower id) and Q8 (hit accounting per unique row of F_L).
//
// Layout in HBM: the cached rows are a dense [C x stride] fp32 table in
// degree-rank order (slot i holds the vertex of rank i); with G shards,
// shard o holds ranks i = j*G + o at row j.  slot_map[v] = rank or -1.
// Misses are read zero-copy from the pinned, device-mapped host table.
// With d_rowidx (trainer, whole table resident on this device) only the dst
// prefix F_{L-1} of X is materialised -- the rows the layer-1 GEMMs read --
// and rowidx[u] = cache row of every F_L row, through which the layer-1
// aggregation reads the cache directly (spmm.cu, k_spmm_fwd<LPR, true>);
// with materialize = false not even that (the TF32 layer-1 GEMMs gather the
// H_dst rows from the table with TMA gather4, gemm_tma.cu).
#include <string.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include <cuda_bf16.h>

#include "common.cuh"

namespace gnnv {

__global__ void k_degree_keys(const int64_t* __restrict__ indptr, int64_t n, uint32_t* keys, int32_t* ids) {
  GNNV_PDL_ENTRY();
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t deg = indptr[v + 1] - indptr[v];
    keys[v] = 0xFFFFFFFFu - (uint32_t)(deg < 0xFFFFFFFFll ? deg : 0xFFFFFFFFll);  // ascending key = degree desc
    ids[v] = (int32_t)v;
  }
}

__global__ void k_slots(const int32_t* __restrict__ order, int64_t n, int64_t C, int32_t* slot) {
  GNNV_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    slot[order[i]] = i < C ? (int32_t)i : -1;
}

// shard rows: row j of shard `o` = vertex order[j*G + o]
__global__ void k_fill_shard(const int32_t* __restrict__ order, int64_t C, int G, int o, const float* src,
                             int32_t stride, float* dst, int64_t rows) {
  GNNV_PDL_ENTRY();
  const int vec = stride / 4;
  const int64_t total = rows * vec;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = t / vec;
    const int c = (int)(t - j * vec);
    const int64_t i = j * G + o;
    if (i >= C) continue;
    const int64_t v = order[i];
    reinterpret_cast<float4*>(dst)[j * vec + c] = reinterpret_cast<const float4*>(src)[v * vec + c];
  }
}

// ----------------------------------------------------------------- gather
// A warp owns 32 consecutive rows of F_L: lane i resolves row base+i's
// source (F -> slot -> shard pointer, or the mapped host row on a miss) in
// one round of parallel loads, then the warp copies the rows RU at a time
// with the lanes striding over float4 columns and all RU loads issued before
// the stores (memory-level parallelism for 400-2400 B rows).  Sources: shard
// ptrs[s % G] row s / G (HBM or NVLink peer) or the pinned host table (PCIe).
template <int RU>
__global__ void __launch_bounds__(256) k_gather(const int32_t* __restrict__ F, const int32_t* sizes, int L,
                                                const int32_t* __restrict__ slot,
                                                const float* const* __restrict__ shards, int G, int me,
                                                const float* __restrict__ host, int32_t stride,
                                                float* __restrict__ X, unsigned long long* stats, int mat_level,
                                                int32_t* __restrict__ rowidx, __nv_bfloat16* __restrict__ X16,
                                                int32_t ldx16, int32_t ones_col) {
  GNNV_PDL_ENTRY();
  const int n = sizes[L];
  const int n_mat = mat_level < 0 ? 0 : sizes[mat_level];  // rows materialised in X (all, the dst prefix, none)
  const int vec = stride >> 2;
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  unsigned long long c_local = 0, c_peer = 0, c_miss = 0;
  for (int base = warp * 32; base < n; base += nwarps * 32) {
    const int row = base + lane;
    const float4* src = nullptr;
    int kind = -1;  // 0 local, 1 peer, 2 host
    if (row < n) {
      const int v = F[row];
      const int s = slot[v];
      if (rowidx) rowidx[row] = s;  // cache row of every F_L row (whole-table cache, one shard)
      if (s >= 0) {
        const int o = s % G;
        src = reinterpret_cast<const float4*>(shards[o]) + (int64_t)(s / G) * vec;
        kind = o == me ? 0 : 1;
      } else {
        src = reinterpret_cast<const float4*>(host) + (int64_t)v * vec;
        kind = 2;
      }
    }
    c_local += __popc(__ballot_sync(0xffffffffu, kind == 0));
    c_peer += __popc(__ballot_sync(0xffffffffu, kind == 1));
    c_miss += __popc(__ballot_sync(0xffffffffu, kind == 2));
    const int nrows = min(32, n_mat - base);
    const uint64_t my = reinterpret_cast<uint64_t>(src);
    for (int r0 = 0; r0 < nrows; r0 += RU) {
      const float4* ps[RU];
#pragma unroll
      for (int j = 0; j < RU; ++j) ps[j] = reinterpret_cast<const float4*>(__shfl_sync(0xffffffffu, my, r0 + j));
      for (int c = lane; c < vec; c += 32) {
        float4 val[RU];
#pragma unroll
        for (int j = 0; j < RU; ++j)
          if (r0 + j < nrows) val[j] = __ldg(ps[j] + c);
        if (X) {
#pragma unroll
          for (int j = 0; j < RU; ++j)
            if (r0 + j < nrows) __stcs(reinterpret_cast<float4*>(X) + (int64_t)(base + r0 + j) * vec + c, val[j]);
        }
        if (X16) {  // bf16 copy for the layer's bf16 dW: column ones_col = 1.0, columns past it 0
          const int e = 4 * c;
#pragma unroll
          for (int j = 0; j < RU; ++j)
            if (r0 + j < nrows) {
              float4 v = val[j];
              if (e + 0 >= ones_col) v.x = e + 0 == ones_col ? 1.f : 0.f;
              if (e + 1 >= ones_col) v.y = e + 1 == ones_col ? 1.f : 0.f;
              if (e + 2 >= ones_col) v.z = e + 2 == ones_col ? 1.f : 0.f;
              if (e + 3 >= ones_col) v.w = e + 3 == ones_col ? 1.f : 0.f;
              const __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
              reinterpret_cast<uint2*>(X16)[((int64_t)(base + r0 + j) * ldx16 + e) >> 2] =
                  make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
            }
        }
      }
      if (X16 && 4 * vec <= ones_col && lane < nrows)  // the ones column lies past the row's stride
        X16[(int64_t)(base + lane) * ldx16 + ones_col] = __float2bfloat16_rn(1.f);
    }
  }
  if (stats && lane == 0) {
    if (c_local) atomicAdd(&stats[1], c_local);
    if (c_peer) atomicAdd(&stats[2], c_peer);
    if (c_miss) atomicAdd(&stats[3], c_miss);
    if (c_local + c_peer + c_miss) atomicAdd(&stats[0], c_local + c_peer + c_miss);
  }
}

void launch_gather(const gnnv_cache* c, const gnnv_blocks* b, float* d_X, int64_t* d_stats, cudaStream_t s,
                   int32_t* d_rowidx, bool materialize, void* d_X16, int32_t ldx16) {
  const gnnv_graph* g = c->g;
  GNNV_REQUIRE(!d_X16 || (materialize && ldx16 % 4 == 0 && ldx16 >= std::max(g->stride, g->d + 1)), GNNV_ERR_UNSUPPORTED,
               "gather: the bf16 copy needs materialised rows and a stride (multiple of 4) covering the ones column");
  GNNV_REQUIRE(d_X || (d_X16 && d_rowidx) || (!materialize && d_rowidx), GNNV_ERR_PARAM, "gather: no output");
  constexpr int RU = 8;
  const int64_t rows_ub = b->max_n[b->L];
  const int64_t warps = ceil_div(rows_ub, 32);
  const int blocks = capped_grid(std::min<int64_t>(ceil_div(warps, 8), (int64_t)num_sms() * 8));
  launch_k(k_gather<RU>, blocks, 256, 0, s, b->d_F, b->d_sizes, b->L, c->d_slot, c->d_shard_ptrs, c->world,
                                                   c->rank, g->d_feats, g->stride, d_X,
                                                   reinterpret_cast<unsigned long long*>(d_stats),
                                                   !materialize ? -1 : d_rowidx ? b->L - 1 : b->L, d_rowidx,
                                                   static_cast<__nv_bfloat16*>(d_X16), ldx16, g->d);
  GNNV_CHECK_LAUNCH();
}

}  // namespace gnnv

namespace gnnv {
static void open_peers(gnnv_cache* c, const cudaIpcMemHandle_t* handles) {
  for (int o = 0; o < c->world; ++o) {
    if (o == c->rank || c->shards[o]) continue;
    void* p = nullptr;
    GNNV_TRY_CUDA(cudaIpcOpenMemHandle(&p, handles[o], cudaIpcMemLazyEnablePeerAccess));
    c->shards[o] = (float*)((char*)p + ipc_offset());
    c->shard_ipc[o] = true;
  }
  GNNV_TRY_CUDA(cudaMemcpy((void*)c->d_shard_ptrs, c->shards.data(), c->world * sizeof(float*),
                           cudaMemcpyHostToDevice));
  c->peers_ready = true;
}
// ------------------------------------------------ dynamic cache (NEXT-3)
// access_batch of SPEC S:203-210 with all-miss admission (reading Q27), as
// one pass per batch after its gather:
//   k_dyn_hits   : LRU stamps the batch's hits with t; flags the misses
//   DeviceSelect : the miss rows, ascending (the admission order)
//   k_dyn_keys   : victim order of all C slots -- free slots first (by
//                  index), then (stamp, seq) for LRU / seq for FIFO
//   RadixSort    : slots sorted by key
//   k_dyn_admit  : miss i takes slot sorted[i mod C] (only the last C misses
//                  of a batch larger than C survive, as in the sequential
//                  rule), evicts its owner, copies its row from X
//   k_dyn_close  : counters (replaced = max(0, M - free slots)), seq += M
__global__ void k_dyn_hits(const int32_t* __restrict__ F, const int32_t* sizes, int L, int64_t cap,
                           const int32_t* __restrict__ slot, int32_t* stamp, int32_t t, int lru,
                           int32_t* __restrict__ mflag) {
  GNNV_PDL_ENTRY();
  const int n = sizes[L];
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < cap; r += (int64_t)gridDim.x * blockDim.x) {
    int f = 0;
    if (r < n) {
      const int s = slot[F[r]];
      if (s >= 0) {
        if (lru) stamp[s] = t;
      } else {
        f = 1;
      }
    }
    mflag[r] = f;
  }
}

__global__ void k_dyn_keys(int64_t C, const int32_t* __restrict__ owner, const int32_t* __restrict__ stamp,
                           const int64_t* __restrict__ seq, int lru, unsigned long long* keys, int32_t* idx) {
  GNNV_PDL_ENTRY();
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < C; s += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long k;
    if (owner[s] < 0) {
      k = (unsigned long long)s;  // free: lowest index first
    } else if (lru) {
      k = ((unsigned long long)(stamp[s] + 1) << 40) | (unsigned long long)seq[s];
    } else {
      k = (1ull << 62) | (unsigned long long)seq[s];
    }
    keys[s] = k;
    idx[s] = (int32_t)s;
  }
}

__global__ void k_dyn_admit(int64_t C, const int32_t* __restrict__ miss, const int64_t* ctr,
                            const int32_t* __restrict__ vslot, const int32_t* __restrict__ F, int32_t* slot,
                            int32_t* owner, int32_t* stamp, int64_t* seq, int32_t t, const float* __restrict__ X,
                            float* __restrict__ cache, int32_t stride) {
  GNNV_PDL_ENTRY();
  const int64_t M = ctr[5], base = ctr[4];
  const int64_t first = M > C ? M - C : 0;
  const int lane = threadIdx.x & 31;
  const int vec = stride >> 2;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = first + warp; i < M; i += nwarps) {
    const int r = miss[i];
    const int v = F[r];
    const int s = vslot[i % C];
    if (lane == 0) {
      const int old = owner[s];
      if (old >= 0) slot[old] = -1;
      owner[s] = v;
      slot[v] = s;
      stamp[s] = t;
      seq[s] = base + i;
    }
    const float4* src = reinterpret_cast<const float4*>(X) + (int64_t)r * vec;
    float4* dst = reinterpret_cast<float4*>(cache) + (int64_t)s * vec;
    for (int c = lane; c < vec; c += 32) dst[c] = __ldg(src + c);
  }
}

__global__ void k_dyn_close(int64_t* ctr, const int32_t* sizes, int L, int64_t C) {
  // ctr: 0 hits, 1 misses, 2 replaced, 3 admitted, 4 seq_next, 5 M, 6 occupied
  // all-miss admission fills the free slots first: M misses evict
  // max(0, M - free) residents and leave min(C, occupied + M) occupied
  const int64_t M = ctr[5], n = sizes[L], fr = C - ctr[6];
  ctr[0] += n - M;
  ctr[1] += M;
  if (C > 0) {
    ctr[2] += M > fr ? M - fr : 0;
    ctr[3] += M;
    ctr[4] += M;
    ctr[6] = ctr[6] + M < C ? ctr[6] + M : C;
  }
}

// bf16 copy of the local table: row r = bf16(table row r), zero-padded to ld16
__global__ void k_table_bf16(const float* __restrict__ src, int32_t stride, int32_t d, int64_t rows,
                             __nv_bfloat16* __restrict__ dst, int32_t ld16) {
  const int64_t total = rows * ld16;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / ld16;
    const int c = (int)(t - r * ld16);
    dst[t] = __float2bfloat16_rn(c < d ? src[r * stride + c] : 0.f);
  }
}

void cache_bf16_table(gnnv_cache* c) {
  if (c->d_table16) return;
  GNNV_REQUIRE(c->world == 1 && c->shards.size() == 1 && c->shards[0] && !c->dynamic, GNNV_ERR_STATE,
               "cache_bf16_table: a single static local table is required");
  const gnnv_graph* g = c->g;
  c->table16_ld = (g->d + 7) / 8 * 8;
  const int64_t rows = c->local_rows;
  c->d_table16 = dmalloc((size_t)std::max<int64_t>(rows, 1) * c->table16_ld * 2, "bf16 feature table");
  k_table_bf16<<<num_sms() * 16, 256>>>(c->shards[0], g->stride, g->d, rows, static_cast<__nv_bfloat16*>(c->d_table16),
                                        c->table16_ld);
  GNNV_CHECK_LAUNCH();
  GNNV_TRY_CUDA(cudaDeviceSynchronize());
}

void launch_cache_update(gnnv_cache* c, const gnnv_blocks* b, const float* d_X, cudaStream_t s) {
  const int L = b->L;
  const int64_t cap = b->max_n[L];
  const int64_t C = c->capacity;
  const int sms = num_sms();
  if (cap > c->miss_cap) {  // grow the miss buffers (setup-time synchronisation)
    GNNV_TRY_CUDA(cudaStreamSynchronize(s));
    dfree(c->d_miss);
    dfree(c->d_mflag);
    dfree(c->d_sel_tmp);
    c->d_miss = (int32_t*)dmalloc(cap * sizeof(int32_t), "cache miss rows");
    c->d_mflag = (int32_t*)dmalloc(cap * sizeof(int32_t), "cache miss flags");
    c->sel_tmp_bytes = 0;
    cub::CountingInputIterator<int32_t> it(0);
    GNNV_TRY_CUDA(cub::DeviceSelect::Flagged(nullptr, c->sel_tmp_bytes, it, c->d_mflag, c->d_miss,
                                             static_cast<int64_t*>(nullptr), (int)cap));
    c->d_sel_tmp = dmalloc(c->sel_tmp_bytes, "cache select temp");
    c->miss_cap = cap;
  }
  launch_k(k_dyn_hits, (int)std::min<int64_t>(ceil_div(cap, 256), sms * 8), 256, 0, s, b->d_F, b->d_sizes, L, cap,
           c->d_slot, c->d_stamp, c->step, c->policy == GNNV_POLICY_LRU ? 1 : 0, c->d_mflag);
  GNNV_CHECK_LAUNCH();
  cub::CountingInputIterator<int32_t> it(0);
  GNNV_TRY_CUDA(cub::DeviceSelect::Flagged(c->d_sel_tmp, c->sel_tmp_bytes, it, c->d_mflag, c->d_miss, c->d_ctr + 5,
                                           (int)cap, s));
  if (C > 0) {
    launch_k(k_dyn_keys, (int)std::min<int64_t>(ceil_div(C, 256), sms * 8), 256, 0, s, C, c->d_owner, c->d_stamp,
             c->d_seq, c->policy == GNNV_POLICY_LRU ? 1 : 0, c->d_keys, c->d_vidx);
    GNNV_CHECK_LAUNCH();
    GNNV_TRY_CUDA(cub::DeviceRadixSort::SortPairs(c->d_sort_tmp, c->sort_tmp_bytes, c->d_keys, c->d_keys + C,
                                                  c->d_vidx, c->d_vidx + C, (int)C, 0, 64, s));
    launch_k(k_dyn_admit, sms * 8, 256, 0, s, C, c->d_miss, c->d_ctr, c->d_vidx + C, b->d_F, c->d_slot, c->d_owner,
             c->d_stamp, c->d_seq, c->step, d_X, c->shards[0], c->g->stride);
    GNNV_CHECK_LAUNCH();
  }
  k_dyn_close<<<1, 1, 0, s>>>(c->d_ctr, b->d_sizes, L, C);
  GNNV_CHECK_LAUNCH();
  ++c->step;
}

}  // namespace gnnv

using namespace gnnv;

extern "C" {

gnnv_status gnnv_cache_ipc_handle(const gnnv_cache* c, void* out64) {
  return guarded([&] {
    GNNV_REQUIRE(c && out64, GNNV_ERR_PARAM, "cache_ipc_handle: null");
    GNNV_REQUIRE(c->placement == GNNV_PLACE_SHARDED, GNNV_ERR_STATE, "cache_ipc_handle: placement is not SHARDED");
    GNNV_TRY_CUDA(cudaSetDevice(c->g->device));
    cudaIpcMemHandle_t h;
    GNNV_TRY_CUDA(cudaIpcGetMemHandle(&h, c->shards[c->rank]));
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    memcpy(out64, &h, sizeof(h));
  });
}

gnnv_status gnnv_cache_open_peers(gnnv_cache* c, const void* handles) {
  return guarded([&] {
    GNNV_REQUIRE(c && handles, GNNV_ERR_PARAM, "cache_open_peers: null");
    GNNV_REQUIRE(c->placement == GNNV_PLACE_SHARDED, GNNV_ERR_STATE, "cache_open_peers: placement is not SHARDED");
    GNNV_TRY_CUDA(cudaSetDevice(c->g->device));
    open_peers(c, static_cast<const cudaIpcMemHandle_t*>(handles));
  });
}

gnnv_status gnnv_cache_build(gnnv_graph* g, double ratio, int32_t policy, int32_t placement, gnnv_comm* comm,
                             int32_t virtual_shards, gnnv_cache** out) {
  return guarded([&] {
    GNNV_REQUIRE(g && out, GNNV_ERR_PARAM, "cache_build: null");
    GNNV_REQUIRE(ratio >= 0.0 && ratio <= 1.0, GNNV_ERR_PARAM, "cache_build: ratio must be in [0,1]");
    GNNV_REQUIRE(policy == GNNV_POLICY_NONE || policy == GNNV_POLICY_DEGREE || policy == GNNV_POLICY_FIFO ||
                     policy == GNNV_POLICY_LRU,
                 GNNV_ERR_PARAM, "cache_build: unknown policy");
    const bool dynamic = policy == GNNV_POLICY_FIFO || policy == GNNV_POLICY_LRU;
    GNNV_REQUIRE(!dynamic || placement == GNNV_PLACE_REPLICA || (placement == GNNV_PLACE_SHARDED && !comm),
                 GNNV_ERR_UNSUPPORTED, "cache_build: dynamic FIFO/LRU caches are built for one device (REPLICA)");
    GNNV_REQUIRE(placement >= GNNV_PLACE_REPLICA && placement <= GNNV_PLACE_SHARDED_LOCAL, GNNV_ERR_PARAM,
                 "cache_build: unknown placement");
    int G = 1, me = 0;
    if (placement == GNNV_PLACE_SHARDED) {
      if (comm) {  // no comm: one rank, one shard
        G = comm->world;
        me = comm->rank;
      }
    } else if (placement == GNNV_PLACE_SHARDED_LOCAL) {
      GNNV_REQUIRE(virtual_shards >= 1 && virtual_shards <= 64, GNNV_ERR_PARAM, "cache_build: virtual_shards in [1,64]");
      G = virtual_shards;
    }
    GNNV_TRY_CUDA(cudaSetDevice(g->device));
    const int64_t n = g->n;
    // C = floor(ratio * N) in IEEE double; NONE => 0
    const int64_t C = policy == GNNV_POLICY_NONE ? 0 : (int64_t)std::floor(ratio * (double)n);
    gnnv_cache* c = new gnnv_cache();
    c->g = g;
    c->capacity = C;
    c->world = G;
    c->rank = me;
    c->placement = placement;
    c->policy = policy;
    c->dynamic = dynamic;
    try {
      c->d_slot = (int32_t*)dmalloc(n * sizeof(int32_t), "cache slot map");
      c->d_order = (int32_t*)dmalloc(n * sizeof(int32_t), "cache order");
      uint32_t* keys = (uint32_t*)dmalloc(n * sizeof(uint32_t), "degree keys");
      uint32_t* keys2 = (uint32_t*)dmalloc(n * sizeof(uint32_t), "degree keys");
      int32_t* ids = (int32_t*)dmalloc(n * sizeof(int32_t), "ids");
      const int sms = num_sms();
      k_degree_keys<<<sms * 8, 256>>>(g->d_indptr, n, keys, ids);
      GNNV_CHECK_LAUNCH();
      size_t tmp_bytes = 0;
      GNNV_TRY_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys2, ids, c->d_order, (int)n));
      void* tmp = dmalloc(tmp_bytes, "sort temp");
      // LSD radix sort is stable: equal degrees keep ascending id order
      GNNV_TRY_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys2, ids, c->d_order, (int)n));
      k_slots<<<sms * 8, 256>>>(c->d_order, n, dynamic ? 0 : C, c->d_slot);  // dynamic: starts empty
      GNNV_CHECK_LAUNCH();
      GNNV_TRY_CUDA(cudaDeviceSynchronize());
      dfree(tmp);
      dfree(keys);
      dfree(keys2);
      dfree(ids);
      c->shards.assign(G, nullptr);
      c->shard_owned.assign(G, false);
      c->shard_ipc.assign(G, false);
      for (int o = 0; o < G; ++o) {
        const int64_t rows = C > o ? (C - o + G - 1) / G : 0;
        const bool resident = placement != GNNV_PLACE_SHARDED || o == me;
        if (!resident) continue;
        const size_t bytes = (size_t)std::max<int64_t>(rows, 1) * g->stride * sizeof(float);
        c->shards[o] = (float*)dmalloc(bytes, "feature cache (Gamma_cache)");
        c->shard_owned[o] = true;
        c->local_rows += rows;
        if (rows && !dynamic) {
          k_fill_shard<<<sms * 16, 256>>>(c->d_order, C, G, o, g->d_feats, g->stride, c->shards[o], rows);
          GNNV_CHECK_LAUNCH();
        }
      }
      if (dynamic) {
        const int64_t Cs = std::max<int64_t>(C, 1);
        c->d_owner = (int32_t*)dmalloc(Cs * sizeof(int32_t), "cache owners");
        c->d_stamp = (int32_t*)dmalloc(Cs * sizeof(int32_t), "cache stamps");
        c->d_seq = (int64_t*)dmalloc(Cs * sizeof(int64_t), "cache sequence numbers");
        c->d_keys = (unsigned long long*)dmalloc(2 * Cs * sizeof(unsigned long long), "cache victim keys");
        c->d_vidx = (int32_t*)dmalloc(2 * Cs * sizeof(int32_t), "cache victim order");
        c->d_ctr = (int64_t*)dmalloc(8 * sizeof(int64_t), "cache counters");
        GNNV_TRY_CUDA(cudaMemset(c->d_owner, 0xFF, Cs * sizeof(int32_t)));
        GNNV_TRY_CUDA(cudaMemset(c->d_stamp, 0xFF, Cs * sizeof(int32_t)));
        GNNV_TRY_CUDA(cudaMemset(c->d_seq, 0xFF, Cs * sizeof(int64_t)));
        GNNV_TRY_CUDA(cudaMemset(c->d_ctr, 0, 8 * sizeof(int64_t)));
        GNNV_TRY_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, c->sort_tmp_bytes, c->d_keys, c->d_keys + Cs,
                                                      c->d_vidx, c->d_vidx + Cs, (int)Cs));
        c->d_sort_tmp = dmalloc(c->sort_tmp_bytes, "cache victim sort temp");
      }
      c->d_shard_ptrs = (const float**)dmalloc(G * sizeof(float*), "shard pointers");
      GNNV_TRY_CUDA(cudaMemcpy((void*)c->d_shard_ptrs, c->shards.data(), G * sizeof(float*), cudaMemcpyHostToDevice));
      GNNV_TRY_CUDA(cudaDeviceSynchronize());
      if (placement == GNNV_PLACE_SHARDED && G > 1) {
        // peers' shards are read in place over NVLink: export this rank's
        // shard as a CUDA IPC handle, all-gather the handles (NCCL), map the
        // others.  A host-only comm leaves this to gnnv_cache_open_peers.
        c->peers_ready = false;
        if (comm->nccl) {
          std::vector<cudaIpcMemHandle_t> all(G);
          cudaIpcMemHandle_t mine;
          GNNV_TRY_CUDA(cudaIpcGetMemHandle(&mine, c->shards[me]));
          comm_allgather_bytes(comm, &mine, all.data(), sizeof(mine));
          open_peers(c, all.data());
        }
      }
    } catch (...) {
      gnnv_cache_free(c);
      throw;
    }
    *out = c;
  });
}

gnnv_status gnnv_cache_free(gnnv_cache* c) {
  if (!c) return GNNV_OK;
  dfree(c->d_slot);
  dfree(c->d_order);
  for (size_t o = 0; o < c->shards.size(); ++o) {
    if (c->shard_owned[o]) dfree(c->shards[o]);
    if (c->shard_ipc[o]) cudaIpcCloseMemHandle((char*)c->shards[o] - ipc_offset());
  }
  dfree((void*)c->d_shard_ptrs);
  dfree(c->d_owner);
  dfree(c->d_stamp);
  dfree(c->d_seq);
  dfree(c->d_keys);
  dfree(c->d_vidx);
  dfree(c->d_sort_tmp);
  dfree(c->d_miss);
  dfree(c->d_mflag);
  dfree(c->d_sel_tmp);
  dfree(c->d_ctr);
  dfree(c->d_table16);
  delete c;
  return GNNV_OK;
}

gnnv_status gnnv_cache_info(const gnnv_cache* c, gnnv_cache_view* o) {
  return guarded([&] {
    GNNV_REQUIRE(c && o, GNNV_ERR_PARAM, "cache_info: null");
    o->capacity = c->capacity;
    o->local_rows = c->local_rows;
    o->bytes = c->local_rows * (int64_t)c->g->stride * (int64_t)sizeof(float);
    o->world = c->world;
    o->rank = c->rank;
    o->placement = c->placement;
    o->d_slot = c->d_slot;
    o->d_order = c->d_order;
  });
}

gnnv_status gnnv_cache_update(gnnv_cache* c, const gnnv_blocks* b, const float* d_X, gnnv_stream s) {
  return guarded([&] {
    GNNV_REQUIRE(c && b && d_X, GNNV_ERR_PARAM, "cache_update: null");
    GNNV_REQUIRE(c->dynamic, GNNV_ERR_STATE, "cache_update: the cache's policy is static (FIFO/LRU only)");
    GNNV_REQUIRE(b->sampled, GNNV_ERR_STATE, "cache_update: gnnv_sample has not run on these blocks");
    GNNV_REQUIRE(c->g == b->g, GNNV_ERR_STATE, "cache_update: cache and blocks belong to different graphs");
    launch_cache_update(c, b, d_X, (cudaStream_t)s);
  });
}

gnnv_status gnnv_cache_counters(const gnnv_cache* c, int64_t* host4) {
  return guarded([&] {
    GNNV_REQUIRE(c && host4, GNNV_ERR_PARAM, "cache_counters: null");
    for (int i = 0; i < 4; ++i) host4[i] = 0;
    if (!c->dynamic) return;
    GNNV_TRY_CUDA(cudaDeviceSynchronize());
    GNNV_TRY_CUDA(cudaMemcpy(host4, c->d_ctr, 4 * sizeof(int64_t), cudaMemcpyDeviceToHost));
  });
}

gnnv_status gnnv_cache_owners(const gnnv_cache* c, const int32_t** d_owner) {
  return guarded([&] {
    GNNV_REQUIRE(c && d_owner, GNNV_ERR_PARAM, "cache_owners: null");
    GNNV_REQUIRE(c->dynamic, GNNV_ERR_STATE, "cache_owners: static cache");
    *d_owner = c->d_owner;
  });
}

gnnv_status gnnv_gather(const gnnv_cache* c, const gnnv_blocks* b, float* d_X, int64_t* d_stats, gnnv_stream s) {
  return guarded([&] {
    GNNV_REQUIRE(c && b && d_X, GNNV_ERR_PARAM, "gather: null");
    GNNV_REQUIRE(b->sampled, GNNV_ERR_STATE, "gather: gnnv_sample has not run on these blocks");
    GNNV_REQUIRE(c->g == b->g, GNNV_ERR_STATE, "gather: cache and blocks belong to different graphs");
    GNNV_REQUIRE(((uintptr_t)d_X & 15) == 0, GNNV_ERR_PARAM, "gather: d_X must be 16-byte aligned");
    GNNV_REQUIRE(c->peers_ready, GNNV_ERR_STATE, "gather: SHARDED peers not mapped (gnnv_cache_open_peers)");
    launch_gather(c, b, d_X, d_stats, (cudaStream_t)s);
  });
}

}  // extern "C"
