// Sampled-block aggregation (SpMM) forward and its transpose.
//
// Paper: Eq.1 Aggregate; Algorithm 1 line 5 and the
// backward of line 8.  Reading Q11/Q15:
//   SAGE mean: A[v] = (1/c_v) sum_{u in N_b(v)} H[u]   (0 when c_v = 0)
//   SAGE sum : A[v] = sum_u H[u]
//   GCN  mean: A[v] = (H[v] + sum_u H[u]) / (c_v + 1);  GCN sum: H[v] + sum_u H[u]
// Backward: dH[u] += w_v dA[v] for every edge (v,u) (and the self term for
// GCN), w_v the same normalisation.
//
// Mapping: a warp owns RPW = 32/LPR dst rows (LPR lanes per row, LPR = 32
// for rows wider than 64 floats); a row's lanes stride over its float4
// columns.  Neighbour ids are fetched cooperatively and broadcast with
// shuffles; four neighbour rows are loaded before they are added, in
// ascending edge order (a fixed summation order).  HBM-bound: compulsory
// bytes are the distinct source rows + the output rows + the indices.
#include "common.cuh"

namespace gnnv {

__device__ __forceinline__ float4 f4add(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ float4 f4scale(float4 a, float s) { return make_float4(a.x * s, a.y * s, a.z * s, a.w * s); }
__device__ __forceinline__ float4 f4div(float4 a, float s) { return make_float4(a.x / s, a.y / s, a.z / s, a.w / s); }
__device__ __forceinline__ float4 mask_tail(float4 a, int col4, int d) {
  const int base = col4 * 4;
  if (base + 4 <= d) return a;
  return make_float4(base + 0 < d ? a.x : 0.f, base + 1 < d ? a.y : 0.f, base + 2 < d ? a.z : 0.f,
                     base + 3 < d ? a.w : 0.f);
}

template <int LPR>
__global__ void __launch_bounds__(256) k_spmm_fwd(const int32_t* __restrict__ indptr,
                                                  const int32_t* __restrict__ indices, const int32_t* d_ndst,
                                                  const float* __restrict__ H, int32_t ldh, float* __restrict__ A,
                                                  int32_t lda, int32_t d, int32_t kind, int32_t aggr) {
  constexpr int RPW = 32 / LPR;
  const int n = *d_ndst;
  const int vec = (d + 3) >> 2;
  const int lane = threadIdx.x & 31, sub = lane / LPR, sl = lane % LPR;
  const unsigned smask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (sub * LPR));
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const float4* H4 = reinterpret_cast<const float4*>(H);
  const int ldh4 = ldh >> 2, lda4 = lda >> 2;
  for (int base = warp * RPW; base < n; base += nwarps * RPW) {
    const int row = base + sub;
    const bool active = row < n;
    const int beg = active ? indptr[row] : 0;
    const int end = active ? indptr[row + 1] : 0;
    const int cnt = end - beg;
    for (int c0 = 0; c0 < vec; c0 += LPR) {
      const int c = c0 + sl;
      const bool cok = active && c < vec;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      if (kind == GNNV_KIND_GCN && cok) acc = __ldg(H4 + (int64_t)row * ldh4 + c);
      for (int e0 = 0; e0 < cnt; e0 += LPR) {
        const int my = (e0 + sl < cnt) ? __ldg(indices + beg + e0 + sl) : 0;
        const int m = min(LPR, cnt - e0);
        int j = 0;
        for (; j + 4 <= m; j += 4) {
          const int u0 = __shfl_sync(smask, my, j, LPR), u1 = __shfl_sync(smask, my, j + 1, LPR);
          const int u2 = __shfl_sync(smask, my, j + 2, LPR), u3 = __shfl_sync(smask, my, j + 3, LPR);
          if (cok) {
            const float4 h0 = __ldg(H4 + (int64_t)u0 * ldh4 + c), h1 = __ldg(H4 + (int64_t)u1 * ldh4 + c);
            const float4 h2 = __ldg(H4 + (int64_t)u2 * ldh4 + c), h3 = __ldg(H4 + (int64_t)u3 * ldh4 + c);
            acc = f4add(acc, h0);
            acc = f4add(acc, h1);
            acc = f4add(acc, h2);
            acc = f4add(acc, h3);
          }
        }
        for (; j < m; ++j) {
          const int u = __shfl_sync(smask, my, j, LPR);
          if (cok) acc = f4add(acc, __ldg(H4 + (int64_t)u * ldh4 + c));
        }
      }
      if (cok) {
        if (aggr == GNNV_AGGR_MEAN) {
          const int denom = cnt + (kind == GNNV_KIND_GCN ? 1 : 0);
          acc = denom ? f4div(acc, (float)denom) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        reinterpret_cast<float4*>(A)[(int64_t)row * lda4 + c] = mask_tail(acc, c, d);
      }
    }
    // zero the padding float4s of the output row (lda may exceed the used width)
    if (active) {
      for (int c = vec + sl; c < lda4; c += LPR)
        reinterpret_cast<float4*>(A)[(int64_t)row * lda4 + c] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
}

template <int LPR>
__global__ void __launch_bounds__(256) k_spmm_bwd(const int32_t* __restrict__ indptr,
                                                  const int32_t* __restrict__ indices, const int32_t* d_ndst,
                                                  const float* __restrict__ dA, int32_t lda, float* dH, int32_t ldh,
                                                  int32_t d, int32_t kind, int32_t aggr) {
  constexpr int RPW = 32 / LPR;
  const int n = *d_ndst;
  const int vec = (d + 3) >> 2;
  const int lane = threadIdx.x & 31, sub = lane / LPR, sl = lane % LPR;
  const unsigned smask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (sub * LPR));
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int ldh4 = ldh >> 2, lda4 = lda >> 2;
  float4* dH4 = reinterpret_cast<float4*>(dH);
  for (int base = warp * RPW; base < n; base += nwarps * RPW) {
    const int row = base + sub;
    const bool active = row < n;
    const int beg = active ? indptr[row] : 0;
    const int end = active ? indptr[row + 1] : 0;
    const int cnt = end - beg;
    float w = 1.f;
    if (aggr == GNNV_AGGR_MEAN) {
      const int denom = cnt + (kind == GNNV_KIND_GCN ? 1 : 0);
      w = denom ? 1.f / (float)denom : 0.f;
    }
    for (int c0 = 0; c0 < vec; c0 += LPR) {
      const int c = c0 + sl;
      const bool cok = active && c < vec;
      float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
      if (cok) g = mask_tail(f4scale(__ldg(reinterpret_cast<const float4*>(dA) + (int64_t)row * lda4 + c), w), c, d);
      if (kind == GNNV_KIND_GCN && cok) atomicAdd(dH4 + (int64_t)row * ldh4 + c, g);
      for (int e0 = 0; e0 < cnt; e0 += LPR) {
        const int my = (e0 + sl < cnt) ? __ldg(indices + beg + e0 + sl) : 0;
        const int m = min(LPR, cnt - e0);
        for (int j = 0; j < m; ++j) {
          const int u = __shfl_sync(smask, my, j, LPR);
          if (cok) atomicAdd(dH4 + (int64_t)u * ldh4 + c, g);
        }
      }
    }
  }
}

__global__ void k_rows_zero(float* X, int32_t ld, const int32_t* d_begin, const int32_t* d_end) {
  const int64_t b = d_begin ? *d_begin : 0, e = *d_end;
  const int ld4 = ld >> 2;
  const int64_t total = (e - b) * ld4;
  float4* X4 = reinterpret_cast<float4*>(X) + b * ld4;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x)
    X4[t] = make_float4(0.f, 0.f, 0.f, 0.f);
}

static int spmm_grid(int64_t max_rows, int rows_per_warp) {
  const int64_t warps = ceil_div(std::max<int64_t>(max_rows, 1), rows_per_warp);
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(warps, 8), (int64_t)num_sms() * 16));
}

void launch_spmm_fwd(const int32_t* d_indptr, const int32_t* d_indices, const int32_t* d_ndst, int64_t max_dst,
                     const float* H, int32_t ldh, float* A, int32_t lda, int32_t d, int32_t kind, int32_t aggr,
                     cudaStream_t s) {
  const int vec = (d + 3) / 4;
  if (vec <= 8) {
    k_spmm_fwd<8><<<spmm_grid(max_dst, 4), 256, 0, s>>>(d_indptr, d_indices, d_ndst, H, ldh, A, lda, d, kind, aggr);
  } else if (vec <= 16) {
    k_spmm_fwd<16><<<spmm_grid(max_dst, 2), 256, 0, s>>>(d_indptr, d_indices, d_ndst, H, ldh, A, lda, d, kind, aggr);
  } else {
    k_spmm_fwd<32><<<spmm_grid(max_dst, 1), 256, 0, s>>>(d_indptr, d_indices, d_ndst, H, ldh, A, lda, d, kind, aggr);
  }
  GNNV_CHECK_LAUNCH();
}

void launch_spmm_bwd(const int32_t* d_indptr, const int32_t* d_indices, const int32_t* d_ndst, int64_t max_dst,
                     const float* dA, int32_t lda, float* dH, int32_t ldh, int32_t d, int32_t kind, int32_t aggr,
                     cudaStream_t s) {
  const int vec = (d + 3) / 4;
  if (vec <= 8) {
    k_spmm_bwd<8><<<spmm_grid(max_dst, 4), 256, 0, s>>>(d_indptr, d_indices, d_ndst, dA, lda, dH, ldh, d, kind, aggr);
  } else if (vec <= 16) {
    k_spmm_bwd<16><<<spmm_grid(max_dst, 2), 256, 0, s>>>(d_indptr, d_indices, d_ndst, dA, lda, dH, ldh, d, kind, aggr);
  } else {
    k_spmm_bwd<32><<<spmm_grid(max_dst, 1), 256, 0, s>>>(d_indptr, d_indices, d_ndst, dA, lda, dH, ldh, d, kind, aggr);
  }
  GNNV_CHECK_LAUNCH();
}

// ---------------------------------------------------------------------
// Gather-form transposed aggregation.  The block is transposed on the device
// (CSC: for each src row u the dst rows v that sampled it), then
//   dH[u] = base(u) + sum_{v -> u} w_v dA[v]
// with base(u) = dH_dst[u] (SAGE, already in dH rows < n_dst from the dX
// GEMM) or w_u dA[u] (GCN self term), 0 for u >= n_dst.  Every dH row is
// written exactly once: no atomics on dH and no separate zeroing pass.

// edges per src row; also the per-dst weight w_v
__global__ void k_csc_count(const int32_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                            const int32_t* d_ndst, int32_t* __restrict__ colcnt, float* __restrict__ wv, int kind,
                            int aggr) {
  const int n = *d_ndst;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int)nthreads) {
    const int c = indptr[v + 1] - indptr[v];
    const int denom = c + (kind == GNNV_KIND_GCN ? 1 : 0);
    wv[v] = aggr == GNNV_AGGR_MEAN ? (denom ? 1.f / (float)denom : 0.f) : 1.f;
  }
  const int nnz = indptr[n];
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int)nthreads) atomicAdd(&colcnt[indices[e]], 1);
}

// exclusive scan of colcnt[0:n) into colptr[0:n] (single pass, decoupled
// look-back over tiles of 2048; status zeroed by the caller)
constexpr int kCscTile = 2048;
__global__ void __launch_bounds__(256) k_csc_scan(const int32_t* __restrict__ colcnt, const int32_t* d_n,
                                                  int32_t* __restrict__ colptr, unsigned long long* status) {
  __shared__ int s_tile;
  __shared__ uint32_t s_w[8], s_prefix;
  const int n = *d_n;
  const int ntiles = (n + kCscTile - 1) / kCscTile;
  if (threadIdx.x == 0) s_tile = (int)atomicAdd(reinterpret_cast<unsigned int*>(status), 1u);
  __syncthreads();
  const int tile = s_tile;
  if (tile >= ntiles) return;
  unsigned long long* st = status + 1;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int i0 = tile * kCscTile + threadIdx.x * 8;
  uint32_t x[8], sum = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    x[j] = (i0 + j < n) ? (uint32_t)colcnt[i0 + j] : 0u;
    sum += x[j];
  }
  uint32_t inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) s_w[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    uint32_t w = lane < 8 ? s_w[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += t;
    }
    if (lane < 8) s_w[lane] = w;
    const uint32_t agg = __shfl_sync(0xffffffffu, w, 7);
    uint32_t prefix = 0;
    if (tile == 0) {
      if (lane == 0) asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&st[0]), "l"((2ull << 62) | agg) : "memory");
    } else {
      if (lane == 0) asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&st[tile]), "l"((1ull << 62) | agg) : "memory");
      int p = tile - 1;
      while (true) {
        const int q = p - lane;
        unsigned long long w2 = 2ull << 62;
        if (q >= 0) {
          do {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(w2) : "l"(&st[q]) : "memory");
          } while ((w2 >> 62) == 0);
        }
        const unsigned pre = __ballot_sync(0xffffffffu, (w2 >> 62) == 2);
        const int stop = pre ? __ffs(pre) - 1 : 31;
        uint32_t v = lane <= stop ? (uint32_t)(w2 & 0xFFFFFFFFull) : 0u;
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        prefix += v;
        if (pre) break;
        p -= 32;
      }
      if (lane == 0)
        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&st[tile]), "l"((2ull << 62) | (prefix + agg))
                     : "memory");
    }
    if (lane == 0) s_prefix = prefix;
  }
  __syncthreads();
  uint32_t run = s_prefix + (wid ? s_w[wid - 1] : 0u) + inc - sum;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (i0 + j < n) colptr[i0 + j] = (int32_t)run;
    run += x[j];
  }
  if (tile == ntiles - 1 && i0 <= n && n <= i0 + 8) colptr[n] = (int32_t)(s_prefix + (wid ? s_w[wid - 1] : 0u) + inc);
}

// dst rows into their src buckets (counting down; order inside a bucket is
// arbitrary, so the fp32 sum order of dH is not fixed)
__global__ void k_csc_fill(const int32_t* __restrict__ indptr, const int32_t* __restrict__ indices, const int32_t* d_ndst,
                           const int32_t* __restrict__ colptr, int32_t* __restrict__ colcnt, int32_t* __restrict__ cscv) {
  const int n = *d_ndst;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const int b = indptr[v], e1 = indptr[v + 1];
    for (int e = b; e < e1; ++e) {
      const int u = indices[e];
      const int pos = colptr[u] + atomicSub(&colcnt[u], 1) - 1;
      cscv[pos] = v;
    }
  }
}

template <int LPR>
__global__ void __launch_bounds__(256) k_spmm_bwd_gather(const int32_t* __restrict__ colptr,
                                                         const int32_t* __restrict__ cscv,
                                                         const float* __restrict__ wv, const int32_t* d_ndst,
                                                         const int32_t* d_nsrc, const float* __restrict__ dA, int32_t lda,
                                                         float* dH, int32_t ldh, int32_t d, int32_t kind) {
  constexpr int RPW = 32 / LPR;
  const int ndst = *d_ndst, nsrc = *d_nsrc;
  const int vec = (d + 3) >> 2, ldh4 = ldh >> 2, lda4 = lda >> 2;
  const int lane = threadIdx.x & 31, sub = lane / LPR, sl = lane % LPR;
  const unsigned smask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (sub * LPR));
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const float4* dA4 = reinterpret_cast<const float4*>(dA);
  float4* dH4 = reinterpret_cast<float4*>(dH);
  for (int base = warp * RPW; base < nsrc; base += nwarps * RPW) {
    const int u = base + sub;
    const bool active = u < nsrc;
    const int beg = active ? colptr[u] : 0;
    const int cnt = active ? colptr[u + 1] - beg : 0;
    const float wself = (active && kind == GNNV_KIND_GCN && u < ndst) ? wv[u] : 0.f;
    for (int c0 = 0; c0 < ldh4; c0 += LPR) {
      const int c = c0 + sl;
      const bool cok = active && c < ldh4;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      if (cok && c < vec && u < ndst) {
        if (kind == GNNV_KIND_GCN) acc = f4scale(__ldg(dA4 + (int64_t)u * lda4 + c), wself);
        else acc = dH4[(int64_t)u * ldh4 + c];
      }
      for (int e0 = 0; e0 < cnt; e0 += LPR) {
        const int myv = (e0 + sl < cnt) ? __ldg(cscv + beg + e0 + sl) : 0;
        const float myw = (e0 + sl < cnt) ? __ldg(wv + myv) : 0.f;
        const int m = min(LPR, cnt - e0);
        for (int j = 0; j < m; ++j) {
          const int v = __shfl_sync(smask, myv, j, LPR);
          const float w = __shfl_sync(smask, myw, j, LPR);
          if (cok && c < vec) {
            const float4 g = __ldg(dA4 + (int64_t)v * lda4 + c);
            acc.x = fmaf(w, g.x, acc.x);
            acc.y = fmaf(w, g.y, acc.y);
            acc.z = fmaf(w, g.z, acc.z);
            acc.w = fmaf(w, g.w, acc.w);
          }
        }
      }
      if (cok) dH4[(int64_t)u * ldh4 + c] = c < vec ? mask_tail(acc, c, d) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
}

size_t spmm_bwd_csc_scratch_bytes(int64_t max_dst, int64_t max_src, int64_t max_nnz) {
  const int64_t tiles = ceil_div(std::max<int64_t>(max_src, 1), kCscTile) + 1;
  return (size_t)(max_src * 4 + (max_src + 1) * 4 + max_nnz * 4 + max_dst * 4 + tiles * 8 + 256);
}

void launch_spmm_bwd_csc(const int32_t* d_indptr, const int32_t* d_indices, const int32_t* d_ndst, const int32_t* d_nsrc,
                         int64_t max_dst, int64_t max_src, int64_t max_nnz, const float* dA, int32_t lda, float* dH,
                         int32_t ldh, int32_t d, int32_t kind, int32_t aggr, void* scratch, cudaStream_t s) {
  char* p = static_cast<char*>(scratch);
  auto take = [&](size_t bytes) {
    char* q = p;
    p += (bytes + 15) & ~(size_t)15;
    return q;
  };
  const int64_t tiles = ceil_div(std::max<int64_t>(max_src, 1), kCscTile) + 1;
  int32_t* colcnt = (int32_t*)take(max_src * 4);
  int32_t* colptr = (int32_t*)take((max_src + 1) * 4);
  int32_t* cscv = (int32_t*)take(std::max<int64_t>(max_nnz, 1) * 4);
  float* wv = (float*)take(std::max<int64_t>(max_dst, 1) * 4);
  unsigned long long* status = (unsigned long long*)take(tiles * 8);
  GNNV_TRY_CUDA(cudaMemsetAsync(colcnt, 0, max_src * 4, s));
  GNNV_TRY_CUDA(cudaMemsetAsync(status, 0, tiles * 8, s));
  const int sms = num_sms();
  k_csc_count<<<sms * 8, 256, 0, s>>>(d_indptr, d_indices, d_ndst, colcnt, wv, kind, aggr);
  GNNV_CHECK_LAUNCH();
  k_csc_scan<<<(unsigned)(tiles - 1 > 0 ? tiles - 1 : 1), 256, 0, s>>>(colcnt, d_nsrc, colptr, status);
  GNNV_CHECK_LAUNCH();
  k_csc_fill<<<sms * 8, 256, 0, s>>>(d_indptr, d_indices, d_ndst, colptr, colcnt, cscv);
  GNNV_CHECK_LAUNCH();
  const int vec = (ldh + 3) / 4;
  if (vec <= 8) {
    k_spmm_bwd_gather<8><<<spmm_grid(max_src, 4), 256, 0, s>>>(colptr, cscv, wv, d_ndst, d_nsrc, dA, lda, dH, ldh, d,
                                                               kind);
  } else if (vec <= 16) {
    k_spmm_bwd_gather<16><<<spmm_grid(max_src, 2), 256, 0, s>>>(colptr, cscv, wv, d_ndst, d_nsrc, dA, lda, dH, ldh, d,
                                                                kind);
  } else {
    k_spmm_bwd_gather<32><<<spmm_grid(max_src, 1), 256, 0, s>>>(colptr, cscv, wv, d_ndst, d_nsrc, dA, lda, dH, ldh, d,
                                                                kind);
  }
  GNNV_CHECK_LAUNCH();
}

void launch_rows_zero(float* X, int32_t ld, const int32_t* d_row_begin, const int32_t* d_row_end, int64_t max_rows,
                      cudaStream_t s) {
  const int64_t total = std::max<int64_t>(max_rows, 1) * (ld / 4);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), (int64_t)num_sms() * 8));
  k_rows_zero<<<grid, 256, 0, s>>>(X, ld, d_row_begin, d_row_end);
  GNNV_CHECK_LAUNCH();
}

}  // namespace gnnv
