// Sampled-block aggregation (SpMM) forward and its transpose.
//
// Paper: Eq.1 Aggregate; Algorithm 1 line 5 and the
// backward of line 8.  Reading Q11/Q15:
//   SAGE mean: A[v] = (1/c_v) sum_{u in N_b(v)} H[u]   (0 when c_v = 0)
//   SAGE sum : A[v] = sum_u H[u]
//   GCN  mean: A[v] = (H[v] + sum_u H[u]) / (c_v + 1);  GCN sum: H[v] + sum_u H[u]
// Backward: dH[u] += w_v dA[v] for every edge (v,u) (and the self term for
// GCN), w_v the same normalisation -- pushed in two passes (owner stores,
// then atomic adds), see k_spmm_bwd.
//
// Mapping: a warp owns RPW = 32/LPR dst rows (LPR lanes per row, LPR = 32
// for rows wider than 64 floats); a row's lanes stride over its float4
// columns.  Neighbour ids are fetched cooperatively and broadcast with
// shuffles; four neighbour rows are loaded before they are added, in
// ascending edge order (a fixed summation order).  HBM-bound: compulsory
// bytes are the distinct source rows + the output rows + the indices.
#include <cuda_bf16.h>

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

__device__ __forceinline__ uint64_t l2_policy_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_normal() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float4 ld_hint(const float4* p, uint64_t pol) {
  float4 v;
  asm("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_hint(float4* p, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w), "l"(pol)
               : "memory");
}

// row u of H (HINT: u carries the evict_first flag in its sign bit)
template <bool HINT>
__device__ __forceinline__ float4 ld_row(const float4* __restrict__ H4, int u, int ldh4, int c, uint64_t pol_first,
                                         uint64_t pol_norm) {
  if (!HINT) return __ldg(H4 + (int64_t)u * ldh4 + c);
  return ld_hint(H4 + (int64_t)(u & 0x7FFFFFFF) * ldh4 + c, u < 0 ? pol_first : pol_norm);
}

// IND: source rows are read through rowidx (row u of the block is row
// rowidx[u] of H = the device cache table), so X need not be materialised.
// HINT (lastv != NULL; the trainer's layer 1): the visit at which a source
// row is read for the last time in this launch (lastv[u] = 1 + the CSR
// position of u's last edge, sampler k_map) loads it with an L2 evict_first
// policy, every other visit with evict_normal, and the aggregate rows are
// stored evict_first: dead rows leave L2 first, so rows still to be
// re-read stay (an LRU replay of the products visit sequence
// gives 1.41 DRAM reads per distinct row at 126 MB, 1.03 with these hints).
// Summation order unchanged (bitwise the same result).
template <int LPR, bool IND, bool HINT>
__global__ void __launch_bounds__(256) k_spmm_fwd(const int32_t* __restrict__ indptr,
                                                  const int32_t* __restrict__ indices, const int32_t* d_ndst,
                                                  const float* __restrict__ H, int32_t ldh, float* __restrict__ A,
                                                  int32_t lda, int32_t d, int32_t kind, int32_t aggr,
                                                  const int32_t* __restrict__ rowidx,
                                                  const uint32_t* __restrict__ lastv) {
  GNNV_PDL_ENTRY();
  uint64_t pol_first = 0, pol_norm = 0;
  if (HINT) {
    pol_first = l2_policy_first();
    pol_norm = l2_policy_normal();
  }

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
      if (kind == GNNV_KIND_GCN && cok) acc = __ldg(H4 + (int64_t)(IND ? __ldg(rowidx + row) : row) * ldh4 + c);
      for (int e0 = 0; e0 < cnt; e0 += LPR) {
        int my = (e0 + sl < cnt) ? __ldg(indices + beg + e0 + sl) : 0;
        bool last = false;
        if (HINT && e0 + sl < cnt) last = __ldg(lastv + my) == (uint32_t)(beg + e0 + sl) + 1u;
        if (IND) my = __ldg(rowidx + my);
        if (HINT && last) my |= (int)0x80000000;  // row ids < 2^31: the sign bit carries the hint
        const int m = min(LPR, cnt - e0);
        int j = 0;
        for (; j + 4 <= m; j += 4) {
          const int u0 = __shfl_sync(smask, my, j, LPR), u1 = __shfl_sync(smask, my, j + 1, LPR);
          const int u2 = __shfl_sync(smask, my, j + 2, LPR), u3 = __shfl_sync(smask, my, j + 3, LPR);
          if (cok) {
            const float4 h0 = ld_row<HINT>(H4, u0, ldh4, c, pol_first, pol_norm);
            const float4 h1 = ld_row<HINT>(H4, u1, ldh4, c, pol_first, pol_norm);
            const float4 h2 = ld_row<HINT>(H4, u2, ldh4, c, pol_first, pol_norm);
            const float4 h3 = ld_row<HINT>(H4, u3, ldh4, c, pol_first, pol_norm);
            acc = f4add(acc, h0);
            acc = f4add(acc, h1);
            acc = f4add(acc, h2);
            acc = f4add(acc, h3);
          }
        }
        for (; j < m; ++j) {
          const int u = __shfl_sync(smask, my, j, LPR);
          if (cok) acc = f4add(acc, ld_row<HINT>(H4, u, ldh4, c, pol_first, pol_norm));
        }
      }
      if (cok) {
        if (aggr == GNNV_AGGR_MEAN) {
          const int denom = cnt + (kind == GNNV_KIND_GCN ? 1 : 0);
          acc = denom ? f4div(acc, (float)denom) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        float4* out = reinterpret_cast<float4*>(A) + (int64_t)row * lda4 + c;
        if (HINT) st_hint(out, mask_tail(acc, c, d), pol_first);
        else *out = mask_tail(acc, c, d);
      }
    }
    // zero the padding float4s of the output row (lda may exceed the used width)
    if (active) {
      for (int c = vec + sl; c < lda4; c += LPR)
        reinterpret_cast<float4*>(A)[(int64_t)row * lda4 + c] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
}

// Transposed aggregation dH[u] += w_v dA[v] over the block's edges (v, u),
// pushed from the dst rows in two passes so that no dH row needs zeroing:
//  phase 1: every OWNER edge -- the edge at which u first appeared in the
//           sampler's scan, own[v] bit i (a src id >= n_dst has exactly one)
//           -- STORES its row: dH[u] = w_v dA[v] (padding columns 0); GCN
//           also stores the self term dH[v] = w_v dA[v] of every dst row.
//  phase 2: every other edge ADDS (red.global.add.v4.f32) into rows written
//           by phase 1 or, for u < n_dst, by the dX GEMM (SAGE dH_dst).
// Every dH row < n_src is therefore written before it is accumulated into;
// phase 2 carries only the repeated ids (products layer 2: ~30% of edges).
// dH row pieces of 4 elements: fp32 (float4) or, with H16, bf16 (8 bytes;
// the phase-2 additions are two red.global.add.noftz.bf16x2)
__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}
template <bool H16>
__device__ __forceinline__ void dh_store4(void* dH, int64_t i4, float4 v) {
  if (!H16) reinterpret_cast<float4*>(dH)[i4] = v;
  else reinterpret_cast<uint2*>(dH)[i4] = make_uint2(pack_bf16x2(v.x, v.y), pack_bf16x2(v.z, v.w));
}
template <bool H16>
__device__ __forceinline__ void dh_add4(void* dH, int64_t i4, float4 v) {
  if (!H16) {
    atomicAdd(reinterpret_cast<float4*>(dH) + i4, v);
  } else {
    uint2* p = reinterpret_cast<uint2*>(dH) + i4;  // one 8-byte bf16x4 reduction
    asm volatile("red.global.add.noftz.v2.bf16x2 [%0], {%1, %2};" ::"l"(p), "r"(pack_bf16x2(v.x, v.y)),
                 "r"(pack_bf16x2(v.z, v.w))
                 : "memory");
  }
}

template <int LPR, bool H16 = false>
__global__ void __launch_bounds__(256) k_spmm_bwd(const int32_t* __restrict__ indptr,
                                                  const int32_t* __restrict__ indices,
                                                  const uint32_t* __restrict__ own, const int32_t* d_ndst,
                                                  const float* __restrict__ dA, int32_t lda, void* dH, int32_t ldh,
                                                  int32_t d, int32_t kind, int32_t aggr, int32_t phase,
                                                  const uint32_t* __restrict__ bits, int32_t bits_ld) {
  GNNV_PDL_ENTRY();
  constexpr int RPW = 32 / LPR;
  const int n = *d_ndst;
  const int vec = (d + 3) >> 2;
  const int lane = threadIdx.x & 31, sub = lane / LPR, sl = lane % LPR;
  const unsigned smask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (sub * LPR));
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int ldh4 = ldh >> 2, lda4 = lda >> 2;
  const int cols = phase == 1 ? ldh4 : vec;  // phase 1 also writes the padding
  const bool gcn = kind == GNNV_KIND_GCN;
  // optional ReLU mask of dH's rows (the previous layer's output bits):
  // dH[u] = relu'(H[u]) * sum, applied to every contribution
  auto masked = [&](float4 g, int64_t u, int c) {
    if (!bits) return g;
    const uint32_t w = __ldg(bits + u * bits_ld + (c >> 3)) >> ((c & 7) * 4);
    return make_float4(w & 1u ? g.x : 0.f, w & 2u ? g.y : 0.f, w & 4u ? g.z : 0.f, w & 8u ? g.w : 0.f);
  };
  for (int base = warp * RPW; base < n; base += nwarps * RPW) {
    const int row = base + sub;
    const bool active = row < n;
    const int beg = active ? indptr[row] : 0;
    const int end = active ? indptr[row + 1] : 0;
    const int cnt = end - beg;
    const uint32_t mine = active ? own[row] : 0u;
    const uint32_t sel = phase == 1 ? mine : ~mine;
    float w = 1.f;
    if (aggr == GNNV_AGGR_MEAN) {
      const int denom = cnt + (gcn ? 1 : 0);
      w = denom ? 1.f / (float)denom : 0.f;
    }
    const uint32_t todo = (cnt >= 32 ? 0xffffffffu : ((1u << cnt) - 1u)) & sel;
    if (!(phase == 1 && gcn) && __ballot_sync(0xffffffffu, todo != 0u) == 0u) continue;  // warp-uniform
    for (int c0 = 0; c0 < cols; c0 += LPR) {
      const int c = c0 + sl;
      const bool cok = active && c < cols;
      float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
      if (cok && c < vec)
        g = mask_tail(f4scale(__ldg(reinterpret_cast<const float4*>(dA) + (int64_t)row * lda4 + c), w), c, d);
      if (phase == 1 && gcn && cok) dh_store4<H16>(dH, (int64_t)row * ldh4 + c, c < vec ? masked(g, row, c) : g);
      for (int e0 = 0; e0 < cnt; e0 += LPR) {
        const int my = (e0 + sl < cnt) ? __ldg(indices + beg + e0 + sl) : 0;
        const int m = min(LPR, cnt - e0);
        // this phase's edges of the chunk, four at a time: their src ids and
        // ReLU-bit words are all requested before any row is written, so
        // the dependent bit loads overlap (uniform within the row's lanes)
        uint32_t pend = (todo >> e0) & (m >= 32 ? 0xffffffffu : ((1u << m) - 1u));
        while (pend) {
          int u[4];
          uint32_t wb[4];
          int k = 0;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int j = pend ? __ffs(pend) - 1 : 0;
            u[q] = __shfl_sync(smask, my, j, LPR);
            if (pend) {
              pend &= pend - 1;
              k = q + 1;
            }
          }
#pragma unroll
          for (int q = 0; q < 4; ++q)
            wb[q] = (bits && q < k && cok && c < vec) ? __ldg(bits + (int64_t)u[q] * bits_ld + (c >> 3)) >> ((c & 7) * 4)
                                                       : 0xFu;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (q < k && cok) {
              const float4 gm = make_float4(wb[q] & 1u ? g.x : 0.f, wb[q] & 2u ? g.y : 0.f, wb[q] & 4u ? g.z : 0.f,
                                            wb[q] & 8u ? g.w : 0.f);
              if (phase == 1) dh_store4<H16>(dH, (int64_t)u[q] * ldh4 + c, gm);
              else dh_add4<H16>(dH, (int64_t)u[q] * ldh4 + c, gm);
            }
          }
        }
      }
    }
  }
}

// The bf16-dH push with 8 columns (16 bytes of dH) per lane: a warp owns a
// whole dst row of up to 256 columns, so every edge is one pass of 16-byte
// stores (phase 1) or four bf16x2 reductions per lane (phase 2), and a
// lane's ReLU bits are one byte of the edge row's mask word.  SAGE only
// (no self term); dH row stride ldh = 8 * lanes used, dA row stride lda.
template <bool DA16>  // dA as bf16 (the dX epilogue's bf16 copy) instead of fp32
__global__ void __launch_bounds__(256) k_spmm_bwd16w(const int32_t* __restrict__ indptr,
                                                     const int32_t* __restrict__ indices,
                                                     const uint32_t* __restrict__ own, const int32_t* d_ndst,
                                                     const void* __restrict__ dA, int32_t lda,
                                                     __nv_bfloat16* __restrict__ dH, int32_t ldh, int32_t d,
                                                     int32_t aggr, int32_t phase, const uint32_t* __restrict__ bits,
                                                     int32_t bits_ld) {
  GNNV_PDL_ENTRY();
  const int n = *d_ndst;
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int c8 = lane, cols8 = ldh >> 3;
  const bool cok = c8 < cols8;
  for (int row = warp; row < n; row += nwarps) {
    const int beg = indptr[row], cnt = indptr[row + 1] - beg;
    const uint32_t mine = own[row];
    const uint32_t todo = (cnt >= 32 ? 0xffffffffu : ((1u << cnt) - 1u)) & (phase == 1 ? mine : ~mine);
    if (!todo) continue;  // warp-uniform (one row per warp)
    const float w = (aggr == GNNV_AGGR_MEAN && cnt) ? 1.f / (float)cnt : 1.f;
    float g[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (cok && 8 * c8 < d) {
      if (DA16) {
        const uint4 q = __ldg(reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(dA) + (int64_t)row * lda) + c8);
        const uint32_t qw[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const __nv_bfloat162 h2 = *reinterpret_cast<const __nv_bfloat162*>(&qw[j]);
          g[2 * j] = __low2float(h2) * w;
          g[2 * j + 1] = __high2float(h2) * w;
        }
      } else {
        const float* dAf = static_cast<const float*>(dA);
        const float4 a = __ldg(reinterpret_cast<const float4*>(dAf + (int64_t)row * lda) + 2 * c8);
        const float4 b = __ldg(reinterpret_cast<const float4*>(dAf + (int64_t)row * lda) + 2 * c8 + 1);
        g[0] = a.x * w; g[1] = a.y * w; g[2] = a.z * w; g[3] = a.w * w;
        g[4] = b.x * w; g[5] = b.y * w; g[6] = b.z * w; g[7] = b.w * w;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (8 * c8 + j >= d) g[j] = 0.f;
    }
    for (int e0 = 0; e0 < cnt; e0 += 32) {
      const int my = (e0 + lane < cnt) ? __ldg(indices + beg + e0 + lane) : 0;
      uint32_t pend = (todo >> e0) & (cnt - e0 >= 32 ? 0xffffffffu : ((1u << (cnt - e0)) - 1u));
      while (pend) {
        int u[4];
        uint32_t wb[4];
        int k = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int j = pend ? __ffs(pend) - 1 : 0;
          u[q] = __shfl_sync(0xffffffffu, my, j);
          if (pend) {
            pend &= pend - 1;
            k = q + 1;
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
          wb[q] = (bits && q < k && cok) ? (__ldg(bits + (int64_t)u[q] * bits_ld + (c8 >> 2)) >> ((c8 & 3) * 8)) : 0xFFu;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (q >= k || !cok) continue;
          uint32_t h[4];
#pragma unroll
          for (int j = 0; j < 4; ++j)
            h[j] = pack_bf16x2(wb[q] & (1u << (2 * j)) ? g[2 * j] : 0.f, wb[q] & (2u << (2 * j)) ? g[2 * j + 1] : 0.f);
          uint4* p = reinterpret_cast<uint4*>(dH + (int64_t)u[q] * ldh) + c8;
          if (phase == 1) {
            *p = make_uint4(h[0], h[1], h[2], h[3]);
          } else {  // one 16-byte bf16x8 reduction (REDG.ADD.BF16x8)
            asm volatile("red.global.add.noftz.v4.bf16x2 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(h[0]), "r"(h[1]),
                         "r"(h[2]), "r"(h[3])
                         : "memory");
          }
        }
      }
    }
  }
}

// w_v of the mean (1/c_v, 1/(c_v+1) for GCN, 0 for an empty row) or 1 (sum)
__device__ __forceinline__ float pull_weight(const int32_t* __restrict__ indptr, int v, bool mean, bool gcn) {
  if (!mean) return 1.f;
  const int denom = __ldg(indptr + v + 1) - __ldg(indptr + v) + (gcn ? 1 : 0);
  return denom ? 1.f / (float)denom : 0.f;
}

// The same transposed aggregation pulled per SRC row through the block's CSC
// (sampler: k_map counts, scan, k_csc_fill):
//   dH[u] = base[u] + relu'(H[u]) * sum_{(v,u)} w_v dA[v]   (+ the GCN self
// term w_u dA[u] for u < n_dst), base = the dX GEMM's dH_dst rows (SAGE,
// u < n_dst) or 0.  Every dH row is written once with coalesced stores, no
// atomics; dA (n_dst rows) is small and read from L2.  A warp takes 32 src
// rows: lane i first fetches row i's column range, first in-edge and its
// weight (independent loads, one round trip), then the warp's LPR-lane
// groups load U rows' first dA rows before storing any (most src rows have a
// single in-edge; further in-edges are added in column order).
template <int LPR, int NC, int U>
__global__ void __launch_bounds__(256) k_spmm_bwd_pull(const int32_t* __restrict__ colptr,
                                                       const int32_t* __restrict__ csc,
                                                       const int32_t* __restrict__ indptr, const int32_t* d_ndst,
                                                       const int32_t* d_nsrc, const float* __restrict__ dA,
                                                       int32_t lda, float* dH, int32_t ldh, int32_t d, int32_t kind,
                                                       int32_t aggr, const uint32_t* __restrict__ bits,
                                                       int32_t bits_ld) {
  GNNV_PDL_ENTRY();
  constexpr int RPW = 32 / LPR;
  static_assert(RPW * U <= 32 && 32 % (RPW * U) == 0, "row groups must tile the warp's 32 rows");
  const int n_dst = *d_ndst, n_src = *d_nsrc;
  const int vec = (d + 3) >> 2;
  const int lane = threadIdx.x & 31, sub = lane / LPR, sl = lane % LPR;
  const unsigned smask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (sub * LPR));
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int ldh4 = ldh >> 2, lda4 = lda >> 2;
  const float4* dA4 = reinterpret_cast<const float4*>(dA);
  float4* dH4 = reinterpret_cast<float4*>(dH);
  const bool gcn = kind == GNNV_KIND_GCN, mean = aggr == GNNV_AGGR_MEAN;
  for (int base = warp * 32; base < n_src; base += nwarps * 32) {
    // lane-parallel row metadata
    const int mu = base + lane;
    int mbeg = 0, mcnt = 0, mv = 0;
    float mw = 0.f;
    if (mu < n_src) {
      mbeg = __ldg(colptr + mu);
      mcnt = __ldg(colptr + mu + 1) - mbeg;
      if (mcnt) {
        mv = __ldg(csc + mbeg);
        mw = pull_weight(indptr, mv, mean, gcn);
      }
    }
    const float mws = (gcn && mu < n_dst) ? pull_weight(indptr, mu, mean, gcn) : 0.f;
#pragma unroll 1
    for (int j0 = 0; j0 < 32; j0 += RPW * U) {
      float4 acc[U][NC];
      int cnt[U], beg[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int j = j0 + q * RPW + sub;
        const int u = base + j;
        beg[q] = __shfl_sync(0xffffffffu, mbeg, j);
        cnt[q] = __shfl_sync(0xffffffffu, mcnt, j);
        const int v = __shfl_sync(0xffffffffu, mv, j);
        const float w = __shfl_sync(0xffffffffu, mw, j);
        const float ws = __shfl_sync(0xffffffffu, mws, j);
#pragma unroll
        for (int k = 0; k < NC; ++k) {
          const int c = k * LPR + sl;
          acc[q][k] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (u < n_src && c < vec) {
            if (cnt[q]) acc[q][k] = f4scale(__ldg(dA4 + (int64_t)v * lda4 + c), w);
            if (gcn && u < n_dst) acc[q][k] = f4add(acc[q][k], f4scale(__ldg(dA4 + (int64_t)u * lda4 + c), ws));
          }
        }
      }
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int u = base + j0 + q * RPW + sub;
        if (u >= n_src) continue;  // subgroup-uniform (one row per LPR lanes)
        // further in-edges (repeated src ids; hubs of the dst prefix collect
        // hundreds): fetched lane-parallel, broadcast, 4 dA rows in flight
        for (int e0 = 1; e0 < cnt[q]; e0 += LPR) {
          int my = 0;
          float myw = 0.f;
          if (e0 + sl < cnt[q]) {
            my = __ldg(csc + beg[q] + e0 + sl);
            myw = pull_weight(indptr, my, mean, gcn);
          }
          const int m = min(LPR, cnt[q] - e0);
          int jj = 0;
          for (; jj + 4 <= m; jj += 4) {
            int v4[4];
            float w4[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              v4[t] = __shfl_sync(smask, my, jj + t, LPR);
              w4[t] = __shfl_sync(smask, myw, jj + t, LPR);
            }
#pragma unroll
            for (int k = 0; k < NC; ++k) {
              const int c = k * LPR + sl;
              if (c < vec) {
                float4 a[4];
#pragma unroll
                for (int t = 0; t < 4; ++t) a[t] = __ldg(dA4 + (int64_t)v4[t] * lda4 + c);
#pragma unroll
                for (int t = 0; t < 4; ++t) acc[q][k] = f4add(acc[q][k], f4scale(a[t], w4[t]));
              }
            }
          }
          for (; jj < m; ++jj) {
            const int v = __shfl_sync(smask, my, jj, LPR);
            const float w = __shfl_sync(smask, myw, jj, LPR);
#pragma unroll
            for (int k = 0; k < NC; ++k) {
              const int c = k * LPR + sl;
              if (c < vec) acc[q][k] = f4add(acc[q][k], f4scale(__ldg(dA4 + (int64_t)v * lda4 + c), w));
            }
          }
        }
        const bool keep = !gcn && u < n_dst;  // the dX GEMM wrote dH_dst[u] (masked)
#pragma unroll
        for (int k = 0; k < NC; ++k) {
          const int c = k * LPR + sl;
          if (c >= ldh4 || (keep && c >= vec)) continue;
          float4 g = acc[q][k];
          if (c < vec) {
            g = mask_tail(g, c, d);
            if (bits) {
              const uint32_t m = __ldg(bits + (int64_t)u * bits_ld + (c >> 3)) >> ((c & 7) * 4);
              g = make_float4(m & 1u ? g.x : 0.f, m & 2u ? g.y : 0.f, m & 4u ? g.z : 0.f, m & 8u ? g.w : 0.f);
            }
            if (keep) g = f4add(dH4[(int64_t)u * ldh4 + c], g);
          }
          __stcs(dH4 + (int64_t)u * ldh4 + c, g);  // streaming: keep dA in L2; padding columns of whole rows: 0
        }
      }
    }
  }
}

static int spmm_grid(int64_t max_rows, int rows_per_warp) {
  const int64_t warps = ceil_div(std::max<int64_t>(max_rows, 1), rows_per_warp);
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(warps, 8), (int64_t)num_sms() * 16));
}

void launch_spmm_fwd(const int32_t* d_indptr, const int32_t* d_indices, const int32_t* d_ndst, int64_t max_dst,
                     const float* H, int32_t ldh, float* A, int32_t lda, int32_t d, int32_t kind, int32_t aggr,
                     cudaStream_t s, const int32_t* rowidx, const uint32_t* lastv) {
  const int vec = (d + 3) / 4;
#define GNNV_SPMM_FWD(LPR, RPWv)                                                                                  \
  do {                                                                                                            \
    const int grid = spmm_grid(max_dst, RPWv);                                                                    \
    if (rowidx && lastv)                                                                                          \
      launch_k(k_spmm_fwd<LPR, true, true>, grid, 256, 0, s, d_indptr, d_indices, d_ndst, H, ldh, A, lda, d, kind,  \
               aggr, rowidx, lastv);                                                                              \
    else if (rowidx)                                                                                              \
      launch_k(k_spmm_fwd<LPR, true, false>, grid, 256, 0, s, d_indptr, d_indices, d_ndst, H, ldh, A, lda, d, kind, \
               aggr, rowidx, (const uint32_t*)nullptr);                                                           \
    else if (lastv)                                                                                               \
      launch_k(k_spmm_fwd<LPR, false, true>, grid, 256, 0, s, d_indptr, d_indices, d_ndst, H, ldh, A, lda, d, kind, \
               aggr, (const int32_t*)nullptr, lastv);                                                             \
    else                                                                                                          \
      launch_k(k_spmm_fwd<LPR, false, false>, grid, 256, 0, s, d_indptr, d_indices, d_ndst, H, ldh, A, lda, d,      \
               kind, aggr, (const int32_t*)nullptr, (const uint32_t*)nullptr);                                    \
  } while (0)
  if (vec <= 8) {
    GNNV_SPMM_FWD(8, 4);
  } else if (vec <= 16) {
    GNNV_SPMM_FWD(16, 2);
  } else {
    GNNV_SPMM_FWD(32, 1);
  }
#undef GNNV_SPMM_FWD
  GNNV_CHECK_LAUNCH();
}

bool spmm_bwd_wide(int32_t ldh, int32_t lda, int32_t kind, bool dh_bf16) {
  return dh_bf16 && kind == GNNV_KIND_SAGE && ldh % 8 == 0 && ldh / 8 <= 32 && ldh / 8 > 16 && lda % 8 == 0 &&
         !env_on("GNNV_BWD_NARROW");
}

void launch_spmm_bwd(const int32_t* d_indptr, const int32_t* d_indices, const uint32_t* d_own, const int32_t* d_ndst,
                     int64_t max_dst, const float* dA, int32_t lda, void* dH, int32_t ldh, int32_t d, int32_t kind,
                     int32_t aggr, const uint32_t* bits, int32_t bits_ld, cudaStream_t s, bool dh_bf16, bool da_bf16) {
  const int ldh4 = ldh / 4;
  if (spmm_bwd_wide(ldh, lda, kind, dh_bf16)) {
    for (int phase = 1; phase <= 2; ++phase) {
      if (da_bf16)
        launch_k(k_spmm_bwd16w<true>, spmm_grid(max_dst, 1), 256, 0, s, d_indptr, d_indices, d_own, d_ndst,
                 (const void*)dA, lda, static_cast<__nv_bfloat16*>(dH), ldh, d, aggr, phase, bits, bits_ld);
      else
        launch_k(k_spmm_bwd16w<false>, spmm_grid(max_dst, 1), 256, 0, s, d_indptr, d_indices, d_own, d_ndst,
                 (const void*)dA, lda, static_cast<__nv_bfloat16*>(dH), ldh, d, aggr, phase, bits, bits_ld);
      GNNV_CHECK_LAUNCH();
    }
    return;
  }
  GNNV_REQUIRE(!da_bf16, GNNV_ERR_PARAM, "spmm_bwd: a bf16 dA needs the wide bf16 push");
  for (int phase = 1; phase <= 2; ++phase) {
#define GNNV_BWD(LPR, RPWv)                                                                                          \
  do {                                                                                                               \
    if (dh_bf16)                                                                                                     \
      launch_k(k_spmm_bwd<LPR, true>, spmm_grid(max_dst, RPWv), 256, 0, s, d_indptr, d_indices, d_own, d_ndst, dA,   \
               lda, dH, ldh, d, kind, aggr, phase, bits, bits_ld);                                                   \
    else                                                                                                             \
      launch_k(k_spmm_bwd<LPR, false>, spmm_grid(max_dst, RPWv), 256, 0, s, d_indptr, d_indices, d_own, d_ndst, dA,  \
               lda, dH, ldh, d, kind, aggr, phase, bits, bits_ld);                                                   \
  } while (0)
    if (ldh4 <= 8) GNNV_BWD(8, 4);
    else if (ldh4 <= 16) GNNV_BWD(16, 2);
    else GNNV_BWD(32, 1);
#undef GNNV_BWD
    GNNV_CHECK_LAUNCH();
  }
}

// The aggregation over bf16 source rows (the trainer's bf16 copy of a hidden
// layer's output): eight elements (16 bytes) per lane and
// unit, fp32 accumulation in the fp32 kernel's edge order, fp32 aggregate.
// d % 8 == 0, row stride ld16 elements (a multiple of 8).
__device__ __forceinline__ void add_bf16x8(float* acc, uint4 q) {
  const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    acc[2 * k] += __uint_as_float(w[k] << 16);
    acc[2 * k + 1] += __uint_as_float(w[k] & 0xFFFF0000u);
  }
}
template <int LPR, int IND>  // IND 0: rows of H; 1: rows rowidx[.] of H; 2: indices are H rows, the self row rowidx[row]
__global__ void __launch_bounds__(256, 8) k_spmm_fwd_h16(const int32_t* __restrict__ indptr,
                                                      const int32_t* __restrict__ indices, const int32_t* d_ndst,
                                                      const __nv_bfloat16* __restrict__ H, int32_t ld16,
                                                      float* __restrict__ A, int32_t lda, int32_t d, int32_t kind,
                                                      int32_t aggr, const int32_t* __restrict__ rowidx,
                                                      __nv_bfloat16* __restrict__ A16, int32_t lda16,
                                                      __nv_bfloat16* __restrict__ X16, int32_t ones_col) {
  GNNV_PDL_ENTRY();
  constexpr int RPW = 32 / LPR;
  const int n = *d_ndst;
  const int vec8 = (d + 7) >> 3;  // 8-element units; elements >= d are zero in H
  const int lane = threadIdx.x & 31, sub = lane / LPR, sl = lane % LPR;
  const unsigned smask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (sub * LPR));
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const uint4* H8 = reinterpret_cast<const uint4*>(H);
  const int ld8 = ld16 >> 3, lda4 = lda >> 2;
  for (int base = warp * RPW; base < n; base += nwarps * RPW) {
    const int row = base + sub;
    const bool active = row < n;
    const int beg = active ? indptr[row] : 0;
    const int cnt = active ? indptr[row + 1] - beg : 0;
    for (int c0 = 0; c0 < vec8; c0 += LPR) {
      const int c = c0 + sl;
      const bool cok = active && c < vec8;
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      if (kind == GNNV_KIND_GCN && cok)
        add_bf16x8(acc, __ldg(H8 + (int64_t)(IND ? __ldg(rowidx + row) : row) * ld8 + c));
      if (X16 && cok) {
        // the dst row's own (bf16) features with the ones column at
        // ones_col: the self operand of the layer's bf16 GEMMs (stride lda16)
        uint4 sv = __ldg(H8 + (int64_t)(IND ? __ldg(rowidx + row) : row) * ld8 + c);
        uint32_t* w = reinterpret_cast<uint32_t*>(&sv);
        const int oh = ones_col & 7;
        if (c == (ones_col >> 3))
          w[oh >> 1] = (oh & 1) ? ((w[oh >> 1] & 0xFFFFu) | 0x3F800000u) : ((w[oh >> 1] & 0xFFFF0000u) | 0x3F80u);
        uint4* xr = reinterpret_cast<uint4*>(X16) + (int64_t)row * (lda16 >> 3);
        xr[c] = sv;
        if (c == vec8 - 1 && (ones_col >> 3) == vec8) xr[vec8] = make_uint4(0x3F80u, 0u, 0u, 0u);
      }
      for (int e0 = 0; e0 < cnt; e0 += LPR) {
        int my = (e0 + sl < cnt) ? __ldg(indices + beg + e0 + sl) : 0;
        if (IND == 1) my = __ldg(rowidx + my);
        const int m = min(LPR, cnt - e0);
        int j = 0;
        for (; j + 4 <= m; j += 4) {
          const int u0 = __shfl_sync(smask, my, j, LPR), u1 = __shfl_sync(smask, my, j + 1, LPR);
          const int u2 = __shfl_sync(smask, my, j + 2, LPR), u3 = __shfl_sync(smask, my, j + 3, LPR);
          if (cok) {
            const uint4 h0 = __ldg(H8 + (int64_t)u0 * ld8 + c), h1 = __ldg(H8 + (int64_t)u1 * ld8 + c);
            const uint4 h2 = __ldg(H8 + (int64_t)u2 * ld8 + c), h3 = __ldg(H8 + (int64_t)u3 * ld8 + c);
            add_bf16x8(acc, h0);
            add_bf16x8(acc, h1);
            add_bf16x8(acc, h2);
            add_bf16x8(acc, h3);
          }
        }
        for (; j < m; ++j) {
          const int u = __shfl_sync(smask, my, j, LPR);
          if (cok) add_bf16x8(acc, __ldg(H8 + (int64_t)u * ld8 + c));
        }
      }
      if (cok) {
        if (aggr == GNNV_AGGR_MEAN) {
          const int denom = cnt + (kind == GNNV_KIND_GCN ? 1 : 0);
#pragma unroll
          for (int k = 0; k < 8; ++k) acc[k] = denom ? acc[k] / (float)denom : 0.f;
        }
        if (A) {
          float4* out = reinterpret_cast<float4*>(A) + (int64_t)row * lda4 + 2 * c;
          out[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
          if (2 * c + 1 < lda4) out[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
        }
        if (A16)  // the bf16 copy the layer's bf16 dW reads (gemm_dw16)
          reinterpret_cast<uint4*>(A16)[(int64_t)row * (lda16 >> 3) + c] =
              make_uint4(pack_bf16x2(acc[0], acc[1]), pack_bf16x2(acc[2], acc[3]), pack_bf16x2(acc[4], acc[5]),
                         pack_bf16x2(acc[6], acc[7]));
      }
    }
    if (active && A)  // padding float4s of the output row
      for (int c4 = 2 * vec8 + sl; c4 < lda4; c4 += LPR)
        reinterpret_cast<float4*>(A)[(int64_t)row * lda4 + c4] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

void launch_spmm_fwd_h16(const int32_t* d_indptr, const int32_t* d_indices, const int32_t* d_ndst, int64_t max_dst,
                         const void* H16, int32_t ld16, float* A, int32_t lda, int32_t d, int32_t kind, int32_t aggr,
                         cudaStream_t s, const int32_t* rowidx, void* A16, int32_t lda16, void* X16,
                         bool rows_direct) {
  const int vec8 = (d + 7) / 8;
  GNNV_REQUIRE(!A16 || (lda16 % 8 == 0 && lda16 >= 8 * vec8), GNNV_ERR_UNSUPPORTED,
               "spmm_fwd_h16: the bf16 output stride must be a multiple of 8 covering d");
  __nv_bfloat16* a16 = static_cast<__nv_bfloat16*>(A16);
  GNNV_REQUIRE(A || a16, GNNV_ERR_PARAM, "spmm_fwd_h16: no output");
  __nv_bfloat16* x16 = static_cast<__nv_bfloat16*>(X16);
  const int32_t ones_col = d;
  GNNV_REQUIRE(!x16 || (a16 && lda16 >= d + 1), GNNV_ERR_PARAM,
               "spmm_fwd_h16: the self copy shares the bf16 aggregate's stride, which must cover the ones column");
  GNNV_REQUIRE(ld16 % 8 == 0 && ld16 >= 8 * vec8 && lda % 4 == 0, GNNV_ERR_UNSUPPORTED,
               "spmm_fwd_h16: the bf16 row stride must be a multiple of 8 covering d");
  const __nv_bfloat16* H = static_cast<const __nv_bfloat16*>(H16);
#define GNNV_H16(LPR, RPWv)                                                                                          \
  do {                                                                                                               \
    if (rowidx && rows_direct)                                                                                       \
      launch_k(k_spmm_fwd_h16<LPR, 2>, spmm_grid(max_dst, RPWv), 256, 0, s, d_indptr, d_indices, d_ndst, H, ld16,    \
               A, lda, d, kind, aggr, rowidx, a16, lda16, x16, ones_col);                                            \
    else if (rowidx)                                                                                                 \
      launch_k(k_spmm_fwd_h16<LPR, 1>, spmm_grid(max_dst, RPWv), 256, 0, s, d_indptr, d_indices, d_ndst, H, ld16,    \
               A, lda, d, kind, aggr, rowidx, a16, lda16, x16, ones_col);                                            \
    else                                                                                                             \
      launch_k(k_spmm_fwd_h16<LPR, 0>, spmm_grid(max_dst, RPWv), 256, 0, s, d_indptr, d_indices, d_ndst, H,          \
               ld16, A, lda, d, kind, aggr, (const int32_t*)nullptr, a16, lda16, x16, ones_col);                     \
  } while (0)
  if (vec8 <= 8) GNNV_H16(8, 4);
  else if (vec8 <= 16) GNNV_H16(16, 2);
  else GNNV_H16(32, 1);
#undef GNNV_H16
  GNNV_CHECK_LAUNCH();
}

void launch_spmm_bwd_pull(const int32_t* d_colptr, const int32_t* d_csc, const int32_t* d_indptr,
                          const int32_t* d_ndst, const int32_t* d_nsrc, int64_t max_src, const float* dA, int32_t lda,
                          float* dH, int32_t ldh, int32_t d, int32_t kind, int32_t aggr, const uint32_t* bits,
                          int32_t bits_ld, cudaStream_t s) {
  const int ldh4 = ldh / 4;
  const int64_t rows = ceil_div(std::max<int64_t>(max_src, 1), 32) * 32;  // a warp per 32 rows
#define GNNV_PULL(LPR, NC, U)                                                                                     \
  launch_k(k_spmm_bwd_pull<LPR, NC, U>, spmm_grid(rows, 32), 256, 0, s, d_colptr, d_csc, d_indptr, d_ndst, d_nsrc, \
           dA, lda, dH, ldh, d, kind, aggr, bits, bits_ld)
  GNNV_REQUIRE(ldh4 <= kPullMaxLd / 4, GNNV_ERR_UNSUPPORTED, "spmm_bwd_pull: rows wider than 512 floats");
  if (ldh4 <= 8) {
    GNNV_PULL(8, 1, 4);
  } else if (ldh4 <= 16) {
    GNNV_PULL(16, 1, 4);
  } else if (ldh4 <= 32) {
    GNNV_PULL(32, 1, 4);
  } else if (ldh4 <= 64) {
    GNNV_PULL(32, 2, 2);
  } else {
    GNNV_PULL(32, 4, 1);
  }
#undef GNNV_PULL
  GNNV_CHECK_LAUNCH();
}


}  // namespace gnnv
