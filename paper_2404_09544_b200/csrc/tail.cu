// Fused output layer of the trainer's step: layer L forward (aggregate +
// combine), the softmax cross-entropy loss and layer L's backward in two
// launches instead of seven.
//
// Paper: Eq.1 Aggregate/Combine for the output layer and
// Algorithm 1 lines 5-8: the mini-batch loss and its backward.
// Same arithmetic as the per-kernel path (spmm.cu, layers.cu k_ce_loss, the
// tf32 layer GEMMs): readings Q11 (SAGE mean/sum), Q15 (empty row -> 0),
// Q22 (tf32 GEMM operands), Q23 (w_v = 0 for c_v = 0), Q25 (1/B_global).
//
// Why: the output layer works on the seeds only (n_0 = 4096 rows on
// products, C = 47 classes); its seven kernels are each a few microseconds
// of work behind a chain of memory round trips (~117 us serially, about
// twice that overlapped with the Eq.4 prefetch's sampler).  Here a CTA owns
// 32 seed rows end to end, and the three small GEMMs run on the tensor
// cores from shared memory (warp-level mma.sync m16n8k8 tf32: the tiles are
// 32 rows wide, far below a tcgen05 tile):
//
// k_tail_a (CTA = 32 seed rows, 16 warps, W^T staged in shared memory):
//   X = [H[v] | a_v], a_v = (1/c_v) sum_u H[u]      (warp per 2 rows, float4 lanes)
//   Z = X W + b                                    (mma, 32 x C8, K = 2d)
//   loss_v, dZ = (softmax(Z) - onehot) / B_global  (warp per 2 rows)
//   dX = dZ W^T:  dH[v] = relu'(H[v]) dX[:, :d],  dA_v = w_v dX[:, d:]  (mma)
//   dH[u] = relu'(H[u]) dA_v for every owner edge (v, u)  (k_spmm_bwd phase 1)
//   P_cta = X^T dZ, colsum dZ                      (mma; per-CTA partial dW, db)
// k_tail_b:
//   dH[u] += relu'(H[u]) dA_v for the other edges  (k_spmm_bwd phase 2)
//   dW, db = sum of the CTA partials in CTA order; loss = sum of partials / B
#include <cuda_bf16.h>

#include "common.cuh"

namespace gnnv {

constexpr int TA_ROWS = 32;   // seed rows per CTA
constexpr int TA_WARPS = 16;  // 512 threads

// fp32 bits as a tf32 operand: the tensor core reads the top 19 bits (the
// same truncation as the tcgen05 kind::tf32 layer GEMMs, reading Q22)
__device__ __forceinline__ uint32_t to_tf32(float x) { return __float_as_uint(x); }
// D(16x8) += A(16x8, row) B(8x8, col); fragments as in the PTX ISA for
// m16n8k8 .tf32: g = lane / 4, t = lane % 4;
//   a0 (g, t) a1 (g+8, t) a2 (g, t+4) a3 (g+8, t+4);  b0 (k=t, n=g) b1 (k=t+4, n=g);
//   d0 (g, 2t) d1 (g, 2t+1) d2 (g+8, 2t) d3 (g+8, 2t+1)
__device__ __forceinline__ void mma_tf32_16x8x8(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                                uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float4 f4add_(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ float4 f4mask(float4 g, uint32_t word, int col) {  // bits col..col+3 of word
  const uint32_t w = word >> (col & 31);
  return make_float4(w & 1u ? g.x : 0.f, w & 2u ? g.y : 0.f, w & 4u ? g.z : 0.f, w & 8u ? g.w : 0.f);
}

// shared-memory strides (floats): K + 4 and C8 + 4 keep the fragment loads
// conflict-free (4 g + t distinct banks)
struct TailSmem {
  int K, C8, xs, ws, zs;
  __host__ __device__ TailSmem(int d, int C) : K(2 * d), C8((C + 7) & ~7), xs(2 * d + 4), ws(2 * d + 4),
                                               zs(((C + 7) & ~7) + 4) {}
  __host__ __device__ size_t floats() const { return (size_t)TA_ROWS * xs + (size_t)C8 * ws + (size_t)TA_ROWS * zs; }
};

// CPL = float4 columns of a d-wide row per lane (d <= 128 CPL)
template <int CPL, bool B16>  // B16: dL/dH^{L-1} as bf16 + db partials (TailArgs::dH16)
__global__ void __launch_bounds__(TA_WARPS * 32, 1) k_tail_a(
    const int32_t* __restrict__ indptr, const int32_t* __restrict__ indices, const uint32_t* __restrict__ own,
    const int32_t* d_ndst, const float* __restrict__ H, int ldh, const uint32_t* __restrict__ hbits, int hbits_ld,
    const float* __restrict__ W, const float* __restrict__ bias, int d, int C, int aggr, float* __restrict__ A,
    int lda, float* __restrict__ Z, float* __restrict__ dZ, int ldz, const int32_t* __restrict__ F,
    const int32_t* __restrict__ labels, int n_global, float* dH, int ldg, float* dAs, float* __restrict__ part,
    float* __restrict__ loss_partial, float* __restrict__ zero, int64_t zero_n, __nv_bfloat16* __restrict__ dH16,
    float* __restrict__ db_part) {
  GNNV_PDL_ENTRY();
  __shared__ float s_db[512];  // dH16: this CTA's column sums of dL/dH^{L-1}
  if (B16)
    for (int c = threadIdx.x; c < d; c += blockDim.x) s_db[c] = 0.f;
  // the earlier layers' dW / db, accumulated atomically by their dW GEMMs
  // later in the step: cleared here instead of by memset nodes
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < zero_n; i += (int64_t)gridDim.x * blockDim.x)
    zero[i] = 0.f;
  extern __shared__ __align__(16) float sm[];
  const TailSmem L(d, C);
  const int K = L.K, C8 = L.C8;
  float* s_x = sm;                      // [32][xs]   X = [H | A] rows
  float* s_w = s_x + TA_ROWS * L.xs;    // [C8][ws]   W^T (zero columns c >= C)
  float* s_z = s_w + (size_t)C8 * L.ws; // [32][zs]   logits, then dZ
  __shared__ float s_loss[TA_WARPS];
  __shared__ uint32_t s_hb[TA_ROWS * 16];  // the seed rows' ReLU-bit words (d <= 512), for the dX pass
  const int n = *d_ndst;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int v0 = blockIdx.x * TA_ROWS;
  const int d4 = d >> 2;  // d % 4 == 0 (tail_supported)
  // ---- W^T into shared memory
  {  // warp w takes W rows k = w + 16 j, lanes the columns; 8 rows in flight
    for (int k0 = wid; k0 < K; k0 += 8 * TA_WARPS) {
      float w8[8][2];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int k = k0 + j * TA_WARPS;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = lane + 32 * h;
          w8[j][h] = (k < K && c < C) ? __ldg(W + (int64_t)k * C + c) : 0.f;
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int k = k0 + j * TA_WARPS;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = lane + 32 * h;
          if (k < K && c < C8) s_w[c * L.ws + k] = w8[j][h];
        }
      }
    }
  }
  // ---- X rows: warp w owns rows 2w, 2w+1 (ascending edge order, EB rows in flight)
  int my[2], cnt[2], yv[2];
  uint32_t ownm[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int r = 2 * wid + q, v = v0 + r;
    const bool ok = v < n;
    const int beg = ok ? indptr[v] : 0;
    cnt[q] = ok ? indptr[v + 1] - beg : 0;  // <= 32 (fanout <= 32)
    my[q] = lane < cnt[q] ? __ldg(indices + beg + lane) : 0;
    ownm[q] = ok ? own[v] : 0u;
    yv[q] = ok ? __ldg(labels + F[v]) : 0;
    if (lane < 16) s_hb[r * 16 + lane] = (ok && 32 * lane < d) ? __ldg(hbits + (int64_t)v * hbits_ld + lane) : 0u;
    float4 hs[CPL], ag[CPL];
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
      const int c4 = lane + 32 * j;
      hs[j] = (ok && c4 < d4) ? __ldg(reinterpret_cast<const float4*>(H + (int64_t)v * ldh) + c4)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
      ag[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    constexpr int EB = CPL <= 2 ? 8 : 4;  // neighbour rows in flight
    for (int e0 = 0; e0 < cnt[q]; e0 += EB) {
      float4 x[EB][CPL];
#pragma unroll
      for (int e = 0; e < EB; ++e) {
        const int u = __shfl_sync(0xffffffffu, my[q], (e0 + e) & 31);
#pragma unroll
        for (int j = 0; j < CPL; ++j) {
          const int c4 = lane + 32 * j;
          x[e][j] = (e0 + e < cnt[q] && c4 < d4) ? __ldg(reinterpret_cast<const float4*>(H + (int64_t)u * ldh) + c4)
                                                 : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
#pragma unroll
      for (int e = 0; e < EB; ++e)
        if (e0 + e < cnt[q]) {
#pragma unroll
          for (int j = 0; j < CPL; ++j) ag[j] = f4add_(ag[j], x[e][j]);
        }
    }
    if (aggr == GNNV_AGGR_MEAN) {
      const float den = (float)cnt[q];
#pragma unroll
      for (int j = 0; j < CPL; ++j)
        ag[j] = cnt[q] ? make_float4(ag[j].x / den, ag[j].y / den, ag[j].z / den, ag[j].w / den)
                       : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
      const int c4 = lane + 32 * j;
      if (c4 < d4) {
        reinterpret_cast<float4*>(s_x + r * L.xs)[c4] = hs[j];
        reinterpret_cast<float4*>(s_x + r * L.xs + d)[c4] = ag[j];
        if (ok) reinterpret_cast<float4*>(A + (int64_t)v * lda)[c4] = ag[j];
      }
    }
    if (ok)
      for (int c = d + lane; c < lda; c += 32) A[(int64_t)v * lda + c] = 0.f;
  }
  __syncthreads();
  // ---- Z = X W + b: 2 x (C8/8) tiles of 16 x 8, K = 2d
  {
    const int ntn = C8 / 8;
    for (int tile = wid; tile < 2 * ntn; tile += TA_WARPS) {
      const int m0 = (tile / ntn) * 16, n0 = (tile % ntn) * 8;
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      const float* xa = s_x + (m0 + g) * L.xs + t;
      const float* wb = s_w + (n0 + g) * L.ws + t;
#pragma unroll 4
      for (int k0 = 0; k0 < K; k0 += 8) {
        mma_tf32_16x8x8(acc, to_tf32(xa[k0]), to_tf32(xa[8 * L.xs + k0]), to_tf32(xa[k0 + 4]),
                        to_tf32(xa[8 * L.xs + k0 + 4]), to_tf32(wb[k0]), to_tf32(wb[k0 + 4]));
      }
      const int c = n0 + 2 * t;
      const float b0 = c < C ? __ldg(bias + c) : 0.f, b1 = c + 1 < C ? __ldg(bias + c + 1) : 0.f;
      s_z[(m0 + g) * L.zs + c] = acc[0] + b0;
      s_z[(m0 + g) * L.zs + c + 1] = acc[1] + b1;
      s_z[(m0 + g + 8) * L.zs + c] = acc[2] + b0;
      s_z[(m0 + g + 8) * L.zs + c + 1] = acc[3] + b1;
    }
  }
  __syncthreads();
  // ---- softmax cross-entropy (as k_ce_loss); dZ replaces Z in s_z
  const float inv = 1.f / (float)n_global;
  float lsum = 0.f;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int r = 2 * wid + q, v = v0 + r;
    float* zr = s_z + r * L.zs;
    if (v >= n) {  // padding rows: dZ = 0 (they still enter the dW MMA)
      for (int c = lane; c < C8; c += 32) zr[c] = 0.f;
      continue;
    }
    float z[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) z[h] = lane + 32 * h < C ? zr[lane + 32 * h] : -INFINITY;
    const float m = warp_max(fmaxf(z[0], z[1]));
    float se = 0.f;
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (lane + 32 * h < C) se += expf(z[h] - m);
    se = warp_sum(se);
    const int y = yv[q];
    const float zy = zr[y];
    if (lane == 0) lsum += (m + logf(se)) - zy;
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = lane + 32 * h;
      const float gz = c < C ? (expf(z[h] - m) / se - (c == y ? 1.f : 0.f)) * inv : 0.f;
      if (c < ldz) {
        Z[(int64_t)v * ldz + c] = c < C ? z[h] : 0.f;
        dZ[(int64_t)v * ldz + c] = gz;
      }
      if (c < C8) zr[c] = gz;
    }
  }
  if (lane == 0) s_loss[wid] = lsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int i = 0; i < TA_WARPS; ++i) s += s_loss[i];
    loss_partial[blockIdx.x] = s;
  }
  // ---- dX = dZ W^T (32 x 2d, K = C8): self columns -> dH[v] (masked),
  //      neighbour columns -> w_v dA_v (global scratch, L2)
  {
    const int ntn = K / 8;
    for (int tile = wid; tile < 2 * ntn; tile += TA_WARPS) {
      const int m0 = (tile / ntn) * 16, n0 = (tile % ntn) * 8;
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      const float* za = s_z + (m0 + g) * L.zs + t;
      for (int k0 = 0; k0 < C8; k0 += 8) {
        const float* wb = s_w + (k0 + t) * L.ws + n0 + g;  // B[k = c][n = col] = W^T[c][col]
        mma_tf32_16x8x8(acc, to_tf32(za[k0]), to_tf32(za[8 * L.zs + k0]), to_tf32(za[k0 + 4]),
                        to_tf32(za[8 * L.zs + k0 + 4]), to_tf32(wb[0]), to_tf32(wb[4 * L.ws]));
      }
      const int col = n0 + 2 * t;
      float cs0 = 0.f, cs1 = 0.f;  // dH16: this lane's part of the tile's column sums
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = m0 + g + 8 * h, v = v0 + r;
        if (v >= n) continue;
        const float x0 = acc[2 * h], x1 = acc[2 * h + 1];
        if (col < d) {
          const uint32_t word = s_hb[r * 16 + (col >> 5)];
          const uint32_t b = word >> (col & 31);
          const float m0 = b & 1u ? x0 : 0.f, m1 = b & 2u ? x1 : 0.f;
          if (B16) {
            const __nv_bfloat162 hv = __floats2bfloat162_rn(m0, m1);
            *reinterpret_cast<__nv_bfloat162*>(dH16 + (int64_t)v * ldg + col) = hv;
            cs0 += m0;
            cs1 += m1;
          } else {
            *reinterpret_cast<float2*>(dH + (int64_t)v * ldg + col) = make_float2(m0, m1);
          }
        } else {  // scaled by w_v by the row's warp below
          *reinterpret_cast<float2*>(dAs + (int64_t)v * d + (col - d)) = make_float2(x0, x1);
        }
      }
      if (B16 && col < d) {  // tile-uniform: sum the 8 row groups (lane bits 2..4), one add per column
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
          cs0 += __shfl_xor_sync(0xffffffffu, cs0, o);
          cs1 += __shfl_xor_sync(0xffffffffu, cs1, o);
        }
        if (g == 0) {
          atomicAdd(&s_db[col], cs0);
          atomicAdd(&s_db[col + 1], cs1);
        }
      }
    }
  }
  __syncthreads();
  // ---- owner edges store w_v dA_v into their row (k_spmm_bwd phase 1);
  //      padding columns of the seeds' own dH rows
  float4 dbs[CPL];
#pragma unroll
  for (int j = 0; j < CPL; ++j) dbs[j] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int r = 2 * wid + q, v = v0 + r;
    if (v >= n) continue;
    for (int c = d + lane; c < ldg; c += 32) {
      if (B16) dH16[(int64_t)v * ldg + c] = __float2bfloat16_rn(0.f);
      else dH[(int64_t)v * ldg + c] = 0.f;
    }
    const float w = aggr == GNNV_AGGR_MEAN ? (cnt[q] ? 1.f / (float)cnt[q] : 0.f) : 1.f;
    float4 da[CPL];
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
      const int c4 = lane + 32 * j;
      if (c4 < d4) {
        const float4 a = reinterpret_cast<const float4*>(dAs + (int64_t)v * d)[c4];
        da[j] = make_float4(a.x * w, a.y * w, a.z * w, a.w * w);
        reinterpret_cast<float4*>(dAs + (int64_t)v * d)[c4] = da[j];  // k_tail_b pushes the scaled rows
      }
    }
    const uint32_t mine = ownm[q] & (cnt[q] >= 32 ? 0xffffffffu : ((1u << cnt[q]) - 1u));
    constexpr int OB = CPL <= 2 ? 16 : 8;  // owner edges whose mask words are loaded together
    for (uint32_t o = mine; o;) {
      int us[OB], nb = 0;
#pragma unroll
      for (int e = 0; e < OB; ++e) {
        us[e] = 0;
        if (o) {
          us[e] = __shfl_sync(0xffffffffu, my[q], __ffs(o) - 1);
          o &= o - 1;
          nb = e + 1;
        }
      }
      uint32_t wd[OB][CPL];
#pragma unroll
      for (int e = 0; e < OB; ++e)
#pragma unroll
        for (int j = 0; j < CPL; ++j) {
          const int c4 = lane + 32 * j;
          wd[e][j] = (e < nb && c4 < d4) ? __ldg(hbits + (int64_t)us[e] * hbits_ld + ((4 * c4) >> 5)) : 0u;
        }
#pragma unroll
      for (int e = 0; e < OB; ++e) {
        if (e >= nb) break;
#pragma unroll
        for (int j = 0; j < CPL; ++j) {
          const int c4 = lane + 32 * j;
          if (c4 >= d4) continue;
          const float4 m = f4mask(da[j], wd[e][j], 4 * c4);
          if (B16) {
            const __nv_bfloat162 lo = __floats2bfloat162_rn(m.x, m.y), hi = __floats2bfloat162_rn(m.z, m.w);
            reinterpret_cast<uint2*>(dH16 + (int64_t)us[e] * ldg)[c4] =
                make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
            dbs[j] = f4add_(dbs[j], m);
          } else {
            reinterpret_cast<float4*>(dH + (int64_t)us[e] * ldg)[c4] = m;
          }
        }
        for (int c = d + lane; c < ldg; c += 32) {
          if (B16) dH16[(int64_t)us[e] * ldg + c] = __float2bfloat16_rn(0.f);
          else dH[(int64_t)us[e] * ldg + c] = 0.f;
        }
      }
    }
  }
  if (B16) {  // this CTA's column sums -> db_part[blockIdx.x]
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
      const int c4 = lane + 32 * j;
      if (c4 < d4) {
        atomicAdd(&s_db[4 * c4 + 0], dbs[j].x);
        atomicAdd(&s_db[4 * c4 + 1], dbs[j].y);
        atomicAdd(&s_db[4 * c4 + 2], dbs[j].z);
        atomicAdd(&s_db[4 * c4 + 3], dbs[j].w);
      }
    }
    __syncthreads();
    for (int c = threadIdx.x; c < d; c += blockDim.x) db_part[(int64_t)blockIdx.x * d + c] = s_db[c];
  }
  // ---- per-CTA partials: P = X^T dZ (2d x C8, K = 32 rows) and colsum dZ
  {
    float* P = part + (size_t)blockIdx.x * ((size_t)K * C + C);
    const int ntn = C8 / 8, ntm = K / 16;
    for (int tile = wid; tile < ntm * ntn; tile += TA_WARPS) {
      const int m0 = (tile / ntn) * 16, n0 = (tile % ntn) * 8;
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int k0 = 0; k0 < TA_ROWS; k0 += 8) {
        const float* xa = s_x + (k0 + t) * L.xs + m0 + g;  // A[m = col][k = row] = X[row][col]
        const float* zb = s_z + (k0 + t) * L.zs + n0 + g;  // B[k = row][n = c] = dZ[row][c]
        mma_tf32_16x8x8(acc, to_tf32(xa[0]), to_tf32(xa[8]), to_tf32(xa[4 * L.xs]), to_tf32(xa[4 * L.xs + 8]),
                        to_tf32(zb[0]), to_tf32(zb[4 * L.zs]));
      }
      const int c = n0 + 2 * t;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int k = m0 + g + 8 * h;
        if (c < C) P[(size_t)k * C + c] = acc[2 * h];
        if (c + 1 < C) P[(size_t)k * C + c + 1] = acc[2 * h + 1];
      }
    }
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
      float s = 0.f;
      for (int r = 0; r < TA_ROWS; ++r) s += s_z[r * L.zs + c];
      P[(size_t)K * C + c] = s;
    }
  }
}

// blocks [0, push_blocks): warp per seed row, its non-owner edges' pushes;
// the rest: thread per element of [dW | db], the CTA partials summed in CTA
// order (deterministic); block 0 warp 0 also reduces the loss
template <int CPL, bool B16>  // B16: dL/dH^{L-1} as bf16 + db partials (TailArgs::dH16)
__global__ void __launch_bounds__(256) k_tail_b(const int32_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                                                const uint32_t* __restrict__ own, const int32_t* d_ndst, int push_blocks,
                                                const uint32_t* __restrict__ hbits, int hbits_ld, int d,
                                                const float* __restrict__ dAs, float* dH, int ldg,
                                                const float* __restrict__ part, int nparts, int K, int C, float* dW,
                                                float* db, const float* __restrict__ loss_partial, int n_global,
                                                float* d_loss, __nv_bfloat16* __restrict__ dH16,
                                                float* __restrict__ db_part, int db_base) {
  GNNV_PDL_ENTRY();
  const int n = *d_ndst;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int used = (n + TA_ROWS - 1) / TA_ROWS;  // CTAs of k_tail_a that had rows
  if (blockIdx.x == 0 && wid == 0) {
    float s = 0.f;
    for (int i = lane; i < used; i += 32) s += loss_partial[i];
    s = warp_sum(s);
    if (lane == 0) *d_loss = s * (1.f / (float)n_global);
  }
  if ((int)blockIdx.x < push_blocks) {
    __shared__ float4 s_dbw[8][128];  // dH16: per-warp column sums (d <= 512)
    const int v = blockIdx.x * 8 + wid;
    const int d4 = d >> 2;
    float4 dbs[CPL];
#pragma unroll
    for (int j = 0; j < CPL; ++j) dbs[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    const int beg = v < n ? indptr[v] : 0, cnt = v < n ? indptr[v + 1] - beg : 0;
    const uint32_t rest = v < n ? ~own[v] & (cnt >= 32 ? 0xffffffffu : ((1u << cnt) - 1u)) : 0u;
    if (rest) {
      const int my = lane < cnt ? __ldg(indices + beg + lane) : 0;
      float4 da[CPL];
#pragma unroll
      for (int j = 0; j < CPL; ++j) {
        const int c4 = lane + 32 * j;
        da[j] = c4 < d4 ? reinterpret_cast<const float4*>(dAs + (int64_t)v * d)[c4] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      for (uint32_t o = rest; o; o &= o - 1) {
        const int u = __shfl_sync(0xffffffffu, my, __ffs(o) - 1);
#pragma unroll
        for (int j = 0; j < CPL; ++j) {
          const int c4 = lane + 32 * j;
          if (c4 >= d4) continue;
          const float4 m = f4mask(da[j], __ldg(hbits + (int64_t)u * hbits_ld + ((4 * c4) >> 5)), 4 * c4);
          if (B16) {
            uint2* p = reinterpret_cast<uint2*>(dH16 + (int64_t)u * ldg) + c4;  // one bf16x4 reduction
            const __nv_bfloat162 lo = __floats2bfloat162_rn(m.x, m.y), hi = __floats2bfloat162_rn(m.z, m.w);
            asm volatile("red.global.add.noftz.v2.bf16x2 [%0], {%1, %2};" ::"l"(p),
                         "r"(*reinterpret_cast<const uint32_t*>(&lo)), "r"(*reinterpret_cast<const uint32_t*>(&hi))
                         : "memory");
            dbs[j] = f4add_(dbs[j], m);
          } else {
            atomicAdd(reinterpret_cast<float4*>(dH + (int64_t)u * ldg) + c4, m);
          }
        }
      }
    }
    if (!B16) return;
    // this block's column sums -> db_part[db_base + blockIdx.x], warps added in order
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
      const int c4 = lane + 32 * j;
      if (c4 < d4) s_dbw[wid][c4] = dbs[j];
    }
    __syncthreads();
    for (int c4 = threadIdx.x; c4 < d4; c4 += blockDim.x) {
      float4 t = s_dbw[0][c4];
      for (int w = 1; w < 8; ++w) t = f4add_(t, s_dbw[w][c4]);
      reinterpret_cast<float4*>(db_part + (int64_t)(db_base + blockIdx.x) * d)[c4] = t;
    }
    return;
  }
  const int i = (blockIdx.x - push_blocks) * blockDim.x + threadIdx.x;
  const int tot = K * C + C;
  if (i >= tot) return;
  float s = 0.f;
  for (int p = 0; p < used && p < nparts; ++p) s += part[(size_t)p * tot + i];
  if (i < K * C) dW[i] = s;
  else db[i - K * C] = s;
}

bool tail_supported(int kind, int d, int C, int fanout0) {
  return kind == GNNV_KIND_SAGE && d >= 8 && d % 8 == 0 && d <= 512 && C >= 1 && C <= 64 && fanout0 <= 32 &&
         TailSmem(d, C).floats() * sizeof(float) <= 220 * 1024;
}

int tail_db_parts(int64_t max_dst) {
  return (int)(ceil_div(std::max<int64_t>(max_dst, 1), TA_ROWS) + ceil_div(std::max<int64_t>(max_dst, 1), 8));
}

size_t tail_partial_floats(int64_t max_dst, int d, int C) {
  return (size_t)ceil_div(std::max<int64_t>(max_dst, 1), TA_ROWS) * ((size_t)2 * d * C + C);
}

template <int CPL, bool B16>
static void launch_tail_cpl(const TailArgs& a, cudaStream_t s, Timeline* tl, const std::string& sfx) {
  const size_t smem = TailSmem(a.d, a.C).floats() * sizeof(float);
  static size_t attr = 0;
  if (smem > attr) {
    GNNV_TRY_CUDA(cudaFuncSetAttribute(k_tail_a<CPL, B16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = smem;
  }
  const int ga = (int)ceil_div(std::max<int64_t>(a.max_dst, 1), TA_ROWS);
  GNNV_REQUIRE(ga <= 4096, GNNV_ERR_PARAM, "output layer: too many seed rows for the loss partials");
  GNNV_REQUIRE(!B16 || (a.db_part && a.d <= 512), GNNV_ERR_PARAM, "output layer: bf16 dH needs the db partials");
  if (tl) tl->mark(s, "tail_a" + sfx);
  launch_k(k_tail_a<CPL, B16>, ga, TA_WARPS * 32, smem, s, a.indptr, a.indices, a.own, a.d_ndst, a.H, a.ldh, a.hbits,
           a.hbits_ld, a.W, a.bias, a.d, a.C, a.aggr, a.A, a.lda, a.Z, a.dZ, a.ldz, a.F, a.labels, a.n_global, a.dH,
           a.ldg, a.dA, a.part, a.loss_partial, a.zero, a.zero ? a.zero_n : (int64_t)0,
           static_cast<__nv_bfloat16*>(a.dH16), a.db_part);
  GNNV_CHECK_LAUNCH();
  const int push_blocks = (int)ceil_div(std::max<int64_t>(a.max_dst, 1), 8);
  const int K = 2 * a.d;
  const int red_blocks = (int)ceil_div((int64_t)K * a.C + a.C, 256);
  if (tl) tl->mark(s, "tail_b" + sfx);
  launch_k(k_tail_b<CPL, B16>, push_blocks + red_blocks, 256, 0, s, a.indptr, a.indices, a.own, a.d_ndst, push_blocks,
           a.hbits, a.hbits_ld, a.d, a.dA, a.dH, a.ldg, a.part, ga, K, a.C, a.dW, a.db, a.loss_partial, a.n_global,
           a.d_loss, static_cast<__nv_bfloat16*>(a.dH16), a.db_part, ga);
  GNNV_CHECK_LAUNCH();
}
template <int CPL>
static void launch_tail_cpl(const TailArgs& a, cudaStream_t s, Timeline* tl, const std::string& sfx) {
  if (a.dH16) launch_tail_cpl<CPL, true>(a, s, tl, sfx);
  else launch_tail_cpl<CPL, false>(a, s, tl, sfx);
}

void launch_tail(const TailArgs& a, cudaStream_t s, Timeline* tl, const std::string& sfx) {
  const int cpl = (a.d / 4 + 31) / 32;
  switch (cpl) {
    case 1: return launch_tail_cpl<1>(a, s, tl, sfx);
    case 2: return launch_tail_cpl<2>(a, s, tl, sfx);
    case 3: case 4: return launch_tail_cpl<4>(a, s, tl, sfx);
  }
  GNNV_REQUIRE(false, GNNV_ERR_UNSUPPORTED, "output layer: width");
}

}  // namespace gnnv
