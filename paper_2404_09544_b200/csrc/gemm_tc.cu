// Dense transform of the GNN layer on the 5th-generation tensor cores
// (tcgen05, sm_100a): bf16 operands (reading Q18: RNE-rounded from the fp32
// activations/weights), fp32 accumulation in TMEM.
//
// Paper: Eq.1 Combine; Algorithm 1 lines 6 and 8.
//   fwd : Y  = act([X1 | X2] W + b)          M = n_dst rows (device-side)
//   dX  : [Y1 | Y2] = G W^T
//   dW  : [dW ; db] = [X1 | X2 | 1]^T G      long reduction over the rows,
//         split over CTAs, fixed-order reduction (deterministic)
//
// Why a producer-converts design (no TMA for the activations): the
// activations are fp32 in HBM (the SpMM that produces them stays fp32), so
// every element is read once by four producer warps, rounded to bf16 and
// stored straight into the UMMA canonical K-major SWIZZLE_NONE layout (8x16B
// core matrices), transposing on the fly for dW.  The weights are tiny: a
// prep kernel writes them once per call as a ready-made bf16 smem image that
// one thread streams per stage with cp.async.bulk (SASS UBLKCP) completing on
// the stage's mbarrier.  One elected thread of warp 4 issues tcgen05.mma
// (M=128, N<=256, K=16) and commits to the stage's "empty" barrier; the
// accumulator tile lives in TMEM and the producer warps drain it with
// tcgen05.ld for the epilogue (bias, ReLU, zero padding / split partials).
//
// Layout of one operand stage (R rows, BK = 64 bf16): byte offset of
// (row r, k) = (k/8) * (R*16) + r*16 + (k%8)*2, i.e. LBO (K direction) =
// R*16 bytes, SBO (8-row groups) = 128 bytes.
#include <cuda_bf16.h>

#include "common.cuh"

namespace gnnv {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int STAGES = 2;
constexpr int NTHREADS = 160;  // warps 0-3 producers/epilogue, warp 4 MMA + TMEM owner
constexpr int A_STAGE_BYTES = BM * BK * 2;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_NONE, sm100 version 1.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// kind::f16 instruction descriptor: D=f32, A=B=bf16, K-major, M=128, N.
__device__ __forceinline__ uint32_t umma_idesc(uint32_t n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ uint4 pack8(const float* f) {
  return make_uint4(pack_bf16(f[0], f[1]), pack_bf16(f[2], f[3]), pack_bf16(f[4], f[5]), pack_bf16(f[6], f[7]));
}
__device__ __forceinline__ void st_shared_16(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

__device__ __forceinline__ float4 ld4_masked(const float* p, int valid) {
  // valid: how many of the 4 elements are in range (0..4)
  if (valid <= 0) return make_float4(0.f, 0.f, 0.f, 0.f);
  float4 v = __ldg(reinterpret_cast<const float4*>(p));
  if (valid < 4) {
    if (valid < 2) v.y = 0.f;
    if (valid < 3) v.z = 0.f;
    v.w = 0.f;
    if (valid < 1) v.x = 0.f;
  }
  return v;
}

// ------------------------------------------------------------ policies
// Row-major fp32 operand split over two sources in a padded k' space:
// k' in [0, K1p) -> X1 col k' (valid < K1); [K1p, 2 K1p) -> X2 col k'-K1p.
struct SplitRows {
  const float *X1, *X2;
  int ld1, ld2, K1, K1p;
  __device__ __forceinline__ float4 load4(int64_t m, int k4) const {  // k4: multiple of 4
    if (k4 < K1p) return ld4_masked(X1 + m * ld1 + k4, K1 - k4);
    if (X2) {
      const int kk = k4 - K1p;
      if (kk < K1p) return ld4_masked(X2 + m * ld2 + kk, K1 - kk);
    }
    return make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __device__ __forceinline__ float load1(int64_t m, int k) const {
    if (k < K1p) return k < K1 ? __ldg(X1 + m * ld1 + k) : 0.f;
    if (X2) {
      const int kk = k - K1p;
      if (kk < K1) return __ldg(X2 + m * ld2 + kk);
    }
    return 0.f;
  }
};

struct FwdPolicy {
  static constexpr int MT = 1;
  SplitRows x;
  const __nv_bfloat16* wimg;  // [nkb][BN*BK] smem images
  const float* bias;
  float* Y;
  int ldy, N, BN, nkb;
  bool relu;
  const int32_t* dM;
  int M, m0;
  __device__ bool setup() {
    M = *dM;
    m0 = blockIdx.x * BM;
    return m0 < M;
  }
  __device__ int kb_begin() const { return 0; }
  __device__ int kb_end() const { return nkb; }
  __device__ int full_count() const { return 128 + 1; }
  __device__ void produce(int kb, uint8_t* sA, uint8_t* sB, uint64_t* full, int t) const {
    if (t == 0) {
      const uint32_t bytes = (uint32_t)BN * BK * 2;
      mbar_arrive_tx(full, bytes);
      bulk_g2s(sB, wimg + (size_t)kb * BN * BK, bytes, full);
    }
    const int64_t m = (int64_t)m0 + t;
    const uint32_t base = smem_u32(sA) + t * 16;
    const bool ok = m < M;
#pragma unroll
    for (int kc = 0; kc < 8; ++kc) {
      const int k4 = kb * BK + kc * 8;
      float f[8];
      float4 a = ok ? x.load4(m, k4) : make_float4(0.f, 0.f, 0.f, 0.f);
      float4 b = ok ? x.load4(m, k4 + 4) : make_float4(0.f, 0.f, 0.f, 0.f);
      f[0] = a.x, f[1] = a.y, f[2] = a.z, f[3] = a.w, f[4] = b.x, f[5] = b.y, f[6] = b.z, f[7] = b.w;
      st_shared_16(base + kc * (BM * 16), pack8(f));
    }
  }
  __device__ void epilogue(int row, int mt, int c, const float* v) const {
    const int64_t m = (int64_t)m0 + row;
    if (m >= M) return;
#pragma unroll
    for (int j = 0; j < 16; j += 4) {
      const int n = c + j;
      if (n >= ldy) break;
      float o[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int nn = n + e;
        float val = 0.f;
        if (nn < N) {
          val = v[j + e] + __ldg(bias + nn);
          if (relu) val = fmaxf(val, 0.f);
        }
        o[e] = val;
      }
      *reinterpret_cast<float4*>(Y + m * ldy + n) = make_float4(o[0], o[1], o[2], o[3]);
    }
  }
};

struct DxPolicy {
  static constexpr int MT = 1;
  const float* G;
  int ldg, K;  // K = d_out of the layer (reduction)
  const __nv_bfloat16* wimg;  // [ntiles][nkb][BN*BK]
  float *Y1, *Y2;
  int ld1, ld2, BN, nkb;
  const int32_t* dM;
  int M, m0, n0;
  __device__ bool setup() {
    M = *dM;
    m0 = blockIdx.x * BM;
    n0 = blockIdx.y * BN;
    return m0 < M;
  }
  __device__ int kb_begin() const { return 0; }
  __device__ int kb_end() const { return nkb; }
  __device__ int full_count() const { return 128 + 1; }
  __device__ void produce(int kb, uint8_t* sA, uint8_t* sB, uint64_t* full, int t) const {
    if (t == 0) {
      const uint32_t bytes = (uint32_t)BN * BK * 2;
      mbar_arrive_tx(full, bytes);
      bulk_g2s(sB, wimg + ((size_t)blockIdx.y * nkb + kb) * BN * BK, bytes, full);
    }
    const int64_t m = (int64_t)m0 + t;
    const uint32_t base = smem_u32(sA) + t * 16;
    const bool ok = m < M;
#pragma unroll
    for (int kc = 0; kc < 8; ++kc) {
      const int k4 = kb * BK + kc * 8;
      float f[8];
      float4 a = ok ? ld4_masked(G + m * ldg + k4, K - k4) : make_float4(0.f, 0.f, 0.f, 0.f);
      float4 b = ok ? ld4_masked(G + m * ldg + k4 + 4, K - k4 - 4) : make_float4(0.f, 0.f, 0.f, 0.f);
      f[0] = a.x, f[1] = a.y, f[2] = a.z, f[3] = a.w, f[4] = b.x, f[5] = b.y, f[6] = b.z, f[7] = b.w;
      st_shared_16(base + kc * (BM * 16), pack8(f));
    }
  }
  __device__ void epilogue(int row, int mt, int c, const float* v) const {
    const int64_t m = (int64_t)m0 + row;
    if (m >= M) return;
#pragma unroll
    for (int j = 0; j < 16; j += 4) {
      const int col = n0 + c + j;
      const float4 o = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      if (col < ld1) {
        *reinterpret_cast<float4*>(Y1 + m * ld1 + col) = o;
      } else if (Y2 && col - ld1 < ld2) {
        *reinterpret_cast<float4*>(Y2 + m * ld2 + (col - ld1)) = o;
      }
    }
  }
};

// dW: MMA rows = feature index i' (padded split space + bias row), MMA cols =
// n (d_out), reduction over graph rows m.  Both operands are transposed on
// load (thread = one row of the smem tile, 64 coalesced scalar loads).
struct DwPolicy {
  static constexpr int MT = 2;  // 128-row i'-tiles per CTA (shares the G tile)
  SplitRows x;
  int rows_p;  // padded i' rows incl. the bias row at index bias_row
  int bias_row;
  const float* G;
  int ldg, N, BN;
  const int32_t* dM;
  int splits;
  float* partial;  // [splits][itiles*128][BN]
  int itiles;
  int M, i0, kb0, kb1;
  __device__ bool setup() {
    M = *dM;
    i0 = blockIdx.y * (BM * MT);
    const int nkb = (M + BK - 1) / BK;
    const int per = (nkb + splits - 1) / splits;
    kb0 = min(nkb, (int)blockIdx.x * per);
    kb1 = min(nkb, kb0 + per);
    return true;  // every CTA writes its partial (zeros if its range is empty)
  }
  __device__ int kb_begin() const { return kb0; }
  __device__ int kb_end() const { return kb1; }
  __device__ int full_count() const { return 128; }
  __device__ void produce(int kb, uint8_t* sA, uint8_t* sB, uint64_t*, int t) const {
    const int mb = kb * BK;
    // A tiles: rows i' = i0 + mt*128 + t, 64 consecutive m
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int i = i0 + mt * BM + t;
      const uint32_t base = smem_u32(sA + mt * A_STAGE_BYTES) + t * 16;
      for (int kc = 0; kc < 8; ++kc) {
        float f[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int m = mb + kc * 8 + e;
          float val = 0.f;
          if (m < M) val = (i == bias_row) ? 1.f : x.load1(m, i);
          f[e] = val;
        }
        st_shared_16(base + kc * (BM * 16), pack8(f));
      }
    }
    // B tile: rows n, 64 consecutive m
    for (int n = t; n < BN; n += 128) {
      const uint32_t base = smem_u32(sB) + n * 16;
      for (int kc = 0; kc < 8; ++kc) {
        float f[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int m = mb + kc * 8 + e;
          f[e] = (m < M && n < N) ? __ldg(G + (int64_t)m * ldg + n) : 0.f;
        }
        st_shared_16(base + kc * (BN * 16), pack8(f));
      }
    }
  }
  __device__ void epilogue(int row, int mt, int c, const float* v) const {
    const int i = i0 + mt * BM + row;
    float* dst = partial + ((int64_t)blockIdx.x * (itiles * BM) + i) * BN + c;
#pragma unroll
    for (int j = 0; j < 16; j += 4) *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
  }
};

template <class P>
__global__ void __launch_bounds__(NTHREADS, 1) k_tc_gemm(P p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int BN = p.BN;
  constexpr int MT = P::MT;
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * MT * A_STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + (size_t)STAGES * BN * BK * 2);
  uint64_t* empty = full + STAGES;
  uint64_t* accf = empty + STAGES;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(accf + 1);
  if (!p.setup()) return;  // block-uniform
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kb0 = p.kb_begin(), kb1 = p.kb_end();
  const int nkb = kb1 - kb0;
  uint32_t ncols = 32;
  while (ncols < (uint32_t)(MT * BN)) ncols <<= 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], p.full_count());
      mbar_init(&empty[s], 1);
    }
    mbar_init(accf, 1);
    fence_barrier_init();
  }
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  if (warp < 4) {
    const int t = threadIdx.x;
    for (int i = 0; i < nkb; ++i) {
      const int s = i % STAGES;
      const uint32_t ph = (uint32_t)(i / STAGES) & 1u;
      if (i >= STAGES) mbar_wait(&empty[s], ph ^ 1u);
      p.produce(kb0 + i, sA + s * MT * A_STAGE_BYTES, sB + (size_t)s * BN * BK * 2, &full[s], t);
      fence_proxy_async();
      mbar_arrive(&full[s]);
    }
    mbar_wait(accf, 0);
    tc_fence_after();
    const int row = warp * 32 + lane;
    for (int mt = 0; mt < MT; ++mt) {
      for (int c = 0; c < BN; c += 16) {
        float v[16];
        if (nkb > 0) {
          tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(mt * BN + c), v);
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = 0.f;
        }
        p.epilogue(row, mt, c, v);
      }
    }
  } else if (lane == 0) {
    const uint32_t idesc = umma_idesc((uint32_t)BN);
    const uint32_t lbo_a = BM * 16, lbo_b = (uint32_t)BN * 16;
    for (int i = 0; i < nkb; ++i) {
      const int s = i % STAGES;
      const uint32_t ph = (uint32_t)(i / STAGES) & 1u;
      mbar_wait(&full[s], ph);
      tc_fence_after();
      const uint32_t b_base = smem_u32(sB + (size_t)s * BN * BK * 2);
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const uint32_t a_base = smem_u32(sA + (s * MT + mt) * A_STAGE_BYTES);
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          const uint64_t ad = umma_desc(a_base + k * 2 * lbo_a, lbo_a, 128);
          const uint64_t bd = umma_desc(b_base + k * 2 * lbo_b, lbo_b, 128);
          umma_bf16(tmem + (uint32_t)(mt * BN), ad, bd, idesc, (i > 0 || k > 0) ? 1u : 0u);
        }
      }
      umma_commit(&empty[s]);
    }
    if (nkb > 0) umma_commit(accf);
    else mbar_arrive(accf);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    __syncwarp();
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols) : "memory");
  }
}

// ------------------------------------------------------- weight images
// Image element (tile, kb, n, k) at ((tile*nkb + kb) * BN + ...) in the
// canonical layout: offset = (k/8)*(BN*8) + n*8 + (k%8) elements.
// fwd: B[n][k'] = W[k(k')][n]   (k' in the split-padded space)
__global__ void k_wimg_fwd(const float* __restrict__ W, int K1, int K1p, bool two, int N, int BN, int nkb,
                           __nv_bfloat16* img) {
  const int total = nkb * BN * BK;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int kb = t / (BN * BK);
    const int r = t - kb * BN * BK;
    const int kc = r / (BN * 8);
    const int r2 = r - kc * BN * 8;
    const int n = r2 / 8, e = r2 % 8;
    const int kp = kb * BK + kc * 8 + e;
    int k = -1;
    if (kp < K1p) {
      if (kp < K1) k = kp;
    } else if (two && kp - K1p < K1) {
      k = K1 + (kp - K1p);
    }
    const float v = (k >= 0 && n < N) ? W[(int64_t)k * N + n] : 0.f;
    img[t] = __float2bfloat16_rn(v);
  }
}

// dx: B[j][k] = W[row(j)][k], j over [0,ld1) (+ [ld1, ld1+ld2)), k < N (d_out)
__global__ void k_wimg_dx(const float* __restrict__ W, int K1, int ld1, int ld2, bool two, int N, int BN, int nkb,
                          int ntiles, __nv_bfloat16* img) {
  const int per_tile = nkb * BN * BK;
  const int total = ntiles * per_tile;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int tile = t / per_tile;
    const int r0 = t - tile * per_tile;
    const int kb = r0 / (BN * BK);
    const int r = r0 - kb * BN * BK;
    const int kc = r / (BN * 8);
    const int r2 = r - kc * BN * 8;
    const int nl = r2 / 8, e = r2 % 8;
    const int j = tile * BN + nl;
    const int k = kb * BK + kc * 8 + e;
    int row = -1;
    if (j < ld1) {
      if (j < K1) row = j;
    } else if (two && j - ld1 < ld2) {
      if (j - ld1 < K1) row = K1 + (j - ld1);
    }
    const float v = (row >= 0 && k < N) ? W[(int64_t)row * N + k] : 0.f;
    img[t] = __float2bfloat16_rn(v);
  }
}

__global__ void k_dw_reduce_tc(const float* __restrict__ partial, int splits, int rows_p, int BN, int K1, int K1p,
                               int Ktot, int bias_row, int N, float* dW, float* db) {
  const int total = (Ktot + 1) * N;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int k = t / N, n = t - k * N;
    const int ip = (k == Ktot) ? bias_row : (k < K1 ? k : K1p + (k - K1));
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += partial[((int64_t)z * rows_p + ip) * BN + n];
    if (k < Ktot) dW[(int64_t)k * N + n] = s;
    else db[n] = s;
  }
}

static int round_up(int x, int m) { return (x + m - 1) / m * m; }

template <class P>
static void launch(const P& p, dim3 grid, int BN, cudaStream_t s) {
  const size_t smem = (size_t)STAGES * P::MT * A_STAGE_BYTES + (size_t)STAGES * BN * BK * 2 + 8 * (2 * STAGES + 1) + 16;
  static bool attr_set = false;
  if (!attr_set) {
    GNNV_TRY_CUDA(cudaFuncSetAttribute(k_tc_gemm<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr_set = true;
  }
  k_tc_gemm<P><<<grid, NTHREADS, smem, s>>>(p);
  GNNV_CHECK_LAUNCH();
}

// Scratch for the weight images / partials: a small per-process arena.
static void* tc_scratch(size_t bytes, cudaStream_t s) {
  static void* buf = nullptr;
  static size_t cap = 0;
  if (bytes > cap) {
    if (buf) {
      GNNV_TRY_CUDA(cudaStreamSynchronize(s));
      dfree(buf);
    }
    cap = std::max(bytes, (size_t)4 << 20);
    buf = dmalloc(cap, "tensor-core weight image");
  }
  return buf;
}

}  // namespace tc

bool gemm_fwd_tc(const GemmFwdArgs& a, cudaStream_t s) {
  using namespace tc;
  const int BN = round_up(a.ldy, 16);
  if (BN > 256) return false;
  const int K1p = (a.K1 + 3) & ~3;
  const int Kp = a.X2 ? 2 * K1p : K1p;
  const int nkb = (Kp + BK - 1) / BK;
  __nv_bfloat16* img = (__nv_bfloat16*)tc_scratch((size_t)nkb * BN * BK * 2, s);
  k_wimg_fwd<<<std::min(1024, (nkb * BN * BK + 255) / 256), 256, 0, s>>>(a.W, a.K1, K1p, a.X2 != nullptr, a.N, BN,
                                                                         nkb, img);
  GNNV_CHECK_LAUNCH();
  FwdPolicy p{};
  p.x = SplitRows{a.X1, a.X2, a.ld1, a.ld2, a.K1, K1p};
  p.wimg = img;
  p.bias = a.bias;
  p.Y = a.Y;
  p.ldy = a.ldy;
  p.N = a.N;
  p.BN = BN;
  p.nkb = nkb;
  p.relu = a.relu;
  p.dM = a.d_M;
  launch(p, dim3((unsigned)ceil_div(std::max<int64_t>(a.max_M, 1), BM)), BN, s);
  return true;
}

bool gemm_dx_tc(const GemmDxArgs& a, cudaStream_t s) {
  using namespace tc;
  const int NC = a.Y2 ? a.ld1 + a.ld2 : a.ld1;
  const int ntiles = (NC + 255) / 256;
  const int BN = round_up((NC + ntiles - 1) / ntiles, 16);
  const int nkb = (a.N + BK - 1) / BK;
  __nv_bfloat16* img = (__nv_bfloat16*)tc_scratch((size_t)ntiles * nkb * BN * BK * 2, s);
  const int total = ntiles * nkb * BN * BK;
  k_wimg_dx<<<std::min(1024, (total + 255) / 256), 256, 0, s>>>(a.W, a.K1, a.ld1, a.ld2, a.Y2 != nullptr, a.N, BN,
                                                                 nkb, ntiles, img);
  GNNV_CHECK_LAUNCH();
  DxPolicy p{};
  p.G = a.G;
  p.ldg = a.ldg;
  p.K = a.N;
  p.wimg = img;
  p.Y1 = a.Y1;
  p.Y2 = a.Y2;
  p.ld1 = a.ld1;
  p.ld2 = a.ld2;
  p.BN = BN;
  p.nkb = nkb;
  p.dM = a.d_M;
  launch(p, dim3((unsigned)ceil_div(std::max<int64_t>(a.max_M, 1), BM), (unsigned)ntiles), BN, s);
  return true;
}

bool gemm_dw_tc(const GemmDwArgs& a, cudaStream_t s) {
  using namespace tc;
  const int BN = round_up(a.N, 16);
  if (BN * DwPolicy::MT > 512) return false;
  const int K1p = (a.K1 + 3) & ~3;
  const int Kp = a.X2 ? 2 * K1p : K1p;
  const int bias_row = Kp;
  const int rows_p = round_up(Kp + 1, BM * DwPolicy::MT);
  const int igroups = rows_p / (BM * DwPolicy::MT);
  const int itiles = rows_p / BM;
  const int64_t nkb_max = ceil_div(std::max<int64_t>(a.max_M, 1), BK);
  int splits = (int)std::max<int64_t>(1, std::min<int64_t>(nkb_max, (int64_t)num_sms() / igroups));
  const size_t part_bytes = (size_t)splits * rows_p * BN * sizeof(float);
  // the SIMT path sized a.partial for its own split count; use our own arena
  float* partial = (float*)tc_scratch(part_bytes, s);
  DwPolicy p{};
  p.x = SplitRows{a.X1, a.X2, a.ld1, a.ld2, a.K1, K1p};
  p.rows_p = rows_p;
  p.bias_row = bias_row;
  p.G = a.G;
  p.ldg = a.ldg;
  p.N = a.N;
  p.BN = BN;
  p.dM = a.d_M;
  p.splits = splits;
  p.partial = partial;
  p.itiles = itiles;
  launch(p, dim3((unsigned)splits, (unsigned)igroups), BN, s);
  const int Ktot = a.X2 ? 2 * a.K1 : a.K1;
  const int total = (Ktot + 1) * a.N;
  k_dw_reduce_tc<<<std::min(1024, (total + 255) / 256), 256, 0, s>>>(partial, splits, rows_p, BN, a.K1, K1p, Ktot,
                                                                     bias_row, a.N, a.dW, a.db);
  GNNV_CHECK_LAUNCH();
  return true;
}

}  // namespace gnnv
