// Dense transform of the GNN layer, fp32 SIMT path (parity mode, reading Q17:
// TF32 would exceed the 1e-5 tolerance, so this is plain FFMA).
//
// Paper: Eq.1 Combine, Algorithm 1 lines 6 and 8.
// Three products, all with the row count M on the device:
//   fwd : Y  = act([X1 | X2] W + b)                       (M x N)
//   dX  : [Y1 | Y2] = G W^T                                (M x 2K1)
//   dW  : [dW ; db] = [X1 | X2 | 1]^T G  (long-K, split-K with a fixed-order
//         reduction so dW/db are deterministic; the ones column folds the
//         bias gradient into the same product)
// Tile 128x128x8, 256 threads, 8x8 outputs per thread, register-prefetched
// double buffer.  The bf16 tcgen05 path is gemm_tc.cu.
#include "common.cuh"

namespace gnnv {

constexpr int TBM = 128, TBN = 128, TBK = 8;

struct ProbFwd {
  const float *X1, *X2, *W, *bias;
  int ld1, ld2, K1, N;
  float* Y;
  int ldy;
  const int32_t* dM;
  bool relu;
  __device__ int M() const { return *dM; }
  __device__ int K() const { return X2 ? 2 * K1 : K1; }
  __device__ int NC() const { return ldy; }  // output columns incl. zero padding
  __device__ float a(int m, int k) const {
    return k < K1 ? __ldg(X1 + (int64_t)m * ld1 + k) : __ldg(X2 + (int64_t)m * ld2 + (k - K1));
  }
  __device__ float b(int k, int n) const { return n < N ? __ldg(W + (int64_t)k * N + n) : 0.f; }
  __device__ void store(int m, int n, float v, int) const {
    if (n < N) {
      v += __ldg(bias + n);
      if (relu) v = fmaxf(v, 0.f);
    } else {
      v = 0.f;
    }
    Y[(int64_t)m * ldy + n] = v;
  }
};

struct ProbDx {
  const float *G, *W;
  int ldg, N, K1;
  float *Y1, *Y2;
  int ld1, ld2;
  const int32_t* dM;
  __device__ int M() const { return *dM; }
  __device__ int K() const { return N; }
  __device__ int NC() const { return Y2 ? ld1 + ld2 : ld1; }
  __device__ float a(int m, int k) const { return __ldg(G + (int64_t)m * ldg + k); }
  __device__ float b(int k, int j) const {
    int r;
    if (j < ld1) {
      if (j >= K1) return 0.f;
      r = j;
    } else {
      const int jj = j - ld1;
      if (jj >= K1) return 0.f;
      r = K1 + jj;
    }
    return __ldg(W + (int64_t)r * N + k);
  }
  __device__ void store(int m, int j, float v, int) const {
    if (j < ld1) Y1[(int64_t)m * ld1 + j] = v;
    else Y2[(int64_t)m * ld2 + (j - ld1)] = v;
  }
};

struct ProbDw {
  const float *X1, *X2, *G;
  int ld1, ld2, K1, ldg, N;
  const int32_t* dRows;  // reduction length (device)
  int rows;              // output rows incl. the bias row: (X2 ? 2K1 : K1) + 1
  float* partial;        // [splits][rows][N]
  __device__ int M() const { return rows; }
  __device__ int K() const { return *dRows; }
  __device__ int NC() const { return N; }
  __device__ float a(int i, int m) const {
    if (i < K1) return __ldg(X1 + (int64_t)m * ld1 + i);
    if (X2 && i < 2 * K1) return __ldg(X2 + (int64_t)m * ld2 + (i - K1));
    return 1.f;
  }
  __device__ float b(int m, int n) const { return __ldg(G + (int64_t)m * ldg + n); }
  __device__ void store(int i, int n, float v, int split) const {
    if (n < N) partial[((int64_t)split * rows + i) * N + n] = v;
  }
};

// A_KFAST: consecutive threads walk k when loading the A tile (A row-major in
// k); otherwise they walk m.  B_NFAST: consecutive threads walk n for B.
template <bool A_KFAST, bool B_NFAST, bool SPLITK, class P>
__global__ void __launch_bounds__(256) k_gemm_simt(P p, int splits) {
  __shared__ __align__(16) float As[2][TBK][TBM];
  __shared__ __align__(16) float Bs[2][TBK][TBN];
  const int M = p.M(), K = p.K(), NC = p.NC();
  const int m0 = blockIdx.x * TBM, n0 = blockIdx.y * TBN;
  if (m0 >= M || n0 >= NC) return;
  int kb = 0, ke = K;
  if (SPLITK) {
    const int chunk = ((K + splits - 1) / splits + TBK - 1) / TBK * TBK;
    kb = min(K, (int)blockIdx.z * chunk);
    ke = min(K, kb + chunk);
  }
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  float ra[4], rb[4];
  auto load = [&](int k0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = tid + 256 * i;
      int m, k;
      if (A_KFAST) {
        k = e & 7;
        m = e >> 3;
      } else {
        m = e & 127;
        k = e >> 7;
      }
      const int gm = m0 + m, gk = k0 + k;
      ra[i] = (gm < M && gk < ke) ? p.a(gm, gk) : 0.f;
      int n, kk;
      if (B_NFAST) {
        n = e & 127;
        kk = e >> 7;
      } else {
        kk = e & 7;
        n = e >> 3;
      }
      const int gn = n0 + n, gk2 = k0 + kk;
      rb[i] = (gn < NC && gk2 < ke) ? p.b(gk2, gn) : 0.f;
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = tid + 256 * i;
      if (A_KFAST) As[buf][e & 7][e >> 3] = ra[i];
      else As[buf][e >> 7][e & 127] = ra[i];
      if (B_NFAST) Bs[buf][e >> 7][e & 127] = rb[i];
      else Bs[buf][e & 7][e >> 3] = rb[i];
    }
  };
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  int buf = 0;
  if (kb < ke) {
    load(kb);
    stash(0);
    __syncthreads();
    for (int k0 = kb; k0 < ke; k0 += TBK) {
      const bool more = k0 + TBK < ke;
      if (more) load(k0 + TBK);
#pragma unroll
      for (int kk = 0; kk < TBK; ++kk) {
        const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
        const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][64 + ty * 4]);
        const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
        const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][64 + tx * 4]);
        const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      }
      if (more) {
        stash(buf ^ 1);
        __syncthreads();
        buf ^= 1;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int n = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
      if (n < NC) p.store(m, n, acc[i][j], SPLITK ? (int)blockIdx.z : 0);
    }
  }
}

__global__ void k_dw_reduce(const float* __restrict__ partial, int splits, int rows, int N, float* dW, float* db) {
  const int total = rows * N;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += partial[(int64_t)z * total + t];
    const int i = t / N, n = t - i * N;
    if (i < rows - 1) dW[t] = s;
    else db[n] = s;
  }
}

void gemm_fwd_simt(const GemmFwdArgs& a, cudaStream_t s) {
  ProbFwd p{a.X1, a.X2, a.W, a.bias, a.ld1, a.ld2, a.K1, a.N, a.Y, a.ldy, a.d_M, a.relu};
  dim3 grid((unsigned)ceil_div(std::max<int64_t>(a.max_M, 1), TBM), (unsigned)ceil_div(a.ldy, TBN));
  k_gemm_simt<true, true, false><<<grid, 256, 0, s>>>(p, 1);
  GNNV_CHECK_LAUNCH();
}

void gemm_dx_simt(const GemmDxArgs& a, cudaStream_t s) {
  ProbDx p{a.G, a.W, a.ldg, a.N, a.K1, a.Y1, a.Y2, a.ld1, a.ld2, a.d_M};
  const int NC = a.Y2 ? a.ld1 + a.ld2 : a.ld1;
  dim3 grid((unsigned)ceil_div(std::max<int64_t>(a.max_M, 1), TBM), (unsigned)ceil_div(NC, TBN));
  k_gemm_simt<true, false, false><<<grid, 256, 0, s>>>(p, 1);
  GNNV_CHECK_LAUNCH();
}

size_t gemm_dw_partial_floats(int32_t rows_plus_bias, int32_t N, int32_t* splits_out, int64_t max_M) {
  // enough splits to fill the machine twice over with 128x128 output tiles
  const int64_t tiles = ceil_div(rows_plus_bias, TBM) * ceil_div(N, TBN);
  int64_t splits = std::max<int64_t>(1, (int64_t)num_sms() * 2 / std::max<int64_t>(tiles, 1));
  splits = std::min<int64_t>(splits, std::max<int64_t>(1, ceil_div(max_M, 256)));
  *splits_out = (int32_t)splits;
  return (size_t)splits * rows_plus_bias * N;
}

void gemm_dw_simt(const GemmDwArgs& a, cudaStream_t s) {
  const int rows = (a.X2 ? 2 * a.K1 : a.K1) + 1;
  ProbDw p{a.X1, a.X2, a.G, a.ld1, a.ld2, a.K1, a.ldg, a.N, a.d_M, rows, a.partial};
  dim3 grid((unsigned)ceil_div(rows, TBM), (unsigned)ceil_div(a.N, TBN), (unsigned)a.splits);
  k_gemm_simt<false, true, true><<<grid, 256, 0, s>>>(p, a.splits);
  GNNV_CHECK_LAUNCH();
  const int total = rows * a.N;
  k_dw_reduce<<<(int)std::min<int64_t>(ceil_div(total, 256), num_sms() * 4), 256, 0, s>>>(a.partial, a.splits, rows,
                                                                                           a.N, a.dW, a.db);
  GNNV_CHECK_LAUNCH();
}

// bf16 tensor-core entry points (gemm_tc.cu); return false if the shape is
// not handled there, in which case the SIMT path runs.
bool gemm_fwd_tc(const GemmFwdArgs& a, cudaStream_t s);
bool gemm_dx_tc(const GemmDxArgs& a, cudaStream_t s);
bool gemm_dw_tc(const GemmDwArgs& a, cudaStream_t s);

bool gemm_fwd_tma(const GemmFwdArgs& a, cudaStream_t s);
bool gemm_dx_tma(const GemmDxArgs& a, cudaStream_t s);
bool gemm_dw_tma(const GemmDwArgs& a, cudaStream_t s);

// Precision dispatch.  A tensor-core path that does not handle a shape is an
// error, never a silent fall back to another precision.
void gemm_fwd(const GemmFwdArgs& a, int prec, cudaStream_t s) {
  GNNV_REQUIRE(!a.x1_rows || prec == GNNV_PREC_TF32, GNNV_ERR_UNSUPPORTED, "fwd: indexed X1 rows need the tf32 path");
  GNNV_REQUIRE(!a.push_out || prec == GNNV_PREC_TF32, GNNV_ERR_UNSUPPORTED, "fwd: the fused push needs the tf32 path");
  GNNV_REQUIRE(!a.X1_16 || prec == GNNV_PREC_TF32, GNNV_ERR_UNSUPPORTED, "fwd: bf16 operand copies need the tf32 path");
  if (prec == GNNV_PREC_FP32) return gemm_fwd_simt(a, s);
  const bool ok = prec == GNNV_PREC_TF32 ? gemm_fwd_tma(a, s) : gemm_fwd_tc(a, s);
  GNNV_REQUIRE(ok, GNNV_ERR_UNSUPPORTED, "tensor-core fwd GEMM: d_out > 252 is not supported");
}
void gemm_dx(const GemmDxArgs& a, int prec, cudaStream_t s) {
  GNNV_REQUIRE(!a.G16 || prec == GNNV_PREC_TF32, GNNV_ERR_UNSUPPORTED, "dX: a bf16 G copy needs the tf32 path");
  if (prec == GNNV_PREC_FP32) return gemm_dx_simt(a, s);
  const bool ok = prec == GNNV_PREC_TF32 ? gemm_dx_tma(a, s) : gemm_dx_tc(a, s);
  GNNV_REQUIRE(ok, GNNV_ERR_UNSUPPORTED, "tensor-core dX GEMM: unsupported shape");
}
// For TF32 this computes dW only; db comes from k_mask_colsum (layers.cu).
void gemm_dw(const GemmDwArgs& a, int prec, cudaStream_t s) {
  GNNV_REQUIRE(!a.x1_rows || prec == GNNV_PREC_TF32, GNNV_ERR_UNSUPPORTED, "dW: indexed X1 rows need the tf32 path");
  if (prec == GNNV_PREC_FP32) return gemm_dw_simt(a, s);
  const bool ok = prec == GNNV_PREC_TF32 ? gemm_dw_tma(a, s) : gemm_dw_tc(a, s);
  GNNV_REQUIRE(ok, GNNV_ERR_UNSUPPORTED, "tensor-core dW GEMM: d_out > 256 is not supported");
}

}  // namespace gnnv
