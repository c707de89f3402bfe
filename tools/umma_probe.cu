// Probe: one tcgen05.mma (M=128, N=32) with hand-built SW128 smem operands,
// K-major or MN-major, tf32 or bf16; prints max |D - A B^T| per variant.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_probe umma_probe.cu
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((a >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

// A[m][k] (M=128), B[n][k] (N=32); K = 8 (tf32) or 16 (bf16)
__device__ float Aval(int m, int k) { return (float)((m % 7) - 3 + k); }
__device__ float Bval(int n, int k) { return (float)((n % 5) - 2 - k); }

// element byte offset in an SW128 atom layout
// K-major: row = mn (128B = 32 tf32 / 64 bf16 of K), 8-row atoms at 1024
// MN-major: row = k (128B = 32 tf32 / 64 bf16 of MN), atoms of 8 k-rows; MN blocks at `mnblk`
__device__ uint32_t off_kmajor(int mn, int k, int esz) {
  const int byte = k * esz;  // within the 128B row
  const int chunk = byte >> 4, in = byte & 15;
  return (uint32_t)(mn * 128 + ((chunk ^ (mn & 7)) << 4) + in);
}
// K-major SWIZZLE_64B: 64B rows (16 tf32), 8-row atoms of 512B, chunk ^= (row>>1)&3
__device__ uint32_t off_kmajor64(int mn, int k, int esz) {
  const int byte = k * esz;
  const int chunk = byte >> 4, in = byte & 15;
  return (uint32_t)(mn * 64 + ((chunk ^ ((mn >> 1) & 3)) << 4) + in);
}
// K-major SWIZZLE_NONE: core matrices 8 rows x 16B; [kchunk][rowgroup][8][16B]
__device__ uint32_t off_knone(int mn, int k, int esz, int M) {
  const int byte = k * esz;
  const int chunk = byte >> 4, in = byte & 15;
  return (uint32_t)(chunk * (M * 16) + mn * 16 + in);
}
__device__ uint32_t off_mnmajor(int mn, int k, int esz, int mnblk_bytes, int kgrp_bytes) {
  const int per_row = 128 / esz;  // MN elements per 128B row
  const int blk = mn / per_row, r = mn % per_row;
  const int byte = r * esz;
  const int chunk = byte >> 4, in = byte & 15;
  const int krow = k & 7, kg = k >> 3;
  return (uint32_t)(blk * mnblk_bytes + kg * kgrp_bytes + krow * 128 + ((chunk ^ krow) << 4) + in);
}

__global__ void probe(int kind /*0 tf32, 1 bf16*/, int a_mn, int b_mn, int klay /*0 sw128 1 sw64 2 none*/, uint32_t lbo_a, uint32_t sbo_a, uint32_t lbo_b,
                      uint32_t sbo_b, float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = base;
  uint8_t* sB = base + 65536;
  __shared__ uint64_t bar;
  __shared__ uint32_t tm;
  const int esz = kind == 0 ? 4 : 2;
  const int K = kind == 0 ? 8 : 16;
  for (int i = threadIdx.x; i < 65536 * 2 / 4; i += blockDim.x) ((uint32_t*)base)[i] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < 128 * K; i += blockDim.x) {
    const int m = i / K, k = i % K;
    const uint32_t o = a_mn ? off_mnmajor(m, k, esz, lbo_a, sbo_a)
                            : (klay == 0 ? off_kmajor(m, k, esz) : klay == 1 ? off_kmajor64(m, k, esz) : off_knone(m, k, esz, 128));
    if (kind == 0) *(float*)(sA + o) = Aval(m, k);
    else *(__nv_bfloat16*)(sA + o) = __float2bfloat16(Aval(m, k));
  }
  for (int i = threadIdx.x; i < 32 * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    const uint32_t o = b_mn ? off_mnmajor(n, k, esz, lbo_b, sbo_b)
                            : (klay == 0 ? off_kmajor(n, k, esz) : klay == 1 ? off_kmajor64(n, k, esz) : off_knone(n, k, esz, 32));
    if (kind == 0) *(float*)(sB + o) = Bval(n, k);
    else *(__nv_bfloat16*)(sB + o) = __float2bfloat16(Bval(n, k));
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tm)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = tm;
  if (threadIdx.x == 0) {
    const uint32_t fmt = kind == 0 ? 2u : 1u;
    const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
                           ((32u >> 3) << 17) | ((128u >> 4) << 24);
    const uint32_t lay = klay == 0 ? 2u : klay == 1 ? 4u : 0u;
    const uint64_t ad = a_mn ? desc(su32(sA), lbo_a, sbo_a, 2)
                             : desc(su32(sA), klay == 2 ? 128 * 16 : 16, klay == 0 ? 1024 : klay == 1 ? 512 : 128, lay);
    const uint64_t bd = b_mn ? desc(su32(sB), lbo_b, sbo_b, 2)
                             : desc(su32(sB), klay == 2 ? 32 * 16 : 16, klay == 0 ? 1024 : klay == 1 ? 512 : 128, lay);
    if (kind == 0)
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 0, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(t),
                   "l"(ad), "l"(bd), "r"(idesc));
    else
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 0, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(t),
                   "l"(ad), "l"(bd), "r"(idesc));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
  }
  asm volatile(
      "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t r[8];
  for (int c = 0; c < 32; c += 8) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(t + ((uint32_t)(w * 32) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 8; ++j) out[(w * 32 + lane) * 32 + c + j] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(t));
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 32 * 4);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  struct V {
    const char* name;
    int kind, amn, bmn, klay;
    uint32_t la, sa, lb, sb;
  } vs[] = {
      {"tf32 K/K sw128", 0, 0, 0, 0, 0, 0, 0, 0},
      {"tf32 K/K sw64", 0, 0, 0, 1, 0, 0, 0, 0},
      {"tf32 K/K none", 0, 0, 0, 2, 0, 0, 0, 0},
      {"tf32 MN/MN lbo=mnblk sbo=kgrp", 0, 1, 1, 0, 4096, 1024, 4096, 1024},
      {"tf32 MN/MN lbo=kgrp sbo=mnblk", 0, 1, 1, 0, 1024, 4096, 1024, 4096},
      {"tf32 MN/K  lbo=mnblk sbo=kgrp", 0, 1, 0, 0, 4096, 1024, 0, 0},
      {"tf32 K/MN  lbo=mnblk sbo=kgrp", 0, 0, 1, 0, 0, 0, 4096, 1024},
      {"bf16 K/K", 1, 0, 0, 0, 0, 0, 0, 0},
      {"bf16 MN/MN lbo=mnblk sbo=kgrp", 1, 1, 1, 0, 8192, 1024, 8192, 1024},
      {"bf16 MN/MN lbo=kgrp sbo=mnblk", 1, 1, 1, 0, 1024, 8192, 1024, 8192},
  };
  float h[128 * 32];
  for (auto& v : vs) {
    cudaMemset(d, 0, sizeof(h));
    probe<<<1, 128, 140 * 1024>>>(v.kind, v.amn, v.bmn, v.klay, v.la, v.sa, v.lb, v.sb, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    const int K = v.kind == 0 ? 8 : 16;
    double maxerr = 0, maxref = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 32; ++n) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += (double)((m % 7) - 3 + k) * (double)((n % 5) - 2 - k);
        maxerr = fmax(maxerr, fabs(ref - h[m * 32 + n]));
        maxref = fmax(maxref, fabs(ref));
      }
    printf("%-34s err=%s maxerr=%g (maxref %g) D[0][0..3]=%g %g %g %g D[40][1]=%g\n", v.name, cudaGetErrorString(e),
           maxerr, maxref, h[0], h[1], h[2], h[3], h[40 * 32 + 1]);
  }
  return 0;
}
