// Microbenchmark: can the layer-2 aggregation live in L2 on B200?
//
// Products layer 2: A2 / dA2 are n_1 x 256 fp32 (~61 MB,
// L2-resident); E_1 ~ 600K sampled edges, each moving one 1 KB row.
//   push_warp   : red.global.add.v4.f32, a warp per edge row (coalesced)
//   push_thread : red.global.add.v4.f32, a thread per edge row (scattered)
//   push_bulk   : cp.reduce.async.bulk .add.f32, 1 KB per edge from smem
//   pull_l2     : warp per src row, gathers its (1-2) dA2 rows from L2
//   store_dram  : the DRAM write it would replace (E_1 rows of 1 KB)
//   read_dram   : the DRAM read it would replace
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench_l2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

__global__ void push_warp(float* A, int rows, int E, int ld) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int e = w; e < E; e += nw) {
    const int v = hsh(e) % rows;
    float4* p = reinterpret_cast<float4*>(A + (int64_t)v * ld);
    for (int c = lane; c < ld / 4; c += 32) atomicAdd(p + c, make_float4(1.f, 1.f, 1.f, 1.f));
  }
}

__global__ void push_thread(float* A, int rows, int E, int ld) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    const int v = hsh(e) % rows;
    float4* p = reinterpret_cast<float4*>(A + (int64_t)v * ld);
    for (int c = 0; c < ld / 4; ++c) atomicAdd(p + c, make_float4(1.f, 1.f, 1.f, 1.f));
  }
}

__global__ void push_bulk(float* A, int rows, int E, int ld) {
  extern __shared__ __align__(128) float sm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  float* row = sm + wib * ld;
  for (int c = lane; c < ld; c += 32) row[c] = 1.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  if (lane == 0) {
    for (int e = w; e < E; e += nw) {
      const int v = hsh(e) % rows;
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(A + (int64_t)v * ld),
                   "r"((uint32_t)__cvta_generic_to_shared(row)), "r"(ld * 4) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

__global__ void pull_l2(const float* A, int rows, int E, int ld, float* sink) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int e = w; e < E; e += nw) {
    const int v = hsh(e) % rows;
    const float4* p = reinterpret_cast<const float4*>(A + (int64_t)v * ld);
    for (int c = lane; c < ld / 4; c += 32) {
      float4 x = __ldg(p + c);
      acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
    }
  }
  if (acc.x == 12345.f) sink[0] = acc.y + acc.z + acc.w;
}

__global__ void store_dram(float* B, int E, int ld) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int e = w; e < E; e += nw) {
    float4* p = reinterpret_cast<float4*>(B + (int64_t)e * ld);
    for (int c = lane; c < ld / 4; c += 32) p[c] = make_float4(1.f, 2.f, 3.f, 4.f);
  }
}

__global__ void read_dram(const float* B, int E, int ld, float* sink) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int e = w; e < E; e += nw) {
    const float4* p = reinterpret_cast<const float4*>(B + (int64_t)e * ld);
    for (int c = lane; c < ld / 4; c += 32) {
      float4 x = __ldg(p + c);
      acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
    }
  }
  if (acc.x == 12345.f) sink[0] = acc.y + acc.z + acc.w;
}

__global__ void flush(float* f, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) f[i] += 1.f;
}

int main() {
  const int ld = 256;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *A, *B, *F, *sink;
  const int E = 600000;
  const int64_t fl = 64ll << 20;  // 256 MB flush buffer
  CK(cudaMalloc(&A, 100000ll * ld * 4));
  CK(cudaMalloc(&B, (int64_t)E * ld * 4));
  CK(cudaMalloc(&F, fl * 4));
  CK(cudaMalloc(&sink, 64));
  CK(cudaMemset(A, 0, 100000ll * ld * 4));
  CK(cudaMemset(B, 0, (int64_t)E * ld * 4));
  CK(cudaFuncSetAttribute(push_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * ld * 4));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = (double)E * ld * 4;
  for (int rows : {30000, 60000, 100000}) {
    for (int k = 0; k < 6; ++k) {
      float best = 1e9;
      for (int it = 0; it < 5; ++it) {
        flush<<<sms * 8, 256>>>(F, fl);
        if (k == 3) {  // make the pulled rows L2-resident, as after the dX GEMM
          push_warp<<<sms * 8, 256>>>(A, rows, rows, ld);
        }
        cudaEventRecord(e0);
        switch (k) {
          case 0: push_warp<<<sms * 8, 256>>>(A, rows, E, ld); break;
          case 1: push_thread<<<sms * 8, 256>>>(A, rows, E, ld); break;
          case 2: push_bulk<<<sms * 4, 256, 8 * ld * 4>>>(A, rows, E, ld); break;
          case 3: pull_l2<<<sms * 8, 256>>>(A, rows, E, ld, sink); break;
          case 4: store_dram<<<sms * 8, 256>>>(B, E, ld); break;
          case 5: read_dram<<<sms * 8, 256>>>(B, E, ld, sink); break;
        }
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      CK(cudaGetLastError());
      const char* nm[] = {"push_warp", "push_thread", "push_bulk", "pull_l2", "store_dram", "read_dram"};
      printf("rows %6d (%5.1f MB) %-12s E=%d x 1KB: %8.1f us  %7.1f GB/s\n", rows, rows * ld * 4 / 1e6, nm[k], E,
             best * 1e3, bytes / (best * 1e-3) / 1e9);
    }
  }
  return 0;
}
