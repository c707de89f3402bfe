// NVLink peer-read microbenchmark for the SHARDED feature cache (north_star:
// "the feature cache is sharded across the GPUs' HBM and read peer-to-peer
// over NVLink"; SURVEY §8(d) "NVLink P2P read GB/s per GPU, at 1 and 8
// concurrent readers").  Ready for a multi-GPU box; with one GPU it says so.
//
//   stream : each reader GPU copies 1 GiB from a peer's buffer with 128-bit
//            SM loads (the gather's access pattern, one-sided, no copy engine)
//   rows   : random 512-byte rows (papers100M rows) gathered from the peer,
//            a warp per 8 rows, as k_gather does for peer-owned slots
// Modes: one reader at a time (GPU 0 <- GPU j) and all GPUs at once
// (GPU i <- GPU (i+1) % G).  Per-launch device time by CUDA events.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvlink_p2p tools/nvlink_p2p.cu
// ncu recipe (one reader, e.g. GPU 0 <- 1; 1 GPU profiled at a time):
//   ncu --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,dram__bytes_read.sum \
//       --clock-control none -k regex:k_peer tools/nvlink_p2p 0 1
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x)                                                                \
  do {                                                                       \
    cudaError_t e_ = (x);                                                    \
    if (e_ != cudaSuccess) {                                                 \
      printf("%s: %s\n", #x, cudaGetErrorString(e_));                        \
      exit(1);                                                               \
    }                                                                        \
  } while (0)

__global__ void k_peer_stream(const float4* __restrict__ src, float4* __restrict__ dst, int64_t n4) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __ldg(src + i);
}

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// rows of 32 float4 (512 B): a warp copies 8 random peer rows, loads first
__global__ void k_peer_rows(const float4* __restrict__ src, int64_t src_rows, float4* __restrict__ dst, int64_t rows) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r0 = w * 8; r0 < rows; r0 += nw * 8) {
    float4 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __ldg(src + (int64_t)(hsh((uint32_t)(r0 + j)) % src_rows) * 32 + lane);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (r0 + j < rows) dst[(r0 + j) * 32 + lane] = v[j];
  }
}

struct Buf {
  float4* src;
  float4* dst;
};

int main(int argc, char** argv) {
  int G = 0;
  CK(cudaGetDeviceCount(&G));
  const int64_t bytes = 1ll << 30, n4 = bytes / 16, rows = bytes / 512;
  if (G < 2) {
    printf("{\"nvlink_p2p\": \"skipped: %d GPU visible (needs >= 2)\"}\n", G);
    return 0;
  }
  int only_r = -1, only_s = -1;
  if (argc == 3) only_r = atoi(argv[1]), only_s = atoi(argv[2]);
  std::vector<Buf> b(G);
  for (int i = 0; i < G; ++i) {
    CK(cudaSetDevice(i));
    CK(cudaMalloc(&b[i].src, bytes));
    CK(cudaMalloc(&b[i].dst, bytes));
    CK(cudaMemset(b[i].src, 1, bytes));
    for (int j = 0; j < G; ++j) {
      int ok = 0;
      if (j != i && cudaDeviceCanAccessPeer(&ok, i, j) == cudaSuccess && ok) {
        cudaError_t e = cudaDeviceEnablePeerAccess(j, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
        cudaGetLastError();
      }
    }
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto run = [&](const std::vector<std::pair<int, int>>& pairs, bool rowmode) {
    std::vector<cudaEvent_t> e0(pairs.size()), e1(pairs.size());
    for (int rep = 0; rep < 3; ++rep) {
      for (size_t k = 0; k < pairs.size(); ++k) {
        const int r = pairs[k].first, s = pairs[k].second;
        CK(cudaSetDevice(r));
        if (rep == 0) {
          CK(cudaEventCreate(&e0[k]));
          CK(cudaEventCreate(&e1[k]));
        }
        CK(cudaEventRecord(e0[k]));
        if (rowmode) k_peer_rows<<<sms * 8, 256>>>(b[s].src, rows, b[r].dst, rows);
        else k_peer_stream<<<sms * 8, 256>>>(b[s].src, b[r].dst, n4);
        CK(cudaEventRecord(e1[k]));
      }
      for (size_t k = 0; k < pairs.size(); ++k) {
        CK(cudaSetDevice(pairs[k].first));
        CK(cudaEventSynchronize(e1[k]));
      }
    }
    double sum = 0, mn = 1e30;
    for (size_t k = 0; k < pairs.size(); ++k) {
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0[k], e1[k]));
      const double gbs = bytes / (ms * 1e-3) / 1e9;
      sum += gbs;
      mn = gbs < mn ? gbs : mn;
    }
    return std::make_pair(sum / pairs.size(), mn);
  };
  printf("{\"gpus\": %d, \"bytes_per_reader\": %lld, \"results\": [\n", G, (long long)bytes);
  bool first = true;
  for (int rowmode = 0; rowmode < 2; ++rowmode) {
    for (int j = 1; j < G; ++j) {
      if (only_r >= 0 && !(only_r == 0 && only_s == j)) continue;
      auto r = run({{0, j}}, rowmode);
      printf("%s  {\"mode\": \"%s\", \"readers\": 1, \"pair\": \"0<-%d\", \"GBps\": %.1f}", first ? "" : ",\n",
             rowmode ? "rows512" : "stream", j, r.first);
      first = false;
    }
    if (only_r < 0) {
      std::vector<std::pair<int, int>> all;
      for (int i = 0; i < G; ++i) all.push_back({i, (i + 1) % G});
      auto r = run(all, rowmode);
      printf(",\n  {\"mode\": \"%s\", \"readers\": %d, \"pattern\": \"i<-(i+1)%%G\", \"GBps_mean\": %.1f, "
             "\"GBps_min\": %.1f}", rowmode ? "rows512" : "stream", G, r.first, r.second);
    }
  }
  printf("\n]}\n");
  return 0;
}
