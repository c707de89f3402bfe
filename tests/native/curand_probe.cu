// Test infrastructure (not part of libgnnv): the library routine the
// oracle's draw() layout claims to equal -- cuRAND's Philox4_32_10 with
// curand_init(seed, subsequence = (hop << 32) | node, offset = s); curand().
// Built by tests/test_gpu_curand.py with nvcc; shares nothing with libgnnv
// or oracle/.
#include <curand_kernel.h>
#include <stdint.h>

__global__ void k_draws(uint64_t seed, const uint32_t* hop, const uint32_t* node, const uint32_t* s, int n,
                        uint32_t* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  curandStatePhilox4_32_10_t st;
  curand_init(seed, ((unsigned long long)hop[i] << 32) | node[i], s[i], &st);
  out[i] = curand(&st);
}

extern "C" int curand_probe_draws(uint64_t seed, const uint32_t* hop, const uint32_t* node, const uint32_t* s, int n,
                                  uint32_t* out_host) {
  uint32_t *dh, *dn, *ds, *dout;
  const size_t b = (size_t)n * 4;
  if (cudaMalloc(&dh, b) || cudaMalloc(&dn, b) || cudaMalloc(&ds, b) || cudaMalloc(&dout, b)) return 1;
  cudaMemcpy(dh, hop, b, cudaMemcpyHostToDevice);
  cudaMemcpy(dn, node, b, cudaMemcpyHostToDevice);
  cudaMemcpy(ds, s, b, cudaMemcpyHostToDevice);
  k_draws<<<(n + 255) / 256, 256>>>(seed, dh, dn, ds, n, dout);
  const int rc = cudaMemcpy(out_host, dout, b, cudaMemcpyDeviceToHost) != cudaSuccess;
  cudaFree(dh);
  cudaFree(dn);
  cudaFree(ds);
  cudaFree(dout);
  return rc;
}
