// Does a concurrent copy-engine D2H slow SM kernels?  read kernel (1 GiB and
// 16 MiB) alone vs with a 1 GiB pinned D2H in flight on another stream.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/interference_micro tools/interference_micro.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_copy(const uint4* a, uint4* b, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
  uint8_t *a, *b, *big, *h;
  const uint64_t N = 1ull << 30;
  cudaMalloc(&a, N); cudaMalloc(&b, N); cudaMalloc(&big, N);
  cudaHostAlloc(&h, N, cudaHostAllocDefault);
  cudaMemset(a, 1, N); cudaMemset(big, 2, N);
  cudaStream_t s, c;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (uint64_t bytes : {16ull << 20, 256ull << 20, 1ull << 30}) {
    for (int conc = 0; conc < 3; ++conc) {
      float best = 1e9;
      for (int r = 0; r < 5; ++r) {
        if (conc == 1) cudaMemcpyAsync(h, big, N, cudaMemcpyDeviceToHost, c);
        if (conc == 2) cudaMemcpyAsync(big, h, N, cudaMemcpyHostToDevice, c);
        cudaEventRecord(e0, s);
        k_copy<<<148 * 8, 256, 0, s>>>((const uint4*)a, (uint4*)b, bytes / 16);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
        cudaDeviceSynchronize();
      }
      printf("copy kernel %5llu MiB %s: %8.1f us  %7.1f GB/s\n", (unsigned long long)(bytes >> 20),
             conc == 0 ? "alone      " : conc == 1 ? "+ D2H 1 GiB" : "+ H2D 1 GiB", best * 1e3, 2.0 * bytes / (best * 1e-3) / 1e9);
    }
  }
  return 0;
}
