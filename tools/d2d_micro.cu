// STW gather candidates beside a running copy-engine D2H (the direct pre-copy's
// host leg): copy-engine D2D of 1024 x 64 KiB chunks (cudaMemcpyBatchAsync) vs
// one contiguous 64 MiB D2D, alone and beside a 1 GiB D2H on another stream.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/d2d_micro tools/d2d_micro.cu
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

#include <cuda_runtime.h>

int main() {
  const uint64_t N = 1ull << 30, piece = 65536, n = 1024;
  uint8_t *a, *b, *big, *h;
  cudaMalloc(&a, N);
  cudaMalloc(&b, 64ull << 20);
  cudaMalloc(&big, N);
  cudaHostAlloc(&h, N, cudaHostAllocDefault);
  cudaMemset(a, 1, N);
  cudaStream_t s, c;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::vector<void*> srcs(n), dsts(n);
  std::vector<size_t> sizes(n, piece);
  for (uint64_t i = 0; i < n; ++i) {
    srcs[i] = a + (i * 977 % (N / piece)) * piece;  // scattered sources
    dsts[i] = b + i * piece;                          // packed destination
  }
  cudaMemcpyAttributes attr{};
  attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
  attr.srcLocHint.type = cudaMemLocationTypeDevice;
  attr.dstLocHint.type = cudaMemLocationTypeDevice;
  for (int conc = 0; conc < 2; ++conc) {
    for (int mode = 0; mode < 2; ++mode) {
      float best = 1e9;
      for (int r = 0; r < 5; ++r) {
        if (conc) cudaMemcpyAsync(h, big, N, cudaMemcpyDeviceToHost, c);
        cudaEventRecord(e0, s);
        if (mode == 0) {
          size_t z = 0, f = 0;
          cudaMemcpyBatchAsync(dsts.data(), srcs.data(), sizes.data(), n, &attr, &z, 1, &f, s);
        } else {
          cudaMemcpyAsync(b, a, n * piece, cudaMemcpyDeviceToDevice, s);
        }
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms);
        cudaDeviceSynchronize();
      }
      printf("%-28s %s: %8.1f us  %7.1f GB/s (read+write)\n", mode ? "CE D2D 64 MiB contiguous" : "CE D2D batch 1024 x 64 KiB",
             conc ? "beside 1 GiB D2H" : "alone           ", best * 1e3, 2.0 * n * piece / (best * 1e-3) / 1e9);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
