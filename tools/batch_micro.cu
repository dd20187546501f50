// Host-leg probe for the direct (into-the-image) pre-copy: how fast can the
// copy engine scatter many chunk-sized D2H copies into a pinned image?
//   cudaMemcpyBatchAsync (CUDA 12.8+) vs a cudaMemcpyAsync loop vs SM stores
//   (zero copy), for 64 KiB chunks and for 400 KiB runs; plus CE + SM
//   concurrently on the link.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/batch_micro tools/batch_micro.cu
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

#include <cuda_runtime.h>

__global__ void k_zc(const uint64_t* src, const uint64_t* dst, const uint64_t* len, int n) {
  const int lane = threadIdx.x & 31;
  for (int i = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); i < n; i += gridDim.x * (blockDim.x / 32)) {
    const uint4* s = (const uint4*)src[i];
    uint4* d = (uint4*)dst[i];
    uint64_t m = len[i] / 16;
    for (uint64_t k = lane; k < m; k += 32 * 4) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = k + u * 32 < m ? s[k + u * 32] : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (k + u * 32 < m) d[k + u * 32] = v[u];
    }
  }
}

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  const uint64_t dev_bytes = 1ull << 30;
  uint8_t *d, *h;
  cudaMalloc(&d, dev_bytes);
  cudaMemset(d, 7, dev_bytes);
  cudaHostAlloc(&h, dev_bytes, cudaHostAllocMapped);
  cudaStream_t s, s2;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  std::mt19937_64 rng(1);
  for (uint64_t piece : {65536ull, 409600ull, 4ull << 20}) {
    for (int n : {100, 400, 1638}) {
      if (piece * n > dev_bytes / 2) continue;
      // distinct random slots
      uint64_t slots = dev_bytes / piece;
      std::vector<uint64_t> pick(slots);
      for (uint64_t i = 0; i < slots; ++i) pick[i] = i;
      std::shuffle(pick.begin(), pick.end(), rng);
      std::vector<void*> srcs(n), dsts(n);
      std::vector<size_t> sizes(n, piece);
      std::vector<uint64_t> hs(n), hd(n), hl(n, piece);
      for (int i = 0; i < n; ++i) {
        srcs[i] = d + pick[i] * piece;
        dsts[i] = h + pick[i] * piece;
        hs[i] = (uint64_t)srcs[i];
        hd[i] = (uint64_t)dsts[i];
      }
      const double bytes = (double)piece * n;
      // 1. batch
      cudaMemcpyAttributes attr{};
      attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
      attr.srcLocHint.type = cudaMemLocationTypeDevice;
      attr.dstLocHint.type = cudaMemLocationTypeHost;
      size_t idx0 = 0, fail = 0;
      double best_dev = 1e9, best_host = 1e9;
      for (int r = 0; r < 4; ++r) {
        cudaStreamSynchronize(s);
        cudaEventRecord(a, s);
        double t0 = now_us();
        cudaError_t e = cudaMemcpyBatchAsync(dsts.data(), srcs.data(), sizes.data(), n, &attr, &idx0, 1, &fail, s);
        double t1 = now_us();
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        if (e != cudaSuccess) {
          printf("batch error %s (fail idx %zu)\n", cudaGetErrorString(e), fail);
          break;
        }
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best_dev = std::min(best_dev, (double)ms * 1e3);
        best_host = std::min(best_host, t1 - t0);
      }
      printf("piece %7llu n %5d  batch : enqueue %8.1f us  device %8.1f us  %6.1f GB/s\n",
             (unsigned long long)piece, n, best_host, best_dev, bytes / best_dev / 1e3);
      // 2. loop of cudaMemcpyAsync
      best_dev = best_host = 1e9;
      for (int r = 0; r < 4; ++r) {
        cudaStreamSynchronize(s);
        cudaEventRecord(a, s);
        double t0 = now_us();
        for (int i = 0; i < n; ++i) cudaMemcpyAsync(dsts[i], srcs[i], piece, cudaMemcpyDeviceToHost, s);
        double t1 = now_us();
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best_dev = std::min(best_dev, (double)ms * 1e3);
        best_host = std::min(best_host, t1 - t0);
      }
      printf("piece %7llu n %5d  loop  : enqueue %8.1f us  device %8.1f us  %6.1f GB/s\n",
             (unsigned long long)piece, n, best_host, best_dev, bytes / best_dev / 1e3);
      // 3. SM zero copy
      uint64_t *ds, *dd, *dl;
      cudaMalloc(&ds, n * 8);
      cudaMalloc(&dd, n * 8);
      cudaMalloc(&dl, n * 8);
      cudaMemcpy(ds, hs.data(), n * 8, cudaMemcpyHostToDevice);
      cudaMemcpy(dd, hd.data(), n * 8, cudaMemcpyHostToDevice);
      cudaMemcpy(dl, hl.data(), n * 8, cudaMemcpyHostToDevice);
      for (int ctas : {8, 16, 32}) {
        best_dev = 1e9;
        for (int r = 0; r < 4; ++r) {
          cudaEventRecord(a, s);
          k_zc<<<ctas, 128, 0, s>>>(ds, dd, dl, n);
          cudaEventRecord(b, s);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          best_dev = std::min(best_dev, (double)ms * 1e3);
        }
        printf("piece %7llu n %5d  zc%-3d :                     device %8.1f us  %6.1f GB/s\n",
               (unsigned long long)piece, n, ctas, best_dev, bytes / best_dev / 1e3);
      }
      cudaFree(ds);
      cudaFree(dd);
      cudaFree(dl);
    }
  }
  // 4. CE + SM on the link at once (256 MiB each; SM side as 4096 x 64 KiB items, 16 CTAs)
  {
    const uint64_t n = 256ull << 20, items = 4096, piece = n / items;
    std::vector<uint64_t> hs(items), hd(items), hl(items, piece);
    for (uint64_t i = 0; i < items; ++i) {
      hs[i] = (uint64_t)(d + n + i * piece);
      hd[i] = (uint64_t)(h + n + i * piece);
    }
    uint64_t *ds, *dd, *dl;
    cudaMalloc(&ds, items * 8);
    cudaMalloc(&dd, items * 8);
    cudaMalloc(&dl, items * 8);
    cudaMemcpy(ds, hs.data(), items * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dd, hd.data(), items * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dl, hl.data(), items * 8, cudaMemcpyHostToDevice);
    cudaEvent_t c;
    cudaEventCreate(&c);
    for (int r = 0; r < 3; ++r) {
      cudaDeviceSynchronize();
      cudaEventRecord(a, s);
      cudaStreamWaitEvent(s2, a, 0);
      cudaMemcpyAsync(h, d, n, cudaMemcpyDeviceToHost, s);
      k_zc<<<16, 128, 0, s2>>>(ds, dd, dl, (int)items);
      cudaEventRecord(c, s2);
      cudaStreamWaitEvent(s, c, 0);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("CE 256 MiB || SM 256 MiB: %.1f GB/s combined\n", 2.0 * n / (ms * 1e-3) / 1e9);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
