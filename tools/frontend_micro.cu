// Why a launch-bound application slows down while the copy engine saturates
// the host link: an iteration of 9 short HBM kernels (125 MB fills, ~25 us
// each) timed alone and beside a continuous D2H into pinned memory, issued
// as 9 stream launches or as one CUDA graph launch; and beside a duty-cycled
// D2H (an idle gap after every slice).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/frontend_micro tools/frontend_micro.cu -lpthread
#include <cuda_runtime.h>
#include <atomic>
#include <chrono>
#include <utility>
#include <cstdint>
#include <cstdio>
#include <thread>
#include <vector>

__global__ void k_fill(uint4* p, size_t n16, uint32_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(seed, (uint32_t)i, seed ^ 0x9e3779b9u, (uint32_t)(i >> 32));
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const size_t fill = 125000000 / 16 * 16, K = 9;
  uint8_t* app_mem;
  cudaMalloc(&app_mem, K * fill);
  const size_t ce_bytes = 4ull << 30, S = 16 << 20;
  uint8_t *ce_src, *ce_dst;
  cudaMalloc(&ce_src, ce_bytes);
  cudaHostAlloc(&ce_dst, ce_bytes, cudaHostAllocMapped);
  cudaStream_t app, ce;
  cudaStreamCreateWithFlags(&app, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&ce, cudaStreamNonBlocking);
  auto launch_iter = [&](cudaStream_t s) {
    for (size_t k = 0; k < K; ++k)
      k_fill<<<nsm * 4, 512, 0, s>>>(reinterpret_cast<uint4*>(app_mem + k * fill), fill / 16, (uint32_t)k);
  };
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(app, cudaStreamCaptureModeThreadLocal);
  launch_iter(app);
  cudaStreamEndCapture(app, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run_app = [&](bool graph, int iters) {
    cudaEventRecord(a, app);
    for (int i = 0; i < iters; ++i) {
      if (graph) cudaGraphLaunch(ge, app);
      else launch_iter(app);
    }
    cudaEventRecord(b, app);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / iters;
  };
  std::atomic<bool> stop{false};
  std::atomic<uint64_t> moved{0};
  int gap_us = 0;  // idle time after every slice (a duty cycle below the link)
  size_t slice = S;
  auto ce_loop = [&]() {  // windowed slices, 3 in flight (1 with a gap), until stopped
    cudaEvent_t ring[3];
    for (auto& e : ring) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    uint64_t k = 0;
    const int W = gap_us ? 1 : 3;
    while (!stop.load()) {
      if (k >= (uint64_t)W) cudaEventSynchronize(ring[k % W]);
      if (gap_us && k) {
        auto t0 = std::chrono::steady_clock::now();
        while (std::chrono::steady_clock::now() - t0 < std::chrono::microseconds(gap_us)) {}
      }
      const size_t o = (k * slice) % (ce_bytes - slice);
      cudaMemcpyAsync(ce_dst + o, ce_src + o, slice, cudaMemcpyDeviceToHost, ce);
      cudaEventRecord(ring[k % W], ce);
      moved += slice;
      ++k;
    }
    cudaStreamSynchronize(ce);
    for (auto& e : ring) cudaEventDestroy(e);
  };
  run_app(false, 20);
  run_app(true, 20);
  const float alone_s = run_app(false, 400), alone_g = run_app(true, 400);
  printf("app iteration (9 x 125 MB fill kernels), ms per iteration: alone %.4f (stream launches), %.4f (graph)\n",
         alone_s, alone_g);
  for (auto [g, sl] : {std::pair<int, size_t>{0, S}, {20, S}, {60, S}, {10, 4 << 20}, {30, 4 << 20}}) {
    gap_us = g;
    slice = sl;
    stop = false;
    moved = 0;
    auto t0 = std::chrono::steady_clock::now();
    std::thread t(ce_loop);
    run_app(false, 20);
    const float ce_s = run_app(false, 400), ce_g = run_app(true, 400);
    stop = true;
    t.join();
    const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    printf("  D2H %2d MiB slices, gap %2d us: link %5.1f GB/s | stream launches %.4f (%.2fx)  graph %.4f (%.2fx)\n",
           (int)(sl >> 20), g, moved.load() / sec / 1e9, ce_s, ce_s / alone_s, ce_g, ce_g / alone_g);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
