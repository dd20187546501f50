// Why a launch-bound application slows down while the copy engine saturates
// the host link: an iteration of 9 short HBM kernels (125 MB fills, ~25 us
// each) timed alone and beside a continuous D2H into pinned memory, issued
// as 9 stream launches or as one CUDA graph launch.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/frontend_micro tools/frontend_micro.cu -lpthread
#include <cuda_runtime.h>
#include <atomic>
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
  auto ce_loop = [&]() {  // windowed 16 MiB slices, 3 in flight, until stopped
    cudaEvent_t ring[3];
    for (auto& e : ring) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    uint64_t k = 0;
    while (!stop.load()) {
      if (k >= 3) cudaEventSynchronize(ring[k % 3]);
      const size_t o = (k * S) % ce_bytes;
      cudaMemcpyAsync(ce_dst + o, ce_src + o, S, cudaMemcpyDeviceToHost, ce);
      cudaEventRecord(ring[k % 3], ce);
      ++k;
    }
    cudaStreamSynchronize(ce);
    for (auto& e : ring) cudaEventDestroy(e);
  };
  run_app(false, 20);
  run_app(true, 20);
  const float alone_s = run_app(false, 400), alone_g = run_app(true, 400);
  std::thread t(ce_loop);
  run_app(false, 20);
  const float ce_s = run_app(false, 400), ce_g = run_app(true, 400);
  stop = true;
  t.join();
  printf("app iteration (9 x 125 MB fill kernels), ms per iteration\n");
  printf("  stream launches : alone %.4f  beside CE D2H %.4f  (%.2fx)\n", alone_s, ce_s, ce_s / alone_s);
  printf("  one graph launch: alone %.4f  beside CE D2H %.4f  (%.2fx)\n", alone_g, ce_g, ce_g / alone_g);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
