// Why the stop-the-world window is longer in direct mode: launch-to-launch
// latency of a kernel chain on one stream (k_stamp: globaltimer into a slot,
// plus one 13 MB gather kernel in the middle) while another stream runs a
// copy-engine D2H of 52 MB, issued as one copy / a cudaMemcpyBatchAsync of N
// runs / N cudaMemcpyAsync calls.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/stw_micro tools/stw_micro.cu
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

#include <cuda_runtime.h>

__global__ void k_stamp(unsigned long long* at) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *at = t;
}

__global__ void k_gather(const uint4* src, uint4* dst, uint64_t n16) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

__global__ void k_spin(uint64_t ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

// The bench's stop sequence: an application stream runs a 300 us kernel and
// records E; the stop is [event 3, stamp, gather, stamp, event 4] either on a
// dump stream that waits on E (cross-stream) or on the application stream
// itself; with and without the CE D2H batch running on a third stream.
static void stop_sequence(uint8_t* d, uint8_t* h, uint64_t D2H, uint8_t* gs, uint8_t* gd, uint64_t G,
                          unsigned long long* st) {
  cudaStream_t app, dump, ce;
  cudaStreamCreateWithFlags(&app, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&dump, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&ce, cudaStreamNonBlocking);
  cudaEvent_t E, e3, e4;
  cudaEventCreateWithFlags(&E, cudaEventDisableTiming);
  cudaEventCreate(&e3);
  cudaEventCreate(&e4);
  const int nruns = 800;
  std::vector<void*> ds(nruns), ss(nruns);
  std::vector<size_t> sz(nruns);
  const uint64_t per = D2H / nruns / 4096 * 4096;
  for (int i = 0; i < nruns; ++i) {
    ds[i] = h + i * per;
    ss[i] = d + i * per;
    sz[i] = per;
  }
  for (int round = 0; round < 3; ++round)
    for (int busy = 0; busy < 2; ++busy)
      for (int same = 0; same < 2; ++same) {
        cudaDeviceSynchronize();
        if (busy) {
          cudaMemcpyAttributes attr{};
          attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
          attr.srcLocHint.type = cudaMemLocationTypeDevice;
          attr.dstLocHint.type = cudaMemLocationTypeHost;
          attr.flags = cudaMemcpyFlagPreferOverlapWithCompute;
          size_t zero = 0, fi = 0;
          cudaMemcpyBatchAsync(ds.data(), ss.data(), sz.data(), nruns, &attr, &zero, 1, &fi, ce);
        }
        k_spin<<<1, 32, 0, app>>>(300000);
        cudaStream_t s = same ? app : dump;
        if (!same) {
          cudaEventRecord(E, app);
          cudaStreamWaitEvent(dump, E, 0);
        }
        cudaEventRecord(e3, s);
        k_stamp<<<1, 1, 0, s>>>(st + 0);
        k_gather<<<148 * 4, 256, 0, s>>>((const uint4*)gs, (uint4*)gd, G / 16);
        k_stamp<<<1, 1, 0, s>>>(st + 1);
        cudaEventRecord(e4, s);
        cudaDeviceSynchronize();
        float ms;
        cudaEventElapsedTime(&ms, e3, e4);
        unsigned long long t[2];
        cudaMemcpy(t, st, sizeof t, cudaMemcpyDeviceToHost);
        if (round == 2)
          std::printf("stop on %-12s %-14s event3->event4 %7.2f us   stamp->stamp (gather) %7.2f us\n",
                      same ? "app stream" : "dump stream", busy ? "CE D2H busy" : "idle", ms * 1e3, (t[1] - t[0]) / 1e3);
      }
}

int main() {
  const uint64_t D2H = 52ull << 20, G = 13ull << 20;
  uint8_t *d, *h, *gs, *gd;
  cudaMalloc(&d, D2H);
  cudaMalloc(&gs, G);
  cudaMalloc(&gd, G);
  cudaHostAlloc((void**)&h, D2H, cudaHostAllocMapped);
  cudaMemset(d, 1, D2H);
  unsigned long long* st;
  cudaMalloc(&st, 64 * 8);
  int lo, hi;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  cudaStream_t sc, ss, ssh;
  cudaStreamCreateWithFlags(&sc, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&ss, cudaStreamNonBlocking);
  cudaStreamCreateWithPriority(&ssh, cudaStreamNonBlocking, hi);
  stop_sequence(d, h, D2H, gs, gd, G, st);
  for (int round = 0; round < 2; ++round)
    for (int mode = 0; mode < 7; ++mode)
      for (int prio = 0; prio < 2; ++prio) {
        cudaStream_t s = prio ? ssh : ss;
        const int nruns = mode == 2 ? 800 : mode == 3 ? 200 : mode == 4 ? 3200 : mode == 5 ? 800 : mode == 6 ? 50 : 1;
        std::vector<void*> ds(nruns), ss2(nruns);
        std::vector<size_t> sz(nruns);
        const uint64_t per = D2H / nruns / 4096 * 4096;
        for (int i = 0; i < nruns; ++i) {
          ds[i] = h + i * per;
          ss2[i] = d + i * per;
          sz[i] = per;
        }
        cudaDeviceSynchronize();
        if (mode == 1) cudaMemcpyAsync(h, d, D2H, cudaMemcpyDeviceToHost, sc);
        if (mode == 2 || mode == 3 || mode == 4 || mode == 6) {
          cudaMemcpyAttributes attr{};
          attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
          attr.srcLocHint.type = cudaMemLocationTypeDevice;
          attr.dstLocHint.type = cudaMemLocationTypeHost;
          attr.flags = cudaMemcpyFlagPreferOverlapWithCompute;
          size_t zero = 0, fi = 0;
          cudaError_t e = cudaMemcpyBatchAsync(ds.data(), ss2.data(), sz.data(), nruns, &attr, &zero, 1, &fi, sc);
          if (e != cudaSuccess) std::printf("batch: %s\n", cudaGetErrorString(e));
        }
        if (mode == 5)
          for (int i = 0; i < nruns; ++i) cudaMemcpyAsync(ds[i], ss2[i], sz[i], cudaMemcpyDeviceToHost, sc);
        for (int i = 0; i < 8; ++i) k_stamp<<<1, 1, 0, s>>>(st + i);
        k_gather<<<148 * 4, 256, 0, s>>>((const uint4*)gs, (uint4*)gd, G / 16);
        for (int i = 8; i < 16; ++i) k_stamp<<<1, 1, 0, s>>>(st + i);
        cudaDeviceSynchronize();
        unsigned long long t[16];
        cudaMemcpy(t, st, sizeof t, cudaMemcpyDeviceToHost);
        std::vector<double> gaps;
        for (int i = 0; i < 7; ++i) gaps.push_back((t[i + 1] - t[i]) / 1e3);
        for (int i = 9; i < 15; ++i) gaps.push_back((t[i + 1] - t[i]) / 1e3);
        std::sort(gaps.begin(), gaps.end());
        static const char* names[] = {"idle", "1 x 52 MB D2H", "batch 800 runs", "batch 200 runs", "batch 3200 runs",
                                      "800 x cudaMemcpyAsync", "batch 50 runs"};
        if (round == 1)
          std::printf("%-24s %s  stamp gap median %7.2f us max %7.2f   stamp7->stamp8 (gather 13 MB) %7.2f us\n",
                      names[mode], prio ? "hi-prio" : "normal ", gaps[gaps.size() / 2], gaps.back(),
                      (t[8] - t[7]) / 1e3);
      }
  return 0;
}
