// Pinned host image allocation: cudaHostAlloc vs mmap + THP + parallel
// first touch + cudaHostRegister.  Prints GB/s of each.
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main(int argc, char** argv) {
  size_t gb = argc > 1 ? atoll(argv[1]) : 16;
  int nt = argc > 2 ? atoi(argv[2]) : 16;
  size_t n = gb << 30;
  cudaFree(0);
  double t = now();
  void* p = nullptr;
  cudaHostAlloc(&p, n, cudaHostAllocMapped | cudaHostAllocPortable);
  double a = now() - t;
  printf("cudaHostAlloc %zu GiB: %.2f s = %.2f GB/s\n", gb, a, n / a / 1e9);
  t = now(); cudaFreeHost(p); printf("cudaFreeHost %.2f s\n", now() - t);
  for (int huge = 0; huge < 2; ++huge) {
    t = now();
    uint8_t* q = (uint8_t*)mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (huge) madvise(q, n, MADV_HUGEPAGE);
    std::vector<std::thread> th;
    for (int i = 0; i < nt; ++i)
      th.emplace_back([=] { size_t lo = n * i / nt, hi = n * (i + 1) / nt; for (size_t o = lo; o < hi; o += 4096) q[o] = 0; });
    for (auto& x : th) x.join();
    double b = now() - t;
    t = now();
    cudaError_t e = cudaHostRegister(q, n, cudaHostRegisterMapped | cudaHostRegisterPortable);
    double c = now() - t;
    printf("mmap huge=%d touch(%d thr) %.2f s + register %.2f s (%s) = %.2f GB/s\n", huge, nt, b, c,
           cudaGetErrorString(e), n / (b + c) / 1e9);
    // D2H bandwidth into it
    void* d; cudaMalloc(&d, 1ull << 30);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 0;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); cudaMemcpyAsync(q + (size_t)r * (1ull << 30), d, 1ull << 30, cudaMemcpyDeviceToHost); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::max(best, (float)((1ull << 30) / (ms * 1e-3) / 1e9));
    }
    printf("  D2H 1 GiB into it: %.2f GB/s\n", best);
    cudaFree(d);
    t = now(); cudaHostUnregister(q); munmap(q, n); printf("  unregister+munmap %.2f s\n", now() - t);
  }
  return 0;
}
