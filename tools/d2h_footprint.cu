// Does the D2H rate depend on the host destination's footprint?  8 GiB of
// D2H (32 x 256 MiB copies) into: the same 256 MiB region, 8 GiB of
// huge-page registered memory, 8 GiB of cudaHostAlloc memory, and 64 GiB of
// huge-page memory (strided).
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <cstdint>
#include <cstdio>
#include <cstring>
static uint8_t* huge(size_t n) {
  uint8_t* p = (uint8_t*)mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  madvise(p, n, MADV_HUGEPAGE);
  memset(p, 0, n);
  cudaHostRegister(p, n, cudaHostRegisterMapped | cudaHostRegisterPortable);
  return p;
}
int main() {
  const size_t piece = 256ull << 20, n = 32;
  uint8_t* dev; cudaMalloc(&dev, piece * n);
  cudaMemset(dev, 3, piece * n);
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, uint8_t* dst, size_t stride) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a, s);
      for (size_t i = 0; i < n; ++i) cudaMemcpyAsync(dst + i * stride, dev + i * piece, piece, cudaMemcpyDeviceToHost, s);
      cudaEventRecord(b, s); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("%-40s rep %d: %.2f GB/s\n", name, rep, piece * n / (ms * 1e-3) / 1e9);
    }
  };
  uint8_t* small; cudaHostAlloc((void**)&small, piece, 0);
  run("same 256 MiB (cudaHostAlloc)", small, 0);
  uint8_t* h8 = huge(piece * n);
  run("8 GiB huge-page registered", h8, piece);
  run("same 256 MiB of the huge-page range", h8, 0);
  uint8_t* c8; cudaHostAlloc((void**)&c8, piece * n, 0);
  run("8 GiB cudaHostAlloc", c8, piece);
  uint8_t* h64 = huge(piece * n * 8);
  run("64 GiB huge-page, every 8th piece", h64, piece * 8);
  run("64 GiB huge-page, first 8 GiB", h64, piece);
  return 0;
}
