// Host-link D2H variants into a huge-page pinned image: one big copy,
// per-run cudaMemcpyAsync on 1/2/4 streams, cudaMemcpyBatchAsync, and the
// same with an HBM-bound kernel running beside it.  GB/s by CUDA events.
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
__global__ void k_hbm(const uint4* a, uint4* b, size_t n, int reps) {
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      uint4 v = a[i]; v.x ^= r; b[i] = v;
    }
}
int main() {
  const size_t run = 125000000, nrun = 64, stride = (run + 255) / 256 * 256, n = stride * nrun;
  uint8_t* img = (uint8_t*)mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  madvise(img, n, MADV_HUGEPAGE);
  memset(img, 0, n);
  cudaHostRegister(img, n, cudaHostRegisterMapped | cudaHostRegisterPortable);
  uint8_t* dev; cudaMalloc(&dev, n);
  cudaMemset(dev, 1, n);
  uint8_t *h1, *h2; cudaMalloc(&h1, 4ull << 30); cudaMalloc(&h2, 4ull << 30);
  cudaStream_t st[4], ks; for (auto& s : st) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&ks, cudaStreamNonBlocking);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEvent_t ej[4]; for (auto& e : ej) cudaEventCreate(&e);
  auto timed = [&](const char* name, auto fn, bool hbm) {
    cudaDeviceSynchronize();
    if (hbm) k_hbm<<<148 * 4, 512, 0, ks>>>((const uint4*)h1, (uint4*)h2, (4ull << 30) / 16, 8);
    cudaEventRecord(e0, st[0]);
    for (int k = 1; k < 4; ++k) cudaStreamWaitEvent(st[k], e0, 0);
    fn();
    for (int k = 1; k < 4; ++k) { cudaEventRecord(ej[k], st[k]); cudaStreamWaitEvent(st[0], ej[k], 0); }
    cudaEventRecord(e1, st[0]);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-44s %s %.2f GB/s (%.1f ms)\n", name, hbm ? "+hbm" : "    ", n / (ms * 1e-3) / 1e9, ms);
    cudaDeviceSynchronize();
  };
  for (int hbm = 0; hbm < 2; ++hbm) {
    timed("one copy", [&] { cudaMemcpyAsync(img, dev, n, cudaMemcpyDeviceToHost, st[0]); }, hbm);
    for (int ns : {1, 2, 4}) {
      char nm[64]; snprintf(nm, 64, "per-run memcpy, %d stream(s)", ns);
      timed(nm, [&] { for (size_t r = 0; r < nrun; ++r)
        cudaMemcpyAsync(img + r * stride, dev + r * stride, run, cudaMemcpyDeviceToHost, st[r % ns]); }, hbm);
    }
    for (size_t piece : {(size_t)2 << 20, (size_t)8 << 20}) {
      char nm[64]; snprintf(nm, 64, "2 MiB..%zu MiB pieces, 2 streams", piece >> 20);
      timed(nm, [&] { size_t k = 0; for (size_t r = 0; r < nrun; ++r) for (size_t o = 0; o < run; o += piece, ++k)
        cudaMemcpyAsync(img + r * stride + o, dev + r * stride + o, std::min(piece, run - o), cudaMemcpyDeviceToHost, st[k % 2]); }, hbm);
    }
    for (int ns : {1, 2}) {
      char nm[64]; snprintf(nm, 64, "cudaMemcpyBatchAsync, %d stream(s)", ns);
      timed(nm, [&] {
        std::vector<void*> d(nrun), s(nrun); std::vector<size_t> b(nrun, run);
        for (size_t r = 0; r < nrun; ++r) { d[r] = img + r * stride; s[r] = dev + r * stride; }
        cudaMemcpyAttributes a{}; a.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
        a.srcLocHint.type = cudaMemLocationTypeDevice; a.dstLocHint.type = cudaMemLocationTypeHost;
        size_t zero = 0, fi = 0;
        size_t per = nrun / ns;
        for (int k = 0; k < ns; ++k)
          cudaMemcpyBatchAsync(d.data() + k * per, s.data() + k * per, b.data() + k * per, per, &a, &zero, 1, &fi, st[k]);
      }, hbm);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
