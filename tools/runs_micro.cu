// Host-leg alternatives for SHORT copy runs (device buffers -> scattered
// places of a huge-page pinned host image), without the copy-engine batch
// API (closed on this pool): per-run cudaMemcpyAsync round-robin over S
// streams, and an SM zero-copy kernel with G CTAs storing into the mapped
// image.  Each also beside an HBM-bound kernel (its slowdown = interference).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/runs_micro tools/runs_micro.cu
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

__global__ void k_hbm(const uint4* a, uint4* b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = a[i];
    v.x ^= 1;
    b[i] = v;
  }
}

// One CTA per run at a time (grid-stride over runs); 16-B loads/stores.
__global__ void k_ship(const uint64_t* src, const uint64_t* dst, const uint64_t* len, uint32_t n) {
  for (uint32_t r = blockIdx.x; r < n; r += gridDim.x) {
    const uint4* s = reinterpret_cast<const uint4*>(src[r]);
    uint4* d = reinterpret_cast<uint4*>(dst[r]);
    const uint64_t n16 = len[r] / 16;
    for (uint64_t i = threadIdx.x; i < n16; i += blockDim.x) {
      uint4 v;
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                   : "l"(s + i));
      d[i] = v;
    }
  }
}

int main() {
  const uint64_t total = 256ull << 20;
  const uint64_t img_bytes = 2 * total;
  uint8_t* img = (uint8_t*)mmap(nullptr, img_bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  madvise(img, img_bytes, MADV_HUGEPAGE);
  memset(img, 0, img_bytes);
  cudaHostRegister(img, img_bytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
  uint8_t* dimg = nullptr;
  cudaHostGetDevicePointer((void**)&dimg, img, 0);
  uint8_t* dev;
  cudaMalloc(&dev, 2 * total);
  cudaMemset(dev, 7, 2 * total);
  const size_t hn = (1ull << 30) / 16;
  uint4 *ha, *hb;
  cudaMalloc(&ha, hn * 16);
  cudaMalloc(&hb, hn * 16);
  cudaStream_t st[8], ks;
  for (auto& s : st) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&ks, cudaStreamNonBlocking);
  cudaEvent_t e0, e1, k0, k1, ej[8];
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventCreate(&k0);
  cudaEventCreate(&k1);
  for (auto& e : ej) cudaEventCreate(&e);
  uint64_t* drun;
  cudaMalloc(&drun, 3 * 65536 * 8);
  int nsm = 148;
  auto hbm_alone = [&]() {
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(k0, ks);
      k_hbm<<<nsm * 4, 512, 0, ks>>>(ha, hb, hn);
      cudaEventRecord(k1, ks);
      cudaEventSynchronize(k1);
      float ms;
      cudaEventElapsedTime(&ms, k0, k1);
      best = std::min(best, ms);
    }
    return best;
  };
  const float hbm0 = hbm_alone();
  printf("hbm kernel alone (1 GiB copy): %.3f ms\n", hbm0);
  for (uint64_t piece : {65536ull, 262144ull, 458752ull, 1ull << 20, 4ull << 20}) {
    const uint32_t n = (uint32_t)(total / piece);
    std::vector<uint64_t> h(3 * n);
    for (uint32_t i = 0; i < n; ++i) {  // every other piece of the device buffer -> every other of the image
      h[i] = (uint64_t)(dev + 2 * i * piece);
      h[n + i] = (uint64_t)(dimg + 2 * i * piece);
      h[2 * n + i] = piece;
    }
    cudaMemcpy(drun, h.data(), 3 * n * 8, cudaMemcpyHostToDevice);
    auto run_ce = [&](int S) {
      cudaEventRecord(e0, st[0]);
      for (int k = 1; k < S; ++k) cudaStreamWaitEvent(st[k], e0, 0);
      for (uint32_t i = 0; i < n; ++i)
        cudaMemcpyAsync((void*)(img + 2 * i * piece), (const void*)h[i], piece, cudaMemcpyDeviceToHost, st[i % S]);
      for (int k = 1; k < S; ++k) {
        cudaEventRecord(ej[k], st[k]);
        cudaStreamWaitEvent(st[0], ej[k], 0);
      }
      cudaEventRecord(e1, st[0]);
    };
    auto run_sm = [&](int G) {
      cudaEventRecord(e0, st[0]);
      k_ship<<<G, 512, 0, st[0]>>>(drun, drun + n, drun + 2 * n, n);
      cudaEventRecord(e1, st[0]);
    };
    auto measure = [&](const char* name, auto fn, int arg) {
      float best = 1e9, kbest = 1e9, kdur = 0;
      for (int r = 0; r < 4; ++r) {
        fn(arg);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms);
      }
      for (int r = 0; r < 3; ++r) {  // beside the HBM kernel (launched right after the copies start)
        fn(arg);
        cudaEventRecord(k0, ks);
        k_hbm<<<nsm * 4, 512, 0, ks>>>(ha, hb, hn);
        cudaEventRecord(k1, ks);
        cudaEventSynchronize(e1);
        cudaEventSynchronize(k1);
        cudaEventElapsedTime(&kdur, k0, k1);
        kbest = std::min(kbest, kdur);
      }
      printf("piece %8llu n %5u %-10s %2d: %8.1f us %6.1f GB/s | hbm kernel beside: %.3f ms (%.2fx)\n",
             (unsigned long long)piece, n, name, arg, best * 1e3, total / (best * 1e-3) / 1e9, kbest, kbest / hbm0);
    };
    for (int S : {1, 2, 4, 8}) measure("ce_streams", run_ce, S);
    for (int G : {2, 4, 8, 16, 32}) measure("sm_ctas", run_sm, G);
  }
  // correctness spot check of the last SM run
  std::vector<uint8_t> chk(64);
  memcpy(chk.data(), img, 64);
  printf("img[0]=%d err=%s\n", chk[0], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
