// Host-link probe: SM-driven writes into mapped pinned host memory (zero copy)
// vs the copy engine (cudaMemcpyAsync D2H), for the pack D2H leg.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/zerocopy_micro tools/zerocopy_micro.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_st(const uint4* src, uint4* dst, uint64_t n16) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// TMA bulk: G->S then S->G (dst may be host-mapped), one elected thread, 4 x 16 KiB ring.
__global__ void k_bulk(const uint8_t* src, uint8_t* dst, uint64_t bytes) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 4 * 16384);
  if (threadIdx.x) return;
  for (int s = 0; s < 4; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar + s)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint32_t phase = 0;
  const uint64_t piece = 16384;
  uint64_t npieces = bytes / piece;
  int k = 0;
  for (uint64_t p = blockIdx.x; p < npieces; p += gridDim.x, ++k) {
    int s = k & 3;
    uint32_t sa = (uint32_t)__cvta_generic_to_shared(sm + s * piece);
    uint32_t ba = (uint32_t)__cvta_generic_to_shared(bar + s);
    asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ba), "r"((uint32_t)piece) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa),
                 "l"(src + p * piece), "r"((uint32_t)piece), "r"(ba) : "memory");
    asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(ba),
                 "r"((phase >> s) & 1) : "memory");
    phase ^= 1u << s;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + p * piece), "r"(sa),
                 "r"((uint32_t)piece) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const uint64_t bytes = 256ull << 20;
  uint8_t *d, *h;
  cudaMalloc(&d, bytes);
  cudaMemset(d, 3, bytes);
  cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
  cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16384 + 64);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](auto f) {
    float best = 1e9;
    for (int r = 0; r < 4; ++r) {
      cudaEventRecord(a);
      f();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    return bytes / (best * 1e-3) / 1e9;
  };
  printf("copy engine D2H: %.1f GB/s\n", timeit([&] { cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost); }));
  for (int blocks : {4, 8, 16, 32, 64, 148, 296}) {
    double st = timeit([&] { k_st<<<blocks, 512>>>((const uint4*)d, (uint4*)h, bytes / 16); });
    double bk = timeit([&] { k_bulk<<<blocks, 32, 4 * 16384 + 64>>>(d, h, bytes); });
    printf("blocks %3d: st.global.v4 %.1f GB/s   TMA bulk S->G %.1f GB/s\n", blocks, st, bk);
  }
  cudaError_t e = cudaGetLastError();
  printf("err: %s\n", cudaGetErrorString(e));
  return 0;
}
