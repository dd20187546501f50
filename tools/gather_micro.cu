// Small STW gathers (config 2: ~200 x 64 KiB DAG-dirty chunks = 13 MB) are
// latency-bound, not HBM-bound.  Variants, event-timed on an idle GPU:
//   bulk P/K : TMA bulk G->S->G, one elected thread, K stages of P bytes, grid-stride over pieces
//   simt U   : 512-thread CTAs, each thread U x 16-B loads in flight, then U stores
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_micro tools/gather_micro.cu
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

struct Item { uint64_t src, dst, len; };

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(b)),
               "r"(parity) : "memory");
}
__device__ __forceinline__ void g2s(void* s, const void* g, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(s)),
               "l"(g), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(b)) : "memory");
}
__device__ __forceinline__ void s2g(void* g, const void* s, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g),
               "r"((uint32_t)__cvta_generic_to_shared(s)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// every item's length is a multiple of P; pieces p = blockIdx.x, +grid, ...
template <uint32_t P, int K>
__global__ void __launch_bounds__(32) k_bulk(const Item* items, uint32_t n, uint32_t ppi) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + K * P);
  if (threadIdx.x) return;
  for (int s = 0; s < K; ++s) mbar_init(bar + s, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const uint64_t np = (uint64_t)n * ppi;
  uint64_t dsts[K];
  uint64_t p = blockIdx.x;
  int issued = 0;
  for (; issued < K && p < np; ++issued, p += gridDim.x) {
    const Item it = items[p / ppi];
    const uint64_t o = (p % ppi) * P;
    dsts[issued] = it.dst + o;
    mbar_expect_tx(bar + issued, P);
    g2s(sm + issued * P, (const void*)(it.src + o), P, bar + issued);
  }
  uint32_t phase = 0;
  int slot = 0;
  for (int done = 0; done < issued; ++done) {
    mbar_wait(bar + slot, (phase >> slot) & 1);
    phase ^= 1u << slot;
    s2g((void*)dsts[slot], sm + slot * P, P);
    if (p < np) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      const Item it = items[p / ppi];
      const uint64_t o = (p % ppi) * P;
      dsts[slot] = it.dst + o;
      mbar_expect_tx(bar + slot, P);
      g2s(sm + slot * P, (const void*)(it.src + o), P, bar + slot);
      p += gridDim.x;
      ++issued;
    }
    slot = (slot + 1) % K;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// all threads: unit = U x 16 B per thread per round, units grid-strided over the concatenation
template <int U>
__global__ void __launch_bounds__(512) k_simt(const Item* items, uint32_t n, uint64_t item_len) {
  const uint64_t per_item16 = item_len / 16;
  const uint64_t total16 = per_item16 * n;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; base < total16; base += stride * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t g = base + u * stride;
      if (g < total16) {
        const Item it = items[g / per_item16];
        v[u] = reinterpret_cast<const uint4*>(it.src)[g % per_item16];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t g = base + u * stride;
      if (g < total16) {
        const Item it = items[g / per_item16];
        reinterpret_cast<uint4*>(it.dst)[g % per_item16] = v[u];
      }
    }
  }
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const uint64_t L = 65536;
  uint8_t *src, *dst, *flush;
  const uint32_t NMAX = 17200;  // config 5's STW delta: 1.125 GB = 17166 x 64 KiB
  cudaMalloc(&src, NMAX * L);
  cudaMalloc(&dst, NMAX * L);
  cudaMalloc(&flush, 256 << 20);
  cudaMemset(src, 5, NMAX * L);
  Item* d_items;
  cudaMalloc(&d_items, NMAX * sizeof(Item));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaFuncSetAttribute(k_bulk<16384, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16384 + 64);
  cudaFuncSetAttribute(k_bulk<4096, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 4096 + 256);
  cudaFuncSetAttribute(k_bulk<8192, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 8192 + 128);
  cudaFuncSetAttribute(k_bulk<4096, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 4096 + 128);
  cudaFuncSetAttribute(k_bulk<32768, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 32768 + 64);
  cudaFuncSetAttribute(k_bulk<16384, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 16384 + 64);
  cudaFuncSetAttribute(k_bulk<16384, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 16384 + 64);
  for (uint32_t n : {50u, 200u, 800u, 2048u, 17166u}) {
    std::vector<Item> h(n);
    for (uint32_t i = 0; i < n; ++i)  // scattered sources (every other chunk of 2n), dense destination
      h[i] = Item{(uint64_t)(src + (uint64_t)((i * 7919ull) % n) * L), (uint64_t)(dst + (uint64_t)i * L), L};
    cudaMemcpy(d_items, h.data(), n * sizeof(Item), cudaMemcpyHostToDevice);
    auto timeit = [&](const char* name, auto fn) {
      std::vector<float> t;
      for (int r = 0; r < 12; ++r) {
        cudaMemsetAsync(flush, r, 256 << 20);  // L2 flush
        cudaEventRecord(a);
        fn();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (r >= 2) t.push_back(ms);
      }
      std::sort(t.begin(), t.end());
      const float med = t[t.size() / 2];
      printf("items %4u (%6.1f MB)  %-22s median %7.2f us  min %7.2f us  %6.0f GB/s (2x bytes)\n", n, n * L / 1e6,
             name, med * 1e3, t[0] * 1e3, 2.0 * n * L / (med * 1e-3) / 1e9);
    };
    timeit("bulk 16K x4, 3/SM", [&] { k_bulk<16384, 4><<<nsm * 3, 32, 4 * 16384 + 64>>>(d_items, n, L / 16384); });
    timeit("bulk 8K x8, 3/SM", [&] { k_bulk<8192, 8><<<nsm * 3, 32, 8 * 8192 + 128>>>(d_items, n, L / 8192); });
    timeit("bulk 4K x16, 3/SM", [&] { k_bulk<4096, 16><<<nsm * 3, 32, 16 * 4096 + 256>>>(d_items, n, L / 4096); });
    timeit("bulk 4K x8, 6/SM", [&] { k_bulk<4096, 8><<<nsm * 6, 32, 8 * 4096 + 128>>>(d_items, n, L / 4096); });
    timeit("bulk 32K x3, 2/SM", [&] { k_bulk<32768, 3><<<nsm * 2, 32, 3 * 32768 + 64>>>(d_items, n, L / 32768); });
    timeit("bulk 16K x6, 2/SM", [&] { k_bulk<16384, 6><<<nsm * 2, 32, 6 * 16384 + 64>>>(d_items, n, L / 16384); });
    timeit("bulk 16K x3, 4/SM", [&] { k_bulk<16384, 3><<<nsm * 4, 32, 3 * 16384 + 64>>>(d_items, n, L / 16384); });
    timeit("simt U=4, 4x148", [&] { k_simt<4><<<nsm * 4, 512>>>(d_items, n, L); });
    timeit("simt U=8, 4x148", [&] { k_simt<8><<<nsm * 4, 512>>>(d_items, n, L); });
    timeit("simt U=2, 4x148", [&] { k_simt<2><<<nsm * 4, 512>>>(d_items, n, L); });
    if (n <= 2048) timeit("cudaMemcpyAsync D2D x n", [&] {
      for (uint32_t i = 0; i < n; ++i) cudaMemcpyAsync((void*)h[i].dst, (const void*)h[i].src, L, cudaMemcpyDeviceToDevice);
    });
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
