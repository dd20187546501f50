// Fixed-cost breakdown of k_hash_chunks: CUDA-event time of single launches
// (after an L2-flushing memset) for an empty kernel, an empty kernel holding
// the hash's 192 KiB of dynamic shared memory, the hash with no work (table
// prologue only), and the hash over 1 / 148 / 1526 chunks.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/hash_micro tools/hash_micro.cu
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <vector>

#define POS_HASH_PROF 1
#include "../paper_2405_12079_b200/csrc/kernels.cuh"

using namespace posdump;

__global__ void k_empty() {}
__global__ void k_empty_smem() {
  extern __shared__ uint8_t s[];
  if (threadIdx.x == 1023) s[0] = 0;
}
__global__ void __launch_bounds__(512) k_empty_512() {}

#define CK(x)                                                             \
  do {                                                                    \
    cudaError_t e = (x);                                                  \
    if (e != cudaSuccess) {                                               \
      std::printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
      return 1;                                                           \
    }                                                                     \
  } while (0)

int main() {
  const uint64_t CS = 65536, NCH = 1526;
  uint8_t* data;
  CK(cudaMalloc(&data, NCH * CS));
  CK(cudaMemset(data, 7, NCH * CS));
  uint8_t* flush;
  const size_t FL = 256u << 20;
  CK(cudaMalloc(&flush, FL));
  std::vector<uint32_t> h(7 * 1024);
  build_advance_table(512, h.data());
  build_advance_table(4, h.data() + 1024);
  for (int k = 0; k < 5; ++k) build_advance_table(16u << k, h.data() + 1024 * (2 + k));
  std::vector<uint32_t> xi(512);
  for (int n = 0; n < 512; ++n) xi[n] = xinv8nmodp(n);
  uint32_t *tables, *xinv, *dcur, *dprev, *bitmap;
  uint8_t* flags;
  CK(cudaMalloc(&tables, h.size() * 4));
  CK(cudaMalloc(&xinv, 2048));
  CK(cudaMemcpy(tables, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(xinv, xi.data(), 2048, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&dcur, NCH * 4));
  CK(cudaMalloc(&dprev, NCH * 4));
  CK(cudaMalloc(&bitmap, NCH));
  CK(cudaMalloc(&flags, NCH));
  // one buffer per 64 chunks
  std::vector<DevBuf> bufs;
  std::vector<uint2> cmap;
  for (uint64_t c0 = 0; c0 < NCH; c0 += 64) {
    DevBuf b{};
    const uint64_t n = std::min<uint64_t>(64, NCH - c0);
    b.ptr = (uint64_t)(data + c0 * CS);
    b.size = n * CS;
    b.handle = bufs.size() + 1;
    b.chunk_base = c0;
    b.nchunks = (uint32_t)n;
    b.k_tail = zeros_crc(CS);
    b.x8_tail = x8nmodp(CS);
    for (uint32_t k = 0; k < n; ++k) cmap.push_back(make_uint2((uint32_t)bufs.size(), k));
    bufs.push_back(b);
  }
  DevBuf* dbufs;
  uint2* dmap;
  CK(cudaMalloc(&dbufs, bufs.size() * sizeof(DevBuf)));
  CK(cudaMalloc(&dmap, cmap.size() * sizeof(uint2)));
  CK(cudaMemcpy(dbufs, bufs.data(), bufs.size() * sizeof(DevBuf), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dmap, cmap.data(), cmap.size() * sizeof(uint2), cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(k_hash_chunks<kModeHash>, cudaFuncAttributeMaxDynamicSharedMemorySize, kHashSmem));
  CK(cudaFuncSetAttribute(k_empty_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, kHashSmem));

  HashParams p{};
  p.bufs = dbufs;
  p.chunk_map = dmap;
  p.chunk_size = CS;
  p.k_full = zeros_crc(CS);
  p.tables = tables;
  p.xinv = xinv;
  p.digest_cur = dcur;
  p.digest_prev = dprev;
  p.flags = flags;
  p.bitmap = bitmap;
  p.nseg = 1;
  p.seg_bytes = (uint32_t)CS;

  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  auto timed = [&](const char* name, auto launch, bool do_flush) {
    std::vector<float> t;
    for (int i = 0; i < 14; ++i) {
      if (do_flush) cudaMemsetAsync(flush, i, FL, s);
      cudaEventRecord(a, s);
      launch();
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (i >= 4) t.push_back(ms * 1e3f);
    }
    std::sort(t.begin(), t.end());
    // back-to-back: 20 launches between one event pair
    cudaEventRecord(a, s);
    for (int i = 0; i < 20; ++i) launch();
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    std::printf("%-34s %s single median %7.2f us  min %7.2f   back-to-back %7.2f us/launch\n", name,
                do_flush ? "flush" : "warm ", t[t.size() / 2], t[0], ms * 1e3f / 20);
    return cudaGetLastError();
  };
  // phase stamps of one flushed launch per size (POS_HASH_PROF)
  static unsigned long long prof[1024][16][5];
  for (uint32_t pf : {0u, 65536u, 16384u, 1u})
  for (uint64_t n : {1ull, 148ull, 1526ull}) {
    HashParams q = p;
    q.n_items = n;
    q.pf_bytes = pf;  // > 1: L2 bulk prefetch of the chunk's first pf bytes at its start; 1: sliding window
    q.pad3 = 32;
    for (int rep = 0; rep < 3; ++rep) {
      std::memset(prof, 0, sizeof prof);
      CK(cudaMemcpyToSymbol(g_hash_prof, prof, sizeof prof));
      cudaMemsetAsync(flush, rep, FL, s);
      k_hash_chunks<kModeHash><<<148, 512, kHashSmem, s>>>(q);
      CK(cudaStreamSynchronize(s));
    }
    CK(cudaMemcpyFromSymbol(prof, g_hash_prof, sizeof prof));
    unsigned long long t0 = ~0ull;
    for (int b = 0; b < 148; ++b)
      for (int w = 0; w < 16; ++w)
        if (prof[b][w][0]) t0 = std::min(t0, prof[b][w][0]);
    std::vector<double> ph[5], chain;
    for (int b = 0; b < 148; ++b)
      for (int w = 0; w < 16; ++w) {
        if (!prof[b][w][2]) continue;
        for (int k = 0; k < 5; ++k) ph[k].push_back((prof[b][w][k] - t0) / 1e3);
        chain.push_back((prof[b][w][3] - prof[b][w][2]) / 1e3);
      }
    auto med = [](std::vector<double> v) { std::sort(v.begin(), v.end()); return v[v.size() / 2]; };
    auto mx = [](const std::vector<double>& v) { return *std::max_element(v.begin(), v.end()); };
    std::printf("pf=%-6u n=%-5llu warps %4zu | entry %5.2f/%5.2f tables %5.2f/%5.2f record %5.2f/%5.2f crc %5.2f/%5.2f "
                "done %5.2f/%5.2f us (median/max from first entry) | chain %5.2f/%5.2f\n",
                pf, (unsigned long long)n, chain.size(), med(ph[0]), mx(ph[0]), med(ph[1]), mx(ph[1]), med(ph[2]),
                mx(ph[2]), med(ph[3]), mx(ph[3]), med(ph[4]), mx(ph[4]), med(chain), mx(chain));
  }
  for (bool fl : {true, false}) {
    CK(timed("empty <<<148,512>>>", [&] { k_empty_512<<<148, 512, 0, s>>>(); }, fl));
    CK(timed("empty + 192 KiB smem", [&] { k_empty_smem<<<148, 512, kHashSmem, s>>>(); }, fl));
    for (uint64_t n : {0ull, 1ull, 148ull, 1526ull}) {
      char name[64];
      std::snprintf(name, sizeof name, "k_hash_chunks n_items=%llu", (unsigned long long)n);
      HashParams q = p;
      q.n_items = n;
      CK(timed(name, [&] { k_hash_chunks<kModeHash><<<148, 512, kHashSmem, s>>>(q); }, fl));
    }
  }
  return 0;
}
