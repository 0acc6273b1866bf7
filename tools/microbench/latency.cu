// Pointer-chase latency probe (one thread): L1-resident, L2-resident and
// DRAM-resident chains, plus a dependent atomicAdd chain and the
// %globaltimer tick.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 latency.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__global__ void chase(const uint32_t* __restrict__ next, int iters, uint32_t* out, long long* cyc) {
  uint32_t p = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) p = __ldcg(next + p);
  long long t1 = clock64();
  *out = p;
  *cyc = t1 - t0;
}
__global__ void chase_l1(const uint32_t* __restrict__ next, int iters, uint32_t* out, long long* cyc) {
  uint32_t p = 0;
  for (int i = 0; i < iters; ++i) p = __ldca(next + p);  // warm L1
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) p = __ldca(next + p);
  long long t1 = clock64();
  *out = p;
  *cyc = t1 - t0;
}
__global__ void atom_chain(unsigned long long* a, int iters, long long* cyc) {
  unsigned long long v = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v = atomicAdd(a + (v & 1), 1ull);
  long long t1 = clock64();
  a[2] = v;
  *cyc = t1 - t0;
}
__global__ void gtimer(unsigned long long* out) {
  unsigned long long prev, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(prev));
  int changes = 0;
  unsigned long long first = prev, last = prev, mind = ~0ull;
  for (int i = 0; i < 200000 && changes < 64; ++i) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t != last) { if (t - last < mind) mind = t - last; last = t; ++changes; }
  }
  out[0] = mind; out[1] = last - first; out[2] = changes;
}

int main() {
  uint32_t *d, *o; long long* c; unsigned long long* a;
  cudaMalloc(&o, 4); cudaMalloc(&c, 8); cudaMalloc(&a, 64); cudaMemset(a, 0, 64);
  for (size_t bytes : {size_t(16) << 10, size_t(4) << 20, size_t(64) << 20, size_t(1) << 30}) {
    size_t n = bytes / 4;
    std::vector<uint32_t> h(n);
    // random cyclic permutation with 128 B stride between consecutive hops
    size_t lines = n / 32;
    std::vector<uint32_t> perm(lines);
    for (size_t i = 0; i < lines; ++i) perm[i] = i;
    uint64_t s = 88172645463325252ull;
    for (size_t i = lines - 1; i > 0; --i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; std::swap(perm[i], perm[s % (i + 1)]); }
    for (size_t i = 0; i < lines; ++i) h[perm[i] * 32] = perm[(i + 1) % lines] * 32;
    cudaMalloc(&d, bytes);
    cudaMemcpy(d, h.data(), bytes, cudaMemcpyHostToDevice);
    int iters = 20000;
    chase<<<1, 1>>>(d, 2000, o, c);  // warm
    chase<<<1, 1>>>(d, iters, o, c);
    long long cy; cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
    printf("chase ldcg %8zu KB: %.1f cycles/hop\n", bytes >> 10, double(cy) / iters);
    if (bytes <= (size_t(16) << 10)) {
      chase_l1<<<1, 1>>>(d, 2000, o, c);
      cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
      printf("chase ldca (L1) %zu KB: %.1f cycles/hop\n", bytes >> 10, double(cy) / 2000);
    }
    cudaFree(d);
  }
  atom_chain<<<1, 1>>>(a, 5000, c);
  long long cy; cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
  printf("dependent atomicAdd: %.1f cycles/op\n", double(cy) / 5000);
  unsigned long long g[3];
  gtimer<<<1, 1>>>(a);
  cudaMemcpy(g, a, 24, cudaMemcpyDeviceToHost);
  printf("globaltimer min tick %llu ns over %llu changes (span %llu ns)\n", g[0], g[2], g[1]);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SM clock attr %d kHz\n", clk);
  return cudaDeviceSynchronize() != cudaSuccess;
}
