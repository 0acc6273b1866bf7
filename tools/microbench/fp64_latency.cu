// Dependent-chain latencies on sm_100a (cycles per op, one warp):
// DADD, DMUL, DSETP+select, LDS, I2F.F64.U64.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
__global__ void k(double* out, long long* cyc, int n, double a) {
  __shared__ double sh[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sh[i] = (double)((i * 7) & 1023);
  __syncthreads();
  double x = a, y = 1.0000001;
  long long t0, t1;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dadd_rn(x, y);
  t1 = clock64(); cyc[0] = (t1 - t0) / n;
  // DMUL chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dmul_rn(x, y);
  t1 = clock64(); cyc[1] = (t1 - t0) / n;
  // DSETP + select chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = (x < y) ? x + 0.0 : y;
  t1 = clock64(); cyc[2] = (t1 - t0) / n;
  // LDS chain (index from loaded value)
  int idx = 3;
  t0 = clock64();
  for (int i = 0; i < n; ++i) idx = (int)sh[idx & 1023];
  t1 = clock64(); cyc[3] = (t1 - t0) / n;
  // I2F.F64.U64 chain
  unsigned long long u = 12345;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { double d = (double)u; u = (unsigned long long)__double_as_longlong(d) >> 11; }
  t1 = clock64(); cyc[4] = (t1 - t0) / n;
  out[threadIdx.x] = x + idx + (double)u;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 64);
  k<<<1, 32>>>(o, c, 4096, 1.0); cudaDeviceSynchronize();
  long long h[5]; cudaMemcpy(h, c, 40, cudaMemcpyDeviceToHost);
  printf("DADD %lld  DMUL %lld  DSETP+sel %lld  LDS %lld  I2F.F64.U64+shift %lld cycles/op\n", h[0], h[1], h[2], h[3], h[4]);
}
