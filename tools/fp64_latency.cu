// Dependent-chain latency of DFMA, DMMA.8x8x4 and LDS.64 on one warp (clock64).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, int n, double a, double b) {
  __shared__ double sm[64];
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  double x = threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  double c0 = x, c1 = 0.0;
  for (int i = 0; i < n; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  long long t2 = clock64();
  int idx = threadIdx.x & 31;
  for (int i = 0; i < n; ++i) { idx = (int)sm[idx] & 31; }
  long long t3 = clock64();
  out[threadIdx.x] = c0 + c1 + idx;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 64);
  int n = 4096;
  lat<<<1, 32>>>(o, c, n, 0.999, 1e-9);
  lat<<<1, 32>>>(o, c, n, 0.999, 1e-9);
  long long h[3]; cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
  printf("{\"dfma_latency_cycles\": %.2f, \"dmma_latency_cycles\": %.2f, \"lds_dep_latency_cycles\": %.2f}\n",
         (double)h[0] / n, (double)h[1] / n, (double)h[2] / n);
  return 0;
}
