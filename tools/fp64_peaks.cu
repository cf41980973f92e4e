// FP64 peak microbenchmarks for the B200 roofline denominators of the ADER-DG path.
//   dfma : CUDA-core DFMA throughput (independent FMA chains per thread)
//   dmma : tensor-core mma.sync.m8n8k4.f64 throughput (DMMA.8x8x4)
//   mixed: DFMA and DMMA interleaved in one warp (do the two pipes add up?)
//   lds  : shared-memory LDS.64 bandwidth (bytes/clk/SM)
// Output: one JSON line per test on stdout.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("{\"error\":\"%s\"}\n", cudaGetErrorString(e)); return 1; } } while (0)

template <int CHAINS>
__global__ void k_dfma(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

template <int CHAINS>
__global__ void k_dmma(double* out, int iters, double a, double b) {
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = threadIdx.x; c[i][1] = i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) dmma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int CM, int CF>
__global__ void k_mixed(double* out, int iters, double a, double b) {
  double c[CM][2];
  double f[CF];
#pragma unroll
  for (int i = 0; i < CM; ++i) { c[i][0] = threadIdx.x; c[i][1] = i; }
#pragma unroll
  for (int i = 0; i < CF; ++i) f[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CM; ++i) dmma(c[i], a, b);
#pragma unroll
    for (int i = 0; i < CF; ++i) f[i] = fma(f[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CM; ++i) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < CF; ++i) s += f[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_lds(double* out, int iters) {
  __shared__ double sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i;
  __syncthreads();
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  int idx = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    volatile double* v = sm;
    s0 += v[(idx) & 4095];
    s1 += v[(idx + 256) & 4095];
    s2 += v[(idx + 512) & 4095];
    s3 += v[(idx + 768) & 4095];
    idx = (idx + 32) & 4095;
  }
  if (s0 + s1 + s2 + s3 == 12345.678) out[0] = s0;
}

int main() {
  int dev = 0; cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  int sms = prop.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  auto timeit = [&](auto launch, int reps) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); return ms / reps;
  };
  const int iters = 4096;
  // DFMA: 8 chains x 256 threads x 4 blocks/SM x sms
  {
    int threads = 256, blocks = sms * 8;
    float ms = timeit([&] { k_dfma<8><<<blocks, threads>>>(out, iters, 0.999999, 1e-7); }, 5);
    double flops = 2.0 * 8 * iters * (double)threads * blocks;
    printf("{\"test\":\"dfma\",\"tflops\":%.3f,\"ms\":%.3f,\"sms\":%d,\"clock_mhz_attr\":%d}\n", flops / ms / 1e9, ms, sms, clk_khz / 1000);
  }
  for (int chains : {4, 8}) {
    int threads = 256, blocks = sms * 8;
    float ms = chains == 4
      ? timeit([&] { k_dmma<4><<<blocks, threads>>>(out, iters, 0.999999, 1e-7); }, 5)
      : timeit([&] { k_dmma<8><<<blocks, threads>>>(out, iters, 0.999999, 1e-7); }, 5);
    double flops = 2.0 * 256 * chains * iters * (double)(threads / 32) * blocks;
    printf("{\"test\":\"dmma_m8n8k4\",\"chains\":%d,\"tflops\":%.3f,\"ms\":%.3f}\n", chains, flops / ms / 1e9, ms);
  }
  {
    int threads = 256, blocks = sms * 8;
    float ms = timeit([&] { k_mixed<4, 8><<<blocks, threads>>>(out, iters, 0.999999, 1e-7); }, 5);
    double fl_m = 2.0 * 256 * 4 * iters * (double)(threads / 32) * blocks;
    double fl_f = 2.0 * 8 * iters * (double)threads * blocks;
    printf("{\"test\":\"mixed_dmma4_dfma8\",\"tflops_total\":%.3f,\"tflops_dmma\":%.3f,\"tflops_dfma\":%.3f,\"ms\":%.3f}\n",
           (fl_m + fl_f) / ms / 1e9, fl_m / ms / 1e9, fl_f / ms / 1e9, ms);
  }
  {
    int threads = 512, blocks = sms * 4;
    float ms = timeit([&] { k_lds<<<blocks, threads>>>(out, iters); }, 5);
    double bytes = 4.0 * 8 * iters * (double)threads * blocks;
    printf("{\"test\":\"lds64\",\"TBps\":%.3f,\"bytes_per_clk_per_sm_at_attr_clock\":%.1f}\n", bytes / ms / 1e9,
           bytes / (ms * 1e-3) / sms / (clk_khz * 1e3));
  }
  return 0;
}
