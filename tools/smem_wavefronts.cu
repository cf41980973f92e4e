// Shared-memory wavefront microbenchmark (run under ncu on the B200):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/smemwf tools/smem_wavefronts.cu
//   ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__inst_executed_op_shared_ld.sum /tmp/smemwf
// One warp, one kernel launch per lane-address pattern; every launch issues REPS
// shared loads of the pattern, so wavefronts / instructions = the cost of one
// warp-wide load with that pattern.  Patterns are in doubles (8-byte words).
#include <cstdio>
#include <cuda_runtime.h>

constexpr int REPS = 256;

template <int W>   // W = 1: 8-byte loads, 2: 16-byte loads
__global__ void probe(const int* __restrict__ pat, double* out) {
  __shared__ __align__(16) double s[4096];
  for (int i = threadIdx.x; i < 4096; i += 32) s[i] = i;
  __syncwarp();
  const int k = pat[threadIdx.x] & 4095;
  const unsigned addr = (unsigned)__cvta_generic_to_shared(s + (W == 2 ? (k & ~1) : k));
  double acc = 0.0;
#pragma unroll 1
  for (int r = 0; r < REPS; ++r) {
    if (W == 1) {
      double x;
      asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(x) : "r"(addr));
      acc += x;
    } else {
      double x, y;
      asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(addr));
      acc += x + y;
    }
  }
  out[threadIdx.x] = acc;
}

int main() {
  struct P { const char* name; int w; int a[32]; };
  P pats[32];
  int np = 0;
  auto add = [&](const char* name, int w, auto f) {
    pats[np].name = name; pats[np].w = w;
    for (int l = 0; l < 32; ++l) pats[np].a[l] = f(l);
    ++np;
  };
  add("same address", 1, [](int) { return 0; });
  add("2 distinct, lane halves, same 128B", 1, [](int l) { return l < 16 ? 0 : 1; });
  add("4 consecutive", 1, [](int l) { return l & 3; });
  add("8 consecutive", 1, [](int l) { return l & 7; });
  add("16 consecutive (one 128B line)", 1, [](int l) { return l & 15; });
  add("16 consecutive, offset 8 (two lines)", 1, [](int l) { return 8 + (l & 15); });
  add("32 consecutive", 1, [](int l) { return l; });
  add("8 distinct, stride 17 (distinct banks)", 1, [](int l) { return 17 * (l & 7); });
  add("16 distinct, stride 17 (distinct banks)", 1, [](int l) { return 17 * (l & 15); });
  add("8 distinct, stride 16 (one bank pair)", 1, [](int l) { return 16 * (l & 7); });
  add("halves: 0..15 | 16..31", 1, [](int l) { return l; });
  add("halves both 0..15", 1, [](int l) { return l & 15; });
  add("lane groups of 4 share (8 distinct, stride 17)", 1, [](int l) { return 17 * (l >> 2); });
  add("lane groups of 2 share (16 distinct, stride 17)", 1, [](int l) { return 17 * (l >> 1); });
  add("2 distinct far apart (0, 1000)", 1, [](int l) { return (l & 1) ? 1001 : 0; });
  add("4 distinct, one per lane quarter, distinct banks", 1, [](int l) { return 49 * (l >> 3); });
  add("16B: same address", 2, [](int) { return 0; });
  add("16B: 8 consecutive chunks", 2, [](int l) { return 2 * (l & 7); });
  add("16B: 32 consecutive chunks", 2, [](int l) { return 2 * l; });
  add("16B: 4 distinct chunks", 2, [](int l) { return 2 * (l & 3); });
  int* dpat;
  double* dout;
  cudaMalloc(&dpat, 32 * sizeof(int));
  cudaMalloc(&dout, 32 * sizeof(double));
  for (int i = 0; i < np; ++i) {
    cudaMemcpy(dpat, pats[i].a, 32 * sizeof(int), cudaMemcpyHostToDevice);
    if (pats[i].w == 1) probe<1><<<1, 32>>>(dpat, dout);
    else probe<2><<<1, 32>>>(dpat, dout);
    cudaDeviceSynchronize();
    printf("launch %2d: %s\n", i, pats[i].name);
  }
  printf("REPS %d\n", REPS);
  return 0;
}
