// Can cp.async.bulk (TMA bulk copy) read from / write to host-mapped pinned memory?
// One CTA per 2560-byte "cell": bulk load -> +1 -> bulk store back, in place, on a
// mapped host buffer.  Prints errors and the GB/s of the in-place round trip.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(double* q, int per) {
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) uint64_t bar;
  double* cell = q + (size_t)blockIdx.x * per;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar)), "r"(per * 8) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(s32(sm)), "l"(cell), "r"(per * 8), "r"(s32(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(s32(&bar)) : "memory");
  for (int i = threadIdx.x; i < per; i += blockDim.x) sm[i] += 1.0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(cell), "r"(s32(sm)), "r"(per * 8) : "memory");
    asm volatile("cp.async.bulk.commit_group;\ncp.async.bulk.wait_group 0;" ::: "memory");
  }
}
int main() {
  const int cells = 19683, per = 320;
  size_t bytes = (size_t)cells * per * 8;
  double* h; cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
  for (size_t i = 0; i < (size_t)cells * per; ++i) h[i] = (double)i;
  double* d; cudaHostGetDevicePointer(&d, h, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k<<<cells, 64, per * 8>>>(d, per);
  cudaError_t e = cudaDeviceSynchronize();
  printf("first launch: %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  const int R = 10;
  cudaEventRecord(a);
  for (int r = 0; r < R; ++r) k<<<cells, 64, per * 8>>>(d, per);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  long bad = 0;
  for (size_t i = 0; i < (size_t)cells * per; ++i) bad += h[i] != (double)i + 1 + R;
  printf("mismatches %ld; in-place round trip %.3f ms per pass (%.1f GB/s each way)\n", bad, ms / R,
         bytes / (ms / R * 1e-3) / 1e9);
  return 0;
}
