// Can cp.async.bulk (TMA bulk copy) read from / write to host-mapped pinned memory?
// One CTA per 2560-byte "cell": bulk load -> +1 -> bulk store back, in place, on a
// mapped host buffer.  Prints errors and the GB/s of the in-place round trip.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const double* qi, double* q, int per) {
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) uint64_t bar;
  double* cell = q + (size_t)blockIdx.x * per;
  const double* icell = qi + (size_t)blockIdx.x * per;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar)), "r"(per * 8) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(s32(sm)), "l"(icell), "r"(per * 8), "r"(s32(&bar)) : "memory");
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
  double* h2; cudaHostAlloc(&h2, bytes, cudaHostAllocMapped);
  for (size_t i = 0; i < (size_t)cells * per; ++i) h[i] = (double)i;
  double* dh; cudaHostGetDevicePointer(&dh, h, 0);
  double *dev, *dev2; cudaMalloc(&dev, bytes); cudaMalloc(&dev2, bytes);
  cudaMemcpy(dev, h, bytes, cudaMemcpyHostToDevice);
  cudaStream_t s1, s2; cudaStreamCreate(&s1); cudaStreamCreate(&s2);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int R = 10;
  auto time = [&](const char* name, auto f) {
    f(); cudaDeviceSynchronize();
    cudaError_t e = cudaGetLastError();
    cudaEventRecord(a, s1);
    for (int r = 0; r < R; ++r) f();
    cudaStreamWaitEvent(s1, b, 0);
    cudaDeviceSynchronize();
    cudaEventRecord(b, s1); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%-44s %s  %.3f ms per pass (50 MB)\n", name, cudaGetErrorString(e), ms / R);
  };
  time("host->host in place (kernel, TMA)", [&] { k<<<cells, 64, per * 8, s1>>>(dh, dh, per); });
  time("host read -> device write (kernel, TMA)", [&] { k<<<cells, 64, per * 8, s1>>>(dh, dev, per); });
  time("device read -> host write (kernel, TMA)", [&] { k<<<cells, 64, per * 8, s1>>>(dev, dh, per); });
  time("device -> device (kernel, TMA)", [&] { k<<<cells, 64, per * 8, s1>>>(dev, dev2, per); });
  time("CE H2D alone", [&] { cudaMemcpyAsync(dev2, h2, bytes, cudaMemcpyHostToDevice, s1); });
  time("CE D2H alone", [&] { cudaMemcpyAsync(h2, dev2, bytes, cudaMemcpyDeviceToHost, s1); });
  time("CE H2D + CE D2H concurrent", [&] {
    cudaMemcpyAsync(dev2, h2, bytes, cudaMemcpyHostToDevice, s2);
    cudaMemcpyAsync(h, dev, bytes, cudaMemcpyDeviceToHost, s1);
    cudaEventRecord(b, s2); cudaStreamWaitEvent(s1, b, 0); });
  time("CE H2D + kernel host write concurrent", [&] {
    cudaMemcpyAsync(dev2, h2, bytes, cudaMemcpyHostToDevice, s2);
    k<<<cells, 64, per * 8, s1>>>(dev, dh, per);
    cudaEventRecord(b, s2); cudaStreamWaitEvent(s1, b, 0); });
  cudaStream_t s3; cudaStreamCreate(&s3);
  std::vector<cudaEvent_t> ei(64), ek(64);
  for (int i = 0; i < 64; ++i) { cudaEventCreateWithFlags(&ei[i], cudaEventDisableTiming); cudaEventCreateWithFlags(&ek[i], cudaEventDisableTiming); }
  for (int c : {1, 4, 8, 16, 23, 32}) {
    char nm[96];
    snprintf(nm, sizeof nm, "CE H2D + CE D2H, %d chunks, no deps", c);
    const size_t cb = bytes / c / 2560 * 2560;
    auto off = [&](int i) { return i == c ? bytes : (size_t)i * cb; };
    time(nm, [&] {
      for (int i = 0; i < c; ++i) {
        cudaMemcpyAsync((char*)dev2 + off(i), (char*)h2 + off(i), off(i + 1) - off(i), cudaMemcpyHostToDevice, s2);
        cudaMemcpyAsync((char*)h + off(i), (char*)dev + off(i), off(i + 1) - off(i), cudaMemcpyDeviceToHost, s1);
      }
      cudaEventRecord(b, s2); cudaStreamWaitEvent(s1, b, 0); });
    snprintf(nm, sizeof nm, "pipeline H2D->kernel->D2H, %d chunks", c);
    time(nm, [&] {
      for (int i = 0; i < c; ++i) {
        cudaMemcpyAsync((char*)dev2 + off(i), (char*)h2 + off(i), off(i + 1) - off(i), cudaMemcpyHostToDevice, s2);
        cudaEventRecord(ei[i], s2);
      }
      for (int i = 0; i < c; ++i) {
        cudaStreamWaitEvent(s3, ei[i], 0);
        const int c0 = off(i) / 2560, c1 = off(i + 1) / 2560;
        k<<<c1 - c0, 64, per * 8, s3>>>(dev2 + (size_t)c0 * per, dev + (size_t)c0 * per, per);
        cudaEventRecord(ek[i], s3);
        cudaStreamWaitEvent(s1, ek[i], 0);
        cudaMemcpyAsync((char*)h + off(i), (char*)dev + off(i), off(i + 1) - off(i), cudaMemcpyDeviceToHost, s1);
      }
      cudaEventRecord(b, s2); cudaStreamWaitEvent(s1, b, 0); });
  }
  return 0;
}
