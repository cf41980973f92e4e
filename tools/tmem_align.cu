// Does tcgen05.ld / st with .x4 / .x8 / .x16 need the column address aligned to the
// access width?  Writes known values column by column (.x1), reads them back with a
// wide load at every offset 0..15 and checks; prints per (width, offset) ok / bad.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int W>
__device__ void ld_wide(uint32_t a, uint32_t (&r)[W]);
template <>
__device__ void ld_wide<4>(uint32_t a, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(a));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
template <>
__device__ void ld_wide<8>(uint32_t a, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "r"(a));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

template <int W>
__global__ void probe(int* out) {
  __shared__ uint32_t base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;\n"
                 "tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::"r"(smem_u32(&base)) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t t = base + ((uint32_t)(32 * warp) << 16);
  for (int c = 0; c < 64; ++c) {
    const uint32_t v = (uint32_t)(lane * 1000 + c);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(t + c), "r"(v) : "memory");
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  for (int off = 0; off < 16; ++off) {
    uint32_t r[W];
    ld_wide<W>(t + off, r);
    int ok = 1;
    for (int i = 0; i < W; ++i) ok &= (r[i] == (uint32_t)(lane * 1000 + off + i));
    ok = __all_sync(0xffffffffu, ok);
    if (threadIdx.x == 0) out[off] = ok;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(base) : "memory");
}

int main() {
  int* d;
  int h[16];
  cudaMalloc(&d, 64);
  probe<4><<<1, 32>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
  printf("x4: %s |", cudaGetErrorString(e));
  for (int i = 0; i < 16; ++i) printf(" %d", h[i]);
  printf("\n");
  probe<8><<<1, 32>>>(d);
  e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
  printf("x8: %s |", cudaGetErrorString(e));
  for (int i = 0; i < 16; ++i) printf(" %d", h[i]);
  printf("\n");
  return 0;
}
