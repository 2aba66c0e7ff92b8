// Bulk-copy (cp.async.bulk global -> shared) throughput per SM and chip-wide:
// one producer thread per CTA issues `copies` copies of `bytes` each into a
// ring of `depth` shared-memory slots (mbarrier per slot, complete_tx), the
// same pattern as conv_ss's producer.  Source: a buffer of `span` bytes read
// round-robin (L2-resident when span << 126 MB).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_bulk tools/ubench_bulk.cu
//   tools/ubench_bulk
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void bulk_kernel(const uint8_t* src, size_t span, int bytes, int copies, int depth, int per_stage,
                            unsigned long long* cycles) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar[16];
  if (threadIdx.x == 0) {
    for (int i = 0; i < depth; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const unsigned long long t0 = clock64();
  size_t off = (size_t)blockIdx.x * 65536 % span;
  uint32_t ph[16] = {0};
  for (int c = 0; c < copies; ++c) {
    const int s = c % depth;
    const uint32_t b = smem_u32(&bar[s]);
    if (c >= depth) {
      // wait for this slot's previous fill
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(b), "r"(ph[s]) : "memory");
      ph[s] ^= 1;
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes * per_stage) : "memory");
    for (int k = 0; k < per_stage; ++k) {
      const uint32_t dst = smem_u32(smem + (size_t)(s * per_stage + k) * bytes);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(dst), "l"(src + off), "r"(bytes), "r"(b) : "memory");
      off += 4099 * 16;
      if (off + bytes > span) off = (off + bytes) % (span - bytes) & ~(size_t)15;
    }
  }
  for (int s = 0; s < depth && s < copies; ++s) {
    uint32_t ok = 0;
    const uint32_t b = smem_u32(&bar[s]);
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(b), "r"(ph[s]) : "memory");
  }
  cycles[blockIdx.x] = clock64() - t0;
}

// all copies of the launch issued back to back (no slot reuse), one
// mbarrier for all: is the TMA engine pipelining independent copies?
__global__ void burst_kernel(const uint8_t* src, size_t span, int bytes, int copies, unsigned long long* cycles,
                             int lanes) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t b = smem_u32(&bar);
  const unsigned long long t0 = clock64();
  if (threadIdx.x == 0)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes * copies) : "memory");
  __syncthreads();
  if ((int)threadIdx.x < lanes) {
    for (int c = threadIdx.x; c < copies; c += lanes) {
      size_t off = ((size_t)blockIdx.x * 131 + c) * 65536 % (span - bytes);
      off &= ~(size_t)15;
      const uint32_t dst = smem_u32(smem + (size_t)c * bytes);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(dst), "l"(src + off), "r"(bytes), "r"(b) : "memory");
    }
  }
  if (threadIdx.x == 0) {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(b), "r"(0) : "memory");
    cycles[blockIdx.x] = clock64() - t0;
  }
}

int main() {
  const size_t span = 32u << 20;
  uint8_t* src;
  cudaMalloc(&src, span);
  cudaMemset(src, 1, span);
  unsigned long long* cyc;
  cudaMalloc(&cyc, 148 * sizeof(unsigned long long));
  unsigned long long h[148];
  cudaFuncSetAttribute(burst_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  printf("burst: grid bytes copies lanes -> total cycles  cycles/copy  B/cyc/SM\n");
  for (int grid : {1, 148})
    for (int bytes : {1024, 5248, 16384})
      for (int copies : {1, 4, 8, 16, 32})
        for (int lanes : {1, 32}) {
          if ((size_t)bytes * copies > 190 * 1024 || lanes > copies) continue;
          for (int rep = 0; rep < 3; ++rep)
            burst_kernel<<<grid, 32, 200 * 1024>>>(src, span, bytes, copies, cyc, lanes);
          cudaDeviceSynchronize();
          cudaMemcpy(h, cyc, grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
          double mx = 0;
          for (int i = 0; i < grid; ++i) mx = mx > h[i] ? mx : (double)h[i];
          printf("%4d %6d %3d %3d -> %8.0f  %8.1f  %7.1f\n", grid, bytes, copies, lanes, mx, mx / copies,
                 (double)bytes * copies / mx);
        }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
