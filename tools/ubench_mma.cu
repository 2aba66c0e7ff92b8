// tcgen05.mma kind::f16 issue rate, M = 128, cta_group::1: cycles per MMA
// issued back to back by one elected thread, for N = 16 .. 256, with
//   ss0: both operands in shared memory, constant descriptors
//   ss1: A descriptor moving by a tap offset per MMA (as conv_ss)
//   ts : A in tensor memory, B in shared memory
//   ss2w: ss1 issued by two warps into two accumulators concurrently
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Ipaper_2509_22857_b200/csrc -Iinclude tools/ubench_mma.cu -o tools/ubench_mma
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_fp16.h>
#include "tc_ptx.cuh"
using namespace pcnn;

__device__ __forceinline__ uint32_t elect1() {
  uint32_t e;
  asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 r;\n\telect.sync r|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(e));
  return e;
}
__device__ __forceinline__ void mma_ss(uint32_t e, uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile("{\n\t.reg .pred p, q;\n\tsetp.ne.b32 q, %0, 0;\n\tsetp.ne.b32 p, 1, 0;\n\t"
               "@q tcgen05.mma.cta_group::1.kind::f16 [%1], %2, %3, %4, p;\n\t}"
               ::"r"(e), "r"(d), "l"(a), "l"(b), "r"(idesc) : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t e, uint32_t d, uint32_t a, uint64_t b, uint32_t idesc) {
  asm volatile("{\n\t.reg .pred p, q;\n\tsetp.ne.b32 q, %0, 0;\n\tsetp.ne.b32 p, 1, 0;\n\t"
               "@q tcgen05.mma.cta_group::1.kind::f16 [%1], [%2], %3, %4, p;\n\t}"
               ::"r"(e), "r"(d), "r"(a), "l"(b), "r"(idesc) : "memory");
}

constexpr int kReps = 16, kTaps = 9;

template <int mode>
__global__ void ubench(unsigned long long* out, int N) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 96 * 1024 / 2; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u;
    h ^= h >> 13;
    reinterpret_cast<__half*>(smem)[i] = __float2half(((h & 0xFFFF) / 32768.f - 1.f));
  }
  if (tid == 0) {
    ptx::mbar_init(ptx::smem_u32(&bar[0]), 1);
    ptx::mbar_init(ptx::smem_u32(&bar[1]), 1);
    ptx::mbar_init(ptx::smem_u32(&bar[2]), 1);
    ptx::mbar_init(ptx::smem_u32(&bar[3]), 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc(ptx::smem_u32(&tbase), 512);
  ptx::fence_proxy_async();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tbase;
  const uint32_t a0 = ptx::smem_u32(smem), b0 = ptx::smem_u32(smem + 32768);
  const uint32_t idesc = ptx::idesc_f16(128, N);
  const uint64_t ad = ptx::smem_desc_noswz(a0, 128 * 16, 128);
  const uint64_t bd = ptx::smem_desc_noswz(b0, 256 * 16, 128);
  constexpr int nw = mode == 3 ? 2 : mode == 4 ? 4 : mode == 5 ? 3 : 1;
  long long c = 0;
  if (warp >= 1 && warp <= nw) {
    const uint32_t e = elect1();
    const uint32_t d = tmem + (warp - 1) * (nw > 2 ? 128 : 256);
    __syncwarp();
    const long long t0 = clock64();
    for (int r = 0; r < kReps; ++r) {
#pragma unroll
      for (int t = 0; t < kTaps; ++t) {
        const uint64_t off = (uint64_t)((t / 3) * 33 + (t % 3) + r);
        if (mode == 0 || mode == 6) mma_ss(e, d, ad, bd, idesc);
        else if (mode == 1 || mode == 3 || mode == 4 || mode == 5) mma_ss(e, d, ad + off, bd + t * 4, idesc);
        else mma_ts(e, d, tmem + 256 + (uint32_t)(t & 3) * 8, bd + t * 4, idesc);
      }
    }
    ptx::mma_commit_warp(ptx::smem_u32(&bar[warp - 1]));
    ptx::mbar_wait(ptx::smem_u32(&bar[warp - 1]), 0);
    c = (clock64() - t0) / (kReps * kTaps);
    if ((tid & 31) == 0) out[warp - 1] = c;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(tmem, 512);
}

template <int mode>
void runm(unsigned long long* d, const char* name) {
  cudaFuncSetAttribute(ubench<mode>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  for (int N : {16, 32, 64, 128, 256}) {
    if (mode >= 3 && mode <= 5 && N > (mode == 3 ? 128 : 64)) continue;
    for (int rep = 0; rep < 2; ++rep) ubench<mode><<<1, 160, 96 * 1024>>>(d, N);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
    unsigned long long h[4] = {0, 0, 0, 0};
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-18s N=%3d  %4llu %4llu %4llu %4llu cycles/MMA (per-warp)  floor %d\n", name, N, h[0], h[1], h[2], h[3], 128 * N / 256);
    cudaMemset(d, 0, 64);
  }
}
int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64 * 8);
  cudaMemset(d, 0, 64);
  runm<0>(d, "ss const");
  runm<1>(d, "ss moving");
  runm<2>(d, "ts (A tmem)");
  runm<3>(d, "ss moving 2 warps");
  runm<5>(d, "ss moving 3 warps");
  runm<4>(d, "ss moving 4 warps");
  runm<6>(d, "ss const lane0");
  return 0;
}
