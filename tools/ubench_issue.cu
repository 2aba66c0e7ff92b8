// Issue-rate microbenchmark: cycles per kind::f16 SS MMA (M=128, N=32 and 16)
// when the A descriptor moves per tap (3x3 taps over a pitch-33 grid), for
// several ways of forming the descriptors:
//   0 constant descriptors (hardware rate)
//   1 64-bit add of a per-tap offset to a base descriptor (as conv_ss.cu)
//   2 32-bit add on the low word + mov.b64 {lo, hi} inside the asm
//   3 nine descriptors precomputed before the timed loop (no arithmetic)
//   4 conv_ss concat pattern: N=2n into one accumulator, N=n into another
//   5 same N, alternating accumulators;  6 alternating N, same accumulator
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Ipaper_2509_22857_b200/csrc -Iinclude tools/ubench_issue.cu -o tools/ubench_issue.bin
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>

#include "tc_ptx.cuh"

using namespace pcnn;

__device__ __forceinline__ uint32_t elect1() {
  uint32_t e;
  asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 r;\n\telect.sync r|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(e));
  return e;
}
__device__ __forceinline__ void mma64(uint32_t e, uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, q;\n\tsetp.ne.b32 q, %0, 0;\n\tsetp.ne.b32 p, %5, 0;\n\t"
               "@q tcgen05.mma.cta_group::1.kind::f16 [%1], %2, %3, %4, p;\n\t}"
               ::"r"(e), "r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc)
               : "memory");
}
__device__ __forceinline__ void mma32(uint32_t e, uint32_t d, uint32_t alo, uint32_t ahi, uint32_t blo, uint32_t bhi,
                                      uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, q;\n\t.reg .b64 ad, bd;\n\tsetp.ne.b32 q, %0, 0;\n\tsetp.ne.b32 p, %7, 0;\n\t"
               "mov.b64 ad, {%2, %3};\n\tmov.b64 bd, {%4, %5};\n\t"
               "@q tcgen05.mma.cta_group::1.kind::f16 [%1], ad, bd, %6, p;\n\t}"
               ::"r"(e), "r"(d), "r"(alo), "r"(ahi), "r"(blo), "r"(bhi), "r"(idesc), "r"(acc)
               : "memory");
}

template <int V>
__device__ long long run(uint32_t tmem, uint32_t a0, uint32_t b0, int N, uint32_t bar, uint32_t& phase, int pitch) {
  const uint32_t idesc = ptx::idesc_f16(128, N);
  const uint64_t ad = ptx::smem_desc_noswz(a0, 128 * 16, 128);
  const uint64_t bd = ptx::smem_desc_noswz(b0, 256 * 16, 128);
  uint64_t offs[9];
#pragma unroll
  for (int t = 0; t < 9; ++t) offs[t] = (uint64_t)((t / 3) * pitch + (t % 3));
  uint64_t pre[9];
#pragma unroll
  for (int t = 0; t < 9; ++t) pre[t] = ad + offs[t];
  const uint32_t e = elect1();
  __syncwarp();
  const long long t0 = clock64();
  for (int r = 0; r < 7; ++r) {
    if (V == 0) {
#pragma unroll
      for (int t = 0; t < 9; ++t) mma64(e, tmem, ad, bd, idesc, 1u);
    } else if (V == 1) {
#pragma unroll
      for (int t = 0; t < 9; ++t) mma64(e, tmem, ad + offs[t] + r, bd + t * 4, idesc, 1u);
    } else if (V == 2) {
      const uint32_t alo = (uint32_t)ad + r, ahi = (uint32_t)(ad >> 32);
      const uint32_t blo = (uint32_t)bd, bhi = (uint32_t)(bd >> 32);
#pragma unroll
      for (int t = 0; t < 9; ++t) mma32(e, tmem, alo + (uint32_t)offs[t], ahi, blo + t * 4, bhi, idesc, 1u);
    } else if (V == 3) {
#pragma unroll
      for (int t = 0; t < 9; ++t) mma64(e, tmem, pre[t], bd, idesc, 1u);
    } else if (V == 4) {  // conv_ss concat pattern: N=2n into D0, N=n into D1
      const uint32_t id2 = ptx::idesc_f16(128, 2 * N);
#pragma unroll
      for (int t = 0; t < 9; ++t) {
        mma64(e, tmem, pre[t], bd, id2, 1u);
        mma64(e, tmem + 256, pre[t] + 1024, bd, idesc, 1u);
      }
    } else if (V == 5) {  // same N, alternating D
#pragma unroll
      for (int t = 0; t < 9; ++t) {
        mma64(e, tmem, pre[t], bd, idesc, 1u);
        mma64(e, tmem + 256, pre[t] + 1024, bd, idesc, 1u);
      }
    } else if (V == 6) {  // alternating N, same D
      const uint32_t id2 = ptx::idesc_f16(128, 2 * N);
#pragma unroll
      for (int t = 0; t < 9; ++t) {
        mma64(e, tmem, pre[t], bd, id2, 1u);
        mma64(e, tmem, pre[t] + 1024, bd, idesc, 1u);
      }
    }
  }
  ptx::mma_commit_warp(bar);
  ptx::mbar_wait(bar, phase);
  phase ^= 1;
  return (clock64() - t0) / (V >= 4 ? 126 : 63);
}

__global__ void ubench(unsigned long long* out, int pitch, int fill) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  // fill 0: zeros; 1: pseudo-random fp16 in (-1, 1)
  for (int i = tid; i < 65536 / 2; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u;
    h ^= h >> 13;
    reinterpret_cast<__half*>(smem)[i] = __float2half(fill ? ((h & 0xFFFF) / 32768.f - 1.f) : 0.f);
  }
  if (tid == 0) {
    ptx::mbar_init(ptx::smem_u32(&bar), 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc(ptx::smem_u32(&tbase), 512);
  ptx::fence_proxy_async();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tbase;
  const uint32_t a0 = ptx::smem_u32(smem), b0 = ptx::smem_u32(smem + 32768);
  uint32_t phase = 0;
  if (warp == 1) {
    for (int ni = 0; ni < 2; ++ni) {
      const int N = ni ? 16 : 32;
      long long c[7];
      c[0] = run<0>(tmem, a0, b0, N, ptx::smem_u32(&bar), phase, pitch);
      c[1] = run<1>(tmem, a0, b0, N, ptx::smem_u32(&bar), phase, pitch);
      c[2] = run<2>(tmem, a0, b0, N, ptx::smem_u32(&bar), phase, pitch);
      c[3] = run<3>(tmem, a0, b0, N, ptx::smem_u32(&bar), phase, pitch);
      c[4] = run<4>(tmem, a0, b0, N, ptx::smem_u32(&bar), phase, pitch);
      c[5] = run<5>(tmem, a0, b0, N, ptx::smem_u32(&bar), phase, pitch);
      c[6] = run<6>(tmem, a0, b0, N, ptx::smem_u32(&bar), phase, pitch);
      if ((tid & 31) == 0)
        for (int v = 0; v < 7; ++v) out[ni * 8 + v] = c[v];
    }
  }
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(tmem, 512);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64 * 8);
  cudaMemset(d, 0, 64 * 8);
  cudaFuncSetAttribute(ubench, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  for (int fill = 0; fill < 2; ++fill) {
    for (int rep = 0; rep < 2; ++rep) ubench<<<1, 64, 65536>>>(d, 33, fill);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("error %s\n", cudaGetErrorString(e));
      return 1;
    }
    unsigned long long h[16];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    const char* names[7] = {"const", "add64", "add32+mov.b64", "precomputed", "N=2n,n alt D", "same N alt D",
                            "N=2n,n same D"};
    for (int ni = 0; ni < 2; ++ni)
      for (int v = 0; v < 7; ++v)
        printf("%s n=%d %-14s %llu cycles/MMA\n", fill ? "random" : "zeros", ni ? 16 : 32, names[v], h[ni * 8 + v]);
  }
  return 0;
}
