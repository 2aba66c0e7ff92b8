// Microbenchmark + layout probe for kind::f16 tcgen05.mma with both operands
// in shared memory (K-major, no swizzle), as used by conv_ss.cu.
//   * cycles per MMA for a chain of 64 dependent MMAs, per (M, N)
//   * where an M=64 accumulator lands in tensor memory (lane -> row)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Ipaper_2509_22857_b200/csrc -Iinclude tools/ubench_ss.cu -o /tmp/ubench_ss
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>

#include "tc_ptx.cuh"

using namespace pcnn;

__global__ void ubench_ss(unsigned long long* out, float* probe) {
  extern __shared__ __align__(1024) uint8_t smem[];
  // A: 128 rows x 16 fp16 (2 core-matrix columns); B: 256 rows x 16 fp16
  __half* A = reinterpret_cast<__half*>(smem);            // [kc8 2][128][8]
  __half* B = reinterpret_cast<__half*>(smem + 4096);     // [kc8 2][256][8]
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // A[m][k] = (k == 0) ? m + 1 : 0 ; B[n][k] = (k == 0) ? 1 : 0  -> D[m][n] = m + 1
  for (int i = tid; i < 2 * 128 * 8; i += blockDim.x) {
    const int g = i / (128 * 8), m = (i / 8) % 128, j = i % 8;
    A[i] = __float2half((g == 0 && j == 0) ? (float)(m + 1) : 0.f);
  }
  for (int i = tid; i < 2 * 256 * 8; i += blockDim.x) {
    const int g = i / (256 * 8), j = i % 8;
    B[i] = __float2half((g == 0 && j == 0) ? 1.f : 0.f);
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
  const uint32_t a0 = ptx::smem_u32(A), b0 = ptx::smem_u32(B);
  const int Ms[2] = {128, 64};
  const int Ns[6] = {16, 32, 64, 128, 256, 0};
  uint32_t phase = 0;
  int slot = 0;
  for (int mi = 0; mi < 2; ++mi) {
    for (int ni = 0; Ns[ni]; ++ni) {
      const int M = Ms[mi], N = Ns[ni];
      const uint64_t ad = ptx::smem_desc_noswz(a0, 128 * 16, 128);
      const uint64_t bd = ptx::smem_desc_noswz(b0, 256 * 16, 128);
      const uint32_t idesc = ptx::idesc_f16(M, N);
      __syncthreads();
      long long t0 = 0, t1 = 0;
      if (warp == 1) {
        t0 = clock64();
        for (int i = 0; i < 64; ++i) ptx::mma_f16_ss_warp(tmem, ad, bd, idesc, i > 0);
        ptx::mma_commit_warp(ptx::smem_u32(&bar));
        ptx::mbar_wait(ptx::smem_u32(&bar), phase);
        t1 = clock64();
        if (lane == 0) out[slot] = (unsigned long long)(t1 - t0) / 64;
      }
      phase ^= 1;
      __syncthreads();
      ptx::tc_fence_after();
      if (M == 64 && N == 64 && warp < 4) {
        // D = 64 * (m + 1) after 64 accumulating MMAs; record column 0 of every lane
        float v[16];
        ptx::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16), v);
        probe[warp * 32 + lane] = v[0];
      }
      ++slot;
    }
  }
  // A start shifted by s x 16 B (s = 0..7), M=128 N=32 and N=16; then taps
  // cycling through shifts 0..8 like a 3x3 conv over a pitch-33 grid
  for (int sh = 0; sh < 10; ++sh) {
    for (int nn = 0; nn < 2; ++nn) {
      const int N = nn ? 16 : 32;
      const uint32_t idesc = ptx::idesc_f16(128, N);
      __syncthreads();
      if (warp == 1) {
        const long long t0 = clock64();
        for (int i = 0; i < 64; ++i) {
          int s16 = sh < 8 ? sh : (sh == 8 ? (i % 9) / 3 * 33 + (i % 3) : (i % 9) / 3 * 32 + (i % 3));
          s16 &= 63;  // stay inside the 4 KB A buffer region (the values do not matter)
          const uint64_t ad = ptx::smem_desc_noswz(a0 + s16 * 16, 128 * 16, 128);
          const uint64_t bd = ptx::smem_desc_noswz(b0, 256 * 16, 128);
          ptx::mma_f16_ss_warp(tmem, ad, bd, idesc, i > 0);
        }
        ptx::mma_commit_warp(ptx::smem_u32(&bar));
        ptx::mbar_wait(ptx::smem_u32(&bar), phase);
        const long long t1 = clock64();
        if (lane == 0) out[20 + sh * 2 + nn] = (unsigned long long)(t1 - t0) / 64;
      }
      phase ^= 1;
    }
  }
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(tmem, 512);
}

int main() {
  unsigned long long* d;
  float* p;
  cudaMalloc(&d, 64 * 8);
  cudaMemset(d, 0, 64 * 8);
  cudaMalloc(&p, 128 * 4);
  cudaMemset(p, 0, 128 * 4);
  cudaFuncSetAttribute(ubench_ss, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  ubench_ss<<<1, 128 + 32, 16384>>>(d, p);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return 1;
  }
  unsigned long long h[64];
  float hp[128];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaMemcpy(hp, p, sizeof(hp), cudaMemcpyDeviceToHost);
  const int Ns[5] = {16, 32, 64, 128, 256};
  for (int mi = 0; mi < 2; ++mi) {
    printf("SS kind::f16 K=16 M=%d cycles/MMA N=16,32,64,128,256:", mi ? 64 : 128);
    for (int ni = 0; ni < 5; ++ni) printf(" %llu", h[mi * 5 + ni]);
    printf("\n");
    (void)Ns;
  }
  printf("A start shifted by s*16 B, cycles/MMA (N=32, N=16):");
  for (int sh = 0; sh < 8; ++sh) printf("  s=%d: %llu %llu", sh, h[20 + 2 * sh], h[21 + 2 * sh]);
  printf("\n3x3 tap shifts, pitch 33: %llu %llu   pitch 32: %llu %llu\n", h[36], h[37], h[38], h[39]);
  printf("M=64 accumulator, column 0 per TMEM lane (value/64 = row+1):\n");
  for (int l = 0; l < 128; ++l) printf("%g%c", hp[l] / 64.f, (l % 32 == 31) ? '\n' : ' ');
  return 0;
}
