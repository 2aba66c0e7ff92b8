// Microbenchmarks of the tcgen05 pipeline primitives on B200 (sm_100a):
// mbarrier hand-off latency, tcgen05.commit latency, MMA latency/throughput
// (kind::tf32, A from TMEM), TMEM store throughput.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2509_22857_b200/csrc \
//        -I include tools/ubench_tc.cu -o build/ubench_tc
#include <cstdio>
#include <cstdint>
#include <cstdlib>

#include "tc_ptx.cuh"

using namespace pcnn;

__device__ __forceinline__ uint64_t clk() { return clock64(); }

__global__ void ubench(uint64_t* out, int iters, int n_mma, int randomize, int getenv_n256) {
  __shared__ __align__(1024) uint8_t bsm[16 * 1024];
  __shared__ uint64_t bar[4];
  __shared__ uint64_t barf;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) ptx::mbar_init(ptx::smem_u32(&bar[i]), 1);
    ptx::mbar_init(ptx::smem_u32(&barf), 1);
    ptx::fence_mbar_init();
  }
  for (int i = threadIdx.x; i < 16 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(bsm)[i] = 0.f;
  if (warp == 0) ptx::tmem_alloc(ptx::smem_u32(&tbase), 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tbase;
  const uint32_t b0 = ptx::smem_u32(&bar[0]), b1 = ptx::smem_u32(&bar[1]), b2 = ptx::smem_u32(&bar[2]);

  // 1. ping-pong between warp 0 lane 0 and warp 1 lane 0
  uint64_t t0 = clk();
  if (lane == 0 && warp < 2) {
    for (int i = 0; i < iters; ++i) {
      if (warp == 0) {
        ptx::mbar_arrive(b0);
        ptx::mbar_wait(b1, i & 1);
      } else {
        ptx::mbar_wait(b0, i & 1);
        ptx::mbar_arrive(b1);
      }
    }
  }
  uint64_t t1 = clk();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
  __syncthreads();

  // 2. commit latency with nothing in flight
  if (threadIdx.x == 0) {
    t0 = clk();
    for (int i = 0; i < iters; ++i) {
      ptx::mma_commit(b2);
      ptx::mbar_wait(b2, i & 1);
    }
    t1 = clk();
    out[1] = (t1 - t0) / iters;
  }
  __syncthreads();

  // 3. MMA latency: n_mma dependent MMAs (same accumulator) + commit + wait
  const uint32_t idesc16 = ptx::idesc_tf32(128, 16), idesc128 = ptx::idesc_tf32(128, 128);
  const uint64_t bd = ptx::smem_desc_sw128(ptx::smem_u32(bsm));
  if (threadIdx.x == 0) {
    for (int cfg = 0; cfg < 2; ++cfg) {
      const uint32_t idesc = cfg ? idesc128 : idesc16;
      t0 = clk();
      for (int i = 0; i < iters; ++i) {
        for (int k = 0; k < n_mma; ++k) ptx::mma_tf32_ts(tmem, tmem + 256 + (k & 7) * 8, bd, idesc, k > 0);
        ptx::mma_commit(b2);
        ptx::mbar_wait(b2, (iters * (1 + cfg) + i) & 1);  // b2 phases continue from step 2
      }
      t1 = clk();
      out[2 + cfg] = (t1 - t0) / iters;
    }
  }
  __syncthreads();

  // 3a. optionally fill A (TMEM cols 256..511) and B (smem) with random data
  if (randomize) {
    if (warp < 4) {
      const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
      uint32_t seed = 0x9E3779B9u * (threadIdx.x + 1);
      for (int c = 256; c < 512; c += 8) {
        uint32_t r[8];
        for (int i = 0; i < 8; ++i) {
          seed = seed * 1664525u + 1013904223u;
          r[i] = __float_as_uint(((seed >> 8) * (1.0f / 16777216.0f)) - 0.5f) & 0xFFFFE000u;
        }
        ptx::tmem_st8(tmem + lane_off + c, r);
      }
      ptx::tmem_st_wait();
    }
    for (int i = threadIdx.x; i < 16 * 1024 / 4; i += blockDim.x) {
      uint32_t x = 0x85EBCA6Bu * (i + 7);
      x ^= x >> 13; x *= 0xC2B2AE35u; x ^= x >> 16;
      reinterpret_cast<float*>(bsm)[i] = __uint_as_float(__float_as_uint(((x >> 8) * (1.0f / 16777216.0f)) - 0.5f) & 0xFFFFE000u);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
  }

  // 3b. MMA throughput vs number of independent accumulators and N (48 MMAs)
  if (threadIdx.x == 0) {
    int slot = 6;
    const int ns[4] = {16, 32, 64, 128};
    uint32_t ph = (iters * 3) & 1;  // b2 completed 3*iters phases so far
    for (int ni = 0; ni < 4; ++ni) {
      const uint32_t idesc = ptx::idesc_tf32(128, ns[ni]);
      for (int R = 1; R <= 8; R *= 2) {
        if (R * ns[ni] > 256) { out[slot++] = 0; continue; }
        t0 = clk();
        for (int i = 0; i < 20; ++i) {
          for (int k = 0; k < 48; ++k)
            ptx::mma_tf32_ts(tmem + (k % R) * ns[ni], tmem + 256 + (k & 7) * 8, bd, idesc, k >= R);
          ptx::mma_commit(b2);
          ptx::mbar_wait(b2, ph);
          ph ^= 1;
        }
        t1 = clk();
        out[slot++] = (t1 - t0) / 20 / 48;
      }
    }
    // patterns of the conv kernel: alternating N (32/16), varying B descriptor
    {
      const uint32_t i32 = ptx::idesc_tf32(128, 32), i16 = ptx::idesc_tf32(128, 16);
      for (int pat = 0; pat < 3; ++pat) {
        t0 = clk();
        for (int i = 0; i < 20; ++i) {
          for (int k = 0; k < 48; ++k) {
            const uint32_t id = pat == 0 ? ((k & 1) ? i16 : i32) : i32;
            const uint64_t b = pat == 1 ? bd + 2 * ((k >> 1) & 3) : bd;
            const uint32_t d = pat == 2 ? tmem + (k & 1) * 16 : tmem;
            ptx::mma_tf32_ts(d, tmem + 256 + (k & 7) * 8, b, id, k > 1);
          }
          ptx::mma_commit(b2);
          ptx::mbar_wait(b2, ph);
          ph ^= 1;
        }
        t1 = clk();
        out[26 + pat] = (t1 - t0) / 20 / 48;
      }
    }
    // the conv kernel's per-K-block pattern: fence, 8 MMAs (concat), commit
    {

      const uint32_t i32 = ptx::idesc_tf32(128, 32), i16 = ptx::idesc_tf32(128, 16);
      for (int var = 0; var < 6; ++var) {
        const uint32_t acol = var == 3 ? 64 : (var == 4 ? 96 : (var == 5 ? 128 : 256));
        t0 = clk();
        for (int i = 0; i < 24; ++i) {
          if (var != 1) ptx::tc_fence_after();
          for (int k4 = 0; k4 < 4; ++k4) {
            ptx::mma_tf32_ts(tmem, tmem + acol + k4 * 8, bd + 2 * k4, i32, i > 0 || k4 > 0);
            ptx::mma_tf32_ts(tmem + 16, tmem + acol + 32 + k4 * 8, bd + 2 * k4, i16, 1);
          }
          if (var != 2) ptx::mma_commit(ptx::smem_u32(&bar[3]));
        }
        ptx::mma_commit(b2);
        ptx::mbar_wait(b2, ph);
        ph ^= 1;
        t1 = clk();
        out[40 + var] = (t1 - t0) / 24;
      }
    }
    // the kernel's asm K-block (warp-collective, elect.sync inside)
    {
      const uint32_t i32 = ptx::idesc_tf32(128, 32), i16 = ptx::idesc_tf32(128, 16);
      out[46] = 0;
    }
    // SS mode (A from smem, same zero image), N=16 and 128, R=1 and 4
    for (int ni = 0; ni < 2; ++ni) {
      const uint32_t idesc = ptx::idesc_tf32(128, ni ? 128 : 16);
      for (int R = 1; R <= 4; R *= 4) {
        t0 = clk();
        for (int i = 0; i < 20; ++i) {
          for (int k = 0; k < 48; ++k)
            ptx::mma_tf32_ss(tmem + (k % R) * (ni ? 64 : 16), bd, bd, idesc, k >= R);
          ptx::mma_commit(b2);
          ptx::mbar_wait(b2, ph);
          ph ^= 1;
        }
        t1 = clk();
        out[slot++] = (t1 - t0) / 20 / 48;
      }
    }
  }
  __syncthreads();

  // 3d. the conv kernel's K-block asm issued by a whole warp (elect.sync)
  if (warp == 0) {
    const uint32_t i32 = ptx::idesc_tf32(128, 32), i16 = ptx::idesc_tf32(128, 16);
    uint32_t ph3 = 0;
    for (int var = 0; var < 2; ++var) {
      const uint64_t t0w = clk();
      for (int i = 0; i < 24; ++i) {
        if (var) ptx::tc_fence_after();
        ptx::mma_kblock_concat(tmem, tmem, tmem, tmem, 16, tmem + 256 + (i & 3) * 64, tmem + 288 + (i & 3) * 64,
                               bd, i32, i16, i ? 0xF : 0xE);
        if (var) ptx::mma_commit_warp(ptx::smem_u32(&bar[3]));
      }
      ptx::mma_commit_warp(ptx::smem_u32(&bar[1]));
      ptx::mbar_wait(ptx::smem_u32(&bar[1]), ph3);
      ph3 ^= 1;
      const uint64_t t1w = clk();
      if (lane == 0) out[47 + var] = (t1w - t0w) / 24;
    }
  }
  __syncthreads();

  // 3e. kind::f16 (fp16 in, fp32 accumulate), K=16 per MMA, A from TMEM
  if (threadIdx.x == 0) {
    uint32_t ph4 = 0;
    const int ns[3] = {32, 128, getenv_n256};
    for (int ni = 0; ni < 3; ++ni) {
      if (ns[ni] == 0) { out[52 + ni] = 0; continue; }
      // f16 idesc: c_format F32 (1<<4), a/b format F16 (0), K-major
      const uint32_t idesc = (1u << 4) | ((uint32_t)(ns[ni] >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      const uint64_t t0f = clk();
      for (int i = 0; i < 20; ++i) {
        for (int k = 0; k < 48; ++k) {
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                       :: "r"(tmem), "r"(tmem + 256 + (k & 7) * 8), "l"(bd), "r"(idesc), "r"((uint32_t)(k > 0)) : "memory");
        }
        ptx::mma_commit(ptx::smem_u32(&barf));
        ptx::mbar_wait(ptx::smem_u32(&barf), ph4);
        ph4 ^= 1;
      }
      const uint64_t t1f = clk();
      out[52 + ni] = (t1f - t0f) / 20 / 48;
    }
  }
  __syncthreads();

  // 3c. N=256 and MMA throughput under concurrent TMEM store/load traffic
  {
    __shared__ volatile int stop;
    if (threadIdx.x == 0) stop = 0;
    __syncthreads();
    uint32_t ph2 = 0;
    for (int mode = 1; mode < 5; ++mode) {   // 1: +STTM, 2: +LDTM, 3: +converter-like mix, 4: alone (real B data)
      if (threadIdx.x == 0) stop = 0;
      __syncthreads();
      if (threadIdx.x == 0) {
        const uint32_t idesc = ptx::idesc_tf32(128, mode == 0 ? 256 : 64);
        if (mode == 4) for (int i = 0; i < 16 * 1024 / 4; ++i) reinterpret_cast<float*>(bsm)[i] = 0.37f * (i % 13);
        t0 = clk();
        for (int i = 0; i < 20; ++i) {
          for (int k = 0; k < 48; ++k) ptx::mma_tf32_ts(tmem, tmem + 256 + (k & 7) * 8, bd, idesc, k > 0);
          ptx::mma_commit(b1);
          ptx::mbar_wait(b1, ph2);
          ph2 ^= 1;
        }
        t1 = clk();
        out[30 + mode] = (t1 - t0) / 20 / 48;
        stop = 1;
      } else if (warp >= 4 && mode > 0) {
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        uint32_t r[8] = {1, 2, 3, 4, 5, 6, 7, 8};
        float v[16];
        while (!stop) {
          if (mode == 1) {
            for (int g = 0; g < 8; ++g) ptx::tmem_st8(tmem + lane_off + 320 + g * 8, r);
            ptx::tmem_st_wait();
          } else if (mode == 3) {
            float4 f[8];
            const uint32_t sb = ptx::smem_u32(bsm) + (threadIdx.x & 31) * 64;
#pragma unroll
            for (int q = 0; q < 8; ++q)
              asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(f[q].x), "=f"(f[q].y), "=f"(f[q].z), "=f"(f[q].w) : "r"(sb + q * 16));
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              uint32_t hi[8], lo[8];
              const float v[8] = {f[2*g].x, f[2*g].y, f[2*g].z, f[2*g].w, f[2*g+1].x, f[2*g+1].y, f[2*g+1].z, f[2*g+1].w};
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                hi[i] = (__float_as_uint(v[i]) + 0x1000u) & 0xFFFFE000u;
                lo[i] = (__float_as_uint(v[i] - __uint_as_float(hi[i])) + 0x1000u) & 0xFFFFE000u;
              }
              ptx::tmem_st8(tmem + lane_off + 320 + g * 8, hi);
              ptx::tmem_st8(tmem + lane_off + 352 + g * 8, lo);
            }
            ptx::tmem_st_wait();
          } else if (mode == 4) {
            break;
          } else {
            ptx::tmem_ld16(tmem + lane_off + 384, v);
            r[0] += __float_as_uint(v[3]);
          }
        }
        if (r[0] == 12345) out[50] = 1;
      }
      __syncthreads();
    }
  }

  // 4. TMEM store throughput: warps 0-3, 16 x STTM.x8 + wait::st per iteration
  if (warp < 4) {
    uint32_t r[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    t0 = clk();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        ptx::tmem_st8(tmem + lane_off + 256 + g * 8, r);
        ptx::tmem_st8(tmem + lane_off + 320 + g * 8, r);
      }
      ptx::tmem_st_wait();
    }
    t1 = clk();
    if (threadIdx.x == 0) out[4] = (t1 - t0) / iters;
  }
  __syncthreads();
  // 5. TMEM load: 4 warps, ld16 x 8 (128 columns)
  if (warp < 4) {
    float v[16];
    float acc = 0.f;
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    t0 = clk();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        ptx::tmem_ld16(tmem + lane_off + g * 16, v);
        acc += v[0];
      }
    }
    t1 = clk();
    if (threadIdx.x == 0) out[5] = (t1 - t0) / iters + (acc == 12345.f);
  }
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

int main() {
  uint64_t* d;
  cudaMalloc(&d, 64 * sizeof(uint64_t));
  cudaMemset(d, 0, 64 * sizeof(uint64_t));
  for (int n_mma : {1, 12, 48}) {
    ubench<<<getenv("UB_BLOCKS") ? atoi(getenv("UB_BLOCKS")) : 1, 384>>>(d, 200, n_mma, getenv("UB_RANDOM") ? 1 : 0, getenv("UB_N256") ? 256 : 0);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("error %s\n", cudaGetErrorString(e));
      return 1;
    }
    uint64_t h[64];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    if (n_mma == 1) {
      const int ns[4] = {16, 32, 64, 128};
      for (int ni = 0; ni < 4; ++ni)
        printf("TS N=%3d cycles/MMA with R=1,2,4,8 accumulators: %llu %llu %llu %llu\n", ns[ni],
               (unsigned long long)h[6 + ni * 4], (unsigned long long)h[7 + ni * 4],
               (unsigned long long)h[8 + ni * 4], (unsigned long long)h[9 + ni * 4]);
      printf("TS N=64 with STTM traffic: %llu; with LDTM traffic: %llu; with converter mix: %llu; real B data: %llu\n",
             (unsigned long long)h[31], (unsigned long long)h[32], (unsigned long long)h[33], (unsigned long long)h[34]);
      printf("alternating N 32/16: %llu; varying B desc: %llu; D alternating (overlapping cols): %llu\n",
             (unsigned long long)h[26], (unsigned long long)h[27], (unsigned long long)h[28]);
      printf("kind::f16 K=16 TS cycles/MMA N=32,64,128: %llu %llu %llu\n", (unsigned long long)h[52],
             (unsigned long long)h[53], (unsigned long long)h[54]);
      printf("asm K-block by a whole warp (8 MMAs): plain %llu, with fence+commit %llu\n",
             (unsigned long long)h[47], (unsigned long long)h[48]);
      printf("kernel pattern per K-block (8 MMAs): fence+commit %llu, commit only %llu, fence only %llu; A at col 64: %llu, 96: %llu, 128: %llu\n",
             (unsigned long long)h[40], (unsigned long long)h[41], (unsigned long long)h[42],
             (unsigned long long)h[43], (unsigned long long)h[44], (unsigned long long)h[45]);
      printf("SS N=16 R=1,4: %llu %llu   SS N=128 R=1,4: %llu %llu\n", (unsigned long long)h[22],
             (unsigned long long)h[23], (unsigned long long)h[24], (unsigned long long)h[25]);
    }
    printf("n_mma=%d: pingpong=%llu commit_empty=%llu mma_chain_N16=%llu mma_chain_N128=%llu "
           "sttm(32KB)+wait=%llu ldtm(4w x 128col)=%llu cycles\n",
           n_mma, (unsigned long long)h[0], (unsigned long long)h[1], (unsigned long long)h[2],
           (unsigned long long)h[3], (unsigned long long)h[4], (unsigned long long)h[5]);
  }
  return 0;
}
