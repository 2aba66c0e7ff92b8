// tcgen05 (5th-gen tensor core) implicit-GEMM convolution with the fused
// polynomial / residual / pool epilogue, fp32-accurate via 3xTF32.
//
// GEMM view: D[M = output pixels, N = output channels] = A[M, K] * B[N, K]^T,
// K = (channel block, ky, kx, channel) of the channel-blocked input.
//
//   * A (activations) never touches shared memory: converter warps gather
//     each pixel's im2col row, split every fp32 value into tf32 hi + lo
//     (x = hi + lo + O(2^-22 x)) and write both straight into tensor memory
//     with tcgen05.st (A operand "from TMEM", lane = pixel row).
//   * B (weights) is pre-split and pre-swizzled by the pack kernel into the
//     exact 128B-swizzled K-major shared-memory image (tc_layout.cuh); a
//     producer thread bulk-copies it (TMA engine, cp.async.bulk) -- once for
//     the whole kernel when it fits ("resident"), else per K-block through a
//     ring of stages.
//   * One thread issues, per 8-deep K step, three tcgen05.mma kind::tf32:
//     A_hi*B_hi into a main accumulator and A_hi*B_lo + A_lo*B_hi into a
//     separate correction accumulator.  The tensor core truncates when it
//     adds into an fp32 accumulator (measured: a bias of ~0.2 ulp per MMA,
//     growing linearly with K), so the main products are also spread over
//     P partial accumulators and everything is summed with round-to-nearest
//     FADDs in the epilogue -- that keeps deep layers (K = 4608) at
//     fp32-class error.
//   * Epilogue warps tcgen05.ld the accumulators (double-buffered in TMEM
//     when the columns allow, so the next tile's MMAs overlap), apply bias ->
//     affine -> residual -> polynomial -> pool and store; 2x2 pools reduce
//     across the four lanes that hold one window (WINDOW pixel order), the
//     global pool reduces a warp and issues one atomic per channel.
//
// Warp roles (384 threads, persistent, one CTA per SM):
//   warp 0: bulk-copy producer for B;  warp 1: MMA issuer;  warp 2: TMEM
//   allocator;  warps 4-7: A converters;  warps 8-11: epilogue.
#include "kernels.cuh"
#include "tc_layout.cuh"
#include "tc_ptx.cuh"

namespace pcnn {

namespace {

constexpr int kThreads = 384;
constexpr int kMaxAStages = 4;   // A hi/lo stages in TMEM (64 columns each)
constexpr int kBStages = 4;      // streamed B stages in smem
constexpr int kBResidentMax = 160 * 1024;
constexpr int kTileM = 128;
constexpr int kMaxPartials = 4;
constexpr int kAddsPerPartial = 96;  // main-accumulator MMAs per partial before splitting

struct TcParams {
  ConvArgs a;
  int nt;          // N tile (UMMA N), 16..128
  int n_tiles;
  int m_tiles;
  int nkb;         // K-blocks of 32
  int resident;    // B image kept in smem for the whole kernel
  int taps;        // kh * kw
  int nseg;        // nblk_in * taps (valid channel segments)
  int a_stages;    // A stages in TMEM
  int acc_bufs;    // accumulator sets (1 or 2)
  int partials;    // main partial accumulators P
  uint32_t b_stage_bytes;
  uint32_t tmem_cols;
};

struct Smem {
  uint64_t a_full[kMaxAStages], a_empty[kMaxAStages];
  uint64_t b_full[kBStages], b_empty[kBStages];
  uint64_t acc_full[2], acc_empty[2];
  uint32_t tmem_base;
};

__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
  hi = f32_to_tf32(x);
  lo = f32_to_tf32(x - __uint_as_float(hi));
}

// ---- converter: im2col row of one pixel -> tf32 hi/lo in TMEM -------------------
__device__ __forceinline__ void convert_kblock(const TcParams& P, int kb, int b, int iy0, int ix0, bool valid,
                                               uint32_t t_hi, uint32_t t_lo) {
  const ConvArgs& a = P.a;
  const TensorView& in = a.in;
  const int cb = in.cb;
  float4 f[8];
  // issue all eight 16-byte loads of the K-block before using any of them
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int k = kb * kTcBK + q * 4;
    const int seg = k / cb, ci = k - seg * cb;
    const int blk = seg / P.taps, tap = seg - blk * P.taps;
    const int ky = tap / a.kw, kx = tap - ky * a.kw;
    const int iy = iy0 + ky, ix = ix0 + kx;
    const bool ok = valid && seg < P.nseg && iy >= 0 && iy < in.h && ix >= 0 && ix < in.w;
    const float* src = in.base + ((((int64_t)b * in.nblk + blk) * in.h + iy) * in.w + ix) * cb + ci;
    f[q] = ok ? __ldg(reinterpret_cast<const float4*>(src)) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const float v[8] = {f[2 * g].x, f[2 * g].y, f[2 * g].z, f[2 * g].w,
                        f[2 * g + 1].x, f[2 * g + 1].y, f[2 * g + 1].z, f[2 * g + 1].w};
    uint32_t hi[8], lo[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) split_tf32(v[i], hi[i], lo[i]);
    ptx::tmem_st8(t_hi + g * 8, hi);
    ptx::tmem_st8(t_lo + g * 8, lo);
  }
}

__device__ __forceinline__ void store4(const EpiParams& e, int b, int ch, int y, int x, const float* o) {
  *reinterpret_cast<float4*>(e.out.pix(b, ch, y, x)) = make_float4(o[0], o[1], o[2], o[3]);
}

__global__ void __launch_bounds__(kThreads, 1) conv_tc_kernel(const __grid_constant__ TcParams P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const ConvArgs& a = P.a;
  const uint32_t b_region = P.resident ? P.b_stage_bytes * P.nkb : P.b_stage_bytes * kBStages;
  Smem* S = reinterpret_cast<Smem*>(smem + b_region);
  const uint32_t b_base = ptx::smem_u32(smem);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int total_tiles = P.m_tiles * P.n_tiles;
  const int64_t M = a.pm.count(a.batch);
  const int SA = P.a_stages, NB = P.acc_bufs, NP = P.partials;
  const uint32_t acc_set_cols = (uint32_t)(NP + 1) * P.nt;  // P main partials + correction

  if (threadIdx.x == 0) {
    for (int i = 0; i < kMaxAStages; ++i) {
      ptx::mbar_init(ptx::smem_u32(&S->a_full[i]), 4);
      ptx::mbar_init(ptx::smem_u32(&S->a_empty[i]), 1);
    }
    for (int i = 0; i < kBStages; ++i) {
      ptx::mbar_init(ptx::smem_u32(&S->b_full[i]), 1);
      ptx::mbar_init(ptx::smem_u32(&S->b_empty[i]), 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(ptx::smem_u32(&S->acc_full[i]), 1);
      ptx::mbar_init(ptx::smem_u32(&S->acc_empty[i]), 4);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc(ptx::smem_u32(&S->tmem_base), P.tmem_cols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = S->tmem_base;
  const uint32_t a_col0 = (uint32_t)NB * acc_set_cols;

  if (warp == 0) {
    // ===== B producer =====
    if (lane == 0) {
      if (P.resident) {
        const uint32_t bar = ptx::smem_u32(&S->b_full[0]);
        ptx::mbar_arrive_tx(bar, P.b_stage_bytes * P.nkb);
        for (int kb = 0; kb < P.nkb; ++kb)
          ptx::bulk_g2s(b_base + kb * P.b_stage_bytes, a.tcw + (size_t)kb * (P.b_stage_bytes / 4),
                        P.b_stage_bytes, bar);
      } else {
        uint32_t it = 0;
        for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
          const int n_tile = tile / P.m_tiles;
          for (int kb = 0; kb < P.nkb; ++kb, ++it) {
            const int s = it % kBStages;
            ptx::mbar_wait(ptx::smem_u32(&S->b_empty[s]), ((it / kBStages) & 1) ^ 1);
            const uint32_t bar = ptx::smem_u32(&S->b_full[s]);
            ptx::mbar_arrive_tx(bar, P.b_stage_bytes);
            const float* src = a.tcw + ((size_t)n_tile * P.nkb + kb) * (P.b_stage_bytes / 4);
            ptx::bulk_g2s(b_base + s * P.b_stage_bytes, src, P.b_stage_bytes, bar);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer =====
    if (lane == 0) {
      const uint32_t idesc = ptx::idesc_tf32(kTileM, P.nt);
      const uint32_t lo_off = P.nt * 128;  // lo image follows the hi image
      uint32_t it = 0, bit = 0, acc_it = 0;
      if (P.resident) ptx::mbar_wait(ptx::smem_u32(&S->b_full[0]), 0);
      for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x, ++acc_it) {
        const uint32_t acc = NB == 2 ? (acc_it & 1) : 0;
        const uint32_t acc_ph = (NB == 2 ? (acc_it >> 1) : acc_it) & 1;
        ptx::mbar_wait(ptx::smem_u32(&S->acc_empty[acc]), acc_ph ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_set = tmem + acc * acc_set_cols;
        const uint32_t d_corr = d_set + NP * P.nt;
        int step = 0;
        for (int kb = 0; kb < P.nkb; ++kb, ++it) {
          const int s = it % SA;
          ptx::mbar_wait(ptx::smem_u32(&S->a_full[s]), (it / SA) & 1);
          uint32_t bsm;
          int bs = 0;
          if (P.resident) {
            bsm = b_base + kb * P.b_stage_bytes;
          } else {
            bs = bit % kBStages;
            ptx::mbar_wait(ptx::smem_u32(&S->b_full[bs]), (bit / kBStages) & 1);
            bsm = b_base + bs * P.b_stage_bytes;
          }
          ptx::tc_fence_after();
          const uint32_t a_hi = tmem + a_col0 + s * 64, a_lo = a_hi + 32;
#pragma unroll
          for (int k4 = 0; k4 < kTcBK / 8; ++k4, ++step) {
            const uint64_t dh = ptx::smem_desc_sw128(bsm + k4 * 32);
            const uint64_t dl = ptx::smem_desc_sw128(bsm + lo_off + k4 * 32);
            const int part = step % NP;
            ptx::mma_tf32_ts(d_corr, a_lo + k4 * 8, dh, idesc, step != 0);
            ptx::mma_tf32_ts(d_corr, a_hi + k4 * 8, dl, idesc, 1);
            ptx::mma_tf32_ts(d_set + part * P.nt, a_hi + k4 * 8, dh, idesc, step >= NP);
          }
          ptx::mma_commit(ptx::smem_u32(&S->a_empty[s]));
          if (!P.resident) {
            ptx::mma_commit(ptx::smem_u32(&S->b_empty[bs]));
            ++bit;
          }
        }
        ptx::mma_commit(ptx::smem_u32(&S->acc_full[acc]));
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ===== A converters: thread r of the warpgroup owns accumulator row r =====
    const int row = threadIdx.x - 128;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    uint32_t it = 0;
    for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
      const int m_tile = tile % P.m_tiles;
      const int64_t m = (int64_t)m_tile * kTileM + row;
      int b = 0, oy = 0, ox = 0;
      const bool valid = m < M;
      if (valid) a.pm.decode(m, b, oy, ox);
      const int iy0 = oy * a.stride - a.pad, ix0 = ox * a.stride - a.pad;
      for (int kb = 0; kb < P.nkb; ++kb, ++it) {
        const int s = it % SA;
        ptx::mbar_wait(ptx::smem_u32(&S->a_empty[s]), ((it / SA) & 1) ^ 1);
        ptx::tc_fence_after();
        const uint32_t t_hi = tmem + lane_off + a_col0 + s * 64;
        convert_kblock(P, kb, b, iy0, ix0, valid, t_hi, t_hi + 32);
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(ptx::smem_u32(&S->a_full[s]));
      }
    }
  } else if (warp >= 8) {
    // ===== epilogue =====
    const EpiParams& e = a.epi;
    const int row = threadIdx.x - 256;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    uint32_t acc_it = 0;
    for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x, ++acc_it) {
      const int m_tile = tile % P.m_tiles, n_tile = tile / P.m_tiles;
      const uint32_t acc = NB == 2 ? (acc_it & 1) : 0;
      const uint32_t acc_ph = (NB == 2 ? (acc_it >> 1) : acc_it) & 1;
      ptx::mbar_wait(ptx::smem_u32(&S->acc_full[acc]), acc_ph);
      ptx::tc_fence_after();
      const int64_t m = (int64_t)m_tile * kTileM + row;
      int b = -1, oy = 0, ox = 0;
      const bool valid = m < M;
      if (valid) a.pm.decode(m, b, oy, ox);
      const uint32_t d_set = tmem + lane_off + acc * acc_set_cols;
      for (int c0 = 0; c0 < P.nt; c0 += 16) {
        float v[16], t[16];
        ptx::tmem_ld16(d_set + NP * P.nt + c0, v);  // correction terms
        for (int p = 0; p < NP; ++p) {
          ptx::tmem_ld16(d_set + p * P.nt + c0, t);
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] += t[i];
        }
        const int chb = n_tile * P.nt + c0;
#pragma unroll
        for (int grp = 0; grp < 4; ++grp) {
          float o[4];
          const int ch0 = chb + grp * 4;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int ch = ch0 + j;
            o[j] = (valid && ch < e.cout) ? epi_point(e, v[grp * 4 + j], b, oy, ox, ch) : 0.f;
          }
          if (e.pool == PCNN_POOL_NONE) {
            if (valid) store4(e, b, ch0, oy, ox, o);
          } else if (e.pool == PCNN_POOL_GLOBAL) {
            const float div = __ldg(e.pool_p);
            const int b0 = __shfl_sync(0xffffffffu, b, 0);
            const bool uniform = __all_sync(0xffffffffu, valid && b == b0);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              float s = o[j] * div;
              if (uniform) {
#pragma unroll
                for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
                if (lane == 0 && ch0 + j < e.cout) atomicAdd(e.out.base + (int64_t)b0 * e.npad + ch0 + j, s);
              } else if (valid && ch0 + j < e.cout) {
                atomicAdd(e.out.base + (int64_t)b * e.npad + ch0 + j, s);
              }
            }
          } else {
            // WINDOW order: lanes 4q..4q+3 hold the (dy, dx) = 00, 01, 10, 11 window pixels
            float q1[4], q2[4], q3[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              q1[j] = __shfl_down_sync(0xffffffffu, o[j], 1);
              q2[j] = __shfl_down_sync(0xffffffffu, o[j], 2);
              q3[j] = __shfl_down_sync(0xffffffffu, o[j], 3);
            }
            if (valid && (lane & 3) == 0) {
              float p[4];
#pragma unroll
              for (int j = 0; j < 4; ++j)
                p[j] = (ch0 + j < e.cout) ? epi_pool4(e, ch0 + j, o[j], q1[j], q2[j], q3[j]) : 0.f;
              store4(e, b, ch0, oy >> 1, ox >> 1, p);
            }
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(ptx::smem_u32(&S->acc_empty[acc]));
    }
  }
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, P.tmem_cols);
  }
}

bool make_params(const ConvArgs& a, TcParams& P) {
  const int cb = a.in.cb;
  if (!(cb == 4 || cb == 8 || cb == 16 || cb == 32)) return false;
  if (a.npad < 16 || a.npad % 16) return false;
  if (!a.tcw) return false;
  P.a = a;
  P.nt = a.npad <= 128 ? a.npad : 128;
  if (a.npad % P.nt) return false;
  P.n_tiles = a.npad / P.nt;
  const int64_t M = host_pixel_count(a.pm, a.batch);
  P.m_tiles = (int)((M + kTileM - 1) / kTileM);
  P.nkb = tc_kblocks(a.kp);
  P.taps = a.kh * a.kw;
  P.nseg = a.in.nblk * P.taps;
  P.b_stage_bytes = (uint32_t)(2 * P.nt * kTcBK * 4);
  P.resident = (P.n_tiles == 1 && (int64_t)P.b_stage_bytes * P.nkb <= kBResidentMax) ? 1 : 0;
  // TMEM budget (512 columns): acc_bufs x (P + 1) x NT accumulators + a_stages x 64
  const int ksteps = P.nkb * (kTcBK / 8);
  int want = (ksteps + kAddsPerPartial - 1) / kAddsPerPartial;
  want = want < 1 ? 1 : (want > kMaxPartials ? kMaxPartials : want);
  const int cfg[4][2] = {{2, 4}, {2, 2}, {1, 4}, {1, 2}};  // (acc_bufs, a_stages), preferred first
  P.partials = 0;
  for (int want_p = want; want_p >= 1 && !P.partials; --want_p) {
    for (auto& c : cfg) {
      if (c[0] * (want_p + 1) * P.nt + c[1] * 64 <= 512) {
        P.acc_bufs = c[0];
        P.a_stages = c[1];
        P.partials = want_p;
        break;
      }
    }
  }
  if (!P.partials) return false;
  const uint32_t need = P.acc_bufs * (P.partials + 1) * P.nt + P.a_stages * 64;
  P.tmem_cols = need <= 128 ? 128 : (need <= 256 ? 256 : 512);
  return true;
}

size_t smem_bytes(const TcParams& P) {
  size_t b = P.resident ? (size_t)P.b_stage_bytes * P.nkb : (size_t)P.b_stage_bytes * kBStages;
  return 1024 + b + sizeof(Smem);
}

}  // namespace

bool conv_tc_supported(const ConvArgs& a) {
  TcParams P;
  return make_params(a, P);
}

void launch_conv_tc(const ConvArgs& a, cudaStream_t s) {
  TcParams P;
  if (!make_params(a, P)) return;
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  const size_t smem = smem_bytes(P);
  cudaFuncSetAttribute(conv_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int tiles = P.m_tiles * P.n_tiles;
  const int grid = tiles < nsm ? tiles : nsm;
  conv_tc_kernel<<<grid, kThreads, smem, s>>>(P);
}

}  // namespace pcnn
