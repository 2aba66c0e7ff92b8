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
// Warp roles (512 threads, persistent, one CTA per SM):
//   warps 0-3: epilogue;  warps 4-11: A converters (staged: 4-7 only; direct:
//   two warpgroups taking alternate K-blocks);  warp 12: TMEM allocator;
//   warp 14: TMA / bulk-copy producer;  warp 15: MMA issuer.
#include <cuda.h>

#include <cstdlib>

#include "epi_tc.cuh"
#include "kernels.cuh"
#include "tc_layout.cuh"
#include "tc_ptx.cuh"

namespace pcnn {

namespace {

constexpr int kThreads = 640;
// warp roles: the warp scheduler favours higher warp ids, so the single MMA
// issuing warp gets the highest id.  Epilogue warpgroups 0-3 / 12-15 (one per
// accumulator buffer) and converter warpgroups 4-7 / 8-11 (alternate A
// stages) each cover TMEM lanes 0-127 (warp w owns lanes 32*(w%4)..+31).
constexpr int kWarpAlloc = 16, kWarpProducer = 18, kWarpMma = 19;
constexpr int kMaxAStages = 4;   // A hi/lo stages in TMEM (64 columns per K-block)
constexpr int kMaxKs = 8;        // K-blocks per A stage
constexpr int kBStages = 4;      // streamed B stages in smem
constexpr int kTileM = 128;
constexpr int kMaxPartials = 4;
constexpr int kAddsPerPartial = 96;  // main-accumulator MMAs per partial before splitting

struct alignas(64) TmaMap {
  uint64_t v[16];  // CUtensorMap (opaque 128 bytes)
};

struct TcParams {
  TmaMap tmap;     // first member: 64-byte aligned in the param space
  ConvArgs a;
  int nt;          // N tile (UMMA N), 16..128
  int n_tiles;
  int m_tiles;
  int nkb;         // K-blocks (32 tf32 or 64 fp16 elements)
  int sub;         // 32-element sub-blocks per K-block (1 tf32, 2 fp16x2)
  int nsub_real;   // sub-blocks holding real K (the rest is K padding)
  const float* tcw;        // weight image for this precision
  const float* wscale;     // fp16x2: 2^-e weight scale (device), else null
  int resident;    // B image kept in smem for the whole kernel
  int taps;        // kh * kw
  int nseg;        // nblk_in * taps (valid channel segments)
  int a_stages;    // A stages in TMEM
  int ks;          // K-blocks per A stage (1..kMaxKs)
  int acc_bufs;    // accumulator sets (1 or 2)
  int partials;    // main partial accumulators P
  uint32_t b_stage_bytes;
  uint32_t tmem_cols;
  EpiTab etab;     // per-channel parameter table staged in smem (epi_tc.cuh)
  int concat;      // N-concatenated hi|lo B operand (NT <= 64): 2 MMAs per K step
  // TMA-staged input (staged = 1): per (tile, channel block) the input rows a
  // tile needs are loaded as <= `pieces` 4-D boxes (one per image), zero
  // padded by the TMA unit, and the converter reads im2col rows from smem.
  int staged;
  int box_w, box_h, pieces, nblk_in;
  int kpc;         // 32-element sub-blocks per channel block
  uint32_t piece_bytes, st_bytes;
  int nbs;         // streamed B stages
  int dbg;         // PCNN_TC_DEBUG bits: 1 no converter loads, 2 no MMA, 4 no epilogue math
};

// PCNN_TC_DEBUG bit 32: CTA 0 records clock64 events here (see pcnn_tc_trace).
// Each role writes its own region with a private counter: plain stores, no
// atomics, so tracing barely perturbs the pipeline.
constexpr int kTraceLen = 1 << 16;
constexpr int kTraceRegion = kTraceLen / 4;
__device__ unsigned long long g_trace[kTraceLen];

struct Tracer {
  uint32_t n = 0;
  __device__ __forceinline__ void operator()(const TcParams& P, int region, uint32_t tag) {
    if ((P.dbg & 32) && blockIdx.x == 0 && n < kTraceRegion)
      g_trace[region * kTraceRegion + n++] = ((unsigned long long)tag << 48) | (clock64() & 0xFFFFFFFFFFFFull);
  }
};

struct Smem {
  uint64_t a_full[kMaxAStages], a_empty[kMaxAStages];
  uint64_t b_full[kBStages], b_empty[kBStages];
  uint64_t acc_full[2], acc_empty[2];
  uint64_t st_full[2], st_empty[2];
  uint32_t tmem_base;
};

// x = hi + lo with hi, lo representable in tf32 (low 13 mantissa bits zero),
// both rounded to nearest (ties away) by an integer add on the bit pattern --
// 5 instructions; cvt.rna.tf32.f32 is emulated on sm_100 and cost ~8x more.
// |x - hi - lo| <= 2^-22 |x| for finite x.
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
  hi = (__float_as_uint(x) + 0x1000u) & 0xFFFFE000u;
  lo = (__float_as_uint(x - __uint_as_float(hi)) + 0x1000u) & 0xFFFFE000u;
}

// ---- converter: im2col row of one pixel -> tf32 hi/lo in TMEM -------------------
// seg[s] (shared): channel segment s of the K axis = cb consecutive channels
// of one (channel block, ky, kx); .x = float offset relative to the pixel's
// (iy0, ix0) origin, .y = ky | kx << 8 (ky = 31 marks K padding).
struct PixelRow {
  const float* base;    // &in[b][0][iy0][ix0][0] (may point outside; only read when valid)
  const __half* hbase;  // the same element in the hi plane of a split tensor
  uint32_t ymask, xmask;
};

__device__ __forceinline__ PixelRow pixel_row(const TcParams& P, int b, int oy, int ox, bool valid) {
  const ConvArgs& a = P.a;
  const TensorView& in = a.in;
  const int iy0 = oy * a.stride - a.pad, ix0 = ox * a.stride - a.pad;
  PixelRow r;
  const int64_t idx = (((int64_t)b * in.nblk * in.h + iy0) * in.w + ix0) * in.cb;
  r.base = in.base + idx;
  r.hbase = in.split ? in.hi() + (1 + ((int64_t)b * in.hp + iy0 + 1) * in.wp + ix0) * 8 : nullptr;
  r.ymask = r.xmask = 0;
  if (valid) {
    for (int k = 0; k < a.kh; ++k) r.ymask |= (uint32_t)(iy0 + k >= 0 && iy0 + k < in.h) << k;
    for (int k = 0; k < a.kw; ++k) r.xmask |= (uint32_t)(ix0 + k >= 0 && ix0 + k < in.w) << k;
  }
  return r;
}

template <int CBS>
__device__ __forceinline__ void load_kblock(const int2* __restrict__ seg, int kb, const PixelRow& px, float4* f) {
  constexpr int CB = 1 << CBS, SEGS = 32 >> CBS, PER = 8 / SEGS;  // float4 per segment
  // eight independent 16-byte loads, all issued before any use
#pragma unroll
  for (int g = 0; g < SEGS; ++g) {
    const int2 e = seg[kb * SEGS + g];
    const bool ok = (px.ymask >> (e.y & 0xFF)) & (px.xmask >> (e.y >> 8)) & 1u;
    const float4* src = reinterpret_cast<const float4*>(px.base + e.x);
#pragma unroll
    for (int q = 0; q < PER; ++q) f[g * PER + q] = ok ? __ldg(src + q) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  (void)CB;
}

__device__ __forceinline__ void store_kblock(const TcParams& P, const float4* f, uint32_t t_hi, uint32_t t_lo) {
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const float v[8] = {f[2 * g].x, f[2 * g].y, f[2 * g].z, f[2 * g].w,
                        f[2 * g + 1].x, f[2 * g + 1].y, f[2 * g + 1].z, f[2 * g + 1].w};
    uint32_t hi[8], lo[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) split_tf32(v[i], hi[i], lo[i]);
    if (P.dbg & 8) continue;
    ptx::tmem_st8(t_hi + g * 8, hi);
    ptx::tmem_st8(t_lo + g * 8, lo);
  }
}

// fp16x2: x = hi + lo with hi, lo fp16 (round to nearest); one 32-bit TMEM
// column holds the K pair (x0 low half, x1 high half).  |x| >= 65520 makes
// hi infinite, which poisons every column of the pixel's accumulator row --
// the epilogue detects that and recomputes the row in fp32.
__device__ __forceinline__ void split_f16x2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(x0, x1);
  const float2 hf = __half22float2(h);
  const __half2 l = __floats2half2_rn(x0 - hf.x, x1 - hf.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}

// one 32-element sub-block -> 16 hi + 16 lo TMEM columns
__device__ __forceinline__ void store_sub16(const TcParams& P, const float4* f, uint32_t t_hi, uint32_t t_lo) {
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    uint32_t hi[8], lo[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float4 a = f[4 * g + i];
      split_f16x2(a.x, a.y, hi[2 * i], lo[2 * i]);
      split_f16x2(a.z, a.w, hi[2 * i + 1], lo[2 * i + 1]);
    }
    if (P.dbg & 8) continue;
    ptx::tmem_st8(t_hi + g * 8, hi);
    ptx::tmem_st8(t_lo + g * 8, lo);
  }
}

// Converter register buffer for one 32-element sub-block: fp32 values to
// split, or (split input) the hi/lo fp16 words ready for tensor memory.
template <int CBS, bool SPL>
struct SubBuf {
  float4 f[8];
  __device__ __forceinline__ void load(const int2* seg, int h, const PixelRow& px, const TensorView&) {
    load_kblock<CBS>(seg, h, px, f);
  }
};
template <int CBS>
struct SubBuf<CBS, true> {
  uint32_t hw[16], lw[16];
  // split layout: a segment's cb channels are cb/8 groups of 16 bytes, one per
  // 8-channel plane (kstride apart); cb = 4 is the first half of a group
  __device__ __forceinline__ void load(const int2* __restrict__ seg, int h, const PixelRow& px, const TensorView& in) {
    constexpr int SEGS = 32 >> CBS, WPS = (1 << CBS) / 2;  // segments, words per segment
    const int64_t plane = in.plane;
#pragma unroll
    for (int g = 0; g < SEGS; ++g) {
      const int2 e = seg[h * SEGS + g];
      const bool ok = (px.ymask >> (e.y & 0xFF)) & (px.xmask >> (e.y >> 8)) & 1u;
      const __half* src = px.hbase + e.x;
      if (WPS >= 4) {
#pragma unroll
        for (int q = 0; q < WPS / 4; ++q) {
          const __half* sq = src + q * in.kstride;
          const uint4 a = ok ? __ldg(reinterpret_cast<const uint4*>(sq)) : make_uint4(0, 0, 0, 0);
          const uint4 b = ok ? __ldg(reinterpret_cast<const uint4*>(sq + plane)) : make_uint4(0, 0, 0, 0);
          uint32_t* H = hw + g * WPS + 4 * q;
          uint32_t* L = lw + g * WPS + 4 * q;
          H[0] = a.x; H[1] = a.y; H[2] = a.z; H[3] = a.w;
          L[0] = b.x; L[1] = b.y; L[2] = b.z; L[3] = b.w;
        }
      } else {
        const uint2 a = ok ? __ldg(reinterpret_cast<const uint2*>(src)) : make_uint2(0, 0);
        const uint2 b = ok ? __ldg(reinterpret_cast<const uint2*>(src + plane)) : make_uint2(0, 0);
        hw[g * 2] = a.x; hw[g * 2 + 1] = a.y;
        lw[g * 2] = b.x; lw[g * 2 + 1] = b.y;
      }
    }
  }
};

// sub-block h of a stage (K-block j = h / SUB of the stage) -> its TMEM columns
template <bool F16, int CBS>
__device__ __forceinline__ void store_buf(const TcParams& P, const SubBuf<CBS, false>& b, uint32_t t_stage, int j,
                                          int hh) {
  if (F16) store_sub16(P, b.f, t_stage + j * 32 + hh * 16, t_stage + 32 * P.ks + j * 32 + hh * 16);
  else store_kblock(P, b.f, t_stage + j * 32, t_stage + 32 * P.ks + j * 32);
}
template <bool F16, int CBS>
__device__ __forceinline__ void store_buf(const TcParams& P, const SubBuf<CBS, true>& b, uint32_t t_stage, int j,
                                          int hh) {
  if (P.dbg & 8) return;
  const uint32_t th = t_stage + j * 32 + hh * 16, tl = t_stage + 32 * P.ks + j * 32 + hh * 16;
  ptx::tmem_st8(th, b.hw);
  ptx::tmem_st8(th + 8, b.hw + 8);
  ptx::tmem_st8(tl, b.lw);
  ptx::tmem_st8(tl + 8, b.lw + 8);
}

template <bool F16>
__device__ __forceinline__ void store_sub(const TcParams& P, const float4* f, uint32_t t_stage, int j, int hh) {
  if (F16) store_sub16(P, f, t_stage + j * 32 + hh * 16, t_stage + 32 * P.ks + j * 32 + hh * 16);
  else store_kblock(P, f, t_stage + j * 32, t_stage + 32 * P.ks + j * 32);
}

template <int CBS, bool F16, bool SPL>
__global__ void __launch_bounds__(kThreads, 1) conv_tc_kernel(const __grid_constant__ TcParams P) {
  static_assert(F16 || !SPL, "split-format input feeds the fp16x2 kernel only");
  constexpr int SUB = F16 ? 2 : 1;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const ConvArgs& a = P.a;
  const uint32_t b_region = P.resident ? P.b_stage_bytes * P.nkb : P.b_stage_bytes * P.nbs;
  const uint32_t st_region = P.staged ? 2 * P.st_bytes : 0;
  uint8_t* st_buf = smem + b_region;
  Smem* S = reinterpret_cast<Smem*>(smem + b_region + st_region);
  int2* seg = reinterpret_cast<int2*>(smem + b_region + st_region + ((sizeof(Smem) + 15) & ~size_t(15)));
  // parameter table: 16-byte aligned (read with ld.shared.v4)
  float* ptab = reinterpret_cast<float*>(
      (reinterpret_cast<uintptr_t>(seg + ((P.nkb * SUB) << (5 - a.in.cbs))) + 15) & ~uintptr_t(15));
  const uint32_t b_base = ptx::smem_u32(smem);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int total_tiles = P.m_tiles * P.n_tiles;
  Tracer tr;
  const int64_t M = a.pm.count(a.batch);
  const int SA = P.a_stages, NB = P.acc_bufs, NP = P.partials, KS = P.ks;
  // accumulator set: concat -> NP blocks [main_p | corr_p] of 2*NT columns;
  // otherwise NP main partials then one correction accumulator
  const uint32_t acc_set_cols = P.concat ? (uint32_t)NP * 2 * P.nt : (uint32_t)(NP + 1) * P.nt;

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
      ptx::mbar_init(ptx::smem_u32(&S->st_full[i]), 1);
      ptx::mbar_init(ptx::smem_u32(&S->st_empty[i]), 8);
    }
    ptx::fence_mbar_init();
  }
  if (warp == kWarpAlloc) ptx::tmem_alloc(ptx::smem_u32(&S->tmem_base), P.tmem_cols);
  {
    const TensorView& in = a.in;
    const int nsegs = (P.nkb * SUB) << (5 - in.cbs);
    for (int s2 = threadIdx.x; s2 < nsegs; s2 += kThreads) {
      int2 e = make_int2(0, 31);
      if (s2 < P.nseg) {
        const int blk = s2 / P.taps, tap = s2 - blk * P.taps;
        const int ky = tap / a.kw, kx = tap - ky * a.kw;
        // staged: float offset inside the staged box; direct: inside the
        // tensor (split: halves from the pixel's first 8-channel group)
        e = P.staged  ? make_int2((ky * P.box_w + kx) * in.cb, ky | (kx << 8))
            : in.split ? make_int2((int)(blk * (in.cb >> 3) * in.kstride + (ky * in.wp + kx) * 8), ky | (kx << 8))
                       : make_int2(((blk * in.h + ky) * in.w + kx) * in.cb, ky | (kx << 8));
      }
      seg[s2] = e;
    }
    epi_fill_tab(a.epi, P.etab, ptab, threadIdx.x, kThreads);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  ptx::griddep_wait();  // activations come from the previous kernel
  ptx::griddep_launch();
  tl_mark(a.tl, 0);
  const uint32_t tmem = S->tmem_base;
  const uint32_t a_col0 = (uint32_t)NB * acc_set_cols;

  if (warp == kWarpProducer) {
    // ===== producer: TMA input staging + B (weights) bulk copies =====
    if (lane == 0) {
      if (P.staged) ptx::prefetch_tmap(&P.tmap);
      if (P.resident) {
        const uint32_t bar = ptx::smem_u32(&S->b_full[0]);
        ptx::mbar_arrive_tx(bar, P.b_stage_bytes * P.nkb);
        for (int kb = 0; kb < P.nkb; ++kb)
          ptx::bulk_g2s(b_base + kb * P.b_stage_bytes, P.tcw + (size_t)kb * (P.b_stage_bytes / 4),
                        P.b_stage_bytes, bar);
      }
      int bs = 0, sb = 0;
      uint32_t bph = 0, sph = 0;
      const uint32_t box_bytes = (uint32_t)P.box_w * P.box_h * a.in.cb * 4;
      for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
        const int n_tile = tile / P.m_tiles, m_tile = tile - n_tile * P.m_tiles;
        int b0 = 0, oy0 = 0, ox0 = 0, b1 = 0, oy1 = 0, ox1 = 0;
        if (P.staged) {
          const int64_t m0 = (int64_t)m_tile * kTileM;
          const int64_t m1 = (m0 + kTileM < M ? m0 + kTileM : M) - 1;
          a.pm.decode(m0, b0, oy0, ox0);
          a.pm.decode(m1, b1, oy1, ox1);
        }
        for (int kb = 0; kb < P.nkb; ++kb) {
          for (int h = kb * SUB; P.staged && h < kb * SUB + SUB; ++h) {
            if (h >= P.nsub_real || h % P.kpc) continue;
            const int blk = h / P.kpc;
            ptx::mbar_wait_sleep(ptx::smem_u32(&S->st_empty[sb]), sph ^ 1);
            const uint32_t bar = ptx::smem_u32(&S->st_full[sb]);
            ptx::mbar_arrive_tx(bar, box_bytes * (uint32_t)(b1 - b0 + 1));
            for (int bi = b0; bi <= b1; ++bi) {
              const int lo = bi == b0 ? oy0 : 0;
              ptx::tma_load_4d(ptx::smem_u32(st_buf + sb * P.st_bytes + (bi - b0) * P.piece_bytes), &P.tmap, 0,
                               -a.pad, lo * a.stride - a.pad, bi * P.nblk_in + blk, bar);
            }
            if (++sb == 2) { sb = 0; sph ^= 1; }
          }
          if (!P.resident) {
            ptx::mbar_wait_sleep(ptx::smem_u32(&S->b_empty[bs]), bph ^ 1);
            const uint32_t bar = ptx::smem_u32(&S->b_full[bs]);
            ptx::mbar_arrive_tx(bar, P.b_stage_bytes);
            const float* src = P.tcw + ((size_t)n_tile * P.nkb + kb) * (P.b_stage_bytes / 4);
            ptx::bulk_g2s(b_base + bs * P.b_stage_bytes, src, P.b_stage_bytes, bar);
            if (++bs == P.nbs) { bs = 0; bph ^= 1; }
          }
        }
      }
    }
  } else if (warp == kWarpMma) {
    // ===== MMA issuer: the whole warp runs the loop with warp-uniform state,
    // one elected lane issues each tcgen05 instruction =====
    {
      const uint32_t idesc = F16 ? ptx::idesc_f16(kTileM, P.nt) : ptx::idesc_tf32(kTileM, P.nt);
      const uint32_t idesc2 = F16 ? ptx::idesc_f16(kTileM, 2 * P.nt) : ptx::idesc_tf32(kTileM, 2 * P.nt);
      const uint32_t lo_enc = (P.nt * 128) >> 4;  // lo image offset in descriptor units
      const uint64_t desc0 = ptx::smem_desc_sw128(b_base);
      const uint32_t a_empty0 = ptx::smem_u32(&S->a_empty[0]), a_full0 = ptx::smem_u32(&S->a_full[0]);
      const uint32_t b_empty0 = ptx::smem_u32(&S->b_empty[0]), b_full0 = ptx::smem_u32(&S->b_full[0]);
      const uint32_t acc_full0 = ptx::smem_u32(&S->acc_full[0]), acc_empty0 = ptx::smem_u32(&S->acc_empty[0]);
      const uint32_t part_cols = P.nt;
      const bool do_mma = !(P.dbg & 2);
      int s = 0, bs = 0;
      uint32_t ph = 0, bph = 0;
      uint32_t acc = 0, acc_ph = 0;
      if (P.resident) ptx::mbar_wait(b_full0, 0);
      for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
        if (!(P.dbg & 256)) ptx::mbar_wait(acc_empty0 + 8 * acc, acc_ph ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_set = tmem + acc * acc_set_cols;
        const uint32_t d_corr = d_set + NP * part_cols;
        uint32_t d_main = d_set;
        const uint32_t d_main_end = d_set + acc_set_cols - (P.concat ? 0 : part_cols);
        uint32_t first_corr = 0;  // accumulate flags
        int main_seen = 0;
        for (int kb0 = 0; kb0 < P.nkb; kb0 += KS) {
          tr(P, 1, 0x400 | kb0);
          if (!(P.dbg & 256)) ptx::mbar_wait(a_full0 + 8 * s, ph);
          tr(P, 1, 0x500 | kb0);
          ptx::tc_fence_after();
          const int kbn = P.nkb - kb0 < KS ? P.nkb - kb0 : KS;
          for (int j = 0; j < kbn; ++j) {
            const int kb = kb0 + j;
            uint64_t dkb;
            if (P.resident) {
              dkb = desc0 + ((kb * P.b_stage_bytes) >> 4);
            } else {
              ptx::mbar_wait(b_full0 + 8 * bs, bph);
              ptx::tc_fence_after();
              dkb = desc0 + ((bs * P.b_stage_bytes) >> 4);
            }
            const uint32_t a_hi = tmem + a_col0 + s * 64 * KS + j * 32, a_lo = a_hi + 32 * KS;
            if (do_mma && P.concat && !(P.dbg & 128)) {
              // the whole K-block in one asm statement (operands go uniform once)
              uint32_t dk[4], accm = 0;
#pragma unroll
              for (int k4 = 0; k4 < 4; ++k4) {
                dk[k4] = d_main;
                accm |= (main_seen >= NP ? 1u : 0u) << k4;
                ++main_seen;
                d_main += 2 * part_cols;
                if (d_main == d_main_end) d_main = d_set;
              }
              ptx::mma_kblock_concat<F16>(dk[0], dk[1], dk[2], dk[3], part_cols, a_hi, a_lo, dkb, idesc2, idesc, accm);
              first_corr = 1;
            } else if (do_mma) {
#pragma unroll
              for (int k4 = 0; k4 < 4; ++k4) {
                const uint64_t dh = dkb + 2 * k4, dl = dh + lo_enc;  // +32 B per K step (8 tf32 / 16 fp16)
                if (P.concat) {
                  // B rows [hi; lo] as one N = 2*NT operand: [main | corr] += A_hi * [B_hi | B_lo],
                  // then corr += A_lo * B_hi -- two MMAs per K step instead of three
                  ptx::mma_ts_warp<F16>(d_main, a_hi + k4 * 8, dh, idesc2, main_seen >= NP);
                  ptx::mma_ts_warp<F16>(d_main + part_cols, a_lo + k4 * 8, dh, idesc, 1);
                  if (P.dbg & 128) tr(P, 3, 0xA00 | k4);
                  d_main += 2 * part_cols;
                } else {
                  ptx::mma_ts_warp<F16>(d_corr, a_lo + k4 * 8, dh, idesc, first_corr);
                  ptx::mma_ts_warp<F16>(d_corr, a_hi + k4 * 8, dl, idesc, 1);
                  ptx::mma_ts_warp<F16>(d_main, a_hi + k4 * 8, dh, idesc, main_seen >= NP);
                  if (P.dbg & 128) tr(P, 3, 0xA00 | k4);
                  d_main += part_cols;
                }
                first_corr = 1;
                ++main_seen;
                if (d_main == d_main_end) d_main = d_set;
              }
            }
            if (!P.resident) {
              ptx::mma_commit_warp(b_empty0 + 8 * bs);
              if (++bs == P.nbs) { bs = 0; bph ^= 1; }
            }
          }
          ptx::mma_commit_warp(a_empty0 + 8 * s);
          tr(P, 1, 0x600 | kb0);
          if (++s == SA) { s = 0; ph ^= 1; }
        }
        ptx::mma_commit_warp(acc_full0 + 8 * acc);
        if (NB == 2) { acc ^= 1; if (acc == 0) acc_ph ^= 1; } else { acc_ph ^= 1; }
      }
    }
  } else if (P.staged && warp >= 4 && warp < 12) {
    // ===== A converters, staged: two warpgroups take alternate A stages and
    // read each pixel's im2col row from the TMA-staged input box in shared
    // memory (swizzled like the TMA wrote it: conflict-free 16-byte reads).
    // Every converter warp waits st_full and arrives st_empty once per
    // channel block, whether or not it converted any of its K-blocks. =====
    constexpr int CB = 1 << CBS, SEGS = 32 >> CBS, PER = 8 / SEGS;
    constexpr uint32_t SWZ = CBS >= 3 ? (1u << (CBS - 2)) - 1 : 0;  // XOR mask of 16B chunks
    const int cw = (warp - 4) >> 2;
    const int row = (threadIdx.x - 128) & 127;
    int gstage = 0;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t st0 = ptx::smem_u32(st_buf);
    int s = 0, sb = 0;
    uint32_t par = 1, sph = 0;
    for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
      const int m_tile = tile % P.m_tiles;
      const int64_t m0 = (int64_t)m_tile * kTileM, m = m0 + row;
      int b0 = 0, oy0 = 0, ox0 = 0, b = 0, oy = 0, ox = 0;
      a.pm.decode(m0, b0, oy0, ox0);
      const bool valid = m < M && !(P.dbg & 1);
      if (valid) a.pm.decode(m, b, oy, ox);
      // logical byte offset of this pixel's tap-(0,0) element inside a staging buffer
      const uint32_t pix0 = (uint32_t)(b - b0) * P.piece_bytes +
                            (uint32_t)((((oy - (b == b0 ? oy0 : 0)) * a.stride) * P.box_w + ox * a.stride) * CB * 4);
      for (int kb0 = 0; kb0 < P.nkb; kb0 += KS, ++gstage) {
        const int kbn = P.nkb - kb0 < KS ? P.nkb - kb0 : KS;
        const bool mine = (gstage & 1) == cw;
        if (!mine) {
          // not this warpgroup's stage: only keep the staging-buffer protocol
          for (int h = kb0 * SUB; h < (kb0 + kbn) * SUB && h < P.nsub_real; ++h) {
            if (h % P.kpc == 0) ptx::mbar_wait_warp(ptx::smem_u32(&S->st_full[sb]), sph);
            if (h % P.kpc == P.kpc - 1 || h == P.nsub_real - 1) {
              __syncwarp();
              if (lane == 0) ptx::mbar_arrive(ptx::smem_u32(&S->st_empty[sb]));
              if (++sb == 2) { sb = 0; sph ^= 1; }
            }
          }
          if (++s == SA) { s = 0; par ^= 1; }
          continue;
        }
        if (lane == 0 && warp == 4) tr(P, 0, 0x200 | kb0);
        ptx::mbar_wait_warp(ptx::smem_u32(&S->a_empty[s]), par);
        if (lane == 0 && warp == 4) tr(P, 0, 0xB00 | kb0);
        ptx::tc_fence_after();
        const uint32_t t_stage = tmem + lane_off + a_col0 + s * 64 * KS;
        for (int hs = 0; hs < kbn * SUB; ++hs) {
          const int j = hs / SUB, hh = hs - j * SUB;
          const int h = kb0 * SUB + hs;
          const bool real = h < P.nsub_real;
          if (real && h % P.kpc == 0) {
            ptx::mbar_wait_warp(ptx::smem_u32(&S->st_full[sb]), sph);
            if (lane == 0 && warp == 4) tr(P, 0, 0xC00 | h);
          }
          float4 f[8];
          const uint32_t buf = st0 + sb * P.st_bytes;
#pragma unroll
          for (int g = 0; g < SEGS; ++g) {
            const int2 e = seg[h * SEGS + g];
            const bool ok = valid && real && (e.y & 0xFF) != 31;
            const uint32_t L0 = pix0 + (uint32_t)e.x * 4;
#pragma unroll
            for (int q = 0; q < PER; ++q) {
              const uint32_t L = L0 + q * 16;
              const uint32_t phys = L ^ (((L >> 7) & SWZ) << 4);
              float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
              if (ok) asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                                   : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(buf + phys));
              f[g * PER + q] = v;
            }
          }
          if (real && (h % P.kpc == P.kpc - 1 || h == P.nsub_real - 1)) {
            // last sub-block of this channel block: release the staging buffer
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(ptx::smem_u32(&S->st_empty[sb]));
            if (++sb == 2) { sb = 0; sph ^= 1; }
          }
          if (!(P.dbg & 512)) store_sub<F16>(P, f, t_stage, j, hh);
        }
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(ptx::smem_u32(&S->a_full[s]));
        if (lane == 0 && warp == 4) tr(P, 0, 0x300 | kb0);
        if (++s == SA) { s = 0; par ^= 1; }
      }
    }
    (void)CB;
  } else if (!P.staged && warp >= 4 && warp < 12) {
    // ===== A converters, direct loads: two warpgroups take alternate A stages
    // (KS K-blocks each); thread r of a warpgroup owns accumulator row r.  All
    // loads of a stage are issued before the stage's wait.  Bookkeeping is
    // incremental -- no divisions in the loop. =====
    const int cw = (warp - 4) >> 2;
    const int row = (threadIdx.x - 128) & 127;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const int nkb = P.nkb;
    const int spt = (nkb + KS - 1) / KS;  // stages per tile
    auto px_for = [&](int tile) {
      const int64_t m = (int64_t)(tile % P.m_tiles) * kTileM + row;
      int b = 0, oy = 0, ox = 0;
      const bool valid = m < M && !(P.dbg & 1);
      if (valid) a.pm.decode(m, b, oy, ox);
      return pixel_row(P, b, oy, ox, valid);
    };
    int tile = blockIdx.x, r = cw;  // r: stage index within the tile
    while (r >= spt) { r -= spt; tile += gridDim.x; }
    int s = cw, par = 1;  // A stage and the parity to wait for on a_empty
    while (s >= SA) { s -= SA; par ^= 1; }
    int px_tile = -1;
    PixelRow px;
    while (tile < total_tiles) {
      if (px_tile != tile) {
        px = px_for(tile);
        px_tile = tile;
      }
      const int kb0 = r * KS;
      const int kbn = nkb - kb0 < KS ? nkb - kb0 : KS;
      const int nsb = kbn * SUB;  // 32-element sub-blocks of this stage
      const int h0 = kb0 * SUB;
      // two register buffers: the next sub-block's loads are in flight while
      // the current one is split and stored
      SubBuf<CBS, SPL> fa, fb;
      fa.load(seg, h0, px, a.in);
      if (nsb > 1) fb.load(seg, h0 + 1, px, a.in);
      if (lane == 0 && warp == 4) tr(P, 0, 0x200 | kb0);
      ptx::mbar_wait_warp(ptx::smem_u32(&S->a_empty[s]), par);
      ptx::tc_fence_after();
      const uint32_t t_stage = tmem + lane_off + a_col0 + s * 64 * KS;
      for (int i = 0; i < nsb; i += 2) {
        store_buf<F16>(P, fa, t_stage, i / SUB, i % SUB);
        if (i + 2 < nsb) fa.load(seg, h0 + i + 2, px, a.in);
        if (i + 1 < nsb) {
          store_buf<F16>(P, fb, t_stage, (i + 1) / SUB, (i + 1) % SUB);
          if (i + 3 < nsb) fb.load(seg, h0 + i + 3, px, a.in);
        }
      }
      if (!(P.dbg & 16)) ptx::tmem_st_wait();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(ptx::smem_u32(&S->a_full[s]));
      if (lane == 0 && warp == 4) tr(P, 0, 0x300 | kb0);
      r += 2;
      while (r >= spt) { r -= spt; tile += gridDim.x; }
      s += 2;
      while (s >= SA) { s -= SA; par ^= 1; }
    }
  } else if (warp < 4 || (warp >= 12 && warp < 16)) {
    // ===== epilogue: warpgroup ew drains accumulator buffer ew (with one
    // buffer, warpgroup 0 takes every tile) =====
    const int ew = warp < 4 ? 0 : 1;
    const EpiParams& e = a.epi;
    const int row = threadIdx.x & 127;
    // fp16 weight scale, and the input's storage scale when it is split
    const float wsc = (F16 ? __ldg(P.wscale) : 1.f) * (a.in.split ? a.in.sload : 1.f);
    EpiTab etab = P.etab;
    etab.ptab = ptab;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    uint32_t acc_it = 0;
    for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x, ++acc_it) {
      const int m_tile = tile % P.m_tiles, n_tile = tile / P.m_tiles;
      const uint32_t acc = NB == 2 ? (acc_it & 1) : 0;
      const uint32_t acc_ph = (NB == 2 ? (acc_it >> 1) : acc_it) & 1;
      if ((int)acc != ew || (NB == 1 && ew == 1)) continue;
      if (lane == 0 && warp == 0) tr(P, 2, 0x700);
      ptx::mbar_wait_warp(ptx::smem_u32(&S->acc_full[acc]), acc_ph);
      if (lane == 0 && warp == 0) tr(P, 2, 0x800);
      ptx::tc_fence_after();
      const int64_t m = (int64_t)m_tile * kTileM + row;
      int b = -1, oy = 0, ox = 0;
      const bool valid = m < M;
      if (valid) a.pm.decode(m, b, oy, ox);
      const uint32_t d_set = tmem + lane_off + acc * acc_set_cols;
      for (int c0 = 0; c0 < ((P.dbg & 4) ? 0 : P.nt); c0 += 16) {
        float v[16], t[16];
        if (P.concat) {
          // [main_p | corr_p] blocks: corr_0 + main_0 + sum_p (corr_p + main_p)
          ptx::tmem_ld16x2(d_set + P.nt + c0, d_set + c0, v, t);
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] += t[i];
          for (int p = 1; p < NP; ++p) {
            float u[16];
            ptx::tmem_ld16x2(d_set + 2 * p * P.nt + P.nt + c0, d_set + 2 * p * P.nt + c0, u, t);
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] += u[i] + t[i];
          }
        } else {
          ptx::tmem_ld16(d_set + NP * P.nt + c0, v);  // correction terms
          for (int p = 0; p < NP; ++p) {
            ptx::tmem_ld16(d_set + p * P.nt + c0, t);
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] += t[i];
          }
        }
        const int chb = n_tile * P.nt + c0;
        if (lane == 0 && warp == 0) tr(P, 2, 0xD00 | c0);
        if (F16) {
          if (valid && !isfinite(v[0]) && !SPL) {
            // an input of this pixel overflowed fp16 (or is inf/nan): redo the
            // row's 16 dot products in fp32 with the unscaled fp32 weights
            // (split inputs cannot overflow here: their producer flagged it)
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = 0.f;
            const TensorView& in = a.in;
            int k = 0;
            for (int blk = 0; blk < in.nblk; ++blk)
              for (int ky = 0; ky < a.kh; ++ky)
                for (int kx = 0; kx < a.kw; ++kx, k += in.cb) {
                  const int iy = oy * a.stride - a.pad + ky, ix = ox * a.stride - a.pad + kx;
                  if (iy < 0 || iy >= in.h || ix < 0 || ix >= in.w) continue;
                  const float* xp = in.at(b, blk << in.cbs, iy, ix);
                  for (int c = 0; c < in.cb; ++c) {
                    const float xv = xp[c];
#pragma unroll
                    for (int j = 0; j < 16; ++j) v[j] = fmaf(xv, __ldg(a.w + (int64_t)(chb + j) * a.kp + k + c), v[j]);
                  }
                }
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] *= wsc;
          }
        }
        float sk[16];
        epi_load_skip(e, chb, valid, b, oy, ox, sk);
        epi_chunk16(e, etab, v, 1.f, sk, chb, valid, b, oy, ox, lane);
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(ptx::smem_u32(&S->acc_empty[acc]));
      if (lane == 0 && warp == 0) tr(P, 2, 0x900);
    }
  }
  __syncthreads();
  tl_mark(a.tl, 1);
  if (warp == kWarpAlloc) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, P.tmem_cols);
  }
}

size_t smem_aux_bytes(const TcParams& P);
void staging_geometry(const ConvArgs& a, TcParams& P);

bool make_params(const ConvArgs& a, TcParams& P) {
  const int cb = a.in.cb;
  if (!(cb == 4 || cb == 8 || cb == 16 || cb == 32)) return false;
  if (a.npad < 16 || a.npad % 16) return false;
  P.tcw = a.f16 ? a.tcw16 : a.tcw;
  P.wscale = a.f16 ? a.tc16_scale + 1 : nullptr;
  if (!P.tcw || (a.f16 && !a.tc16_scale)) return false;
  if (a.kh > 31 || a.kw > 31 || host_pixel_count(a.pm, a.batch) >= (1ll << 31)) return false;
  P.a = a;
  P.nt = a.npad <= 128 ? a.npad : 128;
  if (a.npad % P.nt) return false;
  P.n_tiles = a.npad / P.nt;
  const int64_t M = host_pixel_count(a.pm, a.batch);
  P.m_tiles = (int)((M + kTileM - 1) / kTileM);
  P.sub = a.f16 ? 2 : 1;
  P.nkb = a.f16 ? tc16_kblocks(a.kp) : tc_kblocks(a.kp);
  P.nsub_real = (a.kp + 31) / 32;
  P.taps = a.kh * a.kw;
  P.nseg = a.in.nblk * P.taps;
  P.b_stage_bytes = (uint32_t)(2 * P.nt * kTcBK * 4);
  P.etab = epi_tab_layout(a.epi);
  const size_t aux = smem_aux_bytes(P);
  const size_t budget = 225 * 1024;
  // staged input if a tile needs few boxes and everything fits
  P.staged = 0;
  staging_geometry(a, P);
  const bool stage_ok = a.opt.tc_stage && !a.in.split && P.pieces <= 4 && P.box_w <= 256 &&
                        P.box_h <= 256 &&
                        (a.in.nblk == 1 || a.in.cb == 32);
  P.nbs = kBStages;
  if (stage_ok) {
    for (int nbs = kBStages; nbs >= 2 && !P.staged; --nbs)
      if (1024 + (size_t)P.b_stage_bytes * nbs + 2 * (size_t)P.st_bytes + aux <= budget) {
        P.staged = 1;
        P.nbs = nbs;
      }
  }
  const size_t st = P.staged ? 2 * (size_t)P.st_bytes : 0;
  if (1024 + (size_t)P.b_stage_bytes * P.nbs + st + aux > budget) return false;
  P.resident = (P.n_tiles == 1 && 1024 + (size_t)P.b_stage_bytes * P.nkb + st + aux <= budget) ? 1 : 0;
  // TMEM budget (512 columns): acc_bufs x (P + 1) x NT accumulators + a_stages x 64
  P.dbg = a.opt.dbg;
  const int ksteps = P.nkb * (kTcBK / 8);
  int want = (ksteps + kAddsPerPartial - 1) / kAddsPerPartial;
  want = want < 1 ? 1 : (want > kMaxPartials ? kMaxPartials : want);
  const int cfg[4][2] = {{2, 4}, {2, 2}, {1, 4}, {1, 2}};  // (acc_bufs, a_stages), preferred first
  P.concat = P.nt <= 64 && !(P.dbg & 64);
  P.partials = 0;
  for (int want_p = want; want_p >= 1 && !P.partials; --want_p) {
    const int set_cols = P.concat ? want_p * 2 * P.nt : (want_p + 1) * P.nt;
    for (auto& c : cfg) {
      if (c[0] * set_cols + c[1] * 64 <= 512) {
        P.acc_bufs = c[0];
        P.a_stages = c[1];
        P.partials = want_p;
        break;
      }
    }
  }
  if (!P.partials) return false;
  const uint32_t set_cols = P.concat ? P.partials * 2 * P.nt : (P.partials + 1) * P.nt;
  // two K-blocks per A stage halves the hand-offs (waits, fences, commits)
  // per MMA when TMEM has room for at least two such stages
  const int free_cols = 512 - P.acc_bufs * (int)set_cols;
  // K-blocks per A stage: as many as two stages of TMEM allow (up to the
  // whole K) -- every stage costs a full/empty hand-off through the MMA warp
  P.ks = 1;
  if (!(P.dbg & 1024))
    for (int ks = 2; ks <= P.nkb && ks <= kMaxKs; ++ks)
      if (free_cols >= 2 * 64 * ks) P.ks = ks;
  P.a_stages = free_cols / (64 * P.ks);
  if (P.a_stages > kMaxAStages) P.a_stages = kMaxAStages;
  if (P.a_stages < 2) return false;
  const uint32_t need = P.acc_bufs * set_cols + P.a_stages * 64 * P.ks;
  P.tmem_cols = need <= 128 ? 128 : (need <= 256 ? 256 : 512);
  return true;
}

size_t smem_aux_bytes(const TcParams& P) {
  const size_t segs = (size_t)(P.nkb * P.sub) << (5 - P.a.in.cbs);
  return ((sizeof(Smem) + 15) & ~size_t(15)) + segs * sizeof(int2) + 16 + (size_t)P.etab.rows * P.a.epi.npad * 4;
}

size_t smem_bytes(const TcParams& P) {
  size_t b = P.resident ? (size_t)P.b_stage_bytes * P.nkb : (size_t)P.b_stage_bytes * P.nbs;
  return 1024 + b + (P.staged ? 2 * (size_t)P.st_bytes : 0) + smem_aux_bytes(P);
}

// staging geometry of a layer: box covering the input rows of one tile's
// output rows within one image, all columns incl. padding
void staging_geometry(const ConvArgs& a, TcParams& P) {
  const PixelMap& pm = a.pm;
  const int hw_out = pm.order == kPlain ? pm.ho * pm.wo : pm.hp * pm.wp * 4;
  int rows_out;
  if (pm.order == kPlain) rows_out = (kTileM + pm.wo - 1) / pm.wo + 1;
  else rows_out = 2 * ((kTileM / 4 + pm.wp - 1) / pm.wp + 1);
  if (rows_out > pm.ho) rows_out = pm.ho;
  P.box_h = (rows_out - 1) * a.stride + a.kh;
  P.box_w = (pm.wo - 1) * a.stride + a.kw;
  P.pieces = (kTileM + hw_out - 1) / hw_out + 1;
  if (P.pieces > (int)((host_pixel_count(pm, a.batch) + hw_out - 1) / hw_out)) P.pieces = a.batch;
  P.piece_bytes = (uint32_t)(((size_t)P.box_w * P.box_h * a.in.cb * 4 + 1023) & ~size_t(1023));
  P.st_bytes = P.piece_bytes * P.pieces;
  P.nblk_in = a.in.nblk;
  P.kpc = a.in.nblk == 1 ? P.nsub_real : P.taps;  // sub-blocks per channel block (cb = 32 when nblk > 1)
}

}  // namespace

// debugging aid (not part of pcnn.h): drain the CTA-0 event trace
extern "C" int pcnn_tc_trace(unsigned long long* host, int n) {
  int m = n < kTraceLen ? n : kTraceLen;
  cudaMemcpyFromSymbol(host, g_trace, sizeof(unsigned long long) * m);
  cudaMemset(reinterpret_cast<void*>(0), 0, 0);
  static unsigned long long zeros[kTraceLen];
  cudaMemcpyToSymbol(g_trace, zeros, sizeof(zeros));
  return m;
}

bool conv_tc_supported(const ConvArgs& a) {
  TcParams P;
  return make_params(a, P);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static bool encode_input_map(const ConvArgs& a, TcParams& P) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) != cudaSuccess || !ptr)
      return false;
    fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  const TensorView& in = a.in;
  const cuuint64_t dims[4] = {(cuuint64_t)in.cb, (cuuint64_t)in.w, (cuuint64_t)in.h,
                              (cuuint64_t)a.batch * in.nblk};
  const cuuint64_t strides[3] = {(cuuint64_t)in.cb * 4, (cuuint64_t)in.w * in.cb * 4,
                                 (cuuint64_t)in.h * in.w * in.cb * 4};
  const cuuint32_t box[4] = {(cuuint32_t)in.cb, (cuuint32_t)P.box_w, (cuuint32_t)P.box_h, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUtensorMapSwizzle swz = in.cb == 32 ? CU_TENSOR_MAP_SWIZZLE_128B
                                 : in.cb == 16 ? CU_TENSOR_MAP_SWIZZLE_64B
                                 : in.cb == 8 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = fn(reinterpret_cast<CUtensorMap*>(&P.tmap), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, in.base, dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

void launch_conv_tc(const ConvArgs& a, cudaStream_t s) {
  TcParams P;
  if (!make_params(a, P)) return;
  if (P.staged && !encode_input_map(a, P)) P.staged = 0;
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  const size_t smem = smem_bytes(P);
  const int tiles = P.m_tiles * P.n_tiles;
  const int grid = tiles < nsm ? tiles : nsm;
  const int mode = a.f16 ? (a.in.split ? 2 : 1) : 0;
  switch (a.in.cbs * 4 + mode) {
#define PCNN_TC_LAUNCH(C, H, SP)                                                                              \
  case C * 4 + (H ? (SP ? 2 : 1) : 0):                                                                        \
    cudaFuncSetAttribute(conv_tc_kernel<C, H, SP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);   \
    launch_pdl(conv_tc_kernel<C, H, SP>, grid, kThreads, smem, s, a.opt.pdl, P);                                         \
    break;
    PCNN_TC_LAUNCH(2, false, false)
    PCNN_TC_LAUNCH(3, false, false)
    PCNN_TC_LAUNCH(4, false, false)
    PCNN_TC_LAUNCH(5, false, false)
    PCNN_TC_LAUNCH(2, true, false)
    PCNN_TC_LAUNCH(3, true, false)
    PCNN_TC_LAUNCH(4, true, false)
    PCNN_TC_LAUNCH(5, true, false)
    PCNN_TC_LAUNCH(2, true, true)
    PCNN_TC_LAUNCH(3, true, true)
    PCNN_TC_LAUNCH(4, true, true)
    PCNN_TC_LAUNCH(5, true, true)
#undef PCNN_TC_LAUNCH
    default: break;
  }
}

}  // namespace pcnn
