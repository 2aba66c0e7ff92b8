// Shared device helpers for libpcnn (sm_100a).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "pcnn.h"

namespace pcnn {

constexpr int kMaxPolyDeg = 8;
constexpr int kMaxBiDeg = 4;

// Resolved view of one activation tensor for a given batch.
//
// Storage formats:
//   fp32  (split = 0): channel-blocked [B][C/cb][H][W][cb] floats.
//   split (split = 1): x = hi + lo as two fp16 planes (|x - hi - lo| <=
//         2^-22 |x| + 2^-25), each [C/8][grid][8]: 8 channels = 16 bytes per
//         position of a zero-bordered grid whose border rows and columns are
//         SHARED by neighbours -- row pitch W+1 (column W is zero and is also
//         the left neighbour of the next row), H+1 rows per image (row 0 of
//         each image is zero and is also the previous image's bottom
//         neighbour), one leading zero position: element (b, y, x) at
//         position 1 + (b (H+1) + y + 1)(W+1) + x.  A 3x3 conv's taps are
//         fixed offsets (ky-1)(W+1) + kx-1 in this flattened grid.
//         Written by producers of tensors that only tcgen05 fp16x2 convs
//         read; a value outside |x| < 2^15 (or not finite) sets *flag and the
//         host reruns the batch on fp32 tensors.
//   parity split (split = 2): the same padded grid cut into its four
//         (row, column) parity planes, [C/8][4][B][Hq][Wq][8] with Hq =
//         ceil((H+2)/2): a stride-2 conv's taps become fixed offsets inside
//         one parity plane.  Used when every conv reading the tensor has
//         stride 2.
struct TensorView {
  float* base;
  int c, h, w, cb, nblk, is_vector;
  int cbs;  // log2(cb); cb is a power of two
  int split;
  int hp, wp;       // split 1: rows per image h + 1, pitch w + 1; split 2: parity grid ceil((h+2)/2), ceil((w+2)/2)
  int64_t pstride;  // split 2: halves per parity plane (batch * hp * wp * 8)
  int64_t kstride;  // halves per 8-channel group (batch * hp * wp * 8, x4 planes for split 2)
  int64_t plane;    // split: halves per hi / lo plane
  int* flag;        // split: overflow flag (device)
  float sstore, sload;  // split: stored value = x * sstore; x = stored * sload (powers of two)
  __host__ __device__ int cpad() const { return nblk * cb; }
  __host__ __device__ __forceinline__ int64_t index(int b, int ch, int y, int x) const {
    return ((((int64_t)b * nblk + (ch >> cbs)) * h + y) * w + x) * cb + (ch & (cb - 1));
  }
  // split: half index of (b, ch, y, x) inside a plane
  __host__ __device__ __forceinline__ int64_t sindex(int b, int ch, int y, int x) const {
    if (split == 2) {
      const int yp = y + 1, xp = x + 1;
      return (ch >> 3) * kstride + (((yp & 1) << 1) | (xp & 1)) * pstride +
             (((int64_t)b * hp + (yp >> 1)) * wp + (xp >> 1)) * 8 + (ch & 7);
    }
    return (ch >> 3) * kstride + (1 + ((int64_t)b * hp + y + 1) * wp + x) * 8 + (ch & 7);
  }
  // address of element (b, channel, y, x) of a spatial tensor (fp32 format)
  __device__ __forceinline__ float* at(int b, int ch, int y, int x) const { return base + index(b, ch, y, x); }
  __device__ __forceinline__ __half* hi() const { return reinterpret_cast<__half*>(base); }
  __device__ __forceinline__ __half* lo() const { return reinterpret_cast<__half*>(base) + plane; }
  // address of element (b, channel, y, x) of a spatial tensor (fp32 format)
  __device__ __forceinline__ float* pix(int b, int ch, int y, int x) const { return at(b, ch, y, x); }
};

// floats a tensor occupies in either format (the workspace holds the larger)
__host__ __device__ inline int64_t tensor_storage_floats(int64_t batch, int64_t c, int64_t cpad, int64_t h, int64_t w,
                                                         bool is_vector) {
  const int64_t fp32 = batch * cpad * h * w;
  if (is_vector) return fp32;
  // 2 planes (hi, lo) of halves; the parity layout rounds the padded grid up to even
  const int64_t split = ((cpad + 7) / 8) * 8 * batch * ((h + 3) / 2 * 2) * ((w + 3) / 2 * 2);
  (void)c;
  return fp32 > split ? fp32 : split;
}

// n / d for 0 <= n < 2^31 without a division: q = (umulhi(n, m) + n) >> l
// (Granlund-Montgomery; m, l from make_fastdiv on the host)
struct FastDiv {
  uint32_t d, m, l;
  __device__ __forceinline__ uint32_t div(uint32_t n) const { return (__umulhi(n, m) + n) >> l; }
};
inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f;
  f.d = d;
  f.l = 0;
  while ((1u << f.l) < d) ++f.l;
  f.m = (uint32_t)((((uint64_t)1 << 32) * (((uint64_t)1 << f.l) - d)) / d + 1);
  return f;
}

// 4 consecutive floats from shared memory (p: generic pointer into smem, 16-byte aligned)
__device__ __forceinline__ float4 lds4(const float* p) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"((uint32_t)__cvta_generic_to_shared(p)));
  return v;
}
__device__ __forceinline__ void lds16(const float* p, float* v) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float4 f = lds4(p + 4 * q);
    v[4 * q] = f.x; v[4 * q + 1] = f.y; v[4 * q + 2] = f.z; v[4 * q + 3] = f.w;
  }
}

// ---- split-format element access ------------------------------------------------
__device__ __forceinline__ uint32_t pack_half2(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}
__device__ __forceinline__ float2 unpack_half2(uint32_t u) {
  return __half22float2(*reinterpret_cast<const __half2*>(&u));
}
// ---- packed fp32 pairs (sm_100 FFMA2 / FADD2 / FMUL2: one instruction per two lanes of work) ----
__device__ __forceinline__ float2 f2(const float* v) { return make_float2(v[0], v[1]); }
__device__ __forceinline__ void f2_put(float* v, float2 p) { v[0] = p.x; v[1] = p.y; }
// v[0..n) = v * s + c (elementwise, s and c per element)
template <int N>
__device__ __forceinline__ void fma_n(float* v, const float* s, const float* c) {
#pragma unroll
  for (int i = 0; i < N; i += 2) f2_put(v + i, __ffma2_rn(f2(v + i), f2(s + i), f2(c + i)));
}
// v[0..n) = v * s + c with one scalar s
template <int N>
__device__ __forceinline__ void fma_n(float* v, float s, const float* c) {
  const float2 ss = make_float2(s, s);
#pragma unroll
  for (int i = 0; i < N; i += 2) f2_put(v + i, __ffma2_rn(f2(v + i), ss, f2(c + i)));
}
// v[0..n) += t
template <int N>
__device__ __forceinline__ void add_n(float* v, const float* t) {
#pragma unroll
  for (int i = 0; i < N; i += 2) f2_put(v + i, __fadd2_rn(f2(v + i), f2(t + i)));
}

// hi/lo fp16 pairs of (a, b); returns false if either is outside |x| < 2^15
__device__ __forceinline__ bool split_pair(float a, float b, uint32_t& hi, uint32_t& lo) {
  hi = pack_half2(a, b);
  const float2 h = unpack_half2(hi);
  const float2 d = __fadd2_rn(make_float2(a, b), make_float2(-h.x, -h.y));
  lo = pack_half2(d.x, d.y);
  return fabsf(a) < 32768.f && fabsf(b) < 32768.f;
}

// store 4 consecutive channels (ch % 4 == 0) in the tensor's format
__device__ __forceinline__ void store4_any(const TensorView& t, int b, int ch, int y, int x, float v0, float v1,
                                           float v2, float v3) {
  if (!t.split) {
    *reinterpret_cast<float4*>(t.base + t.index(b, ch, y, x)) = make_float4(v0, v1, v2, v3);
    return;
  }
  const int64_t e = t.sindex(b, ch, y, x);
  uint2 hi, lo;
  const float s = t.sstore;
  const bool ok = split_pair(v0 * s, v1 * s, hi.x, lo.x) & split_pair(v2 * s, v3 * s, hi.y, lo.y);
  *reinterpret_cast<uint2*>(t.hi() + e) = hi;
  *reinterpret_cast<uint2*>(t.lo() + e) = lo;
  if (!ok) atomicExch(t.flag, 1);
}

// 16 consecutive channels of a split tensor at half index e (channel group
// 2j of the row; the second group is kstride further)
// (s: storage scale applied here, 1 when the caller folded it into its math)
__device__ __forceinline__ void store16_split_at(const TensorView& t, int64_t e, const float* v, float s) {
  uint32_t hi[8], lo[8];
  const float2 ss = make_float2(s, s);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float2 x = __fmul2_rn(f2(v + 2 * i), ss);
    split_pair(x.x, x.y, hi[i], lo[i]);
  }
  // range check on the packed hi halves: max |hi| (NaN-propagating) < 2^15
  __half2 m = __habs2(*reinterpret_cast<const __half2*>(&hi[0]));
#pragma unroll
  for (int i = 1; i < 8; ++i) m = __hmax2_nan(m, __habs2(*reinterpret_cast<const __half2*>(&hi[i])));
  const float2 mf = __half22float2(m);
  const bool ok = mf.x < 32768.f && mf.y < 32768.f;
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    *reinterpret_cast<uint4*>(t.hi() + e + g * t.kstride) = make_uint4(hi[4 * g], hi[4 * g + 1], hi[4 * g + 2], hi[4 * g + 3]);
    *reinterpret_cast<uint4*>(t.lo() + e + g * t.kstride) = make_uint4(lo[4 * g], lo[4 * g + 1], lo[4 * g + 2], lo[4 * g + 3]);
  }
  if (!ok) atomicExch(t.flag, 1);
}

// store 8 consecutive channels (ch % 8 == 0) in the tensor's format
__device__ __forceinline__ void store8_any(const TensorView& t, int b, int ch, int y, int x, const float* v) {
  if (!t.split) {
    float4* o = reinterpret_cast<float4*>(t.base + t.index(b, ch, y, x));
    o[0] = make_float4(v[0], v[1], v[2], v[3]);
    o[1] = make_float4(v[4], v[5], v[6], v[7]);
    return;
  }
  const int64_t e = t.sindex(b, ch, y, x);
  const float s = t.sstore;
  uint32_t hi[4], lo[4];
  bool ok = true;
#pragma unroll
  for (int i = 0; i < 4; ++i) ok &= split_pair(v[2 * i] * s, v[2 * i + 1] * s, hi[i], lo[i]);
  *reinterpret_cast<uint4*>(t.hi() + e) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
  *reinterpret_cast<uint4*>(t.lo() + e) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
  if (!ok) atomicExch(t.flag, 1);
}

// store 16 consecutive channels (ch % 16 == 0; one block when fp32, cb >= 16):
// whole 32-byte sectors per thread in both formats
// cb = 4 (pooled convs' scratch maps): four channel blocks, each 16 bytes per
// position with consecutive positions adjacent, so a warp whose lanes hold
// consecutive positions writes 512 contiguous bytes per store instruction
// (cb >= 16 puts a lane's 64 bytes together and the lanes 64 bytes apart:
// 32 wavefronts of the LSU data pipe per instruction instead of 4)
__device__ __forceinline__ void store16_any(const TensorView& t, int b, int ch, int y, int x, const float* v) {
  if (!t.split) {
    float4* o = reinterpret_cast<float4*>(t.base + t.index(b, ch, y, x));
    const int64_t qs = t.cb == 4 ? (int64_t)t.h * t.w : 1;  // float4 stride between 4-channel groups
#pragma unroll
    for (int q = 0; q < 4; ++q) o[q * qs] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    return;
  }
  store16_split_at(t, t.sindex(b, ch, y, x), v, t.sstore);
}

// 8 channels (one 16-byte group) of a split tensor as fp32
__device__ __forceinline__ void load8_split(const TensorView& t, int64_t e, float* v) {
  // .cg (L2 only): inside a chained kernel the tensor is written by other
  // SMs during the same launch, so L1 must not hold stale lines
  const uint4 h = __ldcg(reinterpret_cast<const uint4*>(t.hi() + e));
  const uint4 l = __ldcg(reinterpret_cast<const uint4*>(t.lo() + e));
  const uint32_t hw[4] = {h.x, h.y, h.z, h.w}, lw[4] = {l.x, l.y, l.z, l.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 a = unpack_half2(hw[i]), c = unpack_half2(lw[i]);
    v[2 * i] = a.x + c.x;
    v[2 * i + 1] = a.y + c.y;
  }
}

// load 16 consecutive channels (ch % 16 == 0; one block when fp32) as fp32
__device__ __forceinline__ void load16_any(const TensorView& t, int b, int ch, int y, int x, float* v) {
  if (!t.split) {
    const float4* s = reinterpret_cast<const float4*>(t.base + t.index(b, ch, y, x));
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 f = __ldcg(s + q);
      v[4 * q] = f.x; v[4 * q + 1] = f.y; v[4 * q + 2] = f.z; v[4 * q + 3] = f.w;
    }
    return;
  }
  const int64_t e = t.sindex(b, ch, y, x);
  load8_split(t, e, v);
  load8_split(t, e + t.kstride, v + 8);
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] *= t.sload;
}

// The same 16 channels as raw 16-byte words (fp32: 4 x float4; split: hi/lo
// of group 0, hi/lo of group 1): issue the loads early, decode at use, so the
// load latency overlaps other work instead of stalling on the conversion.
struct Raw16 {
  uint4 q[4];
};
__device__ __forceinline__ void load16_raw(const TensorView& t, int b, int ch, int y, int x, Raw16& r) {
  if (!t.split) {
    const uint4* s = reinterpret_cast<const uint4*>(t.base + t.index(b, ch, y, x));
#pragma unroll
    for (int q = 0; q < 4; ++q) r.q[q] = __ldcg(s + q);
    return;
  }
  const int64_t e = t.sindex(b, ch, y, x);
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    r.q[2 * g] = __ldcg(reinterpret_cast<const uint4*>(t.hi() + e + g * t.kstride));
    r.q[2 * g + 1] = __ldcg(reinterpret_cast<const uint4*>(t.lo() + e + g * t.kstride));
  }
}
// (s: load scale for split words, 1 when the caller folded it into its math)
__device__ __forceinline__ void decode16_raw(const TensorView& t, const Raw16& r, float* v, float s) {
  if (!t.split) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      v[4 * q] = __uint_as_float(r.q[q].x);
      v[4 * q + 1] = __uint_as_float(r.q[q].y);
      v[4 * q + 2] = __uint_as_float(r.q[q].z);
      v[4 * q + 3] = __uint_as_float(r.q[q].w);
    }
    return;
  }
  const float2 ss = make_float2(s, s);
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    const uint32_t hw[4] = {r.q[2 * g].x, r.q[2 * g].y, r.q[2 * g].z, r.q[2 * g].w};
    const uint32_t lw[4] = {r.q[2 * g + 1].x, r.q[2 * g + 1].y, r.q[2 * g + 1].z, r.q[2 * g + 1].w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
      f2_put(v + 8 * g + 2 * i, __fmul2_rn(__fadd2_rn(unpack_half2(hw[i]), unpack_half2(lw[i])), ss));
  }
}

// cp.async (L2 -> shared, no register dependency) of the 16 channels of one
// row into four 16-byte slots dst + q * qstride, zero-filled when !ok; read
// back with lds_raw16 + decode16_raw after cp.async.wait_group
__device__ __forceinline__ void load16_async_src(const char* const* src, bool ok, uint32_t dst, uint32_t qstride) {
  const uint32_t n = ok ? 16u : 0u;
#pragma unroll
  for (int q = 0; q < 4; ++q)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst + q * qstride), "l"(src[q]), "r"(n)
                 : "memory");
  asm volatile("cp.async.commit_group;" ::: "memory");
}
// split tensor, 16 channels at half index e (as store16_split_at)
__device__ __forceinline__ void load16_async_at(const TensorView& t, int64_t e, bool ok, uint32_t dst,
                                                uint32_t qstride) {
  const char* src[4];
  src[0] = reinterpret_cast<const char*>(t.hi() + e);
  src[1] = reinterpret_cast<const char*>(t.lo() + e);
  src[2] = reinterpret_cast<const char*>(t.hi() + e + t.kstride);
  src[3] = reinterpret_cast<const char*>(t.lo() + e + t.kstride);
  load16_async_src(src, ok, dst, qstride);
}
__device__ __forceinline__ void load16_async(const TensorView& t, int b, int ch, int y, int x, bool ok, uint32_t dst,
                                             uint32_t qstride) {
  if (!t.split) {
    const char* src[4];
    const float* p = t.base + (ok ? t.index(b, ch, y, x) : 0);
#pragma unroll
    for (int q = 0; q < 4; ++q) src[q] = reinterpret_cast<const char*>(p + 4 * q);
    load16_async_src(src, ok, dst, qstride);
    return;
  }
  load16_async_at(t, ok ? t.sindex(b, ch, y, x) : 0, ok, dst, qstride);
}
__device__ __forceinline__ void lds_raw16(uint32_t src, uint32_t qstride, Raw16& r) {
#pragma unroll
  for (int q = 0; q < 4; ++q)
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.q[q].x), "=r"(r.q[q].y), "=r"(r.q[q].z), "=r"(r.q[q].w)
                 : "r"(src + q * qstride)
                 : "memory");
}

// Output-pixel enumeration of a conv unit.  PLAIN walks (b, oy, ox);
// WINDOW walks 2x2 pool windows (b, py, px) with the four window pixels at
// consecutive indices (dy, dx) so a fused pool reduces over adjacent rows.
enum PixelOrder { kPlain = 0, kWindow = 1 };

struct PixelMap {
  int order;
  int ho, wo;  // conv output dims
  int hp, wp;  // pooled dims (WINDOW)
  // m < 2^31 for every supported batch (checked at plan creation)
  __device__ __forceinline__ void decode(int64_t m64, int& b, int& oy, int& ox) const {
    const int m = (int)m64;
    if (order == kPlain) {
      const int hw = ho * wo;
      b = m / hw;
      const int r = m - b * hw;
      oy = r / wo;
      ox = r - oy * wo;
    } else {
      const int q = m >> 2, d = m & 3;
      const int hw = hp * wp;
      b = q / hw;
      const int r = q - b * hw;
      const int py = r / wp, px = r - py * wp;
      oy = 2 * py + (d >> 1);
      ox = 2 * px + (d & 1);
    }
  }
  __device__ __forceinline__ int64_t count(int batch) const {
    return order == kPlain ? (int64_t)batch * ho * wo : (int64_t)batch * hp * wp * 4;
  }
};

// ---- launch timeline (pcnn_plan_timeline) ----------------------------------
// tl[0] = max over CTAs of ~start (so ~tl[0] is the earliest start), tl[1] =
// max over CTAs of the exit time, in %globaltimer ns; both zeroed before
// every forward.  One fire-and-forget reduction per CTA and mark.
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void tl_mark(unsigned long long* tl, int end) {
  if (tl && threadIdx.x == 0) {
    const unsigned long long t = global_ns();
    if (end) atomicMax(tl + 1, t);
    else atomicMax(tl, ~t);
  }
}
// start mark at construction, end mark when the kernel body returns (thread 0).
// Kernels using it may be launched with programmatic stream serialization:
// the construction waits for the previous grid (no-op on a plain launch) and
// lets the next grid's CTAs start their prologue on the SMs this one leaves.
struct TlScope {
  unsigned long long* tl;
  __device__ __forceinline__ explicit TlScope(unsigned long long* p) : tl(p) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    tl_mark(tl, 0);
  }
  __device__ __forceinline__ ~TlScope() { tl_mark(tl, 1); }
};

// Horner with per-channel coefficients c_k at coef[k * stride + ch].
__device__ __forceinline__ float horner(const float* __restrict__ coef, int64_t stride, int deg,
                                        int ch, float x) {
  float acc = __ldg(coef + (int64_t)deg * stride + ch);
  for (int k = deg - 1; k >= 0; --k) acc = fmaf(acc, x, __ldg(coef + (int64_t)k * stride + ch));
  return acc;
}

// Bivariate S(x, y) = sum_{i+j<=d} c_ij x^i y^j, c_ij at coef[(i*(d+1)+j)*stride + ch];
// Horner in x over Horner-in-y rows (same nesting as the oracle).
__device__ __forceinline__ float bivariate(const float* __restrict__ coef, int64_t stride, int d,
                                           int ch, float x, float y) {
  float acc = 0.f;
  for (int i = d; i >= 0; --i) {
    const float* row = coef + (int64_t)(i * (d + 1)) * stride + ch;
    float r = __ldg(row + (int64_t)(d - i) * stride);
    for (int j = d - i - 1; j >= 0; --j) r = fmaf(r, y, __ldg(row + (int64_t)j * stride));
    acc = (i == d) ? r : fmaf(acc, x, r);
  }
  return acc;
}

// bivariate() for 4 consecutive channels (ch % 4 == 0, 16-byte aligned rows)
__device__ __forceinline__ float4 bivariate4(const float* __restrict__ coef, int64_t stride, int d, int ch,
                                             float4 x, float4 y) {
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int i = d; i >= 0; --i) {
    const float* row = coef + (int64_t)(i * (d + 1)) * stride + ch;
    float4 r = __ldg(reinterpret_cast<const float4*>(row + (int64_t)(d - i) * stride));
    for (int j = d - i - 1; j >= 0; --j) {
      const float4 c = __ldg(reinterpret_cast<const float4*>(row + (int64_t)j * stride));
      r = make_float4(fmaf(r.x, y.x, c.x), fmaf(r.y, y.y, c.y), fmaf(r.z, y.z, c.z), fmaf(r.w, y.w, c.w));
    }
    acc = (i == d) ? r
                   : make_float4(fmaf(acc.x, x.x, r.x), fmaf(acc.y, x.y, r.y), fmaf(acc.z, x.z, r.z),
                                 fmaf(acc.w, x.w, r.w));
  }
  return acc;
}

// bivariate4 with the degree a compile-time constant: the loops unroll, so
// all coefficient loads issue up front instead of one dependent load per
// Horner step (the band epilogue runs these on few warps)
template <int D>
__device__ __forceinline__ float4 bivariate4_t(const float* __restrict__ coef, int64_t stride, int ch, float4 x,
                                               float4 y) {
  float4 c[D + 1][D + 1];
#pragma unroll
  for (int i = 0; i <= D; ++i)
#pragma unroll
    for (int j = 0; j + i <= D; ++j)
      c[i][j] = __ldg(reinterpret_cast<const float4*>(coef + (int64_t)(i * (D + 1) + j) * stride + ch));
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int i = D; i >= 0; --i) {
    float4 r = c[i][D - i];
#pragma unroll
    for (int j = D - i - 1; j >= 0; --j)
      r = make_float4(fmaf(r.x, y.x, c[i][j].x), fmaf(r.y, y.y, c[i][j].y), fmaf(r.z, y.z, c[i][j].z),
                      fmaf(r.w, y.w, c[i][j].w));
    acc = (i == D) ? r
                   : make_float4(fmaf(acc.x, x.x, r.x), fmaf(acc.y, x.y, r.y), fmaf(acc.z, x.z, r.z),
                                 fmaf(acc.w, x.w, r.w));
  }
  return acc;
}
// two evaluations sharing one coefficient load: (u, w) = (S(x0, y0), S(x1, y1))
template <int D>
__device__ __forceinline__ void bivariate4x2_t(const float* __restrict__ coef, int64_t stride, int ch, float4 x0,
                                               float4 y0, float4 x1, float4 y1, float4& u, float4& w) {
  float4 c[D + 1][D + 1];
#pragma unroll
  for (int i = 0; i <= D; ++i)
#pragma unroll
    for (int j = 0; j + i <= D; ++j)
      c[i][j] = __ldg(reinterpret_cast<const float4*>(coef + (int64_t)(i * (D + 1) + j) * stride + ch));
  auto ev = [&](float4 x, float4 y) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int i = D; i >= 0; --i) {
      float4 r = c[i][D - i];
#pragma unroll
      for (int j = D - i - 1; j >= 0; --j)
        r = make_float4(fmaf(r.x, y.x, c[i][j].x), fmaf(r.y, y.y, c[i][j].y), fmaf(r.z, y.z, c[i][j].z),
                        fmaf(r.w, y.w, c[i][j].w));
      acc = (i == D) ? r
                     : make_float4(fmaf(acc.x, x.x, r.x), fmaf(acc.y, x.y, r.y), fmaf(acc.z, x.z, r.z),
                                   fmaf(acc.w, x.w, r.w));
    }
    return acc;
  };
  u = ev(x0, y0);
  w = ev(x1, y1);
}
__device__ __forceinline__ float4 bivariate4_any(const float* __restrict__ coef, int64_t stride, int d, int ch,
                                                 float4 x, float4 y) {
  switch (d) {
    case 1: return bivariate4_t<1>(coef, stride, ch, x, y);
    case 2: return bivariate4_t<2>(coef, stride, ch, x, y);
    case 3: return bivariate4_t<3>(coef, stride, ch, x, y);
    case 4: return bivariate4_t<4>(coef, stride, ch, x, y);
    default: return bivariate4(coef, stride, d, ch, x, y);
  }
}

// Quadratic join S(x, y) with coefficient vectors x2 y2 xy x y c.
__device__ __forceinline__ float polyskip(const float* __restrict__ c, int64_t stride, int ch,
                                          float x, float y) {
  float x2 = __ldg(c + ch), y2 = __ldg(c + stride + ch), xy = __ldg(c + 2 * stride + ch);
  float cx = __ldg(c + 3 * stride + ch), cy = __ldg(c + 4 * stride + ch);
  float c0 = __ldg(c + 5 * stride + ch);
  return fmaf(x2 * x, x, fmaf(y2 * y, y, fmaf(xy * x, y, fmaf(cx, x, fmaf(cy, y, c0)))));
}

}  // namespace pcnn
