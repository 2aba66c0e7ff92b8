// Shared device helpers for libpcnn (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "pcnn.h"

namespace pcnn {

constexpr int kMaxPolyDeg = 8;
constexpr int kMaxBiDeg = 4;

// Resolved view of one activation tensor for a given batch.
struct TensorView {
  float* base;
  int c, h, w, cb, nblk, is_vector;
  int cbs;  // log2(cb); cb is a power of two
  __host__ __device__ int cpad() const { return nblk * cb; }
  // address of element (b, channel, y, x) of a spatial tensor
  __device__ __forceinline__ float* at(int b, int ch, int y, int x) const {
    return base + ((((int64_t)b * nblk + (ch >> cbs)) * h + y) * w + x) * cb + (ch & (cb - 1));
  }
  // address of the channel group starting at ch (the group stays in a block)
  __device__ __forceinline__ float* pix(int b, int ch, int y, int x) const { return at(b, ch, y, x); }
};

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

// Quadratic join S(x, y) with coefficient vectors x2 y2 xy x y c.
__device__ __forceinline__ float polyskip(const float* __restrict__ c, int64_t stride, int ch,
                                          float x, float y) {
  float x2 = __ldg(c + ch), y2 = __ldg(c + stride + ch), xy = __ldg(c + 2 * stride + ch);
  float cx = __ldg(c + 3 * stride + ch), cy = __ldg(c + 4 * stride + ch);
  float c0 = __ldg(c + 5 * stride + ch);
  return fmaf(x2 * x, x, fmaf(y2 * y, y, fmaf(xy * x, y, fmaf(cx, x, fmaf(cy, y, c0)))));
}

}  // namespace pcnn
