// Weight image of the tcgen05 conv kernel.
//
// The B operand (weights, N = output channels, K = im2col depth) is split
// into tf32 hi and lo parts (3xTF32: a*b ~ ahi*bhi + ahi*blo + alo*bhi) and
// stored exactly as the kernel's shared-memory tiles: K-major, 128-byte
// swizzle (UMMA layout SWIZZLE_128B, 8-row atoms of 1024 B, 16-byte chunk c
// of row r at chunk position c ^ (r & 7)).  One K-block = 32 tf32 of every
// row.  Global order: [n_tile][k_block][hi, lo][NT rows x 32], so one bulk
// copy of 2*NT*128 bytes brings both parts of a K-block.
//
// The fp16x2 variant (kind::f16) uses the same byte geometry with 64 fp16 per
// 128-byte row: x = hi + lo with hi, lo fp16 (22 significant bits), the
// weights pre-scaled by a power of two 2^e so max|w| 2^e lies in [2^13, 2^14)
// (the epilogue multiplies by 2^-e; slot[1] of the op's scale pair).
#pragma once

#include <cuda_fp16.h>
#include <stdint.h>

namespace pcnn {

constexpr int kTcBK = 32;  // tf32 elements per K-block (128 bytes per row)

__host__ __device__ inline int tc_ntile(int npad) { return npad <= 128 ? npad : 128; }
__host__ __device__ inline int tc_kblocks(int kp) { return (kp + kTcBK - 1) / kTcBK; }

__device__ __forceinline__ uint32_t f32_to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// float index of (row n, depth k, part) inside the image
__host__ __device__ inline int64_t tc_image_index(int n, int k, int part, int npad, int kp) {
  const int nt_rows = tc_ntile(npad);
  const int nkb = tc_kblocks(kp);
  const int nt = n / nt_rows, r = n % nt_rows;
  const int kb = k / kTcBK, kk = k % kTcBK;
  const int chunk = (kk >> 2) ^ (r & 7);
  const int64_t base = ((int64_t)(nt * nkb + kb) * 2 + part) * nt_rows * kTcBK;
  return base + (int64_t)r * kTcBK + chunk * 4 + (kk & 3);
}

__host__ __device__ inline int64_t tc_image_floats(int npad, int kp) {
  const int nt_rows = tc_ntile(npad);
  const int ntiles = (npad + nt_rows - 1) / nt_rows;
  return (int64_t)ntiles * tc_kblocks(kp) * 2 * nt_rows * kTcBK;
}

// pack src [rows][k] float64 into the image (zero K padding)
__device__ inline void pack_tc_weights_device(const double* src, float* dst, int rows, int k,
                                              int64_t tid, int64_t nthreads) {
  const int kpad = tc_kblocks(k) * kTcBK;
  const int64_t total = (int64_t)rows * kpad;
  for (int64_t i = tid; i < total; i += nthreads) {
    int n = (int)(i / kpad), kk = (int)(i % kpad);
    double w = kk < k ? src[(int64_t)n * k + kk] : 0.0;
    float wf = (float)w;
    uint32_t hi = f32_to_tf32(wf);
    float lo_f = (float)(w - (double)__uint_as_float(hi));
    uint32_t lo = f32_to_tf32(lo_f);
    dst[tc_image_index(n, kk, 0, rows, k)] = __uint_as_float(hi);
    dst[tc_image_index(n, kk, 1, rows, k)] = __uint_as_float(lo);
  }
}

// ---- fp16x2 image -------------------------------------------------------------------
constexpr int kTc16BK = 64;  // fp16 elements per K-block (128 bytes per row)
__host__ __device__ inline int tc16_kblocks(int kp) { return (kp + kTc16BK - 1) / kTc16BK; }

// half index of (row n, depth k, part) inside the fp16 image
__host__ __device__ inline int64_t tc16_image_index(int n, int k, int part, int npad, int kp) {
  const int nt_rows = tc_ntile(npad);
  const int nkb = tc16_kblocks(kp);
  const int nt = n / nt_rows, r = n % nt_rows;
  const int kb = k / kTc16BK, kk = k % kTc16BK;
  const int chunk = (kk >> 3) ^ (r & 7);
  const int64_t base = ((int64_t)(nt * nkb + kb) * 2 + part) * nt_rows * kTc16BK;
  return base + (int64_t)r * kTc16BK + chunk * 8 + (kk & 7);
}

__host__ __device__ inline int64_t tc16_image_floats(int npad, int kp) {
  const int nt_rows = tc_ntile(npad);
  const int ntiles = (npad + nt_rows - 1) / nt_rows;
  return (int64_t)ntiles * tc16_kblocks(kp) * nt_rows * kTc16BK;  // 2 parts x 2 bytes = 1 float per element
}

// power-of-two exponent e with max|w| 2^e in [2^13, 2^14) (0 for an all-zero tensor)
__device__ inline int tc16_scale_exp(float amax) {
  if (!(amax > 0.f) || !isfinite(amax)) return 0;
  int x;
  frexpf(amax, &x);  // amax in [2^(x-1), 2^x)
  int e = 14 - x;
  return e < -120 ? -120 : (e > 120 ? 120 : e);
}

// pack src [rows][k] float64 (scaled by 2^e) into the fp16 image (zero K padding)
__device__ inline void pack_tc16_weights_device(const double* src, __half* dst, int rows, int k, int e,
                                                int64_t tid, int64_t nthreads) {
  const int kpad = tc16_kblocks(k) * kTc16BK;
  const int64_t total = (int64_t)rows * kpad;
  for (int64_t i = tid; i < total; i += nthreads) {
    int n = (int)(i / kpad), kk = (int)(i % kpad);
    const double w = kk < k ? ldexp(src[(int64_t)n * k + kk], e) : 0.0;
    const __half hi = __double2half(w);
    const __half lo = __double2half(w - (double)__half2float(hi));
    dst[tc16_image_index(n, kk, 0, rows, k)] = hi;
    dst[tc16_image_index(n, kk, 1, rows, k)] = lo;
  }
}

// ---- fp16x2 image of the shared-memory (halo tile) conv kernel ---------------------
// K-block = one (16-channel chunk q, tap t); per block the B operand is
// [kc8 = 2][2 NT rows: hi then lo][8 fp16], K-major without swizzle (core
// matrices of 8 rows x 16 bytes), so [B_hi | B_lo] is one N = 2 NT operand.
// Global order [n_tile][q][tap][block]: a stage streams taps consecutive blocks.
__host__ __device__ inline int64_t tcss_image_floats(int npad, int cpad, int taps) {
  const int nt_rows = tc_ntile(npad);
  const int ntiles = (npad + nt_rows - 1) / nt_rows;
  return (int64_t)ntiles * ((cpad + 15) / 16) * taps * 16 * nt_rows;
}

__device__ inline void pack_tcss_weights_device(const double* src, __half* dst, int rows, int k, int taps, int cb,
                                                int e, int64_t tid, int64_t nthreads) {
  const int NT = tc_ntile(rows);
  const int cpad = k / taps, nq = (cpad + 15) / 16;  // channels >= cpad stay zero
  const int64_t total = (int64_t)rows * cpad * taps;
  for (int64_t i = tid; i < total; i += nthreads) {
    const int n = (int)(i / ((int64_t)cpad * taps));
    const int rem = (int)(i - (int64_t)n * cpad * taps);
    const int t = rem / cpad, ch = rem - t * cpad;
    const double w = ldexp(src[(int64_t)n * k + ((ch / cb) * taps + t) * cb + ch % cb], e);
    const __half hi = __double2half(w);
    const __half lo = __double2half(w - (double)__half2float(hi));
    const int q = ch >> 4, g = (ch >> 3) & 1, j = ch & 7;
    const int nt = n / NT, r = n - nt * NT;
    const int64_t base = (((int64_t)nt * nq + q) * taps + t) * 32 * NT + g * 16 * NT;
    dst[base + r * 8 + j] = hi;
    dst[base + (NT + r) * 8 + j] = lo;
  }
}

}  // namespace pcnn
