// Fused conv epilogue of the tcgen05 kernels for one pixel row and 16
// consecutive output channels: bias -> [affine] -> [residual: + skip |
// S(v, skip)] -> [polynomial] -> [pool] -> store in the output's format.
// Per-channel parameters come from a table staged in shared memory (rows of
// npad floats: bias, [affine scale, shift], [poly c_0..c_d], [join x2 y2 xy x
// y c]).  Restates epilogue.cuh's epi_point / epi_pool4 16 channels at a time.
#pragma once

#include "epilogue.cuh"

namespace pcnn {

struct EpiTab {
  const float* ptab;  // shared memory
  int rows;
  int row_aff, row_poly, row_res;  // -1 if absent
};

inline EpiTab epi_tab_layout(const EpiParams& e) {
  EpiTab t;
  t.ptab = nullptr;
  int rows = 1;
  t.row_aff = e.aff ? rows : -1;
  rows += e.aff ? 2 : 0;
  t.row_poly = e.poly_deg ? rows : -1;
  rows += e.poly_deg ? e.poly_deg + 1 : 0;
  t.row_res = e.residual >= 2 ? rows : -1;
  rows += e.residual >= 2 ? 6 : 0;
  t.rows = rows;
  return t;
}

// Scale folding (halo-tile kernel): yscale multiplies the rows of S's
// skip variable (its powers), so split skip words enter without their load
// scale; oscale multiplies the rows of the last stage (poly, else S), so the
// result comes out already in storage units.  Both are powers of two: the
// folded arithmetic is exact.
// the value epi_fill_tab stores at table index i (read-only loads: callers
// may batch several before their first store)
__device__ __forceinline__ float epi_tab_value(const EpiParams& ep, const EpiTab& T, int i, float yscale, float oscale) {
  const int np = ep.npad;
  const int r = i / np, c = i - r * np;
  float v;
  if (r == 0) v = __ldg(ep.bias + c);
  else if (T.row_aff >= 0 && r < T.row_aff + 2 && r >= T.row_aff) v = __ldg(ep.aff + (r - T.row_aff) * np + c);
  else if (T.row_poly >= 0 && r >= T.row_poly && r <= T.row_poly + ep.poly_deg) {
    v = __ldg(ep.poly + (r - T.row_poly) * np + c) * oscale;
  } else {
    // S rows: x2 y2 xy x y c; the skip is y for residual 2, x for residual 3
    const int k = r - T.row_res;
    v = __ldg(ep.res + k * np + c);
    const int sq = ep.residual == 2 ? 1 : 0, lin = ep.residual == 2 ? 4 : 3;
    if (k == sq) v *= yscale * yscale;
    else if (k == 2 || k == lin) v *= yscale;
    if (!ep.poly_deg) v *= oscale;
  }
  return v;
}

__device__ __forceinline__ void epi_fill_tab(const EpiParams& ep, const EpiTab& T, float* ptab, int tid, int nthreads,
                                             float yscale = 1.f, float oscale = 1.f) {
  for (int i = tid; i < T.rows * ep.npad; i += nthreads) ptab[i] = epi_tab_value(ep, T, i, yscale, oscale);
}

__device__ __forceinline__ void epi_store4(const EpiParams& e, int b, int ch, int y, int x, const float* o) {
  store4_any(e.out, b, ch, y, x, o[0], o[1], o[2], o[3]);
}

// skip values of channels [chb, chb + 16) for a residual epilogue (zeros
// for an invalid row); issued ahead of the accumulator wait by the callers
__device__ __forceinline__ void epi_load_skip(const EpiParams& e, int chb, bool valid, int b, int oy, int ox,
                                              float* sk) {
  if (e.residual && valid) {
    load16_any(e.skip, b, chb, oy, ox, sk);
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j) sk[j] = 0.f;
  }
}

// one transposing butterfly step over 2 * O values: lanes with bit O set keep
// the upper half, the others the lower half, each adding its partner's copy
template <int O>
__device__ __forceinline__ void butterfly_step(float* x, int lane) {
  const bool up = (lane & O) != 0;
#pragma unroll
  for (int i = 0; i < O; ++i) {
    const float send = up ? x[i] : x[i + O];
    const float keep = up ? x[i + O] : x[i];
    x[i] = keep + __shfl_xor_sync(0xffffffffu, send, O);
  }
}

// raw form: issue now, decode (epi_skip_decode) right before the math
__device__ __forceinline__ void epi_load_skip_raw(const EpiParams& e, int chb, bool valid, int b, int oy, int ox,
                                                  Raw16& r) {
  if (e.residual && valid) {
    load16_raw(e.skip, b, chb, oy, ox, r);
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) r.q[q] = make_uint4(0, 0, 0, 0);
  }
}
__device__ __forceinline__ void epi_skip_decode(const EpiParams& e, const Raw16& r, float* sk) {
  if (e.residual) {
    decode16_raw(e.skip, r, sk, e.skip.sload);
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j) sk[j] = 0.f;
  }
}

// ---- the fused epilogue in pieces: epi_point16 (per element), then one of
// epi_store16 / epi_window16 / epi_global16; kernels instantiate only the
// pieces their units use (the instruction cache holds one short path), and
// epi_chunk16 dispatches on e.pool at run time.

// v: accumulator values of channels [chb, chb + 16), times vscale in true
// units; sk: their skip values (epi_load_skip).  bias -> [affine] ->
// [residual: + skip | S(v, skip)] -> [polynomial]; padded channels -> 0.
__device__ __forceinline__ void epi_point16(const EpiParams& e, const EpiTab& T, float* v, float vscale,
                                            const float* sk, int chb) {
  const float* pt = T.ptab + chb;  // per-channel parameters, shared by all rows
  const int np = e.npad;
  // packed fp32 pairs throughout (FFMA2 / FADD2): half the FMA-pipe issue slots
  float c[16];
  lds16(pt, c);
  fma_n<16>(v, vscale, c);
  if (T.row_aff >= 0) {
    float sc[16], sh[16];
    lds16(pt + T.row_aff * np, sc);
    lds16(pt + (T.row_aff + 1) * np, sh);
    fma_n<16>(v, sc, sh);
  }
  if (e.residual == 1) {
    add_n<16>(v, sk);
  } else if (e.residual >= 2) {
    // S(x, y) = x2 x^2 + y2 y^2 + xy x y + cx x + cy y + c, 4 channels at a time:
    // ((x2 x + xy y + cx) x + (y2 y + cy) y + c
    const float* rc = pt + T.row_res * np;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      float k[6][4];
#pragma unroll
      for (int r = 0; r < 6; ++r) {
        const float4 f = lds4(rc + r * np + 4 * g);
        k[r][0] = f.x; k[r][1] = f.y; k[r][2] = f.z; k[r][3] = f.w;
      }
#pragma unroll
      for (int i = 0; i < 4; i += 2) {
        const int j = 4 * g + i;
        const float2 xv = e.residual == 2 ? f2(v + j) : f2(sk + j), yv = e.residual == 2 ? f2(sk + j) : f2(v + j);
        const float2 x2 = make_float2(k[0][i], k[0][i + 1]), y2 = make_float2(k[1][i], k[1][i + 1]);
        const float2 xy = make_float2(k[2][i], k[2][i + 1]), cx = make_float2(k[3][i], k[3][i + 1]);
        const float2 cy = make_float2(k[4][i], k[4][i + 1]), c0 = make_float2(k[5][i], k[5][i + 1]);
        const float2 ax = __ffma2_rn(x2, xv, __ffma2_rn(xy, yv, cx));
        const float2 ay = __ffma2_rn(y2, yv, cy);
        f2_put(v + j, __ffma2_rn(ax, xv, __ffma2_rn(ay, yv, c0)));
      }
    }
  }
  if (e.poly_deg) {
    const float* pc = pt + T.row_poly * np;
    float h[16], ck[16];
    lds16(pc + e.poly_deg * np, h);
    for (int k = e.poly_deg - 1; k >= 0; --k) {
      lds16(pc + k * np, ck);
#pragma unroll
      for (int j = 0; j < 16; j += 2) f2_put(h + j, __ffma2_rn(f2(h + j), f2(v + j), f2(ck + j)));
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = h[j];
  }
  if (chb + 16 > e.cout) {  // padded channels stay zero
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (chb + j >= e.cout) v[j] = 0.f;
  }
}

// epi_point16 for 8 channels (chb % 8 == 0): the block kernel's half items
__device__ __forceinline__ void epi_point8(const EpiParams& e, const EpiTab& T, float* v, float vscale,
                                           const float* sk, int chb) {
  const float* pt = T.ptab + chb;
  const int np = e.npad;
  float c[8];
  {
    const float4 f0 = lds4(pt), f1 = lds4(pt + 4);
    c[0] = f0.x; c[1] = f0.y; c[2] = f0.z; c[3] = f0.w; c[4] = f1.x; c[5] = f1.y; c[6] = f1.z; c[7] = f1.w;
  }
  fma_n<8>(v, vscale, c);
  if (T.row_aff >= 0) {
    float sc[8], sh[8];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const float4 a = lds4(pt + T.row_aff * np + 4 * q), d = lds4(pt + (T.row_aff + 1) * np + 4 * q);
      sc[4 * q] = a.x; sc[4 * q + 1] = a.y; sc[4 * q + 2] = a.z; sc[4 * q + 3] = a.w;
      sh[4 * q] = d.x; sh[4 * q + 1] = d.y; sh[4 * q + 2] = d.z; sh[4 * q + 3] = d.w;
    }
    fma_n<8>(v, sc, sh);
  }
  if (e.residual == 1) {
    add_n<8>(v, sk);
  } else if (e.residual >= 2) {
    const float* rc = pt + T.row_res * np;
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      float k[6][4];
#pragma unroll
      for (int r = 0; r < 6; ++r) {
        const float4 f = lds4(rc + r * np + 4 * g);
        k[r][0] = f.x; k[r][1] = f.y; k[r][2] = f.z; k[r][3] = f.w;
      }
#pragma unroll
      for (int i = 0; i < 4; i += 2) {
        const int j = 4 * g + i;
        const float2 xv = e.residual == 2 ? f2(v + j) : f2(sk + j), yv = e.residual == 2 ? f2(sk + j) : f2(v + j);
        const float2 x2 = make_float2(k[0][i], k[0][i + 1]), y2 = make_float2(k[1][i], k[1][i + 1]);
        const float2 xy = make_float2(k[2][i], k[2][i + 1]), cx = make_float2(k[3][i], k[3][i + 1]);
        const float2 cy = make_float2(k[4][i], k[4][i + 1]), c0 = make_float2(k[5][i], k[5][i + 1]);
        const float2 ax = __ffma2_rn(x2, xv, __ffma2_rn(xy, yv, cx));
        const float2 ay = __ffma2_rn(y2, yv, cy);
        f2_put(v + j, __ffma2_rn(ax, xv, __ffma2_rn(ay, yv, c0)));
      }
    }
  }
  if (e.poly_deg) {
    const float* pc = pt + T.row_poly * np;
    float h[8], ck[8];
    {
      const float4 f0 = lds4(pc + e.poly_deg * np), f1 = lds4(pc + e.poly_deg * np + 4);
      h[0] = f0.x; h[1] = f0.y; h[2] = f0.z; h[3] = f0.w; h[4] = f1.x; h[5] = f1.y; h[6] = f1.z; h[7] = f1.w;
    }
    for (int k = e.poly_deg - 1; k >= 0; --k) {
      const float4 f0 = lds4(pc + k * np), f1 = lds4(pc + k * np + 4);
      ck[0] = f0.x; ck[1] = f0.y; ck[2] = f0.z; ck[3] = f0.w; ck[4] = f1.x; ck[5] = f1.y; ck[6] = f1.z; ck[7] = f1.w;
#pragma unroll
      for (int j = 0; j < 8; j += 2) f2_put(h + j, __ffma2_rn(f2(h + j), f2(v + j), f2(ck + j)));
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = h[j];
  }
  if (chb + 8 > e.cout) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (chb + j >= e.cout) v[j] = 0.f;
  }
}

// PCNN_POOL_NONE: the 16 channels are contiguous (cb >= 16).  opos >= 0:
// the output is a split tensor whose row starts at half index opos (+
// channel-group terms), so no (b, y, x) addressing is needed; then ostore is
// its storage scale (1 when folded into the table, epi_fill_tab)
__device__ __forceinline__ void epi_store16(const EpiParams& e, const float* v, int chb, bool valid, int b, int oy,
                                            int ox, int64_t opos, float ostore) {
  if (!valid) return;
  if (opos >= 0) store16_split_at(e.out, (int64_t)(chb >> 3) * e.out.kstride + opos, v, ostore);
  else store16_any(e.out, b, chb, oy, ox, v);
}

// SUM2 / BI2 in WINDOW order: lanes 4q..4q+3 hold the (dy, dx) = 00, 01, 10,
// 11 pixels of window q.  Lane 4q+j pools channels [4j, 4j+4) of window q,
// so all 32 lanes work: gather those 4 channels of the 4 pixels by shuffles.
__device__ __forceinline__ void epi_window16(const EpiParams& e, float* v, int chb, bool valid, int b, int oy,
                                             int ox, int lane) {
  if (!valid) {
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = 0.f;
  }
  const int j4 = lane & 3, src = lane & ~3;
  float4 px[4];
#pragma unroll
  for (int pix = 0; pix < 4; ++pix) {
    float4 mine = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const float a0 = __shfl_sync(0xffffffffu, v[4 * g], src + pix);
      const float a1 = __shfl_sync(0xffffffffu, v[4 * g + 1], src + pix);
      const float a2 = __shfl_sync(0xffffffffu, v[4 * g + 2], src + pix);
      const float a3 = __shfl_sync(0xffffffffu, v[4 * g + 3], src + pix);
      if (g == j4) mine = make_float4(a0, a1, a2, a3);
    }
    px[pix] = mine;
  }
  const int ch0 = chb + 4 * j4;
  float4 r;
  if (e.pool == PCNN_POOL_SUM2) {
    const float dv = __ldg(e.pool_p);
    r = make_float4((px[0].x + px[1].x + px[2].x + px[3].x) * dv, (px[0].y + px[1].y + px[2].y + px[3].y) * dv,
                    (px[0].z + px[1].z + px[2].z + px[3].z) * dv, (px[0].w + px[1].w + px[2].w + px[3].w) * dv);
  } else {
    // bivariate tree: stage 1 pairs along the first axis, stage 2 across
    const int64_t nc = (int64_t)(e.pool_deg + 1) * (e.pool_deg + 1) * e.npad;
    const float* s1 = e.pool_p;
    const float* s2 = e.pool_p + nc;
    float4 u, w;
    if (e.pool_order == 0) {  // w first: S1(q0,q1), S1(q2,q3) then S2 along h
      u = bivariate4(s1, e.npad, e.pool_deg, ch0, px[0], px[1]);
      w = bivariate4(s1, e.npad, e.pool_deg, ch0, px[2], px[3]);
    } else {                  // h first: S1(q0,q2), S1(q1,q3) then S2 along w
      u = bivariate4(s1, e.npad, e.pool_deg, ch0, px[0], px[2]);
      w = bivariate4(s1, e.npad, e.pool_deg, ch0, px[1], px[3]);
    }
    r = bivariate4(s2, e.npad, e.pool_deg, ch0, u, w);
  }
  // padded channels (>= cout) stay zero; rows past M are not stored
  if (ch0 + 0 >= e.cout) r.x = 0.f;
  if (ch0 + 1 >= e.cout) r.y = 0.f;
  if (ch0 + 2 >= e.cout) r.z = 0.f;
  if (ch0 + 3 >= e.cout) r.w = 0.f;
  if (valid) store4_any(e.out, b, ch0, oy >> 1, ox >> 1, r.x, r.y, r.z, r.w);
}

// GLOBAL: a warp's 32 rows belong to at most two images unless the images
// are tiny.  The 16 channels x 2 images are reduced over the 32 lanes by a
// transposing butterfly (31 shuffles): afterwards lane L holds the sum of
// image lo_b + L / 16, channel chb + L % 16, and all lanes add at once.
__device__ __forceinline__ void epi_global16(const EpiParams& e, const float* v, int chb, bool valid, int b,
                                             int lane) {
  const float div = __ldg(e.pool_p);
  const int lo_b = (int)__reduce_min_sync(0xffffffffu, valid ? (unsigned)b : 0x7fffffffu);
  const int hi_b = (int)__reduce_max_sync(0xffffffffu, valid ? (unsigned)b : 0u);
  if (lo_b == 0x7fffffff) return;  // no valid row in this warp
  if (hi_b - lo_b <= 1) {
    float x[32];
    const bool first = !valid || b == lo_b;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float t = valid ? v[j] * div : 0.f;
      x[j] = first ? t : 0.f;
      x[16 + j] = first ? 0.f : t;
    }
    butterfly_step<16>(x, lane);
    butterfly_step<8>(x, lane);
    butterfly_step<4>(x, lane);
    butterfly_step<2>(x, lane);
    butterfly_step<1>(x, lane);
    const int ch = chb + (lane & 15);
    if (ch < e.cout && (lane < 16 || hi_b != lo_b)) atomicAdd(e.out.base + (int64_t)(lo_b + (lane >> 4)) * e.npad + ch, x[0]);
    return;
  }
#pragma unroll
  for (int j = 0; j < 16; ++j)
    if (valid && chb + j < e.cout) atomicAdd(e.out.base + (int64_t)b * e.npad + chb + j, v[j] * div);
}

// the whole epilogue, pool kind chosen at run time; WINDOW = false drops the
// 2x2 window pools (the halo-tile kernel never runs them: a shorter loop body)
template <bool WINDOW = true>
__device__ __forceinline__ void epi_chunk16(const EpiParams& e, const EpiTab& T, float* v, float vscale,
                                            const float* sk, int chb, bool valid, int b, int oy, int ox, int lane,
                                            int64_t opos = -1, float ostore = 1.f) {
  epi_point16(e, T, v, vscale, sk, chb);
  if (e.pool == PCNN_POOL_NONE) epi_store16(e, v, chb, valid, b, oy, ox, opos, ostore);
  else if (!WINDOW || e.pool == PCNN_POOL_GLOBAL) epi_global16(e, v, chb, valid, b, lane);
  else epi_window16(e, v, chb, valid, b, oy, ox, lane);
}

}  // namespace pcnn
