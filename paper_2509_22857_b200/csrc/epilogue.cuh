// Fused conv epilogue shared by the SIMT and tcgen05 conv kernels:
//   v = acc + bias -> [affine] -> [residual: + skip | S(v, skip)] -> [poly]
//   -> [pool: 2x2 sum | 2x2 bivariate tree | global sum] -> store.
#pragma once

#include "common.cuh"

namespace pcnn {

struct EpiParams {
  const float* bias;      // [Npad]
  const float* aff;       // scale [Npad], shift [Npad] or null
  int residual;           // 0, 1 add, 2 S(v, skip), 3 S(skip, v)
  const float* res;       // polyskip coeffs [6][Npad]
  int poly_deg;           // 0 = none
  const float* poly;      // [(deg+1)][Npad]
  int pool;               // pcnn_pool_kind
  const float* pool_p;    // divisor or bivariate coeffs
  int pool_deg, pool_order;
  int pool_k, pool_s, pool_pad;  // POOL_LOCAL window
  int npad, cout;         // padded / logical output channels
  TensorView skip;        // residual input (same geometry as the conv output)
  TensorView out;         // output tensor (pooled or vector for GLOBAL)
};

// Per-element part before pooling: bias, affine, residual, poly.
__device__ __forceinline__ float epi_point(const EpiParams& e, float acc, int b, int oy, int ox,
                                           int ch) {
  float v = acc + __ldg(e.bias + ch);
  if (e.aff) v = fmaf(v, __ldg(e.aff + ch), __ldg(e.aff + e.npad + ch));
  if (e.residual) {
    float s = *e.skip.at(b, ch, oy, ox);
    v = (e.residual == 1) ? v + s
        : (e.residual == 2 ? polyskip(e.res, e.npad, ch, v, s) : polyskip(e.res, e.npad, ch, s, v));
  }
  if (e.poly_deg) v = horner(e.poly, e.npad, e.poly_deg, ch, v);
  return v;
}

// Reduce the four values of a 2x2 window given in (dy, dx) order
// q0=(0,0) q1=(0,1) q2=(1,0) q3=(1,1).
__device__ __forceinline__ float epi_pool4(const EpiParams& e, int ch, float q0, float q1, float q2,
                                           float q3) {
  if (e.pool == PCNN_POOL_SUM2) return (q0 + q1 + q2 + q3) * __ldg(e.pool_p);
  // bivariate tree: stage-1 pairs along the first axis, stage-2 across
  const int64_t nc = (int64_t)(e.pool_deg + 1) * (e.pool_deg + 1) * e.npad;
  const float* s1 = e.pool_p;
  const float* s2 = e.pool_p + nc;
  float u, w;
  if (e.pool_order == 0) {  // w first: S1(q0,q1), S1(q2,q3) then S2 along h
    u = bivariate(s1, e.npad, e.pool_deg, ch, q0, q1);
    w = bivariate(s1, e.npad, e.pool_deg, ch, q2, q3);
  } else {                  // h first: S1(q0,q2), S1(q1,q3) then S2 along w
    u = bivariate(s1, e.npad, e.pool_deg, ch, q0, q2);
    w = bivariate(s1, e.npad, e.pool_deg, ch, q1, q3);
  }
  return bivariate(s2, e.npad, e.pool_deg, ch, u, w);
}

}  // namespace pcnn
