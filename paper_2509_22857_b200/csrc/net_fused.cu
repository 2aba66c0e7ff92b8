// Whole-network kernel for small sequential poly CNNs (LeNet-5-shaped):
// ONE launch runs ingest -> every conv / pool / dense unit -> logits, each
// CTA taking whole images with all of an image's activations in shared
// memory.  The reference evaluates such a network node by node per image
// (levnet graph.py:413-426 reference_eval, node kernels graph.py:361-410).
// At LeNet's size (0.28 M MACs per image) a layer-per-launch forward is bound
// by latency -- launches, and dependent weight loads missing L1 -- not by
// arithmetic, so here every parameter of the network (182 KB for LeNet) is
// staged into shared memory once per CTA with all loads in flight, and the
// units run back to back with block barriers between them.
//
// Arithmetic: plain fp32 FMA (CUDA cores), accumulation in the reference's
// (c_in, ky, kx) order; the fused epilogue follows epilogue.cuh's epi_point /
// epi_pool4 (bias -> affine -> polynomial, then SUM2 / bivariate 2x2 / local
// k x k / global sum pools).  Activations: dense CHW per image, the order the
// reference's flatten (C-major) reads.
#include "kernels.cuh"
#include "tc_ptx.cuh"

namespace pcnn {
namespace {

// the CTA's shared memory: parameters and activations at float offsets
extern __shared__ __align__(16) float nsm[];

// Horner / bivariate over shared-memory coefficient rows at float offset
// `coef` (common.cuh's horner / bivariate read global memory)
__device__ __forceinline__ float horner_s(int coef, int stride, int deg, int ch, float x) {
  if (deg == 2)  // the common degree, unrolled
    return fmaf(fmaf(nsm[coef + 2 * stride + ch], x, nsm[coef + stride + ch]), x, nsm[coef + ch]);
  float acc = nsm[coef + deg * stride + ch];
  for (int k = deg - 1; k >= 0; --k) acc = fmaf(acc, x, nsm[coef + k * stride + ch]);
  return acc;
}

__device__ __forceinline__ float bivariate_s(int coef, int stride, int d, int ch, float x, float y) {
  float acc = 0.f;
  for (int i = d; i >= 0; --i) {
    const int row = coef + i * (d + 1) * stride + ch;
    float r = nsm[row + (d - i) * stride];
    for (int j = d - i - 1; j >= 0; --j) r = fmaf(r, y, nsm[row + j * stride]);
    acc = (i == d) ? r : fmaf(acc, x, r);
  }
  return acc;
}

__device__ __forceinline__ float net_point(const NetOp& o, float acc, int ch) {
  const int aff = o.aff, deg = o.poly_deg;
  float v = acc + nsm[o.bias + ch];
  if (aff >= 0) v = fmaf(v, nsm[aff + ch], nsm[aff + o.npad + ch]);
  if (deg) v = horner_s(o.poly, o.poly_stride, deg, ch, v);
  return v;
}

__device__ __forceinline__ float net_pool4(const NetOp& o, int ch, float q0, float q1, float q2, float q3) {
  if (o.pool == PCNN_POOL_SUM2) return (q0 + q1 + q2 + q3) * nsm[o.pool_p];
  const int s1 = o.pool_p, s2 = s1 + (o.pool_deg + 1) * (o.pool_deg + 1) * o.npad;
  float u, w;
  if (o.pool_order == 0) {
    u = bivariate_s(s1, o.npad, o.pool_deg, ch, q0, q1);
    w = bivariate_s(s1, o.npad, o.pool_deg, ch, q2, q3);
  } else {
    u = bivariate_s(s1, o.npad, o.pool_deg, ch, q0, q2);
    w = bivariate_s(s1, o.npad, o.pool_deg, ch, q1, q3);
  }
  return bivariate_s(s2, o.npad, o.pool_deg, ch, u, w);
}

// conv unit: CPI output channels at one output position per work item (each
// input value loaded once for the CPI channels), positions fastest so a warp
// reads the same weights (shared-memory broadcast); o is a register copy
template <int CPI>
__device__ __forceinline__ void net_conv(const NetOp& o, int out) {
  // every field the loops use in a register (o lives in kernel parameter space)
  const int c = o.c, h = o.h, w = o.w, co = o.co, wo = o.wo, kh = o.kh, kw = o.kw, cb = o.cb, kp = o.kp;
  const int stride = o.stride, pad = o.pad, wt = o.wt, in_off = o.in_off;
  const int hwo = o.ho * wo, ngrp = (co + CPI - 1) / CPI, taps_cb = kh * kw * cb;
  const int items = ngrp * hwo;
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int grp = it / hwo, pos = it - grp * hwo;
    const int oy = pos / wo, ox = pos - oy * wo;
    const int c0 = grp * CPI;
    const int nch = co - c0 < CPI ? co - c0 : CPI;
    // rows past the last channel repeat the last one (their sums are dropped)
    int row[CPI];
#pragma unroll
    for (int j = 0; j < CPI; ++j) row[j] = wt + (c0 + (j < nch ? j : nch - 1)) * kp;
    float acc[CPI];
#pragma unroll
    for (int j = 0; j < CPI; ++j) acc[j] = 0.f;
    const int iy0 = oy * stride - pad, ix0 = ox * stride - pad;
    const int ky0 = iy0 < 0 ? -iy0 : 0, ky1 = h - iy0 < kh ? h - iy0 : kh;
    const int kx0 = ix0 < 0 ? -ix0 : 0, kx1 = w - ix0 < kw ? w - ix0 : kw;
    for (int ci = 0; ci < c; ++ci) {
      const int ip = in_off + (ci * h + iy0) * w + ix0;
      const int wc = (ci / cb) * taps_cb + (ci % cb);
      for (int ky = ky0; ky < ky1; ++ky) {
        const int ir = ip + ky * w;
        const int wr = wc + ky * kw * cb;
#pragma unroll 5
        for (int kx = kx0; kx < kx1; ++kx) {
          const float xv = nsm[ir + kx];
#pragma unroll
          for (int j = 0; j < CPI; ++j) acc[j] = fmaf(xv, nsm[row[j] + wr + kx * cb], acc[j]);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < CPI; ++j)
      if (j < nch) nsm[out + (c0 + j) * hwo + pos] = net_point(o, acc[j], c0 + j);
  }
}

// net_conv for a compile-time kernel size and channel block: every tap's
// weight offset is an immediate, out-of-image taps are predicated to zero
template <int CPI, int K, int CB>
__device__ __forceinline__ void net_conv_k(const NetOp& o, int out) {
  const int c = o.c, h = o.h, w = o.w, co = o.co, wo = o.wo, kp = o.kp;
  const int stride = o.stride, pad = o.pad, wt = o.wt, in_off = o.in_off;
  const int hwo = o.ho * wo, ngrp = (co + CPI - 1) / CPI;
  const int items = ngrp * hwo;
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int grp = it / hwo, pos = it - grp * hwo;
    const int oy = pos / wo, ox = pos - oy * wo;
    const int c0 = grp * CPI;
    const int nch = co - c0 < CPI ? co - c0 : CPI;
    int row[CPI];
#pragma unroll
    for (int j = 0; j < CPI; ++j) row[j] = wt + (c0 + (j < nch ? j : nch - 1)) * kp;
    float acc[CPI];
#pragma unroll
    for (int j = 0; j < CPI; ++j) acc[j] = 0.f;
    const int iy0 = oy * stride - pad, ix0 = ox * stride - pad;
    bool oky[K], okx[K];
#pragma unroll
    for (int t = 0; t < K; ++t) {
      oky[t] = (unsigned)(iy0 + t) < (unsigned)h;
      okx[t] = (unsigned)(ix0 + t) < (unsigned)w;
    }
    for (int ci = 0; ci < c; ++ci) {
      const int ip = in_off + (ci * h + iy0) * w + ix0;
      const int wc = (ci / CB) * (K * K * CB) + (ci % CB);
#pragma unroll
      for (int ky = 0; ky < K; ++ky) {
#pragma unroll
        for (int kx = 0; kx < K; ++kx) {
          const float xv = (oky[ky] && okx[kx]) ? nsm[ip + ky * w + kx] : 0.f;
#pragma unroll
          for (int j = 0; j < CPI; ++j) acc[j] = fmaf(xv, nsm[row[j] + wc + (ky * K + kx) * CB], acc[j]);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < CPI; ++j)
      if (j < nch) nsm[out + (c0 + j) * hwo + pos] = net_point(o, acc[j], c0 + j);
  }
}

template <int CPI>
__device__ __forceinline__ void net_conv_any(const NetOp& o, int out) {
  if (o.kh == 5 && o.kw == 5 && o.cb == 4) net_conv_k<CPI, 5, 4>(o, out);
  else if (o.kh == 5 && o.kw == 5 && o.cb == 8) net_conv_k<CPI, 5, 8>(o, out);
  else if (o.kh == 3 && o.kw == 3 && o.cb == 8) net_conv_k<CPI, 3, 8>(o, out);
  else if (o.kh == 3 && o.kw == 3 && o.cb == 16) net_conv_k<CPI, 3, 16>(o, out);
  else net_conv<CPI>(o, out);
}

// pooling of the unpooled conv map at `in` (co x ho x wo) into `out`
__device__ __forceinline__ void net_pool(const NetOp& o, int in, int out) {
  const int hwo = o.ho * o.wo;
  if (o.pool == PCNN_POOL_GLOBAL) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const float div = nsm[o.pool_p];
    for (int ch = warp; ch < o.co; ch += nw) {
      float s = 0.f;
      for (int q = lane; q < hwo; q += 32) s += nsm[in + ch * hwo + q];
#pragma unroll
      for (int d = 16; d; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
      if (lane == 0) nsm[out + ch] = s * div;
    }
    return;
  }
  const int n = o.co * o.ph * o.pw;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int ch = i / (o.ph * o.pw), r = i - ch * (o.ph * o.pw);
    const int py = r / o.pw, px = r - py * o.pw;
    const int p = in + ch * hwo;
    float v;
    if (o.pool == PCNN_POOL_LOCAL) {
      float s = 0.f;
      for (int dy = 0; dy < o.pool_k; ++dy) {
        const int y = py * o.pool_s - o.pool_pad + dy;
        if (y < 0 || y >= o.ho) continue;
        for (int dx = 0; dx < o.pool_k; ++dx) {
          const int x = px * o.pool_s - o.pool_pad + dx;
          if (x >= 0 && x < o.wo) s += nsm[p + y * o.wo + x];
        }
      }
      v = s * nsm[o.pool_p];
    } else {
      const int q = p + 2 * py * o.wo + 2 * px;
      v = net_pool4(o, ch, nsm[q], nsm[q + 1], nsm[q + o.wo], nsm[q + o.wo + 1]);
    }
    nsm[out + i] = v;
  }
}

// dense unit: one warp per output, lanes over the inputs
__device__ __forceinline__ void net_linear(const NetOp& o) {
  int x = o.in_off;
  if (o.in_mode == 2) {
    // global-sum view of a spatial input (c x hw)
    const int hw = o.h * o.w;
    const float div = o.in_div >= 0 ? nsm[o.in_div] : 1.f;
    for (int j = threadIdx.x; j < o.n_in; j += blockDim.x) {
      float s = 0.f;
      for (int q = 0; q < hw; ++q) s += nsm[o.in_off + j * hw + q];
      nsm[o.scratch_off + j] = s * div;
    }
    __syncthreads();
    x = o.scratch_off;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int k = warp; k < o.n_out; k += nw) {
    const int wr = o.wt + k * o.n_in;
    float acc = 0.f;
#pragma unroll 4
    for (int j = lane; j < o.n_in; j += 32) acc = fmaf(nsm[wr + j], nsm[x + j], acc);
#pragma unroll
    for (int d = 16; d; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
    if (lane == 0) {
      float v = acc + nsm[o.bias + k];
      if (o.poly_deg) v = horner_s(o.poly, o.poly_stride, o.poly_deg, k, v);
      nsm[o.out_off + k] = v;
    }
  }
}

__global__ void __launch_bounds__(kNetThreads) net_kernel(const __grid_constant__ NetParams P) {
  __shared__ __align__(8) uint64_t bars[kNetMaxOps];
  tl_mark(P.tl, 0);
  // every parameter block into shared memory by bulk copies, one mbarrier per
  // op: op k waits (first image only) for its own blocks, so the big dense
  // weights stream in while the convolutions compute.  Whole 16-byte units
  // are bulk-copied; a block's last n % 4 floats are loaded by threads.
  if (threadIdx.x == 0) {
    for (int k = 0; k < P.nops; ++k) ptx::mbar_init(ptx::smem_u32(&bars[k]), 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0)
      for (int k = 0; k < P.nops; ++k) {
        uint32_t bytes = 0;
        for (int c = 0; c < P.ncopies; ++c)
          if (P.cp[c].op == k) bytes += (uint32_t)(P.cp[c].n & ~3) * 4u;
        ptx::mbar_arrive_tx(ptx::smem_u32(&bars[k]), bytes);
      }
    __syncwarp();
    for (int c = threadIdx.x; c < P.ncopies; c += 32) {
      const NetCopy& cp = P.cp[c];
      if (cp.n >= 4)
        ptx::bulk_g2s(ptx::smem_u32(nsm + cp.dst), cp.src, (uint32_t)(cp.n & ~3) * 4u, ptx::smem_u32(&bars[cp.op]));
    }
  }
  // the last n % 4 floats of every block (ordered before their readers by
  // the barrier after the first image's ingest)
  if (threadIdx.x < 4 * P.ncopies) {
    const NetCopy& cp = P.cp[threadIdx.x >> 2];
    const int j = (cp.n & ~3) + (threadIdx.x & 3);
    if (j < cp.n) nsm[cp.dst + j] = __ldg(cp.src + j);
  }
  bool first = true;
  for (int b = blockIdx.x; b < P.batch; b += gridDim.x) {
    {
      const float* x = P.x + (int64_t)b * P.in_elems;
      for (int i = threadIdx.x; i < P.in_elems; i += blockDim.x) nsm[P.act_off + i] = __ldg(x + i);
    }
    __syncthreads();
    for (int k = 0; k < P.nops; ++k) {
      const NetOp& o = P.op[k];
      if (first) {
        ptx::mbar_wait(ptx::smem_u32(&bars[k]), 0);
        __syncthreads();
      }
      if (o.kind == kNetConv) {
        const int dst = o.pool ? o.scratch_off : o.out_off;
        if (o.cpi == 4) net_conv_any<4>(o, dst);
        else if (o.cpi == 2) net_conv_any<2>(o, dst);
        else net_conv_any<1>(o, dst);
        if (o.pool) {
          __syncthreads();
          net_pool(o, o.scratch_off, o.out_off);
        }
      } else {
        net_linear(o);
      }
      __syncthreads();
    }
    first = false;
    // logits to the user buffer and the plan's output tensor
    for (int i = threadIdx.x; i < P.out_pad; i += blockDim.x) {
      const float v = i < P.n_out ? nsm[P.out_off + i] : 0.f;
      if (i < P.n_out && P.logits) P.logits[(int64_t)b * P.n_out + i] = v;
      if (P.out_ws) P.out_ws[(int64_t)b * P.out_pad + i] = v;
    }
    __syncthreads();
  }
  if (P.tl) {
    __syncthreads();
    tl_mark(P.tl, 1);
  }
}

}  // namespace

void net_launch(const NetParams& P, cudaStream_t s, int grid) {
  const size_t smem = sizeof(float) * (size_t)P.smem_floats;
  if (smem > 48 * 1024) cudaFuncSetAttribute(net_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  net_kernel<<<grid, kNetThreads, smem, s>>>(P);
}

}  // namespace pcnn
