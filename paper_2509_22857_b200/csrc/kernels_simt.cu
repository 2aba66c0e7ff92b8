// SIMT float32 kernels: input ingest, implicit-GEMM conv with the fused
// epilogue (used for small/odd layers and as the tcgen05 cross-check), the
// dense layer, and standalone elementwise/pool kernels so every node kind of
// the graph IR runs on the GPU even when it is not fused.
#include "kernels.cuh"
#include "tc_ptx.cuh"

namespace pcnn {

// ---------------------------------------------------------------------------
// ingest: user NCHW float32 -> channel-blocked [B][nblk][H][W][cb], pad = 0
// ---------------------------------------------------------------------------
__global__ void ingest_kernel(const float* __restrict__ x, TensorView t, int batch, int s2d,
                              unsigned long long* tl) {
  TlScope tls(tl);
  // one thread per (image, 4-channel group, pixel); pixels fastest so the
  // NCHW reads of each channel plane are coalesced, one float4 store each
  const int64_t hw = (int64_t)t.h * t.w;
  const int groups = t.cpad() / 4;
  const int64_t total = (int64_t)batch * groups * hw;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i % hw;
    const int64_t r = i / hw;
    const int g = (int)(r % groups), b = (int)(r / groups);
    const int y = (int)(p / t.w), xw = (int)(p - (int64_t)y * t.w);
    float v[4];
    if (s2d) {
      // channel ch = (dy*2 + dx)*cin + c of block (y, xw) = pixel (2(y-1)+dy,
      // 2(xw-1)+dx); block row 0 and column 0 are zero
      const int cin = t.c / 4, H = 2 * (t.h - 1), W = 2 * (t.w - 1);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int ch = g * 4 + j;
        const int q = ch / cin, c = ch - q * cin;
        v[j] = (ch < t.c && y > 0 && xw > 0)
                   ? __ldg(x + (((int64_t)b * cin + c) * H + 2 * (y - 1) + (q >> 1)) * W + 2 * (xw - 1) + (q & 1))
                   : 0.f;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int ch = g * 4 + j;
        v[j] = ch < t.c ? __ldg(x + ((int64_t)b * t.c + ch) * hw + p) : 0.f;
      }
    }
    store4_any(t, b, g * 4, y, xw, v[0], v[1], v[2], v[3]);
  }
}

// space-to-depth ingest, one thread per block position and all 16 channels:
// per input channel two float2 row reads (coalesced across the warp), one
// 16-channel store (whole 32-byte sectors in the split layout)
// CIN > 0: the channel count at compile time, so v[] stays in registers
// (a runtime channel loop indexes it dynamically: local memory, measured
// 1.4 TB/s on RN18's 38.5 MB input)
template <int CIN>
__global__ void ingest_s2d_kernel(const float* __restrict__ x, TensorView t, int batch, unsigned long long* tl) {
  TlScope tls(tl);
  const int cin = CIN > 0 ? CIN : t.c / 4, H = 2 * (t.h - 1), W = 2 * (t.w - 1);
  const int64_t hw = (int64_t)t.h * t.w;
  const int64_t total = (int64_t)batch * hw;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(i / hw);
    const int64_t p = i - (int64_t)b * hw;
    const int y = (int)(p / t.w), xw = (int)(p - (int64_t)y * t.w);
    float v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = 0.f;
    if (y > 0 && xw > 0) {
#pragma unroll
      for (int c = 0; c < (CIN > 0 ? CIN : 4); ++c) {
        if (CIN == 0 && c >= cin) break;
#pragma unroll
        for (int dy = 0; dy < 2; ++dy) {
          const float2 f = __ldg(reinterpret_cast<const float2*>(
              x + (((int64_t)b * cin + c) * H + 2 * (y - 1) + dy) * W + 2 * (xw - 1)));
          v[(dy * 2) * cin + c] = f.x;       // (dy, dx = 0)
          v[(dy * 2 + 1) * cin + c] = f.y;   // (dy, dx = 1)
        }
      }
    }
    if (CIN > 0 || (t.cpad() >= 16 && (t.cb >= 16 || t.split))) {
      store16_any(t, b, 0, y, xw, v);  // CIN > 0: launched only for this layout
    } else {
      for (int g = 0; g < t.cpad() / 4; ++g) store4_any(t, b, 4 * g, y, xw, v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
    }
  }
}

void launch_ingest(const float* x, const TensorView& t, int batch, bool s2d, cudaStream_t s, int pdl,
                   unsigned long long* tl) {
  if (s2d && t.c <= 16 && (2 * (t.w - 1)) % 2 == 0) {
    const int64_t total = (int64_t)batch * t.h * t.w;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    if (t.c == 12 && t.cpad() >= 16 && (t.cb >= 16 || t.split)) launch_pdl(ingest_s2d_kernel<3>, std::max(blocks, 1), 256, 0, s, pdl, x, t, batch, tl);
    else launch_pdl(ingest_s2d_kernel<0>, std::max(blocks, 1), 256, 0, s, pdl, x, t, batch, tl);
    return;
  }
  int64_t total = (int64_t)batch * (t.cpad() / 4) * t.h * t.w;
  int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  launch_pdl(ingest_kernel, std::max(blocks, 1), 256, 0, s, pdl, x, t, batch, s2d ? 1 : 0, tl);
}

// ---------------------------------------------------------------------------
// SIMT implicit-GEMM conv.  Tile BM pixels x BN channels, 256 threads, each
// thread 4 consecutive pixel rows x 4 consecutive channels, K staged by 16.
// ---------------------------------------------------------------------------
template <int BN>
__global__ void __launch_bounds__(256) conv_simt_kernel(ConvArgs a) {
  TlScope tls(a.tl);
  constexpr int TN = 4, TM = 4, BK = 16;
  constexpr int NTX = BN / TN;          // threads along N
  constexpr int NTY = 256 / NTX;        // threads along M
  constexpr int BM = NTY * TM;
  __shared__ __align__(16) float As[BK][BM];
  __shared__ __align__(16) float Bs[BK][BN];
  __shared__ int pb[BM], piy[BM], pix_[BM];
  __shared__ int kky[BK], kkx[BK];
  __shared__ int64_t koff[BK];

  const int tid = threadIdx.x;
  const int tx = tid % NTX, ty = tid / NTX;
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;
  const TensorView& in = a.in;
  const int64_t M = a.pm.count(a.batch);
  const int KP = a.kp;

  for (int i = tid; i < BM; i += 256) {
    int64_t m = m0 + i;
    int b = -1, oy = 0, ox = 0;
    if (m < M) a.pm.decode(m, b, oy, ox);
    pb[i] = b;
    piy[i] = oy * a.stride - a.pad;
    pix_[i] = ox * a.stride - a.pad;
  }
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;

  const int64_t plane = (int64_t)in.h * in.w * in.cb;
  const int taps_cb = a.kh * a.kw * in.cb;
  for (int k0 = 0; k0 < KP; k0 += BK) {
    __syncthreads();
    if (tid < BK) {
      int k = k0 + tid;
      if (k < KP) {
        int blk = k / taps_cb;
        int r = k - blk * taps_cb;
        int tap = r / in.cb, ci = r - tap * in.cb;
        int ky = tap / a.kw, kx = tap - ky * a.kw;
        kky[tid] = ky;
        kkx[tid] = kx;
        koff[tid] = blk * plane + ((int64_t)ky * in.w + kx) * in.cb + ci;
      } else {
        kky[tid] = -100000;
        kkx[tid] = 0;
        koff[tid] = 0;
      }
    }
    __syncthreads();
    // gather: issue every predicated load of this thread first, then store,
    // so the loads overlap instead of serialising on memory latency
    constexpr int PER = BK * BM / 256;
    float gv[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int e = tid + q * 256;
      const int kk = e / BM, mm = e - kk * BM;
      const int b = pb[mm];
      const int iy = piy[mm] + kky[kk], ix = pix_[mm] + kkx[kk];
      const bool ok = b >= 0 && iy >= 0 && iy < in.h && ix >= 0 && ix < in.w;
      const float* src = in.base + (int64_t)max(b, 0) * in.nblk * plane + koff[kk] +
                         ((int64_t)piy[mm] * in.w + pix_[mm]) * in.cb;
      gv[q] = ok ? __ldg(src) : 0.f;
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int e = tid + q * 256;
      As[e / BM][e % BM] = gv[q];
    }
    for (int e = tid; e < BK * BN; e += 256) {
      int nn = e / BK, kk = e - nn * BK;
      int n = n0 + nn, k = k0 + kk;
      Bs[kk][nn] = (n < a.npad && k < KP) ? __ldg(a.w + (int64_t)n * KP + k) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float4 av = *reinterpret_cast<const float4*>(&As[kk][ty * TM]);
      float4 bv = *reinterpret_cast<const float4*>(&Bs[kk][tx * TN]);
      float ar[4] = {av.x, av.y, av.z, av.w}, br[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(ar[i], br[j], acc[i][j]);
    }
  }

  // epilogue
  const EpiParams& e = a.epi;
  const int nb = n0 + tx * TN;
  if (nb >= a.npad) return;
  float v[TM][TN];
  int bs[TM], oys[TM], oxs[TM];
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    int64_t m = m0 + ty * TM + i;
    bs[i] = -1;
    if (m < M) a.pm.decode(m, bs[i], oys[i], oxs[i]);
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      int ch = nb + j;
      v[i][j] = (bs[i] >= 0 && ch < e.cout) ? epi_point(e, acc[i][j], bs[i], oys[i], oxs[i], ch) : 0.f;
    }
  }
  if (e.pool == PCNN_POOL_NONE) {
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      if (bs[i] < 0) continue;
      float4 o = make_float4(v[i][0], v[i][1], v[i][2], v[i][3]);
      *reinterpret_cast<float4*>(e.out.pix(bs[i], nb, oys[i], oxs[i])) = o;
    }
  } else if (e.pool == PCNN_POOL_GLOBAL) {
    const float div = __ldg(e.pool_p);
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      if (bs[i] < 0) continue;
#pragma unroll
      for (int j = 0; j < TN; ++j)
        if (nb + j < e.cout) atomicAdd(e.out.base + (int64_t)bs[i] * e.npad + nb + j, v[i][j] * div);
    }
  } else {
    // rows ty*4..ty*4+3 are one 2x2 window (WINDOW order, BM % 4 == 0)
    if (bs[0] < 0) return;
    float o[TN];
#pragma unroll
    for (int j = 0; j < TN; ++j)
      o[j] = (nb + j < e.cout) ? epi_pool4(e, nb + j, v[0][j], v[1][j], v[2][j], v[3][j]) : 0.f;
    *reinterpret_cast<float4*>(e.out.pix(bs[0], nb, oys[0] >> 1, oxs[0] >> 1)) =
        make_float4(o[0], o[1], o[2], o[3]);
  }
}

void launch_conv_simt(const ConvArgs& a, cudaStream_t s) {
  int64_t M = host_pixel_count(a.pm, a.batch);
  int bn = a.npad >= 64 ? 64 : (a.npad >= 32 ? 32 : (a.npad >= 16 ? 16 : 8));
  int bm = 4 * 256 / (bn / 4);
  dim3 grid((unsigned)((M + bm - 1) / bm), (unsigned)((a.npad + bn - 1) / bn));
  switch (bn) {
    case 64: conv_simt_kernel<64><<<grid, 256, 0, s>>>(a); break;
    case 32: conv_simt_kernel<32><<<grid, 256, 0, s>>>(a); break;
    case 16: conv_simt_kernel<16><<<grid, 256, 0, s>>>(a); break;
    default: conv_simt_kernel<8><<<grid, 256, 0, s>>>(a); break;
  }
}

// ---------------------------------------------------------------------------
// dense layer: out[b][k] = W[k] . view(b) + bias[k]  [-> poly]
// view: vector, flatten of a blocked spatial tensor (C-major), or global sum.
// Block = 16 outputs x 16 images (one thread each); the block's 16 weight
// rows and 16 input views are staged in shared memory with every thread's
// loads in flight at once (the layer is a few latency-bound round trips, not
// arithmetic: 512 -> 1000 for 64 images is 33 M MACs), then each thread runs
// its dot product from shared memory (rows padded by one float: the 16
// images a half-warp reads sit in different banks).
// ---------------------------------------------------------------------------
constexpr int kLinO = 16, kLinB = 16, kLinK = 1024;  // K staged in chunks of kLinK

__device__ __forceinline__ float linear_view(const LinearArgs& a, int b, int j, float div) {
  const TensorView& in = a.in;
  if (a.in_mode == 0) return __ldg(in.base + (int64_t)b * in.cpad() + j);
  const int hw = in.h * in.w;
  if (a.in_mode == 1) {
    const int c = j / hw, r = j - c * hw;
    return __ldg(in.at(b, c, r / in.w, r % in.w));
  }
  const float* p = in.at(b, j, 0, 0);
  float s = 0.f;
  for (int q = 0; q < hw; ++q) s += __ldg(p + (int64_t)q * in.cb);
  return s * div;
}

__global__ void __launch_bounds__(256) linear_kernel(LinearArgs a) {
  TlScope tls(a.tl);
  extern __shared__ __align__(16) float sm[];
  __shared__ __align__(8) uint64_t bar;
  const int n = a.n_in, kc = n < kLinK ? n : kLinK, ld = (kc + 4) & ~3;  // rows 16-byte aligned
  float* ws = sm;                 // [kLinO][ld]
  float* xs = sm + kLinO * ld;    // [kLinB][ld]
  const int o0 = blockIdx.x * kLinO, b0 = blockIdx.y * kLinB;
  const float div = a.in_div ? __ldg(a.in_div) : 1.f;
  // contiguous rows (vector input or a 1 x 1 flatten, whole K in one chunk,
  // 16-byte aligned rows): every weight row and input row is one bulk copy,
  // all in flight at once -- one memory round trip for the block
  const bool vec = a.in_mode == 0 || (a.in_mode == 1 && a.in.h * a.in.w == 1);
  const bool bulk = vec && kc == n && (n % 4) == 0 && (a.in.cpad() % 4) == 0 &&
                    ((reinterpret_cast<uintptr_t>(a.w) | reinterpret_cast<uintptr_t>(a.in.base)) & 15) == 0;
  // thread (output ko, image bi): bi fastest, so a warp is 2 outputs x 16 images
  const int bi = threadIdx.x & (kLinB - 1), ko = threadIdx.x >> 4;
  float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, acc3 = 0.f;
  if (bulk) {
    const int no = a.n_out - o0 < kLinO ? a.n_out - o0 : kLinO;
    const int nb = a.batch - b0 < kLinB ? a.batch - b0 : kLinB;
    if (threadIdx.x == 0) {
      ptx::mbar_init(ptx::smem_u32(&bar), 1);
      ptx::fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const uint32_t rb = (uint32_t)n * 4u;
      if (threadIdx.x == 0) ptx::mbar_arrive_tx(ptx::smem_u32(&bar), (uint32_t)((no > 0 ? no : 0) + nb) * rb);
      __syncwarp();
      const int r = threadIdx.x;
      if (r < kLinO && r < no)
        ptx::bulk_g2s(ptx::smem_u32(ws + r * ld), a.w + (int64_t)(o0 + r) * n, rb, ptx::smem_u32(&bar));
      else if (r >= kLinO && r - kLinO < nb)
        ptx::bulk_g2s(ptx::smem_u32(xs + (r - kLinO) * ld), a.in.base + (int64_t)(b0 + r - kLinO) * a.in.cpad(), rb,
                      ptx::smem_u32(&bar));
    }
    // rows past n_out / the batch: zeros
    for (int e = threadIdx.x; e < (kLinO - (no > 0 ? no : 0)) * ld; e += blockDim.x) ws[(no > 0 ? no : 0) * ld + e] = 0.f;
    for (int e = threadIdx.x; e < (kLinB - nb) * ld; e += blockDim.x) xs[nb * ld + e] = 0.f;
    ptx::mbar_wait(ptx::smem_u32(&bar), 0);
    __syncthreads();
    const float* wr = ws + ko * ld;
    const float* xr = xs + bi * ld;
    for (int j = 0; j + 4 <= n; j += 4) {
      const float4 w4 = *reinterpret_cast<const float4*>(wr + j), x4 = *reinterpret_cast<const float4*>(xr + j);
      acc0 = fmaf(w4.x, x4.x, acc0);
      acc1 = fmaf(w4.y, x4.y, acc1);
      acc2 = fmaf(w4.z, x4.z, acc2);
      acc3 = fmaf(w4.w, x4.w, acc3);
    }
  } else
  for (int k0 = 0; k0 < n; k0 += kc) {
    const int m = n - k0 < kc ? n - k0 : kc;
    if (k0) __syncthreads();
    // weights: rows o0 .. o0 + 15 (zero past n_out), eight loads in flight per thread
    for (int e0 = threadIdx.x; e0 < kLinO * m; e0 += 8 * blockDim.x) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * blockDim.x;
        const int r = e / m, j = e - r * m;
        v[u] = (e < kLinO * m && o0 + r < a.n_out) ? __ldg(a.w + (int64_t)(o0 + r) * n + k0 + j) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * blockDim.x;
        if (e < kLinO * m) ws[(e / m) * ld + e % m] = v[u];
      }
    }
    // inputs: images b0 .. b0 + 15 (zero past the batch)
    for (int e0 = threadIdx.x; e0 < kLinB * m; e0 += 8 * blockDim.x) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * blockDim.x;
        const int bb = e / m, j = e - bb * m;
        v[u] = (e < kLinB * m && b0 + bb < a.batch) ? linear_view(a, b0 + bb, k0 + j, div) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * blockDim.x;
        if (e < kLinB * m) xs[(e / m) * ld + e % m] = v[u];
      }
    }
    __syncthreads();
    const float* wr = ws + ko * ld;
    const float* xr = xs + bi * ld;
    int j = 0;
    for (; j + 4 <= m; j += 4) {
      acc0 = fmaf(wr[j], xr[j], acc0);
      acc1 = fmaf(wr[j + 1], xr[j + 1], acc1);
      acc2 = fmaf(wr[j + 2], xr[j + 2], acc2);
      acc3 = fmaf(wr[j + 3], xr[j + 3], acc3);
    }
    for (; j < m; ++j) acc0 = fmaf(wr[j], xr[j], acc0);
  }
  const int k = o0 + ko, b = b0 + bi;
  if (b >= a.batch || k >= a.out_stride) return;
  if (k >= a.n_out) {  // zero the padded channels
    a.out[(int64_t)b * a.out_stride + k] = 0.f;
    return;
  }
  float v = (acc0 + acc1) + (acc2 + acc3) + __ldg(a.bias + k);
  if (a.poly_deg) v = horner(a.poly, a.poly_stride, a.poly_deg, k, v);
  a.out[(int64_t)b * a.out_stride + k] = v;
  if (a.out2) a.out2[(int64_t)b * a.n_out + k] = v;
}

void launch_linear(const LinearArgs& a, cudaStream_t s, int pdl) {
  dim3 grid((unsigned)((a.out_stride + kLinO - 1) / kLinO), (unsigned)((a.batch + kLinB - 1) / kLinB));
  const size_t smem = (size_t)(kLinO + kLinB) * ((((a.n_in < kLinK ? a.n_in : kLinK) + 4) & ~3)) * sizeof(float);
  if (smem > 48 * 1024) cudaFuncSetAttribute(linear_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  launch_pdl(linear_kernel, grid, 256, smem, s, pdl, a);
}

// ---------------------------------------------------------------------------
// standalone elementwise / pool kernels (one thread per 4-channel group)
// ---------------------------------------------------------------------------
__global__ void eltwise_kernel(EltArgs a) {
  TlScope tls(a.tl);
  const TensorView& o = a.out;
  const int groups = o.cpad() / 4;
  const int64_t total = (int64_t)a.batch * groups * o.h * o.w;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int xw = (int)(i % o.w);
    int64_t r = i / o.w;
    int y = (int)(r % o.h); r /= o.h;
    int g = (int)(r % groups);
    int b = (int)(r / groups);
    int ch0 = g * 4;
    if (a.kind == PCNN_UNIT_LOCALPOOL) {
      // window sum on 4-channel float4 groups (channels >= c are zero in the input)
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int dy = 0; dy < a.k; ++dy) {
        const int iy = y * a.st - a.pad + dy;
        if (iy < 0 || iy >= a.in.h) continue;
        for (int dx = 0; dx < a.k; ++dx) {
          const int ix = xw * a.st - a.pad + dx;
          if (ix < 0 || ix >= a.in.w) continue;
          const float4 v = __ldg(reinterpret_cast<const float4*>(a.in.pix(b, ch0, iy, ix)));
          acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
      }
      const float dv = __ldg(a.p);
      *reinterpret_cast<float4*>(o.pix(b, ch0, y, xw)) = make_float4(acc.x * dv, acc.y * dv, acc.z * dv, acc.w * dv);
      continue;
    }
    float res[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int ch = ch0 + j;
      float v = 0.f;
      if (ch < o.c) {
        switch (a.kind) {
          case PCNN_UNIT_POLY: v = horner(a.p, a.stride, a.deg, ch, *a.in.at(b, ch, y, xw)); break;
          case PCNN_UNIT_ADD: v = *a.in.at(b, ch, y, xw) + *a.in2.at(b, ch, y, xw); break;
          case PCNN_UNIT_POLYSKIP:
            v = polyskip(a.p, a.stride, ch, *a.in.at(b, ch, y, xw), *a.in2.at(b, ch, y, xw));
            break;
          case PCNN_UNIT_AFFINE:
            v = fmaf(*a.in.at(b, ch, y, xw), __ldg(a.p + ch), __ldg(a.p + a.stride + ch));
            break;
          case PCNN_UNIT_LOCALPOOL: {
            float s = 0.f;
            for (int dy = 0; dy < a.k; ++dy) {
              int iy = y * a.st - a.pad + dy;
              if (iy < 0 || iy >= a.in.h) continue;
              for (int dx = 0; dx < a.k; ++dx) {
                int ix = xw * a.st - a.pad + dx;
                if (ix < 0 || ix >= a.in.w) continue;
                s += *a.in.at(b, ch, iy, ix);
              }
            }
            v = s * __ldg(a.p);
            break;
          }
          case PCNN_UNIT_BIPOOL: {
            float xv, yv;
            if (a.axis == 0) { xv = *a.in.at(b, ch, y, 2 * xw); yv = *a.in.at(b, ch, y, 2 * xw + 1); }
            else { xv = *a.in.at(b, ch, 2 * y, xw); yv = *a.in.at(b, ch, 2 * y + 1, xw); }
            v = bivariate(a.p, a.stride, a.deg, ch, xv, yv);
            break;
          }
          default: break;
        }
      }
      res[j] = v;
    }
    *reinterpret_cast<float4*>(o.pix(b, ch0, y, xw)) = make_float4(res[0], res[1], res[2], res[3]);
  }
}

// global pool / flatten: spatial -> vector [B][c] or [B][c*h*w]
__global__ void to_vector_kernel(EltArgs a) {
  TlScope tls(a.tl);
  const TensorView& in = a.in;
  const int hw = in.h * in.w;
  if (a.kind == PCNN_UNIT_GLOBALPOOL) {
    // one warp per (b, channel)
    const int64_t warps = (int64_t)a.batch * in.c;
    const int lane = threadIdx.x & 31;
    const float div = __ldg(a.p);
    for (int64_t wi = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; wi < warps;
         wi += ((int64_t)gridDim.x * blockDim.x) >> 5) {
      int b = (int)(wi / in.c), ch = (int)(wi % in.c);
      const float* p = in.at(b, ch, 0, 0);
      float s = 0.f;
      for (int q = lane; q < hw; q += 32) s += p[(int64_t)q * in.cb];
#pragma unroll
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) a.out.base[(int64_t)b * a.out.cpad() + ch] = s * div;
    }
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)a.batch * a.out.cpad();
         i += (int64_t)gridDim.x * blockDim.x)
      if ((int)(i % a.out.cpad()) >= in.c) a.out.base[i] = 0.f;
  } else {
    const int64_t n = (int64_t)in.c * hw;
    const int64_t np = a.out.cpad();
    const int64_t total = (int64_t)a.batch * np;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
      int b = (int)(i / np);
      int64_t j = i - (int64_t)b * np;
      float v = 0.f;
      if (j < n) {
        int c = (int)(j / hw), r = (int)(j - (int64_t)c * hw);
        v = *in.at(b, c, r / in.w, r % in.w);
      }
      a.out.base[i] = v;
    }
  }
}

// k x k / stride local sum pool * divisor.  One thread per (4-channel group,
// output pixel) with the channel group fastest, so a warp's loads cover whole
// 128-byte pixel rows of the channel-blocked input; the output may be split.
__global__ void localpool_kernel(EltArgs a) {
  TlScope tls(a.tl);
  const TensorView& in = a.in;
  const TensorView& o = a.out;
  const int gpb = in.cb / 4;  // 4-channel groups per channel block
  const int64_t total = (int64_t)a.batch * o.nblk * o.h * o.w * gpb;
  const float dv = __ldg(a.p);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int gi = (int)(i % gpb);
    int64_t r = i / gpb;
    const int xw = (int)(r % o.w);
    r /= o.w;
    const int y = (int)(r % o.h);
    r /= o.h;
    const int blk = (int)(r % o.nblk);
    const int b = (int)(r / o.nblk);
    const int ch0 = blk * in.cb + gi * 4;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (a.k == 3) {
      // all nine loads in flight at once
      float4 t9[9];
#pragma unroll
      for (int dy = 0; dy < 3; ++dy)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) {
          const int iy = y * a.st - a.pad + dy, ix = xw * a.st - a.pad + dx;
          const bool ok = iy >= 0 && iy < in.h && ix >= 0 && ix < in.w;
          t9[dy * 3 + dx] = ok ? __ldg(reinterpret_cast<const float4*>(in.at(b, ch0, ok ? iy : 0, ok ? ix : 0)))
                               : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
      for (int q = 0; q < 9; ++q) {
        acc.x += t9[q].x; acc.y += t9[q].y; acc.z += t9[q].z; acc.w += t9[q].w;
      }
      store4_any(o, b, ch0, y, xw, acc.x * dv, acc.y * dv, acc.z * dv, acc.w * dv);
      continue;
    }
    for (int dy = 0; dy < a.k; ++dy) {
      const int iy = y * a.st - a.pad + dy;
      if (iy < 0 || iy >= in.h) continue;
      for (int dx = 0; dx < a.k; ++dx) {
        const int ix = xw * a.st - a.pad + dx;
        if (ix < 0 || ix >= in.w) continue;
        const float4 v = __ldg(reinterpret_cast<const float4*>(in.at(b, ch0, iy, ix)));
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
    }
    store4_any(o, b, ch0, y, xw, acc.x * dv, acc.y * dv, acc.z * dv, acc.w * dv);
  }
}

// k x k / stride local sum pool * divisor over a scratch map in 4-channel
// blocks (in.cb = 4, plan_local_pools): one thread per (8-channel group,
// output pixel), x fastest -- a warp reads runs of adjacent 16-byte pixels
// and writes whole 16-byte hi / lo groups of a split output.
__global__ void localpool_cb4_kernel(EltArgs a) {
  TlScope tls(a.tl);
  const TensorView& in = a.in;
  const TensorView& o = a.out;
  const int ng = o.cpad() / 8;
  const int64_t total = (int64_t)a.batch * ng * o.h * o.w;
  const float dv = __ldg(a.p);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int xw = (int)(i % o.w);
    int64_t r = i / o.w;
    const int y = (int)(r % o.h);
    r /= o.h;
    const int g = (int)(r % ng);
    const int b = (int)(r / ng);
    const int ch0 = g * 8;
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.f;
    if (a.k == 3) {
      // all eighteen loads in flight at once
      float4 t9[2][9];
#pragma unroll
      for (int dy = 0; dy < 3; ++dy)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) {
          const int iy = y * a.st - a.pad + dy, ix = xw * a.st - a.pad + dx;
          const bool ok = iy >= 0 && iy < in.h && ix >= 0 && ix < in.w;
#pragma unroll
          for (int h = 0; h < 2; ++h)
            t9[h][dy * 3 + dx] = ok ? __ldg(reinterpret_cast<const float4*>(in.at(b, ch0 + 4 * h, iy, ix)))
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
      for (int q = 0; q < 9; ++q)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          acc[4 * h] += t9[h][q].x; acc[4 * h + 1] += t9[h][q].y; acc[4 * h + 2] += t9[h][q].z; acc[4 * h + 3] += t9[h][q].w;
        }
    } else {
      for (int dy = 0; dy < a.k; ++dy) {
        const int iy = y * a.st - a.pad + dy;
        if (iy < 0 || iy >= in.h) continue;
        for (int dx = 0; dx < a.k; ++dx) {
          const int ix = xw * a.st - a.pad + dx;
          if (ix < 0 || ix >= in.w) continue;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(in.at(b, ch0 + 4 * h, iy, ix)));
            acc[4 * h] += v.x; acc[4 * h + 1] += v.y; acc[4 * h + 2] += v.z; acc[4 * h + 3] += v.w;
          }
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] *= dv;
    store8_any(o, b, ch0, y, xw, acc);
  }
}

// k x k / stride local sum pool over row bands: a block takes kPoolBandRows
// pooled rows of one (image, channel block); the input rows they need are one
// contiguous piece of the channel-blocked map ((rows - 1) * stride + k rows
// of w * cb floats), fetched by ONE bulk copy into shared memory -- every
// input element leaves L2 once per band (9 rows for 4 pooled rows of a
// 3x3/s2 pool instead of 2.25 reads per element through L1), in long
// contiguous reads.  Same per-window summation order as localpool_kernel.
constexpr int kPoolBandRows = 4;  // most pooled rows per block
__global__ void localpool_band_kernel(EltArgs a, int bands, int brows) {
  TlScope tls(a.tl);
  extern __shared__ __align__(128) float pool_sm[];
  __shared__ uint64_t bar;
  const TensorView& in = a.in;
  const TensorView& o = a.out;
  const int cb = in.cb, gpb = cb / 4, rowf = in.w * cb;
  int id = blockIdx.x;
  const int band = id % bands;
  id /= bands;
  const int blk = id % o.nblk, b = id / o.nblk;
  const int y0 = band * brows, y1 = min(y0 + brows, o.h);
  const int r0 = max(y0 * a.st - a.pad, 0), r1 = min((y1 - 1) * a.st - a.pad + a.k, in.h);  // input rows [r0, r1)
  if (threadIdx.x == 0) {
    ptx::mbar_init(ptx::smem_u32(&bar), 1);
    ptx::fence_mbar_init();
    const uint32_t bytes = (uint32_t)(r1 - r0) * (uint32_t)rowf * 4u;
    ptx::mbar_arrive_tx(ptx::smem_u32(&bar), bytes);
    ptx::bulk_g2s(ptx::smem_u32(pool_sm), in.at(b, blk * cb, r0, 0), bytes, ptx::smem_u32(&bar));
  }
  __syncthreads();
  const float dv = __ldg(a.p);
  ptx::mbar_wait(ptx::smem_u32(&bar), 0);
  const int per = (y1 - y0) * o.w * gpb;
  for (int i = threadIdx.x; i < per; i += blockDim.x) {
    const int gi = i % gpb;
    const int r = i / gpb;
    const int xw = r % o.w, y = y0 + r / o.w;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int dy = 0; dy < a.k; ++dy) {
      const int iy = y * a.st - a.pad + dy;
      if (iy < r0 || iy >= r1) continue;
      const float* row = pool_sm + (size_t)(iy - r0) * rowf + gi * 4;
      for (int dx = 0; dx < a.k; ++dx) {
        const int ix = xw * a.st - a.pad + dx;
        if (ix < 0 || ix >= in.w) continue;
        const float4 v = *reinterpret_cast<const float4*>(row + ix * cb);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
    }
    store4_any(o, b, blk * cb + gi * 4, y, xw, acc.x * dv, acc.y * dv, acc.z * dv, acc.w * dv);
  }
}

// 2x2 / stride-2 window through two bivariate polynomials (axis 0: along w,
// then across rows; 1: along h, then across columns), 4 channels per thread,
// consecutive threads on consecutive memory (channel sub-group, then x);
// fp32 blocked input, output in its storage format.  Restates the BI2 pool
// of the conv epilogue (epi_tc.cuh) as a pass of its own.
// D > 0: the degree at compile time (every coefficient load issued up
// front, one load shared by the two first-axis evaluations); D = 0 any degree
template <int D>
__global__ void bipool2_kernel(EltArgs a) {
  TlScope tls(a.tl);
  const TensorView& in = a.in;
  const TensorView& o = a.out;
  const int sub_n = o.cb / 4;
  const int64_t total = (int64_t)a.batch * o.nblk * o.h * o.w * sub_n;
  const int64_t nc = (int64_t)(a.deg + 1) * (a.deg + 1) * a.stride;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i;
    const int sub = (int)(r % sub_n); r /= sub_n;
    const int x = (int)(r % o.w); r /= o.w;
    const int y = (int)(r % o.h); r /= o.h;
    const int blk = (int)(r % o.nblk);
    const int b = (int)(r / o.nblk);
    const int ch0 = blk * o.cb + 4 * sub;
    const float4 q00 = __ldg(reinterpret_cast<const float4*>(in.pix(b, ch0, 2 * y, 2 * x)));
    const float4 q01 = __ldg(reinterpret_cast<const float4*>(in.pix(b, ch0, 2 * y, 2 * x + 1)));
    const float4 q10 = __ldg(reinterpret_cast<const float4*>(in.pix(b, ch0, 2 * y + 1, 2 * x)));
    const float4 q11 = __ldg(reinterpret_cast<const float4*>(in.pix(b, ch0, 2 * y + 1, 2 * x + 1)));
    float4 u, w, v;
    if constexpr (D > 0) {
      if (a.axis == 0) bivariate4x2_t<D>(a.p, a.stride, ch0, q00, q01, q10, q11, u, w);
      else bivariate4x2_t<D>(a.p, a.stride, ch0, q00, q10, q01, q11, u, w);
      v = bivariate4_t<D>(a.p + nc, a.stride, ch0, u, w);
    } else {
      if (a.axis == 0) {
        u = bivariate4(a.p, a.stride, a.deg, ch0, q00, q01);
        w = bivariate4(a.p, a.stride, a.deg, ch0, q10, q11);
      } else {
        u = bivariate4(a.p, a.stride, a.deg, ch0, q00, q10);
        w = bivariate4(a.p, a.stride, a.deg, ch0, q01, q11);
      }
      v = bivariate4(a.p + nc, a.stride, a.deg, ch0, u, w);
    }
    if (ch0 + 0 >= o.c) v.x = 0.f;
    if (ch0 + 1 >= o.c) v.y = 0.f;
    if (ch0 + 2 >= o.c) v.z = 0.f;
    if (ch0 + 3 >= o.c) v.w = 0.f;
    store4_any(o, b, ch0, y, x, v.x, v.y, v.z, v.w);
  }
}

void launch_eltwise(const EltArgs& a, cudaStream_t s, int pdl) {
  if (a.kind == PCNN_UNIT_LOCALPOOL && a.pool == PCNN_POOL_BI2) {
    const int64_t total = (int64_t)a.batch * a.out.nblk * a.out.h * a.out.w * (a.out.cb / 4);
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 32);
    void (*k)(EltArgs) = a.deg == 2   ? bipool2_kernel<2>
                         : a.deg == 3 ? bipool2_kernel<3>
                         : a.deg == 4 ? bipool2_kernel<4>
                                      : bipool2_kernel<0>;
    launch_pdl(k, std::max(blocks, 1), 256, 0, s, pdl, a);
    return;
  }
  if (a.kind == PCNN_UNIT_GLOBALPOOL || a.kind == PCNN_UNIT_FLATTEN) {
    launch_pdl(to_vector_kernel, 148 * 8, 256, 0, s, pdl, a);
    return;
  }
  if (a.kind == PCNN_UNIT_LOCALPOOL && !a.in.split && a.in.cb == 4 && a.out.cb >= 8 && a.pool == 0) {
    const int64_t total = (int64_t)a.batch * (a.out.cpad() / 8) * a.out.h * a.out.w;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 32);
    launch_pdl(localpool_cb4_kernel, std::max(blocks, 1), 256, 0, s, pdl, a);
    return;
  }
  if (a.kind == PCNN_UNIT_LOCALPOOL && !a.in.split && a.in.cb == a.out.cb && a.pool == 0 &&
      (reinterpret_cast<uintptr_t>(a.in.base) & 15) == 0) {
    // row bands through shared memory: the most pooled rows per block (4, 2
    // or 1) whose input rows fit 72 KB, so three blocks share an SM
    for (int brows = kPoolBandRows; brows >= 1; brows >>= 1) {
      const size_t smem = (size_t)((brows - 1) * a.st + a.k) * a.in.w * a.in.cb * sizeof(float);
      if (smem > 72 * 1024 || brows > a.out.h) continue;
      static bool attr_set = false;
      if (!attr_set) {
        cudaFuncSetAttribute(localpool_band_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 72 * 1024);
        attr_set = true;
      }
      const int bands = (a.out.h + brows - 1) / brows;
      launch_pdl(localpool_band_kernel, a.batch * a.out.nblk * bands, 256, smem, s, pdl, a, bands, brows);
      return;
    }
  }
  if (a.kind == PCNN_UNIT_LOCALPOOL && !a.in.split && a.in.cb == a.out.cb) {
    const int64_t total = (int64_t)a.batch * a.out.nblk * a.out.h * a.out.w * (a.in.cb / 4);
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 32);
    launch_pdl(localpool_kernel, std::max(blocks, 1), 256, 0, s, pdl, a);
    return;
  }
  int64_t total = (int64_t)a.batch * (a.out.cpad() / 4) * a.out.h * a.out.w;
  int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  launch_pdl(eltwise_kernel, std::max(blocks, 1), 256, 0, s, pdl, a);
}

// blocked tensor -> user output [B][C][H][W] (logits [B][K] when H = W = 1)
__global__ void copyout_kernel(TensorView t, float* __restrict__ dst, int batch, unsigned long long* tl) {
  TlScope tls(tl);
  const int64_t hw = (int64_t)t.h * t.w;
  const int64_t n = (int64_t)batch * t.c * hw;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i % hw, bc = i / hw;
    int c = (int)(bc % t.c), b = (int)(bc / t.c);
    dst[i] = *t.at(b, c, (int)(r / t.w), (int)(r % t.w));
  }
}

void launch_copyout(const TensorView& t, float* dst, int batch, cudaStream_t s, unsigned long long* tl, int pdl) {
  int64_t n = (int64_t)batch * t.c * t.h * t.w;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  launch_pdl(copyout_kernel, std::max(blocks, 1), 256, 0, s, pdl, t, dst, batch, tl);
}

}  // namespace pcnn
