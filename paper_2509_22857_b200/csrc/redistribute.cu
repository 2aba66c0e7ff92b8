// Weight redistribution as one cooperative kernel, and parameter packing.
//
// Phase (a), block 0 only: run the straight-line scale program (pcnn_scale_op)
// over float64 vectors in the arena, in order -- update terms upsilon
// (reference transforms.py:296-318), their powers/roots/reciprocals, and the
// channelwise scale solve of redistribute_pass (transforms.py:515-659).
// Refusals the reference raises as TransformError are value checks here
// (CHECK_* ops); the first failure is written to status and phase (b) is
// skipped.
// Phase (b), all blocks after a grid barrier: every rewrite descriptor
// rescales one float64 parameter tensor in place, applying its factor chain
// in order (transforms.py:374-485 per donor, :661-704 channelwise).
#include <cooperative_groups.h>

#include <cmath>

#include "kernels.cuh"
#include "tc_layout.cuh"

namespace cg = cooperative_groups;

namespace pcnn {

constexpr int kRwChunk = 4096;  // rewrite elements per phase-(b) work chunk

__device__ __forceinline__ double ipow(double x, long long p) {
  // exact repeated squaring for small positive p matches x*x*... closely;
  // use pow() like numpy for the general case
  if (p == 1) return x;
  if (p == 2) return x * x;  // numpy's square fast path
  if (p == 0) return 1.0;
  return pow(x, (double)p);
}

__device__ void run_program(const double* __restrict__ master_ro, double* master, double* arena,
                            const pcnn_scale_op* ops, int n_ops, int64_t* status, int64_t* flags) {
  __shared__ int failed;
  __shared__ int bad;
  if (threadIdx.x == 0) failed = 0;
  __syncthreads();
  for (int k = 0; k < n_ops; ++k) {
    const pcnn_scale_op o = ops[k];
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    for (int64_t i = threadIdx.x; i < o.n; i += blockDim.x) {
      double A = 0.0, B = 0.0;
      if (o.op != PCNN_OP_FILL && o.op != PCNN_OP_LOAD) A = arena[o.a + i * o.sa];
      if (o.op == PCNN_OP_MUL || o.op == PCNN_OP_DIV || o.op == PCNN_OP_SUB || o.op == PCNN_OP_SOLVE ||
          o.op == PCNN_OP_CHECK_CLOSE || o.op == PCNN_OP_ADD)
        B = arena[o.b + i * o.sb];
      switch (o.op) {
        case PCNN_OP_FILL: arena[o.dst + i] = o.imm; break;
        case PCNN_OP_LOAD: arena[o.dst + i] = master[o.a + i * o.sa]; break;
        case PCNN_OP_MUL: arena[o.dst + i] = A * B; break;
        case PCNN_OP_DIV: arena[o.dst + i] = A / B; break;
        case PCNN_OP_SUB: arena[o.dst + i] = A - B; break;
        case PCNN_OP_ADD: arena[o.dst + i] = A + B; break;
        case PCNN_OP_POWI: arena[o.dst + i] = o.p >= 0 ? ipow(A, o.p) : pow(A, (double)o.p); break;
        case PCNN_OP_SROOT: arena[o.dst + i] = copysign(pow(fabs(A), 1.0 / (double)o.p), A); break;
        case PCNN_OP_AROOT: arena[o.dst + i] = pow(fabs(A), 1.0 / (double)o.p); break;
        case PCNN_OP_RECIP: arena[o.dst + i] = 1.0 / A; break;
        case PCNN_OP_SQRT: arena[o.dst + i] = sqrt(A); break;
        case PCNN_OP_SOLVE: {
          double r = B / A;
          if ((o.p % 2) == 0 && r < 0) bad = 1;
          double s = (r > 0) ? 1.0 : ((r < 0) ? -1.0 : 0.0);
          arena[o.dst + i] = s * pow(fabs(r), 1.0 / (double)o.p);
          break;
        }
        case PCNN_OP_CHECK_UNIFORM:
          if (A != arena[o.a]) bad = 1;
          break;
        case PCNN_OP_CHECK_NONZERO:
          if (A == 0.0) bad = 1;
          break;
        case PCNN_OP_CHECK_NONNEG:
          if (A < 0.0) bad = 1;
          break;
        case PCNN_OP_CHECK_CLOSE:
          if (!(fabs(A - B) <= o.atol + o.rtol * fabs(B))) bad = 1;
          break;
        case PCNN_OP_CHECK_ALLONE:
          if (A != 1.0) bad = 1;
          break;
        case PCNN_OP_STORE: master[o.dst + i * o.sa] = A; break;
        default: bad = 2; break;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (o.op == PCNN_OP_CHECK_ALLONE) {
        flags[o.p] = bad ? 0 : 1;
      } else if (bad) {
        status[0] = bad == 2 ? -1 : o.err;
        status[1] = k;
        failed = 1;
      }
    }
    __syncthreads();
    if (failed) return;
  }
}

// smem_arena: phase (a) keeps the arena and the op table in block 0's shared
// memory (every op is then a few shared-memory accesses and two block
// barriers instead of dependent L2 round trips) and publishes the arena to
// global memory for phase (b)
__global__ void redistribute_kernel(double* master, double* arena, int64_t arena_len, int smem_arena,
                                    const pcnn_scale_op* ops, int n_ops, const pcnn_rewrite_desc* rw, int n_rw,
                                    const int2* chunks, int n_chunks, int64_t* status, int64_t* flags) {
  extern __shared__ double sarena[];
  cg::grid_group grid = cg::this_grid();
  if (blockIdx.x == 0) {
    const pcnn_scale_op* pops = ops;
    if (smem_arena) {
      // the op table after the arena (16-byte aligned)
      pcnn_scale_op* sops = reinterpret_cast<pcnn_scale_op*>(sarena + ((arena_len + 1) & ~int64_t(1)));
      const int64_t words = (int64_t)n_ops * (int64_t)(sizeof(pcnn_scale_op) / 8);
      const int64_t* src = reinterpret_cast<const int64_t*>(ops);
      int64_t* dst = reinterpret_cast<int64_t*>(sops);
      for (int64_t i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
      __syncthreads();
      pops = sops;
    }
    run_program(master, master, smem_arena ? sarena : arena, pops, n_ops, status, flags);
    if (smem_arena) {
      __syncthreads();
      for (int64_t i = threadIdx.x; i < arena_len; i += blockDim.x) arena[i] = sarena[i];
    }
  }
  grid.sync();
  if (status[0] != 0) return;
  // phase (b): the rewrites cut into chunks of kRwChunk elements, chunks
  // spread over the blocks (every rewrite in parallel; a block pays one
  // descriptor load per chunk, not one per rewrite); factor indices in
  // 32-bit arithmetic (every extent < 2^31, checked at create)
  for (int c = blockIdx.x; c < n_chunks; c += gridDim.x) {
    const int2 ch = chunks[c];
    const pcnn_rewrite_desc& r = rw[ch.x];
    const int n = (int)r.n, e1 = min(ch.y + kRwChunk, n), nf = (int)r.n_factors;
    const double* src = r.src_arena ? arena + r.src : master + r.src;
    double* dst = master + r.dst;
    if (r.set_const) {
      for (int e = ch.y + threadIdx.x; e < e1; e += blockDim.x) dst[e] = r.value;
      continue;
    }
    for (int e = ch.y + threadIdx.x; e < e1; e += blockDim.x) {
      double v = src[e];
      for (int f = 0; f < nf; ++f) {
        const pcnn_factor& F = r.f[f];
        const unsigned idx = (((unsigned)e / (unsigned)F.d1) % (unsigned)F.m1) * (unsigned)F.s1 +
                             ((unsigned)e / (unsigned)F.d2) % (unsigned)F.m2;
        const double fv = arena[F.slot + idx];
        v = F.divide ? v / fv : v * fv;
      }
      dst[e] = v;
    }
  }
}

// phase 0 (one block per op): zero the max|w| slot of each fp16x2 image;
// phase 1 (grid n_ops x slices): max|w| by block reduction + one atomicMax
// on the float bits (non-negative floats order like their bit patterns).
__global__ void pack_amax_kernel(const double* __restrict__ master, float* __restrict__ packed,
                                 const pcnn_pack_desc* ops, int n_ops, int phase) {
  const pcnn_pack_desc o = ops[blockIdx.x];
  if (o.kind != PCNN_PACK_TC16_WEIGHTS) return;
  if (phase == 0) {
    if (threadIdx.x == 0) packed[o.aux] = 0.f;
    return;
  }
  const int64_t total = o.rows * o.k;
  float m = 0.f;
  for (int64_t i = blockIdx.y * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.y * blockDim.x)
    m = fmaxf(m, (float)fabs(master[o.src + i]));
  for (int off = 16; off; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
  __shared__ float red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmaxf(m, red[w]);
    atomicMax(reinterpret_cast<int*>(packed + o.aux), __float_as_int(m));
  }
}

// first_block (n_ops + 1 entries, or null): op k is packed by blocks
// [first_block[k], first_block[k + 1]) -- every op in parallel, each by a
// block count proportional to its size; null: all blocks walk every op.
__global__ void pack_kernel(const double* __restrict__ master, float* __restrict__ packed,
                            const pcnn_pack_desc* ops, int n_ops, const int* __restrict__ first_block) {
  int k0 = 0, k1 = n_ops;
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  if (first_block) {
    int lo = 0, hi = n_ops - 1;  // last op whose first block <= blockIdx.x
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (first_block[mid] <= (int)blockIdx.x) lo = mid;
      else hi = mid - 1;
    }
    k0 = lo;
    k1 = lo + 1;
    tid = (blockIdx.x - first_block[lo]) * (int64_t)blockDim.x + threadIdx.x;
    nthreads = (int64_t)(first_block[lo + 1] - first_block[lo]) * blockDim.x;
  }
  for (int k = k0; k < k1; ++k) {
    const pcnn_pack_desc o = ops[k];
    if (o.kind == PCNN_PACK_CAST) {
      for (int64_t i = tid; i < o.n; i += nthreads) packed[o.dst + i] = (float)master[o.src + i];
    } else if (o.kind == PCNN_PACK_BN_AFFINE) {
      const double* g = master + o.src;
      for (int64_t i = tid; i < o.n; i += nthreads) {
        double s = g[i] / g[3 * o.n + i];
        packed[o.dst + i] = (float)s;
        packed[o.dst + o.n + i] = (float)(g[o.n + i] - s * g[2 * o.n + i]);
      }
    } else if (o.kind == PCNN_PACK_TC_WEIGHTS) {
      pack_tc_weights_device(master + o.src, packed + o.dst, (int)o.rows, (int)o.k, tid, nthreads);
    } else if (o.kind == PCNN_PACK_TCSS_WEIGHTS) {
      // shares the fp16x2 image's scale pair (computed by pack_amax_kernel)
      const int e = tc16_scale_exp(packed[o.aux]);
      pack_tcss_weights_device(master + o.src, reinterpret_cast<__half*>(packed + o.dst), (int)o.rows, (int)o.k,
                               (int)(o.reserved & 0xFFFF), (int)(o.reserved >> 16), e, tid, nthreads);
    } else if (o.kind == PCNN_PACK_TC16_WEIGHTS) {
      const int e = tc16_scale_exp(packed[o.aux]);
      if (tid == 0) packed[o.aux + 1] = ldexpf(1.f, -e);
      pack_tc16_weights_device(master + o.src, reinterpret_cast<__half*>(packed + o.dst), (int)o.rows, (int)o.k, e,
                               tid, nthreads);
    }
  }
}

}  // namespace pcnn
