// C ABI of libpcnn: plans, forward (CUDA-graph replay), packing and
// redistribution launches.  See include/pcnn.h for the contract.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "tc_layout.cuh"

namespace pcnn {
__global__ void redistribute_kernel(double*, double*, int64_t, int, const pcnn_scale_op*, int,
                                    const pcnn_rewrite_desc*, int, const int2*, int, int64_t*, int64_t*);
__global__ void pack_kernel(const double*, float*, const pcnn_pack_desc*, int, const int*);
__global__ void pack_amax_kernel(const double*, float*, const pcnn_pack_desc*, int, int);
}  // namespace pcnn

using namespace pcnn;

namespace {

// Per-forward reset of a plan's small device state (status word, stream-K
// and flag counters, launch timeline) in ONE kernel node instead of a
// memset node per buffer.
struct ResetRanges {
  uint32_t* p[4];
  int64_t n[4];  // 32-bit words
};
__global__ void plan_reset_kernel(ResetRanges r) {
  for (int k = 0; k < 4; ++k)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < r.n[k]; i += (int64_t)gridDim.x * blockDim.x)
      r.p[k][i] = 0u;
}

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define PCNN_CUDA(call)                                                                    \
  do {                                                                                     \
    cudaError_t _e = (call);                                                               \
    if (_e != cudaSuccess)                                                                 \
      return fail(PCNN_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e));      \
  } while (0)

struct GraphEntry {
  const float* x;
  float* logits;
  cudaGraphExec_t exec;
};

}  // namespace

struct pcnn_plan {
  std::vector<pcnn_unit_desc> units;
  std::vector<pcnn_tensor_desc> tensors;
  std::vector<TensorView> views;
  std::vector<char> prezeroed;  // unit's global-pool output zeroed by the previous kernel
  std::vector<int> impl;  // per unit: 1 SIMT, 2 tcgen05
  std::vector<ConvArgs> conv_args;
  int batch = 0, input = 0, output = 0;
  int64_t in_elems = 0;  // user input floats per image (NCHW; a space-to-depth ingest's image, not its tensor)
  const float* params = nullptr;
  float* ws = nullptr;
  size_t ws_bytes = 0;
  cudaStream_t capture_stream = nullptr;
  std::vector<GraphEntry> graphs;
  int launches = 0;
  bool any_split = false;
  int* status_dev = nullptr;   // bit 0: a split-format value left the fp16 range
  int* status_host = nullptr;  // pinned copy written by pcnn_forward_host
  pcnn_plan_options opt;
  KOpts kopt;
  // PCNN_POOL_LOCAL convs not run by the halo-tile band epilogue: unpooled
  // output in plan scratch (float32), then this pooling launch
  std::vector<EltArgs> post_pool;
  std::vector<char> has_post_pool;
  float* scratch = nullptr;
  // image-resident runs (build_blocks): blk_of[u] = run index or -1; a run
  // launches with its first unit
  std::vector<BlkRun*> blks;
  std::vector<int> blk_of, blk_first;
  // whole-network launch (build_net): every unit in one net_kernel launch
  bool net_on = false;
  NetParams net = {};
  int net_grid = 0;
  // launch timeline (options.timeline): [n_units][2] (common.cuh tl_mark)
  unsigned long long* tl_dev = nullptr;
  unsigned long long* tl_host = nullptr;
  // flag-synchronised halo-tile launches (build_flags): per-tile completion
  // counters of every signalling unit, zeroed at the start of each forward
  bool flags_on = false;
  int* flags_dev = nullptr;
  size_t flags_n = 0;
  // fused[u]: unit u (a 1x1 projection) runs inside unit u - 1's halo-tile launch;
  // for a copyout: the linear unit before it writes the user's logits itself
  std::vector<char> fused;
  // stream-K halo-tile launches (plan_streamk): per-unit CTA flags, shared partial slots
  int* sk_flags = nullptr;
  size_t sk_flags_n = 0;
  float* sk_slots = nullptr;
  // pcnn_forward_host_many: copy stream, per-buffer events, pinned statuses
  cudaStream_t copy_stream = nullptr, out_stream = nullptr;
  cudaEvent_t h2d_done[2] = {nullptr, nullptr}, x_free[2] = {nullptr, nullptr};
  cudaEvent_t fwd_done[2] = {nullptr, nullptr}, out_free[2] = {nullptr, nullptr};
  float* logits2 = nullptr;    // second logits staging buffer (plan-owned)
  int* status_slots = nullptr; // device: one status word per batch
  int* status_pinned = nullptr;
  int status_pinned_n = 0;
};

namespace {

TensorView make_view(const pcnn_tensor_desc& t, float* ws) {
  TensorView v;
  v.base = ws + t.offset;
  v.c = (int)t.c;
  v.h = (int)t.h;
  v.w = (int)t.w;
  v.cb = (int)t.cb;
  v.nblk = (int)t.nblk;
  v.is_vector = (int)t.is_vector;
  v.cbs = 0;
  while ((1 << v.cbs) < v.cb) ++v.cbs;
  v.split = 0;
  v.sstore = ldexpf(1.f, (int)t.scale_log2);
  v.sload = ldexpf(1.f, -(int)t.scale_log2);
  v.hp = v.wp = 0;
  v.kstride = v.pstride = 0;
  v.plane = 0;
  v.flag = nullptr;
  return v;
}

int64_t tensor_floats(const pcnn_tensor_desc& t, int batch) {
  return tensor_storage_floats(batch, t.c, t.nblk * t.cb, t.h, t.w, t.is_vector != 0);
}

// Storage formats: a tensor is kept split (two fp16 planes, common.cuh) when
// its producer is the ingest, a local pool or an fp16x2 tcgen05 conv writing
// a spatial tensor, and every reader is an fp16x2 tcgen05 conv (input or
// residual skip).  It takes the parity layout when every conv that reads it
// as input has stride 2 and a shape the halo-tile kernel runs.  Everything
// else stays fp32.
void choose_formats(pcnn_plan* p) {
  const int nt = (int)p->tensors.size();
  std::vector<int> ok(nt, 1), produced(nt, 0), s2_only(nt, 1), inputs(nt, 0);
  for (int i = 0; i < (int)p->units.size(); ++i) {
    const pcnn_unit_desc& u = p->units[i];
    const bool tc16 = u.kind == PCNN_UNIT_CONV && p->impl[i] == 3;
    if (u.out >= 0) {
      produced[u.out] = 1;
      const bool pool_split = u.kind == PCNN_UNIT_LOCALPOOL && p->tensors[u.in].cb == p->tensors[u.out].cb;
      if (!(u.kind == PCNN_UNIT_INGEST || pool_split || (tc16 && u.pool != PCNN_POOL_GLOBAL))) ok[u.out] = 0;
    }
    if (u.in >= 0) {
      ++inputs[u.in];
      if (!tc16) ok[u.in] = 0;
      const bool ss2 = tc16 && u.stride == 2 && (u.impl == 0 || u.impl == 3 || u.impl == 5) &&
                       p->opt.halo_tiles && conv_ss_shape_ok(p->conv_args[i]);
      if (!ss2) s2_only[u.in] = 0;
    }
    if (u.in2 >= 0 && !(tc16 && u.residual)) ok[u.in2] = 0;
  }
  if (!p->opt.split) ok.assign(nt, 0);
  for (int t = 0; t < nt; ++t) {
    TensorView& v = p->views[t];
    if (!ok[t] || !produced[t] || v.is_vector || t == p->output) continue;
    if (v.cb < 8 && v.nblk > 1) continue;
    if (s2_only[t] && inputs[t] > 0) {
      v.split = 2;
      v.hp = (v.h + 3) / 2;
      v.wp = (v.w + 3) / 2;
      v.pstride = (int64_t)p->batch * v.hp * v.wp * 8;
      v.kstride = 4 * v.pstride;
    } else {
      v.split = 1;
      v.hp = v.h + 1;
      v.wp = v.w + 1;
      // positions: leading zero, B (H+1) + 1 rows of pitch W+1, one spare
      v.kstride = v.pstride = (2 + ((int64_t)p->batch * v.hp + 1) * v.wp) * 8;
    }
    v.plane = (int64_t)((v.cpad() + 7) / 8) * v.kstride;
    if (v.plane >= (1ll << 31)) {  // 32-bit segment offsets in the conv kernels
      v.split = 0;
      continue;
    }
    v.flag = p->status_dev;
    p->any_split = true;
  }
  for (int i = 0; i < (int)p->units.size(); ++i) {
    const pcnn_unit_desc& u = p->units[i];
    if (u.kind != PCNN_UNIT_CONV) continue;
    ConvArgs& a = p->conv_args[i];
    a.in = p->views[u.in];
    a.epi.out = p->views[u.out];
    if (u.residual) a.epi.skip = p->views[u.in2];
    // fp16x2 convs reading a split tensor: the halo-tile kernel when the
    // shape allows (unit impl 0, 3 or 5)
    if (p->impl[i] == 3 && (u.impl == 0 || u.impl == 3 || u.impl == 5) && p->opt.halo_tiles &&
        conv_ss_supported(a))
      p->impl[i] = 5;
  }
}

const float* P(const pcnn_plan* p, int64_t off) { return off < 0 ? nullptr : p->params + off; }

int build_conv(pcnn_plan* p, int ui, ConvArgs& a) {
  const pcnn_unit_desc& u = p->units[ui];
  const TensorView& in = p->views[u.in];
  const TensorView& out = p->views[u.out];
  a.in = in;
  a.batch = p->batch;
  a.kh = (int)u.kh;
  a.kw = (int)u.kw;
  a.stride = (int)u.stride;
  a.pad = (int)u.pad;
  a.kp = in.nblk * a.kh * a.kw * in.cb;
  int ho = (in.h + 2 * a.pad - a.kh) / a.stride + 1;
  int wo = (in.w + 2 * a.pad - a.kw) / a.stride + 1;
  a.pm.ho = ho;
  a.pm.wo = wo;
  a.pm.hp = ho / 2;
  a.pm.wp = wo / 2;
  a.pm.order = (u.pool == PCNN_POOL_SUM2 || u.pool == PCNN_POOL_BI2) ? kWindow : kPlain;
  a.w = P(p, u.w_off);
  a.tcw = P(p, u.tc_off);
  a.tcw16 = P(p, u.tc16_off);
  a.tc16_scale = P(p, u.tc16_scale_off);
  a.tcwss = P(p, u.tcss_off);
  a.f16 = 0;
  EpiParams& e = a.epi;
  e.cout = (int)u.cout;
  e.npad = out.cpad();
  e.pool_k = (int)(u.pool_geom & 0xff);
  e.pool_s = (int)((u.pool_geom >> 8) & 0xff);
  e.pool_pad = (int)((u.pool_geom >> 16) & 0xff);
  if (u.pool == PCNN_POOL_GLOBAL) {
    if (out.h != 1 || out.w != 1 || out.c != u.cout)
      return fail(PCNN_ERR_INVALID, "global-pool conv needs a (cout,) output");
  } else if (u.pool == PCNN_POOL_LOCAL) {
    if (e.pool_k < 1 || e.pool_s < 1 || e.pool_pad < 0 || e.pool_pad >= e.pool_k)
      return fail(PCNN_ERR_INVALID, "conv unit " + std::to_string(ui) + ": bad local pool geometry");
    if (out.h != (ho + 2 * e.pool_pad - e.pool_k) / e.pool_s + 1 ||
        out.w != (wo + 2 * e.pool_pad - e.pool_k) / e.pool_s + 1 || out.c != u.cout)
      return fail(PCNN_ERR_INVALID, "conv unit " + std::to_string(ui) + ": pooled output tensor shape mismatch");
  } else {
    int ho_o = a.pm.order == kWindow ? a.pm.hp : ho, wo_o = a.pm.order == kWindow ? a.pm.wp : wo;
    if (out.h != ho_o || out.w != wo_o || out.c != u.cout)
      return fail(PCNN_ERR_INVALID, "conv unit " + std::to_string(ui) + ": output tensor shape mismatch");
  }
  a.npad = e.npad;
  if (u.npad && u.npad != e.npad) return fail(PCNN_ERR_INVALID, "unit npad disagrees with its output tensor");
  e.bias = P(p, u.b_off);
  e.aff = P(p, u.affine_off);
  e.residual = (int)u.residual;
  e.res = P(p, u.res_off);
  e.poly_deg = (int)u.poly_deg;
  e.poly = P(p, u.poly_off);
  e.pool = (int)u.pool;
  e.pool_p = P(p, u.pool_off);
  e.pool_deg = (int)u.pool_deg;
  e.pool_order = (int)u.pool_order;
  e.out = out;
  if (u.pool == PCNN_POOL_LOCAL) {
    // the other conv kernels see an unpooled conv: plan_local_pools either
    // hands the pool to the halo-tile kernel's band epilogue or gives the
    // conv a scratch output and a pooling launch
    e.pool = PCNN_POOL_NONE;
    e.out.h = ho;
    e.out.w = wo;
  }
  if (u.residual) {
    if (u.in2 < 0) return fail(PCNN_ERR_INVALID, "residual unit without skip tensor");
    e.skip = p->views[u.in2];
    if (e.skip.h != ho || e.skip.w != wo) return fail(PCNN_ERR_INVALID, "skip tensor shape mismatch");
  }
  if (u.poly_deg > kMaxPolyDeg) return fail(PCNN_ERR_UNSUPPORTED, "polynomial degree > 8");
  if (u.pool == PCNN_POOL_BI2 && u.pool_deg > kMaxBiDeg) return fail(PCNN_ERR_UNSUPPORTED, "bivariate degree > 4");
  if (!a.w || !e.bias) return fail(PCNN_ERR_INVALID, "conv unit without weights");
  return PCNN_OK;
}

void enqueue_unit(pcnn_plan* p, int ui, const float* x, float* logits, cudaStream_t s, bool flags) {
  const pcnn_unit_desc& u = p->units[ui];
  unsigned long long* tl = p->tl_dev ? p->tl_dev + 2 * ui : nullptr;
  switch (u.kind) {
    case PCNN_UNIT_INGEST:
      launch_ingest(x, p->views[u.out], p->batch, (u.flags & PCNN_FLAG_S2D) != 0, s, (int)p->opt.pdl, tl);
      break;
    case PCNN_UNIT_CONV: {
      if (p->fused[ui]) break;  // computed by the previous unit's launch
      if (!p->blk_of.empty() && p->blk_of[ui] >= 0) {
        const int r = p->blk_of[ui];
        if (p->blk_first[r] == ui) {
          int last = ui;
          while (last + 1 < (int)p->units.size() && p->blk_of[last + 1] == r) ++last;
          if (p->units[last].pool == PCNN_POOL_GLOBAL && !p->prezeroed[last]) {
            const ConvArgs& al = p->conv_args[last];
            cudaMemsetAsync(al.epi.out.base, 0, sizeof(float) * (size_t)p->batch * al.epi.out.cpad(), s);
          }
          blk_launch(p->blks[r], s, tl, p->kopt.pdl);
        }
        break;  // the other units of the run are computed by that launch
      }
      ConvArgs a = p->conv_args[ui];
      a.tl = tl;
      if (u.pool == PCNN_POOL_GLOBAL && !p->prezeroed[ui])
        cudaMemsetAsync(a.epi.out.base, 0, sizeof(float) * (size_t)p->batch * a.epi.out.cpad(), s);
      if (p->impl[ui] == 5) {
        if (flags || !p->flags_on) {
          launch_conv_ss(a, s);
        } else {
          // a unit run on its own: plain griddepcontrol ordering, no counters
          ConvArgs& b = a;
          b.sig_done = nullptr;
          b.skip_gridwait = 0;
          b.fin = FlagDep();
          b.fsk = FlagDep();
          launch_conv_ss(b, s);
        }
      } else if (p->impl[ui] >= 2) {
        launch_conv_tc(a, s);
      }
      else launch_conv_simt(a, s);
      if (p->has_post_pool[ui]) {
        EltArgs e = p->post_pool[ui];
        e.tl = tl ? tl + 2 * p->units.size() : nullptr;  // the pass has its own timeline slot
        launch_eltwise(e, s, (int)p->opt.pdl);
      }
      break;
    }
    case PCNN_UNIT_LINEAR: {
      LinearArgs a;
      a.in = p->views[u.in];
      a.in_mode = (int)u.in_mode;
      a.batch = p->batch;
      a.n_in = (int)u.cin;
      a.n_out = (int)u.cout;
      a.in_div = P(p, u.in_div_off);
      a.w = P(p, u.w_off);
      a.bias = P(p, u.b_off);
      a.poly_deg = (int)u.poly_deg;
      a.poly = P(p, u.poly_off);
      a.poly_stride = p->views[u.out].cpad();
      a.out = p->views[u.out].base;
      a.out_stride = p->views[u.out].cpad();
      if (ui + 1 < (int)p->fused.size() && p->fused[ui + 1]) a.out2 = logits;
      a.tl = tl;
      launch_linear(a, s, 0);  // plain launch: measured faster than PDL (RN18 9.3 vs 12.9 us)
      break;
    }
    case PCNN_UNIT_COPYOUT: {
      if (p->fused[ui]) break;  // the linear unit before it wrote the logits
      launch_copyout(p->views[u.in], logits, p->batch, s, tl, 0);  // plain: a tiny grid launched early would crowd the dense layer's blocks
      break;
    }
    default: {
      EltArgs a;
      a.kind = (int)u.kind;
      a.batch = p->batch;
      a.in = p->views[u.in];
      if (u.in2 >= 0) a.in2 = p->views[u.in2];
      a.out = p->views[u.out];
      a.p = P(p, u.pool_off >= 0 ? u.pool_off : (u.poly_off >= 0 ? u.poly_off : (u.res_off >= 0 ? u.res_off : u.affine_off)));
      a.stride = a.out.cpad();
      a.deg = (int)(u.kind == PCNN_UNIT_POLY ? u.poly_deg : u.pool_deg);
      a.k = (int)u.kh;
      a.st = (int)u.stride;
      a.pad = (int)u.pad;
      a.axis = (int)u.pool_order;
      a.pool = (int)u.pool;
      a.tl = tl;
      launch_eltwise(a, s, (int)p->opt.pdl);
      break;
    }
  }
}

void enqueue_all(pcnn_plan* p, const float* x, float* logits, cudaStream_t s) {
  ResetRanges r = {};
  int k = 0;
  if (p->any_split) { r.p[k] = reinterpret_cast<uint32_t*>(p->status_dev); r.n[k++] = 1; }
  if (p->flags_on) { r.p[k] = reinterpret_cast<uint32_t*>(p->flags_dev); r.n[k++] = (int64_t)p->flags_n; }
  if (p->sk_flags) { r.p[k] = reinterpret_cast<uint32_t*>(p->sk_flags); r.n[k++] = (int64_t)p->sk_flags_n; }
  if (p->tl_dev) { r.p[k] = reinterpret_cast<uint32_t*>(p->tl_dev); r.n[k++] = 8 * (int64_t)p->units.size(); }
  if (k) plan_reset_kernel<<<1, 256, 0, s>>>(r);
  if (p->net_on) {
    NetParams P = p->net;
    P.x = x;
    P.logits = logits;
    P.tl = p->tl_dev;  // unit 0's slot: the launch covers every unit
    net_launch(P, s, p->net_grid);
    return;
  }
  for (int i = 0; i < (int)p->units.size(); ++i) enqueue_unit(p, i, x, logits, s, true);
}

// Pooled convs (PCNN_POOL_LOCAL, e.g. ResNet-18's stem followed by its
// 3x3/s2 pool; PCNN_POOL_BI2 on the halo-tile kernel): with options.band_pool
// the pool runs in the halo-tile kernel's band epilogue (conv_ss.cu
// band_item) -- the unpooled map never reaches global memory; otherwise the
// conv writes a float32 scratch map and a pooling launch follows (BI2 on the
// TMEM-A / SIMT kernels keeps its window-order fused epilogue).
int plan_local_pools(pcnn_plan* p) {
  const int n = (int)p->units.size();
  p->post_pool.assign(n, EltArgs());
  p->has_post_pool.assign(n, 0);
  size_t need = 0;
  std::vector<int> fallback;
  for (int i = 0; i < n; ++i) {
    const pcnn_unit_desc& u = p->units[i];
    if (u.kind != PCNN_UNIT_CONV || !(u.pool == PCNN_POOL_LOCAL || u.pool == PCNN_POOL_BI2)) continue;
    ConvArgs& a = p->conv_args[i];
    if (u.pool == PCNN_POOL_BI2 && p->impl[i] != 5) continue;  // window-order epilogue of the other kernels
    ConvArgs b = a;
    b.epi.pool = (int)u.pool;
    b.epi.out = p->views[u.out];
    if (p->impl[i] == 5 && p->opt.band_pool && conv_ss_supported(b)) {
      a = b;
      continue;
    }
    if (u.pool == PCNN_POOL_LOCAL) {
      if (p->impl[i] == 3 && !conv_tc_supported(a)) p->impl[i] = 1;
    } else {
      // BI2 behind a halo-tile conv: conv_ss into scratch, then the bivariate pass
      a.pm.order = kPlain;
      a.epi.pool = PCNN_POOL_NONE;
      if (!conv_ss_supported(a))
        return fail(PCNN_ERR_UNSUPPORTED, "unit " + std::to_string(i) + ": pooled halo-tile conv");
    }
    fallback.push_back(i);
    const TensorView& o = p->views[u.out];
    need += (size_t)p->batch * o.cpad() * a.pm.ho * a.pm.wo;
  }
  if (fallback.empty()) return PCNN_OK;
  if (cudaMalloc(&p->scratch, need * sizeof(float)) != cudaSuccess)
    return fail(PCNN_ERR_CUDA, "local-pool scratch allocation failed");
  size_t off = 0;
  for (int i : fallback) {
    const pcnn_unit_desc& u = p->units[i];
    ConvArgs& a = p->conv_args[i];
    const TensorView& o = p->views[u.out];
    TensorView t = o;
    t.base = p->scratch + off;
    t.h = a.pm.ho;
    t.w = a.pm.wo;
    t.split = 0;
    t.flag = nullptr;
    off += (size_t)p->batch * o.cpad() * t.h * t.w;
    const int kind = (int)u.pool;
    if (kind == PCNN_POOL_LOCAL && p->impl[i] == 5 && p->opt.scratch_cb4 && o.cpad() % 16 == 0) {
      // halo-tile conv -> local pool: the scratch map in 4-channel blocks, so
      // the epilogue's row-per-lane stores are contiguous across a warp
      // (store16_any) and the pool pass reads 16 bytes per pixel per thread
      t.cb = 4;
      t.cbs = 2;
      t.nblk = o.cpad() / 4;
    }
    a.epi.out = t;
    a.epi.pool = PCNN_POOL_NONE;
    a.pm.order = kPlain;
    EltArgs& e = p->post_pool[i];
    e.kind = PCNN_UNIT_LOCALPOOL;
    e.batch = p->batch;
    e.in = t;
    e.out = o;
    e.p = a.epi.pool_p;
    e.stride = o.cpad();
    if (kind == PCNN_POOL_BI2) {  // bipool2_kernel: the 2x2 window through both bivariate stages
      e.k = 2;
      e.st = 2;
      e.pad = 0;
      e.pool = PCNN_POOL_BI2;
      e.deg = a.epi.pool_deg;
      e.axis = a.epi.pool_order;
    } else {
      e.k = a.epi.pool_k;
      e.st = a.epi.pool_s;
      e.pad = a.epi.pool_pad;
      e.pool = PCNN_POOL_NONE;
    }
    p->has_post_pool[i] = 1;
    p->launches += 1;
  }
  return PCNN_OK;
}

// Image-resident runs: maximal sequences of consecutive halo-tile convs, each
// reading the previous one's output, stride 1, 3x3, C = 32 or 64 channels
// in and out, the same small image (whole-image slots fit shared memory), no
// pools but a global pool on the last unit, every residual either produced
// inside the run or one of the two external tensors (the first unit's input
// and residual), and every output but the last read only inside the run.
// Slots are assigned greedily by liveness (a tensor's slot is free after its
// last reader); the run then computes in ONE conv_blk_kernel launch.
void build_blocks(pcnn_plan* p) {
  const int n = (int)p->units.size();
  p->blk_of.assign(n, -1);
  if (!p->opt.image_blocks || p->flags_on) return;
  std::vector<std::vector<int>> readers(p->tensors.size());
  for (int i = 0; i < n; ++i) {
    const pcnn_unit_desc& u = p->units[i];
    if (u.in >= 0) readers[u.in].push_back(i);
    if (u.in2 >= 0) readers[u.in2].push_back(i);
  }
  auto eligible = [&](int i) {
    const pcnn_unit_desc& u = p->units[i];
    if (u.kind != PCNN_UNIT_CONV || p->impl[i] != 5 || p->fused[i]) return false;
    const ConvArgs& a = p->conv_args[i];
    return a.kh == 3 && a.kw == 3 && a.stride == 1 && a.pad == 1 && !a.proj && a.in.split == 1 && !a.sk_flags &&
           (a.npad == 16 || a.npad == 32 || a.npad == 64) && u.cout == a.npad &&
           // a narrow input (ResNet-20's 3-channel stem: one 8-channel group) can only head a 16-channel run
           (a.in.cpad() == a.npad || (a.npad == 16 && a.in.cpad() <= 8 && !(p->opt.debug & 16384)));
  };
  int i = 0;
  while (i < n) {
    if (!eligible(i)) { ++i; continue; }
    const ConvArgs& a0 = p->conv_args[i];
    int j = i + 1;
    while (j < n && j - i < 7 && eligible(j) && p->units[j].in == p->units[j - 1].out &&
           p->conv_args[j].in.h == a0.in.h && p->conv_args[j].in.w == a0.in.w &&
           p->conv_args[j].npad == a0.npad && p->conv_args[j - 1].epi.pool == PCNN_POOL_NONE)
      ++j;
    // shrink until every condition holds
    bool done = false;
    for (; j - i >= 2; --j) {
      const int m = j - i;
      const int64_t ext_in = p->units[i].in, ext_res = p->units[i].residual ? p->units[i].in2 : -1;
      bool ok = p->conv_args[j - 1].epi.pool == PCNN_POOL_NONE || p->conv_args[j - 1].epi.pool == PCNN_POOL_GLOBAL;
      for (int k = i; k < j && ok; ++k) {
        if (k < j - 1)
          for (int rd : readers[p->units[k].out]) ok &= rd > k && rd < j;  // consumed inside the run only
        if (k > i && p->units[k].residual) {
          const int64_t t = p->units[k].in2;
          bool inside = t == ext_in || t == ext_res;
          for (int q = i; q < k; ++q) inside |= p->units[q].out == t;
          ok &= inside;
        }
        if (k < j - 1) ok &= p->conv_args[k].epi.pool == PCNN_POOL_NONE;
      }
      if (!ok) continue;
      // liveness: last unit (index in the run) reading each tensor
      std::vector<int64_t> tens;
      std::vector<int> last_use;
      auto idx = [&](int64_t t) {
        for (size_t q = 0; q < tens.size(); ++q)
          if (tens[q] == t) return (int)q;
        tens.push_back(t);
        last_use.push_back(-1);
        return (int)tens.size() - 1;
      };
      idx(ext_in);
      if (ext_res >= 0) idx(ext_res);
      for (int k = 0; k < m; ++k) {
        const pcnn_unit_desc& u = p->units[i + k];
        last_use[idx(u.in)] = k;
        if (u.residual) last_use[idx(u.in2)] = k;
        if (k < m - 1) idx(u.out);
      }
      // two slots when every residual's last reader writes over it in
      // place (the epilogue thread reads position p's residual, then writes
      // p), else three
      for (int nslots = 2; nslots <= 3; ++nslots) {
      std::vector<int64_t> holder(nslots, -1);
      std::vector<int> slot_of(tens.size(), -1);
      auto place = [&](int64_t t, int k) {
        for (int sidx = 0; sidx < nslots; ++sidx) {
          const int64_t h = holder[sidx];
          if (h < 0 || last_use[idx(h)] < k) {
            holder[sidx] = t;
            slot_of[idx(t)] = sidx;
            return sidx;
          }
        }
        return -1;
      };
      int ext_in_slot = place(ext_in, 0), ext_res_slot = ext_res >= 0 ? place(ext_res, 0) : -1;
      std::vector<int> in_s(m), res_s(m), out_s(m), kind(m, 0);
      for (int k = 0; k < m; ++k) {
        const pcnn_unit_desc& u = p->units[i + k];
        kind[k] = (u.in == ext_in ? 1 : 0) |
                  (u.residual ? (u.in2 == ext_in ? 1 : (u.in2 == ext_res ? 2 : 0)) << 2 : 0);
      }
      bool fit = ext_in_slot >= 0 && (ext_res < 0 || ext_res_slot >= 0);
      for (int k = 0; k < m && fit; ++k) {
        const pcnn_unit_desc& u = p->units[i + k];
        in_s[k] = slot_of[idx(u.in)];
        res_s[k] = u.residual ? slot_of[idx(u.in2)] : -1;
        if (k == m - 1) {
          out_s[k] = -1;
        } else {
          // the output may not take its input's slot, and takes its
          // residual's only when this unit is the residual's last reader
          int sl = -1;
          for (int sidx = 0; sidx < nslots; ++sidx) {
            const int64_t h = holder[sidx];
            if (sidx == in_s[k]) continue;
            if (sidx == res_s[k] ? last_use[idx(h)] == k : (h < 0 || last_use[idx(h)] < k)) { sl = sidx; break; }
          }
          if (sl < 0) { fit = false; break; }
          holder[sl] = u.out;
          slot_of[idx(u.out)] = sl;
          out_s[k] = sl;
        }
      }
      if (!fit) continue;
      std::vector<ConvArgs> layers(p->conv_args.begin() + i, p->conv_args.begin() + j);
      BlkRun* r = blk_create(layers.data(), m, in_s.data(), res_s.data(), out_s.data(), kind.data(), nslots, ext_in_slot,
                             ext_res_slot, p->views[ext_in], ext_res >= 0 ? p->views[ext_res] : p->views[ext_in],
                             p->status_dev, p->batch, (int)p->opt.image_blocks);
      if (!r) continue;
      const int id = (int)p->blks.size();
      p->blks.push_back(r);
      p->blk_first.push_back(i);
      for (int k = i; k < j; ++k) p->blk_of[k] = id;
      p->launches -= m - 1;
      done = true;
      break;
      }
      if (done) break;
    }
    i = j > i + 1 ? j : i + 1;
  }
}

// A residual block's 1x1 projection (unit i + 1) reads the same input with
// the same stride as the block's first 3x3 conv (unit i): on the halo-tile
// kernel its A operand is the 3x3 conv's centre tap, so the 3x3 launch
// computes it too (two more MMAs per chunk, its own epilogue items and
// output) and the projection's launch -- mostly fill / drain latency at
// these sizes -- disappears.  PCNN_NO_PROJ_FUSE=1 keeps separate launches.
// Small sequential networks (LeNet-5-shaped) as ONE launch (net_fused.cu):
// ingest, then convs (no residual; any kernel / stride / pad; fused poly and
// SUM2 / BI2 / local / global pools) and dense layers each reading the unit
// before it, then copyout.  Only where the launch chain, not arithmetic,
// bounds the forward: <= 2 M conv + dense MACs per image, and an image's
// activations fit in shared memory.
void build_net(pcnn_plan* p) {
  if (!p->opt.fused_net) return;
  const int n = (int)p->units.size();
  if (n < 3 || p->units[0].kind != PCNN_UNIT_INGEST || (p->units[0].flags & PCNN_FLAG_S2D) ||
      p->units[n - 1].kind != PCNN_UNIT_COPYOUT || n - 2 > kNetMaxOps)
    return;
  NetParams& NP = p->net;
  NP = NetParams();
  int64_t top = 0;
  bool ok = true;
  auto alloc = [&](int64_t floats) {
    const int64_t off = top;
    top += (floats + 3) & ~int64_t(3);
    return (int)off;
  };
  // a parameter block staged into shared memory by the kernel's prologue
  auto stage = [&](const float* src, int64_t floats) -> int {
    if (!src) return -1;
    if (NP.ncopies == kNetMaxCopies) {
      ok = false;
      return -1;
    }
    if (reinterpret_cast<uintptr_t>(src) & 15) {
      ok = false;
      return -1;
    }
    const int off = alloc(floats);
    NP.cp[NP.ncopies++] = NetCopy{src, off, (int)floats, NP.nops - 1};
    return off;
  };
  const pcnn_tensor_desc& ti = p->tensors[p->units[0].out];
  NP.in_elems = (int)(ti.c * ti.h * ti.w);
  NP.act_off = alloc(NP.in_elems);
  int cur_t = (int)p->units[0].out, cur_off = NP.act_off;
  double macs = 0;
  for (int i = 1; i < n - 1; ++i) {
    const pcnn_unit_desc& u = p->units[i];
    if (u.in != cur_t) return;  // not a chain
    NetOp& o = NP.op[NP.nops++];
    o = NetOp();
    const pcnn_tensor_desc& tin = p->tensors[u.in];
    const pcnn_tensor_desc& tout = p->tensors[u.out];
    o.in_off = cur_off;
    o.aff = o.poly = o.pool_p = o.in_div = -1;
    if (u.kind == PCNN_UNIT_CONV) {
      const ConvArgs& a = p->conv_args[i];
      if (u.residual || u.impl != 0) return;  // a requested kernel keeps its own launch
      o.kind = kNetConv;
      o.c = (int)tin.c; o.h = (int)tin.h; o.w = (int)tin.w;
      o.kh = a.kh; o.kw = a.kw; o.stride = a.stride; o.pad = a.pad;
      o.cb = a.in.cb; o.kp = a.kp;
      o.co = (int)u.cout;
      o.ho = a.pm.ho; o.wo = a.pm.wo;
      o.npad = a.epi.npad; o.poly_deg = a.epi.poly_deg; o.poly_stride = a.epi.npad;
      o.pool = (int)u.pool;
      o.pool_deg = a.epi.pool_deg; o.pool_order = a.epi.pool_order;
      o.pool_k = a.epi.pool_k; o.pool_s = a.epi.pool_s; o.pool_pad = a.epi.pool_pad;
      o.ph = (int)tout.h; o.pw = (int)tout.w;
      if (o.pool == PCNN_POOL_SUM2 || o.pool == PCNN_POOL_BI2) {
        if (o.ph != o.ho / 2 || o.pw != o.wo / 2) return;
      } else if (o.pool == PCNN_POOL_GLOBAL) {
        if (!tout.is_vector) return;
      } else if (o.pool != PCNN_POOL_NONE && o.pool != PCNN_POOL_LOCAL) {
        return;
      }
      o.wt = stage(a.w, (int64_t)o.co * o.kp);
      o.bias = stage(a.epi.bias, o.co);
      if (a.epi.aff) o.aff = stage(a.epi.aff, 2 * (int64_t)o.npad);
      if (o.poly_deg) o.poly = stage(a.epi.poly, (int64_t)(o.poly_deg + 1) * o.npad);
      if (o.pool)
        o.pool_p = stage(a.epi.pool_p, o.pool == PCNN_POOL_BI2 ? 2 * (int64_t)(o.pool_deg + 1) * (o.pool_deg + 1) * o.npad : 1);
      const int hwo = o.ho * o.wo;
      o.cpi = ((o.co + 3) / 4) * hwo >= kNetThreads ? 4 : ((o.co + 1) / 2) * hwo >= kNetThreads ? 2 : 1;
      if (o.pool) o.scratch_off = alloc((int64_t)o.co * o.ho * o.wo);
      o.out_off = alloc(o.pool == PCNN_POOL_GLOBAL ? o.co : (int64_t)o.co * o.ph * o.pw);
      macs += (double)o.co * o.ho * o.wo * o.c * o.kh * o.kw;
    } else if (u.kind == PCNN_UNIT_LINEAR) {
      o.kind = kNetLinear;
      o.in_mode = (int)u.in_mode;
      if (o.in_mode < 0 || o.in_mode > 2) return;
      o.c = (int)tin.c; o.h = (int)tin.h; o.w = (int)tin.w;
      o.n_in = (int)u.cin; o.n_out = (int)u.cout;
      if (o.in_mode == 1 && o.n_in != o.c * o.h * o.w) return;
      if (o.in_mode != 1 && o.n_in != o.c) return;
      if (!P(p, u.w_off) || !P(p, u.b_off)) return;
      o.poly_deg = (int)u.poly_deg;
      o.poly_stride = p->views[u.out].cpad();
      o.wt = stage(P(p, u.w_off), (int64_t)o.n_in * o.n_out);
      o.bias = stage(P(p, u.b_off), o.n_out);
      if (o.poly_deg) o.poly = stage(P(p, u.poly_off), (int64_t)(o.poly_deg + 1) * o.poly_stride);
      if (o.in_mode == 2) o.in_div = stage(P(p, u.in_div_off), 1);
      if (o.in_mode == 2) o.scratch_off = alloc(o.n_in);
      o.out_off = alloc(o.n_out);
      macs += (double)o.n_in * o.n_out;
    } else {
      return;
    }
    cur_t = (int)u.out;
    cur_off = o.out_off;
  }
  if (!ok || p->units[n - 1].in != cur_t || !p->tensors[cur_t].is_vector) return;
  if (macs > 2e6 || (size_t)top * sizeof(float) > 220 * 1024) return;
  NP.out_off = cur_off;
  NP.n_out = (int)p->tensors[cur_t].c;
  NP.out_pad = p->views[cur_t].cpad();
  NP.out_ws = p->views[cur_t].base;
  NP.batch = p->batch;
  NP.smem_floats = (int)top;
  int nsm = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  p->net_grid = std::min(p->batch, nsm);
  p->net_on = true;
  p->launches = 1;
}

void fuse_projections(pcnn_plan* p) {
  const int n = (int)p->units.size();
  p->fused.assign(n, 0);
  for (int i = 0; i + 1 < n; ++i) {
    const pcnn_unit_desc &u = p->units[i], &v = p->units[i + 1];
    if (u.kind != PCNN_UNIT_CONV || v.kind != PCNN_UNIT_CONV || p->impl[i] != 5 || p->impl[i + 1] != 5) continue;
    if (p->fused[i]) continue;
    if (v.in != u.in || v.kh != 1 || v.stride != u.stride || u.kh != 3) continue;
    if (p->prezeroed[i] || p->prezeroed[i + 1] || (i + 2 < n && p->prezeroed[i + 2])) continue;
    if (p->conv_args[i].prezero || p->conv_args[i + 1].prezero) continue;
    if (!conv_ss_proj_ok(p->conv_args[i], p->conv_args[i + 1])) continue;
    p->conv_args[i].proj = &p->conv_args[i + 1];
    p->fused[i + 1] = 1;
    p->launches -= 1;
  }
  // a linear unit whose vector output only the final copyout reads writes
  // the logits directly (one launch less)
  for (int i = 0; i + 1 < n; ++i) {
    const pcnn_unit_desc &u = p->units[i], &v = p->units[i + 1];
    if (u.kind != PCNN_UNIT_LINEAR || v.kind != PCNN_UNIT_COPYOUT || v.in != u.out) continue;
    const TensorView& t = p->views[u.out];
    if (!t.is_vector || t.c != (int)u.cout || !p->opt.linear_out) continue;
    p->fused[i + 1] = 1;
    p->launches -= 1;
  }
}

// Stream-K for halo-tile convs whose tiles fill the grid's last round badly
// (RN20 stage 3: 163 tiles on 148 SMs; RN18 stages 3-4; VGG's 8x8 .. 2x2
// layers): the (tile, chunk) units are spread evenly over all SMs, partial
// tiles meet in per-CTA slots (conv_ss.cu seg_at).  One slot buffer serves
// every such unit (launches are ordered by griddepcontrol.wait); each unit
// has its own CTA flags, zeroed at the start of the forward.
// PCNN_NO_STREAMK=1 keeps whole tiles.
void plan_streamk(pcnn_plan* p) {
  if (p->flags_on) return;  // flag-synchronised launches keep whole tiles
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int n = (int)p->units.size();
  std::vector<int> want(n, 0);
  size_t slot_max = 0, nflags = 0;
  for (int i = 0; i < n; ++i) {
    if (p->units[i].kind != PCNN_UNIT_CONV || p->impl[i] != 5 || p->fused[i]) continue;
    size_t slot = 0;
    if (!conv_ss_streamk_wanted(p->conv_args[i], nsm, &slot)) continue;
    want[i] = 1;
    slot_max = std::max(slot_max, slot);
    nflags += (size_t)nsm;
  }
  if (!nflags) return;
  if (cudaMalloc(&p->sk_flags, sizeof(int) * nflags) != cudaSuccess ||
      cudaMalloc(&p->sk_slots, sizeof(float) * slot_max * (size_t)nsm) != cudaSuccess) {
    if (p->sk_flags) cudaFree(p->sk_flags);
    p->sk_flags = nullptr;
    return;
  }
  cudaMemset(p->sk_flags, 0, sizeof(int) * nflags);
  p->sk_flags_n = nflags;
  size_t off = 0;
  for (int i = 0; i < n; ++i)
    if (want[i]) {
      p->conv_args[i].sk_flags = p->sk_flags + off;
      p->conv_args[i].sk_slots = p->sk_slots;
      off += (size_t)nsm;
    }
}

// Flag-synchronised launches.  A halo-tile conv whose input and residual are
// both written by halo-tile convs skips griddepcontrol.wait: its producer
// warp waits, tile by tile, for the producer tiles covering the input range
// it is about to copy, and its epilogue for the tiles holding the residual
// rows it reads.  Every halo-tile conv signals (per epilogue warp and tile,
// after its stores).  So a layer's first tiles start while the previous
// layer's last tiles (and the launch gap) are still in flight.  Deadlock-free:
// a grid is scheduled only after every CTA of the previous grid has started
// (griddepcontrol.launch_dependents right after the prologue), so the
// producers any waiting CTA depends on are resident and make progress.
// Units that still use griddepcontrol.wait only see their immediate
// predecessor complete, so the plan keeps flags off unless every tensor such
// a unit reads from a signalling conv was written by that predecessor.
// Opt-in (PCNN_FLAGS=1): measured on B200 RN20 b256 0.342 ms vs 0.323 ms
// with griddepcontrol ordering -- with one CTA per SM a layer's CTA still
// starts only when the SM's previous CTA exits, so the overlap is small, and
// the GPU-scope release per tile costs more than it saves (0.324 ms with a
// relaxed, i.e. unordered, signal: the overlap alone gains nothing).
void build_flags(pcnn_plan* p) {
  p->flags_on = false;
  // debug bits 2 / 4 skip the MMAs / the epilogue (no signals)
  if (!p->opt.flag_sync || (p->opt.debug & 6)) return;
  const int n = (int)p->units.size();
  std::vector<int> producer(p->tensors.size(), -1);
  for (int i = 0; i < n; ++i)
    if (p->units[i].out >= 0) producer[p->units[i].out] = p->fused[i] ? i - 1 : i;
  std::vector<char> sig(n, 0), skip(n, 0);
  std::vector<FlagDep> geo(n);
  size_t total = 0;
  std::vector<size_t> off(n, 0);
  for (int i = 0; i < n; ++i) {
    if (p->units[i].kind != PCNN_UNIT_CONV || p->impl[i] != 5 || p->fused[i]) continue;
    if (!conv_ss_flag_geometry(p->conv_args[i], geo[i])) continue;
    sig[i] = 1;
    off[i] = total;
    total += (size_t)geo[i].m_tiles + 1;
  }
  if (!total) return;
  for (int i = 0; i < n; ++i) {
    if (!sig[i]) continue;
    const pcnn_unit_desc& u = p->units[i];
    const int pin = producer[u.in];
    const int psk = u.residual ? producer[u.in2] : -1;
    skip[i] = pin >= 0 && sig[pin] && (!u.residual || (psk >= 0 && sig[psk]));
    if (p->prezeroed[i] && pin != i - 1) skip[i] = 0;  // its sums are zeroed by unit i - 1
  }
  // every griddepcontrol.wait unit reading a signalling conv's output must
  // read it from its immediate predecessor
  for (int i = 0; i < n; ++i) {
    if (skip[i] || p->fused[i]) continue;
    const pcnn_unit_desc& u = p->units[i];
    for (int64_t t : {(int64_t)u.in, (int64_t)u.in2}) {
      if (t < 0 || t >= (int64_t)producer.size()) continue;
      const int q = producer[t];
      if (q >= 0 && sig[q] && q != i - 1) return;
    }
  }
  if (cudaMalloc(&p->flags_dev, sizeof(int) * total) != cudaSuccess) return;
  cudaMemset(p->flags_dev, 0, sizeof(int) * total);
  p->flags_n = total;
  // same-grid stride-1 producer and consumer: wait per tile range, else all tiles
  auto same_grid = [&](int q, int64_t t, const pcnn_unit_desc& u) {
    const pcnn_unit_desc& uq = p->units[q];
    const TensorView& tv = p->views[t];
    const TensorView& qi = p->views[uq.in];
    return u.stride == 1 && uq.stride == 1 && tv.split == 1 && qi.h == tv.h && qi.w == tv.w &&
           p->views[u.in].h == tv.h && p->views[u.in].w == tv.w;
  };
  for (int i = 0; i < n; ++i) {
    if (!sig[i]) continue;
    ConvArgs& a = p->conv_args[i];
    a.sig_done = p->flags_dev + off[i];
    if (!skip[i]) continue;
    const pcnn_unit_desc& u = p->units[i];
    a.skip_gridwait = 1;
    const int pin = producer[u.in];
    a.fin = geo[pin];
    a.fin.done = p->flags_dev + off[pin];
    a.fin.mode = (same_grid(pin, u.in, u) && !p->prezeroed[i]) ? 1 : 2;
    if (u.residual) {
      const int psk = producer[u.in2];
      a.fsk = geo[psk];
      a.fsk.done = p->flags_dev + off[psk];
      a.fsk.mode = same_grid(psk, u.in2, u) ? 1 : 2;
    }
  }
  p->flags_on = true;
}

}  // namespace

extern "C" {

int pcnn_abi_version(void) { return PCNN_ABI_VERSION; }

const char* pcnn_last_error(void) { return g_last_error.c_str(); }

int pcnn_device_ok(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return 0;
  int dev = 0, major = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  return major == 10 ? 1 : 0;
}

size_t pcnn_workspace_bytes(const pcnn_tensor_desc* tensors, int n_tensors, int batch) {
  int64_t end = 0;
  for (int i = 0; i < n_tensors; ++i) end = std::max(end, tensors[i].offset + tensor_floats(tensors[i], batch));
  return (size_t)end * sizeof(float);
}

void pcnn_plan_options_default(pcnn_plan_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->size = sizeof(*o);
  o->split = 1;
  o->halo_tiles = 1;
  o->fuse_projection = 1;
  o->band_pool = 0;  // measured slower than conv + pool pass on RN18 / VGG
  o->streamk = 1;
  o->streamk_fill = 0.3;
  o->flag_sync = 0;
  o->prezero = 1;
  o->linear_out = 1;
  o->pdl = 1;
  o->graph = 1;
  o->ss_mt = 0;
  o->ss_share = -1;
  o->ss_psub = -1;
  o->ss_wres = 1;
  o->tc_stage = 1;
  o->timeline = 1;
  o->image_blocks = 2;
  o->debug = 0;
  o->fused_net = 1;
  o->ss_wide = 1;
  o->epi_pairs = 2;
  o->scratch_cb4 = 0;  // measured: LSU wavefronts of the stem -57 %, step time unchanged
  o->ss_pair = 1;
}

int pcnn_plan_create(const pcnn_unit_desc* units, int n_units, const pcnn_tensor_desc* tensors, int n_tensors,
                     int batch, int input_tensor, int output_tensor, const float* params, void* workspace,
                     size_t ws_bytes, pcnn_plan** plan_out) {
  return pcnn_plan_create_ex(units, n_units, tensors, n_tensors, batch, input_tensor, output_tensor, params,
                             workspace, ws_bytes, nullptr, plan_out);
}

int pcnn_plan_create_ex(const pcnn_unit_desc* units, int n_units, const pcnn_tensor_desc* tensors, int n_tensors,
                        int batch, int input_tensor, int output_tensor, const float* params, void* workspace,
                        size_t ws_bytes, const pcnn_plan_options* opt, pcnn_plan** plan_out) {
  if (!units || !tensors || n_units <= 0 || n_tensors <= 0 || batch <= 0 || !plan_out || !params || !workspace)
    return fail(PCNN_ERR_INVALID, "pcnn_plan_create: null or empty argument");
  if (input_tensor < 0 || input_tensor >= n_tensors || output_tensor < 0 || output_tensor >= n_tensors)
    return fail(PCNN_ERR_INVALID, "pcnn_plan_create: input / output tensor id out of range");
  if (opt && opt->size != (int64_t)sizeof(pcnn_plan_options))
    return fail(PCNN_ERR_INVALID, "pcnn_plan_create: options size mismatch (use pcnn_plan_options_default)");
  if (!pcnn_device_ok()) return fail(PCNN_ERR_NO_DEVICE, "no compute capability 10.x device");
  if (pcnn_workspace_bytes(tensors, n_tensors, batch) > ws_bytes)
    return fail(PCNN_ERR_INVALID, "workspace too small");
  pcnn_plan* p = new pcnn_plan();
  if (opt) p->opt = *opt;
  else pcnn_plan_options_default(&p->opt);
  p->kopt.pdl = (int)p->opt.pdl;
  p->kopt.ss_mt = (int)p->opt.ss_mt;
  p->kopt.ss_share = (int)p->opt.ss_share;
  p->kopt.ss_psub = (int)p->opt.ss_psub;
  p->kopt.ss_wres = (int)p->opt.ss_wres;
  p->kopt.ss_wide = (int)p->opt.ss_wide;
  p->kopt.epi_pairs = (int)p->opt.epi_pairs;
  p->kopt.ss_pair = p->opt.flag_sync ? 0 : (int)p->opt.ss_pair;
  p->kopt.tc_stage = (int)p->opt.tc_stage;
  p->kopt.proj_fuse = (int)p->opt.fuse_projection;
  p->kopt.streamk = (int)p->opt.streamk;
  p->kopt.streamk_fill = (float)p->opt.streamk_fill;
  p->kopt.dbg = (int)p->opt.debug;
  p->units.assign(units, units + n_units);
  p->tensors.assign(tensors, tensors + n_tensors);
  p->batch = batch;
  p->input = input_tensor;
  p->output = output_tensor;
  p->params = params;
  p->ws = static_cast<float*>(workspace);
  p->ws_bytes = ws_bytes;
  for (auto& t : p->tensors) {
    if (!(t.cb == 4 || t.cb == 8 || t.cb == 16 || t.cb == 32) || t.nblk * t.cb < t.c ||
        (t.is_vector && (t.h != 1 || t.w != 1))) {
      pcnn_plan_destroy(p);
      return fail(PCNN_ERR_INVALID, "tensor block size must be 4, 8, 16 or 32");
    }
    p->views.push_back(make_view(t, p->ws));
  }
  {
    const pcnn_tensor_desc& ti = p->tensors[input_tensor];
    p->in_elems = ti.c * ti.h * ti.w;
    for (const auto& u : p->units)
      if (u.kind == PCNN_UNIT_INGEST && u.out == input_tensor && (u.flags & PCNN_FLAG_S2D))
        p->in_elems = (ti.c / 4) * (2 * (ti.h - 1)) * (2 * (ti.w - 1));
  }
  p->impl.assign(n_units, 1);
  p->conv_args.resize(n_units);
  for (int i = 0; i < n_units; ++i) {
    const pcnn_unit_desc& u = p->units[i];
    auto bad = [&](int64_t id) { return id < -1 || id >= n_tensors; };
    if (bad(u.in) || bad(u.in2) || bad(u.out)) {
      pcnn_plan_destroy(p);
      return fail(PCNN_ERR_INVALID, "unit " + std::to_string(i) + ": tensor id out of range");
    }
    if (u.kind == PCNN_UNIT_CONV) {
      p->conv_args[i].opt = p->kopt;
      int rc = build_conv(p, i, p->conv_args[i]);
      if (rc != PCNN_OK) {
        pcnn_plan_destroy(p);
        return rc;
      }
      // auto: fp16x2 tensor cores, else 3xTF32, else SIMT; 4: auto without fp16x2
      ConvArgs& a = p->conv_args[i];
      if ((u.impl == 0 || u.impl == 3 || u.impl == 5) && a.tcw16 && a.tc16_scale) {
        a.f16 = 1;
        if (conv_tc_supported(a)) p->impl[i] = 3;
        else a.f16 = 0;
      }
      if (p->impl[i] == 1 && (u.impl == 0 || u.impl == 2 || u.impl == 4) && a.tcw && conv_tc_supported(a))
        p->impl[i] = 2;
      if (p->impl[i] == 1 && (u.impl == 2 || u.impl == 3 || u.impl == 5)) {
        pcnn_plan_destroy(p);
        return fail(PCNN_ERR_UNSUPPORTED, "unit " + std::to_string(i) + ": tcgen05 conv requested but unsupported");
      }
    }
    p->launches += 1;
  }
  if (cudaMalloc(&p->status_dev, sizeof(int)) != cudaSuccess ||
      cudaMallocHost(&p->status_host, sizeof(int)) != cudaSuccess) {
    pcnn_plan_destroy(p);
    return fail(PCNN_ERR_CUDA, "status allocation failed");
  }
  cudaMemset(p->status_dev, 0, sizeof(int));
  *p->status_host = 0;
  if (p->opt.timeline) {
    // slots [0, n): the units' launches; [n, 2n): a pooled conv's pooling pass
    const size_t tb = sizeof(unsigned long long) * 4 * (size_t)n_units;
    if (cudaMalloc(&p->tl_dev, tb) != cudaSuccess || cudaMallocHost(&p->tl_host, tb) != cudaSuccess) {
      pcnn_plan_destroy(p);
      return fail(PCNN_ERR_CUDA, "timeline allocation failed");
    }
    cudaMemset(p->tl_dev, 0, tb);
  }
  choose_formats(p);
  {
    const int rc = plan_local_pools(p);
    if (rc != PCNN_OK) {
      pcnn_plan_destroy(p);
      return rc;
    }
  }
  // a global-pool conv right after a halo-tile conv: that kernel zeroes the
  // sums in its prologue (keeps the launch chain free of memset nodes, which
  // would break programmatic dependent launch)
  p->prezeroed.assign(n_units, 0);
  for (int i = 1; i < n_units; ++i) {
    const pcnn_unit_desc& u = p->units[i];
    if (u.kind != PCNN_UNIT_CONV || u.pool != PCNN_POOL_GLOBAL) continue;
    if (p->impl[i - 1] != 5 || !p->opt.prezero) continue;
    ConvArgs& prev = p->conv_args[i - 1];
    prev.prezero = p->conv_args[i].epi.out.base;
    prev.prezero_n = (int64_t)p->batch * p->conv_args[i].epi.out.cpad();
    p->prezeroed[i] = 1;
  }
  fuse_projections(p);
  build_flags(p);
  plan_streamk(p);
  build_blocks(p);
  // a run ending in a global pool: its sums were prezeroed by the unit before
  // the pooled conv, which is now inside the run -- zero them before the run
  for (size_t r = 0; r < p->blks.size(); ++r) {
    int last = p->blk_first[r];
    while (last + 1 < n_units && p->blk_of[last + 1] == (int)r) ++last;
    if (p->prezeroed[last]) {
      p->prezeroed[last] = 0;
      p->conv_args[last - 1].prezero = nullptr;
      const int before = p->blk_first[r] - 1;
      int lb = before;
      while (lb > 0 && p->fused[lb]) --lb;  // the launch that computes unit `before`
      if (lb >= 0 && p->impl[lb] == 5 && p->units[lb].kind == PCNN_UNIT_CONV && !p->conv_args[lb].prezero &&
          (p->blk_of[lb] < 0)) {
        p->conv_args[lb].prezero = p->conv_args[last].epi.out.base;
        p->conv_args[lb].prezero_n = (int64_t)p->batch * p->conv_args[last].epi.out.cpad();
        p->prezeroed[last] = 1;
      }
    }
  }
  build_net(p);
  if (cudaStreamCreateWithFlags(&p->capture_stream, cudaStreamNonBlocking) != cudaSuccess) {
    pcnn_plan_destroy(p);
    return fail(PCNN_ERR_CUDA, "cudaStreamCreate failed");
  }
  *plan_out = p;
  return PCNN_OK;
}

int pcnn_plan_destroy(pcnn_plan* p) {
  if (!p) return PCNN_OK;
  for (auto& g : p->graphs) cudaGraphExecDestroy(g.exec);
  if (p->capture_stream) cudaStreamDestroy(p->capture_stream);
  if (p->status_dev) cudaFree(p->status_dev);
  if (p->tl_dev) cudaFree(p->tl_dev);
  if (p->tl_host) cudaFreeHost(p->tl_host);
  if (p->flags_dev) cudaFree(p->flags_dev);
  if (p->sk_flags) cudaFree(p->sk_flags);
  if (p->sk_slots) cudaFree(p->sk_slots);
  if (p->copy_stream) cudaStreamDestroy(p->copy_stream);
  if (p->out_stream) cudaStreamDestroy(p->out_stream);
  for (int i = 0; i < 2; ++i)
    for (cudaEvent_t e : {p->h2d_done[i], p->x_free[i], p->fwd_done[i], p->out_free[i]})
      if (e) cudaEventDestroy(e);
  if (p->logits2) cudaFree(p->logits2);
  if (p->status_slots) cudaFree(p->status_slots);
  if (p->status_pinned) cudaFreeHost(p->status_pinned);
  if (p->status_host) cudaFreeHost(p->status_host);
  if (p->scratch) cudaFree(p->scratch);
  for (BlkRun* b : p->blks) blk_destroy(b);
  delete p;
  return PCNN_OK;
}

int pcnn_plan_timeline(pcnn_plan* p, int64_t* ns, int max_units, void* stream) {
  if (!p || !ns || max_units < 0) return fail(PCNN_ERR_INVALID, "pcnn_plan_timeline: null argument");
  if (!p->tl_dev) return fail(PCNN_ERR_INVALID, "pcnn_plan_timeline: plan created without options.timeline");
  const int n = std::min(max_units, 2 * (int)p->units.size());
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  PCNN_CUDA(cudaMemcpyAsync(p->tl_host, p->tl_dev, sizeof(unsigned long long) * 2 * (size_t)n,
                            cudaMemcpyDeviceToHost, s));
  PCNN_CUDA(cudaStreamSynchronize(s));
  for (int i = 0; i < n; ++i) {
    const unsigned long long a = p->tl_host[2 * i], b = p->tl_host[2 * i + 1];
    ns[2 * i] = b ? (int64_t)~a : 0;
    ns[2 * i + 1] = (int64_t)b;
  }
  return n;
}

int pcnn_plan_unit_launch(const pcnn_plan* p, int unit) {
  if (!p || unit < 0 || unit >= (int)p->units.size()) return -1;
  int u = unit;
  if (p->net_on) return 0;  // one whole-network launch
  if (!p->blk_of.empty() && p->blk_of[u] >= 0) return p->blk_first[p->blk_of[u]];  // an image-resident run
  while (u > 0 && p->fused[u]) --u;  // a fused unit runs in its predecessor's launch
  return u;
}

int pcnn_plan_num_launches(const pcnn_plan* p) { return p ? p->launches : -1; }

// debugging aid (not part of pcnn.h): 1 if the plan runs flag-synchronised launches
int pcnn_plan_flags(const pcnn_plan* p) { return p && p->flags_on ? 1 : 0; }

int pcnn_plan_unit_impl(const pcnn_plan* p, int unit) {
  if (!p || unit < 0 || unit >= (int)p->units.size()) return -1;
  if (p->net_on) return 7;  // whole-network kernel (fp32 CUDA cores)
  if (!p->blk_of.empty() && p->blk_of[unit] >= 0) return 6;  // halo-tile arithmetic inside an image-resident run
  return p->impl[unit];
}

int pcnn_plan_tensor_split(const pcnn_plan* p, int tensor) {
  if (!p || tensor < 0 || tensor >= (int)p->views.size()) return -1;
  return p->views[tensor].split;
}

int pcnn_plan_status(pcnn_plan* p, void* stream) {
  if (!p) return fail(PCNN_ERR_INVALID, "pcnn_plan_status: null plan");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  PCNN_CUDA(cudaMemcpyAsync(p->status_host, p->status_dev, sizeof(int), cudaMemcpyDeviceToHost, s));
  PCNN_CUDA(cudaStreamSynchronize(s));
  return *p->status_host;
}

int pcnn_plan_last_status(const pcnn_plan* p) { return p ? *p->status_host : -1; }

int pcnn_forward(pcnn_plan* p, const float* x, float* logits, void* stream, int use_graph) {
  if (!p || !x || !logits) return fail(PCNN_ERR_INVALID, "pcnn_forward: null argument");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // options.graph = 0: eager launches (ncu cannot replay the extended-launch
  // kernels inside a CUDA graph)
  if (!use_graph || !p->opt.graph) {
    enqueue_all(p, x, logits, s);
    PCNN_CUDA(cudaGetLastError());
    return PCNN_OK;
  }
  for (auto& g : p->graphs)
    if (g.x == x && g.logits == logits) {
      PCNN_CUDA(cudaGraphLaunch(g.exec, s));
      return PCNN_OK;
    }
  // capture on the plan's own stream (the legacy default stream cannot be
  // captured), then replay on the caller's stream
  cudaGraph_t graph;
  PCNN_CUDA(cudaStreamBeginCapture(p->capture_stream, cudaStreamCaptureModeThreadLocal));
  enqueue_all(p, x, logits, p->capture_stream);
  cudaError_t le = cudaGetLastError();
  PCNN_CUDA(cudaStreamEndCapture(p->capture_stream, &graph));
  if (le != cudaSuccess) {
    cudaGraphDestroy(graph);
    return fail(PCNN_ERR_CUDA, std::string("launch during capture: ") + cudaGetErrorString(le));
  }
  cudaGraphExec_t exec;
  cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ie != cudaSuccess) return fail(PCNN_ERR_CUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(ie));
  if (p->graphs.size() >= 4) {
    cudaGraphExecDestroy(p->graphs.front().exec);
    p->graphs.erase(p->graphs.begin());
  }
  p->graphs.push_back({x, logits, exec});
  PCNN_CUDA(cudaGraphLaunch(exec, s));
  return PCNN_OK;
}

int pcnn_forward_host(pcnn_plan* p, const float* x_host, float* logits_host, float* x_dev, float* logits_dev,
                      void* stream) {
  if (!p || !x_host || !logits_host || !x_dev || !logits_dev) return fail(PCNN_ERR_INVALID, "null argument");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t in_bytes = sizeof(float) * (size_t)p->batch * p->in_elems;
  const pcnn_tensor_desc& to = p->tensors[p->output];
  size_t out_bytes = sizeof(float) * (size_t)p->batch * to.c * to.h * to.w;
  PCNN_CUDA(cudaMemcpyAsync(x_dev, x_host, in_bytes, cudaMemcpyHostToDevice, s));
  int rc = pcnn_forward(p, x_dev, logits_dev, stream, 1);
  if (rc != PCNN_OK) return rc;
  PCNN_CUDA(cudaMemcpyAsync(logits_host, logits_dev, out_bytes, cudaMemcpyDeviceToHost, s));
  if (p->any_split) PCNN_CUDA(cudaMemcpyAsync(p->status_host, p->status_dev, sizeof(int), cudaMemcpyDeviceToHost, s));
  return PCNN_OK;
}

int pcnn_forward_host_many(pcnn_plan* p, const float* const* x_hosts, float* const* logits_hosts, int n,
                           float* x_dev0, float* x_dev1, float* logits_dev, int* statuses, void* stream) {
  if (!p || (n > 0 && (!x_hosts || !logits_hosts)) || !x_dev0 || !x_dev1 || !logits_dev || n < 0)
    return fail(PCNN_ERR_INVALID, "pcnn_forward_host_many: null argument");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t in_bytes = sizeof(float) * (size_t)p->batch * p->in_elems;
  const pcnn_tensor_desc& to = p->tensors[p->output];
  const size_t out_bytes = sizeof(float) * (size_t)p->batch * to.c * to.h * to.w;
  if (!p->copy_stream) {
    PCNN_CUDA(cudaStreamCreateWithFlags(&p->copy_stream, cudaStreamNonBlocking));
    PCNN_CUDA(cudaStreamCreateWithFlags(&p->out_stream, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i)
      for (cudaEvent_t* e : {&p->h2d_done[i], &p->x_free[i], &p->fwd_done[i], &p->out_free[i]})
        PCNN_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    PCNN_CUDA(cudaMalloc(&p->logits2, out_bytes));
  }
  if (p->status_pinned_n < n) {
    if (p->status_pinned) cudaFreeHost(p->status_pinned);
    if (p->status_slots) cudaFree(p->status_slots);
    p->status_pinned = nullptr;
    p->status_slots = nullptr;
    p->status_pinned_n = 0;
    // room to spare: a later, longer call does not pay a pinned allocation (~1 ms) again
    const int cap = n < 256 ? 256 : 2 * n;
    PCNN_CUDA(cudaMallocHost(&p->status_pinned, sizeof(int) * (size_t)cap));
    PCNN_CUDA(cudaMalloc(&p->status_slots, sizeof(int) * (size_t)cap));
    p->status_pinned_n = cap;
  }
  float* xd[2] = {x_dev0, x_dev1};
  float* ld[2] = {logits_dev, p->logits2};
  // Three streams: H2D (copy_stream) -> forward (stream) -> D2H (out_stream).
  // Buffers alternate; x_free / out_free say when a buffer may be reused.
  // Both side streams start after everything already queued on `stream`.
  for (int b = 0; b < 2; ++b) {
    PCNN_CUDA(cudaEventRecord(p->x_free[b], s));
    PCNN_CUDA(cudaEventRecord(p->out_free[b], s));
  }
  PCNN_CUDA(cudaStreamWaitEvent(p->out_stream, p->out_free[0], 0));
  for (int i = 0; i < n; ++i) {
    const int b = i & 1;
    PCNN_CUDA(cudaStreamWaitEvent(p->copy_stream, p->x_free[b], 0));
    PCNN_CUDA(cudaMemcpyAsync(xd[b], x_hosts[i], in_bytes, cudaMemcpyHostToDevice, p->copy_stream));
    PCNN_CUDA(cudaEventRecord(p->h2d_done[b], p->copy_stream));
    PCNN_CUDA(cudaStreamWaitEvent(s, p->h2d_done[b], 0));
    PCNN_CUDA(cudaStreamWaitEvent(s, p->out_free[b], 0));  // batch i - 2's logits are on the host
    const int rc = pcnn_forward(p, xd[b], ld[b], stream, 1);
    if (rc != PCNN_OK) return rc;
    if (p->any_split)
      PCNN_CUDA(cudaMemcpyAsync(p->status_slots + i, p->status_dev, sizeof(int), cudaMemcpyDeviceToDevice, s));
    PCNN_CUDA(cudaEventRecord(p->x_free[b], s));
    PCNN_CUDA(cudaEventRecord(p->fwd_done[b], s));
    PCNN_CUDA(cudaStreamWaitEvent(p->out_stream, p->fwd_done[b], 0));
    PCNN_CUDA(cudaMemcpyAsync(logits_hosts[i], ld[b], out_bytes, cudaMemcpyDeviceToHost, p->out_stream));
    PCNN_CUDA(cudaEventRecord(p->out_free[b], p->out_stream));
  }
  if (p->any_split && n)
    PCNN_CUDA(cudaMemcpyAsync(p->status_pinned, p->status_slots, sizeof(int) * (size_t)n, cudaMemcpyDeviceToHost,
                              p->out_stream));
  else
    for (int i = 0; i < n; ++i) p->status_pinned[i] = 0;
  // `stream` completes after the last D2H (callers time and synchronise it)
  PCNN_CUDA(cudaEventRecord(p->out_free[0], p->out_stream));
  PCNN_CUDA(cudaStreamWaitEvent(s, p->out_free[0], 0));
  if (statuses) {
    PCNN_CUDA(cudaStreamSynchronize(s));
    for (int i = 0; i < n; ++i) statuses[i] = p->status_pinned[i];
  }
  return PCNN_OK;
}

int pcnn_forward_unit(pcnn_plan* p, int unit, const float* x, float* logits, void* stream) {
  if (!p || unit < 0 || unit >= (int)p->units.size()) return fail(PCNN_ERR_INVALID, "bad unit");
  if (p->conv_args.size() > (size_t)unit && p->conv_args[unit].sk_flags) {  // run alone: fresh stream-K flags
    int dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaMemsetAsync(p->conv_args[unit].sk_flags, 0, sizeof(int) * nsm, static_cast<cudaStream_t>(stream));
  }
  if (p->prezeroed[unit]) {  // run alone: its global-pool sums need their own zeroing
    const ConvArgs& a = p->conv_args[unit];
    cudaMemsetAsync(a.epi.out.base, 0, sizeof(float) * (size_t)p->batch * a.epi.out.cpad(),
                    static_cast<cudaStream_t>(stream));
  }
  if (p->tl_dev)
    for (size_t slot : {(size_t)unit, p->units.size() + (size_t)unit})
      cudaMemsetAsync(p->tl_dev + 2 * slot, 0, 2 * sizeof(unsigned long long), static_cast<cudaStream_t>(stream));
  enqueue_unit(p, unit, x, logits, static_cast<cudaStream_t>(stream), false);
  PCNN_CUDA(cudaGetLastError());
  return PCNN_OK;
}

struct pcnn_packer {
  pcnn_pack_desc* d_ops = nullptr;
  int* d_first = nullptr;
  int n_ops = 0, blocks = 0;
  bool tc16 = false;
};

struct pcnn_program {
  char* d_tables = nullptr;  // ops then rewrites
  pcnn_scale_op* d_ops = nullptr;
  pcnn_rewrite_desc* d_rw = nullptr;
  int2* d_chunks = nullptr;  // phase-(b) work chunks {rewrite, first element}
  double* arena = nullptr;
  int64_t arena_len = 0;
  int n_ops = 0, n_rw = 0, n_chunks = 0;
  int smem_arena = 0, blocks = 0;
  size_t smem = 0;
};

int pcnn_packer_create(const pcnn_pack_desc* ops, int n_ops, pcnn_packer** out) {
  if (!out || (!ops && n_ops) || n_ops < 0) return fail(PCNN_ERR_INVALID, "pcnn_packer_create: bad argument");
  pcnn_packer* k = new pcnn_packer();
  k->n_ops = n_ops;
  std::vector<int> first(n_ops + 1, 0);
  for (int i = 0; i < n_ops; ++i) {
    k->tc16 |= ops[i].kind == PCNN_PACK_TC16_WEIGHTS;
    // work items of the op (the padded weight images cover rows x padded k)
    const int64_t work = std::max<int64_t>(std::max<int64_t>(ops[i].n, ops[i].rows * ops[i].k), 1);
    const int64_t nb = std::min<int64_t>((work + 256 * 8 - 1) / (256 * 8), 512);
    first[i + 1] = first[i] + (int)nb;
  }
  k->blocks = first[n_ops];
  if (n_ops) {
    if (cudaMalloc(&k->d_ops, sizeof(pcnn_pack_desc) * n_ops) != cudaSuccess ||
        cudaMalloc(&k->d_first, sizeof(int) * (n_ops + 1)) != cudaSuccess) {
      pcnn_packer_destroy(k);
      return fail(PCNN_ERR_CUDA, "pcnn_packer_create: allocation failed");
    }
    cudaMemcpy(k->d_ops, ops, sizeof(pcnn_pack_desc) * n_ops, cudaMemcpyHostToDevice);
    cudaMemcpy(k->d_first, first.data(), sizeof(int) * (n_ops + 1), cudaMemcpyHostToDevice);
  }
  *out = k;
  return PCNN_OK;
}

int pcnn_packer_run(pcnn_packer* k, const double* master, float* packed, void* stream) {
  if (!k || !master || !packed) return fail(PCNN_ERR_INVALID, "pcnn_packer_run: null argument");
  if (!k->n_ops) return PCNN_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (k->tc16) {
    // max|w| of every fp16x2 image first (its power-of-two scale)
    pack_amax_kernel<<<k->n_ops, 1024, 0, s>>>(master, packed, k->d_ops, k->n_ops, 0);
    pack_amax_kernel<<<dim3(k->n_ops, 64), 256, 0, s>>>(master, packed, k->d_ops, k->n_ops, 1);
  }
  pack_kernel<<<k->blocks, 256, 0, s>>>(master, packed, k->d_ops, k->n_ops, k->d_first);
  cudaError_t le = cudaGetLastError();
  if (le != cudaSuccess) return fail(PCNN_ERR_CUDA, std::string("pack_kernel: ") + cudaGetErrorString(le));
  return PCNN_OK;
}

int pcnn_packer_destroy(pcnn_packer* k) {
  if (!k) return PCNN_OK;
  if (k->d_ops) cudaFree(k->d_ops);
  if (k->d_first) cudaFree(k->d_first);
  delete k;
  return PCNN_OK;
}

int pcnn_pack(const double* master, float* packed, const pcnn_pack_desc* ops, int n_ops, void* stream) {
  if (!master || !packed || (!ops && n_ops)) return fail(PCNN_ERR_INVALID, "pcnn_pack: null argument");
  if (n_ops == 0) return PCNN_OK;
  pcnn_packer* k = nullptr;
  int rc = pcnn_packer_create(ops, n_ops, &k);
  if (rc != PCNN_OK) return rc;
  rc = pcnn_packer_run(k, master, packed, stream);
  cudaStreamSynchronize(static_cast<cudaStream_t>(stream));  // the tables are freed below
  pcnn_packer_destroy(k);
  return rc;
}

int pcnn_program_create(const pcnn_scale_op* ops, int n_ops, const pcnn_rewrite_desc* rewrites, int n_rewrites,
                        int64_t arena_len, pcnn_program** out) {
  if (!out || (!ops && n_ops) || (!rewrites && n_rewrites) || n_ops < 0 || n_rewrites < 0 || arena_len < 0)
    return fail(PCNN_ERR_INVALID, "pcnn_program_create: bad argument");
  for (int i = 0; i < n_ops; ++i) {
    const pcnn_scale_op& o = ops[i];
    if (o.op < PCNN_OP_FILL || o.op > PCNN_OP_ADD || o.n < 0 || o.dst < 0)
      return fail(PCNN_ERR_INVALID, "bad scale op " + std::to_string(i));
  }
  pcnn_program* g = new pcnn_program();
  g->n_ops = n_ops;
  g->n_rw = n_rewrites;
  g->arena_len = arena_len;
  std::vector<int2> chunks;
  for (int i = 0; i < n_rewrites; ++i) {
    const pcnn_rewrite_desc& r = rewrites[i];
    bool ok = r.n >= 0 && r.n < (int64_t(1) << 31) && r.n_factors >= 0 && r.n_factors <= PCNN_MAX_FACTORS;
    for (int f = 0; ok && f < (int)r.n_factors; ++f) {
      const pcnn_factor& F = r.f[f];
      ok = F.d1 > 0 && F.m1 > 0 && F.d2 > 0 && F.m2 > 0 && F.d1 < (int64_t(1) << 31) && F.m1 < (int64_t(1) << 31) &&
           F.d2 < (int64_t(1) << 31) && F.m2 < (int64_t(1) << 31) && F.s1 >= 0 &&
           (F.m1 - 1) * F.s1 + F.m2 < (int64_t(1) << 32);
    }
    if (!ok) {
      delete g;
      return fail(PCNN_ERR_INVALID, "bad rewrite descriptor " + std::to_string(i));
    }
    for (int64_t e = 0; e < r.n; e += 4096) chunks.push_back(make_int2(i, (int)e));
  }
  g->n_chunks = (int)chunks.size();
  const size_t ob = sizeof(pcnn_scale_op) * (size_t)std::max(n_ops, 1);
  const size_t rb = sizeof(pcnn_rewrite_desc) * (size_t)std::max(n_rewrites, 1);
  const size_t cb = sizeof(int2) * std::max<size_t>(chunks.size(), 1);
  if (cudaMalloc(&g->d_tables, ob + rb + cb) != cudaSuccess ||
      cudaMalloc(&g->arena, sizeof(double) * (size_t)std::max<int64_t>(arena_len, 1)) != cudaSuccess) {
    pcnn_program_destroy(g);
    return fail(PCNN_ERR_CUDA, "pcnn_program_create: allocation failed");
  }
  g->d_ops = reinterpret_cast<pcnn_scale_op*>(g->d_tables);
  g->d_rw = reinterpret_cast<pcnn_rewrite_desc*>(g->d_tables + ob);
  g->d_chunks = reinterpret_cast<int2*>(g->d_tables + ob + rb);
  if (!chunks.empty()) cudaMemcpy(g->d_chunks, chunks.data(), sizeof(int2) * chunks.size(), cudaMemcpyHostToDevice);
  if (n_ops) cudaMemcpy(g->d_ops, ops, sizeof(pcnn_scale_op) * n_ops, cudaMemcpyHostToDevice);
  if (n_rewrites) cudaMemcpy(g->d_rw, rewrites, sizeof(pcnn_rewrite_desc) * n_rewrites, cudaMemcpyHostToDevice);
  // the arena and the op table in block 0's shared memory when they fit
  const size_t need = sizeof(double) * (size_t)((arena_len + 1) & ~int64_t(1)) + sizeof(pcnn_scale_op) * (size_t)n_ops;
  g->smem_arena = arena_len > 0 && need <= 200 * 1024 ? 1 : 0;
  g->smem = g->smem_arena ? need : 0;
  if (g->smem > 48 * 1024)
    cudaFuncSetAttribute(redistribute_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g->smem);
  int dev = 0, nsm = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, redistribute_kernel, 256, g->smem);
  g->blocks = std::max(1, nsm * std::max(1, std::min(per_sm, 4)));
  *out = g;
  return PCNN_OK;
}

int pcnn_program_run(pcnn_program* g, double* master, int64_t* status_dev, int64_t* flags_dev, void* stream) {
  if (!g || !master || !status_dev) return fail(PCNN_ERR_INVALID, "pcnn_program_run: null argument");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  PCNN_CUDA(cudaMemsetAsync(status_dev, 0, 4 * sizeof(int64_t), s));
  int64_t* flags = flags_dev ? flags_dev : status_dev + 2;
  double* arena = g->arena;
  int64_t arena_len = g->arena_len;
  int smem_arena = g->smem_arena;
  void* args[] = {&master, &arena, &arena_len, &smem_arena, &g->d_ops, &g->n_ops, &g->d_rw, &g->n_rw,
                  &g->d_chunks, &g->n_chunks, &status_dev, &flags};
  cudaError_t le = cudaLaunchCooperativeKernel((void*)redistribute_kernel, dim3(g->blocks), dim3(256), args, g->smem, s);
  if (le != cudaSuccess) return fail(PCNN_ERR_CUDA, std::string("redistribute_kernel: ") + cudaGetErrorString(le));
  return PCNN_OK;
}

int pcnn_program_destroy(pcnn_program* g) {
  if (!g) return PCNN_OK;
  if (g->d_tables) cudaFree(g->d_tables);
  if (g->arena) cudaFree(g->arena);
  delete g;
  return PCNN_OK;
}

int pcnn_redistribute(double* master, double* arena, int64_t arena_len, const pcnn_scale_op* ops, int n_ops,
                      const pcnn_rewrite_desc* rewrites, int n_rewrites, int64_t* status_dev, int64_t* flags_dev,
                      void* stream) {
  if (!master || !arena || !status_dev || (!ops && n_ops) || (!rewrites && n_rewrites))
    return fail(PCNN_ERR_INVALID, "pcnn_redistribute: null argument");
  pcnn_program* g = nullptr;
  int rc = pcnn_program_create(ops, n_ops, rewrites, n_rewrites, arena_len, &g);
  if (rc != PCNN_OK) return rc;
  // the caller's arena, not the program's own
  cudaFree(g->arena);
  g->arena = arena;
  rc = pcnn_program_run(g, master, status_dev, flags_dev, stream);
  cudaStreamSynchronize(static_cast<cudaStream_t>(stream));  // the tables are freed below
  g->arena = nullptr;
  pcnn_program_destroy(g);
  return rc;
}

}  // extern "C"
