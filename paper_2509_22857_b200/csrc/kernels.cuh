// Kernel argument blocks and launchers (internal to libpcnn).
#pragma once

#include <algorithm>
#include <cstdlib>

#include "epilogue.cuh"

namespace pcnn {

// Flag-synchronised halo-tile launches: a consumer waits for the per-tile
// completion counters of the unit that wrote its input / residual instead of
// griddepcontrol.wait on the whole previous grid.  mode 1: the producer tiles
// covering a position range (same grid), 2: every tile.
struct FlagDep {
  const int* done = nullptr;  // producer counters [m_tiles] per tile, [m_tiles] all
  int mode = 0;               // 0 none
  int tm = 0, m_tiles = 0;    // producer tile rows, tiles
  int64_t gtotal = 0;         // producer grid positions
  int per_tile = 0, all = 0;  // counter values meaning "done"
};

// Per-plan kernel switches (from pcnn_plan_options; the library reads no
// environment variables)
struct KOpts {
  int pdl = 1;          // programmatic dependent launch
  int ss_mt = 0;        // halo-tile sub-tiles per tile (0 auto)
  int ss_share = -1;    // shared epilogue (-1 auto)
  int ss_psub = -1;     // parity-plane stages (-1 auto)
  int ss_wres = 1;      // resident weights
  int ss_wide = 1;      // halo-tile producer issues a stage's copies from many lanes (1: narrow layers, 2: all)
  int ss_pair = 1;      // halo-tile CTA pairs (cta_group::2) for 128-channel tiles
  int epi_pairs = 2;    // halo-tile epilogue warpgroup pairs (1 or 2)
  int tc_stage = 1;     // TMA-staged input boxes (TMEM-A kernel)
  int proj_fuse = 1;    // fused projections
  int streamk = 1;      // stream-K
  float streamk_fill = 0.3f;
  int dbg = 0;          // diagnostic bits (pcnn_plan_options.debug)
};

struct ConvArgs {
  TensorView in;
  PixelMap pm;
  int batch;
  int kh, kw, stride, pad;
  int kp;            // padded K = in.nblk * kh * kw * in.cb
  int npad;          // padded output channels
  const float* w;    // [npad][kp] float32
  const float* tcw;  // tcgen05 weight image (3xTF32) or null
  const float* tcw16;       // fp16x2 weight image or null
  const float* tc16_scale;  // {max|w|, 2^-e} of the fp16x2 image
  const float* tcwss;       // fp16x2 image of the shared-memory kernel or null
  int f16;                  // launch_conv_tc: 1 = fp16x2 (kind::f16), 0 = 3xTF32
  EpiParams epi;
  // halo-tile kernel: zero this buffer (the next unit's global-pool sums)
  // in the prologue, instead of a memset node between the two launches
  float* prezero = nullptr;
  int64_t prezero_n = 0;  // floats, a multiple of 4
  // flag-synchronised launches (api.cu build_flags; halo-tile kernel only)
  int* sig_done = nullptr;  // this unit's counters [m_tiles + 1], bumped after its stores
  int skip_gridwait = 0;    // every producer signals: no griddepcontrol.wait
  FlagDep fin, fsk;         // waits before reading the input / the residual
  // halo-tile kernel: a 1x1 conv with the same input and stride (a residual
  // block's projection) computed in the same launch from the centre tap's
  // A operand, into its own output (api.cu fuse_projections); or null
  const ConvArgs* proj = nullptr;
  // halo-tile kernel, stream-K (api.cu plan_streamk): the (tile, 16-channel
  // chunk) units are split evenly over the grid; a CTA whose range ends
  // inside a tile writes that tile's partial sums to its slot and sets its
  // flag, the CTA holding the tile's last chunk adds them before the
  // epilogue.  null: one whole tile per CTA turn.
  int* sk_flags = nullptr;    // [grid], zeroed at the start of every forward
  float* sk_slots = nullptr;  // [grid][items][128][16]
  KOpts opt;
  unsigned long long* tl = nullptr;  // launch timeline slot (common.cuh tl_mark) or null
};

struct LinearArgs {
  TensorView in;
  int in_mode, batch, n_in, n_out;
  const float* in_div;
  const float* w;
  const float* bias;
  int poly_deg;
  const float* poly;
  int64_t poly_stride;
  float* out;
  int64_t out_stride;
  // also the user's [batch][n_out] logits (the copyout unit folded in), or null
  float* out2 = nullptr;
  unsigned long long* tl = nullptr;
};

struct EltArgs {
  int kind, batch;
  TensorView in, in2, out;
  const float* p;
  int64_t stride;
  int deg, k, st, pad, axis;
  int pool = 0;  // LOCALPOOL: PCNN_POOL_BI2 = 2x2 window through two bivariate stages
  unsigned long long* tl = nullptr;
};

inline int64_t host_pixel_count(const PixelMap& pm, int batch) {
  return pm.order == kPlain ? (int64_t)batch * pm.ho * pm.wo : (int64_t)batch * pm.hp * pm.wp * 4;
}

// s2d: x is [B][C/4][2H][2W] and t holds it as 2x2 blocks, channel (dy*2+dx)*(C/4)+c
void launch_ingest(const float* x, const TensorView& t, int batch, bool s2d, cudaStream_t s, int pdl,
                   unsigned long long* tl = nullptr);
void launch_conv_simt(const ConvArgs& a, cudaStream_t s);
void launch_linear(const LinearArgs& a, cudaStream_t s, int pdl = 0);
void launch_eltwise(const EltArgs& a, cudaStream_t s, int pdl = 0);
void launch_copyout(const TensorView& t, float* dst, int batch, cudaStream_t s, unsigned long long* tl = nullptr,
                    int pdl = 0);

// Launch a persistent tcgen05 kernel with programmatic stream serialization:
// its prologue (barriers, TMEM allocation, parameter table) overlaps the tail
// of the previous kernel, and griddep_wait() in the kernel orders the data.
// pdl = 0 launches it plainly.
template <typename... Params, typename... Args>
inline void launch_pdl(void (*kernel)(Params...), dim3 grid, int threads, size_t smem, cudaStream_t s, int pdl,
                       Args... args) {
  const bool off = !pdl;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = off ? 0 : 1;
  cfg.attrs = at;
  cfg.numAttrs = off ? 0 : 1;
  cudaLaunchKernelEx(&cfg, kernel, args...);
}

// tcgen05 path (conv_tc.cu); returns false if the shape is not supported
bool conv_tc_supported(const ConvArgs& a);
void launch_conv_tc(const ConvArgs& a, cudaStream_t s);
void tc_weight_image_dims(int npad, int kp, int64_t* floats);

// fp16x2 conv with A from shared memory (conv_ss.cu): stride-1 3x3/1x1 convs
// reading a split tensor
bool conv_ss_supported(const ConvArgs& a);
// Image-resident residual runs (conv_ss.cu conv_blk_kernel): n consecutive
// stride-1 3x3 convs on one grid in one launch, activations in shared-memory
// slots; in/res/out_slot per layer (res -1: none, out -1: global), the run's
// external input / residual bulk-copied into ext_in_slot / ext_res_slot.
// nullptr if the layers do not fit.
struct BlkRun;
BlkRun* blk_create(const ConvArgs* layers, int n, const int* in_slot, const int* res_slot, const int* out_slot,
                   const int* src_kind, int nslots, int ext_in_slot, int ext_res_slot, const TensorView& ext_in,
                   const TensorView& ext_res, int* flag, int batch, int max_images);
void blk_launch(const BlkRun* r, cudaStream_t s, unsigned long long* tl, int pdl);
void blk_destroy(BlkRun* r);
// the shape/precision part of conv_ss_supported (input format not checked)
bool conv_ss_shape_ok(const ConvArgs& a);
void launch_conv_ss(const ConvArgs& a, cudaStream_t s);
// tile geometry of a halo-tile launch for its consumers' FlagDep (false if
// the unit does not run on the halo-tile kernel)
bool conv_ss_flag_geometry(const ConvArgs& a, FlagDep& d);
// can `proj` (1x1, same input and stride) run inside `a`'s halo-tile launch?
bool conv_ss_proj_ok(const ConvArgs& a, const ConvArgs& proj);
// stream-K for this halo-tile launch pays (whole tiles leave the grid's
// last round mostly idle); slot_floats: the slot size it needs per CTA
bool conv_ss_streamk_wanted(const ConvArgs& a, int nsm, size_t* slot_floats);


// Whole-network kernel (net_fused.cu) for small sequential networks: every
// unit of the plan in one launch, each CTA keeping whole images in shared
// memory (dense CHW fp32) and every parameter staged into shared memory once.
// Offsets are floats into a CTA's shared memory (-1: absent).
constexpr int kNetThreads = 512, kNetMaxOps = 16, kNetMaxCopies = 96, kNetConv = 1, kNetLinear = 2;
struct NetOp {
  int kind;
  int in_off, out_off, scratch_off;  // scratch: a pooled conv's unpooled map / a global-sum view
  int c, h, w;                       // input (conv, in_mode 2 linear)
  int co, ho, wo, cpi;               // conv output before its pool; output channels per work item
  int kh, kw, stride, pad, cb, kp;   // conv weights [co][kp], k = (ci/cb) kh kw cb + (ky kw + kx) cb + ci%cb
  int pool, pool_k, pool_s, pool_pad, pool_deg, pool_order, ph, pw;
  int npad, poly_deg, poly_stride;
  int n_in, n_out, in_mode;          // linear
  int wt, bias, aff, poly, pool_p, in_div;  // parameter offsets in shared memory
};
struct NetCopy {
  const float* src;  // 16-byte aligned
  int dst, n, op;    // shared-memory float offset, floats, the op that first reads it
};
struct NetParams {
  int nops, ncopies;
  NetOp op[kNetMaxOps];
  NetCopy cp[kNetMaxCopies];
  const float* x;          // user NCHW input
  int in_elems, batch;
  int out_off, n_out, out_pad;
  float* logits;           // user [batch][n_out]
  float* out_ws;           // the plan's output vector tensor [batch][out_pad]
  int act_off;             // first activation float (parameters below it)
  int smem_floats;
  unsigned long long* tl;
};
void net_launch(const NetParams& P, cudaStream_t s, int grid);

}  // namespace pcnn
