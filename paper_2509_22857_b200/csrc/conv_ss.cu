// tcgen05 fp16x2 convolution with both operands in shared memory ("halo
// tiles"), for 3x3 / 1x1 convs of stride 1 or 2 whose input is a split tensor
// (stride 2 reads the parity layout: every tap is again a fixed offset, now
// inside one of the four parity planes).
//
// The split layout (common.cuh) stores every 8-channel group as a plane
// [B][H+2][W+2][8] fp16 with a zero border.  Flatten the padded grid: position
// g = (b*(H+2) + y')*(W+2) + x'.  Computing the conv on that grid, output g
// needs input g + (ky-1)*(W+2) + (kx-1) for tap (ky, kx) -- a FIXED offset.
// So a tile of 128 consecutive grid positions needs one contiguous range of
// 128 + 2R input positions (R = (W+2) + 1), and for every tap the A operand
// (M = 128 positions x K = 16 channels) is just that range shifted: a
// shared-memory descriptor at +offset*16 bytes in a K-major, no-swizzle
// layout (core matrices = 8 positions x 16 bytes).  No im2col, no converter
// warps, no A in tensor memory: per 16-channel chunk the producer issues four
// bulk copies (hi/lo plane x two 8-channel groups) plus one for the weights,
// and the MMA warp issues taps x {2 | 3} MMAs.  Positions on the border are
// computed and discarded (waste (H+2)(W+2)/HW - 1).
//
// Precision: x = x_hi + x_lo, w = w_hi + w_lo (fp16, weights scaled by 2^e);
// x*w ~ x_hi w_hi + x_hi w_lo + x_lo w_hi with fp32 accumulation, the main
// products spread over P partial accumulators (the tensor core truncates when
// accumulating) and summed in the epilogue -- the same scheme as conv_tc.cu.
//
// Warp roles (320 threads, persistent, one CTA per SM): warps 0-3 / 4-7
// epilogue warpgroups (one per accumulator buffer), warp 8 TMEM allocator +
// bulk-copy producer, warp 9 MMA issuer.
#include <cuda.h>

#include <cstdlib>
#include <cstring>
#include <vector>

#include "epi_tc.cuh"
#include "kernels.cuh"
#include "tc_layout.cuh"
#include "tc_ptx.cuh"

namespace pcnn {

namespace {

constexpr int kThreads = 320;
constexpr int kWarpProducer = 8, kWarpMma = 9;
constexpr int kSigRing = 8;  // flag mode: tile-stored counters, 2 x the accumulator buffers
constexpr int kTileM = 128;
constexpr int kMaxStages = 8;
constexpr int kMaxPartials = 4;
constexpr int kAddsPerPartial = 96;

struct alignas(64) SsTmap {
  uint64_t v[16];  // CUtensorMap (opaque 128 bytes)
};

struct SsParams {
  SsTmap wmap;           // pair mode: 4-D map of the weight image (first member: 64-byte aligned)
  ConvArgs a;
  int mt;                // 128-row sub-tiles per tile (two for small N: halves the per-tile hand-offs)
  EpiTab etab;
  const __half* w;       // weight image
  const float* wscale;   // 2^-e
  int nt, n_tiles, m_tiles;
  int nq;                // 16-channel chunks
  int last_groups;       // 8-channel groups in the last chunk (1 when cpad is 4 or 8)
  int taps, wp, hp;      // conv taps; output grid = input grid (padded, or one parity grid)
  int halo;              // positions loaded before a tile's first (stride 1, 3x3: wp + 1)
  int span;              // positions per loaded plane: 128 + halo + reach
  int nplanes;           // input planes loaded per stage (4 parity planes for 3x3 / stride 2)
  int plane_id[4];       // which parity plane goes to loaded slot i
  int toff[16];          // tap -> A start in 16-byte units: slot * 4 * span + position offset
  int vy0, vy1, vx0, vx1;  // grid rows / columns holding outputs (output = grid - v*0)
  int shared_grid;         // stride 1: split layout with shared borders (common.cuh)
  FastDiv div_h1;          // shared grid: rows per image (H + 1)
  int64_t gtotal;        // grid positions (batch * hp * wp)
  uint32_t a_bytes;      // one 8-channel group of one plane: span * 16
  uint32_t b_bytes;      // taps * 64 * NT
  uint32_t stage_bytes;  // 4 * a_bytes + b_bytes
  int stages, partials, acc_bufs, concat;
  uint32_t tmem_cols;
  FastDiv div_hw, div_wp, div_mt;  // grid position decode, tile -> n_tile
  int share_epi;         // both epilogue warpgroups drain every tile (alternate chunks)
  int epi_pairs;         // warpgroup pairs draining tiles (2: pairs alternate tiles, 4 warpgroups)
  int b_img_nt;          // rows per tile of the packed weight image (nt, or 128 when nt = 64)
  // psub: 3x3 stride-2 conv staged one parity plane at a time (4 sub-stages
  // per 16-channel chunk, each with that plane's taps): smaller stages, more
  // of them in flight
  int psub;
  int pl_ntaps[4], pl_tap[4][4], pl_toff[4][4];
  int out_pos, skip_pos; // output / residual row of grid position g starts at half index 8 g (split,
                         // same shared-border geometry as the input grid)
  int fold_skip, fold_out;  // storage scales folded into the epilogue table (epi_fill_tab)
  int wide;  // producer: the warp's lanes issue a stage's bulk copies in parallel
  // CTA pair (cta_group::2, cluster of two): one M = 256 tile over two SMs,
  // each CTA staging its own 128 positions and HALF of the tile's weight rows
  // (bn = nt / 2, one 4-D TMA box from wmap), the leader issuing M = 256 MMAs
  // whose accumulators land in both CTAs' TMEM: the weight bytes every SM
  // pulls through L2 per tile halve.  The peer's MMA warp relays its stage
  // hand-offs to the leader (full2), the peer's epilogue releases the
  // leader's accumulator buffers remotely.
  int pair;
  int bn;    // weight rows staged per CTA: nt, or nt / 2 in pair mode
  int dbg;
  int time_slot;         // PCNN_TC_DEBUG bit 64: per-CTA globaltimer stamps slot, else -1
  // wres: the whole weight image (one n-tile, every chunk) stays resident in
  // shared memory after the stage ring, copied once before
  // griddepcontrol.wait; the ring stages then hold activations only
  int wres;
  uint32_t res_bytes;       // resident weight bytes (nq * b_bytes), 0 without wres
  // fused projection (ConvArgs::proj): per chunk two more MMAs on the centre
  // tap's A into 2 nt more TMEM columns, weights appended to the stage's B
  // region, and nt / 16 more epilogue items per sub-tile with its own
  // parameter table, weight scale and output
  int proj;
  EpiParams pe;
  EpiTab petab;
  const __half* pw;         // projection weight image (taps = 1)
  const float* pwscale;
  uint32_t pb_bytes;        // 64 * nt per chunk
  int ptoff;                // centre tap offset (toff of the projection's input position)
  // band mode (a pooled epilogue, PCNN_POOL_LOCAL k x k / s / pad or
  // PCNN_POOL_BI2 2x2 bivariate): CTA c owns the pooled rows [c R / G,
  // (c + 1) R / G) of all R = batch * hpo pooled rows and walks the conv
  // rows they need in order, one tile per `brows` grid rows (a pooled row
  // whose window overlaps the previous band recomputes one conv row).  The
  // epilogue stages each 16-channel item in shared memory, and the thread
  // owning pooled column px folds the item's rows into a two-row ring of
  // window partials (owned per channel chunk by one warpgroup, so no
  // atomics) and stores each pooled row when its last conv row is in.
  int band;
  int brows;                // grid rows per tile (brows * wp <= 128)
  int pk, ps, pp;           // pool window, stride, pad
  int ho, wo;               // conv output rows / columns per image
  int hpo, wpo;             // pooled rows / columns
  int prows;                // batch * hpo
  int nchunk;               // npad / 16 (ring chunks)
  int nbands;               // bands; CTA c runs band c % nbands of n-tile c / nbands
};

// PCNN_TC_DEBUG bit 32: CTA 0 records clock64 events (see pcnn_ss_trace)
constexpr int kTraceLen = 1 << 16;
constexpr int kTraceRegion = kTraceLen / 4;
__device__ unsigned long long g_ss_trace[kTraceLen];

// PCNN_TC_DEBUG bit 64: every CTA's thread 0 stamps %globaltimer at entry,
// after griddepcontrol.wait, after its role loop and at exit (launch slot
// assigned on the host; see pcnn_ss_cta_times)
constexpr int kTimeSlots = 64, kTimeCtas = 160;
__device__ unsigned long long g_cta_time[kTimeSlots][kTimeCtas][4];
static int g_time_next = 0;

__device__ __forceinline__ void cta_stamp(const SsParams& P, int k) {
  if (P.time_slot >= 0 && threadIdx.x == 0 && blockIdx.x < kTimeCtas) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_cta_time[P.time_slot][blockIdx.x][k] = t;
  }
}

// compiled in only with -DPCNN_SS_TRACE (make NVEXTRA=-DPCNN_SS_TRACE)
struct Tracer {
  uint32_t n = 0;
  __device__ __forceinline__ void operator()(const SsParams& P, int region, uint32_t tag) {
#ifdef PCNN_SS_TRACE
    if ((P.dbg & 32) && blockIdx.x == 0 && n < kTraceRegion)
      g_ss_trace[region * kTraceRegion + n++] = ((unsigned long long)tag << 48) | (clock64() & 0xFFFFFFFFFFFFull);
#else
    (void)P; (void)region; (void)tag;
#endif
  }
};

constexpr int kMaxAcc = 4;  // accumulator buffers in TMEM
constexpr int kMaxWChunks = 8;  // resident weights: one barrier per 16-channel chunk

struct Smem {
  uint64_t full[kMaxStages], empty[kMaxStages];
  uint64_t acc_full[kMaxAcc], acc_empty[kMaxAcc];
  uint64_t wfull[kMaxWChunks];  // resident weights: chunk q landed
  uint64_t full2[kMaxStages];   // pair mode, leader: the peer's stage landed (relayed by its MMA warp)
  uint32_t tstored[kSigRing];  // flag mode: draining warps done with a tile (monotonic per slot)
  uint32_t tmem_base;
  int dep_seq;     // flag mode: this CTA's tiles whose producer tiles were acquired
};


// ---- one stage (all taps of one 16-channel chunk) ----
// Descriptor adds in C++ on warp-uniform values (A advances by the tap's grid
// offset in the 16-byte units of the start-address field, B by one (chunk,
// tap) block), one minimal asm per MMA predicated on a lane elected once per
// stage: ~64 cycles per MMA issued, vs ~75 for one asm block per stage.
// concat (NT <= 64): [main | corr] (+)= A_hi [B_hi | B_lo] (N = 2NT);
//   corr += A_lo B_hi.
// split (NT = 128): corr (+)= A_lo B_hi; corr += A_hi B_lo; main (+)= A_hi B_hi.
__device__ __forceinline__ uint32_t elect_one_sync() {
  uint32_t e;
  asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 r;\n\telect.sync r|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(e));
  return e;
}
__device__ __forceinline__ void mma_f16_ss_if(uint32_t e, uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                              uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, q;\n\tsetp.ne.b32 q, %0, 0;\n\tsetp.ne.b32 p, %5, 0;\n\t"
               "@q tcgen05.mma.cta_group::1.kind::f16 [%1], %2, %3, %4, p;\n\t}"
               ::"r"(e), "r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc)
               : "memory");
}
__device__ __forceinline__ void mma_f16_ss2_if(uint32_t e, uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                               uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, q;\n\tsetp.ne.b32 q, %0, 0;\n\tsetp.ne.b32 p, %5, 0;\n\t"
               "@q tcgen05.mma.cta_group::2.kind::f16 [%1], %2, %3, %4, p;\n\t}"
               ::"r"(e), "r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc)
               : "memory");
}
template <bool PAIR>
__device__ __forceinline__ void mma_ss(uint32_t e, uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (PAIR) mma_f16_ss2_if(e, d, a, b, idesc, acc);
  else mma_f16_ss_if(e, d, a, b, idesc, acc);
}
template <int TAPS, bool PAIR = false>
__device__ __forceinline__ void ss_stage(bool concat, uint32_t dm, uint32_t dc, uint64_t ah, uint64_t al,
                                             uint64_t b, uint64_t bstep, uint64_t blo, uint32_t id2, uint32_t id1,
                                             uint32_t accm, uint32_t accc, const uint64_t* o) {
  const uint32_t e = elect_one_sync();
  if (concat) {
    // same-shape MMAs back to back (all N = 2 NT products, then all N = NT):
    // alternating the two shapes tap by tap cost the image-resident kernels
    // 3-5 % (RN20 span 230 -> 223 us, A/B on one box); each accumulator
    // still sees its products in tap order
#pragma unroll
    for (int t = 0; t < TAPS; ++t) mma_ss<PAIR>(e, dm, ah + o[t], b + t * bstep, id2, t ? 1u : accm);
#pragma unroll
    for (int t = 0; t < TAPS; ++t) mma_ss<PAIR>(e, dc, al + o[t], b + t * bstep, id1, 1u);
  } else {
#pragma unroll
    for (int t = 0; t < TAPS; ++t) {
      mma_ss<PAIR>(e, dc, al + o[t], b + t * bstep, id1, t ? 1u : accc);
      mma_ss<PAIR>(e, dc, ah + o[t], b + t * bstep + blo, id1, 1u);
      mma_ss<PAIR>(e, dm, ah + o[t], b + t * bstep, id1, t ? 1u : accm);
    }
  }
}

// ---- work segments: what a CTA computes, in order ----
// Whole tiles: tile = blockIdx.x + i * gridDim.x, all chunks, owner.
// Stream-K: units u = tile * nq + chunk, CTA c owns [c U / G, (c + 1) U / G);
// its segments are visited in descending tile order, so its only partial
// (non-owner) segment -- the prefix of its last tile -- comes first and is
// published early, and the tile it finishes (the suffix of its first tile,
// whose earlier chunks belong to lower CTAs) comes last.
struct Seg {
  int tile, q0, q1;
  int owner;  // holds the tile's last chunk: runs the epilogue
  int c_lo;   // owner: first CTA holding earlier chunks of the tile (-1: none)
  int n_tile;
  int64_t g0;  // grid position of the tile's first output row
  int r, rows;  // band mode: first grid row, grid rows in the tile
};

// band mode: this CTA's pooled rows [P0, P1) and conv grid rows [r0, r1]
struct Band {
  int P0, P1, r0, r1, tiles;
};
__device__ __forceinline__ Band band_of(const SsParams& P) {
  Band bd;
  const int G = P.nbands, c = (int)blockIdx.x % P.nbands;
  bd.P0 = (int)((int64_t)c * P.prows / G);
  bd.P1 = (int)((int64_t)(c + 1) * P.prows / G);
  bd.tiles = 0;
  bd.r0 = bd.r1 = 0;
  if (bd.P1 <= bd.P0) return bd;
  const int b0 = bd.P0 / P.hpo, py0 = bd.P0 - b0 * P.hpo;
  const int b1 = (bd.P1 - 1) / P.hpo, py1 = bd.P1 - 1 - b1 * P.hpo;
  const int y0 = max(0, P.ps * py0 - P.pp), y1 = min(P.ho - 1, P.ps * py1 - P.pp + P.pk - 1);
  bd.r0 = b0 * P.hp + y0 + 1;  // shared grid: image row y of b is grid row b (H + 1) + y + 1
  bd.r1 = b1 * P.hp + y1 + 1;
  bd.tiles = (bd.r1 - bd.r0 + P.brows) / P.brows;
  return bd;
}

__device__ __forceinline__ bool seg_at(int i, int total_tiles, int nq, bool streamk, Seg& s);

// segment i of this CTA in any mode (whole tiles, stream-K, bands)
template <bool BAND, bool PAIR = false>
__device__ __forceinline__ bool seg_get(const SsParams& P, const Band& bd, int i, int total_tiles, bool streamk,
                                        Seg& s) {
  if constexpr (BAND) {
    if (i >= bd.tiles) return false;
    s.n_tile = (int)blockIdx.x / P.nbands;
    const int local = i;
    s.tile = i;
    s.q0 = 0;
    s.q1 = P.nq;
    s.owner = 1;
    s.c_lo = -1;
    s.r = bd.r0 + local * P.brows;
    s.rows = min(P.brows, bd.r1 - s.r + 1);
    s.g0 = 1 + (int64_t)s.r * P.wp;
    return true;
  }
  if constexpr (PAIR) {
    // pair tile pt = (n_tile, m-tile pair) walked by cluster; rank r takes m-tile 2 m + r
    const int ncl = (int)gridDim.x >> 1, mp = P.m_tiles >> 1;
    const int pt = ((int)blockIdx.x >> 1) + i * ncl;
    if (pt >= mp * P.n_tiles) return false;
    s.n_tile = pt / mp;
    const int m = 2 * (pt - s.n_tile * mp) + ((int)blockIdx.x & 1);
    s.tile = s.n_tile * P.m_tiles + m;
    s.q0 = 0;
    s.q1 = P.nq;
    s.owner = 1;
    s.c_lo = -1;
    s.g0 = (int64_t)m * kTileM;
    s.r = s.rows = 0;
    return true;
  }
  if (!seg_at(i, total_tiles, P.nq, streamk, s)) return false;
  s.n_tile = s.tile / P.m_tiles;
  s.g0 = (int64_t)(s.tile - s.n_tile * P.m_tiles) * kTileM * P.mt;
  s.r = s.rows = 0;
  return true;
}

__device__ __forceinline__ bool seg_at(int i, int total_tiles, int nq, bool streamk, Seg& s) {
  if (!streamk) {
    s.tile = (int)blockIdx.x + i * (int)gridDim.x;
    s.q0 = 0;
    s.q1 = nq;
    s.owner = 1;
    s.c_lo = -1;
    return s.tile < total_tiles;
  }
  const int64_t U = (int64_t)total_tiles * nq, G = gridDim.x, c = blockIdx.x;
  const int64_t u0 = c * U / G, u1 = (c + 1) * U / G;
  if (u1 <= u0) return false;
  const int64_t t0 = u0 / nq, t1 = (u1 - 1) / nq, t = t1 - i;
  if (t < t0) return false;
  s.tile = (int)t;
  s.q0 = (int)((u0 > t * nq ? u0 : t * nq) - t * nq);
  s.q1 = (int)((u1 < (t + 1) * nq ? u1 : (t + 1) * nq) - t * nq);
  s.owner = s.q1 == nq;
  // first contributor: the CTA whose range holds unit t * nq
  s.c_lo = (s.owner && s.q0 > 0) ? (int)(((t * nq + 1) * G - 1) / U) : -1;
  return true;
}

// Flag-synchronised launches: wait until the producer tiles covering grid
// positions [lo, hi) (mode 1) or all its tiles (mode 2) have bumped their
// counters (release-ordered after their stores).  Bounded: a missing signal
// traps instead of hanging the GPU.
__device__ __forceinline__ void flag_wait(const FlagDep& d, int64_t lo, int64_t hi, bool& all_done) {
  if (all_done) return;
  {
    // once the whole producer is done, no more per-tile polls
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(d.done + d.m_tiles) : "memory");
    if (v >= d.all) {
      all_done = true;
      return;
    }
  }
  auto wait_ge = [](const int* c, int target) {
    uint32_t spins = 0;
    for (;;) {
      int v;
      asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
      if (v >= target) break;
      __nanosleep(64);
      if (++spins > (1u << 25)) __trap();
    }
  };
  if (d.mode == 1) {
    lo = lo < 0 ? 0 : lo;
    hi = hi > d.gtotal ? d.gtotal : hi;
    if (hi <= lo) return;
    const int first = (int)(lo / d.tm);
    int last = (int)((hi - 1) / d.tm);
    if (last >= d.m_tiles) last = d.m_tiles - 1;
    for (int t = first; t <= last; ++t) wait_ge(d.done + t, d.per_tile);
  } else if (d.mode == 2) {
    wait_ge(d.done + d.m_tiles, d.all);
    all_done = true;
  }
}

constexpr int kStgPitch = 20;  // staged floats per row (16 + 4: conflict-free 16-byte reads)

// Band mode, one item = 16 channels chb..chb+15 of the tile's grid rows
// [r, r + rows) (v: this thread's row = tile position `row`, per-element
// epilogue applied).  Pooled rows finish in the ring of window partials,
// [ns slots][nchunk][wpo][16] (BI2 order 1: two such rings).
//
// POOL_LOCAL (s = 2; k = 3, p = 1 or k = 2, p = 0; one grid row per tile,
//   so tile position = column x): the even lane x = 2 px sums its window
//   row from its neighbours' registers (shuffles; the window of px = 16 w
//   crossing a warp boundary gets lane 31's value through shared memory),
//   then adds it to the ring slot of every pooled row the conv row feeds;
//   the conv row finishing a pooled row scales by the divisor and stores it.
//   The owner of (px, chunk) is always the same thread: no atomics, no
//   other synchronisation.
// POOL_BI2 (2 x 2, any rows per tile): the item is staged; pair (j, px)
//   of the item goes to thread j * wpo + px; even conv rows write their
//   first-stage result (order 0: S1(q00, q01); order 1: q00, q01) to the
//   ring, a second barrier, odd rows finish S2 and store (epi_tc.cuh's tree).
__device__ __forceinline__ void band_item(const SsParams& P, const EpiParams& e, const Band& bd, float* ring,
                                          float* stg, float* bnd, int r, int rows, int row, int lane, int wq, int ew,
                                          int chb, float* v, float pdiv) {
  const int chunk = chb >> 4;
  const int ns = P.brows / 2 + 2;
  if (e.pool == PCNN_POOL_LOCAL) {
    // lane x holds column x of the tile's conv row.  Window px (s = 2):
    // (3, 1): columns 2px-1 .. 2px+1; (2, 0): 2px, 2px+1.  Channels 0-7 of
    // window px belong to lane 2px, channels 8-15 to lane 2px+1, so every
    // lane sums 8 channels of three (two) columns: even lanes x-1, x, x+1,
    // odd lanes x-2, x-1, x (k = 2: x, x+1 / x-1, x).
    const bool odd = row & 1;
    if (row >= P.wo) {  // columns past the image (the shared zero border): padding
#pragma unroll
      for (int c = 0; c < 16; ++c) v[c] = 0.f;
    }
    float l1[16], h8[8];
#pragma unroll
    for (int c = 0; c < 16; ++c) l1[c] = __shfl_up_sync(0xffffffffu, v[c], 1);
    if (P.pk == 3) {
      float r1[8], l2[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) r1[c] = __shfl_down_sync(0xffffffffu, v[c], 1);
#pragma unroll
      for (int c = 0; c < 8; ++c) l2[c] = __shfl_up_sync(0xffffffffu, v[8 + c], 2);
      // lane 31's column for lanes 0 and 1 of the next warp
      if (lane == 31)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          *reinterpret_cast<float4*>(bnd + wq * 16 + 4 * q) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      asm volatile("bar.sync %0, 128;" ::"r"(1 + ew) : "memory");
      if (lane < 2) {
        float pv[16];
        if (wq > 0) {
          lds16(bnd + (wq - 1) * 16, pv);
        } else {
#pragma unroll
          for (int c = 0; c < 16; ++c) pv[c] = 0.f;  // column -1: zero padding
        }
        if (lane == 0) {
#pragma unroll
          for (int c = 0; c < 8; ++c) l1[c] = pv[c];
        } else {
#pragma unroll
          for (int c = 0; c < 8; ++c) l2[c] = pv[8 + c];
        }
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) h8[c] = odd ? v[8 + c] + l1[8 + c] + l2[c] : v[c] + l1[c] + r1[c];
    } else {
      float r1[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) r1[c] = __shfl_down_sync(0xffffffffu, v[c], 1);
#pragma unroll
      for (int c = 0; c < 8; ++c) h8[c] = odd ? v[8 + c] + l1[8 + c] : v[c] + r1[c];
    }
    const int px = row >> 1, ch8 = chb + (odd ? 8 : 0);
    if (px >= P.wpo || r <= 0) return;
    const int b = (int)P.div_h1.div((uint32_t)(r - 1)), y = r - 1 - b * P.hp;
    if (y >= P.ho) return;  // shared border row between images
    // pooled rows fed by conv row y; ring slot = pooled row & 1 (one conv
    // row per tile, so at most two pooled rows are open)
    float* const ring_px = ring + (chunk * P.wpo + px) * 16 + (odd ? 8 : 0);
    const int slot_stride = P.nchunk * P.wpo * 16;
    auto in_band = [&](int py) { const int pr = b * P.hpo + py; return py < P.hpo && pr >= bd.P0 && pr < bd.P1; };
    auto finish = [&](int py, const float* a) {
      float o[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) o[c] = ch8 + c < e.cout ? (a[c] + h8[c]) * pdiv : 0.f;
      store8_any(e.out, b, ch8, py, px, o);
    };
    auto keep = [&](int py, const float* a) {
      float* sl = ring_px + ((b * P.hpo + py) & 1) * slot_stride;
      *reinterpret_cast<float4*>(sl) = make_float4(a[0] + h8[0], a[1] + h8[1], a[2] + h8[2], a[3] + h8[3]);
      *reinterpret_cast<float4*>(sl + 4) = make_float4(a[4] + h8[4], a[5] + h8[5], a[6] + h8[6], a[7] + h8[7]);
    };
    const float zero[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    auto ring_of = [&](int py, float* a) {
      const float* sl = ring_px + ((b * P.hpo + py) & 1) * slot_stride;
      const float4 u = *reinterpret_cast<const float4*>(sl), w = *reinterpret_cast<const float4*>(sl + 4);
      a[0] = u.x; a[1] = u.y; a[2] = u.z; a[3] = u.w; a[4] = w.x; a[5] = w.y; a[6] = w.z; a[7] = w.w;
    };
    if (P.pk == 3) {
      if (!(y & 1)) {  // rows 2py-1, [2py], 2py+1 of pooled row py = y / 2
        const int py = y >> 1;
        if (in_band(py)) {
          float a[8];
          if (py == 0) {
#pragma unroll
            for (int c = 0; c < 8; ++c) a[c] = 0.f;
          } else {
            ring_of(py, a);
          }
          if (y == P.ho - 1) finish(py, a);
          else keep(py, a);
        }
      } else {         // last row of py0 = (y - 1) / 2, first row of py1 = (y + 1) / 2
        const int py0 = (y - 1) >> 1, py1 = (y + 1) >> 1;
        if (in_band(py0)) {
          float a[8];
          ring_of(py0, a);
          finish(py0, a);
        }
        if (in_band(py1)) keep(py1, zero);
      }
    } else {           // (2, 0): rows 2py, 2py+1
      const int py = y >> 1;
      if (in_band(py)) {
        if (!(y & 1)) {
          keep(py, zero);
        } else {
          float a[8];
          ring_of(py, a);
          finish(py, a);
        }
      }
    }
    return;
  }
  // ---- POOL_BI2 ----
#pragma unroll
  for (int q = 0; q < 4; ++q)
    *reinterpret_cast<float4*>(stg + row * kStgPitch + 4 * q) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  asm volatile("bar.sync %0, 128;" ::"r"(1 + ew) : "memory");
  const int w = row, nw = rows * P.wpo;
  int j = 0, px = 0, b = 0, y = -1, py = 0, prow = 0;
  bool mine = false;
  if (w < nw) {
    j = w / P.wpo;
    px = w - j * P.wpo;
    const int R = r + j;
    if (R > 0) {
      b = (int)P.div_h1.div((uint32_t)(R - 1));
      y = R - 1 - b * P.hp;
      py = y >> 1;
      prow = b * P.hpo + py;
      mine = y < P.ho && py < P.hpo && prow >= bd.P0 && prow < bd.P1;
    }
  }
  const int64_t nc = (int64_t)(e.pool_deg + 1) * (e.pool_deg + 1) * e.npad;
  float* sl = ring + (((prow % ns) * P.nchunk + chunk) * P.wpo + px) * 16;
  float* sl2 = sl + ns * P.nchunk * P.wpo * 16;  // order 1: q01 of the even row
  float q0[16], q1[16];
  if (mine) {
    const float* rowp = stg + (j * P.wp + 2 * px) * kStgPitch;
    lds16(rowp, q0);
    lds16(rowp + kStgPitch, q1);
    if (!(y & 1)) {
      if (e.pool_order == 0) {
#pragma unroll
        for (int g = 0; g < 4; ++g)
          *reinterpret_cast<float4*>(sl + 4 * g) =
              bivariate4_any(e.pool_p, e.npad, e.pool_deg, chb + 4 * g,
                         make_float4(q0[4 * g], q0[4 * g + 1], q0[4 * g + 2], q0[4 * g + 3]),
                         make_float4(q1[4 * g], q1[4 * g + 1], q1[4 * g + 2], q1[4 * g + 3]));
      } else {
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          *reinterpret_cast<float4*>(sl + 4 * g) = make_float4(q0[4 * g], q0[4 * g + 1], q0[4 * g + 2], q0[4 * g + 3]);
          *reinterpret_cast<float4*>(sl2 + 4 * g) = make_float4(q1[4 * g], q1[4 * g + 1], q1[4 * g + 2], q1[4 * g + 3]);
        }
      }
    }
  }
  asm volatile("bar.sync %0, 128;" ::"r"(1 + ew) : "memory");
  if (!mine || !(y & 1)) return;
  float o[16];
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const int ch = chb + 4 * g;
    const float4 x0 = make_float4(q0[4 * g], q0[4 * g + 1], q0[4 * g + 2], q0[4 * g + 3]);
    const float4 x1 = make_float4(q1[4 * g], q1[4 * g + 1], q1[4 * g + 2], q1[4 * g + 3]);
    float4 u, ww;
    if (e.pool_order == 0) {
      u = *reinterpret_cast<const float4*>(sl + 4 * g);
      ww = bivariate4_any(e.pool_p, e.npad, e.pool_deg, ch, x0, x1);
    } else {
      u = bivariate4_any(e.pool_p, e.npad, e.pool_deg, ch, *reinterpret_cast<const float4*>(sl + 4 * g), x0);
      ww = bivariate4_any(e.pool_p, e.npad, e.pool_deg, ch, *reinterpret_cast<const float4*>(sl2 + 4 * g), x1);
    }
    const float4 r4 = bivariate4_any(e.pool_p + nc, e.npad, e.pool_deg, ch, u, ww);
    o[4 * g] = ch < e.cout ? r4.x : 0.f;
    o[4 * g + 1] = ch + 1 < e.cout ? r4.y : 0.f;
    o[4 * g + 2] = ch + 2 < e.cout ? r4.z : 0.f;
    o[4 * g + 3] = ch + 3 < e.cout ? r4.w : 0.f;
  }
  store16_any(e.out, b, chb, py, px, o);
}

// SK: stream-K segments (a separate instantiation: the whole-tile kernel
// keeps its registers and its simpler item walk)
// POOL: kPoolNone (store or global sum, fused projection) or kPoolBand (the
// band epilogue).  Global pools stay in the common instantiation: a kernel
// that runs once per forward starts with a cold instruction cache (measured
// +4.4 us on RN20's last conv as its own instantiation), while the code
// shared by every other layer of the network is already resident.
constexpr int kPoolNone = 0, kPoolBand = 2;

// threads: PAIRS pairs of epilogue warpgroups, the producer and the MMA
// warp.  Two pairs (576 threads, <= 112 registers) hide the epilogue's
// latency on narrow layers; wide layers keep one pair and 168 registers
template <int PAIRS>
constexpr int ss_threads() { return PAIRS == 2 ? 576 : 320; }

template <int TAPS, bool SK, int POOL, int PAIRS = 1, bool PAIR = false>
__global__ void __launch_bounds__(ss_threads<PAIRS>(), 1) conv_ss_kernel(const __grid_constant__ SsParams P) {
  constexpr bool BAND = POOL == kPoolBand;
  constexpr int kThreads = ss_threads<PAIRS>();
  constexpr int kWarpProducer = kThreads / 32 - 2, kWarpMma = kThreads / 32 - 1;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  const ConvArgs& a = P.a;
  const size_t ring = (size_t)P.stages * P.stage_bytes;  // resident weights (wres) follow the ring
  Smem* S = reinterpret_cast<Smem*>(smem + ring + P.res_bytes);
  float* ptab = reinterpret_cast<float*>(smem + ring + P.res_bytes + ((sizeof(Smem) + 15) & ~size_t(15)));
  const uint32_t base = ptx::smem_u32(smem);
  const uint32_t wres_base = base + (uint32_t)ring;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int total_tiles = P.m_tiles * P.n_tiles;
  constexpr bool streamk = SK;
  const int NP = P.partials, NB = P.acc_bufs;
  const uint32_t set_a = P.concat ? (uint32_t)NP * 2 * P.nt : (uint32_t)(NP + 1) * P.nt;
  constexpr bool kProj = TAPS == 9 && POOL == kPoolNone;  // projection fusion: 3x3 convs only
  const bool proj = kProj && P.proj;
  const uint32_t set_cols = set_a + (proj ? 2u * P.nt : 0u);  // + projection [main | corr]
  Tracer tr;
  cta_stamp(P, 0);

  if (threadIdx.x == 0) {
    for (int i = 0; i < P.stages; ++i) {
      ptx::mbar_init(ptx::smem_u32(&S->full[i]), 1);
      ptx::mbar_init(ptx::smem_u32(&S->empty[i]), 1);
    }
    for (int i = 0; i < kMaxAcc; ++i) {
      ptx::mbar_init(ptx::smem_u32(&S->acc_full[i]), 1);
      // one arrive per draining warp (pair mode, leader: of both CTAs)
      ptx::mbar_init(ptx::smem_u32(&S->acc_empty[i]), (P.share_epi ? 8 : 4) * (PAIR ? 2 : 1));
    }
    for (int i = 0; i < kMaxStages; ++i) ptx::mbar_init(ptx::smem_u32(&S->full2[i]), 1);
    for (int i = 0; i < kMaxWChunks; ++i) ptx::mbar_init(ptx::smem_u32(&S->wfull[i]), 1);
    for (int i = 0; i < kSigRing; ++i) S->tstored[i] = 0;
    S->dep_seq = 0;
    ptx::fence_mbar_init();
  }
  if (warp == kWarpProducer) {
    if constexpr (PAIR) ptx::tmem_alloc2(ptx::smem_u32(&S->tmem_base), P.tmem_cols);
    else ptx::tmem_alloc(ptx::smem_u32(&S->tmem_base), P.tmem_cols);
  }
  epi_fill_tab(a.epi, P.etab, ptab, threadIdx.x, kThreads, P.fold_skip ? a.epi.skip.sload : 1.f,
               P.fold_out ? a.epi.out.sstore : 1.f);
  float* ptab_p = ptab + P.etab.rows * a.epi.npad;  // projection table (P.proj)
  if (proj) epi_fill_tab(P.pe, P.petab, ptab_p, threadIdx.x, kThreads);
  if (P.last_groups == 1) {
    // cpad 4 / 8: the second 8-channel group of every stage stays zero
    for (int st = 0; st < P.stages; ++st)
      for (int pl = 0; pl < 2 * P.nplanes; ++pl) {  // (plane, hi/lo): its second 8-channel group
        uint4* z = reinterpret_cast<uint4*>(smem + (size_t)st * P.stage_bytes + (2 * pl + 1) * P.a_bytes);
        for (uint32_t i = threadIdx.x; i < P.a_bytes / 16; i += kThreads) z[i] = make_uint4(0, 0, 0, 0);
      }
    ptx::fence_proxy_async();
  }
  // the next unit's global-pool sums (not touched by any kernel of this
  // forward before this one); before the CTA barrier, so the epilogue's
  // completion signals (flag mode) are ordered after these stores
  if (a.prezero) {
    float4* z = reinterpret_cast<float4*>(a.prezero);
    const int64_t n4 = a.prezero_n / 4;
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n4; i += (int64_t)gridDim.x * kThreads)
      z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) ptx::cluster_sync();  // the peer's barriers exist before any remote arrive
  ptx::tc_fence_after();
  const uint32_t tmem = S->tmem_base;
  // resident weights: parameters, not written by the previous kernel, so the
  // copy overlaps its tail
  // copy overlaps its tail; one barrier per chunk, so the first tile's MMAs
  // start after the first chunk
  if (P.wres && warp == kWarpProducer && lane == 0) {
    for (int q = 0; q < P.nq; ++q) {
      const uint32_t wb = ptx::smem_u32(&S->wfull[q]);
      ptx::mbar_arrive_tx(wb, P.b_bytes);
      ptx::bulk_g2s(wres_base + (uint32_t)q * P.b_bytes, reinterpret_cast<const uint8_t*>(P.w) + (size_t)q * P.b_bytes,
                    P.b_bytes, wb);
    }
  }
  // everything above reads only parameters; activations come from the
  // previous kernel (or, flag mode, from producers whose tiles are awaited
  // one by one below)
  if (!a.skip_gridwait) ptx::griddep_wait();
  ptx::griddep_launch();
  cta_stamp(P, 1);
  tl_mark(a.tl, 0);

  if (warp == kWarpProducer) {
    // ===== producer: per (tile, 16-channel chunk) one stage = the tile's
    // input range for both planes and both 8-channel groups + the weights =====
    if constexpr (PAIR) {
      // pair mode: own activation rows (lanes in parallel) + this CTA's half
      // of the tile's weight rows as one 4-D TMA box ([tap][g, hi/lo][bn rows x 16 B])
      const __half* hi = a.in.hi();
      const __half* lo = a.in.lo();
      const int rank = (int)(blockIdx.x & 1);
      if (lane == 0) ptx::prefetch_tmap(&P.wmap);
      int st = 0;
      uint32_t ph = 0;
      Seg sg;
      Band bd = {};
      for (int si = 0; seg_get<false, true>(P, bd, si, total_tiles, false, sg); ++si) {
        const int64_t gs = sg.g0 - P.halo;
        const int64_t cs = gs < 0 ? 0 : gs;
        const int64_t ge = gs + P.span;
        const int64_t ce = ge > P.gtotal ? P.gtotal : ge;
        // an m-tile past the grid (odd m-tile count) stages weights only
        const uint32_t slot0 = (uint32_t)(cs - gs) * 16, bytes = ce > cs ? (uint32_t)(ce - cs) * 16 : 0u;
        for (int q = 0; q < P.nq; ++q) {
          const uint32_t bar = ptx::smem_u32(&S->full[st]);
          const uint32_t sb = base + st * P.stage_bytes;
          const int ng = q == P.nq - 1 ? P.last_groups : 2;
          if (lane == 0) {
            if (P.dbg & 2048) ptx::mbar_wait_nohint(ptx::smem_u32(&S->empty[st]), ph ^ 1);
            else ptx::mbar_wait_sleep(ptx::smem_u32(&S->empty[st]), ph ^ 1);
            ptx::mbar_arrive_tx(bar, 2 * ng * P.nplanes * bytes + P.b_bytes);
          }
          __syncwarp();
          const int na = 2 * ng * P.nplanes;
          if (lane < na) {
            if (bytes) {
              const int pl = lane / (2 * ng), r = lane - pl * 2 * ng, g = r >> 1, hl = r & 1;
              const int64_t off = (2 * q + g) * a.in.kstride + P.plane_id[pl] * a.in.pstride + cs * 8;
              ptx::bulk_g2s(sb + pl * 4 * P.a_bytes + (hl * 2 + g) * P.a_bytes + slot0, (hl ? lo : hi) + off, bytes,
                            bar);
            }
          } else if (lane == 31) {
            ptx::tma_load_4d(sb + P.nplanes * 4 * P.a_bytes, &P.wmap, rank * P.bn * 4, 0, 0, sg.n_tile * P.nq + q, bar);
          }
          __syncwarp();
          if (++st == P.stages) { st = 0; ph ^= 1; }
        }
      }
    } else if (!BAND && P.wide) {
      // the whole warp walks the stages; lane 0 waits for the slot and posts
      // the byte count, then lane j issues copy j of the stage (a single
      // thread pays ~300 cycles per cp.async.bulk, tools/ubench_bulk.cu)
      const __half* hi = a.in.hi();
      const __half* lo = a.in.lo();
      int st = 0;
      uint32_t ph = 0;
      Seg sg;
      Band bd = {};
      for (int si = 0; seg_get<false>(P, bd, si, total_tiles, streamk, sg); ++si) {
        const int n_tile = sg.n_tile;
        const int64_t gs = sg.g0 - P.halo;
        const int64_t cs = gs < 0 ? 0 : gs;
        const int64_t ge = gs + P.span;
        const int64_t ce = ge > P.gtotal ? P.gtotal : ge;
        const uint32_t slot0 = (uint32_t)(cs - gs) * 16, bytes = (uint32_t)(ce - cs) * 16;
        for (int q = sg.q0; q < sg.q1; ++q) {
          const uint32_t bar = ptx::smem_u32(&S->full[st]);
          const uint32_t sb = base + st * P.stage_bytes;
          const int ng = q == P.nq - 1 ? P.last_groups : 2;
          if (lane == 0) {
            if (P.dbg & 2048) ptx::mbar_wait_nohint(ptx::smem_u32(&S->empty[st]), ph ^ 1);
            else ptx::mbar_wait_sleep(ptx::smem_u32(&S->empty[st]), ph ^ 1);
            ptx::mbar_arrive_tx(bar, 2 * ng * P.nplanes * bytes + (P.wres ? 0u : P.b_bytes) + P.pb_bytes);
          }
          __syncwarp();
          const int na = 2 * ng * P.nplanes;  // activation copies: (plane, group, hi / lo)
          if (lane < na) {
            const int pl = lane / (2 * ng), r = lane - pl * 2 * ng, g = r >> 1, hl = r & 1;
            const int64_t off = (2 * q + g) * a.in.kstride + P.plane_id[pl] * a.in.pstride + cs * 8;
            ptx::bulk_g2s(sb + pl * 4 * P.a_bytes + (hl * 2 + g) * P.a_bytes + slot0, (hl ? lo : hi) + off, bytes,
                          bar);
          } else if (lane == na && P.proj) {
            ptx::bulk_g2s(sb + P.nplanes * 4 * P.a_bytes + P.b_bytes, P.pw + ((int64_t)n_tile * P.nq + q) * 32 * P.nt,
                          P.pb_bytes, bar);
          } else if (lane == na + 1 && !P.wres && P.b_img_nt == P.nt) {
            ptx::bulk_g2s(sb + P.nplanes * 4 * P.a_bytes, P.w + ((int64_t)n_tile * P.nq + q) * P.taps * 32 * P.nt,
                          P.b_bytes, bar);
          }
          if (!P.wres && P.b_img_nt != P.nt) {
            // nt of the image's b_img_nt rows: per (tap, group) the hi and lo row ranges
            const int INT = P.b_img_nt, row0 = n_tile * P.nt, it = row0 / INT, r0 = row0 - it * INT;
            const uint32_t rows_bytes = (uint32_t)P.nt * 16;
            for (int j = lane; j < P.taps * 4; j += 32) {
              const int t = j >> 2, g = (j >> 1) & 1, hl = j & 1;
              const __half* blk = P.w + (((int64_t)it * P.nq + q) * P.taps + t) * 32 * INT;
              const uint32_t dst = sb + P.nplanes * 4 * P.a_bytes + (uint32_t)(t * 32 * P.nt + g * 16 * P.nt) * 2;
              ptx::bulk_g2s(dst + hl * rows_bytes, blk + g * 16 * INT + (hl * INT + r0) * 8, rows_bytes, bar);
            }
          }
          __syncwarp();
          if (++st == P.stages) { st = 0; ph ^= 1; }
        }
      }
    } else if (lane == 0) {
      const __half* hi = a.in.hi();
      const __half* lo = a.in.lo();
      int st = 0;
      uint32_t ph = 0;
      bool fin_all = false, fsk_all = false;
      int dep_seq = 0;
      Seg sg;
      Band bd = {};
      if constexpr (BAND) bd = band_of(P);
      for (int si = 0; seg_get<BAND, PAIR>(P, bd, si, total_tiles, streamk, sg); ++si) {
        const int n_tile = sg.n_tile;
        const int64_t gs = sg.g0 - P.halo;  // grid position of buffer slot 0
        const int64_t cs = gs < 0 ? 0 : gs;
        const int64_t ge = gs + P.span;
        const int64_t ce = ge > P.gtotal ? P.gtotal : ge;
        const uint32_t slot0 = (uint32_t)(cs - gs) * 16, bytes = (uint32_t)(ce - cs) * 16;
        if (a.fin.mode || a.fsk.mode) {
          // the producer tiles of this tile's input range and residual rows;
          // dep_seq hands the acquired state to the epilogue (CTA scope)
          if (a.fin.mode) flag_wait(a.fin, cs, ce, fin_all);
          if (a.fsk.mode) {
            const int64_t r0 = sg.g0;
            flag_wait(a.fsk, r0, r0 + kTileM * P.mt, fsk_all);
          }
          asm volatile("fence.proxy.async.global;" ::: "memory");  // generic writes -> bulk-copy reads
          asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(ptx::smem_u32(&S->dep_seq)), "r"(++dep_seq)
                       : "memory");
        }
        if (P.psub) {
          // one parity plane and its taps' weights per stage
          for (int q = sg.q0; q < sg.q1; ++q)
            for (int ps = 0; ps < 4; ++ps) {
              ptx::mbar_wait_sleep(ptx::smem_u32(&S->empty[st]), ph ^ 1);
              const uint32_t bar = ptx::smem_u32(&S->full[st]);
              const uint32_t sb = base + st * P.stage_bytes;
              const int ng = q == P.nq - 1 ? P.last_groups : 2;
              const int ntp = P.pl_ntaps[ps];
              ptx::mbar_arrive_tx(bar, 2 * ng * bytes + (uint32_t)ntp * 64 * P.nt);
              for (int g = 0; g < ng; ++g) {
                const int64_t off = (2 * q + g) * a.in.kstride + P.plane_id[ps] * a.in.pstride + cs * 8;
                ptx::bulk_g2s(sb + g * P.a_bytes + slot0, hi + off, bytes, bar);
                ptx::bulk_g2s(sb + (2 + g) * P.a_bytes + slot0, lo + off, bytes, bar);
              }
              const int INT = P.b_img_nt, row0 = n_tile * P.nt, it = row0 / INT, r0 = row0 - it * INT;
              for (int j = 0; j < ntp; ++j) {
                const int t = P.pl_tap[ps][j];
                const __half* blk = P.w + (((int64_t)it * P.nq + q) * P.taps + t) * 32 * INT;
                const uint32_t dst = sb + 4 * P.a_bytes + (uint32_t)j * 64 * P.nt;
                if (INT == P.nt) {
                  ptx::bulk_g2s(dst, blk, 64 * P.nt, bar);
                } else {
                  const uint32_t rows_bytes = (uint32_t)P.nt * 16;
                  for (int g = 0; g < 2; ++g) {
                    ptx::bulk_g2s(dst + g * 32 * P.nt, blk + g * 16 * INT + r0 * 8, rows_bytes, bar);
                    ptx::bulk_g2s(dst + g * 32 * P.nt + rows_bytes, blk + g * 16 * INT + (INT + r0) * 8, rows_bytes,
                                  bar);
                  }
                }
              }
              if (++st == P.stages) { st = 0; ph ^= 1; }
            }
          continue;
        }
        for (int q = sg.q0; q < sg.q1; ++q) {
          if (P.dbg & 2048) ptx::mbar_wait_nohint(ptx::smem_u32(&S->empty[st]), ph ^ 1);
          else ptx::mbar_wait_sleep(ptx::smem_u32(&S->empty[st]), ph ^ 1);
          tr(P, 0, 0x100 | q);
          const uint32_t bar = ptx::smem_u32(&S->full[st]);
          const uint32_t sb = base + st * P.stage_bytes;
          const int ng = q == P.nq - 1 ? P.last_groups : 2;
          ptx::mbar_arrive_tx(bar, 2 * ng * P.nplanes * bytes + (P.wres ? 0u : P.b_bytes) + P.pb_bytes);
          if (P.proj)
            ptx::bulk_g2s(sb + P.nplanes * 4 * P.a_bytes + P.b_bytes, P.pw + ((int64_t)n_tile * P.nq + q) * 32 * P.nt,
                          P.pb_bytes, bar);
          for (int pl = 0; pl < P.nplanes; ++pl) {
            const uint32_t ps = sb + pl * 4 * P.a_bytes;
            for (int g = 0; g < ng; ++g) {
              const int64_t off = (2 * q + g) * a.in.kstride + P.plane_id[pl] * a.in.pstride + cs * 8;
              ptx::bulk_g2s(ps + g * P.a_bytes + slot0, hi + off, bytes, bar);
              ptx::bulk_g2s(ps + (2 + g) * P.a_bytes + slot0, lo + off, bytes, bar);
            }
          }
          if (P.wres) {
          } else if (P.b_img_nt == P.nt) {
            ptx::bulk_g2s(sb + P.nplanes * 4 * P.a_bytes, P.w + ((int64_t)n_tile * P.nq + q) * P.taps * 32 * P.nt,
                          P.b_bytes, bar);
          } else {
            // nt of the image's b_img_nt rows: per (tap, group) the hi and lo row ranges
            const int INT = P.b_img_nt, row0 = n_tile * P.nt, it = row0 / INT, r0 = row0 - it * INT;
            const uint32_t rows_bytes = (uint32_t)P.nt * 16;
            for (int t = 0; t < P.taps; ++t) {
              const __half* blk = P.w + (((int64_t)it * P.nq + q) * P.taps + t) * 32 * INT;
              for (int g = 0; g < 2; ++g) {
                const uint32_t dst = sb + P.nplanes * 4 * P.a_bytes + (uint32_t)(t * 32 * P.nt + g * 16 * P.nt) * 2;
                ptx::bulk_g2s(dst, blk + g * 16 * INT + r0 * 8, rows_bytes, bar);
                ptx::bulk_g2s(dst + rows_bytes, blk + g * 16 * INT + (INT + r0) * 8, rows_bytes, bar);
              }
            }
          }
          if (++st == P.stages) { st = 0; ph ^= 1; }
        }
      }
    }
  } else if (PAIR && warp == kWarpMma && (blockIdx.x & 1)) {
    // ===== pair mode, peer CTA: relay each landed stage to the leader =====
    const uint32_t full2 = ptx::mapa(ptx::smem_u32(&S->full2[0]), 0);
    int st = 0;
    uint32_t ph = 0;
    Seg sg;
    Band bd = {};
    for (int si = 0; seg_get<false, true>(P, bd, si, total_tiles, false, sg); ++si)
      for (int q = 0; q < P.nq; ++q) {
        if (lane == 0) {
          ptx::mbar_wait(ptx::smem_u32(&S->full[st]), ph);
          ptx::mbar_arrive_cluster(full2 + st * 8);
        }
        __syncwarp();
        if (++st == P.stages) { st = 0; ph ^= 1; }
      }
  } else if (warp == kWarpMma) {
    // ===== MMA issuer: whole warp, one elected lane issues; main products
    // rotate over the NP partial accumulators per stage (pair mode: the
    // leader, M = 256 over both CTAs) =====
    const uint32_t idesc = ptx::idesc_f16(PAIR ? 2 * kTileM : kTileM, P.nt);
    const uint32_t idesc2 = ptx::idesc_f16(PAIR ? 2 * kTileM : kTileM, 2 * P.nt);
    const uint32_t a_lbo = P.a_bytes, b_lbo = 2 * P.bn * 16;
    const bool do_mma = !(P.dbg & 2);
    // tap offsets in the descriptors' 16-byte address units
    uint64_t offs[TAPS];
#pragma unroll
    for (int t = 0; t < TAPS; ++t) offs[t] = (uint64_t)P.toff[t];
    const uint64_t bstep = (uint64_t)(64 * P.bn) >> 4, blo = (uint64_t)(P.bn * 16) >> 4;
    int st = 0;
    uint32_t ph = 0, acc = 0, acc_ph = 0;
    uint32_t w_seen = P.wres ? 0u : ~0u;  // resident chunks already waited for
    Seg sg;
    Band bd = {};
    if constexpr (BAND) bd = band_of(P);
    for (int si = 0; seg_get<BAND, PAIR>(P, bd, si, total_tiles, streamk, sg); ++si) {
      if constexpr (PAIR) ptx::mbar_wait_cluster(ptx::smem_u32(&S->acc_empty[acc]), acc_ph ^ 1);
      else ptx::mbar_wait(ptx::smem_u32(&S->acc_empty[acc]), acc_ph ^ 1);
      ptx::tc_fence_after();
      const uint32_t d_tile = tmem + acc * P.mt * set_cols;
      int p = 0;
      const int nsub = P.psub ? 4 : 1;
      const int q0 = sg.q0;
      for (int q = q0; q < sg.q1; ++q) {
       for (int ps = 0; ps < nsub; ++ps) {
        tr(P, 1, 0x400 | q);
        ptx::mbar_wait(ptx::smem_u32(&S->full[st]), ph);
        if constexpr (PAIR) ptx::mbar_wait_cluster(ptx::smem_u32(&S->full2[st]), ph);
        tr(P, 1, 0x500 | q);
        if (!((w_seen >> q) & 1u)) {
          ptx::mbar_wait(ptx::smem_u32(&S->wfull[q]), 0);
          w_seen |= 1u << q;
        }
        ptx::tc_fence_after();
        const uint32_t sb = base + st * P.stage_bytes;
        const uint64_t a_hi = ptx::smem_desc_noswz(sb, a_lbo, 128);
        const uint64_t a_lo = ptx::smem_desc_noswz(sb + 2 * P.a_bytes, a_lbo, 128);
        const uint64_t b0 = ptx::smem_desc_noswz(P.wres ? wres_base + (uint32_t)q * P.b_bytes : sb + P.nplanes * 4 * P.a_bytes,
                                                 b_lbo, 128);
        // first writes: main partial at its first chunk's first sub-stage,
        // correction at the tile's first sub-stage
        const uint32_t main_acc = (q - q0 >= NP || ps > 0) ? 1u : 0u;
        const uint32_t corr_acc = (q > q0 || ps > 0) ? 1u : 0u;
        if (do_mma) {
          for (int sub = 0; sub < P.mt; ++sub) {
            // sub-tile rows start 128 positions further in the same buffer
            const uint32_t d_set = d_tile + sub * set_cols;
            const uint32_t dm = P.concat ? d_set + p * 2 * P.nt : d_set + p * P.nt;
            const uint32_t dc = P.concat ? dm + P.nt : d_set + NP * P.nt;
            const uint64_t shift = (uint64_t)(sub * kTileM);
            if constexpr (TAPS == 9) {
              if (P.psub) {
                uint64_t o4[4];
#pragma unroll
                for (int t = 0; t < 4; ++t) o4[t] = (uint64_t)P.pl_toff[ps][t];
                const int ntp = P.pl_ntaps[ps];
                if (ntp == 4)
                  ss_stage<4, PAIR>(P.concat, dm, dc, a_hi + shift, a_lo + shift, b0, bstep, blo, idesc2, idesc, main_acc,
                              corr_acc, o4);
                else if (ntp == 2)
                  ss_stage<2, PAIR>(P.concat, dm, dc, a_hi + shift, a_lo + shift, b0, bstep, blo, idesc2, idesc, main_acc,
                              corr_acc, o4);
                else
                  ss_stage<1, PAIR>(P.concat, dm, dc, a_hi + shift, a_lo + shift, b0, bstep, blo, idesc2, idesc, main_acc,
                              corr_acc, o4);
                continue;
              }
            }
            ss_stage<TAPS, PAIR>(P.concat, dm, dc, a_hi + shift, a_lo + shift, b0, bstep, blo, idesc2, idesc,
                                 main_acc, corr_acc, offs);
            if (proj) {
              // projection: the centre tap's A, its weights after the taps'
              const uint64_t po[1] = {(uint64_t)P.ptoff};
              const uint32_t pm = d_set + set_a;
              const uint64_t bp = b0 + ((uint64_t)P.b_bytes >> 4);
              ss_stage<1, PAIR>(P.concat, pm, pm + P.nt, a_hi + shift, a_lo + shift, bp, bstep, blo, idesc2, idesc,
                          q > q0 ? 1u : 0u, q > q0 ? 1u : 0u, po);
            }
          }
        }
        if constexpr (PAIR) ptx::mma_commit2_warp(ptx::smem_u32(&S->empty[st]), 3);
        else ptx::mma_commit_warp(ptx::smem_u32(&S->empty[st]));
        tr(P, 1, 0x600 | q);
        if (++st == P.stages) { st = 0; ph ^= 1; }
       }
        if (++p == NP) p = 0;
      }
      if constexpr (PAIR) ptx::mma_commit2_warp(ptx::smem_u32(&S->acc_full[acc]), 3);
      else ptx::mma_commit_warp(ptx::smem_u32(&S->acc_full[acc]));
      if (++acc == (uint32_t)NB) { acc = 0; acc_ph ^= 1; }
    }
  } else if (warp < 8 * PAIRS) {
    // ===== epilogue: a tile's 16-column chunks (sub-tile, channel chunk)
    // k = 0 .. mt * nt / 16 - 1.  Unshared: warpgroup (buffer % 2) drains
    // the whole buffer; shared: both warpgroups drain every buffer, warpgroup
    // ew taking the chunks k = ew (mod 2), halving a tile's epilogue latency.
    // The warpgroup walks its (tile, chunk) items in order and issues the
    // next item's residual loads (across tiles too) before this item's math. =====
    // pairs (two pairs: 4 warpgroups): pair jp drains the tiles it = jp
    // (mod 2) -- consecutive tiles sit in different accumulator buffers --
    // and within a pair everything runs as with one pair of warpgroups
    const int wg = warp >> 2, ew = wg & 1, jp = wg >> 1, nwg = 2 * PAIRS;
    const EpiParams& e = a.epi;
    const int row = threadIdx.x & 127;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const float wsc = __ldg(P.wscale) * a.in.sload;  // weight scale, input storage scale
    EpiTab etab = P.etab;
    etab.ptab = ptab;
    const int hw = P.hp * P.wp;
    // items per sub-tile: nt / 16 chunks (a power of two), twice that with
    // a fused projection (chunk j >= nch: the projection's channel j - nch)
    const int nch = P.nt >> 4, nchx = proj ? 2 * nch : nch, lg_nch = __ffs(nchx) - 1, nk = P.mt * nchx;
    const int k0 = P.share_epi ? ew : 0, kstep = P.share_epi ? 2 : 1;
    const int lg_nb = __ffs(NB) - 1;
    // residual rows are staged in shared memory by cp.async one item ahead
    // ([buffer][word][thread] x 16 bytes: conflict-free 16-byte reads)
    const uint32_t skq = (uint32_t)nwg * 128 * 16;
    const uint32_t sk_slot = ptx::smem_u32(ptab + P.etab.rows * e.npad) + threadIdx.x * 16;
    // band mode: staging [warpgroup][2][128 rows][kStgPitch] then the ring
    // [2 slots][nchunk][wpo][16] (no residual, so the residual staging area is free)
    float* band_stage = ptab + ((P.etab.rows * e.npad + 3) & ~3);
    float* band_bnd = band_stage + 4 * kTileM * kStgPitch;  // [warpgroup][2][4 warps][16]
    float* band_ring = band_bnd + 4 * 64;
    const float band_div = (BAND && e.pool == PCNN_POOL_LOCAL) ? __ldg(e.pool_p) : 1.f;
    struct Item {
      int tile, k, n_tile, b, oy, ox, g;
      uint32_t it;  // segment index
      bool valid;
      int owner, c_lo;  // segment: runs the epilogue; first contributing CTA
      int nqs;          // segment chunks (partial accumulators beyond them were not written)
      int tn;           // segment's n-tile
      int64_t g0;       // segment's first grid position
      int r, rows;      // band mode: first grid row, grid rows
    };
    Band ebd = {};
    if constexpr (BAND) ebd = band_of(P);
    // this thread's row of sub-tile (k >> lg_nch) of the item's tile -> image, output row / column
    auto locate = [&](Item& x) {
      x.n_tile = x.tn;
      const int g = (int)x.g0 + (x.k >> lg_nch) * kTileM + row;
      x.g = g;
      if constexpr (BAND) {  // the pooled store decodes rows itself (band_pool)
        x.valid = true;
        x.b = x.oy = x.ox = 0;
        return;
      }
      int gy, gx;
      if (P.shared_grid) {
        // position 1 + R (W+1) + x, global row R = b (H+1) + y + 1
        const int g1 = g > 0 ? g - 1 : 0;
        const int R = (int)P.div_wp.div(g1);
        gx = g1 - R * P.wp;
        const int R1 = R > 0 ? R - 1 : 0;
        x.b = (int)P.div_h1.div(R1);
        gy = R1 - x.b * P.hp;
        x.valid = g >= 1 && R >= 1 && g < P.gtotal && gx < P.vx1 && gy < P.vy1 && x.b < a.batch;
      } else {
        x.b = (int)P.div_hw.div(g);
        const int r = g - x.b * hw;
        gy = (int)P.div_wp.div(r);
        gx = r - gy * P.wp;
        x.valid = g < P.gtotal && gy >= P.vy0 && gy < P.vy1 && gx >= P.vx0 && gx < P.vx1;
      }
      x.oy = gy - P.vy0;
      x.ox = gx - P.vx0;
    };
    // next item of this warpgroup; false past the last
    auto advance = [&](Item& x) -> bool {
      x.k += kstep;
      if (x.k < nk) return true;
      for (;;) {
        ++x.it;
        Seg sx;
        if (!seg_get<BAND, PAIR>(P, ebd, (int)x.it, total_tiles, streamk, sx)) return false;
        x.tile = sx.tile;
        x.tn = sx.n_tile;
        x.g0 = sx.g0;
        x.r = sx.r;
        x.rows = sx.rows;
        if constexpr (SK) {
          x.owner = sx.owner;
          x.c_lo = sx.c_lo;
          x.nqs = sx.q1 - sx.q0;
        }
        if (P.share_epi ? (NB == 1 ? jp == 0 : (int)(x.it & (uint32_t)(PAIRS - 1)) == jp)
                        : (int)((x.it & (uint32_t)(NB - 1)) % (uint32_t)nwg) == wg)
          break;
      }
      x.k = k0;
      return true;
    };
    auto chan = [&](const Item& x) { return x.n_tile * P.nt + (x.k & (nch - 1)) * 16; };
    const float pwsc = proj ? __ldg(P.pwscale) * a.in.sload : 0.f;
    EpiTab petab = P.petab;
    petab.ptab = ptab_p;
    int sk_checked = -1;  // flag mode: tile whose residual rows were acquired
    auto skip_async = [&](const Item& x, uint32_t dst) {
      if (a.fsk.mode && x.tile != sk_checked) {
        // the producer warp acquired this tile's residual rows (x.it + 1
        // tiles so far): CTA-scope acquire of its hand-off
        if (lane == 0) {
          uint32_t spins = 0;
          for (;;) {
            int v;
            asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(ptx::smem_u32(&S->dep_seq))
                         : "memory");
            if (v > (int)x.it) break;
            __nanosleep(32);
            if (++spins > (1u << 26)) __trap();
          }
        }
        __syncwarp();
        sk_checked = x.tile;
      }
      if (P.skip_pos)
        load16_async_at(e.skip, (int64_t)(chan(x) >> 3) * e.skip.kstride + (int64_t)x.g * 8, x.valid, dst, skq);
      else
        load16_async(e.skip, x.b, chan(x), x.oy, x.ox, x.valid, dst, skq);
    };
    Item cur;
    cur.tile = -1;
    cur.it = ~0u;
    cur.k = nk;
    cur.owner = 1;
    cur.c_lo = -1;
    cur.nqs = P.nq;
    bool have = advance(cur);
    uint32_t par = 0;  // staging buffer of the current item
    if (have) {
      locate(cur);
      if (e.residual) skip_async(cur, sk_slot);
    }
    while (have) {
      Item nxt = cur;
      const bool have_next = advance(nxt);
      const bool last_of_tile = !have_next || nxt.it != cur.it;
      if (have_next) {
        if (nxt.it != cur.it || (nxt.k >> lg_nch) != (cur.k >> lg_nch)) locate(nxt);
        if (e.residual) skip_async(nxt, sk_slot + (par ^ 1) * 4 * skq);
      }
      const uint32_t acc = cur.it & (NB - 1);  // NB is 1, 2 or 4
      if (cur.k == k0) {
        if (lane == 0 && warp == 0) tr(P, 2, 0x700);
        ptx::mbar_wait_warp(ptx::smem_u32(&S->acc_full[acc]), (cur.it >> lg_nb) & 1);
        if (lane == 0 && warp == 0) tr(P, 2, 0x800);
        ptx::tc_fence_after();
      }
      const int sub = cur.k >> lg_nch, c0 = (cur.k & (nch - 1)) * 16;
      const bool pj = proj && (cur.k & nch);  // a projection item
      const uint32_t d_set = tmem + lane_off + (acc * P.mt + sub) * set_cols + (pj ? set_a : 0u);
      if (!(P.dbg & 4)) {
        float v[16], t[16];
        // the projection has one main partial and its correction; a stream-K
        // segment shorter than NP chunks wrote only its first partials
        const int npi = pj ? 1 : (SK && cur.nqs < NP ? cur.nqs : NP);
        if (P.concat) {
          ptx::tmem_ld16x2(d_set + P.nt + c0, d_set + c0, v, t);
          add_n<16>(v, t);
          for (int p = 1; p < npi; ++p) {
            float u[16];
            ptx::tmem_ld16x2(d_set + 2 * p * P.nt + P.nt + c0, d_set + 2 * p * P.nt + c0, u, t);
            add_n<16>(u, t);
            add_n<16>(v, u);
          }
        } else {
          // correction after all NP main partials (projection: after its one)
          ptx::tmem_ld16x2(d_set + (pj ? 1 : NP) * P.nt + c0, d_set + c0, v, t);
          add_n<16>(v, t);
          for (int p = 1; p < npi; ++p) {
            ptx::tmem_ld16(d_set + p * P.nt + c0, t);
            add_n<16>(v, t);
          }
        }
        if (last_of_tile) {
          // the accumulators are in registers: release the buffer to the MMA warp
          // (pair mode: the leader's)
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (PAIR) ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&S->acc_empty[acc]), 0));
            else ptx::mbar_arrive(ptx::smem_u32(&S->acc_empty[acc]));
          }
        }
        if (lane == 0 && warp == 0) tr(P, 2, 0xD00 | c0);
        float sk[16];
        if (e.residual) {
          // this item's group is complete once at most the next one is pending
          if (have_next) asm volatile("cp.async.wait_group 1;" ::: "memory");
          else asm volatile("cp.async.wait_group 0;" ::: "memory");
          Raw16 r;
          lds_raw16(sk_slot + par * 4 * skq, skq, r);
          decode16_raw(e.skip, r, sk, P.fold_skip ? 1.f : e.skip.sload);
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) sk[i] = 0.f;
        }
        if (streamk && !cur.owner) {
          // stream-K partial: this CTA's chunks of the tile, raw, to its slot;
          // the last draining warp publishes the slot (GPU-scope release,
          // cumulative over the stores the CTA-scope counter ordered before it)
          float4* dst = reinterpret_cast<float4*>(a.sk_slots + (((size_t)blockIdx.x * nk + cur.k) * 128 + row) * 16);
#pragma unroll
          for (int i = 0; i < 4; ++i) __stcg(dst + i, make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]));
          if (last_of_tile) {
            // every lane fences its own slot stores at GPU scope (the CTA
            // counter alone left partials invisible to the owner now and then)
            __threadfence();
            __syncwarp();
            if (lane == 0) {
              const uint32_t nsig = P.share_epi ? 8u : 4u;
              uint32_t old;
              asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                           : "=r"(old) : "r"(ptx::smem_u32(&S->tstored[cur.it & (kSigRing - 1)])) : "memory");
              if (old % nsig == nsig - 1)
                asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(a.sk_flags + blockIdx.x) : "memory");
            }
          }
        } else {
          if (streamk && cur.c_lo >= 0) {
            // owner of a tile whose earlier chunks lower CTAs computed: add
            // their published partials (each published its one partial
            // segment first, so these waits are short)
            if (cur.k == k0) {
              if (lane == 0)
                for (int c = cur.c_lo; c < (int)blockIdx.x; ++c) {
                  uint32_t spins = 0;
                  for (;;) {
                    int f;
                    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(f) : "l"(a.sk_flags + c) : "memory");
                    if (f >= 1) break;
                    __nanosleep(64);
                    if (++spins > (1u << 25)) __trap();
                  }
                }
              __syncwarp();
            }
            for (int c = cur.c_lo; c < (int)blockIdx.x; ++c) {
              const float4* src = reinterpret_cast<const float4*>(a.sk_slots + (((size_t)c * nk + cur.k) * 128 + row) * 16);
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float4 f = __ldcg(src + i);
                v[4 * i] += f.x; v[4 * i + 1] += f.y; v[4 * i + 2] += f.z; v[4 * i + 3] += f.w;
              }
            }
          }
          if constexpr (POOL == kPoolBand) {
            // the item's 128 conv outputs (bias / affine / poly applied):
            // the owner of each pooled column folds them in (band_item)
            epi_point16(e, etab, v, wsc, sk, chan(cur));
            if (!(P.dbg & 4096))
              band_item(P, e, ebd, band_ring, band_stage + ((ew * 2 + par) * kTileM) * kStgPitch,
                        band_bnd + (ew * 2 + par) * 64, cur.r, cur.rows, row, lane, warp & 3, ew, chan(cur), v,
                        band_div);
          } else if (kProj && pj) {
            epi_chunk16<true>(P.pe, petab, v, pwsc, sk, chan(cur), cur.valid, cur.valid ? cur.b : 0, cur.oy,
                               cur.ox, lane, -1, P.pe.out.sstore);
          } else {
            epi_chunk16<true>(e, etab, v, wsc, sk, chan(cur), cur.valid, cur.valid ? cur.b : 0, cur.oy, cur.ox,
                               lane, P.out_pos ? (int64_t)cur.g * 8 : -1, P.fold_out ? 1.f : e.out.sstore);
          }
        }
        if (lane == 0 && warp == 0) tr(P, 2, 0xE00 | c0);
        if (last_of_tile && a.sig_done) {
          // this warp's rows of the tile are stored: __syncwarp orders the
          // lanes' stores before lane 0's CTA-scope acq_rel count; the last
          // draining warp of the tile publishes it with a GPU-scope release
          // (cumulative over the stores the counter ordered before it)
          __syncwarp();
          if (lane == 0) {
            const uint32_t nsig = P.share_epi ? 8u : 4u;
            uint32_t old;
            asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                         : "=r"(old) : "r"(ptx::smem_u32(&S->tstored[cur.it & (kSigRing - 1)])) : "memory");
            if (old % nsig == nsig - 1) {
              const int m_tile = cur.tile - cur.n_tile * P.m_tiles;
              asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(a.sig_done + m_tile) : "memory");
              asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(a.sig_done + P.m_tiles) : "memory");
            }
          }
        }
      } else if (last_of_tile) {
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (PAIR) ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&S->acc_empty[acc]), 0));
          else ptx::mbar_arrive(ptx::smem_u32(&S->acc_empty[acc]));
        }
      }
      if (last_of_tile && lane == 0 && warp == 0) tr(P, 2, 0x900);
      if (!have_next) break;
      par ^= 1;
      if (nxt.it == cur.it && (nxt.k >> lg_nch) == (cur.k >> lg_nch)) {
        nxt.b = cur.b; nxt.oy = cur.oy; nxt.ox = cur.ox; nxt.valid = cur.valid; nxt.n_tile = cur.n_tile;
      }
      cur = nxt;
    }
  }
  cta_stamp(P, 2);
  __syncthreads();
  // pair mode: neither CTA leaves while the other may still arrive on its barriers
  if constexpr (PAIR) ptx::cluster_sync();
  tl_mark(a.tl, 1);
  if (warp == kWarpProducer) {
    ptx::tc_fence_after();
    if constexpr (PAIR) ptx::tmem_dealloc2(tmem, P.tmem_cols);
    else ptx::tmem_dealloc(tmem, P.tmem_cols);
  }
  cta_stamp(P, 3);
}

// residual staging: [2 buffers][4 words][epilogue threads] x 16 bytes
inline uint32_t ss_skip_stage(int pairs) { return 2u * 4u * 256u * 16u * (uint32_t)pairs; }

size_t ss_aux_bytes(const SsParams& P) {
  const size_t band =
      P.band ? 16 + (size_t)(4 * kTileM * kStgPitch + 4 * 64 + 2 * (P.brows / 2 + 2) * P.nchunk * P.wpo * 16) * 4 : 0;
  return ((sizeof(Smem) + 15) & ~size_t(15)) + (size_t)P.etab.rows * P.a.epi.npad * 4 +
         (P.proj ? (size_t)P.petab.rows * P.pe.npad * 4 : 0) + (P.a.epi.residual ? ss_skip_stage(P.epi_pairs) : 0) + band;
}

// nt: output channels per tile (the weight image is packed in tiles of
// min(npad, 128) rows; a smaller nt copies its rows out of that image)
static bool make_ss_params_nt(const ConvArgs& a, SsParams& P, int nt, bool psub, bool allow_wres, int force_mt = 0,
                              int max_np = 0, int pairs = 1, int pair = 0) {
  const TensorView& in = a.in;
  P.epi_pairs = pairs;
  P.pair = pair;
  if (!a.f16 || !a.tcwss || !a.tc16_scale) return false;
  if ((a.stride != 1 && a.stride != 2) || a.kh != a.kw ||
      !((a.kh == 3 && a.pad == 1) || (a.kh == 1 && a.pad == 0) || (a.kh == 4 && a.pad == 1 && a.stride == 1)))
    return false;
  const bool pooled = a.epi.pool == PCNN_POOL_LOCAL || a.epi.pool == PCNN_POOL_BI2;
  if (a.epi.pool != PCNN_POOL_NONE && a.epi.pool != PCNN_POOL_GLOBAL && !pooled) return false;
  if (!(in.cpad() == 4 || in.cpad() == 8 || in.cpad() % 16 == 0) || a.npad < 16 || a.npad % 16) return false;
  // stride 1 reads the padded grid, stride 2 the parity planes
  if (in.split != (a.stride == 2 ? 2 : 1)) return false;
  // band mode (pooled epilogue): stride-1 convs on the shared-border grid
  // whose grid rows fit one 128-row tile, >= 32 channels per tile (an even
  // number of 16-channel chunks: each warpgroup owns fixed chunks)
  if (pooled && (a.stride != 1 || a.epi.residual || a.proj || nt < 32 || in.wp > kTileM || a.epi.out.w > kTileM ||
                 !((a.kh == 3 && a.kw == 3) || (a.kh == 4 && a.kw == 4))))
    return false;
  const int cpad = in.cpad();
  P.a = a;
  P.b_img_nt = a.npad <= 128 ? a.npad : 128;
  P.nt = nt;
  if (a.npad % P.nt || P.b_img_nt % P.nt) return false;
  P.n_tiles = a.npad / P.nt;
  P.hp = in.hp;
  P.wp = in.wp;
  P.shared_grid = a.stride == 1;
  P.gtotal = a.stride == 1 ? in.kstride / 8 : (int64_t)a.batch * in.hp * in.wp;
  if (P.gtotal >= (1ll << 31)) return false;
  // two 128-row sub-tiles per tile for small N: one stage, one weight copy
  // and one set of hand-offs serve 256 positions
  P.mt = a.opt.ss_mt ? a.opt.ss_mt : (P.nt <= 32 ? 2 : 1);
  if (force_mt) P.mt = force_mt;
  if (P.pair) P.mt = 1;
  P.bn = P.pair ? P.nt / 2 : P.nt;
  P.band = 0;
  if (pooled) {
    P.band = 1;
    P.mt = 1;  // an item is a whole tile's rows (band_pool reads them from one staging buffer)
    P.brows = a.epi.pool == PCNN_POOL_LOCAL ? 1 : kTileM / in.wp;  // LOCAL: one grid row per tile (band_item)
    if (a.epi.pool == PCNN_POOL_LOCAL) {
      P.pk = a.epi.pool_k;
      P.ps = a.epi.pool_s;
      P.pp = a.epi.pool_pad;
    } else {
      P.pk = 2;
      P.ps = 2;
      P.pp = 0;
    }
    // LOCAL: s = 2 with (k, p) = (3, 1) or (2, 0) -- a window row is the owner lane and its neighbours
    if (P.ps != 2 || !((P.pk == 3 && P.pp == 1) || (P.pk == 2 && P.pp == 0))) return false;
    P.ho = a.pm.ho;
    P.wo = a.pm.wo;
    P.hpo = a.epi.out.h;
    P.wpo = a.epi.out.w;
    if (P.hpo != (P.ho + 2 * P.pp - P.pk) / P.ps + 1 || P.wpo != (P.wo + 2 * P.pp - P.pk) / P.ps + 1) return false;
    if (a.epi.pool == PCNN_POOL_BI2 && (2 * P.wpo > P.wo || 2 * P.hpo > P.ho)) return false;
    P.prows = a.batch * P.hpo;
    P.nchunk = a.npad / 16;
    P.nbands = 1;  // set per launch (launch_conv_ss)
  }
  if (P.mt < 1 || P.mt > 4) P.mt = 1;
  const int tm = kTileM * P.mt;
  P.m_tiles = (int)((P.gtotal + tm - 1) / tm);
  if (P.pair) P.m_tiles = (P.m_tiles + 1) & ~1;  // whole pairs (a last odd m-tile's partner stores nothing)
  P.nq = (cpad + 15) / 16;
  P.last_groups = cpad % 16 == 0 ? 2 : 1;
  P.taps = a.kh * a.kw;
  if (a.stride == 1) {
    // shared-border grid; tap (ky, kx) of output g reads g + (ky - pad) wp + kx - pad
    // (the 4x4 space-to-depth stem reaches one position back, two forward)
    P.nplanes = 1;
    P.plane_id[0] = 0;
    P.halo = a.pad * in.wp + a.pad;
    P.span = tm + P.halo + (a.kh - 1 - a.pad) * in.wp + (a.kw - 1 - a.pad);
    P.vy0 = P.vx0 = 0;
    P.vy1 = a.pm.ho;  // = in.h for "same" convs; one less for the 4x4 stem
    P.vx1 = a.pm.wo;
    for (int t = 0; t < P.taps; ++t) P.toff[t] = (t / a.kw) * in.wp + t % a.kw;
  } else {
    // parity planes: padded input (2y + ky, 2x + kx) = plane (ky & 1, kx & 1)
    // at (y + ky / 2, x + kx / 2); a 1x1 conv reads plane (1, 1) at (y, x)
    const int ho = (in.h + 2 * a.pad - a.kh) / 2 + 1, wo = (in.w + 2 * a.pad - a.kw) / 2 + 1;
    P.halo = 0;
    P.vy0 = P.vx0 = 0;
    P.vy1 = ho;
    P.vx1 = wo;
    if (a.kh == 1) {
      P.nplanes = 1;
      P.plane_id[0] = 3;
      P.span = tm;
      P.toff[0] = 0;
    } else {
      P.nplanes = 4;
      for (int i = 0; i < 4; ++i) P.plane_id[i] = i;
      P.span = tm + in.wp + 1;
    }
  }
  if (a.stride == 2 && a.kh == 3)
    for (int t = 0; t < 9; ++t) {
      const int ky = t / 3, kx = t % 3;
      P.toff[t] = (((ky & 1) << 1) | (kx & 1)) * 4 * P.span + (ky >> 1) * in.wp + (kx >> 1);
    }
  P.psub = 0;
  if (psub) {
    if (!(a.stride == 2 && a.kh == 3)) return false;
    P.psub = 1;
    P.nplanes = 1;  // stage layout: one plane
    for (int pl = 0; pl < 4; ++pl) P.pl_ntaps[pl] = 0;
    for (int t = 0; t < 9; ++t) {
      const int ky = t / 3, kx = t % 3, pl = ((ky & 1) << 1) | (kx & 1);
      const int j = P.pl_ntaps[pl]++;
      P.pl_tap[pl][j] = t;
      P.pl_toff[pl][j] = (ky >> 1) * in.wp + (kx >> 1);
    }
    for (int pl = 0; pl < 4; ++pl)
      for (int j = P.pl_ntaps[pl]; j < 4; ++j) P.pl_tap[pl][j] = P.pl_toff[pl][j] = 0;
  }
  P.w = reinterpret_cast<const __half*>(a.tcwss);
  P.wscale = a.tc16_scale + 1;
  P.etab = epi_tab_layout(a.epi);
  auto same_grid = [&](const TensorView& t) {
    return P.shared_grid && t.split == 1 && !t.is_vector && t.hp == in.hp && t.wp == in.wp && P.vy0 == 0 &&
           P.vx0 == 0;
  };
  P.out_pos = a.epi.pool == PCNN_POOL_NONE && same_grid(a.epi.out);
  P.skip_pos = a.epi.residual && same_grid(a.epi.skip);
  // split residual read by S: its load scale goes into S's rows; split output
  // at a position (no pool) after a poly or S: its storage scale goes into them
  P.fold_skip = a.epi.residual >= 2 && a.epi.skip.split;
  P.fold_out = P.out_pos && (a.epi.poly_deg > 0 || a.epi.residual >= 2);
  P.a_bytes = (uint32_t)P.span * 16;
  P.b_bytes = (uint32_t)(P.psub ? 4 : P.taps) * 64 * P.bn;  // psub: at most 4 taps per plane
  P.proj = 0;
  P.pb_bytes = 0;
  if (a.proj) {
    // the projection reads the 3x3 conv's centre tap: same input tensor,
    // stride, output channels and tiles; no residual / pool on either side
    const ConvArgs& q = *a.proj;
    if (P.psub || P.b_img_nt != P.nt || a.kh != 3 || a.pad != 1 || q.kh != 1 || q.kw != 1 || q.pad != 0 ||
        q.stride != a.stride || q.npad != a.npad || q.in.base != a.in.base || !q.f16 || !q.tcwss || !q.tc16_scale ||
        a.epi.residual || q.epi.residual || q.epi.pool != PCNN_POOL_NONE || a.epi.pool != PCNN_POOL_NONE)
      return false;
    P.proj = 1;
    P.pe = q.epi;
    P.petab = epi_tab_layout(q.epi);
    P.pw = reinterpret_cast<const __half*>(q.tcwss);
    P.pwscale = q.tc16_scale + 1;
    P.pb_bytes = 64u * P.nt;
    P.ptoff = P.toff[4];
  }
  P.stage_bytes = P.nplanes * 4 * P.a_bytes + P.b_bytes + P.pb_bytes;
  const size_t budget = 225 * 1024 - 128 - ss_aux_bytes(P);
  P.stages = (int)(budget / P.stage_bytes);
  if (P.stages > kMaxStages) P.stages = kMaxStages;
  // resident weights when one n-tile covers every output channel and the
  // image leaves room for at least min(4, streamed stages) activation stages
  P.wres = 0;
  P.res_bytes = 0;
  {
    const bool want = a.opt.ss_wres != 0;
    const uint32_t res = (uint32_t)P.nq * P.b_bytes, sa = P.nplanes * 4 * P.a_bytes;
    if (want && allow_wres && !P.pair && !P.psub && !P.proj && P.b_img_nt == P.nt && P.n_tiles == 1 && P.nq <= kMaxWChunks &&
        res < budget) {
      int st = (int)((budget - res) / sa);
      if (st > kMaxStages) st = kMaxStages;
      if (st >= 2 && st >= (P.stages < 4 ? P.stages : 4)) {
        P.wres = 1;
        P.res_bytes = res;
        P.stage_bytes = sa;
        P.stages = st;
      }
    }
  }
  if (P.stages < 2) return false;  // neither two streamed stages nor resident weights + two stages fit
  P.dbg = a.opt.dbg;
  // multi-lane issue pays on narrow tiles (RN20); on 128-channel tiles the
  // one-lane producer measured faster (RN18 1106 -> 1087 us, VGG 393 -> 383)
  P.wide = (a.opt.ss_wide == 2 || (a.opt.ss_wide == 1 && P.nt <= 64)) && !P.psub && !P.band && !a.fin.mode &&
           !a.fsk.mode;
  P.time_slot = -1;
  // accumulators: as many partials as accuracy asks for, then two buffers
  // main products rotate over the partials per stage (taps MMAs each)
  const int stages_per_partial = kAddsPerPartial / P.taps > 0 ? kAddsPerPartial / P.taps : 1;
  int want = (P.nq + stages_per_partial - 1) / stages_per_partial;
  want = want < 1 ? 1 : (want > kMaxPartials ? kMaxPartials : want);
  if (max_np && want > max_np) want = max_np;
  P.concat = P.nt <= 64;
  P.partials = 0;
  for (int wp = want; wp >= 1 && !P.partials; --wp) {
    const int set = (P.concat ? wp * 2 * P.nt : (wp + 1) * P.nt) + (P.proj ? 2 * P.nt : 0);
    // up to four buffers: the MMA warp runs ahead of two epilogue warpgroups
    for (int nb = kMaxAcc; nb >= 1 && !P.partials; --nb)
      if (nb * P.mt * set <= 512 && nb != 3) { P.partials = wp; P.acc_bufs = nb; }
  }
  if (!P.partials) return false;
  const uint32_t set =
      (P.concat ? P.partials * 2 * P.nt : (P.partials + 1) * P.nt) + (P.proj ? 2u * P.nt : 0u);
  const uint32_t need = P.acc_bufs * P.mt * set;
  P.tmem_cols = need <= 32 ? 32 : need <= 64 ? 64 : need <= 128 ? 128 : need <= 256 ? 256 : 512;
  // shared epilogue when a tile has an even number of 16-column chunks
  P.share_epi = a.opt.ss_share >= 0 ? a.opt.ss_share : ((P.mt * (P.proj ? 2 : 1) * P.nt / 16) % 2 == 0);
  if (P.band) P.share_epi = 1;  // chunk k always drains on warpgroup k % 2 (ring ownership)
  if (P.band) P.epi_pairs = 1;
  P.div_hw = make_fastdiv((uint32_t)(P.hp * P.wp));
  P.div_h1 = make_fastdiv((uint32_t)P.hp);
  P.div_wp = make_fastdiv((uint32_t)P.wp);
  P.div_mt = make_fastdiv((uint32_t)P.m_tiles);
  return true;
}

// Staging choice: whole-chunk stages (a 16-channel chunk of every plane and
// all taps' weights) when two fit; else, for 3x3 stride 2, one parity plane
// per stage (measured: faster than 64-channel tiles, slower than whole-chunk
// stages when those fit); else two 64-channel tiles.  Option ss_psub 0/1 forces.
static bool make_ss_params_pairs(const ConvArgs& a, SsParams& P, bool allow_wres, int pairs) {
  const int nt = a.npad <= 128 ? a.npad : 128;
  const int force = a.opt.ss_psub;
  if (force == 1 && make_ss_params_nt(a, P, nt, true, allow_wres, 0, 0, pairs)) return true;
  if (make_ss_params_nt(a, P, nt, false, allow_wres, 0, 0, pairs)) return true;
  if (force != 0 && make_ss_params_nt(a, P, nt, true, allow_wres, 0, 0, pairs)) return true;
  return nt == 128 && make_ss_params_nt(a, P, 64, false, allow_wres, 0, 0, pairs);
}

// Two epilogue pairs (four warpgroups) for narrow layers (<= 32 output
// channels, or <= 64 with a fused projection, whose tiles carry twice the
// epilogue items): measured per unit, RN20's downsampling convs with their
// projections 17.8 -> 15.3 us and 17.0 -> 14.8 us, while RN18's 64-channel
// 56 x 56 layers and its stem run slower at the 112-register budget (50 ->
// 54 us, 204 -> 234 us).  Only when the same staging choice still holds
// with the larger residual staging area and keeps its pipeline depth.
bool make_ss_params(const ConvArgs& a, SsParams& P, bool allow_wres = true) {
  SsParams P1 = P;
  if (!make_ss_params_pairs(a, P1, allow_wres, 1)) return false;
  // CTA pairs for 128-channel tiles whose weights are re-staged per tile
  // (RN18 stages 2-4, VGG's wide layers): halves every SM's weight traffic
  if (a.opt.ss_pair && P1.nt == 128 && P1.b_img_nt == 128 && !P1.wres && !P1.psub && !P1.proj && !P1.band &&
      P1.taps == 9 && P1.mt == 1 && P1.m_tiles >= 2 && !a.sk_flags && !a.sig_done && !a.fin.mode && !a.fsk.mode &&
      !a.proj) {
    SsParams Q = P;
    if (make_ss_params_nt(a, Q, 128, false, false, 1, 0, 1, 1) && Q.stages >= 2) {
      P = Q;
      return true;
    }
  }
  if (a.opt.epi_pairs >= 2 && (P1.nt <= 32 || (P1.nt <= 64 && (P1.proj || a.opt.epi_pairs >= 3)) || a.opt.epi_pairs >= 4) &&
      !P1.band && !a.sk_flags) {
    SsParams Q = P;
    if (make_ss_params_nt(a, Q, P1.nt, P1.psub != 0, allow_wres, 0, 0, 2) && Q.wres == P1.wres &&
        Q.mt == P1.mt && Q.stages >= (P1.stages < 3 ? P1.stages : 3)) {
      P = Q;
      return true;
    }
  }
  P = P1;
  return true;
}

// =====================================================================
// Image-resident residual stages (conv_blk_kernel): a run of stride-1 3x3
// convs on one grid with C = 32..128 channels (ResNet-20's identity blocks
// and the conv that follows a downsampling block) in ONE launch.  Each CTA
// takes whole images; an image's activations never leave shared memory
// between the run's layers: the run's external input (and external residual)
// are bulk-copied in, every layer's output is written by the epilogue as a
// split hi/lo tensor into a shared-memory slot in the halo layout, and the
// next layer's MMAs read it there (the same fixed-offset tap descriptors as
// conv_ss).  Only the last layer stores to global memory (or into the global
// pool sums).  Whole images need no halo recompute: the shared zero border
// rows / columns of the grid are the padding.
//
// Pipelining inside the CTA.  One resident image (ni = 1): accumulators
// alternate between two TMEM buffers by layer; the epilogue releases output
// chunk q of layer l (16 channels, all positions) through ready[q], so the
// MMA warp starts layer l+1's chunk q while later chunks of layer l are
// still draining.  Two resident images (ni = 2, when both images' slots fit):
// each image owns a slot set and a TMEM buffer, and the MMA warp alternates
// between them layer by layer, so one image's epilogue runs under the other
// image's MMAs (a layer's epilogue is as long as its MMAs; with one image the
// two only overlap per chunk).  Weights stream through a ring (one stage = one
// 16-channel chunk, all taps), in MMA order.
//
// Slot planes are P_img positions long: a sub-tile's A reads run past the
// image into the next plane (or the weight ring) only for rows whose outputs
// are discarded.
// =====================================================================
constexpr int kBlkMaxLayers = 7;  // ResNet-20 stage 1 with its stem: 1 + 6 convs
// the image-resident kernels run four epilogue warpgroups (warps 0-15), the
// producer (16) and the MMA warp (17): an epilogue item is a long dependent
// chain (accumulator wait, TMEM load, table reads, stores, proxy fence,
// arrive), and twice the warps per sub-partition hide it
#ifndef PCNN_BLK_MMA_WARPS
#define PCNN_BLK_MMA_WARPS 2
#endif
// conv_blk_kernel: with two resident images one MMA-issuing warp per image
// (kWaveMma + i), so one image's barrier waits overlap the other's MMA issue
constexpr int kBlkMmaWarps = PCNN_BLK_MMA_WARPS;
constexpr int kWaveProducer = 16, kWaveMma = 17, kWaveThreads = 32 * (kWaveMma + kBlkMmaWarps);
constexpr int kBlkMaxChunks = 8;
constexpr int kBlkStages = 4;

struct BlkLayer {
  EpiParams epi;       // this layer's epilogue; epi.out is the global output (last layer only)
  EpiTab etab;
  const __half* w;     // tcss weight image (one n-tile = all C output channels)
  const float* wscale; // its 2^-e
  int in_slot, res_slot, out_slot;  // res_slot -1: no residual; out_slot -1: global output
  int ptab_off;        // floats into the CTA's parameter-table area
  float in_sload;      // storage load scale of the input (the external input; 1 for slots)
  float res_sload;     // same for the residual
  int res_ext;         // the residual is an external tensor (wait for its copy)
};

struct BlkParams {
  BlkLayer L[kBlkMaxLayers];
  int nl, C, nq;
  int H, W, wp;        // image, grid row pitch W + 1
  int S;               // 128-row sub-tiles per image
  int p_out0, nout;    // first output position (1 + wp), output positions H * wp
  int P_img;           // positions per external copy: (H + 2) wp
  uint32_t plane;      // bytes per (8-channel group, hi | lo) plane of a slot
  uint32_t slot_bytes; // nq * 4 * plane
  uint32_t set_bytes;  // nslots * slot_bytes: one resident image
  int nslots;
  int ni;              // resident images per CTA (1 or 2)
  int ext_in_slot, ext_res_slot;
  int ext_in_groups;   // 8-channel groups the external input stores (wave mode: 1 for a 3-channel stem input)
  TensorView ext_in, ext_res;
  int batch;
  int stages;
  uint32_t b_bytes;    // one chunk of weights: 9 taps x 64 C bytes
  uint32_t tmem_cols;
  uint32_t set_cols;   // accumulator columns per sub-tile: [main C | corr C]
  int ptab_floats;
  int pos_off;         // floats into the table area: [S][128] packed (inside, valid, y, x) of each
                       // epilogue row of each sub-tile (blk_pos_fill; same for every layer and image)
  int wsc_off;         // floats into the table area: every layer's weight scale x input load scale
  int toff[9];         // tap (ky, kx) -> ky wp + kx (A base = first output position - (wp + 1))
  int* flag;           // the plan's status word (an activation left the fp16 range)
  unsigned long long* tl;
  int dbg;             // debug bit 32: CTA-0 event trace (built with -DPCNN_SS_TRACE)
  // wave mode (conv_wave_kernel, C = 16): one image per CTA, every layer's
  // weights resident, accumulators in a ring of R sub-tile buffers
  int wave, R;
};

// position table of the image-resident kernels' epilogue: row `row` of
// sub-tile s is grid position p = p_out0 + 128 s + row, image row y and
// column x; bit 31 = inside the output rows, bit 30 = a real output column
__device__ __forceinline__ void blk_pos_fill(const BlkParams& P, int* tab, int tid, int nthreads) {
  for (int i = tid; i < P.S * 128; i += nthreads) {
    const int p = P.p_out0 + i;
    const int y = (p - 1) / P.wp - 1, x = p - 1 - (y + 1) * P.wp;
    const bool inside = p < P.p_out0 + P.nout, valid = inside && x < P.W;
    tab[i] = (inside ? (1 << 31) : 0) | (valid ? (1 << 30) : 0) | ((y & 0x7FFF) << 15) | (x & 0x7FFF);
  }
}
// Every layer's epilogue table and weight scale in one pass: a thread issues
// all of its (read-only) global loads before its first store, so a cold
// start pays one memory round trip, not one per layer (measured after an L2
// flush: ~0.8 us per layer of launch gap)
__device__ __forceinline__ void blk_fill_tabs(const BlkParams& P, float* ptab, int tid, int nthreads) {
  const int total = P.pos_off;  // the layers' tables (each padded to 4 floats)
  for (int base = tid; base < total + P.nl; base += 4 * nthreads) {
    float v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = base + k * nthreads;
      v[k] = 0.f;
      if (i < total) {
        int l = 0;
        for (int q = 1; q < P.nl; ++q)
          if (i >= P.L[q].ptab_off) l = q;
        const int j = i - P.L[l].ptab_off;
        if (j < P.L[l].etab.rows * P.C) v[k] = epi_tab_value(P.L[l].epi, P.L[l].etab, j, 1.f, 1.f);
      } else if (i < total + P.nl) {
        v[k] = __ldg(P.L[i - total].wscale) * P.L[i - total].in_sload;
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = base + k * nthreads;
      if (i < total) ptab[i] = v[k];
      else if (i < total + P.nl) ptab[P.wsc_off + i - total] = v[k];
    }
  }
}
__device__ __forceinline__ void blk_pos_get(const int* tab, int s, int row, bool& inside, bool& valid, int& y,
                                            int& x) {
  const int v = tab[s * 128 + row];
  inside = v < 0;
  valid = (v >> 30) & 1;
  y = (v >> 15) & 0x7FFF;
  x = v & 0x7FFF;
}

// CTA-0 event trace of the block kernel (region: 0 producer, 1 MMA, 2 epilogue warp 0)
struct BlkTracer {
  uint32_t n = 0;
  __device__ __forceinline__ void operator()(const BlkParams& P, int region, uint32_t tag) {
#ifdef PCNN_SS_TRACE
    if ((P.dbg & 32) && blockIdx.x == 0 && n < kTraceRegion)
      g_ss_trace[region * kTraceRegion + n++] = ((unsigned long long)tag << 48) | (clock64() & 0xFFFFFFFFFFFFull);
#else
    (void)P; (void)region; (void)tag;
#endif
  }
};

struct BlkSmem {
  uint64_t wfull[kBlkStages], wempty[kBlkStages];
  uint64_t acc_full[2], acc_empty[2];
  uint64_t ready[kBlkMaxChunks];
  uint64_t ext_full[2], img_free[2];
  uint32_t tmem_base;
};

__global__ void __launch_bounds__(kWaveThreads, 1) conv_blk_kernel(const __grid_constant__ BlkParams P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  const uint32_t slots = ptx::smem_u32(smem);
  const uint32_t ring = slots + (uint32_t)P.ni * P.set_bytes;
  BlkSmem* S = reinterpret_cast<BlkSmem*>(smem + (size_t)P.ni * P.set_bytes + (size_t)P.stages * P.b_bytes);
  float* ptab = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(S) + ((sizeof(BlkSmem) + 15) & ~size_t(15)));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = (int)gridDim.x;
  if (threadIdx.x == 0) {
    for (int i = 0; i < P.stages; ++i) {
      ptx::mbar_init(ptx::smem_u32(&S->wfull[i]), 1);
      ptx::mbar_init(ptx::smem_u32(&S->wempty[i]), 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(ptx::smem_u32(&S->acc_full[i]), 1);
      ptx::mbar_init(ptx::smem_u32(&S->acc_empty[i]), 16);
    }
    for (int q = 0; q < kBlkMaxChunks; ++q) ptx::mbar_init(ptx::smem_u32(&S->ready[q]), 8);
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(ptx::smem_u32(&S->ext_full[i]), 1);
      ptx::mbar_init(ptx::smem_u32(&S->img_free[i]), 16);
    }
    ptx::fence_mbar_init();
  }
  if (warp == kWaveProducer) ptx::tmem_alloc(ptx::smem_u32(&S->tmem_base), P.tmem_cols);
  // zero the activation slots (their unwritten border rows are the conv padding)
  {
    uint4* z = reinterpret_cast<uint4*>(smem);
    const uint32_t n16 = (uint32_t)P.ni * P.set_bytes / 16;
    for (uint32_t i = threadIdx.x; i < n16; i += kWaveThreads) z[i] = make_uint4(0, 0, 0, 0);
  }
  blk_fill_tabs(P, ptab, threadIdx.x, kWaveThreads);
  blk_pos_fill(P, reinterpret_cast<int*>(ptab + P.pos_off), threadIdx.x, kWaveThreads);
  ptx::fence_proxy_async();  // generic zero stores -> tcgen05 reads of the slots
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = S->tmem_base;
  ptx::griddep_wait();
  ptx::griddep_launch();
  tl_mark(P.tl, 0);

  if (warp == kWaveProducer) {
    // ===== producer: per image the external tensors (after the previous
    // image is drained), then every (layer, chunk) weight stage =====
    int st = 0;
    uint32_t ph = 0;
    int st2[2] = {0, 0};  // per-image half rings (one MMA warp per image)
    uint32_t ph2[2] = {0u, 0u};
    BlkTracer tr;
    for (int g = 0;; ++g) {
      const int b0 = blockIdx.x + G * g * P.ni;
      if (b0 >= P.batch) break;
      const int nv = (P.ni == 2 && b0 + G < P.batch) ? 2 : 1;
      for (int i = 0; i < nv; ++i) {
        const int b = b0 + G * i;
        if (g > 0) {
          if (lane == 0) ptx::mbar_wait_sleep(ptx::smem_u32(&S->img_free[i]), (g - 1) & 1);
          __syncwarp();
        }
        const uint32_t set = slots + (uint32_t)i * P.set_bytes;
        const int nt_ext = (P.ext_in_slot >= 0) + (P.ext_res_slot >= 0);
        const uint32_t bytes = (uint32_t)P.P_img * 16;
        const uint32_t eb = ptx::smem_u32(&S->ext_full[i]);
        if (lane == 0) ptx::mbar_arrive_tx(eb, (uint32_t)nt_ext * P.nq * 4 * bytes);
        __syncwarp();
        // copy k: tensor k / (4 nq), chunk, group, plane -- one copy per lane per round
        const int total = nt_ext * 4 * P.nq;
        for (int k = lane; k < total; k += 32) {
          const int ti = k / (4 * P.nq), r = k - ti * 4 * P.nq, q = r >> 2, gp = r & 3;
          const bool use_in = P.ext_in_slot >= 0 && ti == 0;
          const TensorView& t = use_in ? P.ext_in : P.ext_res;
          const int slot = use_in ? P.ext_in_slot : P.ext_res_slot;
          const int gg = gp & 1, lo = gp >> 1;
          const __half* base = lo ? t.lo() : t.hi();
          const int64_t off = (2 * q + gg) * t.kstride + (int64_t)b * (P.H + 1) * P.wp * 8;
          ptx::bulk_g2s(set + (uint32_t)slot * P.slot_bytes + (uint32_t)(q * 4 + gp) * P.plane, base + off, bytes, eb);
        }
        if (lane == 0) tr(P, 0, 0x100 | g);  // externals issued
      }
      if (lane == 0) {
        // one MMA warp per image (ni = 2): image i's weights go through its
        // own half of the ring, in MMA order per image
        const bool split = kBlkMmaWarps == 2 && P.ni == 2 && P.stages >= 4;
        const int hs = split ? P.stages / 2 : P.stages;
        for (int l = 0; l < P.nl; ++l)
          for (int i = 0; i < nv; ++i)
            for (int q = 0; q < P.nq; ++q) {
              int& rs = split ? st2[i] : st;
              uint32_t& rp = split ? ph2[i] : ph;
              const int sg = (split ? i * hs : 0) + rs;
              ptx::mbar_wait_sleep(ptx::smem_u32(&S->wempty[sg]), rp ^ 1);
              tr(P, 0, 0x200 | (l << 4) | q);
              const uint32_t bar = ptx::smem_u32(&S->wfull[sg]);
              ptx::mbar_arrive_tx(bar, P.b_bytes);
              ptx::bulk_g2s(ring + (uint32_t)sg * P.b_bytes, P.L[l].w + (int64_t)q * 9 * 32 * P.C, P.b_bytes, bar);
              if (++rs == hs) { rs = 0; rp ^= 1; }
            }
      }
      __syncwarp();
    }
  } else if (warp >= kWaveMma && warp < kWaveMma + kBlkMmaWarps && (warp == kWaveMma || (P.ni == 2 && P.stages >= 4))) {
    // ===== MMA issuers: ni = 2 and two warps: warp kWaveMma + i issues image
    // i's layers (its (layer, image) turns of the weight ring; the other
    // image's stages are skipped by count); else warp kWaveMma issues all =====
    // Each image then owns half of the weight ring (stages [i h, (i + 1) h)):
    // a warp only ever waits on barriers whose previous phase it consumed
    // itself, so the one-bit phase parity cannot alias.
    const int mine = warp - kWaveMma;
    const bool split = kBlkMmaWarps == 2 && P.ni == 2 && P.stages >= 4;
    const int hs = split ? P.stages / 2 : P.stages, sbase = split ? mine * hs : 0;
    const int nt = P.C;
    const uint32_t idesc = ptx::idesc_f16(kTileM, nt), idesc2 = ptx::idesc_f16(kTileM, 2 * nt);
    const uint32_t a_lbo = P.plane, b_lbo = 2 * nt * 16;
    uint64_t offs[9];
#pragma unroll
    for (int t = 0; t < 9; ++t) offs[t] = (uint64_t)(P.toff[t] * 16 >> 4);
    const uint64_t bstep = (uint64_t)(64 * nt) >> 4, blo = (uint64_t)(nt * 16) >> 4;
    int st = 0;
    uint32_t ph = 0;
    uint32_t use[2] = {0u, 0u};
    int gl = 0;
    BlkTracer tr;
    for (int g = 0;; ++g) {
      const int b0 = blockIdx.x + G * g * P.ni;
      if (b0 >= P.batch) break;
      const int nv = (P.ni == 2 && b0 + G < P.batch) ? 2 : 1;
      for (int l = 0; l < P.nl; ++l)
        for (int i = 0; i < nv; ++i, ++gl) {
          // ni = 1: buffers by layer parity; ni = 2: by image
          const uint32_t buf = P.ni == 1 ? (uint32_t)(gl & 1) : (uint32_t)i;
          if (split && i != mine) continue;  // the other warp's image
          if (lane == 0 && mine == 0) tr(P, 1, 0x300 | (l << 4) | (i << 3));
          // ni = 2: this also waits for the image's previous layer in its slot
          ptx::mbar_wait(ptx::smem_u32(&S->acc_empty[buf]), (use[buf] & 1) ^ 1);
          if (lane == 0 && mine == 0) tr(P, 1, 0x400 | (l << 4) | (i << 3));
          ptx::tc_fence_after();
          const uint32_t in_base = slots + (uint32_t)i * P.set_bytes + (uint32_t)P.L[l].in_slot * P.slot_bytes;
          for (int q = 0; q < P.nq; ++q) {
            if (l == 0) {
              if (q == 0) ptx::mbar_wait(ptx::smem_u32(&S->ext_full[i]), g & 1);
            } else if (P.ni == 1) {
              ptx::mbar_wait(ptx::smem_u32(&S->ready[q]), (gl - 1) & 1);  // layer l-1's chunk q is in the slot
            }
            if (lane == 0 && mine == 0) tr(P, 1, 0x500 | (l << 4) | (i << 3) | q);  // input chunk ready
            ptx::mbar_wait(ptx::smem_u32(&S->wfull[sbase + st]), ph);
            if (lane == 0 && mine == 0) tr(P, 1, 0x600 | (l << 4) | (i << 3) | q);  // weights ready
            ptx::tc_fence_after();
            const uint32_t cb = in_base + (uint32_t)q * 4 * P.plane;
            const uint64_t b0d = ptx::smem_desc_noswz(ring + (uint32_t)(sbase + st) * P.b_bytes, b_lbo, 128);
            for (int s = 0; s < P.S; ++s) {
              // rows of sub-tile s: positions p_out0 + 128 s + r; tap t reads
              // p - (wp + 1) + toff[t], and p_out0 = wp + 1
              const uint32_t a0 = cb + (uint32_t)(128 * s) * 16;
              const uint64_t ah = ptx::smem_desc_noswz(a0, a_lbo, 128), al = ptx::smem_desc_noswz(a0 + 2 * P.plane, a_lbo, 128);
              const uint32_t dm = tmem + (buf * P.S + s) * P.set_cols;
              ss_stage<9>(true, dm, dm + nt, ah, al, b0d, bstep, blo, idesc2, idesc, q > 0 ? 1u : 0u, 1u, offs);
            }
            ptx::mma_commit_warp(ptx::smem_u32(&S->wempty[sbase + st]));
            if (lane == 0 && mine == 0) tr(P, 1, 0x700 | (l << 4) | (i << 3) | q);  // issued
            if (++st == hs) { st = 0; ph ^= 1; }
          }
          ptx::mma_commit_warp(ptx::smem_u32(&S->acc_full[buf]));
          ++use[buf];
        }
    }
  } else if (warp < 16) {
    // ===== epilogue: every 16-channel chunk k is split between the two
    // warpgroups (warpgroup ew: channels 16k + 8ew .. +8 of every sub-tile),
    // chunks in order, so chunk k of a layer is complete -- and the next
    // layer's MMAs on it can start -- after the shortest time; a layer's
    // output goes to its slot (split hi/lo, the next layer's A operand) or,
    // for the last layer, to global memory =====
    // four warpgroups: pair jp = wg / 2 drains chunks k = jp (mod 2), warpgroup
    // ew = wg % 2 of the pair channels 16 k + 8 ew .. +7 (a 16-channel chunk's
    // ready count stays the 8 warps of its pair)
    const int wg = warp >> 2, ew = wg & 1, jp = wg >> 1, row = threadIdx.x & 127;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const int* postab = reinterpret_cast<const int*>(ptab + P.pos_off);
    uint32_t use[2] = {0u, 0u};
    int gl = 0;
    BlkTracer tr;
    for (int g = 0;; ++g) {
      const int b0 = blockIdx.x + G * g * P.ni;
      if (b0 >= P.batch) break;
      const int nv = (P.ni == 2 && b0 + G < P.batch) ? 2 : 1;
      for (int l = 0; l < P.nl; ++l)
        for (int i = 0; i < nv; ++i, ++gl) {
        const int b = b0 + G * i;
        const uint32_t set = slots + (uint32_t)i * P.set_bytes;
        const BlkLayer& L = P.L[l];
        const EpiParams& e = L.epi;
        const bool last = l == P.nl - 1;
        if (L.res_ext) ptx::mbar_wait_warp(ptx::smem_u32(&S->ext_full[i]), g & 1);
        const uint32_t buf = P.ni == 1 ? (uint32_t)(gl & 1) : (uint32_t)i;
        if (threadIdx.x == 0) tr(P, 2, 0x800 | (l << 4) | (i << 3));
        ptx::mbar_wait_warp(ptx::smem_u32(&S->acc_full[buf]), use[buf] & 1);
        if (threadIdx.x == 0) tr(P, 2, 0x900 | (l << 4) | (i << 3));
        ptx::tc_fence_after();
        EpiTab tab = L.etab;
        tab.ptab = ptab + L.ptab_off;
        const float wsc = ptab[P.wsc_off + l];
        for (int k = jp; k < P.nq; k += 2) {
          const int chb = 16 * k + 8 * ew;
          float psum[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) psum[j] = 0.f;
          for (int s = 0; s < P.S; ++s) {
            const int p = P.p_out0 + 128 * s + row;
            bool inside, valid;
            int y, x;
            blk_pos_get(postab, s, row, inside, valid, y, x);
            float v[8], t[8];
            const uint32_t d = tmem + lane_off + (buf * P.S + s) * P.set_cols;
            ptx::tmem_ld8x2(d + P.C + chb, d + chb, v, t);
            add_n<8>(v, t);
            float sk[8];
            if (L.res_slot >= 0) {
              // this group's hi and lo planes: [g0 hi][g1 hi][g0 lo][g1 lo] per chunk
              const uint32_t rb = set + (uint32_t)L.res_slot * P.slot_bytes + (uint32_t)(k * 4 + ew) * P.plane +
                                  (uint32_t)p * 16;
              uint4 h, q;
              asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                           : "=r"(h.x), "=r"(h.y), "=r"(h.z), "=r"(h.w) : "r"(rb) : "memory");
              asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                           : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w) : "r"(rb + 2 * P.plane) : "memory");
              const uint32_t hw[4] = {h.x, h.y, h.z, h.w}, lw[4] = {q.x, q.y, q.z, q.w};
              const float2 ss = make_float2(L.res_sload, L.res_sload);
#pragma unroll
              for (int i = 0; i < 4; ++i)
                f2_put(sk + 2 * i, __fmul2_rn(__fadd2_rn(unpack_half2(hw[i]), unpack_half2(lw[i])), ss));
            } else {
#pragma unroll
              for (int j = 0; j < 8; ++j) sk[j] = 0.f;
            }
            epi_point8(e, tab, v, wsc, sk, chb);
            if (!last) {
              if (inside) {
                uint32_t hi[4], lo[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  if (valid) split_pair(v[2 * i], v[2 * i + 1], hi[i], lo[i]);
                  else hi[i] = lo[i] = 0u;
                }
                __half2 m = __habs2(*reinterpret_cast<const __half2*>(&hi[0]));
#pragma unroll
                for (int i = 1; i < 4; ++i) m = __hmax2_nan(m, __habs2(*reinterpret_cast<const __half2*>(&hi[i])));
                const float2 mf = __half22float2(m);
                if (!(mf.x < 32768.f && mf.y < 32768.f)) atomicExch(P.flag, 1);
                const uint32_t ob = set + (uint32_t)L.out_slot * P.slot_bytes + (uint32_t)(k * 4 + ew) * P.plane +
                                    (uint32_t)p * 16;
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(ob), "r"(hi[0]), "r"(hi[1]), "r"(hi[2]),
                             "r"(hi[3]) : "memory");
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(ob + 2 * P.plane), "r"(lo[0]), "r"(lo[1]),
                             "r"(lo[2]), "r"(lo[3]) : "memory");
              }
            } else if (e.pool == PCNN_POOL_GLOBAL) {
              if (valid) add_n<8>(psum, v);
            } else if (valid) {
              store8_any(e.out, b, chb, y, x, v);
            }
          }
          if (last && e.pool == PCNN_POOL_GLOBAL) {
            // every row of the tile is image b: reduce the warp's rows, one atomic per channel
#pragma unroll
            for (int j = 0; j < 8; ++j)
#pragma unroll
              for (int o = 16; o; o >>= 1) psum[j] += __shfl_xor_sync(0xffffffffu, psum[j], o);
            if (lane < 8) {
              float mine = psum[0];
#pragma unroll
              for (int j = 1; j < 8; ++j)
                if (lane == j) mine = psum[j];
              if (chb + lane < e.cout) atomicAdd(e.out.base + (int64_t)b * e.npad + chb + lane, mine * __ldg(e.pool_p));
            }
          }
          if (P.ni == 1) {
            // this warp's rows of chunk k are in the slot: hand them to the
            // async proxy (tcgen05.mma reads) and count the warp in (8 warps)
            ptx::fence_proxy_async();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(ptx::smem_u32(&S->ready[k]));
          }
          if (threadIdx.x == 0) tr(P, 2, 0xA00 | (l << 4) | (i << 3) | k);
        }
        // ni = 2: acc_empty also hands the whole output to the image's next layer
        if (P.ni == 2) ptx::fence_proxy_async();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(ptx::smem_u32(&S->acc_empty[buf]));
        ++use[buf];
        if (last && lane == 0) ptx::mbar_arrive(ptx::smem_u32(&S->img_free[i]));
      }
    }
  }
  __syncthreads();
  tl_mark(P.tl, 1);
  if (warp == kWaveProducer) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, P.tmem_cols);
  }
}

// =====================================================================
// Image-resident runs of 16-channel layers (conv_wave_kernel; ResNet-20's
// stage 1: 32 x 32 images, six 3x3 convs).  A 16-channel image needs 72 KB
// per slot, so a CTA keeps ONE image (two slots: the ping-pong output and
// the in-place residual) plus every layer's weights (9 KB each) resident.
// Without a second image to alternate with, the MMA and epilogue overlap
// across sub-tiles instead of across images: job (layer l, sub-tile s)
// needs only sub-tiles s-1..s+1 of layer l-1 (the taps reach one grid row,
// 33 positions, past a 128-row sub-tile), so the MMA warp runs a wavefront
// one layer ahead of the epilogue, through a ring of R TMEM accumulators
// (32 columns each: [main | corr] of the concatenated hi/lo weights).
// ready[s] counts the epilogue warps that stored sub-tile s of the current
// layer (one phase per layer); a job waits for its three neighbours, which
// can never be more than one phase ahead (their next phase needs a later
// job of the in-order MMA warp).
// =====================================================================
constexpr int kWaveMaxSub = 16;  // pairs of epilogue warpgroups take even / odd jobs
// two MMA warps (even / odd jobs): one warp's dependency waits (~200-300
// cycles per mbarrier test) overlap the other warp's MMA issue
#ifndef PCNN_WAVE_MMA_WARPS
#define PCNN_WAVE_MMA_WARPS 2
// Two, not more: ready[layer & 1][s] is reused every second layer and waited
// on by parity.  A warp's previous job (l+1, s-2) waited for layer l at
// s-3 .. s-1, which implies layer l-2 complete at s-5 .. s+1 -- every barrier
// job (l+1, s) tests has finished its previous phase.  With three warps the
// previous job is (l+1, s-3), layer l-2 at s+1 may still be pending, the
// parity aliases and the job reads a stale sub-tile (3 warps: stage-1 run
// 77.9 -> 75.4 us, rn20_fixture golden forward off by 2.5e-4).
#endif
constexpr int kWaveMmaWarps = PCNN_WAVE_MMA_WARPS;  // MMA-issuing warps kWaveMma .. kWaveMma + kWaveMmaWarps - 1
constexpr int kWaveThreads2 = 32 * (kWaveMma + kWaveMmaWarps);

struct WaveSmem {
  uint64_t wfull, ext_full, img_done;
  uint64_t acc_full[kWaveMaxSub], acc_empty[kWaveMaxSub];
  uint64_t ready[2][kWaveMaxSub];  // by layer parity: [global layer & 1][sub-tile]
  uint32_t tmem_base;
};

__global__ void __launch_bounds__(kWaveThreads2, 1) conv_wave_kernel(const __grid_constant__ BlkParams P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  const uint32_t slots = ptx::smem_u32(smem);
  const uint32_t wres = slots + P.set_bytes;
  WaveSmem* S = reinterpret_cast<WaveSmem*>(smem + (size_t)P.set_bytes + (size_t)P.nl * P.b_bytes);
  float* ptab = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(S) + ((sizeof(WaveSmem) + 15) & ~size_t(15)));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = (int)gridDim.x, R = P.R, NS = P.S, NL = P.nl;
  if (threadIdx.x == 0) {
    ptx::mbar_init(ptx::smem_u32(&S->wfull), 1);
    ptx::mbar_init(ptx::smem_u32(&S->ext_full), 1);
    ptx::mbar_init(ptx::smem_u32(&S->img_done), 16);
    for (int i = 0; i < R; ++i) {
      ptx::mbar_init(ptx::smem_u32(&S->acc_full[i]), 1);
      ptx::mbar_init(ptx::smem_u32(&S->acc_empty[i]), 8);
    }
    for (int i = 0; i < NS; ++i) {
      ptx::mbar_init(ptx::smem_u32(&S->ready[0][i]), 8);
      ptx::mbar_init(ptx::smem_u32(&S->ready[1][i]), 8);
    }
    ptx::fence_mbar_init();
  }
  if (warp == kWaveProducer) ptx::tmem_alloc(ptx::smem_u32(&S->tmem_base), P.tmem_cols);
  {
    uint4* z = reinterpret_cast<uint4*>(smem);
    for (uint32_t i = threadIdx.x; i < P.set_bytes / 16; i += kWaveThreads2) z[i] = make_uint4(0, 0, 0, 0);
  }
  blk_fill_tabs(P, ptab, threadIdx.x, kWaveThreads2);
  blk_pos_fill(P, reinterpret_cast<int*>(ptab + P.pos_off), threadIdx.x, kWaveThreads2);
  ptx::fence_proxy_async();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = S->tmem_base;
  // weights are parameters: their copy overlaps the previous kernel's tail
  if (warp == kWaveProducer && lane == 0) {
    const uint32_t wb = ptx::smem_u32(&S->wfull);
    ptx::mbar_arrive_tx(wb, (uint32_t)NL * P.b_bytes);
    for (int l = 0; l < NL; ++l) ptx::bulk_g2s(wres + (uint32_t)l * P.b_bytes, P.L[l].w, P.b_bytes, wb);
  }
  ptx::griddep_wait();
  ptx::griddep_launch();
  tl_mark(P.tl, 0);

  if (warp == kWaveProducer) {
    // ===== producer: each image's external input (+ residual) after the
    // previous image is fully drained =====
    for (int g = 0;; ++g) {
      const int b = blockIdx.x + G * g;
      if (b >= P.batch) break;
      if (g > 0) {
        if (lane == 0) ptx::mbar_wait_sleep(ptx::smem_u32(&S->img_done), (g - 1) & 1);
        __syncwarp();
      }
      const int nt_ext = (P.ext_in_slot >= 0) + (P.ext_res_slot >= 0);
      const uint32_t bytes = (uint32_t)P.P_img * 16;
      const uint32_t eb = ptx::smem_u32(&S->ext_full);
      // a one-group input (the stem's) leaves the slot's second group as the
      // previous image left it: finite values its zero weight rows cancel
      const int planes = (P.ext_in_slot >= 0 ? 2 * P.ext_in_groups : 0) + (P.ext_res_slot >= 0 ? 4 : 0);
      if (lane == 0) ptx::mbar_arrive_tx(eb, (uint32_t)planes * bytes);
      __syncwarp();
      if (lane < 4 * nt_ext) {
        const int ti = lane >> 2, gp = lane & 3;
        const bool use_in = P.ext_in_slot >= 0 && ti == 0;
        const TensorView& t = use_in ? P.ext_in : P.ext_res;
        const int slot = use_in ? P.ext_in_slot : P.ext_res_slot;
        const int gg = gp & 1, lo = gp >> 1;
        const __half* base = lo ? t.lo() : t.hi();
        const int64_t off = gg * t.kstride + (int64_t)b * (P.H + 1) * P.wp * 8;
        if (!use_in || gg < P.ext_in_groups)
          ptx::bulk_g2s(slots + (uint32_t)slot * P.slot_bytes + (uint32_t)gp * P.plane, base + off, bytes, eb);
      }
      __syncwarp();
    }
  } else if (warp >= kWaveMma && warp < kWaveMma + kWaveMmaWarps) {
    // ===== MMA issuers: warp kWaveMma + i the jobs j = i (mod kWaveMmaWarps)
    // (jobs (image, layer, sub-tile) in order).  A job waits for all three
    // of its input sub-tiles (the other warp may have issued the neighbours)
    // on ready[layer & 1]: a neighbour's barrier cannot run a phase ahead,
    // since layer l+1 at sub-tiles s-1 .. s+1 needs this job's output.
    const uint32_t mine = (uint32_t)(warp - kWaveMma);
    const int nt = 16;
    const uint32_t idesc = ptx::idesc_f16(kTileM, nt), idesc2 = ptx::idesc_f16(kTileM, 2 * nt);
    const uint32_t a_lbo = P.plane, b_lbo = 2 * nt * 16;
    uint64_t offs[9];
#pragma unroll
    for (int t = 0; t < 9; ++t) offs[t] = (uint64_t)P.toff[t];
    const uint64_t bstep = (uint64_t)(64 * nt) >> 4, blo = (uint64_t)(nt * 16) >> 4;
    ptx::mbar_wait(ptx::smem_u32(&S->wfull), 0);
    uint32_t j = 0;  // job counter (ring slot j % R, use j / R)
    for (int g = 0;; ++g) {
      const int b = blockIdx.x + G * g;
      if (b >= P.batch) break;
      ptx::mbar_wait(ptx::smem_u32(&S->ext_full), g & 1);
      for (int l = 0; l < NL; ++l) {
        const uint32_t in_base = slots + (uint32_t)P.L[l].in_slot * P.slot_bytes;
        const uint64_t b0d = ptx::smem_desc_noswz(wres + (uint32_t)l * P.b_bytes, b_lbo, 128);
        const int gl = g * NL + l - 1;  // global index of the input's layer
        const uint32_t rb = ptx::smem_u32(&S->ready[gl & 1][0]), rph = (uint32_t)(gl >> 1) & 1u;
        for (int s = 0; s < NS; ++s, ++j) {
          if (j % (uint32_t)kWaveMmaWarps != mine) continue;
          if (l > 0) {
            if (s > 0) ptx::mbar_wait(rb + 8u * (uint32_t)(s - 1), rph);
            ptx::mbar_wait(rb + 8u * (uint32_t)s, rph);
            if (s + 1 < NS) ptx::mbar_wait(rb + 8u * (uint32_t)(s + 1), rph);
          }
          const uint32_t r = j % (uint32_t)R;
          ptx::mbar_wait(ptx::smem_u32(&S->acc_empty[r]), ((j / (uint32_t)R) & 1u) ^ 1u);
          ptx::tc_fence_after();
          const uint32_t a0 = in_base + (uint32_t)(128 * s) * 16;
          const uint64_t ah = ptx::smem_desc_noswz(a0, a_lbo, 128), al = ptx::smem_desc_noswz(a0 + 2 * P.plane, a_lbo, 128);
          const uint32_t dm = tmem + r * 32u;
          ss_stage<9>(true, dm, dm + nt, ah, al, b0d, bstep, blo, idesc2, idesc, 0u, 1u, offs);
          ptx::mma_commit_warp(ptx::smem_u32(&S->acc_full[r]));
        }
      }
    }
  } else if (warp < 16) {
    // ===== epilogue: warpgroup pair jp = wg / 2 drains the jobs j = jp
    // (mod 2); warpgroup ew = wg % 2 of the pair takes channels 8 ew .. +7 =====
    const int wg = warp >> 2, ew = wg & 1, jp = wg >> 1, row = threadIdx.x & 127, chb = 8 * ew;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const int* postab = reinterpret_cast<const int*>(ptab + P.pos_off);
    const uint32_t rmask = (uint32_t)R - 1u, lg_r = (uint32_t)(__ffs(R) - 1);  // R: a power of two
    uint32_t j = 0;
    for (int g = 0;; ++g) {
      const int b = blockIdx.x + G * g;
      if (b >= P.batch) break;
      for (int l = 0; l < NL; ++l) {
        const BlkLayer& L = P.L[l];
        const EpiParams& e = L.epi;
        const bool last = l == NL - 1;
        if (L.res_ext) ptx::mbar_wait_warp(ptx::smem_u32(&S->ext_full), g & 1);
        EpiTab tab = L.etab;
        tab.ptab = ptab + L.ptab_off;
        const float wsc = ptab[P.wsc_off + l];
        float psum[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) psum[q] = 0.f;
        // jobs j0 + s of this layer; this pair's are those with (j0 + s) % 2 == jp
        const uint32_t j0 = j;
        j += (uint32_t)NS;
        for (int s = (int)(((uint32_t)jp ^ j0) & 1u); s < NS; s += 2) {
          const uint32_t jj = j0 + (uint32_t)s;
          const uint32_t r = jj & rmask;
          const int p = P.p_out0 + 128 * s + row;
          bool inside, valid;
          int y, x;
          blk_pos_get(postab, s, row, inside, valid, y, x);
          float sk[8];
          if (L.res_slot >= 0) {
            const uint32_t rb = slots + (uint32_t)L.res_slot * P.slot_bytes + (uint32_t)ew * P.plane + (uint32_t)p * 16;
            uint4 h, q;
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(h.x), "=r"(h.y), "=r"(h.z), "=r"(h.w) : "r"(rb) : "memory");
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w) : "r"(rb + 2 * P.plane) : "memory");
            const uint32_t hw[4] = {h.x, h.y, h.z, h.w}, lw[4] = {q.x, q.y, q.z, q.w};
            const float2 ss = make_float2(L.res_sload, L.res_sload);
#pragma unroll
            for (int i = 0; i < 4; ++i)
              f2_put(sk + 2 * i, __fmul2_rn(__fadd2_rn(unpack_half2(hw[i]), unpack_half2(lw[i])), ss));
          } else {
#pragma unroll
            for (int q = 0; q < 8; ++q) sk[q] = 0.f;
          }
          ptx::mbar_wait_warp(ptx::smem_u32(&S->acc_full[r]), (jj >> lg_r) & 1u);
          ptx::tc_fence_after();
          float v[8], t[8];
          const uint32_t d = tmem + lane_off + r * 32u;
          ptx::tmem_ld8x2(d + 16 + chb, d + chb, v, t);
          // the accumulator is in registers: hand the ring slot back
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(ptx::smem_u32(&S->acc_empty[r]));
          add_n<8>(v, t);
          epi_point8(e, tab, v, wsc, sk, chb);
          if (!last) {
            if (inside) {
              uint32_t hi[4], lo[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                if (valid) split_pair(v[2 * i], v[2 * i + 1], hi[i], lo[i]);
                else hi[i] = lo[i] = 0u;
              }
              __half2 m = __habs2(*reinterpret_cast<const __half2*>(&hi[0]));
#pragma unroll
              for (int i = 1; i < 4; ++i) m = __hmax2_nan(m, __habs2(*reinterpret_cast<const __half2*>(&hi[i])));
              const float2 mf = __half22float2(m);
              if (!(mf.x < 32768.f && mf.y < 32768.f)) atomicExch(P.flag, 1);
              const uint32_t ob = slots + (uint32_t)L.out_slot * P.slot_bytes + (uint32_t)ew * P.plane + (uint32_t)p * 16;
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(ob), "r"(hi[0]), "r"(hi[1]), "r"(hi[2]),
                           "r"(hi[3]) : "memory");
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(ob + 2 * P.plane), "r"(lo[0]), "r"(lo[1]),
                           "r"(lo[2]), "r"(lo[3]) : "memory");
            }
          } else if (e.pool == PCNN_POOL_GLOBAL) {
            if (valid) add_n<8>(psum, v);
          } else if (valid) {
            store8_any(e.out, b, chb, y, x, v);
          }
          // this warp's rows of sub-tile s are stored: to the async proxy
          // (the next layer's tcgen05 reads), then count the warp in
          ptx::fence_proxy_async();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(ptx::smem_u32(&S->ready[(g * NL + l) & 1][s]));
        }
        if (last && e.pool == PCNN_POOL_GLOBAL) {
#pragma unroll
          for (int q = 0; q < 8; ++q)
#pragma unroll
            for (int o = 16; o; o >>= 1) psum[q] += __shfl_xor_sync(0xffffffffu, psum[q], o);
          if (lane < 8) {
            float mine = psum[0];
#pragma unroll
            for (int q = 1; q < 8; ++q)
              if (lane == q) mine = psum[q];
            if (chb + lane < e.cout) atomicAdd(e.out.base + (int64_t)b * e.npad + chb + lane, mine * __ldg(e.pool_p));
          }
        }
      }
      // the image is drained (its last layer's residual reads included)
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(ptx::smem_u32(&S->img_done));
    }
  }
  __syncthreads();
  tl_mark(P.tl, 1);
  if (warp == kWaveProducer) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, P.tmem_cols);
  }
}

}  // namespace

struct BlkRun {
  BlkParams P;
  size_t smem;
};

BlkRun* blk_create(const ConvArgs* layers, int n, const int* in_slot, const int* res_slot, const int* out_slot,
                   const int* src_kind, int nslots, int ext_in_slot, int ext_res_slot, const TensorView& ext_in,
                   const TensorView& ext_res, int* flag, int batch, int max_images) {
  if (n < 2 || n > kBlkMaxLayers) return nullptr;
  BlkRun* r = new BlkRun();
  BlkParams& P = r->P;
  std::memset(&P, 0, sizeof(P));
  const ConvArgs& a0 = layers[0];
  P.nl = n;
  P.C = a0.npad;
  P.nq = P.C / 16;
  P.H = a0.in.h;
  P.W = a0.in.w;
  P.wp = a0.in.wp;
  P.wave = P.C == 16;  // 16 channels: one image per CTA, sub-tile wavefront (conv_wave_kernel)
  if ((P.C % 32 && !P.wave) || P.nq > kBlkMaxChunks || P.wp != P.W + 1) { delete r; return nullptr; }
  P.nout = P.H * P.wp;
  P.p_out0 = 1 + P.wp;
  P.S = (P.nout + kTileM - 1) / kTileM;
  P.P_img = (P.H + 2) * P.wp;
  // planes hold the image (P_img positions, + 1: the bottom-right border
  // corner the last output's taps read); A reads of the last sub-tile run
  // up to (128 S + 2 wp + 2 - P_img - 1) positions past the last plane, into
  // the weight ring (checked below)
  P.plane = (uint32_t)(P.P_img + 1) * 16;
  P.slot_bytes = (uint32_t)P.nq * 4 * P.plane;
  P.set_bytes = (uint32_t)nslots * P.slot_bytes;
  const int over = kTileM * P.S + 2 * (P.wp + 1) - P.P_img - 1;
  const uint32_t overrun = over > 0 ? (uint32_t)over * 16 : 0u;
  P.nslots = nslots;
  P.ext_in_slot = ext_in_slot;
  P.ext_res_slot = ext_res_slot;
  P.ext_in = ext_in;
  P.ext_res = ext_res;
  P.ext_in_groups = a0.in.cpad() <= 8 ? 1 : 2;
  P.batch = batch;
  P.b_bytes = 9u * 64u * (uint32_t)P.C;
  P.set_cols = 2u * (uint32_t)P.C;
  const uint32_t need = P.wave ? 512u : 2u * (uint32_t)P.S * P.set_cols;
  if (need > 512 || (P.wave && P.S > kWaveMaxSub)) { delete r; return nullptr; }
  P.R = P.wave ? 512 / (int)P.set_cols : 0;
  if (P.wave && (P.R & (P.R - 1))) { delete r; return nullptr; }  // the epilogue indexes the ring by masks
  P.tmem_cols = need <= 32 ? 32 : need <= 64 ? 64 : need <= 128 ? 128 : need <= 256 ? 256 : 512;
  for (int t = 0; t < 9; ++t) P.toff[t] = (t / 3) * P.wp + t % 3;
  P.flag = flag;
  P.dbg = a0.opt.dbg;
  int pt = 0;
  for (int l = 0; l < n; ++l) {
    const ConvArgs& a = layers[l];
    const bool narrow_head = l == 0 && P.wave && a.in.cpad() <= 8;  // one stored group, zero weight rows beyond it
    if (a.kh != 3 || a.kw != 3 || a.stride != 1 || a.pad != 1 || a.npad != P.C || (a.in.cpad() != P.C && !narrow_head) ||
        a.in.h != P.H || a.in.w != P.W || !a.tcwss || !a.tc16_scale || a.proj || a.epi.residual > 3 ||
        (a.epi.pool != PCNN_POOL_NONE && !(a.epi.pool == PCNN_POOL_GLOBAL && l == n - 1))) {
      delete r;
      return nullptr;
    }
    BlkLayer& L = P.L[l];
    L.epi = a.epi;
    L.etab = epi_tab_layout(a.epi);
    L.w = reinterpret_cast<const __half*>(a.tcwss);
    L.wscale = a.tc16_scale + 1;
    L.in_slot = in_slot[l];
    L.res_slot = res_slot[l];
    L.out_slot = out_slot[l];
    // src_kind: bit 0 input is the external input; bits 2-3 residual 1 = external input, 2 = external residual
    L.in_sload = (src_kind[l] & 1) ? ext_in.sload : 1.f;
    const int rk = (src_kind[l] >> 2) & 3;
    L.res_sload = rk == 1 ? ext_in.sload : rk == 2 ? ext_res.sload : 1.f;
    L.res_ext = rk != 0;
    L.ptab_off = pt;
    pt += (L.etab.rows * P.C + 3) & ~3;
  }
  P.pos_off = pt;
  pt += P.S * 128;
  P.wsc_off = pt;
  pt += (kBlkMaxLayers + 3) & ~3;
  P.ptab_floats = pt;
  const size_t budget = 225 * 1024 - 128;
  if (P.wave) {
    // one image, every layer's weights resident; A over-reads of the last
    // sub-tile land in the weights (discarded rows)
    P.ni = 1;
    const size_t fixed = (size_t)P.set_bytes + (size_t)n * P.b_bytes + ((sizeof(WaveSmem) + 15) & ~size_t(15)) +
                         (size_t)pt * 4;
    if (fixed > budget || overrun > (size_t)n * P.b_bytes) { delete r; return nullptr; }
    P.stages = 0;
    r->smem = 128 + fixed;
    return r;
  }
  const size_t aux = ((sizeof(BlkSmem) + 15) & ~size_t(15)) + (size_t)pt * 4;
  P.ni = max_images >= 2 ? 2 : 1;
  if (P.ni == 2 && 2 * (size_t)P.set_bytes + aux + 2 * (size_t)P.b_bytes > budget) P.ni = 1;
  const size_t fixed = (size_t)P.ni * P.set_bytes + aux;
  if (fixed + 2 * (size_t)P.b_bytes > budget || overrun > 2 * P.b_bytes) { delete r; return nullptr; }
  P.stages = (int)((budget - fixed) / P.b_bytes);
  if (P.stages > kBlkStages) P.stages = kBlkStages;
  r->smem = 128 + fixed + (size_t)P.stages * P.b_bytes;
  return r;
}

void blk_launch(const BlkRun* r, cudaStream_t s, unsigned long long* tl, int pdl) {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  BlkParams P = r->P;
  P.tl = tl;
  const int grid = P.batch < nsm ? P.batch : nsm;
  if (P.wave) {
    cudaFuncSetAttribute(conv_wave_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)r->smem);
    launch_pdl(conv_wave_kernel, grid, kWaveThreads2, r->smem, s, pdl, P);
    return;
  }
  cudaFuncSetAttribute(conv_blk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)r->smem);
  launch_pdl(conv_blk_kernel, grid, kWaveThreads, r->smem, s, pdl, P);
}

void blk_destroy(BlkRun* r) { delete r; }

// debugging aid (not part of pcnn.h): drain the CTA-0 event trace
extern "C" int pcnn_ss_trace(unsigned long long* host, int n) {
  int m = n < kTraceLen ? n : kTraceLen;
  cudaMemcpyFromSymbol(host, g_ss_trace, sizeof(unsigned long long) * m);
  static unsigned long long zeros[kTraceLen];
  cudaMemcpyToSymbol(g_ss_trace, zeros, sizeof(zeros));
  return m;
}

// debugging aid (not part of pcnn.h): per-CTA stamps [slot][cta][4] in ns;
// reset = 1 zeroes them, reset = 2 also restarts the host slot counter
extern "C" int pcnn_ss_cta_times(unsigned long long* host, int reset) {
  static unsigned long long buf[kTimeSlots][kTimeCtas][4];
  if (host) cudaMemcpyFromSymbol(host, g_cta_time, sizeof(buf));
  if (reset) {
    static unsigned long long zeros[kTimeSlots][kTimeCtas][4];
    cudaMemcpyToSymbol(g_cta_time, zeros, sizeof(zeros));
  }
  if (reset == 2) g_time_next = 0;
  return g_time_next;
}

bool conv_ss_shape_ok(const ConvArgs& a) {
  if (!a.f16 || !a.tcwss || !a.tc16_scale) return false;
  if ((a.stride != 1 && a.stride != 2) || a.kh != a.kw ||
      !((a.kh == 3 && a.pad == 1) || (a.kh == 1 && a.pad == 0) || (a.kh == 4 && a.pad == 1 && a.stride == 1)))
    return false;
  if (a.epi.pool != PCNN_POOL_NONE && a.epi.pool != PCNN_POOL_GLOBAL) return false;
  const int cpad = a.in.cpad();
  if (!(cpad == 4 || cpad == 8 || cpad % 16 == 0) || a.npad < 16 || a.npad % 16) return false;
  // and the tiles fit shared memory, given the input in the layout it would get
  ConvArgs b = a;
  TensorView& in = b.in;
  in.split = a.stride == 2 ? 2 : 1;
  in.hp = a.stride == 2 ? (in.h + 3) / 2 : in.h + 1;
  in.wp = a.stride == 2 ? (in.w + 3) / 2 : in.w + 1;
  in.pstride = a.stride == 2 ? (int64_t)b.batch * in.hp * in.wp * 8 : (2 + ((int64_t)b.batch * in.hp + 1) * in.wp) * 8;
  in.kstride = a.stride == 2 ? 4 * in.pstride : in.pstride;
  SsParams P;
  return make_ss_params(b, P);
}

bool conv_ss_flag_geometry(const ConvArgs& a, FlagDep& d) {
  SsParams P;
  if (!make_ss_params(a, P) || P.band) return false;
  d.tm = kTileM * P.mt;
  d.m_tiles = P.m_tiles;
  d.gtotal = P.gtotal;
  d.per_tile = P.n_tiles;  // one signal per (m-tile, n-tile)
  d.all = P.m_tiles * P.n_tiles;
  return true;
}

bool conv_ss_proj_ok(const ConvArgs& a, const ConvArgs& proj) {
  if (!a.opt.proj_fuse) return false;
  ConvArgs b = a;
  b.proj = &proj;
  SsParams P;
  return make_ss_params(b, P) && P.proj;
}

bool conv_ss_streamk_wanted(const ConvArgs& a, int nsm, size_t* slot_floats) {
  if (!a.opt.streamk) return false;
  SsParams P;
  if (!make_ss_params(a, P) || P.nq < 2 || P.band) return false;
  const int tiles = P.m_tiles * P.n_tiles;
  // Measured on B200 (streamk option A/B): splitting pays only when whole
  // tiles leave most SMs idle (VGG 2x2 layers: 36 tiles for 148 SMs);
  // for 1.1-1.5 rounds of tiles (RN20 stage 3, RN18 stages 3-4) the partial
  // round trips and shorter pipelines cost more than the balance gains
  // (RN20 0.362 vs 0.322 ms).  Option streamk_fill sets the threshold.
  const double fill = a.opt.streamk_fill;
  if (tiles > fill * nsm) return false;
  const int items = P.mt * (P.nt / 16) * (P.proj ? 2 : 1);
  *slot_floats = (size_t)items * 128 * 16;
  return true;
}

bool conv_ss_supported(const ConvArgs& a) {
  SsParams P;
  return make_ss_params(a, P);
}

typedef CUresult (*SsEncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// pair mode: the weight image (tc_layout.cuh pack_tcss_weights_device, 128-row
// tiles: [tile, chunk][tap][g, hi/lo][128 rows][8 fp16]) as a 4-D tensor of
// 32-bit words; a box is one CTA's bn rows of every (tap, g, hi/lo) of a chunk
static bool encode_weight_map(SsParams& P) {
  static SsEncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) != cudaSuccess || !ptr)
      return false;
    fn = reinterpret_cast<SsEncodeTiledFn>(ptr);
  }
  // 4-byte elements, a 128-row block row = 128 x 16 B: the box's inner
  // extent is one CTA's bn rows (1 KB contiguous), not one 16-byte row
  const int INT = P.b_img_nt;
  const cuuint64_t dims[4] = {(cuuint64_t)INT * 4, 4, (cuuint64_t)P.taps, (cuuint64_t)(P.a.npad / INT) * (cuuint64_t)P.nq};
  const cuuint64_t strides[3] = {(cuuint64_t)INT * 16, (cuuint64_t)4 * INT * 16, (cuuint64_t)P.taps * 4 * INT * 16};
  const cuuint32_t box[4] = {(cuuint32_t)P.bn * 4, 4, (cuuint32_t)P.taps, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(reinterpret_cast<CUtensorMap*>(&P.wmap), CU_TENSOR_MAP_DATA_TYPE_UINT32, 4,
                  const_cast<__half*>(P.w), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

void launch_conv_ss(const ConvArgs& a, cudaStream_t s) {
  SsParams P;
  if (!make_ss_params(a, P)) return;
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  const size_t smem = 128 + (size_t)P.stages * P.stage_bytes + P.res_bytes + ss_aux_bytes(P);
  const int tiles = P.m_tiles * P.n_tiles;
  int grid = tiles < nsm ? tiles : nsm;
  if (P.band) {
    // bands of at least one tile's worth of pooled rows, n-tiles on separate CTAs
    const int per_tile = P.brows / P.ps > 0 ? P.brows / P.ps : 1;
    int nb = (P.prows + per_tile - 1) / per_tile;
    const int cap = nsm / P.n_tiles > 0 ? nsm / P.n_tiles : 1;
    P.nbands = nb < cap ? nb : cap;
    grid = P.nbands * P.n_tiles;
  }
  if (a.sk_flags) {
    // stream-K: every SM, at least two chunks each (plan_streamk sized the slots for nsm CTAs)
    const int64_t units = (int64_t)tiles * P.nq;
    grid = units / 2 < nsm ? (int)(units / 2) : nsm;
    if (grid < 1) grid = 1;
  }
  const bool sk = a.sk_flags != nullptr;
  void (*k)(SsParams);
  if (P.pair) {
    if (!encode_weight_map(P)) {
      // no tensor map: the one-CTA kernel
      SsParams Q;
      ConvArgs b = a;
      b.opt.ss_pair = 0;
      if (!make_ss_params(b, Q)) return;
      launch_conv_ss(b, s);
      return;
    }
    const int pairs = P.m_tiles / 2 * P.n_tiles;
    const int ncl = pairs < nsm / 2 ? pairs : nsm / 2;
    k = conv_ss_kernel<9, false, kPoolNone, 1, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (P.dbg & 64) P.time_slot = g_time_next++ % kTimeSlots;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * ncl);
    cfg.blockDim = dim3(ss_threads<1>());
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = a.opt.pdl ? 2 : 1;
    cudaLaunchKernelEx(&cfg, k, P);
    return;
  }
  if (P.band) {
    k = P.taps == 16 ? conv_ss_kernel<16, false, kPoolBand> : conv_ss_kernel<9, false, kPoolBand>;
  } else if (P.epi_pairs == 2) {
    k = P.taps == 16 ? conv_ss_kernel<16, false, kPoolNone, 2>
        : P.taps == 9 ? conv_ss_kernel<9, false, kPoolNone, 2> : conv_ss_kernel<1, false, kPoolNone, 2>;
  } else {
    k = P.taps == 16 ? (sk ? conv_ss_kernel<16, true, kPoolNone> : conv_ss_kernel<16, false, kPoolNone>)
        : P.taps == 9 ? (sk ? conv_ss_kernel<9, true, kPoolNone> : conv_ss_kernel<9, false, kPoolNone>)
                      : (sk ? conv_ss_kernel<1, true, kPoolNone> : conv_ss_kernel<1, false, kPoolNone>);
  }
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (P.dbg & 64) P.time_slot = g_time_next++ % kTimeSlots;
  launch_pdl(k, grid, P.epi_pairs == 2 ? ss_threads<2>() : ss_threads<1>(), smem, s, a.opt.pdl, P);
}

}  // namespace pcnn
