/*
 * pcnn.h -- C ABI of libpcnn.so, the B200 (sm_100a) engine for the
 * redistributed polynomial-CNN hot path of arXiv 2509.22857.
 *
 * The reference (levnet, /root/reference/pkg/src/levnet) is pure Python and
 * has no native boundary; its "operator API" is the Python module API.  Each
 * entry point below replaces the numeric core of one reference function:
 *
 *   pcnn_plan_create / pcnn_forward / pcnn_forward_host
 *       <- levnet.graph.reference_eval            graph.py:413-426
 *          (+ node kernels conv2d / eval_polyact / eval_polyskip / pools /
 *           linear, graph.py:361-410), batched over images
 *   pcnn_redistribute
 *       <- levnet.transforms.redistribute_forward  transforms.py:423-449
 *          levnet.transforms.redistribute_backward transforms.py:452-485
 *          levnet.transforms.redistribute_pass     transforms.py:575-705
 *          (update-term computation transforms.py:287-318, receiver
 *           rewrites transforms.py:374-420, channel scales :492-572)
 *   pcnn_pack
 *       <- the float64 -> compute-layout step the reference does implicitly
 *          by evaluating straight from its float64 node fields
 *
 * Host-side graph walking (receiver discovery transforms.py:321-371, the
 * symbolic part of the scale solver, lowering) stays in Python
 * (paper_2509_22857_b200.transforms / .lowering) and reaches this library
 * only as the flat descriptor tables declared here.
 *
 * Conventions: plain pointers and sizes only.  All buffers are caller-owned
 * device memory unless a name says "host"; the library never allocates
 * inside pcnn_forward.  Every call is stream-ordered on the cudaStream_t
 * passed as a void*.  Functions return PCNN_OK (0) or a negative status;
 * pcnn_last_error() returns the thread-local message of the last failure.
 * One plan may be used by one stream at a time.
 */
#ifndef PCNN_H
#define PCNN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PCNN_ABI_VERSION 3

enum pcnn_status {
  PCNN_OK = 0,
  PCNN_ERR_INVALID = -1,      /* bad descriptor or argument            */
  PCNN_ERR_CUDA = -2,         /* a CUDA runtime/driver call failed      */
  PCNN_ERR_UNSUPPORTED = -3,  /* shape/feature not implemented          */
  PCNN_ERR_TRANSFORM = -4,    /* redistribution refused (see status)    */
  PCNN_ERR_NO_DEVICE = -5     /* no sm_100 device                       */
};

/* ---- activation tensors --------------------------------------------------
 * Tensors are stored channel-blocked: [B][nblk][H][W][cb] float32, cb in
 * {4, 8, 16, 32}, channels >= c are zero.  A vector tensor (shape (c,)) is
 * the 1x1 case, i.e. [B][nblk*cb].  offset is in floats from the workspace
 * base, for the plan's batch size. */
typedef struct pcnn_tensor_desc {
  int64_t c, h, w, cb, nblk, is_vector, offset;
  int64_t scale_log2;  /* split storage keeps x * 2^scale_log2 (large activations
                          are scaled into fp16 range; readers undo it)   */
} pcnn_tensor_desc;

/* ---- fused units ---------------------------------------------------------*/
enum pcnn_unit_kind {
  PCNN_UNIT_INGEST = 1,   /* user NCHW float32 -> blocked tensor `out`      */
  PCNN_UNIT_CONV = 2,     /* conv + fused epilogue                          */
  PCNN_UNIT_LINEAR = 3,   /* dense + fused epilogue; in_mode picks the view */
  PCNN_UNIT_POLY = 4,     /* standalone elementwise kernels ...             */
  PCNN_UNIT_ADD = 5,
  PCNN_UNIT_POLYSKIP = 6,
  PCNN_UNIT_AFFINE = 7,   /* batchnorm b1 x + b0                            */
  PCNN_UNIT_LOCALPOOL = 8,
  PCNN_UNIT_BIPOOL = 9,   /* one pairwise bivariate pool along pool_order   */
  PCNN_UNIT_GLOBALPOOL = 10,
  PCNN_UNIT_FLATTEN = 11,
  PCNN_UNIT_COPYOUT = 12  /* vector tensor -> user logits [B][c]            */
};

enum pcnn_pool_kind {
  PCNN_POOL_NONE = 0,
  PCNN_POOL_SUM2 = 1,     /* 2x2/s2 window sum * divisor                    */
  PCNN_POOL_BI2 = 2,      /* two pairwise bivariate pools over a 2x2 window */
  PCNN_POOL_GLOBAL = 3,   /* sum over H*W * divisor -> vector tensor        */
  PCNN_POOL_LOCAL = 4     /* k x k / stride s / pad p window sum * divisor
                             (k, s, p in pool_geom), e.g. ResNet-18's 3x3/s2
                             stem pool; the halo-tile kernel computes it in
                             its epilogue over row bands, other conv kernels
                             write the unpooled output to plan scratch and
                             pool in a second launch                        */
};

/* Offsets are in floats into the packed float32 parameter buffer; -1 = none.
 * Per-channel vectors are padded to the output tensor's nblk*cb.           */
typedef struct pcnn_unit_desc {
  int64_t kind;
  int64_t in, in2, out;          /* tensor ids (in2: residual/skip input)    */
  int64_t cin, cout;             /* logical channels (linear: n_in, n_out)   */
  int64_t kh, kw, stride, pad;   /* conv / local pool window                 */
  int64_t w_off, b_off;          /* conv [Npad][Kp] (Kp = nblk_in*kh*kw*cb_in),
                                    linear [n_out][n_in]; bias [Npad]        */
  int64_t affine_off;            /* scale [Npad] then shift [Npad]           */
  int64_t residual;              /* 0 none, 1 add skip, 2 S(conv, skip),
                                    3 S(skip, conv)                          */
  int64_t res_off;               /* S coeffs [6][Npad]: x2 y2 xy x y c       */
  int64_t poly_deg, poly_off;    /* Horner coeffs c_0..c_d, each [Npad]      */
  int64_t pool;                  /* pcnn_pool_kind                           */
  int64_t pool_off;              /* SUM2/GLOBAL/LOCALPOOL: divisor (1 float);
                                    BI2/BIPOOL: [(d+1)^2][Npad] first stage,
                                    then second stage                        */
  int64_t pool_deg;              /* bivariate degree d                       */
  int64_t pool_order;            /* BI2: 0 = w then h, 1 = h then w;
                                    BIPOOL: 0 = along w, 1 = along h         */
  int64_t in_mode;               /* linear: 0 vector, 1 flatten, 2 global sum*/
  int64_t in_div_off;            /* linear global sum divisor (1 float)      */
  int64_t impl;                  /* conv: 0 auto (tcgen05 fp16x2 if possible),
                                    1 SIMT fp32, 2 tcgen05 3xTF32,
                                    3 tcgen05 fp16x2 (3 fp16 products),
                                    4 auto without fp16x2 (all tensors fp32),
                                    5 tcgen05 fp16x2 with A from shared memory
                                      (halo tiles of split activations)      */
  int64_t tc_off;                /* conv tcgen05 weight image (hi|lo tf32)   */
  int64_t npad;                  /* padded output channels (vector stride)   */
  int64_t tc16_off;              /* conv fp16x2 weight image (hi|lo fp16)    */
  int64_t tc16_scale_off;        /* its {max|w|, 2^-e} pair (2 floats)       */
  int64_t tcss_off;              /* conv fp16x2 image of the shared-memory
                                    (halo tile) kernel, or -1                */
  int64_t flags;                 /* PCNN_FLAG_*                              */
  int64_t pool_geom;             /* POOL_LOCAL: k | stride << 8 | pad << 16  */
} pcnn_unit_desc;

/* ---- parameter packing (float64 master -> float32 compute images) -------*/
enum pcnn_pack_kind {
  PCNN_PACK_CAST = 1,        /* dst[i] = (float) src[i], i < n                */
  PCNN_PACK_BN_AFFINE = 2,   /* src = gamma,beta,mean,std (each n); dst =
                                scale=gamma/std [n], shift=beta-scale*mean [n]*/
  PCNN_PACK_TC_WEIGHTS = 3,  /* src [rows][k] float64 -> tcgen05 B image     */
  PCNN_PACK_TC16_WEIGHTS = 4,/* src [rows][k] float64 -> fp16x2 B image scaled
                                by 2^e; aux = float index of {max|w|, 2^-e} */
  PCNN_PACK_TCSS_WEIGHTS = 5 /* same weights -> image of the shared-memory
                                conv kernel ([n][16-ch chunk][tap] blocks);
                                aux = the fp16x2 image's scale pair;
                                reserved = taps | cb << 16                  */
};

/* unit flags */
enum pcnn_unit_flag {
  PCNN_FLAG_S2D = 1    /* ingest: write the NCHW image as 2x2 space-to-depth
                          blocks, channel (dy*2 + dx)*C + c at (y/2 + 1,
                          x/2 + 1) -- row 0 and column 0 stay zero         */
};

typedef struct pcnn_pack_desc {
  int64_t kind, src, dst, n;
  int64_t rows, k, aux, reserved;
} pcnn_pack_desc;

/* ---- redistribution programs --------------------------------------------
 * Phase (a): a straight-line program over float64 vectors in an "arena",
 * run in order by one CTA (the update terms upsilon and the channelwise
 * scale solve).  Phase (b): every rewrite descriptor rescales one parameter
 * tensor of the float64 master in parallel (grid-stride).  Both phases run
 * in one cooperative launch of pcnn_redistribute.                          */
enum pcnn_scale_opcode {
  PCNN_OP_FILL = 1,        /* dst[i] = imm                                   */
  PCNN_OP_LOAD = 2,        /* dst[i] = master[a + i*sa]                      */
  PCNN_OP_MUL = 3,         /* dst = A * B                                    */
  PCNN_OP_DIV = 4,         /* dst = A / B                                    */
  PCNN_OP_SUB = 5,         /* dst = A - B                                    */
  PCNN_OP_POWI = 6,        /* dst = A ^ p (integer p, may be negative)       */
  PCNN_OP_SROOT = 7,       /* dst = sign(A) |A|^(1/p)                        */
  PCNN_OP_AROOT = 8,       /* dst = |A|^(1/p)                                */
  PCNN_OP_RECIP = 9,       /* dst = 1 / A                                    */
  PCNN_OP_SOLVE = 10,      /* r = B / A; err if p even and r < 0;
                              dst = sign(r) |r|^(1/p)                        */
  PCNN_OP_CHECK_UNIFORM = 11, /* err if A[i] != A[0]                         */
  PCNN_OP_CHECK_NONZERO = 12, /* err if A[i] == 0                            */
  PCNN_OP_CHECK_NONNEG = 13,  /* err if A[i] < 0                             */
  PCNN_OP_CHECK_CLOSE = 14,   /* err unless |A-B| <= atol + rtol |B|         */
  PCNN_OP_CHECK_ALLONE = 15,  /* flag[p] = all(A == 1) (no error)            */
  PCNN_OP_SQRT = 16,       /* dst = sqrt(A)                                  */
  PCNN_OP_STORE = 17,      /* master[dst + i*sa] = A[i]                      */
  PCNN_OP_ADD = 18         /* dst = A + B (node fusing, transforms.py:62-101) */
};

typedef struct pcnn_scale_op {
  int64_t op, n;
  int64_t dst, a, b;        /* arena slots (LOAD: a is a master offset)      */
  int64_t sa, sb;           /* element strides of A/B (0 = broadcast)        */
  int64_t p;                /* integer exponent / root / flag index          */
  int64_t err;              /* error code reported if a check fails          */
  double imm, rtol, atol;
} pcnn_scale_op;

#define PCNN_MAX_FACTORS 6
/* factor value for element e: arena[slot + ((e / d1) % m1) * s1 + (e / d2) % m2] */
typedef struct pcnn_factor {
  int64_t slot, divide;     /* divide: 0 multiply, 1 divide                  */
  int64_t d1, m1, s1, d2, m2, reserved;
} pcnn_factor;

typedef struct pcnn_rewrite_desc {
  int64_t dst, src, n;
  int64_t src_arena;        /* 1: read src from the arena instead of master  */
  int64_t set_const;        /* 1: dst[e] = value (factors ignored)           */
  int64_t n_factors;
  double value;
  pcnn_factor f[PCNN_MAX_FACTORS];
} pcnn_rewrite_desc;

/* status_dev (device, int64[4]) receives {first error code, op index, 0, 0};
 * flags_dev (device, int64[n_flags]) receives CHECK_ALLONE results.        */

/* ---- plan options ----------------------------------------------------------
 * Every tuning / diagnostic switch of a plan.  The library reads no
 * environment variables: a plan's behaviour is fixed by its descriptors and
 * these options.  pcnn_plan_options_default() fills the defaults (the
 * configuration the benchmarks run); pcnn_plan_create() uses them.        */
typedef struct pcnn_plan_options {
  int64_t size;             /* sizeof(pcnn_plan_options), set by _default  */
  int64_t split;            /* 1: split fp16 hi/lo tensors between fp16x2
                               tensor-core convs; 0: every tensor float32  */
  int64_t halo_tiles;       /* 1: halo-tile conv kernel where the shape
                               allows; 0: the TMEM-A kernel only           */
  int64_t fuse_projection;  /* 1: a block's 1x1 projection inside its 3x3
                               conv's launch                               */
  int64_t band_pool;        /* 1: a conv's local / 2x2 bivariate pool in
                               the halo-tile kernel's band epilogue; 0:
                               conv into plan scratch, then a pool launch  */
  int64_t streamk;          /* 1: stream-K for launches whose whole tiles
                               fill < streamk_fill of the SMs              */
  double streamk_fill;      /* default 0.3                                 */
  int64_t flag_sync;        /* 1: per-tile completion counters instead of
                               whole-grid ordering (experimental, off)     */
  int64_t prezero;          /* 1: a halo-tile conv zeroes the next unit's
                               global-pool sums in its prologue            */
  int64_t linear_out;       /* 1: the last linear writes the logits        */
  int64_t pdl;              /* 1: programmatic dependent launches          */
  int64_t graph;            /* 1: pcnn_forward replays a CUDA graph when
                               use_graph is set; 0: always eager           */
  int64_t ss_mt;            /* halo-tile 128-row sub-tiles per tile, 0 auto*/
  int64_t ss_share;         /* both epilogue warpgroups per tile: -1 auto  */
  int64_t ss_psub;          /* one parity plane per stage: -1 auto         */
  int64_t ss_wres;          /* 1: resident weights where they fit          */
  int64_t tc_stage;         /* 1: TMA-staged input boxes (TMEM-A kernel)   */
  int64_t timeline;         /* 1: every launch stamps %globaltimer at its
                               first CTA's start and last CTA's exit
                               (pcnn_plan_timeline)                        */
  int64_t image_blocks;     /* >0: runs of stride-1 3x3 convs (32-64
                               channels) on small images in ONE launch,
                               each CTA keeping whole images' activations
                               in shared memory between the layers; the
                               value is the most images a CTA keeps
                               resident (1 or 2; default 2)             */
  int64_t debug;            /* diagnostic bits (tests / tools only):
                               2 skip MMAs, 4 skip epilogues, 32 CTA-0
                               trace, 64 per-CTA stamps                    */
  int64_t fused_net;        /* 1: a small sequential network (ingest, convs
                               with fused epilogue and pool, dense layers,
                               copyout; <= 2 M MACs per image) runs as ONE
                               launch, every CTA keeping whole images in
                               shared memory between the units            */
  int64_t ss_wide;          /* the halo-tile producer warp issues a
                               stage's bulk copies from several lanes at
                               once (one lane pays ~300 cycles per copy):
                               1 on tiles of <= 64 channels, 2 always,
                               0 never                                     */
  int64_t epi_pairs;        /* halo-tile kernel epilogue warpgroup pairs:
                               2 (four warpgroups, pairs alternate tiles)
                               or 1                                        */
  int64_t ss_pair;          /* 1: 128-channel halo tiles run on CTA pairs
                               (cluster of two, tcgen05 cta_group::2,
                               M = 256 over two SMs, each SM staging half
                               of the tile's weights); 0: one CTA per tile */
  int64_t scratch_cb4;      /* 1: the float32 scratch map between a halo-tile
                               conv and its local-pool pass in 4-channel
                               blocks (a warp's row-per-lane stores become
                               contiguous); 0 (default; measured equal): the
                               tensor's own block width                    */
  int64_t reserved[3];
} pcnn_plan_options;

/* ---- entry points --------------------------------------------------------*/
typedef struct pcnn_plan pcnn_plan;

int pcnn_abi_version(void);
const char* pcnn_last_error(void);
/* 1 if a device of compute capability 10.x is visible, else 0 */
int pcnn_device_ok(void);

void pcnn_plan_options_default(pcnn_plan_options* opt);

size_t pcnn_workspace_bytes(const pcnn_tensor_desc* tensors, int n_tensors, int batch);

int pcnn_plan_create(const pcnn_unit_desc* units, int n_units,
                     const pcnn_tensor_desc* tensors, int n_tensors,
                     int batch, int input_tensor, int output_tensor,
                     const float* params, void* workspace, size_t ws_bytes,
                     pcnn_plan** plan_out);
/* same with explicit options (null = defaults) */
int pcnn_plan_create_ex(const pcnn_unit_desc* units, int n_units,
                        const pcnn_tensor_desc* tensors, int n_tensors,
                        int batch, int input_tensor, int output_tensor,
                        const float* params, void* workspace, size_t ws_bytes,
                        const pcnn_plan_options* opt, pcnn_plan** plan_out);
/* Device timeline of the last forward (options.timeline): for each unit u,
 * ns[2u] = %globaltimer when its launch's first CTA passed its dependency
 * wait, ns[2u + 1] = when its last CTA exited; both 0 for a unit that ran
 * inside another unit's launch (fused) or launched nothing.  Entries
 * n_units + u (max_units up to 2 n_units) hold the pooling pass that follows
 * a pooled conv unit u (conv into plan scratch, then the pool launch), 0 when
 * the unit has none.  Synchronises `stream`.  Returns the number of entries
 * written (<= max_units).                                                  */
int pcnn_plan_timeline(pcnn_plan* plan, int64_t* ns, int max_units, void* stream);
/* the unit whose launch computes unit u (u itself unless fused) */
int pcnn_plan_unit_launch(const pcnn_plan* plan, int unit);
int pcnn_plan_destroy(pcnn_plan* plan);
/* number of kernel launches one forward issues (for gpu_launches) */
int pcnn_plan_num_launches(const pcnn_plan* plan);
/* conv implementation of unit i: 1 SIMT, 2 tcgen05 3xTF32, 3 tcgen05 fp16x2
 * (A in TMEM), 5 tcgen05 fp16x2 halo tiles, 6 the same inside an
 * image-resident run (options.image_blocks) */
int pcnn_plan_unit_impl(const pcnn_plan* plan, int unit);
/* storage format of tensor t: 0 float32; 1 split (two fp16 planes x = hi +
 * lo on the zero-bordered grid, written by its producer for fp16x2 convs);
 * 2 split in the four (row, column) parity planes (stride-2 readers) */
int pcnn_plan_tensor_split(const pcnn_plan* plan, int tensor);
/* Status of the last forward on `stream` (synchronises it): bit 0 = a value
 * of a split tensor left the fp16 range (|x| >= 2^15 or non-finite), so the
 * result is not fp32-accurate and must be recomputed with float32 tensors
 * (impl 2).  pcnn_forward_host copies the status with the logits;
 * pcnn_plan_last_status returns that copy once the stream is synchronised. */
int pcnn_plan_status(pcnn_plan* plan, void* stream);
int pcnn_plan_last_status(const pcnn_plan* plan);

/* x: device [batch][C][H][W] float32; logits: device [batch][K] float32.
 * use_graph: replay a captured CUDA graph of the whole network.          */
int pcnn_forward(pcnn_plan* plan, const float* x, float* logits, void* stream, int use_graph);
/* same with host buffers (pinned for overlap): H2D, forward, D2H inside  */
int pcnn_forward_host(pcnn_plan* plan, const float* x_host, float* logits_host,
                      float* x_dev_staging, float* logits_dev_staging, void* stream);
/* n host batches in a copy/compute pipeline: batch i+1's H2D (on an
 * internal copy stream, into the other of the two x_dev_staging buffers)
 * overlaps batch i's forward on `stream`; each batch's logits and status
 * word come back with a D2H on `stream`.  Every batch is still copied in
 * and out; only the copies overlap the network.  statuses (host, n ints,
 * may be null) receives each batch's status once `stream` is synchronised.
 * Replaces a loop over check_equivalence / reference_eval batches
 * (reference transforms.py:768-769, graph.py:413). */
int pcnn_forward_host_many(pcnn_plan* plan, const float* const* x_hosts, float* const* logits_hosts, int n,
                           float* x_dev_staging0, float* x_dev_staging1, float* logits_dev_staging,
                           int* statuses, void* stream);
/* launch unit i alone (per-kernel timing / debugging) */
int pcnn_forward_unit(pcnn_plan* plan, int unit, const float* x, float* logits, void* stream);

int pcnn_pack(const double* master, float* packed, const pcnn_pack_desc* ops, int n_ops,
              void* stream);

int pcnn_redistribute(double* master, double* arena, int64_t arena_len,
                      const pcnn_scale_op* ops, int n_ops,
                      const pcnn_rewrite_desc* rewrites, int n_rewrites,
                      int64_t* status_dev, int64_t* flags_dev, void* stream);

/* Device-resident forms of pcnn_redistribute / pcnn_pack for repeated runs
 * (an engine repacking after every transform, a redistribution program run
 * again on new weights): the descriptor tables are uploaded once at create;
 * run is stream-ordered launches only -- no allocation, no host copy, no
 * synchronisation.  A program owns its arena.  Same semantics per run as
 * the one-shot calls above (reference transforms.py:287-705). */
typedef struct pcnn_program pcnn_program;
int pcnn_program_create(const pcnn_scale_op* ops, int n_ops,
                        const pcnn_rewrite_desc* rewrites, int n_rewrites,
                        int64_t arena_len, pcnn_program** program_out);
int pcnn_program_run(pcnn_program* program, double* master, int64_t* status_dev,
                     int64_t* flags_dev, void* stream);
int pcnn_program_destroy(pcnn_program* program);

typedef struct pcnn_packer pcnn_packer;
int pcnn_packer_create(const pcnn_pack_desc* ops, int n_ops, pcnn_packer** packer_out);
int pcnn_packer_run(pcnn_packer* packer, const double* master, float* packed, void* stream);
int pcnn_packer_destroy(pcnn_packer* packer);

#ifdef __cplusplus
}
#endif
#endif /* PCNN_H */
