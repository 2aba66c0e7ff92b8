// Thin inline-PTX wrappers for sm_100a: mbarriers, bulk (TMA) copies and the
// tcgen05 family (TMEM alloc, MMA, commit, ld/st, fences).
#pragma once

#include <stdint.h>

namespace pcnn {
namespace ptx {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarrier ----------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool mbar_test(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
// Bounded wait: a protocol bug traps (kernel error) instead of hanging the GPU.
// Polls with the non-suspending test_wait: hand-offs completed by the async
// proxy (tcgen05.commit, bulk-copy complete_tx) are seen immediately.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t spins = 0;
  while (!mbar_test(bar, parity)) {
    if (++spins > (1u << 30)) __trap();
  }
}

// Waiting with try_wait: the warp is suspended in hardware instead of
// spinning, so it does not steal issue slots from the MMA thread that shares
// its SM sub-partition.  Used by every role except the MMA issuer.
// try_wait with an explicit suspend-time hint: without one the hardware
// returns after a short system-dependent limit, and the waiting warps of a
// 20-warp CTA spent a third of all issued instructions polling (ncu).
__device__ __forceinline__ bool mbar_try_hint(uint32_t bar, uint32_t parity, uint32_t ns) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity), "r"(ns)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity) {
  uint32_t spins = 0;
  while (!mbar_try_hint(bar, parity, 20000)) {
    if (++spins > (1u << 20)) __trap();
  }
}
__device__ __forceinline__ void mbar_wait_nohint(uint32_t bar, uint32_t parity) {
  uint32_t spins = 0;
  while (!mbar_try(bar, parity)) {
    if (++spins > (1u << 28)) __trap();
  }
}

// One lane waits, the warp follows (keeps 31 lanes off the barrier unit).
__device__ __forceinline__ void mbar_wait_warp(uint32_t bar, uint32_t parity) {
  if ((threadIdx.x & 31) == 0) mbar_wait_sleep(bar, parity);
  __syncwarp();
}

// ---- bulk copy (TMA engine, non-tensor) ----------------------------------------
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

// 4-D tiled TMA load (coordinates innermost first; out-of-bounds elements are
// zero-filled, which is how conv padding is produced for free)
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const void* tmap, int c0, int c1, int c2, int c3,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(dst),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}

// 5-D tiled TMA load (the halo-tile kernel's weight half-blocks in CTA-pair mode)
__device__ __forceinline__ void tma_load_5d(uint32_t dst, const void* tmap, int c0, int c1, int c2, int c3, int c4,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
      "%6}], [%7];" ::"r"(dst),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(bar)
      : "memory");
}

// ---- clusters (CTA pairs) ----------------------------------------------------------
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cta address -> the same offset in CTA `rank` of the cluster (shared::cluster)
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// wait with cluster-scope acquire (barriers other CTAs of the cluster arrive on)
__device__ __forceinline__ bool mbar_test_cluster(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  uint32_t spins = 0;
  while (!mbar_test_cluster(bar, parity)) {
    if (++spins > (1u << 30)) __trap();
  }
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// make generic-proxy shared-memory writes visible to the async proxy (tensor core reads)
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ---- programmatic dependent launch ------------------------------------------------
// wait: block until the preceding grid in the stream has completed and its
// writes are visible (no-op without a programmatic dependency); launch: let
// the next PDL-launched grid start its prologue on SMs this grid frees.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---- tcgen05 -----------------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst_smem), "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
// CTA pair (cta_group::2): one warp of EACH CTA of the pair executes these
__device__ __forceinline__ void tmem_alloc2(uint32_t dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst_smem), "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
// leader CTA: arrive on the barrier at this offset in every CTA of `mask` once
// all cta_group::2 tcgen05 ops this thread issued complete
__device__ __forceinline__ void mma_commit2_warp(uint32_t bar, uint16_t mask) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .b32 r;\n\t"
      "elect.sync r|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(bar),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[tmem] * B[smem desc], kind::tf32, fp32 accumulate
__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Warp-collective forms: the whole warp executes them with warp-uniform
// operands (so they live in uniform registers) and elect.sync picks the one
// lane that issues.  Issuing from a lone `if (lane == 0)` thread instead made
// the compiler rebuild every operand with R2UR inside a waterfall loop and
// halved the MMA issue rate.
#define PCNN_MMA_TS_WARP(NAME, KIND)                                                                   \
  __device__ __forceinline__ void NAME(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, \
                                       uint32_t accumulate) {                                           \
    asm volatile(                                                                                       \
        "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\t"                                                   \
        "elect.sync r|e, 0xffffffff;\n\t"                                                              \
        "setp.ne.b32 p, %4, 0;\n\t"                                                                    \
        "@e tcgen05.mma.cta_group::1.kind::" KIND " [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),         \
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)                                           \
        : "memory");                                                                                    \
  }
PCNN_MMA_TS_WARP(mma_tf32_ts_warp, "tf32")
PCNN_MMA_TS_WARP(mma_f16_ts_warp, "f16")
#undef PCNN_MMA_TS_WARP
template <bool F16>
__device__ __forceinline__ void mma_ts_warp(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if (F16) mma_f16_ts_warp(d, a, b, idesc, acc);
  else mma_tf32_ts_warp(d, a, b, idesc, acc);
}
// One K-block (four 8-deep K steps) of the N-concatenated 3xTF32 scheme in a
// single asm statement, so every operand is moved to the uniform datapath
// once per K-block instead of once per MMA:
//   [main_k | corr_k] (+)= A_hi[k] * [B_hi | B_lo][k]   (N = 2*NT, idesc2)
//   corr_k            +=  A_lo[k] * B_hi[k]             (N = NT,   idesc1)
// d[k] = main accumulator of step k (corr at d[k] + corr_off); acc bit k of
// `accm` says whether main_k accumulates; desc = hi image descriptor of the
// K-block (+2 per step = +32 bytes).
#define PCNN_MMA_KBLOCK(NAME, KIND) __device__ __forceinline__ void NAME(uint32_t d0, uint32_t d1, uint32_t d2, uint32_t d3, \
                                                  uint32_t corr_off, uint32_t a_hi, uint32_t a_lo, \
                                                  uint64_t desc, uint32_t idesc2, uint32_t idesc1, \
                                                  uint32_t accm) { \
  asm volatile( \
      "{\n\t" \
      ".reg .pred e, p, t;\n\t.reg .b32 r, dc, ah, al;\n\t.reg .b64 bd;\n\t" \
      "elect.sync r|e, 0xffffffff;\n\t" \
      "setp.eq.u32 t, 0, 0;\n\t" \
      "and.b32 r, %11, 1;\n\tsetp.ne.u32 p, r, 0;\n\t" \
      "@e tcgen05.mma.cta_group::1.kind::" KIND " [%0], [%5], %7, %8, p;\n\t" \
      "add.u32 dc, %0, %4;\n\t" \
      "@e tcgen05.mma.cta_group::1.kind::" KIND " [dc], [%6], %7, %9, t;\n\t" \
      "and.b32 r, %11, 2;\n\tsetp.ne.u32 p, r, 0;\n\t" \
      "add.u32 ah, %5, 8;\n\tadd.u32 al, %6, 8;\n\tadd.s64 bd, %7, 2;\n\t" \
      "@e tcgen05.mma.cta_group::1.kind::" KIND " [%1], [ah], bd, %8, p;\n\t" \
      "add.u32 dc, %1, %4;\n\t" \
      "@e tcgen05.mma.cta_group::1.kind::" KIND " [dc], [al], bd, %9, t;\n\t" \
      "and.b32 r, %11, 4;\n\tsetp.ne.u32 p, r, 0;\n\t" \
      "add.u32 ah, %5, 16;\n\tadd.u32 al, %6, 16;\n\tadd.s64 bd, %7, 4;\n\t" \
      "@e tcgen05.mma.cta_group::1.kind::" KIND " [%2], [ah], bd, %8, p;\n\t" \
      "add.u32 dc, %2, %4;\n\t" \
      "@e tcgen05.mma.cta_group::1.kind::" KIND " [dc], [al], bd, %9, t;\n\t" \
      "and.b32 r, %11, 8;\n\tsetp.ne.u32 p, r, 0;\n\t" \
      "add.u32 ah, %5, 24;\n\tadd.u32 al, %6, 24;\n\tadd.s64 bd, %7, 6;\n\t" \
      "@e tcgen05.mma.cta_group::1.kind::" KIND " [%3], [ah], bd, %8, p;\n\t" \
      "add.u32 dc, %3, %4;\n\t" \
      "@e tcgen05.mma.cta_group::1.kind::" KIND " [dc], [al], bd, %9, t;\n\t" \
      "}\n" ::"r"(d0), \
      "r"(d1), "r"(d2), "r"(d3), "r"(corr_off), "r"(a_hi), "r"(a_lo), "l"(desc), "r"(idesc2), "r"(idesc1), \
      "r"(0), "r"(accm) \
      : "memory"); \
}
PCNN_MMA_KBLOCK(mma_kblock_concat_tf32, "tf32")
PCNN_MMA_KBLOCK(mma_kblock_concat_f16, "f16")
#undef PCNN_MMA_KBLOCK
template <bool F16>
__device__ __forceinline__ void mma_kblock_concat(uint32_t d0, uint32_t d1, uint32_t d2, uint32_t d3,
                                                  uint32_t corr_off, uint32_t a_hi, uint32_t a_lo,
                                                  uint64_t desc, uint32_t idesc2, uint32_t idesc1,
                                                  uint32_t accm) {
  if (F16) mma_kblock_concat_f16(d0, d1, d2, d3, corr_off, a_hi, a_lo, desc, idesc2, idesc1, accm);
  else mma_kblock_concat_tf32(d0, d1, d2, d3, corr_off, a_hi, a_lo, desc, idesc2, idesc1, accm);
}

__device__ __forceinline__ void mma_commit_warp(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .b32 r;\n\t"
      "elect.sync r|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(bar)
      : "memory");
}
// D[tmem] (+)= A[smem desc] * B[smem desc], kind::tf32
__device__ __forceinline__ void mma_tf32_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive on an mbarrier once all previously issued tcgen05 ops of this thread complete
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

// 32 lanes x 32 bit, 16 consecutive columns per thread
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Two x16 loads under one wait::ld (the wait names the destination registers,
// so no use of them can be scheduled above it).
__device__ __forceinline__ void tmem_ld16x2(uint32_t ta, uint32_t tb, float* va, float* vb) {
  uint32_t a[16], b[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]), "=r"(a[7]),
        "=r"(a[8]), "=r"(a[9]), "=r"(a[10]), "=r"(a[11]), "=r"(a[12]), "=r"(a[13]), "=r"(a[14]), "=r"(a[15])
      : "r"(ta));
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3]), "=r"(b[4]), "=r"(b[5]), "=r"(b[6]), "=r"(b[7]),
        "=r"(b[8]), "=r"(b[9]), "=r"(b[10]), "=r"(b[11]), "=r"(b[12]), "=r"(b[13]), "=r"(b[14]), "=r"(b[15])
      : "r"(tb));
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4]), "+r"(a[5]), "+r"(a[6]), "+r"(a[7]),
                 "+r"(a[8]), "+r"(a[9]), "+r"(a[10]), "+r"(a[11]), "+r"(a[12]), "+r"(a[13]), "+r"(a[14]),
                 "+r"(a[15]), "+r"(b[0]), "+r"(b[1]), "+r"(b[2]), "+r"(b[3]), "+r"(b[4]), "+r"(b[5]), "+r"(b[6]),
                 "+r"(b[7]), "+r"(b[8]), "+r"(b[9]), "+r"(b[10]), "+r"(b[11]), "+r"(b[12]), "+r"(b[13]),
                 "+r"(b[14]), "+r"(b[15]));
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    va[i] = __uint_as_float(a[i]);
    vb[i] = __uint_as_float(b[i]);
  }
}

// two 8-column loads (e.g. main and correction accumulators), one wait
__device__ __forceinline__ void tmem_ld8x2(uint32_t ta, uint32_t tb, float* va, float* vb) {
  uint32_t a[8], b[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]), "=r"(a[7])
               : "r"(ta));
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3]), "=r"(b[4]), "=r"(b[5]), "=r"(b[6]), "=r"(b[7])
               : "r"(tb));
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4]), "+r"(a[5]), "+r"(a[6]), "+r"(a[7]),
                 "+r"(b[0]), "+r"(b[1]), "+r"(b[2]), "+r"(b[3]), "+r"(b[4]), "+r"(b[5]), "+r"(b[6]), "+r"(b[7]));
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    va[i] = __uint_as_float(a[i]);
    vb[i] = __uint_as_float(b[i]);
  }
}

// 32 lanes x 32 bit, 8 consecutive columns per thread
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ---- descriptors -------------------------------------------------------------
// K-major operand, 128-byte swizzle, 8-row atoms 1024 B apart (SBO), version 1.
// K-major, no swizzle: core matrices of 8 rows x 16 bytes (rows 16 B apart);
// lbo = bytes between core matrices adjacent in K, sbo = adjacent in M/N.
__device__ __forceinline__ uint64_t smem_desc_noswz(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm_100); layout 0 = SWIZZLE_NONE
  return d;
}

// D[tmem] (+)= A[smem desc] * B[smem desc], kind::f16, issued by one elected lane
__device__ __forceinline__ void mma_f16_ss_warp(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                                uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\t"
      "elect.sync r|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);       // start address
  d |= (uint64_t)(1) << 16;                      // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;              // SBO
  d |= (uint64_t)1 << 46;                        // version (sm_100)
  d |= (uint64_t)2 << 61;                        // SWIZZLE_128B
  return d;
}
// instruction descriptor: kind::tf32, fp32 accumulate, K-major A and B
__host__ __device__ __forceinline__ uint32_t idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
// kind::f16: A, B fp16 (format 0), D fp32, both K-major
__host__ __device__ __forceinline__ uint32_t idesc_f16(int m, int n) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

}  // namespace ptx
}  // namespace pcnn
