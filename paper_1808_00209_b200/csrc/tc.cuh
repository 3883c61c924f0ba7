// tc.cuh -- thin inline-PTX wrappers for the sm_100a tensor-core path (tcgen05 / TMEM / mbarrier).
// Descriptor formats (validated bit-exactly by tools/probes/umma_probe.cu on a B200):
//   shared-memory matrix descriptor, SWIZZLE_NONE, K-major canonical layout
//     ((8 rows, m groups), 2 K-chunks) : ((16 B, SBO), LBO) -- core matrix = 8 rows x 16 B contiguous
//     bits [0,14) start >> 4, [16,30) LBO >> 4, [32,46) SBO >> 4, [46,48) version = 1, layout 0.
//   instruction descriptor kind::i8: c_format S32 (bits 4-5 = 2), a/b format signed (bits 7, 10),
//     K-major A and B, N >> 3 at bit 17, M >> 4 at bit 24.
#pragma once
#include "common.cuh"

namespace bnn {
namespace tc {

BNN_DEV uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

BNN_DEV uint64_t desc_kmajor(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);
}

__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, bool a_signed = true) {
  return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

BNN_DEV void mma_i8(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// Block-scaled e2m1 (kind::mxf4, K = 64 per MMA, scale block 32, UE8M0 scales; validated by
// tools/probes/mxf4_probe.cu): a/b format E2M1 = 1, scale format E8M0 (bit 23), K64 (bit 31 = 0).
__host__ __device__ constexpr uint32_t idesc_mxf4(int M, int N) {
  return (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(M >> 4) << 24);
}

BNN_DEV void mma_mxf4(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t sfa, uint32_t sfb,
                      uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %6, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%4], [%5], p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(sfa), "r"(sfb), "r"(accumulate));
}

// Writes v into 8 consecutive TMEM columns of this warp's 32 lanes (warp w: lanes 32 (w % 4)..).
BNN_DEV void tmem_st8_same(uint32_t taddr, uint32_t v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr), "r"(v));
}
BNN_DEV void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

BNN_DEV void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(bar)));
}

BNN_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}

BNN_DEV void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tBNN_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra BNN_DONE_%=;\n\tbra BNN_WAIT_%=;\n\tBNN_DONE_%=:\n\t}\n" ::"r"(smem_addr(bar)),
      "r"(phase));
}

// The same wait with a suspend-time hint: the thread sleeps in the barrier unit until the phase
// completes (or ~1 ms passes) instead of re-issuing try_wait -- for warps that idle a whole MMA.
BNN_DEV void mbar_wait_sleep(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tBNN_WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@P1 bra BNN_DONES_%=;\n\tbra BNN_WAITS_%=;\n\tBNN_DONES_%=:\n\t}\n" ::"r"(smem_addr(bar)),
      "r"(phase), "r"(1000000u));
}

// 1-D bulk copy global -> this CTA's shared memory (16-byte aligned, size % 16 == 0), completing
// `bytes` transactions on `bar` (arm it with expect_tx first)
BNN_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
BNN_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
// Stages `bytes` of a pre-expanded operand image into shared memory (thread 0 issues; wait on bar)
BNN_DEV void stage_image(void* dst, const uint8_t* src, uint32_t bytes, uint64_t* bar) {
  mbar_arrive_expect_tx(bar, bytes);
  constexpr uint32_t CH = 16384;
  for (uint32_t o = 0; o < bytes; o += CH) bulk_g2s(static_cast<uint8_t*>(dst) + o, src + o, bytes - o < CH ? bytes - o : CH, bar);
}

// Bulk copies of `bytes` (16-byte aligned, multiple of 16) in <= 16 KB pieces onto `bar` (the caller arms the
// barrier with the total expect_tx)
BNN_DEV void stage_chunks(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  constexpr uint32_t CH = 16384;
  for (uint32_t o = 0; o < bytes; o += CH)
    bulk_g2s(static_cast<uint8_t*>(dst) + o, static_cast<const uint8_t*>(src) + o, bytes - o < CH ? bytes - o : CH, bar);
}

BNN_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

BNN_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;"); }
BNN_DEV void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;"); }
BNN_DEV void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;"); }
BNN_DEV void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;"); }

template <uint32_t COLS>
BNN_DEV void tmem_alloc(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(dst_smem)),
               "n"(COLS));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}

template <uint32_t COLS>
BNN_DEV void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(COLS));
}

// 32 consecutive 32-bit columns of this thread's TMEM lane (warp w reads lanes 32*(w%4)..+31).
BNN_DEV void tmem_ld32(uint32_t taddr, int (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}

// 16 consecutive 32-bit columns of this thread's TMEM lane.
BNN_DEV void tmem_ld16(uint32_t taddr, int (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

// 16 consecutive columns of this thread's TMEM lane, low 16 bits of each, packed in pairs: register j
// holds column 2j in bits 0-15 and column 2j+1 in bits 16-31 (.pack::16b).
BNN_DEV void tmem_ld8_p16(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}

BNN_DEV void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 32 consecutive columns of this thread's TMEM lane, low 16 bits of each, packed in pairs (.pack::16b):
// register j holds column 2j in bits 0-15 and column 2j+1 in bits 16-31.
BNN_DEV void tmem_ld16_p16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

// Writes v into 32 consecutive TMEM columns of this warp's 32 lanes.
BNN_DEV void tmem_st32_same(uint32_t taddr, uint32_t v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
      "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr), "r"(v));
}

// ---- variants on precomputed shared-memory addresses, for single-thread-latency-bound loops
BNN_DEV void mbar_wait_at(uint32_t bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tBNN_WAITA_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra BNN_DONEA_%=;\n\tbra BNN_WAITA_%=;\n\tBNN_DONEA_%=:\n\t}\n" ::"r"(bar), "r"(phase) : "memory");
}
// Waits for two barriers at once: both try_waits are in flight together, so the latency is the larger of
// the two, not their sum (the loop re-checks both until both phases have completed)
BNN_DEV void mbar_wait2_at(uint32_t bar1, uint32_t phase1, uint32_t bar2, uint32_t phase2) {
  asm volatile(
      "{\n\t.reg .pred P1, P2;\n\tBNN_WAIT2_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P2, [%2], %3;\n\t"
      "@!P1 bra BNN_WAIT2_%=;\n\t@!P2 bra BNN_WAIT2_%=;\n\t}\n" ::"r"(bar1), "r"(phase1), "r"(bar2), "r"(phase2)
      : "memory");
}
BNN_DEV void mbar_wait_sleep_at(uint32_t bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tBNN_WAITB_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@P1 bra BNN_DONEB_%=;\n\tbra BNN_WAITB_%=;\n\tBNN_DONEB_%=:\n\t}\n" ::"r"(bar), "r"(phase), "r"(1000000u)
      : "memory");
}
BNN_DEV void mbar_arrive_at(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// tcgen05.mma (kind::mxf4, cta_group::1) and tcgen05.commit issued by ONE elected lane of a converged
// warp: every lane runs the loop, so no per-lane issue loop is needed around the instruction
BNN_DEV void mma_mxf4_elect(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t sfa,
                            uint32_t sfb, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %6, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%4], [%5], p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(sfa), "r"(sfb), "r"(accumulate));
}
BNN_DEV void commit_elect(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(bar));
}


// ---- CTA pairs (cta_group::2): two CTAs of a (2, 1, 1) cluster on the two SMs of a TPC run one M = 256 MMA.
// CTA rank r holds A rows [128 r, 128 r + 128) and B columns [N/2 r, N/2 r + N/2) at the SAME shared-memory
// offsets; the leader (rank 0) issues; each CTA's TMEM receives its own 128 rows x all N columns.  So each SM
// reads half of B per MMA (the shared-memory operand path is the bound of an N = 128 SS MMA otherwise).
BNN_DEV uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// address of the same shared-memory variable in CTA `rank` of the cluster
BNN_DEV uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// arrive on an mbarrier anywhere in the cluster (default .release.cta semantics, as a remote arrive of CUTLASS's
// ClusterBarrier: .release.cluster compiles to MEMBAR.ALL.GPU and its acquire side to CCTL.IVALL -- both on the
// per-tile chain).  The peer's operand writes reach the leader's MMA through the async proxy: writers fence
// (fence.proxy.async.shared::cta) before arriving.
BNN_DEV void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
BNN_DEV void mbar_wait_cluster_at(uint32_t bar, uint32_t phase) { mbar_wait_at(bar, phase); }
BNN_DEV void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
template <uint32_t COLS>
BNN_DEV void tmem_alloc_pair(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(dst_smem)), "n"(COLS));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
template <uint32_t COLS>
BNN_DEV void tmem_dealloc_pair(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(COLS));
}
BNN_DEV void mma_mxf4_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t sfa, uint32_t sfb,
                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %6, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%4], [%5], p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(sfa), "r"(sfb), "r"(accumulate));
}
BNN_DEV void mma_mxf4_pair_elect(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t sfa,
                                 uint32_t sfb, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %6, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%4], [%5], p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(sfa), "r"(sfb), "r"(accumulate));
}
// completion of the issuing thread's prior pair MMAs arrives on the barrier at this offset in BOTH CTAs
BNN_DEV void commit_pair(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
               "h"((uint16_t)3));
}
BNN_DEV void commit_pair_elect(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}\n" ::"r"(bar),
      "h"((uint16_t)3));
}

}  // namespace tc
}  // namespace bnn
