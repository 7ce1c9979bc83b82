// gb_tc_common.cuh -- device helpers shared by the tcgen05 sum-of-sum kernels
// (gb_decode_sos_tc.cu: 1-CTA kernels; gb_decode_sos_2cta.cu: CTA-pair kernel):
// mbarrier, TMA, UMMA descriptors, tcgen05 MMA / commit / TMEM load wrappers.
// Product code only (the oracle shares nothing with it).
#pragma once
#include <cuda.h>

#include "gb_internal.h"

namespace gb {
namespace tc {

constexpr int kTM = 128;       // probes per tile = UMMA M
constexpr int kKB = 128;       // K bytes per block = one 128 B swizzle atom

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, uint32_t bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
        ::"r"(dst), "l"((uint64_t)map), "r"(bar), "r"(x), "r"(y) : "memory");
}
// UMMA shared-memory descriptor, K-major, 128-byte swizzle: 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1u << 16) | ((uint64_t)(1024u >> 4) << 32) |
           ((uint64_t)1u << 46) | ((uint64_t)2u << 61);
}
// Instruction descriptor: kind::i8, D = s32, A = B = u8, both K-major, M = 128, N.
__device__ __forceinline__ uint32_t i8_idesc(int n) {
    return (2u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kTM >> 4) << 24);
}
__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
          "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
          "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
          "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// Issue-only variant: the caller waits (tmem_wait_ld) once after several loads.
__device__ __forceinline__ void tmem_ld32_nw(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
          "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
          "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
          "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// After tmem_wait_ld: ties the loaded registers to a volatile asm that follows the
// wait, so no use of them can be scheduled above it.
__device__ __forceinline__ void tmem_regs_ready(uint32_t (&v)[32]) {
    asm volatile(""
                 : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
                   "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]),
                   "+r"(v[15]), "+r"(v[16]), "+r"(v[17]), "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]),
                   "+r"(v[22]), "+r"(v[23]), "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]),
                   "+r"(v[29]), "+r"(v[30]), "+r"(v[31]));
}

// ---- CTA-pair (cta_group::2) helpers: cluster rank, DSMEM addresses, pair TMA / MMA / commit
__device__ __forceinline__ uint32_t cta_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void st_cluster_u32(uint32_t a, uint32_t v) {
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
// Arrive on a barrier of either CTA of the pair (address from mapa).  Default
// .release.cta semantics: the epilogue only has to order its (waited)
// tcgen05.ld's before the arrive, which tcgen05.fence::before_thread_sync does;
// .release.cluster would add a GPU-scope fence behind the output stores.
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t a) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
}
// TMA into this CTA's shared memory, transaction bytes counted on the leader's barrier.
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap *map, uint32_t bar_leader, int x,
                                                 int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"((uint64_t)map), "r"(bar_leader), "r"(x), "r"(y) : "memory");
}
// Instruction descriptor: kind::i8, D = s32, A = B = u8, K-major, M = 256 (pair), N.
__device__ __forceinline__ uint32_t i8_idesc_pair(int n) {
    return (2u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}
__device__ __forceinline__ void umma_i8_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
// Arrive on the barrier at the same offset in both CTAs once the pair's MMAs complete.
__device__ __forceinline__ void umma_commit_pair(uint32_t bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            bar),
        "h"((uint16_t)3) : "memory");
}

// 4 state bits -> 4 bytes of 0/1 (bit i -> byte i).
__device__ __forceinline__ uint32_t spread4(uint32_t nib) { return (nib * 0x00204081u) & 0x01010101u; }

__device__ __forceinline__ uint32_t real_mask(int L, int u) {
    const int nb = min(32, max(0, L - u * 32));
    return nb == 32 ? 0xffffffffu : ((1u << nb) - 1u);
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ uint32_t max_u16x2(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("max.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}

// a4 winner-take-all of one cluster (Eq.(4)-(5); ties kept,
// max 0 keeps every neuron, readings R3/R4): words[g] bit j = (sc[32g+j] == max sc).
// narrow: every score < 0x7FFF (true for the folded-gamma kernels: S <= n_p +
// gamma), so two scores share a register (element i and i+16 of a word, 16-bit
// halves) and max / equality run two at a time:
//   K = (mx + 0x7FFF) in both halves;  e = K - pk  (no borrow: pk <= mx per half)
//   bit 15 (31) of e is clear  <=>  the low (high) score equals mx.
// Otherwise plain 32-bit compares.  The max is a tree (independent chains).
template <int WC>
__device__ __forceinline__ void wta_words(const uint32_t (&sc)[32 * WC], bool narrow, uint32_t (&words)[WC]) {
    constexpr int LP = 32 * WC;
    if (narrow) {
        uint32_t pk[LP / 2];
#pragma unroll
        for (int g = 0; g < WC; ++g)
#pragma unroll
            for (int i = 0; i < 16; ++i) pk[16 * g + i] = __byte_perm(sc[32 * g + i], sc[32 * g + i + 16], 0x5410);
        uint32_t t[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) t[i] = pk[i];
#pragma unroll
        for (int i = 8; i < LP / 2; ++i) t[i & 7] = max_u16x2(t[i & 7], pk[i]);
        t[0] = max_u16x2(max_u16x2(t[0], t[1]), max_u16x2(t[2], t[3]));
        t[4] = max_u16x2(max_u16x2(t[4], t[5]), max_u16x2(t[6], t[7]));
        const uint32_t m2 = max_u16x2(t[0], t[4]);
        const uint32_t mx = max(m2 & 0xffffu, m2 >> 16);
        const uint32_t K = mx * 0x10001u + 0x7FFF7FFFu;
#pragma unroll
        for (int g = 0; g < WC; ++g) {
            uint32_t w0 = 0, w1 = 0;
#pragma unroll
            for (int i = 0; i < 16; i += 2) {
                w0 |= (~(K - pk[16 * g + i]) >> (15 - i)) & (0x10001u << i);
                w1 |= (~(K - pk[16 * g + i + 1]) >> (14 - i)) & (0x20002u << i);
            }
            words[g] = w0 | w1;
        }
    } else {
        uint32_t t[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) t[i] = sc[i];
#pragma unroll
        for (int i = 8; i < LP; ++i) t[i & 7] = max(t[i & 7], sc[i]);
        const uint32_t mx = max(max(max(t[0], t[1]), max(t[2], t[3])), max(max(t[4], t[5]), max(t[6], t[7])));
        const uint32_t mx1 = mx - 1u;   // sc == mx  <=>  (mx - 1 - sc) has the sign bit
#pragma unroll
        for (int g = 0; g < WC; ++g) {
            uint32_t w0 = 0, w1 = 0;
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
                w0 |= ((mx1 - sc[32 * g + j]) >> 31) << j;
                w1 |= ((mx1 - sc[32 * g + j + 1]) >> 31) << (j + 1);
            }
            words[g] = w0 | w1;
        }
    }
}

}  // namespace tc
}  // namespace gb
