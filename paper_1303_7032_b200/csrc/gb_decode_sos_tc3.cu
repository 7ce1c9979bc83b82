// gb_decode_sos_tc3.cu -- sum-of-sum decode on the tensor cores for networks
// whose expanded A tile does not fit in shared memory (1024 < n_p <= 4096,
// Lp <= 256; BASELINE C4: c=16 l=256, n_p = 4096; on the CTA pair also Lp = 512
// up to n_p = 8192, the paper's Scenario 2: c=16 l=512).
//
// Same method and per-probe semantics as sos_tc2_kernel (gb_decode_sos_tc.cu):
// a3 S^t = W V^t + gamma V^t as an exact int8 x int8 -> int32 contraction
// (Eq.(3), Eq.(10)-(11) L328/L349, Alg. 1 line 4) with
// tcgen05.mma.kind::i8 and TMEM accumulators; a4 per-cluster winner-take-all
// with ties kept (Eq.(4)-(5) L220-225, readings R3/R4); per-probe convergence
// and max_iters (Alg. 1); slot refill.
//
// At n_p = 4096 the A operand of a 128-probe tile (V^T as bytes) is 512 KiB,
// so it cannot stay resident as in sos_tc2_kernel.  Instead it is streamed:
// A-producer warps expand each K block of the state bits into a ring of
// swizzled 16 KiB stages, once per pass, in step with the TMA ring of W tiles:
//
//   warp 0      TMA producer: W8 + gamma*I tiles (NP rows x 128 B per K block)
//   warp 1      MMA issuer (one lane) and TMEM owner; two 256-column
//               accumulators so the epilogue of pass p overlaps pass p+1
//   warps 2-5   epilogue (thread = probe = TMEM lane): WTA of the pass's
//               clusters, convergence, output, slot refill
//   warps 6-9   A producers (thread = probe = A row): V bits -> A stage
//
// The current state V lives in shared memory ([word][probe], conflict-free);
// the next state is written to a global scratch (L2) by the epilogue and
// copied back into V at the end of the round (every A stage of the round has
// been consumed by then: the last pass's accumulator is complete).
#include <cuda.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include "gb_internal.h"
#include "gb_tc_common.cuh"

namespace gb {
namespace {
using namespace tc;

constexpr int kThreads3 = 320;

struct Sos3Params {
    int NP;          // columns per pass (whole clusters, <= 256)
    int BR;          // TMA box rows
    int S;           // W (B) stages
    int SA;          // A stages
    int gamma_epi;   // gamma added in the epilogue (0 when folded into B)
    int cyc;         // GB_FLAG_CYCLE_EXIT: stop a probe when V^r == V^{r-2}
    int vglob;       // current state in the global scratch (n_p > 4096: too big for shared memory)
    uint32_t a_off, b_off, v_off, bar_off, b_stage;
};

template <int WC>
__global__ void __launch_bounds__(kThreads3, 1)
sos_tc3_kernel(Shape s, const __grid_constant__ CUtensorMap wmap, Sos3Params P,
               const uint16_t *__restrict__ probes, int64_t k, int T, unsigned long long *queue,
               uint32_t *__restrict__ vscratch, uint32_t *__restrict__ out_state,
               uint16_t *__restrict__ out_iters, uint8_t *__restrict__ out_status) {
    constexpr int LP = 32 * WC;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *gbase = smem_raw + (base - raw);
    const uint32_t A0 = base + P.a_off;     // SA x (128 x 128 B), SW128
    const uint32_t B0 = base + P.b_off;     // S x (NP x 128 B), SW128
    uint32_t *V = reinterpret_cast<uint32_t *>(gbase + P.v_off);   // [nw][128] current state
    uint64_t *bars = reinterpret_cast<uint64_t *>(gbase + P.bar_off);
    const uint32_t bar0 = smem_u32(bars);
    const int S = P.S, SA = P.SA;
    auto full_bar = [&](int i) { return bar0 + 8u * i; };
    auto empty_bar = [&](int i) { return bar0 + 8u * (S + i); };
    auto afull_bar = [&](int i) { return bar0 + 8u * (2 * S + i); };
    auto aempty_bar = [&](int i) { return bar0 + 8u * (2 * S + SA + i); };
    auto tfull_bar = [&](int i) { return bar0 + 8u * (2 * S + 2 * SA + i); };
    auto tempty_bar = [&](int i) { return bar0 + 8u * (2 * S + 2 * SA + 2 + i); };
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * S + 2 * SA + 4);

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const bool epi = warp >= 2 && warp < 6;
    const bool apro = warp >= 6;
    const int m = 32 * (warp & 3) + lane;   // probe row = TMEM lane quarter of the warp (epilogue, A producers)
    const int nw = s.nw, np = s.np;
    const int nkb = (np + kKB - 1) / kKB;
    const int npass = (np + P.NP - 1) / P.NP;
    // next state [nw][128] in a global scratch, two areas: round r writes area r & 1, which
    // holds V^{r-2} until then (V^0 is put in area 0 at refill when the cycle exit is on)
    uint32_t *Vn2 = vscratch + (size_t)blockIdx.x * 2 * nw * kTM;

    if (tid == 0) {
        for (int i = 0; i < S; ++i) { mbar_init(full_bar(i), 1); mbar_init(empty_bar(i), 1); }
        for (int i = 0; i < SA; ++i) { mbar_init(afull_bar(i), 1); mbar_init(aempty_bar(i), 1); }
        for (int i = 0; i < 2; ++i) { mbar_init(tfull_bar(i), 1); mbar_init(tempty_bar(i), 128); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&wmap) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    uint32_t it_p = 0, it_m = 0, it_a = 0, pc_m = 0, pc_e = 0;
    int64_t p = -1;
    int rl = 0;
    bool active = false;
    auto refill = [&]() {
        for (;;) {
            p = (int64_t)atomicAdd(queue, 1ull);
            for (int w = 0; w < nw; ++w) V[w * kTM + m] = 0u;
            rl = 0;
            if (p >= k) { active = false; return; }
            bool valid = true;
            for (int c = 0; c < s.C; ++c) {
                const unsigned sym = __ldg(probes + p * s.C + c);
                if (sym != kErased && sym >= (unsigned)s.L) valid = false;
            }
            if (!valid) {   // GB_INVALID: zero state, 0 rounds; take another probe
                uint32_t *out = out_state + p * nw;
                for (int w = 0; w < nw; ++w) out[w] = 0u;
                out_iters[p] = 0;
                out_status[p] = GB_INVALID;
                continue;
            }
            // ---- a1 ingest: V^0 known one-hot, erased 0
            for (int c = 0; c < s.C; ++c) {
                const unsigned sym = __ldg(probes + p * s.C + c);
                if (sym != kErased) V[(c * WC + (int)(sym >> 5)) * kTM + m] = 1u << (sym & 31);
            }
            if (P.cyc)
                for (int w = 0; w < nw; ++w) Vn2[w * kTM + m] = V[w * kTM + m];
            active = true;
            return;
        }
    };
    if (epi) refill();
    for (;;) {
        if (!__syncthreads_or(epi && active)) break;
        if (warp == 0) {
            if (lane == 0) {   // ---- TMA producer: W rows of each pass, K block by K block
                for (int pass = 0; pass < npass; ++pass) {
                    const int n0 = pass * P.NP, ncols = min(P.NP, np - n0);
                    for (int kb = 0; kb < nkb; ++kb, ++it_p) {
                        const int st = it_p % S;
                        mbar_wait(empty_bar(st), ((it_p / S) & 1u) ^ 1u);
                        mbar_expect_tx(full_bar(st), (uint32_t)ncols * kKB);
                        const uint32_t Bs = B0 + st * P.b_stage;
                        for (int r0 = 0; r0 < ncols; r0 += P.BR)
                            tma_load_2d(Bs + r0 * kKB, &wmap, full_bar(st), kb * kKB, n0 + r0);
                    }
                }
            }
            __syncwarp();
        } else if (warp == 1) {
            if (lane == 0) {   // ---- MMA issuer
                for (int pass = 0; pass < npass; ++pass, ++pc_m) {
                    const int n0 = pass * P.NP, ncols = min(P.NP, np - n0);
                    const uint32_t buf = pc_m & 1u;
                    mbar_wait(tempty_bar(buf), ((pc_m >> 1) & 1u) ^ 1u);
                    tc_fence_after();
                    const uint32_t idesc = i8_idesc(ncols);
                    for (int kb = 0; kb < nkb; ++kb, ++it_m) {
                        const int st = it_m % S, sa = it_m % SA;
                        mbar_wait(afull_bar(sa), (it_m / SA) & 1u);
                        mbar_wait(full_bar(st), (it_m / S) & 1u);
                        tc_fence_after();
                        const uint32_t As = A0 + sa * (kTM * kKB), Bs = B0 + st * P.b_stage;
#pragma unroll
                        for (int ks = 0; ks < kKB / 32; ++ks)
                            umma_i8(tmem + buf * 256, sw128_desc(As + ks * 32), sw128_desc(Bs + ks * 32), idesc,
                                    (kb > 0 || ks > 0) ? 1u : 0u);
                        umma_commit(empty_bar(st));
                        umma_commit(aempty_bar(sa));
                    }
                    umma_commit(tfull_bar(buf));
                }
            }
            __syncwarp();
        } else if (apro) {
            // ---- A producers: K block kb of A = probe m's state bits [128 kb, 128 kb + 128) as
            // bytes, 128-byte swizzle (16-byte chunk ch of row m at ch ^ (m & 7)), once per pass
            for (int pass = 0; pass < npass; ++pass) {
                for (int kb = 0; kb < nkb; ++kb, ++it_a) {
                    const int sa = it_a % SA;
                    mbar_wait(aempty_bar(sa), ((it_a / SA) & 1u) ^ 1u);
                    uint32_t wv[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) wv[q] = (4 * kb + q < nw) ? V[(4 * kb + q) * kTM + m] : 0u;
                    uint8_t *arow = gbase + P.a_off + sa * (kTM * kKB) + m * kKB;
#pragma unroll
                    for (int ch = 0; ch < 8; ++ch) {
                        const uint32_t bits = (wv[ch >> 1] >> ((ch & 1) * 16)) & 0xffffu;
                        *reinterpret_cast<uint4 *>(arow + ((ch ^ (m & 7)) * 16)) =
                            make_uint4(spread4(bits & 15u), spread4((bits >> 4) & 15u), spread4((bits >> 8) & 15u),
                                       spread4(bits >> 12));
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    asm volatile("bar.sync 1, 128;" ::: "memory");   // all 128 rows written
                    if (m == 0) mbar_arrive(afull_bar(sa));
                }
            }
        } else {
            // ---- epilogue: per-cluster max + mask of each pass (a4)
            bool changed = false, cyc = true;
            uint32_t *Vn = Vn2 + (size_t)((rl + 1) & 1) * nw * kTM;   // area of round r = rl + 1
            const uint32_t tl = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
            for (int pass = 0; pass < npass; ++pass, ++pc_e) {
                const int n0 = pass * P.NP, ncols = min(P.NP, np - n0);
                const uint32_t buf = pc_e & 1u;
                mbar_wait(tfull_bar(buf), (pc_e >> 1) & 1u);
                tc_fence_after();
                for (int c = n0 / LP; c < (n0 + ncols) / LP; ++c) {
                    const uint32_t col = buf * 256 + (uint32_t)(c * LP - n0);
                    uint32_t mx = 0;
                    for (int g = 0; g < WC; ++g) {
                        uint32_t v32[32];
                        tmem_ld32(tl + col + 32 * g, v32);
                        const uint32_t vw = P.gamma_epi ? V[(c * WC + g) * kTM + m] : 0u;
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            mx = max(mx, v32[j] + (((vw >> j) & 1u) ? (uint32_t)P.gamma_epi : 0u));
                    }
                    for (int g = 0; g < WC; ++g) {
                        uint32_t v32[32];
                        tmem_ld32(tl + col + 32 * g, v32);
                        const uint32_t vw = V[(c * WC + g) * kTM + m];
                        const uint32_t ve = P.gamma_epi ? vw : 0u;
                        uint32_t word = 0;
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            word |= ((v32[j] + (((ve >> j) & 1u) ? (uint32_t)P.gamma_epi : 0u)) == mx ? 1u : 0u) << j;
                        word &= real_mask(s.L, g);
                        if (word != vw) changed = true;
                        if (P.cyc) cyc &= (Vn[(c * WC + g) * kTM + m] == word);   // V^{r-2}
                        Vn[(c * WC + g) * kTM + m] = word;
                    }
                }
                tc_fence_before();
                mbar_arrive(tempty_bar(buf));
            }
            // ---- convergence (Alg. 1 "until V^{t+1} == V^t"), output, slot refill.  The
            // last pass's accumulator is complete, so every A stage of this round has been
            // consumed: V may be overwritten.
            if (active) {
                ++rl;
                const bool cyc_stop = P.cyc && rl >= 2 && cyc && changed;   // V^r == V^{r-2}
                if (!changed || rl == T || cyc_stop) {   // ---- a7 output
                    uint32_t *out = out_state + p * nw;
                    for (int w = 0; w < nw; ++w) out[w] = Vn[w * kTM + m];
                    out_iters[p] = (uint16_t)rl;
                    out_status[p] = (uint8_t)(!changed ? GB_CONVERGED : cyc_stop ? GB_CYCLE : GB_MAX_ITERS);
                    refill();
                } else {
                    for (int w = 0; w < nw; ++w) V[w * kTM + m] = Vn[w * kTM + m];
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int WC>
cudaError_t launch3_t(Call &cl, const Sos3Params &P, size_t smem, const CUtensorMap *map, const uint16_t *probes,
                      int64_t k, int max_iters, uint32_t *state, uint16_t *iters, uint8_t *status) {
    const gb_net *net = cl.net;
    const cudaStream_t st = cl.st;
    auto fn = sos_tc3_kernel<WC>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t ntiles = (k + kTM - 1) / kTM;
    const int grid = (int)std::min<int64_t>(ntiles, net->sm_count);
    uint32_t *vscratch = cl.alloc_n<uint32_t>((size_t)net->sm_count * 2 * net->s.nw * kTM);
    unsigned long long *queue = cl.counters();
    if (!vscratch || !queue) return cl.err;
    fn<<<grid, kThreads3, smem, st>>>(net->s, *map, P, probes, k, max_iters, queue, vscratch, state,
                                      iters, status);
    cl.launched();
    return cudaGetLastError();
}


// ---------------------------------------------------------------------------
// CTA-pair form (tcgen05 cta_group::2, M = 256 probes per pair): the same roles in
// both CTAs; each CTA streams its own 128 probes' A stages and stages HALF of each
// pass's W rows (the tensor core reads the other half from the peer); the leader's
// warp 1 issues the pair's MMAs.  Barriers: full[S] (leader's, expect_tx of both
// halves), afull[SA] (leader's, 256 arrivals: both CTAs' producers), tempty[2]
// (leader's, 256 arrivals: both epilogues); empty / aempty / tfull receive the
// pair's multicast commits in both CTAs.  Rounds are cluster-wide (flags + cluster
// barrier), as in sos_tc2x2_kernel.
template <int WC, bool VG>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads3, 1)
sos_tc3x2_kernel(Shape s, const __grid_constant__ CUtensorMap wmap, Sos3Params P,
                 const uint16_t *__restrict__ probes, int64_t k, int T, unsigned long long *queue,
                 uint32_t *__restrict__ vscratch, uint32_t *__restrict__ out_state,
                 uint16_t *__restrict__ out_iters, uint8_t *__restrict__ out_status) {
    constexpr int LP = 32 * WC;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;   // same offset in both CTAs
    uint8_t *gbase = smem_raw + (base - raw);
    const uint32_t A0 = base + P.a_off;     // SA x (128 x 128 B): this CTA's probe rows
    const uint32_t B0 = base + P.b_off;     // S x (NP/2 x 128 B): this CTA's half of the W rows
    uint64_t *bars = reinterpret_cast<uint64_t *>(gbase + P.bar_off);
    const uint32_t bar0 = smem_u32(bars);
    const int S = P.S, SA = P.SA;
    auto full_bar = [&](int i) { return bar0 + 8u * i; };
    auto empty_bar = [&](int i) { return bar0 + 8u * (S + i); };
    auto afull_bar = [&](int i) { return bar0 + 8u * (2 * S + i); };
    auto aempty_bar = [&](int i) { return bar0 + 8u * (2 * S + SA + i); };
    auto tfull_bar = [&](int i) { return bar0 + 8u * (2 * S + 2 * SA + i); };
    auto tempty_bar = [&](int i) { return bar0 + 8u * (2 * S + 2 * SA + 2 + i); };
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * S + 2 * SA + 4);
    uint32_t *flags = tmem_slot + 1;   // [2 round parities][2 ranks]: "has an active slot"

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const bool epi = warp >= 2 && warp < 6;
    const bool apro = warp >= 6;
    const int m = 32 * (warp & 3) + lane;
    const uint32_t rank = cta_rank();
    const bool leader = rank == 0;
    const int nw = s.nw, np = s.np;
    const int nkb = (np + kKB - 1) / kKB;
    const int npass = (np + P.NP - 1) / P.NP;
    // global scratch per CTA: two next-state areas (as in sos_tc3_kernel) and, when it does not
    // fit shared memory (n_p > 4096), the current state
    uint32_t *Vn2 = vscratch + (size_t)blockIdx.x * 3 * nw * kTM;
    uint32_t *V = VG ? Vn2 + 2 * nw * kTM : reinterpret_cast<uint32_t *>(gbase + P.v_off);   // compile-time space
    // TMEM: two 256-column accumulators (the epilogue of pass p overlaps pass p+1), or one of 512
    // columns when a cluster is wider than 256 (Lp = 512: one cluster per pass, MMAs of N = 256
    // into its two halves; the epilogue then runs between passes).  Scenario 2 (c=16 l=512, 3*10^4
    // probes) 8.28 ms on the 4-warp sos_tc_kernel -> 4.46 ms here (same-box A/B).  Both counts are
    // compile-time: with runtime sub-tile loops in the MMA issuer C4 ran 28 ms instead of 18.
    constexpr int NB = WC > 8 ? 1 : 2;   // WC = 16 <=> Lp = 512 (plan3)
    constexpr int NSUB = WC > 8 ? 2 : 1;

    if (tid == 0) {
        for (int i = 0; i < S; ++i) { mbar_init(full_bar(i), 1); mbar_init(empty_bar(i), 1); }
        for (int i = 0; i < SA; ++i) { mbar_init(afull_bar(i), 2); mbar_init(aempty_bar(i), 1); }
        for (int i = 0; i < 2; ++i) { mbar_init(tfull_bar(i), 1); mbar_init(tempty_bar(i), 2 * 128); }
        flags[0] = flags[1] = flags[2] = flags[3] = 0u;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&wmap) : "memory");
    }
    if (warp == 1) {   // same warp in both CTAs
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t full_leader0 = mapa(full_bar(0), 0);
    const uint32_t afull_leader0 = mapa(afull_bar(0), 0);
    const uint32_t tempty_leader0 = mapa(tempty_bar(0), 0);
    const uint32_t flags_self = mapa(smem_u32(flags), rank), flags_peer = mapa(smem_u32(flags), rank ^ 1u);

    uint32_t it_p = 0, it_m = 0, it_a = 0, pc_m = 0, pc_e = 0, round = 0;
    int64_t p = -1;
    int rl = 0;
    bool active = false;
    auto refill = [&]() {
        for (;;) {
            p = (int64_t)atomicAdd(queue, 1ull);
            for (int w = 0; w < nw; ++w) V[w * kTM + m] = 0u;
            rl = 0;
            if (p >= k) { active = false; return; }
            bool valid = true;
            for (int c = 0; c < s.C; ++c) {
                const unsigned sym = __ldg(probes + p * s.C + c);
                if (sym != kErased && sym >= (unsigned)s.L) valid = false;
            }
            if (!valid) {
                uint32_t *out = out_state + p * nw;
                for (int w = 0; w < nw; ++w) out[w] = 0u;
                out_iters[p] = 0;
                out_status[p] = GB_INVALID;
                continue;
            }
            for (int c = 0; c < s.C; ++c) {   // a1 ingest: V^0 known one-hot, erased 0
                const unsigned sym = __ldg(probes + p * s.C + c);
                if (sym != kErased) V[(c * WC + (int)(sym >> 5)) * kTM + m] = 1u << (sym & 31);
            }
            if (P.cyc)
                for (int w = 0; w < nw; ++w) Vn2[w * kTM + m] = V[w * kTM + m];
            active = true;
            return;
        }
    };
    if (epi) refill();
    for (;;) {
        const int loc = __syncthreads_or(epi && active);
        if (tid == 0) {
            const uint32_t off = 4u * (2u * (round & 1u) + rank);
            st_cluster_u32(flags_self + off, (uint32_t)loc);
            st_cluster_u32(flags_peer + off, (uint32_t)loc);
        }
        cluster_sync();   // both CTAs' states ready; both flags visible
        const uint32_t any = flags[2 * (round & 1u)] | flags[2 * (round & 1u) + 1];
        ++round;
        if (!any) break;
        if (warp == 0) {
            if (lane == 0) {   // ---- TMA: this CTA's half of each pass's W rows, K block by K block
                for (int pass = 0; pass < npass; ++pass) {
                    // sub-tiles of <= 256 columns (one MMA each); this CTA stages half of each
                    const int n0 = pass * P.NP, ncols = min(P.NP, np - n0);
                    const int nsc = ncols / NSUB, half = nsc >> 1;
                    for (int kb = 0; kb < nkb; ++kb, ++it_p) {
                        const int st = it_p % S;
                        mbar_wait(empty_bar(st), ((it_p / S) & 1u) ^ 1u);
                        if (leader) mbar_expect_tx(full_bar(st), (uint32_t)ncols * kKB);   // both halves
                        const uint32_t Bs = B0 + st * P.b_stage;
#pragma unroll
                        for (int j = 0; j < NSUB; ++j)
                            for (int r0 = 0; r0 < half; r0 += P.BR)
                                tma_load_2d_pair(Bs + (j * half + r0) * kKB, &wmap, full_leader0 + 8u * st, kb * kKB,
                                                 n0 + j * nsc + (int)rank * half + r0);
                    }
                }
            }
            __syncwarp();
        } else if (warp == 1) {
            if (lane == 0 && leader) {   // ---- MMA issuer for the pair
                for (int pass = 0; pass < npass; ++pass, ++pc_m) {
                    const int n0 = pass * P.NP, ncols = min(P.NP, np - n0);
                    const int nsc = ncols / NSUB, half = nsc >> 1;
                    const uint32_t buf = pc_m % NB, use = pc_m / NB;
                    mbar_wait(tempty_bar(buf), (use & 1u) ^ 1u);
                    tc_fence_after();
                    const uint32_t idesc = i8_idesc_pair(nsc);
                    for (int kb = 0; kb < nkb; ++kb, ++it_m) {
                        const int st = it_m % S, sa = it_m % SA;
                        mbar_wait(afull_bar(sa), (it_m / SA) & 1u);
                        mbar_wait(full_bar(st), (it_m / S) & 1u);
                        tc_fence_after();
                        const uint32_t As = A0 + sa * (kTM * kKB), Bs = B0 + st * P.b_stage;
#pragma unroll
                        for (int ks = 0; ks < kKB / 32; ++ks)
#pragma unroll
                            for (int j = 0; j < NSUB; ++j)
                                umma_i8_pair(tmem + buf * 256 + j * 256, sw128_desc(As + ks * 32),
                                             sw128_desc(Bs + j * half * kKB + ks * 32), idesc,
                                             (kb > 0 || ks > 0) ? 1u : 0u);
                        umma_commit_pair(empty_bar(st));
                        umma_commit_pair(aempty_bar(sa));
                    }
                    umma_commit_pair(tfull_bar(buf));
                }
            }
            __syncwarp();
        } else if (apro) {
            // ---- A producers: this CTA's 128 probe rows of K block kb, once per pass
            for (int pass = 0; pass < npass; ++pass) {
                for (int kb = 0; kb < nkb; ++kb, ++it_a) {
                    const int sa = it_a % SA;
                    mbar_wait(aempty_bar(sa), ((it_a / SA) & 1u) ^ 1u);
                    uint32_t wv[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) wv[q] = (4 * kb + q < nw) ? V[(4 * kb + q) * kTM + m] : 0u;
                    uint8_t *arow = gbase + P.a_off + sa * (kTM * kKB) + m * kKB;
#pragma unroll
                    for (int ch = 0; ch < 8; ++ch) {
                        const uint32_t bits = (wv[ch >> 1] >> ((ch & 1) * 16)) & 0xffffu;
                        *reinterpret_cast<uint4 *>(arow + ((ch ^ (m & 7)) * 16)) =
                            make_uint4(spread4(bits & 15u), spread4((bits >> 4) & 15u), spread4((bits >> 8) & 15u),
                                       spread4(bits >> 12));
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    // all 128 rows written and fenced to the async proxy (named barrier of the
                    // producer warps), then one arrive per CTA on the leader's barrier (default
                    // .release.cta, as CUTLASS's cluster barriers; a .release.cluster arrive costs
                    // a MEMBAR per stage and starved the MMA: 32.8 vs 16.8 ms at C4)
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                    if (m == 0) mbar_arrive_cluster(afull_leader0 + 8u * sa);
                }
            }
        } else {
            // ---- epilogue: per-cluster max + mask of each pass (a4), from this CTA's TMEM lanes
            bool changed = false, cyc = true;
            uint32_t *Vn = Vn2 + (size_t)((rl + 1) & 1) * nw * kTM;
            const uint32_t tl = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
            constexpr int GB = WC < 2 ? WC : 2;   // TMEM loads in flight per wait (4: spills at WC >= 4)
            for (int pass = 0; pass < npass; ++pass, ++pc_e) {
                const int n0 = pass * P.NP, ncols = min(P.NP, np - n0);
                const uint32_t buf = pc_e % NB;
                mbar_wait(tfull_bar(buf), (pc_e / NB) & 1u);
                tc_fence_after();
                for (int c = n0 / LP; c < (n0 + ncols) / LP; ++c) {
                    const uint32_t col = buf * 256 + (uint32_t)(c * LP - n0);
                    uint32_t mx = 0;
                    for (int g0 = 0; g0 < WC; g0 += GB) {
                        uint32_t v[GB][32];
#pragma unroll
                        for (int gg = 0; gg < GB; ++gg) tmem_ld32_nw(tl + col + 32 * (g0 + gg), v[gg]);
                        tmem_wait_ld();
#pragma unroll
                        for (int gg = 0; gg < GB; ++gg) {
                            tmem_regs_ready(v[gg]);
                            const uint32_t vw = P.gamma_epi ? V[(c * WC + g0 + gg) * kTM + m] : 0u;
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                mx = max(mx, v[gg][j] + (((vw >> j) & 1u) ? (uint32_t)P.gamma_epi : 0u));
                        }
                    }
                    for (int g0 = 0; g0 < WC; g0 += GB) {
                        uint32_t v[GB][32];
#pragma unroll
                        for (int gg = 0; gg < GB; ++gg) tmem_ld32_nw(tl + col + 32 * (g0 + gg), v[gg]);
                        tmem_wait_ld();
#pragma unroll
                        for (int gg = 0; gg < GB; ++gg) {
                            tmem_regs_ready(v[gg]);
                            const int g = g0 + gg;
                            const uint32_t vw = V[(c * WC + g) * kTM + m];
                            const uint32_t ve = P.gamma_epi ? vw : 0u;
                            uint32_t word = 0;
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                word |= ((v[gg][j] + (((ve >> j) & 1u) ? (uint32_t)P.gamma_epi : 0u)) == mx ? 1u : 0u) << j;
                            word &= real_mask(s.L, g);
                            if (word != vw) changed = true;
                            if (P.cyc) cyc &= (Vn[(c * WC + g) * kTM + m] == word);   // V^{r-2}
                            Vn[(c * WC + g) * kTM + m] = word;
                        }
                    }
                }
                tc_fence_before();
                mbar_arrive_cluster(tempty_leader0 + 8u * buf);
            }
            if (active) {
                ++rl;
                const bool cyc_stop = P.cyc && rl >= 2 && cyc && changed;   // V^r == V^{r-2}
                if (!changed || rl == T || cyc_stop) {   // ---- a7 output
                    uint32_t *out = out_state + p * nw;
                    for (int w = 0; w < nw; ++w) out[w] = Vn[w * kTM + m];
                    out_iters[p] = (uint16_t)rl;
                    out_status[p] = (uint8_t)(!changed ? GB_CONVERGED : cyc_stop ? GB_CYCLE : GB_MAX_ITERS);
                    refill();
                } else {
                    for (int w = 0; w < nw; ++w) V[w * kTM + m] = Vn[w * kTM + m];
                }
            }
        }
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int WC>
cudaError_t launch3x2_t(Call &cl, const Sos3Params &P, size_t smem, const CUtensorMap *map,
                        const uint16_t *probes, int64_t k, int max_iters, uint32_t *state, uint16_t *iters,
                        uint8_t *status) {
    const gb_net *net = cl.net;
    const cudaStream_t st = cl.st;
    auto fn = P.vglob ? sos_tc3x2_kernel<WC, true> : sos_tc3x2_kernel<WC, false>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    static std::atomic<int> max_clusters[17][2];
    std::atomic<int> &mc = max_clusters[WC][P.vglob ? 1 : 0];
    if (mc.load() == 0) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(2 * (unsigned)(net->sm_count / 2), 1, 1);
        cfg.blockDim = dim3(kThreads3, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess || n <= 0) {
            cudaGetLastError();
            n = net->sm_count / 2;
        }
        mc.store(n);
    }
    const int64_t npairs = (k + 2 * kTM - 1) / (2 * kTM);
    const int pairs = (int)std::max<int64_t>(1, std::min<int64_t>(npairs, mc.load()));
    uint32_t *vscratch = cl.alloc_n<uint32_t>((size_t)2 * pairs * 3 * net->s.nw * kTM);
    unsigned long long *queue = cl.counters();
    if (!vscratch || !queue) return cl.err;
    fn<<<2 * pairs, kThreads3, smem, st>>>(net->s, *map, P, probes, k, max_iters, queue, vscratch, state,
                                            iters, status);
    cl.launched();
    return cudaGetLastError();
}

}  // namespace

static bool pair3_enabled(const gb_net *net) {
    return net->opt[kOptSosPair].load(std::memory_order_relaxed) != 0;
}

bool plan3(const gb_net *net, int gamma, void *params, size_t &smem) {
    const Shape &s = net->s;
    Sos3Params &P = *reinterpret_cast<Sos3Params *>(params);
    const bool pair = pair3_enabled(net);
    // 1024 < n_p <= 4096 with Lp <= 256 (both forms); Scenario 2's Lp = 512 up to n_p = 8192 on the
    // CTA pair only (one 512-column accumulator, current state in the global scratch)
    if (s.np <= 1024 || s.np > (pair ? 8192 : 4096)) return false;
    if (s.Wc != 1 && s.Wc != 2 && s.Wc != 4 && s.Wc != 8 && !(pair && s.Wc == 16)) return false;
    P.NP = s.Lp > 256 ? s.Lp : s.Lp * (256 / s.Lp);
    if (P.NP > s.np) P.NP = s.np;
    // pair: each CTA stages half of every <= 256-column sub-tile (whole clusters -> halves of
    // Lp/2 rows, or 128 rows of a 512-column pass)
    const int rows = pair ? P.NP / 2 : P.NP;
    const int unit = pair ? (P.NP > 256 ? 128 : s.Lp / 2) : s.Lp;
    int br = 256;
    while (br > 8 && (unit % br || br > rows)) br >>= 1;
    P.BR = br;
    P.gamma_epi = gamma > 255 ? gamma : 0;
    P.cyc = 0;
    P.vglob = s.np > 4096 ? 1 : 0;
    P.b_stage = (uint32_t)rows * kKB;
    P.b_stage = (P.b_stage + 1023u) & ~1023u;   // SW128 atoms stay 1024-byte aligned
    const size_t vbytes = P.vglob ? 0 : (size_t)s.nw * kTM * 4;
    int s_max = pair ? 6 : 4, sa_max = 3;
    for (P.S = s_max; P.S >= 2; --P.S) {
        for (P.SA = sa_max; P.SA >= 2; --P.SA) {
            P.a_off = 0;
            P.b_off = (uint32_t)P.SA * kTM * kKB;
            P.v_off = P.b_off + P.S * P.b_stage;
            P.bar_off = (uint32_t)(P.v_off + vbytes);
            smem = P.bar_off + 8 * (2 * P.S + 2 * P.SA + 4) + 32 + 1024;
            if (smem <= 227 * 1024) return true;
        }
    }
    return false;
}

static_assert(sizeof(Sos3Params) <= 64, "plan3 params buffer");
int plan3_box_rows(const void *params) { return reinterpret_cast<const Sos3Params *>(params)->BR; }

bool sos_tc3_pair(const gb_net *net) { return sos_tc3_enabled(net) && pair3_enabled(net); }

bool sos_tc3_enabled(const gb_net *net) {
    if (net->opt[kOptSosStreamed].load(std::memory_order_relaxed) == 0) return false;
    Sos3Params P;
    size_t smem;
    return plan3(net, 1, &P, smem);
}

cudaError_t launch_sos_tc3(Call &cl, int gamma, int cyc, const void *map, const uint16_t *probes, int64_t k,
                           int max_iters, uint32_t *state, uint16_t *iters, uint8_t *status) {
    const gb_net *net = cl.net;
    Sos3Params P;
    size_t smem;
    if (!plan3(net, gamma, &P, smem)) return cudaErrorNotSupported;
    P.cyc = cyc;
    const CUtensorMap *m = reinterpret_cast<const CUtensorMap *>(map);
    if (pair3_enabled(net)) {
        if (smem < 120 * 1024) smem = 120 * 1024;   // one CTA per SM (512 TMEM columns each)
        switch (net->s.Wc) {
            case 1: return launch3x2_t<1>(cl, P, smem, m, probes, k, max_iters, state, iters, status);
            case 2: return launch3x2_t<2>(cl, P, smem, m, probes, k, max_iters, state, iters, status);
            case 4: return launch3x2_t<4>(cl, P, smem, m, probes, k, max_iters, state, iters, status);
            case 8: return launch3x2_t<8>(cl, P, smem, m, probes, k, max_iters, state, iters, status);
            default: return launch3x2_t<16>(cl, P, smem, m, probes, k, max_iters, state, iters, status);
        }
    }
    switch (net->s.Wc) {
        case 1: return launch3_t<1>(cl, P, smem, m, probes, k, max_iters, state, iters, status);
        case 2: return launch3_t<2>(cl, P, smem, m, probes, k, max_iters, state, iters, status);
        case 4: return launch3_t<4>(cl, P, smem, m, probes, k, max_iters, state, iters, status);
        default: return launch3_t<8>(cl, P, smem, m, probes, k, max_iters, state, iters, status);
    }
}

}  // namespace gb
