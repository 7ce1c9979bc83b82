// gb_decode_sos_2cta.cu -- sum-of-sum decode on a CTA pair (tcgen05 cta_group::2).
//
// Same method and same per-probe semantics as sos_tc2_kernel (gb_decode_sos_tc.cu):
// a3 S^t = W V^t + gamma V^t as an exact int8 x int8 -> int32 contraction
// (Eq.(3), Eq.(10)-(11) L328/L349, Alg. 1 line 4), a4 per-cluster
// winner-take-all with ties kept (Eq.(4)-(5) L220-225, readings R3/R4) and
// per-probe convergence / max_iters (Alg. 1), slot refill.
//
// What changes is the tile: the two CTAs of a cluster (one TPC) issue one
// UMMA of M = 256 probes (128 per CTA = its TMEM lanes), and each CTA stages
// only HALF of the W rows of a pass (N/2 rows of the B operand); the tensor
// core reads the other half from the peer's shared memory.  Per 256 probes a
// round therefore moves n_p^2 bytes of W from L2 instead of 2 n_p^2, and the
// MMA issue count halves.
//
//   leader (rank 0):  warp 0 TMA (its half of B, arms the pair's full barrier),
//                     warp 1 lane 0 MMA issuer for the pair, warps 2-5 epilogue
//   peer   (rank 1):  warp 0 TMA (its half, completes on the leader's barrier),
//                     warps 2-5 epilogue
// Barriers: full[S] (leader's only: expect_tx both halves), empty[S] and
// tfull[2] in both CTAs (multicast tcgen05.commit), tempty[2] (leader's,
// 256 arrivals: 128 local + 128 remote).  Round boundaries are cluster
// barriers; the pair keeps iterating while either CTA has an active slot.
#include <cuda.h>

#include <stdio.h>
#include <stdlib.h>

#include <algorithm>

#include "gb_internal.h"
#include "gb_tc_common.cuh"


namespace gb {
namespace {
using namespace tc;

struct Pair2Params {
    int NP;          // columns per pass (whole clusters, <= 256)
    int BR;          // TMA box rows (divides NP/2 for every pass)
    int S;           // B stages
    int gamma_epi;   // gamma added in the epilogue (0 when folded into B)
    int cyc;         // GB_FLAG_CYCLE_EXIT: stop a probe when V^r == V^{r-2}
    uint32_t a_off, b_off, v_off, bar_off, b_stage;
};

template <int WC>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
sos_tc2x2_kernel(Shape s, const __grid_constant__ CUtensorMap wmap, Pair2Params P,
                 const uint16_t *__restrict__ probes, int64_t k, int T, unsigned long long *queue,
                 uint32_t *__restrict__ out_state, uint16_t *__restrict__ out_iters,
                 uint8_t *__restrict__ out_status, const int64_t *__restrict__ list,
                 const unsigned long long *__restrict__ list_count) {
    constexpr int LP = 32 * WC;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;   // same offset in both CTAs
    uint8_t *gbase = smem_raw + (base - raw);
    const uint32_t A0 = base + P.a_off;     // nkb x (128 x 128 B), SW128: this CTA's 128 probe rows
    const uint32_t B0 = base + P.b_off;     // S x (NP/2 x 128 B), SW128: this CTA's half of the W rows
    uint32_t *Vs = reinterpret_cast<uint32_t *>(gbase + P.v_off);   // 2 x [nw][128]
    uint64_t *bars = reinterpret_cast<uint64_t *>(gbase + P.bar_off);
    const uint32_t bar0 = smem_u32(bars);
    const int S = P.S;
    auto full_bar = [&](int i) { return bar0 + 8u * i; };
    auto empty_bar = [&](int i) { return bar0 + 8u * (S + i); };
    auto tfull_bar = [&](int i) { return bar0 + 8u * (2 * S + i); };
    auto tempty_bar = [&](int i) { return bar0 + 8u * (2 * S + 2 + i); };
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * S + 4);
    uint32_t *flags = tmem_slot + 1;   // [2 round parities][2 ranks]: "has an active slot"

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const bool epi = warp >= 2;
    const int m = 32 * (warp & 3) + lane;
    const uint32_t rank = cta_rank();
    const bool leader = rank == 0;
    const int nw = s.nw, np = s.np;
    const int nkb = (np + kKB - 1) / kKB;
    const int npass = (np + P.NP - 1) / P.NP;
    auto pass_cols = [&](int pass, int &n0, int &ncols) {   // pass -> (first column, columns)
        n0 = pass * P.NP;
        ncols = min(P.NP, np - n0);
    };
    const bool narrow = P.gamma_epi + np < 0x7FFF;   // scores fit 15 bits (wta_words)

    if (tid == 0) {
        for (int i = 0; i < S; ++i) { mbar_init(full_bar(i), 1); mbar_init(empty_bar(i), 1); }
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
    const uint32_t tempty_leader0 = mapa(tempty_bar(0), 0);
    const uint32_t flags_self = mapa(smem_u32(flags), rank), flags_peer = mapa(smem_u32(flags), rank ^ 1u);

    uint32_t it_p = 0, it_m = 0, pc_m = 0, pc_e = 0;
    uint32_t par = 0, round = 0;
    uint32_t *V = Vs, *Vn = Vs + nw * kTM;
    // list mode: decode the *list_count probes whose indices a preceding kernel queued in list
    if (list) k = (int64_t)*list_count;
    auto pid = [&](int64_t i) { return list ? list[i] : i; };
    int64_t p = -1, pn = -1;
    uint4 qn = make_uint4(0, 0, 0, 0);
    const bool pack = s.C <= 8;
    int rl = 0;
    bool active = false;
    uint32_t dirty = (nkb * 4 >= 32) ? 0xffffffffu : ((1u << (nkb * 4)) - 1u);
    uint32_t nzcur = 0u;
    // The next probe is taken in two steps so neither waits at the round boundary: its
    // queue index when a slot is refilled (fetch), its symbols at the start of the next
    // round's epilogue, where the loads overlap that round's MMAs (fetch_syms).
    bool qready = false;
    auto fetch = [&]() {
        pn = (int64_t)atomicAdd(queue, 1ull);
        qready = false;
    };
    auto fetch_syms = [&]() {
        if (qready) return;
        qready = true;
        if (pack && pn < k) {
            uint32_t w4[4] = {0u, 0u, 0u, 0u};
            const uint16_t *pr = probes + pid(pn) * s.C;
#pragma unroll
            for (int c = 0; c < 8; ++c)
                if (c < s.C) w4[c >> 1] |= (uint32_t)__ldg(pr + c) << (16 * (c & 1));
            qn = make_uint4(w4[0], w4[1], w4[2], w4[3]);
        }
    };
    // refill: zmask = the words of the slot's state that may be nonzero (all at the start, else
    // the nonzero words of the finished probe's state)
    auto refill = [&](uint32_t zmask) {
        for (;;) {
            fetch_syms();
            p = pn;
            const uint4 q = qn;
            fetch();
            uint32_t *Vc = Vs + par * nw * kTM;
            // static predicated loop over the <= 32 state words (n_p <= 1024): no divergent
            // loop, stores independent
#pragma unroll
            for (int w = 0; w < 32; ++w)
                if ((zmask >> w) & 1u) Vc[w * kTM + m] = 0u;
            zmask = 0u;
            rl = 0;
            if (p >= k) { active = false; return; }
            p = pid(p);
            auto sym_of = [&](int c) -> unsigned {
                if (pack) {
                    const uint32_t w = (c >> 1) == 0 ? q.x : (c >> 1) == 1 ? q.y : (c >> 1) == 2 ? q.z : q.w;
                    return (w >> (16 * (c & 1))) & 0xffffu;
                }
                return __ldg(probes + p * s.C + c);
            };
            bool valid = true;
            if (pack) {   // C <= 8: symbols in registers, static unroll
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const unsigned sym = sym_of(c);
                    if (c < s.C && sym != kErased && sym >= (unsigned)s.L) valid = false;
                }
            } else {
                for (int c = 0; c < s.C; ++c) {
                    const unsigned sym = sym_of(c);
                    if (sym != kErased && sym >= (unsigned)s.L) valid = false;
                }
            }
            if (!valid) {   // GB_INVALID: zero state, 0 rounds; take another probe
                uint32_t *out = out_state + p * nw;
                for (int w = 0; w < nw; ++w) out[w] = 0u;
                out_iters[p] = 0;
                out_status[p] = GB_INVALID;
                continue;
            }
            auto ingest = [&](int c) {   // a1 ingest: V^0 known one-hot
                const unsigned sym = sym_of(c);
                if (sym != kErased) {
                    const int w = c * WC + (int)(sym >> 5);
                    Vc[w * kTM + m] = 1u << (sym & 31);
                    dirty |= 1u << w;
                }
            };
            if (pack) {
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    if (c < s.C) ingest(c);
            } else {
                for (int c = 0; c < s.C; ++c) ingest(c);
            }
            active = true;
            return;
        }
    };
    // producer: K block j of a round = (pass j / nkb, K block j % nkb)
    const int nload = npass * nkb;
    int pre = 0;   // K blocks of the coming round already issued
    auto load_block = [&](int j) {
        const int pass = j / nkb, kb = j - pass * nkb;
        int n0, ncols;
        pass_cols(pass, n0, ncols);
        const int half = ncols >> 1;
        const int st = it_p % S;
        mbar_wait(empty_bar(st), ((it_p / S) & 1u) ^ 1u);
        if (leader) mbar_expect_tx(full_bar(st), (uint32_t)ncols * kKB);   // both halves
        const uint32_t Bs = B0 + st * P.b_stage;
        for (int r0 = 0; r0 < half; r0 += P.BR)
            tma_load_2d_pair(Bs + r0 * kKB, &wmap, full_leader0 + 8u * st, kb * kKB, n0 + (int)rank * half + r0);
        ++it_p;
    };
    // A finished probe's state (in the Vn area, untouched until the next round's epilogue) is
    // stored at the start of that epilogue, while the tensor cores run the round's first pass,
    // instead of at the round boundary, and a refill zeroes only the words the finished state had
    // set.  Round boundary at C2 (clock64 trace of CTA 0, GB_SOS_TRACE builds): last pass's
    // epilogue 1.7k cycles, convergence + output + refill 3.4k -> 2.4k, A update 2.2k, cluster
    // barrier 0.6-3k, against 21.5k cycles of MMAs per round; C2 10^6 probes 2.72 -> 2.59 ms.
    // Then the refill's zeroing as a static predicated loop (2.4k -> 1.6k cycles) and the A update
    // four dirty words per iteration (2.2k -> ~1.7k): 2.60 -> 2.47-2.51 ms (same-box A/Bs).
    // Measured and not kept: the A update K block by K block with the next block's state words
    // loaded ahead (5.4k cycles, 2.81 ms), and as a static predicated loop over all 32 words
    // (4.3k cycles).
    int64_t pend = -1;
    auto flush = [&]() {
        if (pend >= 0) {
            uint32_t *out = out_state + pend * nw;
            for (int w = 0; w < nw; ++w) out[w] = Vn[w * kTM + m];
            pend = -1;
        }
    };
    if (epi) fetch();
    if (epi) refill(nw >= 32 ? 0xffffffffu : ((1u << nw) - 1u));
#ifdef GB_SOS_TRACE
    // debug: boundary timestamps of CTA 0 (epilogue thread m = 0, MMA issuer), printed at exit
    long long tr[12][8];
    for (int a = 0; a < 12; ++a) for (int b = 0; b < 8; ++b) tr[a][b] = 0;
    const bool trc = blockIdx.x == 0 && ((warp == 2 && lane == 0) || (warp == 1 && lane == 0));
#define TRACE(slot) do { if (trc && round < 12) tr[round][slot] = clock64(); } while (0)
#else
#define TRACE(slot) do { } while (0)
#endif
    for (;;) {
        TRACE(4);
        const int loc = __syncthreads_or(epi && active);
        TRACE(5);
        if (tid == 0) {
            const uint32_t off = 4u * (2u * (round & 1u) + rank);
            st_cluster_u32(flags_self + off, (uint32_t)loc);
            st_cluster_u32(flags_peer + off, (uint32_t)loc);
        }
        V = Vs + par * nw * kTM;
        Vn = Vs + (par ^ 1u) * nw * kTM;
        bool changed = false;
        bool cyc = true;
        if (epi) {   // incremental A = V^T (bytes, SW128), as in sos_tc2_kernel
            // four dirty words per iteration: their state-word loads and expansions overlap
            // (one word at a time, each store waited on its load: 2.2k cycles per round
            // boundary at C2; two at a time 1.8k)
            constexpr int NA = 4;
            uint32_t d = dirty;
            while (d) {
                int wq[NA];
                uint32_t vq[NA];
#pragma unroll
                for (int q = 0; q < NA; ++q) {
                    wq[q] = d ? __ffs(d) - 1 : -1;
                    d &= d - 1u;
                    vq[q] = (wq[q] >= 0 && wq[q] < nw) ? V[wq[q] * kTM + m] : 0u;
                }
#pragma unroll
                for (int q = 0; q < NA; ++q) {
                    if (wq[q] < 0) continue;
                    const int w = wq[q];
                    uint8_t *arow = gbase + P.a_off + (w >> 2) * (kTM * kKB) + m * kKB;
#pragma unroll
                    for (int h2 = 0; h2 < 2; ++h2) {
                        const int ch = 2 * (w & 3) + h2;
                        const uint32_t bits = (vq[q] >> (h2 * 16)) & 0xffffu;
                        *reinterpret_cast<uint4 *>(arow + ((ch ^ (m & 7)) * 16)) =
                            make_uint4(spread4(bits & 15u), spread4((bits >> 4) & 15u),
                                       spread4((bits >> 8) & 15u), spread4(bits >> 12));
                    }
                }
            }
            dirty = 0u;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        TRACE(6);
        cluster_sync();   // both A tiles ready; both flags visible
        TRACE(7);
        const uint32_t any = flags[2 * (round & 1u)] | flags[2 * (round & 1u) + 1];
        ++round;
        if (!any) break;
        if (warp == 0) {
            if (lane == 0) {   // ---- TMA producer: this CTA's half of each pass's W rows
                // W does not depend on the state, so the first `pre` K blocks of the
                // next round are loaded at the end of this one (they land while the
                // epilogue, the A update and the round barrier run)
                for (int j = pre; j < nload; ++j) load_block(j);
                pre = min(S, nload);
                for (int j = 0; j < pre; ++j) load_block(j);
            }
            __syncwarp();
        } else if (warp == 1) {
            if (lane == 0 && leader) {   // ---- MMA issuer for the pair
                for (int pass = 0; pass < npass; ++pass, ++pc_m) {
                    int n0, ncols;
                    pass_cols(pass, n0, ncols);
                    const uint32_t buf = pc_m & 1u;
                    mbar_wait(tempty_bar(buf), ((pc_m >> 1) & 1u) ^ 1u);
                    tc_fence_after();
                    if (pass == 0) TRACE(0);
                    const uint32_t idesc = i8_idesc_pair(ncols);
                    for (int kb = 0; kb < nkb; ++kb, ++it_m) {
                        const int st = it_m % S;
                        mbar_wait(full_bar(st), (it_m / S) & 1u);
                        tc_fence_after();
                        const uint32_t As = A0 + kb * (kTM * kKB), Bs = B0 + st * P.b_stage;
#pragma unroll
                        for (int ks = 0; ks < kKB / 32; ++ks)
                            umma_i8_pair(tmem + buf * 256, sw128_desc(As + ks * 32), sw128_desc(Bs + ks * 32),
                                         idesc, (kb > 0 || ks > 0) ? 1u : 0u);
                        umma_commit_pair(empty_bar(st));
                    }
                    umma_commit_pair(tfull_bar(buf));
                }
            }
            __syncwarp();
        } else {
            // ---- epilogue: per-cluster max + mask of each pass (a4)
            const uint32_t tl = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
            fetch_syms();
            flush();
            for (int pass = 0; pass < npass; ++pass, ++pc_e) {
                int n0, ncols;
                pass_cols(pass, n0, ncols);
                const uint32_t buf = pc_e & 1u;
                mbar_wait(tfull_bar(buf), (pc_e >> 1) & 1u);
                tc_fence_after();
                if (pass == npass - 1) TRACE(1);
                for (int c = n0 / LP; c < (n0 + ncols) / LP; ++c) {
                    const uint32_t col = buf * 256 + (uint32_t)(c * LP - n0);
                    if constexpr (WC <= 4) {
                        uint32_t sc[LP];
                        {   // all WC loads in flight, one wait
                            uint32_t(&v)[LP] = sc;
#pragma unroll
                            for (int g = 0; g < WC; ++g)
                                tmem_ld32_nw(tl + col + 32 * g, *reinterpret_cast<uint32_t(*)[32]>(&v[32 * g]));
                            tmem_wait_ld();
#pragma unroll
                            for (int g = 0; g < WC; ++g)
                                tmem_regs_ready(*reinterpret_cast<uint32_t(*)[32]>(&v[32 * g]));
                        }
                        if (P.gamma_epi) {
#pragma unroll
                            for (int g = 0; g < WC; ++g) {
                                const uint32_t vw = V[(c * WC + g) * kTM + m];
#pragma unroll
                                for (int j = 0; j < 32; ++j)
                                    sc[32 * g + j] += ((vw >> j) & 1u) ? (uint32_t)P.gamma_epi : 0u;
                            }
                        }
                        uint32_t wds[WC];
                        wta_words<WC>(sc, narrow, wds);
#pragma unroll
                        for (int g = 0; g < WC; ++g) {
                            const uint32_t word = wds[g] & real_mask(s.L, g);
                            const uint32_t old = V[(c * WC + g) * kTM + m];
                            const uint32_t wbit = 1u << (c * WC + g);
                            if (word != old) { changed = true; dirty |= wbit; }
                            if (old) nzcur |= wbit;
                            if (P.cyc) cyc &= (Vn[(c * WC + g) * kTM + m] == word);   // V^{r-2}
                            Vn[(c * WC + g) * kTM + m] = word;
                        }
                    } else {
                        uint32_t mx = 0;
                        for (int g = 0; g < WC; ++g) {
                            uint32_t v32[32];
                            tmem_ld32(tl + col + 32 * g, v32);
                            const uint32_t vw = V[(c * WC + g) * kTM + m];
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                mx = max(mx, v32[j] + (((vw >> j) & 1u) ? (uint32_t)P.gamma_epi : 0u));
                        }
                        for (int g = 0; g < WC; ++g) {
                            uint32_t v32[32];
                            tmem_ld32(tl + col + 32 * g, v32);
                            const uint32_t vw = V[(c * WC + g) * kTM + m];
                            uint32_t word = 0;
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                word |= ((v32[j] + (((vw >> j) & 1u) ? (uint32_t)P.gamma_epi : 0u)) == mx ? 1u : 0u)
                                        << j;
                            word &= real_mask(s.L, g);
                            const uint32_t wbit = 1u << (c * WC + g);
                            if (word != vw) { changed = true; dirty |= wbit; }
                            if (vw) nzcur |= wbit;
                            if (P.cyc) cyc &= (Vn[(c * WC + g) * kTM + m] == word);   // V^{r-2}
                            Vn[(c * WC + g) * kTM + m] = word;
                        }
                    }
                }
                tc_fence_before();
                mbar_arrive_cluster(tempty_leader0 + 8u * buf);
            }
            TRACE(2);
            if (active) {   // convergence (Alg. 1 "until V^{t+1} == V^t") and slot refill
                ++rl;
                const bool cyc_stop = P.cyc && rl >= 2 && cyc && changed;   // V^r == V^{r-2}
                if (!changed || rl == T || cyc_stop) {   // ---- a7 output (state: flush)
                    pend = p;
                    out_iters[p] = (uint16_t)rl;
                    out_status[p] = (uint8_t)(!changed ? GB_CONVERGED : cyc_stop ? GB_CYCLE : GB_MAX_ITERS);
                    dirty |= nzcur;
                    refill(nzcur);
                } else {
                    par ^= 1u;
                }
            }
            nzcur = 0u;
            TRACE(3);
        }
    }
    if (epi) flush();
#ifdef GB_SOS_TRACE
    if (trc)
        for (int a = 0; a < 12; ++a)
            printf("TRACE w%d r%d mma0 %lld lastdone %lld epidone %lld refilled %lld top %lld syncor %lld aupd %lld csync %lld\n",
                   warp, a, tr[a][0], tr[a][1], tr[a][2], tr[a][3], tr[a][4], tr[a][5], tr[a][6], tr[a][7]);
#endif
    // drain the prefetched loads (both halves complete on the leader's full barriers)
    // before either CTA can exit
    if (warp == 0 && lane == 0 && leader)
        for (uint32_t j = it_p - (uint32_t)pre; j < it_p; ++j) mbar_wait(full_bar(j % S), (j / S) & 1u);
    tc_fence_before();
    cluster_sync();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

bool plan_pair(const Shape &s, int gamma_epi, Pair2Params &P, size_t &smem) {
    if (s.Lp > 256 || s.np > 1024) return false;
    if (s.Wc != 1 && s.Wc != 2 && s.Wc != 3 && s.Wc != 4 && s.Wc != 8) return false;
    P.NP = s.Lp * (256 / s.Lp);
    if (P.NP > s.np) P.NP = s.np;
    // every pass is a multiple of Lp columns, so halves are multiples of Lp/2
    int br = 128;
    while (br > 8 && (s.Lp / 2) % br) br >>= 1;
    P.BR = br;
    P.gamma_epi = gamma_epi;
    P.cyc = 0;
    const int nkb = (s.np + kKB - 1) / kKB;
    P.a_off = 0;
    P.b_off = (uint32_t)nkb * kTM * kKB;
    P.b_stage = (uint32_t)(P.NP / 2) * kKB;
    P.b_stage = (P.b_stage + 1023u) & ~1023u;   // SW128 atoms stay 1024-byte aligned
    const size_t vbytes = 2ull * s.nw * kTM * 4;
    for (P.S = 6; P.S >= 2; --P.S) {
        P.v_off = P.b_off + P.S * P.b_stage;
        P.bar_off = (uint32_t)(P.v_off + vbytes);
        smem = P.bar_off + 8 * (2 * P.S + 4) + 32 + 1024;
        if (smem <= 227 * 1024) return true;
    }
    return false;
}

template <int WC>
cudaError_t launch_pair_t(Call &cl, const void *map, const Pair2Params &P, size_t smem, const uint16_t *probes,
                          int64_t k, int max_iters, uint32_t *state, uint16_t *iters, uint8_t *status,
                          const int64_t *list, const unsigned long long *list_count) {
    const gb_net *net = cl.net;
    const cudaStream_t st = cl.st;
    auto fn = sos_tc2x2_kernel<WC>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    // pairs that can be resident at once (TPC pairing can leave SMs unpaired)
    static std::atomic<int> max_clusters[9];
    if (max_clusters[WC].load() == 0) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(2 * (unsigned)(net->sm_count / 2), 1, 1);
        cfg.blockDim = dim3(192, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess || n <= 0) {
            cudaGetLastError();
            n = net->sm_count / 2;
        }
        max_clusters[WC].store(n);
    }
    const int64_t npairs = (k + 2 * kTM - 1) / (2 * kTM);
    const int pairs = (int)std::max<int64_t>(1, std::min<int64_t>(npairs, max_clusters[WC].load()));
    unsigned long long *queue = cl.counters();   // list mode: the second queue ([2])
    if (queue && list) queue += 2;
    if (!queue) return cl.err;
    fn<<<2 * pairs, 192, smem, st>>>(net->s, *reinterpret_cast<const CUtensorMap *>(map), P, probes, k,
                                     max_iters, queue, state, iters, status, list, list_count);
    cl.launched();
    return cudaGetLastError();
}

}  // namespace

bool sos_2cta_enabled(const gb_net *net) {
    if (net->opt[kOptSosPair].load(std::memory_order_relaxed) == 0) return false;
    Pair2Params P;
    size_t smem;
    return plan_pair(net->s, 0, P, smem);
}

int sos_2cta_box_rows(const Shape &s) {
    Pair2Params P;
    size_t smem;
    return plan_pair(s, 0, P, smem) ? P.BR : 0;
}

cudaError_t launch_sos_2cta(Call &cl, const void *map, int gamma_epi, int cyc, const uint16_t *probes, int64_t k,
                            int max_iters, uint32_t *state, uint16_t *iters, uint8_t *status, const int64_t *list,
                            const unsigned long long *list_count) {
    const gb_net *net = cl.net;
    Pair2Params P;
    size_t smem;
    if (!plan_pair(net->s, gamma_epi, P, smem)) return cudaErrorNotSupported;
    P.cyc = cyc;
    // one CTA per SM: two 512-column TMEM allocations on one SM could deadlock across pairs
    if (smem < 120 * 1024) smem = 120 * 1024;
    switch (net->s.Wc) {
        case 1: return launch_pair_t<1>(cl, map, P, smem, probes, k, max_iters, state, iters, status, list, list_count);
        case 2: return launch_pair_t<2>(cl, map, P, smem, probes, k, max_iters, state, iters, status, list, list_count);
        case 3: return launch_pair_t<3>(cl, map, P, smem, probes, k, max_iters, state, iters, status, list, list_count);
        case 4: return launch_pair_t<4>(cl, map, P, smem, probes, k, max_iters, state, iters, status, list, list_count);
        default: return launch_pair_t<8>(cl, map, P, smem, probes, k, max_iters, state, iters, status, list, list_count);
    }
}

}  // namespace gb
