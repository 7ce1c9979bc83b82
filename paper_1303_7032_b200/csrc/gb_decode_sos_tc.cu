// gb_decode_sos_tc.cu -- sum-of-sum decode on the 5th-generation tensor cores.
//
// a3 SOS score (Eq.(3), Eq.(10)-(11) L328/L349, Alg. 1 line 4):
//     S^t = W V^t + gamma V^t
// is an exact integer contraction: V (0/1) and W (0/1) as uint8, products and
// sums in int32 -- tcgen05.mma.kind::i8 with the accumulator in TMEM.  One CTA
// owns a tile of 128 probes (UMMA M = 128, TMEM lane = probe):
//     D[probe, neuron] = sum_j A[probe, j] * B[neuron, j],  A = V^T,  B = W
// (W is symmetric, so its rows are the K-major B operand).  W tiles are TMA
// loaded (128-byte swizzle, K block = 128) from the u8 W8 matrix, double
// buffered against the MMAs; the A tile is expanded from the state bits into
// the same swizzled layout by the CTA's threads.
// a4 WTA + convergence (Eq.(4)-(5) L220-225, Alg. 1): the epilogue
// reads each probe's TMEM row (tcgen05.ld), adds gamma*v_i, takes the max over
// each cluster's real neurons and keeps every neuron that reaches it (ties
// kept, reading R3; max 0 activates all real neurons, R4); the new state bits
// go back to shared memory and feed the next round's A tile.  Per-probe
// convergence (V^{t+1} == V^t) and rounds are tracked in registers; the tile
// iterates until all its probes converged or max_iters rounds ran.  There is
// no host round-trip between rounds.
//
// Passes: TMEM holds 512 int32 columns per lane, so the n_p output columns are
// processed in passes of NP <= 512 columns made of whole clusters (Lp <= 256;
// MMA N <= 256 per instruction).
#include <cuda.h>
#include <string.h>

#include <algorithm>

#include "gb_internal.h"
#include "gb_tc_common.cuh"

namespace gb {
namespace {
using namespace tc;

constexpr int kThreads = 128;  // one thread per probe / TMEM lane

struct SosParams {
    int NP;        // columns per pass (multiple of Lp, <= 512)
    int BR;        // TMA box rows (divides Lp, <= 256)
    int v_global;  // state buffers in a global scratch (L2) instead of shared memory (large n_p)
    uint32_t a_off, b_off, v_off, bar_off;   // shared-memory carve (bytes from the aligned base)
    uint32_t b_stage;                        // bytes per B stage
};

template <int WC>
__global__ void __launch_bounds__(kThreads, 1)
sos_tc_kernel(Shape s, const __grid_constant__ CUtensorMap wmap, SosParams P,
              const uint16_t *__restrict__ probes, int64_t k, int gamma, int T, int cyc_exit,
              unsigned long long *queue,
              uint32_t *vscratch,
              uint32_t *__restrict__ out_state, uint16_t *__restrict__ out_iters,
              uint8_t *__restrict__ out_status) {
    constexpr int LP = 32 * WC;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *gbase = smem_raw + (base - raw);
    const uint32_t A0 = base + P.a_off;                 // 2 stages x (128 x 128 B)
    const uint32_t B0 = base + P.b_off;                 // 2 stages x (NP x 128 B)
    // [nw][128] x 2 state buffers: shared memory, or this CTA's slice of a global scratch
    uint32_t *Vs = P.v_global ? vscratch + (size_t)blockIdx.x * 2 * s.nw * kTM
                              : reinterpret_cast<uint32_t *>(gbase + P.v_off);
    uint64_t *bars = reinterpret_cast<uint64_t *>(gbase + P.bar_off);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 4);
    const uint32_t tma_bar0 = smem_u32(&bars[0]), mma_bar0 = smem_u32(&bars[2]);

    const int m = threadIdx.x;
    const int warp = m >> 5;
    const int nw = s.nw, np = s.np;
    const int nkb = (np + kKB - 1) / kKB;
    const int npass = (np + P.NP - 1) / P.NP;

    if (m == 0) {
        mbar_init(tma_bar0, 1);
        mbar_init(tma_bar0 + 8, 1);
        mbar_init(mma_bar0, 1);
        mbar_init(mma_bar0 + 8, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&wmap) : "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tmem_lane = tmem + ((uint32_t)(warp * 32) << 16);

    uint32_t it_count = 0;   // K-block iterations issued so far (stage/phase bookkeeping)
    // Slot refill (as in sos_tc2_kernel): each TMEM lane holds one probe; a probe
    // that converges or reaches max_iters is written out and replaced by the
    // next probe of the global queue.
    // per-thread double buffer: V = V^{r-1} (current), Vn receives V^r and holds V^{r-2} until
    // then (the period-2 check of GB_FLAG_CYCLE_EXIT reads it before overwriting)
    uint32_t *V = Vs, *Vn = Vs + nw * kTM;
    int64_t p = -1;
    int rl = 0;
    bool active = false;
    bool cyc = false;
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
            // ---- a1 ingest: V^0 = known one-hot, erased clusters 0
            for (int c = 0; c < s.C; ++c) {
                const unsigned sym = __ldg(probes + p * s.C + c);
                if (sym != kErased) V[(c * WC + (sym >> 5)) * kTM + m] = 1u << (sym & 31);
            }
            active = true;
            return;
        }
    };
    refill();
    {
        for (;;) {
            if (!__syncthreads_or(active)) break;
            // ---- a3 score S = W V + gamma V, pass by pass
            for (int pass = 0; pass < npass; ++pass) {
                const int n0 = pass * P.NP;
                const int ncols = min(P.NP, np - n0);
                for (int kb = 0; kb < nkb; ++kb, ++it_count) {
                    const uint32_t st = it_count & 1u;
                    const uint32_t use = it_count >> 1;
                    const uint32_t As = A0 + st * (kTM * kKB);
                    const uint32_t Bs = B0 + st * P.b_stage;
                    if (it_count >= 2) mbar_wait(mma_bar0 + 8 * st, (use - 1) & 1u);   // stage free
                    if (m == 0) {
                        mbar_expect_tx(tma_bar0 + 8 * st, (uint32_t)ncols * kKB);
                        for (int r0 = 0; r0 < ncols; r0 += P.BR)
                            tma_load_2d(Bs + r0 * kKB, &wmap, tma_bar0 + 8 * st, kb * kKB, n0 + r0);
                    }
                    // A tile: probe m's bits [kb*128, kb*128+128) as bytes, 128 B swizzle
                    {
                        const int w0 = kb * 4;
                        uint32_t wv[4];
#pragma unroll
                        for (int q = 0; q < 4; ++q) wv[q] = (w0 + q < nw) ? V[(w0 + q) * kTM + m] : 0u;
                        uint8_t *arow = gbase + (As - base) + m * kKB;
#pragma unroll
                        for (int ch = 0; ch < 8; ++ch) {
                            const uint32_t bits = (wv[ch >> 1] >> ((ch & 1) * 16)) & 0xffffu;
                            uint4 v4 = make_uint4(spread4(bits & 15u), spread4((bits >> 4) & 15u),
                                                  spread4((bits >> 8) & 15u), spread4(bits >> 12));
                            *reinterpret_cast<uint4 *>(arow + ((ch ^ (m & 7)) * 16)) = v4;
                        }
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncthreads();
                    if (m == 0) {
                        mbar_wait(tma_bar0 + 8 * st, use & 1u);
                        tc_fence_after();
#pragma unroll
                        for (int ks = 0; ks < kKB / 32; ++ks) {
                            const uint64_t ad = sw128_desc(As + ks * 32);
                            for (int j = 0; j * 256 < ncols; ++j) {
                                const int n = min(256, ncols - j * 256);
                                const uint64_t bd = sw128_desc(Bs + j * 256 * kKB + ks * 32);
                                umma_i8(tmem + j * 256, ad, bd, i8_idesc(n), (kb > 0 || ks > 0) ? 1u : 0u);
                            }
                        }
                        umma_commit(mma_bar0 + 8 * st);
                    }
                }
                // wait for the pass's last commit (covers all earlier MMAs of this thread)
                {
                    const uint32_t last = it_count - 1;
                    mbar_wait(mma_bar0 + 8 * (last & 1u), (last >> 1) & 1u);
                }
                tc_fence_after();
                // ---- a4 per-cluster max + mask (epilogue) for this pass's clusters
                for (int c = n0 / LP; c < (n0 + ncols) / LP; ++c) {
                    const uint32_t col = (uint32_t)(c * LP - n0);
                    if constexpr (WC <= 4) {
                        uint32_t sc[LP];
#pragma unroll
                        for (int g = 0; g < WC; ++g) {
                            uint32_t v32[32];
                            tmem_ld32(tmem_lane + col + 32 * g, v32);
                            const uint32_t vw = V[(c * WC + g) * kTM + m];
#pragma unroll
                            for (int j = 0; j < 32; ++j) sc[32 * g + j] = v32[j] + (((vw >> j) & 1u) ? (uint32_t)gamma : 0u);
                        }
                        uint32_t mx = 0;
#pragma unroll
                        for (int j = 0; j < LP; ++j) mx = max(mx, sc[j]);
#pragma unroll
                        for (int g = 0; g < WC; ++g) {
                            uint32_t word = 0;
#pragma unroll
                            for (int j = 0; j < 32; ++j) word |= (sc[32 * g + j] == mx ? 1u : 0u) << j;
                            word &= real_mask(s.L, g);
                            if (cyc_exit) cyc &= (Vn[(c * WC + g) * kTM + m] == word);
                            Vn[(c * WC + g) * kTM + m] = word;
                        }
                    } else {
                        uint32_t mx = 0;
                        for (int g = 0; g < WC; ++g) {
                            uint32_t v32[32];
                            tmem_ld32(tmem_lane + col + 32 * g, v32);
                            const uint32_t vw = V[(c * WC + g) * kTM + m];
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                mx = max(mx, v32[j] + (((vw >> j) & 1u) ? (uint32_t)gamma : 0u));
                        }
                        for (int g = 0; g < WC; ++g) {
                            uint32_t v32[32];
                            tmem_ld32(tmem_lane + col + 32 * g, v32);
                            const uint32_t vw = V[(c * WC + g) * kTM + m];
                            uint32_t word = 0;
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                word |= ((v32[j] + (((vw >> j) & 1u) ? (uint32_t)gamma : 0u)) == mx ? 1u : 0u) << j;
                            word &= real_mask(s.L, g);
                            if (cyc_exit) cyc &= (Vn[(c * WC + g) * kTM + m] == word);
                            Vn[(c * WC + g) * kTM + m] = word;
                        }
                    }
                }
                tc_fence_before();
                __syncthreads();   // TMEM free for the next pass; Vn complete
            }
            // ---- convergence (Alg. 1 "until V^{t+1} == V^t") and slot refill
            if (active) {
                ++rl;
                bool changed = false;
                for (int w = 0; w < nw; ++w) changed |= (Vn[w * kTM + m] != V[w * kTM + m]);
                const bool cyc_stop = cyc_exit && rl >= 2 && cyc && changed;   // V^r == V^{r-2}
                uint32_t *t = V; V = Vn; Vn = t;                             // V^r is current
                if (!changed || rl == T || cyc_stop) {   // ---- a7 output
                    uint32_t *out = out_state + p * nw;
                    for (int w = 0; w < nw; ++w) out[w] = V[w * kTM + m];
                    out_iters[p] = (uint16_t)rl;
                    out_status[p] = (uint8_t)(!changed ? GB_CONVERGED : cyc_stop ? GB_CYCLE : GB_MAX_ITERS);
                    refill();
                }
            }
            cyc = true;
            __syncthreads();
        }
        __syncthreads();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// ---------------------------------------------------------------------------
// v2: warp-specialised, for n_p <= 1024 (the whole expanded A tile of a round
// fits in shared memory).  Warp 0 = TMA producer (W tiles, S-stage ring),
// warp 1 = MMA issuer (one elected lane) and TMEM owner, warps 2-5 = the 128
// epilogue threads (probe = TMEM lane).  TMEM holds two 256-column
// accumulators, so the epilogue of pass p overlaps the MMAs of pass p+1.
// gamma*V is folded into the B operand (W8 + gamma*I, built per gamma) when
// gamma <= 255, so the epilogue is max + compare only.
struct Sos2Params {
    int NP;          // columns per pass (whole clusters, <= 256)
    int BR;          // TMA box rows
    int S;           // B stages
    int gamma_epi;   // gamma added in the epilogue (0 when folded into B)
    int cyc;         // GB_FLAG_CYCLE_EXIT: stop a probe when V^r == V^{r-2}
    uint32_t a_off, b_off, v_off, bar_off, b_stage;
};


template <int WC>
__global__ void __launch_bounds__(192, 1)
sos_tc2_kernel(Shape s, const __grid_constant__ CUtensorMap wmap, Sos2Params P,
               const uint16_t *__restrict__ probes, int64_t k, int T, unsigned long long *queue,
               uint32_t *__restrict__ out_state, uint16_t *__restrict__ out_iters,
               uint8_t *__restrict__ out_status) {
    constexpr int LP = 32 * WC;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *gbase = smem_raw + (base - raw);
    const uint32_t A0 = base + P.a_off;     // nkb x (128 x 128 B), SW128
    const uint32_t B0 = base + P.b_off;     // S x (NP x 128 B), SW128
    uint32_t *Vs = reinterpret_cast<uint32_t *>(gbase + P.v_off);   // 2 x [nw][128]
    uint64_t *bars = reinterpret_cast<uint64_t *>(gbase + P.bar_off);
    // bars: full[0..S) empty[S..2S) tfull[2S..2S+2) tempty[2S+2..2S+4); then tmem slot
    const uint32_t bar0 = smem_u32(bars);
    const int S = P.S;
    auto full_bar = [&](int i) { return bar0 + 8u * i; };
    auto empty_bar = [&](int i) { return bar0 + 8u * (S + i); };
    auto tfull_bar = [&](int i) { return bar0 + 8u * (2 * S + i); };
    auto tempty_bar = [&](int i) { return bar0 + 8u * (2 * S + 2 + i); };
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * S + 4);

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const bool epi = warp >= 2;
    const int m = 32 * (warp & 3) + lane;            // probe row = TMEM lane (epilogue warps)
    const int nw = s.nw, np = s.np;
    const int nkb = (np + kKB - 1) / kKB;
    const int npass = (np + P.NP - 1) / P.NP;
    const bool narrow = P.gamma_epi + np < 0x7FFF;   // scores fit 15 bits (wta_words)

    if (tid == 0) {
        for (int i = 0; i < S; ++i) { mbar_init(full_bar(i), 1); mbar_init(empty_bar(i), 1); }
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

    uint32_t it_p = 0, it_m = 0, pc_m = 0, pc_e = 0;   // pipeline counters (per role)
    // Slot refill ("continuous batching", N4): each TMEM lane is a slot holding
    // one probe; when its probe converges or reaches max_iters its result is
    // written and the slot takes the next probe from a global queue, so no
    // slot idles while a straggler in the same tile keeps iterating.  Rounds
    // stay synchronous per probe; a probe's rounds are counted locally.
    // Per-thread double buffer: the slot's current state is in buffer `par`, the
    // epilogue writes the next state into buffer par^1 (no copy between rounds).
    uint32_t par = 0;
    uint32_t *V = Vs, *Vn = Vs + nw * kTM;
    int64_t p = -1, pn = -1;
    uint4 qn = make_uint4(0, 0, 0, 0);   // prefetched symbols of probe pn (C <= 8)
    const bool pack = s.C <= 8;
    int rl = 0;            // rounds run by the slot's current probe
    bool active = false;
    // words of A (this thread's row) that must be re-expanded before the next round;
    // A starts undefined, so every word of every K block is dirty
    uint32_t dirty = (nkb * 4 >= 32) ? 0xffffffffu : ((1u << (nkb * 4)) - 1u);
    uint32_t nzcur = 0u;   // words of the current state that are non-zero
    // next probe index from the global queue; for C <= 8 its symbols are
    // prefetched into registers so a later refill does not wait on memory
    auto fetch = [&]() {
        pn = (int64_t)atomicAdd(queue, 1ull);
        if (pack && pn < k) {
            uint32_t w4[4] = {0u, 0u, 0u, 0u};
            const uint16_t *pr = probes + pn * s.C;
#pragma unroll
            for (int c = 0; c < 8; ++c)
                if (c < s.C) w4[c >> 1] |= (uint32_t)__ldg(pr + c) << (16 * (c & 1));
            qn = make_uint4(w4[0], w4[1], w4[2], w4[3]);
        }
    };
    auto refill = [&]() {
        for (;;) {
            p = pn;
            const uint4 q = qn;
            fetch();
            uint32_t *Vc = Vs + par * nw * kTM;
            for (int w = 0; w < nw; ++w) Vc[w * kTM + m] = 0u;
            rl = 0;
            if (p >= k) { active = false; return; }
            auto sym_of = [&](int c) -> unsigned {
                if (pack) {
                    const uint32_t w = (c >> 1) == 0 ? q.x : (c >> 1) == 1 ? q.y : (c >> 1) == 2 ? q.z : q.w;
                    return (w >> (16 * (c & 1))) & 0xffffu;
                }
                return __ldg(probes + p * s.C + c);
            };
            bool valid = true;
            for (int c = 0; c < s.C; ++c) {
                const unsigned sym = sym_of(c);
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
                const unsigned sym = sym_of(c);
                if (sym != kErased) {
                    const int w = c * WC + (int)(sym >> 5);
                    Vc[w * kTM + m] = 1u << (sym & 31);
                    dirty |= 1u << w;   // A must pick up the new probe's one-hot words
                }
            }
            active = true;
            return;
        }
    };
    if (epi) fetch();
    if (epi) refill();
    for (;;) {
        if (!__syncthreads_or(epi && active)) break;
        V = Vs + par * nw * kTM;
        Vn = Vs + (par ^ 1u) * nw * kTM;
        bool changed = false;
        bool cyc = true;
        if (epi) {
            // A = V^T as bytes (128 x 128 B swizzled tile per K block), kept resident and
            // updated incrementally: only the state words that differ from what A holds
            // (dirty mask, n_p <= 1024 so at most 32 words) are re-expanded.
            uint32_t d = dirty;
            while (d) {
                const int w = __ffs(d) - 1;
                d &= d - 1u;
                const uint32_t wv = (w < nw) ? V[w * kTM + m] : 0u;
                uint8_t *arow = gbase + P.a_off + (w >> 2) * (kTM * kKB) + m * kKB;
#pragma unroll
                for (int h2 = 0; h2 < 2; ++h2) {
                    const int ch = 2 * (w & 3) + h2;
                    const uint32_t bits = (wv >> (h2 * 16)) & 0xffffu;
                    *reinterpret_cast<uint4 *>(arow + ((ch ^ (m & 7)) * 16)) =
                        make_uint4(spread4(bits & 15u), spread4((bits >> 4) & 15u),
                                   spread4((bits >> 8) & 15u), spread4(bits >> 12));
                }
            }
            dirty = 0u;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        __syncthreads();
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
                        const int st = it_m % S;
                        mbar_wait(full_bar(st), (it_m / S) & 1u);
                        tc_fence_after();
                        const uint32_t As = A0 + kb * (kTM * kKB), Bs = B0 + st * P.b_stage;
#pragma unroll
                        for (int ks = 0; ks < kKB / 32; ++ks)
                            umma_i8(tmem + buf * 256, sw128_desc(As + ks * 32), sw128_desc(Bs + ks * 32), idesc,
                                    (kb > 0 || ks > 0) ? 1u : 0u);
                        umma_commit(empty_bar(st));
                    }
                    umma_commit(tfull_bar(buf));
                }
            }
            __syncwarp();
        } else {
            // ---- epilogue: per-cluster max + mask of each pass (a4)
            const uint32_t tl = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
            for (int pass = 0; pass < npass; ++pass, ++pc_e) {
                const int n0 = pass * P.NP, ncols = min(P.NP, np - n0);
                const uint32_t buf = pc_e & 1u;
                mbar_wait(tfull_bar(buf), (pc_e >> 1) & 1u);
                tc_fence_after();
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
                                word |= ((v32[j] + (((vw >> j) & 1u) ? (uint32_t)P.gamma_epi : 0u)) == mx ? 1u : 0u) << j;
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
                mbar_arrive(tempty_bar(buf));
            }
            // ---- convergence (Alg. 1 "until V^{t+1} == V^t") and slot refill
            if (active) {
                ++rl;
                const bool cyc_stop = P.cyc && rl >= 2 && cyc && changed;   // V^r == V^{r-2}
                if (!changed || rl == T || cyc_stop) {   // ---- a7 output
                    uint32_t *out = out_state + p * nw;
                    for (int w = 0; w < nw; ++w) out[w] = Vn[w * kTM + m];
                    out_iters[p] = (uint16_t)rl;
                    out_status[p] = (uint8_t)(!changed ? GB_CONVERGED : cyc_stop ? GB_CYCLE : GB_MAX_ITERS);
                    // A still holds the expansion of the probe's state before this round
                    // (V); the new probe's V^0 goes into the same buffer
                    dirty |= nzcur;
                    refill();
                } else {
                    par ^= 1u;   // V^{r} becomes the current state
                }
            }
            nzcur = 0u;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

bool plan2(const Shape &s, int gamma, Sos2Params &P, size_t &smem) {
    if (s.Lp > 256 || s.np > 1024) return false;
    P.NP = s.Lp * (256 / s.Lp);
    if (P.NP > s.np) P.NP = s.np;
    int br = 256;
    while (br > 32 && s.Lp % br) br >>= 1;
    P.BR = br;
    P.gamma_epi = gamma > 255 ? gamma : 0;
    P.cyc = 0;
    const int nkb = (s.np + kKB - 1) / kKB;
    P.a_off = 0;
    P.b_off = (uint32_t)nkb * kTM * kKB;
    P.b_stage = (uint32_t)P.NP * kKB;
    const size_t vbytes = 2ull * s.nw * kTM * 4;
    for (P.S = 4; P.S >= 2; --P.S) {
        P.v_off = P.b_off + P.S * P.b_stage;
        P.bar_off = (uint32_t)(P.v_off + vbytes);
        smem = P.bar_off + 8 * (2 * P.S + 4) + 16 + 1024;
        if (smem <= 227 * 1024) return true;
    }
    return false;
}

// W8g = W8 + gamma*I on the real neurons (the B operand of sos_tc2_kernel).
__global__ void diag_kernel(Shape s, const uint8_t *__restrict__ w8, uint8_t *__restrict__ w8g, int gamma) {
    const int64_t n16 = (int64_t)s.np * s.np / 16;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x) {
        uint4 v = reinterpret_cast<const uint4 *>(w8)[i];
        const int64_t b0 = i * 16;
        const int64_t row = b0 / s.np, col0 = b0 - row * s.np;
        if (row >= col0 && row < col0 + 16 && (row % s.Lp) < s.L) {
            uint8_t *bytes = reinterpret_cast<uint8_t *>(&v);
            bytes[row - col0] = (uint8_t)gamma;
        }
        reinterpret_cast<uint4 *>(w8g)[i] = v;
    }
}

bool plan(const Shape &s, SosParams &P, size_t &smem) {
    if (s.Lp > 512 || s.np > 8192) return false;
    int br = 256;
    while (br > 32 && s.Lp % br) br >>= 1;
    P.BR = br;
    for (P.v_global = 0; P.v_global < 2; ++P.v_global) {
        P.NP = s.Lp * (512 / s.Lp);
        if (P.NP > s.np) P.NP = s.np;
        const size_t vbytes = P.v_global ? 0 : 2ull * s.nw * kTM * 4;
        for (;;) {
            P.b_stage = (uint32_t)P.NP * kKB;
            P.a_off = 0;
            P.b_off = 2 * kTM * kKB;
            P.v_off = P.b_off + 2 * P.b_stage;
            P.bar_off = (uint32_t)(P.v_off + vbytes);
            smem = P.bar_off + 64 + 1024;   // barriers, tmem slot, alignment slack
            if (smem <= 227 * 1024) return true;
            if (P.NP <= s.Lp) break;
            P.NP -= s.Lp;
        }
    }
    return false;
}

template <int WC>
cudaError_t launch_t(Call &cl, const uint16_t *probes, int64_t k, int gamma, int max_iters, int cyc,
                     uint32_t *state, uint16_t *iters, uint8_t *status) {
    const gb_net *net = cl.net;
    const cudaStream_t st = cl.st;
    SosParams P;
    size_t smem;
    if (!plan(net->s, P, smem)) return cudaErrorNotSupported;
    if (!net->wmap_ok) return cudaErrorNotSupported;
    auto fn = sos_tc_kernel<WC>;
    if (smem < 120 * 1024) smem = 120 * 1024;   // one CTA per SM: it owns all 512 TMEM columns
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t ntiles = (k + kTM - 1) / kTM;
    const int grid = (int)std::min<int64_t>(ntiles, net->sm_count);
    uint32_t *vscratch = nullptr;
    if (P.v_global) {
        vscratch = cl.alloc_n<uint32_t>((size_t)net->sm_count * 2 * net->s.nw * kTM);
        if (!vscratch) return cl.err;
    }
    unsigned long long *queue = cl.counters();
    if (!queue) return cl.err;
    fn<<<grid, kThreads, smem, st>>>(net->s, *reinterpret_cast<const CUtensorMap *>(net->wmap), P, probes, k,
                                     gamma, max_iters, cyc, queue, vscratch, state, iters, status);
    cl.launched();
    return cudaGetLastError();
}

}  // namespace

bool sos_tc_supported(const Shape &s) {
    SosParams P;
    size_t smem;
    if (s.Wc != 1 && s.Wc != 2 && s.Wc != 3 && s.Wc != 4 && s.Wc != 8 && s.Wc != 16) return false;
    return plan(s, P, smem);
}

// TMA descriptor of an n_p x n_p u8 matrix (row-major) at gaddr: box 128 B x box_rows rows,
// 128-byte swizzle.
bool sos_encode_map(const gb_net *net, void *gaddr, int box_rows, unsigned char *out) {
    void *fnp = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fnp) {
        cudaGetLastError();
        return false;
    }
    using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    const cuuint64_t dims[2] = {(cuuint64_t)net->s.np, (cuuint64_t)net->s.np};
    const cuuint64_t strides[1] = {(cuuint64_t)net->s.np};
    const cuuint32_t box[2] = {(cuuint32_t)kKB, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    alignas(64) CUtensorMap map;
    static_assert(sizeof(CUtensorMap) == 128, "CUtensorMap size");
    CUresult r = reinterpret_cast<EncodeFn>(fnp)(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, gaddr, dims, strides, box,
                                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    memcpy(out, &map, sizeof map);
    return r == CUDA_SUCCESS;
}

// TMA descriptor of W8 for the 4-warp kernel (box rows from plan).  Called at gb_create
// (W8's address never changes).
bool sos_tc_make_map(gb_net *net) {
    net->wmap_ok = false;
    SosParams P;
    size_t smem;
    if (!plan(net->s, P, smem)) return false;
    net->wmap_ok = sos_encode_map(net, net->w8, P.BR, net->wmap);
    return net->wmap_ok;
}

namespace {

template <int WC>
cudaError_t launch2_t(Call &cl, const void *map, const Sos2Params &P, size_t smem, const uint16_t *probes, int64_t k,
                      int max_iters, uint32_t *state, uint16_t *iters, uint8_t *status) {
    const gb_net *net = cl.net;
    auto fn = sos_tc2_kernel<WC>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t ntiles = (k + kTM - 1) / kTM;
    const int grid = (int)std::min<int64_t>(ntiles, net->sm_count);
    unsigned long long *queue = cl.counters();
    if (!queue) return cl.err;
    fn<<<grid, 192, smem, cl.st>>>(net->s, *reinterpret_cast<const CUtensorMap *>(map), P, probes, k,
                                   max_iters, queue, state, iters, status);
    cl.launched();
    return cudaGetLastError();
}

}  // namespace

bool sos_tc2_supported(const Shape &s) {
    Sos2Params P;
    size_t smem;
    if (s.Wc != 1 && s.Wc != 2 && s.Wc != 3 && s.Wc != 4 && s.Wc != 8) return false;
    return plan2(s, 1, P, smem);
}

// W8g = W8 + gamma*I, the B operand of the warp-specialised kernels: one variant per
// (seal generation, folded gamma), built by diag_kernel on the first call that needs it and
// shared by later calls on any stream (they wait on its `ready` event).  gamma > 255 is added
// in the epilogue instead (variant gfold = 0, B = W8 with a zero diagonal).  Concurrent
// decodes with different gammas get different variants; a fifth live gamma evicts the least
// recently used variant after a device synchronisation (a kernel may still read it).
cudaError_t gamma_operand(Call &cl, int gamma, int box_rows, const void **map) {
    gb_net *net = cl.net;
    const int gfold = gamma > 255 ? 0 : gamma;
    std::lock_guard<std::mutex> lk(net->gmu);
    GammaVariant *v = nullptr;
    for (auto &g : net->gvar)
        if (g.gfold == gfold && g.gen == net->seal_gen && g.w8g) v = &g;
    if (!v) {
        GammaVariant *stale = nullptr, *lru = nullptr;
        for (auto &g : net->gvar) {
            if (!g.w8g || g.gen != net->seal_gen) {
                if (!stale) stale = &g;
            } else if (!lru || g.last_use < lru->last_use) {
                lru = &g;
            }
        }
        v = stale ? stale : lru;
        if (!stale) {   // evicting a live variant: another stream may still read it
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) return e;
        }
        if (!v->w8g) {
            if (cudaMalloc(&v->w8g, (size_t)net->s.np * net->s.np) != cudaSuccess) {
                cudaGetLastError();
                v->w8g = nullptr;
                return cudaErrorMemoryAllocation;
            }
            if (cudaEventCreateWithFlags(&v->ready, cudaEventDisableTiming) != cudaSuccess) return cudaErrorUnknown;
            v->nmaps = 0;   // maps depend only on the (fixed) w8g address and box rows
        }
        v->gfold = gfold;
        v->gen = net->seal_gen;
        diag_kernel<<<net->sm_count * 4, 256, 0, cl.st>>>(net->s, net->w8, v->w8g, gfold);
        cl.launched();
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        e = cudaEventRecord(v->ready, cl.st);
        if (e != cudaSuccess) return e;
    } else {
        cudaError_t e = cudaStreamWaitEvent(cl.st, v->ready, 0);   // built on another call's stream
        if (e != cudaSuccess) return e;
    }
    v->last_use = ++net->guse;
    int mi = -1;
    for (int i = 0; i < v->nmaps; ++i)
        if (v->map_rows[i] == box_rows) mi = i;
    if (mi < 0) {
        if (v->nmaps == 4) return cudaErrorNotSupported;
        mi = v->nmaps;
        if (!sos_encode_map(net, v->w8g, box_rows, v->maps[mi])) return cudaErrorNotSupported;
        v->map_rows[mi] = box_rows;
        v->nmaps += 1;
    }
    *map = v->maps[mi];
    return cudaSuccess;
}

cudaError_t launch_sos_pair_list(Call &cl, const uint16_t *probes, int64_t k, const int64_t *list,
                                 const unsigned long long *count, int gamma, int max_iters, uint32_t *state,
                                 uint16_t *iters, uint8_t *status) {
    const gb_net *net = cl.net;
    Sos2Params P2;
    size_t smem2;
    if (sos_tc3_enabled(net) || !plan2(net->s, gamma, P2, smem2) || !sos_2cta_enabled(net))
        return cudaErrorNotSupported;
    const void *map = nullptr;
    cudaError_t e = gamma_operand(cl, gamma, sos_2cta_box_rows(net->s), &map);
    if (e != cudaSuccess) return e;
    return launch_sos_2cta(cl, map, gamma > 255 ? gamma : 0, 0, probes, k, max_iters, state, iters, status, list,
                           count);
}

cudaError_t launch_decode_sos_tc(Call &cl, const uint16_t *probes, int64_t k, int gamma, int max_iters,
                                 int cyc, uint32_t *state, uint16_t *iters, uint8_t *status) {
    const gb_net *net = cl.net;
    Sos2Params P2;
    size_t smem2;
    if (sos_tc3_enabled(net)) {   // 1024 < n_p <= 4096: streamed A tile
        alignas(8) unsigned char pb[64];
        size_t smem3;
        if (!plan3(net, gamma, pb, smem3)) return cudaErrorNotSupported;
        const void *map = nullptr;
        cudaError_t e = gamma_operand(cl, gamma, plan3_box_rows(pb), &map);
        if (e != cudaSuccess) return e;
        return launch_sos_tc3(cl, gamma, cyc, map, probes, k, max_iters, state, iters, status);
    }
    if (plan2(net->s, gamma, P2, smem2) &&
        (net->s.Wc == 1 || net->s.Wc == 2 || net->s.Wc == 3 || net->s.Wc == 4 || net->s.Wc == 8)) {
        P2.cyc = cyc;
        const void *map = nullptr;
        if (sos_2cta_enabled(net)) {
            cudaError_t e = gamma_operand(cl, gamma, sos_2cta_box_rows(net->s), &map);
            if (e != cudaSuccess) return e;
            return launch_sos_2cta(cl, map, gamma > 255 ? gamma : 0, cyc, probes, k, max_iters, state, iters, status);
        }
        cudaError_t e = gamma_operand(cl, gamma, P2.BR, &map);
        if (e != cudaSuccess) return e;
        if (smem2 < 120 * 1024) smem2 = 120 * 1024;   // one CTA per SM (512 TMEM columns)
        switch (net->s.Wc) {
            case 1: return launch2_t<1>(cl, map, P2, smem2, probes, k, max_iters, state, iters, status);
            case 2: return launch2_t<2>(cl, map, P2, smem2, probes, k, max_iters, state, iters, status);
            case 3: return launch2_t<3>(cl, map, P2, smem2, probes, k, max_iters, state, iters, status);
            case 4: return launch2_t<4>(cl, map, P2, smem2, probes, k, max_iters, state, iters, status);
            default: return launch2_t<8>(cl, map, P2, smem2, probes, k, max_iters, state, iters, status);
        }
    }
    switch (net->s.Wc) {
        case 1: return launch_t<1>(cl, probes, k, gamma, max_iters, cyc, state, iters, status);
        case 2: return launch_t<2>(cl, probes, k, gamma, max_iters, cyc, state, iters, status);
        case 3: return launch_t<3>(cl, probes, k, gamma, max_iters, cyc, state, iters, status);
        case 4: return launch_t<4>(cl, probes, k, gamma, max_iters, cyc, state, iters, status);
        case 8: return launch_t<8>(cl, probes, k, gamma, max_iters, cyc, state, iters, status);
        case 16: return launch_t<16>(cl, probes, k, gamma, max_iters, cyc, state, iters, status);
        default: return cudaErrorNotSupported;
    }
}

}  // namespace gb
