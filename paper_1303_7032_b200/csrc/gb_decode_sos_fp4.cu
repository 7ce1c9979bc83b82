// gb_decode_sos_fp4.cu -- sum-of-sum on the block-scaled FP4 tensor cores
// (tcgen05.mma.kind::mxf4), n_padded <= 1024, Lp <= 128.
//
// Same method, roles and per-probe semantics as sos_tc2_kernel
// (gb_decode_sos_tc.cu): a3 S^t = W V^t + gamma V^t (Eq.(3),
// Eq.(10)-(11) L328/L349, Alg. 1 line 4), a4 per-cluster winner-take-all with
// ties kept (Eq.(4)-(5), readings R3/R4), per-probe convergence / max_iters,
// slot refill, opt-in period-2 exit.  Only the number format of the exact
// contraction differs: V and W are 0/1 and gamma in {0, 1, 2, 3, 4, 6} is an
// e2m1 value, so with unit E8M0 block scales every product is exact and the
// fp32 sums (<= n_p + gamma < 2^24) are exact integers -- the same S as the
// int8 kernels, at twice their per-SM rate (tools/mb/mxf4_probe.cu: exact,
// 20.4k vs 10.3k ops/clk at M = N = 128) and with half the operand bytes.
//
// Layout: A = V^T as e2m1 (1.0 = 0x2; two per byte, element 2i in the low
// nibble), 256 neurons per 128-byte K block, SW128, resident and updated
// incrementally; B = W4 = W8 + gamma*I as e2m1 (built by w4_kernel per seal /
// gamma); TMEM: two 128-column fp32 accumulators (one cluster of Lp = 128 per
// pass) and the unit scale factors in columns 256..271.
#include <cuda.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include "gb_internal.h"
#include "gb_tc_common.cuh"

namespace gb {
namespace {
using namespace tc;

struct Fp4Params {
    int NP;    // columns per pass (whole clusters, 128)
    int BR;    // TMA box rows
    int S;     // B stages
    int gamma_epi;   // always 0: gamma is folded into W4
    int cyc;   // GB_FLAG_CYCLE_EXIT
    uint32_t a_off, b_off, v_off, bar_off, b_stage;
};

// 8 state bits -> 8 e2m1 nibbles of value 1.0 (0x2) or 0, bit i at nibble i
__device__ __forceinline__ uint32_t nib8(uint32_t x) {
    x &= 0xFFu;
    x = (x | (x << 12)) & 0x000F000Fu;
    x = (x | (x << 6)) & 0x03030303u;
    x = (x | (x << 3)) & 0x11111111u;
    return x << 1;
}

__device__ __forceinline__ void umma_mxf4(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accum, uint32_t sfa, uint32_t sfb) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum), "r"(sfa), "r"(sfb));
}

template <int WC>
__global__ void __launch_bounds__(192, 1)
sos_fp4_kernel(Shape s, const __grid_constant__ CUtensorMap wmap, Fp4Params P,
               const uint16_t *__restrict__ probes, int64_t k, int T, unsigned long long *queue,
               uint32_t *__restrict__ out_state, uint16_t *__restrict__ out_iters,
               uint8_t *__restrict__ out_status) {
    constexpr int LP = 32 * WC;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *gbase = smem_raw + (base - raw);
    const uint32_t A0 = base + P.a_off;     // nkb x (128 x 128 B), SW128, two e2m1 per byte
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
    constexpr uint32_t kSfCol = 256;       // unit scale factors (E8M0 1.0) of A and B: TMEM columns 256..271

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const bool epi = warp >= 2;
    const int m = 32 * (warp & 3) + lane;            // probe row = TMEM lane (epilogue warps)
    const int nw = s.nw, np = s.np;
    const int nkb = (np + 255) / 256;               // K blocks of 256 neurons (128 bytes of e2m1)
    const int npass = (np + P.NP - 1) / P.NP;
    // fp32 accumulators: exact non-negative integers, so their bit patterns order like the
    // values and the 32-bit compares of wta_words apply unchanged (no 16-bit packing)
    const bool narrow = false;

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
    if (epi) {   // unit block scales (E8M0 0x7F = 2^0) for every lane in columns kSfCol .. kSfCol + 15
        const uint32_t ta = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + kSfCol;
        const uint32_t one = 0x7F7F7F7Fu;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};"
                     ::"r"(ta), "r"(one) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

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
    uint32_t dirty = (nkb * 8 >= 32) ? 0xffffffffu : ((1u << (nkb * 8)) - 1u);
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
                // 32 state bits -> 32 e2m1 nibbles (1.0 = 0x2), element 2i in the low nibble of byte i
                uint8_t *arow = gbase + P.a_off + (w >> 3) * (kTM * 128) + m * 128;
                *reinterpret_cast<uint4 *>(arow + (((w & 7) ^ (m & 7)) * 16)) =
                    make_uint4(nib8(wv), nib8(wv >> 8), nib8(wv >> 16), nib8(wv >> 24));
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
                        // one box of NP rows (rows past n_p are zero-filled and still counted)
                        mbar_expect_tx(full_bar(st), (uint32_t)P.NP * 128);
                        const uint32_t Bs = B0 + st * P.b_stage;
                        tma_load_2d(Bs, &wmap, full_bar(st), kb * 128, n0);
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
                    // kind::mxf4 descriptor: A/B E2M1 (MXF4 format 1), scales E8M0, M = 128, N = ncols, K = 64
                    const uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(ncols >> 3) << 17) | (1u << 23) |
                                           ((uint32_t)(kTM >> 4) << 24);
                    for (int kb = 0; kb < nkb; ++kb, ++it_m) {
                        const int st = it_m % S;
                        mbar_wait(full_bar(st), (it_m / S) & 1u);
                        tc_fence_after();
                        const uint32_t As = A0 + kb * (kTM * 128), Bs = B0 + st * P.b_stage;
#pragma unroll
                        for (int ks = 0; ks < 4; ++ks)   // 4 x 64 e2m1 = 128 bytes
                            umma_mxf4(tmem + buf * P.NP, sw128_desc(As + ks * 32), sw128_desc(Bs + ks * 32), idesc,
                                      (kb > 0 || ks > 0) ? 1u : 0u, tmem + kSfCol, tmem + kSfCol + 8);
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
                    const uint32_t col = buf * (uint32_t)P.NP + (uint32_t)(c * LP - n0);
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


// e2m1 code of gamma (0, 1, 2, 3, 4, 6 are exact), -1 otherwise
int e2m1_code(int g) {
    switch (g) {
        case 0: return 0x0;
        case 1: return 0x2;
        case 2: return 0x4;
        case 3: return 0x5;
        case 4: return 0x6;
        case 6: return 0x7;
        default: return -1;
    }
}

// W4 = W8 + gamma*I on the real neurons, two e2m1 per byte (column 2i in the low nibble).
// One thread per 16 output bytes (32 columns).
__global__ void w4_kernel(Shape s, const uint8_t *__restrict__ w8, uint8_t *__restrict__ w4, int gcode) {
    const int64_t n32 = (int64_t)s.np * s.np / 32;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n32; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b0 = i * 32;
        const int64_t row = b0 / s.np, col0 = b0 - row * s.np;
        const uint4 lo = reinterpret_cast<const uint4 *>(w8)[2 * i];
        const uint4 hi = reinterpret_cast<const uint4 *>(w8)[2 * i + 1];
        const uint32_t src[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
        uint32_t out[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            uint32_t v = ((src[j >> 2] >> (8 * (j & 3))) & 0xffu) ? 0x2u : 0x0u;
            if (row == col0 + j && (row % s.Lp) < s.L) v = (uint32_t)gcode;
            out[j >> 3] |= v << (4 * (j & 7));
        }
        reinterpret_cast<uint4 *>(w4)[i] = make_uint4(out[0], out[1], out[2], out[3]);
    }
}

bool plan_fp4(const Shape &s, int gamma, Fp4Params &P, size_t &smem) {
    if (s.np > 1024 || s.Lp > 128 || e2m1_code(gamma) < 0) return false;
    if (s.Wc != 1 && s.Wc != 2 && s.Wc != 4) return false;
    P.NP = std::min(128, s.np);
    P.BR = P.NP;
    P.gamma_epi = 0;
    P.cyc = 0;
    const int nkb = (s.np + 255) / 256;
    P.a_off = 0;
    P.b_off = (uint32_t)nkb * kTM * 128;
    P.b_stage = ((uint32_t)P.NP * 128 + 1023u) & ~1023u;
    const size_t vbytes = 2ull * s.nw * kTM * 4;
    for (P.S = 8; P.S >= 2; --P.S) {
        P.v_off = P.b_off + P.S * P.b_stage;
        P.bar_off = (uint32_t)(P.v_off + vbytes);
        smem = P.bar_off + 8 * (2 * P.S + 4) + 16 + 1024;
        if (smem <= 227 * 1024) return true;
    }
    return false;
}

// Tensor map of W4 (n_p rows of n_p/2 bytes): box 128 B x BR rows, 128-byte swizzle.
bool encode_w4_map(gb_net *net, int box_rows) {
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
    const cuuint64_t dims[2] = {(cuuint64_t)net->s.np / 2, (cuuint64_t)net->s.np};
    const cuuint64_t strides[1] = {(cuuint64_t)net->s.np / 2};
    const cuuint32_t box[2] = {128, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    alignas(64) CUtensorMap map;
    const CUresult r = reinterpret_cast<EncodeFn>(fnp)(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, net->w4, dims, strides,
                                                       box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                                       CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    memcpy(net->w4map, &map, sizeof map);
    return r == CUDA_SUCCESS;
}

template <int WC>
cudaError_t launch_fp4_t(gb_net *net, const Fp4Params &P, size_t smem, const uint16_t *probes, int64_t k,
                         int max_iters, uint32_t *state, uint16_t *iters, uint8_t *status, cudaStream_t st) {
    auto fn = sos_fp4_kernel<WC>;
    if (smem < 120 * 1024) smem = 120 * 1024;   // one CTA per SM (512 TMEM columns)
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t ntiles = (k + kTM - 1) / kTM;
    const int grid = (int)std::min<int64_t>(ntiles, net->sm_count);
    e = cudaMemsetAsync(net->queue, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    fn<<<grid, 192, smem, st>>>(net->s, *reinterpret_cast<const CUtensorMap *>(net->w4map), P, probes, k, max_iters,
                                net->queue, state, iters, status);
    net->launches += 1;
    return cudaGetLastError();
}

}  // namespace

bool sos_fp4_enabled(const Shape &s, int gamma) {
    const char *env = getenv("GB_SOS_FP4");
    if (!env || env[0] != '1') return false;
    Fp4Params P;
    size_t smem;
    return plan_fp4(s, gamma, P, smem);
}

cudaError_t launch_sos_fp4(gb_net *net, int gamma, int cyc, const uint16_t *probes, int64_t k, int max_iters,
                           uint32_t *state, uint16_t *iters, uint8_t *status, cudaStream_t st) {
    Fp4Params P;
    size_t smem;
    if (!plan_fp4(net->s, gamma, P, smem)) return cudaErrorNotSupported;
    P.cyc = cyc;
    if (!net->w4) {
        if (cudaMalloc(&net->w4, (size_t)net->s.np * net->s.np / 2) != cudaSuccess) {
            cudaGetLastError();
            net->w4 = nullptr;
            return cudaErrorMemoryAllocation;
        }
        if (!encode_w4_map(net, P.BR)) return cudaErrorNotSupported;
        net->w4_gen = ~0ull;
    }
    if (net->w4_gen != net->seal_gen || net->w4_gamma != gamma) {
        w4_kernel<<<net->sm_count * 4, 256, 0, st>>>(net->s, net->w8, net->w4, e2m1_code(gamma));
        net->launches += 1;
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        net->w4_gen = net->seal_gen;
        net->w4_gamma = gamma;
    }
    switch (net->s.Wc) {
        case 1: return launch_fp4_t<1>(net, P, smem, probes, k, max_iters, state, iters, status, st);
        case 2: return launch_fp4_t<2>(net, P, smem, probes, k, max_iters, state, iters, status, st);
        default: return launch_fp4_t<4>(net, P, smem, probes, k, max_iters, state, iters, status, st);
    }
}

}  // namespace gb
