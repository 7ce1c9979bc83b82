// gb_decode_som_tc.cu -- exact sum-of-max on the tensor cores (SURVEY.md §8.f
// N2; the paper's future work "emulate sum-of-max using sum-of-sum",
// PAPER.md L855, L862-901).
//
// Eq.(6)-(7) (L259-264): s_i = gamma v_i + sum_{c' != c(i)} max_{l'} v_{c'l'} w_{(c'l'),i}
// and v'_i = [s_i = gamma + C - 1].  The max over a source cluster of 0/1
// products is the test "count_{c'}(i) > 0" with the integer count
//     count_{c'}(i) = sum_{l'} v_{c'l'} w_{(c'l'),i}
// -- a sum-of-sum restricted to the K range of cluster c'.  So one round is C
// exact int8 contractions, one per source cluster, each into its own int32
// TMEM accumulator (the paper's Omega/theta emulation packs them into one
// floating-point number and needs >= 57-bit integers, L895; separate
// accumulators make it exact at any size):
//     D_{c'}[probe, i] = sum_{j in c'} V[probe, j] W[j, i]      (tcgen05.mma.kind::i8)
//     v'_i = v_i AND #{c' : D_{c'}[probe, i] > 0} == C - 1
// (for gamma > 0; own-cluster counts are 0 since W has no intra-cluster edge,
// and every gamma > 0 gives the same rule, Thm 1).  Initial state: erased
// clusters all 1, known one-hot (L270-271); synchronous rounds; convergence,
// rounds and status exactly as the bit kernels (readings R5, R6, R14).
//
// Tile: 128 probes (UMMA M = 128, TMEM lane = probe), V^T resident in shared
// memory as the A operand (n_p <= 1024, updated incrementally like
// sos_tc2_kernel), W8 rows by TMA (B operand).  TMEM holds C accumulators of
// NP = 512 / C columns, so a pass covers NP target neurons; warp 0 = TMA,
// warp 1 = MMA issuer, warps 2-5 = epilogue (hit counts, mask, convergence,
// slot refill).  Selected with GB_SOM_TC=1 (the bit kernels stay the default:
// DESIGN.md §9 N2 has the measured comparison).
#include <cuda.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include "gb_internal.h"
#include "gb_tc_common.cuh"

namespace gb {
namespace {
using namespace tc;

struct SomParams {
    int NP;   // target columns per pass (512 / C, multiple of 32)
    int S;    // B stages
    uint32_t a_off, b_off, v_off, bar_off, b_stage;
};

template <int WC>
__global__ void __launch_bounds__(192, 1)
som_tc_kernel(Shape s, const __grid_constant__ CUtensorMap wmap, SomParams P, const uint16_t *__restrict__ probes,
              int64_t k, int T, unsigned long long *queue, uint32_t *__restrict__ out_state,
              uint16_t *__restrict__ out_iters, uint8_t *__restrict__ out_status) {
    constexpr int LP = 32 * WC;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *gbase = smem_raw + (base - raw);
    const uint32_t A0 = base + P.a_off;   // nkb x (128 x 128 B), SW128
    const uint32_t B0 = base + P.b_off;   // S x (NP x 128 B), SW128
    uint32_t *Vs = reinterpret_cast<uint32_t *>(gbase + P.v_off);   // 2 x [nw][128]
    uint64_t *bars = reinterpret_cast<uint64_t *>(gbase + P.bar_off);
    const uint32_t bar0 = smem_u32(bars);
    const int S = P.S;
    auto full_bar = [&](int i) { return bar0 + 8u * i; };
    auto empty_bar = [&](int i) { return bar0 + 8u * (S + i); };
    const uint32_t tfull = bar0 + 8u * (2 * S), tempty = bar0 + 8u * (2 * S + 1);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * S + 2);

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const bool epi = warp >= 2;
    const int m = 32 * (warp & 3) + lane;
    const int C = s.C, nw = s.nw, np = s.np;
    const int nkb = (np + kKB - 1) / kKB;
    const int nsteps = np / 32;                 // K steps of 32 (np is a multiple of 32)
    const int npass = (np + P.NP - 1) / P.NP;

    if (tid == 0) {
        for (int i = 0; i < S; ++i) { mbar_init(full_bar(i), 1); mbar_init(empty_bar(i), 1); }
        mbar_init(tfull, 1);
        mbar_init(tempty, 128);
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

    uint32_t it_p = 0, it_m = 0, pc_m = 0, pc_e = 0;
    uint32_t par = 0;
    uint32_t *V = Vs, *Vn = Vs + nw * kTM;
    int64_t p = -1;
    int rl = 0;
    bool active = false;
    uint32_t dirty = (nkb * 4 >= 32) ? 0xffffffffu : ((1u << (nkb * 4)) - 1u);
    auto refill = [&]() {
        for (;;) {
            p = (int64_t)atomicAdd(queue, 1ull);
            uint32_t *Vc = Vs + par * nw * kTM;
            rl = 0;
            if (p >= k) {
                for (int w = 0; w < nw; ++w) Vc[w * kTM + m] = 0u;
                dirty = 0xffffffffu;
                active = false;
                return;
            }
            bool valid = true;
            for (int c = 0; c < C; ++c) {
                const unsigned sym = __ldg(probes + p * C + c);
                if (sym != kErased && sym >= (unsigned)s.L) valid = false;
            }
            if (!valid) {   // GB_INVALID: zero state, 0 rounds; take another probe
                uint32_t *out = out_state + p * nw;
                for (int w = 0; w < nw; ++w) out[w] = 0u;
                out_iters[p] = 0;
                out_status[p] = GB_INVALID;
                continue;
            }
            // ---- a1 ingest (SOM): erased clusters all 1, known one-hot
            for (int c = 0; c < C; ++c) {
                const unsigned sym = __ldg(probes + p * C + c);
#pragma unroll
                for (int u = 0; u < WC; ++u) {
                    uint32_t x;
                    if (sym == kErased) x = real_mask(s.L, u);
                    else x = ((int)(sym >> 5) == u) ? (1u << (sym & 31)) : 0u;
                    Vc[(c * WC + u) * kTM + m] = x;
                }
            }
            dirty = 0xffffffffu;
            active = true;
            return;
        }
    };
    if (epi) refill();
    for (;;) {
        if (!__syncthreads_or(epi && active)) break;
        V = Vs + par * nw * kTM;
        Vn = Vs + (par ^ 1u) * nw * kTM;
        bool changed = false;
        if (epi) {   // A = V^T as bytes (SW128 tiles), re-expanded where the state changed
            uint32_t d = dirty & ((nw >= 32) ? 0xffffffffu : ((1u << nw) - 1u));
            while (d) {
                const int w = __ffs(d) - 1;
                d &= d - 1u;
                const uint32_t wv = V[w * kTM + m];
                uint8_t *arow = gbase + P.a_off + (w >> 2) * (kTM * kKB) + m * kKB;
#pragma unroll
                for (int h2 = 0; h2 < 2; ++h2) {
                    const int ch = 2 * (w & 3) + h2;
                    const uint32_t bits = (wv >> (h2 * 16)) & 0xffffu;
                    *reinterpret_cast<uint4 *>(arow + ((ch ^ (m & 7)) * 16)) =
                        make_uint4(spread4(bits & 15u), spread4((bits >> 4) & 15u), spread4((bits >> 8) & 15u),
                                   spread4(bits >> 12));
                }
            }
            if (dirty == 0xffffffffu) {   // words beyond nw inside the last K block: zero
                for (int w = nw; w < nkb * 4; ++w) {
                    uint8_t *arow = gbase + P.a_off + (w >> 2) * (kTM * kKB) + m * kKB;
#pragma unroll
                    for (int h2 = 0; h2 < 2; ++h2)
                        *reinterpret_cast<uint4 *>(arow + (((2 * (w & 3) + h2) ^ (m & 7)) * 16)) = make_uint4(0, 0, 0, 0);
                }
            }
            dirty = 0u;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        __syncthreads();
        if (warp == 0) {
            if (lane == 0) {   // ---- TMA producer: W rows [n0, n0 + ncols) of each pass, K block by K block
                for (int pass = 0; pass < npass; ++pass) {
                    const int n0 = pass * P.NP;
                    for (int kb = 0; kb < nkb; ++kb, ++it_p) {
                        const int st = it_p % S;
                        mbar_wait(empty_bar(st), ((it_p / S) & 1u) ^ 1u);
                        // the box is always NP rows (rows past n_p are zero-filled and counted)
                        mbar_expect_tx(full_bar(st), (uint32_t)P.NP * kKB);
                        tma_load_2d(B0 + st * P.b_stage, &wmap, full_bar(st), kb * kKB, n0);
                    }
                }
            }
            __syncwarp();
        } else if (warp == 1) {
            if (lane == 0) {   // ---- MMA issuer: K step j (32 source neurons) goes to accumulator c' = 32 j / Lp
                for (int pass = 0; pass < npass; ++pass, ++pc_m) {
                    const int n0 = pass * P.NP, ncols = min(P.NP, np - n0);
                    mbar_wait(tempty, (pc_m & 1u) ^ 1u);
                    tc_fence_after();
                    const uint32_t idesc = i8_idesc(ncols);
                    for (int kb = 0; kb < nkb; ++kb, ++it_m) {
                        const int st = it_m % S;
                        mbar_wait(full_bar(st), (it_m / S) & 1u);
                        tc_fence_after();
                        const uint32_t As = A0 + kb * (kTM * kKB), Bs = B0 + st * P.b_stage;
#pragma unroll
                        for (int ks = 0; ks < kKB / 32; ++ks) {
                            const int step = kb * 4 + ks;
                            if (step < nsteps) {
                                const int c2 = (step * 32) / LP;
                                const uint32_t first = ((step * 32) % LP) == 0;
                                umma_i8(tmem + (uint32_t)(c2 * P.NP), sw128_desc(As + ks * 32),
                                        sw128_desc(Bs + ks * 32), idesc, first ? 0u : 1u);
                            }
                        }
                        umma_commit(empty_bar(st));
                    }
                    umma_commit(tfull);
                }
            }
            __syncwarp();
        } else {
            // ---- epilogue: hit counts over the source clusters, Eq.(7) mask (a6)
            const uint32_t tl = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
            for (int pass = 0; pass < npass; ++pass, ++pc_e) {
                const int n0 = pass * P.NP, ncols = min(P.NP, np - n0);
                mbar_wait(tfull, pc_e & 1u);
                tc_fence_after();
                for (int g = 0; g < ncols / 32; ++g) {
                    uint32_t cnt[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) cnt[j] = 0u;
                    for (int c2 = 0; c2 < C; ++c2) {
                        uint32_t v32[32];
                        tmem_ld32(tl + (uint32_t)(c2 * P.NP + 32 * g), v32);
#pragma unroll
                        for (int j = 0; j < 32; ++j) cnt[j] += v32[j] ? 1u : 0u;
                    }
                    const int w = (n0 >> 5) + g;          // state word of target neurons n0 + 32 g + j
                    const uint32_t vw = V[w * kTM + m];
                    uint32_t word = 0u;
#pragma unroll
                    for (int j = 0; j < 32; ++j) word |= (cnt[j] == (uint32_t)(C - 1) ? 1u : 0u) << j;
                    word &= vw;   // v_i = 1 and C - 1 hits <=> s_i = gamma + C - 1 (gamma > 0)
                    if (word != vw) { changed = true; dirty |= 1u << w; }
                    Vn[w * kTM + m] = word;
                }
                tc_fence_before();
                mbar_arrive(tempty);
            }
            if (active) {   // convergence, output, slot refill
                ++rl;
                if (!changed || rl == T) {
                    uint32_t *out = out_state + p * nw;
                    for (int w = 0; w < nw; ++w) out[w] = Vn[w * kTM + m];
                    out_iters[p] = (uint16_t)rl;
                    out_status[p] = (uint8_t)(changed ? GB_MAX_ITERS : GB_CONVERGED);
                    refill();
                } else {
                    par ^= 1u;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

bool plan_som(const Shape &s, SomParams &P, size_t &smem) {
    if (s.np > 1024 || s.C > 16) return false;
    if (s.Wc != 1 && s.Wc != 2 && s.Wc != 4 && s.Wc != 8) return false;
    P.NP = std::min(256, (512 / s.C) & ~31);
    if (P.NP > s.np) P.NP = s.np;
    if (P.NP < 32) return false;
    const int nkb = (s.np + kKB - 1) / kKB;
    P.a_off = 0;
    P.b_off = (uint32_t)nkb * kTM * kKB;
    P.b_stage = ((uint32_t)P.NP * kKB + 1023u) & ~1023u;
    const size_t vbytes = 2ull * s.nw * kTM * 4;
    for (P.S = 6; P.S >= 2; --P.S) {
        P.v_off = P.b_off + P.S * P.b_stage;
        P.bar_off = (uint32_t)(P.v_off + vbytes);
        smem = P.bar_off + 8 * (2 * P.S + 2) + 16 + 1024;
        if (smem <= 227 * 1024) return true;
    }
    return false;
}

template <int WC>
cudaError_t launch_som_t(Call &cl, const SomParams &P, size_t smem, const uint16_t *probes, int64_t k,
                         int max_iters, uint32_t *state, uint16_t *iters, uint8_t *status) {
    gb_net *net = cl.net;
    const cudaStream_t st = cl.st;
    auto fn = som_tc_kernel<WC>;
    if (smem < 120 * 1024) smem = 120 * 1024;   // one CTA per SM: it owns all 512 TMEM columns
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t ntiles = (k + kTM - 1) / kTM;
    const int grid = (int)std::min<int64_t>(ntiles, net->sm_count);
    unsigned long long *queue = cl.counters();
    if (!queue) return cl.err;
    fn<<<grid, 192, smem, st>>>(net->s, *reinterpret_cast<const CUtensorMap *>(net->wmap_som), P, probes, k,
                                max_iters, queue, state, iters, status);
    cl.launched();
    return cudaGetLastError();
}

}  // namespace

bool som_tc_enabled(const gb_net *net) {
    if (net->opt[kOptSomTensor].load(std::memory_order_relaxed) != 1) return false;
    SomParams P;
    size_t smem;
    return plan_som(net->s, P, smem);
}

cudaError_t launch_som_tc(Call &cl, const uint16_t *probes, int64_t k, int max_iters, uint32_t *state,
                          uint16_t *iters, uint8_t *status) {
    gb_net *net = cl.net;
    SomParams P;
    size_t smem;
    if (!plan_som(net->s, P, smem)) return cudaErrorNotSupported;
    {
        std::lock_guard<std::mutex> lk(net->som_mu);
        if (!net->wmap_som_ok) {   // W8 (no gamma: the rule only tests counts > 0), box = NP rows
            net->wmap_som_ok = sos_encode_map(net, net->w8, P.NP, net->wmap_som);
            if (!net->wmap_som_ok) return cudaErrorNotSupported;
        }
    }
    switch (net->s.Wc) {
        case 1: return launch_som_t<1>(cl, P, smem, probes, k, max_iters, state, iters, status);
        case 2: return launch_som_t<2>(cl, P, smem, probes, k, max_iters, state, iters, status);
        case 4: return launch_som_t<4>(cl, P, smem, probes, k, max_iters, state, iters, status);
        default: return launch_som_t<8>(cl, P, smem, probes, k, max_iters, state, iters, status);
    }
}

}  // namespace gb
