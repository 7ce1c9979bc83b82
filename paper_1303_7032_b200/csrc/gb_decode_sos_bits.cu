// gb_decode_sos_bits.cu -- sum-of-sum decode on the CUDA cores for sparse states.
//
// Same method and per-probe semantics as the tensor-core SOS kernels
// (gb_decode_sos_tc.cu): a3 S^t = W V^t + gamma V^t (Eq.(3),
// Eq.(10)-(11) L328/L349, Alg. 1 line 4), a4 per-cluster winner-take-all with
// all ties kept and "max 0 activates the whole cluster" (Eq.(4)-(5) L220-225,
// readings R3/R4), per-probe convergence V^{t+1} == V^t or max_iters
// (Alg. 1), slot refill.  What differs is how S is formed: V^0 holds
// only the C - e known one-hots and, at low W density, a round keeps
// only a few neurons per cluster, so S is the sum of a handful of bit rows
// instead of a dense n_p x n_p contraction.
//
//  * one thread per probe (persistent, a work queue refills a lane whose probe
//    finished: every lane runs one round of its own probe per loop trip);
//  * W bit rows resident in shared memory (n_padded <= 1024: <= 128 KiB);
//  * a round lists the active neurons' row offsets (call-private shared memory,
//    [entry][thread]), then for every target cluster adds the listed rows'
//    blocks into bit-sliced counters -- plane b holds bit b of the score of
//    each of the cluster's neurons, one word per 32 neurons -- seeded with
//    gamma * v, and takes the winner-take-all plane by plane from the top
//    (cand &= plane when that leaves a neuron: the maximizers, ties kept;
//    all planes 0 leaves every real neuron, R4);
//  * the counters get enough planes for the round's largest possible score
//    (active neurons + gamma): 4 or 6, chosen per lane and round; two target
//    clusters share one pass over the list, and a cluster's new state words
//    replace the old ones as soon as it is scored (the list already holds the
//    round's sources; v_t only feeds target t's gamma term);
//  * lane q visits the target clusters in the order (c + q) mod C, so at C = 8
//    the 8 lanes of a quarter-warp read 8 different 16-byte blocks of their
//    rows (row-major: block t is chunk t of a 128-byte row) -- no bank conflicts;
//  * a probe whose active set outgrows the list or 6 planes (more than 32
//    active neurons, or a score that could reach 64 -- e.g. a cluster whose max
//    was 0 turned whole, R4) is queued and decoded from the start by
//    decode_generic_kernel in list mode (rare at the densities this kernel is
//    chosen for; exact either way).
// Scores are exact integers, so the state, rounds and status equal the
// oracle's bit for bit.
#include <stdlib.h>

#include <type_traits>

#include "gb_internal.h"

namespace gb {
namespace {

constexpr int kNTb = 512;      // threads per CTA (one probe each)
constexpr int kList = 32;      // active-neuron list entries per thread

// Two target clusters (one pass over the list; their row blocks load together):
// S = gamma * v_t + sum of the listed rows' block t, then the WTA -> the new state words of each.
// P counter planes hold every score of the round.  Plain (non-volatile) shared loads so the
// compiler overlaps consecutive entries' loads.
template <int WC, int P>
__device__ __forceinline__ void score_wta2(const uint32_t (&va)[WC], const uint32_t (&vb)[WC], uint32_t gamma,
                                           const uint32_t *lst, int cnt, int cntw, uint32_t zoff, const uint8_t *w,
                                           uint32_t ta, uint32_t tbb, int L, uint32_t (&oa)[WC], uint32_t (&ob)[WC]) {
    using Blk = typename std::conditional<WC == 4, uint4, typename std::conditional<WC == 2, uint2, uint32_t>::type>::type;
    uint32_t pa[P][WC], pb[P][WC];
#pragma unroll
    for (int b = 0; b < P; ++b)
#pragma unroll
        for (int u = 0; u < WC; ++u) {
            pa[b][u] = ((gamma >> b) & 1u) ? va[u] : 0u;
            pb[b][u] = ((gamma >> b) & 1u) ? vb[u] : 0u;
        }
    // two rows per step: plane 0 takes both through a full adder (sum = p ^ x ^ y, carry =
    // majority), the carry then ripples up -- 2P logic ops per word for two rows instead of 4P
    auto add2 = [&](uint32_t (&pl)[P][WC], const Blk &bx, const Blk &by) {
        const uint32_t *x = reinterpret_cast<const uint32_t *>(&bx);
        const uint32_t *y = reinterpret_cast<const uint32_t *>(&by);
#pragma unroll
        for (int u = 0; u < WC; ++u) {
            const uint32_t p0 = pl[0][u];
            uint32_t cy = (p0 & x[u]) | (p0 & y[u]) | (x[u] & y[u]);
            pl[0][u] = p0 ^ x[u] ^ y[u];
#pragma unroll
            for (int b = 1; b < P; ++b) {
                const uint32_t t = pl[b][u] & cy;
                pl[b][u] ^= cy;
                cy = t;
            }
        }
    };
    // the warp's largest count for every lane (no divergence); a lane past its own count adds the
    // zero row
    for (int e = 0; e < cntw; e += 2) {
        const uint32_t o0 = e < cnt ? lst[e * kNTb] : zoff;
        const uint32_t o1 = e + 1 < cnt ? lst[(e + 1) * kNTb] : zoff;
        const Blk xa = *reinterpret_cast<const Blk *>(w + o0 + ta);
        const Blk ya = *reinterpret_cast<const Blk *>(w + o1 + ta);
        const Blk xb = *reinterpret_cast<const Blk *>(w + o0 + tbb);
        const Blk yb = *reinterpret_cast<const Blk *>(w + o1 + tbb);
        add2(pa, xa, ya);
        add2(pb, xb, yb);
    }
    auto wta = [&](const uint32_t (&pl)[P][WC], uint32_t (&out)[WC]) {
        uint32_t cand[WC];
#pragma unroll
        for (int u = 0; u < WC; ++u) {
            const int nb = min(32, max(0, L - u * 32));
            cand[u] = nb == 32 ? 0xffffffffu : ((1u << nb) - 1u);
        }
#pragma unroll
        for (int b = P - 1; b >= 0; --b) {
            uint32_t x[WC], any = 0u;
#pragma unroll
            for (int u = 0; u < WC; ++u) {
                x[u] = cand[u] & pl[b][u];
                any |= x[u];
            }
            if (any) {
#pragma unroll
                for (int u = 0; u < WC; ++u) cand[u] = x[u];
            }
        }
#pragma unroll
        for (int u = 0; u < WC; ++u) out[u] = cand[u];
    };
    wta(pa, oa);
    wta(pb, ob);
}

template <int WC>
__global__ void __launch_bounds__(kNTb, 1)
sos_bits_kernel(Shape s, const uint32_t *__restrict__ wb, const uint16_t *__restrict__ probes, int64_t k,
                int gamma, int T, unsigned long long *queue, uint32_t *__restrict__ out_state,
                uint16_t *__restrict__ out_iters, uint8_t *__restrict__ out_status, int64_t *__restrict__ ovf,
                unsigned long long *__restrict__ ovf_count) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    const uint32_t w_s = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const int C = s.C, L = s.L, nw = s.nw, np = s.np;
    const uint32_t rowB = (uint32_t)nw * 4u;
    uint32_t *lst = reinterpret_cast<uint32_t *>(smem_raw + (size_t)np * rowB) + threadIdx.x;   // [entry][thread]
    const uint32_t zoff = (uint32_t)np * rowB + (uint32_t)kList * kNTb * 4u;   // a zero row (rowB bytes)
    for (int i = threadIdx.x; i < nw; i += kNTb) reinterpret_cast<uint32_t *>(smem_raw + zoff)[i] = 0u;
    for (int i = threadIdx.x; i < np * nw / 4; i += kNTb) {
        const uint4 v = __ldg(reinterpret_cast<const uint4 *>(wb) + i);
        asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(w_s + i * 16), "r"(v.x), "r"(v.y), "r"(v.z),
                     "r"(v.w)
                     : "memory");
    }
    __syncthreads();
    const uint32_t q = (uint32_t)((threadIdx.x & 31) % C);
    const uint32_t ug = (uint32_t)gamma;

    uint32_t V[8][WC];   // V[c] = state words of cluster (c + q) mod C
    int64_t p = -1;
    int rl = 0;
    bool active = false;
    // the next probe's symbols are loaded one refill ahead (their latency overlaps the rounds)
    int64_t pn = (int64_t)atomicAdd(queue, 1ull);
    uint32_t nx[4];   // 16 bits per cluster
    auto prefetch = [&]() {
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const uint32_t lo = (pn < k && 2 * h < C) ? (uint32_t)__ldg(probes + pn * C + 2 * h) : 0u;
            const uint32_t hi = (pn < k && 2 * h + 1 < C) ? (uint32_t)__ldg(probes + pn * C + 2 * h + 1) : 0u;
            nx[h] = lo | (hi << 16);
        }
    };
    prefetch();
    auto refill = [&]() {
        for (;;) {
            p = pn;
            uint32_t sy[4];
#pragma unroll
            for (int h = 0; h < 4; ++h) sy[h] = nx[h];
            pn = (int64_t)atomicAdd(queue, 1ull);
            prefetch();
            rl = 0;
            if (p >= k) {
                active = false;
#pragma unroll
                for (int c = 0; c < 8; ++c)
#pragma unroll
                    for (int u = 0; u < WC; ++u) V[c][u] = 0u;
                return;
            }
            bool valid = true;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
#pragma unroll
                for (int u = 0; u < WC; ++u) V[c][u] = 0u;
                if (c < C) {
                    // symbol of cluster (c + q) mod C: a static select over the prefetched words
                    const uint32_t cl = (uint32_t)((c + (int)q) % C);
                    uint32_t wd = sy[0];
#pragma unroll
                    for (int j = 1; j < 4; ++j) wd = (cl >> 1) == (uint32_t)j ? sy[j] : wd;
                    const uint32_t sym = (wd >> (16u * (cl & 1u))) & 0xffffu;
                    if (sym != kErased) {
                        if (sym >= (uint32_t)L) valid = false;
#pragma unroll
                        for (int u = 0; u < WC; ++u) V[c][u] = (sym >> 5) == (uint32_t)u ? 1u << (sym & 31u) : 0u;
                    }
                }
            }
            if (!valid) {   // GB_INVALID: zero state, 0 rounds; take another probe
                for (int w = 0; w < nw; ++w) out_state[p * nw + w] = 0u;
                out_iters[p] = 0;
                out_status[p] = GB_INVALID;
                continue;
            }
            active = true;
            return;
        }
    };
    refill();
    while (__any_sync(0xffffffffu, active)) {
        // ---- the active neurons' row offsets (first kList), and their number (0 when idle)
        int cnt = 0;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            if (c < C) {
                const uint32_t cl = (uint32_t)((c + (int)q) % C);
#pragma unroll
                for (int u = 0; u < WC; ++u) {
                    uint32_t x = V[c][u];
                    while (x) {
                        const uint32_t bi = __ffs(x) - 1;
                        x &= x - 1u;
                        if (cnt < kList) lst[cnt * kNTb] = (cl * (uint32_t)(32 * WC) + (uint32_t)u * 32u + bi) * rowB;
                        ++cnt;
                    }
                }
            }
        }
        const uint32_t smax = (uint32_t)cnt + ug;   // no score of the round exceeds this
        bool go = active;
        if (active && (cnt > kList || smax >= 64u)) {
            // a large active set (e.g. a cluster whose max was 0 turned whole, R4): the probe is
            // queued and decoded from the start by the CTA-pair kernel in list mode (the generic
            // kernel when the pair is off), exact either way
            ovf[atomicAdd(ovf_count, 1ull)] = p;
            refill();
            go = false;
        }
        // warp-uniform list length and plane count; an idle lane scores its (discarded) state
        // against the zero row
        const int cl_n = go ? cnt : 0;
        const int cntw = (int)__reduce_max_sync(0xffffffffu, (unsigned)cl_n);
        const bool wide = __any_sync(0xffffffffu, go && smax >= 16u);
        // two target clusters per pass over the list; a cluster's new words replace its old ones
        // once scored (the list already holds the round's sources, and v_t feeds only target t)
        bool changed = false;
#pragma unroll
        for (int c = 0; c < 8; c += 2) {
            if (c < C) {
                const uint32_t ca = (uint32_t)((c + (int)q) % C), cb = (uint32_t)((c + 1 + (int)q) % C);
                uint32_t na[WC], nb[WC];
                if (!wide)
                    score_wta2<WC, 4>(V[c], V[c + 1], ug, lst, cl_n, cntw, zoff, smem_raw, ca * (WC * 4),
                                      cb * (WC * 4), L, na, nb);
                else
                    score_wta2<WC, 6>(V[c], V[c + 1], ug, lst, cl_n, cntw, zoff, smem_raw, ca * (WC * 4),
                                      cb * (WC * 4), L, na, nb);
                if (go) {
#pragma unroll
                    for (int u = 0; u < WC; ++u) {
                        changed |= na[u] != V[c][u];
                        V[c][u] = na[u];
                        if (c + 1 < C) {
                            changed |= nb[u] != V[c + 1][u];
                            V[c + 1][u] = nb[u];
                        }
                    }
                }
            }
        }
        if (go) {
            ++rl;
            if (!changed || rl == T) {   // ---- a7 output: V^rl (un-rotated by address)
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    if (c < C) {
                        const uint32_t cl = (uint32_t)((c + (int)q) % C);
#pragma unroll
                        for (int u = 0; u < WC; ++u) out_state[p * nw + cl * WC + u] = V[c][u];
                    }
                }
                out_iters[p] = (uint16_t)rl;
                out_status[p] = (uint8_t)(!changed ? GB_CONVERGED : GB_MAX_ITERS);
                refill();
            }
        }
    }
}

template <int WC>
cudaError_t launch_bits_t(Call &cl, const uint16_t *probes, int64_t k, int gamma, int max_iters, uint32_t *state,
                          uint16_t *iters, uint8_t *status, int64_t *ovf, unsigned long long *ovf_count) {
    const gb_net *net = cl.net;
    const size_t smem = (size_t)net->s.np * net->s.nw * 4 + (size_t)kList * kNTb * 4 + (size_t)net->s.nw * 4;
    auto fn = sos_bits_kernel<WC>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    unsigned long long *queue = cl.counters();   // [0] work queue, [1] overflow count
    if (!queue) return cl.err;
    int64_t grid = (k + 63) / 64;   // small batches: spread over more SMs (the queue balances)
    if (grid > net->sm_count) grid = net->sm_count;
    if (grid < 1) grid = 1;
    fn<<<(unsigned)grid, kNTb, smem, cl.st>>>(net->s, net->wb, probes, k, gamma, max_iters, queue, state, iters,
                                              status, ovf, ovf_count);
    cl.launched();
    return cudaGetLastError();
}

}  // namespace

// Shapes the kernel takes: C <= 8 clusters of <= 128 neurons (W bit rows + the lists fit shared
// memory), scores below 2^11 (n_padded + gamma), no period-2 exit (GB_FLAG_CYCLE_EXIT keeps the
// tensor-core kernels).
bool sos_bits_supported(const Shape &s, int gamma, int cyc) {
    return !cyc && s.C <= 8 && (s.Wc == 1 || s.Wc == 2 || s.Wc == 4) && s.np <= 1024 && s.np + gamma < 2048 &&
           (size_t)s.np * s.nw * 4 + (size_t)kList * kNTb * 4 + (size_t)s.nw * 4 <= 227 * 1024;
}

cudaError_t launch_sos_bits(Call &cl, const uint16_t *probes, int64_t k, int gamma, int max_iters,
                            uint32_t *state, uint16_t *iters, uint8_t *status) {
    int64_t *ovf = cl.ovf(k);
    unsigned long long *cnt = cl.counters();
    if (!ovf || !cnt) return cl.err;
    cudaError_t e;
    switch (cl.net->s.Wc) {
        case 1: e = launch_bits_t<1>(cl, probes, k, gamma, max_iters, state, iters, status, ovf, cnt + 1); break;
        case 2: e = launch_bits_t<2>(cl, probes, k, gamma, max_iters, state, iters, status, ovf, cnt + 1); break;
        case 4: e = launch_bits_t<4>(cl, probes, k, gamma, max_iters, state, iters, status, ovf, cnt + 1); break;
        default: return cudaErrorNotSupported;
    }
    if (e != cudaSuccess) return e;
    // the probes whose active set outgrew the list: decoded from the start (exact) by the CTA-pair
    // tensor-core kernel in list mode, else (shapes it does not take) the generic kernel
    e = launch_sos_pair_list(cl, probes, k, ovf, cnt + 1, gamma, max_iters, state, iters, status);
    if (e != cudaErrorNotSupported) return e;
    return launch_decode_generic_list(cl, probes, k, ovf, cnt + 1, GB_SUM_OF_SUM, gamma, max_iters, state, iters,
                                      status);
}

}  // namespace gb
