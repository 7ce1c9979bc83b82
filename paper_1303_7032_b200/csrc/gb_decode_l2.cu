// gb_decode_l2.cu -- SOM / hybrid decode for networks whose bit rows do not
// fit in shared memory (n_padded > 1024 or C > 8; e.g. BASELINE C4,
// c=16 l=256: W bits = 2 MiB, L2-resident).
//
// One warp per probe; the probe's state (old and next) lives in shared
// memory.  The warp is split into NG = 32/WC lane groups of WC lanes: a group
// owns one (source cluster s -> target cluster t) push at a time and lane u of
// the group owns word u of the target block, so the W reads of a group are
// one contiguous 4*WC-byte segment of a bit row (one L2 sector at WC = 8).
//
// Method, the same as the shared-memory kernel:
//  a1 ingest  -- symbols -> erased set; symbol >= L -> GB_INVALID.
//  a5 prune   -- hybrid: X^0 on erased clusters = AND of the known neurons'
//                bit rows (S^0 == C-e, Alg. 2 L2-5, F3 of DESIGN.md); SOM:
//                erased clusters all 1 (L270-271), known one-hot.
//  a6 round   -- Eq.(6)-(7) by bail-out-early (Thm 1): for every in-scope
//                target t and every other in-scope source s, H_{s->t} = OR of
//                block t of the rows j in X_s, accumulated until it covers
//                X_t (L449); X'_t = X_t AND over s of H_{s->t}; a target
//                found empty stops being walked (L450).  Hybrid: scope =
//                erased clusters, known clusters frozen (Alg. 2).
//                Synchronous rounds: every H reads the old state.
//  a7 output  -- state bits, rounds (incl. the confirming round), status.
#include "gb_internal.h"

namespace gb {
namespace {

constexpr int kL2Warps = 8;

__device__ __forceinline__ uint32_t real_mask_w(int L, int u) {
    const int nb = min(32, max(0, L - u * 32));
    return nb == 32 ? 0xffffffffu : ((1u << nb) - 1u);
}

template <int WC, int RULE>
__global__ void __launch_bounds__(kL2Warps * 32)
decode_l2_kernel(Shape s, const uint32_t *__restrict__ wb, const uint16_t *__restrict__ probes, int64_t k,
                 int T, uint32_t *__restrict__ out_state, uint16_t *__restrict__ out_iters,
                 uint8_t *__restrict__ out_status, const int64_t *__restrict__ list,
                 const unsigned long long *__restrict__ list_count) {
    constexpr int NG = 32 / WC;            // lane groups per warp
    constexpr int LP = 32 * WC;
    extern __shared__ uint32_t sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane / WC, u = lane % WC;     // group, word of the target block
    const int C = s.C, nw = s.nw;
    uint32_t *Xa = sm + warp * 2 * nw, *Xb = Xa + nw;
    const unsigned gmask = (WC == 32 ? 0xffffffffu : ((1u << WC) - 1u)) << (g * WC);

    // list mode: decode only the probes queued by decode_l2t_kernel (more erased clusters than its slots)
    const int64_t nprobe = list ? (int64_t)*list_count : k;
    for (int64_t pi = (int64_t)blockIdx.x * kL2Warps + warp; pi < nprobe; pi += (int64_t)gridDim.x * kL2Warps) {
        const int64_t p = list ? list[pi] : pi;
        const uint16_t *pr = probes + p * C;
        // ---- a1 ingest
        unsigned long long em = 0ull;
        bool bad = false;
        for (int c = lane; c < C; c += 32) {
            const unsigned sym = __ldg(pr + c);
            if (sym == kErased) em |= 1ull << c;
            else if (sym >= (unsigned)s.L) bad = true;
        }
        {
            unsigned lo = __reduce_or_sync(0xffffffffu, (unsigned)em);
            unsigned hi = __reduce_or_sync(0xffffffffu, (unsigned)(em >> 32));
            em = ((unsigned long long)hi << 32) | lo;
        }
        bad = __any_sync(0xffffffffu, bad);
        uint32_t *out = out_state + p * nw;
        if (bad) {
            for (int w = lane; w < nw; w += 32) out[w] = 0u;
            if (lane == 0) { out_iters[p] = 0; out_status[p] = GB_INVALID; }
            continue;
        }
        const unsigned long long all = (C == 64) ? ~0ull : ((1ull << C) - 1ull);
        const unsigned long long scope = (RULE == GB_SUM_OF_MAX) ? all : em;
        uint32_t *X = Xa, *Xn = Xb;
        // ---- a5 prune / init
        for (int w = lane; w < nw; w += 32) {
            const int c = w / WC, uu = w - c * WC;
            uint32_t x;
            if ((em >> c) & 1ull) {
                x = real_mask_w(s.L, uu);
                if (RULE == GB_HYBRID) {
                    unsigned long long km = all & ~em;
                    while (km && x) {
                        const int kc = __ffsll((long long)km) - 1;
                        km &= km - 1ull;
                        const int row = kc * LP + __ldg(pr + kc);
                        x &= __ldg(wb + (int64_t)row * nw + w);
                    }
                }
            } else {
                const unsigned sym = __ldg(pr + c);
                x = ((int)(sym >> 5) == uu) ? (1u << (sym & 31)) : 0u;
            }
            X[w] = x;
        }
        __syncwarp();

        int it = 0, status = GB_MAX_ITERS;
        if (RULE == GB_HYBRID && em == 0ull) {
            status = GB_CONVERGED;
        } else {
            while (it < T) {
                for (int w = lane; w < nw; w += 32) Xn[w] = X[w];
                __syncwarp();
                // ---- a6 one synchronous round
                unsigned long long tm = scope;
                while (tm) {
                    const int t = __ffsll((long long)tm) - 1;
                    tm &= tm - 1ull;
                    // next state of word u of cluster t; also the coverage target (it only
                    // shrinks, so covering it is enough for the AND below)
                    uint32_t acc = X[t * WC + u];
                    if (!__any_sync(0xffffffffu, acc)) continue;
                    unsigned long long sm_ = scope & ~(1ull << t);
                    while (sm_) {
                        // the next NG sources, one per lane group
                        int src = -1;
                        {
                            unsigned long long q = sm_;
                            for (int i = 0; i < NG && q; ++i) {
                                const int c2 = __ffsll((long long)q) - 1;
                                q &= q - 1ull;
                                if (i == g) src = c2;
                            }
                            for (int i = 0; i < NG && sm_; ++i) sm_ &= sm_ - 1ull;
                        }
                        uint32_t h = 0u;
                        if (src >= 0) {
                            const uint32_t *xs = X + src * WC;
                            const uint32_t *wcol = wb + (int64_t)(src * LP) * nw + t * WC + u;
                            uint32_t v = 0, cur = xs[0];
                            bool miss = true;
                            while (miss) {
                                if (!cur) {
                                    do { ++v; } while (v < (uint32_t)WC && !(cur = xs[v]));
                                    if (v >= (uint32_t)WC) break;
                                }
                                // two rows per step (ILP); the second may be absent
                                const uint32_t b1 = __ffs(cur) - 1;
                                cur &= cur - 1u;
                                const uint32_t b2 = __ffs(cur) - 1;
                                cur &= cur - 1u;
                                const uint32_t r1 = __ldg(wcol + (int64_t)(v * 32 + b1) * nw);
                                const uint32_t r2 = (b2 != 0xffffffffu) ? __ldg(wcol + (int64_t)(v * 32 + b2) * nw) : 0u;
                                h |= r1 | r2;
                                miss = (__ballot_sync(gmask, (acc & ~h) != 0u) & gmask) != 0u;
                            }
                        } else {
                            h = 0xffffffffu;
                        }
                        // AND the groups' coverage masks into the next state
#pragma unroll
                        for (int off = WC; off < 32; off <<= 1) h &= __shfl_xor_sync(0xffffffffu, h, off);
                        acc &= h;
                        if (!__any_sync(0xffffffffu, acc)) break;   // target cluster empty (L450)
                    }
                    if (g == 0) Xn[t * WC + u] = acc;
                }
                __syncwarp();
                bool diff = false;
                for (int w = lane; w < nw; w += 32) diff |= (Xn[w] != X[w]);
                diff = __any_sync(0xffffffffu, diff);
                uint32_t *tmp = X; X = Xn; Xn = tmp;
                ++it;
                if (!diff) { status = GB_CONVERGED; break; }
            }
        }
        for (int w = lane; w < nw; w += 32) out[w] = X[w];
        if (lane == 0) { out_iters[p] = (uint16_t)it; out_status[p] = (uint8_t)status; }
        __syncwarp();
    }
}

template <int WC, int RULE>
cudaError_t launch_t(Call &cl, const uint16_t *probes, int64_t k, int max_iters, uint32_t *state,
                     uint16_t *iters, uint8_t *status, const int64_t *list = nullptr,
                     const unsigned long long *list_count = nullptr) {
    const gb_net *net = cl.net;
    const cudaStream_t st = cl.st;
    const size_t smem = (size_t)kL2Warps * 2 * net->s.nw * sizeof(uint32_t);
    auto fn = decode_l2_kernel<WC, RULE>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    int64_t grid = (k + kL2Warps - 1) / kL2Warps;
    const int64_t cap = (int64_t)net->sm_count * 8;
    if (grid > cap || list) grid = cap;
    fn<<<(unsigned)grid, kL2Warps * 32, smem, st>>>(net->s, net->wb, probes, k, max_iters, state, iters, status,
                                                    list, list_count);
    cl.launched();
    return cudaGetLastError();
}

}  // namespace

bool decode_l2_supported(const Shape &s, int rule) {
    if (rule == GB_SUM_OF_SUM) return false;
    return s.Wc == 1 || s.Wc == 2 || s.Wc == 4 || s.Wc == 8 || s.Wc == 16;
}

cudaError_t launch_decode_l2(Call &cl, const uint16_t *probes, int64_t k, int rule, int max_iters,
                             uint32_t *state, uint16_t *iters, uint8_t *status) {
    const gb_net *net = cl.net;
    if (!decode_l2_supported(net->s, rule)) return cudaErrorNotSupported;
    const bool h = rule == GB_HYBRID;
    if (decode_l2t_supported(net, rule)) {
        // thread-per-probe kernel; probes with more in-scope clusters than its slots are
        // queued and decoded here by the warp-per-probe kernel in list mode
        int64_t *L = cl.ovf(k);
        unsigned long long *cnt = cl.counters();
        if (!L || !cnt) return cl.err;
        cudaError_t e = launch_decode_l2t(cl, probes, k, rule, max_iters, state, iters, status);
        if (e != cudaSuccess) return e;
        const unsigned long long *LC = cnt + 1;
        switch (net->s.Wc) {
            case 4: return h ? launch_t<4, GB_HYBRID>(cl, probes, k, max_iters, state, iters, status, L, LC)
                             : launch_t<4, GB_SUM_OF_MAX>(cl, probes, k, max_iters, state, iters, status, L, LC);
            case 8: return h ? launch_t<8, GB_HYBRID>(cl, probes, k, max_iters, state, iters, status, L, LC)
                             : launch_t<8, GB_SUM_OF_MAX>(cl, probes, k, max_iters, state, iters, status, L, LC);
            default: return h ? launch_t<16, GB_HYBRID>(cl, probes, k, max_iters, state, iters, status, L, LC)
                              : launch_t<16, GB_SUM_OF_MAX>(cl, probes, k, max_iters, state, iters, status, L, LC);
        }
    }
    switch (net->s.Wc) {
        case 1: return h ? launch_t<1, GB_HYBRID>(cl, probes, k, max_iters, state, iters, status)
                         : launch_t<1, GB_SUM_OF_MAX>(cl, probes, k, max_iters, state, iters, status);
        case 2: return h ? launch_t<2, GB_HYBRID>(cl, probes, k, max_iters, state, iters, status)
                         : launch_t<2, GB_SUM_OF_MAX>(cl, probes, k, max_iters, state, iters, status);
        case 4: return h ? launch_t<4, GB_HYBRID>(cl, probes, k, max_iters, state, iters, status)
                         : launch_t<4, GB_SUM_OF_MAX>(cl, probes, k, max_iters, state, iters, status);
        case 8: return h ? launch_t<8, GB_HYBRID>(cl, probes, k, max_iters, state, iters, status)
                         : launch_t<8, GB_SUM_OF_MAX>(cl, probes, k, max_iters, state, iters, status);
        default: return h ? launch_t<16, GB_HYBRID>(cl, probes, k, max_iters, state, iters, status)
                          : launch_t<16, GB_SUM_OF_MAX>(cl, probes, k, max_iters, state, iters, status);
    }
}

}  // namespace gb
