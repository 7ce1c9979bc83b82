// gb_decode_l2t.cu -- thread-per-probe SOM / hybrid decode for networks whose
// bit rows do not fit in shared memory (C <= 16, Wc in {4, 8, 16}, e.g.
// BASELINE C4 c=16 l=256: W bits = 2 MiB, L2-resident; Scenario 2 l=512).
//
// Same method and result as decode_l2_kernel (gb_decode_l2.cu), which keeps
// the probes needing more slots than this kernel holds (list mode).  Here one
// thread decodes one probe: its in-scope cluster states (erased clusters for
// the hybrid, all clusters for sum-of-max) live in shared memory laid out
// [slot word][thread] (conflict-free), old and next state in two areas
// (synchronous rounds).  W bit-row blocks are read from L2 with 16-byte loads.
//
// Method:
//  a1 ingest  -- symbols -> erased set; symbol >= L -> GB_INVALID.
//  a5 prune   -- hybrid: X^0 on erased clusters = AND of the known neurons'
//                rows (S^0 == C-e, Alg. 2 L2-5 / Thm 4); the known rows are
//                walked once, each loading its blocks of every erased cluster.
//                SOM: erased clusters all 1 (L270-271), known one-hot.
//  a6 round   -- Eq.(6)-(7) by bail-out-early (Thm 1) in push form:
//                for target t and source s != t, H = OR of block t of the rows
//                of X_s, read in stages of up to 4 rows (6 for SOM; the lowest remaining
//                candidate of successive words, all in flight together) until
//                H covers the still-alive part of X_t (L449); X'_t = X_t AND
//                over s of H; an emptied target stops being walked (L450).
//                Hybrid: known clusters frozen (Alg. 2).
//  a7 output  -- state bits, rounds (incl. the confirming round), status.
#include "gb_internal.h"

namespace gb {
namespace {

constexpr int kMaxC16 = 16;

// 32-byte read-only load (sm_100: LDG.256): one sector per lane, half the L1TEX wavefronts of two
// 16-byte loads of the same block (the kernel is bound by the L1TEX data pipe: 93% at C4 with
// 16-byte loads).  Same-box A/B: C4 hybrid 2.05 -> 1.59 ms, C4 sum-of-max (10^6) 10.56 -> 9.13,
// Scenario 2 sum-of-max 1.745 -> 1.689, hybrid 0.174 -> 0.167.
__device__ __forceinline__ void ldg8(const uint32_t *a, uint32_t *v) {
    asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "l"(a));
}
__device__ __forceinline__ void ldg8p(uint32_t p, const uint32_t *a, uint32_t *v) {
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %8, 0;\n\t@q ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%9];\n\t}"
        : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7])
        : "r"(p), "l"(a));
}

template <int WC>
__device__ __forceinline__ void ldg_block(const uint32_t *p, uint32_t (&v)[WC]) {
    if constexpr (WC % 8 == 0) {
#pragma unroll
        for (int q = 0; q < WC / 8; ++q) ldg8(p + 8 * q, v + 8 * q);
    } else if constexpr (WC % 4 == 0) {
#pragma unroll
        for (int q = 0; q < WC / 4; ++q) {
            const uint4 t = __ldg(reinterpret_cast<const uint4 *>(p) + q);
            v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
        }
    } else {
#pragma unroll
        for (int u = 0; u < WC; ++u) v[u] = __ldg(p + u);
    }
}

// Predicated 16-byte read-only load (v unchanged when p == 0): a stage's row loads issue back
// to back without branches, so their L2 latencies overlap.
__device__ __forceinline__ void ldg4p(uint32_t p, const uint32_t *a, uint32_t (&v)[4]) {
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %4, 0;\n\t@q ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%5];\n\t}"
        : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3])
        : "r"(p), "l"(a));
}

template <int WC>
__device__ __forceinline__ void ldg_blockp(uint32_t p, const uint32_t *a, uint32_t (&v)[WC]) {
    static_assert(WC % 4 == 0, "predicated block loads need Wc % 4 == 0");
    if constexpr (WC % 8 == 0) {
#pragma unroll
        for (int q = 0; q < WC / 8; ++q) {
            uint32_t t[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
            ldg8p(p, a + 8 * q, t);
#pragma unroll
            for (int i = 0; i < 8; ++i) v[8 * q + i] = t[i];
        }
    } else {
#pragma unroll
        for (int q = 0; q < WC / 4; ++q) {
            uint32_t t[4] = {0u, 0u, 0u, 0u};
            ldg4p(p, a + 4 * q, t);
            v[4 * q] = t[0]; v[4 * q + 1] = t[1]; v[4 * q + 2] = t[2]; v[4 * q + 3] = t[3];
        }
    }
}

template <int WC, int RULE, int MAXS, int NT>
__global__ void __launch_bounds__(NT, 1)
decode_l2t_kernel(Shape s, const uint32_t *__restrict__ wb, const uint16_t *__restrict__ probes, int64_t k, int T,
                  uint32_t *__restrict__ out_state, uint16_t *__restrict__ out_iters,
                  uint8_t *__restrict__ out_status, int64_t *__restrict__ ovf,
                  unsigned long long *__restrict__ ovf_count, uint32_t *__restrict__ xscratch,
                  const uint32_t *__restrict__ wu) {
    constexpr int LP = 32 * WC;
    // rows per push stage = one word group of G words (the lowest remaining candidate of each),
    // all G loads predicated and in flight together; groups are visited cyclically until the
    // target is covered or the source exhausted.  Sum-of-max's first round covers whole erased
    // clusters from all-ones sources, where wider stages pay.
    constexpr int G = (RULE == GB_SUM_OF_MAX ? 8 : 4) < WC ? (RULE == GB_SUM_OF_MAX ? 8 : 4) : WC;
    static_assert(WC % G == 0, "word groups tile the block");
    extern __shared__ uint32_t sm[];
    const int tid = threadIdx.x;
    const int C = s.C, nw = s.nw;
    uint32_t rmask[WC];
#pragma unroll
    for (int u = 0; u < WC; ++u) {
        const int nb = min(32, max(0, s.L - u * 32));
        rmask[u] = nb == 32 ? 0xffffffffu : ((1u << nb) - 1u);
    }
    for (int64_t p = (int64_t)blockIdx.x * NT + tid; p < k; p += (int64_t)gridDim.x * NT) {
        const uint16_t *pr = probes + p * C;
        // ---- a1 ingest
        uint32_t emask = 0u;
        bool bad = false;
        for (int c = 0; c < C; ++c) {
            const unsigned sym = __ldg(pr + c);
            if (sym == kErased) emask |= 1u << c;
            else if (sym >= (unsigned)s.L) bad = true;
        }
        uint32_t *out = out_state + p * nw;
        if (bad) {
            for (int w = 0; w < nw; ++w) out[w] = 0u;
            out_iters[p] = 0;
            out_status[p] = GB_INVALID;
            continue;
        }
        const uint32_t scope = (RULE == GB_SUM_OF_MAX) ? ((1u << C) - 1u) : emask;
        const int nslot = __popc(scope);
        if (nslot > MAXS) {   // more in-scope clusters than slots: warp-per-probe kernel (list mode)
            ovf[atomicAdd(ovf_count, 1ull)] = p;
            continue;
        }
        uint64_t slots = 0;   // in-scope clusters ascending, 4 bits each
        {
            uint32_t m = scope;
#pragma unroll
            for (int t = 0; t < MAXS; ++t) {
                if (m) {
                    slots |= (uint64_t)(__ffs(m) - 1) << (4 * t);
                    m &= m - 1u;
                }
            }
        }
        auto slot_c = [&](int t) -> int { return (int)((slots >> (4 * t)) & 15u); };
        // current state in shared memory, next state in this CTA's slice of a global scratch
        // ([word][thread], L2): only the current state is read in the push loops, so shared
        // memory holds one copy and twice as many threads fit (latency hiding of the L2 rows)
        uint32_t *X = sm, *Xn = xscratch + (size_t)blockIdx.x * MAXS * WC * NT;
        // bit t set <=> slot t holds every real neuron of its cluster: a push from it covers
        // exactly the cluster union Wu (one block load instead of ~L/4 rows; seal builds Wu)
        uint32_t fullm = 0u;
        // ---- a5 prune (hybrid) / init (SOM)
        if (RULE == GB_HYBRID) {
            uint32_t x[MAXS][WC];
#pragma unroll
            for (int t = 0; t < MAXS; ++t)
#pragma unroll
                for (int u = 0; u < WC; ++u) x[t][u] = rmask[u];
            uint32_t km = ((1u << C) - 1u) & ~emask;
            while (km) {
                const int kc = __ffs(km) - 1;
                km &= km - 1u;
                const uint32_t *row = wb + (size_t)(kc * LP + __ldg(pr + kc)) * nw;
#pragma unroll
                for (int t = 0; t < MAXS; ++t) {
                    if (t < nslot) {
                        uint32_t r[WC];
                        ldg_block<WC>(row + slot_c(t) * WC, r);
#pragma unroll
                        for (int u = 0; u < WC; ++u) x[t][u] &= r[u];
                    }
                }
            }
#pragma unroll
            for (int t = 0; t < MAXS; ++t)
                if (t < nslot) {
                    bool full = true;
#pragma unroll
                    for (int u = 0; u < WC; ++u) {
                        X[(t * WC + u) * NT + tid] = x[t][u];
                        full &= x[t][u] == rmask[u];
                    }
                    if (full) fullm |= 1u << t;
                }
        } else {
            for (int t = 0; t < nslot; ++t) {
                const int c = slot_c(t);
                if ((emask >> c) & 1u) {
#pragma unroll
                    for (int u = 0; u < WC; ++u) X[(t * WC + u) * NT + tid] = rmask[u];
                    fullm |= 1u << t;
                } else {
                    const unsigned sym = __ldg(pr + c);
#pragma unroll
                    for (int u = 0; u < WC; ++u)
                        X[(t * WC + u) * NT + tid] = ((int)(sym >> 5) == u) ? (1u << (sym & 31)) : 0u;
                }
            }
        }
        // ---- a6 synchronous rounds
        int it = 0, status = GB_MAX_ITERS;
        if (RULE == GB_HYBRID && nslot == 0) {
            status = GB_CONVERGED;
        } else {
            // from round 2 on only the pairs whose source slot changed in the previous round: a
            // pair whose source kept its candidates removes nothing (after the round that last
            // evaluated it, the target's candidates lie inside the OR of the rows it read, and
            // those rows are still candidates)
            uint32_t chg = 0xFFFFFFFFu;
            while (it < T) {
                bool changed = false;
                uint32_t chgn = 0u;
                uint32_t fulln = fullm;   // the round's pushes read the old state: update after it
                for (int t = 0; t < nslot; ++t) {
                    const int ct = slot_c(t);
                    uint32_t alive[WC];
                    uint32_t any = 0u;
#pragma unroll
                    for (int u = 0; u < WC; ++u) {
                        alive[u] = X[(t * WC + u) * NT + tid];
                        any |= alive[u];
                    }
                    for (int si = 0; si < nslot && any; ++si) {
                        if (si == t || !((chg >> si) & 1u)) continue;
                        const uint32_t *base = wb + (size_t)(slot_c(si) * LP) * nw + ct * WC;
                        uint32_t rem[WC];
                        uint32_t left = 0u;
#pragma unroll
                        for (int u = 0; u < WC; ++u) {
                            rem[u] = X[(si * WC + u) * NT + tid];
                            left |= rem[u];
                        }
                        uint32_t h[WC];
#pragma unroll
                        for (int u = 0; u < WC; ++u) h[u] = 0u;
                        uint32_t miss = 1u;
                        if ((fullm >> si) & 1u) {   // full source cluster: H = Wu[c_si][c_t]
                            ldg_block<WC>(wu + (size_t)(slot_c(si) * C + ct) * WC, h);
                            left = 0u;
                        }
                        while (miss && left) {
#pragma unroll
                            for (int grp = 0; grp < WC / G; ++grp) {
                                if (!(miss && left)) break;
                                // one stage: the lowest remaining candidate of each word of the group
                                uint32_t r[G][WC];
#pragma unroll
                                for (int q = 0; q < G; ++q) {
                                    const int u = grp * G + q;
                                    const uint32_t x = rem[u];
                                    rem[u] = x & (x - 1u);
#pragma unroll
                                    for (int v = 0; v < WC; ++v) r[q][v] = 0u;
                                    ldg_blockp<WC>(x, base + (size_t)(u * 32 + __ffs(x) - 1) * nw, r[q]);
                                }
                                miss = 0u;
                                left = 0u;
#pragma unroll
                                for (int v = 0; v < WC; ++v) {
                                    uint32_t o = 0u;
#pragma unroll
                                    for (int q = 0; q < G; ++q) o |= r[q][v];
                                    h[v] |= o;
                                    miss |= alive[v] & ~h[v];
                                    left |= rem[v];
                                }
                            }
                        }
                        any = 0u;
#pragma unroll
                        for (int u = 0; u < WC; ++u) {
                            alive[u] &= h[u];
                            any |= alive[u];
                        }
                    }
#pragma unroll
                    for (int u = 0; u < WC; ++u) {
                        if (alive[u] != X[(t * WC + u) * NT + tid]) chgn |= 1u << t;
                        changed |= (alive[u] != X[(t * WC + u) * NT + tid]);
                        Xn[(t * WC + u) * NT + tid] = alive[u];
                        if (alive[u] != rmask[u]) fulln &= ~(1u << t);
                    }
                }
                fullm = fulln;
                chg = chgn;
                if (changed)
                    for (int w = 0; w < nslot * WC; ++w) X[w * NT + tid] = Xn[w * NT + tid];
                ++it;
                if (!changed) { status = GB_CONVERGED; break; }
            }
        }
        // ---- a7 output: in-scope clusters from X, the others the known one-hot
        for (int c = 0; c < C; ++c) {
            uint32_t v[WC];
            if ((scope >> c) & 1u) {
                const int t = __popc(scope & ((1u << c) - 1u));
#pragma unroll
                for (int u = 0; u < WC; ++u) v[u] = X[(t * WC + u) * NT + tid];
            } else {
                const unsigned sym = __ldg(pr + c);
#pragma unroll
                for (int u = 0; u < WC; ++u) v[u] = ((int)(sym >> 5) == u) ? (1u << (sym & 31)) : 0u;
            }
            uint32_t *o = out + c * WC;
            if constexpr (WC % 4 == 0) {
#pragma unroll
                for (int q = 0; q < WC / 4; ++q)
                    reinterpret_cast<uint4 *>(o)[q] = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            } else {
#pragma unroll
                for (int u = 0; u < WC; ++u) o[u] = v[u];
            }
        }
        out_iters[p] = (uint16_t)it;
        out_status[p] = (uint8_t)status;
    }
}

template <int WC, int RULE, int MAXS>
cudaError_t launch_t(Call &cl, const uint16_t *probes, int64_t k, int max_iters, uint32_t *state,
                     uint16_t *iters, uint8_t *status) {
    const gb_net *net = cl.net;
    // threads per CTA: as many slot-state columns as 192 KiB of shared memory hold (128 KiB at
    // Wc = 16), at most 640 (register budget).  Same-box A/B: 128 KiB / 512 ->
    // 192 KiB / 640 took C4 hybrid 2.59 -> 2.32 ms and C4 SOM 3.33 -> 2.32 ms; Scenario 2
    // (Wc = 16) was faster at 128 KiB (0.270 vs 0.289 ms).
    constexpr int kSmemKB = WC >= 16 ? 128 : 192;
    constexpr int NT0 = (kSmemKB * 1024) / (MAXS * WC * 4);
    constexpr int NT = (NT0 > 640 ? 640 : NT0) / 32 * 32;
    const size_t smem = (size_t)MAXS * WC * NT * sizeof(uint32_t);
    uint32_t *xscratch = cl.alloc_n<uint32_t>((size_t)net->sm_count * MAXS * WC * NT);
    int64_t *ovf = cl.ovf(k);
    unsigned long long *cnt = cl.counters();
    if (!xscratch || !ovf || !cnt) return cl.err;
    auto fn = decode_l2t_kernel<WC, RULE, MAXS, NT>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int64_t grid = (k + NT - 1) / NT;
    if (grid > net->sm_count) grid = net->sm_count;
    fn<<<(unsigned)grid, NT, smem, cl.st>>>(net->s, net->wb, probes, k, max_iters, state, iters, status, ovf,
                                            cnt + 1, xscratch, wu_of(net, net->seal_gen));
    cl.launched();
    return cudaGetLastError();
}

}  // namespace

bool decode_l2t_supported(const gb_net *net, int rule) {
    const Shape &s = net->s;
    // measured (round 1, same box, next state in L2 scratch): faster than the warp-per-probe
    // kernel for the hybrid at C4 (2.59 vs 7.92 ms), Scenario 2 (0.270 vs 0.356 ms) and for
    // sum-of-max at C4 (3.33 vs 4.59 ms)
    if (net->opt[kOptL2t].load(std::memory_order_relaxed) == 0) return false;
    if (rule == GB_SUM_OF_SUM || s.C > kMaxC16) return false;
    // sum-of-max at Wc = 16 (16 slots x 64 B per thread, 128 threads per SM) was left to the warp
    // kernel while the stage loads were serial; with them in flight together it is faster
    // (Scenario 2 sum-of-max 2.99 -> 1.74 ms, same-box A/B)
    if (rule == GB_SUM_OF_MAX) return s.Wc == 4 || s.Wc == 8 || s.Wc == 16;
    return s.Wc == 4 || s.Wc == 8 || s.Wc == 16;
}

cudaError_t launch_decode_l2t(Call &cl, const uint16_t *probes, int64_t k, int rule, int max_iters,
                              uint32_t *state, uint16_t *iters, uint8_t *status) {
    const gb_net *net = cl.net;
    if (!decode_l2t_supported(net, rule)) return cudaErrorNotSupported;
    const bool h = rule == GB_HYBRID;
    switch (net->s.Wc) {
        case 4: return h ? launch_t<4, GB_HYBRID, 8>(cl, probes, k, max_iters, state, iters, status)
                         : launch_t<4, GB_SUM_OF_MAX, 16>(cl, probes, k, max_iters, state, iters, status);
        case 8: return h ? launch_t<8, GB_HYBRID, 8>(cl, probes, k, max_iters, state, iters, status)
                         : launch_t<8, GB_SUM_OF_MAX, 16>(cl, probes, k, max_iters, state, iters, status);
        default: return h ? launch_t<16, GB_HYBRID, 8>(cl, probes, k, max_iters, state, iters, status)
                          : launch_t<16, GB_SUM_OF_MAX, 16>(cl, probes, k, max_iters, state, iters, status);
    }
}

}  // namespace gb
