// gb_decode_smem.cu -- thread-per-probe SOM / hybrid decode with W held in
// shared memory (n_padded <= 1024, C <= 8): sum-of-max at the paper's shape,
// the hybrid shapes decode_hyb8_kernel does not take (C != 8 or Wc != 4), and
// the hybrid probes with e > 4 that it queues (8-slot instance, list mode).
//
// Layout (DESIGN.md §Kernels / "smem bit kernel"):
//  * W bit rows copied once per CTA into shared memory (128 KiB at c=8
//    l=128), row-major: block c of row j = words [c*WC, c*WC+WC).  Which
//    bank group a lane's read hits is set by its target cluster; the slot
//    list of each probe is rotated by a lane-dependent amount so the lanes
//    of a quarter-warp work on different targets at the same time.
//  * one thread = one probe.  The probe's in-scope cluster states X[t][WC]
//    (t indexes the slot list: erased clusters for the hybrid, all clusters
//    for sum-of-max) live in a per-thread shared-memory area laid out
//    [word][thread] (bank-conflict free); the next state of each slot is
//    built in registers (static slot unroll) and written back after the
//    round, so rounds are synchronous.
//
// Method:
//  a1 ingest  -- probe symbols -> erased list; symbol >= L -> GB_INVALID.
//  a5 prune   -- hybrid: X^0_c = AND over known clusters k of block c of row
//                (k, p_k): the erased neurons with S^0 = C-e (Alg. 2 L2-5,
//                identity F3 of DESIGN.md).  SOM: erased clusters all 1
//                (L270-271), known one-hot.
//  a6 round   -- Eq.(6)-(7) by bail-out-early (Thm 1) in "push"
//                form: for target slot t and every other source slot s,
//                H = OR of block c_t of the rows j in X_s, accumulated until
//                H covers the still-alive part of X_t (the first signal a
//                candidate receives from cluster c_s is enough, L449);
//                alive &= H; a target found dead stops being walked (L450).
//                Dead neurons stay dead (Lemma 1).  Hybrid: targets and
//                sources are the erased clusters only; known clusters are
//                frozen one-hot (Alg. 2) and every candidate is
//                adjacent to them by the prune.
//  a7 output  -- state bits, rounds (incl. the confirming round), status.
#include "gb_internal.h"

namespace gb {
namespace {

constexpr int kMaxC = 8;
#ifndef GB_NARROW_THREADS
#define GB_NARROW_THREADS 768
#endif

template <int WC>
__device__ __forceinline__ void lds_block(uint32_t addr, uint32_t (&v)[WC]) {
    if constexpr (WC == 4) {
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(addr));
    } else if constexpr (WC == 2) {
        asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v[0]), "=r"(v[1]) : "r"(addr));
    } else {
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v[0]) : "r"(addr));
    }
}

__device__ __forceinline__ uint32_t real_mask_u(int L, int u) {
    const int nb = min(32, max(0, L - u * 32));
    return nb == 32 ? 0xffffffffu : ((1u << nb) - 1u);
}

// MAXS = slots held per thread (4: hybrid probes with e <= 4 -- more threads fit;
// 8: any probe).  A probe needing more slots than MAXS is appended to `ovf` and
// decoded by the MAXS = 8 instance in list mode (`list` != nullptr).
template <int WC, int RULE, int MAXS, int NT>
__global__ void __launch_bounds__(NT, 1)
decode_smem_kernel(Shape s, const uint32_t *__restrict__ wb, const uint16_t *__restrict__ probes,
                   int64_t k, int T, uint32_t *__restrict__ out_state,
                   uint16_t *__restrict__ out_iters, uint8_t *__restrict__ out_status,
                   const int64_t *__restrict__ list, const unsigned long long *__restrict__ list_count,
                   int64_t *__restrict__ ovf, unsigned long long *__restrict__ ovf_count,
                   const uint32_t *__restrict__ wu) {
    extern __shared__ __align__(16) uint32_t smem[];
    constexpr int LP = 32 * WC;
    constexpr int BB = 4 * WC;                      // bytes per block
    const int C = s.C;
    const int nw = C * WC;
    const int np = C * LP;
    const int rowB = nw * 4;                        // bytes per row
    uint32_t *W = smem;
    uint32_t *X = smem + np * nw;                   // [MAXS*WC][threads]
    uint32_t *Z = X + (MAXS == 4 ? 0 : MAXS * WC * NT);   // one all-zero block
    const int tid = threadIdx.x;
    if (list && *list_count == 0ull) return;   // no queued probe: skip the W load
    const uint32_t w_s = (uint32_t)__cvta_generic_to_shared(W);
    const uint32_t zaddr = (uint32_t)__cvta_generic_to_shared(Z);
    if (tid < 4) Z[tid] = 0u;

    // W -> shared memory with the block swizzle.
    for (int i = tid; i < np * C; i += NT) {
        const int j = i / C, c = i - j * C;
        const int pc = c;
#pragma unroll
        for (int u = 0; u < WC; ++u) W[j * nw + pc * WC + u] = __ldg(wb + (int64_t)j * nw + c * WC + u);
    }
    __syncthreads();

    const int64_t nprobe = list ? (int64_t)*list_count : k;
    for (int64_t pi = (int64_t)blockIdx.x * NT + tid; pi < nprobe; pi += (int64_t)gridDim.x * NT) {
        const int64_t p = list ? list[pi] : pi;
        // ---- a1 ingest
        unsigned sym[kMaxC];
        const uint16_t *pr = probes + p * C;
        if (C == 8) {
            const uint4 q = __ldg(reinterpret_cast<const uint4 *>(pr));
            sym[0] = q.x & 0xffffu; sym[1] = q.x >> 16; sym[2] = q.y & 0xffffu; sym[3] = q.y >> 16;
            sym[4] = q.z & 0xffffu; sym[5] = q.z >> 16; sym[6] = q.w & 0xffffu; sym[7] = q.w >> 16;
        } else {
#pragma unroll
            for (int c = 0; c < kMaxC; ++c) sym[c] = (c < C) ? (unsigned)__ldg(pr + c) : 0u;
        }
        unsigned emask = 0, bad = 0;
#pragma unroll
        for (int c = 0; c < kMaxC; ++c) {
            if (c < C) {
                if (sym[c] == kErased) emask |= 1u << c;
                else if (sym[c] >= (unsigned)s.L) bad = 1;
            }
        }
        uint32_t *out = out_state + p * nw;
        if (bad) {
            for (int w = 0; w < nw; ++w) out[w] = 0u;
            out_iters[p] = 0;
            out_status[p] = GB_INVALID;
            continue;
        }
        const unsigned scope = (RULE == GB_SUM_OF_MAX) ? ((1u << C) - 1u) : emask;   // in-scope clusters
        // slot list: erased clusters (hybrid) or all clusters (SOM); 4 bits each
        unsigned slots = 0, nslot = 0;
#pragma unroll
        for (int c = 0; c < kMaxC; ++c) {
            if (c < C && (RULE == GB_SUM_OF_MAX || ((emask >> c) & 1u))) {
                slots |= (unsigned)c << (4 * nslot);
                ++nslot;
            }
        }
        // rotate the slot list by a lane-dependent amount: lanes of a quarter-warp then
        // work on different target clusters at the same static slot, which spreads
        // their bit-row block reads over the shared-memory bank groups
        if (nslot > 1) {
            const unsigned rot = (unsigned)(tid & 7) % nslot;
            const unsigned bits = 4u * nslot;
            const unsigned msk = bits >= 32u ? 0xffffffffu : ((1u << bits) - 1u);
            if (rot) slots = ((slots >> (4u * rot)) | (slots << (bits - 4u * rot))) & msk;
        }
        if (MAXS < kMaxC && (int)nslot > MAXS) {   // needs the wide-slot instance
            ovf[atomicAdd(ovf_count, 1ull)] = p;
            continue;
        }
        // ---- a5 prune / init -> X.  Slots are a static unroll (their count is
        // uniform across a warp when e is); the known clusters are walked in a
        // dynamic loop of C-e trips, one bit row per known neuron.
        uint64_t sp_lo = 0, sp_hi = 0;   // symbols packed 16 bits per cluster
#pragma unroll
        for (int c = 0; c < kMaxC; ++c) {
            if (c < 4) sp_lo |= (uint64_t)(sym[c] & 0xffffu) << (16 * c);
            else sp_hi |= (uint64_t)(sym[c] & 0xffffu) << (16 * (c - 4));
        }
        // known rows: ra[kk] = smem address of row (kc, p_kc)
        uint32_t ra[kMaxC];
        // bit t*WC+u set <=> word u of slot t is non-zero (lets the push skip empty words)
        uint32_t nzall = 0u;
        // bit t set <=> slot t holds every real neuron of its cluster (MAXS = 8 instance): a push
        // from it covers exactly the cluster union Wu (one load; seal builds Wu)
        uint32_t fullm = 0u;
        // 4-slot instance: the slot states live in registers (static slot indices)
        uint32_t xr[MAXS == 4 ? 4 : 1][WC];
        unsigned nk = 0;
        if (RULE == GB_HYBRID) {
            unsigned km = (~emask) & ((1u << C) - 1u);
            nk = __popc(km);
#pragma unroll
            for (int kk = 0; kk < kMaxC; ++kk) {
                const unsigned kc = __ffs(km) - 1;
                km &= km - 1u;
                const unsigned sk = (unsigned)(((kc < 4) ? sp_lo : sp_hi) >> (16 * (kc & 3))) & 0xffffu;
                ra[kk] = w_s + (kc * LP + sk) * rowB;
            }
        }
#pragma unroll
        for (int t = 0; t < MAXS; ++t) {
            if (t < (int)nslot) {
                const unsigned c = (slots >> (4 * t)) & 15u;
                uint32_t x[WC];
                if ((emask >> c) & 1u) {
#pragma unroll
                    for (int u = 0; u < WC; ++u) x[u] = real_mask_u(s.L, u);
                    if (RULE == GB_HYBRID) {
                        const uint32_t cb = c * BB;
#pragma unroll
                        for (int kk = 0; kk < kMaxC; ++kk) {
                            if (kk < (int)nk) {
                                uint32_t r[WC];
                                lds_block<WC>(ra[kk] + cb, r);
#pragma unroll
                                for (int u = 0; u < WC; ++u) x[u] &= r[u];
                            }
                        }
                    }
                } else {
                    const unsigned sc = (unsigned)(((c < 4) ? sp_lo : sp_hi) >> (16 * (c & 3))) & 0xffffu;
#pragma unroll
                    for (int u = 0; u < WC; ++u) x[u] = ((sc >> 5) == (unsigned)u) ? (1u << (sc & 31)) : 0u;
                }
                bool full = true;
#pragma unroll
                for (int u = 0; u < WC; ++u) {
                    if constexpr (MAXS == 4) xr[t][u] = x[u];
                    else X[(t * WC + u) * NT + tid] = x[u];
                    if (x[u]) nzall |= 1u << (t * WC + u);
                    full &= x[u] == real_mask_u(s.L, u);
                }
                if (full) fullm |= 1u << t;
            }
        }

        int it = 0;
        int status = GB_MAX_ITERS;
        if (RULE == GB_HYBRID && nslot == 0) {
            status = GB_CONVERGED;
        } else {
            // ---- a6 rounds.  From round 2 on only the pairs whose source slot changed in the
            // previous round are evaluated: a pair whose source kept its candidates removes
            // nothing (after the round that last evaluated it, the target's candidates lie inside
            // the OR of the rows it read, and those rows are still candidates).
            uint32_t chg = 0xFFu;
            if constexpr (MAXS == 4) {
                while (it < T) {
                    uint32_t xn[4][WC];
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        if (t < (int)nslot) {
                            const uint32_t ckey = (slots >> (4 * t)) & 15u;
                            uint32_t alive[WC];
                            uint32_t any = 0;
#pragma unroll
                            for (int u = 0; u < WC; ++u) {
                                alive[u] = xr[t][u];
                                any |= alive[u];
                            }
#pragma unroll
                            for (int sidx = 0; sidx < 4; ++sidx) {
                                if (sidx < (int)nslot && sidx != t && any && ((chg >> sidx) & 1u)) {
                                    const uint32_t c2 = (slots >> (4 * sidx)) & 15u;
                                    uint32_t h[WC];
#pragma unroll
                                    for (int u = 0; u < WC; ++u) h[u] = 0u;
                                    uint32_t miss = any;
                                    uint32_t nzs = (nzall >> (sidx * WC)) & ((1u << WC) - 1u);
                                    uint32_t u2 = 0, cur = 0, base = 0;
                                    while (miss) {
                                        if (!cur) {
                                            if (!nzs) break;   // source exhausted
                                            u2 = __ffs(nzs) - 1;
                                            nzs &= nzs - 1u;
                                            cur = xr[sidx][0];
#pragma unroll
                                            for (int u = 1; u < WC; ++u)
                                                if (u2 == (uint32_t)u) cur = xr[sidx][u];
                                            base = w_s + (c2 * LP + u2 * 32) * rowB;
                                        }
                                        const uint32_t b1 = __ffs(cur) - 1;
                                        cur &= cur - 1u;
                                        const uint32_t b2 = __ffs(cur) - 1;
                                        cur &= cur - 1u;
                                        uint32_t r[WC], r2[WC];
                                        lds_block<WC>(base + b1 * rowB + ckey * BB, r);
                                        const uint32_t a2 = base + b2 * rowB + ckey * BB;
                                        lds_block<WC>(b2 == 0xffffffffu ? zaddr : a2, r2);
                                        miss = 0u;
#pragma unroll
                                        for (int u = 0; u < WC; ++u) {
                                            h[u] |= r[u] | r2[u];
                                            miss |= alive[u] & ~h[u];
                                        }
                                    }
                                    any = 0u;
#pragma unroll
                                    for (int u = 0; u < WC; ++u) {
                                        alive[u] &= h[u];
                                        any |= alive[u];
                                    }
                                }
                            }
#pragma unroll
                            for (int u = 0; u < WC; ++u) xn[t][u] = alive[u];
                        }
                    }
                    bool changed = false;
                    chg = 0u;
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        if (t < (int)nslot) {
#pragma unroll
                            for (int u = 0; u < WC; ++u) {
                                if (xr[t][u] != xn[t][u]) chg |= 1u << t;
                                changed |= (xr[t][u] != xn[t][u]);
                                xr[t][u] = xn[t][u];
                                if (!xn[t][u]) nzall &= ~(1u << (t * WC + u));
                            }
                        }
                    }
                    ++it;
                    if (!changed) { status = GB_CONVERGED; break; }
                }
            } else
            while (it < T) {
                uint32_t xn[MAXS][WC];
                bool changed = false;
#pragma unroll
                for (int t = 0; t < MAXS; ++t) {
                    if (t < (int)nslot) {
                        const int c = (slots >> (4 * t)) & 15;
                        uint32_t alive[WC];
                        uint32_t any = 0;
#pragma unroll
                        for (int u = 0; u < WC; ++u) {
                            alive[u] = X[(t * WC + u) * NT + tid];
                            any |= alive[u];
                        }
                        for (unsigned sidx = 0; sidx < nslot && any; ++sidx) {
                            if ((int)sidx == t || !((chg >> sidx) & 1u)) continue;
                            const int c2 = (slots >> (4 * sidx)) & 15;
                            uint32_t h[WC];
#pragma unroll
                            for (int u = 0; u < WC; ++u) h[u] = 0u;
                            uint32_t miss = any;
                            const uint32_t ckey = (uint32_t)c;
                            if ((fullm >> sidx) & 1u) {   // full source cluster: H = Wu[c2][c]
                                const uint32_t *ub = wu + (size_t)(c2 * C + c) * WC;
#pragma unroll
                                for (int u = 0; u < WC; ++u) h[u] = __ldg(ub + u);
                                miss = 0u;
                            }
                            // one loop over the source's candidate words (a lane that runs out of
                            // word u2 moves on inside the same loop: no per-word divergent tails)
                            const uint32_t *xs = X + (sidx * WC) * NT + tid;
                            uint32_t nzs = (nzall >> (sidx * WC)) & ((1u << WC) - 1u);
                            uint32_t u2 = 0, cur = 0;
                            uint32_t base = 0;   // row j = c2*LP + u2*32 + b
                            while (miss) {
                                if (!cur) {
                                    if (!nzs) break;   // source exhausted
                                    u2 = __ffs(nzs) - 1;
                                    nzs &= nzs - 1u;
                                    cur = xs[u2 * NT];
                                    base = w_s + (uint32_t)(c2 * LP + u2 * 32) * rowB;
                                }
                                // two rows per check: the second is the zero block when only
                                // one candidate is left in the word (branch-free, ILP 2);
                                const uint32_t b1 = __ffs(cur) - 1;
                                cur &= cur - 1u;
                                const uint32_t b2 = __ffs(cur) - 1;
                                cur &= cur - 1u;
                                uint32_t r[WC], r2[WC];
                                lds_block<WC>(base + b1 * rowB + ckey * BB, r);
                                const uint32_t a2 = base + b2 * rowB + ckey * BB;
                                lds_block<WC>(b2 == 0xffffffffu ? zaddr : a2, r2);
                                miss = 0u;
#pragma unroll
                                for (int u = 0; u < WC; ++u) {
                                    h[u] |= r[u] | r2[u];
                                    miss |= alive[u] & ~h[u];
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
                        for (int u = 0; u < WC; ++u) xn[t][u] = alive[u];
                    }
                }
                chg = 0u;
#pragma unroll
                for (int t = 0; t < MAXS; ++t) {
                    if (t < (int)nslot) {
#pragma unroll
                        for (int u = 0; u < WC; ++u) {
                            uint32_t *a = &X[(t * WC + u) * NT + tid];
                            if (*a != xn[t][u]) chg |= 1u << t;
                            changed |= (*a != xn[t][u]);
                            *a = xn[t][u];
                            if (!xn[t][u]) nzall &= ~(1u << (t * WC + u));
                            if (xn[t][u] != real_mask_u(s.L, u)) fullm &= ~(1u << t);
                        }
                    }
                }
                ++it;
                if (!changed) { status = GB_CONVERGED; break; }
            }
        }
        // ---- a7 output: clusters outside the scope are the known one-hot; slots come from X
#pragma unroll
        for (int c = 0; c < kMaxC; ++c) {
            if (c < C && !((scope >> c) & 1u)) {
                const unsigned sc = (unsigned)(((c < 4) ? sp_lo : sp_hi) >> (16 * (c & 3))) & 0xffffu;
                uint32_t v[WC];
#pragma unroll
                for (int u = 0; u < WC; ++u) v[u] = ((sc >> 5) == (unsigned)u) ? (1u << (sc & 31)) : 0u;
                if constexpr (WC == 4) {
                    *reinterpret_cast<uint4 *>(out + c * WC) = make_uint4(v[0], v[1], v[2], v[3]);
                } else {
#pragma unroll
                    for (int u = 0; u < WC; ++u) out[c * WC + u] = v[u];
                }
            }
        }
#pragma unroll
        for (int t = 0; t < MAXS; ++t) {
            if (t < (int)nslot) {
                const unsigned c = (slots >> (4 * t)) & 15u;
                uint32_t v[WC];
#pragma unroll
                for (int u = 0; u < WC; ++u) {
                    if constexpr (MAXS == 4) v[u] = xr[t][u];
                    else v[u] = X[(t * WC + u) * NT + tid];
                }
                if constexpr (WC == 4) {
                    *reinterpret_cast<uint4 *>(out + c * WC) = make_uint4(v[0], v[1], v[2], v[3]);
                } else {
#pragma unroll
                    for (int u = 0; u < WC; ++u) out[c * WC + u] = v[u];
                }
            }
        }
        out_iters[p] = (uint16_t)it;
        out_status[p] = (uint8_t)status;
    }
}

constexpr int kWideThreads = 640;     // MAXS = 8
#ifndef GB_SOM_THREADS
#define GB_SOM_THREADS 768
#endif
constexpr int kSomThreads = GB_SOM_THREADS;   // sum-of-max instance (MAXS = 8)
constexpr int kNarrowThreads = GB_NARROW_THREADS;   // MAXS = 4

size_t smem_bytes(const Shape &s, int wc, int maxs, int nt) {
    // the 4-slot instance keeps its slot states in registers (no X area)
    return (size_t)s.np * s.nw * 4 + (maxs == 4 ? 0 : (size_t)maxs * wc * nt * 4) + 16;
}

template <int WC, int RULE, int MAXS, int NT>
cudaError_t launch_t(Call &cl, const uint16_t *probes, int64_t k, int max_iters, uint32_t *state,
                     uint16_t *iters, uint8_t *status, const int64_t *list, const unsigned long long *list_count,
                     int64_t *ovf, unsigned long long *ovf_count) {
    const gb_net *net = cl.net;
    const Shape &s = net->s;
    const size_t smem = smem_bytes(s, WC, MAXS, NT);
    auto fn = decode_smem_kernel<WC, RULE, MAXS, NT>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int64_t grid = list ? net->sm_count : (k + NT - 1) / NT;
    if (grid > net->sm_count) grid = net->sm_count;
    fn<<<(unsigned)grid, NT, smem, cl.st>>>(s, net->wb, probes, k, max_iters, state, iters, status, list, list_count,
                                            ovf, ovf_count, wu_of(net, net->seal_gen));
    cl.launched();
    return cudaGetLastError();
}

template <int WC, int RULE>
cudaError_t launch_rule(Call &cl, const uint16_t *probes, int64_t k, int max_iters, uint32_t *state,
                        uint16_t *iters, uint8_t *status) {
    if (RULE == GB_SUM_OF_MAX)   // every probe needs all C slots
        return launch_t<WC, RULE, 8, kSomThreads>(cl, probes, k, max_iters, state, iters, status, nullptr,
                                                  nullptr, nullptr, nullptr);
    if (cl.net->s.C <= 4)
        return launch_t<WC, RULE, 8, kWideThreads>(cl, probes, k, max_iters, state, iters, status, nullptr,
                                                   nullptr, nullptr, nullptr);
    // hybrid: probes with e <= 4 on the narrow (more threads) instance, the rest queued
    // for the wide one (list mode)
    int64_t *ovf = cl.ovf(k);
    unsigned long long *cnt = cl.counters();
    if (!ovf || !cnt) return cl.err;
    cudaError_t e = cudaErrorNotSupported;
    if (WC == 4 && RULE == GB_HYBRID && decode_hyb8_supported(cl.net, RULE, k, state))
        e = launch_decode_hyb8(cl, probes, k, max_iters, state, iters, status, ovf, cnt + 1);
    if (e == cudaErrorNotSupported)   // other shapes, or no tensor map for this output buffer
        e = launch_t<WC, RULE, 4, kNarrowThreads>(cl, probes, k, max_iters, state, iters, status, nullptr, nullptr,
                                                  ovf, cnt + 1);
    if (e != cudaSuccess) return e;
    return launch_t<WC, RULE, 8, kWideThreads>(cl, probes, k, max_iters, state, iters, status, ovf, cnt + 1,
                                               nullptr, nullptr);
}

}  // namespace

bool decode_smem_supported(const Shape &s, int rule) {
    if (s.C > kMaxC || s.np > 1024 || rule == GB_SUM_OF_SUM) return false;
    if (s.Wc != 1 && s.Wc != 2 && s.Wc != 4) return false;
    return smem_bytes(s, s.Wc, 8, kWideThreads) <= 227 * 1024 &&
           smem_bytes(s, s.Wc, 8, kSomThreads) <= 227 * 1024 &&
           smem_bytes(s, s.Wc, 4, kNarrowThreads) <= 227 * 1024;
}

// Returns cudaErrorNotSupported when the shape does not fit this kernel.
cudaError_t launch_decode_smem(Call &cl, const uint16_t *probes, int64_t k, int rule, int max_iters,
                               uint32_t *state, uint16_t *iters, uint8_t *status) {
    const Shape &s = cl.net->s;
    if (!decode_smem_supported(s, rule)) return cudaErrorNotSupported;
    const bool hyb = (rule == GB_HYBRID);
    switch (s.Wc) {
        case 1: return hyb ? launch_rule<1, GB_HYBRID>(cl, probes, k, max_iters, state, iters, status)
                           : launch_rule<1, GB_SUM_OF_MAX>(cl, probes, k, max_iters, state, iters, status);
        case 2: return hyb ? launch_rule<2, GB_HYBRID>(cl, probes, k, max_iters, state, iters, status)
                           : launch_rule<2, GB_SUM_OF_MAX>(cl, probes, k, max_iters, state, iters, status);
        default: return hyb ? launch_rule<4, GB_HYBRID>(cl, probes, k, max_iters, state, iters, status)
                            : launch_rule<4, GB_SUM_OF_MAX>(cl, probes, k, max_iters, state, iters, status);
    }
}

}  // namespace gb
