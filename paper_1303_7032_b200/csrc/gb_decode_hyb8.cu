// gb_decode_hyb8.cu -- hybrid decode (Alg. 2) specialised for the metric
// shape: C = 8 clusters of 97..128 neurons (4 words per cluster block), probes
// with at most 4 erased clusters.  Same method and result as
// decode_smem_kernel (gb_decode_smem.cu, which keeps every other shape and the
// probes with e > 4); what differs is how the work maps to the SM:
//
//  * compile-time C / block size: no per-cluster predicates or runtime loops
//    in ingest, prune and output;
//  * the push of one (source -> target) pair reads candidate rows several at a
//    time instead of walking the source's bits one at a time: when W is dense
//    (decode_hyb8r_kernel) one row per 16-neuron half-word of the source, in a
//    shared-memory layout where those loads never bank-conflict; when sparse
//    (decode_hyb8_kernel) a loop of "the lowest remaining candidate of every
//    word"; each step runs only while some target candidate is still
//    uncovered (bail-out-early), and every source candidate is read
//    at most once, so the cover H is the same OR of rows;
//  * output through a TMA tensor store: each warp writes its 32 probes'
//    128-byte states into a 4 KiB shared-memory box in the 128-byte swizzle
//    (16-byte chunk c of row r at chunk c ^ (r & 7): the lanes of a
//    quarter-warp hit 8 different bank groups) and one lane stores the box
//    with cp.async.bulk.tensor (rows >= k are clipped by the tensor map).
//
// Method: a1 ingest, a5 prune (X^0 of an erased cluster = AND of
// the known neurons' rows, Alg. 2 L2-5 / Thm 4), a6 synchronous sum-of-max
// rounds on the erased clusters with the known clusters frozen (Eq.(6)-(7),
// Alg. 2 L8-13), a7 output (state, rounds incl. the confirming one, status).
#include <cuda.h>
#include <stdlib.h>

#include "gb_internal.h"

namespace gb {
namespace {

// 768 threads (24 warps, 80 registers).  Measured (round 2, same-box A/B): 1024 threads at 64
// registers with half-box output staging (W + 32 boxes of 2 KiB fit 227 KiB) is slower -- C3
// 1.18 vs 1.04 ms, C2 hybrid (10^7) 4.74 vs 3.33 ms: the register cap serialises the staged
// loads, and each half box waits for the TMA unit to read the previous one.
constexpr int kNT = 768;            // threads per CTA (one probe each)

constexpr int kWarps = kNT / 32;
constexpr int kRowB = 128;          // bytes per W bit row (8 clusters x 16 B)
constexpr int kClusterB = 128 * kRowB;   // bytes of the 128 rows of one cluster
constexpr int kBoxRows = 32;             // probes per TMA output box (one warp)
constexpr uint32_t kStageB = kBoxRows * 128;   // one warp's output staging box
constexpr size_t kSmem = 1024 + 1024 * kRowB + (size_t)kWarps * kStageB;

__device__ __forceinline__ void lds4(uint32_t a, uint32_t (&v)[4]) {
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(a));
}
__device__ __forceinline__ void sts4(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
// Predicated load: v unchanged (zero-initialised by the caller) when p == 0.  No branch, so
// the loads of one stage issue back to back and their latencies overlap (with `if (x) lds4`
// the compiler emitted one branch per row and each row's OR waited for its load).
__device__ __forceinline__ void lds4p(uint32_t p, uint32_t a, uint32_t (&v)[4]) {
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %4, 0;\n\t@q ld.shared.v4.u32 {%0,%1,%2,%3}, [%5];\n\t}"
        : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3])
        : "r"(p), "r"(a));
}
__device__ __forceinline__ uint32_t lowbit(uint32_t x) { return __ffs(x) - 1; }
// Sparse W (density <= 0.65, counted by seal): one loop whose every step reads the lowest
// remaining candidate row of each word (up to 4 loads in flight) until the target is covered or
// the source exhausted -- few candidates per cluster, many of them dying.  W in row-major order
// (a row block lies in the bank group of its target cluster).  Same-box A/B (round 2, 10^7
// probes, hybrid, c=8 l=128): M=5k (density 0.26) 2.24 -> 1.74 ms with the loop instead of the
// round-1 stages, M=10k (0.46) 4.11 -> 3.32, M=15k (0.60) 1.19 -> 1.08; the rotated-layout kernel
// below is slower there (M=5k 2.48, M=10k 4.98, M=15k 1.09 ms): with ~2-17 candidates per
// erased cluster most of its 8 half-word loads are empty.
__global__ void __launch_bounds__(kNT, 1)
decode_hyb8_kernel(const uint32_t *__restrict__ wb, const uint16_t *__restrict__ probes, int64_t k, int L,
                   int T, const __grid_constant__ CUtensorMap omap, uint16_t *__restrict__ out_iters,
                   uint8_t *__restrict__ out_status, int64_t *__restrict__ ovf,
                   unsigned long long *__restrict__ ovf_count) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t sbase = ((uint32_t)__cvta_generic_to_shared(smem_raw) + 1023u) & ~1023u;
    const uint32_t w_s = sbase;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t stg = w_s + 1024 * kRowB + warp * kStageB;
    const uint32_t my_row = stg + (lane & (kBoxRows - 1)) * 128;
    const uint32_t sw = (uint32_t)(lane & 7);

    // W bit rows -> shared memory (row-major, 128 B per row)
    for (int i = tid; i < 1024 * kRowB / 16; i += kNT) {
        const uint4 v = __ldg(reinterpret_cast<const uint4 *>(wb) + i);
        sts4(w_s + i * 16, v.x, v.y, v.z, v.w);
    }
    __syncthreads();
    uint32_t rmask[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int nb = min(32, max(0, L - u * 32));
        rmask[u] = nb == 32 ? 0xffffffffu : ((1u << nb) - 1u);
    }

    for (int64_t pb = ((int64_t)blockIdx.x * kWarps + warp) * 32; pb < k; pb += (int64_t)gridDim.x * kNT) {
        const int64_t p = pb + lane;
        // ---- a1 ingest
        uint32_t sym[8];
        uint32_t emask = 0, bad = 0, live = 0;
        if (p < k) {
            const uint4 q = __ldg(reinterpret_cast<const uint4 *>(probes + p * 8));
            const uint32_t w4[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                sym[2 * h] = w4[h] & 0xffffu;
                sym[2 * h + 1] = w4[h] >> 16;
            }
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                if (sym[c] == kErased) emask |= 1u << c;
                else if (sym[c] >= (uint32_t)L) bad = 1;
            }
            live = 1;
        } else {
#pragma unroll
            for (int c = 0; c < 8; ++c) sym[c] = 0;
        }
        const uint32_t nslot = __popc(emask);
        if (live && !bad && nslot > 4) {   // needs more slots: decoded by decode_smem_kernel (list mode)
            ovf[atomicAdd(ovf_count, 1ull)] = p;
            live = 0;
        }
        const bool work = live && !bad;
        // slot list: erased clusters ascending, 4 bits each, rotated by (lane & 7) % nslot so
        // the lanes of a quarter-warp start on different target clusters
        uint32_t slots = 0;
        {
            uint32_t em = emask;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                if (em) {
                    slots |= (uint32_t)(__ffs(em) - 1) << (4 * t);
                    em &= em - 1u;
                }
            }
            const uint32_t tab = nslot == 4 ? 0x32103210u : nslot == 3 ? 0x10210210u : nslot == 2 ? 0x10101010u : 0u;
            const uint32_t rot = (tab >> (4 * sw)) & 15u;
            if (rot) {
                const uint32_t bits = 4u * nslot;
                slots = ((slots >> (4u * rot)) | (slots << (bits - 4u * rot))) & ((1u << bits) - 1u);
            }
        }
        // ---- a5 prune: X^0_c = AND over known clusters kc of block c of row (kc, p_kc)
        uint32_t xr[4][4];
        {
            uint32_t ra[8];
            uint32_t km = (~emask) & 0xffu;
            uint64_t sp_lo = 0, sp_hi = 0;   // symbols packed 16 bits per cluster
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                sp_lo |= (uint64_t)sym[c] << (16 * c);
                sp_hi |= (uint64_t)sym[c + 4] << (16 * c);
            }
            auto next_row = [&]() {   // row address of the next known cluster
                const uint32_t kc = km ? (uint32_t)(__ffs(km) - 1) : 0u;
                km &= km - 1u;
                const uint32_t sk = (uint32_t)(((kc < 4) ? sp_lo : sp_hi) >> (16 * (kc & 3))) & 0xffffu;
                return w_s + kc * kClusterB + sk * kRowB;
            };
            const uint32_t nk = 8u - nslot;
            // e <= 4 here, so at least 4 known clusters: their rows unconditionally, the others
            // (e < 4) in a second pass (same-box A/B: C3 0.962 -> 0.931 ms, M=30k 0.856 -> 0.830)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) ra[kk] = next_row();
#pragma unroll
            for (int t = 0; t < 4; ++t) {
#pragma unroll
                for (int u = 0; u < 4; ++u) xr[t][u] = 0u;
                if (work && t < (int)nslot) {
                    const uint32_t ct = (slots >> (4 * t)) & 15u;
#pragma unroll
                    for (int u = 0; u < 4; ++u) xr[t][u] = rmask[u];
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        uint32_t r[4];
                        lds4(ra[kk] + (ct << 4), r);
#pragma unroll
                        for (int u = 0; u < 4; ++u) xr[t][u] &= r[u];
                    }
                }
            }
            if (work && nk > 4) {
#pragma unroll
                for (int kk = 4; kk < 8; ++kk) ra[kk] = next_row();
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    if (t < (int)nslot) {
                        const uint32_t ct = (slots >> (4 * t)) & 15u;
#pragma unroll
                        for (int kk = 4; kk < 8; ++kk) {
                            if (kk < (int)nk) {
                                uint32_t r[4];
                                lds4(ra[kk] + (ct << 4), r);
#pragma unroll
                                for (int u = 0; u < 4; ++u) xr[t][u] &= r[u];
                            }
                        }
                    }
                }
            }
        }
        // ---- a6 synchronous rounds on the erased clusters (known clusters frozen)
        int it = 0;
        int status = GB_MAX_ITERS;
        if (!work || nslot == 0) {
            status = GB_CONVERGED;
        } else {
            // slots whose candidates changed in the previous round (all, before round 1): a pair
            // whose source kept its candidates removes nothing (after the round that last
            // evaluated it, the target's candidates lie inside the OR of the rows it read, and
            // those rows are still candidates), so only pairs from changed sources are evaluated.
            // Same-box A/B (10^7 probes, c=8 l=128): M=5k 1.687 -> 1.546 ms, M=10k 3.265 -> 2.721,
            // M=15k unchanged; the rotated kernel (1-2 rounds at its densities) does not gain
            // (C3 0.772 vs 0.778, M=30k 0.683 vs 0.694) and keeps evaluating every pair
            uint32_t chg = 0xFu;
            while (it < T) {
                uint32_t xn[4][4];
#pragma unroll
                for (int t = 0; t < 4; ++t) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) xn[t][u] = 0u;
                    if (t < (int)nslot) {
                        const uint32_t ct = (slots >> (4 * t)) & 15u;
                        uint32_t alive[4];
                        uint32_t any = 0u;
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            alive[u] = xr[t][u];
                            any |= alive[u];
                        }
#pragma unroll
                        for (int sidx = 0; sidx < 4; ++sidx) {
                            if (sidx != t && sidx < (int)nslot && any && ((chg >> sidx) & 1u)) {
                                // block c_t of row (c2, 32u + b): rb + (32u + b) * 128
                                const uint32_t rb = w_s + ((slots >> (4 * sidx)) & 15u) * kClusterB + (ct << 4);
                                uint32_t h[4] = {0u, 0u, 0u, 0u};
                                // sparse: the lowest remaining candidate row of every word per
                                // step (4 loads in flight) until covered or exhausted
                                uint32_t rem[4];
#pragma unroll
                                for (int u = 0; u < 4; ++u) rem[u] = xr[sidx][u];
                                uint32_t miss;
                                do {
                                    uint32_t r[4][4];
#pragma unroll
                                    for (int u = 0; u < 4; ++u) {
                                        const uint32_t x = rem[u];
#pragma unroll
                                        for (int v = 0; v < 4; ++v) r[u][v] = 0u;
                                        lds4p(x, rb + (u * 32 + lowbit(x)) * kRowB, r[u]);
                                        rem[u] = x & (x - 1u);
                                    }
                                    miss = 0u;
#pragma unroll
                                    for (int v = 0; v < 4; ++v) {
                                        h[v] |= (r[0][v] | r[1][v]) | (r[2][v] | r[3][v]);
                                        miss |= alive[v] & ~h[v];
                                    }
                                } while (miss && ((rem[0] | rem[1]) | (rem[2] | rem[3])));
                                any = 0u;
#pragma unroll
                                for (int v = 0; v < 4; ++v) {
                                    alive[v] &= h[v];
                                    any |= alive[v];
                                }
                            }
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u) xn[t][u] = alive[u];
                    }
                }
                bool changed = false;
                chg = 0u;
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    bool ct_changed = false;
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        ct_changed |= (xr[t][u] != xn[t][u]);
                        xr[t][u] = xn[t][u];
                    }
                    changed |= ct_changed;
                    chg |= (ct_changed ? 1u : 0u) << t;
                }
                ++it;
                if (!changed) {
                    status = GB_CONVERGED;
                    break;
                }
            }
        }
        // ---- a7 output
        if (live) {
            out_iters[p] = (uint16_t)it;
            out_status[p] = (uint8_t)(bad ? GB_INVALID : status);
        }
        // two half boxes: lanes 0-15, then lanes 16-31 (each waits until the TMA unit has
        // read the previous box out of the staging buffer)
#pragma unroll
        for (int half = 0; half < 32 / kBoxRows; ++half) {
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
            if (live && (lane / kBoxRows) == half) {
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    if (bad || !((emask >> c) & 1u)) {
                        const uint32_t s = bad ? 0xffffffffu : sym[c];
                        const uint32_t b = 1u << (s & 31u), w = s >> 5;
                        sts4(my_row + (((uint32_t)c ^ sw) << 4), w == 0 ? b : 0u, w == 1 ? b : 0u,
                             w == 2 ? b : 0u, w == 3 ? b : 0u);
                    }
                }
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    if (!bad && t < (int)nslot) {
                        const uint32_t c = (slots >> (4 * t)) & 15u;
                        sts4(my_row + ((c ^ sw) << 4), xr[t][0], xr[t][1], xr[t][2], xr[t][3]);
                    }
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                asm volatile(
                    "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                    ::"l"((uint64_t)&omap), "r"(0), "r"((int)pb + half * kBoxRows), "r"(stg) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ---- rotated-layout kernel (dense W) ------------------------------------------------------------
// The push reads one row per 16-neuron half-word of the source's candidates (8 rows per pair, in
// flight together; at C3 ~32 candidates per erased cluster, so the 8 rows cover the target in
// ~99.8% of the pairs and the rest are read one at a time).  W is laid out in shared memory so
// that those 8 loads never conflict: row i's block t sits in 16-byte chunk (i >> 4) of its line,
//   addr(c, i, t) = c * 17 KiB + ((i & 15) + 1) * 1 KiB + t * 128 + (i >> 4) * 16,
// i.e. the bank group of a row block is the half-word its neuron lies in, whatever the target.
// Lane q (= lane & 7) issues half-word (k + q) & 7 as its k-th load, so the 8 lanes of a
// quarter-warp always hit 8 different bank groups.  Group 0 of every cluster is zero: an empty
// half-word reads it (address offset __ffs(0) = 0), so the loads need no predicate and no zeroed
// destination registers.  The prune's loads (known rows) keep random bank groups.
constexpr int kGrpB = 1024;                  // one (cluster, i & 15) group: 8 lines of 128 B
constexpr int kClusterBr = 17 * kGrpB;       // group 0 = zeros, groups 1..16 = i & 15 = 0..15
constexpr int kNTr = 512;                    // threads per CTA (one probe each)
constexpr int kWarpsR = kNTr / 32;
constexpr size_t kSmemR = 1024 + 8 * (size_t)kClusterBr + (size_t)kWarpsR * kStageB;

template <int NR>
__global__ void __launch_bounds__(kNTr, 1)
decode_hyb8r_kernel(const uint32_t *__restrict__ wb, const uint16_t *__restrict__ probes, int64_t k, int L,
                    int T, const __grid_constant__ CUtensorMap omap, uint16_t *__restrict__ out_iters,
                    uint8_t *__restrict__ out_status, int64_t *__restrict__ ovf,
                    unsigned long long *__restrict__ ovf_count) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t sbase = ((uint32_t)__cvta_generic_to_shared(smem_raw) + 1023u) & ~1023u;
    const uint32_t w_s = sbase;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t stg = w_s + 8 * kClusterBr + warp * kStageB;   // 1024-aligned (128-B swizzle)
    const uint32_t my_row = stg + lane * 128;
    const uint32_t sw = (uint32_t)(lane & 7);

    // W bit rows -> shared memory in the rotated layout: smem chunk g = (c, group, t, chunk),
    // consecutive threads store consecutive chunks (conflict-free)
    for (int g = tid; g < 8 * (kClusterBr / 16); g += kNTr) {
        const int c = g / (kClusterBr / 16), rest = g - c * (kClusterBr / 16), grp = rest >> 6;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (grp) {
            const int i = (rest & 7) * 16 + grp - 1, t = (rest >> 3) & 7;
            v = __ldg(reinterpret_cast<const uint4 *>(wb) + ((c * 128 + i) * 8 + t));
        }
        sts4(w_s + g * 16, v.x, v.y, v.z, v.w);
    }
    __syncthreads();
    uint32_t rmask[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int nb = min(32, max(0, L - u * 32));
        rmask[u] = nb == 32 ? 0xffffffffu : ((1u << nb) - 1u);
    }
    // lane constants of the source rotation: the k-th load reads half-word (k + q) & 7
    const uint32_t q = (uint32_t)(lane & 7);
    const bool rot1 = (q >> 1) & 1u, rot2 = (q >> 2) & 1u;
    const uint32_t rots = (q & 1u) * 16u;
    const uint32_t q16 = q << 4;
    auto qk = [&](int kk) { return (q16 + 16u * (uint32_t)kk) & 0x70u; };   // chunk of rotated half-word kk

    const int64_t stride = (int64_t)gridDim.x * kNTr;
    int64_t pb = ((int64_t)blockIdx.x * kWarpsR + warp) * 32;
    uint4 qnext = make_uint4(0u, 0u, 0u, 0u);
    if (pb + lane < k) qnext = __ldg(reinterpret_cast<const uint4 *>(probes + (pb + lane) * 8));
    for (; pb < k; pb += stride) {
        const int64_t p = pb + lane;
        // ---- a1 ingest (the next batch's probe is loaded one batch ahead)
        const uint32_t w4[4] = {qnext.x, qnext.y, qnext.z, qnext.w};
        if (p + stride < k) qnext = __ldg(reinterpret_cast<const uint4 *>(probes + (p + stride) * 8));
        auto sym = [&](int c) { return (w4[c >> 1] >> (16 * (c & 1))) & 0xffffu; };
        uint32_t emask = 0, bad = 0, live = 0;
        if (p < k) {
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                if (sym(c) == kErased) emask |= 1u << c;
                else if (sym(c) >= (uint32_t)L) bad = 1;
            }
            live = 1;
        }
        const uint32_t nslot = __popc(emask);
        if (live && !bad && nslot > 4) {   // needs more slots: decoded by decode_smem_kernel (list mode)
            ovf[atomicAdd(ovf_count, 1ull)] = p;
            live = 0;
        }
        const bool work = live && !bad;
        uint32_t slots = 0;   // erased clusters ascending, 4 bits each
        {
            uint32_t em = emask;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                if (em) {
                    slots |= (uint32_t)(__ffs(em) - 1) << (4 * t);
                    em &= em - 1u;
                }
            }
        }
        // ---- a5 prune: X^0_c = AND over known clusters kc of block c of row (kc, p_kc)
        uint32_t xr[4][4];
        {
            uint32_t ra[8];
            uint32_t km = (~emask) & 0xffu;
            const uint64_t sp_lo = ((uint64_t)w4[1] << 32) | w4[0], sp_hi = ((uint64_t)w4[3] << 32) | w4[2];
            auto next_row = [&]() {
                const uint32_t kc = km ? (uint32_t)(__ffs(km) - 1) : 0u;
                km &= km - 1u;
                const uint32_t sk = (uint32_t)(((kc < 4) ? sp_lo : sp_hi) >> (16 * (kc & 3))) & 0x7fu;
                return w_s + kc * kClusterBr + ((sk & 15u) + 1u) * kGrpB + (sk >> 4) * 16u;
            };
            const uint32_t nk = 8u - nslot;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) ra[kk] = next_row();
#pragma unroll
            for (int t = 0; t < 4; ++t) {
#pragma unroll
                for (int u = 0; u < 4; ++u) xr[t][u] = 0u;
                if (work && t < (int)nslot) {
                    const uint32_t ct = (slots >> (4 * t)) & 15u;
#pragma unroll
                    for (int u = 0; u < 4; ++u) xr[t][u] = rmask[u];
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        uint32_t r[4];
                        lds4(ra[kk] + (ct << 7), r);
#pragma unroll
                        for (int u = 0; u < 4; ++u) xr[t][u] &= r[u];
                    }
                }
            }
            if (work && nk > 4) {
#pragma unroll
                for (int kk = 4; kk < 8; ++kk) ra[kk] = next_row();
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    if (t < (int)nslot) {
                        const uint32_t ct = (slots >> (4 * t)) & 15u;
#pragma unroll
                        for (int kk = 4; kk < 8; ++kk) {
                            if (kk < (int)nk) {
                                uint32_t r[4];
                                lds4(ra[kk] + (ct << 7), r);
#pragma unroll
                                for (int u = 0; u < 4; ++u) xr[t][u] &= r[u];
                            }
                        }
                    }
                }
            }
        }
        // ---- a6 synchronous rounds on the erased clusters (known clusters frozen)
        int it = 0;
        int status = GB_MAX_ITERS;
        if (!work || nslot == 0) {
            status = GB_CONVERGED;
        } else {
            while (it < T) {
                uint32_t xn[4][4];
#pragma unroll
                for (int t = 0; t < 4; ++t)
#pragma unroll
                    for (int u = 0; u < 4; ++u) xn[t][u] = xr[t][u];
#pragma unroll
                for (int s = 0; s < 4; ++s) {
                    if (s < (int)nslot) {
                        const uint32_t sb = w_s + ((slots >> (4 * s)) & 15u) * kClusterBr;
                        // the source's candidate bits rotated right by 16q: half-word kk of c is
                        // half-word (kk + q) & 7 of the source
                        uint32_t c[4];
                        {
                            uint32_t a[4], b[4];
#pragma unroll
                            for (int j = 0; j < 4; ++j) a[j] = rot1 ? xr[s][(j + 1) & 3] : xr[s][j];
#pragma unroll
                            for (int j = 0; j < 4; ++j) b[j] = rot2 ? a[(j + 2) & 3] : a[j];
#pragma unroll
                            for (int j = 0; j < 4; ++j) c[j] = __funnelshift_r(b[j], b[(j + 1) & 3], rots);
                        }
                        uint32_t off[NR];   // lowest candidate of each half-word (group 0 if none)
#pragma unroll
                        for (int kk = 0; kk < NR; ++kk) {
                            const uint32_t hw = (kk & 1) ? (c[kk >> 1] >> 16) : (c[kk >> 1] & 0xffffu);
                            off[kk] = qk(kk) + (uint32_t)__ffs(hw) * kGrpB;
                        }
#pragma unroll
                        for (int t = 0; t < 4; ++t) {
                            if (t != s && t < (int)nslot) {
                                const uint32_t pbase = sb + (((slots >> (4 * t)) & 15u) << 7);
                                uint32_t r[NR][4];
#pragma unroll
                                for (int kk = 0; kk < NR; ++kk) lds4(pbase + off[kk], r[kk]);
                                uint32_t h[4], miss = 0u;
#pragma unroll
                                for (int v = 0; v < 4; ++v) {
                                    h[v] = r[0][v];
#pragma unroll
                                    for (int kk = 1; kk < NR; ++kk) h[v] |= r[kk][v];
                                    miss |= xn[t][v] & ~h[v];
                                }
                                if (miss) {
                                    // the source's other candidates, a step at a time: each step reads the
                                    // next candidate of every half-word (8 loads in flight, still one bank
                                    // group per lane of a quarter-warp) until covered or exhausted
                                    uint32_t hw[8];
#pragma unroll
                                    for (int kk = 0; kk < 8; ++kk) {
                                        uint32_t x = (kk & 1) ? (c[kk >> 1] >> 16) : (c[kk >> 1] & 0xffffu);
                                        if (kk < NR) x &= x - 1u;
                                        hw[kk] = x;
                                    }
                                    while (miss && (((hw[0] | hw[1]) | (hw[2] | hw[3])) | ((hw[4] | hw[5]) | (hw[6] | hw[7])))) {
#pragma unroll
                                        for (int g = 0; g < 2; ++g) {   // two groups of 4 (registers)
                                            uint32_t rr[4][4];
#pragma unroll
                                            for (int kk = 0; kk < 4; ++kk) {
                                                lds4(pbase + qk(4 * g + kk) + (uint32_t)__ffs(hw[4 * g + kk]) * kGrpB, rr[kk]);
                                                hw[4 * g + kk] &= hw[4 * g + kk] - 1u;
                                            }
#pragma unroll
                                            for (int v = 0; v < 4; ++v) h[v] |= (rr[0][v] | rr[1][v]) | (rr[2][v] | rr[3][v]);
                                        }
                                        miss = 0u;
#pragma unroll
                                        for (int v = 0; v < 4; ++v) {
                                            miss |= xn[t][v] & ~h[v];
                                        }
                                    }
#pragma unroll
                                    for (int v = 0; v < 4; ++v) xn[t][v] &= h[v];
                                }
                            }
                        }
                    }
                }
                bool changed = false;
#pragma unroll
                for (int t = 0; t < 4; ++t) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        changed |= (xr[t][u] != xn[t][u]);
                        xr[t][u] = xn[t][u];
                    }
                }
                ++it;
                if (!changed) {
                    status = GB_CONVERGED;
                    break;
                }
            }
        }
        // ---- a7 output
        if (live) {
            out_iters[p] = (uint16_t)it;
            out_status[p] = (uint8_t)(bad ? GB_INVALID : status);
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
        if (live) {
            // clusters in the same order on every lane: lane q's chunk of cluster c is c ^ q, so the
            // 8 stores never bank-conflict (storing the erased slots by slot index put the lanes of a
            // quarter-warp on random chunks: 2.4x the wavefronts; same-box A/B C3 0.777 -> 0.770 ms, M=30k
            // 0.691 -> 0.678); an erased cluster's state is picked from its slot, t = number of erased
            // clusters below c
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const bool er = !bad && ((emask >> c) & 1u);
                const uint32_t s = bad ? 0xffffffffu : sym(c);
                const uint32_t b = 1u << (s & 31u), w = s >> 5;
                const uint32_t t = __popc(emask & ((1u << c) - 1u));
                uint32_t v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    uint32_t x = xr[0][u];
                    if (c >= 1) x = (t & 1u) ? xr[1][u] : x;
                    if (c >= 2) x = (t == 2u) ? xr[2][u] : x;
                    if (c >= 3) x = (t == 3u) ? xr[3][u] : x;
                    v[u] = er ? x : (w == (uint32_t)u ? b : 0u);
                }
                sts4(my_row + (((uint32_t)c ^ sw) << 4), v[0], v[1], v[2], v[3]);
            }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
            asm volatile(
                "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                ::"l"((uint64_t)&omap), "r"(0), "r"((int)pb), "r"(stg) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

}  // namespace

// The rotated-layout kernel for dense W (density > 0.65, counted by seal), the loop kernel for
// sparse W; GB_OPT_HYB8_SPLIT forces either.
bool decode_hyb8_rotated(const gb_net *net) {
    const int fs = net->opt[kOptHyb8Split].load(std::memory_order_relaxed);
    return fs >= 0 ? (fs != 0) : (net->density.load(std::memory_order_relaxed) > 0.65);
}

bool decode_hyb8_supported(const gb_net *net, int rule, int64_t k, const void *state) {
    const Shape &s = net->s;
    return rule == GB_HYBRID && s.C == 8 && s.Wc == 4 && k < (1ll << 31) && ((uintptr_t)state & 15u) == 0 &&
           net->opt[kOptHyb8].load(std::memory_order_relaxed) != 0;
}

// Tensor map of out_state viewed as [k rows][32 words], 32 x kBoxRows boxes, 128-byte swizzle.
static bool encode_out_map(void *state, int64_t k, CUtensorMap *map) {
    static std::atomic<void *> fnp_cache{nullptr};
    void *fnp = fnp_cache.load();
    if (!fnp) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fnp) {
            cudaGetLastError();
            return false;
        }
        fnp_cache.store(fnp);
    }
    using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    const cuuint64_t dims[2] = {32, (cuuint64_t)k};
    const cuuint64_t strides[1] = {128};
    const cuuint32_t box[2] = {32, (cuuint32_t)kBoxRows};
    const cuuint32_t estr[2] = {1, 1};
    return reinterpret_cast<EncodeFn>(fnp)(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, state, dims, strides, box, estr,
                                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                           CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Narrow (e <= 4) pass of the C = 8 hybrid decode; probes with e > 4 are appended
// to `ovf` for decode_smem_kernel's list mode (launched by the caller).
// Rows of the dense kernel's first push step: the fewest (6..8) for which a target's expected
// candidates n_t = 1 + (L - 1) d^4 (e = 4, four known rows) are all covered by n
// random candidate rows except with probability n_t (1 - d)^n <= 0.007 -- the rate at which the
// further steps cost less than the rows saved (same-box A/B, c=8 l=128, 10^7 probes: d = 0.70
// (C3) 7 rows 0.781 ms vs 8: 0.800, 6: 0.902; d = 0.78 6 rows 0.716 vs 5: 0.878, 7: 0.734, 8: 0.780;
// d = 0.84 6 rows 0.695 vs 5: 0.713, 7: 0.732, 8: 0.782 -- 5 rows never won, so 6 is the floor).
static int hyb8_rows(double d, int L) {
    const double nt = 1.0 + (L - 1) * d * d * d * d;
    double miss = nt;
    for (int n = 1; n <= 8; ++n) {
        miss *= 1.0 - d;
        if (n >= 6 && miss <= 0.007) return n;
    }
    return 8;
}

cudaError_t launch_decode_hyb8(Call &cl, const uint16_t *probes, int64_t k, int max_iters, uint32_t *state,
                               uint16_t *iters, uint8_t *status, int64_t *ovf, unsigned long long *ovf_count) {
    const gb_net *net = cl.net;
    // the output tensor map is a kernel parameter (copied at launch): encoded per call
    alignas(64) CUtensorMap map;
    if (!encode_out_map(state, k, &map)) return cudaErrorNotSupported;
    // kernel by W's density (see the kernels' comments); GB_OPT_HYB8_SPLIT forces it
    const double d = net->density.load(std::memory_order_relaxed);
    const bool dense = decode_hyb8_rotated(net);
    int nr = cl.opt(kOptHyb8Rows);
    if (nr == 0) nr = hyb8_rows(d, net->s.L);
    auto fn = !dense ? decode_hyb8_kernel
              : nr == 6 ? decode_hyb8r_kernel<6>
              : nr == 7 ? decode_hyb8r_kernel<7> : decode_hyb8r_kernel<8>;
    const int nt = dense ? kNTr : kNT;
    const size_t smem = dense ? kSmemR : kSmem;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int64_t grid = (k + nt - 1) / nt;
    if (grid > net->sm_count) grid = net->sm_count;
    fn<<<(unsigned)grid, nt, smem, cl.st>>>(net->wb, probes, k, net->s.L, max_iters, map, iters, status, ovf,
                                             ovf_count);
    cl.launched();
    return cudaGetLastError();
}

}  // namespace gb
