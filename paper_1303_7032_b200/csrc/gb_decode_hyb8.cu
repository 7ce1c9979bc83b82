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
//    in stages (the lowest candidate of every non-empty word of the source, then
//    the highest other candidate of every word in two halves, then the rest one
//    at a time), when sparse in a loop of "the lowest remaining candidate of
//    every word"; each step runs only while some target candidate is still
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
__device__ __forceinline__ uint32_t highbit(uint32_t x) { return 31 - __clz(x); }
// Two push variants, chosen by W's density (seal counts the edges):
//  DENSE (density > 0.65): stage 1 = the lowest candidate row of each word of the source;
//    stage 2 = the highest other candidate of each word, in two halves with a cover check
//    between them (at C3 ~32 candidates per erased cluster: stage 1 covers ~77% of the pairs and
//    two more rows usually cover the rest); stage 3 = the remaining rows one at a time;
//  sparse: one loop whose every step reads the lowest remaining candidate row of each word (up to
//    4 loads in flight) until the target is covered or the source exhausted -- few candidates per
//    cluster, many of them dying, so the uniform loop wastes fewer warp slots than the stages.
// Same-box A/B (round 2, 10^7 probes, hybrid, c=8 l=128): M=5k (density 0.26) 2.24 -> 1.74 ms
// with the loop, M=10k (0.46) 4.11 -> 3.32, M=15k (0.60) 1.19 -> 1.08; the staged form stays
// faster when dense: M=20k (C3, 0.70) 0.960 vs 0.973, M=30k (0.84) 0.855 vs 0.870.  A third form,
// stage 1 then one "pull" row per uncovered target candidate (row i's block of the source meets
// the source's remaining candidates, W symmetric), was slower at every density (C3 1.12 ms,
// M=5k 2.11): its loads run on few lanes, so each costs almost a full wavefront.
//
// The kernel is bound by the LSU data pipe (~87% of one shared-memory wavefront per SM per clock
// at C3); half of its wavefronts are bank conflicts, because a row block sits in the bank group of
// its target cluster and the 8 lanes of a quarter-warp target random clusters.  Measured and not
// kept (round 2, same-box A/B at C3):
//  * unpredicated stage loads (empty words read a discarded row, fixed up in a rare branch):
//    11% fewer instructions, ALU pipe 71% -> 55%, but 0.961 vs 0.931 ms -- not ALU-bound;
//  * a conflict-free probe order: each CTA classifies its 768-probe chunk by erasure set and
//    places 4 probes erasing E and 4 erasing ~E on every quarter-warp (counting sort in shared
//    memory, CTA-wide staging of the output rows): conflicts 118M -> 51M per launch, but 1.15 ms
//    (three CTA barriers per chunk and the exposed probe loads: long-scoreboard and barrier
//    stalls).  Host-side ordering of the same probes (no in-kernel cost) gives 0.88 vs 0.97 ms.
template <bool DENSE>
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
                            if (sidx != t && sidx < (int)nslot && any) {
                                // block c_t of row (c2, 32u + b): rb + (32u + b) * 128
                                const uint32_t rb = w_s + ((slots >> (4 * sidx)) & 15u) * kClusterB + (ct << 4);
                                uint32_t h[4] = {0u, 0u, 0u, 0u};
                                if constexpr (!DENSE) {
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
                                } else {
                                    // stage 1: the lowest candidate of each non-empty word, in flight
                                    // together
                                    {
                                        uint32_t r[4][4];
#pragma unroll
                                        for (int u = 0; u < 4; ++u) {
                                            const uint32_t x = xr[sidx][u];
#pragma unroll
                                            for (int v = 0; v < 4; ++v) r[u][v] = 0u;
                                            lds4p(x, rb + (u * 32 + lowbit(x)) * kRowB, r[u]);
                                        }
#pragma unroll
                                        for (int v = 0; v < 4; ++v) h[v] = (r[0][v] | r[1][v]) | (r[2][v] | r[3][v]);
                                    }
                                    uint32_t miss = 0u;
#pragma unroll
                                    for (int v = 0; v < 4; ++v) miss |= alive[v] & ~h[v];
                                    if (miss) {
                                        // stage 2: the highest other candidate of each word holding
                                        // >= 2, words 0-1, a cover check, then words 2-3 (the loads of
                                        // a half predicated and in flight together)
#pragma unroll
                                        for (int g = 0; g < 2; ++g) {
                                            if (g == 1) {
                                                miss = 0u;
#pragma unroll
                                                for (int v = 0; v < 4; ++v) miss |= alive[v] & ~h[v];
                                                if (!miss) break;
                                            }
                                            uint32_t r[2][4];
#pragma unroll
                                            for (int uu = 0; uu < 2; ++uu) {
                                                const int u = 2 * g + uu;
                                                const uint32_t x = xr[sidx][u];
                                                const uint32_t x2 = x & (x - 1u);
#pragma unroll
                                                for (int v = 0; v < 4; ++v) r[uu][v] = 0u;
                                                lds4p(x2, rb + (u * 32 + highbit(x2)) * kRowB, r[uu]);
                                            }
#pragma unroll
                                            for (int v = 0; v < 4; ++v) h[v] |= r[0][v] | r[1][v];
                                        }
                                        miss = 0u;
#pragma unroll
                                        for (int v = 0; v < 4; ++v) miss |= alive[v] & ~h[v];
                                        if (miss) {
                                            // stage 3: the rest, one row at a time
#pragma unroll
                                            for (int u = 0; u < 4; ++u) {
                                                const uint32_t x = xr[sidx][u];
                                                uint32_t rem = x & (x - 1u);                   // minus stage 1
                                                if (rem) rem &= ~(1u << highbit(rem));         // minus stage 2
                                                while (rem && miss) {
                                                    const uint32_t b = lowbit(rem);
                                                    rem &= rem - 1u;
                                                    uint32_t r[4];
                                                    lds4(rb + (u * 32 + b) * kRowB, r);
                                                    miss = 0u;
#pragma unroll
                                                    for (int v = 0; v < 4; ++v) {
                                                        h[v] |= r[v];
                                                        miss |= alive[v] & ~h[v];
                                                    }
                                                }
                                            }
                                        }
                                    }
                                }
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

}  // namespace

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
cudaError_t launch_decode_hyb8(Call &cl, const uint16_t *probes, int64_t k, int max_iters, uint32_t *state,
                               uint16_t *iters, uint8_t *status, int64_t *ovf, unsigned long long *ovf_count) {
    const gb_net *net = cl.net;
    // the output tensor map is a kernel parameter (copied at launch): encoded per call
    alignas(64) CUtensorMap map;
    if (!encode_out_map(state, k, &map)) return cudaErrorNotSupported;
    // push variant by W's density (see the kernel's comment); GB_OPT_HYB8_SPLIT forces it
    const int fs = cl.opt(kOptHyb8Split);
    const bool dense = fs >= 0 ? (fs != 0) : (net->density.load(std::memory_order_relaxed) > 0.65);
    auto fn = dense ? decode_hyb8_kernel<true> : decode_hyb8_kernel<false>;   // compile-time variants
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
    if (e != cudaSuccess) return e;
    int64_t grid = (k + kNT - 1) / kNT;
    if (grid > net->sm_count) grid = net->sm_count;
    fn<<<(unsigned)grid, kNT, kSmem, cl.st>>>(net->wb, probes, k, net->s.L, max_iters, map, iters, status, ovf,
                                              ovf_count);
    cl.launched();
    return cudaGetLastError();
}

}  // namespace gb
