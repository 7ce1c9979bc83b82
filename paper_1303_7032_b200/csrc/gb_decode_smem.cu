// gb_decode_smem.cu -- thread-per-probe SOM / hybrid decode with W held in
// shared memory (n_padded <= 1024, C <= 8): the hot path of the metric
// (hybrid rule, c=8 l=128).
//
// Layout (DESIGN.md §Kernels / "smem bit kernel"):
//  * W bit rows Wb[np][nw] copied once per CTA into shared memory (128 KiB at
//    c=8 l=128); block c of row j = words [c*WC, c*WC+WC).
//  * one thread = one probe.  The probe's in-scope cluster states X[t][WC]
//    (t indexes the slot list: erased clusters for the hybrid, all clusters
//    for sum-of-max) live in a per-thread shared-memory area, two buffers
//    (synchronous rounds), interleaved [word][thread] so accesses are
//    bank-conflict free.
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
//                H covers the still-alive part of X_t (the first time a
//                candidate receives a signal from cluster c_s is enough,
//                L449); alive &= H; a target found dead in one source cluster
//                stops being walked (L450).  Dead neurons stay dead (Lemma 1).
//                Hybrid: targets and sources are the erased clusters only;
//                known clusters are frozen one-hot (Alg. 2) and
//                every candidate is adjacent to them by the prune.
//  a7 output  -- state bits, rounds (incl. the confirming round), status.
#include "gb_internal.h"

namespace gb {
namespace {

constexpr int kSmemThreads = 256;
constexpr int kMaxC = 8;

template <int WC>
__device__ __forceinline__ void load_block(const uint32_t *p, uint32_t (&v)[WC]) {
    if constexpr (WC == 4) {
        const uint4 q = *reinterpret_cast<const uint4 *>(p);
        v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    } else if constexpr (WC == 2) {
        const uint2 q = *reinterpret_cast<const uint2 *>(p);
        v[0] = q.x; v[1] = q.y;
    } else {
#pragma unroll
        for (int u = 0; u < WC; ++u) v[u] = p[u];
    }
}

template <int WC>
__device__ __forceinline__ uint32_t real_mask_u(int L, int u) {
    const int lo = u * 32;
    const int nb = min(32, max(0, L - lo));
    return nb == 32 ? 0xffffffffu : ((1u << nb) - 1u);
}

template <int WC, int RULE>
__global__ void __launch_bounds__(kSmemThreads, 1)
decode_smem_kernel(Shape s, const uint32_t *__restrict__ wb, const uint16_t *__restrict__ probes,
                   int64_t k, int T, uint32_t *__restrict__ out_state,
                   uint16_t *__restrict__ out_iters, uint8_t *__restrict__ out_status) {
    extern __shared__ __align__(16) uint32_t smem[];
    constexpr int LP = 32 * WC;
    const int C = s.C;
    const int nw = C * WC;
    const int np = C * LP;
    uint32_t *W = smem;                                  // [np][nw]
    uint32_t *XA = smem + np * nw;                       // [C*WC][threads]
    uint32_t *XB = XA + kMaxC * WC * kSmemThreads;
    const int tid = threadIdx.x;

    // W -> shared memory, 16 B per thread per step.
    {
        const int n16 = np * nw / 4;
        const uint4 *src = reinterpret_cast<const uint4 *>(wb);
        uint4 *dst = reinterpret_cast<uint4 *>(W);
        for (int i = tid; i < n16; i += kSmemThreads) dst[i] = __ldg(src + i);
    }
    __syncthreads();

    for (int64_t p = (int64_t)blockIdx.x * kSmemThreads + tid; p < k;
         p += (int64_t)gridDim.x * kSmemThreads) {
        // ---- a1 ingest
        unsigned sym[kMaxC];
        const uint16_t *pr = probes + p * C;
#pragma unroll
        for (int c = 0; c < kMaxC; ++c) sym[c] = (c < C) ? (unsigned)__ldg(pr + c) : 0u;
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
        // slot list: erased clusters (hybrid) or all clusters (SOM); 4 bits each
        unsigned slots = 0, nslot = 0;
#pragma unroll
        for (int c = 0; c < kMaxC; ++c) {
            if (c < C && (RULE == GB_SUM_OF_MAX || ((emask >> c) & 1u))) {
                slots |= (unsigned)c << (4 * nslot);
                ++nslot;
            }
        }
        uint32_t *X = XA, *Xn = XB;
        // ---- a5 prune / init
        for (unsigned t = 0; t < nslot; ++t) {
            const int c = (slots >> (4 * t)) & 15;
            uint32_t x[WC];
            if ((emask >> c) & 1u) {
#pragma unroll
                for (int u = 0; u < WC; ++u) x[u] = real_mask_u<WC>(s.L, u);
                if (RULE == GB_HYBRID) {
#pragma unroll
                    for (int kc = 0; kc < kMaxC; ++kc) {
                        if (kc < C && !((emask >> kc) & 1u)) {
                            uint32_t r[WC];
                            load_block<WC>(W + (kc * LP + sym[kc]) * nw + c * WC, r);
#pragma unroll
                            for (int u = 0; u < WC; ++u) x[u] &= r[u];
                        }
                    }
                }
            } else {
#pragma unroll
                for (int u = 0; u < WC; ++u) x[u] = ((int)(sym[c] >> 5) == u) ? (1u << (sym[c] & 31)) : 0u;
            }
#pragma unroll
            for (int u = 0; u < WC; ++u) X[(t * WC + u) * kSmemThreads + tid] = x[u];
        }

        int it = 0;
        int status = GB_MAX_ITERS;
        if (RULE == GB_HYBRID && nslot == 0) {
            status = GB_CONVERGED;
        } else {
            // ---- a6 rounds
            while (it < T) {
                bool changed = false;
                for (unsigned t = 0; t < nslot; ++t) {
                    const int c = (slots >> (4 * t)) & 15;
                    uint32_t x[WC], alive[WC];
#pragma unroll
                    for (int u = 0; u < WC; ++u) {
                        x[u] = X[(t * WC + u) * kSmemThreads + tid];
                        alive[u] = x[u];
                    }
                    uint32_t any = 0;
#pragma unroll
                    for (int u = 0; u < WC; ++u) any |= alive[u];
                    for (unsigned sidx = 0; sidx < nslot && any; ++sidx) {
                        if (sidx == t) continue;
                        const int c2 = (slots >> (4 * sidx)) & 15;
                        uint32_t h[WC];
#pragma unroll
                        for (int u = 0; u < WC; ++u) h[u] = 0u;
                        bool covered = false;
#pragma unroll
                        for (int u2 = 0; u2 < WC; ++u2) {
                            uint32_t bits = X[(sidx * WC + u2) * kSmemThreads + tid];
                            while (bits && !covered) {
                                const int b = __ffs(bits) - 1;
                                bits &= bits - 1u;
                                const int j = c2 * LP + u2 * 32 + b;
                                uint32_t r[WC];
                                load_block<WC>(W + j * nw + c * WC, r);
                                uint32_t miss = 0;
#pragma unroll
                                for (int u = 0; u < WC; ++u) {
                                    h[u] |= r[u];
                                    miss |= alive[u] & ~h[u];
                                }
                                covered = (miss == 0u);
                            }
                        }
                        any = 0;
#pragma unroll
                        for (int u = 0; u < WC; ++u) {
                            alive[u] &= h[u];
                            any |= alive[u];
                        }
                    }
#pragma unroll
                    for (int u = 0; u < WC; ++u) {
                        Xn[(t * WC + u) * kSmemThreads + tid] = alive[u];
                        changed |= (alive[u] != x[u]);
                    }
                }
                uint32_t *tmp = X; X = Xn; Xn = tmp;
                ++it;
                if (!changed) { status = GB_CONVERGED; break; }
            }
        }
        // ---- a7 output (known clusters one-hot, slots from X)
        unsigned slot_of = 0;  // 4 bits per cluster: slot index + 1 (0 = none)
        for (unsigned t = 0; t < nslot; ++t) slot_of |= (t + 1) << (4 * ((slots >> (4 * t)) & 15));
#pragma unroll
        for (int c = 0; c < kMaxC; ++c) {
            if (c >= C) break;
            const unsigned so = (slot_of >> (4 * c)) & 15u;
            uint32_t v[WC];
#pragma unroll
            for (int u = 0; u < WC; ++u)
                v[u] = so ? X[((so - 1) * WC + u) * kSmemThreads + tid]
                          : (((int)(sym[c] >> 5) == u) ? (1u << (sym[c] & 31)) : 0u);
            if constexpr (WC == 4) {
                *reinterpret_cast<uint4 *>(out + c * WC) = make_uint4(v[0], v[1], v[2], v[3]);
            } else {
#pragma unroll
                for (int u = 0; u < WC; ++u) out[c * WC + u] = v[u];
            }
        }
        out_iters[p] = (uint16_t)it;
        out_status[p] = (uint8_t)status;
    }
}

template <int WC, int RULE>
cudaError_t launch_t(gb_net *net, const uint16_t *probes, int64_t k, int max_iters, uint32_t *state,
                     uint16_t *iters, uint8_t *status, cudaStream_t st) {
    const Shape &s = net->s;
    const size_t smem = (size_t)s.np * s.nw * 4 + 2ull * kMaxC * WC * kSmemThreads * 4;
    auto fn = decode_smem_kernel<WC, RULE>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int64_t grid = (k + kSmemThreads - 1) / kSmemThreads;
    if (grid > net->sm_count) grid = net->sm_count;
    fn<<<(unsigned)grid, kSmemThreads, smem, st>>>(s, net->wb, probes, k, max_iters, state, iters, status);
    net->launches += 1;
    return cudaGetLastError();
}

}  // namespace

// Returns cudaErrorNotSupported when the shape does not fit this kernel.
cudaError_t launch_decode_smem(gb_net *net, const uint16_t *probes, int64_t k, int rule, int max_iters,
                               uint32_t *state, uint16_t *iters, uint8_t *status, cudaStream_t st) {
    const Shape &s = net->s;
    if (s.C > kMaxC || s.np > 1024 || rule == GB_SUM_OF_SUM) return cudaErrorNotSupported;
    const size_t smem = (size_t)s.np * s.nw * 4 + 2ull * kMaxC * s.Wc * kSmemThreads * 4;
    if (smem > 227 * 1024) return cudaErrorNotSupported;
    const bool hyb = (rule == GB_HYBRID);
    switch (s.Wc) {
        case 1: return hyb ? launch_t<1, GB_HYBRID>(net, probes, k, max_iters, state, iters, status, st)
                           : launch_t<1, GB_SUM_OF_MAX>(net, probes, k, max_iters, state, iters, status, st);
        case 2: return hyb ? launch_t<2, GB_HYBRID>(net, probes, k, max_iters, state, iters, status, st)
                           : launch_t<2, GB_SUM_OF_MAX>(net, probes, k, max_iters, state, iters, status, st);
        case 4: return hyb ? launch_t<4, GB_HYBRID>(net, probes, k, max_iters, state, iters, status, st)
                           : launch_t<4, GB_SUM_OF_MAX>(net, probes, k, max_iters, state, iters, status, st);
        default: return cudaErrorNotSupported;
    }
}

}  // namespace gb
