// gb_decode_generic.cu -- warp-per-probe decode for any supported shape.
//
// One warp owns one probe at a time; its state V (n_padded bits = nw words)
// and the next state live in shared memory, lane t owning words t, t+32, ...
// W is read as bit rows Wb[i][*] (i = padded neuron index) through L1/L2.
//
//  a1 ingest  : symbols -> known one-hot / erased mask (PAPER.md L165, L197,
//               L270-271, Alg. 2 line 1); a symbol >= L -> GB_INVALID.
//  a5 prune   : hybrid X^0 on erased clusters = AND of the known neurons' bit
//               rows (S^0 == C-e, Alg. 2 lines 2-5; identity F3 of DESIGN.md).
//  a6 round   : SOM / hybrid: v'_i = v_i AND for every other cluster c' in
//               scope, (row_i & V_c') != 0  (Eq.(6)-(7) evaluated by
//               bail-out-early, Thm 1: walk clusters, stop at the
//               first silent one).  Hybrid: only erased clusters update and
//               only erased clusters are walked (known clusters are frozen
//               one-hot and every candidate is adjacent to them by the prune).
//  a3/a4 SOS  : s_i = gamma v_i + popc(row_i & V) (Eq.(3)); keep every
//               per-cluster maximiser (Eq.(4)-(5)).  Exact integer score on
//               the CUDA cores; used for shapes the tensor-core SOS kernel
//               does not take.
//  a7 output  : V, rounds, status; rounds are synchronous (Jacobi) and the
//               count includes the confirming round (readings R5-R7, R14).
#include "gb_internal.h"

namespace gb {
namespace {

constexpr int kWarps = 8;

__device__ __forceinline__ unsigned real_mask(const Shape &s, int u) {
    const int lo = u * 32;
    const int hi = min(s.L, lo + 32);
    if (hi <= lo) return 0u;
    const int nb = hi - lo;
    return nb == 32 ? 0xffffffffu : ((1u << nb) - 1u);
}

__global__ void __launch_bounds__(kWarps * 32)
decode_generic_kernel(Shape s, const uint32_t *__restrict__ wb, const uint16_t *__restrict__ probes,
                      int64_t k, int rule, int gamma, int T, int cyc_exit, uint32_t *__restrict__ out_state,
                      uint16_t *__restrict__ out_iters, uint8_t *__restrict__ out_status,
                      const int64_t *__restrict__ list, const unsigned long long *__restrict__ list_count) {
    extern __shared__ uint32_t smem[];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int nw = s.nw;
    uint32_t *bufA = smem + warp * 3 * nw;
    uint32_t *bufB = bufA + nw;
    int *wmax = reinterpret_cast<int *>(bufB + nw);

    // list mode: decode the list_count probes whose indices another kernel queued in list
    const int64_t n = list ? (int64_t)*list_count : k;
    for (int64_t i = (int64_t)blockIdx.x * kWarps + warp; i < n; i += (int64_t)gridDim.x * kWarps) {
        const int64_t p = list ? list[i] : i;
        const uint16_t *pr = probes + p * s.C;
        unsigned long long em = 0ull;
        bool bad = false;
        for (int c = lane; c < s.C; c += 32) {
            const unsigned sym = __ldg(pr + c);
            if (sym == kErased) em |= 1ull << c;
            else if (sym >= (unsigned)s.L) bad = true;
        }
        unsigned lo = (unsigned)em, hi = (unsigned)(em >> 32);
        lo = __reduce_or_sync(0xffffffffu, lo);
        hi = __reduce_or_sync(0xffffffffu, hi);
        em = ((unsigned long long)hi << 32) | lo;
        bad = __any_sync(0xffffffffu, bad);
        uint32_t *out = out_state + p * nw;
        if (bad) {
            for (int w = lane; w < nw; w += 32) out[w] = 0u;
            if (lane == 0) { out_iters[p] = 0; out_status[p] = GB_INVALID; }
            continue;
        }
        const int e = __popcll(em);
        uint32_t *X = bufA, *Xn = bufB;

        // a1 (+ a5 for hybrid): initial state.
        for (int w = lane; w < nw; w += 32) {
            const int c = w / s.Wc, u = w - c * s.Wc;
            uint32_t x;
            if ((em >> c) & 1ull) {
                if (rule == GB_SUM_OF_MAX) {
                    x = real_mask(s, u);
                } else if (rule == GB_HYBRID) {
                    x = real_mask(s, u);
                    for (int kc = 0; kc < s.C; ++kc) {
                        if ((em >> kc) & 1ull) continue;
                        const int row = kc * s.Lp + __ldg(pr + kc);
                        x &= __ldg(wb + (int64_t)row * nw + w);
                    }
                } else {
                    x = 0u;
                }
            } else {
                const unsigned sym = __ldg(pr + c);
                x = ((int)(sym >> 5) == u) ? (1u << (sym & 31)) : 0u;
            }
            X[w] = x;
        }
        __syncwarp();

        int it = 0;
        int status = GB_MAX_ITERS;
        if (rule == GB_HYBRID && e == 0) {
            status = GB_CONVERGED;
            it = 0;
        } else {
            while (it < T) {
                bool cyc = cyc_exit && it >= 1;   // Xn holds V^{r-2} from round r = it + 1 >= 2 on
                if (rule == GB_SUM_OF_SUM) {
                    // pass 1: per-word max of the scores of real neurons
                    for (int w = lane; w < nw; w += 32) {
                        const int c = w / s.Wc, u = w - c * s.Wc;
                        const unsigned rm = real_mask(s, u);
                        int mx = -1;
                        for (int b = 0; b < 32; ++b) {
                            if (!((rm >> b) & 1u)) continue;
                            const int64_t i = (int64_t)c * s.Lp + u * 32 + b;
                            const uint32_t *row = wb + i * nw;
                            int sc = ((X[w] >> b) & 1u) ? gamma : 0;
                            for (int v = 0; v < nw; ++v) sc += __popc(__ldg(row + v) & X[v]);
                            mx = max(mx, sc);
                        }
                        wmax[w] = mx;
                    }
                    __syncwarp();
                    // pass 2: keep all neurons reaching their cluster max
                    for (int w = lane; w < nw; w += 32) {
                        const int c = w / s.Wc, u = w - c * s.Wc;
                        const unsigned rm = real_mask(s, u);
                        int cm = -1;
                        for (int v = 0; v < s.Wc; ++v) cm = max(cm, wmax[c * s.Wc + v]);
                        uint32_t nx = 0u;
                        for (int b = 0; b < 32; ++b) {
                            if (!((rm >> b) & 1u)) continue;
                            const int64_t i = (int64_t)c * s.Lp + u * 32 + b;
                            const uint32_t *row = wb + i * nw;
                            int sc = ((X[w] >> b) & 1u) ? gamma : 0;
                            for (int v = 0; v < nw; ++v) sc += __popc(__ldg(row + v) & X[v]);
                            if (sc == cm) nx |= 1u << b;
                        }
                        cyc &= (Xn[w] == nx);
                        Xn[w] = nx;
                    }
                } else {
                    const bool hyb = (rule == GB_HYBRID);
                    for (int w = lane; w < nw; w += 32) {
                        const int c = w / s.Wc, u = w - c * s.Wc;
                        const uint32_t xw = X[w];
                        uint32_t nx = xw;
                        if (!hyb || ((em >> c) & 1ull)) {
                            uint32_t bits = xw;
                            while (bits) {
                                const int b = __ffs(bits) - 1;
                                bits &= bits - 1u;
                                const int64_t i = (int64_t)c * s.Lp + u * 32 + b;
                                const uint32_t *row = wb + i * nw;
                                for (int c2 = 0; c2 < s.C; ++c2) {
                                    if (c2 == c) continue;
                                    if (hyb && !((em >> c2) & 1ull)) continue;
                                    uint32_t any = 0u;
                                    for (int v = 0; v < s.Wc; ++v)
                                        any |= __ldg(row + c2 * s.Wc + v) & X[c2 * s.Wc + v];
                                    if (!any) { nx &= ~(1u << b); break; }
                                }
                            }
                        }
                        Xn[w] = nx;
                    }
                }
                __syncwarp();
                bool diff = false;
                for (int w = lane; w < nw; w += 32) diff |= (Xn[w] != X[w]);
                diff = __any_sync(0xffffffffu, diff);
                cyc = __all_sync(0xffffffffu, cyc) && rule == GB_SUM_OF_SUM;
                uint32_t *tmp = X; X = Xn; Xn = tmp;
                ++it;
                if (!diff) { status = GB_CONVERGED; break; }
                if (cyc) { status = GB_CYCLE; break; }   // V^r == V^{r-2} (GB_FLAG_CYCLE_EXIT)
            }
        }
        for (int w = lane; w < nw; w += 32) out[w] = X[w];
        if (lane == 0) {
            out_iters[p] = (uint16_t)it;
            out_status[p] = (uint8_t)status;
        }
        __syncwarp();
    }
}

}  // namespace

cudaError_t launch_decode_generic(Call &cl, const uint16_t *probes, int64_t k, int rule,
                                  int gamma, int max_iters, int cyc, uint32_t *state, uint16_t *iters,
                                  uint8_t *status) {
    const gb_net *net = cl.net;
    const cudaStream_t st = cl.st;
    const size_t smem = (size_t)kWarps * 3 * net->s.nw * sizeof(uint32_t);
    int64_t grid = (k + kWarps - 1) / kWarps;
    const int64_t cap = (int64_t)net->sm_count * 8;
    if (grid > cap) grid = cap;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(decode_generic_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    decode_generic_kernel<<<(unsigned)grid, kWarps * 32, smem, st>>>(
        net->s, net->wb, probes, k, rule, gamma, max_iters, cyc, state, iters, status, nullptr, nullptr);
    cl.launched();
    return cudaGetLastError();
}

// List mode: the *count probes listed in `list` (indices into probes / the outputs), queued by a
// preceding kernel on the same stream; k bounds the count.
cudaError_t launch_decode_generic_list(Call &cl, const uint16_t *probes, int64_t k, const int64_t *list,
                                       const unsigned long long *count, int rule, int gamma, int max_iters,
                                       uint32_t *state, uint16_t *iters, uint8_t *status) {
    const gb_net *net = cl.net;
    const size_t smem = (size_t)kWarps * 3 * net->s.nw * sizeof(uint32_t);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(decode_generic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
    }
    decode_generic_kernel<<<(unsigned)net->sm_count, kWarps * 32, smem, cl.st>>>(
        net->s, net->wb, probes, k, rule, gamma, max_iters, 0, state, iters, status, list, count);
    cl.launched();
    return cudaGetLastError();
}

}  // namespace gb
