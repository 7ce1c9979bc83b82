// gb_symbols.cu -- gb_decode_symbols' output pass: the final state of every probe
// (cluster-padded bits, as the decode kernels write it) -> the retrieved message,
// one uint16 per cluster: the index of the cluster's only active neuron, GB_ERASED
// when none is active, GB_AMBIGUOUS when several are (DESIGN.md
// reading R16).  One thread per (probe, cluster); the cluster's Wc words are read
// together (consecutive threads read consecutive blocks of a state row).
#include "gb_internal.h"

namespace gb {
namespace {

template <int WC>
__global__ void symbols_kernel(const uint32_t *__restrict__ state, int64_t k, int C, int nw,
                               uint16_t *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // probe * C + cluster
    if (i >= k * C) return;
    const int64_t p = i / C;
    const int c = (int)(i - p * C);
    const uint32_t *blk = state + p * nw + c * WC;
    int cnt = 0, idx = 0;
#pragma unroll
    for (int u = 0; u < WC; ++u) {
        const uint32_t x = __ldg(blk + u);
        if (x && cnt == 0) idx = 32 * u + __ffs(x) - 1;
        cnt += __popc(x);
    }
    out[i] = cnt == 0 ? (uint16_t)GB_ERASED : cnt > 1 ? (uint16_t)GB_AMBIGUOUS : (uint16_t)idx;
}

__global__ void symbols_generic_kernel(const uint32_t *__restrict__ state, int64_t k, int C, int wc, int nw,
                                       uint16_t *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= k * C) return;
    const int64_t p = i / C;
    const int c = (int)(i - p * C);
    const uint32_t *blk = state + p * nw + c * wc;
    int cnt = 0, idx = 0;
    for (int u = 0; u < wc; ++u) {
        const uint32_t x = __ldg(blk + u);
        if (x && cnt == 0) idx = 32 * u + __ffs(x) - 1;
        cnt += __popc(x);
    }
    out[i] = cnt == 0 ? (uint16_t)GB_ERASED : cnt > 1 ? (uint16_t)GB_AMBIGUOUS : (uint16_t)idx;
}

}  // namespace

cudaError_t launch_symbols(Call &cl, const uint32_t *state, int64_t k, uint16_t *out) {
    const Shape &s = cl.net->s;
    const int64_t n = k * s.C;
    if (n == 0) return cudaSuccess;
    const int block = 256;
    const unsigned grid = (unsigned)((n + block - 1) / block);
    switch (s.Wc) {
        case 1: symbols_kernel<1><<<grid, block, 0, cl.st>>>(state, k, s.C, s.nw, out); break;
        case 2: symbols_kernel<2><<<grid, block, 0, cl.st>>>(state, k, s.C, s.nw, out); break;
        case 4: symbols_kernel<4><<<grid, block, 0, cl.st>>>(state, k, s.C, s.nw, out); break;
        case 8: symbols_kernel<8><<<grid, block, 0, cl.st>>>(state, k, s.C, s.nw, out); break;
        default: symbols_generic_kernel<<<grid, block, 0, cl.st>>>(state, k, s.C, s.Wc, s.nw, out); break;
    }
    cl.launched();
    return cudaGetLastError();
}

}  // namespace gb
