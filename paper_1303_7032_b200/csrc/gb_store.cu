// gb_store.cu -- clique storage (a2) and seal/pack of W for retrieval.
//
// STORE (Eq.(1)): for each message and each
// ordered cluster pair c != c', W8[(c,m_c)][(c',m_c')] = 1.  One thread per
// (message, c) writes row (c, m_c) at the C-1 other clusters' columns.
// Concurrent writers only ever write the value 1, and the writes are
// st.relaxed.gpu (morally strong), so there is no data race in the PTX
// memory model (SURVEY.md §5 "race detection").
//
// SEAL ("the variables w are fixed"; L381 "W fixed at the
// retrieval stage" / Alg. 2 line 6 "sparsify W"): pack W8 rows into bit rows
// Wb[i][w] (bit b = W8[i][32w+b]) with a warp ballot, and check the
// invariants of Eq.(1): binary entries, w_ij = w_ji (L306), no intra-cluster
// edge (L145), no padding edge.
#include "gb_internal.h"

namespace gb {
namespace {

__device__ __forceinline__ void st_relaxed_u8(uint8_t *p, unsigned v) {
    asm volatile("st.relaxed.gpu.global.u8 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void store_kernel(Shape s, const uint16_t *__restrict__ msgs, int64_t m,
                             uint8_t *__restrict__ w8, unsigned long long *__restrict__ dcount,
                             unsigned *__restrict__ dflag) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m * s.C) return;
    const int64_t msg = t / s.C;
    const int c = (int)(t - msg * s.C);
    const uint16_t *row = msgs + msg * s.C;
    bool ok = true;
    for (int cc = 0; cc < s.C; ++cc) ok &= (__ldg(row + cc) < s.L);
    if (!ok) {
        if (c == 0) {
            atomicAdd(dcount, 1ull);
            atomicOr(dflag, kFlagStoreInvalid);
        }
        return;
    }
    const int64_t i = (int64_t)c * s.Lp + __ldg(row + c);
    uint8_t *wrow = w8 + i * s.np;
    for (int cc = 0; cc < s.C; ++cc) {
        if (cc == c) continue;
        st_relaxed_u8(wrow + (int64_t)cc * s.Lp + __ldg(row + cc), 1u);
    }
}

// One warp per (row i, word w): lane b reads W8[i][32w+b], checks it, and the
// warp ballot forms Wb[i][w].
__global__ void seal_kernel(Shape s, const uint8_t *__restrict__ w8, uint32_t *__restrict__ wb,
                            unsigned *__restrict__ dflag) {
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t total = (int64_t)s.np * s.nw;
    if (warp >= total) return;
    const int i = (int)(warp / s.nw);
    const int w = (int)(warp - (int64_t)i * s.nw);
    const int j = w * 32 + lane;
    const unsigned v = w8[(int64_t)i * s.np + j];
    unsigned bad = 0;
    if (v > 1u) bad |= kFlagNotBinary;
    if (v) {
        const int ci = i / s.Lp, cj = j / s.Lp;
        if (ci == cj) bad |= kFlagIntra;
        if (i - ci * s.Lp >= s.L || j - cj * s.Lp >= s.L) bad |= kFlagPad;
    }
    if (w8[(int64_t)j * s.np + i] != v) bad |= kFlagAsym;
    const unsigned bits = __ballot_sync(0xffffffffu, v != 0u);
    const unsigned anybad = __reduce_or_sync(0xffffffffu, bad);
    if (lane == 0) {
        wb[(int64_t)i * s.nw + w] = bits;
        if (anybad) atomicOr(dflag, anybad);
    }
}

}  // namespace

cudaError_t launch_store(const gb_net *net, const uint16_t *msgs, int64_t m, cudaStream_t st) {
    const int64_t threads = m * net->s.C;
    const int block = 256;
    const int64_t grid = (threads + block - 1) / block;
    store_kernel<<<(unsigned)grid, block, 0, st>>>(net->s, msgs, m, net->w8, net->dcount,
                                                   net->dflag);
    return cudaGetLastError();
}

cudaError_t launch_seal(const gb_net *net, cudaStream_t st) {
    const int64_t warps = (int64_t)net->s.np * net->s.nw;
    const int block = 256;
    const int64_t grid = (warps * 32 + block - 1) / block;
    seal_kernel<<<(unsigned)grid, block, 0, st>>>(net->s, net->w8, net->wb, net->dflag);
    return cudaGetLastError();
}

}  // namespace gb
