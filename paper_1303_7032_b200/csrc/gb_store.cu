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
#include <stdlib.h>

#include <algorithm>

#include "gb_internal.h"

namespace gb {
namespace {

#ifndef GB_PRIV_TILE_KB
#define GB_PRIV_TILE_KB 128
#endif
#ifndef GB_PRIV_NT
#define GB_PRIV_NT 1024
#endif

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

// One warp per 32x32 tile (rows i0.., columns j0..): lane r loads row i0+r of
// the tile and row j0+r of the transposed tile (32 contiguous bytes each), packs
// its row into Wb[i0+r][j0/32], and the warp checks the tile against the
// transpose (32 ballots) and the structural invariants.
__device__ __forceinline__ uint32_t pack32(const uint8_t *p, unsigned &nonbin) {
    const uint4 a = *reinterpret_cast<const uint4 *>(p);
    const uint4 b = *reinterpret_cast<const uint4 *>(p + 16);
    const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    uint32_t bits = 0u;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        nonbin |= w[k] & 0xfefefefeu;
#pragma unroll
        for (int q = 0; q < 4; ++q) bits |= ((w[k] >> (8 * q)) & 0xffu ? 1u : 0u) << (4 * k + q);
    }
    return bits;
}

// Also builds the cluster unions Wu[s][t] = OR over the rows j of cluster s of block t of
// row j: the cover H that a push from a source whose candidate set is the whole cluster
// computes (the sum-of-max state of an erased cluster before its first round, PAPER.md
// L270-271), which the bit kernels then read in one load instead of ~L/4 row loads.  Each
// tile's warp ORs its 32 packed words into Wu (two buffers alternating by seal generation:
// this seal ORs into `wu` and zeroes `wu_next` for the next one).
__global__ void seal_kernel(Shape s, const uint8_t *__restrict__ w8, uint32_t *__restrict__ wb,
                            unsigned long long *__restrict__ dcount, Status *__restrict__ hstat,
                            unsigned long long gen, uint32_t *__restrict__ wu, uint32_t *__restrict__ wu_next) {
    unsigned *dflag = reinterpret_cast<unsigned *>(dcount + 1);   // [0] flags, [1] edges, [2] CTAs done
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int nt = s.np / 32;
    if (warp < (int64_t)nt * nt) {
        const int ti = (int)(warp / nt), tj = (int)(warp - (int64_t)ti * nt);
        const int i0 = 32 * ti, j0 = 32 * tj;
        unsigned nonbin = 0u;
        const uint32_t P = pack32(w8 + (int64_t)(i0 + lane) * s.np + j0, nonbin);   // W8[i0+lane][j0+b]
        const uint32_t T = pack32(w8 + (int64_t)(j0 + lane) * s.np + i0, nonbin);   // W8[j0+lane][i0+b]
        uint32_t R = 0u;                                                             // W8[j0+b][i0+lane]
#pragma unroll 8
        for (int k = 0; k < 32; ++k) {
            const uint32_t x = __ballot_sync(0xffffffffu, (T >> k) & 1u);
            if (lane == k) R = x;
        }
        const int ci = i0 / s.Lp, cj = j0 / s.Lp;
        const int cb = j0 - cj * s.Lp;   // first column slot of the tile inside cluster cj
        const uint32_t realc = cb >= s.L ? 0u : (s.L - cb >= 32 ? 0xffffffffu : ((1u << (s.L - cb)) - 1u));
        const bool realr = (i0 + lane - ci * s.Lp) < s.L;
        unsigned bad = nonbin ? kFlagNotBinary : 0u;
        if (P != R) bad |= kFlagAsym;
        if (P && ci == cj) bad |= kFlagIntra;
        if ((P & ~realc) || (P && !realr)) bad |= kFlagPad;
        wb[(int64_t)(i0 + lane) * s.nw + tj] = P;
        const unsigned anybad = __reduce_or_sync(0xffffffffu, bad);
        if (lane == 0 && anybad) atomicOr(dflag, anybad);
        const unsigned ne = __reduce_add_sync(0xffffffffu, (unsigned)__popc(P));   // edges (both directions)
        if (lane == 0 && ne) atomicAdd(dflag + 1, ne);
        const unsigned un = __reduce_or_sync(0xffffffffu, P);                        // cluster union
        if (lane == 0 && un) atomicOr(wu + (ci * s.C + cj) * s.Wc + (tj - cj * s.Wc), un);
    }
    {
        const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        if (t < (int64_t)s.C * s.C * s.Wc) wu_next[t] = 0u;
    }
    // the last CTA to finish publishes the status to mapped host memory (no host sync in
    // gb_seal) and resets the per-seal words for the next seal
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(dflag + 2, 1u) == gridDim.x - 1) {
            __threadfence();
            const unsigned long long inv = atomicAdd(dcount, 0ull);
            const unsigned flags = atomicOr(dflag, 0u), edges = atomicAdd(dflag + 1, 0u);
            volatile Status *h = hstat;
            h->invalid = inv;
            h->flags = flags;
            h->edges = edges;
            __threadfence_system();
            h->gen = gen;
            __threadfence_system();
            dflag[0] = 0u;
            dflag[1] = 0u;
            dflag[2] = 0u;
        }
    }
}

// ---- privatised store (large m): one CTA = (row cluster c, column-cluster
// group g, message chunk).  The CTA ORs the clique edges of its chunk that
// fall in rows (c, *) x columns of group g into a bit tile in shared memory
// (shared-memory atomics instead of scattered L2 byte writes), then writes the
// tile into partial bit matrix `chunk`; apply_kernel ORs the partials into W8.
// Every tile of every chunk writes its whole region (the c' = c block as
// zeros), so the partials need no clearing.  Same edges as store_kernel:
// W8[(c,m_c)][(c',m_c')] for every ordered pair c != c' (Eq.(1)).
struct PrivPlan {
    int G;        // column clusters per tile
    int ngroups;  // ceil(C / G)
    int tiles;    // C * ngroups
    int chunks;
    int64_t per_chunk;
    size_t tile_bytes;
};

template <int NV>
__global__ void __launch_bounds__(GB_PRIV_NT, 1)
store_priv_kernel(Shape s, const uint16_t *__restrict__ msgs, int64_t m, int G, int ngroups, int tiles,
                  int64_t per_chunk, uint32_t *__restrict__ part, unsigned long long *__restrict__ dcount,
                  unsigned *__restrict__ dflag) {
    extern __shared__ __align__(16) uint32_t tile[];
    const int chunk = blockIdx.x / tiles;
    const int t = blockIdx.x - chunk * tiles;
    const int c = t / ngroups;
    const int g0 = (t - c * ngroups) * G;
    const int g1 = min(s.C, g0 + G);
    const int tw = (g1 - g0) * s.Wc;                 // words per tile row
    // odd row stride: with tw a multiple of 32 every row would start on bank 0, and the
    // lanes of a warp (same column cluster at the same step) would share 8 banks
    const int ts = tw | 1;
    const int nwords = s.Lp * tw;
    for (int i = threadIdx.x; i < s.Lp * ts; i += blockDim.x) tile[i] = 0u;
    __syncthreads();
    const int64_t b = (int64_t)chunk * per_chunk;
    const int64_t e = min(m, b + per_chunk);
    const bool counter = (t == 0);
    for (int64_t mi = b + threadIdx.x; mi < e; mi += blockDim.x) {
        const uint16_t *row = msgs + mi * s.C;
        unsigned mc, sy[NV > 0 ? 8 * NV : 1];
        bool ok = true;
        if constexpr (NV > 0) {
            // the message as NV 16-byte vectors (C = 8*NV, rows 16-byte aligned)
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const uint4 q = __ldg(reinterpret_cast<const uint4 *>(row) + v);
                const uint32_t w4[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    sy[8 * v + 2 * h] = w4[h] & 0xffffu;
                    sy[8 * v + 2 * h + 1] = w4[h] >> 16;
                }
            }
            mc = 0;
#pragma unroll
            for (int cc = 0; cc < 8 * NV; ++cc) {
                ok &= (sy[cc] < (unsigned)s.L);
                if (cc == c) mc = sy[cc];
            }
        } else {
            for (int cc = 0; cc < s.C; ++cc) ok &= (__ldg(row + cc) < s.L);
            mc = ok ? __ldg(row + c) : 0u;
        }
        if (!ok) {
            if (counter) {
                atomicAdd(dcount, 1ull);
                atomicOr(dflag, kFlagStoreInvalid);
            }
            continue;
        }
        uint32_t *trow = tile + mc * ts;
        if constexpr (NV > 0) {
#pragma unroll
            for (int cc = 0; cc < 8 * NV; ++cc) {
                if (cc == c || cc < g0 || cc >= g1) continue;
                const int col = (cc - g0) * s.Lp + (int)sy[cc];
                atomicOr(trow + (col >> 5), 1u << (col & 31));
            }
        } else {
            for (int cc = g0; cc < g1; ++cc) {
                if (cc == c) continue;
                const int col = (cc - g0) * s.Lp + __ldg(row + cc);
                atomicOr(trow + (col >> 5), 1u << (col & 31));
            }
        }
    }
    __syncthreads();
    uint32_t *dst = part + (size_t)chunk * s.np * s.nw + (size_t)c * s.Lp * s.nw + g0 * s.Wc;
    for (int i = threadIdx.x; i < nwords; i += blockDim.x) {
        const int r = i / tw, w = i - r * tw;
        dst[(size_t)r * s.nw + w] = tile[r * ts + w];
    }
}

// One thread per (row i, word w) of the bit matrix: OR the chunk partials and
// set the corresponding W8 bytes (read-modify-write of 32 bytes only when some
// bit is set; W8 keeps every edge it already had).
__global__ void apply_kernel(Shape s, const uint32_t *__restrict__ part, int chunks, uint8_t *__restrict__ w8) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t total = (int64_t)s.np * s.nw;
    if (idx >= total) return;
    uint32_t bits = 0u;
    for (int ch = 0; ch < chunks; ++ch) bits |= __ldg(part + (size_t)ch * total + idx);
    if (!bits) return;
    const int64_t i = idx / s.nw, w = idx - i * s.nw;
    uint4 *p = reinterpret_cast<uint4 *>(w8 + i * s.np + w * 32);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        uint4 v = p[h];
        uint32_t q[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t nib = (bits >> (16 * h + 4 * k)) & 15u;
            q[k] |= (nib & 1u) | ((nib & 2u) << 7) | ((nib & 4u) << 14) | ((nib & 8u) << 21);
        }
        p[h] = make_uint4(q[0], q[1], q[2], q[3]);
    }
}

// ---- upper-triangle exchange: W is symmetric, so the
// cluster-pair blocks (a, b) with a < b carry all of it.  Packed layout: blocks in (a, b)
// lexicographic order, each Lp rows x Wc words of Wb, row-major.
__device__ __forceinline__ void upper_block(const Shape &s, int64_t q, int &a, int &b) {
    a = 0;
    while (q >= s.C - 1 - a) {
        q -= s.C - 1 - a;
        ++a;
    }
    b = a + 1 + (int)q;
}

__global__ void pack_upper_kernel(Shape s, const uint32_t *__restrict__ wb, uint32_t *__restrict__ out) {
    const int64_t per = (int64_t)s.Lp * s.Wc;
    const int64_t total = per * s.C * (s.C - 1) / 2;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t q = idx / per, rem = idx - q * per;
        const int r = (int)(rem / s.Wc), w = (int)(rem - (int64_t)r * s.Wc);
        int a, b;
        upper_block(s, q, a, b);
        out[idx] = __ldg(wb + ((int64_t)a * s.Lp + r) * s.nw + b * s.Wc + w);
    }
}

// OR 32 bits into the 32 W8 bytes at p (bit k -> byte k); read-modify-write only if any bit.
__device__ __forceinline__ void or_bytes32(uint8_t *p, uint32_t bits) {
    if (!bits) return;
    uint4 *q = reinterpret_cast<uint4 *>(p);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        uint4 v = q[h];
        uint32_t x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t nib = (bits >> (16 * h + 4 * k)) & 15u;
            x[k] |= (nib & 1u) | ((nib & 2u) << 7) | ((nib & 4u) << 14) | ((nib & 8u) << 21);
        }
        q[h] = make_uint4(x[0], x[1], x[2], x[3]);
    }
}

// One warp per 32x32 tile of an upper block: lane l ORs row i0+l's word over the `count`
// packed sets, sets W8[i0+l][j0..j0+31], and (after a 32-ballot transpose) the mirror
// W8[j0+l][i0..i0+31].  Every W8 segment is written by exactly one lane.
__global__ void or_upper_kernel(Shape s, const uint32_t *__restrict__ sets, int count, uint8_t *__restrict__ w8) {
    const int64_t per = (int64_t)s.Lp * s.Wc;
    const int64_t set_words = per * s.C * (s.C - 1) / 2;
    const int64_t tiles = set_words / 32;   // (Lp / 32) row groups x Wc words per block
    const int lane = threadIdx.x & 31;
    for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < tiles;
         t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t per_t = per / 32;
        const int64_t q = t / per_t, rem = t - q * per_t;
        const int rg = (int)(rem / s.Wc), w = (int)(rem - (int64_t)rg * s.Wc);
        int a, b;
        upper_block(s, q, a, b);
        const int64_t idx = q * per + (int64_t)(rg * 32 + lane) * s.Wc + w;
        uint32_t bits = 0u;
        for (int k = 0; k < count; ++k) bits |= __ldg(sets + (int64_t)k * set_words + idx);
        const int64_t i0 = (int64_t)a * s.Lp + rg * 32, j0 = (int64_t)b * s.Lp + w * 32;
        or_bytes32(w8 + (i0 + lane) * s.np + j0, bits);
        uint32_t tr = 0u;
#pragma unroll 8
        for (int k = 0; k < 32; ++k) {
            const uint32_t x = __ballot_sync(0xffffffffu, (bits >> k) & 1u);
            if (lane == k) tr = x;
        }
        or_bytes32(w8 + (j0 + lane) * s.np + i0, tr);
    }
}

constexpr size_t kPrivTileMax = GB_PRIV_TILE_KB * 1024;

PrivPlan priv_plan(const Shape &s, int64_t m, int sm_count) {
    PrivPlan p;
    const size_t blk = (size_t)s.Lp * s.Lp / 8;      // one cluster-pair block in bits
    p.G = (int)std::min<size_t>((size_t)s.C, std::max<size_t>(1, kPrivTileMax / blk));
    p.ngroups = (s.C + p.G - 1) / p.G;
    p.tiles = s.C * p.ngroups;
    p.tile_bytes = (size_t)p.G * blk + (size_t)s.Lp * 4;   // + one pad word per row
    const int resident = (int)std::max<size_t>(1, std::min<size_t>(8, (200 * 1024) / p.tile_bytes));
    const int64_t slots = std::max<int64_t>(1, (int64_t)sm_count * resident / p.tiles);
    const int64_t want = std::max<int64_t>(1, (m + 4095) / 4096);
    p.chunks = (int)std::min<int64_t>(slots, want);
    p.per_chunk = (m + p.chunks - 1) / p.chunks;
    return p;
}

}  // namespace

cudaError_t launch_store(Call &cl, const uint16_t *msgs, int64_t m) {
    gb_net *net = cl.net;
    const cudaStream_t st = cl.st;
    const Shape &s = net->s;
    const PrivPlan p = priv_plan(s, m, net->sm_count);
    // small batches: scattered relaxed byte stores (no tile setup / apply pass); also when one
    // cluster-pair block does not fit the privatised tile (Lp > 1024: Lp^2/8 > 128 KiB)
    if (m * s.C * (s.C - 1) < (int64_t)s.np * s.nw * 8 || cl.opt(kOptStoreScatter) == 1 ||
        p.tile_bytes > kPrivTileMax + (size_t)s.Lp * 4) {
        const int64_t threads = m * s.C;
        const int block = 256;
        const int64_t grid = (threads + block - 1) / block;
        store_kernel<<<(unsigned)grid, block, 0, st>>>(s, msgs, m, net->w8, net->dcount, net->dflag);
        cl.launched();
        return cudaGetLastError();
    }
    uint32_t *spart = cl.alloc_n<uint32_t>((size_t)p.chunks * s.np * s.nw);
    if (!spart) return cl.err;
    // vector loads of whole messages when C = 8, 16, 24, 32 and rows are 16-byte aligned
    const int nv = ((s.C % 8) == 0 && s.C <= 32 && ((uintptr_t)msgs & 15u) == 0) ? s.C / 8 : 0;
    auto fn = nv == 1 ? store_priv_kernel<1> : nv == 2 ? store_priv_kernel<2>
            : nv == 3 ? store_priv_kernel<3> : nv == 4 ? store_priv_kernel<4> : store_priv_kernel<0>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.tile_bytes);
    if (e != cudaSuccess) return e;
    fn<<<(unsigned)(p.chunks * p.tiles), GB_PRIV_NT, p.tile_bytes, st>>>(
        s, msgs, m, p.G, p.ngroups, p.tiles, p.per_chunk, spart, net->dcount, net->dflag);
    const int64_t total = (int64_t)s.np * s.nw;
    apply_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(s, spart, p.chunks, net->w8);
    cl.launched(2);
    return cudaGetLastError();
}

// OR `count` packed bit matrices into W8 (the apply pass of the privatised store).
cudaError_t launch_or_bits(Call &cl, const uint32_t *bits, int64_t count) {
    const int64_t total = (int64_t)cl.net->s.np * cl.net->s.nw;
    apply_kernel<<<(unsigned)((total + 255) / 256), 256, 0, cl.st>>>(cl.net->s, bits, (int)count, cl.net->w8);
    cl.launched();
    return cudaGetLastError();
}

// NVLS merge: every rank holds its partial packed rows Wb at the same offset of
// a buffer bound to a multicast object; one multimem.ld_reduce.or per word returns the OR over
// all ranks' copies (reduced in the NVSwitch), and the bits are set in W8 as apply_kernel does.
__global__ void or_multimem_kernel(Shape s, const uint32_t *mc, uint8_t *__restrict__ w8) {
    const int64_t total = (int64_t)s.np * s.nw;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        uint32_t bits;
        asm volatile("multimem.ld_reduce.relaxed.sys.global.or.b32 %0, [%1];" : "=r"(bits) : "l"(mc + idx) : "memory");
        if (!bits) continue;
        const int64_t i = idx / s.nw, w = idx - i * s.nw;
        uint4 *p = reinterpret_cast<uint4 *>(w8 + i * s.np + w * 32);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            uint4 v = p[h];
            uint32_t q[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t nib = (bits >> (16 * h + 4 * k)) & 15u;
                q[k] |= (nib & 1u) | ((nib & 2u) << 7) | ((nib & 4u) << 14) | ((nib & 8u) << 21);
            }
            p[h] = make_uint4(q[0], q[1], q[2], q[3]);
        }
    }
}

cudaError_t launch_or_multimem(Call &cl, const uint32_t *mc) {
    const int64_t total = (int64_t)cl.net->s.np * cl.net->s.nw;
    const int64_t grid = std::min<int64_t>((total + 255) / 256, (int64_t)cl.net->sm_count * 8);
    or_multimem_kernel<<<(unsigned)grid, 256, 0, cl.st>>>(cl.net->s, mc, cl.net->w8);
    cl.launched();
    return cudaGetLastError();
}

int64_t upper_words(const Shape &s) { return (int64_t)s.Lp * s.Wc * s.C * (s.C - 1) / 2; }

cudaError_t launch_pack_upper(Call &cl, uint32_t *out) {
    const int64_t total = upper_words(cl.net->s);
    const int64_t grid = std::min<int64_t>((total + 255) / 256, (int64_t)cl.net->sm_count * 8);
    pack_upper_kernel<<<(unsigned)grid, 256, 0, cl.st>>>(cl.net->s, cl.net->wb, out);
    cl.launched();
    return cudaGetLastError();
}

cudaError_t launch_or_upper(Call &cl, const uint32_t *sets, int64_t count) {
    const int64_t warps = upper_words(cl.net->s) / 32;
    const int64_t grid = std::min<int64_t>((warps * 32 + 255) / 256, (int64_t)cl.net->sm_count * 16);
    or_upper_kernel<<<(unsigned)grid, 256, 0, cl.st>>>(cl.net->s, sets, (int)count, cl.net->w8);
    cl.launched();
    return cudaGetLastError();
}

cudaError_t launch_seal(gb_net *net, cudaStream_t st) {
    const int64_t warps = (int64_t)(net->s.np / 32) * (net->s.np / 32);
    const int block = 256;
    const int64_t grid = (warps * 32 + block - 1) / block;
    const int64_t zthreads = (int64_t)net->s.C * net->s.C * net->s.Wc;   // wu_next zeroing
    const int64_t g2 = std::max<int64_t>(grid, (zthreads + block - 1) / block);
    seal_kernel<<<(unsigned)g2, block, 0, st>>>(net->s, net->w8, net->wb, net->dcount, net->hstat_dev,
                                                net->seal_gen, wu_of(net, net->seal_gen),
                                                wu_of(net, net->seal_gen + 1));
    net->launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}

}  // namespace gb
