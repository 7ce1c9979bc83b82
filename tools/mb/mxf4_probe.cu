// mxf4_probe.cu -- feasibility probe (round-2 groundwork, not product code): is a 0/1 contraction
// exact on block-scaled FP4 (tcgen05.mma kind::mxf4, e2m1 operands 0 / 1.0, unit E8M0 scales,
// fp32 accumulate), and what is its issue rate vs kind::i8?  One CTA, M=128 x N=128 x K=256.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mxf4_probe mxf4_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1u << 16) | ((uint64_t)(1024u >> 4) << 32) |
           ((uint64_t)1u << 46) | ((uint64_t)2u << 61);
}

// A, B: 128 rows x 128 bytes each (K = 256 fp4 or 128 int8), row-major K, host layout unswizzled.
__global__ void probe(const uint8_t *A, const uint8_t *B, float *Dout, int mode, int iters, long long *cycles) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t *sa = sm, *sb = sm + 128 * 128;
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // swizzled copy: 16-byte chunk j of row r goes to chunk j ^ (r & 7)
    for (int i = tid; i < 128 * 8; i += blockDim.x) {
        const int r = i >> 3, j = i & 7;
        *reinterpret_cast<uint4 *>(sa + r * 128 + ((j ^ (r & 7)) << 4)) = reinterpret_cast<const uint4 *>(A)[i];
        *reinterpret_cast<uint4 *>(sb + r * 128 + ((j ^ (r & 7)) << 4)) = reinterpret_cast<const uint4 *>(B)[i];
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    // unit scale factors (E8M0 0x7F = 2^0) in columns 256..271 of every lane
    {
        const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16) + 256;
        const uint32_t one = 0x7F7F7F7Fu;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};"
                     ::"r"(taddr), "r"(one));
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    long long t0 = 0, t1 = 0;
    if (tid == 0) {
        const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
        uint32_t idesc;
        if (mode == 0) {   // kind::mxf4: a/b format E2M1 = 1, scale E8M0, M=128, N=128, K=64 per MMA
            idesc = (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | (1u << 23) | ((128u >> 4) << 24);
        } else {           // kind::i8: D s32 (2 << 4), A/B u8, M=128, N=128, K=32 per MMA
            idesc = (2u << 4) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
        }
        const uint32_t sfa = tmem + 256, sfb = tmem + 264;
        t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            for (int ks = 0; ks < 4; ++ks) {
                const uint64_t ad = sw128_desc(a0 + ks * 32), bd = sw128_desc(b0 + ks * 32);
                const uint32_t acc = (ks > 0) ? 1u : 0u;
                if (mode == 0) {
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}"
                                 ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb));
                } else {
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}"
                                 ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
                }
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
        asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}"
                     ::"r"(smem_u32(&bar)));
        t1 = clock64();
        *cycles = t1 - t0;
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    // read D: lane = row, 128 columns
    for (int g = 0; g < 4; ++g) {
        uint32_t v[32];
        const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16) + 32 * g;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                     "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                       "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                       "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                       "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                     : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int j = 0; j < 32; ++j)
            Dout[(32 * warp + lane) * 128 + 32 * g + j] = mode == 0 ? __uint_as_float(v[j]) : (float)(int)v[j];
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
    srand(7);
    std::vector<uint8_t> a(128 * 128), b(128 * 128);
    std::vector<int> abit(128 * 256), bbit(128 * 256);
    for (int mode = 0; mode < 2; ++mode) {
        const int K = mode == 0 ? 256 : 128;   // elements per 128-byte row
        for (int r = 0; r < 128; ++r)
            for (int kk = 0; kk < K; ++kk) {
                abit[r * 256 + kk] = rand() & 1;
                bbit[r * 256 + kk] = (rand() % 3) == 0;
            }
        for (int r = 0; r < 128; ++r)
            for (int by = 0; by < 128; ++by) {
                if (mode == 0) {   // two e2m1 per byte, element 2i in the low nibble, 1.0 = 0b0010
                    a[r * 128 + by] = (uint8_t)((abit[r * 256 + 2 * by] ? 0x2 : 0) | (abit[r * 256 + 2 * by + 1] ? 0x20 : 0));
                    b[r * 128 + by] = (uint8_t)((bbit[r * 256 + 2 * by] ? 0x2 : 0) | (bbit[r * 256 + 2 * by + 1] ? 0x20 : 0));
                } else {
                    a[r * 128 + by] = (uint8_t)abit[r * 256 + by];
                    b[r * 128 + by] = (uint8_t)bbit[r * 256 + by];
                }
            }
        uint8_t *dA, *dB;
        float *dD;
        long long *dc;
        cudaMalloc(&dA, a.size()); cudaMalloc(&dB, b.size()); cudaMalloc(&dD, 128 * 128 * 4); cudaMalloc(&dc, 8);
        cudaMemcpy(dA, a.data(), a.size(), cudaMemcpyHostToDevice);
        cudaMemcpy(dB, b.data(), b.size(), cudaMemcpyHostToDevice);
        cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 128 * 128);
        probe<<<1, 128, 2 * 128 * 128>>>(dA, dB, dD, mode, 1, dc);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> D(128 * 128);
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int i = 0; i < 128; ++i)
            for (int j = 0; j < 128; ++j) {
                int s = 0;
                for (int kk = 0; kk < K; ++kk) s += abit[i * 256 + kk] * bbit[j * 256 + kk];
                if (D[i * 128 + j] != (float)s) { if (bad < 5) printf("  mismatch (%d,%d): got %f want %d\n", i, j, D[i * 128 + j], s); ++bad; }
            }
        long long cyc = 0;
        probe<<<1, 128, 2 * 128 * 128>>>(dA, dB, dD, mode, 20000, dc);
        cudaDeviceSynchronize();
        cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
        const double ops = 2.0 * 128 * 128 * K * 20000.0;
        printf("%s: status %s, mismatches %d / 16384, %.1f ops/clk per SM (K=%d per 128-B row)\n",
               mode == 0 ? "kind::mxf4 (e2m1, unit E8M0 scales)" : "kind::i8", cudaGetErrorString(e), bad,
               ops / (double)cyc, K);
        cudaFree(dA); cudaFree(dB); cudaFree(dD); cudaFree(dc);
    }
    return 0;
}
