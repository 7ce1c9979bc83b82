// lds_conflicts.cu -- shared-memory wavefronts of 16-byte loads (LDS.128) by bank-group pattern.
// Each lane reads 16 B from a random 128-B row at bank group g(lane) (the W bit-row layout of
// decode_hyb8_kernel).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lds lds_conflicts.cu
// Measured on B200 (ncu l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld / LDS instructions):
//   pattern 0  g = lane & 7 (8 distinct groups per quarter-warp)   4.0 wavefronts (ideal)
//   pattern 1  g = (lane >> 2) & 7                                 16.0
//   pattern 2  g random                                              9.4  (= the decode kernel's 9.2)
//   pattern 3  g = 0                                                32.0
//   pattern 4  2 lanes per group in each quarter-warp                8.0
// i.e. wavefronts are formed per quarter-warp (lanes 8q..8q+7) and a random row pick costs 2.3x.
#include <cstdio>
#include <cstdint>
// each lane reads 16 B from row r (random) at bank group g(lane, pattern)
__global__ void k(int pattern, uint32_t* out, int iters) {
    extern __shared__ __align__(16) uint32_t s[];
    for (int i = threadIdx.x; i < 1024 * 32; i += blockDim.x) s[i] = i * 2654435761u;
    __syncthreads();
    int lane = threadIdx.x & 31;
    uint32_t h = threadIdx.x * 747796405u + blockIdx.x;
    uint32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
        h = h * 1664525u + 1013904223u;
        uint32_t row = (h >> 8) & 1023;
        uint32_t g;
        if (pattern == 0) g = lane & 7;
        else if (pattern == 1) g = (lane >> 2) & 7;
        else if (pattern == 2) g = (h >> 20) & 7;
        else if (pattern == 3) g = 0;
        else g = (lane & 3) | ((lane >> 4) << 2);  // lanes 0-3,16-19 distinct?
        uint32_t a = row * 32 + g * 4;
        uint4 v = *reinterpret_cast<uint4*>(&s[a]);
        acc += v.x ^ v.y ^ v.z ^ v.w;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
    uint32_t* o; cudaMalloc(&o, 148 * 256 * 4);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    for (int p = 0; p < 5; ++p) {
        k<<<148, 256, 131072>>>(p, o, 4096);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        k<<<148, 256, 131072>>>(p, o, 4096);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("pattern %d: %.3f ms\n", p, ms);
    }
    return 0;
}
