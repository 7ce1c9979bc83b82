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
