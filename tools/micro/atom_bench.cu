// Microbenchmark: shared-memory vs global (L2-resident) atomic throughput on
// random addresses, as used by the round-1 neighbour counting.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hsh(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
template <int NODES>
__global__ void k_smem(int iters, unsigned long long* out) {
    extern __shared__ uint32_t c[];
    for (int i = threadIdx.x; i < 2 * NODES; i += blockDim.x) c[i] = 0;
    __syncthreads();
    uint32_t s = hsh(blockIdx.x * 1024 + threadIdx.x);
    for (int i = 0; i < iters; ++i) {
        s = hsh(s);
        atomicAdd(&c[s & (2 * NODES - 1)], 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(out, c[0]);
}
__global__ void k_glob(int iters, uint32_t* c, uint32_t mask) {
    uint32_t s = hsh(blockIdx.x * 1024 + threadIdx.x);
    for (int i = 0; i < iters; ++i) {
        s = hsh(s);
        atomicAdd(&c[s & mask], 1u);
    }
}
// binned: the CTA's atomics stay inside a window that moves with blockIdx
__global__ void k_glob_win(int iters, uint32_t* c, uint32_t win) {
    uint32_t s = hsh(blockIdx.x * 1024 + threadIdx.x);
    uint32_t base = (blockIdx.x / 8) * win;
    for (int i = 0; i < iters; ++i) {
        s = hsh(s);
        atomicAdd(&c[base + (s & (win - 1))], 1u);
    }
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* out; cudaMalloc(&out, 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int iters = 1024; float ms;
    {
        constexpr int NODES = 16384;
        size_t sm = 2 * NODES * 4;
        cudaFuncSetAttribute(k_smem<NODES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        for (int threads : {256, 512, 1024}) {
            int grid = sms * (threads == 1024 ? 1 : 2048 / threads / 2);
            k_smem<NODES><<<grid, threads, sm>>>(iters, out);
            cudaEventRecord(a);
            for (int r = 0; r < 5; ++r) k_smem<NODES><<<grid, threads, sm>>>(iters, out);
            cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
            double ops = 5.0 * grid * threads * iters;
            printf("smem atomics 128KB table, %d thr x %d CTAs: %.1f G atom/s\n", threads, grid, ops / ms / 1e6);
        }
    }
    uint32_t* c; size_t big = 1ull << 30; cudaMalloc(&c, big * 4); cudaMemset(c, 0, big * 4);
    for (uint32_t mb : {4u, 16u, 64u, 1024u, 4096u}) {
        uint32_t mask = mb * 262144u - 1;
        int grid = sms * 4, threads = 512;
        k_glob<<<grid, threads>>>(iters, c, mask);
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) k_glob<<<grid, threads>>>(iters, c, mask);
        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        double ops = 5.0 * grid * threads * iters;
        printf("global RED random over %u MB: %.1f G atom/s\n", mb, ops / ms / 1e6);
    }
    for (uint32_t win : {1u << 15, 1u << 17, 1u << 19}) {
        int grid = sms * 4, threads = 512;
        k_glob_win<<<grid, threads>>>(iters, c, win);
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) k_glob_win<<<grid, threads>>>(iters, c, win);
        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        double ops = 5.0 * grid * threads * iters;
        printf("global RED windowed %u KB per 8 CTAs: %.1f G atom/s\n", win * 4 / 1024, ops / ms / 1e6);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
}
