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
// same, but the old value is used (rank-style ATOMS with return)
template <int NODES>
__global__ void k_smem_ret(int iters, unsigned long long* out) {
    extern __shared__ uint32_t c[];
    for (int i = threadIdx.x; i < 2 * NODES; i += blockDim.x) c[i] = 0;
    __syncthreads();
    uint32_t s = hsh(blockIdx.x * 1024 + threadIdx.x), acc = 0;
    for (int i = 0; i < iters; ++i) {
        s = hsh(s);
        acc += atomicAdd(&c[s & (2 * NODES - 1)], 1u);
    }
    __syncthreads();
    if (acc == 0xFFFFFFFFu) atomicAdd(out, acc);
}
// 8 independent ATOMS with return in flight per thread (the scatter's pattern)
__global__ void k_smem_ret8(int iters, unsigned long long* out, int mask) {
    extern __shared__ uint32_t c[];
    for (int i = threadIdx.x; i <= mask; i += blockDim.x) c[i] = 0;
    __syncthreads();
    uint32_t s = hsh(blockIdx.x * 1024 + threadIdx.x), acc = 0;
    for (int i = 0; i < iters; i += 8) {
        uint32_t r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) { s = hsh(s); r[j] = atomicAdd(&c[s & mask], 1u); }
#pragma unroll
        for (int j = 0; j < 8; ++j) acc += r[j];
    }
    __syncthreads();
    if (acc == 0xFFFFFFFFu) atomicAdd(out, acc);
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
    {
        constexpr int NODES = 16384;
        size_t sm = 2 * NODES * 4;
        cudaFuncSetAttribute(k_smem_ret<NODES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        cudaFuncSetAttribute(k_smem_ret8, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        int threads = 1024, grid = sms;
        k_smem_ret<NODES><<<grid, threads, sm>>>(iters, out);
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) k_smem_ret<NODES><<<grid, threads, sm>>>(iters, out);
        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("smem atomics WITH return (dependent use), 1024 thr: %.1f G atom/s\n", 5.0 * grid * threads * iters / ms / 1e6);
        for (int mask : {2047, 32767}) {
            k_smem_ret8<<<grid, threads, sm>>>(iters, out, mask);
            cudaEventRecord(a);
            for (int r = 0; r < 5; ++r) k_smem_ret8<<<grid, threads, sm>>>(iters, out, mask);
            cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
            printf("smem atomics WITH return, 8 in flight, %d addrs: %.1f G atom/s\n", mask + 1, 5.0 * grid * threads * iters / ms / 1e6);
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
