// Feasibility probe: green contexts (SM partitions) with runtime-API launches,
// pool allocations made on the primary context, graph capture and PDL.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <set>
#include <vector>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)
#define DK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s_; cuGetErrorString(r_, &s_); printf("CU %s at %s:%d\n", s_, __FILE__, __LINE__); return 1; } } while (0)
__global__ void k_work(int* smids, float* data, long n, int iters) {
    unsigned sm; asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    if (threadIdx.x == 0) smids[blockIdx.x] = (int)sm;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        float v = data[i];
        for (int k = 0; k < iters; ++k) v = v * 1.0000001f + 0.5f;
        data[i] = v;
    }
}
__global__ void k_pdl(int* out) {
#if __CUDA_ARCH__ >= 900
    cudaGridDependencySynchronize();
#endif
    if (threadIdx.x == 0) atomicAdd(out, 1);
}
int main() {
    CK(cudaSetDevice(0));
    CK(cudaFree(0));
    CUdevice dev; DK(cuDeviceGet(&dev, 0));
    CUdevResource res; DK(cuDeviceGetDevResource(dev, &res, CU_DEV_RESOURCE_TYPE_SM));
    printf("device SMs: %u\n", res.sm.smCount);
    CUdevResource groups[1], rest; unsigned nb = 1;
    DK(cuDevSmResourceSplitByCount(groups, &nb, &res, &rest, 0, 32));
    printf("group SMs %u, remaining %u\n", groups[0].sm.smCount, rest.sm.smCount);
    CUdevResourceDesc dA, dB;
    DK(cuDevResourceGenerateDesc(&dA, groups, 1));
    DK(cuDevResourceGenerateDesc(&dB, &rest, 1));
    CUgreenCtx gA, gB;
    DK(cuGreenCtxCreate(&gA, dA, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    DK(cuGreenCtxCreate(&gB, dB, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CUstream sA, sB;
    DK(cuGreenCtxStreamCreate(&sA, gA, CU_STREAM_NON_BLOCKING, 0));
    DK(cuGreenCtxStreamCreate(&sB, gB, CU_STREAM_NON_BLOCKING, 0));
    cudaStream_t s0; CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));   // primary context stream
    const long n = 1L << 26; const int blocks = 4 * 148;
    float* data; int *smA, *smB, *cnt;
    CK(cudaMallocAsync((void**)&data, n * 4, s0));
    CK(cudaMallocAsync((void**)&smA, blocks * 4, s0));
    CK(cudaMallocAsync((void**)&smB, blocks * 4, s0));
    CK(cudaMallocAsync((void**)&cnt, 4, s0));
    CK(cudaMemsetAsync(data, 0, n * 4, s0));
    CK(cudaMemsetAsync(cnt, 0, 4, s0));
    CK(cudaStreamSynchronize(s0));
    // runtime launches on green streams, memory from the primary context's pool
    k_work<<<blocks, 256, 0, (cudaStream_t)sA>>>(smA, data, n / 2, 200);
    k_work<<<blocks, 256, 0, (cudaStream_t)sB>>>(smB, data + n / 2, n / 2, 200);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize((cudaStream_t)sA));
    CK(cudaStreamSynchronize((cudaStream_t)sB));
    std::vector<int> a(blocks), b(blocks);
    CK(cudaMemcpy(a.data(), smA, blocks * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(b.data(), smB, blocks * 4, cudaMemcpyDeviceToHost));
    std::set<int> sa(a.begin(), a.end()), sb(b.begin(), b.end());
    int overlap = 0; for (int x : sa) overlap += sb.count(x);
    printf("stream A used %zu SMs, stream B %zu SMs, overlap %d\n", sa.size(), sb.size(), overlap);
    float h[2]; CK(cudaMemcpy(h, data, 4, cudaMemcpyDeviceToHost)); CK(cudaMemcpy(h + 1, data + n - 1, 4, cudaMemcpyDeviceToHost));
    printf("data %f %f\n", h[0], h[1]);
    // pool allocation on a green stream, used by a primary-context kernel
    float* d2; CK(cudaMallocAsync((void**)&d2, 1 << 20, (cudaStream_t)sA));
    CK(cudaMemsetAsync(d2, 0, 1 << 20, (cudaStream_t)sA));
    CK(cudaStreamSynchronize((cudaStream_t)sA));
    k_work<<<4, 256, 0, s0>>>(smA, d2, 1 << 18, 1);
    CK(cudaStreamSynchronize(s0));
    printf("cross-context pool memory ok\n");
    // graph capture on a green stream + PDL launch
    cudaGraph_t g; cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture((cudaStream_t)sA, cudaStreamCaptureModeThreadLocal));
    k_work<<<blocks, 256, 0, (cudaStream_t)sA>>>(smA, data, 1 << 20, 1);
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(8); cfg.blockDim = dim3(32); cfg.stream = (cudaStream_t)sA;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, k_pdl, cnt));
    CK(cudaStreamEndCapture((cudaStream_t)sA, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    CK(cudaGraphLaunch(ge, (cudaStream_t)sA));
    CK(cudaStreamSynchronize((cudaStream_t)sA));
    int c = 0; CK(cudaMemcpy(&c, cnt, 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(a.data(), smA, blocks * 4, cudaMemcpyDeviceToHost));
    sa = std::set<int>(a.begin(), a.end());
    printf("graph on green stream: pdl count %d, SMs used %zu\n", c, sa.size());
    // event sync across a green and a primary stream
    cudaEvent_t ev; CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CK(cudaEventRecord(ev, (cudaStream_t)sA));
    CK(cudaStreamWaitEvent(s0, ev, 0));
    CK(cudaStreamSynchronize(s0));
    printf("ok\n");
    return 0;
}
