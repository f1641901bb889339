// grem_kernels.cu — hand-written sm_100a kernels of the GREM path.
//
// The reference sweep (process_chunk, grem.py:119-155) is sequential: node i
// sees the *live* labels of lower-id chunk neighbours and one shared `sizes`
// pair gates every decision.  It is reproduced exactly in parallel by rounds
// to a fixpoint:
//   counts   per node, lower neighbours read the tentative labels of the
//            previous round, higher neighbours the pre-sweep labels
//            (k_count_init / k_count_delta: edge-parallel, packed u64 REDs);
//   prefs    fp64 averaging (a + c) * 0.5 exactly as Python (k_prefs);
//   sizes    every node's effect on x = sizes[0] is a clamp; clamps compose in
//            O(1), so the exact sequential sizes chain is a parallel scan
//            (k_scan_*); ties (go to the smaller side) are not clamps, so
//            they are speculated, verified, and repaired by a sequential walk
//            only where the speculation was wrong (k_walk);
//   decide   b = [x - o <= t]; labels that changed feed the next round.
// A fixpoint equals the sequential result (by induction over the sweep).
#include <cub/cub.cuh>
#include <climits>
#include <thrust/iterator/counting_iterator.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "grem_core.cuh"
#include "grem_gen.h"
#include "grem_kernels.cuh"

namespace grem {

static int g_num_sms = 0;
int num_sms() {
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    return g_num_sms;
}

static inline unsigned grid_for(int64_t work, int threads, int per_sm = 8) {
    int64_t blocks = (work + threads - 1) / threads;
    int64_t cap = (int64_t)num_sms() * per_sm;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    return (unsigned)blocks;
}

#define GRID_STRIDE(i, n) for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); \
                               i += (int64_t)gridDim.x * blockDim.x)

// Programmatic dependent launch for the round kernels: each is launched with
// programmatic stream serialization (its CTAs may be scheduled while the
// previous kernel drains) and waits at entry (griddepcontrol.wait) until that
// kernel has completed and its writes are visible -- same semantics as a
// plain stream order, minus the launch gap.  GREM_NO_PDL=1: plain launches.
__device__ __forceinline__ void pdl_wait() {
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 900
    cudaGridDependencySynchronize();
#endif
}
static bool pdl_on() {
    static const bool on = getenv("GREM_NO_PDL") == nullptr;
    return on;
}
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
    if (!pdl_on()) {
        kern<<<grid, block, smem, s>>>(args...);
        return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, ((KArgs)args)...);
}

// ------------------------------------------------------------------ scan core

__device__ __forceinline__ Clamp shfl_up_clamp(const Clamp& v, int off) {
    Clamp r;
    r.d = __shfl_up_sync(0xffffffffu, v.d, off);
    r.L = __shfl_up_sync(0xffffffffu, v.L, off);
    r.U = __shfl_up_sync(0xffffffffu, v.U, off);
    return r;
}
__device__ __forceinline__ Clamp shfl_clamp(const Clamp& v, int src) {
    Clamp r;
    r.d = __shfl_sync(0xffffffffu, v.d, src);
    r.L = __shfl_sync(0xffffffffu, v.L, src);
    r.U = __shfl_sync(0xffffffffu, v.U, src);
    return r;
}

__device__ __forceinline__ Clamp warp_incl_scan(Clamp v) {
    int lane = threadIdx.x & 31;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        Clamp o = shfl_up_clamp(v, off);
        if (lane >= off) v = clamp_then(o, v);
    }
    return v;
}

// exclusive, order-respecting block scan of clamps (thread order)
template <int BT>
__device__ __forceinline__ Clamp block_excl_scan(Clamp v, Clamp* smem /* >= BT/32 */, Clamp* total) {
    int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NW = BT / 32;
    Clamp incl = warp_incl_scan(v);
    Clamp excl = shfl_up_clamp(incl, 1);
    if (lane == 0) excl = clamp_identity();
    if (lane == 31) smem[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        Clamp w = lane < NW ? smem[lane] : clamp_identity();
        Clamp wi = warp_incl_scan(w);
        Clamp we = shfl_up_clamp(wi, 1);
        if (lane == 0) we = clamp_identity();
        if (lane < NW) smem[lane] = we;
        if (lane == 31 && total) *total = wi;
    }
    __syncthreads();
    Clamp pre = smem[warp];
    __syncthreads();
    return clamp_then(pre, excl);
}

// map sources -----------------------------------------------------------------

struct ChunkMapSrc {
    const uint8_t* meta;
    const int32_t* newb;
    long long s0, cap;
    __device__ __forceinline__ NodeMap get(int64_t i) const {
        uint8_t m = meta[i];
        long long lift = (meta_active(m) && meta_old(m) != -1) ? 1 : 0;
        return node_map(m, s0 + newb[i] - lift, cap);
    }
};

// seed refinement pass (seed.py:96-116): moves are x-independent wishes gated
// by the receiving side's room; 0->1: x' = max(x-1, s-cap); 1->0: min(x+1, cap)
struct RefineMapSrc {
    const uint8_t* want;
    const int8_t* pre;
    long long s, cap;
    __device__ __forceinline__ NodeMap get(int64_t i) const {
        NodeMap r;
        r.o = 0;
        r.t = 0;
        if (!want[i]) {
            r.f = clamp_identity();
        } else if (pre[i] == 0) {
            r.f = Clamp{-1, s - cap, kInf};
        } else {
            r.f = Clamp{1, -kInf, cap};
        }
        return r;
    }
};

template <class Src>
__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(Src src, int64_t N, Clamp* tile_agg) {
    __shared__ Clamp smem[kScanThreads / 32];
    int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    Clamp acc = clamp_identity();
#pragma unroll 4
    for (int j = 0; j < kScanItems; ++j) {
        int64_t i = base + j;
        if (i < N) acc = clamp_then(acc, src.get(i).f);
    }
    __shared__ Clamp stotal;
    block_excl_scan<kScanThreads>(acc, smem, &stotal);
    __syncthreads();
    if (threadIdx.x == 0) tile_agg[blockIdx.x] = stotal;
}

// single block: exclusive scan over tile aggregates, evaluated at x0
__global__ void __launch_bounds__(1024) k_scan_top(const Clamp* tile_agg, int64_t ntiles, const long long* x0p,
                                                   long long* tile_x) {
    __shared__ Clamp smem[32];
    int64_t per = (ntiles + 1023) / 1024;
    int64_t lo = (int64_t)threadIdx.x * per;
    int64_t hi = lo + per < ntiles ? lo + per : ntiles;
    Clamp acc = clamp_identity();
    for (int64_t t = lo; t < hi; ++t) acc = clamp_then(acc, tile_agg[t]);
    Clamp pre = block_excl_scan<1024>(acc, smem, nullptr);
    long long x = clamp_apply(pre, *x0p);
    for (int64_t t = lo; t < hi; ++t) {
        tile_x[t] = x;
        x = clamp_apply(tile_agg[t], x);
    }
}

// chunk downsweep: x before every node, tie verification
struct ChunkOut {
    int32_t* x;
    uint8_t* bad;
    long long* tile_bad;
    long long* nbad;
    const uint8_t* meta;
};

template <class Src>
__global__ void __launch_bounds__(kScanThreads) k_scan_down_chunk(Src src, int64_t N, const long long* tile_x,
                                                                  ChunkOut out) {
    __shared__ Clamp smem[kScanThreads / 32];
    __shared__ long long sbad;
    if (threadIdx.x == 0) sbad = kInf;
    int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    Clamp acc = clamp_identity();
#pragma unroll 4
    for (int j = 0; j < kScanItems; ++j) {
        int64_t i = base + j;
        if (i < N) acc = clamp_then(acc, src.get(i).f);
    }
    Clamp pre = block_excl_scan<kScanThreads>(acc, smem, nullptr);
    long long x = clamp_apply(pre, tile_x[blockIdx.x]);
    long long mybad = kInf;
    int nb = 0;
    for (int j = 0; j < kScanItems; ++j) {
        int64_t i = base + j;
        if (i >= N) break;
        NodeMap nm = src.get(i);
        out.x[i] = (int32_t)x;
        uint8_t m = out.meta[i];
        uint8_t isbad = 0;
        if (meta_active(m) && meta_pref(m) == 2) {
            if (tie_misspeculated(m, x, nm)) {
                isbad = 1;
                if (i < mybad) mybad = i;
                nb++;
            }
        }
        out.bad[i] = isbad;
        x = clamp_apply(nm.f, x);
        if (i == N - 1) out.x[N] = (int32_t)x;
    }
    if (mybad != kInf) atomicMin(&sbad, mybad);
    if (nb) atomicAdd((unsigned long long*)out.nbad, (unsigned long long)nb);
    __syncthreads();
    if (threadIdx.x == 0) {
        out.tile_bad[blockIdx.x] = sbad;
        if (sbad != kInf) atomicMin(out.nbad + 2, sbad);   // scal[6]: first mis-speculated tie of the chunk
    }
}

template <class Src>
__global__ void __launch_bounds__(kScanThreads) k_scan_down_plain(Src src, int64_t N, const long long* tile_x,
                                                                  int32_t* xo) {
    __shared__ Clamp smem[kScanThreads / 32];
    int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    Clamp acc = clamp_identity();
    for (int j = 0; j < kScanItems; ++j) {
        int64_t i = base + j;
        if (i < N) acc = clamp_then(acc, src.get(i).f);
    }
    Clamp pre = block_excl_scan<kScanThreads>(acc, smem, nullptr);
    long long x = clamp_apply(pre, tile_x[blockIdx.x]);
    for (int j = 0; j < kScanItems; ++j) {
        int64_t i = base + j;
        if (i >= N) break;
        xo[i] = (int32_t)x;
        x = clamp_apply(src.get(i).f, x);
        if (i == N - 1) xo[N] = (int32_t)x;
    }
}

// ------------------------------------------------------------- counting

// ------------------------------------------------------------- hub table
// Hub table: bucketised 2-choice cuckoo hashing (kHubSlots / 2 buckets of two
// slots; built on the host, hub_table_build).  A lookup is two 8-byte shared
// loads and four compares: no probe loop, so no warp divergence.
__device__ __forceinline__ int hub_find(const uint32_t* s_keys, uint32_t u) {
    uint32_t b1 = hub_bucket1(u), b2 = hub_bucket2(u);
    uint2 p = reinterpret_cast<const uint2*>(s_keys)[b1];
    uint2 q = reinterpret_cast<const uint2*>(s_keys)[b2];
    int r = -1;
    r = p.x == u ? (int)(2 * b1) : r;
    r = p.y == u ? (int)(2 * b1 + 1) : r;
    r = q.x == u ? (int)(2 * b2) : r;
    r = q.y == u ? (int)(2 * b2 + 1) : r;
    return r;
}
// One-bit-per-hash prefilter in front of the hub table (64 Kbit, one hash):
// most endpoints are not hubs and leave after one 4-byte shared load instead
// of the table's two 8-byte ones (the table probes were 39% of
// k_bin_scatter's shared wavefronts, ncu r02i).  No false negatives.
constexpr int kBloomWords = 2048;
__device__ __forceinline__ uint32_t hub_bloom_bit(uint32_t u) { return (u * 0x2C1B3C6Du) >> 16; }
__device__ __forceinline__ void hub_bloom_build(uint32_t* s_bloom, const uint32_t* s_keys) {
    for (int k = threadIdx.x; k < kBloomWords; k += blockDim.x) s_bloom[k] = 0u;
    __syncthreads();
    for (int k = threadIdx.x; k < kHubSlots; k += blockDim.x) {
        uint32_t key = s_keys[k];
        if (key != kHubEmpty) {
            uint32_t h = hub_bloom_bit(key);
            atomicOr(&s_bloom[h >> 5], 1u << (h & 31));
        }
    }
}
__device__ __forceinline__ int hub_find_pf(const uint32_t* s_keys, const uint32_t* s_bloom, uint32_t u) {
    uint32_t h = hub_bloom_bit(u);
    if (!((s_bloom[h >> 5] >> (h & 31)) & 1u)) return -1;
    return hub_find(s_keys, u);
}
__device__ __forceinline__ void hub_load(uint32_t* s_keys, const uint32_t* hub_keys) {
    for (int k = threadIdx.x; k < kHubSlots; k += blockDim.x) s_keys[k] = hub_keys ? hub_keys[k] : kHubEmpty;
}

// contiguous edge range of this CTA (keeps the per-CTA hub flush amortised)
__device__ __forceinline__ void cta_range(int64_t m, int64_t& lo, int64_t& hi) {
    int64_t per = (m + gridDim.x - 1) / gridDim.x;
    lo = (int64_t)blockIdx.x * per;
    hi = lo + per < m ? lo + per : m;
}

constexpr int kEdgeThreads = 512;
#ifndef GREM_DELTA_UNROLL
#define GREM_DELTA_UNROLL 4
#endif
constexpr int kDeltaUnroll = GREM_DELTA_UNROLL;

// round 1: every chunk neighbour read with its pre-sweep label (cnt_nbrs,
// grem.py:82-97 / 138-145); nodes whose counts stay zero get a flag so the
// chunk node set (np.unique, model.py:59) still contains them.  Hub endpoints
// accumulate in shared memory.
__global__ void __launch_bounds__(kEdgeThreads) k_count_init(const uint2* __restrict__ e, int64_t m,
                                                             const int8_t* __restrict__ lab,
                                                             unsigned long long* __restrict__ cnt,
                                                             uint8_t* __restrict__ flag,
                                                             const uint32_t* __restrict__ hub_keys) {
    __shared__ __align__(8) uint32_t s_keys[kHubSlots];
    __shared__ unsigned long long s_cnt[kHubSlots];
    __shared__ uint8_t s_flag[kHubSlots];
    hub_load(s_keys, hub_keys);
    for (int k = threadIdx.x; k < kHubSlots; k += blockDim.x) {
        s_cnt[k] = 0ULL;
        s_flag[k] = 0;
    }
    __syncthreads();
    int64_t lo, hi;
    cta_range(m, lo, hi);
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        uint2 ed = e[i];
        uint32_t u = ed.x, v = ed.y;
        int hu = hub_find(s_keys, u);
        if (u == v) {   // self-loops never count (model.py:53-55) but make u a chunk node
            if (hu >= 0) s_flag[hu] = 1;
            else flag[u] = 1;
            continue;
        }
        int hv = hub_find(s_keys, v);
        int lu = lab[u], lv = lab[v];
        if (lv >= 0) {
            unsigned long long inc = lv == 0 ? 1ULL : (1ULL << 32);
            if (hu >= 0) atomicAdd(reinterpret_cast<unsigned int*>(s_cnt + hu) + (lv == 0 ? 0 : 1), 1u);   // native 32-bit half
            else atomicAdd(&cnt[u], inc);
        } else if (hu >= 0) {
            s_flag[hu] = 1;
        } else {
            flag[u] = 1;
        }
        if (lu >= 0) {
            unsigned long long inc = lu == 0 ? 1ULL : (1ULL << 32);
            if (hv >= 0) atomicAdd(reinterpret_cast<unsigned int*>(s_cnt + hv) + (lu == 0 ? 0 : 1), 1u);   // native 32-bit half
            else atomicAdd(&cnt[v], inc);
        } else if (hv >= 0) {
            s_flag[hv] = 1;
        } else {
            flag[v] = 1;
        }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < kHubSlots; k += blockDim.x) {
        uint32_t key = s_keys[k];
        if (key == kHubEmpty) continue;
        if (s_cnt[k]) atomicAdd(&cnt[key], s_cnt[k]);
        if (s_flag[k]) flag[key] = 1;
    }
}

__device__ __forceinline__ uint32_t word_rank(const uint2* __restrict__ rw, uint32_t g) {
    uint2 q = __ldg(rw + (g >> 5));
    return q.y + __popc(q.x & ((1u << (g & 31)) - 1u));
}

__device__ __forceinline__ void mark_changed_coarse(uint32_t* chgc, int shift, uint32_t g) {
    uint32_t c = g >> shift;
    uint32_t bit = 1u << (c & 31);
    if (!(((volatile uint32_t*)chgc)[c >> 5] & bit)) atomicOr(&chgc[c >> 5], bit);   // mostly set already
}

// rounds >= 2: the higher endpoint of every edge sees the lower endpoint's
// tentative label; apply the change since the previous round.
// STAGED (the first delta round of a chunk, where most lower endpoints
// changed): the per-edge chain of dependent gathers (changed bit -> label ->
// chunk index) runs stage by stage across the unrolled edges so each stage's
// loads are in flight together; later rounds (few active edges) keep the
// plain form, which has fewer registers and stays at 4 CTAs per SM.
#ifndef GREM_CD_MINB
#define GREM_CD_MINB 4   // CTAs per SM the plain delta kernel's register budget allows (A/B build knob)
#endif
// a hub's label-code change (prev -> cur) on its two 32-bit count halves
__device__ __forceinline__ void hub_delta_add(uint2* c, int cur, int prev) {
    unsigned int* h = reinterpret_cast<unsigned int*>(c);
    if (cur == 1) atomicAdd(h, 1u);
    else if (cur == 2) atomicAdd(h + 1, 1u);
    if (prev == 1) atomicAdd(h, 0xFFFFFFFFu);
    else if (prev == 2) atomicAdd(h + 1, 0xFFFFFFFFu);
}
template <bool STAGED>
__global__ void __launch_bounds__(kEdgeThreads, STAGED ? 3 : GREM_CD_MINB) k_count_delta(const uint2* __restrict__ e, int64_t m,
                                                              const uint8_t* __restrict__ tl,
                                                              const uint32_t* __restrict__ chg,
                                                              const uint2* __restrict__ rankw,
                                                              unsigned long long* __restrict__ cntc,
                                                              const uint32_t* __restrict__ hub_keys,
                                                              const long long* __restrict__ gate,
                                                              uint8_t* __restrict__ dirty,
                                                              const uint32_t* __restrict__ chgc, int cshift) {
    pdl_wait();
    if (gate && *gate == 0) return;   // previous round changed nothing (converged)
    __shared__ __align__(8) uint32_t s_keys[kHubSlots];
    // per hub slot: {label-0, label-1} count deltas as two 32-bit halves
    // (native shared atomics; a 64-bit shared atomicAdd is a CAS spin loop),
    // merged as hi * 2^32 + (signed) lo -- the same 64-bit packed delta
    __shared__ uint2 s_cnt[kHubSlots];
    __shared__ uint32_t s_chgc[kChgCoarseBits / 32];
    hub_load(s_keys, hub_keys);
    for (int k = threadIdx.x; k < kHubSlots; k += blockDim.x) s_cnt[k] = make_uint2(0u, 0u);
    for (int k = threadIdx.x; k < kChgCoarseBits / 32; k += blockDim.x) s_chgc[k] = chgc[k];
    __syncthreads();
    int64_t lo, hi;
    cta_range(m, lo, hi);
    // kDeltaUnroll independent edge loads in flight per thread before any of
    // them is filtered: the stream is latency bound with one load per thread.
    const int64_t bd = blockDim.x;
    for (int64_t i0 = lo + threadIdx.x; i0 < hi; i0 += kDeltaUnroll * bd) {
        uint2 ed[kDeltaUnroll];
#pragma unroll
        for (int j = 0; j < kDeltaUnroll; ++j) {
            int64_t i = i0 + j * bd;
            ed[j] = i < hi ? __ldcs(&e[i]) : make_uint2(0u, 0u);   // (0,0): a self-loop, skipped
        }
        if constexpr (STAGED) {
            uint32_t A[kDeltaUnroll], B[kDeltaUnroll], w[kDeltaUnroll];
            bool act[kDeltaUnroll];
#pragma unroll
            for (int j = 0; j < kDeltaUnroll; ++j) {
                uint32_t u = ed[j].x, v = ed[j].y;
                A[j] = u < v ? u : v;
                B[j] = u < v ? v : u;
                uint32_t ca = A[j] >> cshift;
                act[j] = u != v && ((s_chgc[ca >> 5] >> (ca & 31)) & 1u);
            }
#pragma unroll
            for (int j = 0; j < kDeltaUnroll; ++j) w[j] = act[j] ? chg[A[j] >> 5] : 0u;
            uint8_t t[kDeltaUnroll];
#pragma unroll
            for (int j = 0; j < kDeltaUnroll; ++j) {
                act[j] = (w[j] >> (A[j] & 31)) & 1u;
                t[j] = act[j] ? tl[A[j]] : (uint8_t)0;
            }
            int hb[kDeltaUnroll];
            uint2 q[kDeltaUnroll];
#pragma unroll
            for (int j = 0; j < kDeltaUnroll; ++j) {
                hb[j] = act[j] ? hub_find(s_keys, B[j]) : -1;
                q[j] = (act[j] && hb[j] < 0) ? __ldg(rankw + (B[j] >> 5)) : make_uint2(0u, 0u);
            }
#pragma unroll
            for (int j = 0; j < kDeltaUnroll; ++j) {
                if (!act[j]) continue;
                int cur = t[j] & 0xF, prev = t[j] >> 4;
                unsigned long long d = enc_label(cur) - enc_label(prev);
                if (hb[j] >= 0) {
                    hub_delta_add(s_cnt + hb[j], cur, prev);
                } else {
                    int32_t pb = (int32_t)(q[j].y + __popc(q[j].x & ((1u << (B[j] & 31)) - 1u)));
                    atomicAdd(&cntc[pb], d);
                    dirty[pb / kRTileC] = 1;
                }
            }
        } else {
#pragma unroll
        for (int j = 0; j < kDeltaUnroll; ++j) {
            uint32_t u = ed[j].x, v = ed[j].y;
            if (u == v) continue;
            uint32_t a = u < v ? u : v, b = u < v ? v : u;
            uint32_t ca = a >> cshift;
            if (!((s_chgc[ca >> 5] >> (ca & 31)) & 1u)) continue;   // coarse filter in shared memory
            if (!((chg[a >> 5] >> (a & 31)) & 1u)) continue;   // L2-resident bitmap of changed labels
            uint8_t t = tl[a];
            int cur = t & 0xF, prev = t >> 4;
            unsigned long long d = enc_label(cur) - enc_label(prev);
            int hb = hub_find(s_keys, b);
            if (hb >= 0) {
                hub_delta_add(s_cnt + hb, cur, prev);
            } else {
                int32_t pb = (int32_t)word_rank(rankw, b);   // L2-resident succinct map
                atomicAdd(&cntc[pb], d);
                dirty[pb / kRTileC] = 1;   // plain byte store: idempotent
            }
        }
        }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < kHubSlots; k += blockDim.x) {
        uint32_t key = s_keys[k];
        uint2 hc = s_cnt[k];
        unsigned long long dk = ((unsigned long long)hc.y << 32) + (unsigned long long)(long long)(int32_t)hc.x;
        if (key != kHubEmpty && dk) {
            int32_t pk = (int32_t)word_rank(rankw, key);
            atomicAdd(&cntc[pk], dk);
            dirty[pk / kRTileC] = 1;
        }
    }
}

static inline unsigned edge_grid(int64_t m, int per_sm = 4) {   // per_sm: resident CTAs of the kernel
    int64_t blocks = (m + 4 * kEdgeThreads - 1) / (4 * kEdgeThreads);
    int64_t cap = (int64_t)num_sms() * per_sm;
    if (blocks > cap) blocks = cap;
    return (unsigned)(blocks < 1 ? 1 : blocks);
}
// the delta pass loads a 24 KB shared-memory prologue per CTA (hub table,
// coarse filter): small chunks get >= 16 edges per thread so that prologue
// does not outweigh their edges (a 2.75M-edge chunk read 14 MB of prologue)
static inline unsigned delta_grid(int64_t m, int per_sm) {
    int64_t blocks = (m + 16 * kEdgeThreads - 1) / (16 * kEdgeThreads);
    int64_t lo = num_sms(), cap = (int64_t)num_sms() * per_sm;
    blocks = blocks < lo ? lo : (blocks > cap ? cap : blocks);
    return (unsigned)blocks;
}

void launch_count_init(const uint2* e, int64_t m, const ChunkBufs& b, cudaStream_t s) {
    k_count_init<<<edge_grid(m), kEdgeThreads, 0, s>>>(e, m, b.lab, b.cnt, b.flag, b.hub_keys);
}
void launch_count_delta(const uint2* e, int64_t m, const ChunkBufs& b, cudaStream_t s, bool staged) {
    if (staged) {
        launch_pdl(k_count_delta<true>, dim3(delta_grid(m, 3)), dim3(kEdgeThreads), 0, s, e, m, b.tl, b.chg, b.rankw, b.cntc, b.hub_keys,
                                                                     b.gate, b.dcur, b.chgc, b.chg_shift);
        return;
    }
    launch_pdl(k_count_delta<false>, dim3(delta_grid(m, GREM_CD_MINB)), dim3(kEdgeThreads), 0, s, e, m, b.tl, b.chg, b.rankw, b.cntc, b.hub_keys, b.gate, b.dcur,
                                                              b.chgc, b.chg_shift);
}

// -------------------------------------------------- binned round-1 counting
__device__ __forceinline__ uint32_t lab2_code(const uint32_t* __restrict__ lab2, uint32_t u) {
    return (lab2[u >> 4] >> ((u & 15) * 2)) & 3u;
}

// (bin offsets, scatter and the fused apply/compact are at the end of the file)

// hub detection: endpoint histogram of a sample, candidates, top-K
__global__ void k_sample_deg(const uint2* __restrict__ e, int64_t sample, int32_t* sdeg) {
    GRID_STRIDE(i, sample) {
        uint2 ed = e[i];
        atomicAdd(&sdeg[ed.x], 1);
        if (ed.y != ed.x) atomicAdd(&sdeg[ed.y], 1);
    }
}
void launch_sample_degrees(const uint2* e, int64_t sample, int32_t* sdeg, cudaStream_t s) {
    k_sample_deg<<<grid_for(sample, 256, 8), 256, 0, s>>>(e, sample, sdeg);
}
struct HubPred {
    const int32_t* sdeg;
    int32_t min_deg;
    __device__ __forceinline__ bool operator()(const uint32_t& i) const { return sdeg[i] >= min_deg; }
};
size_t hub_select_temp_bytes(int64_t n) {
    size_t bytes = 0;
    thrust::counting_iterator<uint32_t> it(0);
    cub::DeviceSelect::If(nullptr, bytes, it, (uint32_t*)nullptr, (long long*)nullptr, (int)n, HubPred{nullptr, 0});
    return bytes;
}
void launch_hub_select(const int32_t* sdeg, int64_t n, int32_t min_deg, uint32_t* ids, long long* d_count, void* temp,
                       size_t temp_bytes, cudaStream_t s) {
    thrust::counting_iterator<uint32_t> it(0);
    cub::DeviceSelect::If(temp, temp_bytes, it, ids, d_count, (int)n, HubPred{sdeg, min_deg}, s);
}
__global__ void k_hub_keys(const uint32_t* ids, int64_t cnt, const int32_t* sdeg, unsigned long long* keys) {
    GRID_STRIDE(j, cnt) keys[j] = ((unsigned long long)(uint32_t)sdeg[ids[j]] << 32) | ids[j];
}
void launch_hub_keys(const uint32_t* ids, int64_t cnt, const int32_t* sdeg, unsigned long long* keys, cudaStream_t s) {
    k_hub_keys<<<grid_for(cnt, 256), 256, 0, s>>>(ids, cnt, sdeg, keys);
}

__global__ void k_mark_all(const uint2* __restrict__ e, int64_t m, uint8_t* __restrict__ flag) {
    GRID_STRIDE(i, m) {
        uint2 ed = e[i];
        flag[ed.x] = 1;
        flag[ed.y] = 1;
    }
}
void launch_mark_all(const uint2* e, int64_t m, uint8_t* flag, cudaStream_t s) {
    k_mark_all<<<grid_for(m, 256, 16), 256, 0, s>>>(e, m, flag);
}

struct PresentPred {
    const uint8_t* flag;
    const unsigned long long* cnt;
    __device__ __forceinline__ bool operator()(const uint32_t& g) const { return flag[g] || cnt[g]; }
};

size_t select_nodes_temp_bytes(int64_t n) {
    size_t bytes = 0;
    thrust::counting_iterator<uint32_t> it(0);
    cub::DeviceSelect::If(nullptr, bytes, it, (uint32_t*)nullptr, (long long*)nullptr, (int)n,
                          PresentPred{nullptr, nullptr});
    return bytes;
}
void launch_select_nodes(const uint8_t* flag, const unsigned long long* cnt, int64_t n, uint32_t* nodes,
                         long long* d_count, void* temp, size_t temp_bytes, cudaStream_t s) {
    thrust::counting_iterator<uint32_t> it(0);
    cub::DeviceSelect::If(temp, temp_bytes, it, nodes, d_count, (int)n, PresentPred{flag, cnt}, s);
}

// ------------------------------------------------------------ node passes

// chunk node i: meta, compact round state (counts, estimates, label codes),
// the id -> index map; the id-indexed counters and flags are cleared for the
// next chunk here.
__global__ void k_node_init(const uint32_t* __restrict__ nodes, int64_t nc, const int8_t* __restrict__ lab,
                            int refine, uint8_t* __restrict__ meta, ChunkBufs b,
                            int32_t* __restrict__ newflag, long long* total_new) {
    int cnt_new = 0;
    GRID_STRIDE(i, nc) {
        uint32_t g = nodes[i];
        int old = lab[g];
        int code = old + 1;
        bool isnew = old == -1;
        bool active = isnew || refine;
        meta[i] = (uint8_t)(code | (active ? M_ACTIVE : 0) | (isnew ? M_NEW : 0));
        b.tlc[i] = (uint8_t)(code | (code << 4));
        b.cntc[i] = b.cnt[g];
        b.cnt[g] = 0ULL;
        b.flag[g] = 0;
        b.nbrc[i] = isnew ? make_double2(0.0, 0.0) : b.nbr[g];
        int nf = (active && isnew) ? 1 : 0;
        newflag[i] = nf;
        cnt_new += nf;
    }
    for (int off = 16; off; off >>= 1) cnt_new += __shfl_down_sync(0xffffffffu, cnt_new, off);
    if ((threadIdx.x & 31) == 0 && cnt_new) atomicAdd((unsigned long long*)total_new, (unsigned long long)cnt_new);
}

void launch_node_init(const ChunkBufs& b, int64_t nc, int refine, cudaStream_t s) {
    k_node_init<<<grid_for(nc, 256), 256, 0, s>>>(b.nodes, nc, b.lab, refine, b.meta, b, b.x, b.scal + 2);
}

__device__ __forceinline__ void averaged(uint8_t m, unsigned long long c, double2 nb, double& a0, double& a1) {
    double c0 = (double)(uint32_t)(c & 0xffffffffULL);
    double c1 = (double)(uint32_t)(c >> 32);
    if (meta_old(m) != -1) {   // (nbr + c) * 0.5 in binary64 (grem.py:147-148)
        a0 = __dmul_rn(__dadd_rn(nb.x, c0), 0.5);
        a1 = __dmul_rn(__dadd_rn(nb.y, c1), 0.5);
    } else {
        a0 = c0;
        a1 = c1;
    }
}


template <class Src>
static void run_scan_chunk(const Src& src, int64_t N, const ChunkBufs& b, cudaStream_t s) {
    int64_t ntiles = (N + kScanTile - 1) / kScanTile;
    k_scan_reduce<Src><<<(unsigned)ntiles, kScanThreads, 0, s>>>(src, N, b.tile_agg);
    k_scan_top<<<1, 1024, 0, s>>>(b.tile_agg, ntiles, b.sizes, b.tile_x);
    ChunkOut out{b.x, b.bad, b.tile_bad, b.scal + 4, b.meta};
    k_scan_down_chunk<Src><<<(unsigned)ntiles, kScanThreads, 0, s>>>(src, N, b.tile_x, out);
}

// The map source needs s_l = s0 + (active new nodes before i) - lift; s0 is
// folded into newb once per chunk so the source stays a plain value.
__global__ void k_add_base(int32_t* a, int64_t n, const long long* sizes) {
    long long s0 = sizes[0] + sizes[1];
    GRID_STRIDE(i, n) a[i] = (int32_t)(a[i] + s0);
}
void launch_add_base(int32_t* a, int64_t n, const long long* sizes, cudaStream_t s) {
    k_add_base<<<grid_for(n, 256), 256, 0, s>>>(a, n, sizes);
}

void launch_chunk_scan(const ChunkBufs& b, int64_t nc, long long cap, cudaStream_t s) {
    // newb already holds s0 + (active new nodes before i)  (see runtime)
    ChunkMapSrc src{b.meta, b.newb, 0, cap};
    run_scan_chunk(src, nc, b, s);
}

// Sequential repair of mis-speculated ties (single warp; all lanes run the
// chain redundantly, lanes prefetch node parameters in batches of 32).
__global__ void __launch_bounds__(32) k_walk(const uint8_t* __restrict__ meta, const int32_t* __restrict__ newb,
                                             int32_t* __restrict__ x, const uint8_t* __restrict__ bad,
                                             const long long* __restrict__ tile_bad, int64_t nc, long long cap,
                                             const long long* nbad, long long* steps_out) {
    if (*nbad == 0) return;
    const int lane = threadIdx.x;
    const int64_t ntiles = (nc + kScanTile - 1) / kScanTile;
    int64_t pos = 0;
    long long steps = 0;
    while (true) {
        // ---- next flagged index >= pos
        int64_t k = -1;
        int64_t t = pos / kScanTile;
        if (t < ntiles && tile_bad[t] != kInf) {
            int64_t lo = pos, hi = (t + 1) * kScanTile < nc ? (t + 1) * kScanTile : nc;
            for (int64_t j = lo; j < hi && k < 0; j += 32) {
                int64_t idx = j + lane;
                unsigned bal = __ballot_sync(0xffffffffu, idx < hi && bad[idx]);
                if (bal) k = j + __ffs(bal) - 1;
            }
        }
        for (int64_t tt = t + 1; k < 0 && tt < ntiles; tt += 32) {
            int64_t mt = tt + lane;
            unsigned bal = __ballot_sync(0xffffffffu, mt < ntiles && tile_bad[mt] != kInf);
            if (bal) {
                int64_t ft = tt + __ffs(bal) - 1;
                k = tile_bad[ft];
            }
        }
        if (k < 0) break;
        // ---- walk from k with the exact x until it re-joins the speculative chain
        long long xe = x[k];
        int64_t i = k;
        bool done = false;
        while (!done) {
            int64_t idx = i + lane;
            uint8_t m = idx < nc ? meta[idx] : 0;
            int32_t nb = idx < nc ? newb[idx] : 0;
            int32_t xs = idx < nc ? x[idx + 1] : 0;   // speculative x after node idx (read before writes)
            __syncwarp();
            for (int j = 0; j < 32; ++j) {
                int64_t p = i + j;
                uint8_t mj = __shfl_sync(0xffffffffu, m, j);
                int32_t nbj = __shfl_sync(0xffffffffu, nb, j);
                int32_t xsj = __shfl_sync(0xffffffffu, xs, j);
                if (p >= nc) { done = true; pos = nc; break; }
                long long lift = (meta_active(mj) && meta_old(mj) != -1) ? 1 : 0;
                NodeMap nm = node_map(mj, (long long)nbj - lift, cap);
                if (lane == 0) x[p] = (int32_t)xe;
                if (meta_active(mj)) xe = xe - nm.o + ((xe - nm.o <= nm.t) ? 1 : 0);
                steps++;
                if (p + 1 == nc) {
                    if (lane == 0) x[nc] = (int32_t)xe;
                    done = true;
                    pos = nc;
                    break;
                }
                if (xe == (long long)xsj) {   // re-joined: the speculative chain is exact again
                    done = true;
                    pos = p + 1;
                    break;
                }
            }
            i += 32;
            __syncwarp();
        }
        if (pos >= nc) break;
    }
    if (lane == 0) atomicAdd((unsigned long long*)steps_out, (unsigned long long)steps);
}

void launch_walk(const ChunkBufs& b, int64_t nc, long long cap, cudaStream_t s) {
    k_walk<<<1, 32, 0, s>>>(b.meta, b.newb, b.x, b.bad, b.tile_bad, nc, cap, b.scal + 4, b.scal + 3);
}

// ------------------------------------------------------- fused round kernels
// One fixpoint round = k_round_reduce (preferences + tile clamp aggregates),
// k_scan_top, k_round_down (exact-or-speculative x, tie verification,
// speculative decisions, next tie guesses) and, only when a tie was
// mis-speculated, the trajectory-bundle repair (which re-decides the repaired
// suffix).  Node arrays are padded to whole tiles with inactive (identity)
// nodes, so every thread moves kRI consecutive nodes with vector loads.
constexpr int kRT = 512;             // threads per tile
constexpr int kRI = 8;               // nodes per thread
constexpr int kRTile = kRT * kRI;    // == kScanTile
static_assert(kRTile == kScanTile, "round tiles reuse the scan tile buffers");
static_assert(kRTile == kRTileC, "dirty-tile granularity");

struct RoundArgs {
    const uint32_t* nodes;
    uint8_t* meta;
    const int32_t* newb;
    const unsigned long long* cnt;
    const double2* nbr;
    const long long* sizes;
    long long cap;
    int64_t nc;
    const long long* gate;   // nullptr or the previous round's changed count (0: converged, skip)
    const uint8_t* dcur;     // incremental rounds: tiles whose inputs changed since the last round
    uint8_t* dnext;          // tiles whose tie guesses changed (dirty in the next round)
    int incremental;         // skip clean tiles (round >= 3)
};

__device__ __forceinline__ void load8_u8(const uint8_t* p, uint8_t* v) {
    uint2 w = *reinterpret_cast<const uint2*>(p);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        v[k] = (uint8_t)(w.x >> (8 * k));
        v[4 + k] = (uint8_t)(w.y >> (8 * k));
    }
}
__device__ __forceinline__ void store8_u8(uint8_t* p, const uint8_t* v) {
    uint2 w;
    w.x = v[0] | (v[1] << 8) | (v[2] << 16) | ((uint32_t)v[3] << 24);
    w.y = v[4] | (v[5] << 8) | (v[6] << 16) | ((uint32_t)v[7] << 24);
    *reinterpret_cast<uint2*>(p) = w;
}
template <class T>
__device__ __forceinline__ void load8_32(const T* p, T* v) {
    int4 a = *reinterpret_cast<const int4*>(p), b = *reinterpret_cast<const int4*>(p + 4);
    v[0] = (T)a.x; v[1] = (T)a.y; v[2] = (T)a.z; v[3] = (T)a.w;
    v[4] = (T)b.x; v[5] = (T)b.y; v[6] = (T)b.z; v[7] = (T)b.w;
}
template <class T>
__device__ __forceinline__ void store8_32(T* p, const T* v) {
    *reinterpret_cast<int4*>(p) = make_int4((int)v[0], (int)v[1], (int)v[2], (int)v[3]);
    *reinterpret_cast<int4*>(p + 4) = make_int4((int)v[4], (int)v[5], (int)v[6], (int)v[7]);
}

__device__ __forceinline__ long long node_sl(uint8_t m, int32_t nb) {
    return (long long)nb - ((meta_active(m) && meta_old(m) != -1) ? 1 : 0);
}

__global__ void __launch_bounds__(kRT) k_round_reduce(RoundArgs a, Clamp* tile_agg, int first_round) {
    pdl_wait();
    if (a.gate && *a.gate == 0) return;
    // a clean tile (no count change, no tie-guess change) keeps its preferences
    // and its aggregate from the previous round
    if (a.incremental && !a.dcur[blockIdx.x]) return;
    __shared__ Clamp smem[kRT / 32];
    __shared__ Clamp stotal;
    int64_t base = (int64_t)blockIdx.x * kRTile + (int64_t)threadIdx.x * kRI;
    uint8_t m[kRI];
    int32_t nb[kRI];
    load8_u8(a.meta + base, m);
    load8_32(a.newb + base, nb);
    long long x0 = a.sizes[0];
    Clamp acc = clamp_identity();
#pragma unroll
    for (int j = 0; j < kRI; ++j) {
        uint8_t mm = m[j];
        if (meta_active(mm)) {   // preferences: assign() inputs (grem.py:138-150)
            unsigned long long c = a.cnt[base + j];
            double2 nbv = make_double2(0.0, 0.0);
            if (meta_old(mm) != -1) nbv = a.nbr[base + j];
            double a0, a1;
            averaged(mm, c, nbv, a0, a1);
            int pref = a0 < a1 ? 1 : (a1 < a0 ? 0 : 2);
            mm = (uint8_t)((mm & ~M_PREF) | (pref << M_PREF_SHIFT));
            if (first_round) {
                long long o = meta_old(mm) == 0 ? 1 : 0;
                bool side0 = (x0 - o) <= (node_sl(mm, nb[j]) >> 1);
                mm = (uint8_t)(side0 ? (mm & ~M_SPEC) : (mm | M_SPEC));
            }
            m[j] = mm;
        }
        acc = clamp_then(acc, node_map(m[j], node_sl(m[j], nb[j]), a.cap).f);
    }
    store8_u8(a.meta + base, m);
    block_excl_scan<kRT>(acc, smem, &stotal);
    __syncthreads();
    if (threadIdx.x == 0) tile_agg[blockIdx.x] = stotal;
}

struct RoundOut {
    int32_t* x;
    int32_t* xalt;
    uint8_t* tlc;      // compact codes (cur | prev << 4)
    uint8_t* tl;       // id-indexed codes, written for changed nodes only
    uint32_t* chg;     // id-indexed changed bits
    uint32_t* chgc;    // coarse changed filter
    int chg_shift;
    long long* scal;   // [1] changed, [4] nbad, [6] first bad
    uint8_t* segbad;   // per bundle segment of segL nodes: a mis-speculated tie (nullptr: not tracked)
    int64_t segL;
};

#ifndef GREM_RD_MINB
#define GREM_RD_MINB 2   // CTAs per SM the register budget of k_round_down allows (2: 647 vs 664 ms/step, r02d)
#endif
__global__ void __launch_bounds__(kRT, GREM_RD_MINB) k_round_down(RoundArgs a, const long long* tile_x, RoundOut out) {
    pdl_wait();
    if (a.gate && *a.gate == 0) return;
    __shared__ Clamp smem[kRT / 32];
    __shared__ long long sbad, sfirst;
    __shared__ int sspec;
    __shared__ unsigned int s_nbad, s_ch;   // block totals: one global atomic per tile, not per warp
    if (threadIdx.x == 0) {
        sbad = sfirst = kInf;
        sspec = 0;
        s_nbad = s_ch = 0u;
    }
    int64_t base = (int64_t)blockIdx.x * kRTile + (int64_t)threadIdx.x * kRI;
    if (a.incremental && !a.dcur[blockIdx.x] && (long long)out.x[(int64_t)blockIdx.x * kRTile] == tile_x[blockIdx.x]) {
        // clean tile entered with last round's exact x: every decision, tie
        // guess and x is what the last round computed; only the second window
        // centre (this round's exact x) needs the copy
        int32_t xs[kRI];
        load8_32(out.x + base, xs);
        store8_32(out.xalt + base, xs);
        if (base + kRI > a.nc && base <= a.nc) out.xalt[a.nc] = out.x[a.nc];
        return;
    }
    uint8_t m[kRI];
    int32_t nb[kRI];
    uint32_t g[kRI];
    load8_u8(a.meta + base, m);
    load8_32(a.newb + base, nb);
    Clamp acc = clamp_identity();
#pragma unroll
    for (int j = 0; j < kRI; ++j) acc = clamp_then(acc, node_map(m[j], node_sl(m[j], nb[j]), a.cap).f);
    Clamp pre = block_excl_scan<kRT>(acc, smem, nullptr);
    long long x = clamp_apply(pre, tile_x[blockIdx.x]);
    load8_32(a.nodes + base, g);
    uint8_t tc[kRI];
    load8_u8(out.tlc + base, tc);
    int32_t xs[kRI];
    int nbad = 0, ch = 0;
    long long mybad = kInf, mybad_ch = kInf;
    // changed bits: the thread's 8 nodes are consecutive chunk nodes (ascending
    // ids), so their bitmap words / coarse blocks repeat; OR them into one
    // RED per word / block instead of one per node, and never wait on a read
    // of the coarse filter (its latency, 8 times per thread in sequence,
    // dominated this kernel in round 1: ncu r02c)
    uint32_t cw = 0xFFFFFFFFu, cmask = 0u, kc = 0xFFFFFFFFu, kc0 = 0xFFFFFFFFu;
#pragma unroll
    for (int j = 0; j < kRI; ++j) {
        xs[j] = (int32_t)x;
        uint8_t mm = m[j];
        if (meta_active(mm)) {
            long long sl = node_sl(mm, nb[j]);
            NodeMap nm = node_map(mm, sl, a.cap);
            int b = (x - nm.o <= nm.t) ? 0 : 1;
            if (meta_pref(mm) == 2 && tie_misspeculated(mm, x, nm)) {   // mis-speculated tie
                nbad++;
                if (base + j < mybad) mybad = base + j;
                if (out.segbad) out.segbad[(base + j) / out.segL] = 1;
            }
            // speculative decision (exact unless a repair follows) and tentative label update
            int cur = tc[j] & 0xF, code = b + 1;
            tc[j] = (uint8_t)(code | (cur << 4));
            if (code != cur) {
                ch++;
                if (base + j < mybad_ch) mybad_ch = base + j;
                out.tl[g[j]] = tc[j];
                uint32_t w = g[j] >> 5;
                if (w != cw) {
                    if (cmask) atomicOr(&out.chg[cw], cmask);
                    cw = w;
                    cmask = 0u;
                }
                cmask |= 1u << (g[j] & 31);
                uint32_t c = g[j] >> out.chg_shift;
                if (c != kc) {   // coarse blocks: the first is OR-ed warp-wide below, later ones directly
                    if (kc0 == 0xFFFFFFFFu) kc0 = c;
                    else atomicOr(&out.chgc[c >> 5], 1u << (c & 31));
                    kc = c;
                }
            }
            // next round's tie guess: the tie rule at this x
            bool tie0 = (x - nm.o) <= (sl >> 1);
            m[j] = (uint8_t)(tie0 ? (mm & ~M_SPEC) : (mm | M_SPEC));
            if (meta_pref(mm) == 2 && m[j] != mm) sspec = 1;   // a tie's map changes next round
            x = clamp_apply(nm.f, x);
        }
    }
    if (cmask) atomicOr(&out.chg[cw], cmask);
    {   // the warp's lanes mostly share one coarse-filter word (a warp spans ~500
        // ids): one RED per distinct word instead of up to 32 on one address
        const bool has = kc0 != 0xFFFFFFFFu;
        const unsigned act = __ballot_sync(0xffffffffu, has);
        if (has) {
            const uint32_t wi = kc0 >> 5;
            const unsigned peers = __match_any_sync(act, wi);
            const uint32_t bits = __reduce_or_sync(peers, 1u << (kc0 & 31));
            if ((int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicOr(&out.chgc[wi], bits);
        }
    }
    store8_32(out.x + base, xs);
    store8_32(out.xalt + base, xs);
    store8_u8(a.meta + base, m);
    store8_u8(out.tlc + base, tc);
    if (base + kRI > a.nc && base <= a.nc) out.x[a.nc] = xs[a.nc - base];   // padding is identity
    for (int off = 16; off; off >>= 1) {
        nbad += __shfl_down_sync(0xffffffffu, nbad, off);
        ch += __shfl_down_sync(0xffffffffu, ch, off);
    }
    if (mybad != kInf) atomicMin(&sbad, mybad);
    if (mybad_ch != kInf) atomicMin(&sfirst, mybad_ch);
    if ((threadIdx.x & 31) == 0) {
        if (nbad) atomicAdd(&s_nbad, (unsigned int)nbad);
        if (ch) atomicAdd(&s_ch, (unsigned int)ch);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (s_nbad) atomicAdd((unsigned long long*)(out.scal + 4), (unsigned long long)s_nbad);
        if (s_ch) atomicAdd((unsigned long long*)(out.scal + 1), (unsigned long long)s_ch);
        if (sbad != kInf) atomicMin(out.scal + 6, sbad);
        if (sfirst != kInf) atomicMin(out.scal + 9, sfirst);   // first changed decision
        if (sspec) a.dnext[blockIdx.x] = 1;
    }
}

// ---- single-pass round (GREM_ROUND_FUSED=1; off by default: measured no faster): preferences, tile
// aggregate, decoupled look-back over round tiles (taken in ticket order) for
// the tile's incoming x, then decisions -- one launch and one read of the
// node state instead of reduce / top / down.  Look-back payloads are clamps
// (3 x 64 bit): written, fenced, then flagged (1: aggregate, 2: inclusive).
__device__ __forceinline__ Clamp ld_clamp_cg(const Clamp* p) {
    Clamp c;
    c.d = __ldcg(&p->d);
    c.L = __ldcg(&p->L);
    c.U = __ldcg(&p->U);
    return c;
}
__device__ Clamp clamp_lookback(const Clamp* agg, const Clamp* inc, const unsigned* flag, int64_t t) {
    const int lane = threadIdx.x & 31;
    Clamp acc = clamp_identity();   // composite of the tiles after the current window, up to t - 1
    int64_t j = t - 1;
    while (true) {
        int64_t q = j - lane;   // lane 0: nearest predecessor
        unsigned f = 2;
        Clamp v = clamp_identity();
        if (q >= 0) {
            do { f = ((volatile const unsigned*)flag)[q]; } while (f == 0);
            __threadfence();
            v = f == 2 ? ld_clamp_cg(inc + q) : ld_clamp_cg(agg + q);
        }
        unsigned incm = __ballot_sync(0xffffffffu, f == 2);
        int stop = incm ? __ffs(incm) - 1 : 31;
        Clamp w = clamp_identity();
        for (int l = stop; l >= 0; --l) w = clamp_then(w, shfl_clamp(v, l));   // tile order: lane stop first
        acc = clamp_then(w, acc);
        if (incm) break;
        j -= 32;
    }
    return acc;
}

struct FusedBufs {
    Clamp* tile_inc;
    unsigned* tflag;
    unsigned* ticket;
};

__global__ void __launch_bounds__(kRT, 2) k_round_fused(RoundArgs a, Clamp* tile_agg, FusedBufs fb, RoundOut out,
                                                     int first_round) {
    if (a.gate && *a.gate == 0) return;
    __shared__ int64_t s_tile;
    __shared__ Clamp smem[kRT / 32];
    __shared__ Clamp stotal, sprefix;
    __shared__ long long sbad, sfirst;
    __shared__ int sspec;
    if (threadIdx.x == 0) {
        s_tile = atomicAdd(fb.ticket, 1u);
        sbad = sfirst = kInf;
        sspec = 0;
    }
    __syncthreads();
    const int64_t t = s_tile;
    const int64_t base = t * kRTile + (int64_t)threadIdx.x * kRI;
    const bool clean = a.incremental && !a.dcur[t];
    uint8_t m[kRI];
    int32_t nb[kRI];
    load8_u8(a.meta + base, m);
    load8_32(a.newb + base, nb);
    const long long x0 = a.sizes[0];
    Clamp acc = clamp_identity();
    if (!clean) {
#pragma unroll
        for (int j = 0; j < kRI; ++j) {
            uint8_t mm = m[j];
            if (meta_active(mm)) {   // preferences: assign() inputs (grem.py:138-150)
                unsigned long long c = a.cnt[base + j];
                double2 nbv = make_double2(0.0, 0.0);
                if (meta_old(mm) != -1) nbv = a.nbr[base + j];
                double a0, a1;
                averaged(mm, c, nbv, a0, a1);
                int pref = a0 < a1 ? 1 : (a1 < a0 ? 0 : 2);
                mm = (uint8_t)((mm & ~M_PREF) | (pref << M_PREF_SHIFT));
                if (first_round) {
                    long long o = meta_old(mm) == 0 ? 1 : 0;
                    bool side0 = (x0 - o) <= (node_sl(mm, nb[j]) >> 1);
                    mm = (uint8_t)(side0 ? (mm & ~M_SPEC) : (mm | M_SPEC));
                }
                m[j] = mm;
            }
        }
    }
#pragma unroll
    for (int j = 0; j < kRI; ++j) acc = clamp_then(acc, node_map(m[j], node_sl(m[j], nb[j]), a.cap).f);
    Clamp pre = block_excl_scan<kRT>(acc, smem, &stotal);
    __syncthreads();
    if (threadIdx.x < 32) {
        Clamp agg = stotal;
        if (threadIdx.x == 0) {
            tile_agg[t] = agg;
            if (t == 0) fb.tile_inc[0] = agg;
            __threadfence();
            atomicExch(fb.tflag + t, t == 0 ? 2u : 1u);
        }
        Clamp prefix = t > 0 ? clamp_lookback(tile_agg, fb.tile_inc, fb.tflag, t) : clamp_identity();
        if (threadIdx.x == 0) {
            if (t > 0) {
                fb.tile_inc[t] = clamp_then(prefix, agg);
                __threadfence();
                atomicExch(fb.tflag + t, 2u);
            }
            sprefix = prefix;
        }
    }
    __syncthreads();
    const long long xin = clamp_apply(sprefix, x0);
    if (clean && (long long)out.x[t * kRTile] == xin) {
        // clean tile entered with last round's exact x: decisions, tie guesses
        // and x are the last round's; only the next window-centre buffer is copied
        int32_t xs[kRI];
        load8_32(out.x + base, xs);
        store8_32(out.xalt + base, xs);
        if (base + kRI > a.nc && base <= a.nc) out.xalt[a.nc] = out.x[a.nc];
        return;
    }
    if (!clean) store8_u8(a.meta + base, m);   // preference bits (tie guesses are rewritten below)
    long long x = clamp_apply(pre, xin);
    uint32_t g[kRI];
    load8_32(a.nodes + base, g);
    uint8_t tc[kRI];
    load8_u8(out.tlc + base, tc);
    int32_t xs[kRI];
    int nbad = 0, ch = 0;
    long long mybad = kInf, mybad_ch = kInf;
#pragma unroll
    for (int j = 0; j < kRI; ++j) {
        xs[j] = (int32_t)x;
        uint8_t mm = m[j];
        if (meta_active(mm)) {
            long long sl = node_sl(mm, nb[j]);
            NodeMap nm = node_map(mm, sl, a.cap);
            int b = (x - nm.o <= nm.t) ? 0 : 1;
            if (meta_pref(mm) == 2 && tie_misspeculated(mm, x, nm)) {   // mis-speculated tie
                nbad++;
                if (base + j < mybad) mybad = base + j;
            }
            int cur = tc[j] & 0xF, code = b + 1;
            tc[j] = (uint8_t)(code | (cur << 4));
            if (code != cur) {
                ch++;
                if (base + j < mybad_ch) mybad_ch = base + j;
                out.tl[g[j]] = tc[j];
                atomicOr(&out.chg[g[j] >> 5], 1u << (g[j] & 31));
                mark_changed_coarse(out.chgc, out.chg_shift, g[j]);
            }
            bool tie0 = (x - nm.o) <= (sl >> 1);
            m[j] = (uint8_t)(tie0 ? (mm & ~M_SPEC) : (mm | M_SPEC));
            if (meta_pref(mm) == 2 && m[j] != mm) sspec = 1;
            x = clamp_apply(nm.f, x);
        }
    }
    store8_32(out.x + base, xs);
    store8_32(out.xalt + base, xs);
    store8_u8(a.meta + base, m);
    store8_u8(out.tlc + base, tc);
    if (base + kRI > a.nc && base <= a.nc) out.x[a.nc] = xs[a.nc - base];   // padding is identity
    for (int off = 16; off; off >>= 1) {
        nbad += __shfl_down_sync(0xffffffffu, nbad, off);
        ch += __shfl_down_sync(0xffffffffu, ch, off);
    }
    if (mybad != kInf) atomicMin(&sbad, mybad);
    if (mybad_ch != kInf) atomicMin(&sfirst, mybad_ch);
    if ((threadIdx.x & 31) == 0) {
        if (nbad) atomicAdd((unsigned long long*)(out.scal + 4), (unsigned long long)nbad);
        if (ch) atomicAdd((unsigned long long*)(out.scal + 1), (unsigned long long)ch);
    }
    __syncthreads();
    if (threadIdx.x == 0 && sbad != kInf) atomicMin(out.scal + 6, sbad);
    if (threadIdx.x == 0 && sfirst != kInf) atomicMin(out.scal + 9, sfirst);
    if (threadIdx.x == 0 && sspec) a.dnext[t] = 1;
}

__global__ void k_scan_top_gated(const Clamp* tile_agg, int64_t ntiles, const long long* x0p, long long* tile_x,
                                 const long long* gate);
void launch_round_scan(const ChunkBufs& b, int64_t nc, long long cap, int first_round, int incremental,
                       cudaStream_t s) {
    RoundArgs a{b.nodes, b.meta, b.newb, b.cntc, b.nbrc, b.sizes, cap, nc, first_round ? nullptr : b.gate,
                b.dcur, b.dnext, incremental};
    int64_t ntiles = (nc + 1 + kRTile - 1) / kRTile;   // x[nc] falls in a tile too
    static const bool fused = getenv("GREM_ROUND_FUSED") != nullptr;   // measured: no gain over 3 launches
    RoundOut o{b.x, b.xnext, b.tlc, b.tl, b.chg, b.chgc, b.chg_shift, b.scal,
               (fused || b.bseg_len <= 0) ? nullptr : b.segbad, b.bseg_len};
    if (fused && b.tflag) {
        cudaMemsetAsync(b.tflag, 0, sizeof(unsigned) * (ntiles + 1), s);   // flags + ticket (last word)
        FusedBufs fb{b.tile_inc, b.tflag, b.tflag + ntiles};
        k_round_fused<<<(unsigned)ntiles, kRT, 0, s>>>(a, b.tile_agg, fb, o, first_round);
        return;
    }
    // kernel marks on full rounds only (incremental rounds skip clean tiles,
    // so their per-launch bytes are not the per-node figure)
    kmark(incremental ? KM_ROUND_REDUCE_ALL : KM_ROUND_REDUCE, 1, s);
    launch_pdl(k_round_reduce, dim3((unsigned)ntiles), dim3(kRT), 0, s, a, b.tile_agg, first_round);
    kmark(incremental ? KM_ROUND_REDUCE_ALL : KM_ROUND_REDUCE, 0, s);
    launch_pdl(k_scan_top_gated, dim3(1), dim3(1024), 0, s, (const Clamp*)b.tile_agg, ntiles, (const long long*)b.sizes, b.tile_x, b.gate);
    kmark(incremental ? KM_ROUND_DOWN_ALL : KM_ROUND_DOWN, 1, s);
    launch_pdl(k_round_down, dim3((unsigned)ntiles), dim3(kRT), 0, s, a, b.tile_x, o);
    kmark(incremental ? KM_ROUND_DOWN_ALL : KM_ROUND_DOWN, 0, s);
}

// ------------------------------------------------------- trajectory bundles
// Exact repair when tie speculation failed.  Ties pull the
// sizes chain toward balance, so trajectories started near the true value
// merge quickly.  Per segment of L nodes a CTA simulates kBundle trajectories
// from two windows of starting values (around this round's speculative x and
// around a second predictor); a single warp then chains the segments exactly
// (a lookup when the exact input falls in a window, a sequential simulation
// otherwise) and every segment replays its exact trajectory.

struct HalfMapSrc {   // half-step predictor: ties count +1/2 (doubled coordinates)
    const uint8_t* meta;
    const int32_t* newb;
    long long cap;
    __device__ __forceinline__ NodeMap get(int64_t i) const {
        NodeMap r;
        r.o = 0;
        r.t = 0;
        uint8_t m = meta[i];
        if (!meta_active(m)) {
            r.f = clamp_identity();
            return r;
        }
        long long o = meta_old(m) == 0 ? 1 : 0;
        long long lift = meta_old(m) != -1 ? 1 : 0;
        long long sl = (long long)newb[i] - lift;
        int pref = meta_pref(m);
        if (pref == 0) r.f = Clamp{2 - 2 * o, -kInf, 2 * cap};
        else if (pref == 1) r.f = Clamp{-2 * o, 2 * (sl - cap + 1), kInf};
        else r.f = Clamp{1 - 2 * o, 2 * (sl + 1 - cap), 2 * cap};
        return r;
    }
};

__global__ void k_double_x0(const long long* sizes, long long* out) { *out = 2 * sizes[0]; }

// gated variants: skip all work when the speculative scan was already exact
template <class Src>
__global__ void __launch_bounds__(kScanThreads) k_scan_reduce_gated(Src src, int64_t N, Clamp* tile_agg,
                                                                     const long long* gate) {
    if (*gate == 0) return;
    __shared__ Clamp smem[kScanThreads / 32];
    int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    Clamp acc = clamp_identity();
    for (int j = 0; j < kScanItems; ++j) {
        int64_t i = base + j;
        if (i < N) acc = clamp_then(acc, src.get(i).f);
    }
    __shared__ Clamp stotal;
    block_excl_scan<kScanThreads>(acc, smem, &stotal);
    __syncthreads();
    if (threadIdx.x == 0) tile_agg[blockIdx.x] = stotal;
}
__global__ void __launch_bounds__(1024) k_scan_top_gated(const Clamp* tile_agg, int64_t ntiles, const long long* x0p,
                                                         long long* tile_x, const long long* gate) {
    pdl_wait();
    if (gate && *gate == 0) return;
    __shared__ Clamp smem[32];
    int64_t per = (ntiles + 1023) / 1024;
    int64_t lo = (int64_t)threadIdx.x * per;
    int64_t hi = lo + per < ntiles ? lo + per : ntiles;
    Clamp acc = clamp_identity();
    for (int64_t t = lo; t < hi; ++t) acc = clamp_then(acc, tile_agg[t]);
    Clamp pre = block_excl_scan<1024>(acc, smem, nullptr);
    long long x = clamp_apply(pre, *x0p);
    for (int64_t t = lo; t < hi; ++t) {
        tile_x[t] = x;
        x = clamp_apply(tile_agg[t], x);
    }
}

template <class Src>
__global__ void __launch_bounds__(kScanThreads) k_scan_down_half(Src src, int64_t N, const long long* tile_x,
                                                                 int32_t* xo, const long long* gate) {
    if (*gate == 0) return;
    __shared__ Clamp smem[kScanThreads / 32];
    int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    Clamp acc = clamp_identity();
    for (int j = 0; j < kScanItems; ++j) {
        int64_t i = base + j;
        if (i < N) acc = clamp_then(acc, src.get(i).f);
    }
    Clamp pre = block_excl_scan<kScanThreads>(acc, smem, nullptr);
    long long x = clamp_apply(pre, tile_x[blockIdx.x]);
    for (int j = 0; j < kScanItems; ++j) {
        int64_t i = base + j;
        if (i >= N) break;
        xo[i] = (int32_t)(x >> 1);
        x = clamp_apply(src.get(i).f, x);
    }
}

void launch_half_predictor(const ChunkBufs& b, int64_t nc, long long cap, int32_t* xalt, cudaStream_t s) {
    HalfMapSrc src{b.meta, b.newb, cap};
    int64_t ntiles = (nc + kScanTile - 1) / kScanTile;
    k_double_x0<<<1, 1, 0, s>>>(b.sizes, b.scal + 5);
    k_scan_reduce_gated<HalfMapSrc><<<(unsigned)ntiles, kScanThreads, 0, s>>>(src, nc, b.tile_agg, b.scal + 4);
    k_scan_top_gated<<<1, 1024, 0, s>>>(b.tile_agg, ntiles, b.scal + 5, b.tile_x, b.scal + 4);
    k_scan_down_half<HalfMapSrc><<<(unsigned)ntiles, kScanThreads, 0, s>>>(src, nc, b.tile_x, xalt, b.scal + 4);
}

// per node: threshold t and lift o packed for the bundle loops:
// pk = t * 4 + o (arithmetic shift recovers t), o = 2 marks an inactive node.
__device__ __forceinline__ int32_t bundle_pack(uint8_t m, int32_t nb, long long cap) {
    if (!meta_active(m)) return 2;
    long long lift = meta_old(m) != -1 ? 1 : 0;
    NodeMap nm = node_map(m, (long long)nb - lift, cap);
    return (int32_t)(nm.t * 4 + nm.o);
}
__device__ __forceinline__ long long bundle_step(long long x, int32_t pk) {
    int o = pk & 3;
    if (o == 2) return x;
    long long xl = x - o;
    return xl + (xl <= (long long)(pk >> 2) ? 1 : 0);
}

constexpr int kBundleWin = 64;      // trajectories per window
constexpr int kBundleMaxWin = 3;    // windows: speculative x, previous exact x / half-step, balance point
constexpr int kBundleMax = kBundleWin * kBundleMaxWin;
constexpr int kBundleBatch = 2048;  // nodes staged in shared memory at a time
constexpr int kCkpt = 64;           // trajectory checkpoint stride (nodes)

__device__ __forceinline__ int64_t bundle_seg0(const long long* first_bad, int64_t L) { return *first_bad / L; }

__global__ void k_bundle_params(const uint8_t* __restrict__ meta, const int32_t* __restrict__ newb, int64_t nc,
                                int64_t L, long long cap, int32_t* __restrict__ bp, const long long* nbad,
                                const long long* first_bad, const uint8_t* __restrict__ segbad,
                                int32_t* __restrict__ segflag) {
    pdl_wait();
    if (*nbad == 0) return;
    int64_t lo = bundle_seg0(first_bad, L) * L;   // from the start of the first repaired segment
    if (segbad) {   // per segment: bit 0 a mis-speculated tie inside, bit 1 simulate (it or its predecessor)
        int64_t nseg = (nc + L - 1) / L;
        for (int64_t sg = lo / L + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; sg < nseg;
             sg += (int64_t)gridDim.x * blockDim.x) {
            bool b0 = segbad[sg], bp1 = sg > 0 && segbad[sg - 1];
            segflag[sg] = (b0 ? 1 : 0) | ((b0 || bp1) ? 2 : 0);
        }
    }
    for (int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nc; i += (int64_t)gridDim.x * blockDim.x)
        bp[i] = bundle_pack(meta[i], newb[i], cap);
}

// Segment simulation in offset coordinates: with O = the number of lifted
// (o = 1) active nodes since the segment start and z = x + O, one node is
// z' = z + [z < K] with K = t + o + O + 1 (inactive nodes: K = INT_MIN), a
// two-deep min/max chain in 32-bit registers; K is built per staged batch by
// a block scan of o.  Checkpoints and segment ends are stored as x = z - O.
template <int NWIN>
__global__ void __launch_bounds__(kBundleWin * NWIN) k_bundle_sim(const int32_t* __restrict__ bp,
                                                                 const int32_t* __restrict__ newb,
                                                                 const int32_t* __restrict__ xspec,
                                                                 const int32_t* __restrict__ xalt, int64_t nc,
                                                                 int64_t L, int32_t* __restrict__ ends,
                                                                 int32_t* __restrict__ ckpt, const long long* nbad,
                                                                 const long long* first_bad,
                                                                 const int32_t* __restrict__ segflag) {
    pdl_wait();
    constexpr int NT = kBundleWin * NWIN;
    constexpr int IPT = (kBundleBatch + NT - 1) / NT;
    if (*nbad == 0) return;
    int64_t seg = blockIdx.x;
    if (seg < bundle_seg0(first_bad, L)) return;
    // only segments holding a mis-speculated tie and the segment after each
    // need tables: elsewhere the exact trajectory is the speculative one as
    // long as it enters on it (the chain checks, a miss replays exactly)
    if (segflag && !(segflag[seg] & 2)) return;
    __shared__ int32_t sK[kBundleBatch];
    __shared__ int32_t sO[kBundleBatch / kCkpt + 1];
    __shared__ int32_t swarp[NT / 32 + 1];
    int64_t lo = seg * L;
    int64_t hi = lo + L < nc ? lo + L : nc;
    int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    int win = tid / kBundleWin;
    long long c = win == 0 ? xspec[lo] : (win == 1 ? xalt[lo] : ((long long)newb[lo] + 1) / 2);
    int32_t z = (int32_t)(c + (tid % kBundleWin) - kBundleWin / 2);
    int32_t ocarry = 0;   // O at the start of the staged batch
    int64_t ncp = (L + kCkpt - 1) / kCkpt;
    int32_t* ck = ckpt + seg * ncp * NT;
    for (int64_t b = lo; b < hi; b += kBundleBatch) {
        int cnt = (int)(hi - b < kBundleBatch ? hi - b : kBundleBatch);
        __syncthreads();
        // stage: o and t of this thread's IPT consecutive nodes, block scan of o
        int32_t pk[IPT];
        int osum = 0;
#pragma unroll
        for (int j = 0; j < IPT; ++j) {
            int k = tid * IPT + j;
            pk[j] = k < cnt ? bp[b + k] : 2;
            osum += (pk[j] & 3) == 1;
        }
        int incl = osum;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            int v = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += v;
        }
        if (lane == 31) swarp[wid] = incl;
        __syncthreads();
        int before = ocarry;
        for (int w = 0; w < wid; ++w) before += swarp[w];
        before += incl - osum;
#pragma unroll
        for (int j = 0; j < IPT; ++j) {
            int k = tid * IPT + j;
            if (k < cnt) {
                int o = pk[j] & 3;
                if ((k & (kCkpt - 1)) == 0) sO[k / kCkpt] = before;
                sK[k] = o == 2 ? INT_MIN : (pk[j] >> 2) + o + before + 1;
                before += o == 1;
            }
        }
        int total = 0;
        for (int w = 0; w < NT / 32; ++w) total += swarp[w];
        __syncthreads();
        for (int k0 = 0; k0 < cnt; k0 += kCkpt) {
            ck[((b - lo + k0) / kCkpt) * NT + tid] = z - sO[k0 / kCkpt];   // x before node b + k0
            int lim = cnt - k0 < kCkpt ? cnt - k0 : kCkpt;
            if (lim == kCkpt) {
#pragma unroll 16
                for (int k = 0; k < kCkpt; ++k) z = min(max(z, sK[k0 + k]), z + 1);
            } else {
                for (int k = 0; k < lim; ++k) z = min(max(z, sK[k0 + k]), z + 1);
            }
        }
        ocarry += total;
    }
    ends[seg * NT + tid] = z - ocarry;
}

// single warp: exact chain over segments.  Segment tables are staged into
// shared memory with cp.async, double buffered, so the dependent lookups of
// the chain overlap the loads of the next batch.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::); }

constexpr int kChainSB = 16;   // segments per staged batch

template <int NWIN>
__global__ void __launch_bounds__(32) k_bundle_chain(const int32_t* __restrict__ bp, const int32_t* __restrict__ newb,
                                                     const int32_t* __restrict__ xspec,
                                                     const int32_t* __restrict__ xalt, const int32_t* __restrict__ ends,
                                                     int64_t nseg, int64_t nc, int64_t L, int32_t* __restrict__ xin,
                                                     int32_t* __restrict__ hit_out, const long long* nbad,
                                                     const long long* first_bad, long long* misses,
                                                     const int32_t* __restrict__ segflag) {
    pdl_wait();
    constexpr int NT = kBundleWin * NWIN;
    if (*nbad == 0) return;
    const int lane = threadIdx.x;
    __shared__ __align__(16) int32_t tab[2][kChainSB * NT];
    __shared__ int32_t cen[2][kChainSB][NWIN];
    __shared__ int32_t sxe[2][kChainSB];   // speculative x at the segment's end
    __shared__ int32_t sflag[2][kChainSB];   // bit 0: mis-speculated tie inside, bit 1: simulated
    int64_t seg0 = bundle_seg0(first_bad, L);
    auto stage = [&](int buf, int64_t s0) {
        int cnt = (int)(nseg - s0 < kChainSB ? nseg - s0 : kChainSB);
        const int32_t* src = ends + s0 * NT;
        int n16 = cnt * NT / 4;
        for (int k = lane; k < n16; k += 32) cp_async16(&tab[buf][k * 4], src + k * 4);
        if (lane < cnt) {
            int64_t lo = (s0 + lane) * L;
            cp_async4(&cen[buf][lane][0], xspec + lo);
            if (NWIN > 1) cp_async4(&cen[buf][lane][1], xalt + lo);
            if (NWIN > 2) cp_async4(&cen[buf][lane][NWIN > 2 ? 2 : 0], newb + lo);   // balance point: (s + 1) / 2
            if (segflag) {
                cp_async4(&sxe[buf][lane], xspec + (lo + L < nc ? lo + L : nc));
                cp_async4(&sflag[buf][lane], segflag + s0 + lane);
            }
        }
        cp_async_commit();
    };
    long long cur = xspec[seg0 * L];   // exact: every tie before first_bad was consistent
    long long nmiss = 0;
    stage(0, seg0);
    int buf = 0;
    for (int64_t s0 = seg0; s0 < nseg; s0 += kChainSB, buf ^= 1) {
        int cnt = (int)(nseg - s0 < kChainSB ? nseg - s0 : kChainSB);
        if (s0 + kChainSB < nseg) {
            stage(buf ^ 1, s0 + kChainSB);
            cp_async_wait1();
        } else {
            cp_async_wait0();
        }
        __syncwarp();
        for (int j = 0; j < cnt; ++j) {
            int64_t seg = s0 + j;
            int hit = -1;
            int fl = segflag ? sflag[buf][j] : 3;   // no flags: every segment may hold a bad tie, all simulated
            if (!(fl & 1) && cur == (long long)cen[buf][j][0]) {
                // no mis-speculated tie and entered on the speculative trajectory:
                // the speculative decisions are exact here (final / fix skip it)
                if (lane == 0) {
                    xin[seg] = (int32_t)cur;
                    hit_out[seg] = -2;
                }
                cur = sxe[buf][j];
                continue;
            }
            if (fl & 2) {
#pragma unroll
                for (int w = 0; w < NWIN; ++w) {
                    long long cw = w == 2 ? ((long long)cen[buf][j][w] + 1) / 2 : (long long)cen[buf][j][w];
                    long long d = cur - cw + kBundleWin / 2;
                    if (hit < 0 && d >= 0 && d < kBundleWin) hit = w * kBundleWin + (int)d;
                }
            }
            if (lane == 0) {
                xin[seg] = (int32_t)cur;
                hit_out[seg] = hit;
            }
            if (hit >= 0) {
                cur = tab[buf][j * NT + hit];
            } else {   // window miss: simulate the segment (lanes prefetch 32 nodes)
                nmiss++;
                int64_t lo = seg * L, hi = lo + L < nc ? lo + L : nc;
                for (int64_t b = lo; b < hi; b += 32) {
                    int64_t idx = b + lane;
                    int32_t pk = idx < hi ? bp[idx] : 2;
                    int lim = (int)(hi - b < 32 ? hi - b : 32);
                    for (int k = 0; k < lim; ++k) cur = bundle_step(cur, __shfl_sync(0xffffffffu, pk, k));
                }
            }
        }
        __syncwarp();
    }
    if (lane == 0) atomicAdd((unsigned long long*)misses, (unsigned long long)nmiss);
}

// parallel replay of the exact trajectory: one thread per checkpoint interval;
// the repaired nodes are re-decided (their speculative decision, tentative
// label and next tie guess from k_round_down are corrected).
struct BundleFix {
    const uint32_t* nodes;
    uint8_t* meta;
    const int32_t* newb;
    uint8_t* tlc;
    uint8_t* tl;
    uint32_t* chg;
    int32_t* xalt;
    long long* changed;
    uint8_t* dnext;   // tie-guess changes make the tile dirty next round
    uint32_t* chgc;
    int chg_shift;
};

template <int NWIN>
__global__ void k_bundle_final(const int32_t* __restrict__ bp, const int32_t* __restrict__ xin,
                               const int32_t* __restrict__ hit, const int32_t* __restrict__ ckpt, int64_t nseg,
                               int64_t nc, int64_t L, int32_t* __restrict__ x, int32_t* __restrict__ xalt,
                               const long long* nbad, const long long* first_bad) {
    pdl_wait();
    constexpr int NT = kBundleWin * NWIN;
    if (*nbad == 0) return;
    int64_t ncp = (L + kCkpt - 1) / kCkpt;
    int64_t seg0 = bundle_seg0(first_bad, L);
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nseg * ncp;
         w += (int64_t)gridDim.x * blockDim.x) {
        int64_t seg = w / ncp, cp = w % ncp;
        if (seg < seg0) continue;
        int64_t lo = seg * L, hi = lo + L < nc ? lo + L : nc;
        int h = hit[seg];
        if (h == -2) continue;   // exact speculative trajectory (k_bundle_chain)
        long long cur;
        int64_t a, e;
        if (h >= 0) {
            a = lo + cp * kCkpt;
            if (a >= hi) continue;
            e = a + kCkpt < hi ? a + kCkpt : hi;
            cur = ckpt[(seg * ncp + cp) * NT + h];
        } else {   // window miss: one thread replays the segment
            if (cp) continue;
            a = lo;
            e = hi;
            cur = xin[seg];
        }
        if (e - a == kCkpt) {
            // a full interval (256-byte aligned): all 64 params in flight at
            // once, the chain in registers, 16-byte stores
            static_assert(kCkpt == 64, "interval = 16 x int4");
            int32_t xs[kCkpt];
#pragma unroll
            for (int q = 0; q < kCkpt / 4; ++q) {
                int4 p4 = __ldg(reinterpret_cast<const int4*>(bp + a) + q);
                int32_t pk[4] = {p4.x, p4.y, p4.z, p4.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    xs[q * 4 + j] = (int32_t)cur;
                    cur = bundle_step(cur, pk[j]);
                }
            }
#pragma unroll
            for (int q = 0; q < kCkpt / 4; ++q) {
                int4 v = make_int4(xs[4 * q], xs[4 * q + 1], xs[4 * q + 2], xs[4 * q + 3]);
                reinterpret_cast<int4*>(x + a)[q] = v;
                if (xalt) reinterpret_cast<int4*>(xalt + a)[q] = v;
            }
        } else {
            for (int64_t i = a; i < e; ++i) {
                x[i] = (int32_t)cur;
                if (xalt) xalt[i] = (int32_t)cur;
                cur = bundle_step(cur, bp[i]);
            }
        }
        if (e == nc) {
            x[nc] = (int32_t)cur;
            if (xalt) xalt[nc] = (int32_t)cur;
        }
    }
}

// the repaired suffix re-decided from its exact x, one thread per node
__global__ void k_bundle_fix(const int32_t* __restrict__ bp, const int32_t* __restrict__ x, int64_t nc, int64_t L,
                             const long long* nbad, const long long* first_bad, BundleFix fx,
                             const int32_t* __restrict__ hit) {
    pdl_wait();
    if (*nbad == 0) return;
    int64_t lo = bundle_seg0(first_bad, L) * L;
    long long dch = 0;
    for (int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nc;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (hit[i / L] == -2) continue;   // decided exactly by k_round_down already
        int32_t pk = bp[i];
        int o = pk & 3;
        if (o == 2) continue;
        long long cur = x[i];
        int b = (cur - o <= (long long)(pk >> 2)) ? 0 : 1;
        uint8_t t8 = fx.tlc[i];
        int spec_code = t8 & 0xF, prev = t8 >> 4;
        if (b + 1 != spec_code) {
            uint8_t nt = (uint8_t)((b + 1) | (prev << 4));
            fx.tlc[i] = nt;
            bool now = b + 1 != prev, was = spec_code != prev;
            dch += (long long)now - (long long)was;
            uint32_t g = fx.nodes[i];
            if (now) {
                fx.tl[g] = nt;
                if (!was) {
                    atomicOr(&fx.chg[g >> 5], 1u << (g & 31));
                    uint32_t cc = g >> fx.chg_shift;
                    atomicOr(&fx.chgc[cc >> 5], 1u << (cc & 31));   // RED: no dependent read of the filter
                }
            } else if (was) {
                atomicAnd(&fx.chg[g >> 5], ~(1u << (g & 31)));
            }
        }
        uint8_t m = fx.meta[i];
        bool tie0 = (cur - o) <= (node_sl(m, fx.newb[i]) >> 1);
        uint8_t m2 = (uint8_t)(tie0 ? (m & ~M_SPEC) : (m | M_SPEC));
        fx.meta[i] = m2;
        if (m2 != m && meta_pref(m) == 2) fx.dnext[i / kRTile] = 1;
    }
    for (int off = 16; off; off >>= 1) dch += __shfl_down_sync(0xffffffffu, dch, off);
    if ((threadIdx.x & 31) == 0 && dch) atomicAdd((unsigned long long*)fx.changed, (unsigned long long)dch);
}

int64_t bundle_segment_len(int64_t nc) {
    // the chain costs ~140 cycles per segment (dependent smem lookups) and a
    // segment's simulation ~6 cycles per node: L ~ sqrt(24 nc) balances them
    static const double kb = getenv("GREM_BUNDLE_K") ? atof(getenv("GREM_BUNDLE_K")) : 24.0;
    int64_t L = (int64_t)std::sqrt(kb * (double)nc);
    if (L < kCkpt) L = kCkpt;
    if ((nc + L - 1) / L > 4096) L = (nc + 4095) / 4096;
    return (L + kCkpt - 1) / kCkpt * kCkpt;
}
int64_t bundle_ckpt_ints(int64_t nc) {
    int64_t L = bundle_segment_len(nc);
    int64_t nseg = (nc + L - 1) / L;
    return nseg * ((L + kCkpt - 1) / kCkpt) * kBundleMax;
}

void launch_bundle(const ChunkBufs& b, int64_t nc, long long cap, const int32_t* xalt, const BundleBufs& bb, int nwin,
                   cudaStream_t s, bool fix_decisions) {
    int64_t L = bundle_segment_len(nc);
    int64_t nseg = (nc + L - 1) / L;
    int64_t ncp = (L + kCkpt - 1) / kCkpt;
    // per-segment mis-speculation flags from k_round_down (same L); without
    // them (fused round kernel, debug entry points) every segment is simulated
    static const bool fused = getenv("GREM_ROUND_FUSED") != nullptr;
    static const bool no_skip = getenv("GREM_BUNDLE_NO_SKIP") != nullptr;   // A/B switch
    const uint8_t* segbad = (!fused && !no_skip && fix_decisions && b.bseg_len == L) ? b.segbad : nullptr;
    const long long* nbad = b.scal + 4;
    const long long* first_bad = b.scal + 6;
    BundleFix fx{b.nodes, b.meta,  b.newb, b.tlc, b.tl, b.chg, fix_decisions ? b.xnext : nullptr,
                 fix_decisions ? b.scal + 1 : nullptr, b.dnext, b.chgc, b.chg_shift};
    int32_t* segflag = segbad ? bb.segflag : nullptr;
    launch_pdl(k_bundle_params, dim3(grid_for(nc, 256)), dim3(256), 0, s, b.meta, b.newb, nc, L, cap, bb.params, nbad, first_bad, segbad,
                                                      segflag);
    unsigned fgrid = (unsigned)((nseg * ncp + 255) / 256);
    int32_t* xalt_out = fix_decisions ? b.xnext : nullptr;
    if (nwin == 3) {
        launch_pdl(k_bundle_sim<3>, dim3((unsigned)nseg), dim3(kBundleWin * 3), 0, s, bb.params, b.newb, b.x, xalt, nc, L, bb.ends, bb.ckpt,
                                                                 nbad, first_bad, segflag);
        launch_pdl(k_bundle_chain<3>, dim3(1), dim3(32), 0, s, bb.params, b.newb, b.x, xalt, bb.ends, nseg, nc, L, bb.xin, bb.hit, nbad,
                                           first_bad, b.scal + 3, segflag);
        launch_pdl(k_bundle_final<3>, dim3(fgrid), dim3(256), 0, s, bb.params, bb.xin, bb.hit, bb.ckpt, nseg, nc, L, b.x, xalt_out, nbad,
                                               first_bad);
    } else {
        launch_pdl(k_bundle_sim<2>, dim3((unsigned)nseg), dim3(kBundleWin * 2), 0, s, bb.params, b.newb, b.x, xalt, nc, L, bb.ends, bb.ckpt,
                                                                 nbad, first_bad, segflag);
        launch_pdl(k_bundle_chain<2>, dim3(1), dim3(32), 0, s, bb.params, b.newb, b.x, xalt, bb.ends, nseg, nc, L, bb.xin, bb.hit, nbad,
                                           first_bad, b.scal + 3, segflag);
        launch_pdl(k_bundle_final<2>, dim3(fgrid), dim3(256), 0, s, bb.params, bb.xin, bb.hit, bb.ckpt, nseg, nc, L, b.x, xalt_out, nbad,
                                               first_bad);
    }
    if (fix_decisions) launch_pdl(k_bundle_fix, dim3(grid_for(nc, 256)), dim3(256), 0, s, bb.params, b.x, nc, L, nbad, first_bad, fx, bb.hit);
}


__global__ void k_commit(const uint32_t* __restrict__ nodes, int64_t nc, const uint8_t* __restrict__ meta,
                         const unsigned long long* __restrict__ cntc, const double2* __restrict__ nbrc,
                         double2* __restrict__ nbr, int8_t* __restrict__ lab, const uint8_t* __restrict__ tlc,
                         uint32_t* __restrict__ lab2) {
    GRID_STRIDE(i, nc) {
        uint8_t m = meta[i];
        if (meta_active(m)) {
            uint32_t g = nodes[i];
            double a0, a1;
            averaged(m, cntc[i], nbrc[i], a0, a1);
            nbr[g] = make_double2(a0, a1);
            int code = tlc[i] & 0xF;
            lab[g] = (int8_t)(code - 1);
            uint32_t diff = (uint32_t)((code ^ (m & M_OLD)) & 3);
            if (diff) atomicXor(&lab2[g >> 4], diff << ((g & 15) * 2));
        }
    }
}

void launch_commit(const ChunkBufs& b, int64_t nc, cudaStream_t s) {
    k_commit<<<grid_for(nc, 256), 256, 0, s>>>(b.nodes, nc, b.meta, b.cntc, b.nbrc, b.nbr, b.lab, b.tlc, b.lab2);
}

// start of a round: one launch instead of five memsets -- per-round scalars
// (changed, mis-speculated ties, first bad / first change = +large), next
// round's dirty tiles cleared, round 1: every tile dirty
// Round r >= 2 also closes round r-1's gate (it ran iff scal[7] != 0; round r
// runs iff round r-1 changed a label) and clears this round's changed-label
// bitmaps (double buffered: round r writes chg[r&1], count_delta(r+1) reads it).
__global__ void k_round_start(long long* scal, uint8_t* dnext, uint8_t* dcur_all, int64_t nt, int first_round,
                              uint32_t* chg, int64_t nchg, uint32_t* chgc, int64_t nchgc, uint8_t* segbad,
                              int64_t nseg) {
    pdl_wait();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (!first_round) {
            if (scal[7]) scal[8] += 1;
            scal[7] = scal[1];
        }
        scal[1] = 0;
        scal[4] = 0;
        scal[6] = 0x7F7F7F7F7F7F7F7FLL;
        scal[9] = 0x7F7F7F7F7F7F7F7FLL;
    }
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nt; i += stride) {
        dnext[i] = 0;
        if (dcur_all) dcur_all[i] = 1;
    }
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nchg; i += stride) chg[i] = 0u;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nchgc; i += stride) chgc[i] = 0u;
    if (segbad)
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nseg; i += stride) segbad[i] = 0;
}
void launch_round_start(const ChunkBufs& b, int64_t nt, bool first_round, int64_t nchg_words, cudaStream_t s) {
    int64_t work = nt > nchg_words ? nt : nchg_words;
    int64_t nseg = b.bseg_len > 0 ? b.bseg_n + 1 : 0;   // (the buffer holds bseg_n + 2 flags)
    launch_pdl(k_round_start, dim3(grid_for(work, 256)), dim3(256), 0, s, b.scal, b.dnext, first_round ? b.dcur : nullptr, nt,
                                                       first_round ? 1 : 0, b.chg, nchg_words, b.chgc,
                                                       kChgCoarseBits / 32, b.bseg_len > 0 ? b.segbad : nullptr,
                                                       nseg);
}

// body tail of the device-side round loop (a conditional WHILE graph node,
// grem_runtime.cu process_chunk): iterate again while the pair's last round
// changed a label, within the round budget the host loop also enforced
__global__ void k_loop_cond(cudaGraphConditionalHandle h, const long long* scal, long long max_rounds) {
    bool again = scal[1] != 0 && scal[8] + 2 < max_rounds;
    cudaGraphSetConditional(h, again ? 1u : 0u);
}
void launch_loop_cond(cudaGraphConditionalHandle h, const long long* scal, long long max_rounds, cudaStream_t s) {
    k_loop_cond<<<1, 1, 0, s>>>(h, scal, max_rounds);
}

// end of a round: the next round runs only if this one changed a label;
// scal[8] counts the rounds that actually ran
__global__ void k_round_gate(long long* scal) {
    if (scal[7]) scal[8] += 1;
    scal[7] = scal[1];
}
void launch_round_gate(const ChunkBufs& b, cudaStream_t s) { k_round_gate<<<1, 1, 0, s>>>(b.scal); }

__global__ void k_sizes_update(long long* sizes, const int32_t* x, int64_t nc, const long long* total_new) {
    long long s0 = sizes[0] + sizes[1];
    long long xe = x[nc];
    sizes[0] = xe;
    sizes[1] = s0 + *total_new - xe;
}
void launch_sizes_update(const ChunkBufs& b, int64_t nc, cudaStream_t s) {
    k_sizes_update<<<1, 1, 0, s>>>(b.sizes, b.x, nc, b.scal + 2);
}

// ----------------------------------------------------------------- seed

__global__ void k_set_rank(const uint32_t* nodes, int64_t nc, int32_t* rank) {
    GRID_STRIDE(i, nc) rank[nodes[i]] = (int32_t)i;
}
void launch_set_rank(const uint32_t* nodes, int64_t nc, int32_t* rank, cudaStream_t s) {
    k_set_rank<<<grid_for(nc, 256), 256, 0, s>>>(nodes, nc, rank);
}

__global__ void __launch_bounds__(kEdgeThreads) k_degrees(const uint2* __restrict__ e, int64_t m,
                                                          const int32_t* __restrict__ rank, int32_t* __restrict__ deg,
                                                          const uint32_t* __restrict__ hub_keys) {
    __shared__ __align__(8) uint32_t s_keys[kHubSlots];
    __shared__ uint32_t s_deg[kHubSlots];
    hub_load(s_keys, hub_keys);
    for (int k = threadIdx.x; k < kHubSlots; k += blockDim.x) s_deg[k] = 0;
    __syncthreads();
    int64_t lo, hi;
    cta_range(m, lo, hi);
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        uint2 ed = e[i];
        if (ed.x == ed.y) continue;
        int hu = hub_find(s_keys, ed.x), hv = hub_find(s_keys, ed.y);
        if (hu >= 0) atomicAdd(&s_deg[hu], 1u);
        else atomicAdd(&deg[rank[ed.x]], 1);
        if (hv >= 0) atomicAdd(&s_deg[hv], 1u);
        else atomicAdd(&deg[rank[ed.y]], 1);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < kHubSlots; k += blockDim.x) {
        uint32_t key = s_keys[k];
        if (key != kHubEmpty && s_deg[k]) atomicAdd(&deg[rank[key]], (int32_t)s_deg[k]);
    }
}
void launch_degrees(const uint2* e, int64_t m, const int32_t* rank, int32_t* deg, const uint32_t* hub_keys,
                    cudaStream_t s) {
    k_degrees<<<edge_grid(m), kEdgeThreads, 0, s>>>(e, m, rank, deg, hub_keys);
}

// CSR fill: hubs reserve one contiguous block per CTA (count pass over the
// CTA's edge range, one global atomic per hub, then fill from the block).
__global__ void __launch_bounds__(kEdgeThreads) k_fill_csr(const uint2* __restrict__ e, int64_t m,
                                                           const int32_t* __restrict__ rank,
                                                           int32_t* __restrict__ cursor, uint32_t* __restrict__ adj,
                                                           uint32_t* __restrict__ row_of,
                                                           const uint32_t* __restrict__ hub_keys) {
    __shared__ __align__(8) uint32_t s_keys[kHubSlots];
    __shared__ int32_t s_pos[kHubSlots];
    hub_load(s_keys, hub_keys);
    for (int k = threadIdx.x; k < kHubSlots; k += blockDim.x) s_pos[k] = 0;
    __syncthreads();
    int64_t lo, hi;
    cta_range(m, lo, hi);
    if (hub_keys) {
        for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
            uint2 ed = e[i];
            if (ed.x == ed.y) continue;
            int hu = hub_find(s_keys, ed.x), hv = hub_find(s_keys, ed.y);
            if (hu >= 0) atomicAdd(&s_pos[hu], 1);
            if (hv >= 0) atomicAdd(&s_pos[hv], 1);
        }
        __syncthreads();
        for (int k = threadIdx.x; k < kHubSlots; k += blockDim.x) {
            uint32_t key = s_keys[k];
            if (key != kHubEmpty && s_pos[k]) s_pos[k] = atomicAdd(&cursor[rank[key]], s_pos[k]);
        }
        __syncthreads();
    }
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        uint2 ed = e[i];
        if (ed.x == ed.y) continue;
        int32_t a = rank[ed.x], c = rank[ed.y];
        int hu = hub_find(s_keys, ed.x), hv = hub_find(s_keys, ed.y);
        int32_t pa = hu >= 0 ? atomicAdd(&s_pos[hu], 1) : atomicAdd(&cursor[a], 1);
        adj[pa] = (uint32_t)c;
        row_of[pa] = (uint32_t)a;
        int32_t pc = hv >= 0 ? atomicAdd(&s_pos[hv], 1) : atomicAdd(&cursor[c], 1);
        adj[pc] = (uint32_t)a;
        row_of[pc] = (uint32_t)c;
    }
}
void launch_fill_csr(const uint2* e, int64_t m, const int32_t* rank, int32_t* cursor, uint32_t* adj,
                     uint32_t* row_of, const uint32_t* hub_keys, cudaStream_t s) {
    k_fill_csr<<<edge_grid(m), kEdgeThreads, 0, s>>>(e, m, rank, cursor, adj, row_of, hub_keys);
}

// Chunk-0 CSR by sorting (no random scatter): both directions of every edge
// as (key = row id, value = column id) pairs, one radix sort over the id bits,
// run-length encoding of the sorted keys -> ascending chunk nodes (= ranks)
// and row lengths, then a gather of ranks.  Self-loops become (x, x) entries
// that every consumer skips (w == row); their count per row is subtracted
// where the reference's degree is used (seed.py:69-75 restart order).
__global__ void k_seed_pairs(const uint2* __restrict__ e, int64_t m, uint2* __restrict__ keys,
                             uint2* __restrict__ vals) {
    GRID_STRIDE(i, m) {
        uint2 ed = e[i];
        keys[i] = ed;
        vals[i] = make_uint2(ed.y, ed.x);
    }
}
// Succinct rank of the chunk-0 node set (ascending ids, the RLE runs): per
// 32-id word {presence bits, members before the word}; rank(g) is one 8-byte
// gather into n/4 bytes (L2-resident) plus a popcount, instead of a 4-byte
// gather from an n x 4 B table in HBM (k_seed_map's column ranks were one
// DRAM sector per CSR entry: 25.7 GB for a papers100M level-0 seed, ncu r02c).
// Thread i owns the words from just after node i-1's word through node i's
// word; the words before the first / after the last member are filled by a
// grid-stride pass of their own (they can be long).
__global__ void k_rank_words(const uint32_t* __restrict__ nodes, int64_t nc, int64_t nwords, uint2* __restrict__ rw) {
    const int64_t wfirst = nodes[0] >> 5, wlast = nodes[nc - 1] >> 5;
    GRID_STRIDE(q, nwords) {
        if (q < wfirst) rw[q] = make_uint2(0u, 0u);
        else if (q > wlast) rw[q] = make_uint2(0u, (uint32_t)nc);
    }
    GRID_STRIDE(i, nc) {
        uint32_t g = nodes[i];
        int64_t w = g >> 5;
        if (i > 0)
            for (int64_t q = (int64_t)(nodes[i - 1] >> 5) + 1; q < w; ++q) rw[q] = make_uint2(0u, (uint32_t)i);
        if (i == 0 || (int64_t)(nodes[i - 1] >> 5) != w) {   // first member of its word: build the mask
            uint32_t bits = 0u;
            for (int64_t k = i; k < nc && (int64_t)(nodes[k] >> 5) == w; ++k) bits |= 1u << (nodes[k] & 31);
            rw[w] = make_uint2(bits, (uint32_t)i);
        }
    }
}
void launch_rank_words(const uint32_t* nodes, int64_t nc, int64_t nwords, uint2* rw, cudaStream_t s) {
    if (nc > 0) k_rank_words<<<grid_for(nc, 256), 256, 0, s>>>(nodes, nc, nwords, rw);
}

__global__ void k_seed_map(const uint32_t* __restrict__ skeys, const uint32_t* __restrict__ svals, int64_t entries,
                           const uint2* __restrict__ rw, uint32_t* row_of, uint32_t* adj,
                           int32_t* __restrict__ selfc) {
    GRID_STRIDE(j, entries) {
        uint32_t r = word_rank(rw, skeys[j]), w = word_rank(rw, svals[j]);
        row_of[j] = r;
        adj[j] = w;
        if (r == w) atomicAdd(&selfc[r], 1);
    }
}
size_t seed_csr_temp_bytes(int64_t entries) {
    size_t a = 0, b = 0;
    cub::DoubleBuffer<uint32_t> dk(nullptr, nullptr), dv(nullptr, nullptr);
    cub::DeviceRadixSort::SortPairs(nullptr, a, dk, dv, entries);
    cub::DeviceRunLengthEncode::Encode(nullptr, b, (uint32_t*)nullptr, (uint32_t*)nullptr, (int32_t*)nullptr,
                                       (long long*)nullptr, entries);
    return a > b ? a : b;
}
// keysA/valsA, keysB/valsB: two entries-sized buffer pairs (A = row_of/adj of
// the SeedBufs); the sorted CSR ends in row_of/adj (a swap is reported).
// nodes <- ascending chunk node ids, counts <- row lengths, nruns -> *d_nruns.
void launch_seed_sort(const uint2* e, int64_t m, uint32_t* keysA, uint32_t* valsA, uint32_t* keysB, uint32_t* valsB,
                      int end_bit, uint32_t* nodes, int32_t* counts, long long* d_nruns, void* temp,
                      size_t temp_bytes, bool* sorted_in_b, cudaStream_t s) {
    int64_t entries = 2 * m;
    k_seed_pairs<<<grid_for(m, 256, 16), 256, 0, s>>>(e, m, reinterpret_cast<uint2*>(keysA),
                                                      reinterpret_cast<uint2*>(valsA));
    cub::DoubleBuffer<uint32_t> dk(keysA, keysB), dv(valsA, valsB);
    cub::DeviceRadixSort::SortPairs(temp, temp_bytes, dk, dv, entries, 0, end_bit, s);
    *sorted_in_b = dk.Current() == keysB;
    cub::DeviceRunLengthEncode::Encode(temp, temp_bytes, dk.Current(), nodes, counts, d_nruns, entries, s);
}
void launch_seed_map(const uint32_t* skeys, const uint32_t* svals, int64_t entries, const uint2* rw,
                     uint32_t* row_of, uint32_t* adj, int32_t* selfc, cudaStream_t s) {
    k_seed_map<<<grid_for(entries, 256, 16), 256, 0, s>>>(skeys, svals, entries, rw, row_of, adj, selfc);
}

// union-find connected components (link larger root under smaller root)
__device__ __forceinline__ uint32_t uf_find(uint32_t* parent, uint32_t x) {
    uint32_t p = ((volatile uint32_t*)parent)[x];
    while (p != x) {
        uint32_t gp = ((volatile uint32_t*)parent)[p];
        if (gp != p) ((volatile uint32_t*)parent)[x] = gp;   // path halving
        x = p;
        p = gp;
    }
    return x;
}

__global__ void k_iota_u32(uint32_t* a, int64_t n) {
    GRID_STRIDE(i, n) a[i] = (uint32_t)i;
}

__global__ void k_cc_link(const uint2* __restrict__ e, int64_t m, const int32_t* __restrict__ rank, uint32_t* parent) {
    GRID_STRIDE(i, m) {
        uint2 ed = e[i];
        if (ed.x == ed.y) continue;
        uint32_t a = (uint32_t)rank[ed.x], b = (uint32_t)rank[ed.y];
        while (true) {
            uint32_t ra = uf_find(parent, a), rb = uf_find(parent, b);
            if (ra == rb) break;
            if (ra > rb) { uint32_t t = ra; ra = rb; rb = t; }
            if (atomicCAS(&parent[rb], rb, ra) == rb) break;
            a = ra;
            b = rb;
        }
    }
}

// After linking the forest is frozen: a read-only walk to the root, written to
// a separate array (writing parent[] in place would race with other threads'
// walks through the same node and can leave a non-root parent behind).
__global__ void k_cc_roots(const uint32_t* __restrict__ parent, int64_t nc, uint32_t* __restrict__ root) {
    GRID_STRIDE(i, nc) {
        uint32_t r = (uint32_t)i, p = parent[r];
        while (p != r) {
            r = p;
            p = parent[r];
        }
        root[i] = r;
    }
}

void launch_cc(const uint2* e, int64_t m, const int32_t* rank, uint32_t* parent, uint32_t* scratch, int64_t nc,
               cudaStream_t s) {
    k_iota_u32<<<grid_for(nc, 256), 256, 0, s>>>(parent, nc);
    k_cc_link<<<grid_for(m, 256, 16), 256, 0, s>>>(e, m, rank, parent);
    k_cc_roots<<<grid_for(nc, 256), 256, 0, s>>>(parent, nc, scratch);
    cudaMemcpyAsync(parent, scratch, sizeof(uint32_t) * nc, cudaMemcpyDeviceToDevice, s);
}

// Components over the chunk-0 CSR with sampled linking (the Afforest scheme):
// link every row to its first two neighbours, flatten, find the most common
// root (the giant component) from a sample, then link the remaining
// neighbours of rows outside it only.  An edge skipped at a giant row is
// linked from its other endpoint's row unless that row was in the giant
// component too, so the final components equal the full union-find's.
__device__ __forceinline__ void uf_link(uint32_t* parent, uint32_t a, uint32_t b) {
    while (true) {
        uint32_t ra = uf_find(parent, a), rb = uf_find(parent, b);
        if (ra == rb) return;
        if (ra > rb) { uint32_t t = ra; ra = rb; rb = t; }
        if (atomicCAS(&parent[rb], rb, ra) == rb) return;
        a = ra;
        b = rb;
    }
}
__global__ void k_cc_link_rows(const int32_t* __restrict__ start, const uint32_t* __restrict__ adj, int64_t nc,
                               uint32_t* parent, int first, int count, const unsigned long long* giant) {
    uint32_t g = giant ? (uint32_t)*giant : 0xFFFFFFFFu;
    GRID_STRIDE(i, nc) {
        int64_t b = start[i] + first, e = start[i + 1];
        if (count > 0 && b + count < e) e = b + count;
        if (b >= e) continue;
        if (giant && uf_find(parent, (uint32_t)i) == g) continue;
        for (int64_t j = b; j < e; ++j) {
            uint32_t w = adj[j];
            if (w != (uint32_t)i) uf_link(parent, (uint32_t)i, w);
        }
    }
}
// the most frequent root among 1024 sampled nodes (flattened forest)
__global__ void k_cc_giant(const uint32_t* __restrict__ parent, int64_t nc, unsigned long long* giant) {
    __shared__ uint32_t smp[1024];
    __shared__ unsigned long long best;
    uint32_t t = threadIdx.x;
    uint64_t h = (uint64_t)(t + 1) * 0x9E3779B97F4A7C15ULL;
    h ^= h >> 29;
    smp[t] = parent[h % (uint64_t)nc];
    if (t == 0) best = 0;
    __syncthreads();
    uint32_t c = 0;
    for (int j = 0; j < 1024; ++j) c += smp[j] == smp[t];
    atomicMax(&best, ((unsigned long long)c << 32) | (0xFFFFFFFFu - smp[t]));   // ties: smaller root
    __syncthreads();
    if (t == 0) *giant = 0xFFFFFFFFu - (uint32_t)(best & 0xFFFFFFFFULL);
}
void launch_cc_csr(const int32_t* start, const uint32_t* adj, int64_t nc, uint32_t* parent, uint32_t* scratch,
                   unsigned long long* d_giant, cudaStream_t s) {
    k_iota_u32<<<grid_for(nc, 256), 256, 0, s>>>(parent, nc);
    k_cc_link_rows<<<grid_for(nc, 256, 16), 256, 0, s>>>(start, adj, nc, parent, 0, 2, nullptr);
    k_cc_roots<<<grid_for(nc, 256), 256, 0, s>>>(parent, nc, scratch);
    cudaMemcpyAsync(parent, scratch, sizeof(uint32_t) * nc, cudaMemcpyDeviceToDevice, s);
    k_cc_giant<<<1, 1024, 0, s>>>(parent, nc, d_giant);
    k_cc_link_rows<<<grid_for(nc, 256, 16), 256, 0, s>>>(start, adj, nc, parent, 2, 0, d_giant);
    k_cc_roots<<<grid_for(nc, 256), 256, 0, s>>>(parent, nc, scratch);
    cudaMemcpyAsync(parent, scratch, sizeof(uint32_t) * nc, cudaMemcpyDeviceToDevice, s);
}

// restart order of _bfs_grow (seed.py:69-75): a component is entered at its
// highest-degree, lowest-index node; key = (~degree << 32) | index, min wins.
__global__ void k_comp_keys(const int32_t* __restrict__ start, const int32_t* __restrict__ selfc,
                            const uint32_t* __restrict__ parent, int64_t nc, unsigned long long* ckey,
                            uint32_t* csize, const unsigned long long* giant) {
    // the giant component's key and size are accumulated per block in shared
    // memory (one atomic per block instead of one per warp on two L2 words:
    // 1.9M same-address atomics per papers100M level-0 seed)
    __shared__ unsigned int s_gcnt;
    __shared__ unsigned long long s_gkey;
    const uint32_t g = giant ? (uint32_t)*giant : 0xFFFFFFFFu;
    if (threadIdx.x == 0) {
        s_gcnt = 0u;
        s_gkey = ~0ULL;
    }
    __syncthreads();
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); base < nc; base += stride) {
        int64_t i = base + (threadIdx.x & 31);
        bool valid = i < nc;
        uint32_t r = valid ? parent[i] : 0xFFFFFFFFu;
        unsigned long long key = ~0ULL;
        if (valid) {
            uint32_t d = (uint32_t)(start[i + 1] - start[i] - selfc[i]);
            key = ((unsigned long long)(0xFFFFFFFFu - d) << 32) | (unsigned long long)i;
        }
        // one update per (warp, component): min of the degree part, then of
        // the index among the lanes holding it
        unsigned peers = __match_any_sync(0xffffffffu, r);
        int leader = __ffs(peers) - 1;
        uint32_t khi = __reduce_min_sync(peers, (uint32_t)(key >> 32));
        uint32_t klo = __reduce_min_sync(peers, (uint32_t)(key >> 32) == khi ? (uint32_t)key : 0xFFFFFFFFu);
        if (valid && (int)(threadIdx.x & 31) == leader) {
            unsigned long long kk = ((unsigned long long)khi << 32) | klo;
            if (r == g) {
                atomicAdd(&s_gcnt, (unsigned int)__popc(peers));
                if (kk < s_gkey) atomicMin(&s_gkey, kk);
            } else {
                atomicMin(&ckey[r], kk);
                atomicAdd(&csize[r], (uint32_t)__popc(peers));
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0 && s_gcnt) {
        atomicAdd(&csize[g], s_gcnt);
        atomicMin(&ckey[g], s_gkey);
    }
}
void launch_comp_keys(const SeedBufs& sb, int64_t nc, cudaStream_t s, const unsigned long long* giant) {
    cudaMemsetAsync(sb.ckey, 0xFF, sizeof(unsigned long long) * nc, s);
    cudaMemsetAsync(sb.csize, 0, sizeof(uint32_t) * nc, s);
    k_comp_keys<<<grid_for(nc, 256), 256, 0, s>>>(sb.start, sb.cursor, sb.parent, nc, sb.ckey, sb.csize, giant);
}

struct RootPred {
    const uint32_t* parent;
    __device__ __forceinline__ bool operator()(const uint32_t& i) const { return parent[i] == i; }
};
void launch_select_roots(const SeedBufs& sb, int64_t nc, void* temp, size_t temp_bytes, cudaStream_t s) {
    thrust::counting_iterator<uint32_t> it(0);
    cub::DeviceSelect::If(temp, temp_bytes, it, sb.roots, sb.scal + 0, (int)nc, RootPred{sb.parent}, s);
}

__global__ void k_root_keys(const uint32_t* roots, int64_t nr, const unsigned long long* ckey,
                            unsigned long long* rkeys, uint32_t* rvals) {
    GRID_STRIDE(j, nr) {
        rkeys[j] = ckey[roots[j]];
        rvals[j] = roots[j];
    }
}
void launch_root_keys(const SeedBufs& sb, int64_t nr, cudaStream_t s) {
    k_root_keys<<<grid_for(nr, 256), 256, 0, s>>>(sb.roots, nr, sb.ckey, sb.rkeys, sb.rvals);
}

// cumulative component sizes in restart order -> boundary component
__global__ void k_csize_sorted(const uint32_t* rvals2, int64_t nr, const uint32_t* csize, int64_t* out) {
    GRID_STRIDE(j, nr) out[j] = csize[rvals2[j]];
}
__global__ void k_find_boundary(const int64_t* cum_excl, const uint32_t* rvals2, const uint32_t* csize,
                                const unsigned long long* rkeys2, int64_t nr, long long target, uint32_t* cpos,
                                long long* scal) {
    GRID_STRIDE(j, nr) {
        long long before = cum_excl[j];
        long long after = before + csize[rvals2[j]];
        cpos[rvals2[j]] = (uint32_t)j;
        if (before < target && after >= target) {
            scal[1] = j;                                  // boundary component position
            scal[2] = target - before;                    // BFS quota inside it
            scal[3] = (long long)(rkeys2[j] & 0xFFFFFFFFULL);   // its start node
        }
    }
}
void launch_boundary(const SeedBufs& sb, int64_t nr, long long target, void* temp, size_t temp_bytes,
                     cudaStream_t s) {
    k_csize_sorted<<<grid_for(nr, 256), 256, 0, s>>>(sb.rvals2, nr, sb.csize, sb.fdeg);
    cub::DeviceScan::ExclusiveSum(temp, temp_bytes, sb.fdeg, sb.cum, (int)nr, s);
    k_find_boundary<<<grid_for(nr, 256), 256, 0, s>>>(sb.cum, sb.rvals2, sb.csize, sb.rkeys2, nr, target, sb.cpos,
                                                       sb.scal);
}

__global__ void k_seed_labels(const uint32_t* parent, const uint32_t* cpos, int64_t nc, const long long* scal,
                              int8_t* slab, uint32_t* disc) {
    long long jb = scal[1];
    long long s0 = scal[3];
    GRID_STRIDE(i, nc) {
        long long p = cpos[parent[i]];
        slab[i] = (int8_t)(p < jb ? 0 : (p > jb ? 1 : 2));
        disc[i] = 0xFFFFFFFFu;
        if (i == s0) slab[i] = 0;   // BFS start is picked first (seed.py:70-74)
    }
}
void launch_seed_labels(const SeedBufs& sb, int64_t nc, cudaStream_t s) {
    k_seed_labels<<<grid_for(nc, 256), 256, 0, s>>>(sb.parent, sb.cpos, nc, sb.scal, sb.slab, sb.disc);
}

__global__ void k_frontier_deg(const uint32_t* frontier, int64_t fsize, const int32_t* start, int64_t* fdeg) {
    GRID_STRIDE(j, fsize) {
        uint32_t v = frontier[j];
        fdeg[j] = start[v + 1] - start[v];
    }
}
void launch_frontier_degrees(const SeedBufs& sb, int64_t fsize, cudaStream_t s) {
    k_frontier_deg<<<grid_for(fsize, 256), 256, 0, s>>>(sb.frontier, fsize, sb.start, sb.fdeg);
}

// level expansion: every (frontier node, neighbour) pair, balanced over
// entries; a candidate keeps its minimum discoverer rank (FIFO order of
// _bfs_grow: queue order, then ascending neighbour id).
__global__ void __launch_bounds__(256) k_bfs_expand(const uint32_t* __restrict__ frontier, int64_t fsize,
                                                    long long rbase, const int64_t* __restrict__ fpre, int64_t total,
                                                    const int32_t* __restrict__ start,
                                                    const uint32_t* __restrict__ adj, const int8_t* __restrict__ slab,
                                                    uint32_t* __restrict__ disc,
                                                    unsigned long long* __restrict__ cand, long long* ncand) {
    // each lane expands 4 consecutive frontier-adjacency slots (one binary
    // search for the first); first discoveries are appended warp-aggregated
    constexpr int Q = 4;
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t wb = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * (32 * Q); wb < total;
         wb += nwarps * 32 * Q) {
        int64_t k0 = wb + (int64_t)lane * Q;
        int64_t lo = 0;
        if (k0 < total) {   // j = last index with fpre[j] <= k0
            int64_t hi = fsize - 1;
            while (lo < hi) {
                int64_t mid = (lo + hi + 1) >> 1;
                if (fpre[mid] <= k0) lo = mid; else hi = mid - 1;
            }
        }
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            int64_t k = k0 + q;
            bool fresh = false;
            uint32_t w = 0;
            if (k < total) {
                while (lo + 1 < fsize && fpre[lo + 1] <= k) ++lo;
                uint32_t v = frontier[lo];
                w = adj[start[v] + (k - fpre[lo])];
                if (slab[w] == 2) {
                    uint32_t r = (uint32_t)(rbase + lo);
                    if (r < ((volatile uint32_t*)disc)[w]) fresh = atomicMin(&disc[w], r) == 0xFFFFFFFFu;
                }
            }
            unsigned bal = __ballot_sync(0xffffffffu, fresh);
            if (bal) {
                unsigned long long base = 0;
                if (lane == __ffs(bal) - 1) base = atomicAdd((unsigned long long*)ncand, (unsigned long long)__popc(bal));
                base = __shfl_sync(0xffffffffu, base, __ffs(bal) - 1);
                if (fresh) cand[base + __popc(bal & ((1u << lane) - 1))] = w;
            }
        }
    }
}
void launch_bfs_expand(const SeedBufs& sb, int64_t fsize, long long rbase, int64_t total, cudaStream_t s) {
    k_bfs_expand<<<grid_for(total / 4 + 1, 256, 16), 256, 0, s>>>(sb.frontier, fsize, rbase, sb.cum, total, sb.start, sb.adj,
                                                         sb.slab, sb.disc, sb.cand_keys, sb.scal + 4);
}

__global__ void k_cand_keys(unsigned long long* cand, int64_t nc, const uint32_t* disc) {
    GRID_STRIDE(c, nc) {
        uint32_t w = (uint32_t)cand[c];
        cand[c] = ((unsigned long long)disc[w] << 32) | w;
    }
}
void launch_cand_keys(const SeedBufs& sb, int64_t ncand, cudaStream_t s) {
    k_cand_keys<<<grid_for(ncand, 256), 256, 0, s>>>(sb.cand_keys, ncand, sb.disc);
}
__global__ void k_bfs_take(const unsigned long long* sorted, int64_t take, int8_t* slab, uint32_t* frontier) {
    GRID_STRIDE(c, take) {
        uint32_t w = (uint32_t)(sorted[c] & 0xFFFFFFFFULL);
        slab[w] = 0;
        frontier[c] = w;
    }
}
void launch_bfs_take(const SeedBufs& sb, int64_t ncand, int64_t take, cudaStream_t s) {
    k_bfs_take<<<grid_for(take, 256), 256, 0, s>>>(sb.cand_keys2, take, sb.slab, sb.frontier);
}

__global__ void k_seed_finalize(int8_t* slab, int64_t nc) {
    GRID_STRIDE(i, nc) if (slab[i] == 2) slab[i] = 1;
}
void launch_seed_finalize(const SeedBufs& sb, int64_t nc, cudaStream_t s) {
    k_seed_finalize<<<grid_for(nc, 256), 256, 0, s>>>(sb.slab, nc);
}

// per-row packed counts over the chunk-0 CSR (entries of a row are
// contiguous): warp-segmented reduction, one atomic per row segment.
//   mode 0 (refinement pass, seed.py:96-116): (same | other<<32) where a
//          neighbour's label is `cur` if its index is lower, else `pre`;
//   mode 1 (estimates, grem.py:166-174): (#label0 | #label1<<32) over `cur`.
__global__ void k_row_counts(const uint32_t* __restrict__ adj, const uint32_t* __restrict__ row_of, int64_t entries,
                             const int8_t* __restrict__ cur, const int8_t* __restrict__ pre, int mode,
                             unsigned long long* __restrict__ pair) {
    int lane = threadIdx.x & 31;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); base < entries; base += stride) {
        int64_t k = base + lane;
        bool valid = k < entries;
        uint32_t row = valid ? row_of[k] : 0xFFFFFFFFu;
        unsigned long long v = 0;
        if (valid) {
            uint32_t w = adj[k];
            if (w == row) {
                v = 0;
            } else if (mode == 0) {
                int lw = w < row ? cur[w] : pre[w];
                v = (lw == pre[row]) ? 1ULL : (1ULL << 32);
            } else {
                int lw = cur[w];
                v = lw == 0 ? 1ULL : (lw == 1 ? (1ULL << 32) : 0ULL);
            }
        }
        // segmented inclusive scan over equal rows (rows are non-decreasing in k)
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            unsigned long long ov = __shfl_up_sync(0xffffffffu, v, off);
            uint32_t orow = __shfl_up_sync(0xffffffffu, row, off);
            if (lane >= off && orow == row) v += ov;
        }
        uint32_t nrow = __shfl_down_sync(0xffffffffu, row, 1);
        bool tail = (lane == 31) || (nrow != row);
        if (valid && tail && v) atomicAdd(&pair[row], v);
    }
}
void launch_row_counts(const SeedBufs& sb, const int8_t* cur, const int8_t* pre, int mode, int64_t entries,
                       int64_t nc, cudaStream_t s) {
    cudaMemsetAsync(sb.pair, 0, sizeof(unsigned long long) * nc, s);
    if (entries > 0)
        k_row_counts<<<grid_for(entries, 256, 16), 256, 0, s>>>(sb.adj, sb.row_of, entries, cur, pre, mode, sb.pair);
}

__global__ void k_want(const unsigned long long* pair, int64_t nc, uint8_t* want) {
    GRID_STRIDE(i, nc) {
        unsigned long long p = pair[i];
        uint32_t same = (uint32_t)(p & 0xFFFFFFFFULL), other = (uint32_t)(p >> 32);
        want[i] = (other > 0 && other > same) ? 1 : 0;
    }
}

// one refinement round's sizes chain: x before every node, starting from the
// pass-start x in scal[6]
void launch_refine_scan(const SeedBufs& sb, const ChunkBufs& b, int64_t nc, long long cap, cudaStream_t s) {
    k_want<<<grid_for(nc, 256), 256, 0, s>>>(sb.pair, nc, sb.want);
    RefineMapSrc src{sb.want, sb.slab, (long long)nc, cap};
    int64_t ntiles = (nc + kScanTile - 1) / kScanTile;
    k_scan_reduce<RefineMapSrc><<<(unsigned)ntiles, kScanThreads, 0, s>>>(src, nc, b.tile_agg);
    k_scan_top<<<1, 1024, 0, s>>>(b.tile_agg, ntiles, sb.scal + 6, b.tile_x);
    k_scan_down_plain<RefineMapSrc><<<(unsigned)ntiles, kScanThreads, 0, s>>>(src, nc, b.tile_x, b.x);
}

// ------------------------------------------- refinement rounds on bitmaps
// Seed labels are 0/1: the pre-pass labels P and the tentative labels T of a
// refinement pass are bitmaps (N_c bits, L2-resident), a thread owns one
// 32-node word, and one round = per-row same/other counts + a fused
// want/clamp-reduce + top scan + fused x/decision pass.
constexpr int kRfT = 256;
constexpr int kRfTile = kRfT * 32;

__device__ __forceinline__ uint32_t bit_of(const uint32_t* __restrict__ bits, uint32_t i) {
    return (bits[i >> 5] >> (i & 31)) & 1u;
}

__global__ void k_row_counts_bits(const uint32_t* __restrict__ adj, const uint32_t* __restrict__ row_of,
                                  int64_t entries, const uint32_t* __restrict__ Pb, const uint32_t* __restrict__ Tb,
                                  int mode, unsigned long long* __restrict__ pair) {
    int lane = threadIdx.x & 31;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); base < entries; base += stride) {
        int64_t k = base + lane;
        bool valid = k < entries;
        uint32_t row = valid ? row_of[k] : 0xFFFFFFFFu;
        unsigned long long v = 0;
        if (valid) {
            uint32_t w = adj[k];
            if (w == row) {
                v = 0;         // self-loop entry: not an adjacency (model.py: loops are skipped)
            } else if (mode == 0) {   // seed.py:99-104: lower index -> this pass's label, else pre-pass
                uint32_t lw = w < row ? bit_of(Tb, w) : bit_of(Pb, w);
                v = (lw == bit_of(Pb, row)) ? 1ULL : (1ULL << 32);
            } else {           // grem.py:166-174 estimates against the final labels
                v = bit_of(Pb, w) == 0 ? 1ULL : (1ULL << 32);
            }
        }
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            unsigned long long ov = __shfl_up_sync(0xffffffffu, v, off);
            uint32_t orow = __shfl_up_sync(0xffffffffu, row, off);
            if (lane >= off && orow == row) v += ov;
        }
        uint32_t nrow = __shfl_down_sync(0xffffffffu, row, 1);
        bool tail = (lane == 31) || (nrow != row);
        if (valid && tail && v) atomicAdd(&pair[row], v);
    }
}

__device__ __forceinline__ Clamp refine_map(uint32_t want, uint32_t p, long long s, long long cap) {
    if (!want) return clamp_identity();
    return p == 0 ? Clamp{-1, s - cap, kInf} : Clamp{1, -kInf, cap};
}

__global__ void __launch_bounds__(kRfT) k_refine_reduce(const unsigned long long* __restrict__ pair,
                                                        const uint32_t* __restrict__ Pb, uint32_t* __restrict__ wantb,
                                                        int64_t nc, long long cap, Clamp* tile_agg) {
    __shared__ Clamp smem[kRfT / 32];
    __shared__ Clamp stotal;
    int64_t w = (int64_t)blockIdx.x * kRfT + threadIdx.x;
    int64_t base = w * 32;
    uint32_t P = 0, wb = 0;
    if (base < nc) {
        P = Pb[w];
#pragma unroll 8
        for (int j = 0; j < 32; ++j) {
            int64_t i = base + j;
            if (i >= nc) break;
            unsigned long long pp = pair[i];
            uint32_t same = (uint32_t)(pp & 0xFFFFFFFFULL), other = (uint32_t)(pp >> 32);
            if (other > same) wb |= 1u << j;   // move iff it strictly reduces the local cut (seed.py:110-111)
        }
        wantb[w] = wb;
    }
    Clamp acc = clamp_identity();
    for (int j = 0; j < 32; ++j) acc = clamp_then(acc, refine_map((wb >> j) & 1u, (P >> j) & 1u, nc, cap));
    block_excl_scan<kRfT>(acc, smem, &stotal);
    __syncthreads();
    if (threadIdx.x == 0) tile_agg[blockIdx.x] = stotal;
}

__global__ void __launch_bounds__(kRfT) k_refine_down(const uint32_t* __restrict__ Pb, uint32_t* __restrict__ Tb,
                                                      const uint32_t* __restrict__ wantb, int64_t nc, long long cap,
                                                      const long long* tile_x, long long* changed, long long* xend,
                                                      uint32_t* __restrict__ Db) {
    __shared__ Clamp smem[kRfT / 32];
    int64_t w = (int64_t)blockIdx.x * kRfT + threadIdx.x;
    int64_t nwords = (nc + 31) / 32;
    uint32_t P = 0, wb = 0;
    if (w < nwords) {
        P = Pb[w];
        wb = wantb[w];
    }
    Clamp acc = clamp_identity();
    for (int j = 0; j < 32; ++j) acc = clamp_then(acc, refine_map((wb >> j) & 1u, (P >> j) & 1u, nc, cap));
    Clamp pre = block_excl_scan<kRfT>(acc, smem, nullptr);
    long long x = clamp_apply(pre, tile_x[blockIdx.x]);
    uint32_t Tn = P;
    for (int j = 0; j < 32; ++j) {
        uint32_t want = (wb >> j) & 1u, p = (P >> j) & 1u;
        if (want) {   // receiving side must have room (seed.py:110)
            bool room = p == 0 ? (x > nc - cap) : (x < cap);
            if (room) Tn ^= 1u << j;
        }
        x = clamp_apply(refine_map(want, p, nc, cap), x);
    }
    int ch = 0;
    if (w < nwords) {
        uint32_t d = Tn ^ Tb[w];
        ch = __popc(d);
        Db[w] = d;
        Tb[w] = Tn;
        if (w == nwords - 1) *xend = x;
    }
    for (int off = 16; off; off >>= 1) ch += __shfl_down_sync(0xffffffffu, ch, off);
    if ((threadIdx.x & 31) == 0 && ch) atomicAdd((unsigned long long*)changed, (unsigned long long)ch);
}

// Incremental row counts between refinement rounds of one pass: only rows
// above a node whose tentative label flipped read it (seed.py:99-104), so
// the flipped nodes' adjacency rows move one count between same and other.
__global__ void k_refine_list(const uint32_t* __restrict__ Db, int64_t nwords, const int32_t* __restrict__ start,
                              uint32_t* __restrict__ list, int64_t* __restrict__ deg, long long* count) {
    GRID_STRIDE(w, nwords) {
        uint32_t d = Db[w];
        while (d) {
            int j = __ffs(d) - 1;
            d &= d - 1;
            uint32_t i = (uint32_t)(w * 32 + j);
            long long idx = (long long)atomicAdd((unsigned long long*)count, 1ULL);
            list[idx] = i;
            deg[idx] = start[i + 1] - start[i];
        }
    }
}
__global__ void k_refine_delta(const uint32_t* __restrict__ list, int64_t cnt, const int64_t* __restrict__ cum,
                               const int32_t* __restrict__ start, const uint32_t* __restrict__ adj,
                               const uint32_t* __restrict__ Pb, const uint32_t* __restrict__ Tb,
                               unsigned long long* __restrict__ pair) {
    int64_t total = cum[cnt];
    GRID_STRIDE(k, total) {
        int64_t lo = 0, hi = cnt - 1;
        while (lo < hi) {
            int64_t mid = (lo + hi + 1) >> 1;
            if (cum[mid] <= k) lo = mid; else hi = mid - 1;
        }
        uint32_t w = list[lo];
        uint32_t row = adj[start[w] + (k - cum[lo])];
        if (row <= w) continue;   // lower rows read the pre-pass label; self-loop entries are skipped
        bool same_now = bit_of(Tb, w) == bit_of(Pb, row);
        atomicAdd(&pair[row], same_now ? 0xFFFFFFFF00000001ULL : 0x00000000FFFFFFFFULL);
    }
}
void launch_refine_delta(const SeedBufs& sb, const uint32_t* Db, int64_t nc, int64_t changed, const uint32_t* Pb,
                         const uint32_t* Tb, void* temp, size_t temp_bytes, cudaStream_t s) {
    int64_t nwords = (nc + 31) / 32;
    cudaMemsetAsync(sb.scal + 12, 0, sizeof(long long), s);
    cudaMemsetAsync(sb.fdeg + changed, 0, sizeof(int64_t), s);
    k_refine_list<<<grid_for(nwords, 256), 256, 0, s>>>(Db, nwords, sb.start, sb.frontier, sb.fdeg, sb.scal + 12);
    cub::DeviceScan::ExclusiveSum(temp, temp_bytes, sb.fdeg, sb.cum, (int)(changed + 1), s);
    k_refine_delta<<<num_sms() * 8, 256, 0, s>>>(sb.frontier, changed, sb.cum, sb.start, sb.adj, Pb, Tb, sb.pair);
}

__global__ void k_pack_bits(const int8_t* __restrict__ lab, int64_t nc, uint32_t* __restrict__ bits, int64_t nwords) {
    GRID_STRIDE(w, nwords) {
        uint32_t b = 0;
        for (int j = 0; j < 32; ++j) {
            int64_t i = w * 32 + j;
            if (i < nc && lab[i] == 1) b |= 1u << j;
        }
        bits[w] = b;
    }
}
__global__ void k_unpack_bits(const uint32_t* __restrict__ bits, int64_t nc, int8_t* __restrict__ lab) {
    GRID_STRIDE(i, nc) lab[i] = (int8_t)((bits[i >> 5] >> (i & 31)) & 1u);
}
__global__ void k_xor_popc(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b, int64_t nwords,
                           long long* out) {
    int d = 0;
    GRID_STRIDE(w, nwords) d += __popc(a[w] ^ b[w]);
    for (int off = 16; off; off >>= 1) d += __shfl_down_sync(0xffffffffu, d, off);
    if ((threadIdx.x & 31) == 0 && d) atomicAdd((unsigned long long*)out, (unsigned long long)d);
}

void launch_pack_bits(const int8_t* lab, int64_t nc, uint32_t* bits, cudaStream_t s) {
    int64_t nw = (nc + 31) / 32;
    k_pack_bits<<<grid_for(nw, 256), 256, 0, s>>>(lab, nc, bits, nw);
}
void launch_unpack_bits(const uint32_t* bits, int64_t nc, int8_t* lab, cudaStream_t s) {
    k_unpack_bits<<<grid_for(nc, 256), 256, 0, s>>>(bits, nc, lab);
}
void launch_xor_popc(const uint32_t* a, const uint32_t* b, int64_t nc, long long* out, cudaStream_t s) {
    int64_t nw = (nc + 31) / 32;
    k_xor_popc<<<grid_for(nw, 256), 256, 0, s>>>(a, b, nw, out);
}
void launch_row_counts_bits(const SeedBufs& sb, const uint32_t* Pb, const uint32_t* Tb, int mode, int64_t entries,
                            int64_t nc, cudaStream_t s) {
    cudaMemsetAsync(sb.pair, 0, sizeof(unsigned long long) * nc, s);
    if (entries > 0)
        k_row_counts_bits<<<grid_for(entries, 256, 16), 256, 0, s>>>(sb.adj, sb.row_of, entries, Pb, Tb, mode,
                                                                    sb.pair);
}
// one refinement round after the row counts: want bits + exact sizes chain +
// decisions; x at pass start in sb.scal[6], changed -> sb.scal[5], x at the
// end of the pass -> sb.scal[9]
void launch_refine_round(const SeedBufs& sb, const ChunkBufs& b, const uint32_t* Pb, uint32_t* Tb, uint32_t* wantb,
                         uint32_t* Db, int64_t nc, long long cap, cudaStream_t s) {
    int64_t nwords = (nc + 31) / 32;
    int64_t ntiles = (nwords + kRfT - 1) / kRfT;
    k_refine_reduce<<<(unsigned)ntiles, kRfT, 0, s>>>(sb.pair, Pb, wantb, nc, cap, b.tile_agg);
    k_scan_top<<<1, 1024, 0, s>>>(b.tile_agg, ntiles, sb.scal + 6, b.tile_x);
    k_refine_down<<<(unsigned)ntiles, kRfT, 0, s>>>(Pb, Tb, wantb, nc, cap, b.tile_x, sb.scal + 5, sb.scal + 9, Db);
}

// x at pass start = number of label-0 chunk nodes, passed via scal[6] (host)
__global__ void k_refine_decide(const uint8_t* want, const int8_t* pre, const int32_t* x, int64_t nc, long long cap,
                                int8_t* tent, long long* changed) {
    int ch = 0;
    GRID_STRIDE(i, nc) {
        int p = pre[i];
        int t = p;
        if (want[i]) {
            long long xi = x[i];
            bool room = (p == 0) ? (xi > nc - cap) : (xi < cap);
            if (room) t = 1 - p;
        }
        ch += (t != tent[i]);
        tent[i] = (int8_t)t;
    }
    for (int off = 16; off; off >>= 1) ch += __shfl_down_sync(0xffffffffu, ch, off);
    if ((threadIdx.x & 31) == 0 && ch) atomicAdd((unsigned long long*)changed, (unsigned long long)ch);
}

void launch_refine_decide(const SeedBufs& sb, const ChunkBufs& b, int64_t nc, long long cap, cudaStream_t s) {
    k_refine_decide<<<grid_for(nc, 256), 256, 0, s>>>(sb.want, sb.slab, b.x, nc, cap, sb.slab2, sb.scal + 5);
}

__global__ void k_seed_commit(const uint32_t* nodes, int64_t nc, const int8_t* slab,
                              const unsigned long long* pair, int8_t* lab, double2* nbr, uint8_t* flag,
                              long long* zeros, uint32_t* lab2) {
    int z = 0;
    GRID_STRIDE(i, nc) {
        uint32_t g = nodes[i];
        lab[g] = slab[i];
        atomicXor(&lab2[g >> 4], (uint32_t)(slab[i] + 1) << ((g & 15) * 2));   // from code 0 (unassigned)
        unsigned long long p = pair[i];
        nbr[g] = make_double2((double)(uint32_t)(p & 0xFFFFFFFFULL), (double)(uint32_t)(p >> 32));
        flag[g] = 0;
        z += (slab[i] == 0);
    }
    for (int off = 16; off; off >>= 1) z += __shfl_down_sync(0xffffffffu, z, off);
    if ((threadIdx.x & 31) == 0 && z) atomicAdd((unsigned long long*)zeros, (unsigned long long)z);
}
void launch_seed_commit(const SeedBufs& sb, const ChunkBufs& b, const uint32_t* nodes, int64_t nc, cudaStream_t s) {
    k_seed_commit<<<grid_for(nc, 256), 256, 0, s>>>(nodes, nc, sb.slab, sb.pair, b.lab, b.nbr, b.flag, sb.scal + 7,
                                                     b.lab2);
}

// ------------------------------------------------------------ after stream

// _fill_unassigned (grem.py:177-189): in ascending id every never-seen node
// goes to the smaller side (ties to 0); capacity can never redirect it when
// 2*cap >= n.  Closed form: with d = sizes[1]-sizes[0], the first |d| go to
// the smaller side, then sides alternate starting with 0.
__global__ void k_unassigned_flags(const int8_t* lab, int64_t n, int32_t* f) {
    GRID_STRIDE(i, n) f[i] = lab[i] == -1 ? 1 : 0;
}
__global__ void k_fill_apply(int8_t* lab, int64_t n, const int32_t* rank, const long long* sizes) {
    long long d = sizes[1] - sizes[0];
    long long ad = d < 0 ? -d : d;
    int first = d > 0 ? 0 : 1;
    GRID_STRIDE(i, n) {
        if (lab[i] != -1) continue;
        long long j = rank[i];
        lab[i] = (int8_t)(j < ad ? first : ((j - ad) & 1));
    }
}
void launch_fill_unassigned(int8_t* lab, int64_t n, const long long* sizes, int32_t* rank_scratch, void* temp,
                            size_t temp_bytes, cudaStream_t s) {
    // rank_scratch must hold 2n int32
    int32_t* f = rank_scratch + n;
    k_unassigned_flags<<<grid_for(n, 256), 256, 0, s>>>(lab, n, f);
    cub::DeviceScan::ExclusiveSum(temp, temp_bytes, f, rank_scratch, (int)n, s);
    k_fill_apply<<<grid_for(n, 256), 256, 0, s>>>(lab, n, rank_scratch, sizes);
}

__global__ void k_labels_to_i32(const int8_t* lab, int64_t n, int32_t* out) {
    GRID_STRIDE(i, n) out[i] = lab[i];
}
void launch_labels_to_i32(const int8_t* lab, int64_t n, int32_t* out, cudaStream_t s) {
    k_labels_to_i32<<<grid_for(n, 256), 256, 0, s>>>(lab, n, out);
}

// count_cuts (grem.py:227-252)
__global__ void k_cut(const uint2* __restrict__ e, int64_t m, const int32_t* __restrict__ lab,
                      unsigned long long* cut, int* neg) {
    unsigned long long c = 0;
    int ng = 0;
    GRID_STRIDE(i, m) {
        uint2 ed = e[i];
        int a = lab[ed.x], b = lab[ed.y];
        ng |= (a < 0) | (b < 0);
        c += (a != b);
    }
    for (int off = 16; off; off >>= 1) {
        c += __shfl_down_sync(0xffffffffu, c, off);
        ng |= __shfl_down_sync(0xffffffffu, ng, off);
    }
    if ((threadIdx.x & 31) == 0) {
        if (c) atomicAdd(cut, c);
        if (ng) atomicOr(neg, 1);
    }
}
__global__ void k_hist(const int32_t* __restrict__ lab, int64_t n, unsigned long long* sizes, int64_t cap,
                       int* mx, int* neg) {
    extern __shared__ unsigned int sh[];   // per-block counts: native 32-bit shared atomics (no CAS loop)
    int64_t nb = cap < 1024 ? cap : 1024;
    for (int64_t j = threadIdx.x; j < nb; j += blockDim.x) sh[j] = 0;
    __syncthreads();
    int lm = -1, anyneg = 0;
    const int lane = threadIdx.x & 31;
    if (nb <= 32 && ((uintptr_t)lab & 15) == 0) {
        // few parts: warp ballots per part instead of same-address atomics;
        // lane b keeps the count of part b
        unsigned long long mine = 0;
        int64_t nw4 = n / 4;
        const int4* l4 = reinterpret_cast<const int4*>(lab);
        for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x - lane; w < nw4;
             w += (int64_t)gridDim.x * blockDim.x) {
            int4 q = w + lane < nw4 ? l4[w + lane] : make_int4(-2, -2, -2, -2);
            int v[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                anyneg |= v[j] == -1 || (v[j] < -2);
                lm = v[j] > lm ? v[j] : lm;
                for (int b = 0; b < nb; ++b) {
                    unsigned bal = __ballot_sync(0xffffffffu, v[j] == b);
                    if (lane == b) mine += __popc(bal);
                }
            }
        }
        if (blockIdx.x == 0 && threadIdx.x < 32) {   // tail
            for (int64_t i = nw4 * 4 + threadIdx.x; i < n; i += 32) {
                int l = lab[i];
                if (l < 0) { anyneg = 1; continue; }
                lm = l > lm ? l : lm;
                if (l < nb) atomicAdd(&sh[l], 1u);
            }
        }
        if (lane < nb && mine) atomicAdd(&sh[lane], (unsigned int)mine);
    } else {
        GRID_STRIDE(i, n) {
            int l = lab[i];
            if (l < 0) {
                anyneg = 1;
                continue;
            }
            lm = l > lm ? l : lm;
            if (l < nb) atomicAdd(&sh[l], 1u);
            else if (l < cap) atomicAdd(&sizes[l], 1ULL);
        }
    }
    for (int off = 16; off; off >>= 1) {
        int o = __shfl_down_sync(0xffffffffu, lm, off);
        lm = o > lm ? o : lm;
    }
    if ((threadIdx.x & 31) == 0 && lm >= 0) atomicMax(mx, lm);
    if (anyneg) atomicOr(neg, 4);   // some node is unlabeled (allowed unless it is an endpoint)
    __syncthreads();
    for (int64_t j = threadIdx.x; j < nb; j += blockDim.x)
        if (sh[j]) atomicAdd(&sizes[j], (unsigned long long)sh[j]);
}
void launch_count_cuts(const uint2* e, int64_t m, const int32_t* lab, int64_t n, unsigned long long* d_cut,
                       unsigned long long* d_sizes, int64_t sizes_cap, int* d_max, int* d_neg, cudaStream_t s) {
    if (m > 0 && d_cut) k_cut<<<grid_for(m, 256, 16), 256, 0, s>>>(e, m, lab, d_cut, d_neg);
    int64_t nb = sizes_cap < 1024 ? sizes_cap : 1024;
    k_hist<<<grid_for(n, 256, 4), 256, nb * sizeof(unsigned int), s>>>(lab, n, d_sizes, sizes_cap, d_max,
                                                                            d_neg);
}

__global__ void k_max_id(const uint2* __restrict__ e, int64_t m, uint32_t* mx) {
    uint32_t v = 0;
    GRID_STRIDE(i, m) {
        uint2 ed = e[i];
        v = max(v, max(ed.x, ed.y));
    }
    for (int off = 16; off; off >>= 1) v = max(v, __shfl_down_sync(0xffffffffu, v, off));
    if ((threadIdx.x & 31) == 0) atomicMax(mx, v);
}
// ingest piece check (edgefile.py:63-65): endpoints >= n are recorded (max)
// and replaced by 0 so that kernels that run before the host sees the error
// stay in bounds; the call then fails with the reference's FormatError.
// bad_max: u64, max bad id + 1 (0 = no bad endpoint); 64-bit so that a bad id
// of 0xFFFFFFFF (the usual -1 sentinel) is still recorded
__global__ void k_check_piece(uint2* e, int64_t m, uint32_t n, unsigned long long* bad_max) {
    uint32_t v = 0;
    bool any = false;
    GRID_STRIDE(i, m) {
        uint2 ed = e[i];
        if (ed.x >= n || ed.y >= n) {
            v = max(v, max(ed.x >= n ? ed.x : 0u, ed.y >= n ? ed.y : 0u));
            any = true;
            e[i] = make_uint2(ed.x >= n ? 0u : ed.x, ed.y >= n ? 0u : ed.y);
        }
    }
    if (any) atomicMax(bad_max, (unsigned long long)v + 1ull);
}
// compute_node_stats (theory.py:97-122), hub-privatised form of the packed
// count (grem_store.cu): the bisection's hub table (detect_hubs) is loaded
// into shared memory and endpoints that are hubs accumulate in per-CTA
// shared counters (flushed once per CTA), so the top nodes' millions of
// endpoints stop serialising on single L2 addresses; the rest are REDs into
// one u64 per node (side 0 low / side 1 high half).
__global__ void __launch_bounds__(512) k_node_side_counts_hub(const uint2* __restrict__ e, int64_t m,
                                                              const uint32_t* __restrict__ packed,
                                                              const uint32_t* __restrict__ hub_keys,
                                                              unsigned long long* __restrict__ cnt, int* bad) {
    __shared__ __align__(16) uint32_t s_keys[kHubSlots];
    __shared__ unsigned long long s_cnt[kHubSlots];
    hub_load(s_keys, hub_keys);
    for (int k = threadIdx.x; k < kHubSlots; k += blockDim.x) s_cnt[k] = 0;
    __syncthreads();
    int64_t lo, hi;
    cta_range(m, lo, hi);
    int b = 0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        uint2 ed = __ldcs(e + i);
        if (ed.x == ed.y) continue;   // theory.py:111
        uint32_t lu = (__ldg(packed + (ed.x >> 4)) >> (2 * (ed.x & 15))) & 3u;
        uint32_t lv = (__ldg(packed + (ed.y >> 4)) >> (2 * (ed.y & 15))) & 3u;
        if ((lu | lv) & 2u) {         // theory.py:114-115
            b = 1;
            continue;
        }
        unsigned long long iu = 1ull << (32 * lv), iv = 1ull << (32 * lu);
        int hu = hub_find(s_keys, ed.x), hv = hub_find(s_keys, ed.y);
        // hub halves with native 32-bit shared atomics (a 64-bit one is a CAS loop)
        if (hu >= 0) atomicAdd(reinterpret_cast<unsigned int*>(s_cnt + hu) + lv, 1u);
        else atomicAdd(cnt + ed.x, iu);
        if (hv >= 0) atomicAdd(reinterpret_cast<unsigned int*>(s_cnt + hv) + lu, 1u);
        else atomicAdd(cnt + ed.y, iv);
    }
    if (__any_sync(0xffffffffu, b) && (threadIdx.x & 31) == 0) atomicOr(bad, 1);
    __syncthreads();
    for (int k = threadIdx.x; k < kHubSlots; k += blockDim.x)
        if (s_cnt[k]) atomicAdd(cnt + s_keys[k], s_cnt[k]);
}

void launch_node_side_counts_hub(const uint2* e, int64_t m, const uint32_t* packed, const uint32_t* hub_keys,
                                 unsigned long long* cnt, int* bad, cudaStream_t s) {
    if (m <= 0) return;
    int64_t g = (m + 511) / 512;
    int cap = num_sms() * 4;
    k_node_side_counts_hub<<<(int)(g < cap ? (g < 1 ? 1 : g) : cap), 512, 0, s>>>(e, m, packed, hub_keys, cnt, bad);
}

void launch_check_piece(uint2* e, int64_t m, uint32_t n, unsigned long long* bad_max, cudaStream_t s) {
    if (m > 0) k_check_piece<<<grid_for(m, 256, 8), 256, 0, s>>>(e, m, n, bad_max);
}
void launch_check_ids(const uint2* e, int64_t m, uint32_t* d_max_id, cudaStream_t s) {
    if (m > 0) k_max_id<<<grid_for(m, 256, 8), 256, 0, s>>>(e, m, d_max_id);
}

// --------------------------------------------------------------- recursion

// ------------------------------------------------ succinct side bitmaps
// After a bisection every node is 0 or 1: side-1 bitmap (n bits) + exclusive
// per-word prefix of popcounts.  Dense id of node g inside its side (rank
// among ascending members, grem.py:265-266) = rank1(g) or g - rank1(g);
// both gathers hit the L2-resident 2 x n/8 bytes instead of an n x 4 B table.
__global__ void k_side_bits(const int8_t* __restrict__ lab, int64_t n, uint32_t* __restrict__ bits,
                            uint32_t* __restrict__ wpop, int64_t nwords) {
    GRID_STRIDE(w, nwords) {
        uint32_t b = 0;
        int64_t base = w * 32;
        if (base + 32 <= n) {
            const uint4* p4 = reinterpret_cast<const uint4*>(lab + base);
            uint4 v0 = p4[0], v1 = p4[1];
            uint32_t words[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
            for (int q = 0; q < 8; ++q)
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (((words[q] >> (8 * k)) & 0xFF) == 1) b |= 1u << (q * 4 + k);
        } else {
            for (int j = 0; j < 32; ++j)
                if (base + j < n && lab[base + j] == 1) b |= 1u << j;
        }
        bits[w] = b;
        wpop[w] = __popc(b);
    }
}
__device__ __forceinline__ uint32_t side_rank1(const uint32_t* __restrict__ bits, const uint32_t* __restrict__ pre,
                                               uint32_t g) {
    uint32_t w = g >> 5;
    return pre[w] + __popc(bits[w] & ((1u << (g & 31)) - 1u));
}
__device__ __forceinline__ uint32_t side_newid(const uint32_t* __restrict__ bits, const uint32_t* __restrict__ pre,
                                               uint32_t g, int side) {
    uint32_t r1 = side_rank1(bits, pre, g);
    return side ? r1 : g - r1;
}
__global__ void k_sub_orig_bits(const int8_t* __restrict__ lab, int64_t n, int side, const uint32_t* __restrict__ bits,
                                const uint32_t* __restrict__ pre, const int32_t* __restrict__ orig,
                                int32_t* __restrict__ sub) {
    GRID_STRIDE(i, n) if (lab[i] == side) sub[side_newid(bits, pre, (uint32_t)i, side)] = orig[i];
}
void launch_side_bits(const int8_t* lab, int64_t n, uint32_t* bits, uint32_t* wpop, uint32_t* pre, void* temp,
                      size_t temp_bytes, cudaStream_t s) {
    int64_t nw = (n + 31) / 32;
    k_side_bits<<<grid_for(nw, 256), 256, 0, s>>>(lab, n, bits, wpop, nw);
    cub::DeviceScan::ExclusiveSum(temp, temp_bytes, wpop, pre, (int)(nw + 1), s);
}
// Both induced subgraphs (grem.py:255-274) in ONE pass over the edges:
// per edge two 8-byte gathers of {side bits, rank prefix} words (L2-resident),
// the edge goes to side 0, side 1 or is cut; order within a side stays the
// file order through a tile-local ballot ranking plus a decoupled look-back
// across tiles (dynamic tile ids, so waiting only ever targets started tiles).
#ifndef GREM_SPLIT_T
#define GREM_SPLIT_T 256
#endif
constexpr int kSplitT = GREM_SPLIT_T;   // threads (and 8x edges) per tile: fewer, larger tiles = fewer look-backs
constexpr int kSplitI = 8;
constexpr int kSplitTile = kSplitT * kSplitI;
constexpr unsigned long long kLbAgg = 1ULL << 62, kLbInc = 2ULL << 62, kLbVal = (1ULL << 62) - 1;

__global__ void k_word_info(const uint32_t* __restrict__ bits, const uint32_t* __restrict__ pre, int64_t nw,
                            uint2* __restrict__ wi) {
    GRID_STRIDE(w, nw) wi[w] = make_uint2(bits[w], pre[w]);
}

__device__ __forceinline__ unsigned long long lb_load(const unsigned long long* p) {
    return *reinterpret_cast<const volatile unsigned long long*>(p);
}
// warp-cooperative look-back: exclusive prefix of tile t's value
__device__ unsigned long long lb_prefix(unsigned long long* status, int64_t t) {
    int lane = threadIdx.x & 31;
    unsigned long long acc = 0;
    int64_t j = t - 1;
    while (j >= 0) {
        int64_t q = j - lane;
        unsigned long long st = 0;
        if (q >= 0) {
            do { st = lb_load(status + q); } while ((st >> 62) == 0);
        } else {
            st = kLbInc;   // before tile 0: an inclusive zero
        }
        unsigned inc = __ballot_sync(0xffffffffu, (st >> 62) == 2);
        int stop = inc ? __ffs(inc) - 1 : 32;
        unsigned long long v = lane <= stop ? (st & kLbVal) : 0;
        for (int off = 16; off; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
        acc += __shfl_sync(0xffffffffu, v, 0);
        if (inc) break;
        j -= 32;
    }
    return acc;
}

__global__ void __launch_bounds__(kSplitT) k_split_edges(const uint2* __restrict__ e, int64_t m,
                                                         const uint2* __restrict__ wi, uint2* __restrict__ out0,
                                                         uint2* __restrict__ out1, unsigned long long* status0,
                                                         unsigned long long* status1, unsigned int* ticket,
                                                         long long* counts, int64_t ntiles) {
    __shared__ int64_t s_tile;
    __shared__ uint32_t s_c[2][kSplitI][kSplitT / 32];
    __shared__ unsigned long long s_pre[2];
    constexpr int NW = kSplitT / 32;
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    int64_t t = s_tile;
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t base = t * kSplitTile;
    uint2 ed[kSplitI];
    int side[kSplitI];
    uint32_t rank[kSplitI];
    // all edge loads, then all side-map gathers, in flight before any use
    uint2 dd[kSplitI], wa[kSplitI], wb[kSplitI];
#pragma unroll
    for (int k = 0; k < kSplitI; ++k) {
        int64_t i = base + (int64_t)k * kSplitT + threadIdx.x;   // warp-striped: coalesced loads
        dd[k] = i < m ? __ldcs(e + i) : make_uint2(0, 0);
    }
#pragma unroll
    for (int k = 0; k < kSplitI; ++k) {
        wa[k] = wi[dd[k].x >> 5];
        wb[k] = wi[dd[k].y >> 5];
    }
#pragma unroll
    for (int k = 0; k < kSplitI; ++k) {
        int64_t i = base + (int64_t)k * kSplitT + threadIdx.x;
        side[k] = 2;
        if (i < m) {
            uint2 d = dd[k];
            uint2 a = wa[k], b = wb[k];
            uint32_t su = (a.x >> (d.x & 31)) & 1u, sv = (b.x >> (d.y & 31)) & 1u;
            if (su == sv) {
                uint32_t r1u = a.y + __popc(a.x & ((1u << (d.x & 31)) - 1u));
                uint32_t r1v = b.y + __popc(b.x & ((1u << (d.y & 31)) - 1u));
                side[k] = (int)su;
                ed[k] = su ? make_uint2(r1u, r1v) : make_uint2(d.x - r1u, d.y - r1v);
            }
        }
        unsigned b0 = __ballot_sync(0xffffffffu, side[k] == 0), b1 = __ballot_sync(0xffffffffu, side[k] == 1);
        unsigned lt = (1u << lane) - 1u;
        rank[k] = side[k] == 0 ? __popc(b0 & lt) : __popc(b1 & lt);
        if (lane == 0) {
            s_c[0][k][wid] = __popc(b0);
            s_c[1][k][wid] = __popc(b1);
        }
    }
    __syncthreads();
    // exclusive prefix over (k, warp) in edge order, per side; warps 0/1 own sides 0/1
    if (wid < 2) {
        int sd = wid;
        constexpr int NE = kSplitI * NW;   // (k, warp) entries in edge order
        constexpr int PER = NE / 32;       // consecutive entries per lane
        static_assert(NE % 32 == 0, "whole entries per lane");
        uint32_t v[PER], sum = 0;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            int en = lane * PER + q;
            v[q] = s_c[sd][en / NW][en % NW];
            sum += v[q];
        }
        uint32_t incl = sum;
        for (int off = 1; off < 32; off <<= 1) {
            uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += o;
        }
        uint32_t excl = incl - sum;
        __syncwarp();
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            int en = lane * PER + q;
            s_c[sd][en / NW][en % NW] = excl;
            excl += v[q];
        }
        uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        unsigned long long* status = sd ? status1 : status0;
        unsigned long long prefix = 0;
        if (t == 0) {
            if (lane == 0) atomicExch(status, kLbInc | total);
        } else {
            if (lane == 0) atomicExch(status + t, kLbAgg | total);
            prefix = lb_prefix(status, t);
            if (lane == 0) atomicExch(status + t, kLbInc | (prefix + total));
        }
        if (lane == 0) {
            s_pre[sd] = prefix;
            if (t == ntiles - 1) counts[sd] = (long long)(prefix + total);
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kSplitI; ++k) {
        if (side[k] == 2) continue;
        unsigned long long p = s_pre[side[k]] + s_c[side[k]][k][wid] + rank[k];
        if (side[k]) out1[-(int64_t)p] = ed[k];   // side 1 grows down from the arena's last slot
        else out0[p] = ed[k];
    }
}

// side 1 was written backwards from the end of the arena: restore file order
__global__ void k_reverse_u64(unsigned long long* a, int64_t n) {
    GRID_STRIDE(i, n / 2) {
        unsigned long long x = a[i], y = a[n - 1 - i];
        a[i] = y;
        a[n - 1 - i] = x;
    }
}
void launch_reverse_edges(uint2* a, int64_t n, cudaStream_t s) {
    if (n > 1) k_reverse_u64<<<grid_for(n / 2, 256, 8), 256, 0, s>>>(reinterpret_cast<unsigned long long*>(a), n);
}
size_t split_edges_tiles(int64_t m) { return (size_t)((m + kSplitTile - 1) / kSplitTile); }
// One arena of m edges holds both induced subgraphs: side 0 from the front in
// file order, side 1 from the back in reverse file order (launch_reverse_edges
// on its e1 edges restores the order), so extraction needs m, not 2m, slots.
void launch_split_edges(const uint2* e, int64_t m, const uint32_t* bits, const uint32_t* pre, int64_t nw, uint2* wi,
                        uint2* arena, unsigned long long* status, unsigned int* ticket, long long* counts,
                        cudaStream_t s) {
    uint2* out0 = arena;
    uint2* out1 = arena + (m > 0 ? m - 1 : 0);
    int64_t ntiles = (int64_t)split_edges_tiles(m);
    k_word_info<<<grid_for(nw, 256), 256, 0, s>>>(bits, pre, nw, wi);
    cudaMemsetAsync(counts, 0, 2 * sizeof(long long), s);
    if (ntiles == 0) return;
    cudaMemsetAsync(status, 0, sizeof(unsigned long long) * 2 * ntiles, s);
    cudaMemsetAsync(ticket, 0, sizeof(unsigned int), s);
    k_split_edges<<<(unsigned)ntiles, kSplitT, 0, s>>>(e, m, wi, out0, out1, status, status + ntiles, ticket, counts,
                                                       ntiles);
}

void launch_sub_orig_bits(const int8_t* lab, int64_t n, int side, const uint32_t* bits, const uint32_t* pre,
                          const int32_t* orig, int32_t* sub, cudaStream_t s) {
    k_sub_orig_bits<<<grid_for(n, 256), 256, 0, s>>>(lab, n, side, bits, pre, orig, sub);
}

// count_cuts with bit-packed labels: 2^lb bits per label (lb <= 5)
__global__ void k_pack_labels(const int32_t* __restrict__ lab, int64_t n, int lb, uint32_t* __restrict__ out,
                              int64_t nwords, int* neg) {
    int per = 32 >> lb, width = 1 << lb;
    int ng = 0;
    GRID_STRIDE(w, nwords) {
        uint32_t v = 0;
        for (int j = 0; j < per; ++j) {
            int64_t i = w * per + j;
            if (i < n) {
                int32_t l = lab[i];
                ng |= l < 0;
                v |= ((uint32_t)l & (width == 32 ? 0xFFFFFFFFu : ((1u << width) - 1))) << (j * width);
            }
        }
        out[w] = v;
    }
    if (ng) atomicOr(neg, 2);
}
__global__ void k_cut_packed(const uint2* __restrict__ e, int64_t m, const uint32_t* __restrict__ pl, int lb,
                             unsigned long long* cut) {
    int width = 1 << lb, lpw = 5 - lb;
    uint32_t mask = width == 32 ? 0xFFFFFFFFu : ((1u << width) - 1);
    unsigned long long c = 0;
    GRID_STRIDE(i, m) {
        uint2 ed = e[i];
        uint32_t a = (pl[ed.x >> lpw] >> ((ed.x & ((1u << lpw) - 1)) << lb)) & mask;
        uint32_t b = (pl[ed.y >> lpw] >> ((ed.y & ((1u << lpw) - 1)) << lb)) & mask;
        c += (a != b);
    }
    for (int off = 16; off; off >>= 1) c += __shfl_down_sync(0xffffffffu, c, off);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(cut, c);
}
void launch_count_cuts_packed(const uint2* e, int64_t m, const int32_t* lab, int64_t n, int lb, uint32_t* packed,
                              unsigned long long* d_cut, int* d_neg, cudaStream_t s) {
    int per = 32 >> lb;
    int64_t nw = (n + per - 1) / per;
    k_pack_labels<<<grid_for(nw, 256), 256, 0, s>>>(lab, n, lb, packed, nw, d_neg);
    if (m > 0) k_cut_packed<<<grid_for(m, 256, 16), 256, 0, s>>>(e, m, packed, lb, d_cut);
}

__global__ void k_side_flags(const int8_t* lab, int64_t n, int side, int32_t* f) {
    GRID_STRIDE(i, n) f[i] = lab[i] == side ? 1 : 0;
}
void launch_side_flags(const int8_t* lab, int64_t n, int side, int32_t* flags, cudaStream_t s) {
    k_side_flags<<<grid_for(n, 256), 256, 0, s>>>(lab, n, side, flags);
}

struct SidePred {
    const int8_t* lab;
    int side;
    __device__ __forceinline__ bool operator()(const uint2& ed) const {
        return lab[ed.x] == side && lab[ed.y] == side;
    }
};
size_t extract_temp_bytes(int64_t m) {
    size_t bytes = 0;
    cub::DeviceSelect::If(nullptr, bytes, (const uint2*)nullptr, (uint2*)nullptr, (long long*)nullptr, m,
                          SidePred{nullptr, 0});
    return bytes;
}
__global__ void k_remap(uint2* e, const long long* cnt, const int32_t* newid) {
    int64_t m = *cnt;
    GRID_STRIDE(i, m) {
        uint2 ed = e[i];
        e[i] = make_uint2((uint32_t)newid[ed.x], (uint32_t)newid[ed.y]);
    }
}
void launch_extract(const uint2* e, int64_t m, const int8_t* lab, int side, const int32_t* newid, uint2* out,
                    long long* d_count, void* temp, size_t temp_bytes, cudaStream_t s) {
    // kept edges in file order (stable selection), dense ids = rank among members
    cub::DeviceSelect::If(temp, temp_bytes, e, out, d_count, m, SidePred{lab, side}, s);
    k_remap<<<grid_for(m, 256, 8), 256, 0, s>>>(out, d_count, newid);
}

__global__ void k_sub_orig(const int8_t* lab, int64_t n, int side, const int32_t* newid, const int32_t* orig,
                           int32_t* sub) {
    GRID_STRIDE(i, n) if (lab[i] == side) sub[newid[i]] = orig[i];
}
void launch_sub_orig(const int8_t* lab, int64_t n, int side, const int32_t* newid, const int32_t* orig,
                     int32_t* sub_orig, cudaStream_t s) {
    k_sub_orig<<<grid_for(n, 256), 256, 0, s>>>(lab, n, side, newid, orig, sub_orig);
}

__global__ void k_leaf_write(const int8_t* lab, int64_t n, const int32_t* orig, int32_t base, int32_t* fin) {
    GRID_STRIDE(i, n) fin[orig[i]] = base + lab[i];
}
void launch_leaf_write(const int8_t* lab, int64_t n, const int32_t* orig, int32_t leaf_base, int32_t* final_lab,
                       cudaStream_t s) {
    k_leaf_write<<<grid_for(n, 256), 256, 0, s>>>(lab, n, orig, leaf_base, final_lab);
}

// cut edges of one bisection (its own edge list and 0/1 labels): edges whose
// endpoints got different sides.  partition() sums these over the leaf
// bisections and adds the edges every extraction drops (grem_runtime.cu
// recurse), which is the final count_cuts' cut (grem.py:235-240) without a
// pass over the original edges after the last leaf.
__global__ void k_bisect_cut(const uint2* __restrict__ e, int64_t m, const int8_t* __restrict__ lab,
                             unsigned long long* out) {
    unsigned long long c = 0;
    GRID_STRIDE(i, m) {
        uint2 ed = __ldcs(e + i);
        c += __ldg(lab + ed.x) != __ldg(lab + ed.y);
    }
    for (int off = 16; off; off >>= 1) c += __shfl_down_sync(0xffffffffu, c, off);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}
void launch_bisect_cut(const uint2* e, int64_t m, const int8_t* lab, unsigned long long* out, cudaStream_t s) {
    cudaMemsetAsync(out, 0, sizeof(unsigned long long), s);
    if (m > 0) k_bisect_cut<<<grid_for(m, 256, 8), 256, 0, s>>>(e, m, lab, out);
}

__global__ void k_iota(int32_t* a, int64_t n) {
    GRID_STRIDE(i, n) a[i] = (int32_t)i;
}
void launch_iota(int32_t* a, int64_t n, cudaStream_t s) { k_iota<<<grid_for(n, 256), 256, 0, s>>>(a, n); }

// ------------------------------------------------------------- CUB helpers

size_t scan_temp_bytes(int64_t n) {
    size_t a = 0, b = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, a, (int32_t*)nullptr, (int32_t*)nullptr, (int)n);
    cub::DeviceScan::ExclusiveSum(nullptr, b, (int64_t*)nullptr, (int64_t*)nullptr, (int)n);
    return a > b ? a : b;
}
void exclusive_sum_i32(const int32_t* in, int32_t* out, int64_t n, void* temp, size_t temp_bytes, cudaStream_t s) {
    cub::DeviceScan::ExclusiveSum(temp, temp_bytes, in, out, (int)n, s);
}
void exclusive_sum_i64(const int64_t* in, int64_t* out, int64_t n, void* temp, size_t temp_bytes, cudaStream_t s) {
    cub::DeviceScan::ExclusiveSum(temp, temp_bytes, in, out, (int)n, s);
}
size_t sort_temp_bytes(int64_t n) {
    size_t a = 0, b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, (unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                    (uint32_t*)nullptr, (uint32_t*)nullptr, (int)n);
    cub::DeviceRadixSort::SortKeys(nullptr, b, (unsigned long long*)nullptr, (unsigned long long*)nullptr, (int)n);
    return a > b ? a : b;
}
void sort_pairs_u64_u32(const unsigned long long* kin, unsigned long long* kout, const uint32_t* vin, uint32_t* vout,
                        int64_t n, void* temp, size_t temp_bytes, cudaStream_t s) {
    cub::DeviceRadixSort::SortPairs(temp, temp_bytes, kin, kout, vin, vout, (int)n, 0, 64, s);
}
void sort_keys_u64_desc(const unsigned long long* kin, unsigned long long* kout, int64_t n, void* temp,
                        size_t temp_bytes, cudaStream_t s) {
    cub::DeviceRadixSort::SortKeysDescending(temp, temp_bytes, kin, kout, (int)n, 0, 64, s);
}
void sort_keys_u64(const unsigned long long* kin, unsigned long long* kout, int64_t n, void* temp, size_t temp_bytes,
                   cudaStream_t s) {
    cub::DeviceRadixSort::SortKeys(temp, temp_bytes, kin, kout, (int)n, 0, 64, s);
}

// ------------------------------------------------------------- generator
__global__ void k_gen(gg_params p, uint64_t e0, uint64_t count, uint32_t* out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t j = 2 * (e0 + i);
        uint2 ed = make_uint2(gg_endpoint(&p, j), gg_endpoint(&p, j + 1));
        reinterpret_cast<uint2*>(out)[i] = ed;
    }
}
void launch_gen_edges(uint64_t n, uint32_t beta, uint64_t seed, double scale, uint64_t perm_mask, uint32_t perm_bits,
                      uint64_t e0, uint64_t count, uint32_t* out, cudaStream_t s) {
    gg_params p;
    p.n = n;
    p.seed = seed;
    p.beta = beta;
    p.scale = scale;
    p.perm_mask = perm_mask;
    p.perm_bits = perm_bits;
    k_gen<<<grid_for((int64_t)count, 256, 32), 256, 0, s>>>(p, e0, count, out);
}


// ===================================================== binned round-1 counts
// Round 1 of a large chunk (cnt_nbrs with pre-sweep labels, grem.py:82-97,
// plus the chunk node set np.unique, model.py:59) in three passes:
//   k_bin_hist     records per (coarse bin of 2^shift node ids, scatter CTA),
//                  scanned into private per-CTA cursors;
//   k_bin_scatter  per 8192-edge batch a block counting sort by coarse bin
//                  (rank = smem atomic return), coalesced record runs out;
//   k_bin_compact  one CTA per 2^kSubShift-node tile, in node order: smem
//                  counters (smem atomics run ~12x faster than L2 REDs),
//                  hub counts merged, chunk membership, block scan and a
//                  decoupled look-back give the chunk index, and the compact
//                  round state is written directly (no n-sized counters, no
//                  select, no separate node init or scan).
// Records: node << 2 | code (1: +c0, 2: +c1, 0: unassigned neighbour, 3: self-loop).

// Per-CTA record histogram (the scatter CTA c covers the same contiguous
// edge range): hist[bin * G + c]; its exclusive scan gives every CTA a private,
// deterministic cursor per bin (no global atomics in the scatter).
// Scatter shape (A/B build knobs): GREM_SCAT_T threads per CTA and
// 1024 / GREM_SCAT_T CTAs per SM; the bin count limit kMaxBins (grem_kernels.cuh)
// must be <= 2 * GREM_SCAT_T (two bins per thread in the batch scan).
#ifndef GREM_SCAT_T
#define GREM_SCAT_T 1024
#endif
constexpr int kScatT = GREM_SCAT_T;
constexpr int kScatPerSM = 1024 / kScatT;   // the 64-register budget: 1024 resident threads
static_assert(kMaxBins <= 2 * kScatT, "two bins per thread in the batch scan");
__global__ void __launch_bounds__(1024) k_bin_hist(const uint2* __restrict__ e, int64_t m,
                                                     const uint32_t* __restrict__ hub_keys, int shift, int nbins,
                                                     int32_t* __restrict__ hist) {
    __shared__ __align__(8) uint32_t s_keys[kHubSlots];
    __shared__ unsigned int s_hist[kMaxBins];
    hub_load(s_keys, hub_keys);
    const int bd = blockDim.x;   // the scatter's CTA decomposition
    for (int k = threadIdx.x; k < nbins; k += bd) s_hist[k] = 0;
    __syncthreads();
    int64_t lo, hi;
    cta_range(m, lo, hi);
    for (int64_t i = lo + threadIdx.x; i < hi; i += 4 * bd) {
        uint2 ed[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) ed[j] = i + j * bd < hi ? __ldcs(e + i + j * bd) : make_uint2(kHubEmpty, kHubEmpty);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (ed[j].x == kHubEmpty) continue;
            if (hub_find(s_keys, ed[j].x) < 0) atomicAdd(&s_hist[ed[j].x >> shift], 1u);
            if (ed[j].x != ed[j].y && hub_find(s_keys, ed[j].y) < 0) atomicAdd(&s_hist[ed[j].y >> shift], 1u);
        }
    }
    __syncthreads();
    for (int k = threadIdx.x; k <= nbins; k += bd)
        hist[(int64_t)k * gridDim.x + blockIdx.x] = k < nbins ? (int32_t)s_hist[k] : 0;   // row nbins: total
}

#ifndef GREM_SCAT_IPT
#define GREM_SCAT_IPT 8
#endif
constexpr int kScatIPT = GREM_SCAT_IPT;
constexpr int kScatBatch = kScatT * kScatIPT;   // edges per batch, <= 2 records each
// Shared-memory footprint (ncu r02i: hub probes 39% and carry-slot reads
// 13.5% of the shared wavefronts).  GREM_SCAT_BLOOM=1 puts a one-bit
// prefilter in front of the hub probes; GREM_CARRY_STRIDE=9 pads the per-bin
// carry slots so the flush loop (thread t: bins 2t, 2t+1) leaves its 16-way
// bank conflict.  Both need 8 KB of shared memory, and with 2048 bins either
// one pushed the kernel (197 -> 205 KB) to the largest carve-out, halving the
// L1 left for the label gathers: 91 -> 116 ms summed
// (profiles/r02_ab_scatter_smem.txt).  With 1024 bins (GREM_MAX_BINS) the
// kernel needs 160 KB, keeps the 164 KB carve-out with 92 KB of L1, and both
// fit: step 570 -> 554 ms (profiles/r02_ab_scatter_bins.txt; the compact
// reads each bin's records from twice as many tiles, 39 -> 49 ms summed).
#ifndef GREM_SCAT_BLOOM
#define GREM_SCAT_BLOOM 1
#endif
#ifndef GREM_CARRY_STRIDE
#define GREM_CARRY_STRIDE 9
#endif
constexpr int kCarryStride = GREM_CARRY_STRIDE;
constexpr size_t kScatSmem = (size_t)kHubSlots * (4 + 8 + 4) + (size_t)kMaxBins * 4 * 4 +
                             (size_t)kMaxBins * 4 * kCarryStride + (size_t)2 * kScatBatch * 4 + 64 * 4 +
                             (GREM_SCAT_BLOOM ? (size_t)kBloomWords * 4 : 0);

__global__ void __launch_bounds__(kScatT, kScatPerSM) k_bin_scatter(const uint2* __restrict__ e, int64_t m,
                                                        const uint32_t* __restrict__ lab2,
                                                        const uint32_t* __restrict__ hub_keys, int shift, int nbins,
                                                        const int32_t* __restrict__ offs,
                                                        uint32_t* __restrict__ recs,
                                                        unsigned long long* __restrict__ hub_cnt,
                                                        uint32_t* __restrict__ hub_flag) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // per hub slot {label-0 count, label-1 count} as two 32-bit halves: native
    // 32-bit shared atomics (a 64-bit shared atomicAdd compiles to a CAS spin
    // loop, which on the hot hub slots was a third of the kernel's shared
    // wavefronts, ncu r02_final)
    unsigned long long* s_hcnt = reinterpret_cast<unsigned long long*>(smem_raw);
    uint32_t* s_keys = reinterpret_cast<uint32_t*>(s_hcnt + kHubSlots);
    uint32_t* s_hflag = s_keys + kHubSlots;
    unsigned int* s_hist = s_hflag + kHubSlots;
    unsigned int* s_start = s_hist + kMaxBins;
    unsigned int* s_cur = s_start + kMaxBins;
    unsigned int* s_beg = s_cur + kMaxBins;       // first record slot of this CTA's region per bin
    uint32_t* s_carry = s_beg + kMaxBins;         // per bin: the open (incomplete) 32-byte sector
    uint32_t* s_out = s_carry + kCarryStride * kMaxBins;
    unsigned int* s_w = s_out + 2 * kScatBatch;
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    hub_load(s_keys, hub_keys);
#if GREM_SCAT_BLOOM
    uint32_t* s_bloom = s_w + 64;
    __syncthreads();
    hub_bloom_build(s_bloom, s_keys);   // visible after the first batch's barrier
#define SCAT_HUB_FIND(x) hub_find_pf(s_keys, s_bloom, (x))
#else
#define SCAT_HUB_FIND(x) hub_find(s_keys, (x))
#endif
    for (int k = t; k < kHubSlots; k += kScatT) {
        s_hcnt[k] = 0ULL;
        s_hflag[k] = 0u;
    }
    for (int k = t; k < nbins; k += kScatT) s_beg[k] = s_cur[k] = (unsigned int)offs[(int64_t)k * gridDim.x + blockIdx.x];
    int64_t lo, hi;
    cta_range(m, lo, hi);
    for (int64_t b0 = lo; b0 < hi; b0 += kScatBatch) {
        for (int k = t; k < nbins; k += kScatT) s_hist[k] = 0u;
        uint2 ed[kScatIPT];
#pragma unroll
        for (int k = 0; k < kScatIPT; ++k) {
            int64_t i = b0 + (int64_t)k * kScatT + t;
            ed[k] = i < hi ? __ldcs(e + i) : make_uint2(kHubEmpty, kHubEmpty);   // streaming: keep L2 for the record runs
        }
        __syncthreads();
        uint32_t rec[2 * kScatIPT], rk[2 * kScatIPT];
#pragma unroll
        for (int k = 0; k < kScatIPT; ++k) {
            rec[2 * k] = 0xFFFFFFFFu;
            rec[2 * k + 1] = 0xFFFFFFFFu;
            uint32_t u = ed[k].x, v = ed[k].y;
            if (u != kHubEmpty) {
                int hu = SCAT_HUB_FIND(u);
                if (u == v) {   // self-loop: u is a chunk node, no count (model.py:53-55)
                    if (hu >= 0) s_hflag[hu] = 1u;
                    else rec[2 * k] = (u << 2) | 3u;
                } else {
                    int hv = SCAT_HUB_FIND(v);
                    uint32_t cu = lab2_code(lab2, u), cv = lab2_code(lab2, v);
                    if (hu >= 0) {
                        if (cv) atomicAdd(reinterpret_cast<unsigned int*>(s_hcnt + hu) + (cv == 1 ? 0 : 1), 1u);
                        else s_hflag[hu] = 1u;
                    } else {
                        rec[2 * k] = (u << 2) | cv;
                    }
                    if (hv >= 0) {
                        if (cu) atomicAdd(reinterpret_cast<unsigned int*>(s_hcnt + hv) + (cu == 1 ? 0 : 1), 1u);
                        else s_hflag[hv] = 1u;
                    } else {
                        rec[2 * k + 1] = (v << 2) | cu;
                    }
                }
            }
#pragma unroll
            for (int h = 0; h < 2; ++h)
                if (rec[2 * k + h] != 0xFFFFFFFFu) rk[2 * k + h] = atomicAdd(&s_hist[(rec[2 * k + h] >> 2) >> shift], 1u);
        }
        __syncthreads();
        // exclusive scan of the batch's bin histogram (nbins <= 2 * kScatT)
        unsigned int v0 = 2 * t < nbins ? s_hist[2 * t] : 0u, v1 = 2 * t + 1 < nbins ? s_hist[2 * t + 1] : 0u;
        {
            unsigned int pr = v0 + v1, incl = pr;
            for (int off = 1; off < 32; off <<= 1) {
                unsigned int o = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= off) incl += o;
            }
            if (lane == 31) s_w[wid] = incl;
            __syncthreads();
            if (wid == 0) {
                unsigned int w = lane < kScatT / 32 ? s_w[lane] : 0u, wi = w;
                for (int off = 1; off < 32; off <<= 1) {
                    unsigned int o = __shfl_up_sync(0xffffffffu, wi, off);
                    if (lane >= off) wi += o;
                }
                if (lane < kScatT / 32) s_w[lane] = wi - w;
                if (lane == 31) s_w[32] = wi;
            }
            __syncthreads();
            unsigned int ex = s_w[wid] + incl - pr;
            if (2 * t < nbins) s_start[2 * t] = ex;
            if (2 * t + 1 < nbins) s_start[2 * t + 1] = ex + v0;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 2 * kScatIPT; ++k)
            if (rec[k] != 0xFFFFFFFFu) s_out[s_start[(rec[k] >> 2) >> shift] + rk[k]] = rec[k];
        // Records leave in whole 32-byte sectors: a bin's open sector waits in
        // shared memory until this CTA's next run of that bin completes it
        // (partial sectors would cost a DRAM read-modify-write).
#pragma unroll
        for (int h = 0; h < 2; ++h) {   // flush open sectors this batch completes
            int k = 2 * t + h;
            unsigned int v = h ? v1 : v0;
            if (k < nbins && v) {
                unsigned int cur = s_cur[k], sec = cur & ~7u;
                if ((cur & 7u) && cur + v >= sec + 8) {
                    unsigned int lo = s_beg[k] > sec ? s_beg[k] : sec;
                    for (unsigned int p = lo; p < cur; ++p) recs[p] = s_carry[kCarryStride * k + (p & 7u)];
                }
            }
        }
        __syncthreads();
        unsigned int nrec = s_w[32];
        for (unsigned int k = t; k < nrec; k += kScatT) {   // runs of a bin are contiguous
            uint32_t r = s_out[k];
            unsigned int bb = (r >> 2) >> shift;
            unsigned int p = s_cur[bb] + (k - s_start[bb]);
            if (p < ((s_cur[bb] + s_hist[bb]) & ~7u)) recs[p] = r;
            else s_carry[kCarryStride * bb + (p & 7u)] = r;
        }
        __syncthreads();
        if (2 * t < nbins) s_cur[2 * t] += v0;
        if (2 * t + 1 < nbins) s_cur[2 * t + 1] += v1;
    }
    __syncthreads();
    for (int k = t; k < nbins; k += kScatT) {   // the last open sectors
        unsigned int cur = s_cur[k], sec = cur & ~7u;
        if (cur & 7u) {
            unsigned int lo = s_beg[k] > sec ? s_beg[k] : sec;
            for (unsigned int p = lo; p < cur; ++p) recs[p] = s_carry[kCarryStride * k + (p & 7u)];
        }
    }
    for (int k = t; k < kHubSlots; k += kScatT) {
        if (s_keys[k] == kHubEmpty) continue;
        if (s_hcnt[k]) atomicAdd(&hub_cnt[k], s_hcnt[k]);
        if (s_hflag[k]) hub_flag[k] = 1u;
    }
}
#undef SCAT_HUB_FIND

constexpr int kCmpSub = 1 << kSubShift;              // nodes per tile
constexpr int kCmpT = kCmpSub / 16;
constexpr int kCmpIPT = kCmpSub / kCmpT;             // 16 consecutive nodes per thread
constexpr size_t kCmpSmem = (size_t)kCmpSub * (8 + 2 + 2) + (size_t)kCmpSub / 8 + 64 * 8;
static_assert(kCmpIPT == 16, "16 nodes per thread (one 16-byte label load)");

__global__ void __launch_bounds__(kCmpT) k_bin_compact(const uint32_t* __restrict__ recs,
                                                       const int32_t* __restrict__ offs, int G, int shift,
                                                       int64_t n, const uint32_t* __restrict__ hub_keys,
                                                       const unsigned long long* __restrict__ hub_cnt,
                                                       const uint32_t* __restrict__ hub_flag, int refine,
                                                       ChunkBufs b, unsigned long long* status,
                                                       unsigned int* ticket, int64_t ntiles) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned long long* s_cnt = reinterpret_cast<unsigned long long*>(smem_raw);
    unsigned long long* s_w = s_cnt + kCmpSub;
    uint32_t* s_pres = reinterpret_cast<uint32_t*>(s_w + 64);
    uint16_t* s_idx = reinterpret_cast<uint16_t*>(s_pres + kCmpSub / 32);   // member k: local id | old code << 14
    uint16_t* s_nwx = s_idx + kCmpSub;                                       // member k: new members before k
    __shared__ int64_t s_tile;
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    if (t == 0) s_tile = atomicAdd(ticket, 1u);
    for (int k = t; k < kCmpSub; k += kCmpT) s_cnt[k] = 0ULL;
    for (int k = t; k < kCmpSub / 32; k += kCmpT) s_pres[k] = 0u;
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t g0 = tile << kSubShift;
    const int64_t cb = g0 >> shift;
    const int64_t rbeg = offs[cb * G], rend = offs[(cb + 1) * G];
    // records of the coarse bin that fall in this tile (16-byte loads, 4 in flight)
    auto apply = [&](uint32_t r) {
        uint32_t node = r >> 2;
        if ((int64_t)(node >> kSubShift) != tile) return;
        uint32_t l = node & (kCmpSub - 1), c = r & 3u;
        if (c == 1) atomicAdd(reinterpret_cast<unsigned int*>(s_cnt + l), 1u);
        else if (c == 2) atomicAdd(reinterpret_cast<unsigned int*>(s_cnt + l) + 1, 1u);
        else atomicOr(&s_pres[l >> 5], 1u << (l & 31));
    };
    int64_t abeg = (rbeg + 3) & ~3LL, aend = rend & ~3LL;
    if (abeg >= aend) {
        for (int64_t k = rbeg + t; k < rend; k += kCmpT) apply(recs[k]);
    } else {
        if (rbeg + t < abeg) apply(recs[rbeg + t]);
        if (aend + t < rend) apply(recs[aend + t]);
        const uint4* q4 = reinterpret_cast<const uint4*>(recs + abeg);
        int64_t nq = (aend - abeg) >> 2;
        for (int64_t k = t; k < nq; k += 4 * kCmpT) {
            uint4 q[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) q[j] = k + j * kCmpT < nq ? q4[k + j * kCmpT] : make_uint4(~0u, ~0u, ~0u, ~0u);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                apply(q[j].x);
                apply(q[j].y);
                apply(q[j].z);
                apply(q[j].w);
            }
        }
    }
    if (hub_keys) {   // hubs never emit records: their counts come from the slot table
        for (int k = t; k < kHubSlots; k += kCmpT) {
            uint32_t key = hub_keys[k];
            if (key == kHubEmpty || (int64_t)(key >> kSubShift) != tile) continue;
            uint32_t l = key & (kCmpSub - 1);
            unsigned long long c = hub_cnt[k];
            if (c) s_cnt[l] = c;
            if (hub_flag[k]) atomicOr(&s_pres[l >> 5], 1u << (l & 31));
        }
    }
    __syncthreads();
    // counted nodes into the presence bits, one 32-node word per warp ballot
    // (conflict-free: lane j reads node 32w + j; reading the counts of a
    // thread's own 16 consecutive nodes below was a 32-way bank conflict)
    for (int q = wid; q < kCmpSub / 32; q += kCmpT / 32) {
        unsigned bal = __ballot_sync(0xffffffffu, s_cnt[q * 32 + lane] != 0ULL);
        if (lane == 0 && bal) s_pres[q] |= bal;
    }
    __syncthreads();
    // this thread's 16 consecutive nodes: membership, old labels, new flags
    const int l0 = t * kCmpIPT;
    const int64_t gt = g0 + l0;
    int8_t lab16[kCmpIPT];
    if (gt + kCmpIPT <= n) {
        uint4 q = *reinterpret_cast<const uint4*>(b.lab + gt);
        const int8_t* qb = reinterpret_cast<const int8_t*>(&q);
#pragma unroll
        for (int j = 0; j < kCmpIPT; ++j) lab16[j] = qb[j];
    } else {
#pragma unroll
        for (int j = 0; j < kCmpIPT; ++j) lab16[j] = gt + j < n ? b.lab[gt + j] : (int8_t)-1;
    }
    uint32_t pw = (s_pres[l0 >> 5] >> (l0 & 31)) & 0xFFFFu;
    uint32_t pmask = 0, nmask = 0;
#pragma unroll
    for (int j = 0; j < kCmpIPT; ++j) {
        bool pres = (gt + j < n) && ((pw >> j) & 1u);
        if (pres) {
            pmask |= 1u << j;
            if (lab16[j] == -1) nmask |= 1u << j;
        }
    }
    // block scan of (members, new members) packed as p | nw << 31
    unsigned long long mine = (unsigned long long)__popc(pmask) | ((unsigned long long)__popc(nmask) << 31);
    unsigned long long incl = mine;
    for (int off = 1; off < 32; off <<= 1) {
        unsigned long long o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += o;
    }
    if (lane == 31) s_w[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        unsigned long long w = lane < kCmpT / 32 ? s_w[lane] : 0ULL, wi = w;
        for (int off = 1; off < 32; off <<= 1) {
            unsigned long long o = __shfl_up_sync(0xffffffffu, wi, off);
            if (lane >= off) wi += o;
        }
        s_w[lane] = wi - w;
        unsigned long long total = __shfl_sync(0xffffffffu, wi, 31);
        unsigned long long prefix = 0;
        if (tile == 0) {
            if (lane == 0) atomicExch(status, kLbInc | total);
        } else {
            if (lane == 0) atomicExch(status + tile, kLbAgg | total);
            prefix = lb_prefix(status, tile);
            if (lane == 0) atomicExch(status + tile, kLbInc | (prefix + total));
        }
        if (lane == 0) {
            s_w[32] = prefix;
            s_w[33] = total;
            if (tile == ntiles - 1) {
                unsigned long long all = prefix + total;
                b.scal[0] = (long long)(all & 0x7FFFFFFFULL);
                b.scal[2] = (long long)(all >> 31);
            }
        }
    }
    __syncthreads();
    int kfirst;   // this thread's first member's index inside the tile
    {   // members of this thread in tile order
        unsigned long long ex = s_w[wid] + incl - mine;
        int k = (int)(ex & 0x7FFFFFFFULL), nw = (int)(ex >> 31);
        kfirst = k;
#pragma unroll
        for (int j = 0; j < kCmpIPT; ++j) {
            if (!((pmask >> j) & 1u)) continue;
            s_idx[k] = (uint16_t)((l0 + j) | ((lab16[j] + 1) << 14));
            s_nwx[k] = (uint16_t)nw;
            nw += (nmask >> j) & 1u;
            ++k;
        }
    }
    __syncthreads();
    // outputs, one member per thread (coalesced chunk-index writes)
    const unsigned long long pre = s_w[32];
    const int64_t i0 = (int64_t)(pre & 0x7FFFFFFFULL);
    const long long nb0 = b.sizes[0] + b.sizes[1] + (long long)(pre >> 31);
    const int cnt = (int)(s_w[33] & 0x7FFFFFFFULL);
    {   // succinct id -> chunk index map: this tile's 512 rank words {bits, members before}
        uint32_t hi = __shfl_down_sync(0xffffffffu, pmask, 1);
        if (!(t & 1)) b.rankw[(g0 >> 5) + (t >> 1)] = make_uint2(pmask | (hi << 16), (uint32_t)(i0 + kfirst));
    }
    for (int k = t; k < cnt; k += kCmpT) {
        uint32_t v = s_idx[k];
        uint32_t l = v & (kCmpSub - 1);
        int code = (int)(v >> 14);
        uint32_t g = (uint32_t)(g0 + l);
        bool isnew = code == 0;
        bool active = isnew || refine;
        int64_t i = i0 + k;
        b.nodes[i] = g;
        b.meta[i] = (uint8_t)(code | (active ? M_ACTIVE : 0) | (isnew ? M_NEW : 0));
        b.tlc[i] = (uint8_t)(code | (code << 4));
        b.cntc[i] = s_cnt[l];
        b.nbrc[i] = isnew ? make_double2(0.0, 0.0) : b.nbr[g];
        b.newb[i] = (int32_t)(nb0 + s_nwx[k]);   // s0 + active new nodes before i (new nodes are always active)
    }
}

// the state-independent half of round 1: per-(bin, CTA) record counts of a
// chunk's edges and their scan (the scatter's private cursors).  Depends only
// on the edges and the hub table, so the runtime computes it for chunk i+1 on
// a side stream while chunk i's rounds run.
void launch_bin_offsets(const uint2* e, int64_t m, const uint32_t* hub_keys, int shift, int nbins, int32_t* hist,
                        int32_t* offs, void* temp, size_t temp_bytes, cudaStream_t s) {
    const int G = binned_scatter_ctas();
    kmark(KM_BIN_HIST, 1, s);
    k_bin_hist<<<G, kScatT, 0, s>>>(e, m, hub_keys, shift, nbins, hist);
    kmark(KM_BIN_HIST, 0, s);
    exclusive_sum_i32(hist, offs, (int64_t)(nbins + 1) * G, temp, temp_bytes, s);
}

void launch_count_init_binned(const uint2* e, int64_t m, int64_t n, int refine, const ChunkBufs& b,
                              const BinBufs& bb, void* temp, size_t temp_bytes, cudaStream_t s, bool have_offs) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_bin_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kScatSmem);
        cudaFuncSetAttribute(k_bin_compact, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCmpSmem);
        attr = true;
    }
    int64_t ntiles = (n + kCmpSub - 1) >> kSubShift;
    const int G = binned_scatter_ctas();
    cudaMemsetAsync(bb.hub_cnt, 0, sizeof(unsigned long long) * kHubSlots, s);
    cudaMemsetAsync(bb.hub_flag, 0, sizeof(uint32_t) * kHubSlots, s);
    cudaMemsetAsync(bb.status, 0, sizeof(unsigned long long) * ntiles, s);
    cudaMemsetAsync(bb.ticket, 0, sizeof(unsigned int), s);
    if (!have_offs) launch_bin_offsets(e, m, b.hub_keys, bb.shift, bb.nbins, bb.hist, bb.offs, temp, temp_bytes, s);
    kmark(KM_BIN_SCATTER, 1, s);
    k_bin_scatter<<<G, kScatT, kScatSmem, s>>>(e, m, b.lab2, b.hub_keys, bb.shift, bb.nbins, bb.offs, bb.recs,
                                               bb.hub_cnt, bb.hub_flag);
    kmark(KM_BIN_SCATTER, 0, s);
    kmark(KM_BIN_COMPACT, 1, s);
    k_bin_compact<<<(unsigned)ntiles, kCmpT, kCmpSmem, s>>>(bb.recs, bb.offs, G, bb.shift, n, b.hub_keys,
                                                           bb.hub_cnt, bb.hub_flag, refine, b, bb.status,
                                                           bb.ticket, ntiles);
    kmark(KM_BIN_COMPACT, 0, s);
}
int binned_scatter_ctas() { return num_sms() * kScatPerSM; }
int64_t binned_hist_entries(int nbins) { return (int64_t)(nbins + 1) * binned_scatter_ctas(); }
int binned_shift(int64_t n) {
    int shift = kSubShift;
    while (((n + (1LL << shift) - 1) >> shift) > kMaxBins) ++shift;
    return shift;
}
int64_t binned_tiles(int64_t n) { return (n + kCmpSub - 1) >> kSubShift; }

// ============================================ expected-cut model (theory.py)
// expected_cuts (theory.py:125-142): per node with k >= 1, p = prob_correct
// (theory.py:78-94) = 1 - Pr(X <= t) for X ~ Hypergeom(k, k0, d), d = draws
// (theory.py:67-75), t = ceil(d/2) - 1, the tail summed term by term as
// exp(log C(k0, j) + log C(k - k0, d - j) - log C(k, d)) with log C from
// log-gamma (theory.py:35-63), same association order.  Log-gamma values
// come from a table lg[i] = lgamma(i), 0 <= i <= max k + 1.
namespace {
__device__ __forceinline__ double th_logc(const double* __restrict__ lg, int64_t n, int64_t r) {
    return lg[n + 1] - lg[r + 1] - lg[n - r + 1];
}
__device__ __forceinline__ int64_t th_draws(int64_t k, double x_eff) {
    int64_t d = (int64_t)rint(x_eff * (double)k);   // Python round(): half to even
    return d < 1 ? 1 : (d > k ? k : d);
}
constexpr int kThBig = 1024;   // tail terms above which a node goes to the block kernel
}  // namespace

__global__ void k_lgamma_table(double* lg, int64_t count) {
    GRID_STRIDE(i, count) lg[i] = lgamma((double)i);
}

// one thread per node: its expected cut endpoints into term[i]; nodes with a
// long tail are queued (big_list) and summed by k_theory_big
__global__ void k_theory_nodes(const int64_t* __restrict__ k, const int64_t* __restrict__ k0, int64_t n,
                               const double* __restrict__ lg, double x_eff, double* __restrict__ term,
                               int64_t* big_list, unsigned long long* big_count) {
    GRID_STRIDE(i, n) {
        int64_t ki = k[i], k0i = k0[i];
        double v = 0.0;
        if (ki >= 1) {
            int64_t d = th_draws(ki, x_eff);
            int64_t t = (d + 1) / 2 - 1;
            int64_t lo = d - (ki - k0i) > 0 ? d - (ki - k0i) : 0;
            int64_t hi = d < k0i ? d : k0i;
            int64_t top = t < hi ? t : hi;
            if (top - lo + 1 > kThBig) {
                big_list[atomicAdd(big_count, 1ULL)] = i;
                term[i] = 0.0;
                continue;
            }
            double ld = th_logc(lg, ki, d), cdf = 0.0;
            for (int64_t j = lo; j <= top; ++j) cdf += exp(th_logc(lg, k0i, j) + th_logc(lg, ki - k0i, d - j) - ld);
            double p = 1.0 - cdf;
            v = (double)(ki - k0i) * p + (double)k0i * (1.0 - p);
        }
        term[i] = v;
    }
}

// one block per queued node: the tail terms in parallel, reduced in a fixed order
__global__ void __launch_bounds__(256) k_theory_big(const int64_t* __restrict__ k, const int64_t* __restrict__ k0,
                                                    const double* __restrict__ lg, double x_eff,
                                                    const int64_t* __restrict__ big_list,
                                                    const unsigned long long* big_count, double* __restrict__ term) {
    __shared__ double sw[8];
    for (unsigned long long b = blockIdx.x; b < *big_count; b += gridDim.x) {
        int64_t i = big_list[b];
        int64_t ki = k[i], k0i = k0[i];
        int64_t d = th_draws(ki, x_eff);
        int64_t t = (d + 1) / 2 - 1;
        int64_t lo = d - (ki - k0i) > 0 ? d - (ki - k0i) : 0;
        int64_t hi = d < k0i ? d : k0i;
        int64_t top = t < hi ? t : hi;
        double ld = th_logc(lg, ki, d), s = 0.0;
        for (int64_t j = lo + threadIdx.x; j <= top; j += blockDim.x)
            s += exp(th_logc(lg, k0i, j) + th_logc(lg, ki - k0i, d - j) - ld);
        for (int off = 16; off; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
        if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
            double cdf = 0.0;
            for (int w = 0; w < 8; ++w) cdf += sw[w];
            double p = 1.0 - cdf;
            term[i] = (double)(ki - k0i) * p + (double)k0i * (1.0 - p);
        }
        __syncthreads();
    }
}

// deterministic sum: fixed per-block partials, then one block in block order
__global__ void __launch_bounds__(256) k_sum_f64_partial(const double* __restrict__ v, int64_t n, double* part) {
    __shared__ double sw[8];
    double s = 0.0;
    GRID_STRIDE(i, n) s += v[i];
    for (int off = 16; off; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
    if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double b = 0.0;
        for (int w = 0; w < 8; ++w) b += sw[w];
        part[blockIdx.x] = b;
    }
}
__global__ void k_sum_f64_final(const double* __restrict__ part, int np, double* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int b = 0; b < np; ++b) s += part[b];
        *out = s;
    }
}

int theory_sum_blocks() { return num_sms() * 4; }
void launch_lgamma_table(double* lg, int64_t count, cudaStream_t s) {
    k_lgamma_table<<<grid_for(count, 256), 256, 0, s>>>(lg, count);
}
void launch_expected_cuts(const int64_t* k, const int64_t* k0, int64_t n, const double* lg, double x_eff,
                          double* term, int64_t* big_list, unsigned long long* big_count, double* part,
                          double* out, cudaStream_t s) {
    cudaMemsetAsync(big_count, 0, sizeof(unsigned long long), s);
    k_theory_nodes<<<grid_for(n, 256), 256, 0, s>>>(k, k0, n, lg, x_eff, term, big_list, big_count);
    k_theory_big<<<num_sms() * 8, 256, 0, s>>>(k, k0, lg, x_eff, big_list, big_count, term);
    int nb = theory_sum_blocks();
    k_sum_f64_partial<<<nb, 256, 0, s>>>(term, n, part);
    k_sum_f64_final<<<1, 32, 0, s>>>(part, nb, out);
}

}  // namespace grem

namespace grem {
// validation and totals for expected_cuts: out[0] = first node with k >= 1,
// out[1] = first such node whose k0 is not its majority side (theory.py:87-88),
// out[2] = max k, out[3] = sum of k (total endpoints); indices as min, -1 = none
__global__ void k_theory_check(const int64_t* __restrict__ k, const int64_t* __restrict__ k0, int64_t n,
                               unsigned long long* out) {
    unsigned long long first = ~0ULL, bad = ~0ULL, mx = 0, sum = 0;
    GRID_STRIDE(i, n) {
        int64_t ki = k[i], k0i = k0[i];
        sum += (unsigned long long)ki;
        if (ki >= 1) {
            if ((unsigned long long)i < first) first = (unsigned long long)i;
            if ((k0i < 0 || k0i > ki || 2 * k0i < ki) && (unsigned long long)i < bad) bad = (unsigned long long)i;
            if ((unsigned long long)ki > mx) mx = (unsigned long long)ki;
        }
    }
    for (int off = 16; off; off >>= 1) {
        first = min(first, __shfl_down_sync(0xffffffffu, first, off));
        bad = min(bad, __shfl_down_sync(0xffffffffu, bad, off));
        mx = max(mx, __shfl_down_sync(0xffffffffu, mx, off));
        sum += __shfl_down_sync(0xffffffffu, sum, off);
    }
    if ((threadIdx.x & 31) == 0) {
        if (first != ~0ULL) atomicMin(out + 0, first);
        if (bad != ~0ULL) atomicMin(out + 1, bad);
        if (mx) atomicMax(out + 2, mx);
        if (sum) atomicAdd(out + 3, sum);
    }
}
void launch_theory_check(const int64_t* k, const int64_t* k0, int64_t n, unsigned long long* out, cudaStream_t s) {
    k_theory_check<<<grid_for(n, 256), 256, 0, s>>>(k, k0, n, out);
}
}  // namespace grem
