// grem_store.cu — the partitioned storage layout on the GPU:
// write_buckets (streamcut/store.py:55-104), a stable p x p scatter of the
// edge list by (label[src], label[dst]), and the partition-grouping
// permutation of reorder_features (store.py:201-235).
//
// Buckets: key = label[u] * p + label[v] per edge (one pass: edge read + two
// label gathers), then one stable LSD radix sort of (key, edge) pairs over
// ceil(log2 p^2) bits (stable: input order inside a bucket, store.py:92), and
// the bucket extents by binary search of the sorted keys.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "grem_kernels.cuh"

namespace grem {

__global__ void k_label_max(const int32_t* __restrict__ lab, int64_t n, int* mx) {   // mx[1]: some label < 0
    int m = -1, neg = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        m = lab[i] > m ? lab[i] : m;
        neg |= lab[i] < 0;
    }
    if (__any_sync(0xffffffffu, neg) && (threadIdx.x & 31) == 0) atomicOr(mx + 1, 1);
    for (int off = 16; off; off >>= 1) {
        int o = __shfl_down_sync(0xffffffffu, m, off);
        m = o > m ? o : m;
    }
    if ((threadIdx.x & 31) == 0 && m >= 0) atomicMax(mx, m);
}

__global__ void k_bucket_keys(const uint2* __restrict__ e, int64_t m, const int32_t* __restrict__ lab, uint32_t p,
                              uint32_t* __restrict__ keys, int* bad) {
    int b = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        uint2 ed = e[i];
        int lu = lab[ed.x], lv = lab[ed.y];
        if (lu < 0 || lv < 0) {   // store.py:77-78
            b = 1;
            keys[i] = 0;
            continue;
        }
        keys[i] = (uint32_t)lu * p + (uint32_t)lv;
    }
    if (__any_sync(0xffffffffu, b) && (threadIdx.x & 31) == 0) atomicOr(bad, 1);
}

// all labels >= 0: labels packed to 2^lb bits (L2-resident for small p), so
// the two gathers per edge hit L2 instead of the int32 array in HBM
__global__ void k_pack_lab(const int32_t* __restrict__ lab, int64_t n, int lb, uint32_t* __restrict__ out,
                           int64_t nwords) {
    const int per = 32 >> lb, width = 1 << lb;
    const uint32_t mask = width == 32 ? 0xFFFFFFFFu : ((1u << width) - 1);
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nwords; w += (int64_t)gridDim.x * blockDim.x) {
        uint32_t v = 0;
        for (int j = 0; j < per; ++j) {
            int64_t i = w * per + j;
            if (i < n) v |= ((uint32_t)lab[i] & mask) << (j * width);
        }
        out[w] = v;
    }
}
__global__ void k_bucket_keys_packed(const uint2* __restrict__ e, int64_t m, const uint32_t* __restrict__ pl,
                                     int lb, uint32_t p, uint32_t* __restrict__ keys) {
    const int lpw = 5 - lb;
    const uint32_t mask = lb == 5 ? 0xFFFFFFFFu : ((1u << (1 << lb)) - 1);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        uint2 ed = __ldcs(e + i);
        uint32_t lu = (__ldg(pl + (ed.x >> lpw)) >> ((ed.x & ((1u << lpw) - 1)) << lb)) & mask;
        uint32_t lv = (__ldg(pl + (ed.y >> lpw)) >> ((ed.y & ((1u << lpw) - 1)) << lb)) & mask;
        keys[i] = lu * p + lv;
    }
}

// counts[b] = upper_bound(b) - lower_bound(b) in the sorted keys
__global__ void k_bucket_counts(const uint32_t* __restrict__ skeys, int64_t m, int64_t nb,
                                unsigned long long* __restrict__ counts) {
    int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= nb) return;
    auto lower = [&](uint64_t key) {
        int64_t lo = 0, hi = m;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if ((uint64_t)skeys[mid] < key) lo = mid + 1;
            else hi = mid;
        }
        return lo;
    };
    counts[b] = (unsigned long long)(lower((uint64_t)b + 1) - lower((uint64_t)b));
}

size_t bucket_sort_temp_bytes(int64_t m) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (const unsigned long long*)nullptr, (unsigned long long*)nullptr, m);   // 64-bit item count
    return bytes;
}

// compute_node_stats (streamcut/theory.py:97-122): per node, the non-self-loop
// neighbour endpoints on side 0 / side 1 of a bisection, with multiplicity.
// One pass over the edges: two label gathers and two 64-bit REDs per edge
// into the node's (side 0, side 1) counter pair; then k = c0 + c1, k0 = max.
__global__ void k_node_side_counts(const uint2* __restrict__ e, int64_t m, const int32_t* __restrict__ lab,
                                   unsigned long long* __restrict__ cnt, int* bad) {
    int b = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        uint2 ed = __ldcs(e + i);
        if (ed.x == ed.y) continue;   // theory.py:111
        int lu = __ldg(lab + ed.x), lv = __ldg(lab + ed.y);
        if (lu < 0 || lv < 0) {       // theory.py:114-115
            b = 1;
            continue;
        }
        atomicAdd(cnt + 2 * (uint64_t)ed.x + lv, 1ull);
        atomicAdd(cnt + 2 * (uint64_t)ed.y + lu, 1ull);
    }
    if (__any_sync(0xffffffffu, b) && (threadIdx.x & 31) == 0) atomicOr(bad, 1);
}

// Packed form for m < 2^32 (a node's per-side count is <= m): labels as 2-bit
// codes (0, 1, 2 = unlabeled; n/4 bytes, L2-resident) and ONE u64 counter per
// node holding side 0 in the low and side 1 in the high 32 bits, so each
// endpoint is one RED into an 8-byte word (half the counter footprint).
__global__ void k_pack_labels2(const int32_t* __restrict__ lab, int64_t n, uint32_t* __restrict__ packed) {
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < (n + 15) / 16;
         w += (int64_t)gridDim.x * blockDim.x) {
        uint32_t word = 0;
        int64_t base = w * 16;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            int64_t i = base + j;
            uint32_t code = 2;
            if (i < n) {
                int l = __ldcs(lab + i);
                code = l < 0 ? 2u : (uint32_t)(l & 1);
            }
            word |= code << (2 * j);
        }
        packed[w] = word;
    }
}

__global__ void k_node_side_counts_packed(const uint2* __restrict__ e, int64_t m, const uint32_t* __restrict__ packed,
                                          unsigned long long* __restrict__ cnt, int* bad) {
    int b = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        uint2 ed = __ldcs(e + i);
        if (ed.x == ed.y) continue;   // theory.py:111
        uint32_t lu = (__ldg(packed + (ed.x >> 4)) >> (2 * (ed.x & 15))) & 3u;
        uint32_t lv = (__ldg(packed + (ed.y >> 4)) >> (2 * (ed.y & 15))) & 3u;
        if ((lu | lv) & 2u) {         // theory.py:114-115
            b = 1;
            continue;
        }
        atomicAdd(cnt + ed.x, 1ull << (32 * lv));
        atomicAdd(cnt + ed.y, 1ull << (32 * lu));
    }
    if (__any_sync(0xffffffffu, b) && (threadIdx.x & 31) == 0) atomicOr(bad, 1);
}

__global__ void k_node_stats_final_packed(const unsigned long long* __restrict__ cnt, int64_t n,
                                          int64_t* __restrict__ k, int64_t* __restrict__ k0) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long c = cnt[i];
        int64_t c0 = (int64_t)(c & 0xffffffffull), c1 = (int64_t)(c >> 32);
        k[i] = c0 + c1;
        k0[i] = c0 > c1 ? c0 : c1;
    }
}

__global__ void k_node_stats_final(const ulonglong2* __restrict__ cnt, int64_t n, int64_t* __restrict__ k,
                                   int64_t* __restrict__ k0) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        ulonglong2 c = cnt[i];
        k[i] = (int64_t)(c.x + c.y);
        k0[i] = (int64_t)(c.x > c.y ? c.x : c.y);
    }
}

// cnt: 2n u64 (the unpacked fallback needs all of it); packed: n/16 + 1 u32
void launch_node_stats(const uint2* e, int64_t m, const int32_t* lab, int64_t n, unsigned long long* cnt,
                       uint32_t* packed, int64_t* k, int64_t* k0, int* bad, cudaStream_t s,
                       const uint32_t* hub_keys) {
    cudaMemsetAsync(bad, 0, sizeof(int), s);
    int cap = num_sms() * 8;
    auto grid_for = [&](int64_t work) {
        int64_t g = (work + 255) / 256;
        return (int)(g > cap ? cap : (g < 1 ? 1 : g));
    };
    static const bool unpacked = getenv("GREM_NODE_STATS_UNPACKED") != nullptr;   // A/B switch
    if (m < (1LL << 32) && !unpacked) {
        cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * n, s);
        k_pack_labels2<<<grid_for((n + 15) / 16), 256, 0, s>>>(lab, n, packed);
        if (hub_keys) launch_node_side_counts_hub(e, m, packed, hub_keys, cnt, bad, s);
        else if (m > 0) k_node_side_counts_packed<<<grid_for(m), 256, 0, s>>>(e, m, packed, cnt, bad);
        k_node_stats_final_packed<<<grid_for(n), 256, 0, s>>>(cnt, n, k, k0);
        return;
    }
    cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * 2 * n, s);
    if (m > 0) k_node_side_counts<<<grid_for(m), 256, 0, s>>>(e, m, lab, cnt, bad);
    k_node_stats_final<<<grid_for(n), 256, 0, s>>>(reinterpret_cast<const ulonglong2*>(cnt), n, k, k0);
}

// external_shuffle (streamcut/edgefile.py:248-327): a uniform random
// permutation of the edge list.  Each edge gets a 64-bit key from a
// counter-based hash of (seed, position) and one radix sort of (key, edge)
// pairs puts the edges in key order: every permutation is equally likely up
// to 64-bit key ties (stable: input order), deterministic per seed.  The
// reference's order comes from numpy's PCG64 Generator and is not
// reproduced (parity is by multiset, determinism and uniformity).
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void k_shuffle_keys(const uint2* __restrict__ e, int64_t m, unsigned long long seed,
                               unsigned long long* __restrict__ keys, unsigned long long* __restrict__ vals) {
    const unsigned long long sk = mix64(seed + 0x9E3779B97F4A7C15ull);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        uint2 ed = __ldcs(e + i);
        keys[i] = mix64(sk ^ mix64((unsigned long long)i));
        vals[i] = ((unsigned long long)ed.y << 32) | ed.x;
    }
}

size_t shuffle_temp_bytes(int64_t m) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                    (const unsigned long long*)nullptr, (unsigned long long*)nullptr, m);
    return bytes;
}

// keys/vals: 2 x m u64 each (ping-pong); the shuffled edges land in vals + m
void launch_shuffle(const uint2* e, int64_t m, unsigned long long seed, unsigned long long* keys,
                    unsigned long long* vals, void* temp, size_t temp_bytes, cudaStream_t s) {
    if (m <= 0) return;
    int cap = num_sms() * 8;
    int64_t g = (m + 255) / 256;
    k_shuffle_keys<<<(int)(g < cap ? g : cap), 256, 0, s>>>(e, m, seed, keys, vals);
    cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys, keys + m, vals, vals + m, m, 0, 64, s);
}

void launch_label_max(const int32_t* lab, int64_t n, int* d_max, cudaStream_t s) {
    cudaMemsetAsync(d_max, 0xFF, sizeof(int), s);
    cudaMemsetAsync(d_max + 1, 0, sizeof(int), s);
    int grid = (int)((n + 255) / 256);
    if (grid > num_sms() * 8) grid = num_sms() * 8;
    if (grid < 1) grid = 1;
    k_label_max<<<grid, 256, 0, s>>>(lab, n, d_max);
}

void launch_write_buckets(const uint2* e, int64_t m, const int32_t* lab, int64_t n, bool any_unlabeled, uint32_t p,
                          uint32_t* keys_a, uint32_t* keys_b, uint32_t* packed, uint2* out,
                          unsigned long long* counts, int* d_bad, void* temp, size_t temp_bytes, cudaStream_t s) {
    cudaMemsetAsync(d_bad, 0, sizeof(int), s);
    int64_t nb = (int64_t)p * p;
    if (m > 0) {
        int grid = (int)((m + 255) / 256);
        if (grid > num_sms() * 16) grid = num_sms() * 16;
        if (!any_unlabeled && packed) {
            int lb = 0;
            while (lb < 5 && ((uint64_t)(p - 1) >> (1 << lb)) != 0) ++lb;
            int64_t nwords = (n + (32 >> lb) - 1) / (32 >> lb);
            int pg = (int)((nwords + 255) / 256);
            if (pg > num_sms() * 16) pg = num_sms() * 16;
            k_pack_lab<<<pg < 1 ? 1 : pg, 256, 0, s>>>(lab, n, lb, packed, nwords);
            k_bucket_keys_packed<<<grid, 256, 0, s>>>(e, m, packed, lb, p, keys_a);
        } else {
            k_bucket_keys<<<grid, 256, 0, s>>>(e, m, lab, p, keys_a, d_bad);
        }
        int end_bit = 1;
        while (end_bit < 32 && ((uint64_t)(nb - 1) >> end_bit) != 0) ++end_bit;
        cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_a, keys_b,
                                        reinterpret_cast<const unsigned long long*>(e),
                                        reinterpret_cast<unsigned long long*>(out), m, 0, end_bit, s);
        k_bucket_counts<<<(unsigned)((nb + 255) / 256), 256, 0, s>>>(keys_b, m, nb, counts);
    } else {
        cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * nb, s);
    }
}

// reorder_features: stable order of nodes by label (ties by node id,
// store.py:221), its inverse (node -> slot) and the per-partition extents
__global__ void k_iota_u32n(uint32_t* a, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = (uint32_t)i;
}
__global__ void k_perm_inverse(const uint32_t* __restrict__ order, int64_t n, long long* __restrict__ perm) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        perm[order[i]] = i;
}
__global__ void k_gather_records(const uint8_t* __restrict__ rec, const uint32_t* __restrict__ order, int64_t n,
                                 int64_t width, uint8_t* __restrict__ out) {
    // one warp per output record, byte-striped (records are small, arbitrary width)
    int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (; w < n; w += nw) {
        const uint8_t* src = rec + (int64_t)order[w] * width;
        uint8_t* dst = out + w * width;
        for (int64_t k = lane; k < width; k += 32) dst[k] = src[k];
    }
}

size_t order_sort_temp_bytes(int64_t n) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (const uint32_t*)nullptr, (uint32_t*)nullptr, n);
    return bytes;
}

void launch_reorder(const int32_t* lab, int64_t n, uint32_t p, uint32_t* keys_b, uint32_t* ids_a, uint32_t* order,
                    long long* perm, unsigned long long* counts, const uint8_t* rec, int64_t width, uint8_t* out,
                    void* temp, size_t temp_bytes, cudaStream_t s) {
    int grid = (int)((n + 255) / 256);
    if (grid > num_sms() * 16) grid = num_sms() * 16;
    if (grid < 1) grid = 1;
    k_iota_u32n<<<grid, 256, 0, s>>>(ids_a, n);
    int end_bit = 1;
    while (end_bit < 32 && ((uint64_t)p >> end_bit) != 0) ++end_bit;
    cub::DeviceRadixSort::SortPairs(temp, temp_bytes, reinterpret_cast<const uint32_t*>(lab), keys_b, ids_a, order,
                                    n, 0, end_bit, s);
    k_perm_inverse<<<grid, 256, 0, s>>>(order, n, perm);
    k_bucket_counts<<<(unsigned)((p + 255) / 256), 256, 0, s>>>(keys_b, n, p, counts);
    if (rec && out && width > 0) {
        int64_t g = (n * 32 + 255) / 256;
        if (g > num_sms() * 16) g = num_sms() * 16;
        k_gather_records<<<(unsigned)(g < 1 ? 1 : g), 256, 0, s>>>(rec, order, n, width, out);
    }
}

}  // namespace grem
