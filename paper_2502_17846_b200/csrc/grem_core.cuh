// grem_core.cuh — device-side building blocks shared by the GREM kernels.
//
// Layout in HBM for one bisection over n nodes:
//   lab  int8[n]      committed labels (-1 / 0 / 1)            PartitionState.parts
//   nbr  double2[n]   running estimates (nbr0, nbr1), fp64      PartitionState.nbr0/1
//   cnt  u64[n]       per-chunk neighbour counts (c0 | c1<<32), zero between chunks
//   tl   u8[n]        tentative label codes of the fixpoint rounds (cur | prev<<4)
//   flag u8[n]       chunk-membership marks for nodes whose counts stay zero
// and per chunk (N_c nodes, ascending ids): nodes u32, meta u8, newb i32, x i32.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace grem {

constexpr long long kInf = 1LL << 60;

// A node's effect on x = sizes[0] is a clamp x -> min(max(x + d, L), U) on the
// feasible domain (note after the table).  Clamps
// compose in O(1): first a then b.
struct Clamp {
    long long d, L, U;
};

__host__ __device__ __forceinline__ long long clampv(long long v, long long lo, long long hi) {
    return v < lo ? lo : (v > hi ? hi : v);
}
__host__ __device__ __forceinline__ Clamp clamp_identity() { return Clamp{0, -kInf, kInf}; }
__host__ __device__ __forceinline__ Clamp clamp_then(const Clamp& a, const Clamp& b) {
    Clamp r;
    r.d = a.d + b.d;
    r.L = clampv(a.L + b.d, b.L, b.U);
    r.U = clampv(a.U + b.d, b.L, b.U);
    return r;
}
__host__ __device__ __forceinline__ long long clamp_apply(const Clamp& f, long long x) {
    return clampv(x + f.d, f.L, f.U);
}

// meta byte of a chunk node
//   bits 0-1 old label code (0: -1, 1: label 0, 2: label 1)
//   bit 2    active (visited by the sweep: new, or refine on)
//   bit 3    new (old == -1)
//   bits 4-5 preference (0: side 0, 1: side 1, 2: tie)
//   bit 6    speculated side of a tie (0/1)
constexpr uint8_t M_OLD = 0x3, M_ACTIVE = 0x4, M_NEW = 0x8, M_PREF_SHIFT = 4, M_PREF = 0x30, M_SPEC = 0x40;

__host__ __device__ __forceinline__ int meta_old(uint8_t m) { return (int)(m & M_OLD) - 1; }
__host__ __device__ __forceinline__ bool meta_active(uint8_t m) { return m & M_ACTIVE; }
__host__ __device__ __forceinline__ int meta_pref(uint8_t m) { return (m & M_PREF) >> M_PREF_SHIFT; }

// Per-node map of process_chunk (grem.py:134-154): lift-out then assign
// (grem.py:100-116).  s_l = total assigned after the lift-out (independent of
// the decisions).  Decision b = 0 iff x - o <= t.
struct NodeMap {
    Clamp f;
    long long o, t;
};

__host__ __device__ __forceinline__ NodeMap node_map(uint8_t m, long long s_l, long long cap) {
    NodeMap r;
    if (!meta_active(m)) {
        r.f = clamp_identity();
        r.o = 0;
        r.t = kInf;
        return r;
    }
    long long o = (meta_old(m) == 0) ? 1 : 0;
    r.o = o;
    int pref = meta_pref(m);
    if (pref == 0) {          // wants side 0: b=0 iff side 0 has room
        r.f = Clamp{1 - o, -kInf, cap};
        r.t = cap - 1;
    } else if (pref == 1) {   // wants side 1: b=0 iff side 1 is full
        r.f = Clamp{-o, s_l - cap + 1, kInf};
        r.t = s_l - cap;
    } else {
        // tie: smaller side, ties to 0.  The exact map x -> x - o + [x - o <= t]
        // is not a clamp; it is speculated as the clamp of the guessed side,
        // which is exact on a one-step-wider region and, like the true map,
        // absorbs a +-1 shift of x at the threshold (so a trajectory perturbed
        // upstream re-merges instead of mis-speculating every later tie):
        //   guess 0: min(x + 1 - o, t + 1), exact iff x - o <= t + 1
        //   guess 1: max(x - o, t + 1),     exact iff x - o >= t
        r.t = s_l >> 1;
        if (m & M_SPEC) r.f = Clamp{-o, r.t + 1, kInf};
        else r.f = Clamp{1 - o, -kInf, r.t + 1};
    }
    return r;
}
// the speculated clamp of a tie was not exact at input x (repair needed)
__host__ __device__ __forceinline__ bool tie_misspeculated(uint8_t m, long long x, const NodeMap& nm) {
    return (m & M_SPEC) ? (x - nm.o < nm.t) : (x - nm.o > nm.t + 1);
}

__device__ __forceinline__ unsigned long long enc_label(int code) {
    // label code (0: -1, 1: label 0, 2: label 1) -> packed counter increment
    return code == 1 ? 1ULL : (code == 2 ? (1ULL << 32) : 0ULL);
}

}  // namespace grem
