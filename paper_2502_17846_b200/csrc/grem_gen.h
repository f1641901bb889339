/*
 * grem_gen.h — deterministic Chung-Lu power-law edge generator, bit-identical
 * on the host (gcc, -ffp-contract=off) and on the device (nvcc, explicit
 * __dmul_rn/__dadd_rn so no FMA contraction can change a rounding).
 *
 * The reference ships no power-law generator (streamcut/synth.py:101-115 has
 * SBM, clique-union, path and star only; power-law is a declared non-goal,
 * SPEC.md:542), so the benchmark shapes of BASELINE.json need one that both the
 * CPU oracle and the GPU path can reproduce exactly without moving a 13 GB file.
 *
 * Model: endpoint weights w_i ∝ (i+1)^(-alpha),
 * alpha = 1/(gamma-1).  Each endpoint is an independent draw: a 64-bit
 * counter hash gives u in [0,1); the continuous inverse CDF on [1, n+1] is
 *     x = (1 + u * ((n+1)^(1/beta) - 1))^beta,   beta = 1/(1-alpha),
 * evaluated with beta an integer (gamma = 2.1 -> beta = 11;
 * gamma = 7/3 ~ 2.33 -> beta = 4), so only correctly-rounded IEEE ops are
 * used.  node = floor(x) - 1.  Ids are then scrambled by a keyed bijection of
 * [0, n) (xorshift-multiply permutation on the next power of two + cycle
 * walking), so hubs land on random ids.  Edges are i.i.d. draws, hence
 * already in random order (the "random order on disk" precondition,
 * PAPER.md:162), and naturally contain duplicates and self-loops.
 */
#ifndef GREM_GEN_H
#define GREM_GEN_H

#include <stdint.h>

#if defined(__CUDACC__)
#define GG_HD __host__ __device__ __forceinline__
#define GG_H __host__ inline
#else
#define GG_HD static inline
#define GG_H static inline
#endif

typedef struct {
    uint64_t n;        /* nodes */
    uint64_t seed;     /* graph seed */
    uint64_t perm_mask;/* next_pow2(n) - 1 */
    uint32_t perm_bits;
    uint32_t beta;     /* integer exponent */
    double   scale;    /* (n+1)^(1/beta) - 1, computed by gg_root_scale */
} gg_params;

GG_HD uint64_t gg_mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

#if defined(__CUDA_ARCH__)
#define GG_MUL(a, b) __dmul_rn((a), (b))
#define GG_ADD(a, b) __dadd_rn((a), (b))
#else
#define GG_MUL(a, b) ((a) * (b))
#define GG_ADD(a, b) ((a) + (b))
#endif

GG_HD double gg_ipow(double v, uint32_t beta) {
    /* fixed left-to-right binary exponentiation: the op sequence depends only
     * on beta, so host and device round identically */
    double r = 1.0;
    for (int bit = 31; bit >= 0; --bit) {
        r = GG_MUL(r, r);
        if ((beta >> bit) & 1u) r = GG_MUL(r, v);
    }
    return r;
}

/* keyed bijection of [0, 2^bits): every step is invertible mod 2^bits */
GG_HD uint64_t gg_perm_step(uint64_t x, uint64_t key, uint32_t bits, uint64_t mask) {
    uint32_t sh = bits / 2 + 1;
    x = (x ^ key) & mask;
    x = (x * 0xD6E8FEB86659FD93ULL) & mask;
    x ^= x >> sh;
    x = (x * 0x9E3779B97F4A7C15ULL + (key | 1ULL)) & mask;
    x ^= x >> sh;
    x = (x * 0xBF58476D1CE4E5B9ULL) & mask;
    x ^= x >> (sh > 2 ? sh - 1 : 1);
    return x & mask;
}

GG_HD uint64_t gg_permute(const gg_params* p, uint64_t x) {
    uint64_t k0 = gg_mix64(p->seed ^ 0x5DEECE66DULL);
    uint64_t k1 = gg_mix64(k0);
    do {   /* cycle walking: stays inside [0, n) */
        x = gg_perm_step(x, k0, p->perm_bits, p->perm_mask);
        x = gg_perm_step(x, k1, p->perm_bits, p->perm_mask);
    } while (x >= p->n);
    return x;
}

/* endpoint j (edge e has endpoints 2e and 2e+1) -> node id in [0, n) */
GG_HD uint32_t gg_endpoint(const gg_params* p, uint64_t j) {
    uint64_t h = gg_mix64(gg_mix64(p->seed) ^ j);
    double u = (double)(h >> 11) * (1.0 / 9007199254740992.0); /* exact: 2^-53 */
    double v = GG_ADD(1.0, GG_MUL(u, p->scale));
    double x = gg_ipow(v, p->beta);
    uint64_t raw = (uint64_t)x;           /* floor, x >= 1 */
    raw = raw >= 1 ? raw - 1 : 0;
    if (raw >= p->n) raw = p->n - 1;
    return (uint32_t)gg_permute(p, raw);
}

/* (n+1)^(1/beta) - 1 by a fixed bisection in plain IEEE ops (no libm),
 * so every host computes the same double. */
GG_H double gg_root_scale(uint64_t n, uint32_t beta) {
    double a = (double)(n + 1);
    double r = 1.0;
    while (gg_ipow(r * 2.0, beta) <= a) r = r * 2.0;   /* bracket */
    double lo = r, hi = r * 2.0;
    for (int it = 0; it < 200; ++it) {                 /* bisection: exact, fixed */
        double mid = (lo + hi) * 0.5;
        if (mid == lo || mid == hi) break;
        if (gg_ipow(mid, beta) <= a) lo = mid; else hi = mid;
    }
    return lo - 1.0;
}

GG_H void gg_init(gg_params* p, uint64_t n, uint32_t beta, uint64_t seed) {
    p->n = n;
    p->seed = seed;
    p->beta = beta;
    uint32_t bits = 1;
    while ((1ULL << bits) < n) ++bits;
    p->perm_bits = bits;
    p->perm_mask = (1ULL << bits) - 1ULL;
    p->scale = gg_root_scale(n, beta);
}

#endif /* GREM_GEN_H */
