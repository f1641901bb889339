// grem_host.cpp — host-side pieces of libgrem_b200.so that need no GPU:
// the deterministic power-law generator (bit-identical to the device one,
// grem_gen.h) and GRPE file helpers used by the chunk-ingest path.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include "grem_gen.h"
#include "../../include/grem_b200.h"

extern "C" double grem_gen_scale(uint64_t n, uint32_t beta) { return gg_root_scale(n, beta); }

extern "C" int grem_gen_edges_host(uint64_t n, uint32_t beta, uint64_t seed, uint64_t e0, uint64_t count,
                                   uint32_t* out, int threads) {
    if (n < 1 || beta < 1 || !out) return GREM_E_FORMAT;
    gg_params p;
    gg_init(&p, n, beta, seed);
    if (threads <= 0) threads = (int)std::thread::hardware_concurrency();
    if (threads < 1) threads = 1;
    if ((uint64_t)threads > count / 65536 + 1) threads = (int)(count / 65536 + 1);
    auto work = [&](uint64_t lo, uint64_t hi) {
        for (uint64_t e = lo; e < hi; ++e) {
            uint64_t j = 2 * (e0 + e);
            out[2 * e] = gg_endpoint(&p, j);
            out[2 * e + 1] = gg_endpoint(&p, j + 1);
        }
    };
    std::vector<std::thread> ts;
    uint64_t per = (count + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        uint64_t lo = t * per, hi = lo + per < count ? lo + per : count;
        if (lo >= hi) break;
        ts.emplace_back(work, lo, hi);
    }
    for (auto& t : ts) t.join();
    return GREM_OK;
}
