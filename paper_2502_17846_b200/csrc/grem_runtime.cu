// grem_runtime.cu — host orchestration and the C ABI of libgrem_b200.so.
//
// Mirrors the reference drivers (paths relative to pkg/src/streamcut/):
//   bisect        grem.py:192-224   chunk loop, seed on pass 0 chunk 0, fill
//   partition     grem.py:277-319   recursive bisection over induced subgraphs
//   count_cuts    grem.py:227-252
//   ingest        edgefile.py:107-126,186-219,371-465 (GRPE u32 -> HBM through
//                 two pinned chunk buffers; ResidencyMeter schedule)
// All edge data stays resident in HBM for the whole call; per-node state is
// O(n) device arrays (grem_core.cuh).  The host only reads a handful of
// scalars per chunk round (N_c, labels changed).
#include <cuda.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <mutex>
#include <condition_variable>
#include <fcntl.h>
#include <unistd.h>
#include <functional>
#include <thread>
#include <atomic>
#include <cstring>
#include <new>
#include <utility>
#include <string>
#include <vector>

#include "../../include/grem_b200.h"
#include "grem_core.cuh"
#include "grem_gen.h"
#include "grem_kernels.cuh"

using namespace grem;

namespace {

thread_local std::string g_err;

struct GremError {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw GremError{code, msg}; }

#define CK(call)                                                                          \
    do {                                                                                  \
        cudaError_t _e = (call);                                                          \
        if (_e != cudaSuccess)                                                            \
            fail(GREM_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e));        \
    } while (0)

template <class T>
struct DBuf {
    const char* name = "";
    T* p = nullptr;
    size_t cap = 0;   // elements
    DBuf() = default;
    explicit DBuf(const char* nm) : name(nm) {}
    // stream-ordered growth from the device memory pool: no device-wide
    // synchronisation, so concurrent sibling contexts never stall each other
    void ensure(size_t n, cudaStream_t s) {
        if (n <= cap) return;
        if (p) CK(cudaFreeAsync(p, s));
        p = nullptr;
        size_t c = n + n / 8 + 64;
        CK(cudaMallocAsync((void**)&p, c * sizeof(T), s));
        cap = c;
        // debug: GREM_DEBUG_POISON=all|name,name fills new buffers with 0xA5 to
        // expose reads of memory that was never written in this call
        static const char* poison = getenv("GREM_DEBUG_POISON");
        if (poison && (strcmp(poison, "all") == 0 || strstr(poison, (std::string(",") + name + ",").c_str())))
            CK(cudaMemsetAsync(p, 0xA5, c * sizeof(T), s));
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    void release_async(cudaStream_t s) {   // stream-ordered: no device-wide synchronisation
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        cap = 0;
    }
};

}  // namespace

// Phase profiler: CUDA events around launch groups on the context stream
// (enabled per call by grem_set_profiling); elapsed times are folded in after
// the call's final synchronisation.
enum Phase {
    PH_COUNT = 0, PH_SELECT, PH_NODE, PH_DELTA, PH_SCAN, PH_BUNDLE, PH_COMMIT,
    PH_SEED, PH_FILL, PH_EXTRACT, PH_CUTS, PH_INGEST, PH_HUBS,
    PH_SEED_CSR, PH_SEED_CC, PH_SEED_BFS, PH_SEED_REFINE, PH_SEED_COMMIT,   // inside "seed"
    PH_K0,   // kernel-level marks (grem_set_profiling(ctx, 2)): PH_K0 + KM_*
    PH_N = PH_K0 + KM_N
};
static const char* kPhaseNames[PH_N] = {"count_init", "select", "node_init", "count_delta", "scan", "bundle",
                                        "commit", "seed", "fill", "extract", "count_cuts", "ingest", "hubs",
                                        "seed.csr", "seed.cc", "seed.bfs", "seed.refine", "seed.commit",
                                        "k.bin_hist", "k.bin_scatter", "k.bin_compact", "k.round_reduce_full",
                                        "k.round_down_full", "k.count_delta", "k.round_reduce", "k.round_down"};

struct grem_ctx {
    int device = 0;
    int profiling = 0;
    // sibling subtrees of partition() run concurrently on child contexts
    // (own stream, workspaces, host thread); the root owns the pool
    grem_ctx* root = nullptr;
    std::mutex pool_mu;
    std::vector<grem_ctx*> pool_all, pool_idle;
    bool busy = false;   // child context: a subtree is running on it (guarded by the root's pool_mu)
    int64_t ws_m = 0;    // child context: edges of the largest subtree its workspaces were sized for
    std::vector<std::pair<long long, grem_ctx*>> pool_keyed;   // subtree position -> context
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> prof_open;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    double phase_ms[PH_N] = {0};
    long long phase_n[PH_N] = {0};
    double phase_bytes[PH_N] = {0};   // algorithmic bytes of the kernel phases
    cudaEvent_t kmark_open[KM_N] = {};
    cudaStream_t s = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // per node
    DBuf<int8_t> lab{"lab"};
    DBuf<uint32_t> lab2{"lab2"}, bin_recs{"bin_recs"};
    DBuf<unsigned int> bin_ticket{"bin_ticket"};
    DBuf<int32_t> bin_hist{"bin_hist"}, bin_offs{"bin_offs"};
    DBuf<unsigned long long> bin_hcnt{"bin_hcnt"}, bin_status{"bin_status"};
    DBuf<uint32_t> bin_hflag{"bin_hflag"};
    DBuf<uint8_t> tl{"tl"}, flag{"flag"};
    DBuf<unsigned long long> cnt{"cnt"};
    DBuf<double2> nbr{"nbr"};
    DBuf<int32_t> rank{"rank"}, scratch{"scratch"}, newid{"newid"};
    DBuf<uint2> rankw{"rankw"};   // chunk-0 succinct rank words {bits, members before}
    // per chunk node
    DBuf<uint32_t> nodes{"nodes"};
    DBuf<uint8_t> meta{"meta"}, bad{"bad"}, want{"want"};
    DBuf<unsigned long long> cntc{"cntc"};
    DBuf<double2> nbrc{"nbrc"};
    DBuf<uint8_t> tlc{"tlc"};
    DBuf<uint32_t> chg{"chg"}, chgc{"chgc"}, chg2{"chg2"}, chgc2{"chgc2"};
    cudaGraphExec_t round_exec = nullptr;   // replayed pair of rounds (process_chunk)
    cudaGraphExec_t loop_exec = nullptr;    // device-side round loop (conditional WHILE node)
    // root context: its stream on the dense SM partition (green context) and
    // the full-GPU stream it started on (see green_parts / recurse)
    cudaStream_t s_full = nullptr, s_dense = nullptr;
    DBuf<uint8_t> dirty0{"dirty0"}, dirty1{"dirty1"};
    DBuf<int32_t> newb{"newb"}, x{"x"}, xalt{"xalt"}, xnext{"xnext"}, bends{"bends"}, bxin{"bxin"}, bhit{"bhit"}, bparams{"bparams"},
        bckpt{"bckpt"};
    DBuf<uint8_t> bsegbad{"bsegbad"};   // per bundle segment: mis-speculated tie this round
    DBuf<int32_t> bsegflag{"bsegflag"};   // per bundle segment: flags for the sim / chain
    DBuf<Clamp> tile_agg{"tile_agg"}, tile_inc{"tile_inc"};
    DBuf<unsigned> tflag{"tflag"};
    DBuf<long long> tile_x{"tile_x"}, tile_bad{"tile_bad"};
    // seed
    DBuf<int32_t> start{"start"}, cursor{"cursor"};
    DBuf<uint32_t> sortk{"sortk"}, sortv{"sortv"};
    DBuf<uint32_t> adj{"adj"}, row_of{"row_of"}, parent{"parent"}, csize{"csize"}, roots{"roots"}, rvals{"rvals"}, rvals2{"rvals2"}, cpos{"cpos"}, disc{"disc"}, frontier{"frontier"};
    DBuf<unsigned long long> ckey{"ckey"}, rkeys{"rkeys"}, rkeys2{"rkeys2"}, cand{"cand"}, cand2{"cand2"}, pair{"pair"};
    DBuf<int8_t> slab{"slab"}, slab2{"slab2"};
    DBuf<int64_t> fdeg{"fdeg"}, cum{"cum"};
    DBuf<uint32_t> bitsP{"bitsP"}, bitsT{"bitsT"}, bitsW{"bitsW"}, bitsD{"bitsD"};
    // hubs
    DBuf<uint32_t> hub_table{"hub_table"}, hub_ids{"hub_ids"};
    DBuf<unsigned long long> hub_k1{"hub_k1"}, hub_k2{"hub_k2"};
    bool hubs_on = false;
    uint32_t hub_host[kHubSlots];
    // scalars
    long long* d_sizes = nullptr;   // [2]
    long long* d_scal = nullptr;    // [8]
    long long* d_sscal = nullptr;   // [16] seed scalars
    // overlapped ingest of a page-locked host edge list: pieces copied on
    // copy_s, each checked and marked with an event; consumers wait only for
    // the pieces covering the edges they read
    cudaStream_t copy_s = nullptr;
    // id checks of the staged pieces on their own stream: a check waiting for
    // SMs behind a long round kernel must not hold back the next piece's DMA
    cudaStream_t check_s = nullptr;
    struct IngestMark {
        int64_t end;
        cudaEvent_t ev;
    };
    std::vector<IngestMark> ingest;
    const uint2* ingest_base = nullptr;
    int64_t ingest_m = 0, ingest_n = 0;
    unsigned long long* d_bad = nullptr;   // ingest: max bad endpoint + 1 (0 = none)
    long long* h_pin = nullptr;     // [32] pinned mirror
    // cub temp
    DBuf<unsigned char> temp{"temp"};
    // next-chunk bin offsets computed on aux_s while this chunk's rounds run
    DBuf<int32_t> bin_hist2{"bin_hist2"}, bin_offs2{"bin_offs2"};
    DBuf<unsigned char> aux_temp{"aux_temp"};
    cudaStream_t aux_s = nullptr;
    cudaEvent_t pref_go = nullptr, pref_done = nullptr;
    const uint2* pref_e = nullptr;   // chunk whose offsets are pending in buffer pref_buf
    int64_t pref_m = 0;
    int pref_buf = 0, pref_nbins = 0;
    bool pref_pending = false;       // pref_done not yet waited on by c->s
    // ingest
    void* pin_buf[2] = {nullptr, nullptr};
    size_t pin_bytes = 0;
    cudaEvent_t pin_ev[2] = {nullptr, nullptr};
    DBuf<uint2> edges_owned;
    // file ingest (load_grpe): a reader thread preads GRPE pieces into a ring
    // of pinned slots and queues their DMA + check on copy_s; ingest marks are
    // published under ing_mu, ing_pub = edges whose mark exists
    static constexpr int RING = 4;
    std::thread ing_thr;
    std::mutex ing_mu;
    std::condition_variable ing_cv;
    bool ing_live = false, ing_done = false, ing_stop = false;
    int64_t ing_pub = 0;
    std::string ing_err;
    void* ring[RING] = {};
    cudaEvent_t ring_ev[RING] = {};
    size_t ring_bytes = 0;
    // partitioned storage (grem_store.cu)
    DBuf<uint32_t> bk_keys_a{"bk_keys_a"}, bk_keys_b{"bk_keys_b"}, bk_order{"bk_order"};
    DBuf<uint2> bk_out{"bk_out"};
    DBuf<unsigned long long> bk_counts{"bk_counts"};
    DBuf<unsigned long long> ns_cnt{"ns_cnt"};   // node stats (theory)
    DBuf<int64_t> ns_k{"ns_k"}, ns_k0{"ns_k0"};
    DBuf<double> th_lg{"th_lg"}, th_term{"th_term"}, th_part{"th_part"};
    DBuf<int64_t> th_big{"th_big"};
    DBuf<unsigned long long> th_scal{"th_scal"};
    DBuf<uint32_t> ns_pack{"ns_pack"};
    DBuf<unsigned long long> sh_keys{"sh_keys"}, sh_vals{"sh_vals"};   // external shuffle
    DBuf<long long> bk_perm{"bk_perm"};
    DBuf<uint8_t> bk_rec{"bk_rec"}, bk_rec_out{"bk_rec_out"};
    bool staged_last = false;   // edges_owned holds the last call's host edge list
    int64_t staged_m = 0;
    // count_cuts
    DBuf<unsigned long long> cc_sizes;
    DBuf<int32_t> lab32;
    DBuf<uint32_t> packed_lab{"packed_lab"}, side_bits{"side_bits"}, side_pop{"side_pop"}, side_pre{"side_pre"};
    // recursion arena: per-level induced-subgraph buffers (reused across calls)
    DBuf<uint2> rec_e[40];   // per recursion level: both induced subgraphs of the level's bisection
    DBuf<uint2> word_info{"word_info"};
    DBuf<unsigned long long> lb_status{"lb_status"};
    DBuf<unsigned int> lb_ticket{"lb_ticket"};
    DBuf<int32_t> rec_o[40];
    DBuf<int32_t> part_fin{"part_fin"}, part_orig{"part_orig"};
    // live state for hooks
    int64_t live_n = 0;
    grem_stats stats{};
    long long kernels = 0;
    int64_t bk_out_m = -1;   // edges of the last write_buckets kept in bk_out (-1: none)
};
void ctx_trim_buffers(grem_ctx* c);   // every device workspace of one context (defined below)


namespace {

void scal_read(grem_ctx* c, const long long* dsrc, int count) {
    CK(cudaMemcpyAsync(c->h_pin, dsrc, sizeof(long long) * count, cudaMemcpyDeviceToHost, c->s));
    CK(cudaStreamSynchronize(c->s));
}

void scal_write(grem_ctx* c, long long* ddst, const long long* vals, int count) {
    // stage through a private pinned slot so the async copy never races the host
    for (int i = 0; i < count; ++i) c->h_pin[16 + i] = vals[i];
    CK(cudaMemcpyAsync(ddst, c->h_pin + 16, sizeof(long long) * count, cudaMemcpyHostToDevice, c->s));
    CK(cudaStreamSynchronize(c->s));
}

void ensure_temp(grem_ctx* c, size_t bytes) { c->temp.ensure(bytes, c->s); }

cudaEvent_t prof_event(grem_ctx* c) {
    if (c->ev_used == c->ev_pool.size()) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        c->ev_pool.push_back(e);
    }
    return c->ev_pool[c->ev_used++];
}

// NVTX ranges mirror the phases (header-only nvtx3; free when no tool is
// attached), so an nsys / ncu --nvtx timeline names every launch group
struct PhaseScope {
    grem_ctx* c;
    int ph;
    cudaEvent_t a = nullptr, b = nullptr;
    PhaseScope(grem_ctx* c_, int ph_) : c(c_), ph(ph_) {
        nvtxRangePushA(kPhaseNames[ph]);
        if (c->profiling) {
            a = prof_event(c);
            b = prof_event(c);
            cudaEventRecord(a, c->s);
        }
    }
    ~PhaseScope() {
        if (c->profiling) {
            cudaEventRecord(b, c->s);
            c->prof_open.push_back({ph, {a, b}});
        }
        nvtxRangePop();
    }
};

// consecutive sub-phases: to(ph) closes the open one and opens ph
struct PhaseSeq {
    grem_ctx* c;
    int ph = -1;
    bool nvtx_open = false;
    cudaEvent_t a = nullptr;
    explicit PhaseSeq(grem_ctx* c_) : c(c_) {}
    void to(int nph) {
        if (ph >= 0 || nph >= 0) {   // NVTX: close the open sub-phase, open the next
            if (nvtx_open) nvtxRangePop();
            nvtx_open = nph >= 0;
            if (nvtx_open) nvtxRangePushA(kPhaseNames[nph]);
        }
        if (!c->profiling) {
            ph = nph;
            return;
        }
        cudaEvent_t e = prof_event(c);
        cudaEventRecord(e, c->s);
        if (ph >= 0) c->prof_open.push_back({ph, {a, e}});
        ph = nph;
        a = e;
    }
    ~PhaseSeq() { to(-1); }
};

void prof_collect(grem_ctx* c) {
    for (auto& p : c->prof_open) {
        float ms = 0;
        if (cudaEventElapsedTime(&ms, p.second.first, p.second.second) == cudaSuccess) {
            c->phase_ms[p.first] += ms;
            c->phase_n[p.first] += 1;
        }
    }
    c->prof_open.clear();
    c->ev_used = 0;
}

thread_local grem_ctx* tl_ctx = nullptr;   // the context whose bisection runs on this host thread

struct CtxBind {   // binds tl_ctx for the kernel marks of one bisection
    grem_ctx* prev;
    explicit CtxBind(grem_ctx* c) : prev(tl_ctx) { tl_ctx = c; }
    ~CtxBind() { tl_ctx = prev; }
};

void kbytes(grem_ctx* c, int km, double bytes) {
    if (c->profiling == 2) c->phase_bytes[PH_K0 + km] += bytes;
}

void ensure_nodes(grem_ctx* c, int64_t n) {
    c->lab.ensure(n, c->s);
    c->lab2.ensure(n / 16 + 2, c->s);
    c->tl.ensure(n, c->s);
    c->flag.ensure(n, c->s);
    c->cnt.ensure(n, c->s);
    c->nbr.ensure(n, c->s);
    // succinct id -> chunk index map of the current chunk (rank words of 32
    // ids, whole 16K-node compact tiles); replaces an n x 4 B index table
    c->rankw.ensure(((n + 16383) / 16384) * 512 + 2, c->s);
    c->chg.ensure(n / 32 + 2, c->s);
    c->chgc.ensure(kChgCoarseBits / 32, c->s);
    c->chg2.ensure(n / 32 + 2, c->s);
    c->chgc2.ensure(kChgCoarseBits / 32, c->s);
    c->scratch.ensure(2 * n + 2, c->s);
    c->newid.ensure(n + 1, c->s);
    ensure_temp(c, select_nodes_temp_bytes(n));
    ensure_temp(c, scan_temp_bytes(n + 1));
}

void ensure_chunk(grem_ctx* c, int64_t nc_cap, int64_t entries_cap) {
    int64_t padded = (nc_cap + 1 + kScanTile - 1) / kScanTile * kScanTile + 16;   // whole round tiles
    c->nodes.ensure(padded, c->s);
    c->meta.ensure(padded, c->s);
    c->bad.ensure(padded, c->s);
    c->want.ensure(nc_cap, c->s);
    c->newb.ensure(padded, c->s);
    c->x.ensure(padded, c->s);
    c->xalt.ensure(padded, c->s);
    c->xnext.ensure(padded, c->s);
    c->cntc.ensure(padded, c->s);
    c->nbrc.ensure(padded, c->s);
    c->tlc.ensure(padded, c->s);
    int64_t nseg = (nc_cap + bundle_segment_len(nc_cap) - 1) / bundle_segment_len(nc_cap) + 2;
    c->bends.ensure(nseg * 192, c->s);
    c->bxin.ensure(nseg, c->s);
    c->bhit.ensure(nseg, c->s);
    c->bsegbad.ensure(nseg + 1, c->s);
    c->bsegflag.ensure(nseg + 1, c->s);
    c->bparams.ensure(nc_cap + 1, c->s);
    c->bckpt.ensure(bundle_ckpt_ints(nc_cap) + 192, c->s);
    int64_t tiles = (nc_cap + kScanTile - 1) / kScanTile + 1;
    c->tile_agg.ensure(tiles, c->s);
    c->tile_inc.ensure(tiles, c->s);
    c->tflag.ensure(tiles + 2, c->s);
    c->tile_x.ensure(tiles, c->s);
    c->tile_bad.ensure(tiles, c->s);
    ensure_temp(c, scan_temp_bytes(nc_cap + 1));
    ensure_temp(c, sort_temp_bytes(nc_cap));
}

void ensure_seed(grem_ctx* c, int64_t nc, int64_t entries) {
    c->start.ensure(nc + 1, c->s);
    c->cursor.ensure(nc + 1, c->s);
    c->adj.ensure(entries + 1, c->s);
    c->row_of.ensure(entries + 1, c->s);
    c->parent.ensure(nc, c->s);
    c->csize.ensure(nc, c->s);
    c->roots.ensure(nc, c->s);
    c->rvals.ensure(nc, c->s);
    c->rvals2.ensure(nc, c->s);
    c->cpos.ensure(nc, c->s);
    c->disc.ensure(nc, c->s);
    c->frontier.ensure(nc, c->s);
    c->ckey.ensure(nc, c->s);
    c->rkeys.ensure(nc, c->s);
    c->rkeys2.ensure(nc, c->s);
    c->cand.ensure(nc, c->s);
    c->cand2.ensure(nc, c->s);
    c->pair.ensure(nc, c->s);
    c->slab.ensure(nc, c->s);
    c->slab2.ensure(nc, c->s);
    c->fdeg.ensure(nc + 1, c->s);
    c->cum.ensure(nc + 1, c->s);
    ensure_temp(c, sort_temp_bytes(nc));
    ensure_temp(c, scan_temp_bytes(nc + 1));
}

void ingest_wait(grem_ctx* c, const uint2* end);
void ingest_wait_all(grem_ctx* c);

ChunkBufs chunk_bufs(grem_ctx* c) {
    ChunkBufs b;
    b.lab = c->lab.p;
    b.tl = c->tl.p;
    b.cnt = c->cnt.p;
    b.flag = c->flag.p;
    b.nbr = c->nbr.p;
    b.nodes = c->nodes.p;
    b.meta = c->meta.p;
    b.newb = c->newb.p;
    b.x = c->x.p;
    b.xalt = c->xalt.p;
    b.xnext = c->xnext.p;
    b.bad = c->bad.p;
    b.cntc = c->cntc.p;
    b.nbrc = c->nbrc.p;
    b.tlc = c->tlc.p;
    b.pos = nullptr;
    b.rankw = c->rankw.p;
    b.chg = c->chg.p;
    b.chgc = c->chgc.p;
    b.chg_shift = chg_coarse_shift(c->live_n);
    b.tile_agg = c->tile_agg.p;
    b.tile_inc = c->tile_inc.p;
    b.tflag = c->tflag.p;
    b.tile_x = c->tile_x.p;
    b.tile_bad = c->tile_bad.p;
    b.sizes = c->d_sizes;
    b.scal = c->d_scal;
    b.hub_keys = c->hubs_on ? c->hub_table.p : nullptr;
    b.lab2 = c->lab2.p;
    b.gate = nullptr;
    b.dcur = c->dirty0.p;
    b.dnext = c->dirty1.p;
    b.segbad = c->bsegbad.p;
    b.bseg_len = 0;   // set per chunk (process_chunk: bundle_segment_len(nc))
    b.bseg_n = 0;
    return b;
}

SeedBufs seed_bufs(grem_ctx* c) {
    SeedBufs sb;
    sb.rank = nullptr;   // (the seed ranks through rankw)
    sb.start = c->start.p;
    sb.cursor = c->cursor.p;
    sb.adj = c->adj.p;
    sb.row_of = c->row_of.p;
    sb.parent = c->parent.p;
    sb.ckey = c->ckey.p;
    sb.csize = c->csize.p;
    sb.roots = c->roots.p;
    sb.rkeys = c->rkeys.p;
    sb.rkeys2 = c->rkeys2.p;
    sb.rvals = c->rvals.p;
    sb.rvals2 = c->rvals2.p;
    sb.cpos = c->cpos.p;
    sb.slab = c->slab.p;
    sb.slab2 = c->slab2.p;
    sb.disc = c->disc.p;
    sb.frontier = c->frontier.p;
    sb.cand_keys = c->cand.p;
    sb.cand_keys2 = c->cand2.p;
    sb.fdeg = c->fdeg.p;
    sb.cum = c->cum.p;
    sb.pair = c->pair.p;
    sb.want = c->want.p;
    sb.scal = c->d_sscal;
    return sb;
}

struct BisectArgs {
    const uint2* e;
    int64_t m, n;
    int64_t chunk;
    long long cap;
    int refine, passes, seed_algo, seed_passes;
    const grem_hooks* hooks;
};

// ------------------------------------------------------------ seed chunk
__global__ void k_count_diff(const int8_t* a, const int8_t* b, int64_t n, long long* out) {
    int d = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        d += a[i] != b[i];
    for (int off = 16; off; off >>= 1) d += __shfl_down_sync(0xffffffffu, d, off);
    if ((threadIdx.x & 31) == 0 && d) atomicAdd((unsigned long long*)out, (unsigned long long)d);
}

void seed_chunk(grem_ctx* c, const BisectArgs& a, const uint2* e, int64_t mc) {
    cudaStream_t s = c->s;
    ChunkBufs b = chunk_bufs(c);
    PhaseSeq seq(c);
    seq.to(PH_SEED_CSR);
    // chunk-0 CSR by one radix sort of (row id, column id) pairs: the sorted
    // keys' runs are the chunk nodes in ascending id order (= ranks)
    int64_t entries = 2 * mc;
    int64_t nc_cap = a.n < entries ? a.n : entries;
    ensure_seed(c, nc_cap, entries);
    c->sortk.ensure(entries + 1, s);
    c->sortv.ensure(entries + 1, s);
    ensure_temp(c, seed_csr_temp_bytes(entries));
    CK(cudaMemsetAsync(c->cursor.p, 0, sizeof(int32_t) * (nc_cap + 1), s));
    int end_bit = 1;
    while (end_bit < 32 && ((uint64_t)(a.n - 1) >> end_bit) != 0) ++end_bit;
    bool in_b = false;
    launch_seed_sort(e, mc, c->row_of.p, c->adj.p, c->sortk.p, c->sortv.p, end_bit, c->nodes.p, c->cursor.p,
                     c->d_scal, c->temp.p, c->temp.cap, &in_b, s);
    c->kernels += 1 + 2 * ((end_bit + 7) / 8) + 3;
    scal_read(c, c->d_scal, 1);
    int64_t nc = c->h_pin[0];
    if (nc == 0) fail(GREM_E_FORMAT, "cannot seed an empty chunk");
    if (2 * a.cap < nc)
        fail(GREM_E_CAPACITY, "capacity " + std::to_string(a.cap) + " infeasible for " + std::to_string(nc) +
                                  " chunk nodes");
    c->stats.visits += nc;
    exclusive_sum_i32(c->cursor.p, c->start.p, nc + 1, c->temp.p, c->temp.cap, s);
    const int64_t nwords = a.n / 32 + 1;
    launch_rank_words(c->nodes.p, nc, nwords, c->rankw.p, s);
    CK(cudaMemsetAsync(c->cursor.p, 0, sizeof(int32_t) * (nc + 1), s));   // now: self-loop entries per row
    launch_seed_map(in_b ? c->sortk.p : c->row_of.p, in_b ? c->sortv.p : c->adj.p, entries, c->rankw.p, c->row_of.p,
                    c->adj.p, c->cursor.p, s);
    c->kernels += 4;
    SeedBufs sb = seed_bufs(c);
    long long target = (nc + 1) / 2;   // ceil(n / 2), seed.py:57

    if (a.seed_algo == 1) {
        // SeedConfig(algorithm="random"): numpy PCG64 permutation on the host (seed.py:48-52)
        if (!a.hooks || !a.hooks->seed) fail(GREM_E_FORMAT, "random seed needs a seed hook");
        std::vector<int8_t> hl(nc);
        if (a.hooks->seed(nc, hl.data(), a.hooks->user)) fail(GREM_E_CALLBACK, "seed hook failed");
        CK(cudaMemcpyAsync(c->slab.p, hl.data(), nc, cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));
    } else {
        // ---- _bfs_grow (seed.py:56-94): components in restart order, BFS only
        // inside the component where the pick count crosses `target`.
        seq.to(PH_SEED_CC);
        launch_cc_csr(c->start.p, c->adj.p, nc, c->parent.p, c->roots.p,
                      reinterpret_cast<unsigned long long*>(c->d_sscal + 13), s);
        launch_comp_keys(sb, nc, s, reinterpret_cast<unsigned long long*>(c->d_sscal + 13));
        ensure_temp(c, select_nodes_temp_bytes(nc));
        launch_select_roots(sb, nc, c->temp.p, c->temp.cap, s);
        c->kernels += 8;
        scal_read(c, c->d_sscal, 1);
        int64_t nr = c->h_pin[0];
        launch_root_keys(sb, nr, s);
        sort_pairs_u64_u32(c->rkeys.p, c->rkeys2.p, c->rvals.p, c->rvals2.p, nr, c->temp.p, c->temp.cap, s);
        launch_boundary(sb, nr, target, c->temp.p, c->temp.cap, s);
        c->kernels += 6;
        scal_read(c, c->d_sscal, 4);
        long long quota = c->h_pin[2];
        long long sstar = c->h_pin[3];
        launch_seed_labels(sb, nc, s);
        c->kernels += 1;
        seq.to(PH_SEED_BFS);
        long long count = 1;
        if (count < quota) {
            long long h = sstar;
            uint32_t s32 = (uint32_t)h;
            c->h_pin[20] = 0;
            memcpy(&c->h_pin[20], &s32, sizeof(uint32_t));
            CK(cudaMemcpyAsync(c->frontier.p, &c->h_pin[20], sizeof(uint32_t), cudaMemcpyHostToDevice, s));
            int64_t fsize = 1;
            long long rbase = 0;
            while (count < quota) {
                launch_frontier_degrees(sb, fsize, s);
                CK(cudaMemsetAsync(c->fdeg.p + fsize, 0, sizeof(int64_t), s));
                exclusive_sum_i64(c->fdeg.p, c->cum.p, fsize + 1, c->temp.p, c->temp.cap, s);
                CK(cudaMemsetAsync(c->d_sscal + 4, 0, sizeof(long long), s));
                CK(cudaMemcpyAsync(&c->h_pin[0], c->cum.p + fsize, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
                int64_t total = c->h_pin[0];
                if (total > 0) launch_bfs_expand(sb, fsize, rbase, total, s);
                c->kernels += 3;
                scal_read(c, c->d_sscal + 4, 1);
                int64_t ncand = c->h_pin[0];
                if (ncand == 0) fail(GREM_E_FORMAT, "internal: BFS frontier exhausted before quota");
                launch_cand_keys(sb, ncand, s);
                sort_keys_u64(c->cand.p, c->cand2.p, ncand, c->temp.p, c->temp.cap, s);
                int64_t take = ncand < quota - count ? ncand : quota - count;
                launch_bfs_take(sb, ncand, take, s);
                c->kernels += 3;
                c->stats.seed_bfs_levels++;
                count += take;
                rbase += fsize;
                fsize = take;
            }
        }
        launch_seed_finalize(sb, nc, s);
        c->kernels += 1;
        // ---- boundary refinement passes (seed.py:96-116): rounds to a
        // fixpoint with the exact sizes scan (moves are clamps, no ties), on
        // 1-bit label maps
        seq.to(PH_SEED_REFINE);
        int64_t nwords = (nc + 31) / 32;
        c->bitsP.ensure(nwords + 8, s);
        c->bitsT.ensure(nwords + 8, s);
        c->bitsW.ensure(nwords + 8, s);
        c->bitsD.ensure(nwords + 8, s);
        uint32_t* Pb = c->bitsP.p;
        uint32_t* Tb = c->bitsT.p;
        launch_pack_bits(sb.slab, nc, Pb, s);
        long long xstart = target;
        for (int pass = 0; pass < a.seed_passes; ++pass) {
            CK(cudaMemcpyAsync(Tb, Pb, sizeof(uint32_t) * nwords, cudaMemcpyDeviceToDevice, s));
            scal_write(c, c->d_sscal + 6, &xstart, 1);
            int64_t changed = -1;
            for (int round = 0;; ++round) {
                if (changed < 0 || changed > nc / 16) {
                    launch_row_counts_bits(sb, Pb, Tb, 0, entries, nc, s);
                } else {
                    launch_refine_delta(sb, c->bitsD.p, nc, changed, Pb, Tb, c->temp.p, c->temp.cap, s);
                    c->kernels += 2;
                }
                CK(cudaMemsetAsync(c->d_sscal + 5, 0, sizeof(long long), s));
                launch_refine_round(sb, b, Pb, Tb, c->bitsW.p, c->bitsD.p, nc, a.cap, s);
                c->kernels += 4;
                scal_read(c, c->d_sscal + 5, 1);
                changed = c->h_pin[0];
                if (changed == 0) break;
                if (round > nc + 2) fail(GREM_E_FORMAT, "internal: refinement rounds did not converge");
            }
            CK(cudaMemsetAsync(c->d_sscal + 7, 0, sizeof(long long), s));
            launch_xor_popc(Pb, Tb, nc, c->d_sscal + 7, s);
            c->kernels += 1;
            scal_read(c, c->d_sscal + 7, 3);
            if (c->h_pin[0] == 0) break;   // "if not moved: break"
            xstart = c->h_pin[2];          // sscal[9]: x at the end of the pass
            std::swap(Pb, Tb);
        }
        launch_unpack_bits(Pb, nc, sb.slab, s);
        c->kernels += 2;
    }
    seq.to(PH_SEED_COMMIT);
    {
        // estimates against the final seed labels (bitmap gathers)
        int64_t nwords = (nc + 31) / 32;
        c->bitsP.ensure(nwords + 8, s);
        launch_pack_bits(c->slab.p, nc, c->bitsP.p, s);
        launch_row_counts_bits(sb, c->bitsP.p, c->bitsP.p, 1, entries, nc, s);
        sb.slab = c->slab.p;
    }
    // ---- _seed_chunk (grem.py:158-174): labels, sizes recount, estimates
    CK(cudaMemsetAsync(c->d_sscal + 7, 0, sizeof(long long), s));
    launch_seed_commit(sb, b, c->nodes.p, nc, s);
    c->kernels += 2;
    scal_read(c, c->d_sscal + 7, 1);
    long long zeros = c->h_pin[0];
    long long sz[2] = {zeros, nc - zeros};
    scal_write(c, c->d_sizes, sz, 2);
}

// ------------------------------------------------------------ process_chunk
bool chunk_binned(const BisectArgs& a, int64_t mc) {
    if (getenv("GREM_NO_BINNING")) return false;
    return getenv("GREM_FORCE_BINNING") || (a.n * 9 > (48LL << 20) && mc >= (1 << 20));
}

// make c->s wait for any offsets prefetch still in flight (its buffer is about to be reused)
void prefetch_join(grem_ctx* c) {
    if (c->pref_pending) {
        CK(cudaStreamWaitEvent(c->s, c->pref_done, 0));
        c->pref_pending = false;
    }
}

// queue the next chunk's bin offsets on aux_s (into the buffer the current
// chunk does not use), ordered after everything queued on c->s so far
void prefetch_offsets(grem_ctx* c, const BisectArgs& a, const uint2* ne, int64_t nm, int cur_buf) {
    static const bool on = !getenv("GREM_NO_PREFETCH");
    c->pref_e = nullptr;
    if (!on || !ne || nm <= 0 || c->ingest_base || !chunk_binned(a, nm)) return;
    int shift = binned_shift(a.n);
    int nbins = (int)((a.n + (1LL << shift) - 1) >> shift);
    int64_t hent = binned_hist_entries(nbins);
    int nb = cur_buf ^ 1;
    DBuf<int32_t>& hist = nb ? c->bin_hist2 : c->bin_hist;
    DBuf<int32_t>& offs = nb ? c->bin_offs2 : c->bin_offs;
    hist.ensure(hent, c->s);
    offs.ensure(hent, c->s);
    c->aux_temp.ensure(scan_temp_bytes(hent), c->s);
    if (!c->aux_s) {
        int lo = 0, hi = 0;
        CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CK(cudaStreamCreateWithPriority(&c->aux_s, cudaStreamNonBlocking, lo));
        CK(cudaEventCreateWithFlags(&c->pref_go, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->pref_done, cudaEventDisableTiming));
    }
    CK(cudaEventRecord(c->pref_go, c->s));
    CK(cudaStreamWaitEvent(c->aux_s, c->pref_go, 0));
    launch_bin_offsets(ne, nm, c->hubs_on ? c->hub_table.p : nullptr, shift, nbins, hist.p, offs.p, c->aux_temp.p,
                       c->aux_temp.cap, c->aux_s);
    CK(cudaEventRecord(c->pref_done, c->aux_s));
    c->kernels += 3;
    c->pref_e = ne;
    c->pref_m = nm;
    c->pref_buf = nb;
    c->pref_nbins = nbins;
    c->pref_pending = true;
}

void process_chunk(grem_ctx* c, const BisectArgs& a, const uint2* e, int64_t mc, const uint2* next_e = nullptr,
                   int64_t next_mc = 0) {
    cudaStream_t s = c->s;
    ChunkBufs b = chunk_bufs(c);
    CK(cudaMemsetAsync(c->d_scal, 0, sizeof(long long) * 16, s));
    CK(cudaMemsetAsync(c->d_scal + 7, 1, 1, s));   // round gate open
    b.gate = c->d_scal + 7;
    bool binned = false;
    {
        PhaseScope ps(c, PH_COUNT);
        // propagation blocking when the per-node counters do not fit in L2
        const char* nb_env = getenv("GREM_NO_BINNING");
        const char* fb_env = getenv("GREM_FORCE_BINNING");   // tests: exercise the binned path on small graphs
        (void)nb_env;
        (void)fb_env;
        binned = chunk_binned(a, mc);
        if (binned) {
            int shift = binned_shift(a.n);
            int nbins = (int)((a.n + (1LL << shift) - 1) >> shift);
            int64_t ntiles = binned_tiles(a.n);
            bool have = c->pref_e == e && c->pref_m == mc && c->pref_nbins == nbins;
            int buf = have ? c->pref_buf : 0;
            prefetch_join(c);
            DBuf<int32_t>& hist = buf ? c->bin_hist2 : c->bin_hist;
            DBuf<int32_t>& offs = buf ? c->bin_offs2 : c->bin_offs;
            c->bin_recs.ensure(2 * mc + 16, s);
            int64_t hent = binned_hist_entries(nbins);
            hist.ensure(hent, s);
            offs.ensure(hent, s);
            ensure_temp(c, scan_temp_bytes(hent));
            c->bin_hcnt.ensure(kHubSlots, s);
            c->bin_hflag.ensure(kHubSlots, s);
            c->bin_status.ensure(ntiles + 1, s);
            c->bin_ticket.ensure(4, s);
            BinBufs bb{c->bin_recs.p, hist.p, offs.p, c->bin_hcnt.p, c->bin_hflag.p, c->bin_status.p,
                       c->bin_ticket.p, shift, nbins};
            launch_count_init_binned(e, mc, a.n, a.refine, b, bb, c->temp.p, c->temp.cap, s, have);
            c->kernels += have ? 6 : 9;
            prefetch_offsets(c, a, next_e, next_mc, buf);   // overlaps this chunk's rounds
        } else {
            prefetch_join(c);
            launch_count_init(e, mc, b, s);
        }
    }
    c->stats.count_bytes += 10 * mc;   // 8 B edge read + 2 x 1 B label gather
    if (!binned) {
        PhaseScope ps(c, PH_SELECT);
        launch_select_nodes(c->flag.p, c->cnt.p, a.n, c->nodes.p, c->d_scal, c->temp.p, c->temp.cap, s);
        c->kernels += 2;
    }
    scal_read(c, c->d_scal, 3);
    int64_t nc = c->h_pin[0];
    // refined (previously assigned) chunk nodes: the binned compact leaves the
    // new-member count in scal[2]; only needed for the kernel byte counters
    int64_t refined = binned ? nc - c->h_pin[2] : nc;
    c->stats.visits += nc;
    if (binned) {
        kbytes(c, KM_BIN_HIST, 8.0 * mc);              // edge read
        kbytes(c, KM_BIN_SCATTER, 16.0 * mc);          // edge read + two 4-byte records out
        kbytes(c, KM_BIN_COMPACT, 8.0 * mc + 38.0 * nc + 16.0 * refined + (double)a.n);   // records in, state out, nbr + lab in
    }
    if (!binned) {   // (the binned path wrote the compact state, newb and the rank words already)
        PhaseScope ps(c, PH_NODE);
        launch_rank_words(c->nodes.p, nc, a.n / 32 + 1, c->rankw.p, s);
        launch_node_init(b, nc, a.refine, s);
        exclusive_sum_i32(c->x.p, c->newb.p, nc, c->temp.p, c->temp.cap, s);
        launch_add_base(c->newb.p, nc, c->d_sizes, s);
        c->kernels += 3;
    }
    b.bseg_len = bundle_segment_len(nc);
    b.bseg_n = (nc + b.bseg_len - 1) / b.bseg_len;
    c->bsegbad.ensure(b.bseg_n + 2, s);   // (sized from the chunk-node capacity already; never less than this chunk)
    c->bsegflag.ensure(b.bseg_n + 2, s);
    b.segbad = c->bsegbad.p;
    // identity padding up to whole round tiles (inactive nodes, meta 0)
    {
        int64_t padded = (nc + 1 + kScanTile - 1) / kScanTile * kScanTile;
        CK(cudaMemsetAsync(c->meta.p + nc, 0, padded - nc, s));
    }
    // Rounds are launched in batches without a host round trip: every round
    // kernel is gated on the device by the previous round's changed count, so
    // rounds after the fixpoint are no-ops; the host checks once per batch.
    static const int batch = getenv("GREM_ROUND_BATCH") ? std::max(1, atoi(getenv("GREM_ROUND_BATCH"))) : 2;
    // Incremental rounds (r >= 3): a round tile whose counts and tie guesses
    // did not change and whose incoming x equals last round's exact x is
    // skipped (its decisions are already the fixpoint's for that input).
    static const bool incr_on = !getenv("GREM_NO_INCREMENTAL");
    int64_t rtiles = (nc + 1 + kRTileC - 1) / kRTileC;
    c->dirty0.ensure(rtiles + 1, s);
    c->dirty1.ensure(rtiles + 1, s);
    uint8_t* dbuf[2] = {c->dirty0.p, c->dirty1.p};
    uint32_t* chgbuf[2] = {c->chg.p, c->chg2.p};
    uint32_t* chgcbuf[2] = {c->chgc.p, c->chgc2.p};
    const int64_t nchg = a.n / 32 + 2;
    auto issue = [&](int r) {   // one round's launches (all device-gated)
        b.dcur = dbuf[r & 1];
        b.dnext = dbuf[(r + 1) & 1];
        b.chg = chgbuf[r & 1];     // written this round (round_down, bundle_fix)
        b.chgc = chgcbuf[r & 1];
        launch_round_start(b, rtiles + 1, r == 1, nchg, s);   // gate, scalars, dirty tiles, this round's bitmaps
        c->kernels++;
        if (r > 1) {
            PhaseScope ps(c, PH_DELTA);
            ChunkBufs bd = b;      // the previous round's changes
            bd.chg = chgbuf[(r - 1) & 1];
            bd.chgc = chgcbuf[(r - 1) & 1];
            kmark(KM_COUNT_DELTA, 1, s);
            static const bool staged_on = !getenv("GREM_NO_STAGED_DELTA");   // A/B switch
            launch_count_delta(e, mc, bd, s, staged_on && r == 2);   // round 2: most lower endpoints changed
            kmark(KM_COUNT_DELTA, 0, s);
            kbytes(c, KM_COUNT_DELTA, 9.0 * mc);   // 8 B edge read + 1 B lower-endpoint label
            c->kernels++;
        }
        {
            PhaseScope ps(c, PH_SCAN);
            launch_round_scan(b, nc, a.cap, r == 1, incr_on && r >= 3, s);
            c->kernels += 3;
            if (!(incr_on && r >= 3)) {   // full rounds (the marked launches), DESIGN.md §5
                kbytes(c, KM_ROUND_REDUCE, 14.0 * nc + 16.0 * refined);   // meta r/w, newb, cnt; nbr of refined nodes
                kbytes(c, KM_ROUND_DOWN, 20.0 * nc);   // meta, newb, nodes, tlc in; x, xalt, meta, tlc out
            }
        }
        {
            // exact repair by trajectory bundles, gated on the device by the
            // number of mis-speculated ties (no host round trip); windows:
            // speculative x, previous round's exact x (round 1: half-step
            // predictor) and, in round 1, the balance point
            PhaseScope ps(c, PH_BUNDLE);
            if (r == 1) {
                launch_half_predictor(b, nc, a.cap, c->xalt.p, s);
                c->kernels += 4;
            }
            BundleBufs bb{c->bparams.p, c->bends.p, c->bckpt.p, c->bxin.p, c->bhit.p, c->bsegflag.p};
            launch_bundle(b, nc, a.cap, c->xalt.p, bb, r == 1 ? 3 : 2, s, true);
            c->kernels += 5;
        }
        if (getenv("GREM_DEBUG_BUNDLE")) {
            scal_read(c, c->d_scal + 1, 9);
            fprintf(stderr, "[bundle] n %lld round %d nc %lld changed %lld first %lld nbad %lld misses(cum) %lld\n",
                    (long long)a.n, r, (long long)nc, c->h_pin[0], c->h_pin[8] > nc ? -1LL : c->h_pin[8], c->h_pin[3],
                    c->h_pin[2]);
        }
        // this round's exact x becomes the next round's second window centre
        // (after the fixpoint the swaps are harmless: nothing reads xalt)
        std::swap(c->xalt.p, c->xnext.p);
        b.xalt = c->xalt.p;
        b.xnext = c->xnext.p;
    };
    // Rounds >= 3 repeat with period 2 (double buffers), so the pair (3, 4) is
    // captured once per chunk as a CUDA graph and replayed: one launch per two
    // rounds instead of ~20 (the small chunks of the sparse subtrees are
    // launch-latency bound).
    static const bool graphs_on = !getenv("GREM_NO_GRAPH") && !getenv("GREM_DEBUG_BUNDLE");
    const bool use_graph = graphs_on && batch == 2 && !c->profiling;
    bool graph_ready = false;
    long long pair_kernels = 0;
    // Device-side convergence: rounds >= 3 run as a conditional WHILE graph
    // node whose body is one round pair plus k_loop_cond, which sets the
    // condition from the pair's last changed count -- one host round trip
    // per chunk (after round 2) instead of one per pair.  The graph is built
    // while rounds 1-2 run.  Off by default (GREM_DEVICE_LOOP=1): instantiating
    // a graph with a conditional node per chunk cost more than the host round
    // trips it saves (papers100M k=16: 664 vs 608 ms, profiles/r02_ab_devloop.txt).
    static const bool dev_loop_on = getenv("GREM_DEVICE_LOOP") != nullptr;
    const bool dev_loop = use_graph && dev_loop_on && !c->root->s_dense;   // (not with green-context streams)
    const long long max_rounds = nc + 6;
    bool looped = false;
    for (int r = 1;;) {
        if (dev_loop && r == 3) {
            cudaGraph_t parent = nullptr;
            CK(cudaGraphCreate(&parent, 0));
            cudaGraphConditionalHandle h;
            CK(cudaGraphConditionalHandleCreate(&h, parent, 1, cudaGraphCondAssignDefault));
            cudaGraphNodeParams np = {};   // (a union with no default constructor: value-initialise)
            np.type = cudaGraphNodeTypeConditional;
            np.conditional.handle = h;
            np.conditional.type = cudaGraphCondTypeWhile;
            np.conditional.size = 1;
            cudaGraphNode_t node;
            CK(cudaGraphAddNode(&node, parent, nullptr, 0, &np));
            cudaGraph_t body = np.conditional.phGraph_out[0];
            long long k0 = c->kernels;
            CK(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
            issue(r);
            issue(r + 1);
            launch_loop_cond(h, c->d_scal, max_rounds, s);
            cudaGraph_t captured = nullptr;
            CK(cudaStreamEndCapture(s, &captured));
            pair_kernels = c->kernels - k0 + 1;
            c->kernels = k0;
            if (c->loop_exec) {
                cudaGraphExecDestroy(c->loop_exec);   // a graph with conditionals: one instance at a time
                c->loop_exec = nullptr;
            }
            CK(cudaGraphInstantiate(&c->loop_exec, parent, 0));
            CK(cudaGraphDestroy(parent));
            // the host check of round 2 (rounds 1-2 ran while the graph was built)
            scal_read(c, c->d_scal + 1, 1);
            if (c->h_pin[0] == 0) break;
            CK(cudaGraphLaunch(c->loop_exec, s));
            looped = true;
            break;
        }
        if (use_graph && r >= 3) {
            if (!graph_ready) {
                long long k0 = c->kernels;
                cudaGraph_t g = nullptr;
                CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
                issue(r);
                issue(r + 1);
                CK(cudaStreamEndCapture(s, &g));
                pair_kernels = c->kernels - k0;
                c->kernels = k0;
                bool ok = false;
                if (c->round_exec) {
                    cudaGraphExecUpdateResultInfo info;
                    ok = cudaGraphExecUpdate(c->round_exec, g, &info) == cudaSuccess;
                    if (!ok) {
                        cudaGetLastError();
                        cudaGraphExecDestroy(c->round_exec);
                        c->round_exec = nullptr;
                    }
                }
                if (!ok) CK(cudaGraphInstantiate(&c->round_exec, g, 0));
                CK(cudaGraphDestroy(g));
                graph_ready = true;
            }
            // GREM_GRAPH_REPLAYS pairs per host check (A/B knob, default 1):
            // rounds past the fixpoint are gated no-ops
            static const int replays = getenv("GREM_GRAPH_REPLAYS") ? std::max(1, atoi(getenv("GREM_GRAPH_REPLAYS"))) : 1;
            for (int q = 0; q < replays; ++q) {
                CK(cudaGraphLaunch(c->round_exec, s));
                c->kernels += pair_kernels;
                r += 2;
            }
        } else {
            issue(r);
            r += 1;
        }
        if ((r - 1) % batch == 0 && !(dev_loop && r == 3)) {   // (the device loop checks round 2 itself)
            scal_read(c, c->d_scal + 1, 1);   // the last round's changed count (the next round's gate)
            if (c->h_pin[0] == 0) break;
        }
        if (r > nc + 4 + batch) fail(GREM_E_FORMAT, "internal: chunk rounds did not converge");
    }
    if (looped) {
        scal_read(c, c->d_scal + 1, 8);   // [0] the last round's changed count, [7] rounds run
        if (c->h_pin[0] != 0) fail(GREM_E_FORMAT, "internal: chunk rounds did not converge");
        long long ran = c->h_pin[7];
        c->kernels += pair_kernels * std::max(1LL, (ran - 1) / 2);
    }
    launch_round_gate(b, s);   // closes the last launched round's gate
    c->kernels++;
    scal_read(c, c->d_scal + 8, 1);
    int64_t rounds = c->h_pin[0];
    c->stats.count_bytes += 9 * mc * (rounds - 1);   // rounds >= 2: 8 B edge read + 1 B tentative-label gather
    c->stats.delta_bytes += 9 * mc * (rounds - 1);
    {
        PhaseScope ps(c, PH_COMMIT);
        launch_commit(b, nc, s);
        launch_sizes_update(b, nc, s);
    }
    c->kernels += 2;
    scal_read(c, c->d_scal + 3, 1);
    c->stats.walk_steps += c->h_pin[0];   // bundle window misses (sequential segment replays)
    c->stats.rounds += rounds;
    if (rounds > c->stats.max_rounds) c->stats.max_rounds = rounds;
}

// meter schedule of stream_chunks/_raw_chunks (edgefile.py:384-391,453-462)
struct Meter {
    const grem_hooks* h;
    int64_t prev = -1;
    void acquire(int64_t n) {
        if (h && h->meter) h->meter(n, h->user);
    }
    void on_chunk(int64_t n) {
        acquire(n);
        if (prev >= 0 && h && h->meter) h->meter(-prev, h->user);
        prev = n;
    }
    void end() {
        if (prev >= 0 && h && h->meter) h->meter(-prev, h->user);
        prev = -1;
    }
};

}  // namespace

void grem::kmark(int km, int begin, cudaStream_t s) {
    grem_ctx* c = tl_ctx;
    if (!c || c->profiling != 2 || s != c->s) return;
    cudaEvent_t e = prof_event(c);
    cudaEventRecord(e, s);
    if (begin) {
        c->kmark_open[km] = e;
    } else if (c->kmark_open[km]) {
        c->prof_open.push_back({PH_K0 + km, {c->kmark_open[km], e}});
        c->kmark_open[km] = nullptr;
    }
}

// Bucketised cuckoo insertion (2 buckets x 2 slots per key); a key that is
// still homeless after the displacement budget drops out of the hub set
// (hubs only change performance, never results).
int grem::hub_table_build(const uint32_t* ids, int count, uint32_t* table) {
    for (int k = 0; k < kHubSlots; ++k) table[k] = kHubEmpty;
    int placed = 0;
    uint32_t rng = 0x12345u;
    for (int i = 0; i < count; ++i) {
        uint32_t key = ids[i];
        bool dup = false;
        for (uint32_t bk : {hub_bucket1(key), hub_bucket2(key)})
            for (int s2 = 0; s2 < 2; ++s2) dup |= table[2 * bk + s2] == key;
        if (dup) continue;
        bool ok = false;
        for (int kick = 0; kick < 256 && !ok; ++kick) {
            uint32_t b1 = hub_bucket1(key), b2 = hub_bucket2(key);
            for (uint32_t bk : {b1, b2})
                for (int s2 = 0; s2 < 2 && !ok; ++s2)
                    if (table[2 * bk + s2] == kHubEmpty) {
                        table[2 * bk + s2] = key;
                        ok = true;
                    }
            if (ok) break;
            rng = rng * 1664525u + 1013904223u;
            uint32_t bk = (rng >> 16) & 1 ? b1 : b2;
            int s2 = (rng >> 17) & 1;
            std::swap(key, table[2 * bk + s2]);   // evict and re-home the victim
        }
        if (ok) ++placed;   // else `key` (the original or a victim) is dropped
    }
    return placed;
}

namespace {

// Hubs of this bisection: top-kMaxHubs endpoints of a 4M-edge sample of the
// level's edge list (edges are in random order, so the sample ranks degrees);
// only worthwhile for large chunks.  Performance only: results never depend
// on which nodes are hubs.
void detect_hubs(grem_ctx* c, const BisectArgs& a) {
    c->hubs_on = false;
    const char* env_min = getenv("GREM_HUB_MIN_CHUNK");   // tests force the hub path on small graphs
    int64_t min_chunk = env_min ? atoll(env_min) : (1LL << 21);
    if (a.chunk < min_chunk || a.m == 0) return;
    cudaStream_t s = c->s;
    PhaseScope ps(c, PH_HUBS);
    int64_t S = a.m < (1LL << 22) ? a.m : (1LL << 22);
    ingest_wait(c, a.e + S);
    CK(cudaMemsetAsync(c->scratch.p, 0, sizeof(int32_t) * a.n, s));
    launch_sample_degrees(a.e, S, c->scratch.p, s);
    c->hub_ids.ensure(1 << 20, c->s);
    ensure_temp(c, hub_select_temp_bytes(a.n));
    const char* env_deg = getenv("GREM_HUB_MIN_DEG");
    launch_hub_select(c->scratch.p, a.n, env_deg ? atoi(env_deg) : 16, c->hub_ids.p, c->d_sscal + 8, c->temp.p, c->temp.cap, s);
    c->kernels += 3;
    scal_read(c, c->d_sscal + 8, 1);
    int64_t cnt = c->h_pin[0];
    if (cnt <= 0) return;
    if (cnt > (1 << 20)) cnt = 1 << 20;
    c->hub_k1.ensure(cnt, c->s);
    c->hub_k2.ensure(cnt, c->s);
    c->hub_table.ensure(kHubSlots, c->s);
    ensure_temp(c, sort_temp_bytes(cnt));
    launch_hub_keys(c->hub_ids.p, cnt, c->scratch.p, c->hub_k1.p, s);
    sort_keys_u64_desc(c->hub_k1.p, c->hub_k2.p, cnt, c->temp.p, c->temp.cap, s);
    int nh = (int)(cnt < kMaxHubs ? cnt : kMaxHubs);
    std::vector<unsigned long long> top(nh);
    CK(cudaMemcpyAsync(top.data(), c->hub_k2.p, sizeof(unsigned long long) * nh, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    std::vector<uint32_t> ids(nh);
    for (int k = 0; k < nh; ++k) ids[k] = (uint32_t)(top[k] & 0xFFFFFFFFULL);
    hub_table_build(ids.data(), nh, c->hub_host);
    CK(cudaMemcpyAsync(c->hub_table.p, c->hub_host, sizeof(uint32_t) * kHubSlots, cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    c->kernels += 4;
    c->hubs_on = true;
}

cudaEvent_t g_dbg_t0 = nullptr;   // GREM_DEBUG_LEVELS timeline origin

// bisect (grem.py:192-224) on device-resident edges; leaves labels in c->lab
void bisect_core(grem_ctx* c, const BisectArgs& a) {
    cudaStream_t s = c->s;
    CtxBind bind(c);
    struct NvtxBisect {
        explicit NvtxBisect(const BisectArgs& a) {
            char buf[96];
            snprintf(buf, sizeof buf, "bisect n=%lld m=%lld", (long long)a.n, (long long)a.m);
            nvtxRangePushA(buf);
        }
        ~NvtxBisect() { nvtxRangePop(); }
    } nvtx_bisect(a);
    static const char* dbg_levels = getenv("GREM_DEBUG_LEVELS");
    cudaEvent_t lv0 = nullptr, lv1 = nullptr;
    int64_t r0 = c->stats.rounds, v0 = c->stats.visits, b0 = c->stats.walk_steps;
    if (dbg_levels) {
        cudaEventCreate(&lv0);
        cudaEventCreate(&lv1);
        cudaEventRecord(lv0, s);
    }
    double ph0[PH_N];
    if (dbg_levels && c->profiling) {   // per-bisection phase split (debug): fold the open events first
        cudaStreamSynchronize(s);
        prof_collect(c);
        for (int k = 0; k < PH_N; ++k) ph0[k] = c->phase_ms[k];
    }
    struct LevelLog {
        grem_ctx* c; cudaEvent_t a, b; const BisectArgs& args; int64_t r0, v0, b0; const double* ph0;
        ~LevelLog() {
            if (!a) return;
            cudaEventRecord(b, c->s);
            cudaEventSynchronize(b);
            if (c->profiling) {
                prof_collect(c);
                std::string line;
                for (int k = 0; k < PH_N; ++k) {
                    double d = c->phase_ms[k] - ph0[k];
                    if (d >= 0.05) line += std::string(" ") + kPhaseNames[k] + "=" + std::to_string(d).substr(0, 6);
                }
                fprintf(stderr, "[phases] n %lld m %lld:%s\n", (long long)args.n, (long long)args.m, line.c_str());
            }
            float ms = 0, t0 = -1, t1 = -1;
            cudaEventElapsedTime(&ms, a, b);
            if (g_dbg_t0) {   // timeline relative to the start of partition()
                cudaEventElapsedTime(&t0, g_dbg_t0, a);
                cudaEventElapsedTime(&t1, g_dbg_t0, b);
            }
            fprintf(stderr, "[level] [%7.1f, %7.1f] n %lld m %lld cap %lld chunk %lld: %.2f ms rounds %lld visits %lld misses %lld\n",
                    t0, t1, (long long)args.n, (long long)args.m, args.cap, (long long)args.chunk, ms,
                    (long long)(c->stats.rounds - r0), (long long)(c->stats.visits - v0),
                    (long long)(c->stats.walk_steps - b0));
            cudaEventDestroy(a);
            cudaEventDestroy(b);
        }
    } level_log{c, lv0, lv1, a, r0, v0, b0, ph0};
    if (a.n < 1) fail(GREM_E_FORMAT, "num_nodes must be >= 1");
    // bundle tables pack a threshold and a lift into one int32 (t * 4 + o)
    if (a.n >= (1LL << 29)) fail(GREM_E_FORMAT, "bisections over 2^29 or more nodes are not supported");
    if (2 * a.cap < a.n)
        fail(GREM_E_CAPACITY, "capacity " + std::to_string(a.cap) + " cannot hold " + std::to_string(a.n) +
                                  " nodes across two parts");
    if (a.chunk < 1) fail(GREM_E_FORMAT, "chunk_size must be >= 1");
    c->stats.bisections++;
    // 8E (edge read) + 2E (label gathers) + 34 V (per visit)
    int64_t v_before = c->stats.visits;
    struct PathBytes {
        grem_ctx* c; int64_t m, v0;
        ~PathBytes() { c->stats.path_bytes += 10 * m + 34 * (c->stats.visits - v0); }
    } path_bytes{c, a.m, v_before};
    ensure_nodes(c, a.n);
    int64_t nc_cap = a.n < 2 * a.chunk ? a.n : 2 * a.chunk;
    ensure_chunk(c, nc_cap, 0);
    CK(cudaMemsetAsync(c->lab.p, 0xFF, a.n, s));
    CK(cudaMemsetAsync(c->lab2.p, 0, sizeof(uint32_t) * (a.n / 16 + 2), s));
    CK(cudaMemsetAsync(c->chg.p, 0, sizeof(uint32_t) * (a.n / 32 + 2), s));
    CK(cudaMemsetAsync(c->chgc.p, 0, kChgCoarseBits / 8, s));
    // id-indexed counters / flags are only used by the unbinned (small-chunk)
    // count path, which leaves them zero behind itself; the estimates nbr[g]
    // are read only for nodes that already have a label, i.e. after a commit
    // wrote them, so they need no clearing at all (1.8 GB at papers100M)
    {
        int64_t last = a.m ? a.m - (a.m - 1) / a.chunk * a.chunk : 0;
        bool all_binned = !getenv("GREM_NO_BINNING") && a.n * 9 > (48LL << 20) && a.chunk >= (1 << 20) &&
                          last >= (1 << 20) && a.passes == 1;
        if (!all_binned) {
            CK(cudaMemsetAsync(c->flag.p, 0, a.n, s));
            CK(cudaMemsetAsync(c->cnt.p, 0, sizeof(unsigned long long) * a.n, s));
        }
    }
    CK(cudaMemsetAsync(c->d_sizes, 0, sizeof(long long) * 2, s));
    c->live_n = a.n;
    prefetch_join(c);      // a prefetch is only ever consumed within its own bisection
    c->pref_e = nullptr;
    detect_hubs(c, a);
    int64_t num_chunks = a.m ? (a.m + a.chunk - 1) / a.chunk : 0;
    for (int pass = 0; pass < a.passes; ++pass) {
        Meter meter{a.hooks};
        for (int64_t ci = 0; ci < num_chunks; ++ci) {
            int64_t lo = ci * a.chunk;
            int64_t mc = a.m - lo < a.chunk ? a.m - lo : a.chunk;
            meter.on_chunk(mc);
            const uint2* e = a.e + lo;
            ingest_wait(c, e + mc);
            const uint2* ne = ci + 1 < num_chunks ? e + mc : nullptr;   // next chunk of this pass
            int64_t nm = ne ? (a.m - (lo + mc) < a.chunk ? a.m - (lo + mc) : a.chunk) : 0;
            if (pass == 0 && ci == 0) {
                PhaseScope ps(c, PH_SEED);
                prefetch_join(c);
                prefetch_offsets(c, a, ne, nm, 1);   // chunk 1's offsets during the seed (into buffer 0)
                seed_chunk(c, a, e, mc);
            } else {
                process_chunk(c, a, e, mc, ne, nm);
            }
            c->stats.chunks++;
            if (a.hooks && a.hooks->on_chunk) {
                scal_read(c, c->d_sizes, 2);
                long long sz[2] = {c->h_pin[0], c->h_pin[1]};
                int64_t sz64[2] = {sz[0], sz[1]};
                if (a.hooks->on_chunk(sz64, a.hooks->user)) {
                    meter.end();
                    fail(GREM_E_CALLBACK, "on_chunk hook raised");
                }
            }
        }
        meter.end();
    }
    // _fill_unassigned (grem.py:177-189)
    PhaseScope ps(c, PH_FILL);
    launch_fill_unassigned(c->lab.p, a.n, c->d_sizes, c->scratch.p, c->temp.p, c->temp.cap, s);
    c->kernels += 3;
}

int64_t plan_chunk(const grem_config* cfg, int64_t m) {
    // ChunkPlan.plan (edgefile.py:338-349); GremConfig.plan_for default 0.1
    if (cfg->chunk_edges > 0) return cfg->chunk_edges;
    double frac = cfg->chunk_frac > 0 ? cfg->chunk_frac : 0.1;
    if (!(frac > 0 && frac <= 1)) fail(GREM_E_FORMAT, "chunk_frac must be in (0, 1]");
    double t = frac * (double)m;
    int64_t ce = (int64_t)std::ceil(t);
    return ce < 1 ? 1 : ce;
}

void validate_cfg(const grem_config* cfg) {
    if (cfg->capacity_slack < 0) fail(GREM_E_FORMAT, "capacity_slack must be >= 0");
    if (cfg->passes < 1) fail(GREM_E_FORMAT, "passes must be >= 1");
    if (cfg->seed_refinement_passes < 0) fail(GREM_E_FORMAT, "refinement_passes must be >= 0");
    if (cfg->seed_algo != 0 && cfg->seed_algo != 1) fail(GREM_E_FORMAT, "unknown seed algorithm");
}

// count_cuts on device edges / int32 device labels
// known_cut >= 0: the caller already knows the cut (partition's incremental
// count); only the sizes / max label / unlabeled checks run
void count_cuts_dev(grem_ctx* c, const uint2* e, int64_t m, const int32_t* lab, int64_t n, grem_report* rep,
                    long long known_cut = -1) {
    cudaStream_t s = c->s;
    ingest_wait_all(c);
    int64_t cap = rep && rep->sizes_cap > 0 ? rep->sizes_cap : 2;
    if (cap < 2) cap = 2;
    c->cc_sizes.ensure(cap + 4, c->s);
    unsigned long long* d = c->cc_sizes.p;   // [0] cut, [1] max|neg, [2..] sizes
    CK(cudaMemsetAsync(d, 0, sizeof(unsigned long long) * (cap + 4), s));
    int* d_max = (int*)(d + 1);
    int* d_neg = d_max + 1;
    CK(cudaMemsetAsync(d_max, 0xFF, sizeof(int), s));   // -1
    PhaseScope ps(c, PH_CUTS);
    // sizes + max label first; the cut pass then gathers labels packed to the
    // narrowest power-of-two width (1 bit for a bisection, 4 for k=16)
    launch_count_cuts(e, m, lab, n, nullptr, d + 2, cap, d_max, d_neg, s);
    c->kernels += 1;
    std::vector<unsigned long long> h(cap + 2);
    CK(cudaMemcpyAsync(h.data(), d, sizeof(unsigned long long) * 2, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    int mx, neg;
    memcpy(&mx, &h[1], sizeof(int));
    memcpy(&neg, ((char*)&h[1]) + sizeof(int), sizeof(int));
    if (neg & 4) {   // unlabeled nodes exist: exact int32 pass also checks endpoints (grem.py:238-239)
        launch_count_cuts(e, m, lab, n, d, nullptr, 0, d_max, d_neg, s);
        c->kernels += 1;
    } else if (known_cut >= 0) {
        h[0] = (unsigned long long)known_cut;
    } else if (m > 0) {
        int bits = 1;
        while (bits < 32 && (uint64_t)mx >= (1ULL << bits)) bits *= 2;
        int lb = 0;
        while ((1 << lb) < bits) ++lb;
        c->packed_lab.ensure(n / (32 >> lb) + 2, s);
        launch_count_cuts_packed(e, m, lab, n, lb, c->packed_lab.p, d, d_neg, s);
        c->kernels += 2;
    }
    unsigned long long cut_known = h[0];
    CK(cudaMemcpyAsync(h.data(), d, sizeof(unsigned long long) * (cap + 2), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (known_cut >= 0 && !(neg & 4)) h[0] = cut_known;
    memcpy(&neg, ((char*)&h[1]) + sizeof(int), sizeof(int));
    if (neg & 1) fail(GREM_E_FORMAT, "unlabeled endpoint encountered");
    int64_t np = mx >= 0 ? (int64_t)mx + 1 : 1;
    if (rep) {
        rep->total_edges = m;
        rep->cut_edges = (int64_t)h[0];
        rep->num_parts = np;
        if (rep->partition_sizes) {
            if (np > rep->sizes_cap) fail(GREM_E_FORMAT, "partition_sizes buffer too small");
            for (int64_t k = 0; k < np; ++k) rep->partition_sizes[k] = (int64_t)h[2 + k];
        }
    }
}

// ------------------------------------------------------------ ingest
// host (pageable) edges -> HBM through two pinned staging buffers, so the
// copy engine overlaps the host-side copy of the next block.
void ensure_pinned(grem_ctx* c, size_t bytes) {
    if (c->pin_bytes >= bytes) return;
    for (int i = 0; i < 2; ++i) {
        if (c->pin_buf[i]) cudaFreeHost(c->pin_buf[i]);
        c->pin_buf[i] = nullptr;
        CK(cudaHostAlloc(&c->pin_buf[i], bytes, cudaHostAllocDefault));
        if (!c->pin_ev[i]) CK(cudaEventCreateWithFlags(&c->pin_ev[i], cudaEventDisableTiming));
    }
    c->pin_bytes = bytes;
}

template <class Fill>
void staged_upload(grem_ctx* c, void* dst, uint64_t total, Fill fill) {
    const size_t block = 64ull << 20;
    ensure_pinned(c, block);
    uint64_t off = 0;
    int k = 0;
    bool used[2] = {false, false};
    while (off < total) {
        size_t len = total - off < block ? (size_t)(total - off) : block;
        int i = k & 1;
        if (used[i]) CK(cudaEventSynchronize(c->pin_ev[i]));
        fill(c->pin_buf[i], off, len);
        CK(cudaMemcpyAsync((char*)dst + off, c->pin_buf[i], len, cudaMemcpyHostToDevice, c->s));
        CK(cudaEventRecord(c->pin_ev[i], c->s));
        used[i] = true;
        off += len;
        k++;
    }
    CK(cudaStreamSynchronize(c->s));
}

// file ingest: wait for / stop the reader thread of load_grpe
void ingest_join(grem_ctx* c) {
    if (!c->ing_live) return;
    c->ing_thr.join();
    c->ing_live = false;
}
void ingest_reader_failed(grem_ctx* c) {
    std::string msg;
    {
        std::lock_guard<std::mutex> lk(c->ing_mu);
        msg = c->ing_err;
    }
    if (!msg.empty()) fail(GREM_E_FORMAT, msg);
}

// make c->s wait until the ingested edges [base, end) are resident and checked
// (file ingest: first block the host until the reader has queued that piece)
void ingest_wait(grem_ctx* c, const uint2* end) {
    if (!c->ingest_base || end <= c->ingest_base || end > c->ingest_base + c->ingest_m) return;
    int64_t idx = end - c->ingest_base;
    {
        std::unique_lock<std::mutex> lk(c->ing_mu);
        if (c->ing_live) c->ing_cv.wait(lk, [&] { return c->ing_pub >= idx || c->ing_done; });
        for (auto& mk : c->ingest)
            if (mk.end >= idx) {
                CK(cudaStreamWaitEvent(c->s, mk.ev, 0));
                return;
            }
    }
    ingest_reader_failed(c);
    fail(GREM_E_FORMAT, "ingest: edges not staged");
}
void ingest_wait_all(grem_ctx* c) {
    if (!c->ingest_base) return;
    ingest_join(c);
    ingest_reader_failed(c);
    if (!c->ingest.empty()) CK(cudaStreamWaitEvent(c->s, c->ingest.back().ev, 0));
}
// end of a call: every piece consumed; raise the reference's FormatError if an
// endpoint was out of range (edgefile.py:63-65)
void ingest_finish(grem_ctx* c) {
    if (!c->ingest_base) return;
    ingest_wait_all(c);
    CK(cudaMemcpyAsync(&c->h_pin[0], c->d_bad, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->s));
    CK(cudaStreamSynchronize(c->s));
    unsigned long long bad = (unsigned long long)c->h_pin[0];
    for (auto& mk : c->ingest) cudaEventDestroy(mk.ev);
    c->ingest.clear();
    int64_t n = c->ingest_n;
    c->ingest_base = nullptr;
    if (bad)
        fail(GREM_E_FORMAT, "edge endpoint " + std::to_string(bad - 1) + " >= num_nodes " + std::to_string(n));
}
void ingest_abort(grem_ctx* c) {
    {
        std::lock_guard<std::mutex> lk(c->ing_mu);
        c->ing_stop = true;
    }
    ingest_join(c);
    if (c->copy_s) cudaStreamSynchronize(c->copy_s);
    if (c->check_s) cudaStreamSynchronize(c->check_s);
    for (auto& mk : c->ingest) cudaEventDestroy(mk.ev);
    c->ingest.clear();
    c->ingest_base = nullptr;
}

// the id check of a piece just queued on copy_s, on check_s; returns the
// event consumers wait for (piece copied and checked)
cudaEvent_t check_piece_async(grem_ctx* c, uint2* piece, int64_t cnt, uint32_t n) {
    cudaEvent_t copied, ev;
    CK(cudaEventCreateWithFlags(&copied, cudaEventDisableTiming));
    CK(cudaEventRecord(copied, c->copy_s));
    CK(cudaStreamWaitEvent(c->check_s, copied, 0));
    cudaEventDestroy(copied);
    launch_check_piece(piece, cnt, n, c->d_bad, c->check_s);
    CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CK(cudaEventRecord(ev, c->check_s));
    return ev;
}

// copy stream + bad-id flag for an overlapped ingest into dst (ordered after
// the buffer's stream-ordered allocation on c->s)
void ingest_begin(grem_ctx* c, const uint2* dst, int64_t m, int64_t n) {
    if (!c->copy_s) {   // highest priority: the per-piece id checks must not queue behind SM-filling round kernels
        int lo = 0, hi = 0;
        CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        static const bool low = getenv("GREM_COPY_PRIO_LOW") != nullptr;   // A/B switch
        CK(cudaStreamCreateWithPriority(&c->copy_s, cudaStreamNonBlocking, low ? lo : hi));
        CK(cudaStreamCreateWithPriority(&c->check_s, cudaStreamNonBlocking, low ? lo : hi));
    }
    if (!c->d_bad) CK(cudaMalloc(&c->d_bad, sizeof(unsigned long long)));
    cudaEvent_t ready;
    CK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    CK(cudaEventRecord(ready, c->s));
    CK(cudaStreamWaitEvent(c->copy_s, ready, 0));
    cudaEventDestroy(ready);
    CK(cudaMemsetAsync(c->d_bad, 0, sizeof(unsigned long long), c->copy_s));
    c->ingest_base = dst;
    c->ingest_m = m;
    c->ingest_n = n;
}

const uint2* stage_edges(grem_ctx* c, const uint32_t* edges, int64_t m, int64_t n, int on_device,
                         bool overlap = false) {
    if (n < 1) fail(GREM_E_FORMAT, "num_nodes must be >= 1");
    if (n >= (1LL << 31)) fail(GREM_E_FORMAT, "num_nodes >= 2^31 is not supported by the GPU path");
    const uint2* d;
    c->staged_last = !(on_device || m == 0);
    c->staged_m = m;
    if (on_device || m == 0) {
        d = reinterpret_cast<const uint2*>(edges);
    } else {
        c->edges_owned.ensure(m, c->s);
        cudaPointerAttributes at{};
        bool pinned = cudaPointerGetAttributes(&at, edges) == cudaSuccess && at.type == cudaMemoryTypeHost;
        cudaGetLastError();
        if (pinned && overlap) {   // page-locked source: DMA pieces overlapped with the first bisection
            uint2* dst = c->edges_owned.p;
            ingest_begin(c, dst, m, n);
            const int64_t piece = 1LL << 24;   // 128 MB of edges per DMA
            for (int64_t off = 0; off < m; off += piece) {
                int64_t cnt = m - off < piece ? m - off : piece;
                CK(cudaMemcpyAsync(dst + off, edges + 2 * off, (size_t)cnt * 8, cudaMemcpyHostToDevice, c->copy_s));
                c->ingest.push_back({off + cnt, check_piece_async(c, dst + off, cnt, (uint32_t)n)});
            }
            return dst;
        } else if (pinned) {   // page-locked source: DMA straight into HBM
            PhaseScope ps(c, PH_INGEST);
            CK(cudaMemcpyAsync(c->edges_owned.p, edges, (size_t)m * 8, cudaMemcpyHostToDevice, c->s));
            CK(cudaStreamSynchronize(c->s));
        } else {        // pageable: two pinned staging buffers, copy engine overlapped with memcpy
            staged_upload(c, c->edges_owned.p, (uint64_t)m * 8,
                          [&](void* buf, uint64_t off, size_t len) { memcpy(buf, (const char*)edges + off, len); });
        }
        d = c->edges_owned.p;
    }
    if (m > 0) {
        // _check_ids (edgefile.py:63-65)
        unsigned long long* tmp;
        c->cc_sizes.ensure(4, c->s);
        tmp = c->cc_sizes.p;
        CK(cudaMemsetAsync(tmp, 0, sizeof(unsigned long long), c->s));
        launch_check_ids(d, m, (uint32_t*)tmp, c->s);
        CK(cudaMemcpyAsync(&c->h_pin[0], tmp, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->s));
        CK(cudaStreamSynchronize(c->s));
        uint32_t mx;
        memcpy(&mx, &c->h_pin[0], sizeof(uint32_t));
        if ((int64_t)mx >= n)
            fail(GREM_E_FORMAT, "edge endpoint " + std::to_string(mx) + " >= num_nodes " + std::to_string(n));
    }
    return d;
}

struct GrpeHeader {
    int64_t n, m;
};

GrpeHeader read_grpe_header(const char* path) {
    FILE* f = fopen(path, "rb");
    if (!f) fail(GREM_E_FORMAT, std::string(path) + ": cannot open");
    unsigned char h[28];
    size_t got = fread(h, 1, 28, f);
    fseek(f, 0, SEEK_END);
    long long size = ftell(f);
    fclose(f);
    if (got < 28) fail(GREM_E_FORMAT, std::string(path) + ": too short for a binary edge header");
    if (memcmp(h, "GRPE", 4) != 0) fail(GREM_E_FORMAT, std::string(path) + ": bad magic");
    uint32_t version, flags;
    uint64_t n, m;
    memcpy(&version, h + 4, 4);
    memcpy(&flags, h + 8, 4);
    memcpy(&n, h + 12, 8);
    memcpy(&m, h + 20, 8);
    if (version != 1) fail(GREM_E_FORMAT, std::string(path) + ": unsupported version");
    if (flags & 1) fail(GREM_E_FORMAT, std::string(path) + ": 64-bit ids are parsed by the Python layer");
    if ((uint64_t)size != 28 + m * 8)
        fail(GREM_E_FORMAT, std::string(path) + ": payload length does not match header num_edges");
    return GrpeHeader{(int64_t)n, (int64_t)m};
}

// GRPE u32 file -> HBM (edgefile.py:107-126,186-219), overlapped with the
// path: a reader thread preads 128 MB pieces with GREM_INGEST_THREADS threads
// into a ring of pinned slots, queues each piece's DMA and id check on copy_s
// and publishes its mark; the bisection waits only for the pieces covering the
// chunk it is about to read (ingest_wait), so reading the file overlaps the
// first chunks' work.  Bad ids raise the reference's FormatError at the end.
void ensure_ring(grem_ctx* c) {
    const size_t bytes = 128ull << 20;
    if (c->ring_bytes == bytes) return;
    for (int i = 0; i < grem_ctx::RING; ++i) {
        CK(cudaHostAlloc(&c->ring[i], bytes, cudaHostAllocDefault));
        CK(cudaEventCreateWithFlags(&c->ring_ev[i], cudaEventDisableTiming));
    }
    c->ring_bytes = bytes;
}

void ingest_reader(grem_ctx* c, std::string path, uint2* dst, int64_t m, uint32_t n) {
    int fd = -1;
    try {
        CK(cudaSetDevice(c->device));
        fd = open(path.c_str(), O_RDONLY);
        if (fd < 0) fail(GREM_E_FORMAT, path + ": cannot open");
        static const int threads = [] {
            const char* v = getenv("GREM_INGEST_THREADS");
            int hw = (int)std::thread::hardware_concurrency();
            int t = v ? atoi(v) : (hw < 16 ? hw : 16);
            return t < 1 ? 1 : t;
        }();
        int64_t piece = (int64_t)(c->ring_bytes / 8);
        if (const char* v = getenv("GREM_INGEST_PIECE")) {   // test knob: piece size in edges
            int64_t pv = atoll(v);
            if (pv > 0 && pv < piece) piece = pv;
        }
        for (int64_t off = 0, i = 0; off < m; off += piece, ++i) {
            {
                std::lock_guard<std::mutex> lk(c->ing_mu);
                if (c->ing_stop) break;
            }
            int64_t cnt = m - off < piece ? m - off : piece;
            int slot = (int)(i % grem_ctx::RING);
            if (i >= grem_ctx::RING) CK(cudaEventSynchronize(c->ring_ev[slot]));   // slot's previous DMA done
            char* buf = (char*)c->ring[slot];
            const size_t bytes = (size_t)cnt * 8;
            const off_t base = 28 + (off_t)off * 8;
            size_t part = (bytes + threads - 1) / threads;
            part = (part + 4095) & ~(size_t)4095;
            std::vector<std::thread> ws;
            std::vector<char> ok(threads, 1);
            for (int t = 0; t < threads; ++t) {
                size_t lo = (size_t)t * part;
                if (lo >= bytes) break;
                size_t hi = lo + part < bytes ? lo + part : bytes;
                ws.emplace_back([=, &ok] {
                    size_t done = lo;
                    while (done < hi) {
                        ssize_t r = pread(fd, buf + done, hi - done, base + (off_t)done);
                        if (r <= 0) {
                            ok[t] = 0;
                            return;
                        }
                        done += (size_t)r;
                    }
                });
            }
            for (auto& w : ws) w.join();
            for (char o : ok)
                if (!o) fail(GREM_E_FORMAT, path + ": truncated payload");
            CK(cudaMemcpyAsync(dst + off, buf, bytes, cudaMemcpyHostToDevice, c->copy_s));
            CK(cudaEventRecord(c->ring_ev[slot], c->copy_s));
            cudaEvent_t ev = check_piece_async(c, dst + off, cnt, n);
            {
                std::lock_guard<std::mutex> lk(c->ing_mu);
                c->ingest.push_back({off + cnt, ev});
                c->ing_pub = off + cnt;
            }
            c->ing_cv.notify_all();
        }
    } catch (const GremError& e) {
        std::lock_guard<std::mutex> lk(c->ing_mu);
        c->ing_err = e.msg;
    } catch (const std::exception& e) {
        std::lock_guard<std::mutex> lk(c->ing_mu);
        c->ing_err = e.what();
    }
    if (fd >= 0) close(fd);
    {
        std::lock_guard<std::mutex> lk(c->ing_mu);
        c->ing_done = true;
    }
    c->ing_cv.notify_all();
}

const uint2* load_grpe(grem_ctx* c, const char* path, GrpeHeader* hd) {
    *hd = read_grpe_header(path);
    int64_t m = hd->m, n = hd->n;
    c->staged_last = false;
    c->staged_m = m;
    if (n < 1) fail(GREM_E_FORMAT, "num_nodes must be >= 1");
    if (n >= (1LL << 31)) fail(GREM_E_FORMAT, "num_nodes >= 2^31 is not supported by the GPU path");
    if (m == 0) return nullptr;
    c->edges_owned.ensure(m, c->s);
    ensure_ring(c);
    uint2* dst = c->edges_owned.p;
    ingest_begin(c, dst, m, n);
    {
        std::lock_guard<std::mutex> lk(c->ing_mu);
        c->ing_pub = 0;
        c->ing_done = false;
        c->ing_stop = false;
        c->ing_err.clear();
    }
    c->ing_live = true;
    c->ing_thr = std::thread(ingest_reader, c, std::string(path), dst, m, (uint32_t)n);
    return dst;
}

void bisect_entry(grem_ctx* c, const uint2* d, int64_t m, int64_t n, const grem_config* cfg, int64_t capacity,
                  const grem_hooks* hooks, int32_t* labels_out, grem_report* rep) {
    validate_cfg(cfg);
    BisectArgs a;
    a.e = d;
    a.m = m;
    a.n = n;
    a.chunk = plan_chunk(cfg, m);
    a.cap = capacity > 0 ? capacity : (long long)std::ceil((1.0 + cfg->capacity_slack) * (double)n / 2);
    a.refine = cfg->refine;
    a.passes = cfg->passes;
    a.seed_algo = cfg->seed_algo;
    a.seed_passes = cfg->seed_refinement_passes;
    a.hooks = hooks;
    bisect_core(c, a);
    c->lab32.ensure(n, c->s);
    launch_labels_to_i32(c->lab.p, n, c->lab32.p, c->s);
    c->kernels++;
    if (rep) count_cuts_dev(c, d, m, c->lab32.p, n, rep);
    if (labels_out) CK(cudaMemcpyAsync(labels_out, c->lab32.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, c->s));
    CK(cudaStreamSynchronize(c->s));
}

// Stream priorities: the root context carries the dense chain of the
// recursion (the larger side always stays on it), child contexts the smaller
// subtrees.  GREM_PRIO: 0 = none, 1 = root high, 2 = children high.
// SM partitions (green contexts, driver API): once a recursion has split into
// the dense chain and its sibling subtrees, the chain runs on a "dense"
// partition and every child context on a "sparse" one, so the
// latency-bound rounds of the sparse subtrees stop queueing behind the
// chain's SM-filling kernels (and vice versa).  GREM_GREEN_SPARSE_SMS (a
// multiple of 8; default 0 = off): the sparse partition's SM count.  Streams
// of both partitions share the device's memory pool with the primary context
// (checked by tools/micro/green_test.cu on a B200).  Measured slower than
// sharing the whole GPU (papers100M k=16: 16 / 32 / 48 SMs -> 1050 / 672 /
// 610 ms vs 588 ms, profiles/r02_ab_green.txt): the sparse subtrees need more
// than a slice, and the chain loses the SMs it would have borrowed.
struct GreenParts {
    bool ok = false;
    CUgreenCtx dense = nullptr, sparse = nullptr;
};
// driver-API entry points through the runtime (the library does not link
// libcuda, so it still loads where no driver is installed)
struct GreenApi {
    decltype(&::cuDeviceGet) deviceGet = nullptr;
    decltype(&::cuDeviceGetDevResource) getDevResource = nullptr;
    decltype(&::cuDevSmResourceSplitByCount) smSplit = nullptr;
    decltype(&::cuDevResourceGenerateDesc) genDesc = nullptr;
    decltype(&::cuGreenCtxCreate) ctxCreate = nullptr;
    decltype(&::cuGreenCtxStreamCreate) streamCreate = nullptr;
    bool load() {
        auto get = [](const char* name, void** fn) {
            cudaDriverEntryPointQueryResult q;
            return cudaGetDriverEntryPointByVersion(name, fn, CUDA_VERSION, cudaEnableDefault, &q) == cudaSuccess &&
                   q == cudaDriverEntryPointSuccess && *fn;
        };
        return get("cuDeviceGet", (void**)&deviceGet) && get("cuDeviceGetDevResource", (void**)&getDevResource) &&
               get("cuDevSmResourceSplitByCount", (void**)&smSplit) &&
               get("cuDevResourceGenerateDesc", (void**)&genDesc) && get("cuGreenCtxCreate", (void**)&ctxCreate) &&
               get("cuGreenCtxStreamCreate", (void**)&streamCreate);
    }
};
GreenApi g_green_api;
GreenParts* green_parts(int device) {
    static std::mutex mu;
    static GreenParts parts[16];
    static bool tried[16] = {false};
    std::lock_guard<std::mutex> lk(mu);
    if (device < 0 || device >= 16) return nullptr;
    GreenParts& g = parts[device];
    if (!tried[device]) {
        tried[device] = true;
        int want = getenv("GREM_GREEN_SPARSE_SMS") ? atoi(getenv("GREM_GREEN_SPARSE_SMS")) : 0;
        CUdevice dev;
        CUdevResource res, grp[1], rest;
        unsigned nb = 1;
        CUdevResourceDesc dd, ds;
        GreenApi& A = g_green_api;
        if (want > 0 && A.load() && A.deviceGet(&dev, device) == CUDA_SUCCESS &&
            A.getDevResource(dev, &res, CU_DEV_RESOURCE_TYPE_SM) == CUDA_SUCCESS &&
            (int)res.sm.smCount > 2 * want &&
            A.smSplit(grp, &nb, &res, &rest, 0, (unsigned)want) == CUDA_SUCCESS && nb == 1 &&
            A.genDesc(&ds, grp, 1) == CUDA_SUCCESS &&
            A.genDesc(&dd, &rest, 1) == CUDA_SUCCESS &&
            A.ctxCreate(&g.sparse, ds, dev, CU_GREEN_CTX_DEFAULT_STREAM) == CUDA_SUCCESS &&
            A.ctxCreate(&g.dense, dd, dev, CU_GREEN_CTX_DEFAULT_STREAM) == CUDA_SUCCESS)
            g.ok = true;
        cudaGetLastError();
    }
    return g.ok ? &g : nullptr;
}

void init_ctx(grem_ctx* c, int device, bool child = false) {
    c->device = device;
    CK(cudaSetDevice(device));
    static const int prio_mode = getenv("GREM_PRIO") ? atoi(getenv("GREM_PRIO")) : 1;
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    bool high = (prio_mode == 1 && !child) || (prio_mode == 2 && child);
    GreenParts* gp = green_parts(device);
    CUstream cs = nullptr;
    if (child && gp && g_green_api.streamCreate(&cs, gp->sparse, CU_STREAM_NON_BLOCKING,
                                              (prio_mode && high) ? hi : lo) == CUDA_SUCCESS)
        c->s = (cudaStream_t)cs;
    else
        CK(cudaStreamCreateWithPriority(&c->s, cudaStreamNonBlocking, (prio_mode && high) ? hi : lo));
    if (!child && gp && g_green_api.streamCreate(&cs, gp->dense, CU_STREAM_NON_BLOCKING,
                                               prio_mode == 1 ? hi : lo) == CUDA_SUCCESS)
        c->s_dense = (cudaStream_t)cs;
    CK(cudaEventCreate(&c->ev0));
    CK(cudaEventCreate(&c->ev1));
    CK(cudaMalloc(&c->d_sizes, sizeof(long long) * 2));
    CK(cudaMalloc(&c->d_scal, sizeof(long long) * 16));
    CK(cudaMalloc(&c->d_sscal, sizeof(long long) * 16));
    CK(cudaHostAlloc(&c->h_pin, sizeof(long long) * 32, cudaHostAllocDefault));
    ensure_temp(c, 1 << 20);
}

// A subtree position (level, leaf base) always gets the same child context,
// so its workspaces are sized once and reused by later calls.
// free device memory below `frac` of the device: deep recursions (k >= 64 on
// the 1.8B-edge Friendster shape) then stop opening concurrent child contexts
// and hand finished children's workspaces back to the pool
// cudaMemGetInfo is not free (it stalled the concurrent subtrees when called
// per recursion node): the partition entry samples it once (mem_sample), and
// recursion nodes only read the pool's reserved size, a host-side query
struct MemModel {
    int device = -1;
    double total = 0, other = 0;   // device bytes; bytes held outside the stream-ordered pool
};
MemModel g_mem;
std::mutex g_mem_mu;
double pool_attr(int device, cudaMemPoolAttr attr) {
    cudaMemPool_t pool;
    unsigned long long r = 0;
    if (cudaDeviceGetDefaultMemPool(&pool, device) != cudaSuccess) return 0;
    if (cudaMemPoolGetAttribute(pool, attr, &r) != cudaSuccess) return 0;
    return (double)r;
}
double pool_reserved(int device) { return pool_attr(device, cudaMemPoolAttrReservedMemCurrent); }
void mem_sample(int device) {
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) return;
    std::lock_guard<std::mutex> lk(g_mem_mu);
    g_mem.device = device;
    g_mem.total = (double)total_b;
    g_mem.other = (double)total_b - (double)free_b - pool_reserved(device);
}
bool mem_low(double frac, int device) {
    MemModel m;
    {
        std::lock_guard<std::mutex> lk(g_mem_mu);
        m = g_mem;
    }
    if (m.device != device || m.total <= 0) return false;
    // memory in use by live allocations (the pool may also hold freed blocks
    // it has not released yet: those are reusable, so they count as free)
    double used = pool_attr(device, cudaMemPoolAttrUsedMemCurrent);
    bool low = m.total - m.other - used < frac * m.total;
    static const bool dbg = getenv("GREM_DEBUG_MEM") != nullptr;
    if (low && dbg)
        fprintf(stderr, "[mem] low: %.1f GB free of %.1f (other %.1f, pool used %.1f)\n",
                (m.total - m.other - used) / 1e9, m.total / 1e9, m.other / 1e9, used / 1e9);
    return low;
}

// A bounded pool of child contexts (GREM_MAX_CTX, default 24): an idle one
// that last ran the same subtree position is preferred (its workspaces have
// the right sizes), else any idle one, else a new one below the cap; at the
// cap the caller runs the sibling on its own context.  One context per subtree
// position (round 1) held k-1 sets of workspaces across calls, which at
// Friendster k=256 filled the device and serialised later calls.
grem_ctx* ctx_acquire(grem_ctx* root, long long key) {
    static const size_t kMaxCtx = getenv("GREM_MAX_CTX") ? (size_t)atoi(getenv("GREM_MAX_CTX")) : 24;
    grem_ctx* ch = nullptr;
    {
        std::lock_guard<std::mutex> lk(root->pool_mu);
        for (auto& kv : root->pool_keyed)
            if (kv.first == key && !kv.second->busy) ch = kv.second;
        if (!ch)
            for (grem_ctx* c2 : root->pool_all)
                if (!c2->busy) {
                    ch = c2;
                    break;
                }
        if (!ch) {
            if (root->pool_all.size() >= kMaxCtx) return nullptr;
            ch = new grem_ctx();
            ch->root = root;
            init_ctx(ch, root->device, true);
            root->pool_all.push_back(ch);
        }
        bool keyed = false;
        for (auto& kv : root->pool_keyed)
            if (kv.second == ch) {
                kv.first = key;
                keyed = true;
            }
        if (!keyed) root->pool_keyed.push_back({key, ch});
        ch->busy = true;
    }
    memset(&ch->stats, 0, sizeof(ch->stats));
    ch->kernels = 0;
    for (int k = 0; k < PH_N; ++k) {
        ch->phase_ms[k] = 0;
        ch->phase_n[k] = 0;
        ch->phase_bytes[k] = 0;
    }
    ch->prof_open.clear();
    ch->ev_used = 0;
    ch->profiling = root->profiling;
    return ch;
}

// fold a finished child's counters into its parent (stream already synchronised)
// Workspaces of child contexts that are not running a subtree go back to the
// pool (a deep recursion leaves one context per subtree position holding its
// buffers: Friendster k=256 otherwise ran its next call with siblings
// serialised for lack of memory, 4.5 s instead of 2.1 s)
void trim_idle_children(grem_ctx* root) {
    std::lock_guard<std::mutex> lk(root->pool_mu);
    for (grem_ctx* ch : root->pool_all) {
        if (ch->busy) continue;
        cudaStreamSynchronize(ch->s);
        if (ch->aux_s) cudaStreamSynchronize(ch->aux_s);
        ctx_trim_buffers(ch);
        ch->ws_m = 0;
    }
}

void ctx_release(grem_ctx* parent, grem_ctx* ch) {
    prof_collect(ch);
    // the finished subtree's induced subgraphs are dead: hand the level arenas
    // back to the pool (stream-ordered; the pool keeps the memory, so the next
    // subtree re-allocates without the OS).  A pooled context otherwise keeps
    // the union of every subtree's arenas it ever ran (Friendster k=256 repeat
    // calls crept into low-memory serialisation).
    // Only when the device is half full: re-allocating the arenas every call
    // made the pool grow and fragment (papers100M k=16 calls 2-3 ran 100 ms
    // slower than the rest)
    if (mem_low(0.5, ch->device))
        for (int l = 0; l < 40; ++l) {
            ch->rec_e[l].release_async(ch->s);
            ch->rec_o[l].release_async(ch->s);
        }
    {
        std::lock_guard<std::mutex> lk(parent->root->pool_mu);
        ch->busy = false;
    }
    grem_ctx* root = parent->root;
    (void)root;
    parent->stats.chunks += ch->stats.chunks;
    parent->stats.rounds += ch->stats.rounds;
    if (ch->stats.max_rounds > parent->stats.max_rounds) parent->stats.max_rounds = ch->stats.max_rounds;
    parent->stats.visits += ch->stats.visits;
    parent->stats.walk_steps += ch->stats.walk_steps;
    parent->stats.seed_bfs_levels += ch->stats.seed_bfs_levels;
    parent->stats.bisections += ch->stats.bisections;
    parent->stats.count_bytes += ch->stats.count_bytes;
    parent->stats.delta_bytes += ch->stats.delta_bytes;
    parent->stats.path_bytes += ch->stats.path_bytes;
    parent->kernels += ch->kernels;
    for (int k = 0; k < PH_N; ++k) {
        parent->phase_ms[k] += ch->phase_ms[k];
        parent->phase_n[k] += ch->phase_n[k];
        parent->phase_bytes[k] += ch->phase_bytes[k];
    }
}

// partition (grem.py:277-319): depth-first like the reference; both sides
// are extracted (device-resident, file order kept) before recursing, so the
// parent's labels can be overwritten by the child bisections.
struct PartCtx {
    int64_t total_nodes;
    const grem_config* cfg;
    const grem_hooks* hooks;
    int32_t* final_lab;
    int shard_rank = 0;   // multi-GPU subtree sharding: this process's rank
    // single-GPU partition: the final cut, accumulated while recursing (edges
    // dropped by every extraction + cut edges of every leaf bisection)
    std::atomic<long long> cut{0};
    bool track_cut = false;
    // GREM_DEFER=1: the smaller sides split off the root context's chain run
    // after that chain (concurrently with each other) instead of alongside it
    struct Deferred {
        grem_ctx* ch;
        cudaEvent_t ready;
        std::function<void()> run;
    };
    std::vector<Deferred> deferred;
};

// ranks [r0, r1) own this recursion node; a node with several owners is
// computed redundantly (bit-identical) by each of them
void recurse(grem_ctx* c, PartCtx& pc, const uint2* e, int64_t m, int64_t n, const int32_t* orig, int64_t p_level,
             int level, int64_t leaf_base, int r0 = 0, int r1 = 1) {
    cudaStream_t s = c->s;
    if (level >= 39) fail(GREM_E_FORMAT, "partition depth exceeds 2^39 parts");
    double capd = std::ceil((1.0 + pc.cfg->capacity_slack) * (double)pc.total_nodes / (double)(1LL << (level + 1)));
    BisectArgs a;
    a.e = e;
    a.m = m;
    a.n = n;
    a.chunk = plan_chunk(pc.cfg, m);
    a.cap = (long long)capd;
    a.refine = pc.cfg->refine;
    a.passes = pc.cfg->passes;
    a.seed_algo = pc.cfg->seed_algo;
    a.seed_passes = pc.cfg->seed_refinement_passes;
    a.hooks = pc.hooks ? pc.hooks : nullptr;
    grem_hooks sub = pc.hooks ? *pc.hooks : grem_hooks{nullptr, nullptr, nullptr, nullptr};
    sub.on_chunk = nullptr;   // partition() passes only the meter down (grem.py:300)
    a.hooks = &sub;
    bisect_core(c, a);
    if (p_level == 2) {
        launch_leaf_write(c->lab.p, n, orig, (int32_t)leaf_base, pc.final_lab, s);
        c->kernels++;
        if (pc.track_cut) {
            ingest_wait_all(c);
            PhaseScope ps(c, PH_CUTS);
            launch_bisect_cut(e, m, c->lab.p, reinterpret_cast<unsigned long long*>(c->d_scal + 12), s);
            c->kernels++;
            scal_read(c, c->d_scal + 12, 1);
            pc.cut += c->h_pin[0];
        }
        return;
    }
    ingest_wait_all(c);
    // extract both sides: one pass over the edges writes both induced subgraphs
    c->rec_e[level].ensure(m > 0 ? m : 1, s);   // both sides in one arena (launch_split_edges)
    c->rec_o[level].ensure(n, s);
    uint2* side_e[2] = {c->rec_e[level].p, nullptr};
    int32_t* sub_o = c->rec_o[level].p;
    int64_t e_off[3] = {0, 0, 0}, n_off[3] = {0, 0, 0};
    int64_t nw = (n + 31) / 32;
    c->side_bits.ensure(nw + 2, s);
    c->side_pop.ensure(nw + 2, s);
    c->side_pre.ensure(nw + 2, s);
    c->word_info.ensure(nw + 2, s);
    c->lb_status.ensure(2 * (int64_t)split_edges_tiles(m) + 2, s);
    c->lb_ticket.ensure(4, s);
    ensure_temp(c, scan_temp_bytes(nw + 2));
    {
        PhaseScope ps(c, PH_EXTRACT);
        CK(cudaMemsetAsync(c->side_pop.p + nw, 0, sizeof(uint32_t), s));
        launch_side_bits(c->lab.p, n, c->side_bits.p, c->side_pop.p, c->side_pre.p, c->temp.p, c->temp.cap, s);
        launch_split_edges(e, m, c->side_bits.p, c->side_pre.p, nw, c->word_info.p, side_e[0],
                           c->lb_status.p, c->lb_ticket.p, c->d_scal + 6, s);
        CK(cudaMemcpyAsync(&c->h_pin[0], c->side_pre.p + nw, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(&c->h_pin[1], c->d_scal + 6, 2 * sizeof(long long), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        c->kernels += 5;
    }
    uint32_t ones;
    memcpy(&ones, &c->h_pin[0], sizeof(uint32_t));
    n_off[1] = n - (int64_t)ones;
    n_off[2] = n;
    e_off[1] = c->h_pin[1];
    e_off[2] = e_off[1] + c->h_pin[2];
    side_e[1] = side_e[0] + (m - c->h_pin[2]);   // side 1 occupies the arena's last e1 slots
    if (pc.track_cut) pc.cut += m - e_off[2];   // edges with endpoints on different sides: cut for good
    {
        PhaseScope ps(c, PH_EXTRACT);
        launch_reverse_edges(side_e[1], e_off[2] - e_off[1], s);
        for (int side = 0; side < 2; ++side)
            launch_sub_orig_bits(c->lab.p, n, side, c->side_bits.p, c->side_pre.p, orig, sub_o + n_off[side], s);
        c->kernels += 3;
    }
    c->stats.path_bytes += 10 * m + 8 * e_off[2];   // extraction: read, gather, write kept edges
    // split the owning ranks between the sides in proportion to their edges
    int W = r1 - r0, split = r1;
    int sr0[2] = {r0, r0}, sr1[2] = {r1, r1};
    if (W >= 2) {
        double m0 = (double)(e_off[1] - e_off[0]), m1 = (double)(e_off[2] - e_off[1]);
        int w0 = (int)std::floor(W * (m0 + 1.0) / (m0 + m1 + 2.0) + 0.5);
        if (w0 < 1) w0 = 1;
        if (w0 > W - 1) w0 = W - 1;
        split = r0 + w0;
        sr1[0] = split;
        sr0[1] = split;
    }
    auto side_call = [&](grem_ctx* cc, int side) {
        int64_t k = n_off[side + 1] - n_off[side];
        if (k == 0) return;   // grem.py:308-309
        if (pc.shard_rank < sr0[side] || pc.shard_rank >= sr1[side]) return;   // another rank's subtree
        int64_t base = leaf_base + side * (p_level / 2);
        recurse(cc, pc, side_e[side], e_off[side + 1] - e_off[side], k, sub_o + n_off[side], p_level / 2,
                level + 1, base, sr0[side], sr1[side]);
    };
    (void)split;
    // The two sides are independent problems: side 1 runs concurrently on a
    // child context (own stream + host thread) unless a meter is attached
    // (the reference's residency accounting is sequential) or disabled.
    bool mine0 = pc.shard_rank >= sr0[0] && pc.shard_rank < sr1[0];
    bool mine1 = pc.shard_rank >= sr0[1] && pc.shard_rank < sr1[1];
    bool both = (n_off[1] > 0) && (n_off[2] - n_off[1] > 0) && mine0 && mine1;
    static const double kSpawnFree = getenv("GREM_SPAWN_FREE") ? atof(getenv("GREM_SPAWN_FREE")) : 0.15;
    bool par = both && !(pc.hooks && pc.hooks->meter) && !getenv("GREM_SERIAL_SIBLINGS");
    if (par && mem_low(kSpawnFree, c->device)) {   // reclaim idle children first, then decide
        trim_idle_children(c->root);
        par = !mem_low(kSpawnFree, c->device);
    }
    static const bool defer = getenv("GREM_DEFER") && atoi(getenv("GREM_DEFER")) > 0;
    int big = (e_off[1] - e_off[0]) >= (e_off[2] - e_off[1]) ? 0 : 1;   // stays on this context
    grem_ctx* dch = nullptr;
    if (par && defer && c == c->root) {
        dch = ctx_acquire(c->root, ((long long)(level + 1) << 40) | (leaf_base + (1 - big) * (p_level / 2)));
        if (!dch) par = false;
    }
    if (par && defer && c == c->root) {
        cudaEvent_t ready;
        CK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
        CK(cudaEventRecord(ready, s));
        int sm = 1 - big;
        grem_ctx* ch = dch;
        const uint2* se = side_e[sm];
        int64_t sm_m = e_off[sm + 1] - e_off[sm], sm_n = n_off[sm + 1] - n_off[sm];
        const int32_t* so = sub_o + n_off[sm];
        int64_t base = leaf_base + sm * (p_level / 2), pl = p_level / 2;
        int r0s = sr0[sm], r1s = sr1[sm], lv = level + 1;
        PartCtx* ppc = &pc;
        pc.deferred.push_back({ch, ready, [=]() {
                                   CK(cudaSetDevice(ch->device));
                                   CK(cudaStreamWaitEvent(ch->s, ready, 0));
                                   recurse(ch, *ppc, se, sm_m, sm_n, so, pl, lv, base, r0s, r1s);
                                   CK(cudaStreamSynchronize(ch->s));
                               }});
        side_call(c, big);
        return;
    }
    grem_ctx* ch = nullptr;
    if (par && !(defer && c == c->root) && c == c->root && c->s_dense && c->s != c->s_dense) {
        // first split of the recursion: from here on the chain runs on the
        // dense SM partition and the spawned subtrees on the sparse one
        cudaEvent_t ev;
        CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        CK(cudaEventRecord(ev, c->s));
        CK(cudaStreamWaitEvent(c->s_dense, ev, 0));
        CK(cudaEventDestroy(ev));
        c->s_full = c->s;
        c->s = c->s_dense;
    }
    if (par && !(defer && c == c->root)) {
        ch = ctx_acquire(c->root, ((long long)(level + 1) << 40) | (leaf_base + (1 - big) * (p_level / 2)));
        par = ch != nullptr;   // context pool at its cap: siblings in sequence
        if (ch) {   // a context sized for a far bigger subtree first gives its workspaces back
            int64_t ms = e_off[(1 - big) + 1] - e_off[1 - big];
            if (ch->ws_m > 2 * ms + (1 << 22)) {
                CK(cudaStreamSynchronize(ch->s));
                if (ch->aux_s) CK(cudaStreamSynchronize(ch->aux_s));
                ctx_trim_buffers(ch);
                ch->ws_m = 0;
            }
            if (ms > ch->ws_m) ch->ws_m = ms;
        }
    }
    if (par) {
        cudaEvent_t ready;
        CK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
        CK(cudaEventRecord(ready, s));
        std::exception_ptr err = nullptr;
        std::thread th([&] {
            try {
                CK(cudaSetDevice(ch->device));
                CK(cudaStreamWaitEvent(ch->s, ready, 0));
                side_call(ch, 1 - big);
                CK(cudaStreamSynchronize(ch->s));
            } catch (...) {
                err = std::current_exception();
                cudaStreamSynchronize(ch->s);
            }
        });
        std::exception_ptr err0 = nullptr;
        try {
            side_call(c, big);
        } catch (...) {
            err0 = std::current_exception();
        }
        th.join();
        cudaEventDestroy(ready);
        ctx_release(c, ch);
        if (mem_low(kSpawnFree + 0.1, c->device)) ctx_trim_buffers(ch);   // (its stream is synchronised)
        if (err0) std::rethrow_exception(err0);
        if (err) std::rethrow_exception(err);
    } else {
        side_call(c, 0);
        side_call(c, 1);
    }
}

void partition_entry(grem_ctx* c, const uint2* d, int64_t m, int64_t n, int64_t p, const grem_config* cfg,
                     const grem_hooks* hooks, int32_t* labels_out, grem_report* rep, int shard_rank = 0,
                     int shard_world = 1) {
    if (p < 2 || (p & (p - 1)) != 0)
        fail(GREM_E_FORMAT, "number of parts must be a power of two >= 2, got " + std::to_string(p));
    validate_cfg(cfg);
    cudaStream_t s = c->s;
    c->part_fin.ensure(n, s);
    c->part_orig.ensure(n, s);
    int32_t* fin = c->part_fin.p;
    int32_t* orig = c->part_orig.p;
    CK(cudaMemsetAsync(fin, 0xFF, sizeof(int32_t) * n, s));
    launch_iota(orig, n, s);
    if (getenv("GREM_DEBUG_LEVELS")) {
        if (!g_dbg_t0) CK(cudaEventCreate(&g_dbg_t0));
        CK(cudaEventRecord(g_dbg_t0, s));
    }
    mem_sample(c->device);
    struct BackToFull {   // the root context leaves the call on its full-GPU stream again
        grem_ctx* c;
        ~BackToFull() {
            if (!c->s_full) return;
            cudaEvent_t ev;
            if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess) {
                cudaEventRecord(ev, c->s);
                cudaStreamWaitEvent(c->s_full, ev, 0);
                cudaEventDestroy(ev);
            } else {
                cudaStreamSynchronize(c->s);
            }
            c->s = c->s_full;
            c->s_full = nullptr;
        }
    } back_to_full{c};
    PartCtx pc{n, cfg, hooks, fin, shard_rank};
    // incremental cut (extraction drops + per-leaf cut passes) only on request:
    // measured slower and noisier than one final pass (the leaf passes compete
    // with the concurrent sibling leaves; 652 vs 655-700 ms, r02k)
    pc.track_cut = shard_world == 1 && getenv("GREM_INCREMENTAL_CUT");
    try {
        recurse(c, pc, d, m, n, orig, p, 0, 0, 0, shard_world);
        if (!pc.deferred.empty()) {   // GREM_DEFER: the split-off subtrees, concurrently
            std::vector<std::thread> ths;
            std::vector<std::exception_ptr> errs(pc.deferred.size());
            for (size_t i = 0; i < pc.deferred.size(); ++i)
                ths.emplace_back([&, i] {
                    try {
                        pc.deferred[i].run();
                    } catch (...) {
                        errs[i] = std::current_exception();
                        cudaStreamSynchronize(pc.deferred[i].ch->s);
                    }
                });
            for (auto& t : ths) t.join();
            for (auto& dfr : pc.deferred) {
                cudaEventDestroy(dfr.ready);
                ctx_release(c, dfr.ch);
            }
            pc.deferred.clear();
            for (auto& e : errs)
                if (e) std::rethrow_exception(e);
        }
        if (shard_world == 1) {
            count_cuts_dev(c, d, m, fin, n, rep, pc.track_cut ? (long long)pc.cut : -1);
            c->stats.path_bytes += 10 * m;   // final cut pass (SURVEY 8(d) formula; done incrementally here)
        }
        // (c->s: the root may have moved to its dense-partition stream)
        if (labels_out) CK(cudaMemcpyAsync(labels_out, fin, sizeof(int32_t) * n, cudaMemcpyDefault, c->s));
        CK(cudaStreamSynchronize(c->s));
    } catch (...) {
        cudaStreamSynchronize(c->s);
        throw;
    }
    CK(cudaStreamSynchronize(c->s));
}

template <class F>
int guarded(grem_ctx* c, F f) {
    g_err.clear();
    try {
        if (c) {
            CK(cudaSetDevice(c->device));
            memset(&c->stats, 0, sizeof(c->stats));
            c->kernels = 0;
            for (int k = 0; k < PH_N; ++k) {
                c->phase_ms[k] = 0;
                c->phase_n[k] = 0;
                c->phase_bytes[k] = 0;
            }
            c->prof_open.clear();
            c->ev_used = 0;
            CK(cudaEventRecord(c->ev0, c->s));
        }
        f();
        if (c) {
            ingest_finish(c);
            CK(cudaEventRecord(c->ev1, c->s));
            CK(cudaEventSynchronize(c->ev1));
            float ms = 0;
            cudaEventElapsedTime(&ms, c->ev0, c->ev1);
            c->stats.ms_total = ms;
            c->stats.kernels = c->kernels;
            prof_collect(c);
        }
        return GREM_OK;
    } catch (const GremError& e) {
        g_err = e.msg;
        if (c) {
            cudaStreamSynchronize(c->s);
            ingest_abort(c);
        }
        return e.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        if (c) ingest_abort(c);
        return GREM_E_NOMEM;
    }
}

}  // namespace

// every device workspace of one context (stream-ordered frees on its stream)
void ctx_trim_buffers(grem_ctx* c) {
    c->lab.release();
    c->lab2.release();
    c->bsegbad.release();
    c->bsegflag.release();
    c->bin_recs.release();
    c->bin_hist.release();
    c->bin_hist2.release();
    c->bin_offs2.release();
    c->aux_temp.release();
    c->bin_offs.release(); c->bin_ticket.release(); c->bin_hcnt.release(); c->bin_status.release();
    c->bin_hflag.release(); c->tl.release(); c->flag.release(); c->cnt.release(); c->nbr.release();
    c->rank.release(); c->scratch.release(); c->newid.release(); c->rankw.release();
    c->nodes.release(); c->meta.release(); c->bad.release(); c->want.release(); c->newb.release(); c->x.release();
    c->tile_agg.release(); c->tile_x.release(); c->tile_bad.release();
    c->start.release(); c->cursor.release(); c->adj.release(); c->row_of.release();
    c->sortk.release(); c->sortv.release(); c->parent.release();
    c->csize.release(); c->roots.release(); c->rvals.release(); c->rvals2.release(); c->cpos.release();
    c->disc.release(); c->frontier.release(); c->ckey.release(); c->rkeys.release(); c->rkeys2.release();
    c->cand.release(); c->cand2.release(); c->pair.release(); c->slab.release(); c->slab2.release();
    c->fdeg.release(); c->cum.release(); c->temp.release(); c->edges_owned.release(); c->cc_sizes.release();
    c->lab32.release();
    c->packed_lab.release();
    c->side_bits.release();
    c->side_pop.release();
    c->side_pre.release();
    for (int l = 0; l < 40; ++l) {
        c->rec_e[l].release();
        c->rec_o[l].release();
    }
    c->part_fin.release();
    c->part_orig.release();
    c->bk_keys_a.release(); c->bk_keys_b.release(); c->bk_order.release(); c->bk_out.release();
    c->bk_counts.release(); c->ns_cnt.release(); c->ns_k.release(); c->ns_k0.release(); c->ns_pack.release();
    c->sh_keys.release(); c->sh_vals.release();
    c->th_lg.release(); c->th_term.release(); c->th_part.release(); c->th_big.release(); c->th_scal.release();
}

// =============================================================== C ABI

extern "C" {

const char* grem_last_error(void) { return g_err.c_str(); }

grem_ctx* grem_create(int device) {
    g_err.clear();
    grem_ctx* c = new grem_ctx();
    c->root = c;
    try {
        init_ctx(c, device);
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    } catch (const GremError& e) {
        g_err = e.msg;
        delete c;
        return nullptr;
    }
    return c;
}

void grem_destroy(grem_ctx* c) {
    if (!c) return;
    for (grem_ctx* ch : c->pool_all) grem_destroy(ch);
    c->pool_all.clear();
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->s);
    if (c->round_exec) cudaGraphExecDestroy(c->round_exec);
    c->round_exec = nullptr;
    if (c->loop_exec) cudaGraphExecDestroy(c->loop_exec);
    c->loop_exec = nullptr;
    if (c->aux_s) cudaStreamSynchronize(c->aux_s);
    ctx_trim_buffers(c);
    if (c->aux_s) cudaStreamDestroy(c->aux_s);
    if (c->pref_go) cudaEventDestroy(c->pref_go);
    if (c->pref_done) cudaEventDestroy(c->pref_done);
    for (int i = 0; i < 2; ++i) {
        if (c->pin_buf[i]) cudaFreeHost(c->pin_buf[i]);
        if (c->pin_ev[i]) cudaEventDestroy(c->pin_ev[i]);
    }
    for (int i = 0; i < grem_ctx::RING; ++i) {
        if (c->ring[i]) cudaFreeHost(c->ring[i]);
        if (c->ring_ev[i]) cudaEventDestroy(c->ring_ev[i]);
    }
    if (c->d_sizes) cudaFree(c->d_sizes);
    if (c->d_scal) cudaFree(c->d_scal);
    if (c->d_sscal) cudaFree(c->d_sscal);
    if (c->h_pin) cudaFreeHost(c->h_pin);
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    if (c->s) cudaStreamDestroy(c->s);
    if (c->copy_s) cudaStreamDestroy(c->copy_s);
    if (c->check_s) cudaStreamDestroy(c->check_s);
    if (c->d_bad) cudaFree(c->d_bad);
    delete c;
}

int grem_set_profiling(grem_ctx* c, int on) {
    if (!c) return GREM_E_FORMAT;
    c->profiling = on >= 2 ? 2 : (on ? 1 : 0);
    return GREM_OK;
}

int grem_get_phase_times(grem_ctx* c, double* ms_out, int64_t* count_out, int cap, const char** names_out) {
    if (!c) return GREM_E_FORMAT;
    int n = cap < PH_N ? cap : PH_N;
    for (int k = 0; k < n; ++k) {
        if (ms_out) ms_out[k] = c->phase_ms[k];
        if (count_out) count_out[k] = c->phase_n[k];
        if (names_out) names_out[k] = kPhaseNames[k];
    }
    return PH_N;
}

int grem_trim(grem_ctx* c) {
    if (!c) return GREM_E_FORMAT;
    return guarded(nullptr, [&] {
        CK(cudaSetDevice(c->device));
        for (grem_ctx* ch : c->pool_all) {
            CK(cudaStreamSynchronize(ch->s));
            if (ch->aux_s) CK(cudaStreamSynchronize(ch->aux_s));
            ctx_trim_buffers(ch);
        }
        CK(cudaStreamSynchronize(c->s));
        if (c->aux_s) CK(cudaStreamSynchronize(c->aux_s));
        ctx_trim_buffers(c);
        CK(cudaDeviceSynchronize());
        cudaMemPool_t pool;
        CK(cudaDeviceGetDefaultMemPool(&pool, c->device));
        CK(cudaMemPoolTrimTo(pool, 0));
    });
}

int grem_bucket_edges(grem_ctx* c, uint32_t* dst, int64_t first, int64_t count) {
    if (!c || !dst || first < 0 || count < 0) return GREM_E_FORMAT;
    return guarded(nullptr, [&] {
        if (c->bk_out_m < 0 || first + count > c->bk_out_m)
            fail(GREM_E_FORMAT, "no bucket-ordered edges of that range on the device");
        CK(cudaSetDevice(c->device));
        if (count)
            CK(cudaMemcpyAsync(dst, c->bk_out.p + first, sizeof(uint2) * count, cudaMemcpyDeviceToHost, c->s));
        CK(cudaStreamSynchronize(c->s));
    });
}

int grem_mem_high_water(grem_ctx* c, int64_t* used_high, int64_t* reserved_high, int reset) {
    if (!c) return GREM_E_FORMAT;
    return guarded(nullptr, [&] {   // (no per-call stats reset)
        CK(cudaSetDevice(c->device));
        cudaMemPool_t pool;
        CK(cudaDeviceGetDefaultMemPool(&pool, c->device));
        unsigned long long u = 0, r = 0;
        CK(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &u));
        CK(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemHigh, &r));
        if (used_high) *used_high = (int64_t)u;
        if (reserved_high) *reserved_high = (int64_t)r;
        if (reset) {
            unsigned long long z = 0;
            CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &z));
            CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReservedMemHigh, &z));
        }
    });
}

int grem_get_phase_bytes(grem_ctx* c, double* bytes_out, int cap) {
    if (!c) return GREM_E_FORMAT;
    int n = cap < PH_N ? cap : PH_N;
    for (int k = 0; k < n && bytes_out; ++k) bytes_out[k] = c->phase_bytes[k];
    return PH_N;
}

int grem_get_stats(grem_ctx* c, grem_stats* out) {
    if (!c || !out) return GREM_E_FORMAT;
    *out = c->stats;
    return GREM_OK;
}

int grem_bisect_u32(grem_ctx* c, const uint32_t* edges, int64_t m, int64_t n, int on_device, const grem_config* cfg,
                    int64_t capacity, const grem_hooks* hooks, int32_t* labels_out, grem_report* rep) {
    if (!c || !cfg) return GREM_E_FORMAT;
    return guarded(c, [&] {
        const uint2* d = stage_edges(c, edges, m, n, on_device, true);
        bisect_entry(c, d, m, n, cfg, capacity, hooks, labels_out, rep);
    });
}

int grem_partition_u32(grem_ctx* c, const uint32_t* edges, int64_t m, int64_t n, int on_device, int64_t p,
                       const grem_config* cfg, const grem_hooks* hooks, int32_t* labels_out, grem_report* rep) {
    if (!c || !cfg) return GREM_E_FORMAT;
    return guarded(c, [&] {
        if (p < 2 || (p & (p - 1)) != 0)
            fail(GREM_E_FORMAT, "number of parts must be a power of two >= 2, got " + std::to_string(p));
        const uint2* d = stage_edges(c, edges, m, n, on_device, true);
        partition_entry(c, d, m, n, p, cfg, hooks, labels_out, rep);
    });
}

// ------------------------------------------------ partitioned storage
namespace {
const int32_t* stage_labels(grem_ctx* c, const int32_t* labels, int64_t n, int on_device) {
    if (on_device) return labels;
    c->lab32.ensure(n > 0 ? n : 1, c->s);
    if (n > 0) CK(cudaMemcpyAsync(c->lab32.p, labels, sizeof(int32_t) * n, cudaMemcpyHostToDevice, c->s));
    return c->lab32.p;
}
int64_t label_parts(grem_ctx* c, const int32_t* lab, int64_t n, bool* any_negative = nullptr) {
    c->cc_sizes.ensure(4, c->s);
    int* d_max = reinterpret_cast<int*>(c->cc_sizes.p);
    launch_label_max(lab, n, d_max, c->s);
    CK(cudaMemcpyAsync(&c->h_pin[0], d_max, 2 * sizeof(int), cudaMemcpyDeviceToHost, c->s));
    CK(cudaStreamSynchronize(c->s));
    int mx[2];
    memcpy(mx, &c->h_pin[0], 2 * sizeof(int));
    if (any_negative) *any_negative = mx[1] != 0;
    return mx[0] >= 0 ? (int64_t)mx[0] + 1 : 1;
}
}  // namespace

// write_buckets body on staged edges / labels (store.py:55-104)
static void write_buckets_dev(grem_ctx* c, const uint2* d, int64_t m, int64_t n, const int32_t* lab,
                              uint32_t* out_edges, int out_on_device, uint64_t* counts_out, int64_t counts_cap,
                              int64_t* p_out) {
    cudaStream_t s = c->s;
    ingest_wait_all(c);
    bool neg = false;
    int64_t p = label_parts(c, lab, n, &neg);   // store.py:71-72
    if (p_out) *p_out = p;
    if (p >= 65536) fail(GREM_E_FORMAT, "write_buckets supports fewer than 65536 partitions");
    int64_t nb = p * p;
    if (nb > counts_cap) fail(GREM_E_FORMAT, "counts buffer holds " + std::to_string(counts_cap) +
                                                  " entries, p*p = " + std::to_string(nb));
    c->bk_keys_a.ensure(m + 1, s);
    c->bk_keys_b.ensure(m + 1, s);
    c->bk_counts.ensure(nb, s);
    uint2* out = out_on_device ? reinterpret_cast<uint2*>(out_edges) : nullptr;
    if (!out) {
        c->bk_out.ensure(m + 1, s);
        out = c->bk_out.p;
    }
    ensure_temp(c, bucket_sort_temp_bytes(m));
    int* d_bad = reinterpret_cast<int*>(c->cc_sizes.p) + 2;
    c->packed_lab.ensure(n / 2 + 2, s);   // <= 16-bit packed labels (p < 65536)
    launch_write_buckets(d, m, lab, n, neg, (uint32_t)p, c->bk_keys_a.p, c->bk_keys_b.p, c->packed_lab.p, out,
                         c->bk_counts.p, d_bad, c->temp.p, c->temp.cap, s);
    c->kernels += 4;
    CK(cudaMemcpyAsync(&c->h_pin[1], d_bad, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    int bad;
    memcpy(&bad, &c->h_pin[1], sizeof(int));
    if (bad) fail(GREM_E_FORMAT, "unlabeled endpoint encountered");
    CK(cudaMemcpyAsync(counts_out, c->bk_counts.p, sizeof(uint64_t) * nb, cudaMemcpyDeviceToHost, s));
    if (!out_on_device && out_edges && m > 0)   // (out_edges NULL: kept on the device, grem_bucket_edges)
        CK(cudaMemcpyAsync(out_edges, out, sizeof(uint2) * m, cudaMemcpyDeviceToHost, s));
    c->bk_out_m = out_on_device ? -1 : m;
    CK(cudaStreamSynchronize(s));
}

int grem_write_buckets_u32(grem_ctx* c, const uint32_t* edges, int64_t m, int64_t n, int edges_on_device,
                           const int32_t* labels, int labels_on_device, uint32_t* out_edges, int out_on_device,
                           uint64_t* counts_out, int64_t counts_cap, int64_t* p_out) {
    if (!c || !labels || !counts_out || (m > 0 && !out_edges && out_on_device)) return GREM_E_FORMAT;
    return guarded(c, [&] {
        const uint2* d = stage_edges(c, edges, m, n, edges_on_device);
        write_buckets_dev(c, d, m, n, stage_labels(c, labels, n, labels_on_device), out_edges, out_on_device,
                          counts_out, counts_cap, p_out);
    });
}

int grem_write_buckets_file(grem_ctx* c, const char* path, const int32_t* labels, int labels_on_device,
                            uint32_t* out_edges, int out_on_device, uint64_t* counts_out, int64_t counts_cap,
                            int64_t* p_out) {
    if (!c || !path || !labels || !counts_out) return GREM_E_FORMAT;
    return guarded(c, [&] {
        GrpeHeader hd = read_grpe_header(path);
        if (hd.m > 0 && !out_edges && out_on_device) fail(GREM_E_FORMAT, "out_edges is NULL");
        const uint2* d = load_grpe(c, path, &hd);
        write_buckets_dev(c, d, hd.m, hd.n, stage_labels(c, labels, hd.n, labels_on_device), out_edges,
                          out_on_device, counts_out, counts_cap, p_out);
    });
}

// external_shuffle (edgefile.py:248-327) on staged edges: the shuffled list
// (device) is returned; see launch_shuffle for the permutation.
static const uint2* shuffle_dev(grem_ctx* c, const uint2* d, int64_t m, uint64_t seed) {
    cudaStream_t s = c->s;
    ingest_wait_all(c);
    if (m <= 0) return nullptr;
    // the permutation is done in HBM (2 x m u64 keys + 2 x m u64 values + the
    // sort's temp space): refuse up front, naming the limit, instead of
    // failing an allocation half way (the reference is an external-memory
    // shuffle, edgefile.py:248-327; here the bound is device memory)
    {
        size_t free_b = 0, total_b = 0;
        CK(cudaMemGetInfo(&free_b, &total_b));
        auto have = [](size_t cap_elems, int64_t want) { return cap_elems >= (size_t)want ? (size_t)want : 0; };
        size_t need = 2 * 2 * sizeof(unsigned long long) * (size_t)m + shuffle_temp_bytes(m);
        size_t held = sizeof(unsigned long long) * (have(c->sh_keys.cap, 2 * m) + have(c->sh_vals.cap, 2 * m));
        if (need > held && need - held > free_b) {   // memory the stream-ordered pool holds but does not use
            int dev = 0;
            cudaMemPool_t pool;
            CK(cudaStreamSynchronize(s));
            CK(cudaGetDevice(&dev));
            CK(cudaDeviceGetDefaultMemPool(&pool, dev));
            CK(cudaMemPoolTrimTo(pool, 0));
            CK(cudaMemGetInfo(&free_b, &total_b));
        }
        if (need > held && need - held > free_b)
            fail(GREM_E_NOMEM, "external_shuffle of " + std::to_string(m) + " edges needs " +
                                   std::to_string((need - held) >> 20) + " MiB more device memory than the " +
                                   std::to_string(free_b >> 20) + " MiB free (limit: ~" +
                                   std::to_string(total_b / 40 / 1000000) + " M edges on this GPU)");
    }
    c->sh_keys.ensure(2 * m, s);
    c->sh_vals.ensure(2 * m, s);
    ensure_temp(c, shuffle_temp_bytes(m));
    launch_shuffle(d, m, (unsigned long long)seed, c->sh_keys.p, c->sh_vals.p, c->temp.p, c->temp.cap, s);
    c->kernels += 5;
    return reinterpret_cast<const uint2*>(c->sh_vals.p + m);
}

int grem_shuffle_u32(grem_ctx* c, const uint32_t* edges, int64_t m, int64_t n, int edges_on_device, uint64_t seed,
                     uint32_t* out_edges, int out_on_device) {
    if (!c || (m > 0 && !out_edges)) return GREM_E_FORMAT;
    return guarded(c, [&] {
        const uint2* d = stage_edges(c, edges, m, n, edges_on_device);
        const uint2* r = shuffle_dev(c, d, m, seed);
        if (m > 0) CK(cudaMemcpyAsync(out_edges, r, sizeof(uint2) * m, cudaMemcpyDefault, c->s));
        CK(cudaStreamSynchronize(c->s));
        (void)out_on_device;
    });
}

// GRPE u32 file -> shuffled GRPE u32 file; the payload is written in 128 MB
// pieces (device -> pinned ring slot -> pwrite by GREM_INGEST_THREADS threads)
int grem_shuffle_file(grem_ctx* c, const char* in_path, uint64_t seed, const char* out_path) {
    if (!c || !in_path || !out_path) return GREM_E_FORMAT;
    return guarded(c, [&] {
        GrpeHeader hd;
        const uint2* d = load_grpe(c, in_path, &hd);
        const uint2* r = shuffle_dev(c, d, hd.m, seed);
        int fd = open(out_path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
        if (fd < 0) fail(GREM_E_FORMAT, std::string(out_path) + ": cannot create");
        struct Unlink {   // a failed call leaves no partial output file behind
            const char* path; int fd; bool keep = false;
            ~Unlink() { if (!keep) { if (fd >= 0) close(fd); unlink(path); } }
        } guard{out_path, fd};
        unsigned char h[28];
        uint32_t version = 1, flags = 0;
        uint64_t n = (uint64_t)hd.n, m = (uint64_t)hd.m;
        memcpy(h, "GRPE", 4);
        memcpy(h + 4, &version, 4);
        memcpy(h + 8, &flags, 4);
        memcpy(h + 12, &n, 8);
        memcpy(h + 20, &m, 8);
        bool ok = pwrite(fd, h, 28, 0) == 28;
        if (hd.m > 0) {
            ensure_ring(c);
            const int threads = [] {
                const char* v = getenv("GREM_INGEST_THREADS");
                int hw = (int)std::thread::hardware_concurrency();
                int t = v ? atoi(v) : (hw < 16 ? hw : 16);
                return t < 1 ? 1 : t;
            }();
            const int64_t piece = (int64_t)(c->ring_bytes / 8);
            for (int64_t off = 0; off < hd.m && ok; off += piece) {
                int64_t cnt = hd.m - off < piece ? hd.m - off : piece;
                char* buf = (char*)c->ring[0];
                CK(cudaMemcpyAsync(buf, r + off, (size_t)cnt * 8, cudaMemcpyDeviceToHost, c->s));
                CK(cudaStreamSynchronize(c->s));
                const size_t bytes = (size_t)cnt * 8;
                size_t part = ((bytes + threads - 1) / threads + 4095) & ~(size_t)4095;
                std::vector<std::thread> ws;
                std::vector<char> wok(threads, 1);
                for (int t = 0; t < threads; ++t) {
                    size_t lo = (size_t)t * part;
                    if (lo >= bytes) break;
                    size_t hi = lo + part < bytes ? lo + part : bytes;
                    ws.emplace_back([=, &wok] {
                        size_t done = lo;
                        while (done < hi) {
                            ssize_t w = pwrite(fd, buf + done, hi - done, 28 + (off_t)off * 8 + (off_t)done);
                            if (w <= 0) {
                                wok[t] = 0;
                                return;
                            }
                            done += (size_t)w;
                        }
                    });
                }
                for (auto& w : ws) w.join();
                for (char o : wok) ok = ok && o;
            }
        }
        if (!ok) fail(GREM_E_FORMAT, std::string(out_path) + ": write failed");
        guard.keep = true;
        close(fd);
    });
}

static void node_stats_dev(grem_ctx* c, const uint2* d, int64_t m, int64_t n, const int32_t* lab, int64_t* k_out,
                    int64_t* k0_out) {
    cudaStream_t s = c->s;
    ingest_wait_all(c);
    if (label_parts(c, lab, n) > 2) fail(GREM_E_FORMAT, "reference labels are not a bisection");   // theory.py:107-108
    c->ns_cnt.ensure(2 * n + 2, s);
    c->ns_k.ensure(n + 1, s);
    c->ns_k0.ensure(n + 1, s);
    int* d_bad = reinterpret_cast<int*>(c->cc_sizes.p) + 2;
    c->ns_pack.ensure(n / 16 + 2, s);
    // hubs of the edge list (a 4M-edge degree sample), privatised in shared memory
    static const bool no_hubs = getenv("GREM_NODE_STATS_NO_HUBS") != nullptr;   // A/B switch
    c->hubs_on = false;
    if (!no_hubs && d) {
        c->scratch.ensure(n + 2, s);
        BisectArgs ha{};
        ha.e = d;
        ha.m = m;
        ha.n = n;
        ha.chunk = m;
        detect_hubs(c, ha);
    }
    launch_node_stats(d, m, lab, n, c->ns_cnt.p, c->ns_pack.p, c->ns_k.p, c->ns_k0.p, d_bad, s,
                      c->hubs_on ? c->hub_table.p : nullptr);
    c->kernels += 3;
    CK(cudaMemcpyAsync(&c->h_pin[1], d_bad, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    int bad;
    memcpy(&bad, &c->h_pin[1], sizeof(int));
    if (bad) fail(GREM_E_FORMAT, "unlabeled endpoint encountered");
    CK(cudaMemcpyAsync(k_out, c->ns_k.p, sizeof(int64_t) * n, cudaMemcpyDefault, s));
    CK(cudaMemcpyAsync(k0_out, c->ns_k0.p, sizeof(int64_t) * n, cudaMemcpyDefault, s));
    CK(cudaStreamSynchronize(s));
}

int grem_node_stats_u32(grem_ctx* c, const uint32_t* edges, int64_t m, int64_t n, int edges_on_device,
                        const int32_t* labels, int labels_on_device, int64_t* k_out, int64_t* k0_out) {
    if (!c || !labels || !k_out || !k0_out) return GREM_E_FORMAT;
    return guarded(c, [&] {
        const uint2* d = stage_edges(c, edges, m, n, edges_on_device);
        node_stats_dev(c, d, m, n, stage_labels(c, labels, n, labels_on_device), k_out, k0_out);
    });
}

int grem_node_stats_file(grem_ctx* c, const char* path, const int32_t* labels, int labels_on_device,
                         int64_t* k_out, int64_t* k0_out) {
    if (!c || !path || !labels || !k_out || !k0_out) return GREM_E_FORMAT;
    return guarded(c, [&] {
        GrpeHeader hd;
        const uint2* d = load_grpe(c, path, &hd);
        node_stats_dev(c, d, hd.m, hd.n, stage_labels(c, labels, hd.n, labels_on_device), k_out, k0_out);
    });
}

int grem_theory_curve(grem_ctx* c, const int64_t* k, const int64_t* k0, int64_t n, int on_device, const double* xs,
                      int64_t nx, double multiplier, double* cuts_out, int64_t* info_out) {
    if (!c || (nx > 0 && (!xs || !cuts_out)) || n < 0) return GREM_E_FORMAT;
    return guarded(c, [&] {
        if (info_out) info_out[0] = info_out[1] = -1, info_out[2] = 0;
        if (nx == 0) return;   // theory.py:145-146: nothing evaluated
        if (n == 0) fail(GREM_E_FORMAT, "empty node stats");   // theory.py:131-132
        if (!k || !k0) fail(GREM_E_FORMAT, "null node stats");
        cudaStream_t s = c->s;
        const int64_t* dk = k;
        const int64_t* dk0 = k0;
        if (!on_device) {
            c->ns_k.ensure(n, s);
            c->ns_k0.ensure(n, s);
            CK(cudaMemcpyAsync(c->ns_k.p, k, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(c->ns_k0.p, k0, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
            dk = c->ns_k.p;
            dk0 = c->ns_k0.p;
        }
        c->th_scal.ensure(8, s);
        unsigned long long init[4] = {~0ULL, ~0ULL, 0ULL, 0ULL};
        CK(cudaMemcpyAsync(c->th_scal.p, init, sizeof(init), cudaMemcpyHostToDevice, s));
        launch_theory_check(dk, dk0, n, c->th_scal.p, s);
        c->kernels++;
        unsigned long long chk[4];
        CK(cudaMemcpyAsync(chk, c->th_scal.p, sizeof(chk), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        int64_t first = chk[0] == ~0ULL ? -1 : (int64_t)chk[0];
        int64_t bad = chk[1] == ~0ULL ? -1 : (int64_t)chk[1];
        if (info_out) info_out[0] = first, info_out[1] = bad, info_out[2] = (int64_t)chk[3];
        if (first < 0) {   // every node has k = 0: nothing is evaluated, no domain check runs
            for (int64_t q = 0; q < nx; ++q) cuts_out[q] = 0.0;
            return;
        }
        // prob_correct's checks in its order at the first evaluated node (theory.py:85-92)
        if (bad == first) fail(GREM_E_FORMAT, "k0 must be the majority side");
        for (int64_t q = 0; q < nx; ++q)
            if (!(xs[q] > 0.0 && xs[q] <= 1.0)) fail(GREM_E_FORMAT, "chunk fraction must be in (0, 1]");
        if (multiplier < 1.0) fail(GREM_E_FORMAT, "multiplier must be >= 1");
        if (bad >= 0) fail(GREM_E_FORMAT, "k0 must be the majority side");
        int64_t maxk = (int64_t)chk[2];
        c->th_lg.ensure(maxk + 2, s);
        launch_lgamma_table(c->th_lg.p, maxk + 2, s);
        c->th_term.ensure(n, s);
        c->th_big.ensure(n, s);
        c->th_part.ensure(theory_sum_blocks() + 1, s);
        for (int64_t q = 0; q < nx; ++q) {
            double x_eff = multiplier * xs[q] < 1.0 ? multiplier * xs[q] : 1.0;   // theory.py:73
            launch_expected_cuts(dk, dk0, n, c->th_lg.p, x_eff, c->th_term.p, c->th_big.p, c->th_scal.p + 4,
                                 c->th_part.p, c->th_part.p + theory_sum_blocks(), s);
            c->kernels += 5;
            CK(cudaMemcpyAsync(cuts_out + q, c->th_part.p + theory_sum_blocks(), sizeof(double),
                               cudaMemcpyDeviceToHost, s));
        }
        c->kernels++;
        CK(cudaStreamSynchronize(s));
    });
}

int grem_reorder_records(grem_ctx* c, const int32_t* labels, int64_t n, int labels_on_device, const uint8_t* records,
                         int64_t record_width, uint8_t* out_records, int64_t* perm_out, uint64_t* counts_out,
                         int64_t counts_cap, int64_t* p_out) {
    if (!c || !labels || !perm_out || !counts_out) return GREM_E_FORMAT;
    return guarded(c, [&] {
        cudaStream_t s = c->s;
        if (n < 1) fail(GREM_E_FORMAT, "num_nodes must be >= 1");
        const int32_t* lab = stage_labels(c, labels, n, labels_on_device);
        bool neg = false;
        int64_t p = label_parts(c, lab, n, &neg);
        if (neg) fail(GREM_E_FORMAT, "all nodes must be labeled");   // store.py:216-217
        if (p_out) *p_out = p;
        if (p > counts_cap) fail(GREM_E_FORMAT, "counts buffer too small");
        c->bk_keys_a.ensure(n + 1, s);
        c->bk_keys_b.ensure(n + 1, s);
        c->bk_order.ensure(n + 1, s);
        c->bk_perm.ensure(n + 1, s);
        c->bk_counts.ensure(p, s);
        ensure_temp(c, order_sort_temp_bytes(n));
        uint8_t* drec = nullptr;
        uint8_t* dout = nullptr;
        if (records && out_records && record_width > 0) {
            c->bk_rec.ensure(n * record_width, s);
            c->bk_rec_out.ensure(n * record_width, s);
            drec = c->bk_rec.p;
            dout = c->bk_rec_out.p;
            CK(cudaMemcpyAsync(drec, records, (size_t)(n * record_width), cudaMemcpyHostToDevice, s));
        }
        launch_reorder(lab, n, (uint32_t)p, c->bk_keys_b.p, c->bk_keys_a.p, c->bk_order.p, c->bk_perm.p,
                       c->bk_counts.p, drec, record_width, dout, c->temp.p, c->temp.cap, s);
        c->kernels += 5;
        CK(cudaMemcpyAsync(perm_out, c->bk_perm.p, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(counts_out, c->bk_counts.p, sizeof(uint64_t) * p, cudaMemcpyDeviceToHost, s));
        if (dout) CK(cudaMemcpyAsync(out_records, dout, (size_t)(n * record_width), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    });
}

int grem_staged_edges(grem_ctx* c, const uint32_t** dev_edges, int64_t* num_edges) {
    if (!c || !dev_edges) return GREM_E_FORMAT;
    *dev_edges = c->staged_last ? reinterpret_cast<const uint32_t*>(c->edges_owned.p) : nullptr;
    if (num_edges) *num_edges = c->staged_last ? c->staged_m : 0;
    return GREM_OK;
}

int grem_partition_shard_u32(grem_ctx* c, const uint32_t* edges, int64_t m, int64_t n, int on_device, int64_t p,
                             const grem_config* cfg, int rank, int world, int32_t* labels_out) {
    if (!c || !cfg || world < 1 || rank < 0 || rank >= world) return GREM_E_FORMAT;
    return guarded(c, [&] {
        if (p < 2 || (p & (p - 1)) != 0)
            fail(GREM_E_FORMAT, "number of parts must be a power of two >= 2, got " + std::to_string(p));
        const uint2* d = stage_edges(c, edges, m, n, on_device, true);
        partition_entry(c, d, m, n, p, cfg, nullptr, labels_out, nullptr, rank, world);
    });
}

int grem_count_cuts_u32(grem_ctx* c, const uint32_t* edges, int64_t m, int64_t n, int on_device,
                        const int32_t* labels, int labels_on_device, grem_report* rep) {
    if (!c) return GREM_E_FORMAT;
    return guarded(c, [&] {
        const uint2* d = stage_edges(c, edges, m, n, on_device);
        const int32_t* dl = labels;
        if (!labels_on_device) {
            c->lab32.ensure(n, c->s);
            CK(cudaMemcpyAsync(c->lab32.p, labels, sizeof(int32_t) * n, cudaMemcpyHostToDevice, c->s));
            dl = c->lab32.p;
        }
        count_cuts_dev(c, d, m, dl, n, rep);
    });
}

int grem_count_cuts_file(grem_ctx* c, const char* path, const int32_t* labels, int labels_on_device,
                         grem_report* rep) {
    if (!c || !path || !labels) return GREM_E_FORMAT;
    return guarded(c, [&] {
        GrpeHeader hd;
        const uint2* d = load_grpe(c, path, &hd);
        const int32_t* dl = stage_labels(c, labels, hd.n, labels_on_device);
        count_cuts_dev(c, d, hd.m, dl, hd.n, rep);
    });
}

int grem_bisect_file(grem_ctx* c, const char* path, const grem_config* cfg, int64_t capacity,
                     const grem_hooks* hooks, int32_t* labels_out, grem_report* rep) {
    if (!c || !cfg || !path) return GREM_E_FORMAT;
    return guarded(c, [&] {
        GrpeHeader hd;
        const uint2* d = load_grpe(c, path, &hd);
        if (hd.n < 1) fail(GREM_E_FORMAT, "num_nodes must be >= 1");
        bisect_entry(c, d, hd.m, hd.n, cfg, capacity, hooks, labels_out, rep);
    });
}

int grem_partition_file(grem_ctx* c, const char* path, int64_t p, const grem_config* cfg, const grem_hooks* hooks,
                        int32_t* labels_out, grem_report* rep) {
    if (!c || !cfg || !path) return GREM_E_FORMAT;
    return guarded(c, [&] {
        if (p < 2 || (p & (p - 1)) != 0)
            fail(GREM_E_FORMAT, "number of parts must be a power of two >= 2, got " + std::to_string(p));
        GrpeHeader hd;
        const uint2* d = load_grpe(c, path, &hd);
        if (hd.n < 1) fail(GREM_E_FORMAT, "num_nodes must be >= 1");
        partition_entry(c, d, hd.m, hd.n, p, cfg, hooks, labels_out, rep);
    });
}

int grem_state_parts(grem_ctx* c, int32_t* out, int64_t n) {
    if (!c || !out) return GREM_E_FORMAT;
    g_err.clear();
    try {
        if (n != c->live_n) fail(GREM_E_FORMAT, "state size mismatch");
        std::vector<int8_t> h(n);
        CK(cudaMemcpyAsync(h.data(), c->lab.p, n, cudaMemcpyDeviceToHost, c->s));
        CK(cudaStreamSynchronize(c->s));
        for (int64_t i = 0; i < n; ++i) out[i] = h[i];
    } catch (const GremError& e) {
        g_err = e.msg;
        return e.code;
    }
    return GREM_OK;
}

int grem_device_alloc(grem_ctx* c, uint64_t bytes, void** out) {
    if (!c || !out) return GREM_E_FORMAT;
    return guarded(nullptr, [&] {
        CK(cudaSetDevice(c->device));
        CK(cudaMalloc(out, bytes ? bytes : 1));
    });
}
int grem_device_free(grem_ctx* c, void* p) {
    if (!c) return GREM_E_FORMAT;
    return guarded(nullptr, [&] { CK(cudaFree(p)); });
}
int grem_memcpy_h2d(grem_ctx* c, void* dst, const void* src, uint64_t bytes) {
    if (!c) return GREM_E_FORMAT;
    return guarded(nullptr, [&] {
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->s));
        CK(cudaStreamSynchronize(c->s));
    });
}
int grem_memcpy_d2h(grem_ctx* c, void* dst, const void* src, uint64_t bytes) {
    if (!c) return GREM_E_FORMAT;
    return guarded(nullptr, [&] {
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->s));
        CK(cudaStreamSynchronize(c->s));
    });
}

int grem_gen_edges_device(grem_ctx* c, uint64_t n, uint32_t beta, uint64_t seed, uint64_t e0, uint64_t count,
                          uint32_t* dev_out) {
    if (!c || n < 1 || beta < 1) return GREM_E_FORMAT;
    return guarded(nullptr, [&] {
        CK(cudaSetDevice(c->device));
        gg_params p;
        gg_init(&p, n, beta, seed);
        launch_gen_edges(p.n, p.beta, p.seed, p.scale, p.perm_mask, p.perm_bits, e0, count, dev_out, c->s);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(c->s));
    });
}

}  // extern "C"

// ---------------------------------------------------------------- debug
// Runs the chunk sizes scan (+ tie verification and walk) on caller-provided
// node maps; used by the GPU unit tests of the scan kernels.
extern "C" int grem_debug_chunk_scan(grem_ctx* c, const uint8_t* meta, const int32_t* newb, int64_t nc, int64_t x0,
                                     int64_t cap, int do_walk, int32_t* x_out, uint8_t* bad_out, int64_t* nbad_out) {
    if (!c) return GREM_E_FORMAT;
    return guarded(c, [&] {
        ensure_chunk(c, nc + 1, 0);
        CK(cudaMemcpyAsync(c->meta.p, meta, nc, cudaMemcpyHostToDevice, c->s));
        CK(cudaMemcpyAsync(c->newb.p, newb, sizeof(int32_t) * nc, cudaMemcpyHostToDevice, c->s));
        long long sz[2] = {x0, 0};
        scal_write(c, c->d_sizes, sz, 2);
        CK(cudaMemsetAsync(c->d_scal, 0, sizeof(long long) * 8, c->s));
        CK(cudaMemsetAsync(c->d_scal + 6, 0x7F, sizeof(long long), c->s));
        ChunkBufs b = chunk_bufs(c);
        launch_chunk_scan(b, nc, cap, c->s);
        if (do_walk == 1) launch_walk(b, nc, cap, c->s);
        if (do_walk >= 2) {   // production repair: half-step predictor + trajectory bundles (2 or 3 windows)
            launch_half_predictor(b, nc, cap, c->xalt.p, c->s);
            BundleBufs bb{c->bparams.p, c->bends.p, c->bckpt.p, c->bxin.p, c->bhit.p, c->bsegflag.p};
            launch_bundle(b, nc, cap, c->xalt.p, bb, do_walk == 2 ? 3 : 2, c->s, false);
        }
        CK(cudaMemcpyAsync(x_out, c->x.p, sizeof(int32_t) * (nc + 1), cudaMemcpyDeviceToHost, c->s));
        CK(cudaMemcpyAsync(bad_out, c->bad.p, nc, cudaMemcpyDeviceToHost, c->s));
        scal_read(c, c->d_scal + 3, 2);
        nbad_out[0] = c->h_pin[1];   // flagged ties
        nbad_out[1] = c->h_pin[0];   // walk steps
    });
}
