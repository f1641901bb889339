// grem_kernels.cuh — launch wrappers of the sm_100a kernels (grem_kernels.cu).
// Every wrapper enqueues on `s` and never synchronises; counts that the host
// needs (N_c, changed, ...) are left in device scalars.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "grem_core.cuh"

namespace grem {

// Kernel-level timing marks (bench.py's roofline rows): the runtime records a
// CUDA event pair around the marked launches when kernel profiling is on
// (grem_set_profiling(ctx, 2)); a no-op otherwise.  Ids index the runtime's
// kernel phases (KM_* -> "k.<name>").
enum KMark { KM_BIN_HIST = 0, KM_BIN_SCATTER, KM_BIN_COMPACT, KM_ROUND_REDUCE, KM_ROUND_DOWN, KM_COUNT_DELTA,
             KM_ROUND_REDUCE_ALL, KM_ROUND_DOWN_ALL, KM_N };   // *_ALL: every launch (share of the step)
void kmark(int km, int begin, cudaStream_t s);

// Hub privatisation (power-law hubs would serialise the counter atomics):
// up to kMaxHubs high-degree nodes, found per bisection by sampling, live in
// an open-addressing table (kHubSlots u32 keys, empty = kHubEmpty); edge
// kernels accumulate their updates in shared memory and flush once per CTA.
constexpr int kHubSlots = 2048;
constexpr int kMaxHubs = 1024;
constexpr uint32_t kHubEmpty = 0xFFFFFFFFu;
// the two candidate buckets (of kHubSlots / 2) of a key
__host__ __device__ __forceinline__ uint32_t hub_bucket1(uint32_t u) { return (u * 0x9E3779B1u) >> 22; }
__host__ __device__ __forceinline__ uint32_t hub_bucket2(uint32_t u) { return ((u ^ (u >> 15)) * 0x85EBCA77u) >> 22; }
static_assert(kHubSlots == 2048, "hub buckets are 10-bit hashes");
// host: cuckoo insertion of ids (most important first) into table[kHubSlots];
// ids that cannot be placed are simply not hubs.  Returns the number placed.
int hub_table_build(const uint32_t* ids, int count, uint32_t* table);

struct ChunkBufs {
    // global per-node state (n)
    int8_t* lab;
    uint8_t* tl;
    unsigned long long* cnt;
    uint8_t* flag;
    double2* nbr;
    // per chunk node (cap = chunk node capacity)
    uint32_t* nodes;
    uint8_t* meta;
    int32_t* newb;      // exclusive count of active new nodes before i
    int32_t* x;         // sizes[0] before node i; x[N_c] = after the chunk
    int32_t* xalt;      // exact x of the previous round (bundle window centre; read-only in a round)
    int32_t* xnext;     // exact x of this round (becomes xalt of the next round)
    uint8_t* bad;       // tie speculation inconsistent at i
    // compact per-chunk-node round state (coalesced in every round)
    unsigned long long* cntc;   // packed counts (c0 | c1 << 32) of chunk node i
    double2* nbrc;              // running estimates of chunk node i (old nodes; 0 for new)
    uint8_t* tlc;               // tentative label codes (cur | prev << 4) of chunk node i
    int32_t* pos;               // (unused by the chunk rounds; see rankw)
    uint2* rankw;               // n/32 words {presence bits, chunk members before}: chunk index of node g
    uint32_t* chg;              // n bits: tentative label changed in the last round (tl[g] valid)
    uint32_t* chgc;             // kChgCoarseBits bits: some node of the 2^chg_shift-id block changed
    int chg_shift;
    uint8_t* segbad;            // per bundle segment (bseg_len nodes): a tie of this round was mis-speculated
    int64_t bseg_len;
    int64_t bseg_n;             // segments of this chunk: ceil(N_c / bseg_len)
    // per scan tile
    Clamp* tile_agg;
    Clamp* tile_inc;            // single-pass round: inclusive look-back prefixes
    unsigned* tflag;            // single-pass round: look-back flags (+1 word: ticket)
    long long* tile_x;
    long long* tile_bad;
    // device scalars
    long long* sizes;   // [2] live sizes (read-only during a chunk)
    long long* scal;    // [16] scratch scalars: 0 n_c, 1 changed, 2 total_new, 3 bundle misses, 4 nbad, 5 2*x0,
                        //     6 first mis-speculated tie, 7 round gate, 8 rounds run
    const uint32_t* hub_keys;   // kHubSlots table or nullptr (no hubs)
    uint32_t* lab2;             // 2-bit mirror of lab (code = label + 1), L2-resident gathers
    const long long* gate;      // scal + 7: changed count of the previous round (round kernels skip on 0)
    uint8_t* dcur;              // per round tile: inputs changed since the last round (incremental rounds)
    uint8_t* dnext;             // per round tile: dirty in the next round
};
constexpr int kChgCoarseBits = 1 << 17;   // coarse changed-label filter (16 KB, staged in shared memory)
__host__ __device__ __forceinline__ int chg_coarse_shift(int64_t n) {
    int sh = 0;
    while ((((n + (1LL << sh) - 1) >> sh)) > kChgCoarseBits) ++sh;
    return sh;
}
constexpr int kRTileC = 4096;   // nodes per round tile (kRT * kRI in grem_kernels.cu)

// Round-1 counts of large chunks (propagation blocking): edges emit
// (node, label code) records binned by coarse node range (2^shift ids,
// <= kMaxBins bins); one CTA per 2^kSubShift-node tile then accumulates its
// records in shared memory and writes the compact chunk state directly.
#ifndef GREM_MAX_BINS
#define GREM_MAX_BINS 1024   // k_bin_scatter's shared footprint, see GREM_SCAT_BLOOM in grem_kernels.cu
#endif
constexpr int kMaxBins = GREM_MAX_BINS;
#ifndef GREM_SUB_SHIFT
#define GREM_SUB_SHIFT 14
#endif
constexpr int kSubShift = GREM_SUB_SHIFT;   // nodes per compact tile = 2^kSubShift (16 per thread)
struct BinBufs {
    uint32_t* recs;          // >= 2 * edges of the chunk
    int32_t* hist;           // binned_hist_entries(nbins): records per (bin, scatter CTA)
    int32_t* offs;           // its exclusive scan: record cursor per (bin, CTA); row nbins = end
    unsigned long long* hub_cnt;   // kHubSlots
    uint32_t* hub_flag;            // kHubSlots
    unsigned long long* status;    // binned_tiles(n) look-back words
    unsigned int* ticket;          // 1
    int shift, nbins;
};
int binned_shift(int64_t n);
int64_t binned_tiles(int64_t n);
int64_t binned_hist_entries(int nbins);
int binned_scatter_ctas();   // CTAs of the round-1 scatter (and its histogram)
// writes nodes, meta, tlc, pos, cntc, nbrc, newb (incl. s0) for the chunk;
// scal[0] = N_c, scal[2] = new nodes
void launch_bin_offsets(const uint2* e, int64_t m, const uint32_t* hub_keys, int shift, int nbins, int32_t* hist,
                        int32_t* offs, void* temp, size_t temp_bytes, cudaStream_t s);
void launch_count_init_binned(const uint2* e, int64_t m, int64_t n, int refine, const ChunkBufs& b,
                              const BinBufs& bb, void* temp, size_t temp_bytes, cudaStream_t s,
                              bool have_offs = false);

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;

int num_sms();

// --- non-seed chunk (process_chunk, grem.py:119-155) ---
void launch_count_init(const uint2* e, int64_t m, const ChunkBufs& b, cudaStream_t s);
void launch_count_delta(const uint2* e, int64_t m, const ChunkBufs& b, cudaStream_t s, bool staged = false);
void launch_node_init(const ChunkBufs& b, int64_t nc, int refine, cudaStream_t s);
void launch_add_base(int32_t* a, int64_t n, const long long* sizes, cudaStream_t s);
void launch_chunk_scan(const ChunkBufs& b, int64_t nc, long long cap, cudaStream_t s);
void launch_walk(const ChunkBufs& b, int64_t nc, long long cap, cudaStream_t s);
// exact repair of mis-speculated ties by trajectory bundles (replaces the walk)
struct BundleBufs {
    int32_t* params;   // nc packed node parameters
    int32_t* ends;     // nseg * 192
    int32_t* ckpt;     // bundle_ckpt_ints(nc)
    int32_t* xin;      // nseg
    int32_t* hit;      // nseg
    int32_t* segflag;  // nseg: bit 0 mis-speculated tie inside, bit 1 simulated (k_bundle_params)
};
int64_t bundle_segment_len(int64_t nc);
int64_t bundle_ckpt_ints(int64_t nc);
void launch_half_predictor(const ChunkBufs& b, int64_t nc, long long cap, int32_t* xalt, cudaStream_t s);
// fix_decisions: the repaired suffix's decisions / tentative labels / tie
// guesses written by k_round_down are corrected (production rounds)
void launch_bundle(const ChunkBufs& b, int64_t nc, long long cap, const int32_t* xalt, const BundleBufs& bb, int nwin,
                   cudaStream_t s, bool fix_decisions);
// fused round: preferences + clamp tile aggregates, top scan, x / tie check /
// speculative decisions (node arrays padded to whole kScanTile tiles)
void launch_round_scan(const ChunkBufs& b, int64_t nc, long long cap, int first_round, int incremental,
                       cudaStream_t s);
void launch_commit(const ChunkBufs& b, int64_t nc, cudaStream_t s);
void launch_round_gate(const ChunkBufs& b, cudaStream_t s);
void launch_round_start(const ChunkBufs& b, int64_t ntiles, bool first_round, int64_t nchg_words, cudaStream_t s);
void launch_sizes_update(const ChunkBufs& b, int64_t nc, cudaStream_t s);

// --- chunk membership ---
void launch_mark_all(const uint2* e, int64_t m, uint8_t* flag, cudaStream_t s);
// nodes = ascending ids with flag or cnt nonzero; count -> *d_count (device)
size_t select_nodes_temp_bytes(int64_t n);
void launch_select_nodes(const uint8_t* flag, const unsigned long long* cnt, int64_t n, uint32_t* nodes,
                         long long* d_count, void* temp, size_t temp_bytes, cudaStream_t s);

// --- seed chunk (seed.py:36-118, grem.py:158-174) ---
struct SeedBufs {
    int32_t* rank;        // n: local index of a chunk node
    int32_t* start;       // nc+1 CSR row starts
    int32_t* cursor;      // nc: self-loop entries per row (chunk-0 CSR by sort)
    uint32_t* adj;        // entries: local neighbour ids (self-loops as w == row)
    uint32_t* row_of;     // entries: owning row
    uint32_t* parent;     // nc: union-find
    unsigned long long* ckey;  // nc: component (-degree, index) min key
    uint32_t* csize;      // nc
    uint32_t* roots;      // nc
    unsigned long long* rkeys;   // nc
    unsigned long long* rkeys2;  // nc
    uint32_t* rvals;      // nc
    uint32_t* rvals2;     // nc
    uint32_t* cpos;       // nc: sorted position of a component root
    int8_t* slab;         // nc: seed labels (0/1; 2 = boundary component, undecided)
    int8_t* slab2;        // nc
    uint32_t* disc;       // nc: BFS min discoverer rank
    uint32_t* frontier;   // nc
    unsigned long long* cand_keys;   // nc
    unsigned long long* cand_keys2;  // nc
    int64_t* fdeg;        // nc+1 frontier row lengths / sorted component sizes
    int64_t* cum;         // nc+1 exclusive prefix of fdeg
    unsigned long long* pair;        // nc: per-row packed counts
    uint8_t* want;        // nc
    long long* scal;      // [16]
};

void launch_set_rank(const uint32_t* nodes, int64_t nc, int32_t* rank, cudaStream_t s);
void launch_degrees(const uint2* e, int64_t m, const int32_t* rank, int32_t* deg, const uint32_t* hub_keys,
                    cudaStream_t s);
void launch_fill_csr(const uint2* e, int64_t m, const int32_t* rank, int32_t* cursor, uint32_t* adj,
                     uint32_t* row_of, const uint32_t* hub_keys, cudaStream_t s);
size_t seed_csr_temp_bytes(int64_t entries);
void launch_seed_sort(const uint2* e, int64_t m, uint32_t* keysA, uint32_t* valsA, uint32_t* keysB, uint32_t* valsB,
                      int end_bit, uint32_t* nodes, int32_t* counts, long long* d_nruns, void* temp,
                      size_t temp_bytes, bool* sorted_in_b, cudaStream_t s);
void launch_rank_words(const uint32_t* nodes, int64_t nc, int64_t nwords, uint2* rw, cudaStream_t s);
void launch_seed_map(const uint32_t* skeys, const uint32_t* svals, int64_t entries, const uint2* rw,
                     uint32_t* row_of, uint32_t* adj, int32_t* selfc, cudaStream_t s);

// hub detection from a sample of the level's edges
void launch_sample_degrees(const uint2* e, int64_t sample, int32_t* sdeg, cudaStream_t s);
void launch_hub_keys(const uint32_t* ids, int64_t cnt, const int32_t* sdeg, unsigned long long* keys,
                     cudaStream_t s);
size_t hub_select_temp_bytes(int64_t n);
void launch_hub_select(const int32_t* sdeg, int64_t n, int32_t min_deg, uint32_t* ids, long long* d_count, void* temp,
                       size_t temp_bytes, cudaStream_t s);
void sort_keys_u64_desc(const unsigned long long* kin, unsigned long long* kout, int64_t n, void* temp,
                        size_t temp_bytes, cudaStream_t s);
void launch_cc(const uint2* e, int64_t m, const int32_t* rank, uint32_t* parent, uint32_t* scratch, int64_t nc,
               cudaStream_t s);
void launch_cc_csr(const int32_t* start, const uint32_t* adj, int64_t nc, uint32_t* parent, uint32_t* scratch,
                   unsigned long long* d_giant, cudaStream_t s);
void launch_comp_keys(const SeedBufs& sb, int64_t nc, cudaStream_t s, const unsigned long long* giant = nullptr);
void launch_select_roots(const SeedBufs& sb, int64_t nc, void* temp, size_t temp_bytes, cudaStream_t s);
void launch_root_keys(const SeedBufs& sb, int64_t nroots, cudaStream_t s);
void launch_boundary(const SeedBufs& sb, int64_t nroots, long long target, void* temp, size_t temp_bytes,
                     cudaStream_t s);
void launch_seed_labels(const SeedBufs& sb, int64_t nc, cudaStream_t s);
// expansion reads frontier row-length prefix from sb.cum
void launch_bfs_expand(const SeedBufs& sb, int64_t fsize, long long rbase, int64_t total, cudaStream_t s);
void launch_cand_keys(const SeedBufs& sb, int64_t ncand, cudaStream_t s);
void launch_frontier_degrees(const SeedBufs& sb, int64_t fsize, cudaStream_t s);
void launch_bfs_take(const SeedBufs& sb, int64_t ncand, int64_t take, cudaStream_t s);
void launch_seed_finalize(const SeedBufs& sb, int64_t nc, cudaStream_t s);
void launch_row_counts(const SeedBufs& sb, const int8_t* cur, const int8_t* pre, int mode, int64_t entries,
                       int64_t nc, cudaStream_t s);
void launch_refine_scan(const SeedBufs& sb, const ChunkBufs& b, int64_t nc, long long cap, cudaStream_t s);
void launch_refine_decide(const SeedBufs& sb, const ChunkBufs& b, int64_t nc, long long cap, cudaStream_t s);
// refinement on bitmaps (preferred path)
void launch_pack_bits(const int8_t* lab, int64_t nc, uint32_t* bits, cudaStream_t s);
void launch_unpack_bits(const uint32_t* bits, int64_t nc, int8_t* lab, cudaStream_t s);
void launch_xor_popc(const uint32_t* a, const uint32_t* b, int64_t nc, long long* out, cudaStream_t s);
void launch_row_counts_bits(const SeedBufs& sb, const uint32_t* Pb, const uint32_t* Tb, int mode, int64_t entries,
                            int64_t nc, cudaStream_t s);
void launch_refine_round(const SeedBufs& sb, const ChunkBufs& b, const uint32_t* Pb, uint32_t* Tb, uint32_t* wantb,
                         uint32_t* Db, int64_t nc, long long cap, cudaStream_t s);
void launch_refine_delta(const SeedBufs& sb, const uint32_t* Db, int64_t nc, int64_t changed, const uint32_t* Pb,
                         const uint32_t* Tb, void* temp, size_t temp_bytes, cudaStream_t s);
void launch_seed_commit(const SeedBufs& sb, const ChunkBufs& b, const uint32_t* nodes, int64_t nc,
                        cudaStream_t s);

// --- after the stream ---
void launch_fill_unassigned(int8_t* lab, int64_t n, const long long* sizes, int32_t* rank_scratch,
                            void* temp, size_t temp_bytes, cudaStream_t s);
void launch_labels_to_i32(const int8_t* lab, int64_t n, int32_t* out, cudaStream_t s);
// count_cuts (grem.py:227-252): cut, per-part sizes (int32 labels), max label
void launch_count_cuts(const uint2* e, int64_t m, const int32_t* lab, int64_t n, unsigned long long* d_cut,
                       unsigned long long* d_sizes, int64_t sizes_cap, int* d_max, int* d_neg, cudaStream_t s);
void launch_count_cuts_i8(const uint2* e, int64_t m, const int8_t* lab, unsigned long long* d_cut, cudaStream_t s);
void launch_loop_cond(cudaGraphConditionalHandle h, const long long* scal, long long max_rounds, cudaStream_t s);
void launch_check_piece(uint2* e, int64_t m, uint32_t n, unsigned long long* bad_max, cudaStream_t s);
void launch_check_ids(const uint2* e, int64_t m, uint32_t* d_max_id, cudaStream_t s);

// --- recursion (_extract_induced, grem.py:255-274) ---
void launch_side_flags(const int8_t* lab, int64_t n, int side, int32_t* flags, cudaStream_t s);
void launch_extract(const uint2* e, int64_t m, const int8_t* lab, int side, const int32_t* newid,
                    uint2* out, long long* d_count, void* temp, size_t temp_bytes, cudaStream_t s);
size_t extract_temp_bytes(int64_t m);
void launch_sub_orig(const int8_t* lab, int64_t n, int side, const int32_t* newid, const int32_t* orig,
                     int32_t* sub_orig, cudaStream_t s);
void launch_leaf_write(const int8_t* lab, int64_t n, const int32_t* orig, int32_t leaf_base, int32_t* final_lab,
                       cudaStream_t s);
void launch_bisect_cut(const uint2* e, int64_t m, const int8_t* lab, unsigned long long* out, cudaStream_t s);
void launch_iota(int32_t* a, int64_t n, cudaStream_t s);
// succinct side maps for the recursion (preferred path)
void launch_side_bits(const int8_t* lab, int64_t n, uint32_t* bits, uint32_t* wpop, uint32_t* pre, void* temp,
                      size_t temp_bytes, cudaStream_t s);
size_t split_edges_tiles(int64_t m);
void launch_split_edges(const uint2* e, int64_t m, const uint32_t* bits, const uint32_t* pre, int64_t nw, uint2* wi,
                        uint2* arena, unsigned long long* status, unsigned int* ticket, long long* counts,
                        cudaStream_t s);
void launch_reverse_edges(uint2* a, int64_t n, cudaStream_t s);
void launch_sub_orig_bits(const int8_t* lab, int64_t n, int side, const uint32_t* bits, const uint32_t* pre,
                          const int32_t* orig, int32_t* sub, cudaStream_t s);
// cut count with labels packed to 2^lb bits (d_neg gets bit 1 on negative labels)
void launch_count_cuts_packed(const uint2* e, int64_t m, const int32_t* lab, int64_t n, int lb, uint32_t* packed,
                              unsigned long long* d_cut, int* d_neg, cudaStream_t s);

// --- partitioned storage (grem_store.cu; store.py:55-104, 201-235) ---
void launch_node_side_counts_hub(const uint2* e, int64_t m, const uint32_t* packed, const uint32_t* hub_keys,
                                 unsigned long long* cnt, int* bad, cudaStream_t s);
size_t shuffle_temp_bytes(int64_t m);
void launch_shuffle(const uint2* e, int64_t m, unsigned long long seed, unsigned long long* keys,
                    unsigned long long* vals, void* temp, size_t temp_bytes, cudaStream_t s);
void launch_node_stats(const uint2* e, int64_t m, const int32_t* lab, int64_t n, unsigned long long* cnt,
                       uint32_t* packed, int64_t* k, int64_t* k0, int* bad, cudaStream_t s,
                       const uint32_t* hub_keys = nullptr);
void launch_label_max(const int32_t* lab, int64_t n, int* d_max, cudaStream_t s);
size_t bucket_sort_temp_bytes(int64_t m);
// stable p x p bucket scatter of the edges (keys_a/keys_b: m u32 scratch);
// counts: p*p extents; *d_bad != 0 when an endpoint is unlabeled
void launch_write_buckets(const uint2* e, int64_t m, const int32_t* lab, int64_t n, bool any_unlabeled, uint32_t p,
                          uint32_t* keys_a, uint32_t* keys_b, uint32_t* packed, uint2* out,
                          unsigned long long* counts, int* d_bad, void* temp, size_t temp_bytes, cudaStream_t s);
size_t order_sort_temp_bytes(int64_t n);
// nodes grouped by label (stable): order (slot -> node), perm (node -> slot),
// counts per label; optionally the records gathered into out
void launch_reorder(const int32_t* lab, int64_t n, uint32_t p, uint32_t* keys_b, uint32_t* ids_a, uint32_t* order,
                    long long* perm, unsigned long long* counts, const uint8_t* rec, int64_t width, uint8_t* out,
                    void* temp, size_t temp_bytes, cudaStream_t s);

// generic CUB helpers
size_t scan_temp_bytes(int64_t n);
void exclusive_sum_i32(const int32_t* in, int32_t* out, int64_t n, void* temp, size_t temp_bytes, cudaStream_t s);
void exclusive_sum_i64(const int64_t* in, int64_t* out, int64_t n, void* temp, size_t temp_bytes, cudaStream_t s);
size_t sort_temp_bytes(int64_t n);
void sort_pairs_u64_u32(const unsigned long long* kin, unsigned long long* kout, const uint32_t* vin,
                        uint32_t* vout, int64_t n, void* temp, size_t temp_bytes, cudaStream_t s);
void sort_keys_u64(const unsigned long long* kin, unsigned long long* kout, int64_t n, void* temp,
                   size_t temp_bytes, cudaStream_t s);

// expected-cut model (theory.py:125-146): lg = lgamma(i) table; term = n
// doubles, big_list = n slots, part = theory_sum_blocks() doubles
int theory_sum_blocks();
// out[4] (pre-set to {~0, ~0, 0, 0}): first node with k >= 1, first with a
// non-majority k0, max k, sum of k
void launch_theory_check(const int64_t* k, const int64_t* k0, int64_t n, unsigned long long* out, cudaStream_t s);
void launch_lgamma_table(double* lg, int64_t count, cudaStream_t s);
void launch_expected_cuts(const int64_t* k, const int64_t* k0, int64_t n, const double* lg, double x_eff,
                          double* term, int64_t* big_list, unsigned long long* big_count, double* part,
                          double* out, cudaStream_t s);

// synthetic generator (grem_gen.h)
void launch_gen_edges(uint64_t n, uint32_t beta, uint64_t seed, double scale, uint64_t perm_mask,
                      uint32_t perm_bits, uint64_t e0, uint64_t count, uint32_t* out, cudaStream_t s);

}  // namespace grem
