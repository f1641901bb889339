/*
 * grem_b200.h — C ABI of libgrem_b200.so, the B200-native GREM partitioner.
 *
 * Drop-in boundary for the reference's GREM path (streamcut, pure Python;
 * paths below are relative to /root/reference/pkg/src/streamcut/).  Plain
 * pointers and sizes only; no torch types.  A reference-side binding (ctypes)
 * is shown in INTEGRATION.md; the package's own binding is
 * paper_2502_17846_b200/_abi.py.
 *
 * Conventions
 *   - return 0 on success; GREM_E_FORMAT mirrors streamcut.errors.FormatError,
 *     GREM_E_CAPACITY mirrors CapacityError (errors.py:4-13), GREM_E_CUDA is a
 *     CUDA/NCCL failure.  grem_last_error() returns a thread-local message.
 *   - edge arrays are (src, dst) u32 pairs in file order (GRPE payload,
 *     edgefile.py:1-14); `edges_on_device` says whether the pointer is device
 *     memory of the context's GPU (no copy) or host memory (chunked,
 *     double-buffered H2D inside the call).
 *   - node ids must be < num_nodes < 2^31 (larger id spaces are rejected with
 *     GREM_E_FORMAT; model.py:18 allows 64-bit ids, no benchmark shape needs
 *     them).
 *   - the caller owns every buffer it passes; the context owns device state.
 */
#ifndef GREM_B200_H
#define GREM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GREM_OK 0
#define GREM_E_FORMAT 1
#define GREM_E_CAPACITY 2
#define GREM_E_CUDA 3
#define GREM_E_NOMEM 4
#define GREM_E_CALLBACK 5

typedef struct grem_ctx grem_ctx;

/* GremConfig + SeedConfig (grem.py:45-75, seed.py:23-33).  chunk_edges > 0
 * selects an absolute chunk size; otherwise chunk_frac (default 0.1) is used
 * exactly as ChunkPlan.plan does (edgefile.py:338-349). */
typedef struct {
    int64_t chunk_edges;
    double chunk_frac;
    double capacity_slack;
    int32_t refine;
    int32_t passes;
    int32_t seed_algo;               /* 0 = bfs_grow, 1 = random (needs hooks.seed) */
    int32_t seed_refinement_passes;  /* SeedConfig.refinement_passes */
} grem_config;

/* CutReport (model.py:115-132).  partition_sizes is a caller buffer of
 * sizes_cap entries; num_parts = max label + 1 (grem.py:243).  The float
 * fields (cut_fraction, balance_ratio) are derived by the caller from these
 * integers with the reference's own expressions (grem.py:245-251). */
typedef struct {
    int64_t total_edges;
    int64_t cut_edges;
    int64_t num_parts;
    int64_t* partition_sizes;
    int64_t sizes_cap;
} grem_report;

/* seed_bisect(..., algorithm="random") labels (seed.py:48-52) are drawn by
 * numpy's PCG64 on the host: the library asks for them through this hook. */
typedef int (*grem_seed_fn)(int64_t n_chunk_nodes, int8_t* labels_out, void* user);
/* bisect(on_chunk=...) (grem.py:219-221): called after every chunk with the
 * live sizes; grem_state_parts() may be called from inside it. */
typedef int (*grem_chunk_fn)(const int64_t* sizes, void* user);
/* ResidencyMeter (edgefile.py:352-368): +n on acquire, -n on release, called
 * with the reference's stream_chunks timing (edgefile.py:384-391,453-462). */
typedef void (*grem_meter_fn)(int64_t delta_edges, void* user);

typedef struct {
    grem_seed_fn seed;
    grem_chunk_fn on_chunk;
    grem_meter_fn meter;
    void* user;
} grem_hooks;

/* Per-call statistics (diagnostics; zeroed per call). */
typedef struct {
    int64_t chunks;          /* chunks processed (all passes, all bisections) */
    int64_t rounds;          /* fixpoint rounds summed over non-seed chunks */
    int64_t max_rounds;      /* worst chunk */
    int64_t visits;          /* chunk-node visits (sum of N_c) */
    int64_t walk_steps;      /* sequential sizes-chain repairs */
    int64_t seed_bfs_levels; /* BFS levels on the boundary component */
    int64_t bisections;
    int64_t kernels;         /* kernel launches issued */
    double ms_total;         /* device time of the call (CUDA events) */
    int64_t count_bytes;     /* algorithmic bytes of the edge count passes (10 B/edge init, 9 B/edge delta) */
    int64_t path_bytes;      /* algorithmic bytes of the whole call, SURVEY.md 8(d) formula */
    int64_t delta_bytes;     /* the k_count_delta share of count_bytes (9 B/edge per launch) */
} grem_stats;

/* ------------------------------------------------------------------ life */
grem_ctx* grem_create(int device);
void grem_destroy(grem_ctx* ctx);
const char* grem_last_error(void);
int grem_get_stats(grem_ctx* ctx, grem_stats* out);
/* Per-phase device time (CUDA events on the context stream) of the last call,
 * when profiling is on.  Returns the number of phases; fills up to `cap`. */
int grem_set_profiling(grem_ctx* ctx, int on);
int grem_get_phase_times(grem_ctx* ctx, double* ms_out, int64_t* count_out, int cap, const char** names_out);
/* Algorithmic bytes of the kernel-level phases ("k.*", profiling level 2:
 * grem_set_profiling(ctx, 2)), same order as grem_get_phase_times; 0 for
 * phases without a byte model.  Returns the number of phases. */
int grem_get_phase_bytes(grem_ctx* ctx, double* bytes_out, int cap);
/* High-water marks (bytes) of the device memory pool all library workspaces
 * come from (cudaMemPoolAttrUsedMemHigh / ReservedMemHigh of the device's
 * default pool); reset != 0 restarts them.  Buffers the caller allocated with
 * grem_device_alloc (plain cudaMalloc) are not included. */
int grem_mem_high_water(grem_ctx* ctx, int64_t* used_high, int64_t* reserved_high, int reset);
/* Release every device workspace of the context and its child contexts (the
 * next call re-allocates them) and trim the memory pool. */
int grem_trim(grem_ctx* ctx);
/* write_buckets with out_edges == NULL (out_on_device 0) keeps the
 * bucket-ordered edges on the device; this copies edges [first, first+count)
 * of them to host memory, so a caller streams the store file in bounded pieces. */
int grem_bucket_edges(grem_ctx* ctx, uint32_t* dst, int64_t first, int64_t count);

/* --------------------------------------------------------------- the path */

/* bisect (grem.py:192-224).  capacity <= 0 => default_capacity(n, slack)
 * (grem.py:78-79).  labels_out: n int32 in {0,1}.  rep may be NULL (the
 * count_cuts pass is then skipped, as partition() discards it). */
int grem_bisect_u32(grem_ctx* ctx, const uint32_t* edges, int64_t num_edges, int64_t num_nodes,
                    int edges_on_device, const grem_config* cfg, int64_t capacity,
                    const grem_hooks* hooks, int32_t* labels_out, grem_report* rep);

/* partition (grem.py:277-319): p a power of two >= 2; level capacity from the
 * original node count; recursion over device-resident induced subgraphs;
 * final count_cuts on the original edges. */
int grem_partition_u32(grem_ctx* ctx, const uint32_t* edges, int64_t num_edges, int64_t num_nodes,
                       int edges_on_device, int64_t p, const grem_config* cfg, const grem_hooks* hooks,
                       int32_t* labels_out, grem_report* rep);

/* Multi-GPU subtree sharding of partition(): every rank calls this with the
 * same edges; the owners of a recursion node are split between its two sides
 * in proportion to their edge counts (ancestors are computed redundantly and
 * bit-identically).  labels_out gets this rank's leaves, -1 elsewhere; the
 * caller merges ranks with an element-wise max (e.g. one NCCL all-reduce) and
 * runs grem_count_cuts_u32 on the merged labels. */
int grem_partition_shard_u32(grem_ctx* ctx, const uint32_t* edges, int64_t num_edges, int64_t num_nodes,
                             int edges_on_device, int64_t p, const grem_config* cfg, int rank, int world,
                             int32_t* labels_out);

/* write_buckets (streamcut/store.py:55-104): stable p x p scatter of the edge
 * list by (labels[src], labels[dst]).  p = 1 + the largest label >= 0 (1 if
 * none; < 65536) -> *p_out.  out_edges (2*num_edges u32, host or device)
 * receives the buckets row-major, input order inside a bucket; counts_out
 * (host, counts_cap >= p*p entries) the bucket sizes.  Errors: FormatError
 * "unlabeled endpoint encountered" (store.py:77-78), or counts_cap too small
 * (then *p_out is still set). */
int grem_write_buckets_u32(grem_ctx* ctx, const uint32_t* edges, int64_t num_edges, int64_t num_nodes,
                           int edges_on_device, const int32_t* labels, int labels_on_device, uint32_t* out_edges,
                           int out_on_device, uint64_t* counts_out, int64_t counts_cap, int64_t* p_out);
/* The same on a GRPE u32 file, streamed in through the overlapped reader
 * (out_edges: header num_edges pairs). */
int grem_write_buckets_file(grem_ctx* ctx, const char* path, const int32_t* labels, int labels_on_device,
                            uint32_t* out_edges, int out_on_device, uint64_t* counts_out, int64_t counts_cap,
                            int64_t* p_out);

/* reorder_features (store.py:201-235): nodes grouped by label, ascending id
 * inside a partition.  perm_out[node] = slot (int64, host); counts_out (host,
 * counts_cap >= p) = nodes per partition; records (host, num_nodes x
 * record_width bytes, optional) gathered into out_records in slot order.
 * Every node must be labeled (FormatError otherwise, store.py:216-217). */
int grem_reorder_records(grem_ctx* ctx, const int32_t* labels, int64_t num_nodes, int labels_on_device,
                         const uint8_t* records, int64_t record_width, uint8_t* out_records, int64_t* perm_out,
                         uint64_t* counts_out, int64_t counts_cap, int64_t* p_out);

/* compute_node_stats (streamcut/theory.py:97-122): per node, k = non-self-loop
 * neighbour endpoints (with multiplicity) and k0 = those on its majority side
 * of the bisection `labels`.  k_out / k0_out: num_nodes int64 (host or
 * device).  Errors: FormatError "reference labels are not a bisection" (a
 * label > 1, theory.py:107-108), "unlabeled endpoint encountered"
 * (theory.py:114-115). */
int grem_node_stats_u32(grem_ctx* ctx, const uint32_t* edges, int64_t num_edges, int64_t num_nodes,
                        int edges_on_device, const int32_t* labels, int labels_on_device, int64_t* k_out,
                        int64_t* k0_out);
/* The same on a GRPE u32 file, streamed in through the overlapped reader. */
int grem_node_stats_file(grem_ctx* ctx, const char* path, const int32_t* labels, int labels_on_device,
                         int64_t* k_out, int64_t* k0_out);

/* expected_cuts / theory_curve (streamcut/theory.py:125-146): for every x in
 * xs, cuts_out = sum over nodes with k >= 1 of (k - k0) p + k0 (1 - p),
 * p = prob_correct(k, k0, x, multiplier) (theory.py:78-94; hypergeometric
 * tail from log-gamma terms, theory.py:35-75).  k, k0: num_nodes int64 (host
 * or device).  info_out (optional, 3 int64): first node with k >= 1, first
 * such node whose k0 is not its majority side (-1 = none), sum of k (total
 * endpoints).  Errors (FormatError, in the reference's order): "empty node
 * stats" (num_nodes = 0 and nx > 0), the majority-side check, x outside
 * (0, 1], multiplier < 1; nothing is checked when every k is 0. */
int grem_theory_curve(grem_ctx* ctx, const int64_t* k, const int64_t* k0, int64_t num_nodes, int on_device,
                      const double* xs, int64_t nx, double multiplier, double* cuts_out, int64_t* info_out);

/* external_shuffle (streamcut/edgefile.py:248-327): a uniform random
 * permutation of the edge list, deterministic per seed (64-bit counter-hash
 * keys + one radix sort; the reference's numpy-PCG64 order is not
 * reproduced).  out_edges: num_edges pairs, host or device. */
int grem_shuffle_u32(grem_ctx* ctx, const uint32_t* edges, int64_t num_edges, int64_t num_nodes,
                     int edges_on_device, uint64_t seed, uint32_t* out_edges, int out_on_device);
/* The same from a GRPE u32 file (overlapped reader) to a GRPE u32 file. */
int grem_shuffle_file(grem_ctx* ctx, const char* in_path, uint64_t seed, const char* out_path);

/* Device copy of the host edge list staged by the last call on this context
 * (edges_on_device = 0); valid until the next call.  Lets a sharded caller run
 * grem_count_cuts_u32 on the merged labels without a second upload.
 * *dev_edges = NULL when the last call used device edges. */
int grem_staged_edges(grem_ctx* ctx, const uint32_t** dev_edges, int64_t* num_edges);

/* count_cuts (grem.py:227-252).  labels_on_device as for edges. */
int grem_count_cuts_u32(grem_ctx* ctx, const uint32_t* edges, int64_t num_edges, int64_t num_nodes,
                        int edges_on_device, const int32_t* labels, int labels_on_device,
                        grem_report* rep);

/* File front ends: stream a GRPE u32 file (edgefile.py:107-126,186-219)
 * through two pinned chunk buffers into HBM (the ingest subsystem), honouring
 * the meter hook, then run the path.  64-bit-id and text files are parsed by
 * the Python layer and passed to the pointer entry points above. */
int grem_bisect_file(grem_ctx* ctx, const char* path, const grem_config* cfg, int64_t capacity,
                     const grem_hooks* hooks, int32_t* labels_out, grem_report* rep);
int grem_partition_file(grem_ctx* ctx, const char* path, int64_t p, const grem_config* cfg,
                        const grem_hooks* hooks, int32_t* labels_out, grem_report* rep);
/* count_cuts (grem.py:227-252) of a GRPE u32 file: the payload streams in
 * through the same overlapped reader; labels (num_nodes int32, host or
 * device) must match the header's num_nodes. */
int grem_count_cuts_file(grem_ctx* ctx, const char* path, const int32_t* labels, int labels_on_device,
                         grem_report* rep);

/* During an on_chunk hook: D2H copy of the live parts (int32, -1 unassigned). */
int grem_state_parts(grem_ctx* ctx, int32_t* out, int64_t n);

/* ------------------------------------------------- device memory helpers */
/* Let a caller keep edges resident across calls (bench, multi-call users). */
int grem_device_alloc(grem_ctx* ctx, uint64_t bytes, void** out);
int grem_device_free(grem_ctx* ctx, void* ptr);
int grem_memcpy_h2d(grem_ctx* ctx, void* dst, const void* src, uint64_t bytes);
int grem_memcpy_d2h(grem_ctx* ctx, void* dst, const void* src, uint64_t bytes);

/* ------------------------------------------------------------- synthetic */
/* Deterministic Chung-Lu power-law edges (grem_gen.h): edges [e0, e0+count)
 * of the graph (n, beta, seed); host and device produce identical bytes. */
double grem_gen_scale(uint64_t n, uint32_t beta);
int grem_gen_edges_host(uint64_t n, uint32_t beta, uint64_t seed, uint64_t e0, uint64_t count,
                        uint32_t* out, int threads);
int grem_gen_edges_device(grem_ctx* ctx, uint64_t n, uint32_t beta, uint64_t seed, uint64_t e0,
                          uint64_t count, uint32_t* dev_out);

#ifdef __cplusplus
}
#endif
#endif /* GREM_B200_H */
