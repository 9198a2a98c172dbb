/*
 * gnncache_b200.h — C-ABI of libgnncache_b200.so, the B200 (sm_100a) data-preparation
 * path of Legion (arXiv 2305.16588): local shuffle, k-hop CSR sampling, sub-graph
 * dedup + relabel, three-tier feature gather, presampling hotness, cache-plan scans.
 *
 * The reference (`gnncache` 0.1.0, /root/reference/pkg/src/gnncache) is pure
 * Python/numpy and has no FFI: its boundary is a set of Python functions over
 * numpy arrays. Each entry point below names the reference function it replaces
 * (file:line, relative to pkg/src/gnncache/). The Python package
 * paper_2305_16588_b200 binds these through ctypes and keeps the reference's
 * Python signatures, dataclasses and exception types on top of them.
 *
 * Conventions
 *  - every function returns int status: GC_OK (0) or a negative GC_ERR_* code;
 *    gc_last_error() returns a thread-local message for the last failure.
 *  - all buffers are caller-owned. "d_" = device pointer (local HBM, a mapped peer
 *    pointer, or a UVA pointer to mapped pinned host memory); sizes are element counts.
 *  - `stream` is a cudaStream_t passed as void*; every call is asynchronous on it
 *    and never synchronises the device (so a caller may capture calls in a CUDA graph).
 *  - vertex ids are uint32 (the reference guarantees n < 2^32, graph.py:158-159);
 *    row offsets are uint64 (graph.py:65-66).
 *  - "batched" entry points process a window of W independent mini-batches in one
 *    launch; batch b's data lives at base + b*stride and its element count is read
 *    from a device array, so no host round trip is needed between hops.
 */
#ifndef GNNCACHE_B200_H
#define GNNCACHE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GC_ABI_VERSION 1

#define GC_OK 0
#define GC_ERR_VALUE (-1)       /* -> ValueError      (sampling.py:42-48, :128-131; planner.py:107,:119) */
#define GC_ERR_OVERFLOW (-2)    /* -> OverflowError   (sampling.py:298-299) */
#define GC_ERR_CUDA (-3)        /* -> RuntimeError    (device failure; no CPU fallback exists) */
#define GC_ERR_UNSUPPORTED (-4) /* -> NotImplementedError */
#define GC_ERR_ASSERT (-5)      /* -> AssertionError  (planner.py:317-318) */

#define GC_MAX_PEERS 8
#define GC_TIER_HOST 0xFFFFFFFFu /* location-table value for host-resident rows */

int gc_abi_version(void);
/* Process-wide options. GC_OPT_EXACT_SELECTION=1 makes hop expansion skip the packed
 * 32-bit REDUX extraction and always use the 64-bit path (a test hook: both paths
 * must give identical output). */
#define GC_OPT_EXACT_SELECTION 1
/* GC_OPT_DEFER_CTAS: CTAs (one warp each, TMA bulk copies) of gc_gather_deferred's
 * host-row kernel (default 296, two per SM); a tuning knob for the PCIe-bound part. */
#define GC_OPT_DEFER_CTAS 2
/* GC_OPT_GATHER_CTAS_PER_SM: grid of the warp-per-row gather in CTAs per SM over the
 * whole window (default 16: the GPU is full). Fewer leave SM room for another lane's
 * kernels while a PCIe-bound gather runs. */
#define GC_OPT_GATHER_CTAS_PER_SM 3
/* GC_OPT_UNIQUE_BATCH_CTAS: gc_unique_compact's dense path runs one CTA per batch (one
 * launch) when the window has at least this many batches, else three per-tile passes
 * (0, the default: the SM count). Both give identical outputs. */
#define GC_OPT_UNIQUE_BATCH_CTAS 4
/* GC_OPT_DEFER_ORDER: 1 (default) = gc_gather_deferred reads the window's host rows in
 * ascending id (address) order (a bucket sort of the deferred list first); 0 = in the
 * order the gather listed them. Both give identical outputs. */
#define GC_OPT_DEFER_ORDER 5
/* GC_OPT_DEFER_ROWS: rows in flight per CTA of gc_gather_deferred's host-row kernel
 * (0, the default: ~32 KB of rows, at most 64). With GC_OPT_DEFER_CTAS, a few CTAs with
 * many rows each hold only a few SMs (shared memory), leaving the others free. */
#define GC_OPT_DEFER_ROWS 6
int gc_set_option(int option, int value);
const char* gc_last_error(void);
/* device ordinal of the calling thread's current device; -1 if none */
int gc_current_device(void);

/* ------------------------------------------------------------------ RNG (rng.py) */

/* mix64_array, rng.py:34-42 */
int gc_mix64(const uint64_t* d_in, uint64_t* d_out, int64_t n, void* stream);
/* KeyedRng.hash_counters, rng.py:64-66 */
int gc_hash_counters(uint64_t key, const int64_t* d_counters, uint64_t* d_out, int64_t n, void* stream);
/* KeyedRng.hash_pairs, rng.py:68-72 */
int gc_hash_pairs(uint64_t key, const int64_t* d_a, const int64_t* d_b, uint64_t* d_out, int64_t n,
                  void* stream);

/* K1: KeyedRng.permutation (rng.py:78-82) = stable argsort of hash_counters(0..n-1),
 * optionally fused with the gather `pool[perm]` of run_sampling_epoch (sampling.py:231).
 * d_pool may be NULL (then d_out receives perm itself). n < 2^31. */
size_t gc_permutation_temp_bytes(int64_t n);
int gc_permutation(uint64_t key, int64_t n, const int64_t* d_pool, int64_t* d_out, void* d_temp,
                   size_t temp_bytes, void* stream);
/* Same, with the shuffle key read from device memory at run time, so a CUDA graph
 * captured once replays every epoch's shuffle (SampleGatherPipeline.run_epoch_graph). */
int gc_permutation_dkey(const uint64_t* d_key, int64_t n, const int64_t* d_pool, int64_t* d_out, void* d_temp,
                        size_t temp_bytes, void* stream);

/* ---------------------------------------------------------- topology (graph.py) */

/* CsrGraph layout, graph.py:62-96: row_offsets u64[n+1], col_indices u32[m]. The
 * pointers may be local HBM or UVA-mapped pinned host memory (the host topology tier). */
typedef struct gc_csr {
    int64_t num_vertices;
    int64_t num_edges;
    const uint64_t* row_offsets;
    const uint32_t* col_indices;
} gc_csr_t;

/* Tiered topology (Legion's topology cache): the neighbour list of v is read from
 *  - `full` when location == NULL (whole CSR in HBM, or UVA-mapped pinned host memory);
 *  - otherwise location[v] == GC_TIER_HOST -> `full` (the host tier, over PCIe), or
 *    location[v] == (g<<28)|slot -> clique GPU g's compact CSR slab
 *    (slab_offsets[g][slot..slot+1] into slab_cols[g]; g == self_rank is local HBM,
 *    any other g is read one-sided over NVLink through a mapped peer pointer).
 * tier_reads (optional, u64[7]) += {positions, sampled edges} served {local, peer, host},
 * and [6] += sum of t(v) = 1 + ceil(deg*4/CLS) over host-tier reads (PCIe transactions,
 * sampling.py:177-187; CLS and the id width come from `hot` when given, else 64 and 4). */
typedef struct gc_topology {
    gc_csr_t full;
    const uint32_t* location;
    const uint64_t* slab_offsets[GC_MAX_PEERS];
    const uint32_t* slab_cols[GC_MAX_PEERS];
    uint32_t self_rank;
    uint32_t full_on_host; /* 1: `full` is pinned host memory (reads of it count as the host tier) */
    uint64_t* tier_reads;
} gc_topology_t;

/* K8 cache fill: copy the neighbour lists of ids[0..count) from `src` (HBM or mapped
 * host CSR) into a compact slab whose offsets d_slab_offsets[0..count] the caller has
 * already laid out (exclusive scan of the degrees, planner.py:310 byte accounting). */
int gc_csr_extract(const gc_csr_t* src, const int64_t* d_ids, int64_t count, const uint64_t* d_slab_offsets,
                   uint32_t* d_slab_cols, void* stream);

/* ------------------------------------------------- hotness (sampling.py:146-289) */

/* Device hotness counters of one GPU (GpuTrace, sampling.py:190-197). Any pointer may
 * be NULL to skip that counter. Counters are u64 (the u32 dump limit, sampling.py:298,
 * only applies when writing the file). */
typedef struct gc_hotness {
    uint64_t* topo_reads;      /* [n] frontier occurrences (sampling.py:238) */
    uint64_t* edge_traversals; /* [n] sampled edges out of v (sampling.py:239-241) */
    uint64_t* feat_lookups;    /* [n] per-batch distinct appearances (sampling.py:242) */
    uint64_t* txn_total;       /* [1] sum of t(v) over reads (sampling.py:284-288) */
    uint32_t cache_line_bytes; /* HardwareSpec.cache_line_bytes (hardware.py:167) */
    uint32_t uint32_bytes;     /* HardwareSpec.uint32_bytes (hardware.py:168) */
} gc_hotness_t;

/* Per-batch visited sets of a window (the dedup state, K3). `bitmap` holds one bit per
 * vertex, `words` u32 per batch (gc_bitmap_words). The optional `summary` holds one bit
 * per 32-word block (1024 vertices), set when a block's first bit is set, so
 * compaction touches only non-empty blocks: O(distinct + n/1024) per batch instead of
 * O(n/32) — what makes 100M-vertex graphs cheap. summary_words = gc_summary_words(n). */
typedef struct gc_visited {
    uint32_t* bitmap;
    uint64_t words;
    uint32_t* summary;
    uint64_t summary_words;
} gc_visited_t;

/* ------------------------------------------- K2: hop expansion (sampling.py:84-143) */

/* One hop of _expand_frontier (sampling.py:84-117) for W batches at once.
 *  frontier of batch b: d_frontier + b*frontier_stride, d_frontier_count[b] entries
 *  hop key of batch b : d_hop_keys[b] = stream.derive(h).key (sampling.py:135)
 *  output offsets     : d_out_offsets + b*offsets_stride, count+1 entries (u32, exclusive scan of take)
 *  output neighbors   : d_out_nbrs + b*nbrs_stride, d_out_count[b] entries
 *  visited (optional)  : per-batch visited sets; every emitted neighbour is marked, and
 *                       the frontier too if mark_frontier.
 *  hot (optional)     : presampling counters of the sampling GPU.
 * Neighbour lists come from the topology tier that holds them (gc_topology_t).
 * Selection is bit-exact with the reference: deg<=fanout copies the CSR slice in order,
 * otherwise the fanout smallest (hash_pairs(i,j), j) are emitted in ascending order.
 * Requires max_frontier*fanout < 2^32. */
size_t gc_hop_expand_temp_bytes(uint32_t num_batches, uint32_t max_frontier);
int gc_hop_expand(const gc_topology_t* topo, const uint32_t* d_frontier, uint64_t frontier_stride,
                  const uint32_t* d_frontier_count, uint32_t max_frontier, uint32_t fanout,
                  const uint64_t* d_hop_keys, uint32_t num_batches, uint32_t* d_out_offsets,
                  uint64_t offsets_stride, uint32_t* d_out_nbrs, uint64_t nbrs_stride, uint32_t* d_out_count,
                  const gc_visited_t* visited, int mark_frontier, const gc_hotness_t* hot,
                  void* d_temp, size_t temp_bytes, void* stream);

/* ------------------------------- K3: dedup + relabel (BatchSample.distinct_vertices) */

/* Words per batch bitmap for n vertices (padded for 16-byte vector access). */
uint64_t gc_bitmap_words(int64_t num_vertices);
/* Words per batch of the block summary (one bit per 32 bitmap words). */
uint64_t gc_summary_words(int64_t num_vertices);
/* np.unique of seeds ∪ all hop neighbors (sampling.py:73-75) from the visited bitmaps:
 * sorted distinct ids of batch b -> d_unique + b*unique_stride, count -> d_unique_count[b];
 * d_rank_table (optional, 2*bitmap_words u32 per batch) receives {exclusive popcount
 * prefix, bitmap word} per word for gc_relabel. feat_lookups (optional) += 1 per
 * distinct id (sampling.py:242). clear_bitmap zeroes the bitmap as it is consumed.
 * At most unique_stride ids are written per batch; d_unique_count[b] always holds the
 * true distinct count, so d_unique_count[b] > unique_stride reports an overflow (the
 * caller raises; the bitmap is still cleared in full). */
size_t gc_unique_temp_bytes(uint32_t num_batches, const gc_visited_t* visited);
int gc_unique_compact(const gc_visited_t* visited, uint32_t num_batches, uint32_t* d_unique,
                      uint64_t unique_stride, uint32_t* d_unique_count, uint32_t* d_rank_table,
                      uint64_t* d_feat_lookups, int clear_bitmap, void* d_temp, size_t temp_bytes,
                      void* stream);
/* Kernels one gc_unique_compact call launches for this window (launch accounting). */
int gc_unique_compact_launches(uint32_t num_batches, const gc_visited_t* visited);
/* Relabel (not in the reference; CPU restatement np.searchsorted(unique, ids)):
 * d_local[b*stride + k] = index of d_ids[b*stride + k] in batch b's unique list. */
int gc_relabel(const uint32_t* d_ids, uint64_t ids_stride, const uint32_t* d_ids_count, uint32_t max_count,
               uint32_t num_batches, const uint32_t* d_rank_table, uint64_t bitmap_words, uint32_t* d_local,
               void* stream);
/* The same with 16-bit local ids (every batch of the window has <= 65536 distinct
 * vertices): d_local holds u16, element stride ids_stride. */
int gc_relabel16(const uint32_t* d_ids, uint64_t ids_stride, const uint32_t* d_ids_count, uint32_t max_count,
                 uint32_t num_batches, const uint32_t* d_rank_table, uint64_t bitmap_words, uint16_t* d_local,
                 void* stream);
/* Mark ids in the per-batch visited sets (seeds of a zero-hop config). */
int gc_mark_visited(const uint32_t* d_ids, uint64_t ids_stride, const uint32_t* d_count, uint32_t max_count,
                    uint32_t num_batches, const gc_visited_t* visited, void* stream);
/* Zero the visited words touched by batch b's unique ids (reset after clear_bitmap=0). */
int gc_bitmap_clear(const gc_visited_t* visited, uint32_t num_batches, const uint32_t* d_unique,
                    uint64_t unique_stride, const uint32_t* d_unique_count, uint32_t max_unique, void* stream);

/* ------------------------------------------------ K4: three-tier feature gather */

/* Feature store of one GPU (the tier rule of account_assignment, simulator.py:161-202).
 * location[v] == GC_TIER_HOST -> host_rows + v*row_bytes (UVA over PCIe)
 * location[v] == (g<<28)|slot -> slabs[g] + slot*row_bytes (g == self_rank: local HBM,
 *                                otherwise the owner's slab read over NVLink/NVSwitch)
 * location == NULL            -> slabs[self_rank] + v*row_bytes (fully resident table) */
typedef struct gc_feature_store {
    uint32_t row_bytes; /* FeatureSpec.row_bytes (graph.py:220-222); multiple of 4 */
    uint32_t self_rank;
    uint32_t num_ranks;
    uint32_t reserved;
    const uint32_t* location;
    const void* slabs[GC_MAX_PEERS];
    const void* host_rows;
} gc_feature_store_t;

/* out[b*out_stride_rows + k] = row(d_ids[b*ids_stride + k]) for k < min(d_count[b], max_count).
 * d_tier_rows (optional, u64[3]) += rows served by local / peer / host. */
int gc_gather(const gc_feature_store_t* store, const uint32_t* d_ids, uint64_t ids_stride,
              const uint32_t* d_count, uint32_t max_count, uint32_t num_batches, void* d_out,
              uint64_t out_stride_rows, uint64_t* d_tier_rows, void* stream);

/* Same result as gc_gather, scheduled for overlap: rows of the local and peer tiers
 * are copied by the full-width kernel, host-tier rows are appended to `d_defer`
 * (gc_gather_defer_bytes(max_count, num_batches) bytes of device memory) and copied
 * by a second, small-grid kernel on `host_stream` (NULL: the same stream; `stream`
 * waits for it either way). The PCIe-bound part then
 * occupies ~1 CTA per SM and runs under the next window's sampling on another
 * stream (Legion's inter-batch pipeline). Falls back to gc_gather's
 * schedule when the store has no host tier or rows are not 16-byte vectors. */
uint64_t gc_gather_defer_bytes(uint32_t max_count, uint32_t num_batches);
int gc_gather_deferred(const gc_feature_store_t* store, const uint32_t* d_ids, uint64_t ids_stride,
                       const uint32_t* d_count, uint32_t max_count, uint32_t num_batches, void* d_out,
                       uint64_t out_stride_rows, uint64_t* d_tier_rows, void* d_defer, uint64_t defer_bytes,
                       void* stream, void* host_stream);

/* Deterministic synthetic feature rows [first_row, first_row+rows) of a dim-wide fp32
 * table: X[v,d] = (mix64(v*dim+d) >> 40) * 2^-24 - 0.5 (bench/test input only). */
int gc_synth_features(uint64_t first_row, uint64_t rows, uint32_t dim, float* d_out, void* stream);

/* ---------------------------------------------- K5: hotness scatter (sampling.py:164-174) */

/* accumulate_hotness's bincount: d_counter[d_ids[k]] += (d_weights ? d_weights[k] : 1). */
/* Trainer helper (not in the reference): out[i] = mean of x[idx[k]] over
 * k in [offsets[i], offsets[i+1]) (0 for an empty segment), fp32, x row-major [*, dim].
 * The first GraphSAGE layer's neighbour mean taken straight from the gathered rows. */
int gc_segment_mean_gather(const float* d_x, int dim, const int64_t* d_idx, const int64_t* d_offsets, int64_t segs,
                           float* d_out, void* stream);
int gc_scatter_add(const uint32_t* d_ids, const uint32_t* d_weights, int64_t count, uint64_t* d_counter,
                   void* stream);

/* ---- Tree trainer (not in the reference; Legion's PyTorch backend).
 * A sampled batch is a position tree: level 0 = seeds, level h+1 = hop h's neighbours
 * (no dedup between hops, sampling.py:123-125), every position relabelled to a row of
 * the batch's gathered feature matrix. Levels are stacked; level k padded to caps[k]. */
#define GC_TREE_MAX_LEVELS 8
typedef struct {
    int32_t hops;                                    /* L; levels 0..L */
    const int32_t* counts;                           /* [L+1, W] real positions per level */
    int64_t counts_stride;                           /* W */
    const int32_t* local[GC_TREE_MAX_LEVELS];        /* level k relabelled ids [W, local_stride[k]] (u16 when local_bits == 16) */
    int64_t local_stride[GC_TREE_MAX_LEVELS];
    const int32_t* offsets[GC_TREE_MAX_LEVELS];      /* hop h child offsets [W, offsets_stride[h]] */
    int64_t offsets_stride[GC_TREE_MAX_LEVELS];
    const int32_t* seeds;                            /* global seed ids [W, seeds_stride] */
    int64_t seeds_stride;
    const int64_t* labels;                           /* class per vertex [n] (nullable) */
    int64_t caps[GC_TREE_MAX_LEVELS];                /* padded slots per level */
    int32_t local_bits;                              /* 16: local[] hold u16 ids (gc_relabel16); else u32 */
} gc_tree_src_t;

/* Stage batch *d_batch (device scalar, so a captured graph replays for any batch):
 * loc[P] feature row of each stacked position (0 when padded); for levels 0..L-1,
 * cbeg/cdeg = stacked first child and child count; level_counts[L+1] = real positions
 * per level; labels[caps[0]] = labels[seed] or -100 for padding. */
int gc_tree_stage(const gc_tree_src_t* src, const int32_t* d_batch, int32_t* d_loc, int32_t* d_cbeg, int32_t* d_cdeg,
                  int32_t* d_level_counts, int64_t* d_labels, void* stream);
/* Neighbour aggregation of one layer for positions [0, p_out). mode 0 (GraphSAGE):
 * out[p] = [in[row(p)], mean of in[row(c)] over children c] (2*dim columns); mode 1
 * (GCN): out[p] = (in[row(p)] + sum in[row(c)]) / (deg(p) + 1); mode + 2: ReLU applied
 * to every input row as it is read (the input is a layer's pre-activations). row(q) =
 * (*d_batch) * batch_rows + (rowmap ? rowmap[q] : q). dtypes: 0 fp32, 1 bf16 (fp32 ->
 * bf16 allowed); sums in fp32 in child order. dim and strides: 16-byte multiples. */
int gc_tree_aggregate(const void* d_in, int in_dtype, int64_t in_stride, int dim, const int32_t* d_rowmap,
                      const int32_t* d_cbeg, const int32_t* d_cdeg, int64_t p_out, int mode, void* d_out, int out_dtype,
                      int64_t out_stride, const int32_t* d_batch, int64_t batch_rows, void* stream);
/* Its backward for input rows [0, p_in), fused with the ReLU mask of the input
 * pre-activations h (nullable): g[q] = [h[q] > 0] * (cs(q) dA[q, self] +
 * cc(parent(q)) dA[parent(q), child]); SAGE cs = 1, cc = 1/deg; GCN 1/(deg+1).
 * Rows [0, p_in) span levels 0..nlevels-1 of level_caps (host array); rows past
 * d_level_counts[k] (padding) are written as zeros. */
int gc_tree_aggregate_backward(const void* d_dA, int dtype, int64_t dA_stride, int dim, int mode,
                               const int32_t* d_cbeg, const int32_t* d_cdeg, int64_t p_out, int64_t p_in,
                               const void* d_h, int64_t h_stride, void* d_g, int64_t g_stride, int nlevels,
                               const int64_t* level_caps, const int32_t* d_level_counts, void* stream);

/* Classifier head of the tree trainer: for seed rows [0, rows) of the top layer's
 * pre-activations z (dtype 0 fp32 / 1 bf16), top = relu(z), logits = top W^T + b
 * (W fp32 [classes, hid], cast to the activation type as operands, fp32 sums),
 * cross entropy over labels (< 0: padding) averaged over *d_nvalid rows -> *d_loss;
 * d_dW [classes, hid] and d_db [classes] receive the gradients and d_g [rows, hid]
 * (dtype) the gradient with respect to z (ReLU mask applied). Deterministic
 * (fixed-order sums); d_work holds gc_tree_head_work_floats(rows, classes, hid) floats. */
size_t gc_tree_head_work_floats(int64_t rows, int classes, int hid);
int gc_tree_head(const void* d_z, int dtype, int64_t z_stride, int hid, int64_t rows, const float* d_W,
                 const float* d_b, int classes, const int64_t* d_labels, const int32_t* d_nvalid, float* d_loss,
                 float* d_dW, float* d_db, void* d_g, int64_t g_stride, float* d_work, size_t work_floats,
                 void* stream);

/* ------------------------------------------- K6/K7: cost model (planner.py:42-261) */

/* Column sums and first argmax over K rows (planner.py:50-55): rows are int64 [K][n]. */
int gc_colsum_argmax(const int64_t* d_rows, uint32_t k_rows, int64_t n, int64_t* d_totals, int32_t* d_owner,
                     void* stream);
/* hotness_descending_order (planner.py:42-45): ids sorted by totals descending, ties by
 * ascending id. totals must be >= 0. */
size_t gc_descending_order_temp_bytes(int64_t n);
int gc_descending_order(const int64_t* d_totals, int64_t n, int64_t* d_order, void* d_temp, size_t temp_bytes,
                        void* stream);
/* Inclusive scans along an order (planner.py:87-95, :239-240):
 *   d_topo_bytes[i] = sum_{k<=i} deg(order[k])*u32_bytes + u64_bytes   (needs graph offsets)
 *   d_hot_cum[i]    = sum_{k<=i} totals[order[k]] */
size_t gc_order_scan_temp_bytes(int64_t n);
int gc_topo_prefix_bytes(const uint64_t* d_row_offsets, const int64_t* d_order, int64_t n, uint32_t u32_bytes,
                         uint32_t u64_bytes, int64_t* d_out, void* d_temp, size_t temp_bytes, void* stream);
int gc_hot_prefix(const int64_t* d_totals, const int64_t* d_order, int64_t n, int64_t* d_out, void* d_temp,
                  size_t temp_bytes, void* stream);
/* np.searchsorted(prefix, budgets, side="right") with float64 budgets compared as
 * (double)prefix <= budget (planner.py:236-237). */
int gc_searchsorted_right(const int64_t* d_prefix, int64_t n, const double* d_budgets, int32_t num_budgets,
                          int64_t* d_out, void* stream);
/* distribute_prefix (planner.py:264-267): stable split of order[0:len) by owner.
 * d_out receives the concatenation of the k_rows queues, d_counts[g] their lengths. */
size_t gc_distribute_prefix_temp_bytes(int64_t len, uint32_t k_rows);
int gc_distribute_prefix(const int64_t* d_order, int64_t len, const int32_t* d_owner, uint32_t k_rows,
                         int64_t* d_out, int64_t* d_counts, void* d_temp, size_t temp_bytes, void* stream);

/* ---------------------------------- K9: tier accounting (simulator.py:132-203) */

/* holders[v] |= 1 << local_gpu for v in ids (clique membership masks, simulator.py:125-129);
 * holders is u8[n] padded to a multiple of 4 bytes. */
int gc_mark_holders(const int64_t* d_ids, int64_t count, uint32_t local_gpu, uint8_t* d_holders, void* stream);
/* One GPU's TrafficReport row from its epoch trace: out u64[10 + 2k] =
 * {topo_reads, topo_local_hits, topo_peer_hits, sampling_cpu_txn, sampling_peer_txn,
 *  feat_lookups, feat_local_hits, feat_peer_hits, feature_cpu_txn, feature_peer_txn,
 *  topology peer txn by serving GPU [k], feature peer txn by serving GPU [k]};
 * the serving peer is the lowest-index holder (simulator.py:168-169). */
int gc_tier_account(const uint64_t* d_row_offsets, int64_t n, const uint64_t* d_topo_reads,
                    const uint64_t* d_feat_lookups, const uint8_t* d_topo_holders, const uint8_t* d_feat_holders,
                    uint32_t local_gpu, uint32_t clique_size, uint32_t cache_line_bytes, uint32_t uint32_bytes,
                    uint32_t row_txns, uint64_t* d_out, void* stream);

/* --------------------------------------- host tier + peer mapping (plumbing) */

/* Register host memory as mapped, read-only pinned memory (UVA host tier). */
int gc_host_register(void* host_ptr, size_t bytes, void** d_alias);
int gc_host_unregister(void* host_ptr);
/* Copy `bytes` (a multiple of 4) from device memory into mapped pinned host memory with
 * SM stores (no DMA engine: small reads that must not queue behind bulk D2H copies). */
int gc_copy_d2h_mapped(const void* d_src, void* h_dst, uint64_t bytes, void* stream);
/* Pack a padded window array for delivery (SampleGatherPipeline.window_to_host): batch
 * b's rows [0, d_ptr[b+1] - d_ptr[b]) of `row_bytes` bytes at d_src + b*src_stride_bytes
 * go to d_dst from row d_ptr[b] on; max_rows bounds every batch's row count (grid size).
 * mode: 0 copy (rows of u32 words), 1 u32 -> u16 (low 16 bits: relabelled ids of a window
 * whose batches have <= 65536 distinct vertices), 2 copy u16, 3 u16 -> u32, 4 u32 offsets
 * -> u8 counts (row i becomes src[i+1] - src[i]; d_ptr counts the rows, i.e. a hop's
 * frontier positions, and src holds one more offset per batch). */
int gc_pack_segments(const void* d_src, uint64_t src_stride_bytes, uint64_t row_bytes, const int64_t* d_ptr,
                     uint32_t num_batches, uint64_t max_rows, int mode, void* d_dst, void* stream);

/* Host tier through the CUDA VMM API (cuMemCreate, CU_MEM_LOCATION_TYPE_HOST_NUMA):
 * pinned host memory mapped for the CPU and every GPU at one address with the
 * allocation granularity as the GPU page size (2 MB), so random UVA row reads over a
 * large host table miss the GPU TLB far less than with cudaHostAlloc's 4 KB pages.
 * `*mapped_bytes` (bytes rounded up to the granularity) must be passed to the free. */
int gc_host_alloc_numa(size_t bytes, int numa_node, void** ptr, size_t* mapped_bytes);
int gc_host_free_numa(void* ptr, size_t mapped_bytes);
/* Synthetic graph targets (generate_synthetic, graph.py:144-177) on the device: edge
 * e in [first_edge, first_edge + count) gets searchsorted(cdf, u_e, side="right")
 * with u_e the e-th numpy Generator.random() double of the PCG64 stream whose 128-bit
 * state/increment the caller passes (Generator.bit_generator.state), self-loops
 * redirected to (t + 1) % n. d_cdf: the reference's float64 Zipf cdf (host-computed).
 * Bit-identical to the reference's column array. */
int gc_synth_zipf_targets(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                          const double* d_cdf, uint64_t num_vertices, uint64_t degree, uint64_t first_edge,
                          uint64_t count, uint32_t* d_out, void* stream);
/* Cross-process NVLink peer slabs: 64-byte cudaIpcMemHandle_t of the allocation
 * holding d_ptr, plus d_ptr's byte offset from that allocation's base (caching
 * allocators sub-allocate). gc_ipc_import maps the allocation and returns its base;
 * the peer address of the exported pointer is base + offset. */
int gc_ipc_export(void* d_ptr, uint8_t* handle64, uint64_t* offset);
int gc_ipc_import(const uint8_t* handle64, void** d_ptr);
int gc_ipc_close(void* d_ptr);
/* Enable peer access from the current device to `peer` (same-process multi-GPU). */
int gc_enable_peer(int peer);

/* Inter-clique LDG partition, host preprocessing (replaces partition_inter_clique's
 * placement + refinement, src/partition.py:85-152). All arrays are HOST memory:
 * the CSR, the BFS root order (KeyedRng(seed).derive(0x5EED).permutation(n), computed
 * by gc_permutation), capacity = the reference's int((1 + eps) * ceil(n / parts)).
 * Writes h_assignment[n]; h_cuts (optional, 2 * refine_passes) receives the edge cut
 * before/after each refinement pass run. GC_ERR_ASSERT if a pass raised the cut. */
int gc_partition_ldg(const uint64_t* h_row_offsets, const uint32_t* h_cols, uint64_t num_vertices,
                     uint64_t num_edges, const int64_t* h_root_order, uint32_t num_parts, int64_t capacity,
                     int refine_passes, int32_t* h_assignment, uint64_t* h_cuts);

#ifdef __cplusplus
}
#endif
#endif /* GNNCACHE_B200_H */
