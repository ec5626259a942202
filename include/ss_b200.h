/*
 * ss_b200.h -- C ABI of the B200 sliding-window GROUP BY engine.
 *
 * One `ss_engine` owns every piece of device state for one GPU: the
 * per-group window rings, the group -> partition (block) assignment with
 * its ordered per-partition lists, and the scratch of the per-batch
 * pipeline.  All entry points take plain pointers and sizes; a pointer
 * may be host memory (pageable or pinned) or device memory -- the engine
 * inspects it with cudaPointerGetAttributes and stages host data itself.
 * Calls are stream-ordered on the engine's stream (ss_set_stream), not
 * thread-safe per handle, and return an `int` status (SS_OK or SS_E_*).
 *
 * Each entry point replaces one function of the reference package
 * `skewstream` (/root/reference/pkg/src/skewstream); the mapping is noted
 * beside it (reference file:line).  The Python shim
 * (paper_1309_0634_b200/_lib.py) binds exactly these symbols with ctypes.
 */
#ifndef SS_B200_H
#define SS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes -> errors.py:4-29 (mapped in paper_1309_0634_b200/errors.py) */
#define SS_OK            0
#define SS_E_DATA        1  /* DataError: group id outside [0, G) (partition.py:119-126) */
#define SS_E_CONFIG      2  /* InvalidConfigError (balance.py:56-65, partition.py:189-197) */
#define SS_E_SPEC        3  /* InvalidSpecError */
#define SS_E_CONSISTENCY 4  /* ConsistencyError (partition.py:170-173, engine.py:283-284) */
#define SS_E_STALE_MOVE  5  /* StaleMoveError (partition.py:198-200) */
#define SS_E_EXEC        6  /* ExecutionError: CUDA / NCCL failure (engine.py:410-416) */

/* aggregate mask: COUNT and SUM are the reference's own state
 * (engine.py:67-70); AVG/MIN/MAX are derived from the same window. */
#define SS_AGG_COUNT 1u
#define SS_AGG_SUM   2u
#define SS_AGG_AVG   4u
#define SS_AGG_MIN   8u
#define SS_AGG_MAX  16u

/* balancer policies, Policy enum of balance.py:28-35 */
#define SS_POLICY_NO         0
#define SS_POLICY_FIRST      1
#define SS_POLICY_ALL        2
#define SS_POLICY_PROB       3
#define SS_POLICY_BEST       4
#define SS_POLICY_SHIFT      5
#define SS_POLICY_SHIFTLOCAL 6

/* move placement, partition.py:23-24 */
#define SS_FRONT 0
#define SS_BACK  1

typedef struct ss_engine ss_engine;

typedef struct {
    int64_t  n_groups;      /* G: dense group ids 0..G-1 (datagen.py:81-103)          */
    int64_t  window;        /* W: per-group window length (harness.py:43, engine.py:60)*/
    int32_t  n_partitions;  /* P: processing units = aggregate-kernel CTAs           */
    int32_t  key_bits;      /* 32: u32 group ids; 64: int64 keys (ss_step_keys64)     */
    uint32_t agg_mask;      /* SS_AGG_* bits that must be maintained                  */
    int32_t  scope;         /* 0: per-group window (the reference semantics);         */
                            /* 1: the stream's last W tuples, grouped (policy 'no')    */
    int32_t  device;        /* CUDA ordinal                                           */
    int32_t  reserved;
    int64_t  max_batch;     /* largest n passed to ss_step (0: 1<<24; <= 2^30)        */
    int64_t  sub_batch;     /* count chunk: tuple granularity at which never-stored   */
                            /* tuples are dropped (power of two >= 2^16; 0: auto)     */
    int64_t  pool_values;   /* ring pool capacity in values (0: auto)                 */
} ss_config;

typedef struct {
    int32_t policy;          /* SS_POLICY_*                                  */
    int32_t reserved;
    int64_t thread_threshold;/* balance.py:48 (>= 1)                         */
    double  pot;             /* balance.py:49, in (0, 1]                     */
    int64_t max_moves;       /* balance.py:50; 0 = 4 * P (balance.py:64-65)  */
    int32_t split;           /* hot-key splitting across blocks (new)        */
    int32_t split_max;       /* max shares per split group (0: P)            */
    double  split_target;    /* max/mean load the splitter aims for (1.2)    */
} ss_balancer;

typedef struct {
    int32_t group;
    int32_t src;
    int32_t dst;
    int32_t placement;       /* SS_FRONT / SS_BACK */
} ss_move;

typedef struct {
    int64_t tuples;          /* IterationReport.tuples (engine.py:173)                 */
    int64_t imbalance;       /* max(tpt) - min(tpt) (engine.py:313,320)                */
    int64_t moves;           /* moves emitted by this batch's policy                   */
    int64_t moves_applied_before; /* harness.py:113 row.moves                           */
    int64_t scanned;         /* MoveList.scanned_tuples (balance.py:68-80)             */
    int64_t max_load;        /* max per-block load incl. split shares (same unit)       */
    int64_t touched;         /* groups with >= 1 tuple in the batch                    */
    int64_t split_groups;    /* groups executed as split shares this batch            */
    double  mean_load;       /* sum of block loads / P (tuples; values to store with split) */
    double  load_ratio;      /* max_load / mean_load                                    */
} ss_step_report;

/* ---- lifecycle ------------------------------------------------------ */
int  ss_create(const ss_config* cfg, ss_engine** out);        /* WindowStore(G, W), engine.py:60-70 */
void ss_destroy(ss_engine* e);
int  ss_set_stream(ss_engine* e, void* cuda_stream);          /* stream the engine enqueues on */
int  ss_sync(ss_engine* e);
const char* ss_last_error(ss_engine* e);
const char* ss_version(void);
/* kernels this library has launched (all engines); reset != 0 zeroes it */
long long ss_launch_count(int reset);
/* replay the fused step as cached CUDA graphs (default on; inputs whose
 * addresses change every batch turn it off automatically) */
int  ss_set_graphs(ss_engine* e, int enable);
/* the engine's count-chunk size (tuples) */
long long ss_sub_batch(ss_engine* e);

/* ---- assignment (partition.py:45-114, 181-203) ------------------------ */
/* order[G]: concatenated per-partition lists; offsets[P+1] into order. */
int  ss_set_assignment(ss_engine* e, const int32_t* order, const int64_t* offsets);
int  ss_get_assignment(ss_engine* e, int32_t* g2t, int32_t* order, int64_t* offsets);
int  ss_apply_moves(ss_engine* e, const ss_move* moves, int64_t n);   /* apply_moves, partition.py:181-203 */

/* ---- partition step (partition.py:117-178) ---------------------------- */
int  ss_count(ss_engine* e, const uint32_t* groups, int64_t n,
              int64_t* group_counts, int64_t* tpt);                   /* count_batch, partition.py:117-130 */
int  ss_reorder(ss_engine* e, const uint32_t* groups, const int32_t* attrs, int64_t n,
                uint32_t* out_groups, int32_t* out_attrs, int64_t* indicator);  /* reorder_batch, 161-178 */

/* ---- aggregate update (engine.py:185-321) ----------------------------- */
/* ingest_sequence (engine.py:253-296): stable per-group arrival order. */
int  ss_ingest(ss_engine* e, const uint32_t* groups, const int32_t* attrs, int64_t n);

/* ---- balancer (balance.py:141-405) ------------------------------------ */
/* Runs the policy on one batch against the current assignment; does not
 * apply the moves (the reference policies are pure, test_balance.py:355). */
int  ss_balance(ss_engine* e, const uint32_t* groups, int64_t n, const ss_balancer* cfg,
                ss_move* moves, int64_t* n_moves, int64_t* scanned, int64_t* final_tpt);

/* ---- fused per-batch step: harness.run loop body (harness.py:99-117) ---
 * count -> policy (device, overlapped) -> stable rank + window update per
 * L2-resident sub-batch -> per-group result emission -> apply moves.  The
 * moves decided on batch t are in force from batch t+1. */
int  ss_step(ss_engine* e, const uint32_t* groups, const int32_t* attrs, int64_t n,
             const ss_balancer* cfg, ss_step_report* rep);
/* report of the last ss_step (synchronises) */
int  ss_last_report(ss_engine* e, ss_step_report* rep);
/* per-partition tuple loads of the last step (incl. split shares) */
int  ss_last_loads(ss_engine* e, int64_t* loads);
/* per-partition aggregate-kernel time (ns, summed over sub-batches) of the
 * last step: IterationReport.per_thread_cost (engine.py:395-398) */
int  ss_last_part_ns(ss_engine* e, int64_t* ns);
/* values stored by each partition's window update in the last batch */
int  ss_last_part_work(ss_engine* e, int64_t* work);
/* moves emitted by the last step */
int  ss_last_moves(ss_engine* e, ss_move* moves, int64_t cap, int64_t* n);

/* ---- state export (engine.py:51-93) ----------------------------------- */
/* Any output pointer may be NULL.  avg = (double)sum / fill, 0 when empty. */
int  ss_snapshot(ss_engine* e, int64_t* fill, int64_t* next_pos, int64_t* window_sum,
                 int32_t* mn, int32_t* mx, double* avg);
/* Window of one group in arrival order, oldest first (WindowStore.contents, engine.py:72-77). */
int  ss_export_values(ss_engine* e, int64_t group, int64_t* out, int64_t cap, int64_t* n);
/* Per-batch emission of the last ss_step: groups touched by the batch and
 * their COUNT/SUM/AVG/MIN/MAX after it.  Sizes: cap entries each. */
int  ss_results(ss_engine* e, int64_t cap, int32_t* groups, int64_t* count, int64_t* sum,
                double* avg, int32_t* mn, int32_t* mx, int64_t* n);

/* ---- int64 group keys (key_bits = 64; BASELINE C4/C5) ------------------
 * Keys map to dense slots 0..G-1 in order of first appearance in the
 * stream (a device hash table); every other entry point then sees slots. */
int  ss_map_keys(ss_engine* e, const int64_t* keys, int64_t n, uint32_t* out_slots);
/* replay ingest: n records of the reference's replay format
 * (8 bytes: u32 group, i32 attr; datagen.py:29,250-296), host (pinned) or
 * device (16-byte aligned); otherwise identical to ss_step */
/* per-tuple trace (AggregateTrace engine.py:125-164): in
 * trace mode every step keeps all tuples and records, per tuple, its group and
 * the window sum after it, in grouped-projection order (group ids ascending,
 * arrival order within a group); ss_trace copies the last batch's records */
int  ss_set_trace(ss_engine* e, int enable);
int  ss_trace(ss_engine* e, int64_t cap, int32_t* groups, int64_t* sums, int64_t* n);
int  ss_step_records(ss_engine* e, const void* records, int64_t n, const ss_balancer* cfg, ss_step_report* rep);
int  ss_step_keys64(ss_engine* e, const int64_t* keys, const int32_t* attrs, int64_t n,
                    const ss_balancer* cfg, ss_step_report* rep);
/* int64 keys, large G: the probe + count of batch t+1 runs on its own
 * stream while batch t finishes.  Host inputs always overlap; device key
 * inputs overlap only when declared ready at call time (ready_inputs = 1:
 * not produced by work still pending on the engine stream). */
int  ss_set_key_pipeline(ss_engine* e, int ready_inputs);
/* key of every assigned slot (keys[n_slots]) */
int  ss_slot_keys(ss_engine* e, int64_t* keys, int64_t* n_slots);

/* ---- multi-GPU: groups shard by key across GPUs ----------- */
/* owner_of[G] in [0, n_dest), n_dest <= 16 */
int  ss_set_owner(ss_engine* e, const int32_t* owner_of, int n_dest);
/* stable split of a batch by owning GPU (arrival order kept per owner);
 * counts[n_dest] tuples per destination */
int  ss_route(ss_engine* e, const uint32_t* groups, const int32_t* attrs, int64_t n,
              uint32_t* out_groups, int32_t* out_attrs, int64_t* counts);
/* per-group counts of the last step's batch */
int  ss_group_counts(ss_engine* e, int32_t* counts);
/* policy on given per-group counts (BatchStats.group_counts, balance.py:175-385) */
int  ss_balance_counts(ss_engine* e, const int32_t* counts, const ss_balancer* cfg, ss_move* moves,
                       int64_t* n_moves, int64_t* scanned, int64_t* final_tpt);
/* window-state migration: meta[5n] = (fill, next_pos, sum, min, max), values
 * = ring images (span = fill if fill < W else W) concatenated */
int  ss_export_state(ss_engine* e, const int32_t* groups, int64_t n, int64_t* meta, int32_t* values,
                     int64_t cap, int64_t* n_values);
int  ss_import_state(ss_engine* e, const int32_t* groups, int64_t n, const int64_t* meta,
                     const int32_t* values);

/* ---- device-resident multi-GPU data plane (no host reads; stream-ordered
 * on the engine's stream, which the sharded host code sets to the stream
 * NCCL runs on).  Replaces the host-staged route / count / policy /
 * migration steps above for ShardedEngine.step (harness.py:99-117 run at
 * GPU level; balance.py:141-172 with threads = GPUs; moves apply at t+1,
 * harness.py:115-116). */
/* stable split by owner into 8-byte (u32 group, i32 attr) records (device);
 * counts_dev[n_dest] per destination, counts_dev[n_dest] = first bad tuple
 * index or -1 (device) */
int  ss_route_records(ss_engine* e, const uint32_t* groups, const int32_t* attrs, int64_t n,
                      void* out_records, int64_t* counts_dev);
/* owner map from a device array */
int  ss_set_owner_dev(ss_engine* e, const int32_t* owner_dev, int n_dest);
/* policy on device counts, moves applied to this engine's assignment on the
 * device; moves (int4 group, src, dst, placement)[cap], their count and the
 * new group -> partition map copied into device buffers */
int  ss_balance_apply_dev(ss_engine* e, const int32_t* counts_dev, const ss_balancer* cfg, void* moves_dev,
                          int32_t* n_moves_dev, int32_t* pmap_dev);
/* window state of the groups this rank gives away (moves with src == rank)
 * into per-destination blob segments: [n] ++ n x (g, fill, next_pos, sum_lo,
 * sum_hi, min, max, span) ++ ring images; sizes_dev[n_dest] words each
 * (-1: blob_cap too small) */
int  ss_export_moves_dev(ss_engine* e, const void* moves_dev, const int32_t* n_moves_dev, int rank,
                         int32_t* blob_dev, int64_t blob_cap_words, int64_t* sizes_dev);
/* received segments (word offsets seg_off[n_seg + 1], host) -> window state */
int  ss_import_blob_dev(ss_engine* e, const int32_t* blob_dev, const int64_t* seg_off, int n_seg,
                        int max_groups);
/* int64 keys across GPUs: keys shard by a 16-bit hash bucket; the GPU-level
 * engine assigns the 2^16 buckets ("groups") to GPUs.  Bucket -> GPU map
 * (host or device, 65536 entries); route into 12-byte (key lo, key hi,
 * attr) records; the step on received records; per-bucket counts of the
 * last batch; migration of the keys of moved buckets (segments per
 * destination: [n] ++ n x (key lo, key hi, fill, next_pos, sum lo, sum hi,
 * min, max, span) ++ ring images); import (keys claim slots at once). */
int  ss_set_bucket_owner(ss_engine* e, const int32_t* owner, int n_dest);
int  ss_route_records64(ss_engine* e, const int64_t* keys, const int32_t* attrs, int64_t n, void* out_records,
                        int64_t* counts_dev);
int  ss_step_records64(ss_engine* e, const void* records, int64_t n, const ss_balancer* cfg, ss_step_report* rep);
int  ss_bucket_counts_dev(ss_engine* e, int32_t* counts_dev);
int  ss_export_moves64_dev(ss_engine* e, const void* moves_dev, const int32_t* n_moves_dev, int rank,
                           int32_t* blob_dev, int64_t blob_cap_words, int64_t* sizes_dev);
int  ss_import_blob64_dev(ss_engine* e, const int32_t* blob_dev, const int64_t* seg_off, int n_seg);

/* ---- measurement ------------------------------------------------------
 * Kernel classes timed with CUDA events on the engine stream while
 * profiling is enabled (bench.py's roofline numbers). */
#define SS_K_COUNT   0   /* k_count                                  */
#define SS_K_STATS   1   /* k_batch_stats + k_scan_*                 */
#define SS_K_PLACE   2   /* k_sort_pass (all passes)                 */
#define SS_K_INGEST  3   /* k_ingest (+ reserve, finalize, rescan)   */
#define SS_K_EMIT    4   /* k_emit                                   */
#define SS_K_APPLY   5   /* k_apply_* + k_report                     */
#define SS_K_BALANCE 6   /* k_balance (side stream)                  */
#define SS_K_NCLASS  7
int  ss_profile(ss_engine* e, int enable);
/* summed milliseconds and launch counts per class since the last reset */
int  ss_profile_read(ss_engine* e, double* ms, int64_t* launches, int reset);
/* algorithmic HBM bytes of the steps since the last reset:
 * B*(key+attr) + 4*sum min(k,W) + 4*sum_{k<W} max(0,f0+k-W) + 76*touched */
int  ss_alg_bytes(ss_engine* e, int64_t* bytes, int reset);
/* streaming emission: when enabled, every ss_step writes its
 * rows -- group id plus the configured aggregate columns (agg_mask: COUNT,
 * SUM, AVG, MIN, MAX) -- straight into mapped pinned host memory
 * (double-buffered); ss_results_pull returns the oldest batch not yet pulled,
 * waiting only for that batch (rows in emission order, unconfigured columns
 * come back as 0).  Pull at least every other batch.  A batch rejected on the
 * device (group id outside [0, G)) is reported by the pull of that batch as
 * SS_E_DATA with its tuple index (partition.py:119-126); it and the batches
 * issued after it are not applied.  With host inputs, ss_step's H2D runs on
 * a copy stream into alternating staging buffers, so the next batch's copy
 * overlaps the current batch's compute (host buffers must stay unchanged
 * until the step after next has been issued). */
int  ss_set_host_emit(ss_engine* e, int enable);
int  ss_results_pull(ss_engine* e, int64_t cap, int32_t* groups, int64_t* count, int64_t* sum,
                     double* avg, int32_t* mn, int32_t* mx, int64_t* n);
/* raw per-batch emission (no ordering): group id and AVG of each touched group */
int  ss_results_raw(ss_engine* e, int64_t cap, int32_t* groups, double* avg, int64_t* n);

#ifdef __cplusplus
}
#endif
#endif /* SS_B200_H */
