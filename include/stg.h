/*
 * stg.h — C-ABI of libstg (strata-on-B200): the per-window analysis hot path
 *   ingest -> symbolize -> aggregate -> diff -> verdict, plus collective alignment,
 * as hand-written sm_100a CUDA behind plain C entry points.
 *
 * The reference ("strata", /root/reference/proj) exposes this path only as C++20
 * free functions in namespace strata; it has no C-ABI, plugin or FFI.  Each entry
 * point below names the reference function(s) it replaces (file:line under
 * proj/core/).  The C++ drop-in shim (paper_2603_29235_b200/csrc/shim/) re-defines
 * those strata:: functions on top of this header, so reference callers relink
 * unchanged; INTEGRATION.md shows the bindings.
 *
 * Conventions
 *  - Every function returns an int status (STG_OK = 0).  On failure the message is
 *    available from stg_last_error() (thread-local).  STG_EINVAL carries exactly
 *    the strata::Error message the reference would throw for the same input.
 *  - Plain pointers and sizes only; no torch or C++ types.  Bulk sample arrays may
 *    live in host memory (copied in by the call) or already in device memory
 *    (stg_window.memory = STG_MEM_DEVICE, pointers valid on the context's GPU;
 *    frame_pc 32-byte and frame_bin 16-byte aligned, as cudaMalloc returns them).
 *  - A context owns device memory, streams and the loaded symbol tables; calls on
 *    one context are serialised by an internal mutex.
 */
#ifndef STG_H
#define STG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STG_ABI_VERSION 1

enum stg_status {
    STG_OK = 0,
    STG_EINVAL = 1, /* input rejected (strata::Error in the reference)      */
    STG_ECUDA = 2,  /* CUDA runtime / kernel failure                         */
    STG_ENOMEM = 3, /* device or host allocation failed                      */
    STG_ESTATE = 4, /* call order violated (no result yet, bad index, ...)    */
    STG_ENOTFOUND = 5
};

/* SymbolFile::LookupMode (symfile.hpp:32) */
enum stg_lookup_mode { STG_LOOKUP_EXACT_RANGE = 0, STG_LOOKUP_NEAREST_LOWER = 1 };

enum stg_memory { STG_MEM_HOST = 0, STG_MEM_DEVICE = 1 };

/* Verdict (diagnosis.hpp:159-167), same numeric order. */
enum stg_verdict {
    STG_VERDICT_HEALTHY = 0,
    STG_VERDICT_GPU_UNIFORM = 1,
    STG_VERDICT_GPU_SPECIFIC = 2,
    STG_VERDICT_CPU_INTERFERENCE = 3,
    STG_VERDICT_OS_INTERFERENCE = 4,
    STG_VERDICT_TEMPORAL = 5,
    STG_VERDICT_INCONCLUSIVE = 6
};

typedef struct stg_ctx stg_ctx;

/* ---------------------------------------------------------------- lifecycle */
const char* stg_last_error(void);
int stg_abi_version(void);
/* sizeof(stg_window), sizeof(stg_config), sizeof(stg_run_stats) as compiled —
 * lets a foreign binding (ctypes, cgo, JNI) verify its struct mirrors. */
void stg_abi_sizes(uint64_t* window, uint64_t* config, uint64_t* stats);
/* stg_create: one context per GPU (device ordinal). */
int stg_create(int device, stg_ctx** out);
void stg_destroy(stg_ctx* ctx);

/* ------------------------------------------------------------------- ingest
 * Replaces SymbolRepository::ingest/load (symrepo.cpp:35-97) + parse_symbols
 * (symfile.cpp:117-157): validates a SYMR payload with the reference's exact
 * rules and messages, and stages its table on the device (sorted starts, packed
 * {size, name}, a bucket index for the search).  Idempotent per build id
 * (IngestOutcome::AlreadyPresent -> *stored = 0).  claimed_id (20 bytes, may be
 * NULL = take the header's id) plays the role of ingest()'s key argument.
 * The 64 MiB segment SHA-1 check of the transport (symrepo.cpp:23-51) is the
 * sender's concern and is not repeated here. */
int stg_symtab_ingest(stg_ctx* ctx, const uint8_t* claimed_id, const uint8_t* symr,
                      uint64_t len, int* stored);
int stg_symtab_count(stg_ctx* ctx, uint32_t* n_tables);

/* --------------------------------------------------------------- symbolize
 * Replaces resolve_stacks (symrepo.cpp:122-143) / resolve_stack (:99-120):
 * frame-wise lookup of (build id, offset) pairs on the GPU.  Each frame gets a
 * name key; stg_name() renders it (real symbol name, or the reference's unknown
 * label "[<hex id>+0x<off>]", symfile.cpp:159-163).  Keys are valid until the
 * next call on the context and are ordered like the names they denote. */
int stg_resolve(stg_ctx* ctx, uint64_t n_frames, const uint64_t* frame_pc,
                const uint16_t* frame_bin, int32_t n_bins, const uint8_t* bin_build_ids,
                int mode, uint32_t* out_keys);
int stg_name(stg_ctx* ctx, uint32_t key, char* buf, uint64_t cap, uint64_t* needed);
int stg_name_count(stg_ctx* ctx, uint32_t* n);

/* ------------------------------------------------------------------ window
 * One analysis window in structure-of-arrays form: the in-memory equivalent of
 * strata::LoadedBundle (bundle.hpp:23-42).  Samples are grouped by rank
 * (rank-major, time-ordered within a rank as in LoadedBundle::samples). */
typedef struct stg_window {
    int32_t memory; /* stg_memory of sample_ts / sample_frame_off / frame_* */
    int32_t group;
    int64_t window_start_ns;
    int64_t window_end_ns;
    int64_t max_skew_ns;

    /* ranks that own a CPU sample stream (keys of LoadedBundle::samples) */
    int32_t n_ranks;
    const int32_t* rank_ids;         /* host, strictly ascending          */
    const uint64_t* rank_sample_off; /* host, n_ranks+1, into samples     */

    /* binaries referenced by frames: frame_bin indexes this list */
    int32_t n_bins;
    const uint8_t* bin_build_ids; /* host, n_bins * 20 bytes */

    /* CPU stack samples (StackSample, samples.hpp:15-21; spaces are ignored
     * downstream by the reference, so they are not carried) */
    uint64_t n_samples;
    const int64_t* sample_ts;         /* [n_samples] rank-local clock        */
    const uint64_t* sample_frame_off; /* [n_samples+1] CSR into frames       */
    uint64_t n_frames;
    const uint64_t* frame_pc;  /* [n_frames] code offsets, leaf first     */
    const uint16_t* frame_bin; /* [n_frames] index into bin_build_ids     */

    /* NCCL collective events (CollectiveEvent, collective.hpp:24-31), host,
     * in LoadedBundle::collectives order */
    uint64_t n_coll;
    const int32_t* coll_rank;
    const int32_t* coll_group;
    const uint8_t* coll_kind; /* CollectiveKind ordinal */
    const int64_t* coll_entry;
    const int64_t* coll_exit;
    const int64_t* coll_gpu_dur;
    int32_t n_group_ranks;
    const int32_t* group_ranks;

    /* GPU kernel events (GpuEvent, scenario.hpp:72-78), host */
    uint64_t n_gpu;
    const int32_t* gpu_rank;
    const uint32_t* gpu_kernel; /* index into kernel_names */
    const int64_t* gpu_start;
    const int64_t* gpu_dur;
    uint32_t n_kernel_names;
    const char* const* kernel_names;

    /* OS counter records (OsCounterRecord, scenario.hpp:80-84), host */
    uint64_t n_os;
    const int32_t* os_rank;
    const int64_t* os_window_start;
    const int64_t* os_p50;
    const int64_t* os_p99;
    const int64_t* os_migrations;
    const uint64_t* os_irq_off; /* n_os+1 CSR over (key, value) */
    const uint32_t* os_irq_key; /* index into counter_names      */
    const int64_t* os_irq_val;
    const uint64_t* os_sirq_off;
    const uint32_t* os_sirq_key;
    const int64_t* os_sirq_val;
    uint32_t n_counter_names;
    const char* const* counter_names;

    /* historical baseline (BaselineProfile, diagnosis.hpp:142-147).  As in a
     * LoadedBundle it is always present: has_baseline = 0 means an empty profile
     * with the default delta 0.005, has_baseline_iteration = 0 means 0.0 ms. */
    int32_t has_baseline;
    double baseline_delta;
    uint32_t n_baseline;
    const char* const* baseline_names;
    const double* baseline_fracs;
    int32_t has_baseline_iteration;
    double baseline_iteration_ms;

    /* stg_memory of the coll_* arrays (group_ranks stays host) */
    int32_t coll_memory;
    /* stg_memory of the gpu_* and os_* arrays (kernel/counter names stay host) */
    int32_t side_memory;

    /* Distributed mode only (stg_dist_init, world > 1): which per-rank streams
     * this context holds for its own ranks only, instead of identically on
     * every context.  Context p owns the ranks in [shard_rank_lo of p,
     * shard_rank_lo of p+1) (the last context: to infinity); the lower bounds
     * must increase with the world rank.  STG_SHARD_COLL: coll_* hold only the
     * owned ranks' events, in LoadedBundle::collectives order (the group's
     * event order is the contexts' lists concatenated in world-rank order) —
     * stage d (match_collectives / align_clocks / entry_lateness /
     * detect_straggler, collective.cpp:29-142, diagnosis.cpp:76-111) then runs
     * rank-sharded with per-instance partials combined over NCCL, and the
     * lateness_per_instance of the GroupData holds the owned ranks only.
     * STG_SHARD_SIDE: gpu_* / os_* likewise (per-rank sums all-reduced).
     * 0 = replicated. */
    int32_t shard_streams;
    int32_t shard_rank_lo;
} stg_window;

#define STG_SHARD_COLL 1
#define STG_SHARD_SIDE 2

/* DiagnosisConfig (diagnosis.hpp:203-210) + GpuDiffConfig (:83-92) + OsDiffConfig
 * (:127-132).  stg_config_default() fills the reference defaults. */
typedef struct stg_config {
    int32_t window_iterations;
    double k;
    double delta;
    double iteration_regression_gate;
    double gpu_median_uniform;
    double gpu_cv_uniform;
    double gpu_top_share_specific;
    double gpu_median_none;
    int64_t gpu_ref_floor_ns;
    char gpu_exclude_prefix[32];
    double os_min_ratio;
    int64_t os_interrupt_floor;
    int64_t os_sched_delay_floor_ns;
    int64_t os_migration_floor;
    int32_t lookup_mode;    /* build_group_data uses ExactRange (bundle.cpp:300) */
    int32_t want_waterline; /* also compute compute_waterline/flag_ranks     */
    /* verify = 1: after the fused symbolize+aggregate kernel, every in-window
     * sample is symbolized again frame by frame (no prefix cache) and compared
     * name by name with the representative of the aggregation slot it landed
     * in, slot counts are recounted, and every folded line's stack is compared
     * with its cross-rank sequence representative — the full compare the
     * reference does on a digest hit (samples.cpp:67-76).  A mismatch (a
     * fingerprint collision) re-runs the stage with re-keyed fingerprints and
     * no prefix cache; stats.verify_retries counts those re-runs. */
    int32_t verify;
    /* tests only: truncate the prefix-cache key to 4 bits so that distinct
     * call chains collide (exercises the verify retry).  Keep 0. */
    int32_t debug_weak_prefix_key;
} stg_config;

void stg_config_default(stg_config* cfg);

/* Counters of one run (sizes of the result, device timings of the stages). */
typedef struct stg_run_stats {
    uint64_t n_samples_in_window;
    uint64_t n_lines;        /* Σ over ranks of folded lines                 */
    uint64_t n_sequences;    /* distinct symbolized stacks across all ranks  */
    uint64_t n_names;        /* size of the result name space                */
    uint64_t n_unknown;      /* distinct unresolved frames                   */
    uint64_t n_instances;    /* matched collective instances                 */
    uint64_t n_windowed;     /* complete instances inside the window         */
    uint64_t n_cpu_ranks;    /* ranks with a CPU profile                     */
    int32_t verdict;
    int32_t n_flagged;
    float ms_collectives;    /* device time per stage (CUDA events)          */
    float ms_symbolize;      /* the fused symbolize+aggregate kernel         */
    float ms_fold;
    float ms_diff;
    float ms_total;
    uint64_t h2d_bytes;
    uint64_t d2h_bytes;
    uint32_t kernel_launches;
    uint32_t agg_attempts;   /* >1 when a rank table had to grow           */
    uint64_t prefix_hits;    /* symbolization memo hits (raw call chains)  */
    uint64_t prefix_misses;
    uint32_t verified;       /* 1 when cfg.verify checked this run clean   */
    uint32_t verify_retries; /* re-runs after a detected collision         */
} stg_run_stats;

/* Replaces build_group_data (bundle.cpp:252-324) followed by diagnose
 * (diagnosis.cpp:301-432): the whole window batch on the GPU, keeping the
 * result (GroupData + DiagnosisReport) in the context for the getters below. */
int stg_window_run(stg_ctx* ctx, const stg_window* win, const stg_config* cfg,
                   stg_run_stats* stats);

/* -------------------------------------------------------------- distributed
 * One communication group spanning several GPUs: one process
 * (one context) per GPU; the window's CPU sample streams are sharded by rank
 * across the contexts (each passes only its ranks in rank_ids / samples), while
 * collectives, GPU events, OS counters and the baseline are passed identically
 * to every context.  Inside stg_window_run the contexts exchange over NCCL only
 * what the verdict needs: exact inclusive fractions of the straggler and the
 * reference rank and the straggler's hottest path (broadcast from their owner),
 * per-GPU merged stack lists for the temporal route (all-gather, re-merged and
 * sorted on each GPU), and the waterline's per-name sums (all-reduce).  Every
 * context ends with the same report.  All contexts must hold the same symbol
 * tables.  stg_dist_unique_id is called on world rank 0; the caller ships the
 * 128 bytes to the others (e.g. torch.distributed.broadcast). */
int stg_dist_unique_id(uint8_t id[128]);
int stg_dist_init(stg_ctx* ctx, int world_size, int world_rank, const uint8_t id[128]);

/* Canonical JSON renderings of the last window's result (for parity tests and
 * tools): GroupData (every field of diagnosis.hpp:192-201), and the report exactly
 * as DiagnosisReport::to_json (diagnosis.cpp:437-455) writes it (nlohmann
 * dump(2), byte-identical).  Two-call size query: pass buf=NULL to get *needed. */
int stg_result_groupdata_json(stg_ctx* ctx, char* buf, uint64_t cap, uint64_t* needed);
/* The same rendering without the bulky parts a binding fetches structurally
 * (parts = STG_GD_ALL & ~STG_GD_CPU: cpu_profiles comes back empty; read the
 * folded lines with stg_result_rank_lines instead). */
#define STG_GD_CPU 1u
#define STG_GD_ALL 0xffffffffu
int stg_result_groupdata_json_parts(stg_ctx* ctx, uint32_t parts, char* buf, uint64_t cap, uint64_t* needed);
int stg_result_report_json(stg_ctx* ctx, char* buf, uint64_t cap, uint64_t* needed);
/* DiagnosisReport::to_text (diagnosis.cpp:457-481) of the last window's report;
 * like stg_result_report_json (which is to_json's nlohmann dump(2)), the same
 * bytes the reference writes. */
int stg_result_report_text(stg_ctx* ctx, char* buf, uint64_t cap, uint64_t* needed);
/* Waterline (compute_waterline, diagnosis.cpp:35-55) + flag_ranks (:57-71) over
 * the last window's CPU profiles, when cfg.want_waterline was set. */
int stg_result_waterline_json(stg_ctx* ctx, char* buf, uint64_t cap, uint64_t* needed);

/* Structured access to the folded profiles of the last window (to_folded,
 * folded.cpp:56-71): per CPU rank, lines in the reference's lexicographic
 * order as name-key sequences (root first) with counts. */
int stg_result_rank_count(stg_ctx* ctx, uint32_t* n);
int stg_result_rank_info(stg_ctx* ctx, uint32_t i, int32_t* rank, uint64_t* n_lines,
                         uint64_t* total, uint64_t* n_keys);
int stg_result_rank_lines(stg_ctx* ctx, uint32_t i, uint64_t* line_key_off /* n_lines+1 */,
                          uint32_t* keys, uint64_t* counts);

/* ---- bundle ingest (load_bundle, bundle.cpp:181-233) ----
 * Loads a bundle directory as written by write_bundle (bundle.cpp:83-164):
 * meta.json, gpu_events.jsonl and os_counters.jsonl on the host (nlohmann::json,
 * as the reference), samples.jsonl and collectives.jsonl decoded on the GPU into
 * a device-resident window, and the binaries' SYMR tables ingested from
 * <dir>/symbols/.  The window stays owned by the context until the next load;
 * stg_bundle_window returns it (memory = coll_memory = STG_MEM_DEVICE) for
 * stg_window_run.  Errors: the reference's messages for missing files
 * ("missing bundle file: <path>"), build ids and collective kinds; nlohmann's own
 * text for the host-parsed files; "<file> line N: <what>" for malformed bulk lines. */
typedef struct stg_bundle_info {
    uint32_t n_ranks, n_bins, n_tables_ingested, pad;
    uint64_t n_samples, n_frames, n_coll, n_gpu, n_os;
    uint64_t bulk_bytes;        /* samples.jsonl + collectives.jsonl */
    double read_s, decode_s;    /* file reads; GPU decode of the bulk files */
    double total_s;
} stg_bundle_info;

int stg_bundle_load(stg_ctx* ctx, const char* dir, stg_bundle_info* info);
int stg_bundle_window(stg_ctx* ctx, stg_window* out);
/* Copy bytes from the context's device memory (e.g. a bundle window's arrays). */
int stg_device_to_host(stg_ctx* ctx, void* dst, const void* src, uint64_t bytes);

/* ---- raw-address ProfileWindow API (aggregate_samples, samples.hpp:38-44) ----
 * One rank's time-ordered sample stream, structure of arrays.  Frames are raw
 * (bin, offset) pairs, leaf first; a bin stands for one build id (callers intern
 * build ids to bins, so equal FrameRefs (vprocess.hpp:48-53) have equal pairs).
 * rank may be NULL (then the mixed-rank check is skipped). */
typedef struct stg_stream {
    int32_t memory;            /* STG_MEM_HOST or STG_MEM_DEVICE */
    uint64_t n_samples;
    const int64_t* ts;         /* [n_samples] StackSample.timestamp_ns */
    const int32_t* rank;       /* [n_samples] StackSample.rank, or NULL */
    const uint64_t* frame_off; /* [n_samples + 1] CSR into the frame arrays */
    const uint64_t* frame_pc;  /* FrameRef.offset */
    const uint16_t* frame_bin; /* FrameRef.build_id as a bin index */
} stg_stream;

enum stg_agg_flags { STG_AGG_FORCE_EXACT = 1 /* tests: skip the fingerprint table */ };

/* aggregate_samples (samples.cpp:31-85) on the GPU: windows on the drain grid,
 * per window the distinct stacks in first-seen order with their counts (counts
 * sum to n_samples).  A record is reported as the index of its first sample (its
 * frames are that sample's frames) and its count.  Errors carry the reference's
 * messages: "drain interval must be positive", "empty sample stack",
 * "aggregate_samples: mixed ranks", "aggregate_samples: timestamps regressed"
 * (first offending sample in stream order). */
int stg_aggregate_samples(stg_ctx* ctx, const stg_stream* stream, int64_t drain_interval_ns, int flags,
                          uint64_t* n_windows, uint64_t* n_records);
/* Window bounds [start, end) and record offsets (n_windows + 1) of the last call. */
int stg_aggregate_windows(stg_ctx* ctx, int64_t* start_ns, int64_t* end_ns, uint64_t* record_off);
/* Records of the last call: first sample index and count (n_records each). */
int stg_aggregate_records(stg_ctx* ctx, uint64_t* first_sample, uint64_t* count);

/* Folded-text artifacts of the last window, rendered on the device (two-call
 * size query like the JSON getters; *needed counts the trailing NUL).
 *   stg_result_folded_text  FoldedProfile::to_string (folded.cpp:33-43) of the
 *                           rank's CPU profile — what `strata flamegraph` writes
 *                           to <out>.folded (tools/strata.cpp:119-131).
 *   stg_result_diff_folded  diff_folded(profile(a), profile(b)) (folded.cpp:83-96)
 *                           — what `strata diagnose` writes per flagged rank
 *                           against the reference rank (tools/strata.cpp:97-109).
 * A rank without a CPU profile fails with "unknown rank id: <rank>" (rank_profile,
 * tools/strata.cpp:111-116).  In a distributed group both ranks must be held by
 * this context. */
int stg_result_folded_text(stg_ctx* ctx, int32_t rank, char* buf, uint64_t cap, uint64_t* needed);
int stg_result_diff_folded(stg_ctx* ctx, int32_t rank_a, int32_t rank_b, char* buf, uint64_t cap,
                           uint64_t* needed);

/* Flame graphs of the last window (render_flamegraph / render_diff_flamegraph,
 * svg.cpp:157-172, options as SvgOptions svg.hpp): the same SVG bytes the
 * reference writes for FoldedProfile(rank) — or for the diff of rank_before's
 * profile against rank_after's — from the device-resident folded lines.  opts
 * NULL = the reference defaults (1200, 16, 0.001, "flame graph").  Two-call size
 * query; "unknown rank id: <rank>" for a rank without a CPU profile. */
typedef struct stg_svg_options {
    int32_t width;
    int32_t row_height;
    double min_fraction;
    const char* title;
} stg_svg_options;
int stg_result_flamegraph_svg(stg_ctx* ctx, int32_t rank, const stg_svg_options* opts, char* buf, uint64_t cap,
                              uint64_t* needed);
int stg_result_diff_flamegraph_svg(stg_ctx* ctx, int32_t rank_before, int32_t rank_after,
                                   const stg_svg_options* opts, char* buf, uint64_t cap, uint64_t* needed);

#ifdef __cplusplus
}
#endif

#endif /* STG_H */
