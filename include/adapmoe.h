/*
 * adapmoe.h — C ABI of the B200-native AdapMoE offloaded-MoE decode path.
 *
 * The reference (moesim, header-only C++20; `inc/` = /root/reference/proj/include/moesim) exposes
 * this path as a C++ header API + file formats + CLI flags and has no C ABI/FFI of its own
 * (SURVEY.md §8(b)).  Every entry point below replaces one reference function or CLI step; the
 * replaced interface is cited on each declaration.  A C++ facade with the reference's own names
 * (adapmoe::simulate_trace, adapmoe::dp_allocate, ...) sits above this ABI in
 * paper_2408_10284_b200/csrc/host/ (C++ headers); the Python mirror is paper_2408_10284_b200/moesim.py.
 *
 * Conventions
 *   - Every call returns an int status in the reference CLI's exit-code classes
 *     (proj/tools/moesim_main.cpp:26-40) plus MOE_E_DEVICE for CUDA failures; exceptions never
 *     cross the ABI.  moe_last_error() returns the calling thread's last message.
 *   - Plain pointers and sizes only.  Arrays are row-major, C-contiguous, host memory unless the
 *     name says `d_`.  The caller owns every buffer it passes; the engine owns device memory, the
 *     pinned host expert store, streams, events and its copy thread.
 *   - An engine handle is re-entrant per handle and must not be shared across threads
 *     concurrently (inc/simulator.hpp:329 is single-threaded).
 *   - Functions marked [host] need no GPU; all others need the CUDA device the engine was
 *     created on and fail with MOE_E_DEVICE (never fall back to CPU) when it is absent.
 */
#ifndef ADAPMOE_H
#define ADAPMOE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (proj/tools/moesim_main.cpp:26-31) ---------------------------------------- */
#define MOE_OK 0
#define MOE_E_USAGE 1        /* std::invalid_argument / std::domain_error / out_of_range  */
#define MOE_E_IO 2           /* io_error (inc/io.hpp:23)                                   */
#define MOE_E_FORMAT 3       /* parse_error / schema_error / version_error (inc/io.hpp:28-37) */
#define MOE_E_VALIDATION 4   /* inputs fail cross-validation (validate_trace, inc/core.hpp:249) */
#define MOE_E_INFEASIBLE 5   /* infeasible budget / allocation                             */
#define MOE_E_DEVICE 6       /* CUDA error or no device (extension; the reference has no GPU) */
#define MOE_E_INTERNAL 7     /* std::logic_error (internal invariant)                     */

/* [host] thread-local message of the last failing call ("" if none) */
const char* moe_last_error(void);
/* [host] library version string */
const char* moe_version(void);

/* ---- value types -------------------------------------------------------------------------- */
/* ModelSpec (inc/core.hpp:22-37) */
typedef struct {
    int32_t num_layers;        /* L */
    int32_t experts_per_layer; /* N (2..64) */
    int32_t top_k;             /* K */
    int32_t hidden_dim;        /* d */
} moe_model_spec;

/* SimConfig + PolicyFlags (inc/simulator.hpp:26-50) */
typedef struct {
    int32_t tile_count_per_expert;
    int64_t tile_transfer_time;
    int64_t tile_compute_time;
    int64_t attention_compute_time;
    int64_t gate_compute_time;
    int32_t lookahead_depth; /* 0..3 */
    int32_t adaptive_gating;
    int32_t prefetch;
    int32_t adaptive_cache;
} moe_sim_config;

/* SimMetrics scalars (inc/simulator.hpp:149-166); per-token/per-layer vectors are separate args */
typedef struct {
    int64_t total_latency;
    int64_t stall_time;
    int64_t on_demand_loads;
    int64_t cache_hits;
    int64_t prefetch_hits;
    int64_t single_expert_decisions;
    int64_t experts_activated_total;
} moe_metrics;

/* TimelineEvent (inc/simulator.hpp:130-141): stream 0=compute 1=comm; kind 0 attention, 1 gate,
 * 2 expert_compute, 3 tile_compute, 4 tile_transfer. */
typedef struct {
    int64_t stream, kind, start, end, token, layer, expert, tile;
} moe_event;

/* SynthConfig + LayerScales (inc/workload.hpp:14-49) */
typedef struct {
    moe_model_spec spec;
    int32_t tokens;
    double dirichlet_concentration;
    double residual_drift;
    uint64_t gate_seed;
    uint64_t token_seed;
    int32_t shared_gates;
    const double* fisher_scales; /* [L] or NULL (all ones) */
    const double* drift_scales;  /* [L] or NULL (all ones) */
} moe_synth_config;

/* ---- [host] policy tools ------------------------------------------------------------------- */
/* calibrate_threshold (inc/gating.hpp:85-122; CLI `calibrate`, moesim_main.cpp:160):
 * scores [T][L][N] post-softmax, fisher [L]; writes tau and the realized single ratio. */
int moe_calibrate_threshold(const moe_model_spec* spec, const double* scores, int32_t tokens,
                            const double* fisher, double target_single_ratio, double* tau,
                            double* realized_single_ratio);

/* build_cost_table (inc/cache_model.hpp:189-204): alpha/beta [L] -> table [L][N+1] */
int moe_build_cost_table(const moe_model_spec* spec, const double* alpha, const double* beta, double* table);

/* dp_allocate (inc/allocator.hpp:66-88; CLI `allocate`, moesim_main.cpp:232): knapsack over the
 * cost table.  budget is clamped to L*N like the reference; capacities [L]. */
int moe_dp_allocate(const moe_model_spec* spec, const double* table, int32_t budget, int32_t* capacities,
                    double* total_cost);

/* uniform_allocation (inc/allocator.hpp:140-153) */
int moe_uniform_allocation(const moe_model_spec* spec, int32_t budget, int32_t* capacities);

/* expected_cost (inc/cache_model.hpp:71-74) */
int moe_expected_cost(int32_t t, int32_t n, double alpha, double beta, double* cost);

/* tile_pipeline_latency (inc/simulator.hpp:55-60) */
int moe_tile_pipeline_latency(int32_t tiles, int64_t transfer, int64_t compute, int64_t* latency);

/* Tick-model policy engine replay over router outputs already computed (by moe_route_trace):
 * the cache/transfer half of simulate_trace (inc/simulator.hpp:343-468).  decisions [T][L][K]
 * (-1 padded), predictions [T][L][3][2+K] rows (target, count, experts..., -1 padded).
 * events may be NULL; *n_events always receives the event count. */
int moe_replay_policy(const moe_model_spec* spec, int32_t tokens, const int32_t* capacities,
                      const moe_sim_config* cfg, uint64_t seed, const int32_t* decisions,
                      const int32_t* decision_single, const int32_t* predictions, moe_metrics* metrics,
                      int64_t* latency_per_token, int64_t* on_demand_per_layer, moe_event* events,
                      int64_t events_capacity, int64_t* n_events);

/* ---- [host] artifact files (inc/io.hpp; CLI file arguments, moesim_main.cpp:91-122) ---------------
 * The reference's JSON / JSON Lines formats (format_version 1), read without a JSON library and
 * written byte-for-byte like the reference (sorted keys, shortest round-trip doubles, dump(2)), plus a
 * binary trace container (magic "MOETRB1") for fast loading of Mixtral-width traces; loaders detect
 * it by content.  Errors: MOE_E_IO (cannot open / write), MOE_E_FORMAT (parse / schema / version),
 * MOE_E_VALIDATION (shapes that contradict the model).  Array arguments may be NULL on a first call
 * to query sizes ("two-call" convention). */
typedef struct moe_trace_file* moe_trace_t;

/* load_trace (inc/io.hpp:146): JSONL or binary by content */
int moe_trace_load(const char* path, moe_trace_t* out);
int moe_trace_info(moe_trace_t trace, moe_model_spec* spec, int32_t* tokens);
/* acts [T][L][d], scores [T][L][N], selected [T][L][K] (-1 padded); any pointer may be NULL */
int moe_trace_read(moe_trace_t trace, double* acts, double* scores, int32_t* selected);
/* validate_trace (inc/core.hpp:249-297): *violations = count; first message copied (truncated) */
int moe_trace_validate(moe_trace_t trace, int64_t* violations, char* first_message, int64_t message_capacity);
int moe_trace_free(moe_trace_t trace);
/* save_trace (inc/io.hpp:127) when binary == 0, else the binary container; selected may be NULL
 * (then the first K entries are not written: pass the generator's selections) */
int moe_trace_save(const char* path, const moe_model_spec* spec, int32_t tokens, const double* acts, const double* scores,
                   const int32_t* selected, int32_t binary);

/* load_gates / save_gates (inc/io.hpp:200-245): gates [L][d][N]; the optional trained first-layer
 * gate [d][N] with its TrainingConfig (learning_rate, steps, seed). */
int moe_gates_load(const char* path, moe_model_spec* spec, double* gates, double* first_gate, int32_t* has_first_gate,
                   double* learning_rate, int32_t* steps, uint64_t* seed);
int moe_gates_save(const char* path, const moe_model_spec* spec, const double* gates, const double* first_gate,
                   double learning_rate, int32_t steps, uint64_t seed);

/* load_profiles / save_profiles (inc/io.hpp:249-287): alpha = single_expert_prob, beta =
 * prefetch_accuracy, fisher = fisher_diag_sum, per layer.  profile_hash (inc/io.hpp:290) = 16 hex
 * characters + NUL. */
int moe_profiles_load(const char* path, moe_model_spec* spec, double* alpha, double* beta, double* fisher);
int moe_profiles_save(const char* path, const moe_model_spec* spec, const double* alpha, const double* beta,
                      const double* fisher, char* profile_hash_out);

/* load_threshold / save_threshold (inc/io.hpp:294-318) */
int moe_threshold_load(const char* path, double* tau, double* target_single_ratio, double* realized_single_ratio);
int moe_threshold_save(const char* path, double tau, double target_single_ratio, double realized_single_ratio);

/* load_allocation / save_allocation (inc/io.hpp:320-350); profile_hash 16 hex + NUL */
int moe_allocation_load(const char* path, int32_t* budget, int32_t* num_layers, int32_t* capacities, double* total_cost,
                        char* profile_hash);
int moe_allocation_save(const char* path, int32_t budget, int32_t num_layers, const int32_t* capacities,
                        double total_cost, const char* profile_hash);

/* load_cost_table / save_cost_table (inc/io.hpp:352-370): loads [L][N+1] */
int moe_cost_table_load(const char* path, int32_t* experts_per_layer, int32_t* num_layers, double* loads);
int moe_cost_table_save(const char* path, int32_t experts_per_layer, int32_t num_layers, const double* loads);

/* ---- device engine ------------------------------------------------------------------------ */
typedef struct moe_engine* moe_engine_t;

/* Creates the per-GPU engine: streams, events, router workspace.  No weights yet. */
int moe_engine_create(const moe_model_spec* spec, int32_t device, moe_engine_t* out);
int moe_engine_destroy(moe_engine_t engine);

/* Upload the per-layer gate matrices (GateMatrix, inc/prefetch.hpp:13-38; io `load_gates`,
 * inc/io.hpp:227) as row-major fp64 [L][d][N], plus the optional trained first-layer gate
 * (PredictiveGate, inc/prefetch.hpp:146) [d][N] or NULL. */
int moe_load_gates(moe_engine_t engine, const double* gates, const double* first_gate);

/* K1 on device-resident hidden states, stream-ordered (SURVEY §8(b) moe_router_forward): the
 * routing step of one layer for B rows inside a caller's decode loop.  x: device fp64 [B][d] (the
 * layer's router input).  scores: device fp64 [B][N] stored post-softmax scores to decide from
 * (trace replay, inc/simulator.hpp:390-396), or NULL to decide from softmax(x . W_layer).  Items per
 * row: the decision, then look-ahead predictions x . W_{layer+1..layer+lookahead} (at the last layer
 * the first-layer predictive gate, if loaded, as item 1), each with the sensitivity gate when
 * flags & MOE_ROUTE_ADAPTIVE (else plain top-K).  Outputs (device, row r = b*(1+lookahead) + item):
 * selected [rows][K] (-1 padded), count [rows], single [rows], perturbation [rows] (may be NULL).
 * fisher: host [L].  stream: a cudaStream_t (NULL = the engine's compute stream).  Returns once the
 * work is enqueued; the caller synchronises its stream before reading the outputs. */
#define MOE_ROUTE_ADAPTIVE 1
typedef struct {
    int32_t* selected;
    int32_t* count;
    int32_t* single;
    double* perturbation;
} moe_route_out;
int moe_router_forward(moe_engine_t engine, int32_t layer, const double* x, int32_t rows, const double* scores,
                       double tau, const double* fisher, int32_t lookahead, int32_t flags, const moe_route_out* out,
                       void* stream);

/* K1 batched router over a whole trace (replaces the reference's per-call GateMatrix::logits +
 * softmax + top_k + gate_decide_sensitivity inside simulate_trace, inc/simulator.hpp:368-444,
 * and the stored-score decision at :390-396).  acts [T][L][d] fp64, scores [T][L][N] fp64, fisher
 * [L].  Writes decisions [T][L][K], decision_single [T][L], perturbation [T][L] (NULL ok) and
 * predictions [T][L][3][2+K] exactly as simulate_trace would evaluate them. */
int moe_route_trace(moe_engine_t engine, const double* acts, const double* scores, int32_t tokens,
                    const double* fisher, double tau, const moe_sim_config* cfg, int32_t* decisions,
                    int32_t* decision_single, double* perturbation, int32_t* predictions);

/* simulate_trace (inc/simulator.hpp:329-468) with the router on the GPU (K1) and the tick-model
 * cache/transfer engine on the host.  Bit-exact drop-in for the reference's metrics + timeline. */
int moe_simulate_trace(moe_engine_t engine, const double* acts, const double* scores, int32_t tokens,
                       const double* fisher, const int32_t* capacities, double tau, const moe_sim_config* cfg,
                       uint64_t seed, moe_metrics* metrics, int64_t* latency_per_token,
                       int64_t* on_demand_per_layer, moe_event* events, int64_t events_capacity,
                       int64_t* n_events);

/* compare_policies (inc/simulator.hpp:476-550; CLI `compare`, moesim_main.cpp:356): the Table-2
 * ablation grid.  For each of the 7 rows (baseline, +gating, +prefetch, +gating+cache,
 * +prefetch+cache, +gating+prefetch, all): alpha masked to 0 without adaptive gating, beta masked to
 * 0 without prefetching, DP allocation (adaptive cache) or uniform split of `budget`, then
 * simulate_trace with the row's flags (K1 on the GPU, tick engine on the host).  rows[7];
 * capacities [7][L]; latency_per_token [7][T] and on_demand_per_layer [7][L] may be NULL. */
typedef struct {
    char name[24];
    int32_t adaptive_gating, prefetch, adaptive_cache;
    moe_metrics metrics;
    double speedup_vs_baseline;
} moe_compare_row;

int moe_compare_policies(moe_engine_t engine, const double* acts, const double* scores, int32_t tokens,
                         const double* fisher, const double* alpha, const double* beta, double tau,
                         const moe_sim_config* cfg, int32_t budget, uint64_t seed, moe_compare_row* rows,
                         int32_t* capacities, int64_t* latency_per_token, int64_t* on_demand_per_layer);

/* generate_trace (inc/workload.hpp:60-112): host mt19937_64 stream (bit-identical draws), gate
 * logits on the GPU via K1 (fp64, reference summation order).  Outputs: gates [L][d][N], acts
 * [T][L][d], scores [T][L][N], selected [T][L][K], fisher [L]. Also loads the gates into the engine. */
int moe_generate_trace(moe_engine_t engine, const moe_synth_config* cfg, double* gates, double* acts,
                       double* scores, int32_t* selected, double* fisher);

/* generate_profiles (inc/workload.hpp:133-181): alpha (single-expert ratio at tau) and beta
 * (reuse-predict top-1 accuracy) per layer; the T*L reuse GEMVs run batched on the GPU.  Uses the
 * engine's gates and first-layer gate. */
int moe_generate_profiles(moe_engine_t engine, const double* acts, const double* scores, int32_t tokens,
                          const double* fisher, double tau, double* alpha, double* beta);

/* first_layer_training_pairs + train_predictive_gate (inc/workload.hpp:186-197,
 * inc/prefetch.hpp:194-213; CLI `profile --train-gate`, moesim_main.cpp:196): full-batch KL gradient
 * descent of the first-layer predictive gate from (token t-1 last-layer activation, token t first-layer
 * log-scores) pairs.  Logits on the GPU (K1 exact fp64 path), softmax with the host libm exp, gradient
 * and update on the GPU in the reference's summation order: bit-exact with the reference.
 * acts [T][L][d], scores [T][L][N]; T >= 2.  first_gate_out [d][N] row-major (load it with
 * moe_load_gates). */
int moe_train_first_gate(moe_engine_t engine, const double* acts, const double* scores, int32_t tokens,
                         double learning_rate, int32_t steps, uint64_t seed, double* first_gate_out);

/* ---- physical offloaded decode (expert FFN + HBM expert cache + copy engine) -------------- */
/* Expert FFN shape: SwiGLU with ffn_dim F, bf16 weights, F % tiles == 0, tiles = the
 * SimConfig tile_count_per_expert.  Creates the pinned host expert store (all L*N experts,
 * tile-major) and fills it with the deterministic counter-based init (same values as the oracle's
 * orc_expert_init).  host_alias > 0 stores only that many distinct experts and maps
 * (l, e) -> (l*N + e) % host_alias (for hosts without L*N*expert_bytes of RAM); 0 = all distinct. */
int moe_experts_init(moe_engine_t engine, int32_t ffn_dim, int32_t tiles, uint64_t seed, int32_t host_alias);

/* Expert-parallel shard store (replaces the reference's per-expert compute placeholder
 * inc/simulator.hpp:446-462 on a shard): as moe_experts_init, but the pinned store holds only the
 * experts with expert_owner[l*N + e] == rank (the same [L][N] table later passed to
 * moe_decode_begin_ex), so a shard pins ~1/G of the L*N experts.  expert_owner == NULL: all experts.
 * Host pages are placed on the GPU's NUMA node (sysfs; ADAPMOE_NUMA=0 disables, =n+1 forces node n)
 * for every store. */
int moe_experts_init_shard(moe_engine_t engine, int32_t ffn_dim, int32_t tiles, uint64_t seed, int32_t host_alias,
                           const int32_t* expert_owner, int32_t rank);
int moe_experts_alloc_shard(moe_engine_t engine, int32_t ffn_dim, int32_t tiles, const int32_t* expert_owner,
                            int32_t rank);
/* Expert store format for the next moe_experts_init* / moe_experts_alloc* on this engine:
 * MOE_STORE_BF16 (default) keeps every tile as raw bf16; MOE_STORE_XB12 keeps each tile as an XB12
 * record (paper_2408_10284_b200/csrc/kernels/xb12.hpp): sign + mantissa bytes, 4-bit exponent
 * codes against a per-tile 15-exponent window and an escape list, 75 % of the bytes for Mixtral-shape
 * weights.  Lossless: tiles land in an HBM staging buffer and a decode kernel restores the exact bf16
 * bits in the slot before anything reads them, so every output and trace is bit-identical to the
 * bf16 store; the host link moves 25 % fewer bytes.  A tile that would not shrink (> n/64 escapes)
 * stays raw.  MOE_STORE_XBH keeps each tile as an XBH record (kernels/xbh.hpp): the same sign +
 * mantissa bytes, the exponents Huffman-coded per tile (canonical, length-limited to 12 bits,
 * 512-value independently decodable segments), ~66 % of the bytes — same lossless contract, same
 * raw fallback.  moe_expert_read decodes; moe_expert_host_ptr needs a bf16 store. */
#define MOE_STORE_BF16 0
#define MOE_STORE_XB12 1
#define MOE_STORE_XBH 2
int moe_experts_set_format(moe_engine_t engine, int32_t format);
/* Format of the current store and the bytes a copy of all its records moves over the host link. */
int moe_experts_format(moe_engine_t engine, int32_t* format, int64_t* link_bytes);
/* One tile's record in the pinned store: host address, bytes, format (0 raw bf16, 1 XB12, 2 XBH), and
 * for XB12 the window base exponent, escape count and section offsets (lo at 0, nibbles, escapes);
 * for XBH the window base, escape count, the segment table's offset (nib_offset; the decode table
 * and the code bits sit at the offsets xbh.hpp derives from the tile's value count) and the escapes'. */
int moe_expert_tile_record(moe_engine_t engine, int32_t layer, int32_t expert, int32_t tile, const void** record,
                           int64_t* bytes, int32_t* format, uint32_t* base, int64_t* n_escapes, int64_t* nib_offset,
                           int64_t* esc_offset);

/* Pinned bytes, distinct stored expert blocks and the host NUMA node (-1: none) of the store. */
int moe_experts_info(moe_engine_t engine, int64_t* pinned_bytes, int32_t* stored_experts, int32_t* numa_node);

/* Real weights instead of the synthetic init (SURVEY §8(b) moe_load_experts): allocate the pinned
 * store (all L*N experts, zero), then hand every expert's weights over in the usual checkpoint
 * layout — bf16 bit patterns, row-major: w1 = gate_proj.weight [ffn][d], w3 = up_proj.weight
 * [ffn][d], w2 = down_proj.weight [d][ffn] — which moe_expert_set packs into the tile-major store
 * (W1/W3 row pairs, W2 transposed; host threads).  Errors: MOE_E_USAGE for an out-of-range expert
 * or while a decode session is active (its HBM slots hold copies of the store). */
int moe_experts_alloc(moe_engine_t engine, int32_t ffn_dim, int32_t tiles);
int moe_expert_set(moe_engine_t engine, int32_t layer, int32_t expert, const uint16_t* w1, const uint16_t* w3,
                   const uint16_t* w2);

/* Bytes of one expert (3 * F * d * 2) in the store. */
int moe_expert_bytes(moe_engine_t engine, int64_t* bytes);

/* Stream-level primitives (SURVEY §8(b) moe_copy_tile / moe_expert_ffn) for callers that manage their
 * own HBM expert buffers.  moe_copy_tiles: tiles [tile0, tile0 + n_tiles) of expert (layer, expert)
 * from the pinned host store into device memory laid out like the store (dst + t * tile_bytes holds
 * tile t), one cudaMemcpyAsync per tile on `stream` (a cudaStream_t; NULL = the engine's copy
 * stream); tile_events (NULL, or n_tiles cudaEvent_t) are recorded after each tile lands — the
 * physical form of the reference CommEngine's per-tile transfer (inc/simulator.hpp:187-320). */
int moe_copy_tiles(moe_engine_t engine, int32_t layer, int32_t expert, int32_t tile0, int32_t n_tiles, void* dst,
                   void* stream, void* const* tile_events);

/* moe_expert_ffn_async: y[b] = (accumulate ? y[b] : 0) + weight[b] * SwiGLU_E(x[b]) for b < rows,
 * on device buffers, stream-ordered on `stream` (NULL = the engine's compute stream): expert = a
 * device copy of one expert block (tile-major, e.g. from moe_copy_tiles), x [rows][d] fp64,
 * y [rows][d] fp32, weights [rows] host doubles (NULL = 1).  tile_events (NULL or `tiles` events):
 * the stream waits for each before computing (tile-granular overlap with moe_copy_tiles).  K2 + the
 * combine kernel per row (batch-1 streaming; the batched grouped tcgen05 path runs inside
 * moe_decode_tokens / moe_decode_layer).  Uses an engine-owned partial buffer: calls on one engine
 * must be ordered on one stream. */
int moe_expert_ffn_async(moe_engine_t engine, const void* expert, const double* x, float* y, int32_t rows,
                         const double* weights, int32_t accumulate, void* const* tile_events, void* stream);

/* Copy one expert's tile-major bf16 weights out of the pinned store (for parity tests). */
int moe_expert_read(moe_engine_t engine, int32_t layer, int32_t expert, uint16_t* out);

/* Read-only address of one expert's tile-major block inside the pinned store (host memory, valid
 * until the store is replaced or the engine destroyed): zero-copy access for host-side consumers,
 * e.g. a CPU expert path next to the GPU one.  MOE_E_USAGE when this (shard's) store does not
 * hold the expert. */
int moe_expert_host_ptr(moe_engine_t engine, int32_t layer, int32_t expert, const void** ptr);

/* Begin a decode session: per-layer HBM slot pool sized by `capacities` (the DP allocation) plus
 * `staging_slots` transfer slots, LRU initial fill from SeededRng(seed) (inc/simulator.hpp:352-360),
 * fisher [L], tau, config.  total_tokens is the trace length (the last-layer first-gate
 * prediction needs tok + 1 < T, inc/simulator.hpp:431). staging_slots <= 0 sizes the staging pool
 * automatically with a logical dry run of the session inputs when those are given to
 * moe_decode_tokens for the first time. */
int moe_decode_begin(moe_engine_t engine, const int32_t* capacities, int32_t staging_slots, const double* fisher,
                     double tau, const moe_sim_config* cfg, uint64_t seed, int32_t total_tokens);

/* Extended session options (moe_decode_begin_ex).  No reference counterpart: the reference is
 * batch-1 and single-process.
 *  batch  : token streams sharing the expert cache (BASELINE config 4).  Per (token, layer) every
 *           stream is routed with the reference rule; the cache/transfer engine sees the union of
 *           the streams' selections and look-ahead lists (builder-defined, oracle/moe_oracle.c
 *           orc_simulate_batch; batch == 1 is exactly moe_decode_begin).  batch > 1 runs the
 *           expert FFN as grouped tcgen05 GEMMs over each expert's routed tokens (bf16 activations,
 *           fp32 accumulation) and needs hidden_dim % 128 == 0 and (ffn / tiles) % 64 == 0.
 *           batch in [1, 256], batch * top_k <= 512.  moe_decode_tokens then takes acts
 *           [count][batch][L][d], scores [count][batch][L][N] and writes hidden_out [count][batch][L][d].
 *  ep_rank, ep_world : expert parallelism (BASELINE config 5).  Shard ep_rank owns the
 *           experts e with e % ep_world == ep_rank of every layer; the logical cache/transfer engine
 *           is replicated (identical trace on every shard); the shard holds, copies and computes only
 *           its own experts and hidden_out receives its partial layer output (shard 0 adds the
 *           residual x).  The layer output is the sum of the shards' partials in shard order
 *           (paper_2408_10284_b200/ep.py does it with torch.distributed).  0 <= ep_rank < ep_world <= N.
 *  free_running : SURVEY §7.2's second mode (no reference counterpart: the reference replays stored
 *           scores, inc/simulator.hpp:392).  Layer l > 0 routes and computes on layer l-1's output,
 *           so the hidden state flows through the offloaded experts; layer 0 takes the caller's
 *           activation; the actual decision uses the layer's gate on that hidden state (softmax of
 *           logits / dirichlet_concentration, like the reference generator, inc/workload.hpp:93-98)
 *           and the stored scores are ignored.  Given the hidden states the GPU produced, every
 *           decision and the cache trace equal the reference rule's. */
typedef struct {
    int32_t batch;
    int32_t ep_rank;
    int32_t ep_world;
    int32_t free_running;            /* see below; 0 = trace replay (the reference's semantics) */
    double dirichlet_concentration;  /* free-running: logits / concentration before softmax (SynthConfig) */
    const int32_t* expert_owner;     /* EP: [L][N] shard of each (layer, expert), the same table on every
                                        shard; NULL = e % ep_world.  Physical placement only: the event
                                        trace does not depend on it (ep.balanced_owners balances it by a
                                        calibration run's transfers) */
} moe_decode_opts;

int moe_decode_begin_ex(moe_engine_t engine, const int32_t* capacities, int32_t staging_slots, const double* fisher,
                        double tau, const moe_sim_config* cfg, uint64_t seed, int32_t total_tokens,
                        const moe_decode_opts* opts);

/* Expert-parallel exchange over peer memory (NVLink P2P; see kernels/ep_exchange.hpp), replacing a
 * host-side all_gather of the shards' partial outputs.  After moe_decode_begin_ex with ep_world > 1:
 * each shard exports its exchange region (device pointer for peers in the same process, 64-byte
 * CUDA IPC handle for other processes), the shards swap them, and each connects.  From then on the
 * combine kernels store each layer's partial output straight into every shard's region and
 * moe_decode_tokens returns the full layer outputs (shard partials summed in shard order, identical
 * on every shard).  All shards must decode the same calls (same counts, same order), concurrently. */
int moe_decode_ep_export(moe_engine_t engine, int32_t max_tokens_per_call, uint64_t* region_ptr, uint8_t* ipc_handle);
int moe_decode_ep_connect(moe_engine_t engine, const uint64_t* peer_ptrs, const uint8_t* peer_ipc_handles);

/* Decode `count` tokens (trace-replay: layer l's router/FFN input is the trace activation).
 * acts [count][L][d] fp64 and scores [count][L][N] fp64 are HOST buffers if inputs_on_device == 0,
 * else device pointers.  hidden_out [count][L][d] fp32 receives x_l + sum_e w_e * E_e(x_l) per
 * layer (host buffer, or device if inputs_on_device; NULL skips the readback).  gpu_ms receives
 * the CUDA-event time of the call on the compute stream. */
int moe_decode_tokens(moe_engine_t engine, const double* acts, const double* scores, int32_t count,
                      int32_t inputs_on_device, float* hidden_out, double* gpu_ms);

/* One MoE layer of the current token on caller DEVICE buffers, stream-ordered with the caller's
 * stream (the per-layer, stream-level entry an inference engine calls between its own
 * attention layers; the reference's per-layer body is inc/simulator.hpp:380-462).  The session's
 * logical engine steps (token, layer) exactly as moe_decode_tokens does, so the event trace is the
 * same; layers must be called in order 0..L-1 per token (MOE_E_USAGE otherwise), and a token must
 * not be split between moe_decode_layer and moe_decode_tokens.
 *  x      : device fp64 [B][d], this layer's router and expert input (B = the session's batch);
 *  scores : device fp64 [B][N] stored post-softmax scores to decide from (the reference's
 *           actual-selection rule, inc/simulator.hpp:390-396), or NULL to decide from the layer's
 *           gate on x (softmax of logits / dirichlet_concentration, as free-running does);
 *  out    : device fp32 [B][d] = (add_input ? x : 0) + sum_e w_e * E_e(x);
 *  stream : a cudaStream_t (NULL = the engine's compute stream).  The layer's work waits for
 *           everything enqueued on `stream` before the call, and `stream` waits for the layer's
 *           output.  The call returns once the layer is enqueued; the host blocks only on the
 *           layer's router result (the policy step needs the decision).
 * Needs a session without free_running / expert parallelism. */
int moe_decode_layer(moe_engine_t engine, int32_t layer, const double* x, const double* scores, float* out,
                     int32_t add_input, void* stream);

/* Physical timeline of the session (SURVEY §5 tracing): enable = 1 starts recording CUDA-event
 * timestamps of every expert tile copy (request class on_demand / prefetch, promotion, the expert
 * its insert evicted), every FFN launch (one record per (expert, tile) segment with the copy job
 * that filled its slot), compute-stream waits on tile copies and router launches, relative to an
 * origin event recorded now; 0 stops.  moe_decode_timeline_write drains the copy engine,
 * synchronises, and writes everything recorded so far as JSONL sorted by start time, in the
 * reference's schema (inc/io.hpp:402-417: stream, kind, start, end, expert, token, layer, tile;
 * times in microseconds) plus physical fields (request, promoted, evicts, job for transfers;
 * launch, fill for computes).  n_events (may be NULL) receives the line count. */
int moe_decode_record_timeline(moe_engine_t engine, int32_t enable);
int moe_decode_timeline_write(moe_engine_t engine, const char* path, int64_t* n_events);

/* Physical counters of the session so far (CUDA-event timed on the engine's streams). */
typedef struct {
    int64_t tokens;
    int64_t kernels_launched;     /* our kernels: router, FFN passes, combine, coded-tile decode + patch */
    int64_t ffn_launches;         /* FFN pass launches (gate/up + down) */
    int64_t tile_copies;          /* expert tile copies issued host -> HBM */
    int64_t copy_bytes;           /* expert bytes moved host -> HBM */
    int64_t input_bytes;          /* activation/score bytes copied host -> HBM (host-input calls) */
    int64_t ffn_bytes;            /* algorithmic expert bytes streamed by the FFN passes */
    double copy_busy_ms;          /* sum of tile-copy durations */
    double ffn_ms;                /* sum of FFN pass durations */
    double ffn_gate_up_ms, ffn_down_ms;
    double ffn_gate_up_bytes, ffn_down_bytes;
    double router_ms;             /* sum of router (K1) durations */
    double stall_ms;              /* compute-stream time blocked on tile copies */
    int64_t router_exact_items;   /* look-ahead items K1 could not certify from fp32 logits (exact fp64 path) */
    double host_sync_ms;          /* host wall time blocked on K1 results */
    double host_step_ms;          /* host wall time in the policy step + launches (incl. copy-issue waits) */
    int32_t slots_total;          /* HBM slots = sum(capacities) + staging */
    int32_t staging_high_water;   /* most staging slots in use at once */
    double prefetch_copy_ms;      /* tile-copy time of prefetches the logical engine never promoted */
    double prefetch_stall_ms;     /* compute-stream time blocked on those prefetch tiles */
    int64_t prefetch_tile_copies; /* tiles copied for them */
    double prefetch_used_copy_ms; /* ... of which the compute stream consumed; hidden = 1 - stall / used copy */
    int64_t router_launches;      /* K1 launches: one per layer (free-running), one per token window (trace replay) */
    int64_t spec_launches;        /* free-running batch 1: speculative next-layer FFN launches (pre-gate top-1) */
    int64_t spec_hits;            /* ... whose expert the layer's decision selected (partials reused) */
    double record_decode_ms;      /* coded stores (XB12 / XBH): summed duration of the tile decode kernels */
    int64_t record_decodes;       /* ... launches (one per coded tile copied) */
    double record_decode_bytes;   /* ... bytes: records read + bf16 tiles written */
} moe_decode_stats;

/* Counters so far without ending the session. */
int moe_decode_stats_snapshot(moe_engine_t engine, moe_decode_stats* stats);

/* End the session: logical metrics/timeline (bit-exact with simulate_trace on the same inputs),
 * physical stats.  Any pointer may be NULL. */
int moe_decode_end(moe_engine_t engine, moe_metrics* metrics, int64_t* latency_per_token,
                   int64_t* on_demand_per_layer, moe_event* events, int64_t events_capacity, int64_t* n_events,
                   moe_decode_stats* stats);

/* Single-expert SwiGLU (parity/profiling entry): y[d] fp32 = W2 (silu(W1 x) * (W3 x)) for expert
 * (layer, expert) of the store, x [d] fp64 host buffer, y [d] fp32 host buffer.  Runs the same
 * K2 passes and tile-order reduction as the decode path. */
int moe_expert_ffn(moe_engine_t engine, int32_t layer, int32_t expert, const double* x, float* y);

#ifdef __cplusplus
}
#endif
#endif /* ADAPMOE_H */
