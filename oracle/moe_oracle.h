/* TEST INFRASTRUCTURE ONLY — the CPU oracle (checker), never the product.
 *
 * A plain-C restatement of the reference algorithm (moesim, /root/reference/proj/include/moesim,
 * abbreviated `inc/` below) for the AdapMoE offloaded-MoE decode path, plus a builder-defined
 * SwiGLU expert FFN (the reference has no FFN arithmetic: inc/simulator.hpp:446-462 is a tick
 * placeholder), used to check the CUDA path.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / reference arm may load this library.
 *
 * Parity status: pinned.  tests/test_oracle_vs_ref.py checks every function here bit-exactly
 * against the unmodified reference compiled by oracle/Makefile (oracle/_ref/moesim_ref) and against
 * the committed golden fixtures under tests/golden/ (produced by that binary, see
 * tests/golden/make_goldens.py), and restates the reference unit tests' known answers
 * (proj/tests/test_*.cpp).  The expert-FFN restatement has no reference counterpart ("parity
 * unpinned" for FFN values; its contract is the north-star tolerance 1e-4 rel fp32 / 2e-2 bf16).
 *
 * Compile with -O2 -ffp-contract=off and no -march (reference build flags: proj/CMakeLists.txt:1-21).
 */
#ifndef MOE_ORACLE_H
#define MOE_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* --- inc/core.hpp:118-188  SeededRng (mt19937_64 + hand-rolled distributions) --------------- */
typedef struct {
    uint64_t mt[312];
    int mti;
    uint64_t seed;
    double spare;
    int have_spare;
} orc_rng;

void orc_rng_init(orc_rng* r, uint64_t seed);
uint64_t orc_rng_u64(orc_rng* r);
double orc_rng_uniform01(orc_rng* r);
double orc_rng_normal(orc_rng* r);
int orc_rng_uniform_int(orc_rng* r, int n);
void orc_rng_sample_subset(orc_rng* r, int n, int t, int* out);
uint64_t orc_splitmix(uint64_t x);

/* --- inc/core.hpp:192-216, inc/gating.hpp:28-65, inc/prefetch.hpp:24-35 ---------------------- */
int orc_top_k(const double* scores, int n, int k, int* out);
int orc_softmax(const double* logits, int n, double* out);
double orc_top1_share(const double* scores, int n);
/* returns 1 if single; selected gets 1 or top_k entries; *count and *perturbation set */
int orc_gate_decide(const double* scores, int n, int top_k, double fisher, double tau, int* selected, int* count,
                    double* perturbation);
void orc_gate_logits(const double* W /*[d][n]*/, int d, int n, const double* x /*[d]*/, double* out /*[n]*/);

/* --- inc/workload.hpp:60-112  generate_trace ------------------------------------------------- */
int orc_generate_trace(int L, int N, int K, int D, int T, double concentration, double drift, uint64_t gate_seed,
                       uint64_t token_seed, int shared_gates, const double* fisher_scales /*[L] or NULL*/,
                       const double* drift_scales /*[L] or NULL*/, double* gates /*[L][D][N]*/,
                       double* acts /*[T][L][D]*/, double* scores /*[T][L][N]*/, int* selected /*[T][L][K]*/,
                       double* fisher_out /*[L]*/);

/* --- inc/gating.hpp:85-122  calibrate_threshold -------------------------------------------- */
double orc_calibrate_threshold(const double* scores, int T, int L, int N, const double* fisher, double target);

/* --- inc/workload.hpp:186-197 + inc/prefetch.hpp:158-213  first-layer predictive gate ------ */
int orc_train_first_gate(const double* acts, const double* scores, int T, int L, int D, int N, double lr, int steps,
                         uint64_t seed, double* W_out /*[D][N]*/);

/* --- inc/workload.hpp:133-181  generate_profiles (alpha, beta) ------------------------------ */
int orc_generate_profiles(const double* acts, const double* scores, const double* gates, const double* first_gate,
                          int T, int L, int N, int K, int D, double tau, const double* fisher, double* alpha,
                          double* beta);

/* --- inc/cache_model.hpp:28-74,189-204 + inc/allocator.hpp:36-88,140-153 ------------------- */
int orc_cost_table(const double* alpha, const double* beta, int L, int N, double* table /*[L][N+1]*/);
int orc_dp_allocate(const double* table, int L, int N, int budget, int* caps, double* total_cost);
int orc_uniform_allocation(int budget, int L, int N, int* caps);
double orc_expected_cost(int t, int n, double alpha, double beta);

/* --- inc/simulator.hpp:55-60, 64-468  tick-model simulator --------------------------------- */
typedef struct {
    int tiles;
    int64_t tile_transfer, tile_compute, attention, gate;
    int lookahead;
    int gating, prefetch;
} orc_simcfg;

typedef struct {
    int64_t total_latency, stall_time, on_demand_loads, cache_hits, prefetch_hits, single_expert_decisions,
        experts_activated_total;
} orc_metrics;

int64_t orc_tile_pipeline_latency(int tiles, int64_t transfer, int64_t compute);

/* timeline rows are 8 int64: stream, kind, start, end, token, layer, expert, tile.
 * predictions (optional, may be NULL): [T][L][3][2+K] = target, count, experts (pad -1).
 * decisions (optional): [T][L][K] selected (pad -1). Returns 0 or a negative error code;
 * -100 means the timeline capacity was too small (*n_events holds the needed count). */
int orc_simulate(const double* acts, const double* scores, const double* gates, const double* first_gate, int T,
                 int L, int N, int K, int D, const double* fisher, const int* caps, double tau, orc_simcfg cfg,
                 uint64_t seed, orc_metrics* metrics, int64_t* latency_per_token, int64_t* od_per_layer,
                 int64_t* timeline, int64_t timeline_cap, int64_t* n_events, int* predictions, int* decisions);

/* Batched decode over B streams sharing one cache (builder-defined; B = 1 == orc_simulate).
 * acts [B][T][L][D], scores [B][T][L][N]; predictions [B][T][L][3][2+K]; decisions [B][T][L][K]. */
int orc_simulate_batch(const double* acts, const double* scores, const double* gates, const double* first_gate,
                       int B, int T, int L, int N, int K, int D, const double* fisher, const int* caps, double tau,
                       orc_simcfg cfg, uint64_t seed, orc_metrics* metrics, int64_t* latency_per_token,
                       int64_t* od_per_layer, int64_t* timeline, int64_t timeline_cap, int64_t* n_events,
                       int* predictions, int* decisions);

/* --- builder-defined expert FFN (no reference counterpart; parity unpinned) --------------- */
/* Deterministic counter-based bf16 init, identical to the CUDA init kernel. Layout is tile-major:
 * for tile t (ffn rows [t*F/T,(t+1)*F/T)): gate_up [F/T][2][D] (W1 row, W3 row interleaved),
 * then down_t [F/T][D] (row r = W2[:, t*F/T + r]).  Element key = (matrix m in {0:W1,1:W3,2:W2},
 * logical row-major index in W1/W3 [F][D] or W2 [D][F]). */
float orc_init_scale(int fan_in);
uint16_t orc_init_value(uint64_t base, uint64_t index, float scale);
uint64_t orc_expert_base(uint64_t seed, int layer, int expert, int matrix);
int orc_expert_init(uint64_t seed, int layer, int expert, int D, int F, int tiles, uint16_t* out);
/* y[D] = W2 (silu(W1 x) * (W3 x)), fp64 accumulation over bf16 weights, x fp32. */
int orc_swiglu(const uint16_t* w, int D, int F, int tiles, const float* x, double* y);

/* FNV-1a (inc/io.hpp:80-87) over raw bytes, for fixture hashes; start with 0xcbf29ce484222325 */
#include <stddef.h>
uint64_t orc_fnv1a(const void* data, size_t n, uint64_t h);

#ifdef __cplusplus
}
#endif
#endif
