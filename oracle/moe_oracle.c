/* TEST INFRASTRUCTURE ONLY — CPU oracle (checker) for the AdapMoE decode path.
 * See moe_oracle.h for scope and parity status. Every function cites the reference
 * lines (/root/reference/proj/include/moesim = `inc/`) it restates. */
#include "moe_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------------ */
/* inc/core.hpp:118-188  SeededRng: std::mt19937_64 + uniform01 (53-bit) + Box-Muller normal  */
/* with cached spare + rejection uniform_int + partial Fisher-Yates sample_subset.             */
/* ------------------------------------------------------------------------------------------ */
#define MT_NN 312
#define MT_MM 156
#define MT_A 0xB5026F5AA96619E9ULL
#define MT_UM 0xFFFFFFFF80000000ULL
#define MT_LM 0x7FFFFFFFULL

void orc_rng_init(orc_rng* r, uint64_t seed) {
    r->seed = seed;
    r->mt[0] = seed;
    for (int i = 1; i < MT_NN; ++i) r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->mti = MT_NN;
    r->spare = 0.0;
    r->have_spare = 0;
}

uint64_t orc_rng_u64(orc_rng* r) {
    if (r->mti >= MT_NN) {
        int i;
        uint64_t x;
        for (i = 0; i < MT_NN - MT_MM; ++i) {
            x = (r->mt[i] & MT_UM) | (r->mt[i + 1] & MT_LM);
            r->mt[i] = r->mt[i + MT_MM] ^ (x >> 1) ^ ((x & 1ULL) ? MT_A : 0ULL);
        }
        for (; i < MT_NN - 1; ++i) {
            x = (r->mt[i] & MT_UM) | (r->mt[i + 1] & MT_LM);
            r->mt[i] = r->mt[i + (MT_MM - MT_NN)] ^ (x >> 1) ^ ((x & 1ULL) ? MT_A : 0ULL);
        }
        x = (r->mt[MT_NN - 1] & MT_UM) | (r->mt[0] & MT_LM);
        r->mt[MT_NN - 1] = r->mt[MT_MM - 1] ^ (x >> 1) ^ ((x & 1ULL) ? MT_A : 0ULL);
        r->mti = 0;
    }
    uint64_t y = r->mt[r->mti++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= (y >> 43);
    return y;
}

double orc_rng_uniform01(orc_rng* r) { return (double)(orc_rng_u64(r) >> 11) * 0x1.0p-53; }

double orc_rng_normal(orc_rng* r) {
    if (r->have_spare) {
        r->have_spare = 0;
        return r->spare;
    }
    const double two_pi = 6.283185307179586476925286766559;
    double u1 = orc_rng_uniform01(r);
    double u2 = orc_rng_uniform01(r);
    while (u1 <= 0.0) u1 = orc_rng_uniform01(r);
    double rr = sqrt(-2.0 * log(u1));
    double theta = two_pi * u2;
    r->spare = rr * sin(theta);
    r->have_spare = 1;
    return rr * cos(theta);
}

int orc_rng_uniform_int(orc_rng* r, int n) {
    if (n <= 0) return -1;
    const uint64_t un = (uint64_t)n;
    const uint64_t limit = (~(uint64_t)0 / un) * un;
    uint64_t x = orc_rng_u64(r);
    while (x >= limit) x = orc_rng_u64(r);
    return (int)(x % un);
}

void orc_rng_sample_subset(orc_rng* r, int n, int t, int* out) {
    int* pool = (int*)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
    for (int i = 0; i < n; ++i) pool[i] = i;
    for (int i = 0; i < t; ++i) {
        int j = i + orc_rng_uniform_int(r, n - i);
        int tmp = pool[i];
        pool[i] = pool[j];
        pool[j] = tmp;
    }
    for (int i = 0; i < t; ++i) out[i] = pool[i];
    free(pool);
}

uint64_t orc_splitmix(uint64_t x) { /* inc/core.hpp:176-181 */
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

/* ------------------------------------------------------------------------------------------ */
/* inc/core.hpp:192-203 top_k_indices: order by score desc, ties -> lowest index.             */
/* Selection by repeated argmax under that total order gives the identical prefix.           */
/* ------------------------------------------------------------------------------------------ */
int orc_top_k(const double* s, int n, int k, int* out) {
    if (k < 0 || k > n) return -1;
    unsigned long long used = 0;  /* n <= 64 */
    for (int r = 0; r < k; ++r) {
        int best = -1;
        for (int j = 0; j < n; ++j) {
            if (used >> j & 1ULL) continue;
            if (best < 0 || s[j] > s[best]) best = j; /* strict > keeps the lowest index on ties */
        }
        used |= 1ULL << best;
        out[r] = best;
    }
    return 0;
}

/* inc/core.hpp:205-216 softmax: first max, exp(l - mx), sequential sum, divide. */
int orc_softmax(const double* l, int n, double* out) {
    if (n <= 0) return -1;
    double mx = l[0];
    for (int i = 1; i < n; ++i)
        if (l[i] > mx) mx = l[i];
    double sum = 0.0;
    for (int i = 0; i < n; ++i) {
        out[i] = exp(l[i] - mx);
        sum += out[i];
    }
    for (int i = 0; i < n; ++i) out[i] /= sum;
    return 0;
}

/* inc/gating.hpp:28-42 normalized_top1_share. */
double orc_top1_share(const double* scores, int n) {
    double s1 = -1.0, s2 = -1.0;
    for (int i = 0; i < n; ++i) {
        double s = scores[i];
        if (s > s1) {
            s2 = s1;
            s1 = s;
        } else if (s > s2) {
            s2 = s;
        }
    }
    double denom = s1 + s2;
    return s1 / denom;
}

/* inc/gating.hpp:46-65: perturbation = (1-alpha)^2 * F; single iff perturbation <= tau. */
int orc_gate_decide(const double* scores, int n, int top_k, double fisher, double tau, int* selected, int* count,
                    double* perturbation) {
    double alpha = orc_top1_share(scores, n);
    double gap = 1.0 - alpha;
    double p = gap * gap * fisher;
    int single = p <= tau;
    int k = single ? 1 : top_k;
    orc_top_k(scores, n, k, selected);
    if (count) *count = k;
    if (perturbation) *perturbation = p;
    return single;
}

/* inc/prefetch.hpp:24-35 GateMatrix::logits: i ascending, skip x == 0, separate mul + add. */
void orc_gate_logits(const double* W, int d, int n, const double* x, double* out) {
    for (int j = 0; j < n; ++j) out[j] = 0.0;
    for (int i = 0; i < d; ++i) {
        const double xi = x[i];
        if (xi == 0.0) continue;
        const double* row = W + (size_t)i * n;
        for (int j = 0; j < n; ++j) out[j] += xi * row[j];
    }
}

/* ------------------------------------------------------------------------------------------ */
/* inc/workload.hpp:60-112 generate_trace.                                                   */
/* ------------------------------------------------------------------------------------------ */
int orc_generate_trace(int L, int N, int K, int D, int T, double concentration, double drift, uint64_t gate_seed,
                       uint64_t token_seed, int shared_gates, const double* fisher_scales, const double* drift_scales,
                       double* gates, double* acts, double* scores, int* selected, double* fisher_out) {
    if (L < 1 || N < 2 || K < 1 || K > N || D < 1 || T < 1 || !(concentration > 0.0) || !(drift >= 0.0)) return -1;
    for (int l = 0; l < L; ++l) fisher_out[l] = fisher_scales ? fisher_scales[l] : 1.0;
    orc_rng grng;
    orc_rng_init(&grng, gate_seed);
    const double weight_scale = 1.0 / sqrt((double)D);
    const size_t gsz = (size_t)D * N;
    for (int l = 0; l < L; ++l) {
        double* g = gates + (size_t)l * gsz;
        if (shared_gates && l > 0) {
            memcpy(g, gates, gsz * sizeof(double));
            continue;
        }
        for (size_t i = 0; i < gsz; ++i) g[i] = weight_scale * orc_rng_normal(&grng);
    }
    orc_rng trng;
    orc_rng_init(&trng, token_seed);
    double* x = (double*)malloc(sizeof(double) * (size_t)D);
    double* logits = (double*)malloc(sizeof(double) * (size_t)N);
    for (int tok = 0; tok < T; ++tok) {
        for (int i = 0; i < D; ++i) x[i] = orc_rng_normal(&trng);
        for (int l = 0; l < L; ++l) {
            orc_gate_logits(gates + (size_t)l * gsz, D, N, x, logits);
            for (int j = 0; j < N; ++j) logits[j] /= concentration;
            size_t tl = (size_t)tok * L + l;
            memcpy(acts + tl * D, x, sizeof(double) * (size_t)D);
            orc_softmax(logits, N, scores + tl * N);
            orc_top_k(scores + tl * N, N, K, selected + tl * K);
            const double scale = drift_scales ? drift_scales[l] : 1.0;
            const double eps = drift * scale;
            if (eps > 0.0) {
                double norm_sq = 0.0;
                for (int i = 0; i < D; ++i) norm_sq += x[i] * x[i];
                const double step = eps * sqrt(norm_sq / (double)D);
                for (int i = 0; i < D; ++i) x[i] += step * orc_rng_normal(&trng);
            }
        }
    }
    free(x);
    free(logits);
    return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* inc/gating.hpp:85-122 calibrate_threshold: sort perturbations; tau = smallest observed     */
/* value whose right-continuous ratio reaches the target (0 if ratio(0) already does).       */
/* ------------------------------------------------------------------------------------------ */
static int cmp_double(const void* a, const void* b) {
    double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}

static size_t upper_bound_d(const double* v, size_t m, double key) {
    size_t lo = 0, hi = m;
    while (lo < hi) {
        size_t mid = lo + (hi - lo) / 2;
        if (key < v[mid])
            hi = mid;
        else
            lo = mid + 1;
    }
    return lo;
}

double orc_calibrate_threshold(const double* scores, int T, int L, int N, const double* fisher, double target) {
    size_t m = (size_t)T * L;
    double* p = (double*)malloc(sizeof(double) * m);
    for (int tok = 0; tok < T; ++tok)
        for (int l = 0; l < L; ++l) {
            double alpha = orc_top1_share(scores + ((size_t)tok * L + l) * N, N);
            double gap = 1.0 - alpha;
            p[(size_t)tok * L + l] = gap * gap * fisher[l];
        }
    qsort(p, m, sizeof(double), cmp_double);
    double result;
    if ((double)upper_bound_d(p, m, 0.0) / (double)m >= target) {
        result = 0.0;
    } else {
        size_t lo = 0, hi = m - 1;
        while (lo < hi) {
            size_t mid = lo + (hi - lo) / 2;
            if ((double)upper_bound_d(p, m, p[mid]) / (double)m >= target)
                hi = mid;
            else
                lo = mid + 1;
        }
        result = p[lo];
    }
    free(p);
    return result;
}

/* ------------------------------------------------------------------------------------------ */
/* inc/workload.hpp:186-197 + inc/prefetch.hpp:121-213 first-layer predictive gate:          */
/* pairs (prev token's last activation, log(max(score,1e-300)) of layer 0), full-batch GD on  */
/* mean KL with grad = x (q - p), init 0.1 * N(0,1) from SeededRng(seed).                     */
/* ------------------------------------------------------------------------------------------ */
int orc_train_first_gate(const double* acts, const double* scores, int T, int L, int D, int N, double lr, int steps,
                         uint64_t seed, double* W) {
    if (T < 2) return -1;
    const int P = T - 1;
    double* tl = (double*)malloc(sizeof(double) * (size_t)P * N);
    for (int tok = 1; tok < T; ++tok) {
        const double* s = scores + ((size_t)tok * L + 0) * N;
        for (int j = 0; j < N; ++j) tl[(size_t)(tok - 1) * N + j] = log(s[j] > 1e-300 ? s[j] : 1e-300);
    }
    orc_rng rng;
    orc_rng_init(&rng, seed);
    for (size_t i = 0; i < (size_t)D * N; ++i) W[i] = 0.1 * orc_rng_normal(&rng);
    double* grad = (double*)malloc(sizeof(double) * (size_t)D * N);
    double* lg = (double*)malloc(sizeof(double) * N);
    double* q = (double*)malloc(sizeof(double) * N);
    double* p = (double*)malloc(sizeof(double) * N);
    const double inv = 1.0 / (double)P;
    for (int step = 0; step < steps; ++step) {
        memset(grad, 0, sizeof(double) * (size_t)D * N);
        for (int k = 0; k < P; ++k) {
            const double* x = acts + ((size_t)k * L + (L - 1)) * D; /* token k's last activation */
            orc_gate_logits(W, D, N, x, lg);
            orc_softmax(lg, N, q);
            orc_softmax(tl + (size_t)k * N, N, p);
            for (int i = 0; i < D; ++i) {
                const double xi = x[i];
                if (xi == 0.0) continue;
                double* row = grad + (size_t)i * N;
                for (int j = 0; j < N; ++j) row[j] += xi * (q[j] - p[j]);
            }
        }
        for (size_t i = 0; i < (size_t)D * N; ++i) grad[i] *= inv;
        for (size_t i = 0; i < (size_t)D * N; ++i) W[i] -= lr * grad[i];
    }
    free(tl);
    free(grad);
    free(lg);
    free(q);
    free(p);
    return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* inc/workload.hpp:133-181 generate_profiles + inc/gating.hpp:124-135 profile_single_prob +  */
/* inc/prefetch.hpp:46-78 reuse_predict / measure_accuracy.                                  */
/* ------------------------------------------------------------------------------------------ */
static int reuse_top1(const double* x, const double* W, int D, int N) {
    double lg[64], sc[64];
    int top;
    orc_gate_logits(W, D, N, x, lg);
    orc_softmax(lg, N, sc);
    orc_top_k(sc, N, 1, &top);
    return top;
}

int orc_generate_profiles(const double* acts, const double* scores, const double* gates, const double* first_gate,
                          int T, int L, int N, int K, int D, double tau, const double* fisher, double* alpha,
                          double* beta) {
    if (T < 1 || N > 64) return -1;
    long long* singles = (long long*)calloc((size_t)L, sizeof(long long));
    long long* hits = (long long*)calloc((size_t)L, sizeof(long long));
    long long* counted = (long long*)calloc((size_t)L, sizeof(long long));
    int sel[64];
    int cnt;
    for (int tok = 0; tok < T; ++tok)
        for (int l = 0; l < L; ++l) {
            const double* s = scores + ((size_t)tok * L + l) * N;
            singles[l] += orc_gate_decide(s, N, K, fisher[l], tau, sel, &cnt, NULL);
            int pred = -1;
            if (l >= 1)
                pred = reuse_top1(acts + ((size_t)tok * L + (l - 1)) * D, gates + (size_t)l * D * N, D, N);
            else if (first_gate && tok >= 1)
                pred = reuse_top1(acts + ((size_t)(tok - 1) * L + (L - 1)) * D, first_gate, D, N);
            if (pred >= 0) {
                ++counted[l];
                for (int k = 0; k < cnt; ++k)
                    if (sel[k] == pred) {
                        ++hits[l];
                        break;
                    }
            }
        }
    for (int l = 0; l < L; ++l) {
        alpha[l] = (double)singles[l] / (double)T;
        beta[l] = counted[l] > 0 ? (double)hits[l] / (double)counted[l] : 0.0;
    }
    free(singles);
    free(hits);
    free(counted);
    return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* inc/cache_model.hpp:28-74 Eq. 10-15 and :189-204 cost table.                               */
/* ------------------------------------------------------------------------------------------ */
double orc_expected_cost(int t, int n, double alpha, double beta) {
    const double phit = (double)t / (double)n;
    const double single = (1.0 - phit) * (1.0 - beta);
    const double dn = (double)n, dt = (double)t;
    double both_miss = (dn - dt) * (dn - dt - 1.0) / (dn * (dn - 1.0));
    if (both_miss < 0.0) both_miss = 0.0;
    const double one_hit = 2.0 * (dn - dt) * dt / (dn * (dn - 1.0));
    const double c0 = 2.0 * both_miss * (1.0 - beta);
    const double c1 = both_miss * beta;
    const double c2 = one_hit * (1.0 - beta);
    const double two = c0 + c1 + c2; /* TwoExpertCost::total, left to right */
    return alpha * single + (1.0 - alpha) * two;
}

int orc_cost_table(const double* alpha, const double* beta, int L, int N, double* table) {
    for (int l = 0; l < L; ++l)
        for (int t = 0; t <= N; ++t) table[(size_t)l * (N + 1) + t] = orc_expected_cost(t, N, alpha[l], beta[l]);
    return 0;
}

/* inc/allocator.hpp:36-88: knapsack over (layer, slots); strict < keeps the smallest k; the
 * table width is min(budget, L*N); backtrace from the last layer. */
int orc_dp_allocate(const double* table, int L, int N, int budget, int* caps, double* total_cost) {
    if (budget < 0) return -1;
    long long eff_ll = (long long)L * N;
    const int eff = budget < eff_ll ? budget : (int)eff_ll;
    const int W = eff + 1;
    double* mc = (double*)calloc((size_t)(L + 1) * W, sizeof(double));
    int* ch = (int*)calloc((size_t)(L + 1) * W, sizeof(int));
    for (int i = 1; i <= L; ++i)
        for (int j = 0; j <= eff; ++j) {
            double best = INFINITY;
            int best_k = 0;
            const int kmax = j < N ? j : N;
            for (int k = 0; k <= kmax; ++k) {
                const double c = mc[(size_t)(i - 1) * W + (j - k)] + table[(size_t)(i - 1) * (N + 1) + k];
                if (c < best) {
                    best = c;
                    best_k = k;
                }
            }
            mc[(size_t)i * W + j] = best;
            ch[(size_t)i * W + j] = best_k;
        }
    int j = eff;
    for (int i = L; i >= 1; --i) {
        const int k = ch[(size_t)i * W + j];
        caps[i - 1] = k;
        j -= k;
    }
    if (total_cost) *total_cost = mc[(size_t)L * W + eff];
    free(mc);
    free(ch);
    return 0;
}

/* inc/allocator.hpp:140-153 uniform_allocation. */
int orc_uniform_allocation(int budget, int L, int N, int* caps) {
    if (budget < 0) return -1;
    const int base = budget / L, extra = budget % L;
    for (int i = 0; i < L; ++i) {
        const int want = base + (i < extra ? 1 : 0);
        caps[i] = want < N ? want : N;
    }
    return 0;
}

/* inc/simulator.hpp:55-60 */
int64_t orc_tile_pipeline_latency(int tiles, int64_t transfer, int64_t compute) {
    if (transfer >= compute) return (int64_t)tiles * transfer + compute;
    return transfer + (int64_t)tiles * compute;
}

/* ------------------------------------------------------------------------------------------ */
/* inc/simulator.hpp:64-107 LruCache (front = MRU, fresh marks, capacity 0 rejects).          */
/* ------------------------------------------------------------------------------------------ */
typedef struct {
    int cap, size;
    int order[64]; /* order[0] = MRU */
    unsigned char fresh[64];
    unsigned char res[64];
} lru_t;

static int lru_pos(const lru_t* c, int e) {
    for (int i = 0; i < c->size; ++i)
        if (c->order[i] == e) return i;
    return -1;
}
static void lru_to_front(lru_t* c, int pos) {
    int e = c->order[pos];
    for (int i = pos; i > 0; --i) c->order[i] = c->order[i - 1];
    c->order[0] = e;
}
static void lru_touch(lru_t* c, int e) {
    lru_to_front(c, lru_pos(c, e));
    c->fresh[e] = 0;
}
static void lru_insert(lru_t* c, int e, int fresh) {
    if (c->cap == 0) return;
    int pos = lru_pos(c, e);
    if (pos >= 0) {
        lru_to_front(c, pos);
        if (!fresh) c->fresh[e] = 0;
        return;
    }
    if (c->size == c->cap) {
        int v = c->order[c->size - 1];
        c->res[v] = 0;
        c->fresh[v] = 0;
        c->size--;
    }
    for (int i = c->size; i > 0; --i) c->order[i] = c->order[i - 1];
    c->order[0] = e;
    c->size++;
    c->res[e] = 1;
    if (fresh) c->fresh[e] = 1;
}

/* ------------------------------------------------------------------------------------------ */
/* inc/simulator.hpp:187-320 CommEngine: serialized tile channel, od FIFO beats pf FIFO when  */
/* ready, promotion moves a queued prefetch to the od back, in-flight tile never pre-empted, */
/* prefetched experts enter the cache (fresh) on arrival.                                     */
/* ------------------------------------------------------------------------------------------ */
typedef struct {
    int layer, expert, tiles_done, on_demand, token, active;
    int64_t ready;
    int64_t* arrivals;
} req_t;

typedef struct {
    int tiles, L, N;
    int64_t tile_time, cursor;
    req_t* reqs;
    int nreq, capreq;
    int *od, *pf;
    int nod, npf, capq;
    int* pending;       /* [L*N] -> req index or -1 */
    int64_t* fin;       /* [L*N][tiles] */
    int* fin_n;         /* [L*N] */
    int inflight;       /* req index or -1 */
    int64_t inflight_end;
    lru_t* caches;
    int64_t* tl;
    int64_t tl_cap, tl_n;
} comm_t;

static void tl_push(comm_t* c, int64_t s, int64_t k, int64_t a, int64_t b, int64_t tok, int64_t l, int64_t e,
                    int64_t t) {
    if (c->tl && c->tl_n < c->tl_cap) {
        int64_t* r = c->tl + c->tl_n * 8;
        r[0] = s; r[1] = k; r[2] = a; r[3] = b; r[4] = tok; r[5] = l; r[6] = e; r[7] = t;
    }
    c->tl_n++;
}

static void q_erase(int* q, int* n, int v) {
    for (int i = 0; i < *n; ++i)
        if (q[i] == v) {
            memmove(q + i, q + i + 1, sizeof(int) * (size_t)(*n - i - 1));
            (*n)--;
            return;
        }
}

static int comm_new_req(comm_t* c) {
    for (int i = 0; i < c->nreq; ++i)
        if (!c->reqs[i].active) return i;
    if (c->nreq == c->capreq) {
        c->capreq *= 2;
        c->reqs = (req_t*)realloc(c->reqs, sizeof(req_t) * (size_t)c->capreq);
    }
    c->reqs[c->nreq].arrivals = (int64_t*)malloc(sizeof(int64_t) * (size_t)c->tiles);
    return c->nreq++;
}

static void comm_enqueue(comm_t* c, int layer, int expert, int on_demand, int64_t ready, int token) {
    int r = comm_new_req(c);
    req_t* q = &c->reqs[r];
    q->layer = layer; q->expert = expert; q->tiles_done = 0; q->on_demand = on_demand;
    q->token = token; q->active = 1; q->ready = ready;
    c->pending[layer * c->N + expert] = r;
    if (on_demand) c->od[c->nod++] = r; else c->pf[c->npf++] = r;
}

static void comm_promote(comm_t* c, int layer, int expert) {
    int r = c->pending[layer * c->N + expert];
    if (c->reqs[r].on_demand) return;
    c->reqs[r].on_demand = 1;
    q_erase(c->pf, &c->npf, r);
    c->od[c->nod++] = r;
}

static int comm_next_pick(const comm_t* c, int64_t* start) {
    int64_t best = INT64_MAX;
    if (c->nod) best = c->reqs[c->od[0]].ready < best ? c->reqs[c->od[0]].ready : best;
    if (c->npf) best = c->reqs[c->pf[0]].ready < best ? c->reqs[c->pf[0]].ready : best;
    if (best == INT64_MAX) return -1;
    *start = c->cursor > best ? c->cursor : best;
    if (c->nod && c->reqs[c->od[0]].ready <= *start) return c->od[0];
    return c->pf[0];
}

static void comm_start_tile(comm_t* c, int r, int64_t start) {
    req_t* q = &c->reqs[r];
    const int64_t end = start + c->tile_time;
    tl_push(c, 1, 4, start, end, q->token, q->layer, q->expert, q->tiles_done);
    c->inflight = r;
    c->inflight_end = end;
}

static void comm_finish_tile(comm_t* c) {
    const int r = c->inflight;
    req_t* q = &c->reqs[r];
    q->arrivals[q->tiles_done] = c->inflight_end;
    q->tiles_done++;
    if (q->tiles_done == c->tiles) {
        if (q->on_demand) q_erase(c->od, &c->nod, r); else q_erase(c->pf, &c->npf, r);
        const int key = q->layer * c->N + q->expert;
        c->pending[key] = -1;
        memcpy(c->fin + (size_t)key * c->tiles, q->arrivals, sizeof(int64_t) * (size_t)c->tiles);
        c->fin_n[key] = c->tiles;
        if (!q->on_demand) lru_insert(&c->caches[q->layer], q->expert, 1);
        q->active = 0;
    }
    c->cursor = c->inflight_end;
    c->inflight = -1;
}

static void comm_advance_until(comm_t* c, int64_t t) {
    for (;;) {
        if (c->inflight >= 0) {
            if (c->inflight_end > t) return;
            comm_finish_tile(c);
            continue;
        }
        int64_t start;
        int r = comm_next_pick(c, &start);
        if (r < 0 || start > t) return;
        comm_start_tile(c, r, start);
    }
}

static int comm_lookup(const comm_t* c, int layer, int expert, int tile, int64_t* out) {
    const int key = layer * c->N + expert;
    const int r = c->pending[key];
    if (r >= 0) {
        if (tile < c->reqs[r].tiles_done) {
            *out = c->reqs[r].arrivals[tile];
            return 1;
        }
        return 0;
    }
    if (tile < c->fin_n[key]) {
        *out = c->fin[(size_t)key * c->tiles + tile];
        return 1;
    }
    return 0;
}

static int comm_wait_for_tile(comm_t* c, int layer, int expert, int tile, int64_t* arrival) {
    for (;;) {
        if (comm_lookup(c, layer, expert, tile, arrival)) return 0;
        if (c->inflight >= 0) {
            comm_finish_tile(c);
            continue;
        }
        int64_t start;
        int r = comm_next_pick(c, &start);
        if (r < 0) return -3;
        comm_start_tile(c, r, start);
    }
}

/* ------------------------------------------------------------------------------------------ */
/* inc/simulator.hpp:329-468 simulate_trace (per token, per layer).                           */
/* ------------------------------------------------------------------------------------------ */
static int predicted_selection(const double* x, const double* W, int D, int N, int K, int gating, double fisher,
                               double tau, int* out, int* cnt) {
    double lg[64], sc[64];
    orc_gate_logits(W, D, N, x, lg);
    orc_softmax(lg, N, sc);
    if (gating) return orc_gate_decide(sc, N, K, fisher, tau, out, cnt, NULL), 0;
    orc_top_k(sc, N, K, out);
    *cnt = K;
    return 0;
}

/* Batched decode (BASELINE config 4) has no reference counterpart: the reference is batch-1
 * (SPEC.md:531).  Builder-defined extension, B independent token streams sharing one expert cache:
 * per (token, layer) every stream is routed with the reference rule; the cache sees the UNION of
 * the streams' selections (order of first appearance: stream-major, rank order), and each
 * look-ahead target's prediction list is the union of the streams' lists (same order), fed to the
 * unchanged plan_prefetch/dedupe.  single_expert_decisions counts per stream; experts_activated
 * counts union members (so activated = hits + prefetch hits + on-demand still holds).  With B = 1
 * every union is the stream's own list, i.e. exactly simulate_trace (pinned by the goldens). */
static void union_add(int* u, int* n, const int* src, int cnt) {
    for (int k = 0; k < cnt; ++k) {
        int seen = 0;
        for (int i = 0; i < *n; ++i)
            if (u[i] == src[k]) { seen = 1; break; }
        if (!seen) u[(*n)++] = src[k];
    }
}

int orc_simulate_batch(const double* acts, const double* scores, const double* gates, const double* first_gate,
                       int B, int T, int L, int N, int K, int D, const double* fisher, const int* caps, double tau,
                       orc_simcfg cfg, uint64_t seed, orc_metrics* m, int64_t* latency_per_token,
                       int64_t* od_per_layer, int64_t* timeline, int64_t timeline_cap, int64_t* n_events,
                       int* predictions, int* decisions) {
    if (N > 64 || K > N || B < 1 || cfg.tiles < 1 || cfg.lookahead < 0 || cfg.lookahead > 3) return -1;
    memset(m, 0, sizeof(*m));
    for (int l = 0; l < L; ++l) od_per_layer[l] = 0;
    const int prefetch_on = cfg.prefetch && cfg.lookahead > 0;

    lru_t* caches = (lru_t*)calloc((size_t)L, sizeof(lru_t));
    orc_rng rng;
    orc_rng_init(&rng, seed);
    int sub[64];
    for (int l = 0; l < L; ++l) {
        caches[l].cap = caps[l];
        orc_rng_sample_subset(&rng, N, caps[l], sub);
        for (int i = 0; i < caps[l]; ++i) lru_insert(&caches[l], sub[i], 0);
    }

    comm_t c;
    memset(&c, 0, sizeof c);
    c.tiles = cfg.tiles; c.L = L; c.N = N; c.tile_time = cfg.tile_transfer; c.cursor = 0;
    c.capreq = 16;
    c.reqs = (req_t*)malloc(sizeof(req_t) * (size_t)c.capreq);
    c.capq = L * N + 1;
    c.od = (int*)malloc(sizeof(int) * (size_t)c.capq);
    c.pf = (int*)malloc(sizeof(int) * (size_t)c.capq);
    c.pending = (int*)malloc(sizeof(int) * (size_t)L * N);
    for (int i = 0; i < L * N; ++i) c.pending[i] = -1;
    c.fin = (int64_t*)calloc((size_t)L * N * cfg.tiles, sizeof(int64_t));
    c.fin_n = (int*)calloc((size_t)L * N, sizeof(int));
    c.inflight = -1;
    c.caches = caches;
    c.tl = timeline; c.tl_cap = timeline ? timeline_cap : 0; c.tl_n = 0;

    int rc = 0;
    int64_t cur = 0;
    const int PW = 2 + K;
    for (int tok = 0; tok < T && rc == 0; ++tok) {
        const int64_t token_start = cur;
        for (int layer = 0; layer < L && rc == 0; ++layer) {
            tl_push(&c, 0, 0, cur, cur + cfg.attention, tok, layer, -1, -1);
            cur += cfg.attention;
            tl_push(&c, 0, 1, cur, cur + cfg.gate, tok, layer, -1, -1);
            cur += cfg.gate;
            comm_advance_until(&c, cur);

            /* route every stream; union of the selections */
            int sel[64], cnt = 0;
            int pl[3], pc[3], pe[3][64], np = 0;
            for (int b = 0; b < B; ++b) {
                const size_t tl_idx = ((size_t)b * T + tok) * L + layer;
                const double* x = acts + tl_idx * D;
                int sb[64], cb, single;
                if (cfg.gating) {
                    single = orc_gate_decide(scores + tl_idx * N, N, K, fisher[layer], tau, sb, &cb, NULL);
                } else {
                    orc_top_k(scores + tl_idx * N, N, K, sb);
                    cb = K;
                    single = K == 1;
                }
                if (decisions)
                    for (int k = 0; k < K; ++k) decisions[tl_idx * K + k] = k < cb ? sb[k] : -1;
                m->single_expert_decisions += single;
                union_add(sel, &cnt, sb, cb);

                /* this stream's look-ahead predictions (inc/simulator.hpp:422-436) */
                int bl[3], bc[3], be[3][64], bn = 0;
                if (prefetch_on) {
                    if (layer + 1 < L) {
                        for (int depth = 1; depth <= cfg.lookahead; ++depth) {
                            const int tgt = layer + depth;
                            if (tgt >= L) break;
                            bl[bn] = tgt;
                            predicted_selection(x, gates + (size_t)tgt * D * N, D, N, K, cfg.gating, fisher[tgt], tau,
                                                be[bn], &bc[bn]);
                            bn++;
                        }
                    } else if (first_gate && tok + 1 < T) {
                        bl[bn] = 0;
                        predicted_selection(x, first_gate, D, N, K, cfg.gating, fisher[0], tau, be[bn], &bc[bn]);
                        bn++;
                    }
                }
                if (b == 0) {
                    np = bn;
                    for (int s = 0; s < bn; ++s) { pl[s] = bl[s]; pc[s] = 0; }
                }
                for (int s = 0; s < bn; ++s) union_add(pe[s], &pc[s], be[s], bc[s]);
                if (predictions) {
                    int* p = predictions + tl_idx * 3 * PW;
                    for (int s = 0; s < 3; ++s) {
                        int* row = p + s * PW;
                        row[0] = s < bn ? bl[s] : -1;
                        row[1] = s < bn ? bc[s] : 0;
                        for (int k = 0; k < K; ++k) row[2 + k] = (s < bn && k < bc[s]) ? be[s][k] : -1;
                    }
                }
            }
            m->experts_activated_total += cnt;

            int res_now[64], miss_now[64], nres = 0, nmiss = 0;
            lru_t* cache = &caches[layer];
            for (int k = 0; k < cnt; ++k) {
                const int e = sel[k];
                if (cache->res[e]) {
                    if (cache->fresh[e]) m->prefetch_hits++; else m->cache_hits++;
                    lru_touch(cache, e);
                    res_now[nres++] = e;
                } else {
                    m->on_demand_loads++;
                    od_per_layer[layer]++;
                    if (c.pending[layer * N + e] >= 0) comm_promote(&c, layer, e);
                    else comm_enqueue(&c, layer, e, 1, cur, tok);
                    miss_now[nmiss++] = e;
                }
            }

            if (prefetch_on) {
                /* inc/prefetch.hpp:101-119 plan_prefetch, then dedupe against pending (:437-443) */
                const int targets = np < cfg.lookahead ? np : cfg.lookahead;
                for (int idx = 0; idx < targets; ++idx) {
                    int any_missing = 0;
                    for (int k = 0; k < pc[idx]; ++k) {
                        const int e = pe[idx][k];
                        if (caches[pl[idx]].res[e]) continue;
                        any_missing = 1;
                        if (c.pending[pl[idx] * N + e] < 0) comm_enqueue(&c, pl[idx], e, 0, cur, tok);
                    }
                    if (any_missing) break;
                }
            }

            for (int i = 0; i < nres; ++i) {
                const int64_t dur = (int64_t)cfg.tiles * cfg.tile_compute;
                tl_push(&c, 0, 2, cur, cur + dur, tok, layer, res_now[i], -1);
                cur += dur;
            }
            for (int i = 0; i < nmiss; ++i) {
                const int e = miss_now[i];
                for (int tile = 0; tile < cfg.tiles; ++tile) {
                    int64_t arrival;
                    if (comm_wait_for_tile(&c, layer, e, tile, &arrival) != 0) {
                        rc = -3;
                        break;
                    }
                    const int64_t start = cur > arrival ? cur : arrival;
                    m->stall_time += start - cur;
                    tl_push(&c, 0, 3, start, start + cfg.tile_compute, tok, layer, e, tile);
                    cur = start + cfg.tile_compute;
                }
                comm_advance_until(&c, cur);
                lru_insert(&caches[layer], e, 0);
            }
        }
        latency_per_token[tok] = cur - token_start;
    }
    m->total_latency = cur;
    *n_events = c.tl_n;
    if (rc == 0 && timeline && c.tl_n > timeline_cap) rc = -100;

    for (int i = 0; i < c.nreq; ++i) free(c.reqs[i].arrivals);
    free(c.reqs); free(c.od); free(c.pf); free(c.pending); free(c.fin); free(c.fin_n); free(caches);
    return rc;
}

int orc_simulate(const double* acts, const double* scores, const double* gates, const double* first_gate, int T,
                 int L, int N, int K, int D, const double* fisher, const int* caps, double tau, orc_simcfg cfg,
                 uint64_t seed, orc_metrics* m, int64_t* latency_per_token, int64_t* od_per_layer, int64_t* timeline,
                 int64_t timeline_cap, int64_t* n_events, int* predictions, int* decisions) {
    return orc_simulate_batch(acts, scores, gates, first_gate, 1, T, L, N, K, D, fisher, caps, tau, cfg, seed, m,
                              latency_per_token, od_per_layer, timeline, timeline_cap, n_events, predictions, decisions);
}

/* ------------------------------------------------------------------------------------------ */
/* Builder-defined expert weights + SwiGLU (no reference counterpart).                        */
/* ------------------------------------------------------------------------------------------ */
float orc_init_scale(int fan_in) { return (float)(1.0 / (37837.22 * sqrt((double)fan_in))); }

uint64_t orc_expert_base(uint64_t seed, int layer, int expert, int matrix) {
    return orc_splitmix(orc_splitmix(seed) ^ ((uint64_t)(uint32_t)layer << 24) ^ ((uint64_t)(uint32_t)expert << 4) ^
                        (uint64_t)(uint32_t)matrix);
}

uint16_t orc_init_value(uint64_t base, uint64_t index, float scale) {
    const uint64_t h = orc_splitmix(base + index);
    const int32_t u = (int32_t)(h & 0xffff) + (int32_t)((h >> 16) & 0xffff) + (int32_t)((h >> 32) & 0xffff) +
                      (int32_t)((h >> 48) & 0xffff);
    const float v = (float)(u - 131070) * scale;
    uint32_t bits;
    memcpy(&bits, &v, 4);
    bits += 0x7fffu + ((bits >> 16) & 1u); /* round to nearest even */
    return (uint16_t)(bits >> 16);
}

int orc_expert_init(uint64_t seed, int layer, int expert, int D, int F, int tiles, uint16_t* out) {
    if (tiles < 1 || F % tiles) return -1;
    const int Ft = F / tiles;
    const uint64_t b1 = orc_expert_base(seed, layer, expert, 0), b3 = orc_expert_base(seed, layer, expert, 1),
                   b2 = orc_expert_base(seed, layer, expert, 2);
    const float s13 = orc_init_scale(D), s2 = orc_init_scale(F);
    size_t o = 0;
    for (int t = 0; t < tiles; ++t) {
        for (int rl = 0; rl < Ft; ++rl) {
            const uint64_t r = (uint64_t)t * Ft + rl;
            for (int c = 0; c < D; ++c) out[o++] = orc_init_value(b1, r * D + c, s13);
            for (int c = 0; c < D; ++c) out[o++] = orc_init_value(b3, r * D + c, s13);
        }
        for (int rl = 0; rl < Ft; ++rl) /* down_t [Ft][D]: row rl = W2[:, t*Ft + rl] */
            for (int j = 0; j < D; ++j) out[o++] = orc_init_value(b2, (uint64_t)j * F + (uint64_t)t * Ft + rl, s2);
    }
    return 0;
}

static double bf16_to_d(uint16_t b) {
    uint32_t bits = (uint32_t)b << 16;
    float f;
    memcpy(&f, &bits, 4);
    return (double)f;
}

int orc_swiglu(const uint16_t* w, int D, int F, int tiles, const float* x, double* y) {
    if (tiles < 1 || F % tiles) return -1;
    const int Ft = F / tiles;
    double* h = (double*)malloc(sizeof(double) * (size_t)Ft);
    for (int j = 0; j < D; ++j) y[j] = 0.0;
    const size_t tile_elems = (size_t)3 * Ft * D;
    for (int t = 0; t < tiles; ++t) {
        const uint16_t* gu = w + (size_t)t * tile_elems;
        const uint16_t* dn = gu + (size_t)2 * Ft * D;
        for (int rl = 0; rl < Ft; ++rl) {
            double a = 0.0, b = 0.0;
            const uint16_t* r1 = gu + (size_t)rl * 2 * D;
            const uint16_t* r3 = r1 + D;
            for (int c = 0; c < D; ++c) {
                a += bf16_to_d(r1[c]) * (double)x[c];
                b += bf16_to_d(r3[c]) * (double)x[c];
            }
            h[rl] = a / (1.0 + exp(-a)) * b;
        }
        for (int j = 0; j < D; ++j) {
            double acc = 0.0;
            for (int rl = 0; rl < Ft; ++rl) acc += bf16_to_d(dn[(size_t)rl * D + j]) * h[rl];
            y[j] += acc;
        }
    }
    free(h);
    return 0;
}

/* FNV-1a over raw bytes (fixture hashing; same as inc/io.hpp:80-87 over a byte string). */
uint64_t orc_fnv1a(const void* data, size_t n, uint64_t h) {
    const unsigned char* p = (const unsigned char*)data;
    for (size_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ULL;
    }
    return h;
}
