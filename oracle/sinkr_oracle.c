/*
 * sinkr_oracle.c — TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * Plain-C restatement of the reference's CPU algorithm for the SinkRouter
 * decode hot path (routing probe -> Split-K online softmax -> LSE merge).
 * Every function cites the reference file:line it follows
 * (/root/reference/proj/...).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load this library.  It is pinned against the
 * compiled reference itself (oracle/_ref/libsinkr_ref.so, built from the
 * reference sources by oracle/Makefile) and against the SPEC.md known-answer
 * examples; see tests/test_oracle.py.
 *
 * Arithmetic is kept identical to the reference: sequential fp64 sums over f32
 * products, libm exp/sqrt, no FMA contraction (compiled with
 * -ffp-contract=off; the reference is built without -march so g++ emits no
 * FMA either).  Results are therefore bit-identical to the reference.
 *
 * Error codes: 0 ok, 1 invalid_argument, 2 out_of_range, 3 runtime_error,
 * 4 logic_error (same numbering as include/sinkr_cuda.h).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_INVALID 1
#define ORC_RANGE 2
#define ORC_RUNTIME 3
#define ORC_LOGIC 4

/* std::clamp semantics (returns v unchanged when v is NaN). */
static double clampd(double v, double lo, double hi) {
    return v < lo ? lo : (hi < v ? hi : v);
}
/* std::max(a, b) == (a < b) ? b : a */
static double maxd(double a, double b) { return a < b ? b : a; }

/* attention.cpp:25-29 — sequential fp64 dot of f32 vectors. */
static double dot_f32(const float* a, const float* b, size_t n) {
    double s = 0.0;
    for (size_t i = 0; i < n; ++i) s += (double)a[i] * (double)b[i];
    return s;
}

/* kv_cache.cpp:19-23,71-77 — anchor norm captured at first append, stored as
 * float; < 1e-12 is a degenerate anchor (runtime_error). */
int orc_anchor_norm(const float* k, size_t d, float* norm) {
    double s = 0.0;
    for (size_t i = 0; i < d; ++i) s += (double)k[i] * (double)k[i];
    double n = sqrt(s);
    if (n < 1e-12) return ORC_RUNTIME;
    *norm = (float)n;
    return ORC_OK;
}

/* router.cpp:36-48 — cosine proxy against the group anchor. */
int orc_proxy_score(const float* q, const float* k0, float k0_norm, size_t d, double* score,
                    int* degenerate) {
    double dot = 0.0, q_sq = 0.0;
    for (size_t i = 0; i < d; ++i) {
        dot += (double)q[i] * (double)k0[i];
        q_sq += (double)q[i] * (double)q[i];
    }
    const double q_norm = sqrt(q_sq);
    if (q_norm < 1e-12) {
        *score = 0.0;
        *degenerate = 1;
        return ORC_OK;
    }
    const double c = dot / (q_norm * (double)k0_norm);
    *score = clampd(c, -1.0, 1.0);
    *degenerate = 0;
    return ORC_OK;
}

/* router.cpp:50-57 — arithmetic mean, sequential sum then divide by r. */
int orc_group_score(const double* scores, size_t n, size_t width, double* out) {
    if (n != width) return ORC_INVALID;
    double sum = 0.0;
    for (size_t i = 0; i < n; ++i) sum += scores[i];
    *out = sum / (double)width;
    return ORC_OK;
}

/* router.cpp:59-65 — tau = clamp(((a x + b) x + c) x + d), x = L / normalizer. */
int orc_threshold_for_length(size_t len, const double* c, double normalizer, double lo,
                             double hi, double* out) {
    if (len == 0) return ORC_INVALID;
    const double x = (double)len / normalizer;
    const double tau = ((c[0] * x + c[1]) * x + c[2]) * x + c[3];
    *out = clampd(tau, lo, hi);
    return ORC_OK;
}

/* calibration.cpp:29-35 — ThresholdProfile::constant. */
void orc_profile_constant(double tau, double* coeffs, double* normalizer, double* lo,
                          double* hi) {
    coeffs[0] = coeffs[1] = coeffs[2] = 0.0;
    coeffs[3] = tau;
    *normalizer = 1.0;
    *lo = tau < 0.0 ? tau : 0.0; /* std::min(tau, 0.0) */
    *hi = 1.0 < tau ? tau : 1.0; /* std::max(tau, 1.0) */
}

/* router.cpp:31-34 — excluded-layer membership. */
static int layer_excluded(size_t layer, const size_t* excl, size_t n) {
    for (size_t i = 0; i < n; ++i)
        if (excl[i] == layer) return 1;
    return 0;
}

/* router.cpp:67-75 — strict S > tau (>= with sink_on_tie), excluded layers never sink. */
int orc_route(size_t layer, double score, size_t len, const double* coeffs, double normalizer,
              double lo, double hi, const size_t* excluded, size_t n_excluded, int sink_on_tie,
              int* sink, double* threshold) {
    int rc = orc_threshold_for_length(len, coeffs, normalizer, lo, hi, threshold);
    if (rc) return rc;
    const int over = sink_on_tie ? (score >= *threshold) : (score > *threshold);
    *sink = over && !layer_excluded(layer, excluded, n_excluded);
    return ORC_OK;
}

/* router.cpp:77-80 */
size_t orc_auto_num_splits(size_t len) {
    size_t s = (len + 8191) / 8192;
    return s < 1 ? 1 : (s > 16 ? 16 : s);
}

/* attention.cpp:185-202 — even-remainder chunking. */
int orc_split_ranges(size_t len, size_t n, size_t* from_to) {
    if (n == 0 || n > len) return ORC_INVALID;
    const size_t base = len / n, rem = len % n;
    size_t start = 0;
    for (size_t c = 0; c < n; ++c) {
        const size_t sz = base + (c < rem ? 1 : 0);
        from_to[2 * c] = start;
        from_to[2 * c + 1] = start + sz;
        start += sz;
    }
    return ORC_OK;
}

/* attention.cpp:33-40 — logit scale 1.0f / sqrtf(D). */
static float qg_scale(size_t dim) { return 1.0f / sqrtf((float)dim); }

/* attention.cpp:101-142 — single-pass blocked online softmax over one chunk.
 * m, l: heads; acc: heads x dim; fp64 state, f32 data. */
int orc_attend_chunk(const float* q, size_t heads, size_t dim, const float* k, const float* v,
                     size_t len, size_t block, double* m, double* l, double* acc) {
    if (heads == 0 || dim == 0 || len == 0 || block == 0) return ORC_INVALID;
    const float scale = qg_scale(dim);
    for (size_t g = 0; g < heads; ++g) {
        m[g] = -INFINITY;
        l[g] = 0.0;
    }
    memset(acc, 0, heads * dim * sizeof(double));
    double* z = (double*)malloc((block < len ? block : len) * sizeof(double));
    if (!z) return ORC_RUNTIME;
    for (size_t b0 = 0; b0 < len; b0 += block) {
        const size_t b1 = (b0 + block < len) ? b0 + block : len;
        for (size_t g = 0; g < heads; ++g) {
            const float* qq = q + g * dim;
            double block_max = -INFINITY;
            for (size_t i = b0; i < b1; ++i) {
                z[i - b0] = (double)scale * dot_f32(qq, k + i * dim, dim);
                block_max = maxd(block_max, z[i - b0]);
            }
            const double new_m = maxd(m[g], block_max);
            const double rescale = exp(m[g] - new_m);
            l[g] *= rescale;
            double* a = acc + g * dim;
            for (size_t j = 0; j < dim; ++j) a[j] *= rescale;
            for (size_t i = b0; i < b1; ++i) {
                const double p = exp(z[i - b0] - new_m);
                l[g] += p;
                const float* vv = v + i * dim;
                for (size_t j = 0; j < dim; ++j) a[j] += p * (double)vv[j];
            }
            m[g] = new_m;
        }
    }
    free(z);
    return ORC_OK;
}

/* attention.cpp:159-183 — LSE combine; partials with tokens == 0 are skipped.
 * Layout: n_parts x m[heads], l[heads], acc[heads*dim]. */
int orc_merge_partials(size_t n_parts, const double* m, const double* l, const double* acc,
                       const size_t* tokens, size_t heads, size_t dim, float* out) {
    size_t live = 0;
    for (size_t p = 0; p < n_parts; ++p) live += tokens[p] != 0;
    if (live == 0) return ORC_INVALID;
    for (size_t g = 0; g < heads; ++g) {
        double m_star = -INFINITY;
        for (size_t p = 0; p < n_parts; ++p)
            if (tokens[p]) m_star = maxd(m_star, m[p * heads + g]);
        double l_star = 0.0;
        for (size_t p = 0; p < n_parts; ++p)
            if (tokens[p]) l_star += l[p * heads + g] * exp(m[p * heads + g] - m_star);
        for (size_t j = 0; j < dim; ++j) {
            double s = 0.0;
            for (size_t p = 0; p < n_parts; ++p)
                if (tokens[p])
                    s += acc[(p * heads + g) * dim + j] * exp(m[p * heads + g] - m_star);
            out[g * dim + j] = (float)(s / l_star);
        }
    }
    return ORC_OK;
}

/* attention.cpp:42-73 — two-pass exact softmax reference. */
int orc_dense_attention(const float* q, size_t heads, size_t dim, const float* k, const float* v,
                        size_t len, float* out) {
    if (heads == 0 || dim == 0 || len == 0) return ORC_INVALID;
    const float scale = qg_scale(dim);
    double* logits = (double*)malloc(len * sizeof(double));
    double* row = (double*)malloc(dim * sizeof(double));
    if (!logits || !row) {
        free(logits);
        free(row);
        return ORC_RUNTIME;
    }
    for (size_t g = 0; g < heads; ++g) {
        const float* qq = q + g * dim;
        double max_logit = -INFINITY;
        for (size_t i = 0; i < len; ++i) {
            logits[i] = (double)scale * dot_f32(qq, k + i * dim, dim);
            max_logit = maxd(max_logit, logits[i]);
        }
        double denom = 0.0;
        for (size_t i = 0; i < len; ++i) {
            logits[i] = exp(logits[i] - max_logit);
            denom += logits[i];
        }
        for (size_t j = 0; j < dim; ++j) row[j] = 0.0;
        for (size_t i = 0; i < len; ++i) {
            const double w = logits[i] / denom;
            const float* vv = v + i * dim;
            for (size_t j = 0; j < dim; ++j) row[j] += w * (double)vv[j];
        }
        for (size_t j = 0; j < dim; ++j) out[g * dim + j] = (float)row[j];
    }
    free(logits);
    free(row);
    return ORC_OK;
}

/* ---- routed_decode_step (router.cpp:82-188) --------------------------------
 * One layer of one sequence.  k, v: [H_kv][len][D] f32 (the slot-major layout
 * of kv_cache.cpp:41-49 restricted to this layer and to the filled rows);
 * k0: [H_kv][D]; k0_norm: [H_kv].  Task-level parallelism over
 * (active group, chunk) with `threads` pthreads mirrors the reference's
 * ThreadPool fan-out (router.cpp:147-165); results do not depend on it. */
typedef struct {
    const float* q;
    const float* k;
    const float* v;
    size_t r, d, len, block;
    const size_t* task_group;
    const size_t* task_from;
    const size_t* task_to;
    double* pm;
    double* pl;
    double* pacc;
    size_t n_tasks;
    size_t next;
    pthread_mutex_t mu;
} orc_tasks;

static void run_task(orc_tasks* t, size_t i) {
    const size_t g = t->task_group[i], from = t->task_from[i], to = t->task_to[i];
    const size_t off = (g * t->len + from) * t->d;
    orc_attend_chunk(t->q + g * t->r * t->d, t->r, t->d, t->k + off, t->v + off, to - from,
                     t->block, t->pm + i * t->r, t->pl + i * t->r, t->pacc + i * t->r * t->d);
}

static void* worker(void* arg) {
    orc_tasks* t = (orc_tasks*)arg;
    for (;;) {
        pthread_mutex_lock(&t->mu);
        size_t i = t->next++;
        pthread_mutex_unlock(&t->mu);
        if (i >= t->n_tasks) break;
        run_task(t, i);
    }
    return NULL;
}

int orc_routed_decode_step(const float* k, const float* v, const float* k0,
                           const float* k0_norm, size_t hq, size_t hkv, size_t d, size_t len,
                           size_t layer, const float* queries, const double* coeffs,
                           double normalizer, double lo, double hi, const size_t* excluded,
                           size_t n_excluded, int sink_on_tie, size_t num_splits, size_t block,
                           int observe_only, int threads, float* outputs, double* group_scores,
                           double* thresholds, int* sink, int* degenerate,
                           uint64_t* group_kv_floats, double* head_scores,
                           uint64_t* counters_u64) {
    if (hkv == 0 || hq == 0 || hq % hkv != 0 || d == 0) return ORC_INVALID;
    if (len == 0) return ORC_RUNTIME; /* router.cpp:90 */
    const size_t r = hq / hkv;
    memset(outputs, 0, hq * d * sizeof(float)); /* router.cpp:97 */
    int* run = (int*)calloc(hkv, sizeof(int));
    uint64_t anchor_floats = 0, groups_active = 0, groups_skipped = 0;

    /* routing (router.cpp:100-125) */
    for (size_t g = 0; g < hkv; ++g) {
        anchor_floats += d; /* kv_cache.cpp:102 */
        int degen = 0;
        for (size_t i = 0; i < r; ++i) {
            int dg = 0;
            orc_proxy_score(queries + (g * r + i) * d, k0 + g * d, k0_norm[g], d,
                            &head_scores[g * r + i], &dg);
            degen = degen || dg;
        }
        double s;
        orc_group_score(head_scores + g * r, r, r, &s);
        int sk;
        double tau;
        int rc = orc_route(layer, s, len, coeffs, normalizer, lo, hi, excluded, n_excluded,
                           sink_on_tie, &sk, &tau);
        if (rc) {
            free(run);
            return rc;
        }
        if (degen) sk = 0; /* router.cpp:114-117 */
        group_scores[g] = s;
        thresholds[g] = tau;
        sink[g] = sk;
        degenerate[g] = degen;
        run[g] = observe_only || !sk;
        group_kv_floats[g] = 0;
    }

    /* splits (router.cpp:127-129) */
    size_t splits = num_splits == 0 ? orc_auto_num_splits(len) : num_splits;
    if (splits < 1) splits = 1;
    if (splits > len) splits = len;
    size_t* ranges = (size_t*)malloc(2 * splits * sizeof(size_t));
    orc_split_ranges(len, splits, ranges);

    /* tasks (router.cpp:131-145) */
    size_t n_tasks = 0;
    for (size_t g = 0; g < hkv; ++g) n_tasks += run[g] ? splits : 0;
    orc_tasks T;
    memset(&T, 0, sizeof(T));
    size_t* tg = (size_t*)malloc((n_tasks + 1) * sizeof(size_t));
    size_t* tf = (size_t*)malloc((n_tasks + 1) * sizeof(size_t));
    size_t* tt = (size_t*)malloc((n_tasks + 1) * sizeof(size_t));
    size_t n = 0;
    for (size_t g = 0; g < hkv; ++g) {
        if (!run[g]) continue;
        for (size_t c = 0; c < splits; ++c, ++n) {
            tg[n] = g;
            tf[n] = ranges[2 * c];
            tt[n] = ranges[2 * c + 1];
        }
    }
    T.q = queries;
    T.k = k;
    T.v = v;
    T.r = r;
    T.d = d;
    T.len = len;
    T.block = block;
    T.task_group = tg;
    T.task_from = tf;
    T.task_to = tt;
    T.n_tasks = n_tasks;
    T.pm = (double*)malloc((n_tasks + 1) * r * sizeof(double));
    T.pl = (double*)malloc((n_tasks + 1) * r * sizeof(double));
    T.pacc = (double*)malloc((n_tasks + 1) * r * d * sizeof(double));
    pthread_mutex_init(&T.mu, NULL);
    if (threads > 1 && n_tasks > 1) {
        pthread_t* th = (pthread_t*)malloc((size_t)threads * sizeof(pthread_t));
        for (int i = 0; i < threads; ++i) pthread_create(&th[i], NULL, worker, &T);
        for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
        free(th);
    } else {
        for (size_t i = 0; i < n_tasks; ++i) run_task(&T, i);
    }
    pthread_mutex_destroy(&T.mu);

    /* merge (router.cpp:168-186) */
    size_t* tok = (size_t*)malloc(splits * sizeof(size_t));
    for (size_t c = 0; c < splits; ++c) tok[c] = ranges[2 * c + 1] - ranges[2 * c];
    uint64_t kv_total = 0;
    size_t part = 0;
    for (size_t g = 0; g < hkv; ++g) {
        if (!run[g]) {
            ++groups_skipped;
            continue;
        }
        ++groups_active;
        orc_merge_partials(splits, T.pm + part * r, T.pl + part * r, T.pacc + part * r * d, tok,
                           r, d, outputs + g * r * d);
        group_kv_floats[g] = 2ull * len * d; /* kv_cache.cpp:116 summed over chunks */
        kv_total += group_kv_floats[g];
        part += splits;
    }
    counters_u64[0] = kv_total;
    counters_u64[1] = anchor_floats;
    counters_u64[2] = groups_active;
    counters_u64[3] = groups_skipped;

    free(tok);
    free(T.pm);
    free(T.pl);
    free(T.pacc);
    free(tg);
    free(tf);
    free(tt);
    free(ranges);
    free(run);
    return ORC_OK;
}

/* ---- synthetic K/V rows --------------------------------------------------
 * Counter-based access to the reference's SplitMix64 stream (tensor.hpp:15-25):
 * draw(key, n) is the n-th output of SplitMix64{key}.  Streams are keyed with
 * the reference's mix_seed rule (tensor.cpp:53-61).  Approximately normal
 * values come from an Irwin-Hall sum of 12 exact 24-bit uniforms, evaluated in
 * integer arithmetic, so the CPU restatement and the device generator in
 * paper_2604_16883_b200/csrc/workload.cu produce bit-identical rows. */
static uint64_t sm64_final(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static uint64_t sm64_draw(uint64_t key, uint64_t n) {
    return sm64_final(key + (n + 1) * 0x9E3779B97F4A7C15ull);
}
uint64_t orc_mix_seed(uint64_t seed, const uint64_t* tags, size_t n) {
    uint64_t h = sm64_draw(seed, 0);
    for (size_t i = 0; i < n; ++i) h = sm64_draw(h ^ (tags[i] + 0x9E3779B97F4A7C15ull), 0);
    return h;
}
float orc_gauss12(uint64_t key, uint64_t e) {
    uint64_t s = 0;
    for (uint64_t j = 0; j < 6; ++j) {
        const uint64_t h = sm64_draw(key, e * 6 + j);
        s += (h >> 40) + ((h >> 16) & 0xFFFFFFull);
    }
    return (float)((double)s * 0x1.0p-24 - 6.0);
}
/* f32 -> bf16 (round to nearest even) -> f32. */
float orc_round_bf16(float x) {
    uint32_t b;
    memcpy(&b, &x, 4);
    if ((b & 0x7F800000u) == 0x7F800000u) {
        b &= 0xFFFF0000u;
        if (x != x) b |= 0x00400000u;
    } else {
        b = (b + 0x7FFFu + ((b >> 16) & 1u)) & 0xFFFF0000u;
    }
    float y;
    memcpy(&y, &b, 4);
    return y;
}
/* rows [row0, row0+rows) of one slot: value = bf16(scale * gauss12(key, row*d + j)). */
void orc_fill_rows(uint64_t key, size_t row0, size_t rows, size_t d, float scale, float* out) {
    for (size_t t = 0; t < rows; ++t)
        for (size_t j = 0; j < d; ++j)
            out[t * d + j] =
                orc_round_bf16(scale * orc_gauss12(key, (uint64_t)(row0 + t) * d + j));
}
