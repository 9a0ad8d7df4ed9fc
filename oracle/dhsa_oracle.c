/*
 * dhsa_oracle.c -- CPU restatement of the reference super point detector's hot
 * path (scan -> zero counts -> hot sets -> candidate restore -> re-estimate and
 * threshold filter).
 *
 * THIS IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, the smoke check
 * in __graft_entry__.py and bench.py's cpu_baseline / --impl reference legs may
 * load it.  The product path (paper_1803_11449_b200/) never links, imports or
 * executes anything under oracle/.
 *
 * Parity status: PINNED.  tests/test_oracle_golden.py checks every function
 * below against (a) the constants the reference's own tests hold
 * (pkg/tests/test_dhla.py:43,86; pkg/tests/test_estimator.py:57-62) and (b)
 * fixtures under tests/golden/ produced by importing the reference package in
 * the build container (tests/golden/make_golden.py).
 *
 * Every function cites the reference file:line (relative to /root/reference)
 * whose behaviour it restates.  Nothing here is copied: the reference is
 * Python/Cython, this is plain C written from the algorithm's definition.
 *
 * Build: see oracle/Makefile  (gcc -O3 -fPIC -shared -pthread).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_OK 0
#define ORACLE_ECAPACITY 4
#define ORACLE_ENOMEM (-2)

typedef struct {
    int32_t r;          /* estimator arrays                    pkg/src/dhsa/dhg.py:70 */
    int32_t g;          /* bits per estimator                  pkg/src/dhsa/dhg.py:71 */
    int32_t k;          /* log2 estimators per array           pkg/src/dhsa/dhg.py:72 */
    int32_t alpha;      /* block stride                        pkg/src/dhsa/dhg.py:73 */
    int32_t key_width;  /* bits in a host key                  pkg/src/dhsa/dhg.py:74 */
    int32_t pad_;
    uint64_t state_dh0; /* mix64(seed_dh0 ^ tag)               pkg/src/dhsa/dhg.py:112-114 */
    uint64_t state_h1;  /* mix64(seed_h1 ^ tag)                pkg/src/dhsa/dhg.py:116-118 */
} oracle_params;

/* splitmix64 finaliser.  pkg/src/dhsa/dhg.py:36-44, pkg/src/dhsa/_core.pyx:35-40 */
uint64_t oracle_mix64(uint64_t z)
{
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}

/* Seed -> state, with the two domain-separation tags.  pkg/src/dhsa/dhg.py:29-30,112-118 */
void oracle_states(uint64_t seed_dh0, uint64_t seed_h1, uint64_t *state_dh0, uint64_t *state_h1)
{
    *state_dh0 = oracle_mix64(seed_dh0 ^ 0x9E3779B97F4A7C15ULL);
    *state_h1 = oracle_mix64(seed_h1 ^ 0xD1B54A32D192ED03ULL);
}

/* pkg/src/dhsa/dhg.py:126-128 */
static inline uint64_t dh0_of(const oracle_params *p, uint64_t a)
{
    return oracle_mix64(p->state_dh0 ^ a) & ((1ULL << p->k) - 1);
}

/* pkg/src/dhsa/dhg.py:142-144 */
static inline uint64_t h1_of(const oracle_params *p, uint64_t b)
{
    return oracle_mix64(p->state_h1 ^ b) & ((uint64_t)p->g - 1);
}

/* All r indices of one host.  pkg/src/dhsa/dhg.py:152-158 */
void oracle_forward(const oracle_params *p, uint64_t a, uint64_t *idx)
{
    uint64_t kmask = (1ULL << p->k) - 1, d0 = dh0_of(p, a);
    idx[0] = d0;
    for (int i = 1; i < p->r; i++)
        idx[i] = ((a >> ((i - 1) * p->alpha)) & kmask) ^ d0;
}

uint64_t oracle_h1(const oracle_params *p, uint64_t b) { return h1_of(p, b); }

/*
 * Scalar inverse with its accept predicate.  pkg/src/dhsa/dhg.py:161-185.
 * Returns 1 and stores the key when the r indices are consistent, else 0.
 */
int oracle_reconstruct_key(const oracle_params *p, const uint64_t *idx, uint64_t *key_out)
{
    int k = p->k, a = p->alpha;
    uint64_t omask = (1ULL << (k - a)) - 1;
    uint64_t cl0 = idx[0], blk = cl0 ^ idx[1], key = blk;
    for (int i = 2; i < p->r; i++) {
        uint64_t nxt = cl0 ^ idx[i];
        if ((blk >> a) != (nxt & omask))
            return 0;
        key |= (nxt >> (k - a)) << (k + (i - 2) * a);
        blk = nxt;
    }
    if (key >> p->key_width)
        return 0;
    if (dh0_of(p, key) != cl0)
        return 0;
    *key_out = key;
    return 1;
}

/* ------------------------------------------------------------------ scan -- */

static inline size_t cell_bytes(const oracle_params *p) { return (size_t)p->g / 8; }
static inline size_t cells_per_array(const oracle_params *p) { return (size_t)1 << p->k; }

size_t oracle_sketch_bytes(const oracle_params *p) /* pkg/src/dhsa/dhg.py:120-123 */
{
    return (size_t)p->r * cells_per_array(p) * cell_bytes(p);
}

/*
 * One pair -> r bit sets, all at bit position h1(opp): byte h>>3, mask 1<<(h&7).
 * pkg/src/dhsa/_core.pyx:75-86 (loop body), pkg/src/dhsa/dhla.py:80-85 (scalar form).
 * `atomic` selects the relaxed atomic OR used when threads share one sketch
 * (pkg/src/dhsa/_core.pyx:17-23).
 */
static inline void apply_pair(const oracle_params *p, uint8_t *bits, uint32_t cand, uint32_t opp,
                              int atomic)
{
    const size_t bpe = cell_bytes(p), m = cells_per_array(p);
    const uint64_t kmask = (1ULL << p->k) - 1;
    uint64_t a = cand;
    uint64_t h = h1_of(p, opp);
    uint64_t d0 = oracle_mix64(p->state_dh0 ^ a) & kmask;
    size_t byte_idx = (size_t)(h >> 3);
    uint8_t mask = (uint8_t)(1u << (h & 7));
    for (int i = 0; i < p->r; i++) {
        uint64_t row = (i == 0) ? d0 : (((a >> ((i - 1) * p->alpha)) & kmask) ^ d0);
        uint8_t *cell = bits + ((size_t)i * m + (size_t)row) * bpe + byte_idx;
        if (atomic)
            __atomic_fetch_or(cell, mask, __ATOMIC_RELAXED);
        else
            *cell |= mask;
    }
}

/* Single-threaded batch update.  pkg/src/dhsa/_core.pyx:52-86 */
void oracle_update_batch(const oracle_params *p, uint8_t *bits, const uint32_t *cand,
                         const uint32_t *opp, size_t n)
{
    for (size_t t = 0; t < n; t++)
        apply_pair(p, bits, cand[t], opp[t], 0);
}

typedef struct {
    const oracle_params *p;
    uint8_t *bits;
    const uint32_t *cand, *opp;
    size_t lo, hi;
} scan_job;

static void *scan_worker(void *arg)
{
    scan_job *j = (scan_job *)arg;
    for (size_t t = j->lo; t < j->hi; t++)
        apply_pair(j->p, j->bits, j->cand[t], j->opp[t], 1);
    return NULL;
}

/*
 * Threads sharing one sketch, as the reference's window engine does with its
 * pool (pkg/src/dhsa/engine.py:81-86) on top of the atomic byte OR
 * (pkg/src/dhsa/_core.pyx:82-86).  Contiguous slices per thread.
 */
int oracle_update_batch_mt(const oracle_params *p, uint8_t *bits, const uint32_t *cand,
                           const uint32_t *opp, size_t n, int nthreads)
{
    if (nthreads <= 1 || n < 4096) {
        oracle_update_batch(p, bits, cand, opp, n);
        return ORACLE_OK;
    }
    pthread_t *tid = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    scan_job *jobs = (scan_job *)malloc(sizeof(scan_job) * (size_t)nthreads);
    if (!tid || !jobs) {
        free(tid);
        free(jobs);
        return ORACLE_ENOMEM;
    }
    size_t per = (n + (size_t)nthreads - 1) / (size_t)nthreads;
    int started = 0;
    for (int w = 0; w < nthreads; w++) {
        size_t lo = per * (size_t)w, hi = lo + per;
        if (lo > n) lo = n;
        if (hi > n) hi = n;
        jobs[w] = (scan_job){p, bits, cand, opp, lo, hi};
        if (pthread_create(&tid[w], NULL, scan_worker, &jobs[w]) != 0) {
            scan_worker(&jobs[w]);
            tid[w] = 0;
            continue;
        }
        started |= 1;
    }
    (void)started;
    for (int w = 0; w < nthreads; w++)
        if (tid[w]) pthread_join(tid[w], NULL);
    free(tid);
    free(jobs);
    return ORACLE_OK;
}

/* -------------------------------------------------------------- read-out -- */

/*
 * g - popcount(cell) for every cell, (r, 2^k) row-major int64.
 * pkg/src/dhsa/_core.pyx:89-118 (word path when g/8 % 8 == 0, byte path else).
 */
void oracle_zero_counts(const oracle_params *p, const uint8_t *bits, int64_t *out)
{
    const size_t bpe = cell_bytes(p), ncell = (size_t)p->r * cells_per_array(p);
    for (size_t c = 0; c < ncell; c++) {
        const uint8_t *cell = bits + c * bpe;
        int64_t ones = 0;
        if (bpe % 8 == 0) {
            for (size_t q = 0; q < bpe; q += 8) {
                uint64_t w;
                memcpy(&w, cell + q, 8);
                ones += __builtin_popcountll(w);
            }
        } else {
            for (size_t q = 0; q < bpe; q++)
                ones += __builtin_popcount(cell[q]);
        }
        out[c] = (int64_t)p->g - ones;
    }
}

/* Zmin = g * exp(-theta / g).  pkg/src/dhsa/dhla.py:45-47 */
double oracle_hot_threshold(int32_t g, double theta) { return g * exp(-theta / g); }

/*
 * HE(i) = { j : zc[i][j] < Zmin }, ascending.  pkg/src/dhsa/dhla.py:111-119.
 * lists: r * 2^k u64 (row i starts at i * 2^k), counts: r.
 */
void oracle_hot_sets(const oracle_params *p, const int64_t *zc, double theta, uint64_t *lists,
                     uint64_t *counts)
{
    const size_t m = cells_per_array(p);
    double zmin = oracle_hot_threshold(p->g, theta);
    for (int i = 0; i < p->r; i++) {
        uint64_t n = 0;
        for (size_t j = 0; j < m; j++)
            if ((double)zc[(size_t)i * m + j] < zmin)
                lists[(size_t)i * m + n++] = (uint64_t)j;
        counts[i] = n;
    }
}

/* Per array ZR(i) = sum_j zc[i][j].  pkg/src/dhsa/dhla.py:126 */
void oracle_zero_totals(const oracle_params *p, const int64_t *zc, int64_t *zr)
{
    const size_t m = cells_per_array(p);
    for (int i = 0; i < p->r; i++) {
        int64_t s = 0;
        for (size_t j = 0; j < m; j++) s += zc[(size_t)i * m + j];
        zr[i] = s;
    }
}

/*
 * Linear counting over each whole array, averaged.  ZR == 0 is evaluated at one
 * zero bit and flagged saturated.
 * pkg/src/dhsa/estimator.py:26-34, pkg/src/dhsa/dhla.py:121-128.
 */
double oracle_flow_count(const oracle_params *p, const int64_t *zr, int *saturated)
{
    double cap = (double)p->g * (double)cells_per_array(p), acc = 0.0;
    int sat = 0;
    for (int i = 0; i < p->r; i++) {
        int64_t z = zr[i];
        if (z == 0) {
            sat = 1;
            z = 1;
        }
        acc += -cap * log((double)z / cap);
    }
    if (saturated) *saturated = sat;
    return acc / p->r;
}

/* psi = 1 - exp(-w / (g 2^k)).  pkg/src/dhsa/dhla.py:130-134 */
double oracle_bit_set_probability(const oracle_params *p, double flow_count)
{
    return 1.0 - exp(-flow_count / ((double)p->g * (double)cells_per_array(p)));
}

/* --------------------------------------------------------------- restore -- */

typedef struct {
    uint64_t *sub, *cl0;
    size_t n, cap;
} partials;

static int partials_push(partials *b, uint64_t sub, uint64_t cl0)
{
    if (b->n == b->cap) {
        size_t ncap = b->cap ? b->cap * 2 : 1024;
        uint64_t *ns = (uint64_t *)realloc(b->sub, ncap * 8);
        if (!ns) return -1;
        b->sub = ns;
        uint64_t *nc = (uint64_t *)realloc(b->cl0, ncap * 8);
        if (!nc) return -1;
        b->cl0 = nc;
        b->cap = ncap;
    }
    b->sub[b->n] = sub;
    b->cl0[b->n] = cl0;
    b->n++;
    return 0;
}

static void partials_free(partials *b)
{
    free(b->sub);
    free(b->cl0);
    memset(b, 0, sizeof *b);
}

static int cmp_u64(const void *x, const void *y)
{
    uint64_t a = *(const uint64_t *)x, b = *(const uint64_t *)y;
    return (a > b) - (a < b);
}

/*
 * Candidate hosts from the hot sets: the reference's literal enumeration --
 * the full cross product HE0 x HE1 x HE2, then partials x HE_i -- NOT the
 * 2^alpha-extension shortcut the CUDA path uses, so the two check each other.
 *
 *   empty hot set -> no candidates               pkg/src/dhsa/dhla.py:208-209
 *   stage 1                                      pkg/src/dhsa/dhla.py:252-274
 *   stage i >= 3                                 pkg/src/dhsa/dhla.py:277-299
 *   key-width cut, dh0 verification, unique      pkg/src/dhsa/dhla.py:213-217
 *
 * A stage whose survivor count exceeds max_candidates aborts with
 * ORACLE_ECAPACITY; *fail_stage gets the reference's stage number (1, then
 * i - 1) and *fail_count the survivor count, the two numbers in the
 * reference's CapacityError text (dhla.py:269-273, 294-298).
 * stage_counts (optional, r - 2 entries) receives the survivor count per stage.
 * hosts_out holds hosts_cap entries (ORACLE_ENOMEM if the verified keys exceed it).
 */
int oracle_candidate_hosts(const oracle_params *p, const uint64_t *lists, const uint64_t *counts,
                           uint64_t max_candidates, uint64_t *hosts_out, uint64_t hosts_cap,
                           uint64_t *n_hosts, int32_t *fail_stage, uint64_t *fail_count,
                           uint64_t *stage_counts)
{
    const size_t m = cells_per_array(p);
    const int k = p->k, al = p->alpha, r = p->r;
    const uint64_t omask = (1ULL << (k - al)) - 1;
    *n_hosts = 0;
    if (fail_stage) *fail_stage = 0;
    if (fail_count) *fail_count = 0;
    if (stage_counts) memset(stage_counts, 0, sizeof(uint64_t) * (size_t)(r - 2));
    for (int i = 0; i < r; i++)
        if (counts[i] == 0) return ORACLE_OK;

    partials cur = {0}, nxt = {0};
    const uint64_t *he0 = lists, *he1 = lists + m, *he2 = lists + 2 * m;
    for (uint64_t x = 0; x < counts[0]; x++) {
        uint64_t cl0 = he0[x];
        for (uint64_t y = 0; y < counts[1]; y++) {
            uint64_t b1 = cl0 ^ he1[y];
            for (uint64_t z = 0; z < counts[2]; z++) {
                uint64_t b2 = cl0 ^ he2[z];
                if ((b1 >> al) == (b2 & omask))
                    if (partials_push(&cur, b1 | ((b2 >> (k - al)) << k), cl0)) goto nomem;
            }
        }
    }
    if (stage_counts) stage_counts[0] = cur.n;
    if (cur.n > max_candidates) {
        if (fail_stage) *fail_stage = 1;
        if (fail_count) *fail_count = cur.n;
        partials_free(&cur);
        return ORACLE_ECAPACITY;
    }
    for (int i = 3; i < r; i++) {
        const uint64_t *he = lists + (size_t)i * m;
        const int sh_chk = (i - 1) * al, sh_put = k + (i - 2) * al;
        nxt.n = 0;
        for (size_t q = 0; q < cur.n; q++) {
            uint64_t sp = cur.sub[q], cl0 = cur.cl0[q];
            for (uint64_t z = 0; z < counts[i]; z++) {
                uint64_t blk = cl0 ^ he[z];
                if ((sp >> sh_chk) == (blk & omask))
                    if (partials_push(&nxt, sp | ((blk >> (k - al)) << sh_put), cl0)) goto nomem;
            }
        }
        partials t = cur;
        cur = nxt;
        nxt = t;
        if (stage_counts) stage_counts[i - 2] = cur.n;
        if (cur.n > max_candidates) {
            if (fail_stage) *fail_stage = i - 1;
            if (fail_count) *fail_count = cur.n;
            partials_free(&cur);
            partials_free(&nxt);
            return ORACLE_ECAPACITY;
        }
    }
    {
        const int w = p->key_width;
        const uint64_t wmask = (w >= 64) ? ~0ULL : ((1ULL << w) - 1);
        uint64_t n = 0;
        for (size_t q = 0; q < cur.n; q++) {
            if (cur.sub[q] >> w) continue;
            uint64_t key = cur.sub[q] & wmask;
            if (dh0_of(p, key) != cur.cl0[q]) continue;
            if (n == hosts_cap) goto nomem;
            hosts_out[n++] = key;
        }
        qsort(hosts_out, n, 8, cmp_u64);
        uint64_t u = 0;
        for (uint64_t q = 0; q < n; q++)
            if (u == 0 || hosts_out[u - 1] != hosts_out[q]) hosts_out[u++] = hosts_out[q];
        *n_hosts = u;
    }
    partials_free(&cur);
    partials_free(&nxt);
    return ORACLE_OK;
nomem:
    partials_free(&cur);
    partials_free(&nxt);
    return ORACLE_ENOMEM;
}

/*
 * SZ(host) = g - popcount(AND of the host's r cells).  pkg/src/dhsa/dhla.py:136-143
 */
void oracle_shared_zero_counts(const oracle_params *p, const uint8_t *bits, const uint64_t *hosts,
                               size_t n, int64_t *sz)
{
    const size_t bpe = cell_bytes(p), m = cells_per_array(p);
    uint64_t idx[64];
    for (size_t t = 0; t < n; t++) {
        oracle_forward(p, hosts[t], idx);
        int64_t ones = 0;
        for (size_t q = 0; q < bpe; q++) {
            uint8_t acc = 0xFF;
            for (int i = 0; i < p->r; i++)
                acc &= bits[((size_t)i * m + (size_t)idx[i]) * bpe + q];
            ones += __builtin_popcount(acc);
        }
        sz[t] = (int64_t)p->g - ones;
    }
}

/*
 * Sharing-corrected estimate of one SZ value.
 *   denom = g (1 - psi^r); SZ == 0 -> saturated, evaluate at 1;
 *   SZ >= denom -> 0.0; else -g ln(SZ / denom).
 * pkg/src/dhsa/dhla.py:183-189 (vector form), 145-160 (scalar form).
 */
double oracle_corrected_estimate(const oracle_params *p, int64_t sz, double psi, int *saturated)
{
    double denom = p->g * (1.0 - pow(psi, p->r));
    int sat = (sz == 0);
    if (sat) sz = 1;
    if (saturated) *saturated = sat;
    if ((double)sz >= denom) return 0.0;
    return -(double)p->g * log((double)sz / denom);
}

typedef struct {
    uint64_t host;
    double est;
    int32_t sat;
} report_row;

static int cmp_report(const void *x, const void *y) /* pkg/src/dhsa/dhla.py:195 */
{
    const report_row *a = (const report_row *)x, *b = (const report_row *)y;
    if (a->est != b->est) return (a->est < b->est) ? 1 : -1; /* descending estimate */
    return (a->host > b->host) - (a->host < b->host);         /* ascending host */
}

/*
 * Whole read-out: zero counts -> candidates -> psi -> SZ -> estimate ->
 * keep est >= theta -> sort by (-estimate, host).  pkg/src/dhsa/dhla.py:164-196.
 * Outputs hold max_candidates entries.  Returns ORACLE_OK / ORACLE_ECAPACITY.
 */
int oracle_restore_superpoints(const oracle_params *p, const uint8_t *bits, double theta,
                               uint64_t max_candidates, uint64_t *hosts_out, double *est_out,
                               uint8_t *sat_out, uint64_t *n_out, int32_t *fail_stage,
                               uint64_t *fail_count)
{
    const size_t m = cells_per_array(p), ncell = (size_t)p->r * m;
    *n_out = 0;
    int64_t *zc = (int64_t *)malloc(ncell * 8);
    uint64_t *lists = (uint64_t *)malloc(ncell * 8);
    uint64_t cand_cap = max_candidates ? max_candidates : 1;
    uint64_t *cand = (uint64_t *)malloc((size_t)cand_cap * 8);
    uint64_t counts[64];
    int64_t zr[64];
    int rc = ORACLE_ENOMEM;
    if (!zc || !lists || !cand) goto done;
    oracle_zero_counts(p, bits, zc);
    oracle_hot_sets(p, zc, theta, lists, counts);
    uint64_t nh = 0;
    rc = oracle_candidate_hosts(p, lists, counts, max_candidates, cand, cand_cap, &nh, fail_stage,
                                fail_count, NULL);
    if (rc != ORACLE_OK || nh == 0) goto done;
    oracle_zero_totals(p, zc, zr);
    double psi = oracle_bit_set_probability(p, oracle_flow_count(p, zr, NULL));
    int64_t *sz = (int64_t *)malloc((size_t)nh * 8);
    report_row *rows = (report_row *)malloc((size_t)nh * sizeof(report_row));
    if (!sz || !rows) {
        free(sz);
        free(rows);
        rc = ORACLE_ENOMEM;
        goto done;
    }
    oracle_shared_zero_counts(p, bits, cand, (size_t)nh, sz);
    uint64_t kept = 0;
    for (uint64_t t = 0; t < nh; t++) {
        int sat;
        double e = oracle_corrected_estimate(p, sz[t], psi, &sat);
        if (e >= theta) rows[kept++] = (report_row){cand[t], e, sat};
    }
    qsort(rows, (size_t)kept, sizeof(report_row), cmp_report);
    for (uint64_t t = 0; t < kept; t++) {
        hosts_out[t] = rows[t].host;
        est_out[t] = rows[t].est;
        sat_out[t] = (uint8_t)rows[t].sat;
    }
    *n_out = kept;
    free(sz);
    free(rows);
done:
    free(zc);
    free(lists);
    free(cand);
    return rc;
}

/* Union of two sketches with equal parameters.  pkg/src/dhsa/dhla.py:305-318 */
void oracle_merge(uint8_t *dst, const uint8_t *a, const uint8_t *b, size_t nbytes)
{
    for (size_t q = 0; q < nbytes; q++) dst[q] = a[q] | b[q];
}
