/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously correct CPU implementation of throttLL'eM's
 * per-iteration frequency-selection path (arXiv 2408.05235), written from
 * PAPER.md.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  It shares no code, header, table or
 * constant generator with the CUDA path (paper_2408_05235_b200/csrc); it reads
 * the same input BYTES (instance header 48 B, request record 16 B, fp64
 * deadlines, model blob v1) that paper_2408_05235_b200/workload.py writes, and
 * declares its own structs for them.
 *
 * Step numbering O0..O9 follows SURVEY.md §8(c); every step cites the passage it
 * implements.  Readings of ambiguous passages (A-1 .. A-20) are listed in
 * DESIGN.md §3.  No blocking, fusion or reordering: loops run in the paper's
 * order (per instance; per frequency; per future iteration; per tree).
 *
 * Pins: tests/test_oracle_*.py (W1 golden example, SPEC examples, token-by-token
 * brute force, Fraction sums, closed-form ensembles, box-membership tree
 * evaluation, invariants, zero-drift replay, binary-search equivalence).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- input records (byte layout documented in include/tp.h; declared here independently) ---- */
typedef struct {
    int64_t k;        /* current iteration k (unused by the arithmetic; a = k - s_i is given) */
    double t_cur;     /* current time t_cur, seconds (Eq. 4) */
    int32_t req_begin, n_run, n_queue, N, kv_cap, max_batch, tp, pad;
} o_inst;
typedef struct { int32_t a, q, r, flags; } o_req;   /* a = k - s_i, q = |q_i|, r = r^_i */

typedef struct { int32_t feature; float threshold; int32_t left, right; float leaf; } o_node;
typedef struct {
    int32_t n_trees, max_depth;
    float base;
    int32_t* first;   /* first node of each tree in nodes[] */
    int32_t* count;
    o_node* nodes;
} o_model;

enum { O_EMPTY = 1, O_BYPASS_LOST = 2, O_INFEASIBLE = 4, O_KV_OVER = 8, O_QUEUE_BLOCKED = 16,
       O_IPS_CLAMPED = 32, O_BAD_INPUT = 64 };
#define O_LOST 1
#define O_FEAT_LIMIT 16777216LL     /* features must be exact in fp32 (< 2^24) */

/* ============================== model (PAPER §4.3.1) ============================== */

static uint32_t rd32(const unsigned char* p) { uint32_t v; memcpy(&v, p, 4); return v; }

static int check_tree(const o_node* nd, int32_t cnt, int32_t at, int depth, int max_depth, unsigned char* seen) {
    if (at < 0 || at >= cnt || seen[at]) return -1;   /* out of range, cycle or shared child */
    seen[at] = 1;
    if (nd[at].feature == -1) {
        if (!isfinite(nd[at].leaf) || fabsf(nd[at].leaf) > 0x1p60f) return -1;
        return 0;
    }
    if (nd[at].feature < 0 || nd[at].feature > 3 || !isfinite(nd[at].threshold)) return -1;
    if (depth + 1 > max_depth) return -1;
    if (check_tree(nd, cnt, nd[at].left, depth + 1, max_depth, seen)) return -1;
    return check_tree(nd, cnt, nd[at].right, depth + 1, max_depth, seen);
}

/* Parse blob v1 (include/tp.h).  Returns 0 or -4 (malformed). */
int oracle_model_parse(const void* blob, size_t nbytes, o_model** out) {
    const unsigned char* p = (const unsigned char*)blob;
    *out = NULL;
    if (nbytes < 24 || memcmp(p, "TPGB", 4) != 0) return -4;
    if (rd32(p + 4) != 1 || rd32(p + 8) != 4) return -4;
    uint32_t nt = rd32(p + 12), md = rd32(p + 16);
    if (nt > (1u << 20) || md > 12) return -4;
    o_model* m = (o_model*)calloc(1, sizeof(o_model));
    m->n_trees = (int32_t)nt;
    m->max_depth = (int32_t)md;
    memcpy(&m->base, p + 20, 4);
    m->first = (int32_t*)calloc(nt + 1, sizeof(int32_t));
    m->count = (int32_t*)calloc(nt + 1, sizeof(int32_t));
    size_t off = 24, total = 0;
    for (uint32_t t = 0; t < nt; ++t) {               /* first pass: sizes */
        if (off + 4 > nbytes) goto bad;
        uint32_t c = rd32(p + off);
        if (c < 1 || c > (1u << 13) || off + 4 + (size_t)c * 20 > nbytes) goto bad;
        m->first[t] = (int32_t)total;
        m->count[t] = (int32_t)c;
        total += c;
        off += 4 + (size_t)c * 20;
    }
    if (off != nbytes || !isfinite(m->base)) goto bad;
    m->nodes = (o_node*)calloc(total + 1, sizeof(o_node));
    off = 24;
    for (uint32_t t = 0; t < nt; ++t) {
        off += 4;
        for (int32_t i = 0; i < m->count[t]; ++i, off += 20) memcpy(&m->nodes[m->first[t] + i], p + off, 20);
        unsigned char* seen = (unsigned char*)calloc((size_t)m->count[t], 1);
        int rc = check_tree(&m->nodes[m->first[t]], m->count[t], 0, 0, (int)md, seen);
        for (int32_t i = 0; i < m->count[t] && rc == 0; ++i) if (!seen[i]) rc = -1;   /* unreachable node */
        free(seen);
        if (rc) goto bad;
    }
    *out = m;
    return 0;
bad:
    free(m->first); free(m->count); free(m->nodes); free(m);
    return -4;
}

void oracle_model_free(o_model* m) {
    if (!m) return;
    free(m->first); free(m->count); free(m->nodes); free(m);
}

/* Recursive walk: "x[feature] < threshold -> left" (XGBoost convention; reading A-7). */
static float walk(const o_node* nd, int32_t at, const float x[4]) {
    if (nd[at].feature == -1) return nd[at].leaf;
    if (x[nd[at].feature] < nd[at].threshold) return walk(nd, nd[at].left, x);
    return walk(nd, nd[at].right, x);
}

/* M(x) = base + sum_t leaf_t(x), fp32, added one tree at a time in tree order (reading A-7). */
float oracle_predict_raw(const o_model* m, const float x[4]) {
    float acc = m->base;
    for (int32_t t = 0; t < m->n_trees; ++t) {
        float leaf = walk(&m->nodes[m->first[t]], 0, x);
        acc = acc + leaf;
    }
    return acc;
}

/* ============================== per-instance decision ============================== */

/* Eq. 1 at j = k + m - 1, so j - s_i = a + m - 1 (reading A-1):
 *   KV_qi[j] = ceil((j - s_i + |q_i|) / N) for s_i <= j < s_i + r^_i, else 0. */
static int64_t eq1_blocks(int64_t a, int64_t q, int64_t r, int64_t N, int64_t m) {
    int64_t j_minus_s = a + m - 1;
    if (j_minus_s < 0 || j_minus_s >= r) return 0;
    int64_t tokens = j_minus_s + q;
    return (tokens + N - 1) / N;   /* ceil, tokens >= 1 */
}

typedef struct {
    const o_model* m;
    const o_inst* inst;
    const o_req* req;
    const double* t_dead;
    int64_t n_req;
    int32_t H, F;
    const float* freq;
    float tbt;
    /* outputs (any may be NULL) */
    int32_t *B, *KV, *n, *n_adm, *level;
    uint32_t* status;
    float* ips;
    int64_t* tr;
    /* admission = 0: check 1 + batch cap gate (reading A-2); 1: the paper's full admission control
     * (checks 1-3 at f_max, "lost" marking; reading A-23) */
    int admission;
    int adm_limit;        /* admission = 1: at most this many candidates (<= 32) per decision (A-23) */
    uint32_t* adm_lost;   /* out (admission = 1): bit c = queued candidate c admitted as lost */
    int search;           /* 0: exhaustive over all F levels (A-13); 1: the paper's binary search (A-24) */
} o_job;

/* T_R at level u over m = 1..n for the curves (Bv, KVv): O6 + O7.  Returns 1 if a model
 * output was clamped. */
static int level_times(const o_job* J, const o_inst* in, const int64_t* Bv, const int64_t* KVv, int32_t n,
                       int32_t u, float* tcol, int64_t* trv, float* ips_out, int64_t* tr_out) {
    int clamped = 0;
    for (int32_t m = 1; m <= n; ++m) {
        float x[4] = {(float)in->tp, (float)Bv[m], (float)KVv[m], J->freq[u]};
        float acc = oracle_predict_raw(J->m, x);
        float ips = acc;
        if (isnan(acc)) ips = 0x1p-4f;                               /* reading A-8 */
        else if (acc < 0x1p-4f) ips = 0x1p-4f;
        else if (acc > 0x1p17f) ips = 0x1p17f;
        if (isnan(acc) || ips != acc) clamped = 1;
        if (ips_out) ips_out[m - 1] = ips;
        tcol[m] = 1.0f / ips;
    }
    int64_t acc_ticks = 0;
    for (int32_t m = 1; m <= n; ++m) {
        double scaled = (double)tcol[m] * 0x1p40;
        int64_t ticks = (int64_t)scaled;
        if ((double)ticks != scaled) abort();   /* cannot happen for T' in [2^-17, 16] */
        acc_ticks += ticks;
        trv[m] = acc_ticks;
        if (tr_out) tr_out[m - 1] = acc_ticks;
    }
    return clamped;
}

/* O6..O8 at level u for an instance with horizon n and n_adm admitted requests: returns 1 if the
 * TBT check and Eq. 4 for every scheduled request pass; ORs IPS_CLAMPED into *st (reading A-8);
 * writes the level's ips / T_R rows when the caller asked for the grid. */
static int level_passes(const o_job* J, int64_t i, const o_inst* in, const int64_t* Bv, const int64_t* KVv,
                        int32_t n, int32_t n_adm, int32_t u, float* tcol, int64_t* trv, uint32_t* st) {
    const int32_t F = J->F, H = J->H;
    /* O6: T[m] = M(tp, B[m], KV[m], f_u); T'[m] = 1 / T[m] in fp32 (A-9).
     * O7: Eq. 3 T_R[l] = sum_{m<=l} T'[m], exactly (A-10): each T' is an fp32 in
     * [2^-17, 16], hence an integer multiple of 2^-40 s, so the sum is kept in such ticks. */
    if (level_times(J, in, Bv, KVv, n, u, tcol, trv, J->ips ? J->ips + ((int64_t)i * F + u) * H : NULL,
                    J->tr ? J->tr + ((int64_t)i * F + u) * H : NULL))
        *st |= O_IPS_CLAMPED;
    /* O8: TBT check 2: mean(T') = T_R[n] / n must not exceed the SLO (tie passes). */
    long double tr_n = (long double)trv[n];
    int pass = tr_n <= (long double)n * (long double)J->tbt * 0x1p40L;
    /* E2E, Eq. 4: T_R[l] + t_cur < t_dead for every scheduled request, compared
     * as T_R[l] < fl64(t_dead - t_cur) (A-12).  Lost requests are ignored by SLO validation
     * (P:529), but their presence already took the bypass, so none is here. */
    for (int32_t e = 0; pass && e < in->n_run + n_adm; ++e) {
        const o_req* q = &J->req[in->req_begin + e];
        int32_t l = q->r - q->a;
        double slack = J->t_dead[in->req_begin + e] - in->t_cur;
        if (!((long double)trv[l] < (long double)slack * 0x1p40L)) pass = 0;
    }
    return pass;
}

static void decide_one(const o_job* J, int64_t i, int64_t* Bv, int64_t* KVv, float* tcol, int64_t* trv) {
    const o_inst* in = &J->inst[i];
    const int32_t H = J->H, F = J->F;
    uint32_t st = 0;
    int32_t n = 0, n_adm = 0, level = 0;
    uint32_t marked = 0;     /* admission = 1: candidates admitted as "lost" */
    for (int32_t m = 0; m <= H; ++m) Bv[m] = KVv[m] = 0;

    /* ---- O1 validate (reading A-3: every remaining length l in [1, H]) ---- */
    int bad = 0;
    if (in->N < 1 || in->tp < 1 || in->tp >= O_FEAT_LIMIT || in->n_run < 0 || in->n_queue < 0 ||
        in->kv_cap < 0 || in->max_batch < 0 || in->req_begin < 0 ||
        (int64_t)in->req_begin + in->n_run + in->n_queue > J->n_req)
        bad = 1;
    int64_t footprint = 0;
    for (int64_t e = 0; !bad && e < (int64_t)in->n_run + in->n_queue; ++e) {
        const o_req* q = &J->req[in->req_begin + e];
        int64_t l = (int64_t)q->r - q->a;
        if (q->a < 0 || q->q < 1 || q->r < 1 || q->a >= O_FEAT_LIMIT || q->q >= O_FEAT_LIMIT || l < 1 || l > H) bad = 1;
        if (e >= in->n_run && q->a != 0) bad = 1;     /* queued: virtual append at s_a = k */
        if (!bad) footprint += eq1_blocks(q->a, q->q, q->r, in->N, l);   /* last in-window block count */
    }
    if (!bad && footprint >= O_FEAT_LIMIT) bad = 1;   /* KV must stay exact as an fp32 feature */
    if (bad) {
        st = O_BAD_INPUT; level = F - 1;
        goto write;
    }

    /* ---- O2/O3 running totals, Eq. 2: B[m] = #active, KV[m] = sum_i KV_qi ---- */
    for (int32_t m = 1; m <= H; ++m) {
        for (int32_t e = 0; e < in->n_run; ++e) {
            const o_req* q = &J->req[in->req_begin + e];
            int64_t b = eq1_blocks(q->a, q->q, q->r, in->N, m);
            if (b > 0) { Bv[m] += 1; KVv[m] += b; }
        }
    }
    for (int32_t m = 1; m <= H; ++m) if (KVv[m] > in->kv_cap) st |= O_KV_OVER;

    /* ---- O4 FIFO gate: check 1 + batch cap, one at a time, FIFO head-of-line ---- */
    int32_t n_cur = 0;       /* horizon of the scheduled set so far */
    for (int32_t e = 0; e < in->n_run; ++e) {
        const o_req* q = &J->req[in->req_begin + e];
        if (q->r - q->a > n_cur) n_cur = q->r - q->a;
    }
    for (int32_t c = 0; c < in->n_queue; ++c) {
        const o_req* q = &J->req[in->req_begin + in->n_run + c];
        if (J->admission && c >= J->adm_limit) { st |= O_QUEUE_BLOCKED; break; }   /* reading A-23 */
        int ok = (Bv[1] + 1 <= in->max_batch);
        for (int32_t m = 1; ok && m <= H; ++m)      /* virtual append at s = k */
            if (KVv[m] + eq1_blocks(0, q->q, q->r, in->N, m) > in->kv_cap) ok = 0;
        if (!ok) { st |= O_QUEUE_BLOCKED; break; }
        int as_lost = 0;
        if (J->admission) {
            /* checks 2-3 at the maximum frequency on the virtual state */
            for (int32_t m = 1; m <= H; ++m) {      /* the candidate's curves added virtually */
                int64_t b = eq1_blocks(0, q->q, q->r, in->N, m);
                Bv[m] += b > 0; KVv[m] += b;
            }
            int32_t nv = q->r > n_cur ? q->r : n_cur;
            level_times(J, in, Bv, KVv, nv, F - 1, tcol, trv, NULL, NULL);
            int tbt_ok = (long double)trv[nv] <= (long double)nv * (long double)J->tbt * 0x1p40L;
            int others_fail = 0, self_fail = 0;
            for (int32_t e = 0; e <= in->n_run + c; ++e) {
                const o_req* r = &J->req[in->req_begin + e];
                int is_self = e == in->n_run + c;
                int lost_e = (r->flags & O_LOST) || (e >= in->n_run && !is_self && ((marked >> (e - in->n_run)) & 1));
                if (lost_e) continue;               /* lost requests are ignored */
                int32_t l = r->r - r->a;
                double slack = J->t_dead[in->req_begin + e] - in->t_cur;
                int fails = !((long double)trv[l] < (long double)slack * 0x1p40L);
                if (fails) { if (is_self) self_fail = 1; else others_fail = 1; }
            }
            for (int32_t m = 1; m <= H; ++m) {      /* roll back */
                int64_t b = eq1_blocks(0, q->q, q->r, in->N, m);
                Bv[m] -= b > 0; KVv[m] -= b;
            }
            if (!tbt_ok || others_fail) { st |= O_QUEUE_BLOCKED; break; }
            as_lost = self_fail;                    /* schedulable, but its own deadline fails */
        }
        for (int32_t m = 1; m <= H; ++m) {          /* commit */
            int64_t b = eq1_blocks(0, q->q, q->r, in->N, m);
            if (b > 0) { Bv[m] += 1; KVv[m] += b; }
        }
        if (as_lost) marked |= 1u << c;
        if (q->r > n_cur) n_cur = q->r;
        n_adm++;
    }

    /* ---- O5 horizon and early exits ---- */
    int lost = 0;
    for (int32_t e = 0; e < in->n_run + n_adm; ++e) {
        const o_req* q = &J->req[in->req_begin + e];
        int32_t l = q->r - q->a;     /* completes at s_i + r^_i, i.e. l = s_i + r^_i - k */
        if (l > n) n = l;
        if (q->flags & O_LOST) lost = 1;
        if (e >= in->n_run && ((marked >> (e - in->n_run)) & 1)) lost = 1;
    }
    if (n == 0) { st |= O_EMPTY; level = 0; goto write; }                 /* reading A-15 */
    if (lost) { st |= O_BYPASS_LOST; level = F - 1; goto write; }

    /* ---- O6..O9: lowest SLO-meeting level ---- */
    if (J->search == 0) {
        /* exhaustive (reading A-13): every level, ascending; the answer is the lowest passing one */
        level = -1;
        for (int32_t u = 0; u < F; ++u)
            if (level_passes(J, i, in, Bv, KVv, n, n_adm, u, tcol, trv, &st) && level < 0) level = u;
        if (level < 0) { level = F - 1; st |= O_INFEASIBLE; }               /* reading A-14 */
    } else {
        /* the paper's binary search over the frequency range (reading A-24): the maximum
         * level must pass (the scheduler's guarantee), then lo/hi with pass(hi) invariant */
        if (!level_passes(J, i, in, Bv, KVv, n, n_adm, F - 1, tcol, trv, &st)) {
            level = F - 1; st |= O_INFEASIBLE;
        } else {
            int32_t lo = 0, hi = F - 1;
            while (lo < hi) {
                int32_t mid = (lo + hi) / 2;
                if (level_passes(J, i, in, Bv, KVv, n, n_adm, mid, tcol, trv, &st)) hi = mid;
                else lo = mid + 1;
            }
            level = lo;
        }
    }

write:
    if (J->B) for (int32_t m = 1; m <= H; ++m) J->B[(int64_t)i * H + m - 1] = (int32_t)Bv[m];
    if (J->KV) for (int32_t m = 1; m <= H; ++m) J->KV[(int64_t)i * H + m - 1] = (int32_t)KVv[m];
    if (J->n) J->n[i] = n;
    if (J->n_adm) J->n_adm[i] = n_adm;
    if (J->level) J->level[i] = level;
    if (J->status) J->status[i] = st;
    if (J->adm_lost) J->adm_lost[i] = marked;
}

typedef struct { const o_job* J; int64_t lo, hi, stride; } o_slice;

static void* worker(void* arg) {
    const o_slice* s = (const o_slice*)arg;
    int32_t H = s->J->H;
    int64_t* Bv = (int64_t*)malloc(sizeof(int64_t) * (H + 1));
    int64_t* KVv = (int64_t*)malloc(sizeof(int64_t) * (H + 1));
    float* tcol = (float*)malloc(sizeof(float) * (H + 1));
    int64_t* trv = (int64_t*)malloc(sizeof(int64_t) * (H + 1));
    for (int64_t i = s->lo; i < s->hi; i += s->stride) decide_one(s->J, i, Bv, KVv, tcol, trv);
    free(Bv); free(KVv); free(tcol); free(trv);
    return NULL;
}

/* Decide every instance.  Instances are independent, so threads take interleaved instances.
 * Returns 0, or -1 for arguments the path defines as invalid (include/tp.h conventions). */
int oracle_decide(const o_model* m, const o_inst* inst, int64_t n_inst, const o_req* req, int64_t n_req,
                  const double* t_dead, int32_t H, const float* freq, int32_t F, float tbt,
                  int32_t* B, int32_t* KV, int32_t* n, int32_t* n_adm, float* ips, int64_t* tr,
                  int32_t* level, uint32_t* status, int n_threads, int admission, uint32_t* adm_lost,
                  int adm_limit, int search) {
    if (!m || H < 1 || H > 16384 || F < 1 || F > 32 || n_inst < 0) return -1;
    if (!(tbt >= 0x1p-17f && tbt <= 16.0f)) return -1;
    for (int32_t u = 0; u < F; ++u) {
        if (!isfinite(freq[u]) || freq[u] <= 0.0f) return -1;
        if (u > 0 && !(freq[u] > freq[u - 1])) return -1;
    }
    if (adm_limit < 1 || adm_limit > 32) adm_limit = 32;
    if (search != 0 && search != 1) return -1;
    o_job J = {m, inst, req, t_dead, n_req, H, F, freq, tbt, B, KV, n, n_adm, level, status, ips, tr,
               admission, adm_limit, adm_lost, search};
    if (n_threads < 1) n_threads = 1;
    if (n_threads > 256) n_threads = 256;
    if (n_threads == 1) {
        o_slice s = {&J, 0, n_inst, 1};
        worker(&s);
        return 0;
    }
    pthread_t th[256];
    o_slice sl[256];
    for (int t = 0; t < n_threads; ++t) {
        sl[t].J = &J; sl[t].lo = t; sl[t].hi = n_inst; sl[t].stride = n_threads;
        pthread_create(&th[t], NULL, worker, &sl[t]);
    }
    for (int t = 0; t < n_threads; ++t) pthread_join(th[t], NULL);
    return 0;
}
