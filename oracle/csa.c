/*
 * oracle/csa.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * Plain serial Connection-Scan Algorithm (CSA) for the earliest-arrival-time
 * (EAT) problem, written from the paper:
 *
 *   Haryan, Ramakrishna, Nasre, Reddy, "GPU Algorithm for Earliest Arrival
 *   Time Problem in Public Transport Networks", arXiv 1912.00966.
 *   PAPER.md:96-118 (Sec. I-A Preliminaries, Algorithm 1 "Connection-Scan").
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this file.  It shares no code, header,
 * table or helper with the CUDA path (paper_1912_00966_b200/csrc/); the two
 * meet only at plain arrays produced by the seeded generator (synth/).
 *
 * What it computes: e[v] = the minimum of t_k + lambda_k
 * over all time-respecting connection sequences (s=v0,v1,t1,l1), ...,
 * (v_{k-1},v,t_k,l_k) with t_1 >= t_s and t_{i+1} >= t_i + l_i; e[s] = t_s;
 * e[v] = INF when no such sequence exists.
 *
 * Algorithm 1 as printed, with ONE reading (reading R1, SURVEY
 * 8(c) #1): connections with equal departure time t form a group; inside a
 * group the lambda = 0 members are relaxed repeatedly until none improves
 * (a closure at one instant), then the lambda > 0 members are relaxed once.
 * With all lambda > 0 this is exactly Algorithm 1: a
 * lambda > 0 member arrives at t + lambda > t and so cannot enable any other
 * member departing at t.
 *
 * Relax test (Algorithm 3):
 *     if (e[u] <= t && t + lambda < e[v]) e[v] = t + lambda;
 *
 * Integer model (reading R2): times are uint32 seconds, INF = 0x7FFFFFFF;
 * callers guarantee dep + dur < INF.
 *
 * Sort: stable LSD radix sort on dep (two 16-bit passes), so equal
 * departures keep input order (SPEC ties "stable by input order").
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_INF 0x7FFFFFFFu

/* one connection, 16 bytes: departure-sorted array of these is "C" in Alg. 1 */
typedef struct {
    uint32_t u, v, dep, arr; /* arr = dep + lambda */
} oracle_conn;

typedef struct {
    uint32_t n;        /* |V| */
    uint64_t m;        /* |C| */
    oracle_conn *c;    /* C sorted by departure, stable */
    uint64_t *orig;    /* orig[i] = input index of c[i] (for parent witnesses) */
} oracle_tt;

/* Stable sort of connection indices by departure time (LSD radix, 2x16 bit). */
static int sort_by_departure(uint64_t m, const uint32_t *dep, uint64_t *out)
{
    uint64_t *tmp = (uint64_t *)malloc((m ? m : 1) * sizeof(uint64_t));
    uint64_t *cnt = (uint64_t *)malloc(65537 * sizeof(uint64_t));
    if (!tmp || !cnt) { free(tmp); free(cnt); return -1; }
    for (uint64_t i = 0; i < m; ++i) tmp[i] = i;
    for (int pass = 0; pass < 2; ++pass) {
        int shift = 16 * pass;
        uint64_t *src = pass == 0 ? tmp : out;
        uint64_t *dst = pass == 0 ? out : tmp;
        memset(cnt, 0, 65537 * sizeof(uint64_t));
        for (uint64_t i = 0; i < m; ++i) cnt[((dep[src[i]] >> shift) & 0xFFFFu) + 1]++;
        for (int b = 0; b < 65536; ++b) cnt[b + 1] += cnt[b];
        for (uint64_t i = 0; i < m; ++i) dst[cnt[(dep[src[i]] >> shift) & 0xFFFFu]++] = src[i];
    }
    memcpy(out, tmp, m * sizeof(uint64_t));
    free(tmp);
    free(cnt);
    return 0;
}

/* Build the departure-sorted connection array C (the input of Alg. 1,
 * "arranged in non-decreasing order based on their departure
 * time").  Returns NULL on allocation failure. */
void *oracle_prepare(uint32_t n, uint64_t m, const uint32_t *u, const uint32_t *v,
                     const uint32_t *dep, const uint32_t *dur)
{
    oracle_tt *tt = (oracle_tt *)calloc(1, sizeof(oracle_tt));
    if (!tt) return NULL;
    tt->n = n;
    tt->m = m;
    tt->c = (oracle_conn *)malloc((m ? m : 1) * sizeof(oracle_conn));
    tt->orig = (uint64_t *)malloc((m ? m : 1) * sizeof(uint64_t));
    if (!tt->c || !tt->orig || sort_by_departure(m, dep, tt->orig) != 0) {
        free(tt->c); free(tt->orig); free(tt);
        return NULL;
    }
    for (uint64_t i = 0; i < m; ++i) {
        uint64_t k = tt->orig[i];
        tt->c[i].u = u[k];
        tt->c[i].v = v[k];
        tt->c[i].dep = dep[k];
        tt->c[i].arr = dep[k] + dur[k];
    }
    return tt;
}

void oracle_free(void *p)
{
    oracle_tt *tt = (oracle_tt *)p;
    if (!tt) return;
    free(tt->c);
    free(tt->orig);
    free(tt);
}

/* First index i with c[i].dep >= t (connections departing earlier can never
 * pass the test e[u] <= t, because every finite e[u] >= t_s). */
static uint64_t first_departing_at_or_after(const oracle_tt *tt, uint32_t t)
{
    uint64_t lo = 0, hi = tt->m;
    while (lo < hi) {
        uint64_t mid = lo + (hi - lo) / 2;
        if (tt->c[mid].dep < t) lo = mid + 1; else hi = mid;
    }
    return lo;
}

/* Algorithm 3 Relax: returns 1 when e[v] was lowered. */
static int relax(uint32_t *e, int64_t *parent, const oracle_conn *c, uint64_t orig)
{
    if (e[c->u] <= c->dep && c->arr < e[c->v]) {
        e[c->v] = c->arr;
        if (parent) parent[c->v] = (int64_t)orig;
        return 1;
    }
    return 0;
}

/* One query (s, t_s).  e[] has n entries; parent[] (optional, may be NULL)
 * receives, for each v with finite e[v] != t_s-at-source, the input index of
 * the connection that set e[v] last (-1 otherwise).
 * Returns 0, or -1 if s >= n or t_s >= INF. */
int oracle_csa_query(const void *p, uint32_t s, uint32_t t_s, uint32_t *e, int64_t *parent)
{
    const oracle_tt *tt = (const oracle_tt *)p;
    if (s >= tt->n || t_s >= ORACLE_INF) return -1;
    /* Initialize (Alg. 1 lines 1-4, Alg. 2). */
    for (uint32_t x = 0; x < tt->n; ++x) e[x] = ORACLE_INF;
    if (parent) for (uint32_t x = 0; x < tt->n; ++x) parent[x] = -1;
    e[s] = t_s;
    /* Scan (Alg. 1 lines 5-9), grouped by equal departure time (reading R1). */
    uint64_t i = first_departing_at_or_after(tt, t_s);
    while (i < tt->m) {
        uint32_t t = tt->c[i].dep;
        uint64_t j = i;
        while (j < tt->m && tt->c[j].dep == t) ++j;
        /* (a) lambda = 0 members: closure at instant t */
        int changed = 1;
        while (changed) {
            changed = 0;
            for (uint64_t k = i; k < j; ++k)
                if (tt->c[k].arr == t && relax(e, parent, &tt->c[k], tt->orig[k])) changed = 1;
        }
        /* (b) lambda > 0 members: once, in order */
        for (uint64_t k = i; k < j; ++k)
            if (tt->c[k].arr != t) relax(e, parent, &tt->c[k], tt->orig[k]);
        i = j;
    }
    return 0;
}

/* Many queries on one prepared timetable; out is row-major nq x n. */
int oracle_csa_many(const void *p, const uint32_t *src, const uint32_t *ts, uint64_t nq, uint32_t *out)
{
    const oracle_tt *tt = (const oracle_tt *)p;
    for (uint64_t q = 0; q < nq; ++q)
        if (oracle_csa_query(p, src[q], ts[q], out + q * (uint64_t)tt->n, NULL) != 0) return -1;
    return 0;
}

/* One-shot convenience: prepare + query + free. */
int oracle_csa(uint32_t n, uint64_t m, const uint32_t *u, const uint32_t *v, const uint32_t *dep,
               const uint32_t *dur, uint32_t s, uint32_t t_s, uint32_t *e, int64_t *parent)
{
    void *tt = oracle_prepare(n, m, u, v, dep, dur);
    if (!tt) return -2;
    int rc = oracle_csa_query(tt, s, t_s, e, parent);
    oracle_free(tt);
    return rc;
}
