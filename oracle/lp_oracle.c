/*
 * oracle/lp_oracle.c -- CPU ORACLE.  TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, single-threaded C that computes what the B200 path computes, written
 * from the paper's definitions.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load it.  It shares no code with
 * paper_2009_10247_b200/ (the product) and the product never calls it.
 *
 * Citations: PAPER.md line numbers (the LaTeX source of arXiv 2009.10247).
 *
 * Input program (same flat layout as lpgen.Rules / include/lp.h lp_rules):
 *   n atoms 0..n-1; R rules; rule r has head head[r] and body literals
 *   atom[ptr[r] .. ptr[r+1]-1]; neg[j] = 1 marks a negative literal "not atom[j]"
 *   (normal programs only).  A rule with an empty body is a fact.
 *
 * Conventions:
 *   - I_0 = v0 ∪ facts(P).  I_{k+1} = I_k ∪ T_P(I_k) with T_P over the ORIGINAL rules
 *     (PAPER.md:70-72).  k* = least k with I_{k+1} = I_k.  iters = k*+1 = the number of
 *     T_P evaluations Algorithm 1 performs (one at PAPER.md:165 plus k* in the loop at
 *     PAPER.md:167-169) -- convention (B).
 *   - Normal programs: positive form P+ (Eq. 4) with the negated atoms
 *     a_0 < a_1 < ... < a_{k-1} mapped to fresh atoms n+j (abar_j).  A guess fixes the
 *     abar values; column g of the initial matrix (Def. 8) is
 *     facts(P) ∪ {abar_j : guess bit j = 1}.  The column is iterated by T_{P+}
 *     (abar atoms have no rules -- their rows are the self-loops of Def. 7)
 *     to its fixpoint and accepted iff every pair (a_j, abar_j) sums to exactly 1
 *     (Algorithm 3, read as in DESIGN.md reading R7).
 */
#define _POSIX_C_SOURCE 199309L
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define ORC_OK 0
#define ORC_E_NOMEM 1
#define ORC_E_ARG 2

/* ---------------------------------------------------------------------------------
 * O-LM: the definition, literally.  Jacobi iteration of the immediate-consequence
 * operator over the original rules, inflationary, from I_0.
 *   v0        : optional uint8[n] start set (NULL = empty)
 *   model     : out uint8[n] (1 = atom in the least model)
 *   popcounts : optional out int32[cap]: |I_0|, |I_1|, ..., |I_k*|
 *   max_iters : 0 = run to the fixpoint; else stop after that many T_P evaluations
 *               (bounded CPU sample for bench.py; *converged_out says which)
 * ------------------------------------------------------------------------------- */
int orc_lm_jacobi(int32_t n, int64_t R, const int32_t *head, const int64_t *ptr,
                  const int32_t *atom, const uint8_t *v0, uint8_t *model,
                  int32_t *popcounts, int32_t cap, int32_t max_iters,
                  int32_t *iters_out, int32_t *converged_out)
{
    uint8_t *I = (uint8_t *)calloc((size_t)n + 1, 1);
    uint8_t *J = (uint8_t *)calloc((size_t)n + 1, 1);
    if (!I || !J) { free(I); free(J); return ORC_E_NOMEM; }
    if (v0) memcpy(I, v0, (size_t)n);
    for (int64_t r = 0; r < R; ++r)              /* facts: body(r) = ∅ */
        if (ptr[r] == ptr[r + 1]) I[head[r]] = 1;

    int64_t pop = 0;
    for (int32_t a = 0; a < n; ++a) pop += I[a];
    if (popcounts && cap > 0) popcounts[0] = (int32_t)pop;

    int32_t evals = 0, converged = 0;
    for (;;) {
        /* J = I ∪ T_P(I):  T_P(I) = { h | h <- b1..bm in P, {b1..bm} ⊆ I } */
        memcpy(J, I, (size_t)n);
        for (int64_t r = 0; r < R; ++r) {
            int all = 1;
            for (int64_t j = ptr[r]; j < ptr[r + 1]; ++j)
                if (!I[atom[j]]) { all = 0; break; }
            if (all) J[head[r]] = 1;
        }
        ++evals;
        if (memcmp(I, J, (size_t)n) == 0) { converged = 1; break; }   /* u = v */
        uint8_t *t = I; I = J; J = t;
        pop = 0;
        for (int32_t a = 0; a < n; ++a) pop += I[a];
        if (popcounts && evals < cap) popcounts[evals] = (int32_t)pop;
        if (max_iters > 0 && evals >= max_iters) break;
    }
    memcpy(model, I, (size_t)n);
    *iters_out = evals;
    if (converged_out) *converged_out = converged;
    free(I); free(J);
    return ORC_OK;
}

/* ---------------------------------------------------------------------------------
 * O-STAGE: level-synchronous forward chaining with per-rule counters (the same
 * least model and the same stage of every atom).  Used where the
 * Jacobi loop is too slow (C3/C4, and per guess for C5).
 *   stage : out int32[n]; 0 for I_0, k for atoms first in I_k, -1 if not in the model.
 *   iters : k* + 1 with k* = max stage (0 if the model is empty).
 * ------------------------------------------------------------------------------- */
static int stage_core(int32_t n, int64_t R, const int32_t *head, const int64_t *ptr,
                      const int32_t *atom, const uint8_t *v0, int32_t *stage,
                      int32_t *iters_out, const int64_t *occ_ptr, const int64_t *occ_rule,
                      int64_t *cnt, int32_t *queue)
{
    int64_t qh = 0, qt = 0;
    for (int32_t a = 0; a < n; ++a) stage[a] = -1;
    if (v0)
        for (int32_t a = 0; a < n; ++a)
            if (v0[a]) { stage[a] = 0; queue[qt++] = a; }
    for (int64_t r = 0; r < R; ++r) {
        cnt[r] = ptr[r + 1] - ptr[r];
        if (cnt[r] == 0 && stage[head[r]] < 0) { stage[head[r]] = 0; queue[qt++] = head[r]; }
    }
    int32_t kmax = 0;
    while (qh < qt) {                       /* FIFO = non-decreasing stage order */
        int32_t a = queue[qh++];
        int32_t s = stage[a];
        for (int64_t o = occ_ptr[a]; o < occ_ptr[a + 1]; ++o) {
            int64_t r = occ_rule[o];
            if (--cnt[r] == 0) {             /* body(r) ⊆ I_s: head(r) ∈ I_{s+1} */
                int32_t h = head[r];
                if (stage[h] < 0) {
                    stage[h] = s + 1;
                    if (s + 1 > kmax) kmax = s + 1;
                    queue[qt++] = h;
                }
            }
        }
    }
    *iters_out = kmax + 1;
    return ORC_OK;
}

/* occurrence lists: for every atom a, the rules whose body contains a (one entry per
 * body position, so duplicate body atoms decrement the counter once per position). */
static int build_occ(int32_t n, int64_t R, const int64_t *ptr, const int32_t *atom,
                     int64_t **occ_ptr_out, int64_t **occ_rule_out)
{
    int64_t nnz = ptr[R];
    int64_t *op = (int64_t *)calloc((size_t)n + 2, sizeof(int64_t));
    int64_t *orr = (int64_t *)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(int64_t));
    if (!op || !orr) { free(op); free(orr); return ORC_E_NOMEM; }
    for (int64_t j = 0; j < nnz; ++j) op[atom[j] + 1]++;
    for (int32_t a = 0; a < n; ++a) op[a + 1] += op[a];
    int64_t *fill = (int64_t *)malloc(((size_t)n + 1) * sizeof(int64_t));
    if (!fill) { free(op); free(orr); return ORC_E_NOMEM; }
    memcpy(fill, op, ((size_t)n + 1) * sizeof(int64_t));
    for (int64_t r = 0; r < R; ++r)
        for (int64_t j = ptr[r]; j < ptr[r + 1]; ++j) orr[fill[atom[j]]++] = r;
    free(fill);
    *occ_ptr_out = op; *occ_rule_out = orr;
    return ORC_OK;
}

int orc_lm_stage(int32_t n, int64_t R, const int32_t *head, const int64_t *ptr,
                 const int32_t *atom, const uint8_t *v0, int32_t *stage, int32_t *iters_out)
{
    int64_t *op = NULL, *orr = NULL;
    if (build_occ(n, R, ptr, atom, &op, &orr)) return ORC_E_NOMEM;
    int64_t *cnt = (int64_t *)malloc((size_t)(R > 0 ? R : 1) * sizeof(int64_t));
    int32_t *queue = (int32_t *)malloc(((size_t)n + 1) * sizeof(int32_t));
    int rc = ORC_E_NOMEM;
    if (cnt && queue)
        rc = stage_core(n, R, head, ptr, atom, v0, stage, iters_out, op, orr, cnt, queue);
    free(op); free(orr); free(cnt); free(queue);
    return rc;
}

/* Timing entry for bench.py's cpu_baseline (BASELINE.md "CPU-baseline plan"): the
 * occurrence lists are built once (ingest, untimed), then the fixpoint phase --
 * stage_core, unchanged -- runs `trials` times, each timed with CLOCK_MONOTONIC into
 * secs[t].  The caller pins the thread (single core).  Results as orc_lm_stage. */
int orc_lm_stage_timed(int32_t n, int64_t R, const int32_t *head, const int64_t *ptr,
                       const int32_t *atom, const uint8_t *v0, int32_t *stage,
                       int32_t *iters_out, int32_t trials, double *secs)
{
    int64_t *op = NULL, *orr = NULL;
    if (build_occ(n, R, ptr, atom, &op, &orr)) return ORC_E_NOMEM;
    int64_t *cnt = (int64_t *)malloc((size_t)(R > 0 ? R : 1) * sizeof(int64_t));
    int32_t *queue = (int32_t *)malloc(((size_t)n + 1) * sizeof(int32_t));
    int rc = ORC_E_NOMEM;
    if (cnt && queue) {
        for (int32_t t = 0; t < trials; ++t) {
            struct timespec t0, t1;
            clock_gettime(CLOCK_MONOTONIC, &t0);
            rc = stage_core(n, R, head, ptr, atom, v0, stage, iters_out, op, orr, cnt, queue);
            clock_gettime(CLOCK_MONOTONIC, &t1);
            secs[t] = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
            if (rc) break;
        }
    }
    free(op); free(orr); free(cnt); free(queue);
    return rc;
}

/* ---------------------------------------------------------------------------------
 * O-STABLE: Algorithms 2-3 per guess column, via P+ (Eq. 4).
 *   neg        : uint8[nnz] literal polarity (NULL = definite program, k = 0)
 *   G          : number of guesses
 *   guess      : uint8[G][k] abar values (1 = a_j assumed false), or NULL to enumerate
 *                all 2^f assignments of the FREE negated atoms in binary counting order
 *                (bit i of g = abar of the i-th free negated atom); the abar row of a
 *                negated atom that is a fact is forced 0 (Def. 8 item 3).
 *                With guess == NULL the caller passes G = 2^f (checked).
 *   accepted   : out uint8[G]
 *   kstar      : out int32[G]  (k*_g: the column's fixpoint step, max stage)
 *   models     : optional out uint64[G][ceil(n/64)] -- the column's fixpoint restricted
 *                to original atoms, LSB-first bits (atom a: word a>>6, bit a&63)
 *   passes_out : max_g k*_g + 1 = the number of whole-matrix products Algorithm 2
 *                performs
 *   k_out, f_out : number of negated atoms / free negated atoms
 * ------------------------------------------------------------------------------- */
int orc_stable(int32_t n, int64_t R, const int32_t *head, const int64_t *ptr,
               const int32_t *atom, const uint8_t *neg, int64_t G, const uint8_t *guess,
               uint8_t *accepted, int32_t *kstar, uint64_t *models,
               int32_t *passes_out, int32_t *k_out, int32_t *f_out)
{
    int64_t nnz = ptr[R];
    int rc = ORC_E_NOMEM;
    int32_t *na = NULL, *freej = NULL, *patom = NULL, *queue = NULL, *stage = NULL;
    int64_t *op = NULL, *orr = NULL, *cnt = NULL;
    uint8_t *v0 = NULL, *bar = NULL;
    /* negated atoms, ascending */
    uint8_t *isneg = (uint8_t *)calloc((size_t)n + 1, 1);
    uint8_t *isfact = (uint8_t *)calloc((size_t)n + 1, 1);
    int32_t *jof = (int32_t *)malloc(((size_t)n + 1) * sizeof(int32_t));
    if (!isneg || !isfact || !jof) goto done;
    if (neg)
        for (int64_t j = 0; j < nnz; ++j) if (neg[j]) isneg[atom[j]] = 1;
    for (int64_t r = 0; r < R; ++r) if (ptr[r] == ptr[r + 1]) isfact[head[r]] = 1;
    int32_t k = 0, f = 0;
    for (int32_t a = 0; a < n; ++a) { jof[a] = isneg[a] ? k++ : -1; }
    na = (int32_t *)malloc(((size_t)k + 1) * sizeof(int32_t));
    freej = (int32_t *)malloc(((size_t)k + 1) * sizeof(int32_t));
    if (!na || !freej) goto done;
    for (int32_t a = 0; a < n; ++a)
        if (isneg[a]) { na[jof[a]] = a; if (!isfact[a]) freej[f++] = jof[a]; }
    *k_out = k; *f_out = f;
    if (!guess && G != ((int64_t)1 << f)) { rc = ORC_E_ARG; goto done; }

    /* positive form P+: atoms 0..n-1 original, n+j = abar_j */
    int32_t np = n + k;
    patom = (int32_t *)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(int32_t));
    if (!patom) goto done;
    for (int64_t j = 0; j < nnz; ++j)
        patom[j] = (neg && neg[j]) ? n + jof[atom[j]] : atom[j];

    if (build_occ(np, R, ptr, patom, &op, &orr)) goto done;
    cnt = (int64_t *)malloc((size_t)(R > 0 ? R : 1) * sizeof(int64_t));
    queue = (int32_t *)malloc(((size_t)np + 1) * sizeof(int32_t));
    stage = (int32_t *)malloc(((size_t)np + 1) * sizeof(int32_t));
    v0 = (uint8_t *)calloc((size_t)np + 1, 1);
    bar = (uint8_t *)calloc((size_t)k + 1, 1);
    if (!cnt || !queue || !stage || !v0 || !bar) goto done;
    int64_t words = ((int64_t)n + 63) / 64;
    int32_t kmax_all = 0;

    for (int64_t g = 0; g < G; ++g) {
        /* initial-matrix column g (Def. 8): facts are added by stage_core; abar rows */
        for (int32_t j = 0; j < k; ++j) bar[j] = 0;
        if (guess) {
            for (int32_t j = 0; j < k; ++j) bar[j] = guess[g * k + j] ? 1 : 0;
        } else {
            for (int32_t i = 0; i < f; ++i) bar[freej[i]] = (uint8_t)((g >> i) & 1);
        }
        memset(v0, 0, (size_t)np);
        for (int32_t j = 0; j < k; ++j) v0[n + j] = bar[j];
        int32_t it = 0;
        stage_core(np, R, head, ptr, patom, v0, stage, &it, op, orr, cnt, queue);
        kstar[g] = it - 1;
        if (it - 1 > kmax_all) kmax_all = it - 1;
        /* Algorithm 3: accept iff a_l + abar_j = 1 for every negated atom */
        int ok = 1;
        for (int32_t j = 0; j < k; ++j) {
            int in_lm = stage[na[j]] >= 0;
            if (in_lm + (int)bar[j] != 1) { ok = 0; break; }
        }
        accepted[g] = (uint8_t)ok;
        if (models) {
            uint64_t *m = models + g * words;
            for (int64_t w = 0; w < words; ++w) m[w] = 0;
            for (int32_t a = 0; a < n; ++a)
                if (stage[a] >= 0) m[a >> 6] |= (uint64_t)1 << (a & 63);
        }
    }
    *passes_out = G > 0 ? kmax_all + 1 : 0;
    rc = ORC_OK;
done:
    free(isneg); free(isfact); free(jof); free(na); free(freej); free(patom);
    free(op); free(orr); free(cnt); free(queue); free(stage); free(v0); free(bar);
    return rc;
}

/* ---------------------------------------------------------------------------------
 * O-CERT: linear-time certificate check of a claimed (model M, stage s, iters) for a
 * definite program from start set I_0 = v0 ∪ facts (SURVEY.md §8(c) O-CERT):
 *   1. I_0 ⊆ M with s = 0 on I_0; s = -1 exactly off M;
 *   2. closure: no rule with body ⊆ M and head ∉ M  (=> LM ⊆ M);
 *   3. exactness: for a ∈ M \ I_0, s(a) = 1 + min over rules r with head a and
 *      body ⊆ M of max_{b ∈ body(r)} s(b)  (=> M ⊆ LM by induction on s, and s is the
 *      Jacobi stage, so the pass count is exact);
 *   4. iters = max s + 1.
 * Returns 0 if valid, else the number (1..4) of the first failed condition.
 * ------------------------------------------------------------------------------- */
int orc_certify(int32_t n, int64_t R, const int32_t *head, const int64_t *ptr,
                const int32_t *atom, const uint8_t *v0, const uint8_t *model,
                const int32_t *stage, int32_t iters)
{
    uint8_t *i0 = (uint8_t *)calloc((size_t)n + 1, 1);
    int32_t *best = (int32_t *)malloc(((size_t)n + 1) * sizeof(int32_t));
    if (!i0 || !best) { free(i0); free(best); return -1; }
    if (v0) for (int32_t a = 0; a < n; ++a) i0[a] = v0[a] ? 1 : 0;
    for (int64_t r = 0; r < R; ++r) if (ptr[r] == ptr[r + 1]) i0[head[r]] = 1;
    int rc = 0;
    for (int32_t a = 0; a < n && !rc; ++a) {
        if (i0[a] && (!model[a] || stage[a] != 0)) rc = 1;
        if (!model[a] && stage[a] != -1) rc = 1;
        if (model[a] && stage[a] < 0) rc = 1;
    }
    for (int32_t a = 0; a < n; ++a) best[a] = INT32_MAX;
    for (int64_t r = 0; r < R && !rc; ++r) {
        int in = 1; int32_t mx = -1;
        for (int64_t j = ptr[r]; j < ptr[r + 1]; ++j) {
            if (!model[atom[j]]) { in = 0; break; }
            if (stage[atom[j]] > mx) mx = stage[atom[j]];
        }
        if (!in) continue;
        if (!model[head[r]]) rc = 2;
        else if (mx + 1 < best[head[r]]) best[head[r]] = mx + 1;
    }
    int32_t smax = 0;
    for (int32_t a = 0; a < n && !rc; ++a) {
        if (!model[a]) continue;
        if (stage[a] > smax) smax = stage[a];
        if (i0[a]) continue;
        if (best[a] == INT32_MAX || stage[a] != best[a]) rc = 3;
    }
    if (!rc && iters != smax + 1) rc = 4;
    free(i0); free(best);
    return rc;
}
