/*
 * lp.h -- C ABI of the B200 (sm_100a) least-model / stable-model engine
 * (paper_2009_10247_b200/liblp_b200.so).
 *
 * The method (arXiv 2009.10247, PAPER.md = its LaTeX source):
 *   - least model of a definite program = fixpoint of the immediate-consequence
 *     operator T_P iterated from the initial vector, computed as the thresholded
 *     sparse mat-vec v_{k+1} = θ(M_P v_k)   (Algorithm 1, PAPER.md:152-173;
 *     T_P PAPER.md:70-72; θ Def. 5; M_P Def. 2);
 *   - stable models of a normal program = the same iteration batched over an initial
 *     matrix of guesses on the negated atoms, followed by a complementarity check
 *     (Algorithms 2-3; positive form Eq. 4 PAPER.md:188-194;
 *     initial matrix Def. 8).
 *
 * Plain C types only: host or device pointers and sizes.  Every call returns an
 * lp_status; lp_last_error() gives a thread-local detail string for the last failure.
 *
 * Bit conventions (all bit vectors): LSB-first little-endian uint64 words; atom a is
 * word a>>6, bit a&63; guess g is word g>>6, bit g&63.  Padding bits are written as 0
 * and ignored on input.  Model outputs cover the original atoms 0..n_atoms-1 only.
 *
 * Ownership: inputs are borrowed for the duration of the call (lp_load copies what it
 * keeps); outputs are caller-allocated.  Device memory is owned by the lp_program
 * handle until lp_free() and comes from the lp_options alloc/free hooks (the Python
 * binding passes PyTorch's caching allocator) or cudaMalloc by default.  A handle must
 * not be used by two threads at once; distinct handles are independent.
 *
 * Synchronisation: without LP_PTR_DEVICE every pointer argument of a run call is a host
 * pointer and the call returns after the results are in host memory.  With
 * LP_PTR_DEVICE every pointer argument of that call (v0, outputs, guesses, counters)
 * is a device pointer and the call is asynchronous on lp_run.stream.
 */
#ifndef LP_B200_H
#define LP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lp_program lp_program; /* opaque */

typedef enum {
    LP_OK = 0,
    LP_E_INVALID = 1,        /* bad argument: NULL required pointer, atom id out of
                                range, non-monotone body_ptr, size overflow          */
    LP_E_PARSE = 2,          /* reserved (no text loader in this library)            */
    LP_E_SEMANTIC = 3,       /* lp_least_model on a program with negation            */
    LP_E_CAP = 4,            /* guesses == NULL and free negated atoms > guess_cap   */
    LP_E_NOMEM = 5,          /* host or device allocation failed                     */
    LP_E_CUDA = 6,           /* CUDA runtime error (detail in lp_last_error)         */
    LP_E_NOT_CONVERGED = 7,  /* pass guard exceeded (cannot happen for valid input)  */
    LP_E_NODEVICE = 8        /* run call on a host-only handle (lp_options.device<0) */
} lp_status;

/* A ground normal program (Eq. 3; definite when body_neg is NULL
 * or all zero, Eq. 1).  Rule r: head[r] <- the literals
 * body_atom[body_ptr[r] .. body_ptr[r+1]-1], literal j negative ("not atom") iff
 * body_neg[j] = 1.  An empty body is a fact.  Duplicate body literals
 * are removed (footnote PAPER.md:54); duplicate rules are kept (harmless).  Several
 * rules with one head are the paper's multi-rule heads, standardized into AND-rows +
 * an OR-row by lp_load. */
typedef struct {
    int32_t n_atoms;          /* atoms 0..n_atoms-1 (>= 0)                      */
    int64_t n_rules;          /* >= 0                                           */
    const int32_t *head;      /* [n_rules]                                      */
    const int64_t *body_ptr;  /* [n_rules+1], body_ptr[0] = 0, non-decreasing   */
    const int32_t *body_atom; /* [body_ptr[n_rules]]                            */
    const uint8_t *body_neg;  /* [body_ptr[n_rules]] or NULL (definite)         */
} lp_rules;

typedef void *(*lp_alloc_fn)(size_t bytes, void *ctx);
typedef void (*lp_free_fn)(void *ptr, size_t bytes, void *ctx);

#define LP_LOAD_NO_FRONTIER 0x1u /* do not build the transposed occurrence lists */
#define LP_LOAD_PAPER_LAYOUT 0x4u /* standardize into P^δ first: a head with
                                    k >= 2 rules gets auxiliary atoms x_1..x_k and the
                                    OR-row h <- x_1 ∨ ... ∨ x_k, as in the paper's matrix
                                    M_{P^δ}; pass counts and popcount traces (which then
                                    count the auxiliaries too) follow Algorithms 1-2
                                    literally (convention (A), R4).  Models,
                                    stages, v0 and guesses stay over the original atoms */
#define LP_LOAD_KEY8 0x8u        /* summary mode: stream 8-bit key codes (1.25 B/row) instead
                                    of 16-bit ones (2.125 B/row).  On C4 the per-pass plane
                                    then stays L2-resident: 17% faster, L2/latency-bound
                                    rather than HBM-bound       */
/* (flag 0x2u, the former TMA-ring full θ-pass, was removed: lp_load rejects unknown
    flag bits with LP_E_INVALID) */

typedef struct {
    int device;             /* CUDA device ordinal; -1 = host-only handle: encode and
                               validate only (lp_info works, run calls fail with
                               LP_E_NODEVICE) -- used by CPU tests                 */
    int guess_cap;          /* max free negated atoms when guesses == NULL (<=0: 20) */
    uint32_t flags;         /* LP_LOAD_*                                           */
    int32_t smem_bits_cap;  /* test hook: max truth/summary bits kept in shared
                               memory per CTA (0 = automatic)                      */
    int32_t grid_blocks;    /* test hook: CTAs of the persistent kernels (0 = all
                               co-resident CTAs)                                   */
    lp_alloc_fn alloc;      /* device allocator hook (NULL = cudaMalloc)           */
    lp_free_fn free;
    void *alloc_ctx;
    const uint8_t *derivable; /* optional [n_atoms] layout hint, 1 = the atom may become
                               true from the facts (D2);
                               NULL = computed from this program.  Never affects a
                               result.  A head-range shard of a larger program passes
                               the whole program's D2 (shard.py), so atoms derived on
                               other GPUs keep fine key groups.  Ignored with
                               LP_LOAD_PAPER_LAYOUT.                                */
} lp_options;

#define LP_PTR_DEVICE 0x1u /* pointer args of this call are device pointers; async */
#define LP_FRONTIER 0x2u   /* least model: frontier (semi-naive) variant            */
#define LP_FULL_STREAM 0x4u /* full θ-pass: stream every body position in every pass
                               (default: LEAD passes -- stream the lead atom of each
                               row, verify the survivors -- until a pass queues more
                               than 1/16 of the rows or verifies more than 1/8 of the
                               body entries; programs whose bodies average more than
                               32 atoms start with STREAM passes).  Same results.    */
#define LP_FULL_LEAD 0x8u   /* full θ-pass: LEAD passes only (never switch)          */
#define LP_FULL_NO_PIPE 0x10u /* full θ-pass, key-space LEAD passes: do not pipeline
                               (default: pass k+1's lead stream, filtered by v_k,
                               runs while pass k's rows are verified; the rows whose
                               lead atom became true in pass k are added from the
                               lead-occurrence lists).  Same results.               */

typedef struct {
    void *stream;            /* cudaStream_t (NULL = legacy default stream)          */
    uint32_t flags;          /* LP_PTR_DEVICE | LP_FRONTIER                          */
    int32_t *popcounts_out;  /* optional [popcounts_cap]: |I_0|, |I_1|, ..., |I_k*|   */
    int32_t popcounts_cap;
    int32_t *stage_out;      /* optional [n_atoms]: k if the atom first appears in
                                I_k, -1 if it is not in the least model             */
    void *ev_begin;          /* optional cudaEvent_t recorded on stream immediately
                                before the fixpoint kernel, ev_end right after it   */
    void *ev_end;
    uint64_t *stats_out;     /* optional [6], full θ-pass only (zeros otherwise):
                                [0] algorithmic bytes the fixpoint kernel moved (planes
                                streamed + 4 B per verified body entry / head + 12 B
                                per derived atom), [1] LEAD passes, [2] rows queued for
                                verification, [3] body entries verification loaded,
                                [4] SM clock cycles and [5] ns the launch took
                                (%clock64 / %globaltimer of one thread)              */
    int32_t max_passes;      /* lp_least_model: stop after this many θ-passes even if the
                                last one derived something (0 = run to the fixpoint);
                                not an error -- iters_out = passes run.  One pass from a
                                v0 is one T_P evaluation over this program's rules: the
                                step of the head-range-sharded multi-GPU loop (shard.py) */
    int32_t *converged_out;  /* optional (host pointer, host-mode calls only): 1 if the
                                last pass derived nothing (u = v), else 0            */
    int64_t guess_offset;    /* lp_stable_models with guesses == NULL: guess i of this
                                call is global guess guess_offset + i of the binary
                                counting order (a multiple of 64; 0 = from the first).
                                Lets ranks split the 2^f guesses      */
    int32_t *status_out;     /* optional: the run's final status word, bit flags
                                LP_ST_* (0 = reached the fixpoint, nothing dropped).
                                Host mode: a host pointer, filled before the call
                                returns (the lp_status return value already reflects
                                it).  LP_PTR_DEVICE: a DEVICE pointer written by the
                                kernel's epilogue on lp_run.stream -- the only way an
                                asynchronous call reports LP_ST_OVERFLOW or
                                LP_ST_GUARD; callers must check it once the stream
                                has been synchronised.                               */
    int64_t out_word_lo;     /* lp_least_model: with out_word_count > 0, only model  */
    int64_t out_word_count;  /* words [out_word_lo, out_word_lo + out_word_count) are
                                written, to model_out[0 .. out_word_count) (a head-
                                range shard's owned words, shard.py); 0 = the whole
                                model                                               */
} lp_run;

/* lp_run.status_out bit flags (sticky; an overflow is never masked by a cap):      */
#define LP_ST_GUARD 0x1     /* pass guard (n_ext + 2 passes) hit: LP_E_NOT_CONVERGED  */
#define LP_ST_OVERFLOW 0x2  /* internal candidate queue overflow: LP_E_CUDA; results
                               are invalid (cannot happen by construction)           */
#define LP_ST_CAPPED 0x4    /* stopped at lp_run.max_passes before the fixpoint (not
                               an error)                                             */

typedef struct {
    int32_t n_atoms;
    int64_t n_rules;
    int64_t nnz;              /* body literals after de-duplication, + 1 per fact (⊤) */
    int64_t n_heads;          /* distinct heads                                       */
    int32_t n_negated;        /* k: distinct atoms under negation (abar atoms)         */
    int32_t n_free_negated;   /* f: negated atoms that are not facts (Def. 8 item 3)   */
    int32_t max_body;
    int32_t n_segments;       /* body-length buckets of the device layout              */
    int64_t n_prime_paper;    /* side of the paper's standardized matrix (n + k + aux) */
    double sparsity_eq5;      /* Eq. 5, over the input rules         */
    int64_t device_bytes;     /* device memory held by the handle                      */
    int64_t pass_bytes;       /* algorithmic bytes one full θ-pass streams */
    int32_t truth_mode;       /* 0: exact truth vector in shared memory; 1: summary    */
    int32_t summary_shift;    /* atoms per summary bit = 1 << summary_shift            */
    int32_t grid_blocks;      /* CTAs of the persistent kernels                        */
    int32_t block_threads;
    int64_t lead_pass_bytes;  /* program bytes a LEAD full θ-pass streams                */
    int64_t stream_pass_bytes;/* program bytes a STREAM full θ-pass streams              */
    int32_t key_shift;        /* summary mode: keys per key-summary bit = 1 << key_shift;
                                 -1 when there is no key plane                         */
    int32_t n_aux;            /* LP_LOAD_PAPER_LAYOUT: auxiliary atoms of P^δ (else 0)  */
    int32_t cluster_ctas;     /* > 0: the full θ-pass (auto schedule) runs in ONE thread-
                                 block cluster of this many CTAs (truth in shared memory,
                                 DSMEM exchange); 0: the persistent grid kernel         */
    int32_t frontier_cluster_ctas; /* > 0: the frontier variant runs as ONE cluster of
                                 this many CTAs (cluster barriers); 0: the grid         */
    int32_t stable_cluster_ctas;   /* the same for lp_stable_models / lp_stable_search */
    int32_t armed_list_cap;   /* > 0: LEAD passes of the full θ-pass are armed (rows whose
                                 lead atom is true and head is not, kept per CTA in lists
                                 of this many entries);
                                 0: they stream the lead / head (or key) planes        */
    int32_t stable_compact_atoms; /* > 0: lp_stable_models runs the compact kernel: |A*|, the
                                 atoms that can be true in some guess (the least model of P+
                                 with every abar_j true, computed by lp_load), held with
                                 the live rows in shared memory, a CTA per guess word
                                 (DESIGN.md "Compact stable kernel"); 0: the batched kernel */
    int32_t stable_compact_rows;  /* live rows (body within A*, head not a fact)        */
    int32_t small_rows;       /* > 0: the full θ-pass (auto schedule) runs the small-program
                                 kernel: ONE CTA, the rows (this many, at least 1) in shared
                                 memory, semi-naive row lists (DESIGN.md "Small-program
                                 kernel"); 0: the cluster / persistent grid kernels      */
} lp_info_t;

/* Validate, standardize and encode a program, upload it (PAPER.md:62, 82-95,
 * 188-192, 197-210).  opt may be NULL (device 0). */
lp_status lp_load(const lp_rules *rules, const lp_options *opt, lp_program **out);

/* Shapes and layout statistics of a loaded program. */
lp_status lp_info(const lp_program *p, lp_info_t *out);

/* The k negated atoms in ascending id: abar_j of the positive form (Eq. 4) and row j
 * of the guess matrix.  out: int32[k] host array. */
lp_status lp_negated_atoms(const lp_program *p, int32_t *out);

/* Least model of a definite program (Algorithm 1).
 *   v0        : optional start set, bits over the original atoms ([ceil(n/64)] words);
 *               NULL = the paper's initial vector (facts only, Def. 4).  The computed
 *               model is LM(P ∪ {a <- : a ∈ v0}); facts are always included.
 *   model_out : [ceil(n/64)] words, required.  Host mode: a page-locked host buffer
 *               (cudaHostAlloc, pinned torch tensor) is written by the kernel itself
 *               over PCIe; pageable memory is filled by a staged copy.
 *   iters_out : required; the number of T_P evaluations (θ-passes) including the
 *               final one that finds no change (reading R4).
 * Identical results (model, iters, popcounts, stages) with and without LP_FRONTIER.
 * LP_E_SEMANTIC if the program has a negative literal. */
lp_status lp_least_model(lp_program *p, const uint64_t *v0, uint64_t *model_out,
                         int32_t *iters_out, const lp_run *run);

/* Stable models (Algorithms 2-3) over a batch of guesses.
 *   guesses    : bit-sliced guess matrix, [k][W] words with W = ceil(n_guesses/64):
 *                bit g of row j is the value of abar_j (1 = a_j assumed false) in
 *                guess g.  NULL = the 2^f assignments of the free negated atoms in
 *                binary counting order (bit i of g = abar of the i-th free negated
 *                atom; abar of a negated fact fixed to 0, Def. 8 item 3), starting at
 *                lp_run.guess_offset; n_guesses <= 0 takes all the remaining ones,
 *                n_guesses > 0 at most that many (LP_E_CAP if f > guess_cap).
 *                Local guess i (bit i of accepted_out) is global guess offset + i.
 *   accepted_out : [W] words, bit g set iff guess g's fixpoint column satisfies
 *                a_j + abar_j = 1 for every negated atom (Algorithm 3, reading R7).
 *   n_accepted_out : number of accepted guesses (int64).
 *   passes_out : whole-matrix θ-passes until the matrix stopped changing
 *                (= max over guesses of the column's pass count).
 * The fixpoint matrix stays on the device for lp_stable_matrix / lp_guess_model. */
lp_status lp_stable_models(lp_program *p, const uint64_t *guesses, int64_t n_guesses,
                           uint64_t *accepted_out, int64_t *n_accepted_out,
                           int32_t *passes_out, const lp_run *run);

/* Guess-space reduction by sampling + local search (Conclusion: "prepare
 * some manageable size of the initial matrix, and if all guesses fail we do some local
 * search and replace column vectors by new assignments then repeat it until a stable
 * model is found"; details fixed by DESIGN.md reading R23).  For programs whose 2^f
 * guesses cannot be enumerated (lp_stable_models returns LP_E_CAP).
 *   h          : columns of the initial matrix per round (>= 1), W = ceil(h/64) words.
 *                Round 0: column g gives abar_j the bit rand64(seed, 0, g, j) >> 63 for
 *                every free negated atom j, 0 for a negated fact (Def. 8 item 3).
 *   seed       : of the counter-based generator rand64(seed, r, g, j) =
 *                mix(mix(mix(mix(seed) ^ r) ^ g) ^ j), mix = SplitMix64's output function.
 *   max_rounds : >= 1.  Each round is Algorithms 2-3 on the h columns (as
 *                lp_stable_models with explicit guesses); the search stops at the first
 *                round with an accepted column, else every column g is moved: the
 *                violated pairs V_g = {j : [a_j in LM_g] + abar_j != 1} with
 *                rand64(seed, r+1, g, j) >> 63 = 1 are flipped, or, if none is, the one
 *                V_g[rand64(seed, r+1, g, k) mod |V_g|].
 *   guesses_out    : optional [k][W] words: the last round's columns (bit g of row j =
 *                    abar_j in column g), the assignments behind accepted_out.
 *   accepted_out   : [W] words: the last round's accepted columns (all zero if none).
 *   n_accepted_out : accepted columns of the last round (0 = no stable model found
 *                    within max_rounds; not an error).
 *   rounds_out     : rounds run (the accepting round's number + 1, or max_rounds).
 *   passes_out     : whole-matrix θ-passes summed over the rounds.
 * All rounds run in ONE cooperative launch.  Afterwards lp_stable_matrix and
 * lp_guess_model read the last round's fixpoint matrix. */
lp_status lp_stable_search(lp_program *p, int64_t h, uint64_t seed, int32_t max_rounds,
                           uint64_t *guesses_out, uint64_t *accepted_out,
                           int64_t *n_accepted_out, int32_t *rounds_out, int32_t *passes_out,
                           const lp_run *run);

/* After lp_stable_models / lp_stable_search: the fixpoint rows of the original atoms,
 * [n_atoms][W] words (row a, bit g = atom a true in guess g's fixpoint column). */
lp_status lp_stable_matrix(lp_program *p, uint64_t *out, const lp_run *run);

/* After lp_stable_models / lp_stable_search: column `guess` of the fixpoint as a model bit vector over
 * the original atoms, [ceil(n/64)] words. */
lp_status lp_guess_model(lp_program *p, int64_t guess, uint64_t *model_out,
                         const lp_run *run);

/* Multi-GPU least model: the exchange step of one pass
 * over head-range shards.  Rank r loads the rules whose head lies in its 64-aligned atom
 * range (owned model words [word_lo[r], word_lo[r] + word_cnt[r])), runs ONE θ-pass
 * from the common v_k (lp_least_model with max_passes = 1, its owned words written via
 * lp_run.out_word_lo/count and its status word via lp_run.status_out into its payload),
 * and the payloads are all-gathered (NCCL; the caller's plumbing).  This call then
 * computes, on the device, v_{k+1} = v_k OR every rank's owned words -- T_P's OR clause
 * across GPUs -- and whether any rank's pass derived an atom (u != v of Algorithm 1,
 * PAPER.md:167).
 *   gathered      : device [world][stride] words; rank r's row: its owned words at
 *                   0 .. word_cnt[r]-1, its pass's lp_run.status_out word in the low 32
 *                   bits of word stride-1 (LP_ST_CAPPED = the pass derived an atom).
 *   word_lo, word_cnt : HOST [world] arrays; the ranges tile [0, n_words) in rank order,
 *                   word_cnt[r] <= stride - 1.  world in [1, 64].
 *   v, v_next     : device [n_words] model words (distinct buffers).
 *   changed_out   : device or mapped pinned host int32, set to 1/0.
 *   popcount_inout: optional device int32, |v_{k+1}| is ADDED to it (zero it first).
 *   stream        : cudaStream_t; asynchronous. */
lp_status lp_shard_combine(const uint64_t *gathered, int32_t world, int64_t stride,
                           const int64_t *word_lo, const int64_t *word_cnt,
                           const uint64_t *v, uint64_t *v_next, int64_t n_words,
                           int32_t *changed_out, int32_t *popcount_inout, void *stream);

/* Release the handle and its device memory (NULL is a no-op). */
void lp_free(lp_program *p);

const char *lp_status_str(lp_status s);
const char *lp_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* LP_B200_H */
